"""ctypes client for the CPU checkers under oracle/ -- TEST INFRASTRUCTURE ONLY.

`Oracle()` wraps our restatement (oracle/build/liboracle.so); `Reference()` wraps the
compiled reference core (oracle/_ref/librespec_ref.so). Both speak the same JSON schema.
"""
import ctypes
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class CheckerError(Exception):
    def __init__(self, kind, what):
        super().__init__(f"{kind}: {what}")
        self.kind = kind
        self.what = what


class _JsonLib:
    _sym = None

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = ctypes.CDLL(path)
        call = getattr(self.lib, self._sym + "_call")
        call.restype = ctypes.c_void_p
        call.argtypes = [ctypes.c_char_p]
        free = getattr(self.lib, self._sym + "_free")
        free.argtypes = [ctypes.c_void_p]
        self._call, self._free = call, free

    def __call__(self, op, **kw):
        kw["op"] = op
        ptr = self._call(json.dumps(kw).encode())
        try:
            out = json.loads(ctypes.string_at(ptr).decode())
        finally:
            self._free(ptr)
        if isinstance(out, dict) and "error" in out:
            raise CheckerError(out["error"]["type"], out["error"]["what"])
        return out


class Oracle(_JsonLib):
    _sym = "oracle"

    def __init__(self):
        super().__init__(os.path.join(ROOT, "oracle", "build", "liboracle.so"))


class Reference(_JsonLib):
    _sym = "ref"

    def __init__(self):
        super().__init__(os.path.join(ROOT, "oracle", "_ref", "librespec_ref.so"))


def fnv1a_responses(responses):
    """SURVEY.md Appendix B fingerprint: FNV-1a-64 over each response token as 4 LE bytes,
    with a -1 separator token after each response, requests in request order."""
    h = 1469598103934665603
    for resp in responses:
        for t in list(resp) + [-1]:
            for b in int(t).to_bytes(4, "little", signed=True):
                h ^= b
                h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"
