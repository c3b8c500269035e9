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
        self.lib.oracle_lookup_new.restype = ctypes.c_int
        self.lib.oracle_lookup_new.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int]
        self.lib.oracle_lookup_add_f32.restype = ctypes.c_int
        self.lib.oracle_lookup_add_f32.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                                   ctypes.c_int, ctypes.c_void_p]
        self.lib.oracle_lookup_free.argtypes = [ctypes.c_int]

    def lookup(self, vocab, temperature=1.0, depth_aware=False):
        return LookupHandle(self, vocab, temperature, depth_aware)


class LookupHandle:
    """A LookupModel inside liboracle filled through the binary entry (fp32 rows at V ~ 152K
    do not fit the JSON transport). Use `.json()` as the model in a request."""

    def __init__(self, oracle, vocab, temperature=1.0, depth_aware=False):
        self.lib = oracle.lib
        self.vocab = vocab
        self.id = self.lib.oracle_lookup_new(vocab, ctypes.c_double(temperature), 1 if depth_aware else 0)
        self.added = self.duplicates = 0

    def add(self, ctx, depth, logits_f32):
        import numpy as np
        row = np.ascontiguousarray(logits_f32, dtype=np.float32)
        assert row.shape == (self.vocab,)
        c = (ctypes.c_int * len(ctx))(*ctx)
        r = self.lib.oracle_lookup_add_f32(self.id, c, len(ctx), depth, ctypes.c_void_p(row.ctypes.data))
        if r < 0:
            raise AssertionError("same context produced a different logit row (row invariance broken)"
                                 if r == -1 else "unknown lookup id")
        self.added += r == 0
        self.duplicates += r == 1

    def json(self):
        return {"kind": "lookup_ref", "id": self.id}

    def __del__(self):
        try:
            self.lib.oracle_lookup_free(self.id)
        except Exception:
            pass


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
