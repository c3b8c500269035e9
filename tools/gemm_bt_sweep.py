"""Token-tile (BT) sweep of the SM-pair GEMM at the verify shapes (M tokens)."""
import ctypes
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2510_26475_b200 as rb  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1344
shapes = {"qkv": (2560, 2048, 0), "o": (2048, 2048, 2), "gate_up": (22016, 2048, 4), "down": (2048, 11008, 2),
          "lm_head": (151936, 2048, 1)}
dev = rb.default_device()
s = torch.cuda.Stream()
dev.set_stream(s.cuda_stream)
for name, (N, K, epi) in shapes.items():
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    out = torch.zeros(M, N // 2 if epi == 4 else N, device="cuda", dtype=torch.float32 if epi in (1, 2) else torch.bfloat16)
    bias = torch.zeros(N, device="cuda").bfloat16()
    res = []
    for bt in (0, 64, 96, 128, 160, 192, 224, 256):
        for splits in ((1, 2, 3) if epi == 2 else (1,)):
            def run():
                rb._check(rb.lib().rs_gemm_bf16(dev.handle, ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                                ctypes.c_void_p(out.data_ptr()),
                                                ctypes.c_void_p(bias.data_ptr()) if epi == 0 else None, M, N, K, epi,
                                                1.0, bt, splits))
            torch.cuda.synchronize()
            for _ in range(3):
                run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 5 if N > 100000 else 20
            with torch.cuda.stream(s):
                e0.record(s)
                for _ in range(reps):
                    run()
                e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            res.append(f"bt{bt}s{splits}:{2.0 * M * N * K / (ms * 1e-3) / 1e12:.0f}")
    print(name, " ".join(res), flush=True)
