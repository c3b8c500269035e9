"""Split-K sweep of the SM-pair residual GEMM at drafter sizes. Usage: python tools/gemm_split_sweep.py [M]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_26475_b200 as rb  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dev = rb.default_device()
s = torch.cuda.Stream()
dev.set_stream(s.cuda_stream)
for name, (N, K) in {"o": (2048, 2048), "fc": (2048, 6144), "down": (2048, 11008)}.items():
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    res = []
    for bt in (0, 64, 128, 256):
        for splits in (1, 2, 4, 6, 8, 12):
            def run():
                rb._check(rb.lib().rs_gemm_bf16(dev.handle, ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                                ctypes.c_void_p(out.data_ptr()), None, M, N, K, 2, 1.0, bt, splits))
            torch.cuda.synchronize()
            for _ in range(3):
                run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                for _ in range(20):
                    run()
                e1.record(s)
            torch.cuda.synchronize()
            res.append(f"bt{bt}s{splits}:{e0.elapsed_time(e1) / 20 * 1000:.1f}us")
    print(name, " ".join(res), flush=True)
