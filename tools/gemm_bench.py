"""Microbenchmark of the tcgen05 GEMM at the verify shapes (Qwen2.5-3B, M = tokens per round)."""
import ctypes
import json
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
res = {}
for name, (N, K, epi) in shapes.items():
    for bn in ("pair", "single"):
        rb.set_tuning("gemm2", 0 if bn == "pair" else -1)
        A = torch.randn(M, K, device="cuda").bfloat16()
        B = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
        out = torch.zeros(M, N // 2 if epi in (3, 4) else N, device="cuda",
                          dtype=torch.float32 if epi in (1, 2) else torch.bfloat16)
        bias = torch.zeros(N, device="cuda").bfloat16()

        def run():
            rb._check(rb.lib().rs_gemm_bf16(dev.handle, ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                            ctypes.c_void_p(out.data_ptr()),
                                            ctypes.c_void_p(bias.data_ptr()) if epi == 0 else None, M, N, K, epi, 1.0,
                                            0, 1))
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
        ms = e0.elapsed_time(e1) / 20
        tf = 2.0 * M * N * K / (ms * 1e-3) / 1e12
        ref = torch.matmul(A, B.t())
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(20):
            torch.matmul(A, B.t())
        t1.record()
        torch.cuda.synchronize()
        cub = 2.0 * M * N * K / (t0.elapsed_time(t1) / 20 * 1e-3) / 1e12
        res[f"{name}_bn{bn}"] = {"ms": round(ms, 4), "tflops": round(tf, 1), "cublas_tflops": round(cub, 1)}
        print(name, bn, f"{ms:.4f} ms {tf:.1f} TF/s (cuBLAS {cub:.1f})", flush=True)
print(json.dumps(res))
