"""SM-pair GEMM at the verify shapes (Qwen2.5-3B, M = tokens per round) per token tile, next to
cuBLAS (torch.matmul, warmed up). Each GEMM runs 20x back to back (weights L2-warm except the
LM head). Usage: python tools/gemm_cublas_bench.py [M]"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_26475_b200 as rb  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1344
shapes = {"qkv": (2560, 2048, 0), "o": (2048, 2048, 2), "gate_up": (22016, 2048, 4), "down": (2048, 11008, 2),
          "lm_head": (151936, 2048, 1)}
dev = rb.default_device()
s = torch.cuda.Stream()
dev.set_stream(s.cuda_stream)
res = {}
for name, (N, K, epi) in shapes.items():
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    out = torch.zeros(M, N // 2 if epi in (3, 4) else N, device="cuda",
                      dtype=torch.float32 if epi in (1, 2) else torch.bfloat16)
    bias = torch.zeros(N, device="cuda").bfloat16()

    def timed(bn):

        def run():
            rb._check(rb.lib().rs_gemm_bf16(dev.handle, ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                            ctypes.c_void_p(out.data_ptr()),
                                            ctypes.c_void_p(bias.data_ptr()) if epi == 0 else None, M, N, K, epi, 1.0,
                                            bn, 1))
        torch.cuda.synchronize()
        for _ in range(3):
            run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(20):
            run()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 20 * 1e3

    row = {}
    for bn in (0, 64, 96, 128, 160, 192, 224, 256):
        row[f"bt{bn}"] = round(timed(bn), 2)
    for _ in range(3):
        torch.matmul(A, B.t())
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record()
    for _ in range(20):
        torch.matmul(A, B.t())
    t1.record()
    torch.cuda.synchronize()
    row["cublas_us"] = round(t0.elapsed_time(t1) / 20 * 1e3, 2)
    fl = 2.0 * M * N * K
    row["tflops_auto"] = round(fl / (row["bt0"] * 1e-6) / 1e12, 1)
    row["cublas_tflops"] = round(fl / (row["cublas_us"] * 1e-6) / 1e12, 1)
    res[name] = row
    print(name, json.dumps(row), flush=True)
print(json.dumps({"M": M, "shapes": res}))
