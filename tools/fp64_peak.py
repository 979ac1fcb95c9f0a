#!/usr/bin/env python
"""Calibrate the fp64 ceiling for the setup GEMMs: cuBLAS complex128 GEMM
(torch.matmul) at the C2 Gram shape, 2048 x 16384 x 2048, best of 5, CUDA
events.  Prints TFLOP/s (8 real flops per complex multiply-add)."""
import json

import torch

m, k = 2048, 16384
a = torch.randn(m, k, dtype=torch.complex128, device="cuda")
b = a.conj().T.contiguous()
for _ in range(2):
    torch.matmul(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"zgemm_ms": best, "tflops": 8.0 * m * m * k / best / 1e9, "shape": [m, k, m]}))
