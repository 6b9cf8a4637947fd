"""Measure the FP64 roofline denominators on the GPU box: cuBLAS DGEMM and ZGEMM via torch.

Burst = best of 10; sustained = back-to-back for ~4 s.  Prints one JSON line per probe.
"""
import json
import time

import torch


def probe(dtype, n, flop_mult):
    a = torch.randn(n, n, dtype=dtype, device="cuda")
    b = torch.randn(n, n, dtype=dtype, device="cuda")
    c = torch.empty(n, n, dtype=dtype, device="cuda")
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    flops = flop_mult * n**3
    burst = flops / (best * 1e-3) / 1e12
    t_end = time.time() + 4.0
    count = 0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() < t_end:
        for _ in range(4):
            torch.matmul(a, b, out=c)
        count += 4
        torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    sustained = flops * count / (e0.elapsed_time(e1) * 1e-3) / 1e12
    return burst, sustained


if __name__ == "__main__":
    for name, dtype, n, mult in (("dgemm", torch.float64, 8192, 2.0), ("zgemm", torch.complex128, 4096, 8.0)):
        burst, sus = probe(dtype, n, mult)
        print(json.dumps({"probe": name, "n": n, "tflops_burst": round(burst, 3), "tflops_sustained": round(sus, 3)}))
