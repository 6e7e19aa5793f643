"""Measures the B200's dense FP64 / FP32 / TF32 GEMM rates with cuBLAS (torch.matmul), the
denominators SURVEY.md §8(d) asks for besides MEASURED_PEAKS.json's HBM and BF16 figures.

N^3 GEMMs, 2 N^3 flops each; best of 10 (burst) and back to back for ~3 s (sustained),
CUDA events on the current stream.  Prints one JSON object."""
import json
import time

import torch


def rate(dtype, n, tf32=False, secs=3.0):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, dtype=dtype, device="cuda")
    b = torch.randn(n, n, dtype=dtype, device="cuda")
    c = a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    reps = max(1, int(secs * 1e3 / best))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        torch.matmul(a, b, out=c)
    e1.record()
    e1.synchronize()
    flops = 2.0 * n ** 3
    return {"burst_tflops": flops / best / 1e9, "sustained_tflops": flops * reps / e0.elapsed_time(e1) / 1e9,
            "n": n, "reps": reps}


out = {"gpu": torch.cuda.get_device_name(), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
       "how": "torch.matmul (cuBLAS) N^3, 2 N^3 flops; best of 10 and back to back ~3 s",
       "fp64": rate(torch.float64, 8192), "fp32_no_tf32": rate(torch.float32, 8192, tf32=False),
       "tf32": rate(torch.float32, 8192, tf32=True)}
print(json.dumps(out))
