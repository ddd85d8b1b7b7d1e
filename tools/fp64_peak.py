"""cuBLAS DGEMM / ZGEMM throughput via torch (the FP64 analog of the driver's
bf16 cuBLAS figure), plus the DFMA/DMMA probes of tools/fp64_peak.cu."""
import json
import os
import subprocess
import sys

import torch

res = {}
if not os.path.exists("tools/fp64_peak"):  # probe binary (not versioned): build it for sm_100a
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", "tools/fp64_peak",
                    "tools/fp64_peak.cu"], check=True)
out = subprocess.run(["./tools/fp64_peak"], capture_output=True, text=True).stdout.strip()
res.update(json.loads(out))
for name, dt, mult in (("dgemm", torch.float64, 2), ("zgemm", torch.complex128, 8)):
    n = 8192 if dt == torch.float64 else 6144
    a = torch.randn(n, n, dtype=dt, device="cuda")
    b = torch.randn(n, n, dtype=dt, device="cuda")
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[f"cublas_{name}_tflops"] = round(mult * n ** 3 / (best * 1e-3) / 1e12, 2)
res["gpu"] = torch.cuda.get_device_name()
print(json.dumps(res))
