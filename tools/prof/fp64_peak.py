"""FP64 peak on this B200: cuBLAS DGEMM 8192^3 (torch.matmul float64, 2 N^3 flops; best of 10 = burst,
back to back for ~4 s = sustained) and the register-only DFMA / DMMA issue microbenchmark
(tools/microbench/fp64_peak.cu). Writes profiles/r2_fp64_peak.json -- the FP64 roofline denominator
bench.py and DESIGN.md cite (MEASURED_PEAKS.json carries no FP64 entry).

usage: python tools/prof/fp64_peak.py [out.json]
"""
import json
import re
import subprocess
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]


def dgemm(n=8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    flops = 2.0 * n ** 3
    # sustained: back to back for ~4 s
    reps = max(1, int(4000 / best))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        torch.matmul(a, b, out=c)
    e1.record()
    e1.synchronize()
    sus = e0.elapsed_time(e1) / reps
    return flops / best / 1e9, flops / sus / 1e9


def main():
    out = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "profiles" / "r2_fp64_peak.json"
    burst, sustained = dgemm()
    mb = ROOT / "tools" / "microbench" / "fp64_peak"
    src = mb.with_suffix(".cu")
    subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(mb), str(src)], check=True)
    txt = subprocess.run([str(mb)], capture_output=True, text=True, check=True).stdout
    dfma = [float(x) for x in re.findall(r"DFMA blocks/SM=\d+: ([\d.]+) TFLOP/s", txt)]
    dmma = [float(x) for x in re.findall(r"DMMA blocks/SM=\d+: ([\d.]+) TFLOP/s", txt)]
    smi = subprocess.run(["nvidia-smi", "--query-gpu=name,clocks.sm,clocks.max.sm", "--format=csv,noheader"],
                         capture_output=True, text=True).stdout.strip()
    rec = {"dgemm_8192_tflops_burst": burst, "dgemm_8192_tflops_sustained": sustained,
           "dfma_tflops": max(dfma) if dfma else None, "dmma_tflops": max(dmma) if dmma else None,
           "microbench_output": txt.strip().splitlines(), "gpu": smi, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "how": "torch.matmul float64 8192^3 (cuBLAS DGEMM), best of 10 and ~4 s back to back; "
                  "tools/microbench/fp64_peak.cu register-only DFMA / mma.sync.m8n8k4.f64 issue loops"}
    out.write_text(json.dumps(rec, indent=1) + "\n")
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
