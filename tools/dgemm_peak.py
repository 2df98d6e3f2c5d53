"""cuBLAS DGEMM throughput (torch.matmul on float64 CUDA tensors): the second FP64 peak
figure beside the DFMA loop (tools/fp64_peak.cu), as SURVEY 8(d) asks.  Prints JSON:
burst = best of 10 single launches, sustained = back to back for ~4 s (CUDA events).

    python tools/dgemm_peak.py > profiles/r02/dgemm_peak.json
"""
import json

import torch


def main():
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(10):
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    flop = 2.0 * n ** 3
    # sustained: back to back for about 4 s
    k = max(1, int(4000 / best))
    e0.record()
    for _ in range(k):
        torch.matmul(a, b, out=c)
    e1.record()
    torch.cuda.synchronize()
    sus = e0.elapsed_time(e1) / k
    print(json.dumps({"dgemm_tflops": flop / (best * 1e-3) / 1e12, "dgemm_tflops_sustained": flop / (sus * 1e-3) / 1e12,
                      "n": n, "how": f"torch.matmul float64 {n}^3 (cuBLAS DGEMM), best of 10 / {k} back to back",
                      "device": torch.cuda.get_device_name(), "torch": torch.__version__}))


if __name__ == "__main__":
    main()
