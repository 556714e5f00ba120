"""Measured dense TF32 tensor-core peak on this B200 (BASELINE.md §2 asked for
it on the first GPU run): cuBLAS fp32 matmul with TF32 allowed, 8192^3
(2 N^3 FLOP), best of 10 (burst) and back to back for 4 s (sustained), the
same recipe the driver used for the bf16 figure in MEASURED_PEAKS.json.
Writes one JSON line to stdout."""
import json
import time

import torch


def main():
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        a @ b
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    t0, k = time.time(), 0
    s = torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < 4.0:
        for _ in range(10):
            a @ b
        k += 10
        torch.cuda.synchronize()
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    torch.cuda.synchronize()
    sustained = 2 * n ** 3 * k / (s.elapsed_time(e) / 1e3) / 1e12
    print(json.dumps({"tf32_tflops": 2 * n ** 3 / (best / 1e3) / 1e12, "tf32_tflops_sustained": sustained,
                      "how": "torch.matmul fp32 with allow_tf32 (cuBLAS) 8192^3, best of 10 / back to back 4 s",
                      "gpu": torch.cuda.get_device_name()}))


if __name__ == "__main__":
    main()
