"""Measured tensor-core peaks on this pool's B200 (cuBLAS through torch): TF32 (fp32 matmul with
TF32 allowed) and int8 (torch._int_mm, cuBLASLt IMMA), 8192^3, best of 10 after warm-up, CUDA
events.  The roofline denominators of bench.py's tensor-pipe kernels (the 3xTF32 contraction
GEMMs, the int8 digit GEMM of dW_F) -> profiles/r2_tc_peaks.json.

    python tools/measure_tc_peaks.py [out.json]
"""
import json
import sys
from pathlib import Path

import torch


def best_tflops(fn, flops, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return flops / (best * 1e-3) / 1e12


def main():
    n = 8192
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    tf32 = best_tflops(lambda: a @ b, 2.0 * n ** 3)
    ai = torch.randint(-128, 127, (n, n), device="cuda", dtype=torch.int8)
    bi = torch.randint(-128, 127, (n, n), device="cuda", dtype=torch.int8).t().contiguous().t()
    try:
        i8 = best_tflops(lambda: torch._int_mm(ai, bi), 2.0 * n ** 3)
    except RuntimeError as e:  # noqa: BLE001
        i8, err = None, str(e)
    else:
        err = None
    out = {"tf32_tflops": tf32, "int8_tops": i8, "int8_error": err, "n": n,
           "gpu": torch.cuda.get_device_name(0),
           "how": "cuBLAS via torch: fp32 matmul with allow_tf32 (TF32 tcgen05) and torch._int_mm (int8), "
                  "8192^3, 2*n^3 ops, best of 10 after 3 warm-up, CUDA events"}
    path = Path(sys.argv[1]) if len(sys.argv) > 1 else Path("profiles/r2_tc_peaks.json")
    path.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
