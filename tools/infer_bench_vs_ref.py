"""Side-by-side infer-bench: the GPU driver (paper_1702_08597_b200.infer_bench) and the
reference's compress + sparse_forward<float> (oracle/_ref, all host cores) on the same inputs,
density by density.  Prints both CSVs' key columns and whether the checksums agree bitwise.

    python tools/infer_bench_vs_ref.py --layers tools/layers_vgg.cfg --batch 8 --density-sweep 0.1:1:log4
"""
from __future__ import annotations

import argparse
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from oracle import ref  # noqa: E402  (checker / CPU baseline only)
from paper_1702_08597_b200 import infer_bench as ib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", required=True)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--density-sweep", default="0.1:1:log4")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--ref-workers", type=int, default=os.cpu_count())
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    layers = ib.layers_from_config(a.layers)
    grid = ib.parse_density_grid(a.density_sweep)
    rows = ib.run(layers, grid, a.batch, "f32", 1, a.seed)
    print("layer,density,gpu_wall_ns,gpu_gflops,ref_wall_ns,ref_gflops,speedup,checksum_equal")
    for d, row in zip([d for d in layers for _ in grid], rows):
        name, x, _, ns, gf, cs = row
        if a.no_ref:
            print(f"{name},{x:g},{ns},{gf:g},,,,")
            continue
        b, w_f = ib.bench_inputs(d, a.batch, a.seed)
        w = ib.magnitude_threshold_to_density(w_f, x)
        t0 = time.perf_counter_ns()
        out = ref.sparse_forward(b, w, m=d.m, workers=a.ref_workers, precision=32)
        rns = time.perf_counter_ns() - t0
        rgf = d.flops_baseline() * a.batch / rns
        print(f"{name},{x:g},{ns},{gf:g},{rns},{rgf:g},{rns / ns:.1f},{ib.checksum(out) == cs}")


if __name__ == "__main__":
    main()
