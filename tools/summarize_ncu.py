"""Summarise ncu captures into profiles/ (run in the build container; ncu -i needs no GPU).

    python tools/summarize_ncu.py --round r1 --launches gpurun_out/launches_c1.csv \
        --full c1=gpurun_out/full_c1.ncu-rep --full c3=gpurun_out/full_c3.ncu-rep

Writes profiles/<round>_launches_c1.csv (copy), profiles/<round>_launch_shares.md,
profiles/<round>_kernels.md (per-kernel key counters from the full captures) and updates
profiles/ncu_traffic.json with dram read+write bytes per launch for each kernel.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import shutil
import subprocess
from collections import OrderedDict, defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"

KIND = [("input_transform_digits", "input_transform"), ("input_transform", "input_transform"),
        ("grad_z_digits", "grad_z"), ("output_transform", "output_transform"), ("input_grad", "input_grad"),
        ("plane_amax", "amax"), ("xdw::gemm_kernel", "dw_gemm_i8"), ("reduce_sparse", "dw_reduce"),
        ("reduce_dense", "dw_reduce"), ("spmm_hyb", "spmm"), ("spmm_tmem", "spmm"), ("spmm_kernel", "spmm"),
        ("gemm_3xtf32", "dense_tc"), ("tm_", "stream_build"), ("stage_bounds", "stream_build")]

METRICS = OrderedDict([
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("lts__t_sectors.sum", "l2_sectors"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_pipe_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("sm__pipe_tensor_op_tcgen05_cycles_active.avg.pct_of_peak_sustained_active", "tensor_%"),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc_inst_%"),
])


def kind_of(name: str) -> str:
    for key, k in KIND:
        if key in name:
            return k
    return name.split("(")[0][:40]


def to_bytes(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return x * scale.get(unit, 1)


def launches(path: Path, rnd: str, what: str):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0.0, 0])
    for r in rows[hi + 1:]:
        k = kind_of(r[ki])
        agg[k][0] += float(r[vi].replace(",", ""))
        agg[k][1] += 1
    shutil.copy(path, PROF / f"{rnd}_{path.name}")
    ours = {k: v for k, v in agg.items() if "at::" not in k and "vectorized" not in k}
    tot = sum(v[0] for v in ours.values())
    lines = [f"# {rnd}: ncu launch list of `{what}`",
             "", "Cold-cache, serialised per-launch times (`gpu__time_duration.sum`, `--clock-control none`);",
             "compare shares, not absolutes. Torch's L2-flush fills are excluded from the shares.", "",
             "| kernel | launches | mean µs | share |", "|---|---|---|---|"]
    for k, (t, n) in sorted(ours.items(), key=lambda kv: -kv[1][0]):
        lines.append(f"| {k} | {n} | {t / n / 1e3:.1f} | {t / tot:.1%} |")
    (PROF / f"{rnd}_launch_shares_{path.stem}.md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(tag: str, path: Path, rnd: str, traffic: dict, cfg_key: str):
    raw = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    seen = set()
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        name = d.get("Kernel Name", "?")
        k = kind_of(name)
        key = (k, d.get("Block Size"), d.get("Grid Size"))
        if k in seen:
            continue
        seen.add(k)
        rec = OrderedDict(kernel=k)
        for m, short in METRICS.items():
            if m in d and d[m] not in ("", "n/a"):
                if short.startswith(("dram_read", "dram_write", "l2_bytes")):
                    rec[short] = to_bytes(d[m], u[m])
                elif short == "duration":
                    x = float(d[m].replace(",", ""))
                    rec[short] = "{:.1f}".format(x * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                                                      "msecond": 1e3, "nsecond": 1e-3}.get(u[m], 1.0))
                else:
                    try:
                        rec[short] = "{:.1f}".format(float(d[m].replace(",", "")))
                    except ValueError:
                        rec[short] = d[m]
        if "dram_read" in rec:
            tb = rec["dram_read"] + rec.get("dram_write", 0.0)
            rec["dram_total"] = tb
            traffic[f"{cfg_key}:{k if k != 'spmm' else 'spmm_fwd'}"] = tb
        out.append(rec)
    lines = [f"## {tag} — `ncu --set full` ({path.name})", "",
             "| kernel | µs | DRAM MB (r+w) | DRAM %peak | L2 MB | smem wavefronts | smem pipe % | SM % | issue % | occupancy % | regs | tensor % |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for rec in out:
        dur = rec.get("duration", "")
        lines.append("| {} | {} | {:.1f} | {} | {:.1f} | {} | {} | {} | {} | {} | {} | {} |".format(
            rec["kernel"], dur, rec.get("dram_total", 0) / 1e6, rec.get("dram_%peak", ""),
            rec.get("l2_bytes", 0) / 1e6, rec.get("smem_wavefronts", ""), rec.get("smem_pipe_%", ""),
            rec.get("sm_%", ""), rec.get("issue_%", ""), rec.get("occupancy_%", ""), rec.get("regs", ""),
            rec.get("tensor_%", rec.get("tc_inst_%", ""))))
    return lines


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r1")
    ap.add_argument("--launches")
    ap.add_argument("--launches-cmd", default="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-sweep")
    ap.add_argument("--full", action="append", default=[], help="tag=path[:cfgkey]")
    a = ap.parse_args()
    PROF.mkdir(exist_ok=True)
    if a.launches:
        launches(Path(a.launches), a.round, a.launches_cmd)
    tfile = PROF / "ncu_traffic.json"
    traffic = json.loads(tfile.read_text()) if tfile.exists() else {}
    md = [f"# {a.round}: per-kernel counters from single `ncu --set full --clock-control none` captures", "",
          "Durations here are under ncu replay (cold caches, serialised); bench.py's CUDA-event times are",
          "the reported numbers. DRAM MB = dram__bytes_read.sum + dram__bytes_write.sum per launch.", ""]
    for spec in a.full:
        tag, rest = spec.split("=", 1)
        path, _, cfgkey = rest.partition(":")
        md += full(tag, Path(path), a.round, traffic, cfgkey or tag) + [""]
    if a.full:
        (PROF / f"{a.round}_kernels.md").write_text("\n".join(md) + "\n")
        print("\n".join(md))
    tfile.write_text(json.dumps(traffic, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
