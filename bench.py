#!/usr/bin/env python
"""Benchmark of the Winograd-layer fwd+bwd hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--sparsity S]
    python bench.py --impl reference ...      # the reference's own CPU path on the host cores

A step = forward (with ForwardCache) + backward (dW_F and dI) of one layer over one batch of the
config, inputs resident in HBM.  Default workload: configs[3] at 90% W_F sparsity (N=64,
C=K=256, H=W=56, F(4x4,3x3), pad 1) — the metric's own sweep config; the line's "sweep" key
carries the metric's sweep (c3 fwd+bwd at 0/50/80/90/95%, CSR and 'auto' contraction, c2 fwd at
80/90/95%, c1) with each point's dominant kernel and its roofline fraction.  With N>1 GPUs every
rank runs its own batch (weak scaling: batch sharding) and dW_F (nnz-compact) is all-reduced over
NCCL inside the step; `--gpus N` without WORLD_SIZE re-launches itself under
torch.distributed.run.  Effective GFLOP/s follows the reference convention (tools/wino.cpp:362,
perfmodel.cpp:6-9): 2·C·K·H²·9 per image and pass, 3 passes.

Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA events on the
launching stream, with a 256 MB write between steps (outside the events) to flush the 126 MB
L2; barrier + synchronize around the timed region; the max over ranks is reported.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_1702_08597_b200.synth import CONFIGS, make_inputs, with_sparsity  # noqa: E402

METRIC_FWD = "Winograd layer fwd effective GFLOP/s"
METRIC = "Winograd layer fwd+bwd effective GFLOP/s"


def flops_per_image(cfg) -> float:
    """perfmodel.cpp:6-9 (flops_baseline) for one pass of one image."""
    return 2.0 * cfg.c * cfg.k * cfg.h * cfg.w * cfg.r * cfg.r


def workload_name(cfg, passes):
    return (f"{cfg.name}: N={cfg.n}/GPU C={cfg.c} K={cfg.k} H=W={cfg.h} F({cfg.m}x{cfg.m},3x3) "
            f"pad {cfg.pad}, W_F sparsity {cfg.sparsity:.0%}, {passes}")


def peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver-written: HBM copy, cuBLAS bf16), and the
    tcgen05 TF32 / int8 rates measured with cuBLAS on this pool (profiles/r2_tc_peaks.json,
    tools/measure_tc_peaks.py); int8 falls back to 2× bf16 (B200 dense int8 = 2× bf16), TF32 to
    bf16 / 2."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        out = {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"], "source": "measured"}
    else:
        out = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}
    out["tf32_tflops"], out["tf32_source"] = out["bf16_tflops"] / 2, out["source"] + " bf16/2"
    out["int8_tops"], out["int8_source"] = out["bf16_tflops"] * 2, out["source"] + " bf16x2"
    tc = ROOT / "profiles" / "r2_tc_peaks.json"
    if tc.exists():
        d = json.loads(tc.read_text())
        if d.get("tf32_tflops"):
            out["tf32_tflops"], out["tf32_source"] = d["tf32_tflops"], "measured (cuBLAS tf32, profiles/r2_tc_peaks.json)"
        if d.get("int8_tops"):
            out["int8_tops"], out["int8_source"] = d["int8_tops"], "measured (cuBLAS int8, profiles/r2_tc_peaks.json)"
    return out


# -------------------------------------------------------------------------------------
# clocks during the timed region
# -------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# -------------------------------------------------------------------------------------
# CPU side: the reference's own path (oracle/_ref) or the numpy port
# -------------------------------------------------------------------------------------
def cpu_fwd_bwd(cfg, img, w_f, go, n_img, threads):
    """One bounded sample of the reference's fwd+bwd: n_img images through the reference API
    (winograd_forward -> backward_weights -> backward_input per image, train.cpp:169-202),
    spread over `threads` host threads.  Returns (seconds, kind)."""
    from oracle import ref

    pad = cfg.pad
    imgp = np.pad(img[:n_img].astype(np.float64), ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    gop = go[:n_img].astype(np.float64)
    if ref.available():
        t0 = time.perf_counter()
        ref.layer_fwd_bwd_batch(imgp, w_f, gop, m=cfg.m, threads=threads, want_outputs=False)
        return time.perf_counter() - t0, "reference"
    from oracle import wino_oracle as wo  # numpy port, single process

    t0 = time.perf_counter()
    for i in range(n_img):
        _, cache = wo.forward_f64(imgp[i], w_f, cfg.m)
        wo.backward_weights_f64(gop[i], cache)
        wo.backward_input_f64(cache, w_f)
    return time.perf_counter() - t0, "port"


def cpu_sample_size(cfg, threads):
    return int(max(1, min(cfg.n, threads)))


def run_reference(args, cfg, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n_img = cpu_sample_size(cfg, threads)
    img, w_f, go = make_inputs(cfg, n=n_img)
    flops = 3 * flops_per_image(cfg) * n_img
    for _ in range(args.warmup):
        cpu_fwd_bwd(cfg, img, w_f, go, n_img, threads)
    times = []
    kind = "reference"
    for _ in range(args.steps):
        t, kind = cpu_fwd_bwd(cfg, img, w_f, go, n_img, threads)
        times.append(t)
    tot = sum(times)
    value = flops * args.steps / tot / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded splitmix64 normals)",
        "config": {"workload": workload_name(cfg, "fwd+bwd") + f"; CPU sample {n_img} images/step",
                   "n_images_per_step": n_img},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": threads, "kind": kind,
                         "sample": f"{n_img} of {cfg.n} images per step through the reference's "
                                   "dense f64 per-image fwd+bwd API on a thread pool"},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------------------------
# GPU arm
# -------------------------------------------------------------------------------------
def capture(step, args):
    """CUDA-graph the step (paper_1702_08597_b200.graph.GraphedStep) unless --no-graph; falls
    back to eager launches if capture fails (reported in the JSON line)."""
    if args.no_graph:
        return step, "eager"
    from paper_1702_08597_b200.graph import GraphedStep

    try:
        g = GraphedStep(step)
        return g.replay, "cuda-graph (one graph launch per step)"
    except Exception as e:  # noqa: BLE001
        return step, f"eager (graph capture failed: {type(e).__name__}: {e})"


def kernel_work(cfg, layer, n):
    """Algorithmic HBM bytes and tensor-pipe operations per STEP of each kernel
    kind.  input_transform / grad_z: K1 / K4 fused with the exact dW_F digits (5 int8 digits per
    value of Ĩ_F / dZ besides the fp32 value); amax: the max|I| / max|dO| pre-pass; dw_gemm_i8: 15
    exact digit-pair MACs per (k, c, column) on tcgen05 kind::i8."""
    g = layer.geometry
    nt = n * g["t"]
    ntd = -(-nt // 64) * 64
    p2 = g["p"] ** 2
    f = 4
    I = n * cfg.c * cfg.h * cfg.w * f
    O = n * cfg.k * g["h_o"] * g["w_o"] * f
    V = p2 * cfg.c * nt * f
    Z = p2 * cfg.k * nt * f
    nnz = layer.nnz
    Wb = 8 * nnz + 4 * p2 * (cfg.k + 1)
    Wt = 8 * nnz + 4 * p2 * (cfg.c + 1)
    dig_v, dig_z = 5 * p2 * cfg.c * ntd, 5 * p2 * cfg.k * ntd
    dig = dig_v + dig_z
    dense_w = 2 * 4 * p2 * cfg.k * cfg.c  # tf32 hi/lo weight operands
    fwd_only = not cfg.backward
    return {
        "input_transform": {"bytes": I + V + (0 if fwd_only else dig_v)}, "spmm_fwd": {"bytes": V + Z + Wb},
        "output_transform": {"bytes": Z + O}, "grad_z": {"bytes": O + Z + dig_z},
        "amax": {"bytes": I + O},
        "dw_gemm_i8": {"bytes": dig, "ops": 2.0 * 15 * p2 * cfg.k * cfg.c * ntd, "pipe": "int8"},
        "dw_reduce": {"bytes": 8 * p2 * cfg.k * cfg.c + (nnz * 12 if not layer.is_dense else 4 * nnz)},
        "spmm_bwd_data": {"bytes": Z + Wt + V}, "input_grad": {"bytes": V + I},
        "dense_fwd_tc": {"bytes": V + Z + dense_w, "ops": 3 * 2.0 * p2 * cfg.k * cfg.c * nt, "pipe": "tf32"},
        "dense_dv_tc": {"bytes": V + Z + dense_w, "ops": 3 * 2.0 * p2 * cfg.k * cfg.c * nt, "pipe": "tf32"},
    }


# On-chip operand bounds of the CSR kernels (tools/microbench/tmem_bw.cu, spmm_hybrid_bw.cu, one
# B200): a multiply-add needs 4 bytes of the dense operand per lane; tcgen05.ld.32x32b.x4 delivers
# 156 B/clk/SM (the TMEM SpMM), LDS.128 101 B/clk/SM (the shared-memory SpMM).
TMEM_MAC_PER_CLK = 156.3 / 4
LDS_MAC_PER_CLK = 101.3 / 4


def kernel_table(prof, steps, cfg, layer, n, pk, sm_mhz=None):
    """Per-kind time per step (profiled steps, CUDA events on the launching stream) with its
    roofline: tensor-pipe kinds against the measured TF32 / int8 rate, the rest against HBM; the
    CSR kinds also against their on-chip operand bound (multiply-adds per clock per SM)."""
    work = kernel_work(cfg, layer, n)
    nt = n * layer.geometry["t"]
    clk = (sm_mhz or 1965.0) * 1e6
    tot = sum(v[0] for v in prof.values()) or 1.0
    out = {}
    for name, (ms_tot, cnt) in prof.items():
        ms = ms_tot / steps
        k = {"ms_per_step": ms, "launches_per_step": cnt / steps, "share": ms_tot / tot}
        w = work.get(name)
        if w:
            k["alg_bytes"] = w["bytes"]
            k["GBps"] = w["bytes"] / (ms * 1e-3) / 1e9
            if "ops" in w:
                peak = pk["tf32_tflops"] if w["pipe"] == "tf32" else pk["int8_tops"]
                ach = w["ops"] / (ms * 1e-3) / 1e12
                k["roofline"] = {"bound": "tensor", "achieved": ach, "peak": peak, "frac": ach / peak,
                                 "unit": "TFLOP/s" if w["pipe"] == "tf32" else "TOPS",
                                 "peak_source": pk[w["pipe"] + "_source"],
                                 "note": ("issued TF32 FLOPs of the 3xTF32 GEMM (useful = 1/3)" if w["pipe"] == "tf32"
                                          else "issued int8 digit-pair ops (15 pairs per product)")}
            else:
                k["roofline"] = {"bound": "hbm", "achieved": k["GBps"], "peak": pk["hbm_gbs"],
                                 "frac": k["GBps"] / pk["hbm_gbs"], "unit": "GB/s", "peak_source": pk["source"]}
        if name.startswith("spmm"):
            mac = layer.nnz * nt / (ms * 1e-3) / (148 * clk)
            k["on_chip"] = {"mac_per_clk_sm": mac, "tmem_bound": TMEM_MAC_PER_CLK, "lds_bound": LDS_MAC_PER_CLK,
                            "frac_of_tmem_bound": mac / TMEM_MAC_PER_CLK,
                            "frac_of_tmem_plus_lds_bound": mac / (TMEM_MAC_PER_CLK + LDS_MAC_PER_CLK),
                            "note": "nnz·n·T multiply-adds per pass / time / (148 SMs · SM clock); the "
                                    "operand bytes per multiply-add come from TMEM and/or shared memory, not "
                                    "HBM (the hybrid kernel, 128 < C,K <= 256 with a staged stream, reads "
                                    "half its operands through each: its bound is the sum)"}
        out[name] = k
    return out


def dominant_roofline(kernels, traffic_key=None):
    dom = max(kernels.items(), key=lambda kv: kv[1]["ms_per_step"])[0]
    r = dict(kernels[dom].get("roofline") or {})
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if traffic_key and tfile.exists():
        traffic = json.loads(tfile.read_text()).get(f"{traffic_key}:{dom}")
    r.update({"kernel": dom, "traffic": traffic,
              "note": "algorithmic bytes (or issued ops) per step of the kind / its CUDA-event time per step "
                      "(serialised profiled steps, launching stream)"})
    return r


class LayerBench:
    """One layer configuration on the device: inputs, buffers, and the step variants."""

    def __init__(self, cfg, dev, local_rank, contraction="csr", rank=0, world=1):
        import torch

        import paper_1702_08597_b200 as wb

        self.cfg, self.dev = cfg, dev
        n = cfg.n
        img, w_f, go = make_inputs(cfg)
        if world > 1:  # every rank draws its own shard of the global batch
            from paper_1702_08597_b200.synth import Stream

            img = Stream(cfg.seed + 1000 * rank, "shard/I").normal(img.shape).astype(np.float32)
            go = Stream(cfg.seed + 1000 * rank, "shard/dO").normal(go.shape).astype(np.float32)
        self.img, self.w_f, self.go = img, w_f, go
        self.dense = cfg.sparsity == 0.0
        layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=cfg.pad, m=cfg.m, device=local_rank)
        layer.set_weights(w_f, dense="tc" if self.dense else False)
        if contraction != "csr" and not self.dense:
            layer.set_contraction(contraction)
        self.contraction = contraction
        self.layer = layer
        self.fwd_only = not cfg.backward
        self.cache = layer.new_cache(n) if not self.fwd_only else None
        self.x = torch.from_numpy(img).to(dev)
        self.g = torch.from_numpy(go).to(dev)
        self.out = torch.empty((n, cfg.k, layer.ho, layer.wo), device=dev)
        self.dw = torch.empty(layer.grad_w_shape(), device=dev)
        self.di = torch.empty((n, cfg.c, cfg.h, cfg.w), device=dev)

    def path(self):
        if self.dense:
            return "dense plan: tcgen05 3xTF32 Z/dĨ_F"
        return {"csr": "csr (reference order)", "tc": "tcgen05 3xTF32 on zero-filled W_F",
                "auto": "auto (tcgen05 at density >= 11% for 128 < C,K <= 256, >= 8% otherwise; else csr)"}[self.contraction]

    def compute(self):  # one call, scheduled by data dependence (wino_forward_backward)
        if self.fwd_only:
            self.layer.forward(self.x, None, out=self.out)
        else:
            self.layer.forward_backward(self.x, self.g, self.cache, out=self.out, out_w=self.dw, out_i=self.di)

    def serial(self):  # the same kernels one after another (per-kernel attribution)
        lay = self.layer
        lay.forward(self.x, self.cache, out=self.out)
        if not self.fwd_only:
            lay.backward_weights(self.g, self.cache, out=self.dw)
            lay.backward_input(self.cache, out=self.di)

    def profile(self, flush, steps=3):
        import torch

        self.layer.profile(True)
        for _ in range(steps):
            flush.zero_()
            self.serial()
        torch.cuda.synchronize()
        prof = self.layer.profile_read()
        self.layer.profile(False)
        return prof

    def close(self):
        self.layer.close()


def time_steps(run, flush, steps):
    import torch

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:
        flush.zero_()
        a.record()
        run()
        b.record()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def sweep_point(cfg, dev, local_rank, flush, pk, args, contraction="csr"):
    """One point of the metric's sweep: device-resident step time (CUDA graph, L2 flushed), the
    serialised per-kernel table and the dominant kernel's roofline."""
    import torch

    lb = LayerBench(cfg, dev, local_rank, contraction)
    for _ in range(3):
        lb.compute()
    run, _ = capture(lb.compute, args)
    ms = statistics.median(time_steps(run, flush, args.sweep_steps))
    kernels = kernel_table(lb.profile(flush), 3, cfg, lb.layer, cfg.n, pk)
    passes = 1 if lb.fwd_only else 3
    pt = {"sparsity": cfg.sparsity, "path": lb.path(), "nnz": lb.layer.nnz, "ms": ms,
          "eff_tflops": passes * flops_per_image(cfg) * cfg.n / (ms * 1e-3) / 1e12,
          "dominant": dominant_roofline(kernels, f"{cfg.name}:{cfg.sparsity}"),
          "kernels": {k: {"ms": v["ms_per_step"], "frac": (v.get("roofline") or {}).get("frac"),
                          "bound": (v.get("roofline") or {}).get("bound"),
                          **({"mac_per_clk_sm": v["on_chip"]["mac_per_clk_sm"]} if "on_chip" in v else {})}
                      for k, v in kernels.items()}}
    lb.close()
    del lb, run
    torch.cuda.empty_cache()
    return pt


def run_sweep(args, dev, local_rank, flush, pk):
    """BASELINE metric: 'fwd+bwd effective GFLOP/s and ms/layer vs W_F sparsity, % roofline' —
    configs[3] at 0/50/80/90/95% (CSR; and the 'auto' contraction where it differs), configs[2]
    forward at 80/90/95%, configs[1]."""
    sw = {"c3": [], "c3_auto": [], "c2_fwd": [], "c1": None}
    for s in (0.0, 0.5, 0.8, 0.9, 0.95):
        sw["c3"].append(sweep_point(with_sparsity(CONFIGS["c3"], s), dev, local_rank, flush, pk, args))
        print(f"# sweep c3 {s:.2f}: {sw['c3'][-1]['ms']:.3f} ms", file=sys.stderr, flush=True)
    for s in (0.5, 0.8, 0.9):
        sw["c3_auto"].append(sweep_point(with_sparsity(CONFIGS["c3"], s), dev, local_rank, flush, pk, args, "auto"))
    for s in (0.8, 0.9, 0.95):
        sw["c2_fwd"].append(sweep_point(with_sparsity(CONFIGS["c2"], s), dev, local_rank, flush, pk, args))
    sw["c1"] = sweep_point(CONFIGS["c1"], dev, local_rank, flush, pk, args)
    return sw


def run_gpu(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n = cfg.n
    lb = LayerBench(cfg, dev, local_rank, args.contraction, rank, world)
    layer, dw = lb.layer, lb.dw
    img, w_f, go = lb.img, lb.w_f, lb.go
    dense, fwd_only = lb.dense, lb.fwd_only
    flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)
    if args.call_order and not fwd_only:
        def compute():
            layer.forward(lb.x, lb.cache, out=lb.out)
            layer.backward(lb.g, lb.cache, out_w=lb.dw, out_i=lb.di)
    else:
        compute = lb.compute

    exchange = "none (1 GPU)"
    if world > 1 and not fwd_only:
        # the step's one exchange runs inside the backward call (wino_set_dw_allreduce): NCCL on
        # the dW_F stream right after the dW_F kernels, overlapping the dI chain and the forward
        from paper_1702_08597_b200.dist import nccl_comm_ptr

        layer.set_dw_allreduce(nccl_comm_ptr(device=local_rank))
        exchange = "NCCL all-reduce of nnz-compact dW_F inside the backward call (dW_F stream, overlaps dI)"

    def step():
        compute()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    layer.reset_launch_count()
    step()
    torch.cuda.synchronize()
    per_step_launches = layer.launch_count()
    # the step as one CUDA graph (N > 1: the in-backward NCCL exchange is captured with it; if the
    # capture fails the step runs eagerly and the line says so)
    run, graph_note = capture(compute, args)
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times = time_steps(run, flush, args.steps)
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    launches = per_step_launches * args.steps
    prof = lb.profile(flush)
    ms = sum(times) / args.steps
    ms_t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    allreduce = None
    if world > 1 and not fwd_only:  # the exchange's own cost, timed alone
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        dist.barrier()
        for a, b in evs:
            a.record()
            dist.all_reduce(dw)
            b.record()
        torch.cuda.synchronize()
        ar = torch.tensor([sum(a.elapsed_time(b) for a, b in evs) / len(evs)], device=dev, dtype=torch.float64)
        dist.all_reduce(ar, op=dist.ReduceOp.MAX)
        allreduce = {"ms": float(ar.item()), "bytes": dw.numel() * 4, "share_of_step": float(ar.item()) / ms_max,
                     "backend": dist.get_backend(), "placement": exchange}
    passes = 1 if fwd_only else 3
    flops_step = passes * flops_per_image(cfg) * n
    value = world * flops_step / (ms_max * 1e-3) / 1e9

    e2e = None
    if not args.no_e2e:
        # ---- end to end through the public API with host buffers (pinned) ----
        x, g_o, out, di = lb.x, lb.g, lb.out, lb.di
        h_img = torch.from_numpy(img).pin_memory()
        h_go = torch.from_numpy(go).pin_memory()
        h_out = torch.empty(out.shape, dtype=torch.float32).pin_memory()
        h_dw = torch.empty(dw.shape, dtype=torch.float32).pin_memory()
        h_di = torch.empty(di.shape, dtype=torch.float32).pin_memory()

        if fwd_only:
            def e2e_step():
                x.copy_(h_img, non_blocking=True)
                run()
                h_out.copy_(out, non_blocking=True)
            e2e_mode = "serial copies + forward"
        elif world == 1 and not dense and args.contraction == "csr" and not args.no_pipeline:
            # public API: image chunks so every copy overlaps compute (paper_1702_08597_b200/pipeline.py)
            from paper_1702_08597_b200.graph import GraphedStep
            from paper_1702_08597_b200.pipeline import PipelinedHostStep

            ps = PipelinedHostStep(layer, lb.cache, x, g_o, out, dw, di, chunks=("auto" if args.e2e_chunks == "auto"
                                           else [int(v) for v in args.e2e_chunks.split(",")] if "," in args.e2e_chunks
                                           else int(args.e2e_chunks)))
            # the whole pipelined step (copies on 3 streams + range kernels) as one CUDA graph
            e2e_step = GraphedStep(lambda: ps(h_img, h_go, h_out, h_dw, h_di)).replay
            e2e_mode = (f"PipelinedHostStep in one CUDA graph: pinned host buffers, {len(ps.bounds)} image chunks, "
                        "copies overlapped with the range kernels, dW_F once over the batch")
        elif world == 1 and not args.no_graph:
            # public API: HostStep overlaps dO upload with the forward and the O / dW downloads
            # with the backward (paper_1702_08597_b200/pipeline.py)
            from paper_1702_08597_b200.pipeline import HostStep

            hs = HostStep(layer, lb.cache, x, g_o, out, dw, di)

            def e2e_step():
                hs(h_img, h_go, h_out, h_dw, h_di)
            e2e_mode = "HostStep: pinned host buffers, 3 streams, copies overlapped with compute"
        else:
            def e2e_step():
                x.copy_(h_img, non_blocking=True)
                g_o.copy_(h_go, non_blocking=True)
                run()
                h_out.copy_(out, non_blocking=True)
                h_dw.copy_(dw, non_blocking=True)
                h_di.copy_(di, non_blocking=True)
            e2e_mode = "serial copies + step"

        for _ in range(max(1, args.warmup)):
            e2e_step()
        torch.cuda.synchronize()
        ms_e2e = sum(time_steps(e2e_step, flush, args.steps)) / args.steps
        t2 = torch.tensor([ms_e2e], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        e2e_value = world * flops_step / (float(t2.item()) * 1e-3) / 1e9
        h2d = h_img.numel() * 4 + (0 if fwd_only else h_go.numel() * 4)
        d2h = (h_out.numel() + (0 if fwd_only else h_dw.numel() + h_di.numel())) * 4
        del h_img, h_go, h_out, h_dw, h_di
        e2e = {"value": e2e_value, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": float(t2.item()), "mode": e2e_mode}

    if rank != 0:
        return
    pk = peaks()
    kernels = kernel_table(prof, 3, cfg, layer, n, pk, clocks.get("sm_mhz"))
    roofline = dominant_roofline(kernels, f"{cfg.name}:{cfg.sparsity}")
    line = {
        "metric": METRIC_FWD if fwd_only else METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded splitmix64 normals)",
        "config": {"workload": workload_name(cfg, "fwd" if fwd_only else "fwd+bwd"), "global_batch": n * world,
                   "n_per_gpu": n, "sparsity": cfg.sparsity, "nnz": layer.nnz, "path": lb.path(),
                   "dw": "exact: f64 digits fused into K1/K4 + int8 tcgen05 digit-pair GEMM (strict vs the f64 reference)",
                   "l2_flush": "256 MB write between timed steps (inputs also exceed L2 at c2/c3)",
                   "parallelism": f"dp{world} (batch shards; {exchange})"},
        "ms_per_layer": ms_max,
        "roofline": roofline,
        "kernels": kernels,
        "e2e": e2e,
        "gpu_launches": launches,
        "allreduce": allreduce,
        "launch_mode": graph_note,
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline and fwd_only:
        # the reference's sparse inference (compress + sparse_forward<float>, all host cores),
        # best of 3 after a warm-up call (acceptance.cpp:313-320 style), on a sample of images
        from oracle import ref

        threads = os.cpu_count() or 1
        n_img = min(n, 8)
        imgp = np.pad(img[:n_img].astype(np.float64), ((0, 0), (0, 0), (cfg.pad, cfg.pad), (cfg.pad, cfg.pad)))
        ref.sparse_forward(imgp[:1], w_f, m=cfg.m, workers=threads, precision=32)
        best = float("inf")
        for _ in range(3):
            t0 = time.perf_counter()
            ref.sparse_forward(imgp, w_f, m=cfg.m, workers=threads, precision=32)
            best = min(best, time.perf_counter() - t0)
        line["cpu_baseline"] = {"value": flops_per_image(cfg) * n_img / best / 1e9, "unit": "GFLOP/s",
                                "cores": threads, "kind": "reference",
                                "sample": f"{n_img} of {cfg.n} images through the reference's "
                                          "compress + sparse_forward<float>, best of 3"}
    elif world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        n_img = cpu_sample_size(cfg, threads)
        t, kind = cpu_fwd_bwd(cfg, img, w_f, go, n_img, threads)
        line["cpu_baseline"] = {"value": 3 * flops_per_image(cfg) * n_img / t / 1e9, "unit": "GFLOP/s",
                                "cores": threads, "kind": kind,
                                "sample": f"{n_img} of {cfg.n} images (one per host thread) through the "
                                          "reference's dense f64 per-image fwd+bwd API"}
    lb.close()
    del lb
    torch.cuda.empty_cache()
    if world == 1 and not args.no_sweep:
        line["sweep"] = run_sweep(args, dev, local_rank, flush, pk)
    print(json.dumps(line), flush=True)


def run_gpu_stack(args, cfg, rank, world, local_rank):
    """BASELINE configs[4]: data-parallel training step of a 4-layer stack (C=K=256, H=W=28,
    ReLU between layers, 90% fixed masks), global batch 512 sharded by rank, one bucketed
    NCCL all-reduce of the nnz-compact dW_F, masked SGD.  Effective FLOPs: 4 forward + 4
    backward-weights + 3 backward-input passes (no dI for layer 0, train.cpp:201)."""
    import torch
    import torch.distributed as dist

    from paper_1702_08597_b200.dist import shard
    from paper_1702_08597_b200.stack import WinogradStack
    from paper_1702_08597_b200.synth import LayerConfig, Stream

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n_global = CONFIGS["c4"].n
    _, n = shard(n_global, rank, world)
    layers = 4
    weights = [make_inputs(LayerConfig("c4", 1, cfg.c, cfg.k, cfg.h, cfg.sparsity, seed=cfg.seed), layer=l)[1]
               for l in range(layers)]
    img = Stream(cfg.seed + 1000 * rank, "c4/I").normal((n, cfg.c, cfg.h, cfg.w)).astype(np.float32)
    go = Stream(cfg.seed + 1000 * rank, "c4/dO").normal((n, cfg.k, cfg.h, cfg.w)).astype(np.float32)
    st = WinogradStack(weights, cfg.c, cfg.h, cfg.w, pad=cfg.pad, m=cfg.m, device=local_rank, n_max=n)
    x = torch.from_numpy(img).to(dev)
    g_o = torch.from_numpy(go).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)

    if world > 1:  # each layer's dW_F exchange inside its backward, overlapping its dI chain
        from paper_1702_08597_b200.dist import nccl_comm_ptr

        st.set_dw_allreduce(nccl_comm_ptr(device=local_rank))

    def step():
        st.step(x, g_o, lr=1e-4, n_global=n_global)

    # the same step in parts (WinogradStack.step with mode=None): forward + backward and the
    # masked SGD update each as a CUDA graph, the bucket's one all-reduce issued eagerly between
    # them (no NCCL call is graph-captured)
    def fwd_bwd():
        st.forward(x)
        st.backward(g_o)

    def update():
        for lay, gr in zip(st.layers, st.grads):
            lay.sgd_step(gr, lr=1e-4, scale=1.0 / float(n_global), l2=0.0)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    for lay in st.layers:
        lay.reset_launch_count()
    step()
    torch.cuda.synchronize()
    per_step_launches = st.launch_count()
    run_fb, graph_note = capture(fwd_bwd, args)
    run_up, _ = capture(update, args)

    def run():
        run_fb()
        if not st.in_backward_exchange:
            st.bucket.allreduce()
        run_up()
    if world > 1:
        graph_note += " (forward+backward graph with each layer's NCCL dW_F exchange inside its backward, update graph)"
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in ev:
        flush.zero_()
        a.record()
        run()
        b.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    launches = per_step_launches * args.steps
    # per-kernel times: one step with dW_F and dI serialised (concurrent kernels would share the
    # GPU and inflate each other's event times)
    for lay in st.layers:
        lay.profile(True)
    flush.zero_()
    st.forward(x)
    st.backward(g_o, serial=True)
    torch.cuda.synchronize()
    prof = {}
    for lay in st.layers:
        for k, (t, c) in lay.profile_read().items():
            a0 = prof.get(k, (0.0, 0))
            prof[k] = (a0[0] + t, a0[1] + c)
        lay.profile(False)
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    allreduce = None
    if world > 1:  # the exchange's own cost (the bucket of all layers' dW_F as one collective), timed alone
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        dist.barrier()
        for a, b in evs:
            a.record()
            st.bucket.allreduce()
            b.record()
        torch.cuda.synchronize()
        ar = torch.tensor([sum(a.elapsed_time(b) for a, b in evs) / len(evs)], device=dev, dtype=torch.float64)
        dist.all_reduce(ar, op=dist.ReduceOp.MAX)
        allreduce = {"ms": float(ar.item()), "bytes": st.bucket.flat.numel() * 4,
                     "share_of_step": float(ar.item()) / ms_max, "backend": dist.get_backend()}
    passes = 3 * layers - 1
    value = passes * flops_per_image(cfg) * n_global / (ms_max * 1e-3) / 1e9
    # end to end: host shard in, reduced gradient bucket out
    h_img = torch.from_numpy(img).pin_memory()
    h_go = torch.from_numpy(go).pin_memory()
    h_b = torch.empty(st.bucket.flat.shape, dtype=torch.float32).pin_memory()

    def e2e_step():
        x.copy_(h_img, non_blocking=True)
        g_o.copy_(h_go, non_blocking=True)
        run()
        h_b.copy_(st.bucket.flat, non_blocking=True)

    e2e_step()
    torch.cuda.synchronize()
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in ev2:
        flush.zero_()
        a.record()
        e2e_step()
        b.record()
    torch.cuda.synchronize()
    t2 = torch.tensor([sum(a.elapsed_time(b) for a, b in ev2) / args.steps], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
    if rank != 0:
        return
    tot = sum(v[0] for v in prof.values())
    kernels = {k: {"ms_per_step": v[0], "launches_per_step": v[1], "share": v[0] / tot}
               for k, v in prof.items()}
    line = {
        "metric": METRIC.replace("layer", "4-layer training step"), "value": value, "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded splitmix64 normals)",
        "config": {"workload": f"c4: 4-layer Winograd stack C=K=256 H=W=28 F(4x4,3x3) pad 1, ReLU, "
                               f"90% fixed masks, global batch {n_global} sharded over {world} GPU(s), "
                               "masked SGD, NCCL all-reduce of each layer's nnz-compact dW_F inside its backward",
                   "global_batch": n_global, "n_per_gpu": n, "parallelism": f"dp{world}",
                   "l2_flush": "256 MB write between timed steps"},
        "kernels": kernels,
        "e2e": {"value": passes * flops_per_image(cfg) * n_global / (float(t2.item()) * 1e-3) / 1e9,
                "unit": "GFLOP/s", "h2d_bytes_per_step": (h_img.numel() + h_go.numel()) * 4,
                "d2h_bytes_per_step": h_b.numel() * 4, "ms_per_step": float(t2.item())},
        "gpu_launches": launches, "launch_mode": graph_note, "clocks": clocks, "allreduce": allreduce,
    }
    print(json.dumps(line), flush=True)


def free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn_ranks(args) -> int:
    """`--gpus N` (N > 1) without a torchrun environment: re-launch this script as N ranks under
    torch.distributed.run on 127.0.0.1 — the same command line the driver uses."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", str(Path(__file__).resolve())]
    cmd += sys.argv[1:]
    print(f"# spawning {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def run_dry(args, cfg, rank, world):
    """--dry-run: the multi-rank plumbing of the GPU arm on CPU (gloo): every rank holds the
    nnz-compact dW_F of the config, the step's one exchange (a sum all-reduce) runs, rank 0
    checks the sum and prints one JSON line.  Exercised by tests/test_bench_cpu.py."""
    import torch
    import torch.distributed as dist

    from paper_1702_08597_b200.dist import shard

    _, w_f, _ = make_inputs(cfg, n=1)
    nnz = int(np.count_nonzero(w_f))
    dw = torch.full((nnz,), float(rank + 1))
    if world > 1:
        dist.all_reduce(dw)
    want = world * (world + 1) / 2
    ok = bool(torch.all(dw == want))
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "backend": dist.get_backend() if world > 1 else None,
                          "allreduce_ok": ok, "nnz": nnz, "shards": [shard(cfg.n * world, r, world) for r in range(world)]}),
              flush=True)
    if not ok:
        raise SystemExit("all-reduce sum mismatch")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--sparsity", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the metric's sparsity sweep (the 'sweep' key)")
    ap.add_argument("--sweep-steps", type=int, default=10, help="timed steps per sweep point")
    ap.add_argument("--no-graph", action="store_true", help="launch kernels eagerly (no CUDA graph)")
    ap.add_argument("--no-pipeline", action="store_true", help="e2e through HostStep (whole-batch calls)")
    ap.add_argument("--e2e-chunks", default="auto",
                    help="image chunks of the pipelined e2e step: auto, a count (equal chunks) or a comma list of "
                         "image counts, e.g. 16,16,16,8,4,4")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end (host buffers) measurement (profiling runs)")
    ap.add_argument("--call-order", action="store_true",
                    help="forward then backward as two calls (default: one wino_forward_backward call "
                         "scheduled by data dependence)")
    ap.add_argument("--contraction", default="csr", choices=["csr", "tc", "auto"],
                    help="sparse plan: CSR kernels (bitwise reference order) or tcgen05 on zero-filled W_F")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU only: the rank plumbing and the dW_F all-reduce over gloo (tests)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" and not args.dry_run else args.warmup
    cfg = CONFIGS[args.config]
    if args.sparsity is not None:
        cfg = with_sparsity(cfg, args.sparsity)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        if args.dry_run:
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
            if rank == 0:
                print(f"# NCCL communicator: {dist.get_world_size()} ranks", file=sys.stderr, flush=True)
    try:
        if args.dry_run:
            run_dry(args, cfg, rank, world)
        elif args.config == "c4":
            run_gpu_stack(args, cfg, rank, world, local_rank)
        else:
            run_gpu(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
