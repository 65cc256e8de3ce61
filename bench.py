#!/usr/bin/env python
"""Benchmark of the Winograd-layer fwd+bwd hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1] [--sparsity S]
    python bench.py --impl reference ...      # the reference's own CPU path on the host cores

A step = forward (with ForwardCache) + backward_weights + backward_input of one layer over
one batch of the config (configs[1] by default: N=32, C=256, K=384, H=W=13, F(4x4,3x3),
pad 1, 90% W_F sparsity), inputs resident in HBM.  With N>1 GPUs (torchrun) every rank runs
its own batch (weak scaling: batch sharding) and dW_F (nnz-compact) is all-reduced over NCCL
inside the step.  Effective GFLOP/s follows the reference convention
(tools/wino.cpp:362, perfmodel.cpp:6-9): 2·C·K·H²·9 per image and pass, 3 passes.

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
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"], "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


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


def kernel_bytes(cfg, layer, n):
    """Algorithmic HBM bytes per launch of each kernel."""
    g = layer.geometry
    nt = n * g["t"]
    p2 = g["p"] ** 2
    f = 4
    I = n * cfg.c * cfg.h * cfg.w * f
    O = n * cfg.k * g["h_o"] * g["w_o"] * f
    V = p2 * cfg.c * nt * f
    Z = p2 * cfg.k * nt * f
    nnz = layer.nnz
    Wb = 8 * nnz + 4 * p2 * (cfg.k + 1)
    Wt = 8 * nnz + 4 * p2 * (cfg.c + 1)
    dw = nnz * f
    return {
        "input_transform": I + V, "spmm_fwd": V + Z + Wb, "output_transform": Z + O,
        "grad_z": O + Z, "sddmm_dw": Z + V + dw + 8 * nnz + 4 * p2 * (cfg.k + 1),
        "spmm_bwd_data": Z + Wt + V, "input_grad": V + I,
    }


def run_gpu(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1702_08597_b200 as wb

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n = cfg.n
    img, w_f, go = make_inputs(cfg)
    if world > 1:  # every rank draws its own shard of the global batch
        from paper_1702_08597_b200.synth import Stream

        img = Stream(cfg.seed + 1000 * rank, "shard/I").normal(img.shape).astype(np.float32)
        go = Stream(cfg.seed + 1000 * rank, "shard/dO").normal(go.shape).astype(np.float32)
    layer = wb.WinogradLayer(cfg.c, cfg.k, cfg.h, cfg.w, pad=cfg.pad, m=cfg.m, device=local_rank)
    dense = cfg.sparsity == 0.0
    layer.set_weights(w_f, dense=(args.dense or "tc") if dense else False)
    if args.dw == "tc" and not dense:
        layer.set_dw_mode("tc")
    elif args.dw == "precise":
        layer.set_dw_mode("precise")
    elif args.dw == "int8" and not dense:
        layer.set_dw_mode("int8")
    if args.contraction != "csr" and not dense:
        layer.set_contraction(args.contraction)
    cache = layer.new_cache(n)
    x = torch.from_numpy(img).to(dev)
    g_o = torch.from_numpy(go).to(dev)
    out = torch.empty((n, cfg.k, layer.ho, layer.wo), device=dev)
    dw = torch.empty(layer.grad_w_shape(), device=dev)
    di = torch.empty((n, cfg.c, cfg.h, cfg.w), device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)

    fwd_only = not cfg.backward  # c2: the reference's sparse inference pass

    def compute():
        layer.forward(x, cache, out=out)
        if fwd_only:
            return
        if args.separate_bwd:
            layer.backward_weights(g_o, cache, out=dw)
            layer.backward_input(cache, out=di)
        else:  # dW_F concurrently with dI (wino_backward)
            layer.backward(g_o, cache, out_w=dw, out_i=di)

    if not fwd_only and not args.separate_bwd and not args.call_order:
        def compute():  # one call, scheduled by data dependence (wino_forward_backward)
            layer.forward_backward(x, g_o, cache, out=out, out_w=dw, out_i=di)

    def step():
        compute()
        if world > 1 and not fwd_only:
            dist.all_reduce(dw)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    layer.reset_launch_count()
    step()
    torch.cuda.synchronize()
    per_step_launches = layer.launch_count()
    # the layer's kernels as one CUDA graph; the step's one collective (N > 1) is issued eagerly
    # after the replay, on the same stream, so no NCCL call is ever graph-captured
    run_c, graph_note = capture(compute, args)
    if world > 1 and not fwd_only:
        def run():
            run_c()
            dist.all_reduce(dw)
        graph_note += " + eager NCCL all-reduce of dW_F"
    else:
        run = run_c
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    sampler = ClockSampler(local_rank)
    sampler.start()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
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
    # per-kernel times for the roofline: eager steps with CUDA events around every launch, the
    # backward serialised (in the timed step dW_F runs concurrently with dI, which would blur the
    # attribution of time to kernels)
    def step_serial():
        layer.forward(x, cache, out=out)
        if not fwd_only:
            layer.backward_weights(g_o, cache, out=dw)
            layer.backward_input(cache, out=di)

    layer.profile(True)
    for _ in range(3):
        flush.zero_()
        step_serial()
    torch.cuda.synchronize()
    prof = layer.profile_read()
    layer.profile(False)
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    ms_t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    allreduce = None
    if world > 1 and not fwd_only:  # the one exchange of the step, timed alone
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
                     "backend": dist.get_backend()}
    passes = 1 if fwd_only else 3
    flops_step = passes * flops_per_image(cfg) * n
    value = world * flops_step / (ms_max * 1e-3) / 1e9

    # ---- end to end through the public API with host buffers (pinned) ----
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
    elif world == 1 and not dense and args.contraction == "csr" and args.dw == "sddmm" and not args.no_pipeline:
        # public API: image chunks so every copy overlaps compute (paper_1702_08597_b200/pipeline.py)
        from paper_1702_08597_b200.pipeline import PipelinedHostStep

        ps = PipelinedHostStep(layer, cache, x, g_o, out, dw, di, chunks=args.e2e_chunks)
        from paper_1702_08597_b200.graph import GraphedStep

        # the whole pipelined step (copies on 3 streams + range kernels) as one CUDA graph
        e2e_step = GraphedStep(lambda: ps(h_img, h_go, h_out, h_dw, h_di)).replay
        e2e_mode = (f"PipelinedHostStep in one CUDA graph: pinned host buffers, {len(ps.bounds)} image chunks, "
                    "copies overlapped with the range kernels, dW_F once over the batch")
    elif world == 1 and not args.no_graph:
        # public API: HostStep overlaps dO upload with the forward and the O / dW downloads
        # with the backward (paper_1702_08597_b200/pipeline.py)
        from paper_1702_08597_b200.pipeline import HostStep

        hs = HostStep(layer, cache, x, g_o, out, dw, di)

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
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for a, b in ev2:
        flush.zero_()
        a.record()
        e2e_step()
        b.record()
    torch.cuda.synchronize()
    ms_e2e = sum(a.elapsed_time(b) for a, b in ev2) / args.steps
    t2 = torch.tensor([ms_e2e], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
    e2e_value = world * flops_step / (float(t2.item()) * 1e-3) / 1e9
    h2d = h_img.numel() * 4 + (0 if fwd_only else h_go.numel() * 4)
    d2h = (h_out.numel() + (0 if fwd_only else h_dw.numel() + h_di.numel())) * 4

    if rank != 0:
        return
    pk = peaks()
    kb = kernel_bytes(cfg, layer, n)
    kernels = {}
    # a kind can launch more than once per step (SDDMM + its split_sum, the dW GEMM + its fp64
    # reduce): times and achieved bandwidth are per STEP of the kind (3 profiled steps), i.e. the
    # algorithmic bytes of one pass over the kernel's data ÷ all of that pass's launches
    for name, (tot_ms, cnt) in prof.items():
        avg = tot_ms / 3
        bytes_ = kb.get(name)
        kernels[name] = {"ms_per_step": avg, "launches_per_step": cnt / 3,
                         "share": tot_ms / sum(v[0] for v in prof.values())}
        if bytes_:
            kernels[name]["alg_bytes"] = bytes_
            kernels[name]["GBps"] = bytes_ / (avg * 1e-3) / 1e9
    dom = max(prof.items(), key=lambda kv: kv[1][0])[0]
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get(f"{cfg.name}:{cfg.sparsity}:{dom}")
    if dom.startswith("dense_"):
        # tensor-pipe roofline: 3xTF32 issues 3 TF32 products per useful MAC; TF32 dense peak is
        # taken as half the measured bf16 GEMM peak (MEASURED_PEAKS.json)
        g = layer.geometry
        useful = 2.0 * (g["p"] ** 2) * cfg.k * cfg.c * n * g["t"]
        avg_s = prof[dom][0] / 3 * 1e-3
        issued_tf = 3 * useful / avg_s / 1e12
        peak_tf = pk["bf16_tflops"] / 2
        roofline = {"bound": "tensor", "kernel": dom, "achieved": issued_tf, "peak": peak_tf,
                    "unit": "TFLOP/s", "frac": issued_tf / peak_tf, "traffic": traffic,
                    "peak_source": pk["source"] + " (bf16/2 for tf32)",
                    "note": "issued TF32 FLOP/s of the 3xTF32 GEMM (useful = 1/3); time = the kind's launches per step"}
    else:
        dom_gbs = kernels[dom].get("GBps")
        roofline = {"bound": "hbm", "kernel": dom, "achieved": dom_gbs, "peak": pk["hbm_gbs"],
                    "unit": "GB/s", "frac": (dom_gbs / pk["hbm_gbs"]) if dom_gbs else None,
                    "traffic": traffic, "peak_source": pk["source"],
                    "note": ("algorithmic bytes per step / CUDA-event time of the kind's launches in the step (on the launching stream); "
                             "c1's per-kernel working set (<64 MB) is L2-resident within a step")}
    # the on-chip pipe that bounds the CSR contraction kernels: the SDDMM converts
    # one fp32 operand to fp64 per exact product on the XU pipe (16 lanes/clk/SM); the SpMMs read
    # one 4-byte Ĩ_F/dZ operand per product from shared memory (128 B/clk/SM = 32 products/clk/SM)
    pipe_roofline = None
    g_ = layer.geometry
    products = float(layer.nnz) * n * g_["t"]
    clk = (clocks.get("sm_mhz") or 1965.0) * 1e6
    pipes = {"sddmm_dw": ("XU: F2F.F64.F32, one per exact product", 16.0),
             "spmm_fwd": ("shared-memory pipe: 4 B per product", 32.0),
             "spmm_bwd_data": ("shared-memory pipe: 4 B per product", 32.0)}
    if dom in pipes and not dense:
        name_, peak_ = pipes[dom]
        # sddmm_dw's two launches per step (SDDMM + split_sum) are both counted: a lower bound
        t_dom = prof[dom][0] / 3 * 1e-3
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        ach = products / t_dom / sms / clk
        pipe_roofline = {"kernel": dom, "pipe": name_, "unit": "products/clk/SM", "achieved": ach,
                         "peak": peak_, "frac": ach / peak_,
                         "note": "products = nnz·N·T per launch; time from the same CUDA events"}
    line = {
        "metric": METRIC_FWD if fwd_only else METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded splitmix64 normals)",
        "config": {"workload": workload_name(cfg, "fwd" if fwd_only else "fwd+bwd"), "global_batch": n * world,
                   "n_per_gpu": n, "sparsity": cfg.sparsity, "nnz": layer.nnz,
                   "path": ({"tc": "dense-tcgen05-3xtf32-fp64fold", "tc-fast": "dense-tcgen05-3xtf32-fast",
                             "exact": "dense-exact-simt"}[args.dense or "tc"]) if dense else
                           {"csr": "csr", "tc": "tcgen05-3xtf32-fp64fold on zero-filled W_F",
                            "auto": "auto (tensor cores at density >= 8%, else csr)"}[args.contraction],
                   "dw": {"sddmm": "masked-sddmm-exact", "tc": "tcgen05-3xtf32-fp64fold+mask-gather",
                          "precise": "masked-sddmm-exact on fp32 hi+lo operands",
                          "int8": "int8-tcgen05-exact-digit-products+mask-gather"}[args.dw],
                   "l2_flush": "256 MB write between timed steps",
                   "parallelism": f"dp{world} (batch shards, NCCL all-reduce of nnz-compact dW_F)"},
        "ms_per_layer": ms_max,
        "roofline": roofline,
        "pipe_roofline": pipe_roofline,
        "kernels": kernels,
        "e2e": {"value": e2e_value, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": float(t2.item()), "mode": e2e_mode},
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
                                "sample": f"{n_img} of {cfg.n} images (one step's worth per thread) "
                                          "through the reference's dense f64 fwd+bwd API"}
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

    def step():
        st.step(x, g_o, lr=1e-4, n_global=n_global)

    # the same step in three parts (WinogradStack.step with mode=None): forward + backward and the
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
        st.bucket.allreduce()
        run_up()
    if world > 1:
        graph_note += " (forward+backward and update graphs, eager NCCL all-reduce between)"
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
    if world > 1:  # the step's one exchange (the bucket of all layers' dW_F), timed alone
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
                               "masked SGD, one NCCL all-reduce of nnz-compact dW_F per step",
                   "global_batch": n_global, "n_per_gpu": n, "parallelism": f"dp{world}",
                   "l2_flush": "256 MB write between timed steps"},
        "kernels": kernels,
        "e2e": {"value": passes * flops_per_image(cfg) * n_global / (float(t2.item()) * 1e-3) / 1e9,
                "unit": "GFLOP/s", "h2d_bytes_per_step": (h_img.numel() + h_go.numel()) * 4,
                "d2h_bytes_per_step": h_b.numel() * 4, "ms_per_step": float(t2.item())},
        "gpu_launches": launches, "launch_mode": graph_note, "clocks": clocks, "allreduce": allreduce,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c1", choices=sorted(CONFIGS))
    ap.add_argument("--sparsity", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch kernels eagerly (no CUDA graph)")
    ap.add_argument("--no-pipeline", action="store_true", help="e2e through HostStep (whole-batch calls)")
    ap.add_argument("--e2e-chunks", type=int, default=4, help="image chunks of the pipelined e2e step")
    ap.add_argument("--call-order", action="store_true",
                    help="forward then backward as two calls (default: one wino_forward_backward call "
                         "scheduled by data dependence)")
    ap.add_argument("--separate-bwd", action="store_true",
                    help="backward_weights then backward_input instead of the concurrent wino_backward")
    ap.add_argument("--contraction", default="csr", choices=["csr", "tc", "auto"],
                    help="sparse plan: CSR kernels (bitwise reference order) or tcgen05 on zero-filled W_F")
    ap.add_argument("--dw", default="sddmm", choices=["sddmm", "tc", "precise", "int8"],
                    help="sparse dW_F: exact masked SDDMM (default) or tensor-core GEMM + mask gather")
    ap.add_argument("--dense", default=None, choices=["tc", "tc-fast", "exact"],
                    help="dense path at 0%% sparsity: 'tc' (default: 3xTF32 tcgen05, per-k-block fp64 "
                         "folding), 'tc-fast' (one TMEM chain), 'exact' (reference-order SIMT)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    cfg = CONFIGS[args.config]
    if args.sparsity is not None:
        cfg = with_sparsity(cfg, args.sparsity)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.config == "c4":
            run_gpu_stack(args, cfg, rank, world, local_rank)
        else:
            run_gpu(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
