"""`infer-bench` on the GPU: the reference CLI's sparse-inference sweep (tools/wino.cpp:321-381)
with the contraction served by the B200 kernels.

For every layer of a `--layers` config ([name] c=, k=, h=, r=3, m=2; wino.cpp:269-287) it builds
the reference's exact inputs — a batch N×C×(h+r−1)² and W_F K×C×p×p drawn, in that order, from
one mt19937_64 seeded with stream_seed(seed, "bench/<name>") through libstdc++'s
uniform_real_distribution(-1, 1) — then for each density of the sweep keeps the top-|w|
floor(x·size) weights (train.cpp:419-429), and times compress + sparse forward.  The CSV has
the reference's columns and formatting:

    layer,density,workers,wall_ns,effective_gflops,checksum

`checksum` (sequential double sum of the output) equals the reference's f32 run bit for bit,
because the forward is bitwise the reference's sparse_forward<float>.
`wall_ns` is host wall time of one drop-in call: CSR build on the GPU from the host W_F, the
batch's H2D copy, the forward, and the output's D2H copy.  `workers` is reported as the
reference computes it (effective_workers, harness.cpp:144-151); it does not affect the GPU.
"""
from __future__ import annotations

import argparse
import math
import os
import sys
import time
from dataclasses import dataclass

import numpy as np

from .io import Config, ConfigError

_M64 = (1 << 64) - 1


# -- the reference's seeded streams (train.cpp:15-29, 104-106) ------------------------------
def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def fnv1a(s: str) -> int:
    h = 0xCBF29CE484222325
    for c in s.encode():
        h = ((h ^ c) * 0x100000001B3) & _M64
    return h


def stream_seed(seed: int, name: str) -> int:
    return splitmix64((seed & _M64) ^ fnv1a(name))


class MT19937_64:
    """std::mt19937_64 (the published MT19937-64 recurrence and tempering), one 312-word
    block regenerated per numpy step."""

    N, M = 312, 156
    _A = np.uint64(0xB5026F5AA96619E9)
    _UM = np.uint64(0xFFFFFFFF80000000)
    _LM = np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = [seed & _M64]
        for i in range(1, self.N):
            prev = mt[-1]
            mt.append((6364136223846793005 * (prev ^ (prev >> 62)) + i) & _M64)
        self.mt = np.array(mt, dtype=np.uint64)
        self.pending = np.zeros(0, dtype=np.uint64)

    def _step(self, cur, nxt, far):
        y = (cur & self._UM) | (nxt & self._LM)
        return far ^ (y >> np.uint64(1)) ^ ((y & np.uint64(1)) * self._A)

    def _twist(self):
        x, n, m = self.mt, self.N, self.M
        x[0:n - m] = self._step(x[0:n - m], x[1:n - m + 1], x[m:n])
        x[n - m:n - 1] = self._step(x[n - m:n - 1], x[n - m + 1:n], x[0:m - 1])
        x[n - 1:n] = self._step(x[n - 1:n], x[0:1], x[m - 1:m])

    @staticmethod
    def _temper(z):
        z = z ^ ((z >> np.uint64(29)) & np.uint64(0x5555555555555555))
        z = z ^ ((z << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000))
        z = z ^ ((z << np.uint64(37)) & np.uint64(0xFFF7EEE000000000))
        return z ^ (z >> np.uint64(43))

    def next_u64(self, n: int) -> np.ndarray:
        out = [self.pending[:n]]
        have = out[0].size
        self.pending = self.pending[have:]
        blocks = []
        while have < n:
            self._twist()
            blocks.append(self.mt.copy())
            have += self.N
        if blocks:
            z = self._temper(np.concatenate(blocks))
            need = n - out[0].size
            out.append(z[:need])
            self.pending = z[need:]
        return np.concatenate(out)


def uniform(rng: MT19937_64, n: int, a: float = -1.0, b: float = 1.0) -> np.ndarray:
    """libstdc++ uniform_real_distribution<double>: generate_canonical<double,53> with one 64-bit
    draw (double(x) / 2^64, clamped below 1), then u·(b−a) + a."""
    u = rng.next_u64(n).astype(np.float64) / 18446744073709551616.0
    u[u >= 1.0] = np.nextafter(1.0, 0.0)
    return u * (b - a) + a


def uniform_stream(seed: int, name: str, n: int) -> np.ndarray:
    return uniform(MT19937_64(stream_seed(seed, name)), n)


def magnitude_threshold_to_density(w: np.ndarray, density: float) -> np.ndarray:
    """train.cpp:419-429: keep the floor(x·size) largest |w| (stable order), zero the rest."""
    flat = np.array(w, dtype=np.float64).ravel()
    keep = int(math.floor(density * float(flat.size)))
    if keep >= flat.size:
        return flat.reshape(np.shape(w))
    order = np.argsort(-np.abs(flat), kind="stable")
    flat[order[keep:]] = 0.0
    return flat.reshape(np.shape(w))


# -- harness helpers (harness.cpp:92-151) ---------------------------------------------------
def csv_field(s: str) -> str:
    if not any(ch in s for ch in ',"\n\r'):
        return s
    return '"' + s.replace('"', '""') + '"'


def csv_row(fields) -> str:
    return ",".join(csv_field(f) for f in fields)


def parse_density_grid(spec: str) -> list[float]:
    c1 = spec.find(":")
    c2 = spec.find(":", c1 + 1) if c1 >= 0 else -1
    if c1 < 0 or c2 < 0:
        raise ConfigError(f"density grid must be lo:hi:count or lo:hi:logN, got {spec}")
    lo, hi = float(spec[:c1]), float(spec[c1 + 1:c2])
    tail = spec[c2 + 1:]
    log_spaced, count = False, 20
    if tail.startswith("log"):
        log_spaced = True
        if tail[3:]:
            count = int(tail[3:])
    else:
        count = int(tail)
    if lo <= 0.0 or hi < lo or count == 0:
        raise ConfigError(f"bad density grid {spec}")
    if count == 1 or hi == lo:
        return [lo]
    out = []
    for i in range(count):
        f = i / (count - 1)
        out.append(lo * math.pow(hi / lo, f) if log_spaced else lo + f * (hi - lo))
    return out


def effective_workers(requested: int) -> int:
    env = os.environ.get("WINO_THREADS")
    if env:
        try:
            cap = int(env.strip().split()[0]) if env.strip() else 0
        except ValueError:
            cap = 0
        if 0 < cap < requested:
            return cap
    return 1 if requested == 0 else requested


def fmt_g(x: float) -> str:
    """std::ostream << double with default flags (precision 6, %g)."""
    return "%g" % x


@dataclass
class LayerDims:
    """perf::LayerDims (perfmodel.hpp)."""

    name: str
    c: int
    k: int
    h: int
    r: int = 3
    m: int = 2

    @property
    def p(self):
        return self.m + self.r - 1

    def flops_baseline(self) -> float:
        """perfmodel.cpp:6-9."""
        return 2.0 * self.c * self.k * float(self.h * self.h) * float(self.r * self.r)


def layers_from_config(path) -> list[LayerDims]:
    """wino.cpp:269-287."""
    cfg = Config.parse_file(path)
    layers = []
    for section in cfg.sections():
        if not section:
            continue
        d = LayerDims(section, cfg.get_int(section, "c", 0), cfg.get_int(section, "k", 0),
                      cfg.get_int(section, "h", 0), cfg.get_int(section, "r", 3), cfg.get_int(section, "m", 2))
        if not (d.c and d.k and d.h):
            raise ConfigError(f"layer {section} needs c, k, and h")
        layers.append(d)
    if not layers:
        raise ConfigError(f"no layers in {path}")
    return layers


def bench_inputs(d: LayerDims, batch: int, seed: int):
    """(batch N×C×Hi×Hi, W_F K×C×p×p) exactly as wino.cpp:336-342 draws them."""
    hi = d.h + d.r - 1
    rng = MT19937_64(stream_seed(seed, "bench/" + d.name))
    nb = batch * d.c * hi * hi
    v = uniform(rng, nb + d.k * d.c * d.p * d.p)
    return v[:nb].reshape(batch, d.c, hi, hi), v[nb:].reshape(d.k, d.c, d.p, d.p)


def checksum(out: np.ndarray) -> float:
    """Sequential left-to-right double sum (wino.cpp:362-363); np.cumsum never reassociates."""
    flat = np.asarray(out, dtype=np.float64).ravel()
    return float(np.cumsum(flat)[-1]) if flat.size else 0.0


def run(layers, grid, batch=8, precision="f32", workers=1, seed=1, warmup=True):
    """Rows of (layer, density, workers, wall_ns, effective_gflops, checksum)."""
    import torch

    from .layer import WinogradLayer
    from ._lib import CapabilityError

    if precision not in ("f32", "f64"):
        raise ConfigError("precision must be f32 or f64")
    if precision != "f32":
        raise CapabilityError("the B200 path computes in fp32; use --precision f32")
    workers = effective_workers(workers)
    rows = []
    for d in layers:
        b, w_f = bench_inputs(d, batch, seed)
        layer = WinogradLayer(d.c, d.k, b.shape[2], b.shape[3], pad=0, m=d.m, r=d.r)
        h_in = torch.from_numpy(b.astype(np.float32)).pin_memory()
        x = torch.empty(h_in.shape, dtype=torch.float32, device="cuda")
        out = torch.empty((batch, d.k, layer.ho, layer.wo), dtype=torch.float32, device="cuda")
        h_out = torch.empty(out.shape, dtype=torch.float32).pin_memory()
        if warmup:  # context, module load and kernel attributes, outside every timed call
            layer.set_weights(w_f, dense=False)
            x.copy_(h_in, non_blocking=True)
            layer.forward(x, out=out)
            torch.cuda.synchronize()
        for dens in grid:
            w = magnitude_threshold_to_density(w_f, dens)
            torch.cuda.synchronize()
            t0 = time.perf_counter_ns()
            layer.set_weights(w, dense=False)
            x.copy_(h_in, non_blocking=True)
            layer.forward(x, out=out)
            h_out.copy_(out, non_blocking=True)
            torch.cuda.synchronize()
            wall_ns = time.perf_counter_ns() - t0
            gflops = d.flops_baseline() * float(batch) / float(wall_ns)
            rows.append((d.name, dens, workers, wall_ns, gflops, checksum(h_out.numpy())))
        layer.close()
    return rows


def format_csv(rows) -> str:
    lines = [csv_row(["layer", "density", "workers", "wall_ns", "effective_gflops", "checksum"])]
    for name, dens, wk, ns, gf, cs in rows:
        lines.append(csv_row([name, fmt_g(dens), str(wk), str(ns), fmt_g(gf), fmt_g(cs)]))
    return "\n".join(lines) + "\n"


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="infer-bench", description=__doc__.splitlines()[0])
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--layers", required=True)
    ap.add_argument("--density-sweep", default="0.02:1.0:log")
    ap.add_argument("--precision", default="f32")
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--csv", default="")
    ap.add_argument("--seed", type=int, default=1)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:  # usage errors are validation errors (wino.cpp:482-486)
        return 0 if e.code == 0 else 1
    try:
        rows = run(layers_from_config(a.layers), parse_density_grid(a.density_sweep), a.batch,
                   a.precision, a.workers, a.seed)
    except Exception as e:  # std::exception -> kExitValidation (wino.cpp:493-496)
        print(f"error: {e}", file=sys.stderr)
        return 1
    text = format_csv(rows)
    if a.csv:
        with open(a.csv, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
