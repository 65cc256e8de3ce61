"""Portable seeded synthetic inputs for the BASELINE.json configs.

A splitmix64 counter stream (the mixer the reference uses for its named streams,
train.cpp:15-20) feeds uniforms in [0,1) and Box–Muller normals, so inputs are
reproducible without depending on a library-defined distribution
(std::normal_distribution / numpy Generator algorithms may change).

Configs (BASELINE.json:configs, F(4×4,3×3), pad 1, fp32):
    c0  N=1   C=16  K=16  H=12  70%  fwd+bwd  seed 0
    c1  N=32  C=256 K=384 H=13  90%  fwd+bwd
    c2  N=64  C=512 K=512 H=28  80/90/95%  fwd only
    c3  N=64  C=256 K=256 H=56  0/50/80/90/95%  fwd+bwd
    c4  N=512 (global) C=K=256 H=28, 4 layers, 90% fixed masks, DP step
I, dL/dO ~ N(0,1); W_F nonzeros ~ N(0, 2/(9C)) under an independent Bernoulli
keep-mask (keep = 1 − sparsity) per element of each K×C slice.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def _fnv1a(s: str) -> int:
    h = 0xCBF29CE484222325
    for ch in s.encode():
        h ^= ch
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def stream_seed(seed: int, name: str) -> int:
    """train.cpp:104-106: splitmix64(seed ^ fnv1a(name))."""
    return int(_splitmix64(np.array([(seed ^ _fnv1a(name)) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0])


class Stream:
    """Counter-based splitmix64 stream: value i = splitmix64(key + i·golden)."""

    def __init__(self, seed: int, name: str):
        self.key = np.uint64(stream_seed(seed, name))
        self.ctr = 0

    def _bits(self, n: int) -> np.ndarray:
        idx = np.arange(self.ctr, self.ctr + n, dtype=np.uint64)
        self.ctr += n
        with np.errstate(over="ignore"):
            return _splitmix64(self.key + idx * np.uint64(0xD1B54A32D192ED03))

    def uniform(self, shape) -> np.ndarray:
        n = int(np.prod(shape))
        return ((self._bits(n) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)).reshape(shape)

    def normal(self, shape) -> np.ndarray:
        n = int(np.prod(shape))
        m = (n + 1) // 2
        u1 = 1.0 - self.uniform((m,))          # (0,1]
        u2 = self.uniform((m,))
        rad = np.sqrt(-2.0 * np.log(u1))
        z = np.concatenate([rad * np.cos(2 * np.pi * u2), rad * np.sin(2 * np.pi * u2)])
        return z[:n].reshape(shape)


@dataclass(frozen=True)
class LayerConfig:
    name: str
    n: int
    c: int
    k: int
    h: int
    sparsity: float
    pad: int = 1
    m: int = 4
    r: int = 3
    backward: bool = True
    seed: int = 0

    @property
    def w(self):
        return self.h


CONFIGS = {
    "c0": LayerConfig("c0", 1, 16, 16, 12, 0.70, seed=0),
    "c1": LayerConfig("c1", 32, 256, 384, 13, 0.90, seed=1),
    "c2": LayerConfig("c2", 64, 512, 512, 28, 0.90, backward=False, seed=2),
    "c3": LayerConfig("c3", 64, 256, 256, 56, 0.90, seed=3),
    "c4": LayerConfig("c4", 512, 256, 256, 28, 0.90, seed=4),
}


def with_sparsity(cfg: LayerConfig, s: float) -> LayerConfig:
    return LayerConfig(cfg.name, cfg.n, cfg.c, cfg.k, cfg.h, s, cfg.pad, cfg.m, cfg.r,
                       cfg.backward, cfg.seed)


def make_inputs(cfg: LayerConfig, n: int | None = None, layer: int = 0, dtype=np.float32):
    """(I N×C×H×W, W_F K×C×p×p with exact zeros, dL/dO N×K×Ho×Wo) for a config."""
    n = cfg.n if n is None else n
    p = cfg.m + cfg.r - 1
    tag = f"{cfg.name}/L{layer}"
    img = Stream(cfg.seed, tag + "/I").normal((n, cfg.c, cfg.h, cfg.w)).astype(dtype)
    wv = Stream(cfg.seed, tag + "/W").normal((cfg.k, cfg.c, p, p)) * np.sqrt(2.0 / (9.0 * cfg.c))
    keep = Stream(cfg.seed, tag + "/M").uniform((cfg.k, cfg.c, p, p)) >= cfg.sparsity
    w_f = np.where(keep, wv, 0.0).astype(np.float32).astype(np.float64)
    ho = cfg.h + 2 * cfg.pad - cfg.r + 1
    go = Stream(cfg.seed, tag + "/dO").normal((n, cfg.k, ho, ho)).astype(dtype)
    return img, w_f, go
