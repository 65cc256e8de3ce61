"""On-disk formats shared with the reference.

* WGT1 tensors (tensor.hpp:109-114, tensor.cpp:166-216): magic "WGT1", u8 dtype (1 = f64,
  2 = f32), u8 ndim, ndim × u32 little-endian extents, then little-endian row-major elements.
  Files are byte-identical to the reference's writer and readable by its reader.
* key=value configs with [sections] and # comments (harness.cpp:23-90).
* Layer checkpoints (harness.cpp:152-212): a directory of WGT1 weights/masks + manifest.cfg in
  the reference's layout.  The manifest additionally records the tile size `m` of each
  Winograd layer — the reference's load_checkpoint hard-codes F(2x2,3x3) (harness.cpp:192), so
  an F(4x4,3x3) checkpoint could not be reloaded faithfully; a manifest without `m` (one the
  reference wrote) loads as m = 2, exactly as the reference does.
"""
from __future__ import annotations

import os
import re
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np


class IoError(IOError):
    """wino::IoError (tensor.hpp:17-20) -> IOError, as bindings.cpp:202."""


class ConfigError(ValueError):
    """wino::harness::ConfigError."""


_DT = {1: np.dtype("<f8"), 2: np.dtype("<f4")}


def write_wgt1(path, array, dtype: str = "f64") -> None:
    """tensor.cpp:166-184."""
    a = np.asarray(array, dtype=np.float64)
    code = {"f64": 1, "f32": 2}.get(dtype)
    if code is None:
        raise ValueError("dtype must be f64 or f32")
    if a.ndim > 255 or any(e == 0 or e >= 2 ** 32 for e in a.shape):
        raise IoError(f"cannot write shape {a.shape}")
    try:
        with open(path, "wb") as f:
            f.write(b"WGT1" + bytes([code, a.ndim]) + struct.pack(f"<{a.ndim}I", *a.shape))
            f.write(np.ascontiguousarray(a, dtype=_DT[code]).tobytes())
    except OSError as e:
        raise IoError(f"write failed for {path}: {e}") from e


def read_wgt1(path, return_dtype: bool = False):
    """tensor.cpp:186-216 (returns f64, like the reference's Tensor)."""
    try:
        data = Path(path).read_bytes()
    except OSError as e:
        raise IoError(f"cannot open {path}") from e
    if len(data) < 4 or data[:4] != b"WGT1":
        raise IoError(f"{path}: bad WGT1 magic")
    if len(data) < 6:
        raise IoError(f"{path}: truncated header")
    code, ndim = data[4], data[5]
    if code not in _DT:
        raise IoError(f"{path}: unknown dtype code")
    off = 6 + 4 * ndim
    if len(data) < off:
        raise IoError("truncated WGT1 header")
    shape = struct.unpack(f"<{ndim}I", data[6:off])
    if any(e == 0 for e in shape):
        raise IoError(f"{path}: zero extent")
    n = int(np.prod(shape, dtype=np.int64)) if ndim else 1
    nbytes = n * _DT[code].itemsize
    if len(data) < off + nbytes:
        raise IoError(f"{path}: truncated payload")
    arr = np.frombuffer(data, dtype=_DT[code], count=n, offset=off).astype(np.float64).reshape(shape)
    return (arr, {1: "f64", 2: "f32"}[code]) if return_dtype else arr


class Config:
    """harness.cpp:23-90: [section] headers, key=value, # comments; later keys win."""

    def __init__(self):
        self.values: dict[str, dict[str, str]] = {}

    @staticmethod
    def parse_string(text: str) -> "Config":
        cfg = Config()
        section = ""
        ws = " \t\r\n"  # the reference's trim() set
        for lineno, line in enumerate(text.split("\n"), 1):
            line = line.split("#", 1)[0].strip(ws)
            if not line:
                continue
            if line.startswith("["):
                if not line.endswith("]"):
                    raise ConfigError(f"malformed section header at line {lineno}")
                section = line[1:-1].strip(ws)
                continue
            if "=" not in line:
                raise ConfigError(f"expected key=value at line {lineno}")
            k, v = line.split("=", 1)
            cfg.values.setdefault(section, {})[k.strip(ws)] = v.strip(ws)
        return cfg

    @staticmethod
    def parse_file(path) -> "Config":
        try:
            return Config.parse_string(Path(path).read_text())
        except OSError as e:
            raise ConfigError(f"cannot open config file {path}") from e

    def has(self, section, key):
        return key in self.values.get(section, {})

    def get(self, section, key):
        if not self.has(section, key):
            raise ConfigError(f"missing config key [{section}] {key}")
        return self.values[section][key]

    def get_or(self, section, key, fallback):
        return self.get(section, key) if self.has(section, key) else fallback

    def get_int(self, section, key, fallback=0):
        """std::stoll semantics: the leading integer prefix; ValueError (std::invalid_argument) if none."""
        if not self.has(section, key):
            return fallback
        mt = re.match(r"\s*[+-]?\d+", self.get(section, key))
        if not mt:
            raise ValueError(f"stoll: [{section}] {key}")
        return int(mt.group(0))

    def get_double(self, section, key, fallback=0.0):
        """std::stod semantics: leading floating-point prefix."""
        if not self.has(section, key):
            return fallback
        mt = re.match(r"\s*[+-]?(inf(inity)?|nan|(\d+\.?\d*|\.\d+)([eE][+-]?\d+)?)",
                      self.get(section, key), re.IGNORECASE)
        if not mt:
            raise ValueError(f"stod: [{section}] {key}")
        return float(mt.group(0))

    def sections(self):
        return sorted(self.values)  # std::map order, as the reference iterates


@dataclass
class LayerRecord:
    """One conv layer of a checkpoint (train.hpp ConvLayer fields the manifest stores)."""

    name: str
    w: np.ndarray                      # K×C×p×q (winograd) or K×C×r×s (spatial)
    domain: str = "winograd"
    in_c: int = 0
    out_c: int = 0
    lmbda: float = 0.0
    norm: int = 1
    mask: np.ndarray | None = None     # 1 = pruned (frozen zero), train.cpp:331-337
    m: int = 2


@dataclass
class Checkpoint:
    in_c: int
    in_h: int
    in_w: int
    classes: int
    convs: list = field(default_factory=list)
    dense_w: np.ndarray | None = None
    dense_b: np.ndarray | None = None


def _g(v):
    """The reference prints with ostream defaults (%g, 6 digits, harness.cpp:166); that is
    kept whenever it round-trips, otherwise the shortest exact repr (the reference's stod reads
    both)."""
    s = "%g" % float(v)
    return s if float(s) == float(v) else repr(float(v))


def save_checkpoint(directory, ck: Checkpoint) -> None:
    """harness.cpp:152-186 layout + `m=` per Winograd layer."""
    d = Path(directory)
    os.makedirs(d, exist_ok=True)
    lines = ["[network]", f"in_c={ck.in_c}", f"in_h={ck.in_h}", f"in_w={ck.in_w}",
             f"classes={ck.classes}", f"convs={len(ck.convs)}"]
    for conv in ck.convs:
        write_wgt1(d / f"{conv.name}.wgt", conv.w)
        lines += [f"[{conv.name}]", f"domain={conv.domain}", f"file={conv.name}.wgt", f"in_c={conv.in_c}",
                  f"out_c={conv.out_c}", f"lambda={_g(conv.lmbda)}", f"norm={conv.norm}", f"m={conv.m}"]
        if conv.mask is not None and conv.mask.shape == conv.w.shape:
            write_wgt1(d / f"{conv.name}.mask.wgt", conv.mask)
            lines.append(f"mask={conv.name}.mask.wgt")
    if ck.dense_w is not None:
        write_wgt1(d / "dense.wgt", ck.dense_w)
        write_wgt1(d / "dense_bias.wgt", np.asarray(ck.dense_b))
        lines += ["[dense]", "file=dense.wgt", "bias=dense_bias.wgt"]
    try:
        (d / "manifest.cfg").write_text("\n".join(lines) + "\n")
    except OSError as e:
        raise IoError(f"cannot write manifest in {d}") from e


def load_checkpoint(directory) -> Checkpoint:
    """harness.cpp:188-212, with the tile size read from `m=` (default 2, the reference's)."""
    d = Path(directory)
    m = Config.parse_file(d / "manifest.cfg")
    ck = Checkpoint(m.get_int("network", "in_c"), m.get_int("network", "in_h"), m.get_int("network", "in_w"),
                    m.get_int("network", "classes"))
    for i in range(m.get_int("network", "convs")):
        name = f"conv{i + 1}"
        rec = LayerRecord(name=name, w=read_wgt1(d / m.get(name, "file")),
                          domain="winograd" if m.get(name, "domain") == "winograd" else "spatial",
                          in_c=m.get_int(name, "in_c"), out_c=m.get_int(name, "out_c"),
                          lmbda=m.get_double(name, "lambda"), norm=m.get_int(name, "norm", 1),
                          m=m.get_int(name, "m", 2))
        if m.has(name, "mask"):
            rec.mask = read_wgt1(d / m.get(name, "mask"))
        ck.convs.append(rec)
    if m.has("dense", "file"):
        ck.dense_w = read_wgt1(d / m.get("dense", "file"))
        ck.dense_b = read_wgt1(d / m.get("dense", "bias"))
    return ck
