"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no outer products, no sums over
workers, no scheme choice, no sharding). It only:
  * draws seeded random arrays (numpy PCG64, one stream per (config, layer, rank)),
  * rounds them to the device dtype on the host (bf16 round-to-nearest-even on the
    fp32 bit pattern), so the GPU receives the identical bits the oracle widens to
    fp64,
  * describes the workload shapes (synth_inputs/shapes.json, dumped from torchvision
    architectures on the `meta` device by scripts/dump_shapes.py).

Input recipes (DESIGN.md §"Inputs"):
  exact regime   u ∈ {-4..4}, v ∈ {0..4} (integers), W = j/256 with j ∈ [-128,127],
                 alpha = -2^-12, dense grads g ∈ {-64..64}.  Every bf16 product is exact
                 in fp32 and every partial sum stays below 2^24, so any summation order
                 gives the same fp32 result.
  stat regime    u = 2^-5·N(0,1), v = max(0, N(0,1)) (ReLU activations),
                 W ~ U(-1/sqrt(N), 1/sqrt(N)), dense grads 2^-5·N(0,1);
                 rounded to the device dtype at generation.
Seed = 1000*base + 10*layer + rank.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

__all__ = [
    "seed_of", "rng", "bf16_round", "bf16_bits_to_f32", "to_device_dtype",
    "exact_factors", "exact_weights", "exact_dense_grad", "EXACT_ALPHA",
    "stat_factors", "stat_weights", "stat_dense_grad",
    "load_model", "Layer", "MODELS",
]

EXACT_ALPHA = -(2.0 ** -12)

_HERE = os.path.dirname(os.path.abspath(__file__))


def seed_of(base: int, layer: int, rank: int) -> int:
    return 1000 * base + 10 * layer + rank


def rng(base: int, layer: int = 0, rank: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed_of(base, layer, rank)))


# ---------------------------------------------------------------------------
# dtype rounding (host side, bit exact)
# ---------------------------------------------------------------------------

def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit patterns (uint16), round-to-nearest-even. Finite inputs only."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return b.astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def to_device_dtype(x: np.ndarray, dtype: str) -> np.ndarray:
    """Return fp32 values that are exactly representable in `dtype` ('bf16' | 'f32' | 'tf32').

    'tf32' inputs stay fp32: the tensor core rounds them (mode unpinned).
    """
    x = np.asarray(x, dtype=np.float32)
    if dtype == "bf16":
        return bf16_bits_to_f32(bf16_round(x)).reshape(x.shape)
    if dtype in ("f32", "tf32"):
        return x.copy()
    raise ValueError(dtype)


# ---------------------------------------------------------------------------
# exact regime
# ---------------------------------------------------------------------------

def exact_factors(g: np.random.Generator, K: int, M: int, N: int):
    """u: [K][M] in {-4..4}, v: [K][N] in {0..4}, as float32 (exact in bf16)."""
    u = g.integers(-4, 5, size=(K, M)).astype(np.float32)
    v = g.integers(0, 5, size=(K, N)).astype(np.float32)
    return u, v


def exact_weights(g: np.random.Generator, *shape: int) -> np.ndarray:
    return (g.integers(-128, 128, size=shape).astype(np.float32) / np.float32(256.0))


def exact_dense_grad(g: np.random.Generator, n: int) -> np.ndarray:
    return g.integers(-64, 65, size=n).astype(np.float32)


# ---------------------------------------------------------------------------
# statistical regime
# ---------------------------------------------------------------------------

def stat_factors(g: np.random.Generator, K: int, M: int, N: int, dtype: str = "bf16"):
    u = (g.standard_normal((K, M), dtype=np.float32) * np.float32(2.0 ** -5))
    v = np.maximum(g.standard_normal((K, N), dtype=np.float32), np.float32(0.0))
    return to_device_dtype(u, dtype), to_device_dtype(v, dtype)


def stat_weights(g: np.random.Generator, M: int, N: int) -> np.ndarray:
    a = np.float32(1.0 / np.sqrt(N))
    return g.uniform(-a, a, size=(M, N)).astype(np.float32)


def stat_dense_grad(g: np.random.Generator, n: int) -> np.ndarray:
    return g.standard_normal(n, dtype=np.float32) * np.float32(2.0 ** -5)


# ---------------------------------------------------------------------------
# workload shapes
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Layer:
    name: str
    kind: str          # "fc" | "dense"
    M: int = 0         # fc: out_features
    N: int = 0         # fc: in_features
    bias: bool = False
    n: int = 0         # dense: parameter count (weights + bias flattened)

    @property
    def params(self) -> int:
        if self.kind == "fc":
            return self.M * self.N + (self.M if self.bias else 0)
        return self.n


@dataclass(frozen=True)
class Model:
    name: str
    total_params: int
    layers: tuple      # forward order l = 1..L


def _load_all():
    with open(os.path.join(_HERE, "shapes.json")) as f:
        raw = json.load(f)
    out = {}
    for k, v in raw.items():
        ls = tuple(Layer(**l) for l in v["layers"])
        out[k] = Model(k, v["total_params"], ls)
    return out


MODELS = _load_all()

# BASELINE.json configs -> (model, per-GPU batch K)
CONFIGS = {
    "c0": None,  # single FC M=N=64, K=8, P=2 simulated (tests only)
    "c1": ("alexnet", 128),
    "c2": ("vgg19", 32),
    "c3": ("vgg19_22k", 32),
    "c4": ("inception_v3", 32),
}


def load_model(name: str) -> Model:
    return MODELS[name]
