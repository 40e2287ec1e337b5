"""Seeded synthetic input generators shared by the tests, the bench and the
oracle-side checks.

This module holds NO arithmetic of the method (no packing, no tables, no
quantization, no GEMM): it only draws random numbers with numpy's PCG64 and
describes the workload shapes of BASELINE.json.  It is the one module both the
CUDA path's tests and the oracle's tests use.

Recipe: config c uses seed base 1000*c; weights are iid
ternary (config 2: P(-1)=P(+1)=0.3, P(0)=0.4; otherwise uniform), activations
are N(0,1) fp32 drawn as [N][K] (feature-major, as a framework holds them) and
returned token-contiguous [K][N].  The per-token int8 quantization
of those activations is method arithmetic and lives in the oracle (CPU) and in
the quantize kernel (GPU), not here.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

W_SCALE = 0.02  # per-tensor weight scale (BASELINE.json config 1; reading c7)


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def ternary_weights(M: int, K: int, seed: int, p_zero: float | None = None) -> np.ndarray:
    """int8 [M][K] with entries in {-1,0,+1}.  p_zero=None -> uniform thirds;
    otherwise P(0)=p_zero and P(-1)=P(+1)=(1-p_zero)/2."""
    r = rng(seed)
    if p_zero is None:
        return r.integers(-1, 2, size=(M, K), dtype=np.int8)
    p = (1.0 - p_zero) / 2.0
    return r.choice(np.array([-1, 0, 1], dtype=np.int8), size=(M, K),
                    p=[p, p_zero, p])


def activations_f32(K: int, N: int, seed: int) -> np.ndarray:
    """fp32 N(0,1) activations, drawn [N][K], returned token-contiguous [K][N]."""
    x = rng(seed).standard_normal((N, K), dtype=np.float32)
    return np.ascontiguousarray(x.T)


def int8_activations(K: int, N: int, seed: int, lo: int = -128, hi: int = 127) -> np.ndarray:
    """Uniform int8 [K][N] over [lo, hi] (full range incl. -128 by default):
    exercises the kernel's accumulation bounds harder than quantized data."""
    return rng(seed).integers(lo, hi + 1, size=(K, N), dtype=np.int16).astype(np.int8)


def token_scales(N: int, seed: int) -> np.ndarray:
    """Positive fp32 per-token scales (for GEMM tests that skip quantization)."""
    return (rng(seed).random(N, dtype=np.float32) * 0.05 + 1e-3).astype(np.float32)


# ----------------------------------------------------------------- configs
@dataclass
class Linear:
    name: str
    M: int  # out features
    K: int  # in features


@dataclass
class Config:
    idx: int
    name: str
    linears: List[Linear]
    N: List[int]
    g: List[int]
    p_zero: float | None = None
    layers: int = 1
    notes: str = ""
    seed_base: int = field(init=False)

    def __post_init__(self):
        self.seed_base = 1000 * self.idx


CONFIGS = {
    1: Config(1, "single ternary mpGeMM 256x512", [Linear("W", 256, 512)], [8], [4]),
    2: Config(2, "BitNet-2B FFN-up", [Linear("ffn_up", 6912, 2560)], [256], [4],
              p_zero=0.4),
    3: Config(3, "Llama3-8B-shaped layer (5 linears)",
              [Linear("qkv", 6144, 4096), Linear("o", 4096, 4096),
               Linear("gate", 14336, 4096), Linear("up", 14336, 4096),
               Linear("down", 4096, 14336)], [1024], [4]),
    4: Config(4, "Falcon3-10B-shaped FFN-down", [Linear("down", 3072, 23040)],
              [1, 16, 64, 256, 1024, 4096], [4, 5]),
    5: Config(5, "30-layer BitNet-2B-shaped prefill (linears only)",
              [Linear("qkv", 3840, 2560), Linear("o", 2560, 2560),
               Linear("gate", 6912, 2560), Linear("up", 6912, 2560),
               Linear("down", 2560, 6912)], [2048], [4], layers=30),
}


def weight_seed(cfg: Config, layer: int, j: int) -> int:
    if cfg.idx == 5:
        return 5000 + 10 * layer + j
    return cfg.seed_base + j


def act_seed(cfg: Config, N: int, j: int = 0) -> int:
    if cfg.idx == 5:
        return 5999
    if cfg.idx == 4:
        return 4000 + N
    return cfg.seed_base + 100 + j


def config_weights(cfg: Config, layer: int = 0) -> List[Tuple[Linear, np.ndarray]]:
    return [(lin, ternary_weights(lin.M, lin.K, weight_seed(cfg, layer, j), cfg.p_zero))
            for j, lin in enumerate(cfg.linears)]
