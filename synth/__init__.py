"""Seeded synthetic inputs shared by the oracle side and the CUDA side of the tests/bench.

This module holds NO arithmetic of the method (no products, no sums of the LoRA
operands).  It only draws i.i.d. Gaussian tensors with the laws that
BASELINE.json gives for its configs and rounds them once to the dtype the GPU
consumes, so that the fp64 oracle and the CUDA path see exactly the same values
(SURVEY.md §8(d) "Synthetic inputs", reading #12/#13).

Generator: NumPy PCG64, ``np.random.default_rng([2312, cfg, sub, t])``,
``standard_normal`` in fp64, times the std, cast fp64 -> fp32 -> target dtype
(round-to-nearest-even at each step).  Large tensors are drawn in row chunks from
the same generator (sequential draws continue one stream, so a chunked draw is
identical to a single draw; tests/test_synth.py checks it).

Tensor ids ``t``: X=0, W=1, A=2, B=3, dY=4.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

T_X, T_W, T_A, T_B, T_DY = 0, 1, 2, 3, 4
_CHUNK_ELEMS = 1 << 24

_TORCH_DTYPE = {"f32": torch.float32, "bf16": torch.bfloat16}


@dataclass(frozen=True)
class Case:
    """One LoRA-linear problem: n tokens, k = in, m = out, rank r (paper: b·s, i, o, r)."""

    name: str
    cfg: int          # BASELINE.json configs index + 1 (C1..C5); 0 = ad-hoc test case
    sub: int          # sub-configuration index within the config (seed component)
    n: int
    k: int
    m: int
    r: int
    dtype: str        # "f32" | "bf16"
    std: dict = field(default_factory=dict)   # per tensor id

    @property
    def torch_dtype(self):
        return _TORCH_DTYPE[self.dtype]


def _law(k: int, r: int, x_std: float = 1.0) -> dict:
    """BASELINE.json init law: X, dY ~ N(0,1); W, A ~ N(0, 1/k); B ~ N(0, 1/r).

    For C1 the config states W and A scaled by 1/sqrt(256) (= 1/sqrt(k)) and B by
    1/sqrt(8) (= 1/sqrt(r)); for C2/C3-up it states Var 1/4096 (= 1/k).  C3-down and
    C4 give no law; reading R13 takes the same fan-in law.
    """
    return {T_X: x_std, T_W: 1.0 / math.sqrt(k), T_A: 1.0 / math.sqrt(k),
            T_B: 1.0 / math.sqrt(r), T_DY: 1.0}


def case(name, cfg, sub, n, k, m, r, dtype) -> Case:
    return Case(name, cfg, sub, n, k, m, r, dtype, _law(k, r))


# --- BASELINE.json configs -------------------------------------------------------
C1 = case("C1_fp32_256", 1, 0, 256, 256, 256, 8, "f32")
C2 = {r: case(f"C2_llama_attn_r{r}", 2, i, 8192, 4096, 4096, r, "bf16")
      for i, r in enumerate((8, 16, 64, 128))}
C3_UP = case("C3_llama_mlp_up", 3, 0, 8192, 4096, 11008, 16, "bf16")
C3_DOWN = case("C3_llama_mlp_down", 3, 1, 8192, 11008, 4096, 16, "bf16")
C4 = {(r, n): case(f"C4_opt_r{r}_n{n}", 4, 3 * ri + ni, n, 2048, 2048, r, "bf16")
      for ri, r in enumerate((8, 32, 128)) for ni, n in enumerate((4096, 32768, 131072))}

ALL_CONFIGS = [C1, *C2.values(), C3_UP, C3_DOWN, *C4.values()]

# --- C5: stack of LoRA-adapted linears with Llama-7B projection shapes -------------
# Per layer (reading R15): q, k, v, o: d -> d; gate, up: d -> f; down: f -> d.
C5_LINEARS = ("q", "k", "v", "o", "gate", "up", "down")
C5_D, C5_F, C5_R = 4096, 11008, 16


def c5_dims(name: str, d: int = C5_D, f: int = C5_F):
    """(in, out) of linear ``name`` in a layer of width d and MLP width f."""
    return {"gate": (d, f), "up": (d, f), "down": (f, d)}.get(name, (d, d))


def c5_linear(layer: int, name: str, n: int, d: int = C5_D, f: int = C5_F, r: int = C5_R, dtype: str = "bf16"):
    """The Case of one linear of the stack; seeds [2312, 5, layer*8 + index, t]."""
    k, m = c5_dims(name, d, f)
    return case(f"C5_L{layer}_{name}", 5, layer * 8 + C5_LINEARS.index(name), n, k, m, r, dtype)


def c5_weights(layers: int, n: int, d: int = C5_D, f: int = C5_F, r: int = C5_R, dtype: str = "bf16"):
    """[{name: {"W", "A", "B"}}] per layer (CPU tensors), same law as C2/C3 (Var 1/k, 1/r)."""
    out = []
    for layer in range(layers):
        lw = {}
        for name in C5_LINEARS:
            c = c5_linear(layer, name, n, d, f, r, dtype)
            lw[name] = {"W": draw(c, T_W, (c.k, c.m)), "A": draw(c, T_A, (c.k, c.r)), "B": draw(c, T_B, (c.r, c.m))}
        out.append(lw)
    return out


def c5_io(n: int, d: int = C5_D, dtype: str = "bf16"):
    """Stack input X [n, d] ~ N(0, 1) and the synthetic output gradient dY [n, d] ~ N(0, 1)."""
    c = case("C5_io", 5, 1000, n, d, d, 1, dtype)
    return draw(c, T_X, (n, d)), draw(c, T_DY, (n, d))


def draw(c: Case, t: int, shape) -> torch.Tensor:
    """Draw tensor ``t`` of case ``c``; returns a CPU torch tensor in c's dtype."""
    rng = np.random.default_rng([2312, c.cfg, c.sub, t])
    rows, cols = shape
    out = torch.empty(rows, cols, dtype=c.torch_dtype)
    std = c.std[t]
    step = max(1, _CHUNK_ELEMS // max(cols, 1))
    for r0 in range(0, rows, step):
        r1 = min(rows, r0 + step)
        z = rng.standard_normal((r1 - r0, cols))
        z *= std
        out[r0:r1] = torch.from_numpy(z).to(torch.float32).to(c.torch_dtype)
    return out


def operands(c: Case, zero=()):
    """All five operands of case ``c`` (X, W, A, B, dY) as CPU tensors in c's dtype.

    ``zero`` names operands to replace by exact zeros (special-case tests)."""
    shapes = {"X": (c.n, c.k), "W": (c.k, c.m), "A": (c.k, c.r), "B": (c.r, c.m), "dY": (c.n, c.m)}
    tid = {"X": T_X, "W": T_W, "A": T_A, "B": T_B, "dY": T_DY}
    out = {}
    for name, shp in shapes.items():
        if name in zero:
            out[name] = torch.zeros(shp, dtype=c.torch_dtype)
        else:
            out[name] = draw(c, tid[name], shp)
    return out


def sample_rows(n: int, P: int = 1, count: int = 512, seed_cfg: int = 0) -> np.ndarray:
    """Row indices used for sampled parity at large n (SURVEY §8(c) "Row sampling").

    Always includes rows 0 and n-1, every shard boundary p*n/P +- {0,1}, and rows on
    128-row tile edges (== 0, 127 mod 128) near the start and end; the rest are drawn
    without replacement from ``default_rng([2312, seed_cfg, 99])``."""
    must = {0, n - 1}
    for p in range(1, P):
        b = p * n // P
        must.update({b - 1, b, b + 1})
    for base in (0, 128, n - 256, n - 128):
        if 0 <= base < n:
            must.update({base, min(n - 1, base + 127)})
    must = {i for i in must if 0 <= i < n}
    rng = np.random.default_rng([2312, seed_cfg, 99])
    want = max(0, min(count, n) - len(must))
    pool = np.setdiff1d(np.arange(n), np.fromiter(must, dtype=np.int64))
    extra = rng.choice(pool, size=min(want, pool.size), replace=False) if want else []
    return np.sort(np.concatenate([np.fromiter(must, dtype=np.int64), np.asarray(extra, dtype=np.int64)]))
