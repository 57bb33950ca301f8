"""Seeded input generators (recipe = DESIGN.md "Input recipe", reading c12).

* Downward factor  B [k x n] ~ N(0, 1/n)   (so B x has unit-scale entries)
* Upward factor    A [m x k] ~ N(0, 1/k)
* RMSNorm gain     gamma ~ 1 + U(-0.1, 0.1) (so a dropped gain is visible)
* Activations x ~ N(0, 1); cached K/V ~ N(0, 1); token ids ~ U[0, V)
* Seeds: 20260417 + config_id, mixed with (layer, matrix name) by a fixed
  string hash so TP=1 and TP=P ranks see identical full matrices.

Model shapes: LLaMA-3-8B / -70B (Table 1 footnote gives the 70B dims;
the 8B dims are the public LLaMA-3 architecture, reading c9).  Ranks: the
paper's explicit 70B@40% ranks 4916/614, otherwise
round-half-up((1 - rho) * min(m, n)) (readings c1, c2).
"""
from __future__ import annotations

import dataclasses
import zlib

import torch

__all__ = ["ModelShape", "LLAMA3_8B", "LLAMA3_70B", "LLAMA2_7B", "OPT_6_7B", "rank_for", "block_ranks",
           "seed_for", "gen_factor_pair", "gen_block_weights", "gen_normal",
           "MATRICES", "matrix_dims"]

BASE_SEED = 20260417


@dataclasses.dataclass(frozen=True)
class ModelShape:
    name: str
    h: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    m: int          # MLP intermediate
    n_layers: int
    vocab: int
    rope_theta: float = 500000.0
    rms_eps: float = 1e-5
    glu: bool = True       # SiLU-GLU MLP (LLaMA); False = ReLU on up alone (OPT)
    rope: bool = True      # rotary position embedding on q, k

    @property
    def h_kv(self) -> int:
        return self.n_kv_heads * self.head_dim

    @property
    def matrices(self):
        return MATRICES if self.glu else tuple(nm for nm in MATRICES if nm != "gate")


LLAMA3_8B = ModelShape("llama3-8b", 4096, 32, 8, 128, 14336, 32, 128256)
LLAMA3_70B = ModelShape("llama3-70b", 8192, 64, 8, 128, 28672, 80, 128256)
# Table 2 families at their published layer shapes; OPT modelled as
# its MLP (non-GLU ReLU) and position handling (no RoPE) -- reading c16.
LLAMA2_7B = ModelShape("llama2-7b", 4096, 32, 32, 128, 11008, 32, 32000, rope_theta=10000.0)
OPT_6_7B = ModelShape("opt-6.7b", 4096, 32, 32, 128, 16384, 32, 50272, glu=False, rope=False)

MATRICES = ("q", "k", "v", "o", "gate", "up", "down")


def matrix_dims(s: ModelShape, name: str):
    """(m_out, n_in) of each weight in the math convention W in R^{m x n}."""
    return {"q": (s.h, s.h), "k": (s.h_kv, s.h), "v": (s.h_kv, s.h), "o": (s.h, s.h),
            "gate": (s.m, s.h), "up": (s.m, s.h), "down": (s.h, s.m)}[name]


def rank_for(ratio: float, m: int, n: int) -> int:
    """Rank retained at compression ratio rho (rank ratio, P:205 footnote)."""
    if not (0.0 <= ratio < 1.0):
        raise ValueError("compression ratio must be in [0, 1)")
    mn = min(m, n)
    if abs(ratio - 0.4) < 1e-12 and mn in (8192, 1024):
        return {8192: 4916, 1024: 614}[mn]          # printed ranks
    return max(1, int((1.0 - ratio) * mn + 0.5))      # round half up (c2)


def block_ranks(s: ModelShape, ratio: float) -> dict:
    """Retained rank per matrix; a non-GLU shape has no gate (rank 0)."""
    r = {nm: rank_for(ratio, *matrix_dims(s, nm)) for nm in s.matrices}
    r.setdefault("gate", 0)
    return r


def seed_for(config_id: int, layer: int, name: str) -> int:
    return (BASE_SEED + config_id + 1_000_003 * layer + zlib.crc32(name.encode())) % (2**62)


def gen_normal(shape, std: float, seed: int, device="cpu", dtype=torch.float32) -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    t = torch.randn(shape, generator=g, device=device, dtype=torch.float32 if dtype == torch.float64 else dtype)
    if std != 1.0:
        t.mul_(std)
    return t.to(dtype)


def gen_factor_pair(m: int, n: int, k: int, seed: int, device="cpu", dtype=torch.bfloat16):
    """(A [m x k] ~ N(0,1/k), B [k x n] ~ N(0,1/n)) rounded to `dtype`."""
    A = gen_normal((m, k), k ** -0.5, seed * 2 + 1, device, dtype)
    B = gen_normal((k, n), n ** -0.5, seed * 2 + 2, device, dtype)
    return A, B


def gen_block_weights(s: ModelShape, ranks: dict, config_id: int, layer: int,
                      device="cpu", dtype=torch.bfloat16) -> dict:
    """Per-matrix factors A_<name>, B_<name> plus the two RMSNorm gains."""
    w = {}
    for nm in s.matrices:
        mo, ni = matrix_dims(s, nm)
        A, B = gen_factor_pair(mo, ni, ranks[nm], seed_for(config_id, layer, nm), device, dtype)
        w["A_" + nm] = A
        w["B_" + nm] = B
    for nm in ("g_attn", "g_mlp"):
        g = torch.Generator(device=device)
        g.manual_seed(seed_for(config_id, layer, nm))
        u = torch.rand((s.h,), generator=g, device=device, dtype=torch.float32)
        w[nm] = (1.0 + 0.2 * (u - 0.5)).to(dtype)
    return w
