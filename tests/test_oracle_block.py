"""Pins for the oracle's block pieces and census (-m "not gpu").

Independent references used here: torch (float64) library routines --
F.rms_norm, F.scaled_dot_product_attention, complex-multiplication RoPE
(torch.polar) -- closed forms, and Table 1's printed integers.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from conftest import golden


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ---- RMSNorm -------------------------------------------------------------------
def test_rmsnorm_closed_form(orc):
    x = np.full((2, 8), 3.0)
    y = orc.rmsnorm(x, np.ones(8), 1e-5)
    assert np.abs(y - 3.0 / math.sqrt(9.0 + 1e-5)).max() < 1e-15


def test_rmsnorm_vs_torch(orc):
    r = np.random.default_rng(0)
    x, g = r.standard_normal((5, 16)), 1 + 0.1 * r.standard_normal(16)
    ref = F.rms_norm(torch.tensor(x), (16,), torch.tensor(g), eps=1e-5).numpy()
    assert rel(orc.rmsnorm(x, g, 1e-5), ref) < 1e-14


# ---- RoPE -----------------------------------------------------
def test_rope_position_zero_identity(orc):
    v = np.random.default_rng(1).standard_normal((3, 2, 8))
    np.testing.assert_array_equal(orc.rope(v, [0, 0, 0], 10000.0), v)


def test_rope_closed_form_first_pair(orc):
    for p in (1, 5, 37):
        out = orc.rope(np.array([[[1.0, 0.0]]]), [p], 10000.0)
        np.testing.assert_allclose(out[0, 0], [math.cos(p), math.sin(p)], atol=1e-15)


def test_rope_vs_complex_polar(orc):
    """Meta-LLaMA formulation: pairs as complex numbers times exp(i pos theta^(-2i/d))."""
    r = np.random.default_rng(2)
    T, nh, d, theta = 6, 3, 16, 500000.0
    v = r.standard_normal((T, nh, d))
    pos = np.array([0, 1, 2, 100, 511, 2047])
    freqs = 1.0 / theta ** (torch.arange(0, d, 2, dtype=torch.float64) / d)
    ang = torch.outer(torch.tensor(pos, dtype=torch.float64), freqs)
    rot = torch.polar(torch.ones_like(ang), ang)
    vc = torch.view_as_complex(torch.tensor(v).reshape(T, nh, d // 2, 2))
    ref = torch.view_as_real(vc * rot[:, None, :]).reshape(T, nh, d).numpy()
    out = orc.rope(v, pos, theta)
    assert rel(out, ref) < 1e-13
    np.testing.assert_allclose(np.linalg.norm(out, axis=-1), np.linalg.norm(v, axis=-1), rtol=1e-12)


def test_rope_relative_position(orc):
    """<rope(q,p1), rope(k,p2)> depends only on p1 - p2."""
    r = np.random.default_rng(3)
    q, k = r.standard_normal((1, 1, 8)), r.standard_normal((1, 1, 8))
    dots = [float(np.sum(orc.rope(q, [p + 7], 10.0) * orc.rope(k, [p], 10.0))) for p in (0, 3, 50)]
    assert max(dots) - min(dots) < 1e-12


# ---- attention ---------------------------------------------------------
def test_attention_single_token_returns_v(orc):
    r = np.random.default_rng(4)
    q, k, v = r.standard_normal((1, 8)), r.standard_normal((1, 4)), r.standard_normal((1, 4))
    out = orc.attention(q, k, v, [0, 1], H=2, Hkv=1, d=4)
    np.testing.assert_allclose(out, np.concatenate([v, v], 1), atol=1e-15)


def test_attention_equal_keys_causal_prefix_mean(orc):
    """All keys equal -> uniform softmax over the visible prefix -> running mean of v."""
    r = np.random.default_rng(5)
    T, d = 6, 4
    q = r.standard_normal((T, d))
    k = np.tile(r.standard_normal((1, d)), (T, 1))
    v = r.standard_normal((T, d))
    out = orc.attention(q, k, v, [0, T], H=1, Hkv=1, d=d)
    ref = np.cumsum(v, 0) / np.arange(1, T + 1)[:, None]
    assert np.abs(out - ref).max() < 1e-14


def test_attention_gqa_mapping(orc):
    """H=4, Hkv=2: heads 0,1 read kv head 0; heads 2,3 read kv head 1."""
    T, d = 3, 2
    q = np.zeros((T, 4 * d))
    k = np.zeros((T, 2 * d))
    v = np.zeros((T, 2 * d))
    v[:, :d] = 1.0
    v[:, d:] = 2.0
    out = orc.attention(q, k, v, [0, T], H=4, Hkv=2, d=d).reshape(T, 4, d)
    np.testing.assert_array_equal(out[:, :2], 1.0)
    np.testing.assert_array_equal(out[:, 2:], 2.0)


@pytest.mark.parametrize("H,Hkv", [(4, 4), (4, 2), (8, 1)])
def test_attention_vs_torch_sdpa(orc, H, Hkv):
    r = np.random.default_rng(H * 10 + Hkv)
    d, lens = 8, [5, 1, 7]
    cu = np.concatenate([[0], np.cumsum(lens)])
    T = cu[-1]
    q, k, v = r.standard_normal((T, H * d)), r.standard_normal((T, Hkv * d)), r.standard_normal((T, Hkv * d))
    out = orc.attention(q, k, v, cu, H, Hkv, d)
    for s in range(len(lens)):
        a, b = cu[s], cu[s + 1]
        tq = torch.tensor(q[a:b]).reshape(b - a, H, d).transpose(0, 1)
        tk = torch.tensor(k[a:b]).reshape(b - a, Hkv, d).transpose(0, 1).repeat_interleave(H // Hkv, 0)
        tv = torch.tensor(v[a:b]).reshape(b - a, Hkv, d).transpose(0, 1).repeat_interleave(H // Hkv, 0)
        ref = F.scaled_dot_product_attention(tq, tk, tv, is_causal=True).transpose(0, 1).reshape(b - a, H * d)
        assert rel(out[a:b], ref.numpy()) < 1e-13


# ---- whole block -----------------------------------------------------------------
SMALL = dict(h=32, n_heads=4, n_kv_heads=2, head_dim=8, m=48)


def _dense_block_torch(x, W, g1, g2, pos, cu, H, Hkv, d, theta, eps, glu=True, use_rope=True):
    """Independent dense block in torch float64 (used only in the lossless-rank pins).

    Default = LLaMA (SiLU-GLU MLP, RoPE); glu=False = OPT-style ReLU MLP,
    use_rope=False = no rotary embedding (Table 2 variants)."""
    x = torch.tensor(x)
    T, h = x.shape
    a = F.rms_norm(x, (h,), torch.tensor(g1), eps=eps)
    q, k, v = a @ torch.tensor(W["q"]).T, a @ torch.tensor(W["k"]).T, a @ torch.tensor(W["v"]).T
    freqs = 1.0 / theta ** (torch.arange(0, d, 2, dtype=torch.float64) / d)
    rot = torch.polar(torch.ones(T, d // 2, dtype=torch.float64), torch.outer(torch.tensor(pos, dtype=torch.float64), freqs))

    def rope(t, nh):
        c = torch.view_as_complex(t.reshape(T, nh, d // 2, 2).contiguous())
        return torch.view_as_real(c * rot[:, None]).reshape(T, nh * d)
    if use_rope:
        q, k = rope(q, H), rope(k, Hkv)
    att = torch.zeros(T, H * d, dtype=torch.float64)
    for s in range(len(cu) - 1):
        lo, hi = cu[s], cu[s + 1]
        tq = q[lo:hi].reshape(-1, H, d).transpose(0, 1)
        tk = k[lo:hi].reshape(-1, Hkv, d).transpose(0, 1).repeat_interleave(H // Hkv, 0)
        tv = v[lo:hi].reshape(-1, Hkv, d).transpose(0, 1).repeat_interleave(H // Hkv, 0)
        att[lo:hi] = F.scaled_dot_product_attention(tq, tk, tv, is_causal=True).transpose(0, 1).reshape(-1, H * d)
    x = x + att @ torch.tensor(W["o"]).T
    b = F.rms_norm(x, (h,), torch.tensor(g2), eps=eps)
    if glu:
        y = F.silu(b @ torch.tensor(W["gate"]).T) * (b @ torch.tensor(W["up"]).T)
    else:
        y = F.relu(b @ torch.tensor(W["up"]).T)
    return (x + y @ torch.tensor(W["down"]).T).numpy()


def _small_block(orc, lossless, seed=0, n_kv_heads=None, glu=True, use_rope=True, layout=0):
    r = np.random.default_rng(seed)
    s = dict(SMALL)
    if n_kv_heads is not None:
        s["n_kv_heads"] = n_kv_heads
    h, hkv, m = s["h"], s["n_kv_heads"] * s["head_dim"], s["m"]
    dims = {"q": (h, h), "k": (hkv, h), "v": (hkv, h), "o": (h, h), "gate": (m, h), "up": (m, h), "down": (h, m)}
    if not glu:
        del dims["gate"]
    ranks = {nm: (min(mn) if lossless else max(1, int(0.6 * min(mn) + 0.5))) for nm, mn in dims.items()}
    W, w = {}, {}
    for nm, (mo, ni) in dims.items():
        W[nm] = r.standard_normal((mo, ni)) / math.sqrt(ni)
        U, sg, Vt = np.linalg.svd(W[nm], full_matrices=False)
        kk = ranks[nm]
        w["A_" + nm] = U[:, :kk] * np.sqrt(sg[:kk])
        w["B_" + nm] = np.sqrt(sg[:kk])[:, None] * Vt[:kk]
    w["g_attn"] = 1 + 0.1 * r.standard_normal(h)
    w["g_mlp"] = 1 + 0.1 * r.standard_normal(h)
    cfg = orc.BlockCfg(h, s["n_heads"], s["n_kv_heads"], s["head_dim"], m, ranks["q"], ranks["k"], ranks["v"],
                       ranks["o"], ranks.get("gate", 0), ranks["up"], ranks["down"], rope_theta=10000.0,
                       rms_eps=1e-5, mlp_glu=int(glu), use_rope=int(use_rope), layout=layout)
    return cfg, w, W


def test_block_lossless_equals_dense(orc):
    """North-star self-check (3) at block level: full ranks -> dense block."""
    cfg, w, W = _small_block(orc, lossless=True)
    r = np.random.default_rng(9)
    cu = [0, 5, 6, 13]
    T = cu[-1]
    pos = np.concatenate([np.arange(5), np.arange(1), np.arange(7)])
    x = r.standard_normal((T, cfg.h))
    out, _, _ = orc.block_prefill(cfg, w, x, pos, cu)
    ref = _dense_block_torch(x, W, w["g_attn"], w["g_mlp"], pos, cu, cfg.n_heads, cfg.n_kv_heads,
                             cfg.head_dim, cfg.rope_theta, cfg.rms_eps)
    assert rel(out, ref) < 1e-12


VARIANTS = [  # (n_kv_heads, glu, use_rope): Table 2 model families
    (4, True, True),     # MHA (LLaMA-2-7B-like)
    (1, True, True),     # MQA
    (4, False, False),   # OPT-like: MHA, ReLU MLP, no RoPE
    (2, False, True),    # GQA + ReLU
    (2, True, False),    # GQA without RoPE
]


@pytest.mark.parametrize("hkv,glu,use_rope", VARIANTS)
def test_block_variant_lossless_equals_dense(orc, hkv, glu, use_rope):
    """Same lossless pin for the attention / MLP / RoPE variants of the N4 row."""
    cfg, w, W = _small_block(orc, lossless=True, seed=11, n_kv_heads=hkv, glu=glu, use_rope=use_rope)
    r = np.random.default_rng(12)
    cu = [0, 4, 11]
    T = cu[-1]
    pos = np.concatenate([np.arange(4), np.arange(7)])
    x = r.standard_normal((T, cfg.h))
    out, _, _ = orc.block_prefill(cfg, w, x, pos, cu)
    ref = _dense_block_torch(x, W, w["g_attn"], w["g_mlp"], pos, cu, cfg.n_heads, cfg.n_kv_heads,
                             cfg.head_dim, cfg.rope_theta, cfg.rms_eps, glu=glu, use_rope=use_rope)
    assert rel(out, ref) < 1e-12


def test_no_rope_is_position_free(orc):
    """use_rope=0: a single-sequence prefill does not depend on the position ids."""
    cfg, w, _ = _small_block(orc, lossless=False, seed=13, use_rope=False)
    x = np.random.default_rng(14).standard_normal((5, cfg.h))
    o1, k1, _ = orc.block_prefill(cfg, w, x, np.arange(5), [0, 5])
    o2, k2, _ = orc.block_prefill(cfg, w, x, np.arange(5) + 100, [0, 5])
    np.testing.assert_array_equal(o1, o2)
    np.testing.assert_array_equal(k1, k2)


def test_block_params_non_glu(orc):
    """Non-GLU MLP carries no gate factors ((m+n)k per factor pair): the oracle's
    count equals the number of elements actually stored in the block's factor tensors
    (counted from the tensors, not from a formula), and dropping the gate removes exactly
    the gate pair's elements."""
    cfg, w, _ = _small_block(orc, lossless=False, seed=15, glu=False)
    stored = sum(v.size for k, v in w.items() if k.startswith(("A_", "B_")))
    assert "A_gate" not in w and orc.block_params(cfg) == stored
    cfg_g, w_g, _ = _small_block(orc, lossless=False, seed=15, glu=True)
    gate = w_g["A_gate"].size + w_g["B_gate"].size
    assert orc.block_params(cfg_g) == sum(v.size for k, v in w_g.items() if k.startswith(("A_", "B_")))
    assert orc.block_params(cfg_g) - orc.block_params(cfg) == gate


@pytest.mark.parametrize("hkv,glu,use_rope", VARIANTS)
def test_variant_decode_equals_recompute(orc, hkv, glu, use_rope):
    cfg, w, _ = _small_block(orc, lossless=False, seed=16, n_kv_heads=hkv, glu=glu, use_rope=use_rope)
    r = np.random.default_rng(17)
    lens = [3, 6]
    hk = cfg.n_kv_heads * cfg.head_dim
    ck, cv = np.zeros((2, 8, hk)), np.zeros((2, 8, hk))
    xs, ref = [], []
    for b, L in enumerate(lens):
        x = r.standard_normal((L + 1, cfg.h))
        out, kk, vv = orc.block_prefill(cfg, w, x, np.arange(L + 1), [0, L + 1])
        ck[b, :L], cv[b, :L] = kk[:L], vv[:L]
        xs.append(x[L])
        ref.append(out[L])
    o, _, _ = orc.block_decode(cfg, w, np.stack(xs), ck, cv, lens)
    assert rel(o, np.stack(ref)) < 1e-12


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("glu", [True, False])
def test_block_deinfer_layout_p_invariance(orc, world, glu):
    """N1 (Fig. 3): the DeInfer rearrangement -- concat-split B with a
    latent all-gather, row-sharded A, input-sharded B + latent reduce-sum with a
    replicated A -- equals the unsharded block at every world size (uneven
    splits included: ranks 0.6*min(m,n) are odd, m=48 / h=32 split 3 ways)."""
    cfg, w, _ = _small_block(orc, lossless=False, seed=21, glu=glu, layout=orc.LAYOUT_DEINFER)
    r = np.random.default_rng(22)
    x = r.standard_normal((7, cfg.h))
    cu = [0, 3, 7]
    pos = np.array([0, 1, 2, 0, 1, 2, 3])
    o1, k1, v1 = orc.block_prefill(cfg, w, x, pos, cu)
    op, kp, vp = orc.block_prefill(cfg, w, x, pos, cu, world=world)
    assert rel(op, o1) < 1e-12 and rel(kp, k1) < 1e-12 and rel(vp, v1) < 1e-12
    part, _, _ = orc.block_prefill(cfg, w, x, pos, cu, rows=[6, 2], world=world)
    assert rel(part, o1[[6, 2]]) < 1e-12


def test_block_deinfer_lossless_equals_dense(orc):
    cfg, w, W = _small_block(orc, lossless=True, seed=23, layout=orc.LAYOUT_DEINFER)
    r = np.random.default_rng(24)
    x = r.standard_normal((6, cfg.h))
    pos = np.arange(6)
    out, _, _ = orc.block_prefill(cfg, w, x, pos, [0, 6], world=4)
    ref = _dense_block_torch(x, W, w["g_attn"], w["g_mlp"], pos, [0, 6], cfg.n_heads, cfg.n_kv_heads,
                             cfg.head_dim, cfg.rope_theta, cfg.rms_eps)
    assert rel(out, ref) < 1e-12


def test_deinfer_decode_p_invariance(orc):
    cfg, w, _ = _small_block(orc, lossless=False, seed=25, layout=orc.LAYOUT_DEINFER)
    r = np.random.default_rng(26)
    hk = cfg.n_kv_heads * cfg.head_dim
    ck, cv = r.standard_normal((3, 6, hk)), r.standard_normal((3, 6, hk))
    x = r.standard_normal((3, cfg.h))
    o1, k1, _ = orc.block_decode(cfg, w, x, ck, cv, [0, 2, 5])
    o2, k2, _ = orc.block_decode(cfg, w, x, ck, cv, [0, 2, 5], world=2)
    assert rel(o2, o1) < 1e-12 and rel(k2, k1) < 1e-12


@pytest.mark.parametrize("world,align", [(2, 1), (4, 1), (4, 8), (8, 1)])
def test_block_p_invariance(orc, world, align):
    """North-star self-check (4) at block level: rank-sharded block == TP=1 block."""
    cfg, w, _ = _small_block(orc, lossless=False, seed=1)
    r = np.random.default_rng(2)
    x = r.standard_normal((6, cfg.h))
    pos = np.arange(6)
    o1, k1, v1 = orc.block_prefill(cfg, w, x, pos, [0, 6])
    op, kp, vp = orc.block_prefill(cfg, w, x, pos, [0, 6], world=world, align=align)
    assert rel(op, o1) < 1e-12 and rel(kp, k1) < 1e-12 and rel(vp, v1) < 1e-12


def test_block_sampled_rows_equal_full(orc):
    cfg, w, _ = _small_block(orc, lossless=False, seed=3)
    x = np.random.default_rng(4).standard_normal((9, cfg.h))
    pos = np.arange(9)
    full, _, _ = orc.block_prefill(cfg, w, x, pos, [0, 9])
    rows = [8, 0, 4]
    part, _, _ = orc.block_prefill(cfg, w, x, pos, [0, 9], rows=rows)
    np.testing.assert_array_equal(part, full[rows])


def test_decode_with_cache_equals_recompute(orc):
    """decoding token t with the cache of tokens < t == prefill row t."""
    cfg, w, _ = _small_block(orc, lossless=False, seed=5)
    r = np.random.default_rng(6)
    lens = [4, 1, 7]
    hkv = cfg.n_kv_heads * cfg.head_dim
    max_seq = 8
    xs, ck, cv, ref_out, ref_k = [], np.zeros((3, max_seq, hkv)), np.zeros((3, max_seq, hkv)), [], []
    for b, L in enumerate(lens):
        x = r.standard_normal((L + 1, cfg.h))
        out, kk, vv = orc.block_prefill(cfg, w, x, np.arange(L + 1), [0, L + 1])
        ck[b, :L], cv[b, :L] = kk[:L], vv[:L]
        xs.append(x[L])
        ref_out.append(out[L])
        ref_k.append(kk[L])
    o, kn, vn = orc.block_decode(cfg, w, np.stack(xs), ck, cv, lens)
    assert rel(o, np.stack(ref_out)) < 1e-12
    assert rel(kn, np.stack(ref_k)) < 1e-12


# ---- census, Table 1 ------------------------------------------------------
def test_census_table1(orc):
    g = golden("table1_census.json")
    c = orc.census(**g["inputs"])
    for key, val in g["expected"].items():
        assert c[key] == val, key
    assert round(100 * (1 - c["deinfer_block_printed"] / c["unopt_block"])) == g["printed_saving_percent"]


def test_census_build_collectives(orc):
    """This build's collective volume (165,888 ring units, 5 collectives),
    and bench.py's own census (which reports it without importing oracle/) agrees."""
    g = golden("build_census.json")
    c = orc.census(**g["inputs"])
    for key, val in g["expected"].items():
        assert c[key] == val, key
    import argparse
    import bench
    from synthetic import LLAMA3_70B, block_ranks
    args = argparse.Namespace(layout="rp", batch=1)
    bc = bench.collective_census(LLAMA3_70B, block_ranks(LLAMA3_70B, 0.4), 1, 8, args)
    assert bc["units_per_token_layer_nvls"] == g["nvls_units_per_token"]
    assert bc["units_per_token_layer_ring"] == c["build_block"]
    assert bc["collectives_per_layer"] == c["build_collectives"]


# ---- low-rank KV cache (N3: P:111) ---------------------------------------
def test_lowrank_kv_decode_equals_prefill(orc):
    """Decoding token L with the LATENT cache z_k = B_k a_j, z_v = B_v a_j of tokens j < L
    (reconstructed K = RoPE(A_k z_k), V = A_v z_v) == prefill row L."""
    for variant in ({}, {"n_kv_heads": 4}, {"use_rope": False}):
        cfg, w, _ = _small_block(orc, lossless=False, seed=41, **variant)
        r = np.random.default_rng(42)
        lens = [3, 0, 6]
        max_seq = 8
        zk = np.zeros((3, max_seq, cfg.r_k))
        zv = np.zeros((3, max_seq, cfg.r_v))
        xs, ref, ref_zk = [], [], []
        for b, L in enumerate(lens):
            x = r.standard_normal((L + 1, cfg.h))
            out, _, _ = orc.block_prefill(cfg, w, x, np.arange(L + 1), [0, L + 1])
            a = orc.rmsnorm(x, w["g_attn"], cfg.rms_eps)
            zk[b, :L] = orc.matmul(a, w["B_k"].T)[:L]
            zv[b, :L] = orc.matmul(a, w["B_v"].T)[:L]
            xs.append(x[L])
            ref.append(out[L])
            ref_zk.append(orc.matmul(a[L:L + 1], w["B_k"].T)[0])
        o, zk_new, _ = orc.block_decode_lowrank(cfg, w, np.stack(xs), zk, zv, lens)
        assert rel(o, np.stack(ref)) < 1e-12, variant
        assert rel(zk_new, np.stack(ref_zk)) < 1e-13


def _brute_min_runs(phys):
    """Minimal order-preserving partition into ascending-by-one runs (exhaustive)."""
    n = len(phys)
    best = None
    for mask in range(1 << max(n - 1, 0)):
        cuts = [i + 1 for i in range(n - 1) if mask >> i & 1]
        parts, lo = [], 0
        for c in cuts + [n]:
            parts.append(phys[lo:c])
            lo = c
        if all(all(p[i + 1] == p[i] + 1 for i in range(len(p) - 1)) for p in parts):
            if best is None or len(parts) < len(best):
                best = parts
    return [(p[0], len(p)) for p in best] if n else []


def test_kv_runs_examples_and_minimality(orc):
    """P:226 contiguous-run scan: SPEC examples and a brute-force minimal partition."""
    assert orc.kv_runs([5, 6, 7]) == [(5, 3)]
    assert orc.kv_runs([5, 7, 6]) == [(5, 1), (7, 1), (6, 1)]
    assert orc.kv_runs([]) == []
    r = np.random.default_rng(43)
    for _ in range(60):
        n = int(r.integers(1, 9))
        phys = [int(v) for v in r.permutation(12)[:n]] if r.random() < 0.5 else \
            [int(v) for v in np.sort(r.choice(12, n, replace=False))]
        runs = orc.kv_runs(phys)
        assert runs == _brute_min_runs(phys), phys
        assert sum(ln for _, ln in runs) == n
