"""Pins for the oracle's linear-algebra functions (-m "not gpu").

Each test pins the oracle to something other than itself: values the paper
or SPEC print (tests/golden/*), closed forms, special cases that reduce to a
library routine (numpy SVD / matmul), or invariants fixed by the mathematics.
"""
import numpy as np
import pytest

from conftest import golden


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ---- matmul -------------------------------------------------------
def test_matmul_spec_examples(orc):
    g = golden("spec_matmul.json")
    np.testing.assert_array_equal(orc.matmul(g["a"], g["b"]), np.array(g["c"], float))
    M = np.random.default_rng(0).standard_normal((3, 3))
    np.testing.assert_array_equal(orc.matmul(np.eye(3), M), M)


def test_matmul_vs_numpy(orc):
    r = np.random.default_rng(1)
    a, b = r.standard_normal((5, 4)), r.standard_normal((4, 3))
    assert rel(orc.matmul(a, b), a @ b) < 1e-14


# ---- low-rank linear, Eq. 1 --------------------------------------
def test_lowrank_hand_example(orc):
    g = golden("lowrank_hand.json")
    Y = orc.lowrank_linear(g["X"], g["A"], g["B"])
    np.testing.assert_array_equal(Y, np.array(g["Y"], float))
    # y = Wx with W = AB printed in the fixture (catches an A/B swap)
    np.testing.assert_array_equal(Y, np.array(g["X"], float) @ np.array(g["W"], float).T)


@pytest.mark.parametrize("m,n", [(7, 5), (5, 9), (16, 16)])
def test_lowrank_full_rank_equals_dense(orc, m, n):
    """North-star self-check (3): at k = min(m,n), A(Bx) = Wx exactly (to rounding)."""
    r = np.random.default_rng(m * 100 + n)
    W = r.standard_normal((m, n))
    X = r.standard_normal((6, n))
    U, s, Vt = np.linalg.svd(W, full_matrices=False)          # independent library SVD
    k = min(m, n)
    A = U[:, :k] * np.sqrt(s[:k])
    B = np.sqrt(s[:k])[:, None] * Vt[:k]
    assert rel(orc.lowrank_linear(X, A, B), X @ W.T) < 1e-12
    A2, B2, _ = orc.truncated_svd(W, k)                       # oracle SVD factors
    assert rel(orc.lowrank_linear(X, A2, B2), X @ W.T) < 1e-12


def test_lowrank_empty_tokens(orc):
    r = np.random.default_rng(2)
    Y = orc.lowrank_linear(np.zeros((0, 6)), r.standard_normal((4, 3)), r.standard_normal((3, 6)))
    assert Y.shape == (0, 4)


# ---- truncated SVD ---------------------------------------------------
def test_svd_diag_exact(orc):
    W = np.diag([3.0, 2.0, 1.0])
    A, B, s = orc.truncated_svd(W, 3)
    assert np.abs(A @ B - W).max() < 1e-12
    np.testing.assert_allclose(s, [3, 2, 1], atol=1e-12)


def test_svd_rank1_exact(orc):
    r = np.random.default_rng(3)
    u, v = r.standard_normal(6), r.standard_normal(4)
    W = np.outer(u, v)
    A, B, s = orc.truncated_svd(W, 1)
    assert np.abs(A @ B - W).max() < 1e-12
    assert abs(s[0] - np.linalg.norm(u) * np.linalg.norm(v)) < 1e-12


@pytest.mark.parametrize("seed", range(10))
def test_svd_tail_energy_eckart_young(orc, seed):
    """||W - AB||_F^2 = sum_{i>k} sigma_i^2 against numpy's independent SVD."""
    r = np.random.default_rng(100 + seed)
    m, n = r.integers(2, 24, size=2)
    W = r.standard_normal((m, n))
    sig = np.linalg.svd(W, compute_uv=False)
    errs = []
    for k in range(1, min(m, n) + 1):
        A, B, s = orc.truncated_svd(W, k)
        e = np.linalg.norm(W - A @ B) ** 2
        tail = float(np.sum(sig[k:] ** 2))
        assert abs(e - tail) <= 1e-9 * max(np.linalg.norm(W) ** 2, 1.0)
        np.testing.assert_allclose(s, sig, rtol=1e-10, atol=1e-12)
        errs.append(e)
        # factor symmetry: ||A[:,j]|| = ||B[j,:]|| = sqrt(sigma_j)
        np.testing.assert_allclose(np.linalg.norm(A, axis=0), np.sqrt(sig[:k]), rtol=1e-9)
        np.testing.assert_allclose(np.linalg.norm(B, axis=1), np.sqrt(sig[:k]), rtol=1e-9)
    assert all(errs[i] >= errs[i + 1] - 1e-12 for i in range(len(errs) - 1))  # S:62 monotone


def test_svd_rank_errors(orc):
    with pytest.raises(ValueError):
        orc.truncated_svd(np.eye(3), 4)
    with pytest.raises(ValueError):
        orc.truncated_svd(np.eye(3), 0)


# ---- parameter count ----------------------------------------------------
def test_param_count_identity(orc):
    """North-star self-check (2): stored elements of (A, B) = (m+n)k exactly."""
    r = np.random.default_rng(4)
    for m, n, k in [(9, 5, 3), (4, 11, 4), (8, 8, 1)]:
        A, B, _ = orc.truncated_svd(r.standard_normal((m, n)), k)
        assert A.size + B.size == orc.factor_params(m, n, k) == (m + n) * k


def test_param_count_paper_blocks(orc):
    from synthetic import LLAMA3_70B, LLAMA3_8B, block_ranks
    g = golden("param_counts.json")
    for shape, ratio, key in [(LLAMA3_70B, 0.4, "llama3_70b_40"), (LLAMA3_8B, 0.2, "llama3_8b_20")]:
        rk = block_ranks(shape, ratio)
        cfg = orc.BlockCfg(shape.h, shape.n_heads, shape.n_kv_heads, shape.head_dim, shape.m,
                           rk["q"], rk["k"], rk["v"], rk["o"], rk["gate"], rk["up"], rk["down"])
        assert orc.block_params(cfg) == g[key]


# ---- rank sharding -------------------------------
@pytest.mark.parametrize("k", [1, 7, 64, 614, 4916, 6144, 9832])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_ranges_cover_once(orc, k, world):
    if k < world:
        pytest.skip("fewer ranks than ranks-of-k")
    cover = np.zeros(k, int)
    lens = []
    for r in range(world):
        b, ln, lp = orc.shard_range(k, world, r, 1)
        cover[b:b + ln] += 1
        lens.append(ln)
        assert lp == ln
    assert (cover == 1).all()
    assert max(lens) - min(lens) <= 1          # "evenly split"


def test_shard_strict_and_padding(orc):
    with pytest.raises(ValueError):
        orc.shard_range(614, 8, 0, 0)           # strict mode rejects 614 % 8 != 0
    assert orc.shard_range(6144, 8, 7, 0) == (5376, 768, 768)  # QKV concat 70B@40%, TP=8
    b, ln, lp = orc.shard_range(614, 8, 7, 64)
    assert (b, ln, lp) == (538, 76, 128)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("align", [1, 8, 64])
def test_sharded_equals_unsharded(orc, world, align):
    """North-star self-check (4): sum_r A_r(B_r x) = A(Bx) incl. padded odd ranks."""
    r = np.random.default_rng(world * 10 + align)
    m, n, k, T = 24, 20, 37, 5
    X, A, B = r.standard_normal((T, n)), r.standard_normal((m, k)), r.standard_normal((k, n))
    Y1 = orc.lowrank_linear(X, A, B)
    Yp = orc.lowrank_linear_sharded(X, A, B, world, align)
    assert rel(Yp, Y1) < 1e-12
    assert rel(Y1, X @ (A @ B).T) < 1e-12      # and both equal the dense product (numpy)
