"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle, element by
element on the same seeded inputs.  Tolerances (north_star): relative L2
<= 2e-2 for bf16, <= 1e-5 for fp32.  Block outputs are compared on the
block's contribution x_out - x_in (stricter than comparing x_out).
"""
import numpy as np
import pytest
import torch

from synthetic import LLAMA3_8B, ModelShape, block_ranks, gen_block_weights, gen_factor_pair, gen_normal

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2
TOL_F32 = 1e-5


def rel(a, b):
    a, b = (t.detach().cpu().double().numpy() if isinstance(t, torch.Tensor) else t for t in (a, b))
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def dl():
    import paper_2604_17709_b200 as dl
    from paper_2604_17709_b200 import build
    build.build()
    dl.load()
    assert dl.dl_device_ok(), "needs an sm_100 GPU"
    return dl


def _lin_inputs(T, m, n, k, dtype, seed):
    X = gen_normal((T, n), 1.0, seed, dtype=dtype)
    A, B = gen_factor_pair(m, n, k, seed + 7, dtype=dtype)
    return X, A, B


# ---- dl_lowrank_linear --------------------------------------------------------
def test_linear_config1_fp32(dl, orc):
    """BASELINE config 1: m=n=256, k=64, T=4, fp32 vs CPU oracle (1e-5)."""
    X, A, B = _lin_inputs(4, 256, 256, 64, torch.float32, 1)
    Y = torch.empty(4, 256, device="cuda")
    dl.dl_lowrank_linear(X.cuda(), A.cuda(), B.cuda(), Y)
    torch.cuda.synchronize()
    assert rel(Y.cpu(), orc.lowrank_linear(X, A, B)) <= TOL_F32


@pytest.mark.parametrize("T,m,n,k,dt", [(4, 256, 256, 64, torch.float32), (16, 200, 120, 96, torch.float32),
                                        (7, 180, 180, 180, torch.float32), (16, 200, 96, 88, torch.bfloat16),
                                        (1, 64, 512, 64, torch.bfloat16)])
def test_linear_simt_small_chain(dl, orc, T, m, n, k, dt):
    """Fused small chain (Z in shared memory; several CTAs each recompute Z and own a
    64-row slice of Y): ragged m, T up to 16, fp32 and bf16."""
    X, A, B = _lin_inputs(T, m, n, k, dt, 30 + T + m)
    Y = torch.empty(T, m, device="cuda", dtype=dt)
    dl.dl_lowrank_linear(X.cuda(), A.cuda(), B.cuda(), Y)
    torch.cuda.synchronize()
    assert rel(Y.cpu(), orc.lowrank_linear(X, A, B)) <= (TOL_F32 if dt == torch.float32 else TOL_BF16)


@pytest.mark.parametrize("T", [1, 3, 16])
def test_linear_fp32_simt_large(dl, orc, T):
    """fp32 SIMT chain at a size that takes the two-kernel path (k > 1024 is not needed: (m+n)k > 64K)."""
    X, A, B = _lin_inputs(T, 1000, 520, 300, torch.float32, 2 + T)
    Y = torch.empty(T, 1000, device="cuda")
    dl.dl_lowrank_linear(X.cuda(), A.cuda(), B.cuda(), Y)
    torch.cuda.synchronize()
    assert rel(Y.cpu(), orc.lowrank_linear(X, A, B)) <= TOL_F32


@pytest.mark.parametrize("T", [1, 5, 16, 17, 64, 100, 256, 257, 300, 1000])
@pytest.mark.parametrize("accumulate", [False, True])
def test_linear_bf16_paths(dl, orc, T, accumulate):
    """SIMT (T<=16), swap-AB stream-K (17..256) and wide whole-tile (>256) paths.
    m spans 5 M-tiles, n and k are ragged (not multiples of the 64-wide K block)."""
    m, n, k = 640, 520, 200
    X, A, B = _lin_inputs(T, m, n, k, torch.bfloat16, 10 + T)
    Y0 = gen_normal((T, m), 1.0, 99, dtype=torch.bfloat16)
    Y = Y0.clone().cuda()
    dl.dl_lowrank_linear(X.cuda(), A.cuda(), B.cuda(), Y, accumulate=accumulate)
    torch.cuda.synchronize()
    ref = orc.lowrank_linear(X, A, B)
    got = Y.cpu().double().numpy()
    if accumulate:
        got = got - Y0.double().numpy()
    assert rel(got, ref) <= TOL_BF16


def test_linear_bf16_large_shapes(dl, orc):
    """70B o-projection shape (n=m=8192, k=4916) at decode batch 64, sampled via all rows (oracle is fast here)."""
    T, m, n, k = 64, 8192, 8192, 4916
    X, A, B = _lin_inputs(T, m, n, k, torch.bfloat16, 5)
    Y = torch.empty(T, m, dtype=torch.bfloat16, device="cuda")
    A_pad = torch.zeros(m, 4920, dtype=torch.bfloat16, device="cuda")   # ld must be a 16-byte multiple
    A_pad[:, :k] = A.cuda()
    dl.dl_lowrank_linear(X.cuda(), A_pad[:, :k], B.cuda(), Y)
    torch.cuda.synchronize()
    rows = [0, 17, 63]
    ref = orc.lowrank_linear(X[rows], A, B)
    assert rel(Y.cpu()[rows], ref) <= TOL_BF16


@pytest.mark.parametrize("P,T", [(2, 64), (4, 17), (8, 100)])
def test_linear_reads_rank_major_gather(dl, orc, P, T):
    """The TP o projection reads the attention all-gather [P][T][h/P] in place
    through a 3-D TMA map (no un-permute pass): same result as the logical
    [T x h] operand."""
    from paper_2604_17709_b200 import _lib
    w, m, k = 128, 384, 96
    n = P * w
    X, A, B = _lin_inputs(T, m, n, k, torch.bfloat16, 40 + P)
    Xg = X.view(T, P, w).permute(1, 0, 2).contiguous()
    Y = torch.empty(T, m, dtype=torch.bfloat16, device="cuda")
    _lib.dl_debug_linear_gathered(Xg.cuda(), A.cuda(), B.cuda(), Y)
    torch.cuda.synchronize()
    assert rel(Y.cpu(), orc.lowrank_linear(X, A, B)) <= TOL_BF16


@pytest.mark.parametrize("T", [4, 64, 300])
def test_linear_degenerate_ranks(dl, T):
    """Degenerate decompositions with closed forms (Eq. 1, y = A(Bx)):
    B = I (k = n) reduces to the dense product X Aᵀ, and k = 1 to the outer
    product (X b) aᵀ -- checked against float64 torch, not the oracle."""
    n, m = 256, 384
    X = gen_normal((T, n), 1.0, 60 + T, dtype=torch.bfloat16)
    A = gen_normal((m, n), n ** -0.5, 61, dtype=torch.bfloat16)
    Y = torch.empty(T, m, dtype=torch.bfloat16, device="cuda")
    dl.dl_lowrank_linear(X.cuda(), A.cuda(), torch.eye(n, dtype=torch.bfloat16, device="cuda"), Y)
    torch.cuda.synchronize()
    assert rel(Y.cpu(), X.double() @ A.double().T) <= TOL_BF16
    a = gen_normal((m, 1), 1.0, 62, dtype=torch.bfloat16)
    b = gen_normal((1, n), n ** -0.5, 63, dtype=torch.bfloat16)
    Y1 = torch.empty(T, m, dtype=torch.bfloat16, device="cuda")
    a8 = torch.zeros(m, 8, dtype=torch.bfloat16, device="cuda")   # ld must be a 16-byte multiple
    a8[:, :1] = a.cuda()
    dl.dl_lowrank_linear(X.cuda(), a8[:, :1], b.cuda(), Y1)
    torch.cuda.synchronize()
    z = (X.double() @ b.double().T).to(torch.bfloat16).double()   # the kernel's Z is bf16
    assert rel(Y1.cpu(), z @ a.double().T) <= TOL_BF16


def test_dense_lm_head_shape(dl):
    """dl_dense (used for the LM head) vs a float64 torch matmul of the same bf16 values."""
    T, N, K = 64, 1000, 512
    X = gen_normal((T, K), 1.0, 3, dtype=torch.bfloat16)
    W = gen_normal((N, K), K ** -0.5, 4, dtype=torch.bfloat16)
    C = torch.empty(T, N, dtype=torch.bfloat16, device="cuda")
    dl.dl_dense(X.cuda(), W.cuda(), C)
    torch.cuda.synchronize()
    ref = X.double() @ W.double().T
    assert rel(C.cpu(), ref) <= TOL_BF16


# ---- decomposed block ------------------------------------------------------------
SMALL = ModelShape("small", h=512, n_heads=4, n_kv_heads=2, head_dim=128, m=1024, n_layers=1, vocab=1000,
                   rope_theta=500000.0)


def _oracle_cfg(orc, s, rk):
    return orc.BlockCfg(s.h, s.n_heads, s.n_kv_heads, s.head_dim, s.m, rk["q"], rk["k"], rk["v"], rk["o"],
                        rk["gate"], rk["up"], rk["down"], rope_theta=s.rope_theta, rms_eps=s.rms_eps,
                        mlp_glu=int(s.glu), use_rope=int(s.rope))


def _cache_to_oracle(c, S, L):
    # GPU [S, Hk, max_seq, d] -> oracle [S, max_seq, Hk*d]
    return c[:S].permute(0, 2, 1, 3).reshape(S, c.shape[2], -1)[:, :L].cpu()


def _run_prefill(dl, orc, s, ratio, lens, seed):
    rk = block_ranks(s, ratio)
    w = gen_block_weights(s, rk, 0, seed)
    T = sum(lens)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    pos = np.concatenate([np.arange(L) for L in lens]).astype(np.int32)
    x = gen_normal((T, s.h), 1.0, seed + 100, dtype=torch.bfloat16)
    max_seq = max(lens) + 8
    cfg = dl.make_block_config(s, rk, max_tokens=T, max_seqs=len(lens))
    wdev = dl.BlockWeights({k: v.cuda() for k, v in w.items()})
    ws = torch.zeros(dl.dl_block_workspace(cfg), dtype=torch.uint8, device="cuda")
    kc = torch.zeros(len(lens), s.n_kv_heads, max_seq, s.head_dim, dtype=torch.bfloat16, device="cuda")
    vc = torch.zeros_like(kc)
    xd = x.cuda()
    dl.dl_decomposed_block_forward(cfg, wdev, xd, torch.from_numpy(pos).cuda(), torch.from_numpy(cu).cuda(),
                                   len(lens), dl.DL_PREFILL, kc, vc, torch.zeros(len(lens), dtype=torch.int32,
                                                                                  device="cuda"), None, ws)
    torch.cuda.synchronize()
    return w, rk, x, xd.cpu(), pos, cu, kc, vc


@pytest.mark.parametrize("lens", [[100], [60, 1, 39], [300], [129, 200, 71]])
def test_block_prefill_small(dl, orc, lens):
    s = SMALL
    w, rk, x, xo, pos, cu, kc, vc = _run_prefill(dl, orc, s, 0.4, lens, seed=len(lens) * 7 + lens[0])
    ref, rk_, rv_ = orc.block_prefill(_oracle_cfg(orc, s, rk), w, x, pos, cu)
    assert rel(xo.double() - x.double(), ref - x.double().numpy()) <= TOL_BF16
    # KV cache written by the kernel == oracle's post-RoPE keys / values
    for si in range(len(lens)):
        a, b = cu[si], cu[si + 1]
        kg = kc[si, :, :b - a].permute(1, 0, 2).reshape(b - a, -1).cpu()
        vg = vc[si, :, :b - a].permute(1, 0, 2).reshape(b - a, -1).cpu()
        assert rel(kg, rk_[a:b]) <= TOL_BF16
        assert rel(vg, rv_[a:b]) <= TOL_BF16


@pytest.mark.parametrize("first,second", [([70], [60]), ([1, 128, 33], [64, 5, 200]), ([129, 0], [1, 77])])
def test_block_prefill_continues_cached_prefix(dl, orc, first, second):
    """Chunked prefill (include/dl.h: PREFILL token i of sequence s sits at position
    cache_lens[s] + i and attends to the cached prefix too): prefill chunk 1, then
    chunk 2 with cache_lens = len(chunk 1).  Chunk 2's rows must equal the
    oracle's one-shot causal prefill of the concatenated sequences (PAPER.md
    eq. 1-3 attention is causal over all earlier keys), and the cache must hold
    the keys of both chunks."""
    s = SMALL
    rk = block_ranks(s, 0.4)
    w = gen_block_weights(s, rk, 0, 21)
    S = len(first)
    full = [a + b for a, b in zip(first, second)]
    x_full = gen_normal((sum(full), s.h), 1.0, 22, dtype=torch.bfloat16)
    cu_full = np.concatenate([[0], np.cumsum(full)]).astype(np.int32)
    pos_full = np.concatenate([np.arange(L) for L in full]).astype(np.int32)
    ref, rk_, _ = orc.block_prefill(_oracle_cfg(orc, s, rk), w, x_full, pos_full, cu_full)

    max_seq = max(full) + 8
    cfg = dl.make_block_config(s, rk, max_tokens=sum(full), max_seqs=S)
    wdev = dl.BlockWeights({k: v.cuda() for k, v in w.items()})
    ws = torch.zeros(dl.dl_block_workspace(cfg), dtype=torch.uint8, device="cuda")
    kc = torch.zeros(S, s.n_kv_heads, max_seq, s.head_dim, dtype=torch.bfloat16, device="cuda")
    vc = torch.zeros_like(kc)
    outs = []
    for chunk, before in ((first, [0] * S), (second, first)):
        rows = np.concatenate([np.arange(cu_full[i] + before[i], cu_full[i] + before[i] + chunk[i])
                               for i in range(S)]).astype(np.int64)
        if len(rows) == 0:
            continue
        pos = np.concatenate([np.arange(before[i], before[i] + chunk[i]) for i in range(S)]).astype(np.int32)
        cu = np.concatenate([[0], np.cumsum(chunk)]).astype(np.int32)
        xd = x_full[rows].clone().cuda()
        cl = torch.tensor(before, dtype=torch.int32, device="cuda")
        dl.dl_decomposed_block_forward(cfg, wdev, xd, torch.from_numpy(pos).cuda(), torch.from_numpy(cu).cuda(),
                                       S, dl.DL_PREFILL, kc, vc, cl, None, ws)
        torch.cuda.synchronize()
        outs.append((rows, xd.cpu()))
    rows2, xo2 = outs[-1]
    xin2 = x_full[rows2].double()
    assert rel(xo2.double() - xin2, ref[rows2] - xin2.numpy()) <= TOL_BF16
    for i in range(S):
        a, L = cu_full[i], full[i]
        kg = kc[i, :, :L].permute(1, 0, 2).reshape(L, -1).cpu()
        assert rel(kg, rk_[a:a + L]) <= TOL_BF16


@pytest.mark.parametrize("first,second", [([300, 1], [129, 250]), ([0, 127], [385, 1])])
def test_block_prefill_cached_prefix_nan_tail(dl, orc, first, second):
    """The tcgen05 prefill attention reads whole 128-key tiles of the cache: key
    rows past the visible range (unwritten slots, here NaN) must neither leak
    through the masked scores nor through 0 x NaN in P.V.  Chunked prefill over
    NaN-initialised caches, query tiles spanning several key tiles, ragged ends."""
    s = SMALL
    rk = block_ranks(s, 0.4)
    w = gen_block_weights(s, rk, 0, 31)
    S = len(first)
    full = [a + b for a, b in zip(first, second)]
    x_full = gen_normal((sum(full), s.h), 1.0, 32, dtype=torch.bfloat16)
    cu_full = np.concatenate([[0], np.cumsum(full)]).astype(np.int32)
    pos_full = np.concatenate([np.arange(L) for L in full]).astype(np.int32)
    ref, _, _ = orc.block_prefill(_oracle_cfg(orc, s, rk), w, x_full, pos_full, cu_full)
    max_seq = max(full) + 200
    cfg = dl.make_block_config(s, rk, max_tokens=sum(full), max_seqs=S)
    wdev = dl.BlockWeights({k: v.cuda() for k, v in w.items()})
    ws = torch.zeros(dl.dl_block_workspace(cfg), dtype=torch.uint8, device="cuda")
    kc = torch.full((S, s.n_kv_heads, max_seq, s.head_dim), float("nan"), dtype=torch.bfloat16, device="cuda")
    vc = torch.full_like(kc, float("nan"))
    last = None
    for chunk, before in ((first, [0] * S), (second, first)):
        rows = np.concatenate([np.arange(cu_full[i] + before[i], cu_full[i] + before[i] + chunk[i])
                               for i in range(S)]).astype(np.int64)
        pos = np.concatenate([np.arange(before[i], before[i] + chunk[i]) for i in range(S)]).astype(np.int32)
        cu = np.concatenate([[0], np.cumsum(chunk)]).astype(np.int32)
        xd = x_full[rows].clone().cuda()
        cl = torch.tensor(before, dtype=torch.int32, device="cuda")
        dl.dl_decomposed_block_forward(cfg, wdev, xd, torch.from_numpy(pos).cuda(), torch.from_numpy(cu).cuda(),
                                       S, dl.DL_PREFILL, kc, vc, cl, None, ws)
        torch.cuda.synchronize()
        last = (rows, xd.cpu())
    rows2, xo2 = last
    assert torch.isfinite(xo2.float()).all()
    xin2 = x_full[rows2].double()
    assert rel(xo2.double() - xin2, ref[rows2] - xin2.numpy()) <= TOL_BF16


@pytest.mark.parametrize("cache_lens", [[0, 5, 17, 1, 33, 2, 7, 100], [511] * 4])
def test_block_decode_small(dl, orc, cache_lens):
    s = SMALL
    rk = block_ranks(s, 0.4)
    w = gen_block_weights(s, rk, 0, 3)
    S = len(cache_lens)
    max_seq = max(cache_lens) + 1
    x = gen_normal((S, s.h), 1.0, 5, dtype=torch.bfloat16)
    kc = gen_normal((S, s.n_kv_heads, max_seq, s.head_dim), 1.0, 6, dtype=torch.bfloat16)
    vc = gen_normal((S, s.n_kv_heads, max_seq, s.head_dim), 1.0, 7, dtype=torch.bfloat16)
    ko, vo = _cache_to_oracle(kc, S, max_seq), _cache_to_oracle(vc, S, max_seq)
    cl = torch.tensor(cache_lens, dtype=torch.int32)
    cfg = dl.make_block_config(s, rk, max_tokens=S, max_seqs=S)
    wdev = dl.BlockWeights({k: v.cuda() for k, v in w.items()})
    ws = torch.zeros(dl.dl_block_workspace(cfg), dtype=torch.uint8, device="cuda")
    xd, kcd, vcd = x.cuda(), kc.cuda(), vc.cuda()
    dl.dl_decomposed_block_forward(cfg, wdev, xd, cl.cuda(), None, S, dl.DL_DECODE, kcd, vcd, cl.cuda(), None, ws)
    torch.cuda.synchronize()
    ref, kn, vn = orc.block_decode(_oracle_cfg(orc, s, rk), w, x, ko, vo, cache_lens)
    assert rel(xd.cpu().double() - x.double(), ref - x.double().numpy()) <= TOL_BF16
    kg = torch.stack([kcd[b, :, cache_lens[b]].reshape(-1) for b in range(S)]).cpu()
    assert rel(kg, kn) <= TOL_BF16


@pytest.mark.parametrize("S", [100, 200, 256, 300])
def test_block_decode_wide_batches(dl, orc, S):
    """Decode batches on the 128- and 256-token swap-AB configurations (the bench runs 64)
    and beyond (300: whole-tile GEMMs): bf16x2 latent / gate|up reductions, stream-K
    attention over S sequences, run twice."""
    s = SMALL
    rk = block_ranks(s, 0.4)
    w = gen_block_weights(s, rk, 0, 50 + S)
    rng = np.random.default_rng(S)
    cache_lens = [int(v) for v in rng.integers(0, 90, S)]
    max_seq = max(cache_lens) + 1
    x = gen_normal((S, s.h), 1.0, 51, dtype=torch.bfloat16)
    kc = gen_normal((S, s.n_kv_heads, max_seq, s.head_dim), 1.0, 52, dtype=torch.bfloat16)
    vc = gen_normal((S, s.n_kv_heads, max_seq, s.head_dim), 1.0, 53, dtype=torch.bfloat16)
    ko, vo = _cache_to_oracle(kc, S, max_seq), _cache_to_oracle(vc, S, max_seq)
    cl = torch.tensor(cache_lens, dtype=torch.int32)
    cfg = dl.make_block_config(s, rk, max_tokens=S, max_seqs=S)
    wdev = dl.BlockWeights({k: v.cuda() for k, v in w.items()})
    ws = torch.zeros(dl.dl_block_workspace(cfg), dtype=torch.uint8, device="cuda")
    ref, _, _ = orc.block_decode(_oracle_cfg(orc, s, rk), w, x, ko, vo, cache_lens)
    for _ in range(2):
        xd, kcd, vcd = x.cuda(), kc.cuda(), vc.cuda()
        dl.dl_decomposed_block_forward(cfg, wdev, xd, cl.cuda(), None, S, dl.DL_DECODE, kcd, vcd, cl.cuda(), None,
                                       ws)
        torch.cuda.synchronize()
        assert rel(xd.cpu().double() - x.double(), ref - x.double().numpy()) <= TOL_BF16


@pytest.mark.parametrize("cache_lens", [[4000, 3, 700], [63, 64, 127, 128, 0]])
def test_block_decode_long_ragged_nan_tail(dl, orc, cache_lens):
    """Stream-K decode attention: one long item spread over many CTAs next to short ones,
    tile-boundary lengths, and NaN in the unwritten cache slots past each sequence
    (masked keys must contribute exactly nothing). Two calls: the merge counters reset."""
    s = SMALL
    rk = block_ranks(s, 0.4)
    w = gen_block_weights(s, rk, 0, 21)
    S = len(cache_lens)
    max_seq = max(cache_lens) + 70
    x = gen_normal((S, s.h), 1.0, 22, dtype=torch.bfloat16)
    kc = gen_normal((S, s.n_kv_heads, max_seq, s.head_dim), 1.0, 23, dtype=torch.bfloat16)
    vc = gen_normal((S, s.n_kv_heads, max_seq, s.head_dim), 1.0, 24, dtype=torch.bfloat16)
    ko, vo = _cache_to_oracle(kc, S, max_seq), _cache_to_oracle(vc, S, max_seq)
    for b, L in enumerate(cache_lens):          # garbage past the appended slot
        kc[b, :, L + 1:] = float("nan")
        vc[b, :, L + 1:] = float("nan")
    cl = torch.tensor(cache_lens, dtype=torch.int32)
    cfg = dl.make_block_config(s, rk, max_tokens=S, max_seqs=S)
    wdev = dl.BlockWeights({k: v.cuda() for k, v in w.items()})
    ws = torch.zeros(dl.dl_block_workspace(cfg), dtype=torch.uint8, device="cuda")
    ref, _, _ = orc.block_decode(_oracle_cfg(orc, s, rk), w, x, ko, vo, cache_lens)
    for _ in range(2):
        xd, kcd, vcd = x.cuda(), kc.cuda(), vc.cuda()
        dl.dl_decomposed_block_forward(cfg, wdev, xd, cl.cuda(), None, S, dl.DL_DECODE, kcd, vcd, cl.cuda(), None,
                                       ws)
        torch.cuda.synchronize()
        got = xd.cpu().double() - x.double()
        assert torch.isfinite(got).all()
        assert rel(got, ref - x.double().numpy()) <= TOL_BF16


def test_block_workspace_left_zeroed_and_repeatable(dl, orc):
    """Consume-and-clear: two identical decode calls give identical results."""
    s = SMALL
    rk = block_ranks(s, 0.4)
    w = gen_block_weights(s, rk, 0, 4)
    S = 16
    cl = torch.full((S,), 9, dtype=torch.int32, device="cuda")
    cfg = dl.make_block_config(s, rk, max_tokens=S, max_seqs=S)
    wdev = dl.BlockWeights({k: v.cuda() for k, v in w.items()})
    ws = torch.zeros(dl.dl_block_workspace(cfg), dtype=torch.uint8, device="cuda")
    x = gen_normal((S, s.h), 1.0, 8, dtype=torch.bfloat16).cuda()
    kc = torch.zeros(S, s.n_kv_heads, 16, s.head_dim, dtype=torch.bfloat16, device="cuda")
    vc = torch.zeros_like(kc)
    outs = []
    for _ in range(2):
        xx = x.clone()
        dl.dl_decomposed_block_forward(cfg, wdev, xx, cl, None, S, dl.DL_DECODE, kc, vc, cl, None, ws)
        outs.append(xx)
    torch.cuda.synchronize()
    assert float((outs[0].float() - outs[1].float()).abs().max()) < 0.05
    # everything except the bf16 staging must be zero again
    assert rel(outs[0].cpu(), outs[1].cpu()) < 1e-2


@pytest.mark.slow
def test_block_8b_prefill_2048_sampled(dl, orc):
    """BASELINE config 2 at full size (8B @20%, one sequence of 2048 tokens):
    sampled output rows vs the oracle (which recomputes K/V for all tokens)."""
    s = LLAMA3_8B
    w, rk, x, xo, pos, cu, kc, vc = _run_prefill(dl, orc, s, 0.2, [2048], seed=11)
    rows = [0, 1, 511, 1024, 2047]
    ref, _, _ = orc.block_prefill(_oracle_cfg(orc, s, rk), w, x, pos, cu, rows=rows)
    assert rel(xo[rows].double() - x[rows].double(), ref - x[rows].double().numpy()) <= TOL_BF16


@pytest.mark.slow
def test_block_8b_decode_b64_sampled(dl, orc):
    """Config 3 layer shape: 8B @20%, decode batch 64, context 512; 4 sampled sequences."""
    s = LLAMA3_8B
    rk = block_ranks(s, 0.2)
    w = gen_block_weights(s, rk, 0, 12)
    S, L = 64, 512
    x = gen_normal((S, s.h), 1.0, 13, dtype=torch.bfloat16)
    kc = gen_normal((S, s.n_kv_heads, L + 1, s.head_dim), 1.0, 14, dtype=torch.bfloat16)
    vc = gen_normal((S, s.n_kv_heads, L + 1, s.head_dim), 1.0, 15, dtype=torch.bfloat16)
    cl = torch.full((S,), L, dtype=torch.int32)
    cfg = dl.make_block_config(s, rk, max_tokens=S, max_seqs=S)
    wdev = dl.BlockWeights({k: v.cuda() for k, v in w.items()})
    ws = torch.zeros(dl.dl_block_workspace(cfg), dtype=torch.uint8, device="cuda")
    xd, kcd, vcd = x.cuda(), kc.cuda(), vc.cuda()
    dl.dl_decomposed_block_forward(cfg, wdev, xd, cl.cuda(), None, S, dl.DL_DECODE, kcd, vcd, cl.cuda(), None, ws)
    torch.cuda.synchronize()
    pick = [0, 21, 42, 63]
    ref, _, _ = orc.block_decode(_oracle_cfg(orc, s, rk), w, x[pick], _cache_to_oracle(kc[pick], 4, L + 1),
                                 _cache_to_oracle(vc[pick], 4, L + 1), [L] * 4)
    got = xd.cpu()[pick].double() - x[pick].double()
    assert rel(got, ref - x[pick].double().numpy()) <= TOL_BF16


# ---- model-family variants (N4: Table 2) -------------------------------------
VARIANT_SHAPES = {
    "mha": ModelShape("mha", h=512, n_heads=4, n_kv_heads=4, head_dim=128, m=1024, n_layers=1, vocab=1000,
                      rope_theta=10000.0),
    "mqa32": ModelShape("mqa32", h=4096, n_heads=32, n_kv_heads=1, head_dim=128, m=1024, n_layers=1,
                        vocab=1000),
    "opt": ModelShape("opt", h=512, n_heads=4, n_kv_heads=4, head_dim=128, m=2048, n_layers=1, vocab=1000,
                      glu=False, rope=False),
    "gqa_relu": ModelShape("gqa_relu", h=1024, n_heads=8, n_kv_heads=2, head_dim=128, m=1024, n_layers=1,
                           vocab=1000, glu=False),
}


@pytest.mark.parametrize("name", sorted(VARIANT_SHAPES))
@pytest.mark.parametrize("lens", [[70], [300, 45]])
def test_variant_block_prefill(dl, orc, name, lens):
    s = VARIANT_SHAPES[name]
    w, rk, x, xo, pos, cu, kc, vc = _run_prefill(dl, orc, s, 0.4, lens, seed=31 + len(lens))
    ref, rk_, _ = orc.block_prefill(_oracle_cfg(orc, s, rk), w, x, pos, cu)
    assert rel(xo.double() - x.double(), ref - x.double().numpy()) <= TOL_BF16
    kg = kc[0, :, :lens[0]].permute(1, 0, 2).reshape(lens[0], -1).cpu()
    assert rel(kg, rk_[:lens[0]]) <= TOL_BF16


@pytest.mark.parametrize("name", sorted(VARIANT_SHAPES))
@pytest.mark.parametrize("S", [5, 40])
def test_variant_block_decode(dl, orc, name, S):
    s = VARIANT_SHAPES[name]
    rk = block_ranks(s, 0.4)
    w = gen_block_weights(s, rk, 0, 41)
    cache_lens = [(17 * i + 3) % 150 for i in range(S)]
    max_seq = max(cache_lens) + 1
    x = gen_normal((S, s.h), 1.0, 42, dtype=torch.bfloat16)
    kc = gen_normal((S, s.n_kv_heads, max_seq, s.head_dim), 1.0, 43, dtype=torch.bfloat16)
    vc = gen_normal((S, s.n_kv_heads, max_seq, s.head_dim), 1.0, 44, dtype=torch.bfloat16)
    cl = torch.tensor(cache_lens, dtype=torch.int32)
    cfg = dl.make_block_config(s, rk, max_tokens=S, max_seqs=S)
    wdev = dl.BlockWeights({k: v.cuda() for k, v in w.items()})
    ws = torch.zeros(dl.dl_block_workspace(cfg), dtype=torch.uint8, device="cuda")
    xd, kcd, vcd = x.cuda(), kc.cuda(), vc.cuda()
    dl.dl_decomposed_block_forward(cfg, wdev, xd, cl.cuda(), None, S, dl.DL_DECODE, kcd, vcd, cl.cuda(), None, ws)
    torch.cuda.synchronize()
    ref, kn, _ = orc.block_decode(_oracle_cfg(orc, s, rk), w, x, _cache_to_oracle(kc, S, max_seq),
                                  _cache_to_oracle(vc, S, max_seq), cache_lens)
    assert rel(xd.cpu().double() - x.double(), ref - x.double().numpy()) <= TOL_BF16
    kg = torch.stack([kcd[b, :, cache_lens[b]].reshape(-1) for b in range(S)]).cpu()
    assert rel(kg, kn) <= TOL_BF16


@pytest.mark.parametrize("world", [2, 4])
def test_deinfer_shard_factors_match_slices(dl, world):
    """dl_deinfer_shard_factors: sublayer 1 = concat-split B rows + A row
    shards; sublayer 2 = B input-column shard + full A.  Byte-exact copies."""
    As = [gen_normal((m, k), 1.0, 50 + i, dtype=torch.bfloat16).cuda() for i, (m, k) in
          enumerate([(512, 307), (256, 77), (256, 77)])]
    Bs = [gen_normal((a.shape[1], 512), 1.0, 60 + i, dtype=torch.bfloat16).cuda() for i, a in enumerate(As)]
    Bcat = torch.cat(Bs, 0)
    start = 0
    for r in range(world):
        A_sh, B_sh = dl.dl_deinfer_shard_factors(1, As, Bs, world, r)
        kloc = B_sh.shape[0]
        assert torch.equal(B_sh, Bcat[start:start + kloc])
        start += kloc
        for a, s in zip(As, A_sh):
            ml = a.shape[0] // world
            assert torch.equal(s, a[r * ml:(r + 1) * ml])
        A2, B2 = dl.dl_deinfer_shard_factors(2, As[:1], Bs[:1], world, r)
        nl = 512 // world
        assert torch.equal(B2, Bs[0][:, r * nl:(r + 1) * nl]) and torch.equal(A2[0], As[0])
    assert start == Bcat.shape[0]


@pytest.mark.parametrize("P,T,vloc", [(1, 64, 1000), (4, 7, 333), (8, 64, 16032)])
def test_argmax_over_vocab_shards(dl, P, T, vloc):
    """Greedy next token over P vocab shards (bit-exact index work): equals argmax of
    the concatenated logits, ties to the smallest id."""
    g = torch.Generator().manual_seed(P * 100 + T)
    lg = (torch.randn(P, T, vloc, generator=g) * 3).round().to(torch.bfloat16)   # many ties
    ids = torch.empty(T, dtype=torch.int32, device="cuda")
    dl.dl_argmax(lg.cuda() if P > 1 else lg[0].cuda(), ids)
    torch.cuda.synchronize()
    full = lg.permute(1, 0, 2).reshape(T, P * vloc).float()
    mx = full.max(dim=1, keepdim=True).values
    ref = torch.where(full == mx, torch.arange(P * vloc).float(), float("inf")).min(dim=1).values.long()
    assert torch.equal(ids.cpu().long(), ref)


def test_model_decode_variadic_layer_ranks(dl, orc):
    """N4 variadic per-layer ranks through the whole-model decode step: two
    layers compressed at 40% and 20%; hidden state after the blocks vs the
    oracle applied layer by layer (the embedding row is the first input)."""
    from paper_2604_17709_b200.model import DecomposedLlama
    s = SMALL
    rks = [block_ranks(s, 0.4), block_ranks(s, 0.2)]
    ws_ = [gen_block_weights(s, rk, 5, li) for li, rk in enumerate(rks)]
    S, L = 6, 9
    embed = gen_normal((s.vocab, s.h), 1.0, 70, dtype=torch.bfloat16).cuda()
    lm = gen_normal((s.vocab, s.h), s.h ** -0.5, 71, dtype=torch.bfloat16).cuda()
    model = DecomposedLlama(s, rks, [{k: v.cuda() for k, v in w.items()} for w in ws_], embed,
                            torch.ones(s.h, dtype=torch.bfloat16, device="cuda"), lm, batch=S, max_seq=L + 1)
    model.cache.copy_(gen_normal(tuple(model.cache.shape), 1.0, 72, dtype=torch.bfloat16))
    model.cache_lens.fill_(L)
    ids = torch.arange(S, dtype=torch.int32) * 37 % s.vocab
    model.ids.copy_(ids)
    cache0 = model.cache.cpu()
    model.decode_step()
    torch.cuda.synchronize()
    x = embed.cpu()[ids.long()].double()
    for li, (rk, w) in enumerate(zip(rks, ws_)):
        ko = _cache_to_oracle(cache0[li, 0], S, L + 1)
        vo = _cache_to_oracle(cache0[li, 1], S, L + 1)
        x, _, _ = orc.block_decode(_oracle_cfg(orc, s, rk), w, x, ko, vo, [L] * S)
        x = torch.tensor(x)
    x0 = embed.cpu()[ids.long()].double()
    assert rel(model.x.cpu().double() - x0, (x - x0).numpy()) <= TOL_BF16


def test_model_decode_uniform_stack_three_layers(dl, orc):
    """Uniform ranks: the model's decode step goes through dl_decomposed_stack_forward
    (the residual ending block l fused with block l+1's pre-norm). Three layers with
    distinct norms vs the oracle applied layer by layer."""
    from paper_2604_17709_b200.model import DecomposedLlama
    s = SMALL
    rk = block_ranks(s, 0.4)
    ws_ = [gen_block_weights(s, rk, 6, li) for li in range(3)]
    S, L = 5, 70
    embed = gen_normal((s.vocab, s.h), 1.0, 80, dtype=torch.bfloat16).cuda()
    lm = gen_normal((s.vocab, s.h), s.h ** -0.5, 81, dtype=torch.bfloat16).cuda()
    model = DecomposedLlama(s, rk, [{k: v.cuda() for k, v in w.items()} for w in ws_], embed,
                            torch.ones(s.h, dtype=torch.bfloat16, device="cuda"), lm, batch=S, max_seq=L + 1)
    assert model.stack is not None
    model.cache.copy_(gen_normal(tuple(model.cache.shape), 1.0, 82, dtype=torch.bfloat16))
    model.cache_lens.fill_(L)
    ids = torch.arange(S, dtype=torch.int32) * 53 % s.vocab
    model.ids.copy_(ids)
    cache0 = model.cache.cpu()
    x0 = embed.cpu()[ids.long()].double()
    x = x0
    for li, w in enumerate(ws_):
        ko = _cache_to_oracle(cache0[li, 0], S, L + 1)
        vo = _cache_to_oracle(cache0[li, 1], S, L + 1)
        x, _, _ = orc.block_decode(_oracle_cfg(orc, s, rk), w, x, ko, vo, [L] * S)
        x = torch.tensor(x)
    for _ in range(2):                      # twice: the stack leaves its workspace zeroed
        model.decode_step()
        torch.cuda.synchronize()
        assert rel(model.x.cpu().double() - x0, (x - x0).numpy()) <= TOL_BF16
        model.cache.copy_(cache0.cuda())


# ---- low-rank KV cache (N3: P:111) -------------------------------------------
def _kvlr_case(dl, orc, s, cache_lens, seed, block_size=16):
    rk = block_ranks(s, 0.4)
    w = gen_block_weights(s, rk, 0, seed)
    S = len(cache_lens)
    max_seq = max(cache_lens) + 1
    lk, lv = rk["k"], rk["v"]
    zk = gen_normal((S, max_seq, lk), 1.0, seed + 1, dtype=torch.bfloat16)
    zv = gen_normal((S, max_seq, lv), 1.0, seed + 2, dtype=torch.bfloat16)
    x = gen_normal((S, s.h), 1.0, seed + 3, dtype=torch.bfloat16)
    mbps = -(-max_seq // block_size)
    nblk = [-(-(L + 1) // block_size) for L in cache_lens]
    num_blocks = sum(nblk) + 7
    perm = np.random.default_rng(seed).permutation(num_blocks).astype(np.int32)
    tables = np.zeros((S, mbps), np.int32)
    k = 0
    for b, nb in enumerate(nblk):
        if b % 3 == 0:                                   # a physically contiguous sequence
            tables[b, :nb] = np.sort(perm[k:k + nb])
        else:
            tables[b, :nb] = perm[k:k + nb]
        k += nb
    cap = sum(nblk) + 2
    kv = dl.LowRankKVCache(lk, lv, s.n_kv_heads * s.head_dim, num_blocks, block_size, S, mbps, cap)
    kv.block_tables.copy_(torch.from_numpy(tables))
    pool = kv.pool.view(num_blocks, block_size, kv.ld_slot)
    pos = kv.slot_pos.view(num_blocks, block_size)
    for b, L in enumerate(cache_lens):                   # history latents into their slots
        for p in range(L):
            blk, off = tables[b, p // block_size], p % block_size
            pool[blk, off, :lk] = zk[b, p].cuda()
            pool[blk, off, kv.zv_off:kv.zv_off + lv] = zv[b, p].cuda()
            pos[blk, off] = p
    nr = kv.prepare(tables, [L + 1 for L in cache_lens])
    cfg = dl.make_block_config(s, rk, max_tokens=S, max_seqs=S)
    wdev = dl.BlockWeights({kk: v.cuda() for kk, v in w.items()})
    ws = torch.zeros(dl.dl_block_workspace(cfg), dtype=torch.uint8, device="cuda")
    cl = torch.tensor(cache_lens, dtype=torch.int32, device="cuda")
    xd = x.cuda()
    dl.dl_decomposed_block_forward_kvlr(cfg, wdev, xd, cl, kv, cl, None, ws)
    torch.cuda.synchronize()
    ref, zk_new, _ = orc.block_decode_lowrank(_oracle_cfg(orc, s, rk), w, x, zk, zv, cache_lens)
    got_new = torch.stack([pool[tables[b, L // block_size], L % block_size, :lk] for b, L in
                           enumerate(cache_lens)]).cpu()
    return rel(xd.cpu().double() - x.double(), ref - x.double().numpy()), rel(got_new, zk_new), nr


@pytest.mark.parametrize("name", ["small", "mha", "opt"])
def test_lowrank_kv_decode_vs_oracle(dl, orc, name):
    s = SMALL if name == "small" else VARIANT_SHAPES[name]
    err, err_new, nr = _kvlr_case(dl, orc, s, [0, 5, 17, 40, 1, 63, 16, 100], seed=81)
    assert nr > 8                                        # scrambled blocks -> several runs
    assert err <= TOL_BF16 and err_new <= TOL_BF16, (err, err_new)


def test_lowrank_kv_decode_batch64(dl, orc):
    """Decode batch 64 (the bench's shape family) with ragged contexts."""
    err, err_new, _ = _kvlr_case(dl, orc, SMALL, [(37 * i) % 130 for i in range(64)], seed=91)
    assert err <= TOL_BF16 and err_new <= TOL_BF16, (err, err_new)


@pytest.mark.parametrize("knob", ["DL_FA_CLUSTER=2", "DL_FA_CLUSTER=8", "DL_ATTN_PREFILL_MMA=1", "DL_GLU_FUSE=0",
                                  "DL_ROPE_EPI=0"])
def test_prefill_attention_variants(knob):
    """The A/B variants of the prefill path against the oracle:
    K/V tiles multicast to 2- and 8-CTA clusters (GQA heads of one KV head), the
    previous mma.sync attention kernel, and the separate SiLU.up kernel instead of
    the gate|up GLU epilogue, the RoPE + cache-append kernel instead of RoPE in the
    q|k|v stage-2 epilogue -- every prefill parity test of this file, run
    against the instrumented library in a subprocess."""
    import os
    import subprocess
    import sys
    name, _, val = knob.partition("=")
    env = dict(os.environ, DL_LIBRARY="ab", **{name: val})
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_parity.py"), "-k",
                        "prefill and not test_prefill_attention_variants"],
                       capture_output=True, text=True, env=env, timeout=900, cwd=root)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
