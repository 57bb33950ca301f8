"""P > 1 parity of the tensor-parallel CUDA path on ONE GPU.

An in-process group communicator (include/dl.h: dl_comm_create_group) runs
P ranks in one process, each rank in its own host thread with its own stream
and its own weight shards / workspace / KV cache; the collectives are the
library's peer-memory kernels, so every reduce-scatter slab with owner > 0,
every all-reduce sum and every all-gather un-permute is really executed by
CUDA code with P contributors.  Results are compared with the fp64 oracle's
sharded evaluation (`world=P`, PAPER.md:121-123 reduce-sum of the rank
partials; PAPER.md:174-183 DeInfer low-rank communication), and the ranks'
copies of the replicated residual stream must be bit-identical.
"""
import numpy as np
import pytest
import torch

from synthetic import ModelShape, block_ranks, gen_block_weights, gen_factor_pair, gen_normal

pytestmark = pytest.mark.gpu
TOL_BF16 = 2e-2
TOL_F32 = 1e-5


def rel(a, b):
    a = np.asarray(a.detach().cpu().double().numpy() if isinstance(a, torch.Tensor) else a, dtype=np.float64)
    b = np.asarray(b.detach().cpu().double().numpy() if isinstance(b, torch.Tensor) else b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def dl():
    import paper_2604_17709_b200 as dl
    from paper_2604_17709_b200 import build
    build.build()
    dl.load()
    assert dl.dl_device_ok(), "needs an sm_100 GPU"
    return dl


def group(dl, P, sym=8 << 20):
    return dl.Comm.group(P, sym)


def test_window_bytes_query(dl):
    """dl_block_window_bytes: rank-parallel configs need X + Y + G in the window; 0 for DeInfer."""
    s = SHAPE
    rk = block_ranks(s, 0.4)
    cfg = dl.make_block_config(s, rk, max_tokens=64, max_seqs=64)
    W = (s.h + 2 * s.h_kv) // 4
    exp = 64 * max(W, 2 * s.m) * 2 + 2 * 64 * s.h * 2
    assert dl.dl_block_window_bytes(cfg, 4) == exp
    assert dl.dl_block_window_bytes(dl.make_block_config(s, rk, 64, 64, layout=1), 4) == 0


def same_stream(layout, a, b):
    """Rank-parallel: every rank adds the same all-reduced bytes -> bit-identical
    residual streams.  DeInfer: the replicated second-sub-layer up-projection runs
    on every rank with stream-K (atomic, order-nondeterministic) accumulation, so
    the ranks' copies agree to rounding, not bitwise (reading c11)."""
    if layout == 0:
        return torch.equal(a, b)
    return rel(a, b) <= 4e-3


# ---- dl_lowrank_linear with a communicator -------------------------------------
@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("T", [1, 8, 40, 300])
def test_linear_reduce_modes_multirank(dl, orc, P, T):
    """Rank k-shards from dl_tp_shard_factors; ALLREDUCE = the full A(Bx) on every
    rank (bit-identical), SCATTER = rank r's m/P slab of it, NONE = the rank's own
    partial A[:, K_r](B[K_r, :] x) with K_r from the oracle's independent planner."""
    m, n, k = 512, 384, 200
    X = gen_normal((T, n), 1.0, 300 + T, dtype=torch.bfloat16)
    A, B = gen_factor_pair(m, n, k, 301 + P, dtype=torch.bfloat16)
    full = orc.lowrank_linear(X, A, B)
    comms = group(dl, P)

    def body(r, s):
        A_sh, B_sh, lens = dl.dl_tp_shard_factors([A.cuda()], [B.cuda()], P, r)
        Xd = X.cuda()
        out = {}
        for red, mo in ((dl.DL_REDUCE_ALLREDUCE, m), (dl.DL_REDUCE_SCATTER, m // P), (dl.DL_REDUCE_NONE, m)):
            Y = torch.zeros(T, mo, dtype=torch.bfloat16, device="cuda")
            dl.dl_lowrank_linear(Xd, A_sh[0], B_sh, Y, comm=comms[r], reduce=red)
            out[red] = Y
        # accumulate (Y += A(Bx)) through the all-reduce
        Y0 = gen_normal((T, m), 1.0, 77, dtype=torch.bfloat16).cuda()
        dl.dl_lowrank_linear(Xd, A_sh[0], B_sh, Y0, accumulate=True, comm=comms[r], reduce=dl.DL_REDUCE_ALLREDUCE)
        out["acc"] = Y0
        return {kk: v.cpu() for kk, v in out.items()}

    res = dl.run_ranks(body, P)
    for c in comms:
        c.close()
    Y0 = gen_normal((T, m), 1.0, 77, dtype=torch.bfloat16).double().numpy()
    for r in range(P):
        assert rel(res[r][dl.DL_REDUCE_ALLREDUCE], full) <= TOL_BF16
        assert torch.equal(res[r][dl.DL_REDUCE_ALLREDUCE], res[0][dl.DL_REDUCE_ALLREDUCE])
        sl = slice(r * m // P, (r + 1) * m // P)
        assert rel(res[r][dl.DL_REDUCE_SCATTER], full[:, sl]) <= TOL_BF16
        b0, ln, _ = orc.shard_range(k, P, r, 1)
        part = orc.lowrank_linear(X, A[:, b0:b0 + ln], B[b0:b0 + ln])
        assert rel(res[r][dl.DL_REDUCE_NONE], part) <= TOL_BF16
        assert rel(res[r]["acc"].double().numpy() - Y0, full) <= TOL_BF16


@pytest.mark.parametrize("P", [2, 3])
def test_linear_fp32_allreduce_multirank(dl, orc, P):
    """fp32 SIMT chain with a collective (true FFMA, fp32 all-reduce): 1e-5."""
    T, m, n, k = 4, 256, 256, 64
    X = gen_normal((T, n), 1.0, 5, dtype=torch.float32)
    A, B = gen_factor_pair(m, n, k, 6, dtype=torch.float32)
    full = orc.lowrank_linear(X, A, B)
    comms = group(dl, P)

    def body(r, s):
        A_sh, B_sh, _ = dl.dl_tp_shard_factors([A.cuda()], [B.cuda()], P, r)
        Y = torch.zeros(T, m, device="cuda")
        dl.dl_lowrank_linear(X.cuda(), A_sh[0], B_sh, Y, comm=comms[r], reduce=dl.DL_REDUCE_ALLREDUCE)
        Ys = torch.zeros(T, m // P if m % (32 * P) == 0 else m, device="cuda")
        if m % (32 * P) == 0:
            dl.dl_lowrank_linear(X.cuda(), A_sh[0], B_sh, Ys, comm=comms[r], reduce=dl.DL_REDUCE_SCATTER)
        return Y.cpu(), Ys.cpu()

    res = dl.run_ranks(body, P)
    for c in comms:
        c.close()
    for r in range(P):
        assert rel(res[r][0], full) <= TOL_F32
        if m % (32 * P) == 0:
            assert rel(res[r][1], full[:, r * m // P:(r + 1) * m // P]) <= TOL_F32


# ---- rank-shard planner, world > 1, byte-exact ------------------------------------
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_shard_factors_byte_exact_multirank(dl, orc, world):
    """dl_tp_shard_factors / dl_deinfer_shard_factors copies equal the slices the
    oracle's planner names (concatenated group range split evenly)."""
    ranks = [300, 70, 70]
    ms = [512, 128, 128]
    n = 384
    As = [gen_normal((mm, rk), 1.0, 10 + i, dtype=torch.bfloat16) for i, (mm, rk) in enumerate(zip(ms, ranks))]
    Bs = [gen_normal((rk, n), 1.0, 20 + i, dtype=torch.bfloat16) for i, rk in enumerate(ranks)]
    Bcat = torch.cat(Bs, 0)
    R = sum(ranks)
    offs = np.cumsum([0] + ranks)
    for r in range(world):
        A_sh, B_sh, lens = dl.dl_tp_shard_factors([a.cuda() for a in As], [b.cuda() for b in Bs], world, r)
        b0, ln, _ = orc.shard_range(R, world, r, 1)
        assert torch.equal(B_sh.cpu(), Bcat[b0:b0 + ln])
        for g in range(3):
            lo, hi = max(b0, offs[g]), min(b0 + ln, offs[g + 1])
            exp = As[g][:, max(lo - offs[g], 0):max(hi - offs[g], 0)] if hi > lo else As[g][:, :0]
            assert lens[g] == exp.shape[1]
            assert torch.equal(A_sh[g].cpu(), exp)
        if all(mm % world == 0 for mm in ms):
            A1, B1 = dl.dl_deinfer_shard_factors(1, [a.cuda() for a in As], [b.cuda() for b in Bs], world, r)
            assert torch.equal(B1.cpu(), Bcat[b0:b0 + ln])
            for g in range(3):
                ml = ms[g] // world
                assert torch.equal(A1[g].cpu(), As[g][r * ml:(r + 1) * ml])
        if n % world == 0:
            A2, B2 = dl.dl_deinfer_shard_factors(2, [As[0].cuda()], [Bs[0].cuda()], world, r)
            nl = n // world
            assert torch.equal(B2.cpu(), Bs[0][:, r * nl:(r + 1) * nl])
            assert torch.equal(A2[0].cpu(), As[0])


# ---- decomposed block, P ranks ----------------------------------------------------
# GQA like LLaMA-3-70B (8 q heads per kv head... here 2 per kv head so P = 8 still
# leaves a whole kv head per rank), scaled so the fp64 oracle stays fast.
SHAPE = ModelShape("mr", h=2048, n_heads=16, n_kv_heads=8, head_dim=128, m=4096, n_layers=2, vocab=10)


def _ocfg(orc, s, rk, layout):
    return orc.BlockCfg(s.h, s.n_heads, s.n_kv_heads, s.head_dim, s.m, rk["q"], rk["k"], rk["v"], rk["o"],
                        rk["gate"], rk["up"], rk["down"], rope_theta=s.rope_theta, rms_eps=s.rms_eps,
                        mlp_glu=int(s.glu), use_rope=int(s.rope), layout=layout)


@pytest.fixture(scope="module")
def block_case():
    s = SHAPE
    rk = block_ranks(s, 0.4)
    w = gen_block_weights(s, rk, 3, 0)
    w2 = gen_block_weights(s, rk, 3, 1)
    return s, rk, w, w2


def _run_block(dl, s, rk, w, layout, P, mode, T=None, lens=None, w2=None, window=8 << 20):
    """Runs one block (or a 2-block stack) on P group ranks; returns per-rank
    (x_out, k_cache, v_cache) on the host.  window: the group's symmetric window;
    a window >= dl_block_window_bytes selects the fused epilogue collectives of
    the skinny rank-parallel path, a smaller one the collective kernels."""
    comms = group(dl, P, window)
    hk = s.n_kv_heads // P

    def body(r, st):
        wd = dl.BlockWeights({a: b.cuda() for a, b in w.items()}, world=P, rank=r, layout=layout)
        wd2 = dl.BlockWeights({a: b.cuda() for a, b in w2.items()}, world=P, rank=r, layout=layout) if w2 else None
        if mode == "prefill":
            x = gen_normal((T, s.h), 1.0, 500 + T, dtype=torch.bfloat16).cuda()
            cfg = dl.make_block_config(s, rk, max_tokens=T, max_seqs=1, layout=layout)
            ws = torch.zeros(dl.dl_block_workspace(cfg, P), dtype=torch.uint8, device="cuda")
            kc = torch.zeros(1, hk, T, s.head_dim, dtype=torch.bfloat16, device="cuda")
            vc = torch.zeros_like(kc)
            pos = torch.arange(T, dtype=torch.int32, device="cuda")
            cu = torch.tensor([0, T], dtype=torch.int32, device="cuda")
            dl.dl_decomposed_block_forward(cfg, wd, x, pos, cu, 1, dl.DL_PREFILL, kc, vc,
                                           torch.zeros(1, dtype=torch.int32, device="cuda"), comms[r], ws)
            return x.cpu(), kc.cpu(), vc.cpu()
        S, L = len(lens), max(lens) + 1
        x0 = gen_normal((S, s.h), 1.0, 600, dtype=torch.bfloat16).cuda()
        kfull = gen_normal((S, s.n_kv_heads, L, s.head_dim), 1.0, 601, dtype=torch.bfloat16)
        vfull = gen_normal((S, s.n_kv_heads, L, s.head_dim), 1.0, 602, dtype=torch.bfloat16)
        kc = kfull[:, r * hk:(r + 1) * hk].contiguous().cuda()
        vc = vfull[:, r * hk:(r + 1) * hk].contiguous().cuda()
        cl = torch.tensor(lens, dtype=torch.int32, device="cuda")
        cfg = dl.make_block_config(s, rk, max_tokens=S, max_seqs=S, layout=layout)
        ws = torch.zeros(dl.dl_block_workspace(cfg, P), dtype=torch.uint8, device="cuda")
        if mode == "stack":
            kc2, vc2 = kc.clone(), vc.clone()
            args = dl.StackArgs([wd, wd2], [kc, kc2], [vc, vc2])
            x = x0.clone()
            dl.dl_decomposed_stack_forward(cfg, args, x, cl, None, S, dl.DL_DECODE, cl, comms[r], ws)
            return x.cpu(), kc.cpu(), kc2.cpu()
        outs = []
        for _ in range(2):   # twice: reduction / collective buffers are left zeroed
            x = x0.clone()
            k1, v1 = kc.clone(), vc.clone()
            dl.dl_decomposed_block_forward(cfg, wd, x, cl, None, S, dl.DL_DECODE, k1, v1, cl, comms[r], ws)
            outs.append(x)
        return outs[0].cpu(), k1.cpu(), v1.cpu(), outs[1].cpu()

    res = dl.run_ranks(body, P)
    for c in comms:
        c.close()
    return res


@pytest.mark.parametrize("layout,fused", [(0, True), (0, False), (1, False)])
@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("T", [40, 300])
def test_block_prefill_multirank(dl, orc, block_case, layout, fused, P, T):
    """Prefill (skinny stream-K path at T = 40, whole-tile path at T = 300) with P
    ranks: RS slabs of every owner, attention all-gather, AR sums (rank-parallel) /
    latent all-gather + latent all-reduce (DeInfer); K/V of each rank's heads."""
    if T > 256 and fused:
        pytest.skip("the wide prefill path always uses the collective kernels")
    s, rk, w, _ = block_case
    res = _run_block(dl, s, rk, w, layout, P, "prefill", T=T, window=(8 << 20) if fused else 256)
    x = gen_normal((T, s.h), 1.0, 500 + T, dtype=torch.bfloat16)
    ref, kref, vref = orc.block_prefill(_ocfg(orc, s, rk, layout), w, x, np.arange(T), [0, T], world=P)
    d0 = ref - x.double().numpy()
    hk, dd = s.n_kv_heads // P, s.head_dim
    for r in range(P):
        xr, kc, vc = res[r]
        assert same_stream(layout, xr, res[0][0]), "ranks' residual streams differ"
        assert rel(xr.double() - x.double(), d0) <= TOL_BF16
        kr = kc[0].permute(1, 0, 2).reshape(T, hk * dd)
        vr = vc[0].permute(1, 0, 2).reshape(T, hk * dd)
        assert rel(kr, kref[:, r * hk * dd:(r + 1) * hk * dd]) <= TOL_BF16
        assert rel(vr, vref[:, r * hk * dd:(r + 1) * hk * dd]) <= TOL_BF16


@pytest.mark.parametrize("layout,fused", [(0, True), (0, False), (1, False)])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_block_decode_multirank(dl, orc, block_case, layout, fused, P):
    """Decode of 8 sequences with mixed cache lengths (empty included), called twice
    (the window / collective buffers must be left zeroed).  fused: the rank-parallel
    stage-2 epilogues reduce straight into the ranks' windows."""
    s, rk, w, _ = block_case
    lens = [5, 0, 17, 3, 9, 1, 30, 12]
    res = _run_block(dl, s, rk, w, layout, P, "decode", lens=lens, window=(8 << 20) if fused else 256)
    S, L = len(lens), max(lens) + 1
    x = gen_normal((S, s.h), 1.0, 600, dtype=torch.bfloat16)
    kf = gen_normal((S, s.n_kv_heads, L, s.head_dim), 1.0, 601, dtype=torch.bfloat16)
    vf = gen_normal((S, s.n_kv_heads, L, s.head_dim), 1.0, 602, dtype=torch.bfloat16)
    ko = kf.permute(0, 2, 1, 3).reshape(S, L, -1)
    vo = vf.permute(0, 2, 1, 3).reshape(S, L, -1)
    ref, kn, vn = orc.block_decode(_ocfg(orc, s, rk, layout), w, x, ko, vo, lens, world=P)
    d0 = ref - x.double().numpy()
    hk, dd = s.n_kv_heads // P, s.head_dim
    for r in range(P):
        x1, kc, vc, x2 = res[r]
        assert same_stream(layout, x1, res[0][0]) and same_stream(layout, x2, res[0][3])
        assert rel(x1.double() - x.double(), d0) <= TOL_BF16
        assert rel(x2.double() - x.double(), d0) <= TOL_BF16   # the second call: buffers were left zeroed
        knew = torch.stack([kc[i, :, lens[i]] for i in range(S)]).reshape(S, hk * dd)
        vnew = torch.stack([vc[i, :, lens[i]] for i in range(S)]).reshape(S, hk * dd)
        assert rel(knew, kn[:, r * hk * dd:(r + 1) * hk * dd]) <= TOL_BF16
        assert rel(vnew, vn[:, r * hk * dd:(r + 1) * hk * dd]) <= TOL_BF16


@pytest.mark.parametrize("layout,fused", [(0, True), (0, False), (1, False)])
@pytest.mark.parametrize("P", [2, 8])
def test_stack_decode_multirank(dl, orc, block_case, layout, fused, P):
    """Two-block stack (cross-block residual + norm fusion after the last all-reduce)."""
    s, rk, w, w2 = block_case
    lens = [4, 11, 0, 7]
    res = _run_block(dl, s, rk, w, layout, P, "stack", lens=lens, w2=w2, window=(8 << 20) if fused else 256)
    S, L = len(lens), max(lens) + 1
    x = gen_normal((S, s.h), 1.0, 600, dtype=torch.bfloat16)
    kf = gen_normal((S, s.n_kv_heads, L, s.head_dim), 1.0, 601, dtype=torch.bfloat16)
    vf = gen_normal((S, s.n_kv_heads, L, s.head_dim), 1.0, 602, dtype=torch.bfloat16)
    ko = kf.permute(0, 2, 1, 3).reshape(S, L, -1)
    vo = vf.permute(0, 2, 1, 3).reshape(S, L, -1)
    oc = _ocfg(orc, s, rk, layout)
    x1, _, _ = orc.block_decode(oc, w, x, ko, vo, lens, world=P)
    x2, _, _ = orc.block_decode(oc, w2, x1, ko, vo, lens, world=P)
    for r in range(P):
        assert same_stream(layout, res[r][0], res[0][0])
        assert rel(res[r][0].double() - x.double(), x2 - x.double().numpy()) <= TOL_BF16


def test_block_relu_deinfer_multirank(dl, orc):
    """Non-GLU ReLU MLP (OPT family, no RoPE) in the DeInfer layout at P = 2."""
    s = ModelShape("mr-relu", h=1024, n_heads=8, n_kv_heads=8, head_dim=128, m=2048, n_layers=1, vocab=10,
                   glu=False, rope=False)
    rk = block_ranks(s, 0.4)
    w = gen_block_weights(s, rk, 4, 0)
    for mode, T in (("prefill", 40), ("prefill", 300)):
        res = _run_block(dl, s, rk, w, 1, 2, mode, T=T)
        x = gen_normal((T, s.h), 1.0, 500 + T, dtype=torch.bfloat16)
        ref, _, _ = orc.block_prefill(_ocfg(orc, s, rk, 1), w, x, np.arange(T), [0, T], world=2)
        for r in range(2):
            assert rel(res[r][0].double() - x.double(), ref - x.double().numpy()) <= TOL_BF16


@pytest.mark.parametrize("mode", ["prefill", "decode"])
@pytest.mark.parametrize("ranks", [{"k": 1}, {"v": 2}, {"up": 1}])
def test_block_tiny_segment_tp1(dl, orc, mode, ranks):
    """Regression (found by the P = 4 runs, whose balanced split hands a rank a
    1-row piece of a segment): a group with a segment of rank 1-2 gives single-k-
    block stream-K tiles; more than 8 such jobs inside a CTA's first 9 units used to
    deadlock the GEMM producer against its own deferred (pre-PDL-wait) loads."""
    s = SHAPE
    rk = dict(block_ranks(s, 0.4), **ranks)
    w = gen_block_weights(s, rk, 5, 0)
    res = _run_block_single(dl, s, rk, w, mode)
    oc = _ocfg(orc, s, rk, 0)
    if mode == "prefill":
        T = 40
        x = gen_normal((T, s.h), 1.0, 500 + T, dtype=torch.bfloat16)
        ref, _, _ = orc.block_prefill(oc, w, x, np.arange(T), [0, T])
    else:
        lens = [5, 0, 17, 3, 9, 1, 30, 12]
        S, L = len(lens), max(lens) + 1
        x = gen_normal((S, s.h), 1.0, 600, dtype=torch.bfloat16)
        kf = gen_normal((S, s.n_kv_heads, L, s.head_dim), 1.0, 601, dtype=torch.bfloat16)
        vf = gen_normal((S, s.n_kv_heads, L, s.head_dim), 1.0, 602, dtype=torch.bfloat16)
        ref, _, _ = orc.block_decode(oc, w, x, kf.permute(0, 2, 1, 3).reshape(S, L, -1),
                                     vf.permute(0, 2, 1, 3).reshape(S, L, -1), lens)
    assert rel(res.double() - x.double(), ref - x.double().numpy()) <= TOL_BF16


def _run_block_single(dl, s, rk, w, mode):
    wd = dl.BlockWeights({a: b.cuda() for a, b in w.items()})
    if mode == "prefill":
        T = 40
        x = gen_normal((T, s.h), 1.0, 500 + T, dtype=torch.bfloat16).cuda()
        cfg = dl.make_block_config(s, rk, max_tokens=T, max_seqs=1)
        ws = torch.zeros(dl.dl_block_workspace(cfg), dtype=torch.uint8, device="cuda")
        kc = torch.zeros(1, s.n_kv_heads, T, s.head_dim, dtype=torch.bfloat16, device="cuda")
        dl.dl_decomposed_block_forward(cfg, wd, x, torch.arange(T, dtype=torch.int32, device="cuda"),
                                       torch.tensor([0, T], dtype=torch.int32, device="cuda"), 1, dl.DL_PREFILL,
                                       kc, torch.zeros_like(kc), torch.zeros(1, dtype=torch.int32, device="cuda"),
                                       None, ws)
    else:
        lens = [5, 0, 17, 3, 9, 1, 30, 12]
        S, L = len(lens), max(lens) + 1
        x = gen_normal((S, s.h), 1.0, 600, dtype=torch.bfloat16).cuda()
        kc = gen_normal((S, s.n_kv_heads, L, s.head_dim), 1.0, 601, dtype=torch.bfloat16).cuda()
        vc = gen_normal((S, s.n_kv_heads, L, s.head_dim), 1.0, 602, dtype=torch.bfloat16).cuda()
        cl = torch.tensor(lens, dtype=torch.int32, device="cuda")
        cfg = dl.make_block_config(s, rk, max_tokens=S, max_seqs=S)
        ws = torch.zeros(dl.dl_block_workspace(cfg), dtype=torch.uint8, device="cuda")
        dl.dl_decomposed_block_forward(cfg, wd, x, cl, None, S, dl.DL_DECODE, kc, vc, cl, None, ws)
    torch.cuda.synchronize()
    return x.cpu()
