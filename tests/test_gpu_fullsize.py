"""Parity of exactly what bench.py times.

* One decomposed LLaMA-3-70B @ 40 % layer (P:205 ranks 4916 / 614) at the bench's
  full sizes: decode B = 64 at context 512 through dl_decomposed_stack_forward
  (the bench's call, cross-block residual + norm fusion: two layers sharing the
  weights), every row vs the fp64 oracle; prefill of one 2048-token sequence
  through dl_decomposed_block_forward, sampled rows (the oracle recomputes K / V
  for all tokens, reading c15).
* CUDA-graph replay (the decode step is captured once and
  replayed with fixed buffers): a captured decode step -- full KV cache through the
  stack, and the low-rank KV cache with its two-stage reconstruction -- replayed
  twice with new inputs written into the captured buffers between replays, each
  replay vs the oracle.
"""
import numpy as np
import pytest
import torch

from synthetic import LLAMA3_70B, ModelShape, block_ranks, gen_block_weights, gen_normal

pytestmark = pytest.mark.gpu
TOL_BF16 = 2e-2


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


def _ocfg(orc, s, rk):
    return orc.BlockCfg(s.h, s.n_heads, s.n_kv_heads, s.head_dim, s.m, rk["q"], rk["k"], rk["v"], rk["o"],
                        rk["gate"], rk["up"], rk["down"], rope_theta=s.rope_theta, rms_eps=s.rms_eps,
                        mlp_glu=int(s.glu), use_rope=int(s.rope))


def _to_oracle(c, L):
    # GPU cache [S, Hk, max_seq, d] -> oracle [S, L, Hk * d]
    return c.permute(0, 2, 1, 3)[:, :L].reshape(c.shape[0], L, -1).cpu()


@pytest.fixture(scope="module")
def w70():
    s = LLAMA3_70B
    rk = block_ranks(s, 0.4)
    assert (rk["q"], rk["k"]) == (4916, 614)
    return s, rk, gen_block_weights(s, rk, 4, 0)


@pytest.mark.slow
def test_70b_layer_decode_b64_ctx512_stack(dl, orc, w70):
    """Bench decode shape: 64 sequences at context 512 through the stack call (two
    layers, the residual of layer 0 fused with layer 1's pre-norm); all 64 rows of
    both layers' outputs and layer 0's appended K / V vs the oracle."""
    s, rk, w = w70
    S, L = 64, 512
    x = gen_normal((S, s.h), 1.0, 41, dtype=torch.bfloat16)
    kc = gen_normal((S, s.n_kv_heads, L + 1, s.head_dim), 1.0, 42, dtype=torch.bfloat16)
    vc = gen_normal((S, s.n_kv_heads, L + 1, s.head_dim), 1.0, 43, dtype=torch.bfloat16)
    cfg = dl.make_block_config(s, rk, max_tokens=S, max_seqs=S)
    wd = dl.BlockWeights({k: v.cuda() for k, v in w.items()})
    ws = torch.zeros(dl.dl_block_workspace(cfg), dtype=torch.uint8, device="cuda")
    k0, v0 = kc.cuda(), vc.cuda()
    k1, v1 = kc.cuda(), vc.cuda()
    cl = torch.full((S,), L, dtype=torch.int32, device="cuda")
    xd = x.cuda()
    args = dl.StackArgs([wd, wd], [k0, k1], [v0, v1])
    x1d = xd.clone()
    dl.dl_decomposed_block_forward(cfg, wd, x1d, cl, None, S, dl.DL_DECODE, kc.cuda(), vc.cuda(), cl, None, ws)
    dl.dl_decomposed_stack_forward(cfg, args, xd, cl, None, S, dl.DL_DECODE, cl, None, ws)
    torch.cuda.synchronize()
    oc = _ocfg(orc, s, rk)
    ko, vo = _to_oracle(kc, L + 1), _to_oracle(vc, L + 1)
    x1, kn, vn = orc.block_decode(oc, w, x, ko, vo, [L] * S)
    assert rel(x1d.cpu().double() - x.double(), x1 - x.double().numpy()) <= TOL_BF16
    knew = k0[:, :, L].reshape(S, -1).cpu()
    vnew = v0[:, :, L].reshape(S, -1).cpu()
    assert rel(knew, kn) <= TOL_BF16 and rel(vnew, vn) <= TOL_BF16
    x2, _, _ = orc.block_decode(oc, w, torch.tensor(x1), ko, vo, [L] * S)
    assert rel(xd.cpu().double() - torch.tensor(x1), x2 - x1) <= TOL_BF16


@pytest.mark.slow
def test_70b_layer_prefill_2048_sampled(dl, orc, w70):
    """Bench prefill shape: one 2048-token sequence (pair-kernel GEMMs with the
    DP + stream-K tail, FA2 causal attention); sampled rows vs the oracle."""
    s, rk, w = w70
    T = 2048
    x = gen_normal((T, s.h), 1.0, 44, dtype=torch.bfloat16)
    cfg = dl.make_block_config(s, rk, max_tokens=T, max_seqs=1)
    wd = dl.BlockWeights({k: v.cuda() for k, v in w.items()})
    ws = torch.zeros(dl.dl_block_workspace(cfg), dtype=torch.uint8, device="cuda")
    kc = torch.zeros(1, s.n_kv_heads, T, s.head_dim, dtype=torch.bfloat16, device="cuda")
    vc = torch.zeros_like(kc)
    pos = np.arange(T, dtype=np.int32)
    xd = x.cuda()
    dl.dl_decomposed_block_forward(cfg, wd, xd, torch.from_numpy(pos).cuda(),
                                   torch.tensor([0, T], dtype=torch.int32, device="cuda"), 1, dl.DL_PREFILL, kc, vc,
                                   torch.zeros(1, dtype=torch.int32, device="cuda"), None, ws)
    torch.cuda.synchronize()
    rows = [0, 1, 63, 777, 1500, 2047]
    ref, kref, vref = orc.block_prefill(_ocfg(orc, s, rk), w, x, pos, [0, T], rows=rows)
    got = xd.cpu()[rows].double() - x[rows].double()
    assert rel(got, ref - x[rows].double().numpy()) <= TOL_BF16
    assert rel(_to_oracle(kc, T)[0], kref) <= TOL_BF16 and rel(_to_oracle(vc, T)[0], vref) <= TOL_BF16


# ---- CUDA-graph replay ----------------------------------------------------------
SMALL = ModelShape("g", h=1024, n_heads=8, n_kv_heads=2, head_dim=128, m=2048, n_layers=3, vocab=1000)


def test_graph_replay_decode_step_full_kv(dl, orc):
    """The bench's decode step (embedding -> 3-layer stack -> final norm -> LM head ->
    greedy ids) captured once, replayed for two steps with new ids / cache lengths
    written into the captured buffers: hidden states vs the oracle layer by layer."""
    from paper_2604_17709_b200.model import DecomposedLlama
    s = SMALL
    rk = block_ranks(s, 0.4)
    ws_ = [gen_block_weights(s, rk, 9, li) for li in range(3)]
    S, L = 16, 40
    embed = gen_normal((s.vocab, s.h), 1.0, 90, dtype=torch.bfloat16).cuda()
    lm = gen_normal((s.vocab, s.h), s.h ** -0.5, 91, dtype=torch.bfloat16).cuda()
    model = DecomposedLlama(s, rk, [{k: v.cuda() for k, v in w.items()} for w in ws_], embed,
                            torch.ones(s.h, dtype=torch.bfloat16, device="cuda"), lm, batch=S, max_seq=L + 2)
    assert model.stack is not None
    model.cache.copy_(gen_normal(tuple(model.cache.shape), 1.0, 92, dtype=torch.bfloat16))
    lens0 = torch.tensor([(7 * i) % L for i in range(S)], dtype=torch.int32)
    model.cache_lens.copy_(lens0)
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):          # warm-up (module loads, attributes) outside the capture
        model.decode_step()
    stream.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        model.decode_step()
    for step in range(2):
        ids = (torch.arange(S, dtype=torch.int32) * (31 + 17 * step) + step) % s.vocab
        lens = lens0 + step
        model.ids.copy_(ids)
        model.cache_lens.copy_(lens)
        torch.cuda.synchronize()
        cache0 = model.cache.cpu()
        graph.replay()
        torch.cuda.synchronize()
        x0 = embed.cpu()[ids.long()].double()
        x = x0
        for li, w in enumerate(ws_):
            Lm = int(lens.max()) + 1
            ko = _to_oracle(cache0[li, 0], Lm)
            vo = _to_oracle(cache0[li, 1], Lm)
            x, _, _ = orc.block_decode(_ocfg(orc, s, rk), w, x, ko, vo, lens.numpy())
            x = torch.tensor(x)
        assert rel(model.x.cpu().double() - x0, (x - x0).numpy()) <= TOL_BF16, step
        # the step's greedy ids come from the replayed LM head + argmax
        logits = (torch.nn.functional.rms_norm(model.x.cpu().float(), (s.h,), eps=s.rms_eps).bfloat16().double()
                  @ lm.cpu().double().T)
        top2 = logits.topk(2, dim=1).values
        sure = (top2[:, 0] - top2[:, 1]) > 0.05          # compare ids only where the argmax is not a near tie
        assert torch.equal(model.next_ids.cpu()[sure].long(), logits.argmax(1)[sure])


def test_graph_replay_lowrank_kv_decode(dl, orc):
    """Low-rank KV decode of one block captured once; two steps replayed, the second
    after the host preparation stage re-planned the squeeze for the grown sequences
    (new run list, same device arrays: "dynamic shape but fixed memory address",
    P:222); each replay vs the oracle on the latent history incl. step 1's append."""
    s = SMALL
    rk = block_ranks(s, 0.4)
    w = gen_block_weights(s, rk, 10, 0)
    S, bs = 8, 16
    lens0 = [0, 5, 17, 40, 1, 31, 16, 60]
    max_seq = max(lens0) + 3
    lk, lv = rk["k"], rk["v"]
    mbps = -(-max_seq // bs)
    num_blocks = S * mbps + 5
    perm = np.random.default_rng(3).permutation(num_blocks).astype(np.int32)
    tables = perm[:S * mbps].reshape(S, mbps).copy()
    tables[0] = np.sort(tables[0])
    kv = dl.LowRankKVCache(lk, lv, s.n_kv_heads * s.head_dim, num_blocks, bs, S, mbps, S * mbps)
    kv.block_tables.copy_(torch.from_numpy(tables))
    zk = gen_normal((S, max_seq, lk), 1.0, 101, dtype=torch.bfloat16)
    zv = gen_normal((S, max_seq, lv), 1.0, 102, dtype=torch.bfloat16)
    pool = kv.pool.view(num_blocks, bs, kv.ld_slot)
    pos = kv.slot_pos.view(num_blocks, bs)
    for b, L in enumerate(lens0):
        for p in range(L):
            blk, off = tables[b, p // bs], p % bs
            pool[blk, off, :lk] = zk[b, p].cuda()
            pool[blk, off, kv.zv_off:kv.zv_off + lv] = zv[b, p].cuda()
            pos[blk, off] = p
    cfg = dl.make_block_config(s, rk, max_tokens=S, max_seqs=S)
    wd = dl.BlockWeights({k: v.cuda() for k, v in w.items()})
    ws = torch.zeros(dl.dl_block_workspace(cfg), dtype=torch.uint8, device="cuda")
    cl = torch.tensor(lens0, dtype=torch.int32, device="cuda")
    xd = torch.zeros(S, s.h, dtype=torch.bfloat16, device="cuda")
    kv.prepare(tables, [L + 1 for L in lens0])
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        dl.dl_decomposed_block_forward_kvlr(cfg, wd, xd, cl, kv, cl, None, ws)
    stream.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        dl.dl_decomposed_block_forward_kvlr(cfg, wd, xd, cl, kv, cl, None, ws)
    oc = _ocfg(orc, s, rk)
    lens = list(lens0)
    for step in range(2):
        x = gen_normal((S, s.h), 1.0, 200 + step, dtype=torch.bfloat16)
        xd.copy_(x)
        cl.copy_(torch.tensor(lens, dtype=torch.int32))
        kv.prepare(tables, [L + 1 for L in lens])        # host planning stage, outside the replay
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        ref, zk_new, zv_new = orc.block_decode_lowrank(oc, w, x, zk, zv, lens)
        assert rel(xd.cpu().double() - x.double(), ref - x.double().numpy()) <= TOL_BF16, step
        for b, L in enumerate(lens):                      # the history grows by the appended latents
            zk[b, L] = torch.from_numpy(zk_new[b]).bfloat16()
            zv[b, L] = torch.from_numpy(zv_new[b]).bfloat16()
            got = pool[tables[b, L // bs], L % bs, :lk].cpu()
            assert rel(got, zk_new[b]) <= TOL_BF16
        lens = [L + 1 for L in lens]


@pytest.mark.parametrize("chunks", [2, 4])
def test_prefill_chunk_wavefront(dl, orc, chunks):
    """Chunked prefill wavefront (model.py `_prefill_wavefront`): the sequence split into
    `chunks` chunks, block (layer i, chunk c) on chunk c's stream after block (i, c - 1),
    captured in a CUDA graph and replayed.  Every token's final hidden state vs the
    oracle's one-shot causal prefill of the whole sequence, layer by layer (chunks
    continue each other's cached prefix: include/dl.h, PREFILL)."""
    from paper_2604_17709_b200.model import DecomposedLlama
    s = SMALL
    rk = block_ranks(s, 0.4)
    ws_ = [gen_block_weights(s, rk, 11, li) for li in range(3)]
    T = 384
    embed = gen_normal((s.vocab, s.h), 1.0, 95, dtype=torch.bfloat16).cuda()
    lm = gen_normal((s.vocab, s.h), s.h ** -0.5, 96, dtype=torch.bfloat16).cuda()
    model = DecomposedLlama(s, rk, [{k: v.cuda() for k, v in w.items()} for w in ws_], embed,
                            torch.ones(s.h, dtype=torch.bfloat16, device="cuda"), lm, batch=1, max_seq=8,
                            prefill_tokens=T, prefill_chunks=chunks)
    ids = (torch.arange(T, dtype=torch.int32) * 37 + 5) % s.vocab
    model.pre_ids.copy_(ids)
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        model.prefill_step()
    stream.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        model.prefill_step()
    model.pre_x.zero_()
    torch.cuda.synchronize()
    graph.replay()
    torch.cuda.synchronize()
    x0 = embed.cpu()[ids.long()].double()
    x = x0
    pos = np.arange(T, dtype=np.int32)
    cu = np.array([0, T], dtype=np.int32)
    for w in ws_:
        x, _, _ = orc.block_prefill(_ocfg(orc, s, rk), w, x, pos, cu)
        x = torch.tensor(x)
    assert rel(model.pre_x.cpu().double() - x0, (x - x0).numpy()) <= TOL_BF16
