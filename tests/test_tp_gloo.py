"""World-size-2 CPU (gloo) coverage of the tensor-parallel host logic
(-m "not gpu").  Each process plays one TP rank:

* it asks the C-ABI planner (dl_tp_plan) for its share of the concatenated
  group rank ("concatenated and then evenly split"),
* slices its factor shards exactly as dl_tp_shard_factors does (rows of B,
  columns of A per segment),
* computes its partial with the fp64 oracle and reduces over gloo
  (all-reduce), or lays the q|k|v partial out rank-major by head and
  reduce-scatters it (the build's RS step), then all-gathers local
  attention outputs and un-permutes them,

and checks the result against the unsharded oracle.  The CUDA kernels are not
involved (no GPU here); this pins the partition / layout logic the kernels
implement.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import paper_2604_17709_b200 as dl
        rng = np.random.default_rng(0)        # identical full factors on every rank
        T, h, hkv, H, Hk, d = 5, 64, 32, 4, 2, 16
        ranks = [37, 11, 13]                 # odd ranks: uneven split
        mats = [(h, ranks[0]), (hkv, ranks[1]), (hkv, ranks[2])]
        A = [rng.standard_normal((m, k)) for m, k in mats]
        B = [rng.standard_normal((k, h)) for _, k in mats]
        X = rng.standard_normal((T, h))
        full = [oracle.lowrank_linear(X, a, b) for a, b in zip(A, B)]

        beg, lens, kloc = dl.dl_tp_plan(ranks, world, rank)
        parts = []
        for g in range(3):
            a_s = A[g][:, beg[g]:beg[g] + lens[g]]
            b_s = B[g][beg[g]:beg[g] + lens[g], :]
            parts.append(oracle.lowrank_linear(X, a_s, b_s) if lens[g] else np.zeros((T, mats[g][0])))
        # 1) all-reduce of the concatenated partial == unsharded result
        cat = torch.tensor(np.concatenate(parts, 1))
        dist.all_reduce(cat)
        err_ar = float((cat - torch.tensor(np.concatenate(full, 1))).abs().max())

        # 2) reduce-scatter by head: [P][T][W], slab = local q | local k | local v heads
        rpr = [h // world, hkv // world, hkv // world]
        slab = sum(rpr)
        lay = torch.zeros(world, T, slab, dtype=torch.float64)
        off = 0
        for g in range(3):
            for owner in range(world):
                lay[owner, :, off:off + rpr[g]] = torch.tensor(parts[g][:, owner * rpr[g]:(owner + 1) * rpr[g]])
            off += rpr[g]
        mine = torch.zeros(T, slab, dtype=torch.float64)
        dist.reduce_scatter_tensor(mine, lay.reshape(world * T, slab))
        exp = np.concatenate([full[g][:, rank * rpr[g]:(rank + 1) * rpr[g]] for g in range(3)], 1)
        err_rs = float((mine - torch.tensor(exp)).abs().max())
        # local heads: q heads [rank*H/P, ...) read kv heads [rank*Hk/P, ...) (GQA map)
        qh = list(range(rank * H // world, (rank + 1) * H // world))
        kvh = sorted({g * Hk // H for g in qh})
        ok_heads = kvh == list(range(rank * Hk // world, (rank + 1) * Hk // world))

        # 3) all-gather of local attention outputs + un-permute == full rows
        att_full = rng.standard_normal((T, h))
        local = torch.tensor(att_full[:, rank * h // world:(rank + 1) * h // world]).contiguous()
        gathered = torch.zeros(world * T, h // world, dtype=torch.float64)
        dist.all_gather_into_tensor(gathered, local)
        gathered = gathered.view(world, T, h // world)
        unperm = gathered.permute(1, 0, 2).reshape(T, h)
        err_ag = float((unperm - torch.tensor(att_full)).abs().max())
        q.put((rank, err_ar, err_rs, err_ag, ok_heads, kloc))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", repr(e)))


@pytest.mark.timeout(300)
def test_tp_world2_gloo():
    from paper_2604_17709_b200 import build
    build.build()
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
    klocs = 0
    for r in res:
        assert r[1] != "error", r
        _, err_ar, err_rs, err_ag, ok_heads, kloc = r
        assert err_ar < 1e-10 and err_rs < 1e-10 and err_ag == 0.0 and ok_heads
        klocs += kloc
    assert klocs == 37 + 11 + 13


def _deinfer_worker(rank, world, port, q):
    """DeInfer layout (Fig. 3) host logic: concat-split B rows per
    dl_tp_plan, latent all-gather + un-permute, row-sharded A; input-sharded
    B + latent all-reduce with the full A."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import paper_2604_17709_b200 as dl
        rng = np.random.default_rng(1)
        T, h, hkv = 4, 64, 32
        ranks = [37, 11, 13]
        mats = [(h, ranks[0]), (hkv, ranks[1]), (hkv, ranks[2])]
        A = [rng.standard_normal((m, k)) for m, k in mats]
        B = [rng.standard_normal((k, h)) for _, k in mats]
        X = rng.standard_normal((T, h))
        full = [oracle.lowrank_linear(X, a, b) for a, b in zip(A, B)]
        # first sub-layer: the rank's rows of the concatenated B
        beg, lens, kloc = dl.dl_tp_plan(ranks, world, rank)
        Bcat = np.concatenate(B, 0)
        L = Bcat.shape[0]
        start = sum(dl.dl_tp_plan(ranks, world, r)[2] for r in range(rank))
        mine = oracle.matmul(X, Bcat[start:start + kloc].T)             # latent slice [T x kloc]
        slot = -(-L // world)
        send = torch.zeros(T, slot, dtype=torch.float64)
        send[:, :kloc] = torch.tensor(mine)
        recv = [torch.zeros_like(send) for _ in range(world)]
        dist.all_gather(recv, send)
        kl = [dl.dl_tp_plan(ranks, world, r)[2] for r in range(world)]
        Z = np.concatenate([recv[r][:, :kl[r]].numpy() for r in range(world)], 1)   # un-permute
        off = np.concatenate([[0], np.cumsum(ranks)])
        err1 = 0.0
        for g, (m, k) in enumerate(mats):
            rows = slice(rank * m // world, (rank + 1) * m // world)
            yl = oracle.matmul(Z[:, off[g]:off[g + 1]], A[g][rows].T)
            err1 = max(err1, float(np.abs(yl - full[g][:, rows]).max()))
        # second sub-layer (o): input-column shard of B, latent reduce-sum, full A
        Ao, Bo = rng.standard_normal((h, 29)), rng.standard_normal((29, h))
        cols = slice(rank * h // world, (rank + 1) * h // world)
        part = torch.tensor(oracle.matmul(X[:, cols], Bo[:, cols].T))
        dist.all_reduce(part)
        yo = oracle.matmul(part.numpy(), Ao.T)
        err2 = float(np.abs(yo - oracle.lowrank_linear(X, Ao, Bo)).max())
        q.put((rank, err1, err2, kloc))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", repr(e)))


@pytest.mark.timeout(300)
def test_deinfer_layout_world2_gloo():
    from paper_2604_17709_b200 import build
    build.build()
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_deinfer_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
    assert sum(r[3] for r in res if r[1] != "error") == 37 + 11 + 13, res
    for r in res:
        assert r[1] != "error", r
        assert r[1] < 1e-10 and r[2] < 1e-10, r
