"""C-ABI checks that run without a GPU (-m "not gpu"):
the library builds/loads, exports every symbol include/dl.h declares, the
host-side planner agrees with the oracle's independent range computation,
argument validation rejects bad calls before touching the device, and a
valid compute call on a GPU-less host fails loudly (no CPU fallback).
"""
import ctypes
import os
import re

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2604_17709_b200 import build
    build.build()
    import paper_2604_17709_b200 as dl
    dl.load()
    return dl


def header_functions():
    src = open(os.path.join(ROOT, "include", "dl.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dl_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_header_symbol(lib):
    so = ctypes.CDLL(lib._lib.LIB_PATH)
    names = header_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(so, n), f"libdl.so does not export {n}"
    assert set(names) == set(lib.EXPORTS)


def test_version(lib):
    assert lib.dl_version() == 100


@pytest.mark.parametrize("ranks", [[4916, 614, 614], [4916, 4916], [4916], [3277, 819, 819], [7, 5, 3], [64]])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_plan_matches_oracle_concat_split(lib, orc, ranks, world):
    """dl_tp_plan: concatenate the segment ranks, split evenly, map back."""
    R = sum(ranks)
    if R < world:
        pytest.skip("R < world")
    seen = [0] * R
    for r in range(world):
        beg, lens, kloc = lib.dl_tp_plan(ranks, world, r)
        b0, l0, _ = orc.shard_range(R, world, r, 1)          # independent oracle plan
        assert kloc == l0
        off = 0
        got = []
        for g, rk in enumerate(ranks):
            for j in range(lens[g]):
                got.append(off + beg[g] + j)
            off += rk
        assert got == list(range(b0, b0 + l0))
        for i in got:
            seen[i] += 1
    assert all(s == 1 for s in seen)


def test_plan_70b_qkv_tp8(lib):
    beg, lens, kloc = lib.dl_tp_plan([4916, 614, 614], 8, 6)
    assert kloc == 768 and lens == [308, 460, 0] and beg[:2] == [4608, 0]
    beg, lens, kloc = lib.dl_tp_plan([4916, 614, 614], 8, 7)
    assert kloc == 768 and lens == [0, 154, 614] and beg[1:] == [460, 0]


def test_plan_strict_rejects_uneven(lib):
    with pytest.raises(lib.DLError) as e:
        lib.dl_tp_plan([614], 8, 0, strict=True)
    assert e.value.name == "DL_ERR_PARTITION"
    with pytest.raises(lib.DLError):
        lib.dl_tp_plan([3], 4, 0)          # fewer ranks than world


def _call_linear(lib, T=4, m=256, n=256, k=64, ldx=256, lda=64, ldb=256, ldy=256, dt=0, X=256, ws=1 << 20,
                 acc=0, comm=None, reduce=0):
    L = lib.load()
    return L.dl_lowrank_linear(ctypes.c_void_p(X), ldx, ctypes.c_void_p(4096), lda, ctypes.c_void_p(8192), ldb,
                               ctypes.c_void_p(16384), ldy, T, m, n, k, dt, acc, comm, reduce,
                               ctypes.c_void_p(65536), ws, None)


def test_linear_validation_codes(lib):
    assert _call_linear(lib, k=0) == 3            # DL_ERR_RANK
    assert _call_linear(lib, k=300) == 3          # k > min(m, n)
    assert _call_linear(lib, m=0) == 2            # DL_ERR_SHAPE
    assert _call_linear(lib, ldx=100) == 2        # ld < row
    assert _call_linear(lib, X=8) == 6            # DL_ERR_ALIGN (pointer)
    assert _call_linear(lib, lda=66) == 6         # ld not 16-byte multiple (fp32)
    assert _call_linear(lib, T=32, dt=0) == 5     # fp32 beyond the SIMT path
    assert _call_linear(lib, ws=16) == 7          # DL_ERR_WORKSPACE
    assert _call_linear(lib, T=0) == 0            # empty input is a no-op
    assert _call_linear(lib, reduce=3) == 1       # DL_ERR_INVALID_ARG: unknown dl_reduce


def test_linear_reduce_validation(lib):
    """dl_reduce modes (include/dl.h): argument errors are reported before any launch,
    also on a GPU-less host (loopback communicators need no device)."""
    c = lib.Comm.loopback(0, 2)
    h = c.handle
    assert _call_linear(lib, m=96, ldy=48, comm=h, reduce=2) == 4         # SCATTER: m % (32 * world) != 0
    assert _call_linear(lib, comm=h, reduce=1, acc=1) == 10               # fp32 Y += with a collective
    assert _call_linear(lib, comm=h, reduce=2, ldy=130) == 6              # ldy checked against m / P (fp32: 16 B)
    assert _call_linear(lib, comm=h, reduce=2, ldy=100) == 2              # ldy < m / P
    assert _call_linear(lib, comm=h, reduce=2, ldy=128, ws=16) == 7       # workspace includes the RS buffer
    sz = {}
    for red in (0, 1, 2):
        b = ctypes.c_size_t()
        assert lib.load().dl_lowrank_linear_workspace(64, 256, 256, 64, 1, h, red, ctypes.byref(b)) == 0
        sz[red] = b.value
    assert sz[2] > sz[1] > 0 and sz[1] >= sz[0]
    # bf16, T <= 16 with a collective takes the tensor path: its workspace holds the bf16 Z
    b16, b16n = ctypes.c_size_t(), ctypes.c_size_t()
    lib.load().dl_lowrank_linear_workspace(8, 256, 256, 64, 1, h, 1, ctypes.byref(b16))
    lib.load().dl_lowrank_linear_workspace(8, 256, 256, 64, 1, None, 0, ctypes.byref(b16n))
    assert b16.value > b16n.value
    c.close()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the GPU-less failure mode")
def test_group_comm_needs_gpu(lib):
    arr = (ctypes.c_void_p * 2)()
    assert lib.load().dl_comm_create_group(2, 1 << 20, ctypes.cast(arr, ctypes.c_void_p)) == 8   # DL_ERR_CUDA
    assert lib.load().dl_comm_create_group(9, 1 << 20, ctypes.cast(arr, ctypes.c_void_p)) == 1   # world > 8


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the GPU-less failure mode")
def test_no_cpu_fallback(lib):
    """A valid call on a host without an sm_100 GPU must fail loudly."""
    assert _call_linear(lib) == 8                 # DL_ERR_CUDA
    assert "device" in lib.load().dl_last_error().decode().lower() or \
        "cuda" in lib.load().dl_last_error().decode().lower()
    assert not lib.dl_device_ok()


def test_block_workspace_and_validation(lib):
    from synthetic import LLAMA3_70B, block_ranks
    rk = block_ranks(LLAMA3_70B, 0.4)
    cfg = lib.make_block_config(LLAMA3_70B, rk, max_tokens=64, max_seqs=64)
    for world in (1, 2, 4, 8):
        assert lib.dl_block_workspace(cfg, world) > 0
    with pytest.raises(lib.DLError) as e:
        lib.dl_block_workspace(cfg, 16)           # 8 kv heads do not split 16 ways
    assert e.value.name == "DL_ERR_PARTITION"
    bad = lib.make_block_config(LLAMA3_70B, dict(rk, q=9000), max_tokens=64, max_seqs=64)
    with pytest.raises(lib.DLError) as e:
        lib.dl_block_workspace(bad, 1)
    assert e.value.name == "DL_ERR_RANK"


def test_block_variant_validation(lib):
    """mlp_act / no_rope fields (appended to dl_block_config): ReLU MLP must carry no gate."""
    import dataclasses
    from synthetic import OPT_6_7B, LLAMA2_7B, block_ranks
    rk = block_ranks(OPT_6_7B, 0.4)
    assert rk["gate"] == 0
    cfg = lib.make_block_config(OPT_6_7B, rk, max_tokens=64, max_seqs=64)
    assert cfg.mlp_act == lib.DL_MLP_RELU and cfg.no_rope == 1
    assert lib.dl_block_workspace(cfg, 1) > 0
    with pytest.raises(lib.DLError) as e:
        lib.dl_block_workspace(lib.make_block_config(OPT_6_7B, dict(rk, gate=100), 64, 64), 1)
    assert e.value.name == "DL_ERR_RANK"
    cfg.mlp_act = 7
    with pytest.raises(lib.DLError) as e:
        lib.dl_block_workspace(cfg, 1)
    assert e.value.name == "DL_ERR_INVALID_ARG"
    mha = lib.make_block_config(LLAMA2_7B, block_ranks(LLAMA2_7B, 0.2), 64, 64)
    assert mha.mlp_act == lib.DL_MLP_SILU_GLU and mha.no_rope == 0
    for world in (1, 2, 4, 8, 32):
        assert lib.dl_block_workspace(mha, world) > 0
    glu_as_relu = lib.make_block_config(dataclasses.replace(LLAMA2_7B, glu=False), block_ranks(LLAMA2_7B, 0.2),
                                        64, 64)
    with pytest.raises(lib.DLError):
        lib.dl_block_workspace(glu_as_relu, 1)      # LLaMA ranks include a gate


def test_block_layout_validation(lib):
    """DL_LAYOUT_DEINFER workspace sizing and its divisibility / enum checks."""
    from synthetic import LLAMA3_70B, block_ranks
    rk = block_ranks(LLAMA3_70B, 0.4)
    rp = lib.make_block_config(LLAMA3_70B, rk, 64, 64)
    di = lib.make_block_config(LLAMA3_70B, rk, 64, 64, layout=lib.DL_LAYOUT_DEINFER)
    for world in (1, 2, 4, 8):
        assert lib.dl_block_workspace(di, world) > 0
    # latent all-gather buffers: the DeInfer workspace holds [T x slot] + [P x T x slot]
    assert lib.dl_block_workspace(di, 8) > lib.dl_block_workspace(rp, 8)
    di.layout = 9
    with pytest.raises(lib.DLError) as e:
        lib.dl_block_workspace(di, 1)
    assert e.value.name == "DL_ERR_INVALID_ARG"
    import dataclasses
    odd = dataclasses.replace(LLAMA3_70B, m=64 * 7)      # m not divisible by 64 * 2
    bad = lib.make_block_config(odd, block_ranks(odd, 0.4), 64, 64, layout=lib.DL_LAYOUT_DEINFER)
    with pytest.raises(lib.DLError) as e:
        lib.dl_block_workspace(bad, 2)
    assert e.value.name == "DL_ERR_PARTITION"


def test_kv_prepare_matches_oracle_scan(lib, orc):
    """Preparation stage of the low-rank KV cache: the library's host planner
    yields, per sequence, the oracle's contiguous runs, placed at consecutive buffer
    blocks (remapping index list = prefix sums of block counts)."""
    r = np.random.default_rng(7)
    bs, mbps, ns = 16, 6, 5
    for _ in range(20):
        perm = r.permutation(64).astype(np.int32)
        tables = np.full((ns, mbps), -1, np.int32)
        toks = r.integers(0, mbps * bs + 1, ns).astype(np.int32)
        k = 0
        for s in range(ns):
            nb = -(-int(toks[s]) // bs)
            if r.random() < 0.5:                      # some sequences physically contiguous
                start = int(r.integers(100, 200))
                tables[s, :nb] = np.arange(start, start + nb)
            else:
                tables[s, :nb] = perm[k:k + nb]
                k += nb
        rs, rd, rl, nr, sb = lib.dl_kv_prepare(tables, toks, bs, 64, 64)
        got = list(zip(rs[:nr].tolist(), rl[:nr].tolist()))
        exp, dst, exp_dst = [], 0, []
        for s in range(ns):
            nb = -(-int(toks[s]) // bs)
            assert sb[s] == dst
            runs = orc.kv_runs(tables[s, :nb])
            for (st, ln) in runs:
                exp_dst.append(dst)
                dst += ln
            exp += runs
        assert got == exp
        assert rd[:nr].tolist() == exp_dst
    with pytest.raises(lib.DLError) as e:                 # over the buffer capacity
        lib.dl_kv_prepare(np.arange(12, dtype=np.int32).reshape(2, 6), [96, 96], 16, 8, 11)
    assert e.value.name == "DL_ERR_WORKSPACE"
    with pytest.raises(lib.DLError) as e:                 # over max_runs
        lib.dl_kv_prepare(np.array([[0, 2, 4, 6]], np.int32), [64], 16, 3, 8)
    assert e.value.name == "DL_ERR_WORKSPACE"
