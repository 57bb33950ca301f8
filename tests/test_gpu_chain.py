"""GPU parity of the fused two-stage chain (SURVEY §8 row a2+a3): stage 1
Z = X B^T and stage 2 Y = Z A^T in ONE persistent launch, stage 2 waiting on an
in-kernel arrival counter instead of a kernel boundary (Eq. 1,
y = A(Bx)).  Compared element by element with the fp64 oracle (rel-L2 2e-2,
north_star) through the C ABI.

Covers: every swap-AB tile configuration (T in 17..64 -> BN 64 / 9 stages,
65..128 -> BN 128 / 6 stages, 129..256 -> BN 256 / 4 stages, two CTAs per SM),
problems with fewer work units than SMs in either stage (the idle CTAs must
still arrive), stage 2 with many more / many fewer units than stage 1, ragged
k, repeated calls on one workspace (the counters are reset by the last CTA),
and CUDA-graph replays of the chain.
"""
import numpy as np
import pytest
import torch

from synthetic import gen_factor_pair, gen_normal

pytestmark = pytest.mark.gpu

TOL = 2e-2


def rel(a, b):
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


def _inputs(T, m, n, k, seed):
    X = gen_normal((T, n), 1.0, seed, dtype=torch.bfloat16)
    A, B = gen_factor_pair(m, n, k, seed + 7, dtype=torch.bfloat16)
    return X, A, B


# (m, n, k): stage-1 units = ceil(k/128) * ceil(n/64), stage-2 units = ceil(m/128) * ceil(k/64)
SHAPES = [
    (640, 520, 200),      # both stages < 148 units
    (4096, 4096, 616),    # TP=8-like o projection: 320 / 320 units
    (8192, 1024, 96),     # stage 2 >> stage 1 (16 vs 128 units)
    (256, 8192, 248),     # stage 1 >> stage 2 (256 vs 8 units)
    (256, 64, 8),         # tiny: 1 unit in stage 1, 2 in stage 2
]


@pytest.mark.parametrize("T", [17, 40, 64, 65, 128, 129, 200, 256])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_chain_linear(dl, orc, T, shape):
    m, n, k = shape
    X, A, B = _inputs(T, m, n, k, 1000 + T + m)
    Y = torch.empty(T, m, dtype=torch.bfloat16, device="cuda")
    dl.dl_lowrank_linear(X.cuda(), A.cuda(), B.cuda(), Y)
    torch.cuda.synchronize()
    assert rel(Y.cpu().double().numpy(), orc.lowrank_linear(X, A, B)) <= TOL


def test_chain_repeated_calls_one_workspace(dl, orc):
    """Back-to-back chain launches on one workspace (PDL-overlapped on one
    stream): the arrival counters must be reset by each launch's last CTA."""
    T, m, n, k = 64, 2048, 1536, 304
    ws = torch.zeros(dl.dl_lowrank_linear_workspace(T, m, n, k), dtype=torch.uint8, device="cuda")
    outs, refs = [], []
    for i in range(6):
        X, A, B = _inputs(T, m, n, k, 50 + i)
        Y = torch.empty(T, m, dtype=torch.bfloat16, device="cuda")
        dl.dl_lowrank_linear(X.cuda(), A.cuda(), B.cuda(), Y, workspace=ws)
        outs.append(Y)
        refs.append(orc.lowrank_linear(X, A, B))
    torch.cuda.synchronize()
    for Y, r in zip(outs, refs):
        assert rel(Y.cpu().double().numpy(), r) <= TOL


def test_chain_graph_replay(dl, orc):
    """The chain captured in a CUDA graph and replayed with new inputs (P:147-150:
    fixed addresses, no per-replay state left behind)."""
    T, m, n, k = 100, 1024, 2048, 400
    X, A, B = _inputs(T, m, n, k, 77)
    Xd, Ad, Bd = X.cuda(), A.cuda(), B.cuda()
    Y = torch.empty(T, m, dtype=torch.bfloat16, device="cuda")
    ws = torch.zeros(dl.dl_lowrank_linear_workspace(T, m, n, k), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        dl.dl_lowrank_linear(Xd, Ad, Bd, Y, workspace=ws, stream=s)   # warm-up (attributes, maps)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        dl.dl_lowrank_linear(Xd, Ad, Bd, Y, workspace=ws, stream=s)
    for i in range(3):
        Xi = gen_normal((T, n), 1.0, 300 + i, dtype=torch.bfloat16)
        Xd.copy_(Xi.cuda())
        g.replay()
        torch.cuda.synchronize()
        assert rel(Y.cpu().double().numpy(), orc.lowrank_linear(Xi, A, B)) <= TOL
