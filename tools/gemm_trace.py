"""Per-CTA timeline of one tcgen05 GEMM launch (debug).  python tools/gemm_trace.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_17709_b200 as dl
from paper_2604_17709_b200 import _lib

def show(name, fn):
    buf = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
    fn(); torch.cuda.synchronize()
    _lib.dl_debug_gemm_trace(buf)
    fn(); torch.cuda.synchronize()
    _lib.dl_debug_gemm_trace(None)
    t = buf.view(148, 8).cpu()
    used = t[:, 0] > 0
    t = t[used]
    t0 = t[:, 0].min()
    rel = (t[:, :7] - t0).double() / 1000.0
    rel[t[:, :7] == 0] = float("nan")
    labels = ["entry", "setup", "tma0", "land0", "mmaEnd", "accRdy", "epiEnd"]
    print(f"== {name}: {int(used.sum())} CTAs; us relative to first entry (min / median / max)")
    for i, l in enumerate(labels):
        c = rel[:, i]
        c = c[~torch.isnan(c)]
        if len(c): print(f"   {l:7s} {c.min():8.2f} {c.median():8.2f} {c.max():8.2f}")

T = 64
for N, K in [(1024, 8192), (8192, 8192), (65536, 8192)]:
    X = torch.randn(T, K, device="cuda", dtype=torch.bfloat16)
    W = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    C = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    show(f"dense N={N} K={K}", lambda: dl.dl_dense(X, W, C))
m, k, n = 8192, 4928, 8192
X = torch.randn(T, n, device="cuda", dtype=torch.bfloat16)
A = torch.randn(m, k, device="cuda", dtype=torch.bfloat16) * 0.01
B = torch.randn(k, n, device="cuda", dtype=torch.bfloat16) * 0.01
Y = torch.empty(T, m, device="cuda", dtype=torch.bfloat16)
ws = torch.zeros(dl.dl_lowrank_linear_workspace(T, m, n, k), dtype=torch.uint8, device="cuda")
show("lowrank (2 stream-K GEMMs; trace shows the last)", lambda: dl.dl_lowrank_linear(X, A, B, Y, workspace=ws))
