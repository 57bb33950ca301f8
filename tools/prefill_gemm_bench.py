"""Prefill GEMM throughput: dl_dense and dl_lowrank_linear at T=2048 (tokens).
python tools/prefill_gemm_bench.py   (DL_PREFILL_PAIR=0 selects the 1-CTA kernel)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_17709_b200 as dl

def bench(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps): fn()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(s):
        g.replay()
        e0.record(s); g.replay(); e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3

T = 2048
for N, K in [(8192, 8192), (28672, 8192), (8192, 28672), (57344, 4928), (10240, 6144)]:
    X = torch.randn(T, K, device="cuda", dtype=torch.bfloat16)
    W = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.01
    C = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    us = bench(lambda: dl.dl_dense(X, W, C))
    ref = (X.float() @ W.float().T)
    err = ((C.float() - ref).norm() / ref.norm()).item()
    print(f"dense T={T} N={N:6d} K={K:6d}: {us:8.1f} us {2*T*N*K/us/1e6:8.1f} TFLOP/s  relerr {err:.2e}")
