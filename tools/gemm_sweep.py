"""Decode-GEMM overhead sweep: time dl_dense (whole-tile swap-AB) and
dl_lowrank_linear (stream-K chain) at T=64 for growing weight sizes and fit
t = t0 + bytes / BW.  Run on a B200: python tools/gemm_sweep.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_17709_b200 as dl

def bench(fn, reps=50):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(10): fn()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(s):
        g.replay()
        e0.record(s)
        for _ in range(reps // 10): g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps // 10 * 10) * 1e3  # us


def main():
    T = 64
    print("dense (whole-tile swap): N x K, MB, us, GB/s")
    for N, K in [(1024, 8192), (2048, 8192), (4096, 8192), (8192, 8192), (16384, 8192), (32768, 8192), (65536, 8192)]:
        X = torch.randn(T, K, device="cuda", dtype=torch.bfloat16)
        W = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
        C = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
        us = bench(lambda: dl.dl_dense(X, W, C))
        mb = N * K * 2 / 1e6
        print(f"{N:6d} {K:6d} {mb:8.1f} {us:8.1f} {mb / us * 1e3:8.0f}")
    print("lowrank chain (stream-K both stages): m=n, k, MB, us, GB/s")
    for m, k in [(2048, 1024), (4096, 2048), (8192, 4096), (8192, 4928), (16384, 4928), (28672, 4928)]:
        n = 8192
        X = torch.randn(T, n, device="cuda", dtype=torch.bfloat16)
        A = torch.randn(m, k, device="cuda", dtype=torch.bfloat16) * 0.01
        B = torch.randn(k, n, device="cuda", dtype=torch.bfloat16) * 0.01
        Y = torch.empty(T, m, device="cuda", dtype=torch.bfloat16)
        ws = torch.zeros(dl.dl_lowrank_linear_workspace(T, m, n, k), dtype=torch.uint8, device="cuda")
        us = bench(lambda: dl.dl_lowrank_linear(X, A, B, Y, workspace=ws))
        mb = (m + n) * k * 2 / 1e6
        print(f"{m:6d} {k:6d} {mb:8.1f} {us:8.1f} {mb / us * 1e3:8.0f}")


if __name__ == "__main__":
    main()
