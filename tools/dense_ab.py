"""A/B: dense T=64 GEMM, whole-tile bf16 vs stream-K fp32-red (DL_DENSE_SK=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_17709_b200 as dl
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_sweep import bench
T = 64
mode = "streamK" if os.environ.get("DL_DENSE_SK") == "1" else "whole"
for N, K in [(8192, 8192), (4928, 8192), (8192, 4928), (28672, 4928), (57344, 4928), (128256, 8192)]:
    X = torch.randn(T, K, device="cuda", dtype=torch.bfloat16)
    W = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    C = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    ws = torch.zeros(T * N * 4 + 256, dtype=torch.uint8, device="cuda")
    us = bench(lambda: dl.dl_dense(X, W, C, workspace=ws))
    mb = N * K * 2 / 1e6
    print(f"{mode:8s} N={N:6d} K={K:5d} {mb:7.1f} MB {us:8.1f} us {mb / us * 1e3:7.0f} GB/s")
