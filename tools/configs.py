"""BASELINE configs 1 and 2 on one B200 (measurement; bench.py times config 4 at TP = 1).

config 1: one decomposed linear m = n = 256, k = 64, T = 4 tokens, fp32 (SIMT chain,
          Z kept in shared memory): microseconds per call, eager launches and CUDA-Graph
          replays, and rel-L2 against the fp64 oracle.
config 2: one LLaMA-3-8B decomposed block @ 20 % (ranks 3277 / 819), bf16 prefill of
          one 2048-token sequence: ms per block, tokens/s, and the tensor-roofline
          fraction of its algorithmic flops (2 T sum (m+n)k + causal attention).
python tools/configs.py   -> one JSON line per config
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2604_17709_b200 as dl
from synthetic import LLAMA3_8B, block_ranks, gen_block_weights, gen_factor_pair, gen_normal

PEAKS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json")))
dl.load()
dev = torch.device("cuda")
st = torch.cuda.Stream()


def time_it(fn, n):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(n):
            fn()
        e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


# ---- config 1 -------------------------------------------------------------------
T, m, n, k = 4, 256, 256, 64
X = gen_normal((T, n), 1.0, 1, dtype=torch.float32)
A, B = gen_factor_pair(m, n, k, 2, dtype=torch.float32)
Xd, Ad, Bd = X.to(dev), A.to(dev), B.to(dev)
Y = torch.empty(T, m, dtype=torch.float32, device=dev)
ws = torch.zeros(dl.dl_lowrank_linear_workspace(T, m, n, k, torch.float32), dtype=torch.uint8, device=dev)
call = lambda: dl.dl_lowrank_linear(Xd, Ad, Bd, Y, workspace=ws, stream=st)  # noqa: E731
eager_ms = time_it(call, 200)
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(st):
    call()
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=st):
    for _ in range(100):
        call()
graph_ms = time_it(g.replay, 20) / 100
ref = X.double().numpy() @ B.double().numpy().T @ A.double().numpy().T
relerr = float(np.linalg.norm(Y.cpu().double().numpy() - ref) / np.linalg.norm(ref))
print(json.dumps({"config": 1, "workload": "single decomposed linear m=n=256 k=64 T=4 fp32",
                  "us_per_call_eager": round(eager_ms * 1e3, 2), "us_per_call_graph": round(graph_ms * 1e3, 2),
                  "algorithmic_bytes": (m + n) * k * 4 + T * (m + n) * 4, "rel_l2_vs_fp64": relerr}), flush=True)

# ---- config 2 -------------------------------------------------------------------
s = LLAMA3_8B
rk = block_ranks(s, 0.2)
w = gen_block_weights(s, rk, 2, 0, device=dev)
Tp = 2048
cfg = dl.make_block_config(s, rk, max_tokens=Tp, max_seqs=1)
wd = dl.BlockWeights(w)
wsb = torch.zeros(dl.dl_block_workspace(cfg), dtype=torch.uint8, device=dev)
x0 = gen_normal((Tp, s.h), 1.0, 3, device=dev, dtype=torch.bfloat16)
x = x0.clone()
pos = torch.arange(Tp, dtype=torch.int32, device=dev)
cu = torch.tensor([0, Tp], dtype=torch.int32, device=dev)
lens = torch.zeros(1, dtype=torch.int32, device=dev)
kc = torch.zeros(1, s.n_kv_heads, Tp, s.head_dim, dtype=torch.bfloat16, device=dev)
vc = torch.zeros_like(kc)


def block():
    x.copy_(x0)   # same input every call (16 MB copy, timed separately and subtracted)
    dl.dl_decomposed_block_forward(cfg, wd, x, pos, cu, 1, dl.DL_PREFILL, kc, vc, lens, None, wsb, stream=st)


copy_ms = time_it(lambda: x.copy_(x0), 20)
ms = time_it(block, 10) - copy_ms
mats = {"q": (s.h, s.h), "k": (s.h_kv, s.h), "v": (s.h_kv, s.h), "o": (s.h, s.h), "gate": (s.m, s.h),
        "up": (s.m, s.h), "down": (s.h, s.m)}
lin = 2 * Tp * sum((mm + nn) * rk[name] for name, (mm, nn) in mats.items())
att = 4 * (Tp * (Tp + 1) / 2) * s.h
tf = (lin + att) / (ms * 1e-3) / 1e12
print(json.dumps({"config": 2, "workload": "llama3-8b block @20% prefill 2048 tokens, bf16",
                  "ms_per_block": round(ms, 4), "tokens_per_s": round(Tp / ms * 1e3),
                  "algorithmic_gflop": round((lin + att) / 1e9, 1), "achieved_tflops": round(tf, 1),
                  "frac_of_bf16_sustained": round(tf / PEAKS["bf16_tflops_sustained"], 3),
                  "peak_tflops": PEAKS["bf16_tflops_sustained"]}), flush=True)
