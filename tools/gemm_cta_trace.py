"""Per-CTA phase percentiles of the tcgen05 GEMM launches of one captured decode
step (debug).  python tools/gemm_cta_trace.py [--tp 8] [--layers 2]
Fields (us from the launch's first CTA entry): entry, setup done, first TMA
issued, first stage landed (MMA side), last MMA issued, last accumulator ready,
epilogue done; p10 / p50 / p90 / max over CTAs, for the first layer's 8 GEMMs."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_17709_b200 as dl
from paper_2604_17709_b200 import _lib
from paper_2604_17709_b200.model import DecomposedLlama
from synthetic import LLAMA3_70B, block_ranks, gen_block_weights, gen_normal

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--tp", type=int, default=1)
a = ap.parse_args()
s = LLAMA3_70B
rk = block_ranks(s, 0.4)
dev = torch.device("cuda")
m = DecomposedLlama(s, rk, (gen_block_weights(s, rk, 3, i, device=dev) for i in range(a.layers)),
                    gen_normal((s.vocab, s.h), 1.0, 1, device=dev, dtype=torch.bfloat16),
                    torch.ones(s.h, dtype=torch.bfloat16, device=dev),
                    gen_normal((s.vocab // a.tp, s.h), s.h ** -0.5, 2, device=dev, dtype=torch.bfloat16), batch=64,
                    max_seq=513, comm=dl.Comm.loopback(0, a.tp) if a.tp > 1 else None)
m.cache.normal_()
m.cache_lens.fill_(512)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    m.decode_step()
torch.cuda.synchronize()
slots = 16 * a.layers + 16
buf = torch.zeros(slots * 148 * 8, dtype=torch.int64, device=dev)
_lib.dl_debug_gemm_trace(buf)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    m.decode_step()
for _ in range(2):
    buf.zero_()
    with torch.cuda.stream(st):
        g.replay()
    torch.cuda.synchronize()
_lib.dl_debug_gemm_trace(None)
t = buf.view(slots, 148, 8).cpu().double()
names = ["qkv s1", "qkv s2", "o s1", "o s2", "gu s1", "gu s2", "down s1", "down s2"]
labels = ["entry", "setup", "tma0", "land0", "mmaEnd", "accRdy", "epiEnd"]
k = 0
for i in range(slots):
    c = t[i]
    used = c[:, 0] > 0
    if not used.any() or not (c[:, 5] > 2 ** 48).any():
        continue
    c = c[used]
    t0 = c[:, 0].min()
    print(f"== {names[k] if k < 8 else 'gemm'} (slot {i}), {c.shape[0]} CTAs: p10 p50 p90 max (us)")
    for f, l in enumerate(labels):
        v = c[:, f]
        v = ((v[v > 0] - t0) / 1e3).sort().values
        n = len(v)
        if n:
            print(f"   {l:7s} " + " ".join(f"{v[int(q * (n - 1))]:6.1f}" for q in (.1, .5, .9, 1)))
    k += 1
    if k >= 8:
        break
