"""In-graph timeline of one 70B@40% prefill step (2,048 tokens, a few layers; debug).
python tools/prefill_timeline.py [--layers 2]
GEMM launches (first CTA entry, last CTA epilogue end) and the traced non-GEMM
kernels (entry, after griddepcontrol.wait, end), in launch order, microseconds
from the first GEMM entry, with the idle gap before each."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_17709_b200 import _lib
from paper_2604_17709_b200.model import DecomposedLlama
from synthetic import LLAMA3_70B, block_ranks, gen_block_weights, gen_normal

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=2)
a = ap.parse_args()
s = LLAMA3_70B
rk = block_ranks(s, 0.4)
dev = torch.device("cuda")
m = DecomposedLlama(s, rk, (gen_block_weights(s, rk, 3, i, device=dev) for i in range(a.layers)),
                    gen_normal((s.vocab, s.h), 1.0, 1, device=dev, dtype=torch.bfloat16),
                    torch.ones(s.h, dtype=torch.bfloat16, device=dev),
                    gen_normal((s.vocab, s.h), s.h ** -0.5, 2, device=dev, dtype=torch.bfloat16), batch=64,
                    max_seq=513, prefill_tokens=2048)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    m.prefill_step()
torch.cuda.synchronize()
slots = 16 * a.layers + 8
buf = torch.zeros(slots * 148 * 8, dtype=torch.int64, device=dev)
ew = torch.zeros(64 * a.layers * 4, dtype=torch.int64, device=dev)
_lib.dl_debug_gemm_trace(buf)
_lib.dl_debug_ew_trace(ew)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    m.prefill_step()
with torch.cuda.stream(st):
    g.replay()
torch.cuda.synchronize()
buf.zero_()
ew.zero_()
ew.view(-1, 4)[:, 1:3] = -1
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
with torch.cuda.stream(st):
    e0.record(st); g.replay(); e1.record(st)
torch.cuda.synchronize()
_lib.dl_debug_gemm_trace(None)
_lib.dl_debug_ew_trace(None)
ev = []
t = buf.view(slots, 148, 8).cpu()
for i in range(slots):
    c = t[i]
    used = c[:, 0] > 0
    if used.any():
        ev.append(("gemm", c[used, 0].min().item(), None, c[used, 6][c[used, 6] > 0].max().item()))
names = {1: "silu", 2: "res+norm", 3: "rope", 4: "attn-dec", 5: "attn-prefill"}
for r in ew.view(-1, 4).cpu():
    if int(r[0]) == 0:
        continue
    ev.append((names.get(int(r[0]), str(int(r[0]))), r[1].item(), r[2].item(), r[3].item()))
ev.sort(key=lambda x: x[1])
t0 = ev[0][1]
print(f"step {e0.elapsed_time(e1) * 1e3:.0f} us in graph ({a.layers} layers + LM head)")
prev_end = None
for name, st_, wt, en in ev:
    gap = (st_ - prev_end) / 1e3 if prev_end else 0.0
    w = f"{(wt - t0) / 1e3:9.1f}" if wt else "        -"
    print(f"  {name:12s} entry {(st_ - t0) / 1e3:9.1f} wait {w} end {(en - t0) / 1e3:9.1f}  run {(en - (wt or st_)) / 1e3:8.1f}"
          f"  gap-from-prev-end {gap:7.1f}")
    prev_end = en if prev_end is None else max(prev_end, en)
