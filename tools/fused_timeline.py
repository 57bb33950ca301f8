"""In-graph timeline of the fused decode kernels of one decode step (debug).
python tools/fused_timeline.py [--layers 4]
Per fused launch and phase: when the CTAs started / finished the phase
(min / median / max over CTAs, us from the step start) and when the producers
issued the phase's activation loads.  Launch i = 2*layer (+1: post-attention)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_17709_b200 import _lib
from paper_2604_17709_b200.model import DecomposedLlama
from synthetic import LLAMA3_70B, block_ranks, gen_block_weights, gen_normal

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--batch", type=int, default=64)
a = ap.parse_args()
s = LLAMA3_70B
rk = block_ranks(s, 0.4)
dev = torch.device("cuda")
m = DecomposedLlama(s, rk, (gen_block_weights(s, rk, 3, i, device=dev) for i in range(a.layers)),
                    gen_normal((s.vocab, s.h), 1.0, 1, device=dev, dtype=torch.bfloat16),
                    torch.ones(s.h, dtype=torch.bfloat16, device=dev),
                    gen_normal((s.vocab, s.h), s.h ** -0.5, 2, device=dev, dtype=torch.bfloat16), batch=a.batch,
                    max_seq=513)
m.cache.normal_()
m.cache_lens.fill_(512)
torch.cuda.synchronize()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    m.decode_step()
torch.cuda.synchronize()
W = 48
sms = torch.cuda.get_device_properties(0).multi_processor_count
slots = 2 * a.layers
buf = torch.zeros(slots * sms * W, dtype=torch.int64, device=dev)
_lib.dl_debug_fused_trace(buf)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    m.decode_step()
with torch.cuda.stream(st):
    g.replay()
torch.cuda.synchronize()
buf.zero_()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
with torch.cuda.stream(st):
    e0.record(st)
    g.replay()
    e1.record(st)
torch.cuda.synchronize()
_lib.dl_debug_fused_trace(None)
print(f"step {e0.elapsed_time(e1) * 1e3:.1f} us ({a.layers} layers + embedding/LM head)")
t = buf.view(slots, sms, W).cpu().double()
base = t[0, :, 46].min().item()
names = {0: ["rmsnorm", "qkv.s1", "cvt", "qkv.s2", "rope"],
         1: ["o.s1", "cvt", "o.s2", "res+norm", "gu.s1", "cvt", "gu.s2", "silu", "down.s1", "cvt", "down.s2", "res"]}
us = lambda v: (v - base) / 1e3
prev_end = None
for i in range(slots):
    c = t[i]
    ent = c[:, 46]
    print(f"launch {i} (layer {i // 2}, {'pre' if i % 2 == 0 else 'post'}): entry min {us(ent.min()):8.1f} "
          f"max {us(ent.max()):8.1f}" + (f"  (gap after prev end {us(ent.min()) - prev_end:6.1f})" if prev_end else ""))
    for p, nm in enumerate(names[i % 2]):
        st_, en = c[:, 2 * p], c[:, 2 * p + 1]
        rd = c[:, 28 + p]
        has = st_ > 0
        line = f"   {p:2d} {nm:9s} start med {us(st_[has].median()) if has.any() else float('nan'):8.1f} " \
               f"end min {us(en.min()):8.1f} med {us(en.median()):8.1f} max {us(en.max()):8.1f}"
        if (rd > 0).any():
            r = rd[rd > 0]
            line += f"   act-issue min {us(r.min()):8.1f} max {us(r.max()):8.1f}"
        print(line)
    prev_end = us(c[:, 2 * (len(names[i % 2]) - 1) + 1].max())
