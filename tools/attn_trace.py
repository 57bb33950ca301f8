"""Per-CTA timeline of the stream-K decode attention inside a captured decode
step (debug).  python tools/attn_trace.py [--tp 8] [--layers 2]
The attention writes 8 u64 per CTA into the GEMM trace buffer (2 slots for its
296 CTAs): entry, prologue done, griddepcontrol.wait returned, first tile
landed, last item's tile loop done, -, end, SM id.  Printed relative to the
launch's first CTA entry (us): min / p10 / median / p90 / max over CTAs."""
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
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--ctx", type=int, default=512)
a = ap.parse_args()
s = LLAMA3_70B
rk = block_ranks(s, 0.4)
dev = torch.device("cuda")
m = DecomposedLlama(s, rk, (gen_block_weights(s, rk, 3, i, device=dev) for i in range(a.layers)),
                    gen_normal((s.vocab, s.h), 1.0, 1, device=dev, dtype=torch.bfloat16),
                    torch.ones(s.h, dtype=torch.bfloat16, device=dev),
                    gen_normal((s.vocab // a.tp, s.h), s.h ** -0.5, 2, device=dev, dtype=torch.bfloat16),
                    batch=a.batch, max_seq=a.ctx + 1, comm=dl.Comm.loopback(0, a.tp) if a.tp > 1 else None)
m.cache.normal_()
m.cache_lens.fill_(a.ctx)
torch.cuda.synchronize()
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
_lib.dl_debug_gemm_trace(None)
for rep in range(2):
    buf.zero_()
    with torch.cuda.stream(st):
        g.replay()
    torch.cuda.synchronize()
t = buf.view(slots, 148, 8).cpu().double()
labels = ["entry", "prolog", "wait", "tile0", "loop", "-", "end"]
i = 0
while i < slots:
    c = t[i]
    used = c[:, 0] > 0
    if not used.any():
        i += 1
        continue
    # attention launches fill two consecutive slots with 296 CTAs and leave field 5 empty
    # attention slots carry tile / item / merge counts in field 5 (< 2^48), GEMM slots a timestamp
    if used.all() and (c[:, 5] < 2 ** 48).all():
        two = i + 1 < slots and (t[i + 1][:, 0] > 0).all() and (t[i + 1][:, 5] < 2 ** 48).all()
        c = torch.cat([t[i], t[i + 1]]) if two else t[i]
        t0 = c[:, 0].min()
        print(f"== attention (slot {i}{'-%d' % (i + 1) if two else ''}), {c.shape[0]} CTAs; us from first entry: "
              "min p10 p50 p90 max")
        for f, l in enumerate(labels):
            if l == "-":
                continue
            v = c[:, f]
            v = ((v[v > 0] - t0) / 1e3).sort().values
            n = len(v)
            if n:
                print(f"   {l:7s} " + " ".join(f"{v[int(q * (n - 1))]:7.1f}" for q in (0, .1, .5, .9, 1)))
        d = ((c[:, 6] - c[:, 2]) / 1e3).sort().values
        print(f"   run (end - wait) per CTA: p10 {d[len(d) // 10]:.1f} p50 {d[len(d) // 2]:.1f} max {d[-1]:.1f}")
        info = c[:, 5].long()
        tiles, items, merges = info & 0xFFFF, (info >> 16) & 0xFFFF, (info >> 32) & 0xFFFF
        run = (c[:, 6] - c[:, 2]) / 1e3
        order = run.argsort(descending=True)[:8]
        print("   slowest CTAs: run_us tiles items merges smid")
        for k in order.tolist():
            print(f"     {run[k]:6.1f} {int(tiles[k]):5d} {int(items[k]):5d} {int(merges[k]):6d} {int(c[k, 7]):4d}")
        print(f"   merges: CTAs with >=1 merge {(merges > 0).sum().item()}, mean run {run[merges > 0].mean():.1f} "
              f"vs {run[merges == 0].mean():.1f} us without")
        i += 2 if two else 1
        continue
    i += 1
