"""In-graph timeline of the GEMM launches of one decode step (debug).
python tools/decode_timeline.py [--layers 4]
Prints per GEMM launch: start (first CTA entry), first tile landed (median),
end (last CTA epilogue done), duration, and the gap since the previous GEMM
ended (time spent in non-GEMM kernels / dependencies), in microseconds."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_17709_b200 as dl
from paper_2604_17709_b200 import _lib
from paper_2604_17709_b200.model import DecomposedLlama
from synthetic import LLAMA3_70B, block_ranks, gen_block_weights, gen_normal

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--tp", type=int, default=1, help="P > 1: one rank of TP = P through the loopback communicator")
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
torch.cuda.synchronize()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    m.decode_step()
torch.cuda.synchronize()
slots = 16 * a.layers + 8
buf = torch.zeros(slots * 148 * 8, dtype=torch.int64, device=dev)
_lib.dl_debug_gemm_trace(buf)
ew = torch.zeros(256 * a.layers * 4, dtype=torch.int64, device=dev)
_lib.dl_debug_ew_trace(ew)                       # slots are assigned at capture
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    m.decode_step()
with torch.cuda.stream(st):
    g.replay()
torch.cuda.synchronize()
buf.zero_()
ew.zero_()
ew.view(-1, 4)[:, 1:3] = -1                      # 0xffff... for the atomicMin fields
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
with torch.cuda.stream(st):
    e0.record(st); g.replay(); e1.record(st)
torch.cuda.synchronize()
_lib.dl_debug_gemm_trace(None)
_lib.dl_debug_ew_trace(None)
step_us = e0.elapsed_time(e1) * 1e3
t = buf.view(slots, 148, 8).cpu().double()
rows = []
for i in range(slots):
    c = t[i]
    used = c[:, 0] > 0
    if not used.any():
        continue
    c = c[used]
    rows.append((i, c[:, 0].min().item(), c[:, 3][c[:, 3] > 0].median().item() if (c[:, 3] > 0).any() else float("nan"),
                 c[:, 6].max().item(), c[:, 6].min().item(), int(used.sum())))
t0 = rows[0][1]
prev_end = None
tot_gemm = 0.0
print(f"step {step_us:.1f} us in graph ({a.layers} layers); GEMM launches {len(rows)}")
print(" slot   start   land0     end  spanUS  firstEndUS  gapUS  ctas")
for i, st_, land, end, first_end, n in rows:
    gap = (st_ - prev_end) / 1e3 if prev_end is not None else 0.0
    span = (end - st_) / 1e3
    tot_gemm += span
    print(f"{i:5d} {(st_ - t0) / 1e3:7.1f} {(land - t0) / 1e3:7.1f} {(end - t0) / 1e3:7.1f} {span:7.1f} "
          f"{(first_end - t0) / 1e3:11.1f} {gap:6.1f} {n:5d}")
    prev_end = end
print(f"sum of GEMM spans {tot_gemm:.1f} us; last end {(rows[-1][3] - t0) / 1e3:.1f} us")
names = {1: "silu", 2: "res+norm", 3: "rope", 4: "attention"}
ev = ew.view(-1, 4).cpu()
print("non-GEMM kernels (us from the first GEMM start): entry / after-wait / end")
for r in ev:
    if int(r[0]) == 0:
        continue
    f = lambda v: (v.item() - t0) / 1e3 if v.item() > 0 else float("nan")  # noqa: E731
    print(f"  {names.get(int(r[0]), r[0])}: {f(r[1]):8.1f} {f(r[2]):8.1f} {f(r[3]):8.1f}  run {f(r[3]) - f(r[2]):6.1f}")
