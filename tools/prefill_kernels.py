"""Per-launch event timing of the prefill step's GEMMs (kind 0) and DP+SK tail
finalize kernels (kind 2) in an instrumented CUDA-Graph replay (debug)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_17709_b200 as dl
from paper_2604_17709_b200.model import DecomposedLlama
from synthetic import LLAMA3_70B, block_ranks, gen_block_weights, gen_normal
L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
s = LLAMA3_70B
rk = block_ranks(s, 0.4)
dev = torch.device("cuda")
m = DecomposedLlama(s, rk, (gen_block_weights(s, rk, 3, i, device=dev) for i in range(L)),
                    gen_normal((s.vocab, s.h), 1.0, 1, device=dev, dtype=torch.bfloat16),
                    torch.ones(s.h, dtype=torch.bfloat16, device=dev),
                    gen_normal((s.vocab, s.h), s.h ** -0.5, 2, device=dev, dtype=torch.bfloat16), batch=64,
                    max_seq=513, prefill_tokens=2048)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    m.prefill_step()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    m.prefill_step()
gi = torch.cuda.CUDAGraph()
dl.dl_profile_begin(64 * L + 16)
with torch.cuda.graph(gi, stream=st):
    m.prefill_step()
dl.dl_profile_end()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
with torch.cuda.stream(st):
    g.replay(); e0.record(st); g.replay(); e1.record(st)
    gi.replay(); gi.replay()
torch.cuda.synchronize()
rec = dl.dl_profile_records()
k0 = [r for r in rec if r[3] == 0]
k2 = [r for r in rec if r[3] == 2]
print(f"prefill step ({L} layers) {e0.elapsed_time(e1):.2f} ms; GEMMs {len(k0)} {sum(r[0] for r in k0):.2f} ms "
      f"{sum(r[2] for r in k0) / (sum(r[0] for r in k0) * 1e-3) / 1e12:.0f} TFLOP/s; tail finalize {len(k2)} "
      f"{sum(r[0] for r in k2):.3f} ms")
for r in k0[:9]:
    print(f"   gemm {r[0] * 1e3:8.1f} us  {r[2] / (r[0] * 1e-3) / 1e12:7.0f} TFLOP/s")
