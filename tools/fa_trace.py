"""Per-CTA cycle breakdown of the tcgen05 prefill attention (debug): one eager
70B@40% prefill layer (2,048 tokens) with the GEMM trace buffer on; the
attention writes 8 u64 per CTA: softmax warp 2 {wait S, load S + max, exp +
P store, wait P slot}, MMA thread {wait K, wait P, wait other}, total."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_17709_b200 import _lib
from paper_2604_17709_b200.model import DecomposedLlama
from synthetic import LLAMA3_70B, block_ranks, gen_block_weights, gen_normal
s = LLAMA3_70B
rk = block_ranks(s, 0.4)
dev = torch.device("cuda")
m = DecomposedLlama(s, rk, (gen_block_weights(s, rk, 3, i, device=dev) for i in range(1)),
                    gen_normal((s.vocab, s.h), 1.0, 1, device=dev, dtype=torch.bfloat16),
                    torch.ones(s.h, dtype=torch.bfloat16, device=dev),
                    gen_normal((s.vocab, s.h), s.h ** -0.5, 2, device=dev, dtype=torch.bfloat16), batch=64,
                    max_seq=513, prefill_tokens=2048)
m.prefill_step(); torch.cuda.synchronize()
buf = torch.zeros(64 * 148 * 8, dtype=torch.int64, device=dev)
_lib.dl_debug_gemm_trace(buf)
m.prefill_step(); torch.cuda.synchronize()
_lib.dl_debug_gemm_trace(None)
t = buf.view(64, 148, 8).cpu().double()
for i in range(64):
    c = t[i]
    if (c[:, 7] > 0).sum() > 100 and (c[:, 4] > 0).any():
        names = ["sm.waitS", "sm.ldS+max", "sm.exp+P", "sm.waitP", "mma.waitK", "mma.waitP", "K.latency", "total"]
        for j, nme in enumerate(names):
            v = c[:, j]
            print(f"{nme:11s} mean {v.mean() / 1e3:8.1f} kcyc  max {v.max() / 1e3:8.1f}")
        break
