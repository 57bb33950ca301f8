"""Eager decode + prefill steps of a few 70B@40% layers (for ncu / nsys-less
profiling).  python tools/step_profile.py [--layers 2] [--no-decode] [--no-prefill]
Under ncu:  ncu --cache-control none --metrics gpu__time_duration.sum --csv \
            -k regex:"tc_gemm|rmsnorm|ew4|rope|attn|embedding" python tools/step_profile.py"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_17709_b200.model import DecomposedLlama
from synthetic import LLAMA3_70B, block_ranks, gen_block_weights, gen_normal

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--no-decode", action="store_true")
ap.add_argument("--no-prefill", action="store_true")
ap.add_argument("--prefill-tokens", type=int, default=2048)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--kv", default="full", choices=["full", "lowrank"])
a = ap.parse_args()
s = LLAMA3_70B
rk = block_ranks(s, 0.4)
dev = torch.device("cuda")
layers = (gen_block_weights(s, rk, 3, i, device=dev) for i in range(a.layers))
emb = gen_normal((s.vocab, s.h), 1.0, 1, device=dev, dtype=torch.bfloat16)
lm = gen_normal((s.vocab, s.h), s.h ** -0.5, 2, device=dev, dtype=torch.bfloat16)
m = DecomposedLlama(s, rk, layers, emb, torch.ones(s.h, dtype=torch.bfloat16, device=dev), lm, batch=64,
                    max_seq=513, prefill_tokens=0 if a.no_prefill else a.prefill_tokens, kv=a.kv)
m.cache_lens.fill_(512)
if a.kv == "lowrank":
    for kvl in m.kv_layers:
        kvl.pool.normal_()
    m.kv_prepare([512] * 64)
else:
    m.cache.normal_()
torch.cuda.synchronize()
for _ in range(a.reps):
    if not a.no_decode:
        m.decode_step()
    if not a.no_prefill:
        m.prefill_step()
torch.cuda.synchronize()
print("done")
