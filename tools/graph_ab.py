"""Alternating A/B of the 70B@40% decode step: CUDA-Graph replay vs eager launches
(the N2 graph on/off question), same process, same stream, 4 rounds."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_17709_b200.model import DecomposedLlama
from synthetic import LLAMA3_70B, block_ranks, gen_block_weights, gen_normal

s = LLAMA3_70B
rk = block_ranks(s, 0.4)
dev = torch.device("cuda")
m = DecomposedLlama(s, rk, (gen_block_weights(s, rk, 3, i, device=dev) for i in range(s.n_layers)),
                    gen_normal((s.vocab, s.h), 1.0, 1, device=dev, dtype=torch.bfloat16),
                    torch.ones(s.h, dtype=torch.bfloat16, device=dev),
                    gen_normal((s.vocab, s.h), s.h ** -0.5, 2, device=dev, dtype=torch.bfloat16), batch=64,
                    max_seq=513)
m.cache.normal_()
m.cache_lens.fill_(512)
torch.cuda.synchronize()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    m.decode_step()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    m.decode_step()


def run(fn, n=5):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(st):
        fn()
        e0.record(st)
        for _ in range(n):
            fn()
        e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for r in range(4):
    print(f"round {r}: graph {run(g.replay):.3f} ms  eager {run(m.decode_step):.3f} ms", flush=True)
