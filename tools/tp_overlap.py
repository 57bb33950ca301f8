"""Where the TP reductions go: GPU kernel time of one rank of a TP = P decode step,
P ranks emulated on ONE B200 (measurement only; no NVLink on a 1-GPU box).

Three runs of the same layers (70B@40 %, B = 64, context 512 by default):
  loopback    per-rank compute only (collectives are local copies; tools/tp_emulate.py)
  collective  group communicator, the reductions as separate peer-memory kernels
              (reduce-scatter / two-shot all-reduce / all-gather passes over the data)
  fused       group communicator with the symmetric window: the stage-2 epilogues
              red.add into the ranks' windows, the attention output is pushed, and
              each collective is a barrier
Kernel durations come from CUPTI (torch.profiler), summed per kernel family and
divided by P, so host-side barrier gaps of the emulation do not count.

python tools/tp_overlap.py [--P 8] [--layers 4] [--model 70b|8b]
"""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_17709_b200 as dl  # noqa: E402
from synthetic import LLAMA3_70B, LLAMA3_8B, block_ranks, gen_block_weights, gen_normal  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=8)
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--ctx", type=int, default=512)
ap.add_argument("--model", default="70b", choices=["70b", "8b"])
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
s = LLAMA3_70B if a.model == "70b" else LLAMA3_8B
rk = block_ranks(s, 0.4)
P, B, Lc = a.P, a.batch, a.ctx
hk = s.n_kv_heads // P
full = [gen_block_weights(s, rk, 3, i, device="cuda") for i in range(a.layers)]
cfg = dl.make_block_config(s, rk, max_tokens=B, max_seqs=B)


def family(name):
    for key, fam in (("tc_gemm", "gemm"), ("peer_", "collective kernels"), ("fan_copy", "window push"), ("fan_push", "window push"),
                     ("attn", "attention"), ("Memcpy", "collective kernels"), ("memcpy", "collective kernels")):
        if key in name:
            return fam
    return "elementwise"


def setup(r, comm):
    ws_ = [dl.BlockWeights(w, world=P, rank=r) for w in full]
    kc = [torch.randn(B, hk, Lc + 1, s.head_dim, device="cuda").bfloat16() for _ in range(a.layers)]
    vc = [torch.randn(B, hk, Lc + 1, s.head_dim, device="cuda").bfloat16() for _ in range(a.layers)]
    return {"w": ws_, "args": dl.StackArgs(ws_, kc, vc), "kc": kc, "vc": vc,
            "ws": torch.zeros(dl.dl_block_workspace(cfg, P), dtype=torch.uint8, device="cuda"),
            "x": gen_normal((B, s.h), 1.0, 5, device="cuda", dtype=torch.bfloat16),
            "cl": torch.full((B,), Lc, dtype=torch.int32, device="cuda"), "comm": comm}


def step(st):
    dl.dl_decomposed_stack_forward(cfg, st["args"], st["x"], st["cl"], None, B, dl.DL_DECODE, st["cl"], st["comm"],
                                   st["ws"])


def profile(run):
    run()                                      # warm-up
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(a.reps):
            run()
        torch.cuda.synchronize()
    fam = collections.Counter()
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            fam[family(ev.name)] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    return {k: v / a.reps / 1e3 for k, v in fam.items()}     # ms per step, all ranks


out = {"model": a.model, "P": P, "layers": a.layers, "batch": B, "ctx": Lc}
# loopback: rank 0's kernels alone
lb = setup(0, dl.Comm.loopback(0, P))
fam = profile(lambda: step(lb))
out["loopback"] = {k: round(v, 4) for k, v in fam.items()}
out["loopback"]["total"] = round(sum(fam.values()), 4)
del lb
torch.cuda.empty_cache()
need = dl.dl_block_window_bytes(cfg, P)
for name, window in (("collective", 256), ("fused", need)):
    comms = dl.Comm.group(P, window)
    states = [setup(r, comms[r]) for r in range(P)]
    torch.cuda.synchronize()
    fam = profile(lambda: dl.run_ranks(lambda r, _s: step(states[r]), P))
    per_rank = {k: round(v / P, 4) for k, v in fam.items()}
    per_rank["total"] = round(sum(fam.values()) / P, 4)
    out[name] = per_rank
    del states
    for c in comms:
        c.close()
    torch.cuda.empty_cache()
out["unit"] = "GPU ms per rank per step of these layers (CUPTI kernel durations / P)"
out["window_bytes"] = need
print(json.dumps(out))
