"""Debug driver: one multi-rank block call (group communicator), prints OK / error.
usage: python tools/mr_debug.py MODE P T LAYOUT"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17709_b200 as dl  # noqa: E402
from synthetic import ModelShape, block_ranks, gen_block_weights, gen_normal  # noqa: E402

mode, P, T, layout = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
s = ModelShape("mr", h=2048, n_heads=16, n_kv_heads=8, head_dim=128, m=4096, n_layers=2, vocab=10)
rk = block_ranks(s, 0.4)
if os.environ.get("RANKS"):
    rk.update(eval(os.environ["RANKS"]))
w = gen_block_weights(s, rk, 3, 0)
if os.environ.get("NOCOMM"):
    comms = [None]
elif os.environ.get("LOOP"):
    comms = [dl.Comm.loopback(r, P) for r in range(P)]
else:
    comms = dl.Comm.group(P, 8 << 20)
hk = s.n_kv_heads // P


def body(r, st):
    wd = dl.BlockWeights({a: b.cuda() for a, b in w.items()}, world=P, rank=r, layout=layout)
    x = gen_normal((T, s.h), 1.0, 500 + T, dtype=torch.bfloat16).cuda()
    cfg = dl.make_block_config(s, rk, max_tokens=T, max_seqs=1 if mode == "prefill" else T, layout=layout)
    ws = torch.zeros(dl.dl_block_workspace(cfg, P), dtype=torch.uint8, device="cuda")
    if mode == "prefill":
        kc = torch.zeros(1, hk, T, s.head_dim, dtype=torch.bfloat16, device="cuda")
        vc = torch.zeros_like(kc)
        pos = torch.arange(T, dtype=torch.int32, device="cuda")
        cu = torch.tensor([0, T], dtype=torch.int32, device="cuda")
        dl.dl_decomposed_block_forward(cfg, wd, x, pos, cu, 1, dl.DL_PREFILL, kc, vc,
                                       torch.zeros(1, dtype=torch.int32, device="cuda"), comms[r], ws)
    else:
        kc = torch.zeros(T, hk, 32, s.head_dim, dtype=torch.bfloat16, device="cuda")
        vc = torch.zeros_like(kc)
        cl = torch.full((T,), 5, dtype=torch.int32, device="cuda")
        dl.dl_decomposed_block_forward(cfg, wd, x, cl, None, T, dl.DL_DECODE, kc, vc, cl, comms[r], ws)
    print(f"rank {r} enqueued {dl.dl_launch_count()}", flush=True)
    torch.cuda.current_stream().synchronize()
    print(f"rank {r} done", flush=True)
    return x.float().norm().item()


print(mode, P, T, layout, dl.run_ranks(body, P), "OK", flush=True)
