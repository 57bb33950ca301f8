"""Per-rank decode-step compute of TP = P on ONE B200 (measurement only).

A loopback communicator (dl_comm_create_loopback) gives the library P-rank
shapes while the collectives become local copies, so each configuration runs
exactly the kernels one rank runs in a real TP = P step (its shards, its local
heads, the layout's replicated A matrices) -- everything except the NVLink
transfers.  Prints per-rank step time and the per-rank collective payload of
each layout (the bytes a real run moves over NVLink).

python tools/tp_emulate.py [--layers 80] [--ps 1,2,4,8] [--layouts rp,deinfer]
                          [--model 70b|8b] [--ratios 0.4[,0.1,...]]   (BASELINE configs 3-5)
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_17709_b200 as dl
from paper_2604_17709_b200.model import DecomposedLlama
from synthetic import LLAMA3_70B, LLAMA3_8B, block_ranks, gen_block_weights, gen_normal

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=0, help="0: all layers of the model")
ap.add_argument("--ps", default="1,2,4,8")
ap.add_argument("--layouts", default="rp,deinfer")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--ctx", type=int, default=512)
ap.add_argument("--model", default="70b", choices=["70b", "8b"])
ap.add_argument("--ratios", default="0.4")
a = ap.parse_args()
s = LLAMA3_70B if a.model == "70b" else LLAMA3_8B
a.layers = a.layers or s.n_layers
dev = torch.device("cuda")
B = a.batch


def comm_elems(layout, P, rk):
    """Elements per token per layer this rank sends/receives in its collectives (bf16 unless noted)."""
    if P == 1:
        return 0
    if layout == "rp":   # RS(q|k|v) AG(att) AR(o) AR(gate|up) AR(down)
        return (s.h + 2 * s.h_kv) + s.h + s.h + 2 * s.m + s.h
    return (rk["q"] + rk["k"] + rk["v"]) + rk["o"] + (rk["gate"] + rk["up"]) + rk["down"]


res = []
import itertools
for ratio, layout, P in itertools.product([float(r) for r in a.ratios.split(",")], a.layouts.split(","),
                                         [int(p) for p in a.ps.split(",")]):
    rk = block_ranks(s, ratio)
    if True:
        lay = dl.DL_LAYOUT_DEINFER if layout == "deinfer" else dl.DL_LAYOUT_RANK_PARALLEL
        print(f"[tp_emulate] {layout} P={P}: {torch.cuda.memory_allocated() / 1e9:.1f} GB allocated", file=sys.stderr)
        comm = dl.Comm.loopback(0, P) if P > 1 else None
        vloc = s.vocab // P
        m = DecomposedLlama(s, rk, (gen_block_weights(s, rk, 3, i, device=dev) for i in range(a.layers)),
                            gen_normal((s.vocab, s.h), 1.0, 1, device=dev, dtype=torch.bfloat16),
                            torch.ones(s.h, dtype=torch.bfloat16, device=dev),
                            gen_normal((vloc, s.h), s.h ** -0.5, 2, device=dev, dtype=torch.bfloat16), batch=B,
                            max_seq=a.ctx + 1, comm=comm, device=dev, layout=lay)
        m.cache.normal_()
        m.cache_lens.fill_(a.ctx)
        torch.cuda.synchronize()       # setup ran on the default stream; the step runs on `st`
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            m.decode_step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            m.decode_step()
        with torch.cuda.stream(st):
            for _ in range(3):
                g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        with torch.cuda.stream(st):
            e0.record(st)
            for _ in range(a.steps):
                g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        cb = comm_elems(layout, P, rk) * B * a.layers * 2
        weights_gb = sum(t.numel() * t.element_size() for lw in m.layers for t in lw.tensors.values()) / 1e9
        wbytes = sum(t.numel() * t.element_size() for lw in m.layers for t in lw.tensors.values())
        kvb = m.cache.numel() * m.cache.element_size() * a.ctx / (a.ctx + 1)
        lmb = m.lm_head.numel() * 2
        hbm_ms = (wbytes + kvb + lmb) / 6553.6e9 * 1e3      # MEASURED_PEAKS hbm_gbs
        r = {"model": a.model, "ratio": ratio, "ranks": rk, "layout": layout, "P": P, "layers": a.layers,
             "batch": B, "ctx": a.ctx, "rank_ms_per_step": round(ms, 3),
             "rank_tok_s": round(B / ms * 1e3, 1), "hbm_ideal_ms": round(hbm_ms, 3),
             "frac_of_hbm": round(hbm_ms / ms, 3),
             "rank_weight_gb": round(weights_gb, 2), "collective_mb_per_step_per_rank": round(cb / 1e6, 1)}
        res.append(r)
        print(json.dumps(r), flush=True)
        del m, g
        if comm:
            comm.close()
        torch.cuda.empty_cache()
