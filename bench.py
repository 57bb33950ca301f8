#!/usr/bin/env python
"""Benchmark: decomposed LLaMA-3-70B (random init, 40% compression) tokens/s on
N B200s (tensor parallel over the rank dimension), decode and prefill.

    python bench.py [--gpus N --steps K --warmup W]            # our arm
    python bench.py --impl reference ...                       # fp64 CPU oracle arm
    torchrun --nproc-per-node N bench.py --gpus N ...          # TP = N

A "step" is one full-model decode step: embedding -> 80 decomposed blocks
(every row of SURVEY.md section 8(a): RMSNorm, stage-1/stage-2 low-rank
chains, TP reductions, RoPE + cache append, causal GQA attention, SiLU*up,
residual) -> final RMSNorm -> LM head, for a batch of 64 sequences at
context 512, captured in one CUDA Graph.  `value` is decode tokens/s of the
whole job; the prefill line (one 2048-token sequence) rides in "prefill".
Weights (~115 GB at TP=1) and caches are larger than L2, so every step
streams from HBM (no L2 flush needed; stated in config).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decomposed LLaMA-3-70B tokens/s (decode, prefill) at 1/2/4/8 B200; % roofline"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--model", default="70b", choices=["70b", "8b"])
    p.add_argument("--ratio", type=float, default=0.4)
    p.add_argument("--batch", type=int, default=64)
    p.add_argument("--ctx", type=int, default=512)
    p.add_argument("--prefill-tokens", type=int, default=2048)
    p.add_argument("--prefill-steps", type=int, default=3)
    p.add_argument("--prefill-chunks", type=int, default=1,
                   help="prefill as a wavefront of this many chunks on as many streams (model.py)")
    p.add_argument("--layers", type=int, default=0, help="debug only: fewer layers (invalid for reporting)")
    p.add_argument("--layout", default="rp", choices=["rp", "deinfer"],
                   help="TP sharding layout: rank-parallel (north star) or DeInfer low-rank communication")
    p.add_argument("--kv", default="full", choices=["full", "lowrank"],
                   help="decode KV cache: post-RoPE K/V, or the paged low-rank (latent) cache with the "
                        "two-stage reconstruction (P:111, P:219-237)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--tp-window", action="store_true",
                   help="TP > 1: fused epilogue reductions through CUDA-IPC symmetric windows over NVLink "
                        "(include/dl.h dl_comm_window_*; verified with two processes on one GPU, not yet on "
                        "a multi-GPU node) instead of NCCL collectives")
    p.add_argument("--cpu-sample-seqs", type=int, default=64)
    return p.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk["hbm_gbs"], pk["bf16_tflops"], pk.get("bf16_tflops_sustained", pk["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


def collective_census(shape, ranks, n_layers, world, args):
    """Collectives one rank issues per decode step and their bf16 payload:
    rank-parallel RS(q|k|v) + AG(attention) + AR(o) + AR(gate|up) + AR(down) per layer;
    DeInfer AG(latent q|k|v) + AR(latent o) + AG(latent gate|up) + AR(latent down); plus the
    logits all-gather."""
    if world == 1:
        return {"count_per_step": 0, "payload_mb_per_step": 0.0}
    if args.layout == "rp":
        per_tok = (shape.h + 2 * shape.h_kv) + shape.h + shape.h + 2 * shape.m + shape.h
        ar = shape.h + 2 * shape.m + shape.h          # all-reduced elements (cost 2n on a ring)
        n_coll = 5
    else:
        per_tok = (ranks["q"] + ranks["k"] + ranks["v"]) + ranks["o"] + (ranks["gate"] + ranks["up"]) + ranks["down"]
        ar = ranks["o"] + ranks["down"]
        n_coll = 4
    payload = (per_tok * n_layers + shape.vocab) * args.batch * 2
    return {"count_per_step": n_coll * n_layers + 1, "collectives_per_layer": n_coll,
            "units_per_token_layer_nvls": per_tok, "units_per_token_layer_ring": per_tok + ar,
            "payload_mb_per_step": payload / 1e6, "layout": args.layout}


def load_traffic():
    """ncu DRAM bytes of the dominant launch (profiles/traffic.json, from one --set full capture)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = f"/tmp/dl_clocks_{os.getpid()}.csv"

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
            rows = [[c.strip() for c in r] for r in rows if len(r) >= 8]
            if not rows:
                return out
            sm = [float(r[0]) for r in rows]
            out["sm_mhz"] = statistics.median(sm)
            out["sm_max_mhz"] = float(rows[0][1])
            out["samples"] = len(rows)
            out["power_w_max"] = max(float(r[2]) for r in rows if r[2] not in ("[N/A]", ""))
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for i, n in enumerate(names):
                if any(r[4 + i].lower() == "active" for r in rows):
                    out["reasons"].append(n)
        except Exception as e:  # noqa: BLE001
            out["error"] = str(e)
        return out


# ---------------------------------------------------------------------------
def cpu_baseline(shape, ranks, ctx: int, sample_seqs: int, layer0_w=None, min_s: float = 10.0):
    """The fp64 oracle, as it stands, on one decomposed layer for `sample_seqs`
    decode tokens (context ctx), scaled to full-model tokens/s (÷ n_layers)."""
    import numpy as np
    import torch

    import oracle
    from synthetic import gen_block_weights, gen_normal
    oracle.build()
    if layer0_w is None:
        layer0_w = gen_block_weights(shape, ranks, 3, 0, device="cpu")
    w = {k: v.detach().to("cpu") for k, v in layer0_w.items()}
    cfg = oracle.BlockCfg(shape.h, shape.n_heads, shape.n_kv_heads, shape.head_dim, shape.m, ranks["q"],
                          ranks["k"], ranks["v"], ranks["o"], ranks["gate"], ranks["up"], ranks["down"],
                          rope_theta=shape.rope_theta, rms_eps=shape.rms_eps)
    S = sample_seqs
    x = gen_normal((S, shape.h), 1.0, 41)
    kc = gen_normal((S, ctx + 1, shape.h_kv), 1.0, 42, dtype=torch.bfloat16)
    vc = gen_normal((S, ctx + 1, shape.h_kv), 1.0, 43, dtype=torch.bfloat16)
    w64 = {k: v.double().numpy() for k, v in w.items()}
    t0 = time.perf_counter()
    reps = 0
    while True:      # repeat the one-layer sample until >= min_s of CPU work
        oracle.block_decode(cfg, w64, x, kc, vc, np.full(S, ctx, dtype=np.int32))
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= min_s:
            break
    return {"value": S * reps / (dt * shape.n_layers), "unit": "tokens/s", "cores": oracle.num_threads(),
            "kind": "oracle",
            "sample": f"{reps} x (1 of {shape.n_layers} decomposed layers, {S} decode tokens at context {ctx}), "
                      f"fp64; {dt:.2f} s, scaled x{shape.n_layers} layers"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synthetic import LLAMA3_70B, LLAMA3_8B, block_ranks
    shape = LLAMA3_70B if args.model == "70b" else LLAMA3_8B
    ranks = block_ranks(shape, args.ratio)
    from synthetic import gen_block_weights
    w = gen_block_weights(shape, ranks, 3, 0, device="cpu")
    S = max(1, min(args.cpu_sample_seqs, args.batch))
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(shape, ranks, args.ctx, S, w, min_s=2.0)
        if i >= args.warmup:
            vals.append(r["value"])
    v = statistics.mean(vals)
    step_ms = args.batch / v * 1e3
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded random-init factors)",
            "impl": "reference",
            "config": {"workload": f"llama3-{args.model} @{int(args.ratio * 100)}% decode B={args.batch} "
                                   f"ctx={args.ctx}", "global_batch": args.batch, "seq_len": args.ctx,
                       "parallelism": "cpu"},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": r["cores"], "kind": "oracle",
                             "sample": r["sample"]},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2604_17709_b200 as dl
    from paper_2604_17709_b200.model import DecomposedLlama
    from synthetic import LLAMA3_70B, LLAMA3_8B, block_ranks, gen_block_weights, gen_normal

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        comm = dl.Comm.from_process_group()
    dl.load()
    if not dl.dl_device_ok():
        raise SystemExit("libdl.so: no sm_100 device")
    shape = LLAMA3_70B if args.model == "70b" else LLAMA3_8B
    ranks = block_ranks(shape, args.ratio)
    n_layers = args.layers or shape.n_layers
    cfg_id = 3 if args.model == "70b" else 2

    t_init = time.time()
    keep0 = {}

    def layer_iter():
        for li in range(n_layers):
            w = gen_block_weights(shape, ranks, cfg_id, li, device=dev)
            if li == 0 and rank == 0 and world == 1:
                keep0["w"] = {k: v.to("cpu") for k, v in w.items()}
            yield w

    vloc = shape.vocab // world
    embed = gen_normal((shape.vocab, shape.h), 1.0, 7001, device=dev, dtype=torch.bfloat16)
    lm_full_rows = gen_normal((shape.vocab, shape.h), shape.h ** -0.5, 7002, device=dev, dtype=torch.bfloat16)
    lm_head = lm_full_rows[rank * vloc:(rank + 1) * vloc].clone()
    del lm_full_rows
    final_norm = torch.ones(shape.h, dtype=torch.bfloat16, device=dev)
    # TP > 1, rank-parallel: a symmetric window per rank mapped into every peer (CUDA IPC over
    # NVLink) so the decode path's reductions run inside the stage-2 epilogues
    tp_coll = "nccl" if world > 1 else "none"
    if world > 1 and args.layout == "rp" and args.tp_window:
        # every rank must take the same path: agree on success after each stage
        def agree(flag):
            t = torch.tensor([1 if flag else 0], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            return bool(t.item())
        err, hs = "", None
        try:
            wcfg = dl.make_block_config(shape, ranks, max_tokens=args.batch, max_seqs=args.batch)
            comm.window_alloc(dl.dl_block_window_bytes(wcfg, world))
            hs = [None] * world
            dist.all_gather_object(hs, comm.window_handle())
        except Exception as e:   # noqa: BLE001
            err = str(e)[:120]
        if agree(not err):
            try:
                comm.window_connect(hs)
            except Exception as e:   # noqa: BLE001
                err = str(e)[:120]
            if not agree(not err):
                raise SystemExit(f"TP window: connect failed on some rank ({err or 'peer'}); rerun without --tp-window")
            tp_coll = "fused-window (decode) + nccl (prefill)"
        else:
            tp_coll = f"nccl (window setup failed: {err or 'on a peer'})"
    model = DecomposedLlama(shape, ranks, layer_iter(), embed, final_norm, lm_head, batch=args.batch,
                            max_seq=args.ctx + 1, prefill_tokens=args.prefill_tokens, comm=comm, device=dev,
                            prefill_chunks=args.prefill_chunks,
                            layout=dl.DL_LAYOUT_DEINFER if args.layout == "deinfer" else dl.DL_LAYOUT_RANK_PARALLEL,
                            kv=args.kv)
    # context: ctx tokens already cached per sequence (random K/V), fixed for every step
    model.cache_lens.fill_(args.ctx)
    if args.kv == "lowrank":
        for kvl in model.kv_layers:            # latent history N(0, 1), positions 0..ctx-1
            kvl.pool.normal_()
            kvl.slot_pos.copy_(torch.arange(kvl.slot_pos.numel(), device=dev, dtype=torch.int32)
                               % (model.kv_layers[0].block_tables.shape[1] * kvl.block_size))
        model.kv_prepare([args.ctx] * args.batch)      # preparation stage (host), before capture
    else:
        model.cache.normal_()
    g = torch.Generator(device=dev)
    g.manual_seed(7003)
    model.ids.copy_(torch.randint(0, shape.vocab, (args.batch,), generator=g, device=dev, dtype=torch.int32))
    if args.prefill_tokens:
        model.pre_ids.copy_(torch.randint(0, shape.vocab, (args.prefill_tokens,), generator=g, device=dev,
                                          dtype=torch.int32))
    torch.cuda.synchronize()
    init_s = time.time() - t_init
    print(f"[bench] init {init_s:.1f}s, {torch.cuda.memory_allocated(dev) / 1e9:.1f} GB allocated", file=sys.stderr,
          flush=True)

    stream = torch.cuda.Stream(device=dev)
    hbm_gbs, bf16_burst, bf16_sust, peak_src = load_peaks()

    def capture(fn, n_gemm_cap=0):
        """CUDA-Graph capture of one step.  n_gemm_cap > 0: the library records a CUDA
        event pair around each tcgen05 GEMM (event nodes inside the graph); that graph is
        only replayed for the per-kernel roofline, the timed graph has no event nodes
        (they would break the programmatic-dependent-launch overlap between kernels)."""
        with torch.cuda.stream(stream):
            fn()                                   # eager warm-up (sets kernel attributes)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        c0 = dl.dl_launch_count()
        if n_gemm_cap:
            dl.dl_profile_begin(n_gemm_cap)
        with torch.cuda.graph(graph, stream=stream):
            fn()
        if n_gemm_cap:
            dl.dl_profile_end()
        launches = dl.dl_launch_count() - c0
        return graph, launches

    def gemm_in_graph(fn, n_layers, roof):
        """The GEMM class timed inside the un-instrumented step: the graph is captured with
        the per-CTA debug timeline on (globaltimer at each CTA's entry and epilogue end,
        dl_debug_gemm_trace), replayed, and the union of the GEMM launches' [first entry,
        last epilogue end] spans is the time at least one GEMM was streaming; no events sit
        between the launches, so PDL overlap is kept (the event-timed class figure above is a
        lower bound for that reason).  Attention launches share the buffer but never write
        the accumulator-ready field, which tells them apart."""
        from paper_2604_17709_b200 import _lib
        slots = 32 * n_layers + 64
        buf = torch.zeros(slots * 148 * 8, dtype=torch.int64, device=dev)
        _lib.dl_debug_gemm_trace(buf)   # slots are assigned at capture, the buffer is read at replay
        try:
            g, _ = capture(fn)
            for _ in range(2):
                buf.zero_()
                with torch.cuda.stream(stream):
                    g.replay()
                torch.cuda.synchronize()
        finally:
            _lib.dl_debug_gemm_trace(None)
        spans = []
        t = buf.view(slots, 148, 8).cpu()
        for i in range(slots):
            c = t[i]
            used = c[:, 0] > 0
            if not used.any() or not (c[:, 5] > 2 ** 48).any():   # GEMM slots: field 5 is a timestamp
                continue
            c = c[used]
            spans.append((int(c[:, 0].min()), int(c[:, 6].max())))
        del g
        spans.sort()
        union, cur0, cur1 = 0, None, None
        for a0, a1 in spans:
            if cur1 is None or a0 > cur1:
                if cur1 is not None:
                    union += cur1 - cur0
                cur0, cur1 = a0, a1
            else:
                cur1 = max(cur1, a1)
        if cur1 is not None:
            union += cur1 - cur0
        ms = union / 1e6
        byt = roof["achieved"] * 1e9 * roof["kernel_ms_per_step"] * 1e-3   # the class's algorithmic bytes
        ach = byt / (ms * 1e-3) / 1e9
        return {"achieved": ach, "frac": ach / roof["peak"], "launches": len(spans), "union_ms_per_step": ms,
                "method": "union of the GEMM launches' in-graph spans (per-CTA globaltimer trace), "
                          "same algorithmic bytes as the class figure"}

    def kernel_timing(fn, n_gemm_cap, replays=2):
        """Replay the instrumented graph; per-launch GEMM event times of the last replay."""
        g, _ = capture(fn, n_gemm_cap)
        with torch.cuda.stream(stream):
            for _ in range(replays):
                g.replay()
        torch.cuda.synchronize()
        return g

    def timed(graph, steps, warmup):
        with torch.cuda.stream(stream):
            for _ in range(warmup):
                graph.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk, torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(steps):
                graph.replay()
            e1.record(stream)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms, clk.summary()

    def graph_ms(graph, steps):
        with torch.cuda.stream(stream):
            graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(steps):
                graph.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    def eager_ms(fn, steps):
        """Same step launched eagerly (no CUDA Graph): the graph on/off study of
        P:441-470 (Table 6), N2.  Device time between events on the stream."""
        with torch.cuda.stream(stream):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(steps):
                fn()
            e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    def gemm_roofline(kind, bound, extra_kinds=()):
        """kind 0/1 = wide / swap-AB GEMM launches; extra_kinds (2 = DP+SK tail finalize)
        add their time (no algorithmic work of their own) to the GEMM class."""
        recs = [r for r in dl.dl_profile_records() if r[3] == kind or r[3] in extra_kinds]
        if not recs:
            return None
        ms = sum(r[0] for r in recs)
        if bound == "hbm":
            ach = sum(r[1] for r in recs) / (ms * 1e-3) / 1e9
            peak = hbm_gbs
            unit = "GB/s"
        else:
            ach = sum(r[2] for r in recs) / (ms * 1e-3) / 1e12
            peak = bf16_sust
            unit = "TFLOP/s"
        tr = load_traffic().get("decode" if bound == "hbm" else "prefill", {})
        return {"bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                "traffic": tr.get("dram_bytes"), "traffic_launch": tr.get("launch"),
                "traffic_algorithmic_bytes": tr.get("algorithmic_bytes"), "traffic_source": tr.get("source"),
                "kernel": "tc_gemm (tcgen05 low-rank stage-1/stage-2 GEMMs, all launches of one step)",
                "launches_per_step": len(recs), "kernel_ms_per_step": ms,
                "peak_source": f"{peak_src} ({'hbm_gbs' if bound == 'hbm' else 'bf16_tflops_sustained'})",
                # secondary denominator: the B200 data-sheet peak (8 TB/s HBM3e,
                # 2.25 PFLOP/s dense bf16)
                "frac_of_spec": ach / (8000.0 if bound == "hbm" else 2250.0),
                # a launch timed alone (events around it) is held against the burst figure
                "largest_launch": largest_launch(recs, bound, peak if bound == "hbm" else bf16_burst)}

    def largest_launch(recs, bound, peak):
        """The GEMM shape with the most time in the step (70B decode: gate|up stage 2), averaged
        over its launches: same event timing, same algorithmic count as the class."""
        key = (lambda r: r[1]) if bound == "hbm" else (lambda r: r[2])
        groups = {}
        for r in recs:
            if key(r) > 0:
                groups.setdefault(round(key(r) / 1e6), []).append(r)
        sel = max(groups.values(), key=lambda g: sum(r[0] for r in g))
        ms = sum(r[0] for r in sel) / len(sel)
        ach = (key(sel[0]) / (ms * 1e-3)) / (1e9 if bound == "hbm" else 1e12)
        return {"achieved": ach, "peak": peak, "frac": ach / peak, "launches": len(sel), "ms_per_launch": ms,
                "algorithmic_per_launch": key(sel[0]),
                "note": "CUDA events around each launch serialise it (no PDL overlap with its neighbours)"}

    # ---- decode -------------------------------------------------------------
    n_cap = 24 * n_layers + 16         # 8 GEMMs (+ up to 8 tail finalizes) per layer + LM head
    dgraph, dlaunch = capture(model.decode_step)
    dms, dclk = timed(dgraph, args.steps, args.warmup)
    step_ms = dms / args.steps
    dec_tps = args.batch / (step_ms * 1e-3)
    # graph on/off (N2): alternate short graph and eager runs so both see the same
    # power / clock state (a graph run followed by an eager run favours the later one)
    ge, ee = [], []
    for _ in range(3):
        ge.append(graph_ms(dgraph, min(args.steps, 5)))
        ee.append(eager_ms(model.decode_step, min(args.steps, 5)))
    ge.sort()
    ee.sort()
    graph_study = {"graph_ms_per_step": ge[1], "eager_ms_per_step": ee[1], "graph_speedup": ee[1] / ge[1],
                   "method": "median of 3 alternating 5-step runs each"}
    ig = kernel_timing(model.decode_step, n_cap)
    roof = gemm_roofline(1, "hbm")
    del ig
    roof["gemm_class_in_graph"] = gemm_in_graph(model.decode_step, n_layers, roof)
    # algorithmic bytes per decode step per GPU: factors + LM head + KV reads
    pl = (2 * shape.h * ranks["q"] + (shape.h + shape.h_kv) * (ranks["k"] + ranks["v"]) + 2 * shape.h * ranks["o"]
          + (shape.h + shape.m) * (ranks["gate"] + ranks["up"] + ranks["down"]))
    kv_row = 2 * shape.h_kv if args.kv == "full" else ranks["k"] + ranks["v"]   # cached elements per token
    step_bytes = (2 * (n_layers * pl + shape.vocab * shape.h) + args.batch * args.ctx * n_layers * kv_row * 2) \
        / world
    if args.layout == "deinfer" and world > 1:   # A_o and A_down are replicated on every rank
        step_bytes += 2 * n_layers * shape.h * (ranks["o"] + ranks["down"]) * (1 - 1 / world)
    step_gbs = step_bytes / (step_ms * 1e-3) / 1e9

    # ---- e2e: the autoregressive loop a serving user runs: H2D of the step's token ids
    # from pinned host memory, the captured step, D2H of its result (the greedy next token
    # of every sequence, argmax over the gathered logits on the device), and the host
    # round trip that turns those tokens into the next step's input -----------------
    ids_h = model.ids.to("cpu").pin_memory()
    out_dev = model.next_ids
    out_h = torch.empty(out_dev.shape, dtype=out_dev.dtype, pin_memory=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(args.steps):
            model.ids.copy_(ids_h, non_blocking=True)
            dgraph.replay()
            out_h.copy_(out_dev, non_blocking=True)
            stream.synchronize()        # the host needs this step's tokens ...
            ids_h.copy_(out_h)          # ... to feed them back as the next step's input
        e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # ---- prefill ------------------------------------------------------------
    prefill = None
    if args.prefill_tokens:
        pgraph, plaunch = capture(model.prefill_step)
        psteps = max(1, args.prefill_steps)
        pms, pclk = timed(pgraph, psteps, min(args.warmup, 3))
        p_step_ms = pms / psteps
        ig = kernel_timing(model.prefill_step, n_cap, replays=1)
        proof = gemm_roofline(0, "tensor", extra_kinds=(2,))
        del ig
        T = args.prefill_tokens
        pf = (2 * T * n_layers * pl + n_layers * 4 * (T * (T + 1) / 2) * shape.h) / world
        prefill = {"value": T / (p_step_ms * 1e-3), "unit": "tokens/s", "ms_per_step": p_step_ms,
                   "tokens_per_step": T, "steps": psteps, "algorithmic_tflop_per_gpu": pf / 1e12,
                   "achieved_tflops": pf / (p_step_ms * 1e-3) / 1e12,
                   "frac_of_bf16_sustained": pf / (p_step_ms * 1e-3) / 1e12 / bf16_sust,
                   "roofline": proof, "gpu_launches": plaunch * psteps, "clocks": pclk,
                   "chunks": args.prefill_chunks}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(shape, ranks, args.ctx, min(args.cpu_sample_seqs, args.batch), keep0.get("w"))
        except Exception as e:  # noqa: BLE001
            cpu = {"error": str(e)}

    if rank == 0:
        if roof is not None:
            roof["step_algorithmic_gbs"] = step_gbs
            roof["step_frac_of_hbm"] = step_gbs / hbm_gbs
        line = {"metric": METRIC, "value": dec_tps, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded random-init factors, random KV)",
                "config": {"workload": f"llama3-{args.model} @{int(round(args.ratio * 100))}% decode "
                                       f"B={args.batch} ctx={args.ctx} (+ prefill {args.prefill_tokens})",
                           "global_batch": args.batch, "seq_len": args.ctx, "parallelism": f"tp{world}",
                           "tp_layout": "deinfer" if args.layout == "deinfer" else "rank-parallel",
                           "tp_collectives": tp_coll,
                           "kv_cache": "post-RoPE K/V" if args.kv == "full" else
                           "paged low-rank latent, block 16, two-stage reconstruction",
                           "layers": n_layers, "ranks": ranks,
                           "l2": "inputs larger than L2 (weights+KV stream from HBM every step)",
                           "cuda_graph": True},
                "roofline": roof, "cpu_baseline": cpu,
                "e2e": {"value": args.batch / (e2e_ms * 1e-3), "unit": "tokens/s",
                        "h2d_bytes_per_step": ids_h.numel() * ids_h.element_size(),
                        "d2h_bytes_per_step": out_h.numel() * out_h.element_size()},
                "gpu_launches": dlaunch * args.steps, "clocks": dclk, "prefill": prefill,
                "graph_study": graph_study,
                "step_algorithmic_gb_per_gpu": step_bytes / 1e9, "init_s": init_s,
                "collectives": collective_census(shape, ranks, n_layers, world, args)}
        if args.layers:
            line["invalid"] = f"debug run with {n_layers} layers"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
