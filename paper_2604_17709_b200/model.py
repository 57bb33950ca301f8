"""Whole-model decode / prefill steps of a rank-sharded decomposed LLaMA-3,
driving only this library's C ABI (embedding gather, decomposed blocks,
final RMSNorm, dense LM head).  PyTorch supplies device memory, streams,
CUDA-Graph capture and (for the vocab-sharded logits) the all-gather.
"""
from __future__ import annotations

import torch

from . import _lib as L


class DecomposedLlama:
    """Rank `comm.rank` of a TP=`comm.world` decomposed LLaMA-3 (world 1 if comm is None).

    layer_weights: iterable of per-layer dicts {A_<m>, B_<m>, g_attn, g_mlp}
    (full, unsharded factors on this device; sharded here and then dropped).
    ranks: one dict for every layer, or a list of per-layer dicts (variadic
    per-layer ranks); each layer then gets its own block config and
    the workspaces are sized for the largest.
    embed [V x h], final_norm [h], lm_head_local [V/P x h] (this rank's vocab rows).
    """

    def __init__(self, shape, ranks: dict, layer_weights, embed: torch.Tensor, final_norm: torch.Tensor,
                 lm_head_local: torch.Tensor, batch: int, max_seq: int, prefill_tokens: int = 0,
                 comm: L.Comm | None = None, device="cuda", layout: int = L.DL_LAYOUT_RANK_PARALLEL,
                 kv: str = "full", kv_block_size: int = 16, prefill_chunks: int = 1):
        """kv = "full": head-major post-RoPE K/V cache; "lowrank": paged latent cache
         with the two-stage reconstruction (decode only; uniform ranks).
        prefill_chunks > 1: the prefill sequence is split into that many chunks that run
        as a wavefront over (layer, chunk) on one stream per chunk (prefill_step)."""
        self.shape, self.ranks, self.comm, self.layout, self.kv_mode = shape, ranks, comm, layout, kv
        self.world = comm.world if comm else 1
        self.rank = comm.rank if comm else 0
        self.device = torch.device(device)
        self.batch, self.max_seq = batch, max_seq
        self.layers = []
        for w in layer_weights:
            self.layers.append(L.BlockWeights(w, self.world, self.rank, layout=layout))
            del w
        self.embed, self.final_norm, self.lm_head = embed, final_norm, lm_head_local
        s = shape
        hk_loc = s.n_kv_heads // self.world
        nl = len(self.layers)
        bf = torch.bfloat16
        per_layer = ranks if isinstance(ranks, (list, tuple)) else [ranks] * nl
        if kv == "lowrank":
            self.cache = None
            bs = kv_block_size
            mbps = -(-max_seq // bs)
            nblocks = batch * mbps
            self.kv_layers = []
            for r in per_layer:
                self.kv_layers.append(L.LowRankKVCache(r["k"], r["v"], hk_loc * s.head_dim, nblocks, bs, batch, mbps,
                                                       cap_blocks=nblocks, device=self.device,
                                                       shared=self.kv_layers[0] if self.kv_layers else None))
            # default allocation: each sequence owns a contiguous range of blocks
            self.kv_tables_host = torch.arange(nblocks, dtype=torch.int32).view(batch, mbps).numpy()
            self.kv_layers[0].block_tables.copy_(torch.from_numpy(self.kv_tables_host))
        elif kv == "full":
            self.cache = torch.zeros((nl, 2, batch, hk_loc, max_seq, s.head_dim), dtype=bf, device=self.device)
        else:
            raise ValueError(f"kv mode {kv!r}")
        if len(per_layer) != nl:
            raise ValueError(f"{len(per_layer)} rank dicts for {nl} layers")
        # a workspace's layout is tied to its config (include/dl.h): one per distinct rank set
        keys = [tuple(sorted(r.items())) for r in per_layer]
        self.dec_cfgs = [L.make_block_config(s, r, max_tokens=batch, max_seqs=batch, layout=layout)
                         for r in per_layer]
        self.dec_cfg = self.dec_cfgs[0]
        dws = {}
        for k, c in zip(keys, self.dec_cfgs):
            if k not in dws:
                dws[k] = torch.zeros(L.dl_block_workspace(c, self.world), dtype=torch.uint8, device=self.device)
        self.dec_wss = [dws[k] for k in keys]
        self.dec_ws = self.dec_wss[0]
        # uniform ranks, full KV: one stack call (cross-block residual + norm fusion)
        self.stack = None
        import os
        if kv == "full" and len(dws) == 1 and nl > 0 and not os.environ.get("DL_NO_STACK"):   # A/B switch
            self.stack = L.StackArgs(self.layers, [self.cache[i, 0] for i in range(nl)],
                                     [self.cache[i, 1] for i in range(nl)])
        # decode-step static buffers
        self.ids = torch.zeros(batch, dtype=torch.int32, device=self.device)
        self.cache_lens = torch.zeros(batch, dtype=torch.int32, device=self.device)
        self.x = torch.zeros(batch, s.h, dtype=bf, device=self.device)
        self.xn = torch.zeros(batch, s.h, dtype=bf, device=self.device)
        vloc = lm_head_local.shape[0]
        self.logits_local = torch.zeros(batch, vloc, dtype=bf, device=self.device)
        self.logits = torch.zeros(self.world, batch, vloc, dtype=bf, device=self.device)
        self.next_ids = torch.zeros(batch, dtype=torch.int32, device=self.device)   # greedy tokens of the step
        self.prefill_tokens = prefill_tokens
        if prefill_tokens:
            self.pre_cfgs = [L.make_block_config(s, r, max_tokens=prefill_tokens, max_seqs=1, layout=layout)
                             for r in per_layer]
            self.pre_cfg = self.pre_cfgs[0]
            pws = {}
            for k, c in zip(keys, self.pre_cfgs):
                if k not in pws:
                    pws[k] = torch.zeros(L.dl_block_workspace(c, self.world), dtype=torch.uint8,
                                         device=self.device)
            self.pre_wss = [pws[k] for k in keys]
            self.pre_ws = self.pre_wss[0]
            self.pre_cache = torch.zeros((nl, 2, 1, hk_loc, prefill_tokens, s.head_dim), dtype=bf,
                                         device=self.device)
            self.pre_ids = torch.zeros(prefill_tokens, dtype=torch.int32, device=self.device)
            self.pre_pos = torch.arange(prefill_tokens, dtype=torch.int32, device=self.device)
            self.pre_cu = torch.tensor([0, prefill_tokens], dtype=torch.int32, device=self.device)
            self.pre_lens = torch.zeros(1, dtype=torch.int32, device=self.device)
            self.pre_last = torch.tensor([prefill_tokens - 1], dtype=torch.int32, device=self.device)
            self.pre_x = torch.zeros(prefill_tokens, s.h, dtype=bf, device=self.device)
            self.pre_xl = torch.zeros(1, s.h, dtype=bf, device=self.device)
            self.pre_xn = torch.zeros(1, s.h, dtype=bf, device=self.device)
            self.pre_logits = torch.zeros(1, vloc, dtype=bf, device=self.device)
            # chunked wavefront (prefill_chunks > 1): chunk c = tokens [c*Tc, (c+1)*Tc) of the
            # sequence, continuing the cached prefix of chunks < c (cache_lens = c*Tc), with its
            # own workspaces and stream
            C = max(1, int(prefill_chunks))
            if prefill_tokens % C:
                raise ValueError("prefill_chunks must divide prefill_tokens")
            self.pre_chunks = C
            if C > 1:
                Tc = prefill_tokens // C
                self.chunk_cfgs = [L.make_block_config(s, r, max_tokens=Tc, max_seqs=1, layout=layout)
                                   for r in per_layer]
                self.chunk_wss = []
                for c in range(C):
                    cws = {}
                    for k, cf in zip(keys, self.chunk_cfgs):
                        if k not in cws:
                            cws[k] = torch.zeros(L.dl_block_workspace(cf, self.world), dtype=torch.uint8,
                                                 device=self.device)
                    self.chunk_wss.append([cws[k] for k in keys])
                self.chunk_cu = torch.tensor([0, Tc], dtype=torch.int32, device=self.device)
                self.chunk_lens = [torch.tensor([c * Tc], dtype=torch.int32, device=self.device) for c in range(C)]
                self.chunk_streams = [None] + [torch.cuda.Stream(device=self.device) for _ in range(C - 1)]

    def kv_prepare(self, cache_lens_host, tables_host=None):
        """Preparation stage of the low-rank KV cache (host; outside the graph replay):
        plan the squeeze of every sequence's blocks for a step appending at cache_lens."""
        if tables_host is not None:
            self.kv_tables_host = tables_host
            self.kv_layers[0].block_tables.copy_(torch.as_tensor(tables_host, dtype=torch.int32))
        return self.kv_layers[0].prepare(self.kv_tables_host, [int(c) + 1 for c in cache_lens_host])

    # one decode token for each of the `batch` sequences, at position cache_lens[b]
    def decode_step(self):
        s = self.shape
        L.dl_embedding(self.embed, self.ids, self.x)
        if self.kv_mode == "lowrank":
            for i, lw in enumerate(self.layers):
                L.dl_decomposed_block_forward_kvlr(self.dec_cfgs[i], lw, self.x, self.cache_lens, self.kv_layers[i],
                                                   self.cache_lens, self.comm, self.dec_wss[i])
        if self.kv_mode == "full" and self.stack is not None:
            L.dl_decomposed_stack_forward(self.dec_cfg, self.stack, self.x, self.cache_lens, None, self.batch,
                                          L.DL_DECODE, self.cache_lens, self.comm, self.dec_ws)
        for i, lw in enumerate(self.layers if self.kv_mode == "full" and self.stack is None else ()):
            L.dl_decomposed_block_forward(self.dec_cfgs[i], lw, self.x, self.cache_lens, None, self.batch, L.DL_DECODE,
                                          self.cache[i, 0], self.cache[i, 1], self.cache_lens, self.comm,
                                          self.dec_wss[i])
        L.dl_rmsnorm(self.x, self.final_norm, self.xn, s.rms_eps)
        L.dl_dense(self.xn, self.lm_head, self.logits_local)
        if self.world > 1 and getattr(self.comm, "is_loopback", False):
            self.logits[self.rank].copy_(self.logits_local)      # measurement-only emulation
        elif self.world > 1:
            import torch.distributed as dist
            dist.all_gather_into_tensor(self.logits, self.logits_local)
        # greedy next token over the (gathered) vocab shards, on the device
        L.dl_argmax(self.logits_local if self.world == 1 else self.logits, self.next_ids)
        return self.logits_local if self.world == 1 else self.logits

    # one sequence of prefill_tokens tokens; logits of its last token
    def prefill_step(self):
        s = self.shape
        T = self.prefill_tokens
        L.dl_embedding(self.embed, self.pre_ids, self.pre_x)
        if self.pre_chunks > 1:
            self._prefill_wavefront()
        for i, lw in enumerate(self.layers if self.pre_chunks == 1 else ()):
            L.dl_decomposed_block_forward(self.pre_cfgs[i], lw, self.pre_x, self.pre_pos, self.pre_cu, 1, L.DL_PREFILL,
                                          self.pre_cache[i, 0], self.pre_cache[i, 1], self.pre_lens, self.comm,
                                          self.pre_wss[i])
        L.dl_embedding(self.pre_x, self.pre_last, self.pre_xl)        # row gather of the last token
        L.dl_rmsnorm(self.pre_xl, self.final_norm, self.pre_xn, s.rms_eps)
        L.dl_dense(self.pre_xn, self.lm_head, self.pre_logits)
        del T
        return self.pre_logits

    def _prefill_wavefront(self):
        """Block (layer i, chunk c) runs on chunk c's stream after block (i, c - 1) -- its keys
        and values are the cached prefix chunk c attends to (chunked prefill, include/dl.h) --
        and after block (i - 1, c) (stream order).  Block (i, c) therefore overlaps block
        (i + 1, c - 1): one chunk's TP collectives (NCCL on its stream) run while another
        chunk's GEMMs stream (the communication / computation overlap of PAPER.md:224), and on
        one GPU the second stream's kernels fill the SMs the first stream's small kernels and
        GEMM tails leave idle.  Capturable in a CUDA graph (fork / join through events)."""
        C = self.pre_chunks
        Tc = self.prefill_tokens // C
        main = torch.cuda.current_stream(self.device)
        streams = [main] + self.chunk_streams[1:]
        fork = torch.cuda.Event()
        fork.record(main)
        for st in streams[1:]:
            st.wait_event(fork)
        done = [[None] * C for _ in self.layers]
        for i, lw in enumerate(self.layers):
            for c in range(C):
                st = streams[c]
                if c > 0:
                    st.wait_event(done[i][c - 1])
                rows = slice(c * Tc, (c + 1) * Tc)
                with torch.cuda.stream(st):
                    L.dl_decomposed_block_forward(self.chunk_cfgs[i], lw, self.pre_x[rows], self.pre_pos[rows],
                                                  self.chunk_cu, 1, L.DL_PREFILL, self.pre_cache[i, 0],
                                                  self.pre_cache[i, 1], self.chunk_lens[c], self.comm,
                                                  self.chunk_wss[c][i], stream=st)
                ev = torch.cuda.Event()
                ev.record(st)
                done[i][c] = ev
        for c in range(1, C):   # join: the last token's row comes from the last chunk
            main.wait_event(done[-1][c])

