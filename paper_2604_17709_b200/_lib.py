"""ctypes binding of libdl.so (include/dl.h).  Argument marshalling only:
every computation runs in the library's sm_100a kernels.  There is no CPU
or PyTorch fallback -- if libdl.so is missing or the device is not an
sm_100 GPU, calls raise.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
# DL_LIBRARY=ab loads the instrumented build whose A/B timing switches read the
# environment (build.py); the default is the release library.
LIB_PATH = os.path.join(HERE, "libdl_ab.so" if os.environ.get("DL_LIBRARY") == "ab" else "libdl.so")

DL_F32, DL_BF16 = 0, 1
DL_REDUCE_NONE, DL_REDUCE_ALLREDUCE, DL_REDUCE_SCATTER = 0, 1, 2
DL_PREFILL, DL_DECODE = 0, 1
STATUS = {0: "DL_OK", 1: "DL_ERR_INVALID_ARG", 2: "DL_ERR_SHAPE", 3: "DL_ERR_RANK", 4: "DL_ERR_PARTITION",
          5: "DL_ERR_DTYPE", 6: "DL_ERR_ALIGN", 7: "DL_ERR_WORKSPACE", 8: "DL_ERR_CUDA", 9: "DL_ERR_NCCL",
          10: "DL_ERR_UNSUPPORTED"}
EXPORTS = ("dl_last_error", "dl_version", "dl_device_ok", "dl_comm_create", "dl_comm_destroy",
           "dl_lowrank_linear_workspace", "dl_lowrank_linear", "dl_tp_plan", "dl_tp_shard_factors",
           "dl_block_workspace", "dl_decomposed_block_forward", "dl_embedding", "dl_rmsnorm",
           "dl_dense_workspace", "dl_dense", "dl_launch_count", "dl_profile_begin", "dl_profile_end",
           "dl_profile_count", "dl_profile_get", "dl_debug_gemm_trace", "dl_deinfer_shard_factors",
           "dl_kv_prepare", "dl_decomposed_block_forward_kvlr", "dl_comm_create_loopback",
           "dl_decomposed_stack_forward", "dl_debug_ew_trace", "dl_debug_linear_gathered", "dl_argmax",
           "dl_comm_create_group", "dl_block_window_bytes", "dl_comm_create_peer", "dl_comm_window_alloc",
           "dl_comm_window_handle", "dl_comm_window_connect")


class DLError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
I = ctypes.c_int


class dl_block_config(ctypes.Structure):
    _fields_ = [(n, I64) for n in ("h", "n_heads", "n_kv_heads", "head_dim", "m", "rank_q", "rank_k", "rank_v",
                                   "rank_o", "rank_gate", "rank_up", "rank_down")] + \
               [("rope_theta", ctypes.c_float), ("rms_eps", ctypes.c_float), ("max_tokens", I64),
                ("max_seqs", I64), ("mlp_act", I32), ("no_rope", I32), ("layout", I32)]

DL_MLP_SILU_GLU, DL_MLP_RELU = 0, 1
DL_LAYOUT_RANK_PARALLEL, DL_LAYOUT_DEINFER = 0, 1


class dl_segment(ctypes.Structure):
    _fields_ = [("A", P), ("lda", I64), ("k", I64)]


class dl_factor_group(ctypes.Structure):
    _fields_ = [("B", P), ("ldb", I64), ("seg", dl_segment * 3)]


class dl_block_weights(ctypes.Structure):
    _fields_ = [("attn_norm", P), ("mlp_norm", P), ("qkv", dl_factor_group), ("o", dl_factor_group),
                ("gu", dl_factor_group), ("down", dl_factor_group)]


class dl_kv_lowrank(ctypes.Structure):
    _fields_ = [("pool", P), ("slot_pos", P), ("num_blocks", I64), ("block_size", I64), ("ld_slot", I64),
                ("block_tables", P), ("max_blocks_per_seq", I64), ("run_src", P), ("run_dst", P), ("run_len", P),
                ("n_runs", P), ("seq_block", P), ("squeeze", P), ("squeeze_pos", P), ("recon", P),
                ("cap_blocks", I64)]


_lock = threading.Lock()
_lib = None


IPC_HANDLE_BYTES = 64   # DL_IPC_HANDLE_BYTES


def load():
    """Load libdl.so (fails loudly if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2604_17709_b200.build` "
                                   "(there is no fallback implementation)")
            lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
            lib.dl_last_error.restype = ctypes.c_char_p
            lib.dl_version.restype = I
            lib.dl_device_ok.restype = I
            lib.dl_comm_create.argtypes = [P, I, I, ctypes.POINTER(P)]
            lib.dl_comm_destroy.argtypes = [P]
            lib.dl_lowrank_linear_workspace.argtypes = [I64, I64, I64, I64, I, P, I, ctypes.POINTER(ctypes.c_size_t)]
            lib.dl_lowrank_linear.argtypes = [P, I64, P, I64, P, I64, P, I64, I64, I64, I64, I64, I, I, P, I, P,
                                              ctypes.c_size_t, P]
            lib.dl_comm_create_group.argtypes = [I, ctypes.c_size_t, P]
            lib.dl_tp_plan.argtypes = [P, I, I, I, I, P, P, P]
            lib.dl_tp_shard_factors.argtypes = [I, P, P, P, P, P, P, I64, I, I, I, I, P, I64, P, P, P, P]
            lib.dl_block_workspace.argtypes = [ctypes.POINTER(dl_block_config), I, ctypes.POINTER(ctypes.c_size_t)]
            lib.dl_block_window_bytes.argtypes = [ctypes.POINTER(dl_block_config), I,
                                                  ctypes.POINTER(ctypes.c_size_t)]
            lib.dl_decomposed_block_forward.argtypes = [ctypes.POINTER(dl_block_config),
                                                        ctypes.POINTER(dl_block_weights), P, I64, P, P, I32, I,
                                                        P, P, P, I64, P, P, ctypes.c_size_t, P]
            lib.dl_decomposed_stack_forward.argtypes = [ctypes.POINTER(dl_block_config),
                                                        ctypes.POINTER(ctypes.POINTER(dl_block_weights)), I32, P,
                                                        I64, P, P, I32, I, ctypes.POINTER(P), ctypes.POINTER(P), P,
                                                        I64, P, P, ctypes.c_size_t, P]
            lib.dl_embedding.argtypes = [P, I64, I64, P, I64, P, P]
            lib.dl_argmax.argtypes = [P, I64, I64, I32, I64, I64, P, P]
            lib.dl_rmsnorm.argtypes = [P, P, P, I64, I64, ctypes.c_float, P]
            lib.dl_dense_workspace.argtypes = [I64, I64, I64, ctypes.POINTER(ctypes.c_size_t)]
            lib.dl_dense.argtypes = [P, I64, P, I64, P, I64, I64, I64, I64, P, ctypes.c_size_t, P]
            lib.dl_profile_begin.argtypes = [I]
            lib.dl_profile_get.argtypes = [I, P, P, P, P]
            lib.dl_debug_gemm_trace.argtypes = [P]
            lib.dl_debug_ew_trace.argtypes = [P]
            lib.dl_debug_linear_gathered.argtypes = [P, I, P, I64, P, I64, P, I64, I64, I64, I64, I64, P,
                                                     ctypes.c_size_t, P]
            lib.dl_deinfer_shard_factors.argtypes = [I, I, P, P, P, P, P, P, I64, I, I, I, P, I64, P, P, P]
            lib.dl_comm_create_loopback.argtypes = [I, I, ctypes.POINTER(P)]
            lib.dl_comm_create_peer.argtypes = [I, I, ctypes.POINTER(P)]
            lib.dl_comm_window_alloc.argtypes = [P, ctypes.c_size_t]
            lib.dl_comm_window_handle.argtypes = [P, P]
            lib.dl_comm_window_connect.argtypes = [P, P]
            lib.dl_kv_prepare.argtypes = [P, I64, P, I32, I64, I64, I64, P, P, P, P, P]
            lib.dl_decomposed_block_forward_kvlr.argtypes = [ctypes.POINTER(dl_block_config),
                                                             ctypes.POINTER(dl_block_weights), P, I64, P,
                                                             ctypes.POINTER(dl_kv_lowrank), P, P, P, ctypes.c_size_t, P]
            for name in EXPORTS[3:]:
                getattr(lib, name).restype = I
            lib.dl_launch_count.restype = ctypes.c_longlong
            _lib = lib
    return _lib


def _check(status: int):
    if status != 0:
        raise DLError(status, load().dl_last_error().decode())


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ld(t: torch.Tensor) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError("expected a row-major 2-D tensor with unit column stride")
    return t.stride(0)


def _dtype(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return DL_F32
    if t.dtype == torch.bfloat16:
        return DL_BF16
    raise ValueError(f"unsupported dtype {t.dtype}")


def dl_version() -> int:
    return load().dl_version()


def dl_device_ok() -> bool:
    return bool(load().dl_device_ok())


# ---------------------------------------------------------------------------
class Comm:
    """dl_comm wrapper around an ncclComm_t (e.g. from a torch NCCL process group)."""

    def __init__(self, nccl_comm_ptr: int, rank: int, world: int):
        h = P()
        _check(load().dl_comm_create(ctypes.c_void_p(nccl_comm_ptr), rank, world, ctypes.byref(h)))
        self.handle = h
        self.rank, self.world = rank, world
        self.is_loopback = False

    @classmethod
    def from_process_group(cls, pg=None):
        import torch.distributed as dist
        pg = pg or dist.group.WORLD
        backend = pg._get_backend(torch.device("cuda"))
        return cls(backend._comm_ptr(), dist.get_rank(pg), dist.get_world_size(pg))

    @classmethod
    def loopback(cls, rank: int, world: int):
        """Measurement-only communicator: TP=`world` shapes on one GPU, collectives
        replaced by local copies (include/dl.h: dl_comm_create_loopback)."""
        self = cls.__new__(cls)
        h = P()
        _check(load().dl_comm_create_loopback(rank, world, ctypes.byref(h)))
        self.handle, self.rank, self.world = h, rank, world
        self.is_loopback = True
        return self

    @classmethod
    def group(cls, world: int, sym_bytes: int = 16 << 20):
        """`world` in-process ranks on the current GPU (include/dl.h:
        dl_comm_create_group); returns one Comm per rank.  Drive rank r from
        its own host thread, all ranks on one shared stream (see run_ranks)."""
        arr = (P * world)()
        _check(load().dl_comm_create_group(world, sym_bytes, ctypes.cast(arr, P)))
        out = []
        for r in range(world):
            self = cls.__new__(cls)
            self.handle, self.rank, self.world = P(arr[r]), r, world
            self.is_loopback = False
            out.append(self)
        return out

    @classmethod
    def peer(cls, rank: int, world: int):
        """Rank `rank` of `world` processes with only the fused decode collectives
        (include/dl.h: dl_comm_create_peer); needs window_alloc + window_connect."""
        self = cls.__new__(cls)
        h = P()
        _check(load().dl_comm_create_peer(rank, world, ctypes.byref(h)))
        self.handle, self.rank, self.world = h, rank, world
        self.is_loopback = False
        return self

    def window_alloc(self, nbytes: int):
        """Allocate this rank's symmetric window (dl_comm_window_alloc)."""
        _check(load().dl_comm_window_alloc(self.handle, nbytes))

    def window_handle(self) -> bytes:
        """This rank's window IPC handle (DL_IPC_HANDLE_BYTES bytes) to exchange with the peers."""
        buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        _check(load().dl_comm_window_handle(self.handle, ctypes.cast(buf, P)))
        return buf.raw

    def window_connect(self, handles):
        """Map every rank's window (handles: one bytes object per rank, rank order)."""
        blob = b"".join(handles)
        if len(blob) != IPC_HANDLE_BYTES * self.world:
            raise ValueError("need one IPC handle per rank")
        buf = ctypes.create_string_buffer(blob, len(blob))
        _check(load().dl_comm_window_connect(self.handle, ctypes.cast(buf, P)))

    def window_exchange(self, nbytes: int, pg=None):
        """window_alloc + an all-gather of the handles over a torch.distributed
        process group (any backend) + window_connect."""
        import torch.distributed as dist
        self.window_alloc(nbytes)
        hs = [None] * self.world
        dist.all_gather_object(hs, self.window_handle(), group=pg)
        self.window_connect(hs)

    def close(self):
        if self.handle:
            load().dl_comm_destroy(self.handle)
            self.handle = None


def run_ranks(fn, world: int):
    """Run fn(rank, stream) for every rank of a group communicator, each in its
    own host thread; the ranks share ONE CUDA stream (include/dl.h:
    dl_comm_create_group).  Returns the per-rank results, re-raising the first
    error."""
    dev = torch.cuda.current_device()
    shared = torch.cuda.Stream()
    out, errs = [None] * world, [None] * world

    def body(r):
        try:
            torch.cuda.set_device(dev)
            with torch.cuda.stream(shared):
                out[r] = fn(r, shared)
        except BaseException as e:   # noqa: BLE001 -- re-raised below
            errs[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    shared.synchronize()
    for e in errs:
        if e is not None:
            raise e
    return out


def dl_comm_create(nccl_comm_ptr: int, rank: int, world: int) -> Comm:
    return Comm(nccl_comm_ptr, rank, world)


def _comm(c):
    return None if c is None else c.handle


# ---------------------------------------------------------------------------
def dl_lowrank_linear_workspace(T: int, m: int, n: int, k: int, dtype=torch.bfloat16, comm: Comm | None = None,
                                reduce: int = DL_REDUCE_ALLREDUCE) -> int:
    b = ctypes.c_size_t()
    _check(load().dl_lowrank_linear_workspace(T, m, n, k, DL_F32 if dtype == torch.float32 else DL_BF16,
                                              _comm(comm), reduce, ctypes.byref(b)))
    return b.value


def dl_lowrank_linear(X: torch.Tensor, A: torch.Tensor, B: torch.Tensor, Y: torch.Tensor, accumulate: bool = False,
                      comm: Comm | None = None, reduce: int = DL_REDUCE_ALLREDUCE,
                      workspace: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Y (+)= A (B x) per token row; with a communicator the
    rank partials are combined per `reduce` (DL_REDUCE_*; SCATTER: Y is [T x m/P]).
    Tensors are device tensors."""
    T, n = X.shape
    m, k = A.shape
    scat = comm is not None and reduce == DL_REDUCE_SCATTER
    m_out = m // comm.world if scat else m
    if B.shape[0] != k or B.shape[1] != n or Y.shape[0] != T or Y.shape[1] != m_out:
        raise ValueError("shape mismatch")
    dt = _dtype(X)
    if workspace is None:
        workspace = torch.empty(dl_lowrank_linear_workspace(T, m, n, k, X.dtype, comm, reduce), dtype=torch.uint8,
                                device=X.device)
    _check(load().dl_lowrank_linear(_ptr(X), _ld(X), _ptr(A), _ld(A), _ptr(B), _ld(B), _ptr(Y), _ld(Y), T, m, n, k,
                                    dt, int(accumulate), _comm(comm), reduce, _ptr(workspace), workspace.numel(),
                                    _stream(stream)))
    return Y


# ---------------------------------------------------------------------------
def dl_tp_plan(seg_ranks, world: int, rank: int, strict: bool = False):
    """Host planner: returns (seg_begin list, seg_len list, k_loc)."""
    n = len(seg_ranks)
    r = (I64 * n)(*seg_ranks)
    b = (I64 * n)()
    ln = (I64 * n)()
    kl = I64()
    _check(load().dl_tp_plan(ctypes.cast(r, P), n, world, rank, int(strict), ctypes.cast(b, P), ctypes.cast(ln, P),
                             ctypes.byref(kl)))
    return list(b), list(ln), kl.value


def _pad8(x: int) -> int:
    return (x + 7) // 8 * 8


def dl_tp_shard_factors(As, Bs, world: int, rank: int, strict: bool = False, stream=None):
    """Shard a factor group (lists of A_g [m_g x r_g], B_g [r_g x n]) for `rank`.

    Returns (A_shards, B_shard, seg_lens).  Output buffers are allocated here
    (torch = memory plumbing); the copy runs in the library on `stream`.
    """
    ng = len(As)
    dt = _dtype(As[0])
    n = Bs[0].shape[1]
    ranks = [a.shape[1] for a in As]
    _, lens, kloc = dl_tp_plan(ranks, world, rank, strict)
    dev = As[0].device
    B_shard = torch.zeros((kloc, _pad8(n)), dtype=As[0].dtype, device=dev)[:, :n]
    A_shards = [torch.zeros((a.shape[0], max(_pad8(ln), 8)), dtype=a.dtype, device=dev)[:, :ln]
                for a, ln in zip(As, lens)]
    arr = lambda vals, ty=I64: (ty * ng)(*vals)  # noqa: E731
    a_p = (P * ng)(*[a.data_ptr() for a in As])
    b_p = (P * ng)(*[b.data_ptr() for b in Bs])
    as_p = (P * ng)(*[a.data_ptr() for a in A_shards])
    out_len = (I64 * ng)()
    _check(load().dl_tp_shard_factors(ng, ctypes.cast(a_p, P), ctypes.cast(arr([_ld(a) for a in As]), P),
                                      ctypes.cast(b_p, P), ctypes.cast(arr([_ld(b) for b in Bs]), P),
                                      ctypes.cast(arr([a.shape[0] for a in As]), P), ctypes.cast(arr(ranks), P),
                                      n, dt, world, rank, int(strict), _ptr(B_shard), B_shard.stride(0),
                                      ctypes.cast(as_p, P), ctypes.cast(arr([a.stride(0) for a in A_shards]), P),
                                      ctypes.cast(out_len, P), _stream(stream)))
    return A_shards, B_shard, list(out_len)


def dl_deinfer_shard_factors(sublayer: int, As, Bs, world: int, rank: int, stream=None):
    """DeInfer shard of a factor group (Fig. 3).  sublayer 1 (q|k|v, gate|up):
    B = the rank's concat-split rows, A_g = its output-row shard (all latent
    columns); sublayer 2 (o, down): B = its input-column shard, A = full copy.
    Returns (A_shards, B_shard)."""
    ng = len(As)
    dt = _dtype(As[0])
    n = Bs[0].shape[1]
    ranks = [a.shape[1] for a in As]
    dev = As[0].device
    if sublayer == 1:
        _, _, kloc = dl_tp_plan(ranks, world, rank)
        B_shard = torch.zeros((kloc, _pad8(n)), dtype=As[0].dtype, device=dev)[:, :n]
        A_shards = [torch.zeros((a.shape[0] // world, _pad8(a.shape[1])), dtype=a.dtype, device=dev)[:, :a.shape[1]]
                    for a in As]
    else:
        nl = n // world
        B_shard = torch.zeros((ranks[0], _pad8(nl)), dtype=As[0].dtype, device=dev)[:, :nl]
        A_shards = [torch.zeros((As[0].shape[0], _pad8(ranks[0])), dtype=As[0].dtype, device=dev)[:, :ranks[0]]]
    arr = lambda vals, ty=I64: (ty * ng)(*vals)  # noqa: E731
    a_p = (P * ng)(*[a.data_ptr() for a in As])
    b_p = (P * ng)(*[b.data_ptr() for b in Bs])
    as_p = (P * ng)(*[a.data_ptr() for a in A_shards])
    _check(load().dl_deinfer_shard_factors(sublayer, ng, ctypes.cast(a_p, P), ctypes.cast(arr([_ld(a) for a in As]), P),
                                           ctypes.cast(b_p, P), ctypes.cast(arr([_ld(b) for b in Bs]), P),
                                           ctypes.cast(arr([a.shape[0] for a in As]), P), ctypes.cast(arr(ranks), P),
                                           n, dt, world, rank, _ptr(B_shard), B_shard.stride(0),
                                           ctypes.cast(as_p, P), ctypes.cast(arr([a.stride(0) for a in A_shards]), P),
                                           _stream(stream)))
    return A_shards, B_shard


# ---------------------------------------------------------------------------
def make_block_config(shape, ranks: dict, max_tokens: int, max_seqs: int,
                      layout: int = DL_LAYOUT_RANK_PARALLEL) -> dl_block_config:
    return dl_block_config(shape.h, shape.n_heads, shape.n_kv_heads, shape.head_dim, shape.m, ranks["q"],
                           ranks["k"], ranks["v"], ranks["o"], ranks["gate"], ranks["up"], ranks["down"],
                           float(shape.rope_theta), float(shape.rms_eps), max_tokens, max_seqs,
                           DL_MLP_SILU_GLU if getattr(shape, "glu", True) else DL_MLP_RELU,
                           0 if getattr(shape, "rope", True) else 1, layout)


class BlockWeights:
    """Rank shard of one block's factors in the library's group layout
    (B of a group concatenated, A per segment), built with dl_tp_shard_factors."""

    GROUPS = (("qkv", ("q", "k", "v")), ("o", ("o",)), ("gu", ("gate", "up")), ("down", ("down",)))

    SUBLAYER = {"qkv": 1, "o": 2, "gu": 1, "down": 2}   # DeInfer roles

    def __init__(self, w: dict, world: int = 1, rank: int = 0, stream=None, layout: int = DL_LAYOUT_RANK_PARALLEL):
        self.tensors = {"attn_norm": w["g_attn"].contiguous(), "mlp_norm": w["g_mlp"].contiguous()}
        self.c = dl_block_weights()
        self.c.attn_norm = self.tensors["attn_norm"].data_ptr()
        self.c.mlp_norm = self.tensors["mlp_norm"].data_ptr()
        self.seg_lens = {}
        for gname, mats in self.GROUPS:
            if gname == "gu" and "A_gate" not in w:
                mats = ("up",)          # non-GLU MLP: the group holds up alone
            As, Bs = [w["A_" + m] for m in mats], [w["B_" + m] for m in mats]
            if layout == DL_LAYOUT_DEINFER:
                A_sh, B_sh = dl_deinfer_shard_factors(self.SUBLAYER[gname], As, Bs, world, rank, stream=stream)
                lens = [a.shape[1] for a in As]          # every latent column stays on the rank
            else:
                A_sh, B_sh, lens = dl_tp_shard_factors(As, Bs, world, rank, stream=stream)
            self.tensors["B_" + gname] = B_sh
            grp = getattr(self.c, gname)
            grp.B = B_sh.data_ptr()
            grp.ldb = B_sh.stride(0)
            for i, (mname, a, ln) in enumerate(zip(mats, A_sh, lens)):
                self.tensors["A_" + mname] = a
                grp.seg[i].A = a.data_ptr() if ln > 0 else None
                grp.seg[i].lda = a.stride(0)
                grp.seg[i].k = ln
            self.seg_lens[gname] = lens


def dl_block_window_bytes(cfg: dl_block_config, world: int = 1) -> int:
    """Group-window bytes the fused collectives of this config need (include/dl.h)."""
    b = ctypes.c_size_t()
    _check(load().dl_block_window_bytes(ctypes.byref(cfg), world, ctypes.byref(b)))
    return b.value


def dl_block_workspace(cfg: dl_block_config, world: int = 1) -> int:
    b = ctypes.c_size_t()
    _check(load().dl_block_workspace(ctypes.byref(cfg), world, ctypes.byref(b)))
    return b.value


def dl_decomposed_block_forward(cfg: dl_block_config, weights: BlockWeights, x: torch.Tensor,
                                positions: torch.Tensor, cu_seqlens: torch.Tensor | None, num_seqs: int,
                                phase: int, k_cache: torch.Tensor, v_cache: torch.Tensor,
                                cache_lens: torch.Tensor, comm: Comm | None, workspace: torch.Tensor,
                                stream=None) -> torch.Tensor:
    T = x.shape[0]
    _check(load().dl_decomposed_block_forward(ctypes.byref(cfg), ctypes.byref(weights.c), _ptr(x), T,
                                              _ptr(positions), _ptr(cu_seqlens), num_seqs, phase, _ptr(k_cache),
                                              _ptr(v_cache), _ptr(cache_lens), k_cache.shape[2], _comm(comm),
                                              _ptr(workspace), workspace.numel(), _stream(stream)))
    return x


class StackArgs:
    """Host pointer arrays for dl_decomposed_stack_forward (built once; the
    weight structs and caches must outlive it)."""

    def __init__(self, weights, k_caches, v_caches):
        n = len(weights)
        self.n = n
        self.w = (ctypes.POINTER(dl_block_weights) * n)(*[ctypes.pointer(bw.c) for bw in weights])
        self.k = (P * n)(*[_ptr(t) for t in k_caches])
        self.v = (P * n)(*[_ptr(t) for t in v_caches])
        self.max_seq = k_caches[0].shape[2] if n else 1


def dl_decomposed_stack_forward(cfg: dl_block_config, args: StackArgs, x: torch.Tensor, positions: torch.Tensor,
                                cu_seqlens: torch.Tensor | None, num_seqs: int, phase: int,
                                cache_lens: torch.Tensor, comm: Comm | None, workspace: torch.Tensor,
                                stream=None) -> torch.Tensor:
    """args.n consecutive blocks sharing cfg and workspace (include/dl.h)."""
    T = x.shape[0]
    _check(load().dl_decomposed_stack_forward(ctypes.byref(cfg), args.w, args.n, _ptr(x), T, _ptr(positions),
                                              _ptr(cu_seqlens), num_seqs, phase, args.k, args.v, _ptr(cache_lens),
                                              args.max_seq, _comm(comm), _ptr(workspace), workspace.numel(),
                                              _stream(stream)))
    return x


def dl_kv_prepare(block_tables, seq_tokens, block_size: int, max_runs: int, cap_blocks: int):
    """Preparation stage of the low-rank KV cache: contiguous-run scan and
    remapping index list.  Host int32 arrays in; returns (run_src, run_dst, run_len,
    n_runs, seq_block) as numpy int32 arrays (length max_runs / num_seqs)."""
    import numpy as np
    bt = np.ascontiguousarray(np.asarray(block_tables, dtype=np.int32))
    st = np.ascontiguousarray(np.asarray(seq_tokens, dtype=np.int32))
    ns = len(st)
    rs, rd, rl = (np.zeros(max(max_runs, 1), np.int32) for _ in range(3))
    nr = np.zeros(1, np.int32)
    sb = np.zeros(max(ns, 1), np.int32)
    p = lambda a: a.ctypes.data_as(P)  # noqa: E731
    _check(load().dl_kv_prepare(p(bt), bt.shape[1] if bt.ndim == 2 else 1, p(st), ns, block_size, max_runs,
                                cap_blocks, p(rs), p(rd), p(rl), p(nr), p(sb)))
    return rs, rd, rl, int(nr[0]), sb[:ns]


class LowRankKVCache:
    """Paged low-rank KV cache of ONE layer plus the step's fixed buffers
    (squeeze / reconstruction buffers may be shared by all layers: pass them in).

    pool slot = [z_k (l_k) | pad to rup(l_k, 64) | z_v (l_v)] bf16; see include/dl.h."""

    def __init__(self, l_k: int, l_v: int, hkv_local: int, num_blocks: int, block_size: int, max_seqs: int,
                 max_blocks_per_seq: int, cap_blocks: int, max_runs: int | None = None, device="cuda",
                 shared: "LowRankKVCache | None" = None):
        dev = torch.device(device)
        self.l_k, self.l_v, self.block_size = l_k, l_v, block_size
        self.zv_off = -(-l_k // 64) * 64
        self.ld_slot = _pad8(self.zv_off + l_v)
        self.pool = torch.zeros(num_blocks * block_size, self.ld_slot, dtype=torch.bfloat16, device=dev)
        self.slot_pos = torch.zeros(num_blocks * block_size, dtype=torch.int32, device=dev)
        if shared is None:
            self.block_tables = torch.zeros(max_seqs, max_blocks_per_seq, dtype=torch.int32, device=dev)
            self.max_runs = max_runs or max_seqs * max_blocks_per_seq
            self.run_src = torch.zeros(self.max_runs, dtype=torch.int32, device=dev)
            self.run_dst = torch.zeros_like(self.run_src)
            self.run_len = torch.zeros_like(self.run_src)
            self.n_runs = torch.zeros(1, dtype=torch.int32, device=dev)
            self.seq_block = torch.zeros(max_seqs, dtype=torch.int32, device=dev)
            rows = cap_blocks * block_size
            self.squeeze = torch.zeros(rows, self.ld_slot, dtype=torch.bfloat16, device=dev)
            self.squeeze_pos = torch.zeros(rows, dtype=torch.int32, device=dev)
            self.recon = torch.zeros(rows, 2 * hkv_local, dtype=torch.bfloat16, device=dev)
        else:
            # one block table and one plan serve every layer (same allocation pattern);
            # the squeeze / reconstruction buffers are per-step scratch
            for k in ("run_src", "run_dst", "run_len", "n_runs", "seq_block", "squeeze", "squeeze_pos", "recon",
                      "block_tables", "max_runs"):
                setattr(self, k, getattr(shared, k))
        self.cap_blocks = cap_blocks
        self.c = dl_kv_lowrank(self.pool.data_ptr(), self.slot_pos.data_ptr(), num_blocks, block_size, self.ld_slot,
                               self.block_tables.data_ptr(), max_blocks_per_seq, self.run_src.data_ptr(),
                               self.run_dst.data_ptr(), self.run_len.data_ptr(), self.n_runs.data_ptr(),
                               self.seq_block.data_ptr(), self.squeeze.data_ptr(), self.squeeze_pos.data_ptr(),
                               self.recon.data_ptr(), cap_blocks)

    def prepare(self, block_tables_host, seq_tokens):
        """Preparation stage: plan on the host, copy into the fixed device plan arrays."""
        rs, rd, rl, nr, sb = dl_kv_prepare(block_tables_host, seq_tokens, self.block_size, self.max_runs,
                                           self.cap_blocks)
        self.run_src.copy_(torch.from_numpy(rs[:self.max_runs]))
        self.run_dst.copy_(torch.from_numpy(rd[:self.max_runs]))
        self.run_len.copy_(torch.from_numpy(rl[:self.max_runs]))
        self.n_runs.fill_(nr)
        self.seq_block[:len(sb)].copy_(torch.from_numpy(sb))
        return nr


def dl_decomposed_block_forward_kvlr(cfg: dl_block_config, weights: BlockWeights, x: torch.Tensor,
                                     positions: torch.Tensor, kv: LowRankKVCache, cache_lens: torch.Tensor,
                                     comm: Comm | None, workspace: torch.Tensor, stream=None) -> torch.Tensor:
    _check(load().dl_decomposed_block_forward_kvlr(ctypes.byref(cfg), ctypes.byref(weights.c), _ptr(x), x.shape[0],
                                                   _ptr(positions), ctypes.byref(kv.c), _ptr(cache_lens),
                                                   _comm(comm), _ptr(workspace), workspace.numel(),
                                                   _stream(stream)))
    return x


def dl_embedding(table: torch.Tensor, ids: torch.Tensor, out: torch.Tensor, stream=None):
    _check(load().dl_embedding(_ptr(table), table.shape[0], table.shape[1], _ptr(ids), ids.numel(), _ptr(out),
                               _stream(stream)))
    return out


def dl_rmsnorm(x: torch.Tensor, gamma: torch.Tensor, out: torch.Tensor, eps: float, stream=None):
    _check(load().dl_rmsnorm(_ptr(x), _ptr(gamma), _ptr(out), x.shape[0], x.shape[1], eps, _stream(stream)))
    return out


def dl_dense(X: torch.Tensor, W: torch.Tensor, C: torch.Tensor, stream=None, workspace: torch.Tensor | None = None):
    T, K = X.shape
    N = W.shape[0]
    _check(load().dl_dense(_ptr(X), _ld(X), _ptr(W), _ld(W), _ptr(C), _ld(C), T, N, K, _ptr(workspace),
                           0 if workspace is None else workspace.numel(), _stream(stream)))
    return C


def dl_launch_count() -> int:
    """Kernels this library has enqueued since load (captured launches count once)."""
    return int(load().dl_launch_count())


def dl_profile_begin(capacity: int):
    _check(load().dl_profile_begin(capacity))


def dl_profile_end():
    _check(load().dl_profile_end())


def dl_profile_records():
    """[(ms, bytes, flops, kind)] for the instrumented tcgen05 GEMM launches."""
    L = load()
    out = []
    for i in range(L.dl_profile_count()):
        ms, b, f, k = ctypes.c_float(), ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
        _check(L.dl_profile_get(i, ctypes.byref(ms), ctypes.byref(b), ctypes.byref(f), ctypes.byref(k)))
        out.append((ms.value, b.value, f.value, k.value))
    return out


def dl_argmax(logits: torch.Tensor, ids: torch.Tensor, stream=None) -> torch.Tensor:
    """Greedy next token over vocab shards: logits [P, T, vloc] or [T, vloc] (bf16) -> ids [T] int32."""
    lg = logits if logits.dim() == 3 else logits.unsqueeze(0)
    P, T, vloc = lg.shape
    _check(load().dl_argmax(_ptr(lg), T, vloc, P, lg.stride(0), lg.stride(1), _ptr(ids), _stream(stream)))
    return ids


def dl_debug_linear_gathered(Xg: torch.Tensor, A: torch.Tensor, B: torch.Tensor, Y: torch.Tensor, stream=None):
    """Test hook (include/dl.h): Y = A(B X) with X rank-major [P][T][n/P]."""
    P, T, w = Xg.shape
    m, k = A.shape
    n = P * w
    ws = torch.zeros(dl_lowrank_linear_workspace(max(T, 17), m, n, k), dtype=torch.uint8, device=Xg.device)
    _check(load().dl_debug_linear_gathered(_ptr(Xg), P, _ptr(A), A.stride(0), _ptr(B), B.stride(0), _ptr(Y),
                                           Y.stride(0), T, m, n, k, _ptr(ws), ws.numel(), _stream(stream)))
    return Y


def dl_debug_ew_trace(buf: torch.Tensor | None):
    """Timeline of the non-GEMM decode kernels (see include/dl.h); None disables."""
    _check(load().dl_debug_ew_trace(_ptr(buf)))


def dl_debug_gemm_trace(buf: torch.Tensor | None):
    """Enable (int64 device tensor, >= 8 per CTA) or disable (None) the GEMM CTA timeline."""
    _check(load().dl_debug_gemm_trace(_ptr(buf)))
