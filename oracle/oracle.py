"""ctypes marshalling for oracle/dl_oracle.c (no arithmetic here).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.  Every function converts
its inputs to contiguous float64 numpy arrays (exact for bf16/fp32 values),
calls the C routine and returns numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dl_oracle.c")
_LIB = os.path.join(_HERE, "libdl_oracle.so")
_lock = threading.Lock()
_lib = None

__all__ = [
    "build", "load", "matmul", "lowrank_linear", "shard_range",
    "lowrank_linear_sharded", "truncated_svd", "factor_params", "rmsnorm",
    "rope", "attention", "BlockCfg", "block_prefill", "block_decode",
    "block_params", "census", "num_threads", "block_decode_lowrank", "kv_runs", "LAYOUT_RANK_PARALLEL", "LAYOUT_DEINFER",
]


def build(force: bool = False) -> str:
    """Compile dl_oracle.c -> libdl_oracle.so with gcc (-O2, OpenMP, no fast-math)."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp",
           "-shared", "-fPIC", "-std=c11", "-o", tmp, _SRC, "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, _LIB)
    return _LIB


def load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            I64 = ctypes.c_int64
            I = ctypes.c_int
            D = ctypes.c_double
            lib.oracle_matmul.argtypes = [P, P, P, I64, I64, I64]
            lib.oracle_lowrank_linear.argtypes = [P, P, P, P, I64, I64, I64, I64]
            lib.oracle_shard_range.argtypes = [I64, I, I, I64, P, P, P]
            lib.oracle_lowrank_linear_sharded.argtypes = [P, P, P, P, I64, I64, I64, I64, I, I64]
            lib.oracle_truncated_svd.argtypes = [P, I64, I64, I64, P, P, P]
            lib.oracle_factor_params.argtypes = [I64, I64, I64]
            lib.oracle_factor_params.restype = I64
            lib.oracle_rmsnorm.argtypes = [P, P, D, P, I64, I64]
            lib.oracle_rmsnorm.restype = None
            lib.oracle_rope.argtypes = [P, P, I64, I64, I64, D]
            lib.oracle_rope.restype = None
            lib.oracle_attention.argtypes = [P, P, P, P, I64, P, ctypes.c_int32, I64, I64, I64]
            lib.oracle_block_prefill.argtypes = [P, P, P, I64, P, P, ctypes.c_int32, P, I64, P, P, P, I, I64]
            lib.oracle_block_decode.argtypes = [P, P, P, I64, P, P, I64, P, P, P, P, I, I64]
            lib.oracle_block_decode_lowrank.argtypes = [P, P, P, I64, P, P, I64, P, P, P, P]
            lib.oracle_kv_runs.argtypes = [P, I64, P, P]
            lib.oracle_kv_runs.restype = I64
            lib.oracle_block_params.argtypes = [P]
            lib.oracle_block_params.restype = I64
            lib.oracle_census.argtypes = [I64] * 10 + [P]
            lib.oracle_census.restype = None
            _lib = lib
    return _lib


def num_threads() -> int:
    """Threads OpenMP will use for the oracle (OMP_NUM_THREADS or all cores)."""
    env = os.environ.get("OMP_NUM_THREADS")
    return int(env) if env else (os.cpu_count() or 1)


def _f64(a) -> np.ndarray:
    if hasattr(a, "detach"):  # torch tensor (CPU)
        a = a.detach().to("cpu").double().numpy()
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i32(a) -> np.ndarray:
    if hasattr(a, "detach"):
        a = a.detach().to("cpu").numpy()
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"oracle {what} failed with code {rc}")


def matmul(A, B) -> np.ndarray:
    A, B = _f64(A), _f64(B)
    M, K = A.shape
    K2, N = B.shape
    if K != K2:
        raise ValueError("shape")
    C = np.empty((M, N))
    _check(load().oracle_matmul(_p(A), _p(B), _p(C), M, K, N), "matmul")
    return C


def lowrank_linear(X, A, B) -> np.ndarray:
    """Y[T x m] = rows of A (B x_t)   (Eq. 1)."""
    X, A, B = _f64(X), _f64(A), _f64(B)
    T, n = X.shape
    m, k = A.shape
    if B.shape != (k, n):
        raise ValueError("shape")
    Y = np.empty((T, m))
    _check(load().oracle_lowrank_linear(_p(X), _p(A), _p(B), _p(Y), T, m, n, k), "lowrank_linear")
    return Y


def shard_range(k: int, world: int, rank: int, align: int = 1):
    b = ctypes.c_int64()
    ln = ctypes.c_int64()
    lp = ctypes.c_int64()
    rc = load().oracle_shard_range(k, world, rank, align, ctypes.byref(b), ctypes.byref(ln), ctypes.byref(lp))
    _check(rc, "shard_range")
    return b.value, ln.value, lp.value


def lowrank_linear_sharded(X, A, B, world: int, align: int = 1) -> np.ndarray:
    X, A, B = _f64(X), _f64(A), _f64(B)
    T, n = X.shape
    m, k = A.shape
    Y = np.empty((T, m))
    _check(load().oracle_lowrank_linear_sharded(_p(X), _p(A), _p(B), _p(Y), T, m, n, k, world, align),
           "lowrank_linear_sharded")
    return Y


def truncated_svd(W, k: int):
    """Returns (A [m x k], B [k x n], sigma_all [min(m,n)])."""
    W = _f64(W)
    m, n = W.shape
    A = np.empty((m, k))
    B = np.empty((k, n))
    s = np.empty((min(m, n),))
    _check(load().oracle_truncated_svd(_p(W), m, n, k, _p(A), _p(B), _p(s)), "truncated_svd")
    return A, B, s


def factor_params(m: int, n: int, k: int) -> int:
    return int(load().oracle_factor_params(m, n, k))


def rmsnorm(x, g, eps: float) -> np.ndarray:
    x, g = _f64(x), _f64(g)
    T, h = x.shape
    y = np.empty_like(x)
    load().oracle_rmsnorm(_p(x), _p(g), eps, _p(y), T, h)
    return y


def rope(v, pos, theta: float) -> np.ndarray:
    """v [T x nh x d] -> rotated copy."""
    v = _f64(v).copy()
    pos = _i32(pos)
    T, nh, d = v.shape
    load().oracle_rope(_p(v), _p(pos), T, nh, d, theta)
    return v


def attention(q, k, v, cu_seqlens, H: int, Hkv: int, d: int) -> np.ndarray:
    q, k, v = _f64(q), _f64(k), _f64(v)
    cu = _i32(cu_seqlens)
    T = q.shape[0]
    out = np.empty((T, H * d))
    _check(load().oracle_attention(_p(q), _p(k), _p(v), _p(out), T, _p(cu), len(cu) - 1, H, Hkv, d),
           "attention")
    return out


class _CCfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in
                ("h", "n_heads", "n_kv_heads", "head_dim", "m",
                 "r_q", "r_k", "r_v", "r_o", "r_gate", "r_up", "r_down")] + \
               [("rope_theta", ctypes.c_double), ("rms_eps", ctypes.c_double), ("mlp_glu", ctypes.c_int64),
                ("use_rope", ctypes.c_int64), ("layout", ctypes.c_int64)]

LAYOUT_RANK_PARALLEL, LAYOUT_DEINFER = 0, 1


_WNAMES = ("g_attn", "g_mlp", "A_q", "B_q", "A_k", "B_k", "A_v", "B_v", "A_o", "B_o",
           "A_gate", "B_gate", "A_up", "B_up", "A_down", "B_down")


class _CW(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in _WNAMES]


class BlockCfg:
    """Plain record of block dimensions / ranks (names as in Table 1)."""

    def __init__(self, h, n_heads, n_kv_heads, head_dim, m, r_q, r_k, r_v, r_o,
                 r_gate, r_up, r_down, rope_theta=500000.0, rms_eps=1e-5, mlp_glu=1, use_rope=1, layout=0):
        self.__dict__.update(locals())
        del self.__dict__["self"]

    def _c(self):
        return _CCfg(*(getattr(self, n) for n, _ in _CCfg._fields_))


def _pack_w(w: dict):
    w = dict(w)
    if "A_gate" not in w:          # non-GLU MLP: no gate factors (never read by the C code)
        w["A_gate"] = w["B_gate"] = np.zeros((1, 1))
    arrs = {n: _f64(w[n]) for n in _WNAMES}
    cw = _CW(*(arrs[n].ctypes.data for n in _WNAMES))
    return cw, arrs


def block_prefill(cfg: BlockCfg, w: dict, x, pos, cu_seqlens, rows=None,
                  world: int = 1, align: int = 1):
    """Returns (x_out [n_rows x h], k [T x hkv], v [T x hkv])."""
    x = _f64(x)
    pos = _i32(pos)
    cu = _i32(cu_seqlens)
    T, h = x.shape
    hkv = cfg.n_kv_heads * cfg.head_dim
    if rows is None:
        rows_a = None
        n_rows = T
    else:
        rows_a = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
        n_rows = len(rows_a)
    xo = np.empty((n_rows, h))
    ko = np.empty((T, hkv))
    vo = np.empty((T, hkv))
    cc = cfg._c()
    cw, keep = _pack_w(w)
    rc = load().oracle_block_prefill(ctypes.byref(cc), ctypes.byref(cw), _p(x), T, _p(pos), _p(cu),
                                     len(cu) - 1, None if rows_a is None else _p(rows_a), n_rows,
                                     _p(xo), _p(ko), _p(vo), world, align)
    _check(rc, "block_prefill")
    del keep
    return xo, ko, vo


def block_decode(cfg: BlockCfg, w: dict, x, cache_k, cache_v, cache_len,
                 world: int = 1, align: int = 1):
    """x [B x h]; cache_k/v [B x max_seq x hkv] -> (x_out, k_new, v_new)."""
    x = _f64(x)
    ck, cv = _f64(cache_k), _f64(cache_v)
    cl = _i32(cache_len)
    Bn, h = x.shape
    max_seq = ck.shape[1]
    hkv = cfg.n_kv_heads * cfg.head_dim
    xo = np.empty((Bn, h))
    kn = np.empty((Bn, hkv))
    vn = np.empty((Bn, hkv))
    cc = cfg._c()
    cw, keep = _pack_w(w)
    rc = load().oracle_block_decode(ctypes.byref(cc), ctypes.byref(cw), _p(x), Bn, _p(ck), _p(cv),
                                    max_seq, _p(cl), _p(xo), _p(kn), _p(vn), world, align)
    _check(rc, "block_decode")
    del keep
    return xo, kn, vn


def block_decode_lowrank(cfg: BlockCfg, w: dict, x, zk_cache, zv_cache, cache_len):
    """Decode with a low-rank KV cache.  zk_cache [B x max_seq x r_k],
    zv_cache [B x max_seq x r_v] -> (x_out, zk_new [B x r_k], zv_new [B x r_v])."""
    x = _f64(x)
    zk, zv = _f64(zk_cache), _f64(zv_cache)
    cl = _i32(cache_len)
    Bn, h = x.shape
    xo = np.empty((Bn, h))
    kn = np.empty((Bn, cfg.r_k))
    vn = np.empty((Bn, cfg.r_v))
    cc = cfg._c()
    cw, keep = _pack_w(w)
    rc = load().oracle_block_decode_lowrank(ctypes.byref(cc), ctypes.byref(cw), _p(x), Bn, _p(zk), _p(zv),
                                            zk.shape[1], _p(cl), _p(xo), _p(kn), _p(vn))
    _check(rc, "block_decode_lowrank")
    del keep
    return xo, kn, vn


def kv_runs(phys):
    """Contiguous-run scan of a block list -> [(start, length)]."""
    ph = _i32(phys)
    n = len(ph)
    st = np.zeros(max(n, 1), dtype=np.int32)
    ln = np.zeros(max(n, 1), dtype=np.int32)
    r = int(load().oracle_kv_runs(_p(ph), n, _p(st), _p(ln)))
    return [(int(st[i]), int(ln[i])) for i in range(r)]


def block_params(cfg: BlockCfg) -> int:
    cc = cfg._c()
    return int(load().oracle_block_params(ctypes.byref(cc)))


_CENSUS_KEYS = ("unopt_attn", "unopt_mlp", "unopt_block", "deinfer_ag_attn", "deinfer_ag_mlp",
                "deinfer_ag_total", "deinfer_block_rowsum", "deinfer_block_printed",
                "deinfer_block_text", "build_block", "build_collectives", "base_attn_reduce_sums",
                "base_mlp_reduce_sums")


def census(h, h_kv, m, l_q, l_k, l_v, l_o, l_gate, l_up, l_down) -> dict:
    out = np.zeros(13, dtype=np.int64)
    load().oracle_census(h, h_kv, m, l_q, l_k, l_v, l_o, l_gate, l_up, l_down, _p(out))
    return dict(zip(_CENSUS_KEYS, (int(v) for v in out)))
