// C ABI (include/dl.h): argument validation, path selection, the rank-shard
// planner, NCCL plumbing and the decomposed-block orchestration.  Every
// arithmetic step runs in this library's kernels (tc_gemm.cu,
// simt_chain.cu, elementwise.cu, attention.cu); there is no CPU fallback.
#include <dlfcn.h>
#include <stdlib.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <string>

#include "dl_internal.h"

namespace dl {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

dl_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return DL_OK;
  set_error("%s: %s", what, cudaGetErrorString(e));
  return DL_ERR_CUDA;
}

dl_status check_device_sm100() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
  int major = 0;
  e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaDeviceGetAttribute");
  if (major != 10) {
    set_error("device compute capability %d.x is not sm_100 (B200)", major);
    return DL_ERR_CUDA;
  }
  return DL_OK;
}

int num_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return kNumSMsB200;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
    return kNumSMsB200;
  return n;
}

}  // namespace dl

using namespace dl;

#define DL_TRY(expr) DL_TRY_INTERNAL(expr)

namespace {

// ---------------------------------------------------------------------------
// validation helpers
// ---------------------------------------------------------------------------
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
size_t esize(dl_dtype t) { return t == DL_F32 ? 4 : 2; }
int64_t rup(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
size_t rup_sz(size_t x) { return (x + 255) & ~size_t(255); }

dl_status check_ld(int64_t ld, int64_t row, dl_dtype dt, const char* name) {
  if (ld < row) {
    set_error("%s: leading dimension %lld < row length %lld", name, (long long)ld, (long long)row);
    return DL_ERR_SHAPE;
  }
  if ((ld * static_cast<int64_t>(esize(dt))) % 16 != 0) {
    set_error("%s: leading dimension %lld is not a 16-byte multiple", name, (long long)ld);
    return DL_ERR_ALIGN;
  }
  return DL_OK;
}
dl_status check_ptr(const void* p, const char* name) {
  if (!p) {
    set_error("%s is NULL", name);
    return DL_ERR_INVALID_ARG;
  }
  if (!aligned16(p)) {
    set_error("%s is not 16-byte aligned", name);
    return DL_ERR_ALIGN;
  }
  return DL_OK;
}
dl_status check_device() { return check_device_sm100(); }

// path of dl_lowrank_linear
enum LinPath { PATH_SIMT, PATH_SKINNY, PATH_WIDE };
// Skinny stage 1 -> stage 2 as ONE fused chain launch (tc_gemm_chain).
// dl_lowrank_linear uses it by default (DL_CHAIN=0: two launches).  Inside the
// PDL-chained block the two-launch form measured faster (70B@40% decode:
// 25.8 vs 26.5 ms/step at TP = 1, 9.85 vs 10.1-10.2 ms per rank at TP = 8;
// DESIGN.md §6), so the block path takes the chain only with DL_CHAIN=1.
bool use_chain() {
  static const bool on = !DL_ENV("DL_CHAIN") || atoi(DL_ENV("DL_CHAIN")) != 0;
  return on;
}
bool use_chain_block() {
  static const bool on = DL_ENV("DL_CHAIN") && atoi(DL_ENV("DL_CHAIN")) != 0;
  return on;
}

LinPath lin_path(int64_t T, dl_dtype dt) {
  if (dt == DL_F32 || T <= 16) return PATH_SIMT;
  if (T <= 256) return PATH_SKINNY;
  return PATH_WIDE;
}

// workspace carving
struct Carver {
  uint8_t* base;
  size_t off = 0;
  explicit Carver(void* b) : base(static_cast<uint8_t*>(b)) {}
  template <typename T>
  T* take(size_t count) {
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += rup_sz(count * sizeof(T));
    return p;
  }
};

struct LinWs {
  float* zf;           // [T x ldz32] fp32: skinny stage-1 reduction target / SIMT z
  __nv_bfloat16* zb;   // [T x ldzb] bf16 stage-2 operand (tensor-core paths)
  float* yf;           // [T x ldy32] fp32 rank partial (skinny, or any collective)
  float* yr;           // [T x m/P] fp32 reduce-scatter receive buffer (DL_REDUCE_SCATTER)
  unsigned int* chain; // fused-chain arrival counters (skinny tensor path)
  int64_t ldz32, ldzb, ldy32;
};

// Which work a dl_lowrank_linear call does: `coll` = a collective runs
// (communicator given and reduce != NONE); `tensor` = the bf16 tensor-core
// kernels run (T > 16, or a bf16 collective: the rank partial then comes from
// the skinny tensor path, whose fp32 output the collective reduces).
struct LinPlan {
  LinPath path;
  bool coll, tensor;
  int P;
};
LinPlan lin_plan(int64_t T, dl_dtype dt, const dl_comm_s* comm, dl_reduce reduce) {
  LinPlan p{};
  p.path = lin_path(T, dt);
  p.P = comm ? comm->world : 1;
  p.coll = comm != nullptr && reduce != DL_REDUCE_NONE;
  p.tensor = p.path != PATH_SIMT || (p.coll && dt == DL_BF16);
  return p;
}

LinWs carve_lin(Carver& c, int64_t T, int64_t m, int64_t k, const LinPlan& pl, dl_reduce reduce) {
  LinWs w{};
  w.ldz32 = rup(k, 4);
  w.ldzb = rup(k, 8);
  w.ldy32 = rup(m, 4);
  w.zf = c.take<float>(static_cast<size_t>(T) * w.ldz32);
  if (pl.tensor) w.zb = c.take<__nv_bfloat16>(static_cast<size_t>(T) * w.ldzb);
  if (pl.path == PATH_SKINNY || pl.coll) w.yf = c.take<float>(static_cast<size_t>(T) * w.ldy32);
  if (pl.coll && reduce == DL_REDUCE_SCATTER) w.yr = c.take<float>(static_cast<size_t>(T) * (m / pl.P));
  if (pl.tensor) w.chain = c.take<unsigned int>(2);
  return w;
}

GemmProblem one_seg(const void* act, int64_t ld_act, int64_t T, int64_t k_act, const void* w, int64_t ldw,
                    int64_t rows, int64_t klen, GemmOut out) {
  GemmProblem p{};
  p.act = act;
  p.ld_act = ld_act;
  p.T = T;
  p.k_act = k_act;
  p.nseg = 1;
  p.seg[0] = GemmSeg{w, ldw, rows, klen, 0, 0};
  p.n_feat = rows;
  p.out = out;
  return p;
}

GemmOut out_plain(void* ptr, int64_t ld, int mode, int accumulate) {
  GemmOut o{};
  o.ptr = ptr;
  o.ld = ld;
  o.mode = mode;
  o.accumulate = accumulate;
  o.scatter_p = 0;
  return o;
}

}  // namespace

extern "C" {

const char* dl_last_error(void) { return g_last_error.c_str(); }
int dl_version(void) { return 100; }
int dl_device_ok(void) { return check_device() == DL_OK ? 1 : 0; }

// ---------------------------------------------------------------------------
dl_status dl_lowrank_linear_workspace(int64_t T, int64_t m, int64_t n, int64_t k, dl_dtype dtype, dl_comm comm,
                                      dl_reduce reduce, size_t* bytes) {
  (void)n;
  if (!bytes) {
    set_error("bytes is NULL");
    return DL_ERR_INVALID_ARG;
  }
  if (reduce < DL_REDUCE_NONE || reduce > DL_REDUCE_SCATTER) {
    set_error("unknown reduce mode %d", (int)reduce);
    return DL_ERR_INVALID_ARG;
  }
  Carver c(nullptr);
  const LinPlan pl = lin_plan(T, dtype, comm, reduce);
  carve_lin(c, T > 0 ? T : 1, m, k, pl, reduce);
  *bytes = c.off;
  return DL_OK;
}

dl_status dl_lowrank_linear(const void* X, int64_t ldx, const void* A, int64_t lda, const void* B, int64_t ldb,
                            void* Y, int64_t ldy, int64_t T, int64_t m, int64_t n, int64_t k, dl_dtype dtype,
                            int accumulate, dl_comm comm, dl_reduce reduce, void* workspace, size_t workspace_bytes,
                            void* stream) {
  if (dtype != DL_F32 && dtype != DL_BF16) {
    set_error("unknown dtype %d", (int)dtype);
    return DL_ERR_INVALID_ARG;
  }
  if (reduce < DL_REDUCE_NONE || reduce > DL_REDUCE_SCATTER) {
    set_error("unknown reduce mode %d", (int)reduce);
    return DL_ERR_INVALID_ARG;
  }
  if (T < 0 || m <= 0 || n <= 0) {
    set_error("bad shape T=%lld m=%lld n=%lld", (long long)T, (long long)m, (long long)n);
    return DL_ERR_SHAPE;
  }
  if (k < 1 || (!comm && k > std::min(m, n))) {
    set_error("rank k=%lld outside [1, min(m,n)=%lld]", (long long)k, (long long)std::min(m, n));
    return DL_ERR_RANK;
  }
  const LinPlan pl = lin_plan(T, dtype, comm, reduce);
  const bool scatter = pl.coll && reduce == DL_REDUCE_SCATTER;
  if (scatter && m % (32 * pl.P) != 0) {
    set_error("DL_REDUCE_SCATTER needs m %% (32 * world) == 0 (m=%lld, world=%d)", (long long)m, pl.P);
    return DL_ERR_PARTITION;
  }
  if (T == 0) return DL_OK;
  const int64_t m_out = scatter ? m / pl.P : m;   // features this rank receives
  DL_TRY(check_ptr(X, "X"));
  DL_TRY(check_ptr(A, "A"));
  DL_TRY(check_ptr(B, "B"));
  DL_TRY(check_ptr(Y, "Y"));
  DL_TRY(check_ld(ldx, n, dtype, "ldx"));
  DL_TRY(check_ld(lda, k, dtype, "lda"));
  DL_TRY(check_ld(ldb, n, dtype, "ldb"));
  DL_TRY(check_ld(ldy, m_out, dtype, "ldy"));
  if (dtype == DL_F32 && T > 16) {
    set_error("fp32 runs on the exact-FFMA SIMT path, limited to T <= 16 (got %lld)", (long long)T);
    return DL_ERR_DTYPE;
  }
  if (dtype == DL_F32 && pl.coll && accumulate) {
    set_error("fp32 accumulate (Y +=) with a collective is not supported");
    return DL_ERR_UNSUPPORTED;
  }
  if (pl.tensor && m % 4 != 0) {
    set_error("tensor-core path requires m %% 4 == 0 (got m=%lld)", (long long)m);
    return DL_ERR_UNSUPPORTED;
  }
  size_t need = 0;
  dl_lowrank_linear_workspace(T, m, n, k, dtype, comm, reduce, &need);
  if (!workspace || workspace_bytes < need) {
    set_error("workspace %zu B < required %zu B", workspace_bytes, need);
    return DL_ERR_WORKSPACE;
  }
  DL_TRY(check_device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Carver cv(workspace);
  const LinWs ws = carve_lin(cv, T, m, k, pl, reduce);
  __nv_bfloat16* Yb = static_cast<__nv_bfloat16*>(Y);

  if (!pl.tensor) {
    // SIMT chain (T <= 16 bf16 without a collective, or fp32)
    if (!pl.coll) return simt_lowrank(X, ldx, A, lda, B, ldb, Y, ldy, T, m, n, k, dtype, accumulate, ws.zf, st);
    // fp32 collective: partial into the fp32 scratch, all-reduce, copy this rank's columns
    DL_TRY(simt_lowrank(X, ldx, A, lda, B, ldb, ws.yf, ws.ldy32, T, m, n, k, dtype, 0, ws.zf, st));
    DL_TRY(coll_all_reduce(comm, ws.yf, static_cast<size_t>(T) * ws.ldy32, kCollF32, st));
    const int64_t c0 = scatter ? comm->rank * m_out : 0;
    return cuda_status(cudaMemcpy2DAsync(Y, ldy * 4, ws.yf + c0, ws.ldy32 * 4, m_out * 4, T, cudaMemcpyDeviceToDevice,
                                         st), "copy");
  }

  // ---- tensor-core paths (bf16) ----
  // rank partial output: plain [T x m] fp32, or rank-major slabs [P][T][m/P]
  // for the reduce-scatter (feature f goes to rank f / (m/P))
  auto partial_out = [&](int mode) {
    GemmOut o = out_plain(ws.yf, ws.ldy32, mode, 0);
    if (scatter) {
      o.scatter_p = pl.P;
      o.slab = m_out;
      o.seg_rpr[0] = m_out;
    }
    return o;
  };
  // finish: reduce the fp32 partial, then Y (+)= result
  auto finish = [&]() -> dl_status {
    float* res = ws.yf;
    int64_t ldr = ws.ldy32;
    if (scatter) {
      DL_TRY(coll_reduce_scatter(comm, ws.yf, ws.yr, static_cast<size_t>(T) * m_out, kCollF32, st));
      res = ws.yr;
      ldr = m_out;
    } else if (pl.coll) {
      DL_TRY(coll_all_reduce(comm, ws.yf, static_cast<size_t>(T) * ws.ldy32, kCollF32, st));
    }
    const int clear = pl.path == PATH_SKINNY || pl.path == PATH_SIMT ? 1 : 0;   // stream-K targets stay zeroed
    if (accumulate) return launch_residual_add_f32(res, ldr, Yb, ldy, T, m_out, clear, st);
    return launch_f32_to_bf16(res, ldr, Yb, ldy, T, m_out, clear, st);
  };
  if (pl.path == PATH_SKINNY || pl.path == PATH_SIMT) {
    // The fused chain (one launch): stage 1 reduces bf16x2 partials of
    // Z = X B^T into the zeroed L2-resident bf16 Z (stream-K), stage 2 reduces
    // the fp32 rank partial Z A^T once every CTA's stage-1 share has landed.
    // Z, the fp32 partial and the chain counters are zeroed by one memset.
    uint8_t* z0 = reinterpret_cast<uint8_t*>(ws.zb);
    DL_TRY(cuda_status(cudaMemsetAsync(z0, 0, static_cast<uint8_t*>(workspace) + cv.off - z0, st), "memset"));
    GemmProblem p1 = one_seg(X, ldx, T, n, B, ldb, k, n, out_plain(ws.zb, ws.ldzb, OUT_BF16_RED, 0));
    GemmProblem p2 = one_seg(ws.zb, ws.ldzb, T, k, A, lda, m, k, partial_out(OUT_F32_RED));
    if (use_chain()) {
      DL_TRY(tc_gemm_chain(p1, p2, ws.chain, st));
    } else {
      DL_TRY(tc_gemm(p1, true, st));
      DL_TRY(tc_gemm(p2, true, st));
    }
    return finish();
  }
  // PATH_WIDE: whole-tile, bf16 Z straight from the epilogue
  DL_TRY(tc_gemm(one_seg(X, ldx, T, n, B, ldb, k, n, out_plain(ws.zb, ws.ldzb, OUT_BF16, 0)), false, st));
  if (!pl.coll)
    return tc_gemm(one_seg(ws.zb, ws.ldzb, T, k, A, lda, m, k, out_plain(Y, ldy, OUT_BF16, accumulate)), false, st);
  DL_TRY(tc_gemm(one_seg(ws.zb, ws.ldzb, T, k, A, lda, m, k, partial_out(OUT_F32_STORE)), false, st));
  return finish();
}

// Test hook for the rank-major activation layout the TP o projection reads
// straight from the attention all-gather (3-D TMA map; include/dl.h).
dl_status dl_debug_linear_gathered(const void* Xg, int P, const void* A, int64_t lda, const void* B, int64_t ldb,
                                   void* Y, int64_t ldy, int64_t T, int64_t m, int64_t n, int64_t k, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  if (P < 1 || T < 1 || T > 256 || n % P || (n / P) % 64 || m % 4) {
    set_error("dl_debug_linear_gathered: need 1 <= T <= 256, n / P a multiple of 64, m %% 4 == 0");
    return DL_ERR_SHAPE;
  }
  // the skinny tensor path at every T (workspace: dl_lowrank_linear_workspace with T >= 17)
  const LinPlan pl{PATH_SKINNY, false, true, 1};
  Carver need(nullptr);
  carve_lin(need, T, m, k, pl, DL_REDUCE_NONE);
  if (!workspace || workspace_bytes < need.off) {
    set_error("workspace too small (%zu < %zu)", workspace_bytes, need.off);
    return DL_ERR_WORKSPACE;
  }
  DL_TRY(check_device());
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Carver cv(workspace);
  const LinWs ws = carve_lin(cv, T, m, k, pl, DL_REDUCE_NONE);
  DL_TRY(cuda_status(cudaMemsetAsync(ws.zf, 0, sizeof(float) * T * ws.ldz32, st), "memset"));
  DL_TRY(cuda_status(cudaMemsetAsync(ws.yf, 0, sizeof(float) * T * ws.ldy32, st), "memset"));
  GemmProblem p1 = one_seg(Xg, n, T, n, B, ldb, k, n, out_plain(ws.zf, ws.ldz32, OUT_F32_RED, 0));
  p1.act_p = P;
  p1.act_w = n / P;
  DL_TRY(tc_gemm(p1, true, st));
  DL_TRY(launch_f32_to_bf16(ws.zf, ws.ldz32, ws.zb, ws.ldzb, T, rup(k, 4), 1, st));
  DL_TRY(tc_gemm(one_seg(ws.zb, ws.ldzb, T, k, A, lda, m, k, out_plain(ws.yf, ws.ldy32, OUT_F32_RED, 0)), true, st));
  return launch_f32_to_bf16(ws.yf, ws.ldy32, static_cast<__nv_bfloat16*>(Y), ldy, T, m, 1, st);
}

// ---------------------------------------------------------------------------
// rank-shard planner
// ---------------------------------------------------------------------------
dl_status dl_tp_plan(const int64_t* seg_ranks, int n_seg, int world, int rank, int strict, int64_t* seg_begin,
                     int64_t* seg_len, int64_t* k_loc) {
  if (!seg_ranks || !seg_begin || !seg_len || n_seg < 1 || n_seg > 3) {
    set_error("dl_tp_plan: bad arguments");
    return DL_ERR_INVALID_ARG;
  }
  if (world < 1 || rank < 0 || rank >= world) {
    set_error("dl_tp_plan: bad rank %d / world %d", rank, world);
    return DL_ERR_PARTITION;
  }
  int64_t R = 0;
  for (int g = 0; g < n_seg; ++g) {
    if (seg_ranks[g] < 1) {
      set_error("dl_tp_plan: segment %d rank %lld < 1", g, (long long)seg_ranks[g]);
      return DL_ERR_RANK;
    }
    R += seg_ranks[g];
  }
  if (R < world) {
    set_error("dl_tp_plan: total rank %lld < world %d", (long long)R, world);
    return DL_ERR_PARTITION;
  }
  if (strict && R % world != 0) {
    set_error("dl_tp_plan: strict split of %lld over %d ranks is uneven", (long long)R, world);
    return DL_ERR_PARTITION;
  }
  // balanced contiguous split of the concatenated range [0, R)
  const int64_t base = R / world, extra = R % world;
  const int64_t lo = rank * base + std::min<int64_t>(rank, extra);
  const int64_t hi = lo + base + (rank < extra ? 1 : 0);
  int64_t off = 0, total = 0;
  for (int g = 0; g < n_seg; ++g) {
    const int64_t a = std::max(lo, off), b = std::min(hi, off + seg_ranks[g]);
    seg_begin[g] = std::max<int64_t>(0, a - off);
    seg_len[g] = std::max<int64_t>(0, b - a);
    if (seg_len[g] == 0) seg_begin[g] = 0;
    total += seg_len[g];
    off += seg_ranks[g];
  }
  if (k_loc) *k_loc = total;
  return DL_OK;
}

dl_status dl_tp_shard_factors(int n_seg, const void* const* A, const int64_t* lda, const void* const* B,
                              const int64_t* ldb, const int64_t* m, const int64_t* r, int64_t n, dl_dtype dtype,
                              int world, int rank, int strict, void* B_shard, int64_t ldb_shard,
                              void* const* A_shard, const int64_t* lda_shard, int64_t* seg_len_out, void* stream) {
  if (!A || !lda || !B || !ldb || !m || !r || !A_shard || !lda_shard || !B_shard) {
    set_error("dl_tp_shard_factors: null argument");
    return DL_ERR_INVALID_ARG;
  }
  int64_t beg[3], len[3], kloc = 0;
  DL_TRY(dl_tp_plan(r, n_seg, world, rank, strict, beg, len, &kloc));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t es = esize(dtype);
  DL_TRY(check_ld(ldb_shard, n, dtype, "ldb_shard"));
  int64_t row = 0;
  for (int g = 0; g < n_seg; ++g) {
    if (len[g] > 0) {
      DL_TRY(check_ld(lda_shard[g], len[g], dtype, "lda_shard"));
      const uint8_t* bsrc = static_cast<const uint8_t*>(B[g]) + beg[g] * ldb[g] * es;
      uint8_t* bdst = static_cast<uint8_t*>(B_shard) + row * ldb_shard * es;
      DL_TRY(launch_copy2d(bsrc, ldb[g] * es, bdst, ldb_shard * es, len[g], n * es, st));
      const uint8_t* asrc = static_cast<const uint8_t*>(A[g]) + beg[g] * es;
      DL_TRY(launch_copy2d(asrc, lda[g] * es, A_shard[g], lda_shard[g] * es, m[g], len[g] * es, st));
      row += len[g];
    }
    if (seg_len_out) seg_len_out[g] = len[g];
  }
  return DL_OK;
}

dl_status dl_deinfer_shard_factors(int sublayer, int n_seg, const void* const* A, const int64_t* lda,
                                   const void* const* B, const int64_t* ldb, const int64_t* m, const int64_t* r,
                                   int64_t n, dl_dtype dtype, int world, int rank, void* B_shard, int64_t ldb_shard,
                                   void* const* A_shard, const int64_t* lda_shard, void* stream) {
  if (!A || !lda || !B || !ldb || !m || !r || !A_shard || !lda_shard || !B_shard) {
    set_error("dl_deinfer_shard_factors: null argument");
    return DL_ERR_INVALID_ARG;
  }
  if ((sublayer != 1 && sublayer != 2) || n_seg < 1 || n_seg > 3 || (sublayer == 2 && n_seg != 1)) {
    set_error("dl_deinfer_shard_factors: sublayer %d / n_seg %d invalid", sublayer, n_seg);
    return DL_ERR_INVALID_ARG;
  }
  if (world < 1 || rank < 0 || rank >= world) {
    set_error("dl_deinfer_shard_factors: rank %d / world %d invalid", rank, world);
    return DL_ERR_PARTITION;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t es = esize(dtype);
  if (sublayer == 1) {
    // B: the rank's balanced share of the concatenated rows (as dl_tp_shard_factors)
    int64_t beg[3], len[3], kloc = 0;
    DL_TRY(dl_tp_plan(r, n_seg, world, rank, 0, beg, len, &kloc));
    DL_TRY(check_ld(ldb_shard, n, dtype, "ldb_shard"));
    int64_t row = 0;
    for (int g = 0; g < n_seg; ++g) {
      if (m[g] % world != 0) {
        set_error("dl_deinfer_shard_factors: m[%d] = %lld not divisible by world %d", g, (long long)m[g], world);
        return DL_ERR_PARTITION;
      }
      if (len[g] > 0) {
        const uint8_t* bsrc = static_cast<const uint8_t*>(B[g]) + beg[g] * ldb[g] * es;
        uint8_t* bdst = static_cast<uint8_t*>(B_shard) + row * ldb_shard * es;
        DL_TRY(launch_copy2d(bsrc, ldb[g] * es, bdst, ldb_shard * es, len[g], n * es, st));
        row += len[g];
      }
      // A: rows of the rank's output features, every latent column
      const int64_t ml = m[g] / world;
      DL_TRY(check_ld(lda_shard[g], r[g], dtype, "lda_shard"));
      const uint8_t* asrc = static_cast<const uint8_t*>(A[g]) + rank * ml * lda[g] * es;
      DL_TRY(launch_copy2d(asrc, lda[g] * es, A_shard[g], lda_shard[g] * es, ml, r[g] * es, st));
    }
    return DL_OK;
  }
  if (n % world != 0) {
    set_error("dl_deinfer_shard_factors: n = %lld not divisible by world %d", (long long)n, world);
    return DL_ERR_PARTITION;
  }
  const int64_t nl = n / world;
  DL_TRY(check_ld(ldb_shard, nl, dtype, "ldb_shard"));
  DL_TRY(check_ld(lda_shard[0], r[0], dtype, "lda_shard"));
  const uint8_t* bsrc = static_cast<const uint8_t*>(B[0]) + rank * nl * es;
  DL_TRY(launch_copy2d(bsrc, ldb[0] * es, B_shard, ldb_shard * es, r[0], nl * es, st));
  return launch_copy2d(A[0], lda[0] * es, A_shard[0], lda_shard[0] * es, m[0], r[0] * es, st);
}

// ---------------------------------------------------------------------------
// decomposed block
// ---------------------------------------------------------------------------
namespace {

struct BlockDims {
  int64_t h, hkv, m, H, Hk, d, P;
  int64_t Hq_loc, Hk_loc, W;       // local heads, RS slab width
  int64_t k_qkv, k_o, k_gu, k_down, kmax;
  int64_t nmax;                    // widest stage-2 output (features)
  bool glu;                        // SiLU-GLU MLP (else ReLU on up alone)
  int layout;                      // DL_LAYOUT_*
  int64_t lat_slot;                // DeInfer: per-rank latent slice width in the all-gather
};

dl_status block_dims(const dl_block_config* c, int world, BlockDims* d) {
  if (!c) {
    set_error("cfg is NULL");
    return DL_ERR_INVALID_ARG;
  }
  if (c->h <= 0 || c->n_heads <= 0 || c->n_kv_heads <= 0 || c->head_dim <= 0 || c->m <= 0) {
    set_error("bad block dims");
    return DL_ERR_SHAPE;
  }
  if (c->n_heads * c->head_dim != c->h || c->n_heads % c->n_kv_heads != 0) {
    set_error("h must equal n_heads*head_dim and n_heads %% n_kv_heads == 0");
    return DL_ERR_SHAPE;
  }
  if (c->head_dim != 128) {
    set_error("head_dim %lld unsupported (128)", (long long)c->head_dim);
    return DL_ERR_UNSUPPORTED;
  }
  if (world < 1 || c->n_heads % world != 0 || c->n_kv_heads % world != 0) {
    set_error("heads (%lld q, %lld kv) not divisible by world %d", (long long)c->n_heads,
              (long long)c->n_kv_heads, world);
    return DL_ERR_PARTITION;
  }
  if (c->mlp_act != DL_MLP_SILU_GLU && c->mlp_act != DL_MLP_RELU) {
    set_error("mlp_act %d unknown", c->mlp_act);
    return DL_ERR_INVALID_ARG;
  }
  const bool glu = c->mlp_act == DL_MLP_SILU_GLU;
  if (!glu && c->rank_gate != 0) {
    set_error("DL_MLP_RELU has no gate: rank_gate must be 0");
    return DL_ERR_RANK;
  }
  const int64_t hkv = c->n_kv_heads * c->head_dim;
  const int64_t ranks[7] = {c->rank_q, c->rank_k, c->rank_v, c->rank_o, c->rank_gate, c->rank_up, c->rank_down};
  const int64_t mins[7] = {c->h, hkv, hkv, c->h, std::min(c->h, c->m), std::min(c->h, c->m), std::min(c->h, c->m)};
  for (int i = 0; i < 7; ++i)
    if (!(i == 4 && !glu) && (ranks[i] < 1 || ranks[i] > mins[i])) {
      set_error("rank %d = %lld outside [1, %lld]", i, (long long)ranks[i], (long long)mins[i]);
      return DL_ERR_RANK;
    }
  if (c->h % 64 || c->m % 64) {
    set_error("h and m must be multiples of 64");
    return DL_ERR_UNSUPPORTED;
  }
  d->h = c->h; d->hkv = hkv; d->m = c->m; d->H = c->n_heads; d->Hk = c->n_kv_heads; d->d = c->head_dim;
  d->P = world;
  d->Hq_loc = c->n_heads / world;
  d->Hk_loc = c->n_kv_heads / world;
  d->W = (c->h + 2 * hkv) / world;
  auto cdiv = [](int64_t a, int64_t b) { return (a + b - 1) / b; };
  d->k_qkv = cdiv(c->rank_q + c->rank_k + c->rank_v, world);
  d->k_o = cdiv(c->rank_o, world);
  d->k_gu = cdiv(c->rank_gate + c->rank_up, world);
  d->k_down = cdiv(c->rank_down, world);
  // Z columns: every segment starts on a 64-column (one K block) boundary
  d->kmax = std::max(std::max(d->k_qkv, d->k_o), std::max(d->k_gu, d->k_down)) + 3 * 64;
  d->nmax = std::max(c->h + 2 * hkv, (glu ? 2 : 1) * c->m);
  d->glu = glu;
  d->layout = c->layout;
  d->lat_slot = 0;
  if (c->layout != DL_LAYOUT_RANK_PARALLEL && c->layout != DL_LAYOUT_DEINFER) {
    set_error("layout %d unknown", c->layout);
    return DL_ERR_INVALID_ARG;
  }
  if (c->layout == DL_LAYOUT_DEINFER) {
    if (c->m % (64 * world) || c->h % (64 * world)) {
      set_error("DeInfer layout needs h and m divisible by 64 * world");
      return DL_ERR_PARTITION;
    }
    // stage 2 of q|k|v and gate|up reads the FULL latent (all-gathered);
    // o / down stage 2 reads the full reduced latent
    auto zw = [](std::initializer_list<int64_t> ks) {
      int64_t w = 0;
      for (int64_t k : ks) w += rup(k, 64);
      return w;
    };
    const int64_t Lqkv = c->rank_q + c->rank_k + c->rank_v;
    const int64_t Lgu = c->rank_gate + c->rank_up;
    d->lat_slot = rup(cdiv(std::max(Lqkv, Lgu), world), 64);
    d->kmax = std::max({zw({c->rank_q, c->rank_k, c->rank_v}), zw({c->rank_gate, c->rank_up}),
                        rup(c->rank_o, 64), rup(c->rank_down, 64), d->lat_slot}) + 64;
  }
  return DL_OK;
}

// Stream-K launches rotate over kSchedSlots counter pairs.  A kernel touches
// its pair only after griddepcontrol.wait (transitively: every earlier kernel
// has completed and its last CTA has reset the pair it used), so reuse is safe
// at any distance; the rotation is margin.  Small grids let many PDL-launched
// kernels be resident at once: a dynamic-chunk grab before the wait once stole
// units of a still-running launch two chain kernels back (fixed in tc_gemm.cu).
constexpr int kSchedSlots = 8;
// prefill tail scratch: up to 56 tiles of 256 x 256 fp32 (>= 75% of 74 clusters)
constexpr size_t kTailBytes = static_cast<size_t>(56) * 256 * 256 * 4;
// The rotation is per host thread: a stream is driven by one thread, so a
// process-wide counter would let another thread's launches (group ranks, one
// thread each) hand two consecutive launches of one stream the same slot.
unsigned int* next_sched(unsigned int* base) {
  static thread_local unsigned slot = 0;
  return base + 2 * (slot++ % kSchedSlots);
}
unsigned int* next_chain(unsigned int* base) {
  static thread_local unsigned slot = 0;
  return base + 2 * (slot++ % kSchedSlots);
}


struct BlockWs {
  float* zf; float* yf;              // fp32 reduction targets (zero-maintained)
  __nv_bfloat16 *xn, *zb, *yb, *rs, *q, *att, *att_full, *ag, *act;
  __nv_bfloat16* zr;                 // skinny stage-1 Z, bf16 red.add target (zero-maintained)
  __nv_bfloat16* yr;                 // skinny TP stage-2 partials, bf16 red.add target = collective buffer (zero-maintained)
  __nv_bfloat16* yr2;                // [Ts x h] the same for the o / down outputs of the skinny TP path
  float* apart;                      // split-KV attention partials (decode)
  size_t apart_bytes;
  void* ask;                         // stream-K decode attention: counters + partial slots
  int64_t ask_items;
  unsigned int* sched;               // kSchedSlots x 2 stream-K work counters
  unsigned int* chain;               // kSchedSlots x 2 fused-chain arrival counters (tc_gemm_chain)
  unsigned int* tile_cnt;            // stream-K fixup arrival counters (one per output tile)
  float* tail;                       // prefill DP + stream-K tail scratch (zero-maintained)
  size_t tail_bytes;
  __nv_bfloat16 *lat_send, *lat_recv;   // DeInfer latent all-gather [T x slot] / [P][T][slot]
  __nv_bfloat16* lat_red;                // DeInfer skinny: stage-1 latent slice, bf16x2 red.add target (zero-maintained)
  int64_t ldz32, ldzb, ldy32;
};

// Fused collectives of the skinny rank-parallel path (group communicator):
// three zero-maintained bf16 buffers in every rank's symmetric window, at the
// same offsets on every rank.  X = reduce-scatter target [T x W] and, later in
// the block, the gate|up all-reduce [T x 2m]; Y = the o and down all-reduces
// [T x h]; G = the attention all-gather [P][T][h/P].  Consecutive collectives
// alternate X / Y, so a rank writes a buffer only after a barrier that every
// rank reached after consuming (and clearing) that buffer's previous use.
struct FanBufs {
  bool on = false;
  __nv_bfloat16 *X = nullptr, *Y = nullptr, *G = nullptr;
  int64_t delta[8] = {};
};
size_t fan_window_bytes(const BlockDims& d, int64_t Tmax) {
  const size_t Ts = static_cast<size_t>(std::min<int64_t>(Tmax, 256));
  const size_t nx = static_cast<size_t>(std::max<int64_t>(d.W, (d.glu ? 2 : 1) * d.m));
  return rup_sz(Ts * nx * 2) + 2 * rup_sz(Ts * static_cast<size_t>(d.h) * 2);
}

BlockWs carve_block(Carver& c, const BlockDims& d, int64_t Tmax) {
  BlockWs w{};
  const int64_t Ts = std::min<int64_t>(Tmax, 256);   // skinny path bound
  w.ldz32 = rup(d.kmax, 64);
  w.ldzb = rup(d.kmax, 64);
  w.ldy32 = rup(d.nmax, 4);
  w.zf = c.take<float>(static_cast<size_t>(Ts) * w.ldz32);
  w.yf = c.take<float>(static_cast<size_t>(Ts) * w.ldy32);
  w.xn = c.take<__nv_bfloat16>(static_cast<size_t>(Tmax) * d.h);
  w.zb = c.take<__nv_bfloat16>(static_cast<size_t>(Tmax) * w.ldzb);
  // bf16 red.add targets of the skinny stage 1, zero-maintained: two column
  // slots per row ([t][slot][ldzb]) so the gate|up latent (slot 1) may stay
  // live until the down group's finalize clears both
  w.zr = c.take<__nv_bfloat16>(static_cast<size_t>(Ts) * 2 * w.ldzb);
  w.yr = c.take<__nv_bfloat16>(static_cast<size_t>(Ts) * rup(d.nmax, 8));
  w.yr2 = c.take<__nv_bfloat16>(static_cast<size_t>(Ts) * d.h);
  w.yb = c.take<__nv_bfloat16>(static_cast<size_t>(Tmax) * rup(d.nmax, 8));
  w.rs = c.take<__nv_bfloat16>(static_cast<size_t>(Tmax) * d.W);
  w.q = c.take<__nv_bfloat16>(static_cast<size_t>(Tmax) * d.Hq_loc * d.d);
  w.att = c.take<__nv_bfloat16>(static_cast<size_t>(Tmax) * d.Hq_loc * d.d);
  // all-gather buffers (TP path; also present at P = 1 so the TP path can be tested)
  w.att_full = c.take<__nv_bfloat16>(static_cast<size_t>(Tmax) * d.h);
  w.ag = c.take<__nv_bfloat16>(static_cast<size_t>(Tmax) * d.h);
  w.act = c.take<__nv_bfloat16>(static_cast<size_t>(Tmax) * d.m);
  w.apart_bytes = attention_workspace(Ts, static_cast<int>(d.Hq_loc), static_cast<int>(d.d));
  w.apart = c.take<float>(w.apart_bytes / sizeof(float));
  w.ask_items = Tmax * d.Hq_loc;
  w.ask = c.take<float>(attention_sk_workspace(Tmax, static_cast<int>(d.Hq_loc)) / sizeof(float));
  w.sched = c.take<unsigned int>(2 * kSchedSlots);
  w.chain = c.take<unsigned int>(2 * kSchedSlots);
  w.tile_cnt = c.take<unsigned int>(static_cast<size_t>((d.nmax + d.kmax) / 128 + 64));
  w.tail_bytes = Tmax > 256 ? kTailBytes : 0;
  w.tail = w.tail_bytes ? c.take<float>(w.tail_bytes / sizeof(float)) : nullptr;
  if (d.layout == DL_LAYOUT_DEINFER) {
    w.lat_send = c.take<__nv_bfloat16>(static_cast<size_t>(Tmax) * d.lat_slot);
    w.lat_red = c.take<__nv_bfloat16>(static_cast<size_t>(Ts) * d.lat_slot);   // skinny bf16x2 target, zero-maintained
    w.lat_recv = c.take<__nv_bfloat16>(static_cast<size_t>(Tmax) * d.P * d.lat_slot);
  }
  return w;
}

dl_status check_group(const dl_factor_group& g, int nseg, int64_t n, const char* name, int64_t* k_loc) {
  int64_t k = 0;
  for (int s = 0; s < nseg; ++s) {
    if (g.seg[s].k < 0) {
      set_error("%s: negative segment rank", name);
      return DL_ERR_RANK;
    }
    if (g.seg[s].k > 0) {
      DL_TRY(check_ptr(g.seg[s].A, name));
      DL_TRY(check_ld(g.seg[s].lda, g.seg[s].k, DL_BF16, name));
    }
    k += g.seg[s].k;
  }
  if (k < 1) {
    set_error("%s: rank shard is empty", name);
    return DL_ERR_PARTITION;
  }
  DL_TRY(check_ptr(g.B, name));
  DL_TRY(check_ld(g.ldb, n, DL_BF16, name));
  *k_loc = k;
  return DL_OK;
}

// Z column layout of a group: segment g occupies [off_g, off_g + rup(k_g, 64)),
// so every stage-2 TMA box starts on a K-block boundary of its own segment.
struct ZLayout {
  int64_t off[3];
  int64_t width;
};
ZLayout zlayout(const dl_factor_group& g, int nseg) {
  ZLayout z{};
  int64_t o = 0;
  for (int s = 0; s < nseg; ++s) {
    z.off[s] = o;
    o += rup(g.seg[s].k, 64);
  }
  z.width = o;
  return z;
}

// stage 1: Z[:, off_g + j] = act . B_g[j]^T for the rows of B belonging to segment g
GemmProblem stage1(const dl_factor_group& grp, int nseg, const void* act, int64_t ld_act, int64_t T, int64_t n,
                   const ZLayout& zl, GemmOut out) {
  GemmProblem p{};
  p.act = act;
  p.ld_act = ld_act;
  p.T = T;
  p.k_act = n;
  p.nseg = nseg;
  int64_t row = 0;
  out.remap_cols = 1;
  for (int s = 0; s < nseg; ++s) {
    const int64_t k = grp.seg[s].k;
    p.seg[s] = GemmSeg{static_cast<const __nv_bfloat16*>(grp.B) + row * grp.ldb, grp.ldb, k, n, row, 0};
    out.seg_col_off[s] = zl.off[s];
    out.seg_write_rows[s] = rup(k, 64);
    row += k;
  }
  p.n_feat = row;
  p.out = out;
  return p;
}

// stage 2: segment g writes features [begin_g, begin_g + rows_g) from Z[:, off_g ...]
GemmProblem stage2(const dl_factor_group& grp, int nseg, const int64_t* rows, const __nv_bfloat16* zb, int64_t ldzb,
                   int64_t T, const ZLayout& zl, GemmOut out) {
  GemmProblem p{};
  p.act = zb;
  p.ld_act = ldzb;
  p.T = T;
  p.k_act = zl.width;
  p.nseg = nseg;
  int64_t fb = 0;
  for (int s = 0; s < nseg; ++s) {
    p.seg[s] = GemmSeg{grp.seg[s].A, grp.seg[s].lda, rows[s], grp.seg[s].k, fb, zl.off[s]};
    fb += rows[s];
  }
  p.n_feat = fb;
  p.out = out;
  return p;
}

// One factor group: Z = act . B^T (Z kept as bf16 in the workspace), then
// Y = Z . A_g^T into `out2` (skinny: stream-K fp32 reduction; wide: bf16).
// Stream-K last-contributor fixups are opt-in (DL_FIXUP=1).  Measured on B200
// (tools/decode_timeline.py, 4 x 70B layers): 2.2-2.5 ms with fixups vs
// 1.8-1.9 ms with separate finalize kernels -- under static stream-K every
// tile's last contributor finishes at the end of its range, so all finalizes
// (and their fence / counter round trips) pile onto the kernel's tail, while a
// PDL-launched finalize kernel overlaps the GEMM drain.
bool use_fixup() {
  static const bool on = DL_ENV("DL_FIXUP") && atoi(DL_ENV("DL_FIXUP")) != 0;
  return on;
}

// One factor group: Z = act . B^T (bf16 Z in the workspace), then
// Y = Z . A_g^T into `out2` (skinny: stream-K fp32 reduction; wide: bf16).
// Skinny path: stage 1 finalizes Z to bf16 in its last-contributor fixup; a
// stage-2 fixup `fix2` (op != FIX_NONE) finalizes the group output in place
// of a separate kernel (then `out2` only supplies the output pointer/layout).
bool use_zred() {
  static const bool on = !DL_ENV("DL_ZRED") || atoi(DL_ENV("DL_ZRED")) != 0;   // A/B switch (default on)
  return on;
}

// zero_out != NULL (skinny path): stage 1 red.adds its partials straight into
// the bf16 Z buffer ws.zr (no fp32 -> bf16 pass); *zero_out is then the clear
// of that buffer, which the caller hands to the kernel that follows stage 2.
// In-kernel activation of a stage 1 (GemmProblem::xform): mode, reduced
// gate|up rows and their layout.
struct Xform {
  int mode = XFORM_NONE;
  const __nv_bfloat16* src = nullptr;
  int64_t ld = 0, m = 0;
};

dl_status run_group(const dl_factor_group& grp, int nseg, const int64_t* rows, const __nv_bfloat16* act,
                    int64_t ld_act, int64_t n, int64_t T, bool skinny, const BlockWs& ws, const GemmOut& out2,
                    cudaStream_t st, const GemmFixup* fix2 = nullptr, SideZero* zero_out = nullptr,
                    int zslot = 0, int act_p = 0, int64_t act_w = 0, const Xform& xf = Xform{}, int glu = 0) {
  // act_p > 1 (skinny only): act is a rank-major all-gather output read through a 3-D map
  const ZLayout zl = zlayout(grp, nseg);
  if (zero_out) *zero_out = SideZero{};
  if (skinny && zero_out && use_zred() && !use_fixup()) {
    __nv_bfloat16* z = ws.zr + zslot * ws.ldzb;
    const int64_t ldz = 2 * ws.ldzb;
    GemmProblem p1 = stage1(grp, nseg, act, ld_act, T, n, zl, out_plain(z, ldz, OUT_BF16_RED, 0));
    p1.sched = next_sched(ws.sched);
    p1.act_p = act_p;
    p1.act_w = act_w;
    p1.xform = xf.mode;
    p1.xsrc = xf.src;
    p1.xld = xf.ld;
    p1.xm = xf.m;
    GemmProblem p2 = stage2(grp, nseg, rows, z, ldz, T, zl, out2);
    p2.sched = next_sched(ws.sched);
    if (fix2 && fix2->op != FIX_NONE) p2.fix = *fix2;
    if (use_chain_block()) {
      DL_TRY(tc_gemm_chain(p1, p2, next_chain(ws.chain), st));
    } else {
      DL_TRY(tc_gemm(p1, true, st));
      DL_TRY(tc_gemm(p2, true, st));
    }
    zero_out->p = z;
    zero_out->ld = ldz * 2;
    zero_out->rows = T;
    zero_out->row_bytes = zl.width * 2;
    return DL_OK;
  }
  if (skinny) {
    if (use_fixup()) {
      GemmProblem p1 = stage1(grp, nseg, act, ld_act, T, n, zl, out_plain(ws.zb, ws.ldzb, OUT_BF16, 0));
      p1.sched = next_sched(ws.sched);
      p1.act_p = act_p;
      p1.act_w = act_w;
      p1.fix.op = FIX_BF16;
      p1.fix.acc32 = ws.zf;
      p1.fix.acc_ld = ws.ldz32;
      p1.fix.tile_cnt = ws.tile_cnt;
      DL_TRY(tc_gemm(p1, true, st));
    } else {
      GemmProblem p1 = stage1(grp, nseg, act, ld_act, T, n, zl, out_plain(ws.zf, ws.ldz32, OUT_F32_RED, 0));
      p1.sched = next_sched(ws.sched);
      p1.act_p = act_p;
      p1.act_w = act_w;
      DL_TRY(tc_gemm(p1, true, st));
      DL_TRY(launch_f32_to_bf16(ws.zf, ws.ldz32, ws.zb, ws.ldzb, T, zl.width, 1, st));
    }
  } else {
    GemmProblem p1 = stage1(grp, nseg, act, ld_act, T, n, zl, out_plain(ws.zb, ws.ldzb, OUT_BF16, 0));
    p1.tail_acc = ws.tail;
    p1.tail_bytes = ws.tail_bytes;
    DL_TRY(tc_gemm(p1, false, st));
  }
  GemmProblem p2 = stage2(grp, nseg, rows, ws.zb, ws.ldzb, T, zl, out2);
  if (skinny) {
    p2.sched = next_sched(ws.sched);
    if (fix2 && fix2->op != FIX_NONE) p2.fix = *fix2;
  } else {
    p2.tail_acc = ws.tail;
    p2.tail_bytes = ws.tail_bytes;
    p2.glu = glu;   // out2 is then the [T x m] activation
  }
  return tc_gemm(p2, skinny, st);
}

// DeInfer first sub-layer (Fig. 3) of a q|k|v or gate|up group:
// stage 1 on the rank's concat-split B rows -> latent slice [T x k_loc];
// all-gather of the slices (the low-rank communication); un-permute into the
// group's Z layout; stage 2 with the rank's row shards of A (all l columns).
// out2 receives the rank's local features [T x sum rows_loc].
// Stage 1 + latent all-gather + un-permute: the full latent Z of the group in
// ws.zb (segment-aligned layout zlayout(grp, nseg)).
dl_status deinfer_latent(const dl_factor_group& grp, int nseg, const __nv_bfloat16* act, int64_t ld_act, int64_t n,
                         int64_t T, bool skinny, const BlockWs& ws, const BlockDims& d, dl_comm comm, cudaStream_t st) {
  int64_t lens[3], beg[3], len[3], kloc = 0;
  for (int s = 0; s < nseg; ++s) lens[s] = grp.seg[s].k;
  DL_TRY(dl_tp_plan(lens, nseg, comm->world, comm->rank, 0, beg, len, &kloc));
  const bool red16 = skinny && use_zred();   // latent slice reduced as bf16x2 straight into the send buffer
  if (red16) {
    GemmProblem p1 = one_seg(act, ld_act, T, n, grp.B, grp.ldb, kloc, n, out_plain(ws.lat_red, d.lat_slot, OUT_BF16_RED, 0));
    p1.sched = next_sched(ws.sched);
    DL_TRY(tc_gemm(p1, true, st));
  } else if (skinny) {
    GemmProblem p1 = one_seg(act, ld_act, T, n, grp.B, grp.ldb, kloc, n, out_plain(ws.zf, ws.ldz32, OUT_F32_RED, 0));
    p1.sched = next_sched(ws.sched);
    DL_TRY(tc_gemm(p1, true, st));
    DL_TRY(launch_f32_to_bf16(ws.zf, ws.ldz32, ws.lat_send, d.lat_slot, T, rup(kloc, 4), 1, st));
  } else {
    GemmProblem p1 = one_seg(act, ld_act, T, n, grp.B, grp.ldb, kloc, n, out_plain(ws.lat_send, d.lat_slot, OUT_BF16, 0));
    p1.tail_acc = ws.tail;
    p1.tail_bytes = ws.tail_bytes;
    DL_TRY(tc_gemm(p1, false, st));
  }
  DL_TRY(coll_all_gather(comm, red16 ? ws.lat_red : ws.lat_send, ws.lat_recv, static_cast<size_t>(T) * d.lat_slot,
                    kCollBF16, st));
  const ZLayout zl = zlayout(grp, nseg);
  LatentMap mp{};
  mp.nseg = nseg;
  mp.P = comm->world;
  mp.T = T;
  mp.slot = d.lat_slot;
  int64_t L = 0;
  for (int s = 0; s < nseg; ++s) {
    mp.seg_beg[s] = L;
    mp.seg_len[s] = lens[s];
    mp.zoff[s] = zl.off[s];
    L += lens[s];
  }
  mp.base = L / comm->world;
  mp.extra = L % comm->world;
  mp.width = zl.width;
  SideZero z;   // the un-permute runs after the all-gather read the send buffer: clear it there
  if (red16) {
    z.p = ws.lat_red;
    z.rows = 1;
    z.row_bytes = z.ld = static_cast<int64_t>(T) * d.lat_slot * 2;
  }
  return launch_latent_unpermute(ws.lat_recv, ws.zb, ws.ldzb, mp, st, z);
}

dl_status deinfer_first(const dl_factor_group& grp, int nseg, const int64_t* rows_loc, const __nv_bfloat16* act,
                        int64_t ld_act, int64_t n, int64_t T, bool skinny, const BlockWs& ws, const BlockDims& d,
                        dl_comm comm, const GemmOut& out2, cudaStream_t st) {
  DL_TRY(deinfer_latent(grp, nseg, act, ld_act, n, T, skinny, ws, d, comm, st));
  const ZLayout zl = zlayout(grp, nseg);
  GemmProblem p2 = stage2(grp, nseg, rows_loc, ws.zb, ws.ldzb, T, zl, out2);
  if (skinny) {
    p2.sched = next_sched(ws.sched);
  } else {
    p2.tail_acc = ws.tail;
    p2.tail_bytes = ws.tail_bytes;
  }
  return tc_gemm(p2, skinny, st);
}

// DeInfer second sub-layer (o or down): stage 1 with the rank's input-column
// shard of B on its local activations -> partial latent [T x l]; reduce-sum
// of the latent (bf16 payload: decode partials red.add-ed as bf16x2 into the
// all-reduce buffer, prefill bf16 epilogue stores; fp32 only with the
// DL_ZRED=0 A/B switch); stage 2
// with the replicated A, residual added into x.
dl_status deinfer_second(const dl_factor_group& grp, const __nv_bfloat16* act, int64_t n_loc, int64_t m_out,
                         int64_t T, bool skinny, const BlockWs& ws, dl_comm comm, __nv_bfloat16* x, cudaStream_t st) {
  const int64_t l = grp.seg[0].k;
  if (skinny && use_zred()) {
    // latent partial as bf16x2 straight into the all-reduce buffer (contiguous
    // [T x rup(l, 8)] in ws.yr), reduced in place, read by stage 2, cleared by
    // the residual kernel
    const int64_t ldl = rup(l, 8);
    GemmProblem p1 = one_seg(act, n_loc, T, n_loc, grp.B, grp.ldb, l, n_loc, out_plain(ws.yr, ldl, OUT_BF16_RED, 0));
    p1.sched = next_sched(ws.sched);
    DL_TRY(tc_gemm(p1, true, st));
    DL_TRY(coll_all_reduce(comm, ws.yr, static_cast<size_t>(T) * ldl, kCollBF16, st));
    GemmProblem p2 = one_seg(ws.yr, ldl, T, l, grp.seg[0].A, grp.seg[0].lda, m_out, l,
                             out_plain(ws.yf, ws.ldy32, OUT_F32_RED, 0));
    p2.sched = next_sched(ws.sched);
    DL_TRY(tc_gemm(p2, true, st));
    SideZero z;
    z.p = ws.yr;
    z.rows = 1;
    z.row_bytes = z.ld = T * ldl * 2;
    return launch_residual_add_f32(ws.yf, ws.ldy32, x, m_out, T, m_out, 1, st, z);
  }
  if (skinny) {
    GemmProblem p1 = one_seg(act, n_loc, T, n_loc, grp.B, grp.ldb, l, n_loc, out_plain(ws.zf, ws.ldz32, OUT_F32_RED, 0));
    p1.sched = next_sched(ws.sched);
    DL_TRY(tc_gemm(p1, true, st));
    DL_TRY(coll_all_reduce(comm, ws.zf, static_cast<size_t>(T) * ws.ldz32, kCollF32, st));
    DL_TRY(launch_f32_to_bf16(ws.zf, ws.ldz32, ws.zb, ws.ldzb, T, rup(l, 4), 1, st));
    GemmProblem p2 = one_seg(ws.zb, ws.ldzb, T, l, grp.seg[0].A, grp.seg[0].lda, m_out, l,
                             out_plain(ws.yf, ws.ldy32, OUT_F32_RED, 0));
    p2.sched = next_sched(ws.sched);
    DL_TRY(tc_gemm(p2, true, st));
    return launch_residual_add_f32(ws.yf, ws.ldy32, x, m_out, T, m_out, 1, st);
  }
  GemmProblem p1 = one_seg(act, n_loc, T, n_loc, grp.B, grp.ldb, l, n_loc, out_plain(ws.zb, ws.ldzb, OUT_BF16, 0));
  p1.tail_acc = ws.tail;
  p1.tail_bytes = ws.tail_bytes;
  DL_TRY(tc_gemm(p1, false, st));
  DL_TRY(coll_all_reduce(comm, ws.zb, static_cast<size_t>(T) * ws.ldzb, kCollBF16, st));
  GemmProblem p2 = one_seg(ws.zb, ws.ldzb, T, l, grp.seg[0].A, grp.seg[0].lda, m_out, l, out_plain(x, m_out, OUT_BF16, 1));
  p2.tail_acc = ws.tail;
  p2.tail_bytes = ws.tail_bytes;
  return tc_gemm(p2, false, st);
}

// Low-rank KV cache decode attention (N3): latent of
// the new tokens -> pool; squeeze the runs; ONE fixed-size reconstruction GEMM
// over the buffer capacity; in-place RoPE; q projection; attention through the
// remapping index list.  Output: ws.att [T x Hq_loc*d].
dl_status kvlr_attention(const dl_block_config* cfg, const BlockDims& d, const dl_block_weights* w, const BlockWs& ws,
                         const dl_kv_lowrank* kv, int64_t T, const int32_t* positions, const int32_t* cache_lens,
                         bool tp, dl_comm comm, AttnArgs aa, RopeCacheArgs rc, cudaStream_t st) {
  const dl_factor_group& g = w->qkv;
  const ZLayout zl = zlayout(g, 3);
  // 1. latent z = xn . B^T of q|k|v (DeInfer: all-gathered)
  if (tp) {
    DL_TRY(deinfer_latent(g, 3, ws.xn, d.h, d.h, T, true, ws, d, comm, st));
  } else {
    GemmProblem p1 = stage1(g, 3, ws.xn, d.h, T, d.h, zl, out_plain(ws.zf, ws.ldz32, OUT_F32_RED, 0));
    p1.sched = next_sched(ws.sched);
    DL_TRY(tc_gemm(p1, true, st));
    DL_TRY(launch_f32_to_bf16(ws.zf, ws.ldz32, ws.zb, ws.ldzb, T, zl.width, 1, st));
  }
  const int64_t lk = g.seg[1].k, lv = g.seg[2].k, zv_off = zl.off[2] - zl.off[1];
  // 2. append [z_k | pad | z_v] of each new token to its pool slot
  DL_TRY(launch_kv_append(ws.zb, ws.ldzb, zl.off[1], zv_off + lv, static_cast<__nv_bfloat16*>(kv->pool), kv->ld_slot,
                          kv->slot_pos, kv->block_size, kv->block_tables, kv->max_blocks_per_seq, cache_lens,
                          positions, T, st));
  // 3. squeeze the contiguous runs into the compact buffer
  DL_TRY(launch_kv_squeeze(static_cast<const __nv_bfloat16*>(kv->pool), kv->slot_pos,
                           static_cast<__nv_bfloat16*>(kv->squeeze), kv->squeeze_pos, kv->ld_slot, kv->block_size,
                           kv->run_src, kv->run_dst, kv->run_len, kv->n_runs, kv->cap_blocks, st));
  // 4. reconstruction K | V = [z_k | z_v] . [A_k | A_v]^T at the buffer capacity
  const int64_t hkl = d.hkv / d.P, rows = kv->cap_blocks * kv->block_size;
  GemmProblem pr{};
  pr.act = kv->squeeze;
  pr.ld_act = kv->ld_slot;
  pr.T = rows;
  pr.k_act = kv->ld_slot;
  pr.nseg = 2;
  pr.seg[0] = GemmSeg{g.seg[1].A, g.seg[1].lda, hkl, lk, 0, 0};
  pr.seg[1] = GemmSeg{g.seg[2].A, g.seg[2].lda, hkl, lv, hkl, zv_off};
  pr.n_feat = 2 * hkl;
  pr.out = out_plain(kv->recon, 2 * hkl, OUT_BF16, 0);
  // 5. RoPE of the reconstructed keys with the stored positions ("in-place rotary
  //    position embedding ... to the reconstruction results"), applied in
  //    the reconstruction GEMM's epilogue; the separate in-place kernel is kept
  //    for key widths the vectorised epilogue does not cover
  static const bool sep_rope = DL_ENV("DL_RECON_ROPE_SEP") && atoi(DL_ENV("DL_RECON_ROPE_SEP")) != 0;   // A/B: RoPE as its own pass
  const bool epi_rope = !cfg->no_rope && hkl % 128 == 0 && !sep_rope;
  if (epi_rope) {
    pr.out.rope_pos = kv->squeeze_pos;
    pr.out.rope_end = hkl;
    pr.out.rope_theta = cfg->rope_theta;
  }
  DL_TRY(tc_gemm(pr, false, st));
  if (!cfg->no_rope && !epi_rope)
    DL_TRY(launch_rope_rows(static_cast<__nv_bfloat16*>(kv->recon), 2 * hkl, static_cast<int>(d.Hk_loc),
                            kv->squeeze_pos, rows, cfg->rope_theta, st));
  // 6. q = z_q . A_q^T (local heads) + RoPE
  const int64_t q_rows[1] = {d.h / d.P};
  GemmProblem pq = stage2(g, 1, q_rows, ws.zb, ws.ldzb, T, zl, out_plain(ws.yf, ws.ldy32, OUT_F32_RED, 0));
  pq.sched = next_sched(ws.sched);
  DL_TRY(tc_gemm(pq, true, st));
  rc.acc = ws.yf;
  rc.ld_src = ws.ldy32;
  rc.clear = 1;
  rc.Hk = 0;   // q only: keys come from the reconstruction buffer
  DL_TRY(launch_rope_cache(rc, st));
  // 7. attention over the buffer through the remapping index list
  const __nv_bfloat16* recon = static_cast<const __nv_bfloat16*>(kv->recon);
  aa.k_cache = recon;
  aa.v_cache = recon + hkl;
  aa.kv_ld = 2 * hkl;
  aa.kv_blk0 = kv->seq_block;
  aa.kv_bs = kv->block_size;
  aa.kv_rows = rows;
  return launch_attention(aa, st);
}

}  // namespace

dl_status dl_block_window_bytes(const dl_block_config* cfg, int world, size_t* bytes) {
  if (!bytes) {
    set_error("bytes is NULL");
    return DL_ERR_INVALID_ARG;
  }
  BlockDims d;
  DL_TRY(block_dims(cfg, world, &d));
  *bytes = d.layout == DL_LAYOUT_RANK_PARALLEL ? fan_window_bytes(d, std::max<int64_t>(cfg->max_tokens, 1)) : 0;
  return DL_OK;
}

dl_status dl_block_workspace(const dl_block_config* cfg, int world, size_t* bytes) {
  if (!bytes) {
    set_error("bytes is NULL");
    return DL_ERR_INVALID_ARG;
  }
  BlockDims d;
  DL_TRY(block_dims(cfg, world, &d));
  Carver c(nullptr);
  carve_block(c, d, std::max<int64_t>(cfg->max_tokens, 1));
  *bytes = c.off;
  return DL_OK;
}

namespace {
dl_status block_forward_impl(const dl_block_config* cfg, const dl_block_weights* w, void* x_, int64_t T,
                             const int32_t* positions, const int32_t* cu_seqlens, int32_t num_seqs, dl_phase phase,
                             void* k_cache, void* v_cache, const int32_t* cache_lens, int64_t max_seq, dl_comm comm,
                             void* workspace, size_t workspace_bytes, void* stream, const dl_kv_lowrank* kv,
                             const void* next_norm = nullptr, bool* next_normed = nullptr, bool prenormed = false) {
  // Stack chaining (dl_decomposed_stack_forward): with next_norm, a decode
  // block whose last step is the skinny residual add fuses it with the next
  // block's attention RMSNorm into ws.xn and sets *next_normed; with
  // prenormed, ws.xn already holds rmsnorm(x) * attn_norm.
  if (next_normed) *next_normed = false;
  const int P = comm ? comm->world : 1;
  BlockDims d;
  DL_TRY(block_dims(cfg, P, &d));
  if (!w) {
    set_error("weights NULL");
    return DL_ERR_INVALID_ARG;
  }
  if (T < 0 || T > cfg->max_tokens) {
    set_error("T=%lld outside [0, max_tokens=%lld]", (long long)T, (long long)cfg->max_tokens);
    return DL_ERR_SHAPE;
  }
  if (T == 0) return DL_OK;
  if (phase != DL_PREFILL && phase != DL_DECODE) {
    set_error("bad phase");
    return DL_ERR_INVALID_ARG;
  }
  if (num_seqs < 1 || num_seqs > cfg->max_seqs || (phase == DL_DECODE && num_seqs != T)) {
    set_error("num_seqs=%d invalid (max_seqs=%lld, decode requires num_seqs == T)", num_seqs,
              (long long)cfg->max_seqs);
    return DL_ERR_SHAPE;
  }
  if (!positions || !cache_lens || (phase == DL_PREFILL && !cu_seqlens) || max_seq < 1) {
    set_error("positions / cache_lens / cu_seqlens / max_seq missing");
    return DL_ERR_INVALID_ARG;
  }
  DL_TRY(check_ptr(x_, "x"));
  if (!kv) {
    DL_TRY(check_ptr(k_cache, "k_cache"));
    DL_TRY(check_ptr(v_cache, "v_cache"));
  }
  DL_TRY(check_ptr(w->attn_norm, "attn_norm"));
  DL_TRY(check_ptr(w->mlp_norm, "mlp_norm"));
  int64_t kq, ko, kg, kd;
  const int n_gu = d.glu ? 2 : 1;
  const bool deinfer = comm && d.layout == DL_LAYOUT_DEINFER;
  // DeInfer o / down hold the rank's input-column shard of B: [l x n/P]
  DL_TRY(check_group(w->qkv, 3, d.h, "qkv", &kq));
  DL_TRY(check_group(w->o, 1, deinfer ? d.h / P : d.h, "o", &ko));
  DL_TRY(check_group(w->gu, n_gu, d.h, d.glu ? "gate|up" : "up", &kg));
  DL_TRY(check_group(w->down, 1, deinfer ? d.m / P : d.m, "down", &kd));
  if (deinfer) {
    // segments carry the full ranks (the A shards keep every latent column)
    const int64_t want[7] = {cfg->rank_q, cfg->rank_k, cfg->rank_v, cfg->rank_o, cfg->rank_gate, cfg->rank_up,
                             cfg->rank_down};
    const int64_t have[7] = {w->qkv.seg[0].k, w->qkv.seg[1].k, w->qkv.seg[2].k, w->o.seg[0].k,
                             d.glu ? w->gu.seg[0].k : 0, w->gu.seg[d.glu ? 1 : 0].k, w->down.seg[0].k};
    for (int i = 0; i < 7; ++i)
      if (want[i] != have[i]) {
        set_error("DeInfer layout: segment %d rank %lld != config rank %lld", i, (long long)have[i],
                  (long long)want[i]);
        return DL_ERR_RANK;
      }
  } else if (kq > d.k_qkv || ko > d.k_o || kg > d.k_gu || kd > d.k_down) {
    set_error("group shard larger than the balanced split allows");
    return DL_ERR_PARTITION;
  }
  size_t need = 0;
  dl_block_workspace(cfg, P, &need);
  if (!workspace || workspace_bytes < need) {
    set_error("workspace %zu B < required %zu B", workspace_bytes, need);
    return DL_ERR_WORKSPACE;
  }
  DL_TRY(check_device());

  cudaStream_t st = static_cast<cudaStream_t>(stream);
  __nv_bfloat16* x = static_cast<__nv_bfloat16*>(x_);
  Carver cv(workspace);
  const BlockWs ws = carve_block(cv, d, cfg->max_tokens);
  const bool skinny = T <= 256;
  // Any real communicator (NCCL or group, world >= 1) selects the
  // tensor-parallel branch (bf16 partials, RS / AG / AR); at world 1 its
  // collectives are identities.  A loopback communicator of world 1 is TP = 1.
  const bool tp = comm && (P > 1 || comm->kind != kCommLoopback);
  if (kv) {
    if (phase != DL_DECODE || !skinny) {
      set_error("low-rank KV cache: decode only (T <= 256)");
      return DL_ERR_INVALID_ARG;
    }
    if (tp && d.layout != DL_LAYOUT_DEINFER) {
      set_error("low-rank KV cache needs the full latent: TP = 1 or DL_LAYOUT_DEINFER");
      return DL_ERR_UNSUPPORTED;
    }
    const int64_t zv_need = rup(w->qkv.seg[1].k, 64) + w->qkv.seg[2].k;
    if (!kv->pool || !kv->slot_pos || !kv->block_tables || !kv->run_src || !kv->run_dst || !kv->run_len ||
        !kv->n_runs || !kv->seq_block || !kv->squeeze || !kv->squeeze_pos || !kv->recon || kv->block_size < 1 ||
        kv->cap_blocks < 1 || kv->max_blocks_per_seq < 1 || kv->ld_slot % 8 || kv->ld_slot < zv_need ||
        (kv->block_size * kv->ld_slot) % 8) {
      set_error("dl_kv_lowrank: missing buffer or bad sizes (ld_slot >= rup(l_k, 64) + l_v, multiple of 8)");
      return DL_ERR_INVALID_ARG;
    }
  }
  const int64_t qkv_rows[3] = {d.h, d.hkv, d.hkv};
  const int64_t gu_rows[2] = {d.m, d.m};
  const int64_t h_rows[1] = {d.h};
  const int64_t NQKV = d.h + 2 * d.hkv;
  const int red_mode = skinny ? OUT_F32_RED : OUT_BF16;
  // skinny TP: stage-2 partials red.add-ed as bf16x2 straight into the
  // collective's buffer ws.yr (no fp32 -> bf16 pass before each collective);
  // the kernel that consumes the collective's result clears it
  const bool tpr = tp && skinny && use_zred();
  // Fused collectives: with a group communicator the skinny
  // rank-parallel path red.adds its stage-2 partials straight into the ranks'
  // symmetric windows (all-reduce: every rank's copy; reduce-scatter: the
  // owner's) and pushes the attention output into every rank's all-gather slot,
  // so each collective is a barrier, not a pass over the data.
  FanBufs fan;
  if (tpr && d.layout == DL_LAYOUT_RANK_PARALLEL &&
      comm_window_bytes(comm) >= fan_window_bytes(d, cfg->max_tokens)) {
    fan.on = true;
    Carver fc(comm_window(comm, comm->rank));
    const int64_t Ts = std::min<int64_t>(cfg->max_tokens, 256);
    fan.X = fc.take<__nv_bfloat16>(static_cast<size_t>(Ts) * std::max<int64_t>(d.W, n_gu * d.m));
    fan.Y = fc.take<__nv_bfloat16>(static_cast<size_t>(Ts) * d.h);
    fan.G = fc.take<__nv_bfloat16>(static_cast<size_t>(Ts) * d.h);
    for (int j = 0; j < P; ++j) fan.delta[j] = (comm_window(comm, j) - comm_window(comm, comm->rank)) / 2;
  }
  // Two-shot all-reduce fused into the epilogue: the columns of an all-reduced
  // output are split into P slabs; the stage-2 epilogue red.adds each partial
  // into the slab owner's copy only (reduce-scatter, the transfer overlapping
  // the GEMM), then each owner pushes its finished slab into the others' copies.
  // Per rank (P-1)/P of the output is sent twice, as in a ring / two-shot
  // all-reduce (a one-shot fan-out into all P copies would send P-1 times it).
  auto ar_slab = [&](int64_t n) { return rup((n + P - 1) / P, 8); };
  auto fan_ar = [&](GemmOut o, int64_t n) {
    if (fan.on) {
      o.fan_n = P;
      o.fan_cols = ar_slab(n);
      for (int j = 0; j < P; ++j) o.fan_delta[j] = fan.delta[j];
    }
    return o;
  };
  auto fan_all = [&](GemmOut o) {   // reduce-scatter by owner (scatter layout)
    if (fan.on) {
      o.fan_n = P;
      for (int j = 0; j < P; ++j) o.fan_delta[j] = fan.delta[j];
    }
    return o;
  };
  // the bf16 all-reduce target of the skinny TP path: Y / X of the window, else ws.yr
  // (o / down outputs in their own buffer: the down stage 1 may still read the
  // gate|up rows in ws.yr while the down stage 2 reduces, DL_XACT_TP)
  __nv_bfloat16* const arY = fan.on ? fan.Y : ws.yr2;
  __nv_bfloat16* const arX = fan.on ? fan.X : ws.yr;
  auto all_reduce_bf16 = [&](__nv_bfloat16* buf, int64_t n) -> dl_status {
    if (!fan.on) return coll_all_reduce(comm, buf, static_cast<size_t>(T) * n, kCollBF16, st);
    DL_TRY(comm_barrier(comm, st));               // every slab holds the sum of all partials
    const int64_t sl = ar_slab(n), c0 = std::min<int64_t>(n, comm->rank * sl), c1 = std::min<int64_t>(n, c0 + sl);
    DL_TRY(launch_fan_push(buf, n, T, c0, c1, fan.delta, P, comm->rank, st));
    return comm_barrier(comm, st);                // every copy holds every slab
  };

  // ---- q|k|v: one group; partials laid out rank-major by head for the RS ----
  GemmOut qkv_out{};
  qkv_out.mode = red_mode;
  qkv_out.scatter_p = tp ? P : 0;   // TP: rank-major [P][T][W] slabs, also at P = 1
  qkv_out.slab = d.W;
  qkv_out.seg_slab_off[0] = 0;
  qkv_out.seg_slab_off[1] = d.h / P;
  qkv_out.seg_slab_off[2] = d.h / P + d.hkv / P;
  qkv_out.seg_rpr[0] = d.h / P;
  qkv_out.seg_rpr[1] = d.hkv / P;
  qkv_out.seg_rpr[2] = d.hkv / P;
  qkv_out.ptr = skinny ? static_cast<void*>(ws.yf) : static_cast<void*>(ws.yb);
  qkv_out.ld = skinny ? ws.ldy32 : NQKV;
  if (tpr) {
    qkv_out.mode = OUT_BF16_RED;
    qkv_out.ptr = ws.yr;
    qkv_out.ld = NQKV;
    if (fan.on) {   // reduce-scatter by owner: [T][W] in the owner's window
      qkv_out.ptr = fan.X;
      qkv_out = fan_all(qkv_out);
    }
  }
  // Opt-in (DL_ROPE_FUSE=1): TP = 1 decode with the q|k|v partials as bf16x2
  // in ws.yr and RoPE + cache append done by the stream-K attention kernel
  // itself; the o group's residual + MLP-norm kernel clears ws.yr's q|k|v rows.
  // Measured 0.2-0.3 ms/step slower: without the small RoPE kernel between
  // them, the attention CTAs only become resident once the q|k|v stage-2
  // GEMM's CTAs (216 KB of shared memory each) exit, so the old-key tiles are
  // no longer streamed while the predecessor drains.
  static const bool no_rope_fuse = !(DL_ENV("DL_ROPE_FUSE") && atoi(DL_ENV("DL_ROPE_FUSE")) != 0);
  static const bool no_fuse_rn = DL_ENV("DL_NO_FUSE_RESNORM") != nullptr;
  const bool rope_attn = skinny && !tp && !kv && use_zred() && !use_fixup() && !no_rope_fuse && !no_fuse_rn &&
                         phase == DL_DECODE && num_seqs <= 1024 && d.d == 128;
  // TP decode (skinny rank-parallel / DeInfer-free path): the attention reads the
  // reduce-scattered q|k|v rows of the rank's heads and does RoPE + cache
  // append itself -- one launch (and one dependent boundary) less per layer
  // (DL_ROPE_FUSE_TP=0: separate RoPE kernel)
  static const bool rope_fuse_tp = !DL_ENV("DL_ROPE_FUSE_TP") || atoi(DL_ENV("DL_ROPE_FUSE_TP")) != 0;
  const bool rope_attn_tp = tpr && !kv && rope_fuse_tp && phase == DL_DECODE && num_seqs <= 1024 && d.d == 128 &&
                            d.layout == DL_LAYOUT_RANK_PARALLEL && d.W % 8 == 0;
  if (rope_attn) {
    qkv_out.mode = OUT_BF16_RED;
    qkv_out.ptr = ws.yr;
    qkv_out.ld = NQKV;
  }
  // prefill, TP = 1: RoPE of q and k in the q|k|v stage-2 epilogue (whole tiles
  // and the K-split tail finalize, one bf16 rounding); the attention reads q in
  // place from the q|k|v output and a copy-only kernel appends k, v to the
  // caches (DL_ROPE_EPI=0: the RoPE + cache-append kernel, A/B)
  static const bool rope_epi_env = !DL_ENV("DL_ROPE_EPI") || atoi(DL_ENV("DL_ROPE_EPI")) != 0;
  const bool rope_epi = rope_epi_env && phase == DL_PREFILL && !skinny && !tp && !kv && d.d == 128 && NQKV % 8 == 0;
  if (rope_epi && !cfg->no_rope) {
    qkv_out.rope_pos = positions;
    qkv_out.rope_end = (d.Hq_loc + d.Hk_loc) * d.d;
    qkv_out.rope_theta = cfg->rope_theta;
  }

  // skinny, single rank: every group's finalize (RoPE + cache append, residual,
  // SiLU*up) runs in the stage-2 GEMM's last-contributor fixup
  const bool fx = skinny && !tp && use_fixup();
  auto fixup = [&](int op) {
    GemmFixup f{};
    f.op = op;
    f.acc32 = ws.yf;
    f.acc_ld = ws.ldy32;
    f.tile_cnt = ws.tile_cnt;
    f.resid = x;
    f.ld_resid = d.h;
    f.act_out = ws.act;
    f.ld_act_out = d.m;
    return f;
  };

  RopeCacheArgs rc{};
  rc.q_out = ws.q;
  rc.k_cache = static_cast<__nv_bfloat16*>(k_cache);
  rc.v_cache = static_cast<__nv_bfloat16*>(v_cache);
  rc.max_seq = max_seq;
  rc.positions = positions;
  rc.cu_seqlens = cu_seqlens;
  rc.cache_lens = cache_lens;
  rc.num_seqs = num_seqs;
  rc.decode = phase == DL_DECODE;
  rc.T = T;
  rc.Hq = static_cast<int>(d.Hq_loc);
  rc.Hk = static_cast<int>(d.Hk_loc);
  rc.d = static_cast<int>(d.d);
  rc.theta = cfg->rope_theta;
  rc.rope = cfg->no_rope ? 0 : 1;

  AttnArgs aa{};
  aa.q = ws.q;
  aa.out = ws.att;
  aa.k_cache = rc.k_cache;
  aa.v_cache = rc.v_cache;
  aa.max_seq = max_seq;
  aa.cu_seqlens = cu_seqlens;
  aa.cache_lens = cache_lens;
  aa.num_seqs = num_seqs;
  aa.T = T;
  aa.Hq = static_cast<int>(d.Hq_loc);
  aa.Hk = static_cast<int>(d.Hk_loc);
  aa.d = static_cast<int>(d.d);
  aa.decode = phase == DL_DECODE;
  aa.partial = ws.apart;
  aa.partial_bytes = ws.apart_bytes;
  aa.sk_ws = ws.ask;
  aa.sk_items_cap = ws.ask_items;

  if (tp && d.layout == DL_LAYOUT_DEINFER) {
    // ---- DeInfer low-rank communication (Fig. 3) ----------
    const int64_t qkv_loc[3] = {d.h / P, d.hkv / P, d.hkv / P};
    const int64_t m_loc = d.m / P, ngu_loc = n_gu * m_loc;
    const int64_t gu_loc[2] = {m_loc, m_loc};
    DL_TRY(launch_rmsnorm(x, static_cast<const __nv_bfloat16*>(w->attn_norm), ws.xn, T, d.h, cfg->rms_eps, st));
    if (kv) {
      DL_TRY(kvlr_attention(cfg, d, w, ws, kv, T, positions, cache_lens, true, comm, aa, rc, st));
    } else {
      const GemmOut qo = skinny ? out_plain(ws.yf, ws.ldy32, OUT_F32_RED, 0) : out_plain(ws.yb, d.W, OUT_BF16, 0);
      DL_TRY(deinfer_first(w->qkv, 3, qkv_loc, ws.xn, d.h, d.h, T, skinny, ws, d, comm, qo, st));
      if (skinny) {
        rc.acc = ws.yf;
        rc.ld_src = ws.ldy32;
        rc.clear = 1;
      } else {
        rc.src = ws.yb;
        rc.ld_src = d.W;
      }
      DL_TRY(launch_rope_cache(rc, st));
      DL_TRY(launch_attention(aa, st));
    }
    DL_TRY(deinfer_second(w->o, ws.att, d.h / P, d.h, T, skinny, ws, comm, x, st));
    DL_TRY(launch_rmsnorm(x, static_cast<const __nv_bfloat16*>(w->mlp_norm), ws.xn, T, d.h, cfg->rms_eps, st));
    const GemmOut go = skinny ? out_plain(ws.yf, ws.ldy32, OUT_F32_RED, 0) : out_plain(ws.yb, ngu_loc, OUT_BF16, 0);
    DL_TRY(deinfer_first(w->gu, n_gu, gu_loc, ws.xn, d.h, d.h, T, skinny, ws, d, comm, go, st));
    if (skinny) {
      if (d.glu) DL_TRY(launch_silu_mul_f32(ws.yf, ws.ldy32, ws.act, m_loc, T, m_loc, 1, st));
      else DL_TRY(launch_relu_f32(ws.yf, ws.ldy32, ws.act, m_loc, T, m_loc, 1, st));
    } else {
      if (d.glu) DL_TRY(launch_silu_mul_bf16(ws.yb, ngu_loc, ws.act, m_loc, T, m_loc, st));
      else DL_TRY(launch_relu_bf16(ws.yb, ngu_loc, ws.act, m_loc, T, m_loc, st));
    }
    return deinfer_second(w->down, ws.act, m_loc, d.h, T, skinny, ws, comm, x, st);
  }

  if (!prenormed)
    DL_TRY(launch_rmsnorm(x, static_cast<const __nv_bfloat16*>(w->attn_norm), ws.xn, T, d.h, cfg->rms_eps, st));
  SideZero zq;
  static const bool fix_rope = DL_ENV("DL_FIXUP_ROPE") && atoi(DL_ENV("DL_FIXUP_ROPE")) != 0;   // A/B switch
  const bool fx_rope = !fx && !kv && !tp && skinny && fix_rope && !rope_attn && phase == DL_DECODE && num_seqs <= 1024;
  if (kv) {
    DL_TRY(kvlr_attention(cfg, d, w, ws, kv, T, positions, cache_lens, false, comm, aa, rc, st));
  } else if (fx) {
    GemmFixup f = fixup(FIX_ROPE_CACHE);
    f.rope = rc;
    DL_TRY(run_group(w->qkv, 3, qkv_rows, ws.xn, d.h, d.h, T, skinny, ws, qkv_out, st, &f));
  } else if (fx_rope) {
    // RoPE + cache append by the q|k|v stage-2 last-contributor fixup alone
    // (DL_FIXUP_ROPE=1); the latent clear moves to the attention kernel
    GemmFixup f = fixup(FIX_ROPE_CACHE);
    f.rope = rc;
    DL_TRY(run_group(w->qkv, 3, qkv_rows, ws.xn, d.h, d.h, T, skinny, ws, qkv_out, st, &f, &zq));
  } else {
    DL_TRY(run_group(w->qkv, 3, qkv_rows, ws.xn, d.h, d.h, T, skinny, ws, qkv_out, st, nullptr, &zq));
  }

  if (fx || kv) {
    // RoPE + cache append done by the q|k|v stage-2 fixup / low-rank KV path
  } else if (!tp) {
    if (skinny) {
      rc.acc = ws.yf;
      rc.ld_src = ws.ldy32;
      rc.clear = 1;
      rc.zero = zq;
    } else {
      rc.src = ws.yb;
      rc.ld_src = NQKV;
      if (rope_epi) {
        rc.kv_only = 1;
        rc.rope = 0;
        aa.q = ws.yb;
        aa.ld_q = NQKV;
      }
    }
  } else if (fan.on) {
    DL_TRY(comm_barrier(comm, st));   // every rank's q|k|v partials are in the owners' windows
    rc.src = fan.X;
    rc.ld_src = d.W;
    rc.zero = zq;
  } else if (tpr) {
    DL_TRY(coll_reduce_scatter(comm, ws.yr, ws.rs, static_cast<size_t>(T) * d.W, kCollBF16, st));
    rc.src = ws.rs;
    rc.ld_src = d.W;
    rc.zero = zq;
    rc.zero2.p = ws.yr;                         // contiguous [P][T][W] partials
    rc.zero2.rows = 1;
    rc.zero2.row_bytes = rc.zero2.ld = static_cast<int64_t>(T) * NQKV * 2;
  } else {
    if (skinny) DL_TRY(launch_f32_to_bf16(ws.yf, NQKV, ws.yb, NQKV, 1, T * NQKV, 1, st, zq));   // contiguous [P][T][W]
    DL_TRY(coll_reduce_scatter(comm, ws.yb, ws.rs, static_cast<size_t>(T) * d.W, kCollBF16, st));
    rc.src = ws.rs;
    rc.ld_src = d.W;
  }
  if (rope_attn) {
    aa.qkv = ws.yr;
    aa.ld_qkv = NQKV;
    aa.positions = positions;
    aa.theta = cfg->rope_theta;
    aa.rope = cfg->no_rope ? 0 : 1;
    aa.zero = zq;
    DL_TRY(launch_attention(aa, st));
  } else if (rope_attn_tp) {
    aa.qkv = rc.src;   // [T x W] rows of the rank's q | k | v heads
    aa.ld_qkv = rc.ld_src;
    aa.positions = positions;
    aa.theta = cfg->rope_theta;
    aa.rope = cfg->no_rope ? 0 : 1;
    aa.zero = rc.zero;
    aa.zero2 = rc.zero2;
    DL_TRY(launch_attention(aa, st));
  } else {
    if (fx_rope) aa.zero = zq;
    if (!fx && !kv && !fx_rope) DL_TRY(launch_rope_cache(rc, st));
    if (!kv) DL_TRY(launch_attention(aa, st));
  }

  const __nv_bfloat16* att_in = ws.att;
  int o_act_p = 0;
  int64_t o_act_w = 0;
  static const bool no_ag3d = DL_ENV("DL_NO_AG3D") != nullptr;   // A/B switch
  if (tp) {
    const int64_t wl = d.Hq_loc * d.d;
    const __nv_bfloat16* ag = ws.ag;
    if (fan.on) {
      // all-gather by push into every rank's slot [rank][T][wl]; the reduce-
      // scatter buffer X (consumed by RoPE) is cleared on the side
      SideZero zx;
      zx.p = fan.X;
      zx.rows = 1;
      zx.row_bytes = zx.ld = static_cast<int64_t>(T) * d.W * 2;
      DL_TRY(launch_fan_copy(ws.att, wl, fan.G + static_cast<int64_t>(comm->rank) * T * wl, fan.delta, P, T, wl, st,
                             zx));
      DL_TRY(comm_barrier(comm, st));
      ag = fan.G;
    } else {
      DL_TRY(coll_all_gather(comm, ws.att, ws.ag, static_cast<size_t>(T) * wl, kCollBF16, st));
    }
    if (skinny && !no_ag3d && wl % 64 == 0) {
      // o's stage-1 TMA reads the rank-major [P][T][wl] all-gather output directly
      att_in = ag;
      o_act_p = P;
      o_act_w = wl;
    } else {
      DL_TRY(launch_unpermute(ag, ws.att_full, P, T, wl, st));
      att_in = ws.att_full;
    }
  }

  // Finish a [T x n] group output: + residual (o, down) with the TP reduction.
  auto finish_residual = [&](int64_t n, const SideZero& z, const SideZero& z2 = SideZero{}) -> dl_status {
    if (!tp) return skinny ? launch_residual_add_f32(ws.yf, ws.ldy32, x, d.h, T, n, 1, st, z, z2) : DL_OK;
    if (tpr) {
      DL_TRY(all_reduce_bf16(arY, n));
      return launch_residual_add_bf16(arY, n, x, d.h, T, n, st, 1, z, z2);
    }
    if (skinny) DL_TRY(launch_f32_to_bf16(ws.yf, ws.ldy32, ws.yb, n, T, n, 1, st, z));
    DL_TRY(coll_all_reduce(comm, ws.yb, static_cast<size_t>(T) * n, kCollBF16, st));
    return launch_residual_add_bf16(ws.yb, n, x, d.h, T, n, st);
  };
  // wide & TP=1: the stage-2 epilogue adds straight into x (fused residual)
  auto resid_out = [&]() -> GemmOut {
    if (tpr) return fan_ar(out_plain(arY, d.h, OUT_BF16_RED, 0), d.h);
    if (skinny) return out_plain(ws.yf, ws.ldy32, OUT_F32_RED, 0);
    if (!tp) return out_plain(x, d.h, OUT_BF16, 1);
    return out_plain(ws.yb, d.h, OUT_BF16, 0);
  };

  // ---- o projection + residual ----------------------------------------------
  const GemmFixup fres = fixup(fx ? FIX_RESIDUAL : FIX_NONE);
  SideZero zo, zg, zd;
  DL_TRY(run_group(w->o, 1, h_rows, att_in, d.h, d.h, T, skinny, ws, resid_out(), st, &fres, fx ? nullptr : &zo, 0,
                   o_act_p, o_act_w));
  const __nv_bfloat16* mlp_norm = static_cast<const __nv_bfloat16*>(w->mlp_norm);
  static const bool no_fuse = DL_ENV("DL_NO_FUSE_RESNORM") != nullptr;   // A/B timing switch
  if (!fx && !tp && skinny && !no_fuse) {
    // residual add of the o projection fused with the MLP pre-norm
    SideZero zqkv;
    if (rope_attn) {
      zqkv.p = ws.yr;
      zqkv.rows = 1;
      zqkv.row_bytes = zqkv.ld = static_cast<int64_t>(T) * NQKV * 2;
    }
    DL_TRY(launch_residual_rmsnorm(ws.yf, ws.ldy32, x, mlp_norm, ws.xn, T, d.h, cfg->rms_eps, st, zo, zqkv));
  } else if (tpr && !no_fuse) {
    // TP: all-reduce of the bf16 partials, then residual + MLP pre-norm in one pass
    DL_TRY(all_reduce_bf16(arY, d.h));
    DL_TRY(launch_residual_rmsnorm_bf16(arY, d.h, x, mlp_norm, ws.xn, T, d.h, cfg->rms_eps, st, zo));
  } else {
    if (!fx) DL_TRY(finish_residual(d.h, zo));
    DL_TRY(launch_rmsnorm(x, mlp_norm, ws.xn, T, d.h, cfg->rms_eps, st));
  }

  // ---- MLP: gate|up group, SiLU(gate)*up (or ReLU(up)), down + residual ---------
  const int64_t ngu = n_gu * d.m;
  // SiLU(gate)*up by the gate|up stage-2 last-contributor fixup: with all
  // fixups (DL_FIXUP) or alone (DL_FIXUP_SILU; the latent stays in Z slot 1
  // until the down group's finalize clears it)
  static const bool fix_silu = DL_ENV("DL_FIXUP_SILU") && atoi(DL_ENV("DL_FIXUP_SILU")) != 0;
  const bool fx_gu = (fx || (fix_silu && skinny && !tp)) && d.glu;
  GemmOut gu_out = skinny ? out_plain(ws.yf, ws.ldy32, OUT_F32_RED, 0) : out_plain(ws.yb, ngu, OUT_BF16, 0);
  // skinny TP = 1: gate|up partials as bf16x2 reductions too (the SiLU input is
  // bf16-rounded anyway); halves the reduction and finalize traffic (DL_GU_F32 A/B)
  static const bool gu_f32 = DL_ENV("DL_GU_F32") != nullptr;
  const bool gur = skinny && !tp && use_zred() && !fx_gu && !gu_f32;
  // the MLP activation inside the down projection's stage 1 instead of the SiLU kernel
  // (DL_XACT=1, A/B): measured 29.7 vs 26.2 ms/step -- every one of the 39 feature tiles
  // of the down stage 1 recomputes the activation of its k-range (71.6 M SiLUs per layer
  // for 1.8 M outputs), DESIGN.md §6
  static const bool xact_env = DL_ENV("DL_XACT") && atoi(DL_ENV("DL_XACT")) != 0;
  const bool xact = gur && xact_env && d.m % 8 == 0 && ngu % 8 == 0;
  // TP (DL_XACT_TP=1, A/B): the activation in the down stage 1 is recomputed
  // by only the rank's k-shard feature tiles (5 x at TP = 8 for 70B, 39 x at
  // TP = 1) and removes the SiLU kernel and its boundary, but each stage-1 unit
  // then waits on an L2 round trip for its gate|up tile: measured 9.9 vs 8.8 ms
  // per rank at TP = 8 (down stage 1 29 vs 16 us), DESIGN.md §6
  static const bool xact_tp_env = DL_ENV("DL_XACT_TP") && atoi(DL_ENV("DL_XACT_TP")) != 0;
  const bool xact_tp = tpr && !fan.on && xact_tp_env && P > 1 && d.layout == DL_LAYOUT_RANK_PARALLEL &&
                       d.m % 8 == 0 && ngu % 8 == 0;
  if (tpr || gur) gu_out = fan_ar(out_plain(arX, ngu, OUT_BF16_RED, 0), ngu);
  // prefill (whole-tile pair GEMM), TP = 1: SiLU(gate)*up in the gate|up stage-2
  // epilogue (GemmProblem::glu): the [T x 2m] gate|up output never reaches HBM
  // and the SiLU.up kernel is gone (DL_GLU_FUSE=0: separate kernel, A/B)
  static const bool glu_env = !DL_ENV("DL_GLU_FUSE") || atoi(DL_ENV("DL_GLU_FUSE")) != 0;
  const bool glu_fuse = glu_env && !skinny && !tp && d.glu && !fx_gu && n_gu == 2 && d.m % 256 == 0 &&
                        w->gu.seg[0].k == w->gu.seg[1].k && w->gu.seg[0].k > 0;
  if (glu_fuse) gu_out = out_plain(ws.act, d.m, OUT_BF16, 0);
  const GemmFixup fsilu = fixup(fx_gu ? FIX_SILU : FIX_NONE);
  DL_TRY(run_group(w->gu, n_gu, gu_rows, ws.xn, d.h, d.h, T, skinny, ws, gu_out, st, &fsilu, fx ? nullptr : &zg, 1,
                   0, 0, Xform{}, glu_fuse ? 1 : 0));
  if (glu_fuse) {
    // SiLU(gate)*up written by the gate|up stage-2 epilogue
  } else if (fx_gu) {
    // SiLU(gate)*up done by the gate|up stage-2 fixup
  } else if (!tp && gur && xact) {
    // SiLU(gate)*up / ReLU(up) computed by the down projection's stage 1 itself
    // (in-kernel activation); its gate|up source and latent are cleared below
  } else if (!tp && gur) {
    if (d.glu) DL_TRY(launch_silu_mul_bf16(ws.yr, ngu, ws.act, d.m, T, d.m, st, 1, zg));
    else DL_TRY(launch_relu_bf16(ws.yr, ngu, ws.act, d.m, T, d.m, st, 1, zg));
  } else if (!tp && skinny) {
    if (d.glu) DL_TRY(launch_silu_mul_f32(ws.yf, ws.ldy32, ws.act, d.m, T, d.m, 1, st, zg));
    else DL_TRY(launch_relu_f32(ws.yf, ws.ldy32, ws.act, d.m, T, d.m, 1, st, zg));
  } else if (tpr && xact_tp) {
    DL_TRY(all_reduce_bf16(arX, ngu));   // the down stage 1 reads (and a later kernel clears) it
  } else if (tpr) {
    DL_TRY(all_reduce_bf16(arX, ngu));
    if (d.glu) DL_TRY(launch_silu_mul_bf16(arX, ngu, ws.act, d.m, T, d.m, st, 1, zg));
    else DL_TRY(launch_relu_bf16(arX, ngu, ws.act, d.m, T, d.m, st, 1, zg));
  } else {
    if (skinny) DL_TRY(launch_f32_to_bf16(ws.yf, ws.ldy32, ws.yb, ngu, T, ngu, 1, st, zg));
    if (tp) DL_TRY(coll_all_reduce(comm, ws.yb, static_cast<size_t>(T) * ngu, kCollBF16, st));
    if (d.glu) DL_TRY(launch_silu_mul_bf16(ws.yb, ngu, ws.act, d.m, T, d.m, st));
    else DL_TRY(launch_relu_bf16(ws.yb, ngu, ws.act, d.m, T, d.m, st));
  }
  Xform xf;
  SideZero zyr;   // in-kernel activation: the gate|up rows, cleared once the down stage 1 has read them
  if ((!tp && gur && xact) || xact_tp) {
    xf.mode = d.glu ? XFORM_SILU : XFORM_RELU;
    xf.src = ws.yr;
    xf.ld = ngu;
    xf.m = d.m;
    zyr.p = ws.yr;
    zyr.rows = 1;
    zyr.row_bytes = zyr.ld = static_cast<int64_t>(T) * ngu * 2;
  }
  DL_TRY(run_group(w->down, 1, h_rows, ws.act, d.m, d.m, T, skinny, ws, resid_out(), st, &fres, fx ? nullptr : &zd, 0,
                   0, 0, xf));
  if ((fx_gu || xf.mode) && zg.p && zd.p) zd.row_bytes = ws.ldzb * 2 + zg.row_bytes;   // slot 0 + the gate|up latent in slot 1
  if (next_norm && !fx && !tp && skinny && !no_fuse) {
    // residual add of the down projection fused with the next block's pre-norm
    DL_TRY(launch_residual_rmsnorm(ws.yf, ws.ldy32, x, static_cast<const __nv_bfloat16*>(next_norm), ws.xn, T, d.h,
                                   cfg->rms_eps, st, zd, zyr));
    *next_normed = true;
    return DL_OK;
  }
  if (next_norm && tpr && !no_fuse && d.layout != DL_LAYOUT_DEINFER) {
    DL_TRY(all_reduce_bf16(arY, d.h));
    DL_TRY(launch_residual_rmsnorm_bf16(arY, d.h, x, static_cast<const __nv_bfloat16*>(next_norm), ws.xn, T, d.h,
                                        cfg->rms_eps, st, zd, zyr));
    *next_normed = true;
    return DL_OK;
  }
  if (!fx) DL_TRY(finish_residual(d.h, zd, zyr));
  return DL_OK;
}
}  // namespace

dl_status dl_decomposed_stack_forward(const dl_block_config* cfg, const dl_block_weights* const* w, int32_t n_layers,
                                      void* x, int64_t T, const int32_t* positions, const int32_t* cu_seqlens,
                                      int32_t num_seqs, dl_phase phase, void* const* k_caches, void* const* v_caches,
                                      const int32_t* cache_lens, int64_t max_seq, dl_comm comm, void* workspace,
                                      size_t workspace_bytes, void* stream) {
  if (!w || n_layers < 0 || (n_layers > 0 && (!k_caches || !v_caches))) {
    set_error("stack: weights / caches missing");
    return DL_ERR_INVALID_ARG;
  }
  bool normed = false;
  for (int32_t l = 0; l < n_layers; ++l) {
    if (!w[l]) {
      set_error("stack: layer %d weights NULL", l);
      return DL_ERR_INVALID_ARG;
    }
    const void* nn = l + 1 < n_layers ? w[l + 1]->attn_norm : nullptr;
    bool out_normed = false;
    DL_TRY(block_forward_impl(cfg, w[l], x, T, positions, cu_seqlens, num_seqs, phase, k_caches[l], v_caches[l],
                              cache_lens, max_seq, comm, workspace, workspace_bytes, stream, nullptr, nn, &out_normed,
                              normed));
    normed = out_normed;
  }
  return DL_OK;
}

dl_status dl_decomposed_block_forward(const dl_block_config* cfg, const dl_block_weights* w, void* x_, int64_t T,
                                      const int32_t* positions, const int32_t* cu_seqlens, int32_t num_seqs,
                                      dl_phase phase, void* k_cache, void* v_cache, const int32_t* cache_lens,
                                      int64_t max_seq, dl_comm comm, void* workspace, size_t workspace_bytes,
                                      void* stream) {
  return block_forward_impl(cfg, w, x_, T, positions, cu_seqlens, num_seqs, phase, k_cache, v_cache, cache_lens,
                            max_seq, comm, workspace, workspace_bytes, stream, nullptr);
}

dl_status dl_decomposed_block_forward_kvlr(const dl_block_config* cfg, const dl_block_weights* w, void* x, int64_t T,
                                           const int32_t* positions, const dl_kv_lowrank* kv,
                                           const int32_t* cache_lens, dl_comm comm, void* workspace,
                                           size_t workspace_bytes, void* stream) {
  if (!kv) {
    set_error("kv is NULL");
    return DL_ERR_INVALID_ARG;
  }
  return block_forward_impl(cfg, w, x, T, positions, nullptr, static_cast<int32_t>(T), DL_DECODE, nullptr, nullptr,
                            cache_lens, 1, comm, workspace, workspace_bytes, stream, kv);
}

dl_status dl_kv_prepare(const int32_t* block_tables, int64_t max_blocks_per_seq, const int32_t* seq_tokens,
                        int32_t num_seqs, int64_t block_size, int64_t max_runs, int64_t cap_blocks, int32_t* run_src,
                        int32_t* run_dst, int32_t* run_len, int32_t* n_runs, int32_t* seq_block) {
  if (!block_tables || !seq_tokens || !run_src || !run_dst || !run_len || !n_runs || !seq_block || num_seqs < 0 ||
      block_size < 1 || max_blocks_per_seq < 1) {
    set_error("dl_kv_prepare: bad arguments");
    return DL_ERR_SHAPE;
  }
  int64_t nr = 0, dst = 0;
  for (int32_t s = 0; s < num_seqs; ++s) {
    const int64_t nblk = (static_cast<int64_t>(seq_tokens[s]) + block_size - 1) / block_size;
    if (seq_tokens[s] < 0 || nblk > max_blocks_per_seq) {
      set_error("dl_kv_prepare: sequence %d has %d tokens (max %lld blocks)", s, seq_tokens[s],
                (long long)max_blocks_per_seq);
      return DL_ERR_SHAPE;
    }
    seq_block[s] = static_cast<int32_t>(dst);     // remapping index list: consecutive buffer blocks
    const int32_t* row = block_tables + static_cast<int64_t>(s) * max_blocks_per_seq;
    for (int64_t i = 0; i < nblk; ++i) {
      if (row[i] < 0) {
        set_error("dl_kv_prepare: negative block id");
        return DL_ERR_SHAPE;
      }
      if (i == 0 || row[i] != row[i - 1] + 1) {    // a new physically contiguous run
        if (nr == max_runs) {
          set_error("dl_kv_prepare: more than max_runs = %lld runs", (long long)max_runs);
          return DL_ERR_WORKSPACE;
        }
        run_src[nr] = row[i];
        run_dst[nr] = static_cast<int32_t>(dst + i);
        run_len[nr] = 0;
        ++nr;
      }
      run_len[nr - 1] += 1;
    }
    dst += nblk;
  }
  if (dst > cap_blocks) {
    set_error("dl_kv_prepare: %lld blocks exceed the buffer capacity %lld", (long long)dst, (long long)cap_blocks);
    return DL_ERR_WORKSPACE;
  }
  *n_runs = static_cast<int32_t>(nr);
  return DL_OK;
}
// ---------------------------------------------------------------------------
// model-level helpers
// ---------------------------------------------------------------------------
dl_status dl_argmax(const void* logits, int64_t T, int64_t vloc, int32_t P, int64_t rank_stride, int64_t ld,
                    int32_t* ids, void* stream) {
  if (T == 0) return DL_OK;
  DL_TRY(check_ptr(logits, "logits"));
  if (!ids || vloc < 1 || P < 1 || ld < vloc || (P > 1 && rank_stride < T * ld) || P * vloc > 0x7fffffff) {
    set_error("dl_argmax: bad arguments");
    return DL_ERR_INVALID_ARG;
  }
  DL_TRY(check_device());
  return launch_argmax(static_cast<const __nv_bfloat16*>(logits), T, vloc, P, rank_stride, ld, ids,
                       static_cast<cudaStream_t>(stream));
}

dl_status dl_embedding(const void* table, int64_t vocab, int64_t h, const int32_t* ids, int64_t T, void* out,
                       void* stream) {
  if (T == 0) return DL_OK;
  DL_TRY(check_ptr(table, "table"));
  DL_TRY(check_ptr(out, "out"));
  if (!ids || h % 8 || vocab < 1) {
    set_error("dl_embedding: bad arguments");
    return DL_ERR_INVALID_ARG;
  }
  DL_TRY(check_device());
  return launch_embedding(static_cast<const __nv_bfloat16*>(table), vocab, h, ids, T,
                          static_cast<__nv_bfloat16*>(out), static_cast<cudaStream_t>(stream));
}

dl_status dl_rmsnorm(const void* x, const void* gamma, void* out, int64_t T, int64_t h, float eps, void* stream) {
  if (T == 0) return DL_OK;
  DL_TRY(check_ptr(x, "x"));
  DL_TRY(check_ptr(gamma, "gamma"));
  DL_TRY(check_ptr(out, "out"));
  if (h % 8) {
    set_error("h must be a multiple of 8");
    return DL_ERR_ALIGN;
  }
  DL_TRY(check_device());
  return launch_rmsnorm(static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(gamma),
                        static_cast<__nv_bfloat16*>(out), T, h, eps, static_cast<cudaStream_t>(stream));
}

dl_status dl_dense_workspace(int64_t T, int64_t N, int64_t K, size_t* bytes) {
  (void)T; (void)N; (void)K;
  if (!bytes) return DL_ERR_INVALID_ARG;
  *bytes = 0;
  return DL_OK;
}

dl_status dl_dense(const void* X, int64_t ldx, const void* W, int64_t ldw, void* C, int64_t ldc, int64_t T,
                   int64_t N, int64_t K, void* workspace, size_t workspace_bytes, void* stream) {
  (void)workspace; (void)workspace_bytes;
  if (T == 0) return DL_OK;
  if (T < 0 || N <= 0 || K <= 0) {
    set_error("dl_dense: bad shape");
    return DL_ERR_SHAPE;
  }
  DL_TRY(check_ptr(X, "X"));
  DL_TRY(check_ptr(W, "W"));
  DL_TRY(check_ptr(C, "C"));
  DL_TRY(check_ld(ldx, K, DL_BF16, "ldx"));
  DL_TRY(check_ld(ldw, K, DL_BF16, "ldw"));
  DL_TRY(check_ld(ldc, N, DL_BF16, "ldc"));
  DL_TRY(check_device());
  // debug A/B switch (DL_DENSE_SK=1): stream-K with an fp32 reduction into the
  // (zeroed, T*N*4 + 256 bytes) workspace, then conversion -- the decode path's
  // scheme applied to a dense GEMM.
  static const bool sk = DL_ENV("DL_DENSE_SK") && atoi(DL_ENV("DL_DENSE_SK")) != 0;
  if (sk && workspace && workspace_bytes >= static_cast<size_t>(T) * N * 4 + 256 && T <= 256 && N % 4 == 0) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    float* acc = static_cast<float*>(workspace);
    GemmProblem p = one_seg(X, ldx, T, K, W, ldw, N, K, out_plain(acc, N, OUT_F32_RED, 0));
    p.sched = reinterpret_cast<unsigned int*>(static_cast<uint8_t*>(workspace) + static_cast<size_t>(T) * N * 4);
    DL_TRY(tc_gemm(p, true, st));
    return launch_f32_to_bf16(acc, N, static_cast<__nv_bfloat16*>(C), ldc, T, N, 1, st);
  }
  return tc_gemm(one_seg(X, ldx, T, K, W, ldw, N, K, out_plain(C, ldc, OUT_BF16, 0)), false,
                 static_cast<cudaStream_t>(stream));
}

}  // extern "C"
