// Internal interfaces between the C-ABI layer (api.cu) and the kernels.
// Product code only: nothing here is shared with oracle/.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/dl.h"

#define DL_TRY_INTERNAL(expr)   \
  do {                          \
    dl_status _s = (expr);      \
    if (_s != DL_OK) return _s; \
  } while (0)

// A/B timing switches.  Alternatives that were measured and lost stay
// selectable by environment variable for re-measurement, but only in the
// instrumented build (libdl_ab.so, compiled with -DDL_AB_SWITCHES); the
// release library libdl.so ignores the environment entirely and always runs
// the measured defaults, so its behaviour is fixed by include/dl.h alone.
#ifdef DL_AB_SWITCHES
#define DL_ENV(name) getenv(name)
#else
#define DL_ENV(name) (static_cast<const char*>(nullptr))
#endif

namespace dl {
struct CommGroup;   // comm.cu
enum CommKind { kCommNccl = 0, kCommLoopback = 1, kCommGroup = 2, kCommPeer = 3 };
constexpr int kMaxPeers = 8;
// Multi-process symmetric window (dl_comm_window_*): this rank's window and
// its peers' windows mapped into this process (CUDA IPC), plus a flag area
// after each window for the device-side barrier.
struct PeerWindow {
  uint8_t* own = nullptr;                 // cudaMalloc'd: bytes of buffers + kFlagBytes of flags
  size_t bytes = 0;                       // buffer bytes (the flags follow)
  uint8_t* peer[kMaxPeers] = {};          // rank j's window in this address space (peer[rank] = own)
  bool connected = false;
};
constexpr size_t kFlagBytes = 256;        // [kMaxPeers] u32 arrival epochs, then this rank's u32 epoch counter
// NCCL dtype codes (ncclFloat32 / ncclBfloat16), also used by the other kinds
constexpr int kCollF32 = 7;
constexpr int kCollBF16 = 9;
typedef int (*nccl_allreduce_fn)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_reducescatter_fn)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_allgather_fn)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef const char* (*nccl_errstr_fn)(int);
}  // namespace dl

struct dl_comm_s {
  int kind;            // dl::CommKind
  void* nccl;          // kCommNccl: the caller's ncclComm_t
  int rank, world;
  dl::nccl_allreduce_fn allreduce;
  dl::nccl_reducescatter_fn reducescatter;
  dl::nccl_allgather_fn allgather;
  dl::nccl_errstr_fn errstr;
  dl::CommGroup* group;   // kCommGroup: shared by the group's ranks
  dl::PeerWindow* win;    // kCommNccl / kCommPeer: multi-process symmetric window (null: none)
};

namespace dl {

void set_error(const char* fmt, ...);
dl_status cuda_status(cudaError_t e, const char* what);
// DL_OK if the current device is sm_100 (B200), else DL_ERR_CUDA
dl_status check_device_sm100();

// collectives (comm.cu), NCCL semantics for every communicator kind
dl_status coll_all_reduce(dl_comm c, void* buf, size_t count, int dtype, cudaStream_t st);
dl_status coll_reduce_scatter(dl_comm c, const void* src, void* dst, size_t recv_count, int dtype,
                              cudaStream_t st);
dl_status coll_all_gather(dl_comm c, const void* src, void* dst, size_t send_count, int dtype, cudaStream_t st);
// group communicator symmetric window (comm.cu): per-rank bytes (0: the
// communicator has none), rank j's window base, and the barrier that orders
// every rank's preceding stream work before every rank's following work.
size_t comm_window_bytes(dl_comm c);
uint8_t* comm_window(dl_comm c, int rank);
dl_status comm_barrier(dl_comm c, cudaStream_t st);

constexpr int kNumSMsB200 = 148;
int num_sms();

// profile.cu: count a kernel launch and check it; event pair around a GEMM.
dl_status launched(const char* what);
int prof_begin(cudaStream_t st);
void prof_end(int idx, cudaStream_t st, double bytes, double flops, int kind);

// Programmatic dependent launch (PDL).  Every kernel of this library is
// launched with programmatic stream serialization: it may start while its
// predecessor drains, runs pdl_trigger() early so its own successor can do
// the same, and calls pdl_wait() before touching anything a predecessor
// produced (the GEMMs stream their static weights before that point).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// sin / cos of a RoPE angle (pos * theta^(-2i/d), up to ~1e5 rad).  Library
// sincosf takes a Payne-Hanek slow path with a local-memory stack for
// |x| > 105615 and a long fast path otherwise (ncu on the low-rank KV
// reconstruction epilogue: local loads/stores, 30 % tensor utilisation).  Here:
// Cody-Waite reduction by 2*pi in two fp32 parts (2*pi rounded to fp32 exceeds
// 2*pi by 1.7484556e-7), then the SFU __sincosf on [-pi, pi] (abs error
// ~2^-21).  The reduction adds |n| * 2^-24-ish rad, below the fp32 rounding of
// the angle itself (|x| * 2^-24), far below bf16 resolution.
__device__ __forceinline__ void rope_sincos(float x, float* s, float* c) {
  const float n = rintf(x * 0.159154943091895336f);
  float r = fmaf(n, -6.28318548202514648f, x);
  r = fmaf(n, 1.7484556e-7f, r);
  __sincosf(r, s, c);
}

template <typename... KArgs, typename... Args>
dl_status launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     const char* what, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) return cuda_status(e, what);
  return launched(what);
}

// ---------------------------------------------------------------------------
// tcgen05 GEMM family (tc_gemm.cu).
//   C[token][feature] = sum_k act[token][act_koff + k] * W_seg[feature - begin][k]
// act is bf16 row-major [T x Kact] (ld in elements); each segment's weight is
// bf16 row-major [rows x klen] (K-major).  Tiles never straddle segments.
// ---------------------------------------------------------------------------
// q|k|v local rows [T x (Hq + 2 Hk) * d] (fp32 acc or bf16): RoPE on q, k;
// q written (bf16) to q_out [T x Hq*d]; k, v appended to the cache at
// position cache_lens[seq(t)] + (t - cu[seq]) (decode: seq = t).
// Side job of a finalize kernel: zero `rows` rows of `row_bytes` (multiple of
// 16) at p (row stride ld bytes), spread over the kernel's whole grid.
struct SideZero {
  void* p = nullptr;
  int64_t ld = 0, rows = 0, row_bytes = 0;
};

struct RopeCacheArgs {
  const float* acc; const __nv_bfloat16* src; int64_t ld_src; int clear;
  __nv_bfloat16* q_out;
  __nv_bfloat16* k_cache; __nv_bfloat16* v_cache; int64_t max_seq;
  const int32_t* positions; const int32_t* cu_seqlens; const int32_t* cache_lens;
  int32_t num_seqs; int decode;
  int64_t T; int Hq, Hk, d; float theta;
  int rope;            // 0: no rotary embedding (q, k pass through)
  SideZero zero, zero2;   // side jobs (see SideZero)
  int kv_only;         // prefill: q (and RoPE) handled elsewhere -- only append k and v to the caches
};

// Last-contributor finalize of a stream-K GEMM (FixupOp); buffers zeroed on entry,
// left zeroed on exit.
struct GemmFixup {
  int op;                       // FixupOp
  float* acc32;                 // fp32 reduction scratch, output layout (plain rows: acc_ld)
  int64_t acc_ld;
  unsigned int* tile_cnt;       // >= number of output tiles, zeroed
  __nv_bfloat16* resid;         // FIX_RESIDUAL: x += y
  int64_t ld_resid;
  __nv_bfloat16* act_out;       // FIX_SILU: act = silu(seg0) * seg1
  int64_t ld_act_out;
  RopeCacheArgs rope;           // FIX_ROPE_CACHE
};

struct GemmSeg {
  const void* w;      // [rows x klen] bf16 (may be null iff klen == 0)
  int64_t ldw;        // elements
  int64_t rows;       // features in this segment
  int64_t klen;       // K extent of this segment (0 allowed -> zeros)
  int64_t feat_begin; // first global output feature of the segment
  int64_t act_koff;   // column offset of this segment's K range inside act
};

// OUT_BF16_RED: stream-K partials red.add-ed straight into a zeroed bf16
// buffer (red.global.add.noftz.bf16) -- the stage-1 latent Z of the skinny
// path, which needs no fp32 -> bf16 pass; the buffer is zeroed again by the
// kernel that follows the group's stage 2 (SideZero).
enum OutMode { OUT_BF16 = 0, OUT_F32_RED = 1, OUT_F32_STORE = 2, OUT_BF16_RED = 3 };
// Finalize applied by the last stream-K contributor of each output tile.
enum FixupOp { FIX_NONE = 0, FIX_BF16 = 1, FIX_RESIDUAL = 2, FIX_SILU = 3, FIX_ROPE_CACHE = 4 };

struct GemmOut {
  void* ptr;
  int64_t ld;          // elements (row stride of [T x features] output)
  int mode;            // OutMode
  int accumulate;      // OUT_BF16 only: out = bf16(acc + out)
  // reduce-scatter layout (P > 1): feature f of segment g goes to
  //   owner = (f - begin_g) / rpr_g, col = slab_off_g + (f - begin_g) % rpr_g,
  //   index = owner * T * slab + token * slab + col
  int scatter_p;       // 0: plain [token][feature] with ld; >= 1: [P][T][slab]
  int64_t slab;
  int64_t seg_slab_off[3];
  int64_t seg_rpr[3];
  // plain layout only: remap_cols != 0 -> feature f of segment g is stored
  // at column seg_col_off[g] + (f - begin_g) (else column f); the first
  // seg_write_rows[g] (> rows: zero-padded) features of a segment are stored.
  int remap_cols;
  int64_t seg_col_off[3];
  int64_t seg_write_rows[3];
  // whole-tile bf16 outputs only: rope_pos != null -> features [0, rope_end)
  // are 128-wide heads rotated in the epilogue by rope_pos[token] (RoPE of
  // reconstructed keys)
  const int32_t* rope_pos;
  int64_t rope_end;
  float rope_theta;
  // fused collective (swap-AB OUT_BF16_RED only): fan_n > 0 -> the bf16x2
  // partials are red.add-ed into other ranks' buffers (group window, same
  // offset in every window; fan_delta[j] = element offset from ptr to rank j's
  // copy).  scatter_p > 0 (reduce-scatter): only the owner's buffer, laid out
  // [T][slab] (element tok * slab + col); else fan_cols > 0: plain layout,
  // column c goes to the copy of owner c / fan_cols only (the reduce-scatter
  // half of a two-shot all-reduce); else all fan_n copies (one-shot).
  int fan_n;
  int64_t fan_cols;
  int64_t fan_delta[8];
};

struct GemmProblem {
  const void* act; int64_t ld_act; int64_t T; int64_t k_act;  // act [T x k_act]
  int nseg; GemmSeg seg[3];
  int64_t n_feat;      // total output features (sum of seg rows)
  GemmOut out;
  // stream-K only: 2 zero-initialised uint32 counters (work, done) in device
  // memory enabling the hybrid static + dynamic split; null -> static split.
  // Launches that may overlap (PDL) must use different counter pairs.
  unsigned int* sched;
  // stream-K + swap only: last-arriver finalize (requires sched)
  GemmFixup fix;
  // prefill (CTA-pair) only: zeroed fp32 scratch for the DP + stream-K tail
  // (<= 44 tiles x 256 x 256 x 4 B); left zeroed.  null -> whole tiles only.
  float* tail_acc;
  size_t tail_bytes;
  // act_p > 1 (swap-AB decode path only): act is the rank-major all-gather
  // output [act_p][T][act_w] and column c of the logical [T x act_p*act_w]
  // operand is (c / act_w, c % act_w); act_w % 64 == 0.  The TMA reads it
  // through a 3-D map, so no un-permute pass is needed.
  int act_p;
  int64_t act_w;
  // xform != 0 (swap-AB stream-K only): the activation operand is not read by
  // TMA but computed by the kernel's epilogue warps from xsrc [T x xld] bf16
  // (the reduced gate|up output of the previous group): XFORM_SILU: act[t][c] =
  // silu(xsrc[t][c]) * xsrc[t][xm + c]; XFORM_RELU: act[t][c] = relu(xsrc[t][c]);
  // columns c >= k_act read as zero.  Replaces the SiLU / ReLU kernel between
  // the MLP's gate|up and down projections (the down group's stage 1).
  int xform;
  const __nv_bfloat16* xsrc;
  int64_t xld, xm;
  // glu != 0 (prefill CTA-pair path only): segment 0 = gate, segment 1 = up
  // (equal rows m, m % 256 == 0, equal klen); the epilogue writes only
  // out[t][f] = bf16(silu(gate[t][f]) * up[t][f]) ([T x m], plain bf16 layout
  // with out.ld), from the fp32 accumulators -- the SiLU.up pass and the
  // [T x 2m] gate|up round trip through HBM are gone (the MLP of
  // the decomposed block).
  int glu;
};
enum XformMode { XFORM_NONE = 0, XFORM_SILU = 1, XFORM_RELU = 2 };

// Picks the tile configuration (swap-AB for T <= 256, stream-K when the
// output is fp32-reduced) and launches.  `stream_k` requires OUT_F32_RED.
dl_status tc_gemm(const GemmProblem& p, bool stream_k, cudaStream_t st);
// Fused two-stage chain of one factor group in ONE persistent launch (skinny
// swap-AB stream-K path, T <= 256): p1 = stage 1 (its reduction output is p2's
// activation), p2 = stage 2.  Stage-2 weight tiles stream while stage 1 is
// still reducing; stage-2 activation loads wait on the in-kernel arrival
// counter `chain` (2 zero-initialised uint32, left zeroed; launches that may
// overlap under PDL must use different pairs).
dl_status tc_gemm_chain(const GemmProblem& p1, const GemmProblem& p2, unsigned int* chain, cudaStream_t st);
// debug timeline: when buf != NULL every GEMM CTA writes 8 u64 at buf[cta*8]
// (globaltimer ns at entry, setup done, first TMA, first stage landed, last
// MMA issued, epilogue done, exit; and its SM id)
dl_status set_gemm_trace(void* buf);
// per-CTA debug timeline of a non-GEMM launch in the GEMM trace buffer:
// nslots consecutive 148-CTA slots (8 u64 per CTA), or null when tracing is off
unsigned long long* gemm_trace_cta_slots(int nslots);
// Debug timeline of selected non-GEMM kernels (dl_debug_ew_trace): per launch
// slot 4 u64 = {kind, min entry, min start after griddepcontrol.wait, max end}.
dl_status set_ew_trace(void* buf);
int ew_trace_slot();   // next slot (host), -1 when tracing is off
struct EwTrace {
  unsigned long long* buf;   // null: off
  int slot, kind;
};
EwTrace ew_trace(int kind);
__device__ __forceinline__ unsigned long long ew_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void ew_mark(const EwTrace& tr, int field) {   // field 1 entry, 2 start, 3 end
  if (!tr.buf || threadIdx.x != 0) return;
  unsigned long long* r = tr.buf + static_cast<long long>(tr.slot) * 4;
  if (field == 1) r[0] = static_cast<unsigned long long>(tr.kind);
  if (field == 3) atomicMax(r + 3, ew_now());
  else atomicMin(r + field, ew_now());
}

// 2-D bf16 TMA map over a row-major [rows x cols] matrix (ld elements), box
// {64 cols, box_rows}, 128B swizzle, out-of-bounds elements read as zero.
bool encode_map_bf16(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows);

// ---------------------------------------------------------------------------
// SIMT skinny chain (simt_chain.cu): Y[T x m] (+)= (X B^T) A^T, T <= 16.
// ---------------------------------------------------------------------------
dl_status simt_lowrank(const void* X, int64_t ldx, const void* A, int64_t lda,
                       const void* B, int64_t ldb, void* Y, int64_t ldy,
                       int64_t T, int64_t m, int64_t n, int64_t k, dl_dtype dt,
                       int accumulate, void* zbuf, cudaStream_t st);

// ---------------------------------------------------------------------------
// Elementwise (elementwise.cu); bf16 storage, fp32 math.
// ---------------------------------------------------------------------------
dl_status launch_rmsnorm(const __nv_bfloat16* x, const __nv_bfloat16* g,
                         __nv_bfloat16* y, int64_t T, int64_t h, float eps,
                         cudaStream_t st);
// out_bf16[t][c] = bf16(acc[t][c]) ; acc zeroed afterwards (consume-and-clear)
dl_status launch_f32_to_bf16(float* acc, int64_t ld_acc, __nv_bfloat16* out,
                             int64_t ld_out, int64_t T, int64_t n, int clear,
                             cudaStream_t st, const SideZero& z = SideZero{});
// x[t][c] = bf16(x + acc) ; acc cleared
dl_status launch_residual_add_f32(float* acc, int64_t ld_acc, __nv_bfloat16* x,
                                  int64_t ldx, int64_t T, int64_t n,
                                  int clear, cudaStream_t st, const SideZero& z = SideZero{},
                                  const SideZero& z2 = SideZero{});
// x[t][c] = bf16(x + acc) (acc cleared), then y = rmsnorm(x) * g   (h % 8 == 0)
dl_status launch_residual_rmsnorm(float* acc, int64_t lda, __nv_bfloat16* x, const __nv_bfloat16* g,
                                  __nv_bfloat16* y, int64_t T, int64_t h, float eps, cudaStream_t st,
                                  const SideZero& z = SideZero{}, const SideZero& z2 = SideZero{});
// the same with a bf16 accumulator (a TP collective's result, consumed and cleared)
dl_status launch_residual_rmsnorm_bf16(__nv_bfloat16* acc, int64_t lda, __nv_bfloat16* x, const __nv_bfloat16* g,
                                       __nv_bfloat16* y, int64_t T, int64_t h, float eps, cudaStream_t st,
                                       const SideZero& z = SideZero{}, const SideZero& z2 = SideZero{});
// x[t][c] = bf16(x + y)
// clear != 0: y is zeroed as it is read (a bf16 reduction target)
dl_status launch_residual_add_bf16(const __nv_bfloat16* y, int64_t ldy, __nv_bfloat16* x,
                                   int64_t ldx, int64_t T, int64_t n, cudaStream_t st, int clear = 0,
                                   const SideZero& z = SideZero{}, const SideZero& z2 = SideZero{});
// act[t][i] = bf16(silu(g) * u) with g = src[t][i], u = src[t][m + i]
dl_status launch_silu_mul_f32(float* acc, int64_t ld_acc, __nv_bfloat16* act,
                              int64_t ld_act, int64_t T, int64_t m, int clear,
                              cudaStream_t st, const SideZero& z = SideZero{});
dl_status launch_silu_mul_bf16(const __nv_bfloat16* src, int64_t ld_src,
                               __nv_bfloat16* act, int64_t ld_act, int64_t T,
                               int64_t m, cudaStream_t st, int clear = 0, const SideZero& z = SideZero{});
// act[t][i] = bf16(relu(u)), u = src[t][i] (non-GLU MLP)
dl_status launch_relu_f32(float* acc, int64_t ld_acc, __nv_bfloat16* act, int64_t ld_act, int64_t T,
                          int64_t m, int clear, cudaStream_t st, const SideZero& z = SideZero{});
dl_status launch_relu_bf16(const __nv_bfloat16* src, int64_t ld_src, __nv_bfloat16* act, int64_t ld_act,
                           int64_t T, int64_t m, cudaStream_t st, int clear = 0, const SideZero& z = SideZero{});
// RoPE + cache append as a standalone kernel (see RopeCacheArgs)
dl_status launch_rope_cache(const RopeCacheArgs& a, cudaStream_t st);
dl_status launch_argmax(const __nv_bfloat16* logits, int64_t T, int64_t vloc, int P, int64_t rank_stride,
                        int64_t ld, int32_t* ids, cudaStream_t st);
dl_status launch_embedding(const __nv_bfloat16* table, int64_t vocab, int64_t h,
                           const int32_t* ids, int64_t T, __nv_bfloat16* out,
                           cudaStream_t st);
// all-gather by push (fused collective): src [T x w] (ld_src) -> dst + delta[j]
// + t * w for j < P (dst = this rank's slot of its own window); `z` side clear
dl_status launch_fan_copy(const __nv_bfloat16* src, int64_t ld_src, __nv_bfloat16* dst, const int64_t* delta,
                          int P, int64_t T, int64_t w, cudaStream_t st, const SideZero& z = SideZero{});
// all-gather half of a fused two-shot all-reduce: this rank's finished columns
// [c0, c1) of buf [T x ld] (its window) copied into the same place of every
// other rank's window (buf + delta[j]); `z` side clear
dl_status launch_fan_push(__nv_bfloat16* buf, int64_t ld, int64_t T, int64_t c0, int64_t c1, const int64_t* delta,
                          int P, int self, cudaStream_t st, const SideZero& z = SideZero{});
// [P][T][w] -> [T][P*w]
dl_status launch_unpermute(const __nv_bfloat16* src, __nv_bfloat16* dst,
                           int P, int64_t T, int64_t w, cudaStream_t st);
// DeInfer latent all-gather result [P][T][slot] -> group Z layout (see elementwise.cu)
struct LatentMap {
  int nseg, P; int64_t T, slot;
  int64_t base, extra;                     // balanced split of the group rank L over P
  int64_t seg_beg[3], seg_len[3], zoff[3]; // latent start / length / Z column offset per segment
  int64_t width;                           // Z layout width
};
dl_status launch_latent_unpermute(const __nv_bfloat16* recv, __nv_bfloat16* zb, int64_t ldzb,
                                  const LatentMap& mp, cudaStream_t st, const SideZero& z = SideZero{});
// Low-rank KV cache (N3).  append: latent row zb[t][zoff .. zoff + ncopy) of
// decode token t -> pool slot of (seq t, position cache_lens[t]) through the
// block table; slot_pos[slot] = positions[t].
dl_status launch_kv_append(const __nv_bfloat16* zb, int64_t ldzb, int64_t zoff, int64_t ncopy,
                           __nv_bfloat16* pool, int64_t ld_slot, int32_t* slot_pos, int64_t block_size,
                           const int32_t* block_tables, int64_t max_blocks_per_seq, const int32_t* cache_lens,
                           const int32_t* positions, int64_t T, cudaStream_t st);
// squeeze: copy the contiguous runs (device plan) of the pool into the
// compact buffer, whole blocks (rows of ld_slot bf16 + positions)
dl_status launch_kv_squeeze(const __nv_bfloat16* pool, const int32_t* slot_pos, __nv_bfloat16* squeeze,
                            int32_t* squeeze_pos, int64_t ld_slot, int64_t block_size, const int32_t* run_src,
                            const int32_t* run_dst, const int32_t* run_len, const int32_t* n_runs,
                            int64_t cap_blocks, cudaStream_t st);
// in-place RoPE of the first `heads` 128-wide heads of each row (positions pos[row])
dl_status launch_rope_rows(__nv_bfloat16* buf, int64_t ld, int heads, const int32_t* pos, int64_t rows, float theta,
                           cudaStream_t st);
dl_status launch_copy2d(const void* src, int64_t lds, void* dst, int64_t ldd,
                        int64_t rows, int64_t cols_bytes, cudaStream_t st);

// ---------------------------------------------------------------------------
// Attention (attention.cu).  Cache layout [S][Hk][max_seq][d] bf16.
// q [T x Hq*d] bf16 (post-RoPE), out [T x Hq*d] bf16.
// ---------------------------------------------------------------------------
struct AttnArgs {
  const __nv_bfloat16* q; __nv_bfloat16* out;
  int64_t ld_q;                           // prefill: row stride of q (0: Hq * d)
  const __nv_bfloat16* k_cache; const __nv_bfloat16* v_cache; int64_t max_seq;
  const int32_t* cu_seqlens; const int32_t* cache_lens; int32_t num_seqs;
  int64_t T; int Hq, Hk, d; int decode;
  float* partial; size_t partial_bytes;   // split-KV scratch (decode)
  // decode only: kv_ld != 0 -> K/V rows are token-major with stride kv_ld
  // (elements); sequence s starts at row kv_blk0[s] * kv_bs; kv head g at +g*d
  int64_t kv_ld; const int32_t* kv_blk0; int64_t kv_bs; int64_t kv_rows;
  // stream-K decode kernel: zero-maintained counters + partial slots
  // (attention_sk_workspace(sk_items_cap / Hq, Hq) bytes)
  void* sk_ws; int64_t sk_items_cap;
  // fused RoPE + cache append (decode, head-major cache, stream-K kernel only):
  // qkv != null -> q|k|v rows [T x ld_qkv] bf16 straight from the q|k|v group
  // (the kernel rotates q and the new key with positions[t], appends k and v at
  // cache_lens[t]); `zero`, `zero2` are side clears done once the kernel has waited.
  // The kernel returns DL_ERR_UNSUPPORTED if it cannot take them.
  const __nv_bfloat16* qkv; int64_t ld_qkv; const int32_t* positions; float theta; int rope;
  SideZero zero, zero2;
};
dl_status launch_attention(const AttnArgs& a, cudaStream_t st);
// prefill (a.decode == 0) on tcgen05 / TMEM / TMA (attn_tc.cu)
dl_status launch_attention_prefill_tc(const AttnArgs& a, cudaStream_t st);
size_t attention_workspace(int64_t max_tokens, int Hq, int d);
size_t attention_sk_workspace(int64_t max_tokens, int Hq);

}  // namespace dl
