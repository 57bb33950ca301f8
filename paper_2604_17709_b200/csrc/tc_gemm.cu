// tcgen05 / TMEM / TMA GEMM family for the two stages of the low-rank chain
// y = A (B x)  (Section 2.1, Eq. 1):
//
//   stage 1  Z[T x k] = X[T x n] . B[k x n]^T      (downward projection x_v)
//   stage 2  Y[T x m] = Z[T x k] . A_g[m_g x k_g]^T (upward projection x_u,
//            grouped: each output segment g reads its own K range of Z)
//
// Both operands are K-major (row-major activations, row-major A and B), the
// layout tcgen05.mma consumes directly from 128B-swizzled shared memory.
//
// One persistent, warp-specialised kernel (1 CTA / SM, 192 threads):
//   warp 0      TMA producer: STAGES-deep smem ring (full/empty mbarriers)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> global
// The fp32 accumulator is double-buffered in TMEM (2 x BN columns) so the
// epilogue of job i overlaps the main loop of job i+1.
//
// Orientation:
//   SWAP = false (prefill, T > 256): MMA M = 128 tokens, N = BN features.
//   SWAP = true  (decode, T <= 256): "swap-AB": MMA M = 128 weight rows
//                (features), N = BN >= T tokens.  The weights are the
//                streamed operand; tokens ride along as the narrow N.
// Work split:
//   whole-tile  : tiles dealt round-robin to CTAs, output written once
//                 (bf16, optional fused "+= out" residual).
//   stream-K    : the (tile, k-block) iteration space is cut into equal
//                 contiguous ranges, one per CTA (one wave, perfect balance
//                 for the memory-bound decode); partial tiles are reduced
//                 with red.global.add.f32 into a zeroed fp32 buffer.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>

#include <mutex>

#include "dl_internal.h"
#include "sm100_ptx.cuh"

namespace dl {
namespace {

constexpr int BK = 64;   // K elements per stage = one 128-byte swizzle row
constexpr int BM = 128;  // MMA M = TMEM lanes
constexpr int kThreads = 320;   // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue
constexpr int kJobRing = 8;     // producer -> MMA / epilogue job queue depth
constexpr int kStageOutWarp = 32 * 64;   // pair epilogue: per-warp staging of 32 rows x 32 bf16 features
constexpr int kL2Prefetch = 0;  // weight tiles pulled into L2 before griddepcontrol.wait (DL_L2PF); measured: 24 costs ~1 ms per 70B decode step

struct KSeg {
  int feat_begin, feat_end;  // global output features [begin, end)
  int act_koff;              // K offset of this segment inside the activation
  int nkb;                   // k-blocks (ceil(klen / 64))
  int tile_first;            // first global tile index of the segment
  int ntiles;                // tiles in the segment (feature tiles * token tiles)
  long long unit_first;      // stream-K: first unit (tile, kb) of the segment
  long long slab_off, rpr;   // reduce-scatter layout
  int write_end;             // features < write_end are stored (>= feat_end: zeros)
  long long col_off;         // plain layout: column of feature feat_begin
};

struct KArgs {
  int T;
  int tiles_tok;
  int nseg;
  KSeg seg[3];
  int total_tiles;
  long long total_units;
  int stream_k;
  void* out;
  long long ldo;
  int mode;
  int accumulate;
  int scatter_p;
  long long slab;
  int trace_slot;            // debug timeline slot of this launch (-1: none)
  // hybrid stream-K: CTA c first takes units [c*static_units, (c+1)*static_units),
  // then grabs `chunk`-unit pieces of [dyn_begin, total_units) from sched[0];
  // sched[1] counts CTAs done grabbing (the last one resets both).  sched == null:
  // purely static stream-K.
  unsigned int* sched;
  long long static_units, dyn_begin;
  int chunk;
  int l2pf;                  // weight tiles prefetched into L2 before griddepcontrol.wait
  int chain_pf;              // chain stage 2: units whose weights are staged before the in-kernel wait (DL_CHAIN_PF)
  int chain_warp;            // chain: stage-1 arrivals per epilogue warp instead of per CTA (DL_CHAIN_WARP)
  int relaxed_acce;
  int stage_out;             // pair kernel: bf16 stores through the shared-memory transpose (bit 0 plain, bit 1 Y +=; DL_STAGE_OUT)          // accumulator-empty arrivals without release semantics (DL_ACCE_RELEASE=1: off)
  int act_w;                 // > 0: 3-D activation map, column c -> (c % act_w, token, c / act_w)
  int xform;                 // XformMode: activation computed in-kernel from xsrc (GemmProblem::xform)
  const __nv_bfloat16* xsrc;
  long long xld;
  int xm, xcols;
  int wpol;                  // pair kernel weight L2 policy: 0 evict_first, 1 evict_normal, 2 evict_last
  int tail_vec;              // tail finalize: 8-byte stores, Y += old values loaded up front (DL_TAIL_VEC=0: scalar)
  // pair kernel GLU mode (GemmProblem::glu): seg 0 = gate, seg 1 = up; the
  // whole-tile schedule runs over tile PAIRS (total_tiles / dp_tiles count
  // pairs), each emitted as the gate job (accumulator 0) then the up job of the
  // same features (accumulator 1); tail pieces go to tail_acc slots 2p, 2p + 1
  int glu;
  int glu_spol;              // GLU act stores: 0 plain, 1 L2 evict_last hint (the down stage 1 re-reads them)
  // DP + stream-K tail (whole-tile kernels): tiles [0, dp_tiles) whole, each of
  // the remaining tiles split in tail_split K-pieces accumulated in fp32 into
  // tail_acc [tail tile][256][256], finalized by tc_tail_finalize_kernel.
  int dp_tiles, tail_split;
  float* tail_acc;
  // Stream-K fixup (swap-AB stream-K only): contributors red.add fp32 partials
  // into acc32 (same layout as the output, plain rows use acc_ld), bump
  // tile_cnt[tile]; the last contributor applies `fixup` to the reduced tile,
  // writes the final output and zeroes acc32 / the counter.
  int fixup;                 // FixupOp
  float* acc32;
  long long acc_ld;
  unsigned int* tile_cnt;
  __nv_bfloat16* resid;      // FIX_RESIDUAL target x [T x ld_resid]
  long long ld_resid;
  __nv_bfloat16* act_out;    // FIX_SILU output [T x ld_act_out] (gate = seg 0, up = seg 1)
  long long ld_act_out;
  RopeCacheArgs rope;        // FIX_ROPE_CACHE (q|k|v segments, one 128-feature head per tile)
  // epilogue RoPE of whole-tile bf16 outputs (GemmOut::rope_pos)
  const int32_t* rope_pos;
  int rope_end;
  float rope_l2t;
  // fused collective targets (GemmOut::fan_n / fan_cols / fan_delta)
  int fan_n;
  long long fan_cols;
  long long fan_delta[8];
};

// RoPE of 8 consecutive output features f..f+7 (4 pairs (2i, 2i+1) of a
// 128-wide head) of token `tok`: angle = pos * theta^(-dim/128), the same
// expression as rope_cache_kernel.
// `pos` = rope_pos[tok] as float, loaded once per tile row (rope_pos_of).
__device__ __forceinline__ float rope_pos_of(const KArgs& a, int tok) {
  return (a.rope_pos != nullptr && tok < a.T) ? static_cast<float>(a.rope_pos[tok]) : 0.f;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float2 unpack_bf16(uint32_t v) {
  return make_float2(__uint_as_float(v << 16), __uint_as_float(v & 0xffff0000u));
}
// SiLU through one MUFU op (as elementwise.cu's silu_tanh): g sigmoid(g) =
// r + r tanh(r), r = g / 2 (tanh.approx, relative error ~2^-11)
__device__ __forceinline__ float silu_tanh_f(float g) {
  const float r = 0.5f * g;
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(r));
  return fmaf(r, t, r);
}

__device__ __forceinline__ void rope8(const KArgs& a, float pos, int f, float* v) {
  if (a.rope_pos == nullptr || f >= a.rope_end) return;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int dim = (f + 2 * e) & 127;
    float sn, cs;
    rope_sincos(pos * exp2f(-a.rope_l2t * static_cast<float>(dim) / 128.f), &sn, &cs);
    const float x = v[2 * e], y = v[2 * e + 1];
    v[2 * e] = x * cs - y * sn;
    v[2 * e + 1] = x * sn + y * cs;
  }
}

__device__ __forceinline__ long long acc_index(const KArgs& a, const KSeg& s, int tok, int f) {
  if (a.scatter_p <= 0) return static_cast<long long>(tok) * a.acc_ld + s.col_off + (f - s.feat_begin);
  long long loc = f - s.feat_begin;
  long long owner = loc / s.rpr;
  return owner * static_cast<long long>(a.T) * a.slab + static_cast<long long>(tok) * a.slab + s.slab_off +
         loc % s.rpr;
}

// Number of stream-K pieces (jobs) covering the unit interval [lo, hi) under
// the hybrid partition: static range starts c*S (1 <= c <= grid) and dynamic
// chunk starts dyn_begin + i*chunk (i >= 1) that fall strictly inside.
__device__ __forceinline__ int pieces_in(const KArgs& a, long long lo, long long hi, int grid) {
  int n = 1;
  const long long S = a.static_units;
  if (S > 0) {
    long long c0 = lo / S + 1;                       // first c with c*S > lo
    long long c1 = (hi - 1) / S;                     // last c with c*S < hi
    if (c1 > grid) c1 = grid;
    if (c1 >= c0) n += static_cast<int>(c1 - c0 + 1);
  }
  const long long D = a.dyn_begin, C = a.chunk;
  long long i0 = lo < D ? 1 : (lo - D) / C + 1;      // first i >= 1 with D + i*C > lo
  long long i1 = hi - 1 < D ? 0 : (hi - 1 - D) / C;  // last i with D + i*C < hi
  if (i1 >= i0) n += static_cast<int>(i1 - i0 + 1);
  return n;
}

struct Job {
  int seg, feat0, tok0, kb0, kb1;
  int part;   // >= 0: K-split piece of tail tile `part` (fp32 partial into tail_acc)
  int ph;     // chain kernel: 0 = stage 1, 1 = stage 2
};

__device__ __forceinline__ long long out_index(const KArgs& a, const KSeg& s, int tok, int f) {
  if (a.scatter_p <= 0) return static_cast<long long>(tok) * a.ldo + s.col_off + (f - s.feat_begin);
  long long loc = f - s.feat_begin;
  long long owner = loc / s.rpr;
  long long col = s.slab_off + loc % s.rpr;
  return owner * static_cast<long long>(a.T) * a.slab + static_cast<long long>(tok) * a.slab + col;
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }   // 8 epilogue warps

__device__ __forceinline__ float silu_f(float g) { return g / (1.f + __expf(-g)); }

__device__ __forceinline__ float4 ldcg4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4zero(float* p) { *reinterpret_cast<float4*>(p) = make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void st_bf16x4(__nv_bfloat16* p, float a, float b, float c, float d) {
  uint2 o;
  reinterpret_cast<__nv_bfloat162*>(&o)[0] = __floats2bfloat162_rn(a, b);
  reinterpret_cast<__nv_bfloat162*>(&o)[1] = __floats2bfloat162_rn(c, d);
  *reinterpret_cast<uint2*>(p) = o;
}

// Stream-K fixup for one finished job of the swap-AB kernel (feature tile of
// 128 rows, all tokens).  Runs on the 256 epilogue threads (etid 0..255).
// Release: the CTA's red.add partials are ordered before the counter update by
// bar.sync + one thread's gpu-scope fence (cumulative, as in split-K
// semaphores).  The last contributor of the tile (or of the gate/up tile pair
// for FIX_SILU) then reads the reduced fp32 tile from L2 (float4, 8 loads in
// flight per thread), applies the finalize op, writes the final output and
// zeroes the scratch and the counter.
__device__ __noinline__ void fixup_tile(const KArgs& a, const struct Job& j, int etid, int& last_flag) {
  epi_bar();
  const KSeg& s = a.seg[j.seg];
  const int tl = (j.feat0 - s.feat_begin) / 128;   // tile index inside its segment
  const int ci = a.fixup == FIX_SILU ? tl : s.tile_first + tl;
  if (etid == 0) {
    int expected;
    if (a.fixup == FIX_SILU) {
      const KSeg& g0 = a.seg[0];
      const KSeg& g1 = a.seg[1];
      expected = pieces_in(a, g0.unit_first + static_cast<long long>(tl) * g0.nkb,
                           g0.unit_first + static_cast<long long>(tl + 1) * g0.nkb, gridDim.x) +
                 pieces_in(a, g1.unit_first + static_cast<long long>(tl) * g1.nkb,
                           g1.unit_first + static_cast<long long>(tl + 1) * g1.nkb, gridDim.x);
    } else {
      expected = pieces_in(a, s.unit_first + static_cast<long long>(tl) * s.nkb,
                           s.unit_first + static_cast<long long>(tl + 1) * s.nkb, gridDim.x);
    }
    unsigned old;
    asm volatile("fence.acq_rel.gpu;\n\tatom.add.acq_rel.gpu.global.u32 %0, [%1], 1;"
                 : "=r"(old) : "l"(a.tile_cnt + ci) : "memory");
    last_flag = (static_cast<int>(old) == expected - 1) ? 1 : 0;
  }
  epi_bar();
  if (!last_flag) return;
  asm volatile("fence.acq_rel.gpu;" ::: "memory");   // acquire: all contributors' partials visible
  const int T = a.T;
  constexpr int V = 8;                               // float4 loads in flight per thread
  const int nq = 32 * T;                             // float4 quads in a 128-feature x T tile
  if (a.fixup == FIX_BF16 || a.fixup == FIX_RESIDUAL) {
    const int nf = min(128, s.write_end - j.feat0);
    for (int base = etid; base < nq; base += 256 * V) {
      float4 v[V];
      float* pa[V];
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const int q = base + k * 256, fl = (q & 31) * 4, t = q >> 5;
        pa[k] = (q < nq && fl < nf) ? a.acc32 + acc_index(a, s, t, j.feat0 + fl) : nullptr;
        v[k] = pa[k] ? ldcg4(pa[k]) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < V; ++k) {
        if (!pa[k]) continue;
        st4zero(pa[k]);
        const int q = base + k * 256, fl = (q & 31) * 4, t = q >> 5;
        const int f = j.feat0 + fl;
        if (a.fixup == FIX_BF16) {
          st_bf16x4(static_cast<__nv_bfloat16*>(a.out) + out_index(a, s, t, f), v[k].x, v[k].y, v[k].z, v[k].w);
        } else {
          __nv_bfloat16* px = a.resid + static_cast<long long>(t) * a.ld_resid + f;
          const uint2 xo = *reinterpret_cast<const uint2*>(px);
          const float2 x0 = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(&xo)[0]);
          const float2 x1 = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(&xo)[1]);
          st_bf16x4(px, x0.x + v[k].x, x0.y + v[k].y, x1.x + v[k].z, x1.y + v[k].w);
        }
      }
    }
  } else if (a.fixup == FIX_SILU) {
    const KSeg& g0 = a.seg[0];
    const KSeg& g1 = a.seg[1];
    const int fg0 = g0.feat_begin + tl * 128, fu0 = g1.feat_begin + tl * 128;
    const int nf = min(128, g0.feat_end - fg0);
    for (int base = etid; base < nq; base += 256 * (V / 2)) {
      float4 gv[V / 2], uv[V / 2];
      float *pg[V / 2], *pu[V / 2];
#pragma unroll
      for (int k = 0; k < V / 2; ++k) {
        const int q = base + k * 256, fl = (q & 31) * 4, t = q >> 5;
        const bool ok = q < nq && fl < nf;
        pg[k] = ok ? a.acc32 + acc_index(a, g0, t, fg0 + fl) : nullptr;
        pu[k] = ok ? a.acc32 + acc_index(a, g1, t, fu0 + fl) : nullptr;
        gv[k] = ok ? ldcg4(pg[k]) : make_float4(0.f, 0.f, 0.f, 0.f);
        uv[k] = ok ? ldcg4(pu[k]) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < V / 2; ++k) {
        if (!pg[k]) continue;
        st4zero(pg[k]);
        st4zero(pu[k]);
        const int q = base + k * 256, fl = (q & 31) * 4, t = q >> 5;
        st_bf16x4(a.act_out + static_cast<long long>(t) * a.ld_act_out + tl * 128 + fl, silu_f(gv[k].x) * uv[k].x,
                  silu_f(gv[k].y) * uv[k].y, silu_f(gv[k].z) * uv[k].z, silu_f(gv[k].w) * uv[k].w);
      }
    }
  } else if (a.fixup == FIX_ROPE_CACHE) {
    const RopeCacheArgs& r = a.rope;
    const int hh = tl;                         // head index inside the q / k / v segment
    const float l2t = log2f(r.theta);
    for (int base = etid; base < nq; base += 256 * V) {
      float4 v[V];
      float* pa[V];
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const int q = base + k * 256, e = (q & 31) * 4, t = q >> 5;
        pa[k] = q < nq ? a.acc32 + acc_index(a, s, t, j.feat0 + e) : nullptr;
        v[k] = pa[k] ? ldcg4(pa[k]) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < V; ++k) {
        if (!pa[k]) continue;
        st4zero(pa[k]);
        const int q = base + k * 256, e = (q & 31) * 4, t = q >> 5;
        float4 o = v[k];
        if (r.rope && j.seg < 2) {   // rotate pairs (e, e+1), (e+2, e+3) by pos * theta^(-e/d)
          const float pos = static_cast<float>(r.positions[t]);
          float s0, c0, s1, c1;
          rope_sincos(pos * exp2f(-l2t * static_cast<float>(e) / r.d), &s0, &c0);
          rope_sincos(pos * exp2f(-l2t * static_cast<float>(e + 2) / r.d), &s1, &c1);
          o = make_float4(v[k].x * c0 - v[k].y * s0, v[k].x * s0 + v[k].y * c0, v[k].z * c1 - v[k].w * s1,
                          v[k].z * s1 + v[k].w * c1);
        }
        if (j.seg == 0) {
          st_bf16x4(r.q_out + static_cast<long long>(t) * r.Hq * r.d + static_cast<long long>(hh) * r.d + e, o.x, o.y,
                    o.z, o.w);
        } else {
          int sq;
          long long cpos;
          if (r.decode) {
            sq = t;
            cpos = r.cache_lens[t];
          } else {
            int lo = 0, hi = r.num_seqs - 1;
            while (lo < hi) {
              const int mid = (lo + hi + 1) >> 1;
              if (r.cu_seqlens[mid] <= t) lo = mid; else hi = mid - 1;
            }
            sq = lo;
            cpos = r.cache_lens[sq] + (t - r.cu_seqlens[sq]);
          }
          st_bf16x4((j.seg == 1 ? r.k_cache : r.v_cache) +
                        ((static_cast<long long>(sq) * r.Hk + hh) * r.max_seq + cpos) * r.d + e,
                    o.x, o.y, o.z, o.w);
        }
      }
    }
  }
  epi_bar();
  if (etid == 0) atomicExch(a.tile_cnt + ci, 0u);
}

struct __align__(64) KMaps {
  CUtensorMap act;
  CUtensorMap w[3];
};

__device__ unsigned long long* g_trace = nullptr;
bool g_trace_host_on = false;   // host: assign a slot to every launch while tracing
int g_trace_next = 0;
unsigned long long* g_trace_host_buf = nullptr;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %smid;" : "=r"(s));
  return s;
}


// Job enumeration shared by the three roles (pure function of blockIdx).
struct JobIter {
  const KArgs& a;
  int cta, grid;
  int next_tile;            // whole-tile mode
  bool tail_taken = false;  // DP + stream-K tail piece already issued
  bool glu_up = false;      // GLU: the up job of the last gate job is next
  long long u, u_end;       // stream-K mode
  __device__ JobIter(const KArgs& args, int c, int g) : a(args), cta(c), grid(g) {
    next_tile = c;
    if (a.stream_k) {
      u = (a.total_units * c) / g;
      u_end = (a.total_units * (c + 1)) / g;
    } else {
      u = u_end = 0;
    }
  }
  __device__ void set_range(long long b, long long e) {
    u = b;
    u_end = e;
  }
  __device__ bool next(Job& j, int FEAT_TILE, int TOK_TILE) {
    if (a.glu && glu_up) {
      // the up tile of the same features / tokens / K range as the gate job in j
      glu_up = false;
      j.feat0 += a.seg[1].feat_begin - a.seg[0].feat_begin;
      j.seg = 1;
      if (j.part >= 0) ++j.part;
      return true;
    }
    if (!a.stream_k) {
      // data-parallel whole tiles, then (DP + stream-K tail) one K-split piece
      // of the last partial wave's tiles per CTA / cluster
      int t, part = -1;
      if (next_tile < a.dp_tiles) {
        t = next_tile;
        next_tile += grid;
      } else if (a.tail_split > 0 && !tail_taken && cta < (a.total_tiles - a.dp_tiles) * a.tail_split) {
        tail_taken = true;
        part = cta / a.tail_split;
        t = a.dp_tiles + part;
      } else {
        return false;
      }
      int g = 0;
      while (g + 1 < a.nseg && t >= a.seg[g + 1].tile_first) ++g;
      int local = t - a.seg[g].tile_first;
      j.seg = g;
      j.feat0 = a.seg[g].feat_begin + (local / a.tiles_tok) * FEAT_TILE;
      j.tok0 = (local % a.tiles_tok) * TOK_TILE;
      j.part = part;
      if (a.glu) {   // t is a pair: its gate job now, the up job next
        j.part = part < 0 ? -1 : 2 * part;
        glu_up = true;
      }
      if (part < 0) {
        j.kb0 = 0;
        j.kb1 = a.seg[g].nkb;
      } else {
        const int piece = cta % a.tail_split, nkb = a.seg[g].nkb;
        j.kb0 = piece * nkb / a.tail_split;
        j.kb1 = (piece + 1) * nkb / a.tail_split;
      }
      return true;
    }
    while (u < u_end) {
      int g = 0;
      while (g + 1 < a.nseg && u >= a.seg[g + 1].unit_first) ++g;
      const KSeg& s = a.seg[g];
      if (s.nkb == 0) { u = (g + 1 < a.nseg) ? a.seg[g + 1].unit_first : u_end; continue; }
      long long local = u - s.unit_first;
      int tile = static_cast<int>(local / s.nkb);
      int kb0 = static_cast<int>(local % s.nkb);
      long long rem = u_end - u;
      int kb1 = static_cast<int>(kb0 + rem < s.nkb ? kb0 + rem : s.nkb);
      j.seg = g;
      j.feat0 = s.feat_begin + (tile / a.tiles_tok) * FEAT_TILE;
      j.tok0 = (tile % a.tiles_tok) * TOK_TILE;
      j.kb0 = kb0;
      j.kb1 = kb1;
      j.part = -1;
      u += kb1 - kb0;
      return true;
    }
    return false;
  }
};


// Epilogue of one job (warps 2..9): drain this warp's quarter of TMEM lanes
// and column half of the accumulator `acc` into the output described by `a`.
template <int BN, bool SWAP>
__device__ __forceinline__ void epilogue_job(const KArgs& a, const Job& j, uint32_t tmem_base, int acc, int warp,
                                             int lane) {
  const int quarter = warp & 3;              // TMEM lane quarter this warp may access
  const int half = (warp - 2) >> 2;
  const int row = quarter * 32 + lane;       // accumulator row (M index)
  constexpr int HALF_COLS = BN / 2;
  const KSeg& s = a.seg[j.seg];
  const bool has_k = j.kb1 > j.kb0;
#pragma unroll 1
  for (int c0 = half * HALF_COLS; c0 < (half + 1) * HALF_COLS; c0 += 32) {
    uint32_t r[32];
    if (has_k) {
      ptx::tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN + c0, r);
      ptx::tmem_ld_wait();
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = 0u;
    }
    if (SWAP) {
      // row = feature, the 32 columns = consecutive tokens (stride tstride)
      const int f = j.feat0 + row;
      const int tok0 = j.tok0 + c0;
      const int ntok = a.T - tok0;
      if (a.mode == OUT_BF16_RED && a.fixup == FIX_NONE) {
        // bf16x2 reductions: the lane pair (even row, odd row) = two
        // adjacent output columns swaps token halves, so the even lane
        // adds (row, row + 1) for tokens 0-15 and the odd lane for 16-31
        const bool odd = lane & 1;
        const int fe = j.feat0 + (row & ~1);
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float mine_lo = __uint_as_float(r[i]), mine_hi = __uint_as_float(r[i + 16]);
          const float other = __shfl_xor_sync(0xffffffffu, odd ? mine_lo : mine_hi, 1);
          float lo = odd ? other : mine_lo, hi = odd ? mine_hi : other;   // (column fe, column fe + 1)
          if (fe + 1 >= s.write_end) hi = 0.f;
          const __nv_bfloat162 h2 = __floats2bfloat162_rn(lo, hi);
          pk[i] = *reinterpret_cast<const uint32_t*>(&h2);
        }
        const int t0 = odd ? 16 : 0;
        if (fe < s.write_end && ntok > t0) {
          // plain rows: stride ldo; reduce-scatter slabs [P][T][slab]: stride slab (rows per
          // rank and slab offsets are even, so columns fe, fe + 1 stay adjacent)
          const long long tstr = a.scatter_p <= 0 ? a.ldo : a.slab;
          if (a.fan_n > 0 && a.scatter_p > 0) {
            // fused reduce-scatter: the owner's [T][slab] buffer in its window
            const long long loc = fe - s.feat_begin, owner = loc / s.rpr;
            __nv_bfloat16* p = static_cast<__nv_bfloat16*>(a.out) + a.fan_delta[owner] +
                               static_cast<long long>(tok0 + t0) * a.slab + s.slab_off + loc % s.rpr;
#pragma unroll
            for (int i = 0; i < 16; ++i, p += tstr)
              if (t0 + i < ntok) ptx::red_add_bf16x2(p, pk[i]);
          } else {
            __nv_bfloat16* p0 = static_cast<__nv_bfloat16*>(a.out) + out_index(a, s, tok0 + t0, fe);
            // fused all-reduce: two-shot (fan_cols > 0: the column owner's copy only, its
            // finished slab is pushed to the others after a barrier) or one-shot (every
            // rank's copy); fan_n == 0: own buffer
            const bool owner_only = a.fan_n > 0 && a.fan_cols > 0;
            const int nd = a.fan_n > 0 && !owner_only ? a.fan_n : 1;
            for (int dj = 0; dj < nd; ++dj) {
              const long long dlt =
                  a.fan_n == 0 ? 0
                  : owner_only ? a.fan_delta[(s.col_off + (fe - s.feat_begin)) / a.fan_cols] : a.fan_delta[dj];
              __nv_bfloat16* p = p0 + dlt;
#pragma unroll
              for (int i = 0; i < 16; ++i, p += tstr)
                if (t0 + i < ntok) ptx::red_add_bf16x2(p, pk[i]);
            }
          }
        }
      } else if (f < s.write_end && ntok > 0) {
        const bool fx = a.fixup != FIX_NONE;
        const long long tstride = a.scatter_p <= 0 ? (fx ? a.acc_ld : a.ldo) : a.slab;
        const long long base = fx ? acc_index(a, s, tok0, f) : out_index(a, s, tok0, f);
        if (fx || a.mode == OUT_F32_RED) {
          float* p = (fx ? a.acc32 : static_cast<float*>(a.out)) + base;
#pragma unroll
          for (int i = 0; i < 32; ++i, p += tstride)
            if (i < ntok) ptx::red_add_f32(p, __uint_as_float(r[i]));
        } else if (a.mode == OUT_F32_STORE) {
          float* p = static_cast<float*>(a.out) + base;
#pragma unroll
          for (int i = 0; i < 32; ++i, p += tstride)
            if (i < ntok) *p = __uint_as_float(r[i]);
        } else {
          __nv_bfloat16* p = static_cast<__nv_bfloat16*>(a.out) + base;
          const bool accum = a.accumulate != 0;
#pragma unroll
          for (int i0 = 0; i0 < 32; i0 += 8) {
            float old[8];
            __nv_bfloat16* q = p;
#pragma unroll
            for (int i = 0; i < 8; ++i, q += tstride)
              old[i] = (accum && i0 + i < ntok) ? __bfloat162float(*q) : 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i, p += tstride)
              if (i0 + i < ntok) *p = __float2bfloat16_rn(__uint_as_float(r[i0 + i]) + old[i]);
          }
        }
      }
    } else {
      // row = token, columns = features f0 .. f0+31 (same segment, same owner)
      const int tok = j.tok0 + row;
      const int f0 = j.feat0 + c0;
      if (tok < a.T && f0 < s.write_end) {
        const long long idx0 = out_index(a, s, tok, f0);
        const bool full = (f0 + 32 <= s.write_end);
        if (a.mode == OUT_BF16) {
          __nv_bfloat16* o = static_cast<__nv_bfloat16*>(a.out) + idx0;
          if (full && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float v[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(r[q * 8 + e]);
              rope8(a, rope_pos_of(a, tok), f0 + q * 8, v);
              if (a.accumulate) {
                uint4 old = *reinterpret_cast<const uint4*>(o + q * 8);
                const __nv_bfloat162* ob = reinterpret_cast<const __nv_bfloat162*>(&old);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  float2 f2 = __bfloat1622float2(ob[e]);
                  v[2 * e] += f2.x;
                  v[2 * e + 1] += f2.y;
                }
              }
              uint4 pk;
              __nv_bfloat162* pb = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
              for (int e = 0; e < 4; ++e) pb[e] = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
              *reinterpret_cast<uint4*>(o + q * 8) = pk;
            }
          } else {
            const int nf = s.write_end - f0;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              if (i < nf) {
                float w = __uint_as_float(r[i]);
                if (a.accumulate) w += __bfloat162float(o[i]);
                o[i] = __float2bfloat16_rn(w);
              }
            }
          }
        } else {
          float* o = static_cast<float*>(a.out) + idx0;
          const int nf = s.write_end - f0;
          if (a.mode == OUT_F32_RED) {
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              if (i + 4 <= nf) ptx::red_add_v4_f32(o + i, __uint_as_float(r[i]), __uint_as_float(r[i + 1]),
                                                   __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
              else
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  if (i + e < nf) ptx::red_add_f32(o + i + e, __uint_as_float(r[i + e]));
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < nf) o[i] = __uint_as_float(r[i]);
          }
        }
      }
    }
  }
}

// One activation tile of the xform mode (GemmProblem::xform) into the act half
// of a ring slot: BN token rows x 64 k columns, K-major with the 128-byte
// swizzle TMA would have used (16-byte chunk c of row t at chunk c ^ (t & 7)).
// One warp; each lane loads 8 chunks' gate / up rows (all in flight), then
// computes and stores them (the same fp32 expression and bf16 rounding as the
// SiLU kernel it replaces).
template <int BN>
__device__ __forceinline__ void xform_tile(const KArgs& a, uint8_t* dst, int tok0, int k0, int lane) {
  constexpr int CH = BN * 8;   // 16-byte chunks in the tile
  constexpr int PER = 8;       // chunks per lane per batch
#pragma unroll 1
  for (int base = 0; base < CH; base += 32 * PER) {
    uint4 g[PER], u[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int i = base + q * 32 + lane, t = i >> 3, c = i & 7;
      const int tok = tok0 + t, k = k0 + c * 8;
      g[q] = u[q] = make_uint4(0u, 0u, 0u, 0u);
      if (i < CH && tok < a.T && k < a.xcols) {
        const __nv_bfloat16* row = a.xsrc + static_cast<long long>(tok) * a.xld + k;
        u[q] = __ldcg(reinterpret_cast<const uint4*>(row + a.xm));
        if (a.xform == XFORM_SILU) g[q] = __ldcg(reinterpret_cast<const uint4*>(row));
      }
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int i = base + q * 32 + lane, t = i >> 3, c = i & 7;
      if (i >= CH) continue;
      const __nv_bfloat162* gb = reinterpret_cast<const __nv_bfloat162*>(&g[q]);
      const __nv_bfloat162* ub = reinterpret_cast<const __nv_bfloat162*>(&u[q]);
      uint4 o;
      __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 uf = __bfloat1622float2(ub[e]);
        float2 r;
        if (a.xform == XFORM_SILU) {
          const float2 gf = __bfloat1622float2(gb[e]);
          r.x = __fdividef(gf.x, 1.f + __expf(-gf.x)) * uf.x;
          r.y = __fdividef(gf.y, 1.f + __expf(-gf.y)) * uf.y;
        } else {
          r.x = fmaxf(uf.x, 0.f);
          r.y = fmaxf(uf.y, 0.f);
        }
        ob[e] = __floats2bfloat162_rn(r.x, r.y);
      }
      *reinterpret_cast<uint4*>(dst + t * 128 + ((c ^ (t & 7)) << 4)) = o;
    }
  }
}

// A {counter, done} pair is reset for the next launch by the last of the
// grid's CTAs to be finished with c[0]: each calls this once, after its last
// access to c[0] (release: that access is ordered before the done count).
// Called by the producer mid-kernel, so no atomic round trip sits on the
// kernel's exit path (the successor's griddepcontrol.wait waits for it).
__device__ __forceinline__ void release_pair(unsigned int* c) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(c + 1) : "memory");
  if (old == gridDim.x - 1) {
    atomicExch(c, 0u);
    atomicExch(c + 1, 0u);
  }
}

// Shallow (<= 4-stage) swap-AB configurations are register-capped for two
// CTAs per SM, so a successor GEMM's CTA can become resident (and prefetch
// its weights) while this one still runs.
//
// CHAIN (swap-AB stream-K only): the fused two-stage chain of one factor group
// in ONE persistent launch (y = A(Bx)).  Phase 0 is stage 1
// (maps / a: Z = X.B^T, bf16x2 partials reduced into the L2-resident Z
// buffer), phase 1 is stage 2 (maps2 / a2: Y = Z.A_g^T reading that Z).  The
// producer streams phase-1 weight tiles into the ring while phase 0 is still
// being reduced; only their Z halves wait, on a grid-wide arrival counter
// (chain[0] = CTAs whose phase-0 epilogue has retired, released by each CTA
// after its last phase-0 red.add) instead of a kernel boundary.  All CTAs are
// co-resident (one wave), so the in-kernel wait cannot deadlock.
template <int BN, bool SWAP, int STAGES, bool CHAIN>
__global__ void __launch_bounds__(kThreads, (SWAP && STAGES <= 4) ? 2 : 1)
    tc_gemm_kernel(const __grid_constant__ KMaps maps, const __grid_constant__ KArgs a,
                   const __grid_constant__ KMaps maps2, const __grid_constant__ KArgs a2, unsigned int* chain) {
  constexpr int P_ROWS = BM;                 // MMA A operand rows
  constexpr int Q_ROWS = BN;                 // MMA B operand rows
  constexpr int P_BYTES = P_ROWS * BK * 2;
  constexpr int Q_BYTES = Q_ROWS * BK * 2;
  constexpr int STAGE_BYTES = P_BYTES + Q_BYTES;
  constexpr int FEAT_TILE = SWAP ? BM : BN;
  constexpr int TOK_TILE = SWAP ? BN : BM;
  constexpr uint32_t TMEM_COLS = 2 * BN;
  constexpr uint32_t IDESC = ptx::idesc_bf16_f32(BM, BN);
  constexpr int kPhaseMark = -2;             // job-ring marker: end of phase 0 (CHAIN)

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t accf_bar[2];
  __shared__ __align__(8) uint64_t acce_bar[2];
  __shared__ __align__(8) uint64_t jfull_bar[kJobRing];
  __shared__ __align__(8) uint64_t jempty_bar[kJobRing];
  __shared__ Job jobs[kJobRing];
  __shared__ int fix_last;
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  // debug timeline (dl_debug_gemm_trace); a chain launch traces its stage 2
  // in a second slot whose "entry" is the release of the in-kernel wait
  unsigned long long* tr = (g_trace && a.trace_slot >= 0) ? g_trace + (static_cast<long long>(a.trace_slot) * 148 + blockIdx.x) * 8 : nullptr;
  unsigned long long* tr2 = (CHAIN && g_trace && a2.trace_slot >= 0) ? g_trace + (static_cast<long long>(a2.trace_slot) * 148 + blockIdx.x) * 8 : nullptr;
  if (tr && threadIdx.x == 0) { tr[0] = gtime(); tr[7] = smid(); }
  if (tr2 && threadIdx.x == 0) { tr2[1] = gtime(); tr2[7] = smid(); }

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&maps.act);
    for (int g = 0; g < a.nseg; ++g) ptx::prefetch_tmap(&maps.w[g]);
    if (CHAIN) {
      ptx::prefetch_tmap(&maps2.act);
      for (int g = 0; g < a2.nseg; ++g) ptx::prefetch_tmap(&maps2.w[g]);
    }
    for (int s = 0; s < STAGES; ++s) {
      // xform: the producer's weight bytes and one epilogue warp's activation tile
      ptx::mbar_init(&full_bar[s], (SWAP && a.xform) ? 2 : 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&accf_bar[b], 1);
      ptx::mbar_init(&acce_bar[b], 8);
    }
    for (int b = 0; b < kJobRing; ++b) {
      ptx::mbar_init(&jfull_bar[b], 1);
      ptx::mbar_init(&jempty_bar[b], 8);   // released by the 8 epilogue warps
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(&tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = tmem_slot;
  if (tr && threadIdx.x == 0) tr[1] = gtime();

  pdl_trigger();   // let the next kernel launch and prefetch its own weights early
  Job j;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const uint64_t pol_w = ptx::policy_evict_first();   // weights: streamed once
      const uint64_t pol_a = ptx::policy_evict_last();    // activations: re-read
      int stage = 0;
      uint32_t phase = 0;
      int jslot = 0;
      uint32_t jphase = 0;
      // One phase of work (the whole kernel unless CHAIN).  The static weight
      // tiles of the phase's first STAGES units are requested before its
      // dependency wait (phase 0: griddepcontrol.wait on the predecessor kernel;
      // phase 1: the grid-wide stage-1 arrival counter); their activation
      // halves follow once the dependency is met.
      auto run_phase = [&](const KArgs& A, const KMaps& M, int ph) {
        unsigned long long* tp = ph ? tr2 : tr;
        if (tp) tp[2] = gtime();
        JobIter it(A, blockIdx.x, gridDim.x);
        int u = 0, njobs = 0;
        bool waited = false;
        int pend_c0[STAGES], pend_c1[STAGES], pend_st[STAGES];
        // Before waiting on the predecessor, also pull the weight tiles of the
        // next kL2Prefetch units (beyond the STAGES staged in smem) into L2, so
        // the dependency gap is spent streaming HBM instead of idling.
        JobIter pf_it = it;
        if (A.stream_k && A.sched)
          pf_it.set_range(blockIdx.x * A.static_units, (blockIdx.x + 1) * A.static_units);
        auto l2_prefetch = [&]() {
          int skipped = 0, issued = 0;
          Job pj;
          while (issued < A.l2pf && pf_it.next(pj, FEAT_TILE, TOK_TILE)) {
            const KSeg& ps = A.seg[pj.seg];
            for (int kb = pj.kb0; kb < pj.kb1 && issued < A.l2pf; ++kb) {
              if (skipped < STAGES) { ++skipped; continue; }   // these go to smem
              ptx::tma_prefetch_2d(&M.w[pj.seg], kb * BK, pj.feat0 - ps.feat_begin);
              ++issued;
            }
          }
        };
        auto act_load = [&](void* dst, uint64_t* bar, int c, int tok) {
          if (A.act_w > 0) ptx::tma_load_3d(dst, &M.act, bar, c % A.act_w, tok, c / A.act_w, pol_a);
          else ptx::tma_load_2d(dst, &M.act, bar, c, tok, pol_a);
        };
        auto flush_pending = [&]() {
          if (ph == 0) {
            if (SWAP) l2_prefetch();
            pdl_wait();
          } else {
            // stage 2 reads Z: every CTA's stage-1 partials must have landed
            const unsigned need = gridDim.x * (A.chain_warp ? 8u : 1u);
            for (;;) {
              unsigned v;
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(chain) : "memory");
              if (v >= need) break;
              __nanosleep(32);
            }
            // generic-proxy writes (the red.adds) before async-proxy (TMA) reads
            asm volatile("fence.proxy.async.global;" ::: "memory");
            if (tp) tp[0] = gtime();
            release_pair(chain);
          }
          waited = true;
          for (int i = 0; i < u && i < STAGES && !A.xform; ++i) {
            uint8_t* dst = smem + pend_st[i] * STAGE_BYTES + (SWAP ? P_BYTES : 0);
            act_load(dst, &full_bar[pend_st[i]], pend_c0[i], pend_c1[i]);
          }
        };
        auto push = [&](const Job& jb) {
          // The ring slot frees only when the epilogue has finished the job that
          // held it, which needs that job's deferred activation loads: issue them
          // before the first push that may wait (more than kJobRing jobs -- e.g.
          // single-k-block tiles -- within the first STAGES units would otherwise
          // deadlock the producer against its own deferred loads).
          if (!waited && njobs >= kJobRing) flush_pending();
          ++njobs;
          ptx::mbar_wait(&jempty_bar[jslot], jphase ^ 1);
          jobs[jslot] = jb;
          ptx::mbar_arrive(&jfull_bar[jslot]);
          if (++jslot == kJobRing) { jslot = 0; jphase ^= 1; }
        };
        auto emit = [&](Job jb) {
          jb.ph = ph;
          push(jb);
          const KSeg& s = A.seg[jb.seg];
          const int pf_limit = ph && A.chain_pf < STAGES ? A.chain_pf : STAGES;
          for (int kb = jb.kb0; kb < jb.kb1; ++kb, ++u) {
            if (u >= pf_limit && !waited) flush_pending();
            ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
            uint8_t* sp = smem + stage * STAGE_BYTES;
            uint8_t* sq = sp + P_BYTES;
            ptx::mbar_arrive_expect_tx(&full_bar[stage], (SWAP && A.xform) ? P_BYTES : STAGE_BYTES);
            const int kx = kb * BK;
            uint8_t* sw = SWAP ? sp : sq;
            uint8_t* sa = SWAP ? sq : sp;
            ptx::tma_load_2d(sw, &M.w[jb.seg], &full_bar[stage], kx, jb.feat0 - s.feat_begin, pol_w);
            if (SWAP && A.xform) {
              // the activation half is written by an epilogue warp (xform_tile)
            } else if (waited) {
              act_load(sa, &full_bar[stage], s.act_koff + kx, jb.tok0);
            } else {
              pend_c0[u] = s.act_koff + kx;
              pend_c1[u] = jb.tok0;
              pend_st[u] = stage;
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        };
        if (A.stream_k && A.sched) {
          it.set_range(blockIdx.x * A.static_units, (blockIdx.x + 1) * A.static_units);
          while (it.next(j, FEAT_TILE, TOK_TILE)) emit(j);
          for (;;) {   // dynamic tail: fast SMs take more pieces
            // the counter pairs rotate over launches: touch one only after every
            // earlier kernel has completed (griddepcontrol.wait is transitive)
            if (ph == 0 && !waited) flush_pending();
            const long long g = A.dyn_begin + static_cast<long long>(atomicAdd(A.sched, static_cast<unsigned>(A.chunk)));
            if (g >= A.total_units) {
              release_pair(A.sched);
              break;
            }
            it.set_range(g, g + A.chunk < A.total_units ? g + A.chunk : A.total_units);
            while (it.next(j, FEAT_TILE, TOK_TILE)) emit(j);
          }
        } else {
          while (it.next(j, FEAT_TILE, TOK_TILE)) emit(j);
        }
        Job end;
        end.seg = (CHAIN && ph == 0) ? kPhaseMark : -1;
        end.ph = ph;
        push(end);
        // phase 1: every CTA passes the chain wait once (it resets the counter)
        if (!waited && (ph == 0 || u > 0 || CHAIN)) flush_pending();
      };
      run_phase(a, maps, 0);
      if (CHAIN) run_phase(a2, maps2, 1);
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread) =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int jslot = 0;
      uint32_t jphase = 0;
      for (;;) {
        ptx::mbar_wait(&jfull_bar[jslot], jphase);
        j = jobs[jslot];
        if (++jslot == kJobRing) { jslot = 0; jphase ^= 1; }
        if (j.seg == kPhaseMark) {
          if (tr) tr[4] = gtime();
          continue;
        }
        if (j.seg < 0) break;
        unsigned long long* tj = (CHAIN && j.ph) ? tr2 : tr;
        ptx::mbar_wait(&acce_bar[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = j.kb0; kb < j.kb1; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          if (tj && tj[3] == 0) tj[3] = gtime();
          ptx::tc_fence_after();
          const uint32_t sp = ptx::smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sq = sp + P_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // advance 16 bf16 = 32 B along K inside the 128 B swizzle row
            const uint64_t ad = ptx::sdesc_sw128(sp + k * 32);
            const uint64_t bd = ptx::sdesc_sw128(sq + k * 32);
            ptx::umma_bf16(d_tmem, ad, bd, IDESC, (kb > j.kb0 || k > 0) ? 1u : 0u);
          }
          ptx::umma_commit(&empty_bar[stage]);   // smem slot free once these MMAs retire
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        ptx::umma_commit(&accf_bar[acc]);        // accumulator ready for the epilogue
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      if (CHAIN ? tr2 : tr) (CHAIN ? tr2 : tr)[4] = gtime();
    }
  } else {
    // ===================== epilogue (warps 2..9) =====================
    // 8 warps = 2 per SM sub-partition so the per-element store latency of
    // one warp hides behind the other; warp e handles TMEM lane quarter
    // (warp & 3) and column half (e / 4) of the accumulator.
    pdl_wait();                                // outputs may alias a predecessor's buffers
    int acc = 0;
    uint32_t acc_phase = 0;
    int jslot = 0;
    uint32_t jphase = 0;
    if (SWAP && !CHAIN && a.xform) {
      // The activation operand is computed here (GemmProblem::xform): for every
      // unit of a job, epilogue warp (unit % 8) waits for the ring slot, writes
      // the activation tile act[tok][k] = silu(gate) * up (or relu(up)) from the
      // reduced gate|up rows into the slot's swizzled act half and arrives on its
      // full barrier next to the producer's weight bytes.  Each job's accumulator
      // epilogue runs after the NEXT job's tiles are out, so the MMA never waits
      // for an epilogue to get its activations.
      const int ew = warp - 2;
      int xs = 0, xu = 0;
      uint32_t xph = 0;
      Job prev{};
      int prev_slot = -1;
      auto epilogue_of = [&](const Job& jb, int slot) {
        ptx::mbar_wait(&accf_bar[acc], acc_phase);
        ptx::tc_fence_after();
        epilogue_job<BN, SWAP>(a, jb, tmem_base, acc, warp, lane);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (a.relaxed_acce) ptx::mbar_arrive_relaxed(&acce_bar[acc]);
          else ptx::mbar_arrive(&acce_bar[acc]);
          ptx::mbar_arrive(&jempty_bar[slot]);
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      };
      for (;;) {
        ptx::mbar_wait(&jfull_bar[jslot], jphase);
        j = jobs[jslot];
        const int my_slot = jslot;
        if (++jslot == kJobRing) { jslot = 0; jphase ^= 1; }
        if (j.seg < 0) break;
        const KSeg& s = a.seg[j.seg];
        for (int kb = j.kb0; kb < j.kb1; ++kb) {
          if ((xu & 7) == ew) {
            ptx::mbar_wait(&empty_bar[xs], xph ^ 1);
            xform_tile<BN>(a, smem + xs * STAGE_BYTES + P_BYTES, j.tok0, s.act_koff + kb * BK, lane);
            ptx::fence_async_smem();   // generic stores before the MMA's async-proxy reads
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&full_bar[xs]);
          }
          ++xu;
          if (++xs == STAGES) { xs = 0; xph ^= 1; }
        }
        if (prev_slot >= 0) epilogue_of(prev, prev_slot);
        prev = j;
        prev_slot = my_slot;
      }
      if (prev_slot >= 0) epilogue_of(prev, prev_slot);
    } else
    for (;;) {
      ptx::mbar_wait(&jfull_bar[jslot], jphase);
      j = jobs[jslot];
      const int my_slot = jslot;
      if (++jslot == kJobRing) { jslot = 0; jphase ^= 1; }
      if (j.seg == kPhaseMark) {
        // every epilogue warp has retired its phase-0 (stage-1) reductions:
        // publish this CTA's arrival (bar.sync + one thread's release, the
        // grid-barrier pattern; the fence is cumulative over the CTA's stores)
        if (a2.chain_warp) {
          __syncwarp();
          if (lane == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(chain) : "memory");
        } else {
          epi_bar();
          if (threadIdx.x == 64)
            asm volatile("fence.acq_rel.gpu;\n\tred.release.gpu.global.add.u32 [%0], 1;" :: "l"(chain) : "memory");
        }
        if (tr && threadIdx.x == 64) tr[6] = gtime();
        if (lane == 0) ptx::mbar_arrive(&jempty_bar[my_slot]);
        continue;
      }
      if (j.seg < 0) break;
      ptx::mbar_wait(&accf_bar[acc], acc_phase);
      if (warp == 2 && lane == 0) {   // accumulator of this job ready
        unsigned long long* tj = (CHAIN && j.ph) ? tr2 : tr;
        if (tj) tj[5] = gtime();
      }
      ptx::tc_fence_after();
      if (CHAIN && j.ph) epilogue_job<BN, SWAP>(a2, j, tmem_base, acc, warp, lane);
      else epilogue_job<BN, SWAP>(a, j, tmem_base, acc, warp, lane);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (a.relaxed_acce) ptx::mbar_arrive_relaxed(&acce_bar[acc]);
        else ptx::mbar_arrive(&acce_bar[acc]);
        ptx::mbar_arrive(&jempty_bar[my_slot]);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      if (SWAP) {
        if (CHAIN && j.ph) { if (a2.fixup != FIX_NONE) fixup_tile(a2, j, threadIdx.x - 64, fix_last); }
        else if (a.fixup != FIX_NONE) fixup_tile(a, j, threadIdx.x - 64, fix_last);
      }
    }
    if (warp == 2 && lane == 0 && (CHAIN ? tr2 : tr)) (CHAIN ? tr2 : tr)[6] = gtime();   // epilogue done
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc<TMEM_COLS>(tmem_base);
}


// ---------------------------------------------------------------------------
// CTA-pair prefill kernel (cta_group::2): a cluster of 2 CTAs computes a
// 256-token x 256-feature tile with M=256, N=256 MMAs issued by the leader.
// Each CTA stages only its own 128 token rows and 128 weight rows per
// k-block (32 KB / stage), halving per-SM shared-memory operand traffic
// relative to the 1-CTA 128x256 tile.  Whole tiles, bf16 (+ fused residual)
// epilogue; every CTA drains its own TMEM half (its 128 token rows).
// ---------------------------------------------------------------------------
template <int STAGES, bool GLU = false>   // GLU: KArgs::glu launches (gate|up pairs, SiLU.up epilogue)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    tc_gemm_pair_kernel(const __grid_constant__ KMaps maps, const __grid_constant__ KArgs a,
                        const __grid_constant__ KMaps, const __grid_constant__ KArgs, unsigned int*) {
  constexpr int HALF = 128;                       // rows per CTA of both operands
  constexpr int TILE = 256;                       // cluster tile (tokens and features)
  constexpr int A_BYTES = HALF * BK * 2;
  constexpr int STAGE_BYTES = 2 * A_BYTES;        // own A half + own B half
  constexpr uint32_t TMEM_COLS = 2 * TILE;        // double-buffered 256-column accumulator
  constexpr uint32_t IDESC = ptx::idesc_bf16_f32(256, TILE);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t accf_bar[2];
  __shared__ __align__(8) uint64_t acce_bar[2];
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  unsigned long long* tr = (g_trace && a.trace_slot >= 0 && blockIdx.x < 148)
                               ? g_trace + (static_cast<long long>(a.trace_slot) * 148 + blockIdx.x) * 8
                               : nullptr;   // debug timeline: [0] entry, [6] epilogue done
  if (tr && threadIdx.x == 0) { tr[0] = gtime(); tr[7] = smid(); }

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&maps.act);
    for (int g = 0; g < a.nseg; ++g) ptx::prefetch_tmap(&maps.w[g]);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&accf_bar[b], 1);
      ptx::mbar_init(&acce_bar[b], 16);           // 8 epilogue warps x 2 CTAs
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc_pair<TMEM_COLS>(&tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = tmem_slot;

  pdl_trigger();
  JobIter it(a, blockIdx.x / 2, gridDim.x / 2);
  Job j;

  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if (lane == 0) {
      // weights: every feature tile is read by all T/256 token tiles of the
      // cluster schedule, so they are kept in L2 (evict_first -- right for the
      // decode stream -- made the prefill gate|up GEMM read 1.69x its bytes)
      const uint64_t pol_w = a.wpol == 0 ? ptx::policy_evict_first()
                             : a.wpol == 1 ? ptx::policy_evict_normal() : ptx::policy_evict_last();
      const uint64_t pol_a = ptx::policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      int u = 0;
      bool waited = false;
      int pend_c0[STAGES], pend_c1[STAGES];
      auto flush_pending = [&]() {
        pdl_wait();
        waited = true;
        for (int i = 0; i < u && i < STAGES; ++i)
          ptx::tma_load_2d_pair(smem + i * STAGE_BYTES, &maps.act, &full_bar[i], pend_c0[i], pend_c1[i], pol_a);
      };
      while (it.next(j, TILE, TILE)) {
        const KSeg& s = a.seg[j.seg];
        for (int kb = j.kb0; kb < j.kb1; ++kb, ++u) {
          if (u >= STAGES && !waited) flush_pending();
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sw = sa + A_BYTES;
          if (leader) ptx::mbar_arrive_expect_tx(&full_bar[stage], 2 * STAGE_BYTES);
          const int kx = kb * BK;
          ptx::tma_load_2d_pair(sw, &maps.w[j.seg], &full_bar[stage], kx,
                                j.feat0 - s.feat_begin + static_cast<int>(rank) * HALF, pol_w);
          if (waited) {
            ptx::tma_load_2d_pair(sa, &maps.act, &full_bar[stage], s.act_koff + kx,
                                  j.tok0 + static_cast<int>(rank) * HALF, pol_a);
          } else {
            pend_c0[u] = s.act_koff + kx;
            pend_c1[u] = j.tok0 + static_cast<int>(rank) * HALF;
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
      if (!waited) flush_pending();
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA, one thread) =====================
    if (leader && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      while (it.next(j, TILE, TILE)) {
        ptx::mbar_wait(&acce_bar[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * TILE;
        for (int kb = j.kb0; kb < j.kb1; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sw = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            ptx::umma_bf16_pair(d_tmem, ptx::sdesc_sw128(sa + k * 32), ptx::sdesc_sw128(sw + k * 32), IDESC,
                                (kb > j.kb0 || k > 0) ? 1u : 0u);
          ptx::umma_commit_pair(&empty_bar[stage], 0x3);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        ptx::umma_commit_pair(&accf_bar[acc], 0x3);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ===================== epilogue (warps 2..9, both CTAs) =====================
    pdl_wait();
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;          // this CTA's token row within its half
    const uint32_t acce0 = ptx::mapa(ptx::smem_u32(&acce_bar[0]), 0);
    uint8_t* stg = smem + STAGES * STAGE_BYTES + (warp - 2) * kStageOutWarp;   // this warp's store staging
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t gpk[64];   // GLU: silu(gate) of this thread's row, 128 columns as bf16 pairs
    while (it.next(j, TILE, TILE)) {
      const KSeg& s = a.seg[j.seg];
      const int tok = j.tok0 + static_cast<int>(rank) * HALF + row;
      const float rpos = rope_pos_of(a, tok);   // issued before the accumulator wait
      ptx::mbar_wait(&accf_bar[acc], acc_phase);
      ptx::tc_fence_after();
      const bool has_k = j.kb1 > j.kb0;
      const uint32_t tacc = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * TILE + half * 128;
      if (GLU && j.part < 0 && j.seg == 0) {
        // gate job: keep silu(gate) in registers, release the accumulator at once
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t r[32];
          ptx::tmem_ld32(tacc + c * 32, r);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e)
            gpk[c * 16 + e] = pack_bf16(silu_tanh_f(__uint_as_float(r[2 * e])), silu_tanh_f(__uint_as_float(r[2 * e + 1])));
        }
      } else if (GLU && j.part < 0) {
        // up job: act = silu(gate) * up, staged through the per-warp transpose
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(a.out);
        const int fg = j.feat0 - a.seg[1].feat_begin + half * 128;   // gate feature of column 0 of this warp
        const uint64_t spol = ptx::policy_evict_last();
        uint4* sw = reinterpret_cast<uint4*>(stg);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t r[32];
          ptx::tmem_ld32(tacc + c * 32, r);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 pk;
            uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int i0 = q * 8 + 2 * e;
              const float2 g2 = unpack_bf16(gpk[c * 16 + q * 4 + e]);
              pw[e] = pack_bf16(g2.x * __uint_as_float(r[i0]), g2.y * __uint_as_float(r[i0 + 1]));
            }
            sw[lane * 4 + (q ^ ((lane >> 1) & 3))] = pk;
          }
          __syncwarp();
          const int cc = lane & 3;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int rr = 8 * q + (lane >> 2);
            const uint4 val = sw[rr * 4 + (cc ^ ((rr >> 1) & 3))];
            const int t2 = j.tok0 + static_cast<int>(rank) * HALF + quarter * 32 + rr;
            if (t2 < a.T) {
              uint4* dst = reinterpret_cast<uint4*>(out + static_cast<long long>(t2) * a.ldo + fg + c * 32 + cc * 8);
              if (a.glu_spol)
                asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(dst), "r"(val.x),
                             "r"(val.y), "r"(val.z), "r"(val.w), "l"(spol)
                             : "memory");
              else
                *dst = val;
            }
          }
          __syncwarp();
        }
      } else
#pragma unroll 1
      for (int c0 = half * 128; c0 < (half + 1) * 128; c0 += 32) {
        uint32_t r[32];
        if (has_k) {
          ptx::tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * TILE + c0, r);
          ptx::tmem_ld_wait();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = 0u;
        }
        const int f0 = j.feat0 + c0;
        if (j.part >= 0) {
          // K-split tail piece: fp32 partial of tile row (rank*128 + row), columns c0..c0+31
          if (has_k) {
            float* pt = a.tail_acc + (static_cast<long long>(j.part) * TILE + rank * HALF + row) * TILE + c0;
#pragma unroll
            for (int q = 0; q < 32; q += 4)
              ptx::red_add_v4_f32(pt + q, __uint_as_float(r[q]), __uint_as_float(r[q + 1]), __uint_as_float(r[q + 2]),
                                  __uint_as_float(r[q + 3]));
          }
        } else if ((a.stage_out & 1) && !a.accumulate && f0 + 32 <= s.write_end &&
                   __all_sync(0xffffffffu, tok >= a.T || ((reinterpret_cast<uintptr_t>(static_cast<__nv_bfloat16*>(a.out) +
                                                                                     out_index(a, s, tok, f0)) & 15) == 0))) {
          // Coalesced store through a per-warp 2 KB shared-memory transpose: the
          // accumulator gives each lane one token row (32 features = 64 B), so a
          // direct store writes 32 half-sectors per instruction.  Staged, each
          // instruction writes 8 rows x 64 B (whole sectors).  16-byte units are
          // XOR-swizzled by row so both the writes and the reads are conflict-free.
          uint4* sw = reinterpret_cast<uint4*>(stg);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(r[q * 8 + e]);
            rope8(a, rpos, f0 + q * 8, v);
            uint4 pk;
            __nv_bfloat162* pb = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
            for (int e = 0; e < 4; ++e) pb[e] = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
            sw[lane * 4 + (q ^ ((lane >> 1) & 3))] = pk;
          }
          __syncwarp();
          const int c = lane & 3;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int rr = 8 * q + (lane >> 2);
            const uint4 val = sw[rr * 4 + (c ^ ((rr >> 1) & 3))];
            const int t2 = j.tok0 + static_cast<int>(rank) * HALF + quarter * 32 + rr;
            if (t2 < a.T)
              *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.out) + out_index(a, s, t2, f0) + c * 8) = val;
          }
          __syncwarp();   // the next column block reuses the staging buffer
        } else if ((a.stage_out & 2) && a.accumulate && f0 + 32 <= s.write_end &&
                   __all_sync(0xffffffffu, tok >= a.T || ((reinterpret_cast<uintptr_t>(static_cast<__nv_bfloat16*>(a.out) +
                                                                                     out_index(a, s, tok, f0)) & 15) == 0))) {
          // Same transpose for Y += result (the residual-fused stage 2): fp32
          // staging in two 16-column halves, so the old value is added before
          // the one bf16 rounding, exactly as on the direct path.
          float vv[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) vv[i] = __uint_as_float(r[i]);
#pragma unroll
          for (int q = 0; q < 4; ++q) rope8(a, rpos, f0 + q * 8, vv + q * 8);
          float4* sw = reinterpret_cast<float4*>(stg);
          const int c = lane & 3;
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              sw[lane * 4 + (q ^ ((lane >> 1) & 3))] =
                  make_float4(vv[h2 * 16 + q * 4], vv[h2 * 16 + q * 4 + 1], vv[h2 * 16 + q * 4 + 2], vv[h2 * 16 + q * 4 + 3]);
            __syncwarp();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int rr = 8 * q + (lane >> 2);
              const float4 val = sw[rr * 4 + (c ^ ((rr >> 1) & 3))];
              const int t2 = j.tok0 + static_cast<int>(rank) * HALF + quarter * 32 + rr;
              if (t2 < a.T) {
                uint2* o2 = reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(a.out) + out_index(a, s, t2, f0) +
                                                     h2 * 16 + c * 4);
                const uint2 old = *o2;
                const float2 a0 = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(&old)[0]);
                const float2 a1 = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(&old)[1]);
                uint2 pk;
                reinterpret_cast<__nv_bfloat162*>(&pk)[0] = __floats2bfloat162_rn(val.x + a0.x, val.y + a0.y);
                reinterpret_cast<__nv_bfloat162*>(&pk)[1] = __floats2bfloat162_rn(val.z + a1.x, val.w + a1.y);
                *o2 = pk;
              }
            }
            __syncwarp();
          }
        } else if (tok < a.T && f0 < s.write_end) {
          __nv_bfloat16* o = static_cast<__nv_bfloat16*>(a.out) + out_index(a, s, tok, f0);
          if (f0 + 32 <= s.write_end && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float v[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(r[q * 8 + e]);
              rope8(a, rpos, f0 + q * 8, v);
              if (a.accumulate) {
                uint4 old = *reinterpret_cast<const uint4*>(o + q * 8);
                const __nv_bfloat162* ob = reinterpret_cast<const __nv_bfloat162*>(&old);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  float2 f2 = __bfloat1622float2(ob[e]);
                  v[2 * e] += f2.x;
                  v[2 * e + 1] += f2.y;
                }
              }
              uint4 pk;
              __nv_bfloat162* pb = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
              for (int e = 0; e < 4; ++e) pb[e] = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
              *reinterpret_cast<uint4*>(o + q * 8) = pk;
            }
          } else {
            const int nf = s.write_end - f0;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < nf) {
                float w = __uint_as_float(r[i]);
                if (a.accumulate) w += __bfloat162float(o[i]);
                o[i] = __float2bfloat16_rn(w);
              }
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {   // leader's acce_bar[acc]
        if (a.relaxed_acce) ptx::mbar_arrive_cluster_relaxed(acce0 + acc * 8);
        else ptx::mbar_arrive_cluster(acce0 + acc * 8);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  if (tr && warp == 2 && lane == 0) tr[6] = gtime();
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc_pair<TMEM_COLS>(tmem_base);
}

// DP + stream-K tail finalize: grid (tail tiles, 8 row blocks of 32 token rows),
// 256 threads = 64 float4 column groups x 4 row lanes; each thread issues its
// 8 float4 loads before using them.  out = bf16(sum of K-pieces (+ out));
// scratch cleared.  ~100 CTAs: one resident wave, so the next GEMM launches early.
__global__ void __launch_bounds__(256) tc_tail_finalize_kernel(KArgs a) {
  pdl_trigger();
  pdl_wait();
  const int tt = blockIdx.x, rb = blockIdx.y;
  const int t = a.dp_tiles + tt;
  int g = 0;
  while (g + 1 < a.nseg && t >= a.seg[g + 1].tile_first) ++g;
  const KSeg& s = a.seg[g];
  const int local = t - s.tile_first;
  const int feat0 = s.feat_begin + (local / a.tiles_tok) * 256;
  const int tok0 = (local % a.tiles_tok) * 256 + rb * 32;
  const int c4 = (threadIdx.x & 63) * 4, lane_r = threadIdx.x >> 6;
  const int f = feat0 + c4;
  float4 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = rb * 32 + lane_r + 4 * i;
    v[i] = __ldcg(reinterpret_cast<const float4*>(a.tail_acc + (static_cast<long long>(tt) * 256 + r) * 256 + c4));
  }
  // 4 features per thread go out as one 8-byte store when they are whole and
  // aligned; for Y += the old values of all 8 rows are loaded up front (one
  // round trip instead of 8 dependent ones)
  const bool vec = a.tail_vec && f + 4 <= s.write_end;
  uint2 old[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    old[i] = make_uint2(0u, 0u);
    const int tok = tok0 + lane_r + 4 * i;
    if (a.accumulate && vec && tok < a.T) {
      const __nv_bfloat16* o = static_cast<const __nv_bfloat16*>(a.out) + out_index(a, s, tok, f);
      if ((reinterpret_cast<uintptr_t>(o) & 7) == 0) old[i] = *reinterpret_cast<const uint2*>(o);
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = rb * 32 + lane_r + 4 * i;
    *reinterpret_cast<float4*>(a.tail_acc + (static_cast<long long>(tt) * 256 + r) * 256 + c4) =
        make_float4(0.f, 0.f, 0.f, 0.f);
    const int tok = tok0 + lane_r + 4 * i;
    if (tok >= a.T) continue;
    float vv[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
    if (a.rope_pos != nullptr && f < a.rope_end) {
      // the epilogue RoPE of the whole tiles (rope8), on the summed K-pieces
      const float pos = static_cast<float>(a.rope_pos[tok]);
#pragma unroll
      for (int e = 0; e < 4; e += 2) {
        const int dim = (f + e) & 127;
        float sn, cs;
        rope_sincos(pos * exp2f(-a.rope_l2t * static_cast<float>(dim) / 128.f), &sn, &cs);
        const float x = vv[e], y = vv[e + 1];
        vv[e] = x * cs - y * sn;
        vv[e + 1] = x * sn + y * cs;
      }
    }
    __nv_bfloat16* o4 = static_cast<__nv_bfloat16*>(a.out) + out_index(a, s, tok, f);
    if (vec && (reinterpret_cast<uintptr_t>(o4) & 7) == 0) {
      if (a.accumulate) {
        const float2 o01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&old[i].x));
        const float2 o23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&old[i].y));
        vv[0] += o01.x;
        vv[1] += o01.y;
        vv[2] += o23.x;
        vv[3] += o23.y;
      }
      __nv_bfloat162 p01 = __floats2bfloat162_rn(vv[0], vv[1]), p23 = __floats2bfloat162_rn(vv[2], vv[3]);
      *reinterpret_cast<uint2*>(o4) =
          make_uint2(*reinterpret_cast<uint32_t*>(&p01), *reinterpret_cast<uint32_t*>(&p23));
      continue;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (f + e >= s.write_end) break;
      __nv_bfloat16* o = static_cast<__nv_bfloat16*>(a.out) + out_index(a, s, tok, f + e);
      *o = __float2bfloat16_rn(a.accumulate ? vv[e] + __bfloat162float(*o) : vv[e]);
    }
  }
}

// GLU mode: tail pair tt has the gate partial sums in tail_acc slot 2 tt and the
// up ones in slot 2 tt + 1 (gate features seg[0].feat_begin + f, f in the
// pair's 256-feature tile); out = bf16(silu(gate) * up) [T x m], both slots
// cleared.  256 threads = 64 float4 column groups x 4 row lanes, 8 rows each.
__global__ void __launch_bounds__(256) tc_tail_finalize_glu_kernel(KArgs a) {
  pdl_trigger();
  pdl_wait();
  const int tt = blockIdx.x, rb = blockIdx.y;
  const int local = a.dp_tiles + tt;   // pair index = gate tile index
  const int f0 = (local / a.tiles_tok) * 256;
  const int tok0 = (local % a.tiles_tok) * 256 + rb * 32;
  const int c4 = (threadIdx.x & 63) * 4, lane_r = threadIdx.x >> 6;
  float* gs = a.tail_acc + static_cast<long long>(2 * tt) * 256 * 256;
  float* us = gs + 256 * 256;
#pragma unroll 2
  for (int i = 0; i < 8; ++i) {
    const int r = rb * 32 + lane_r + 4 * i;
    const float4 g = __ldcg(reinterpret_cast<const float4*>(gs + r * 256 + c4));
    const float4 u = __ldcg(reinterpret_cast<const float4*>(us + r * 256 + c4));
    *reinterpret_cast<float4*>(gs + r * 256 + c4) = make_float4(0.f, 0.f, 0.f, 0.f);
    *reinterpret_cast<float4*>(us + r * 256 + c4) = make_float4(0.f, 0.f, 0.f, 0.f);
    const int tok = tok0 + lane_r + 4 * i;
    if (tok >= a.T) continue;
    uint2 pk;
    pk.x = pack_bf16(silu_tanh_f(g.x) * u.x, silu_tanh_f(g.y) * u.y);
    pk.y = pack_bf16(silu_tanh_f(g.z) * u.z, silu_tanh_f(g.w) * u.w);
    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(a.out) + static_cast<long long>(tok) * a.ldo + f0 + c4) = pk;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

bool get_encode() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

// 2-D bf16 map over a row-major [rows x cols] matrix (ld elements), box
// {64 cols, box_rows}, 128B swizzle, OOB elements read as zero.
bool make_map(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// CTAs per SM of the shallow (<= 4-stage) swap-AB configurations: 2 fills the
// SM; 1 leaves room for the successor's CTA to become resident early (A/B knob)
int small_per_sm() {
  static const int v = DL_ENV("DL_DECODE_PER_SM") ? atoi(DL_ENV("DL_DECODE_PER_SM")) : 2;
  return v == 1 ? 1 : 2;
}

template <int BN, bool SWAP, int STAGES, bool PAIR>
struct Cfg {
  // PAIR: cta_group::2 kernel, cluster tile 256 tokens x 256 features, each CTA
  // loads 128-row boxes of both operands.
  static constexpr int FEAT_TILE = PAIR ? 256 : (SWAP ? BM : BN);
  static constexpr int TOK_TILE = PAIR ? 256 : (SWAP ? BN : BM);
  static constexpr int BOX_W = PAIR ? 128 : FEAT_TILE;
  static constexpr int BOX_A = PAIR ? 128 : TOK_TILE;
  static constexpr int SMEM =
      PAIR ? STAGES * 2 * 128 * BK * 2 + 8 * kStageOutWarp + 1024 : STAGES * (BM + BN) * BK * 2 + 1024;
  // stream-K grid cap: shallow configurations (<= 4 stages) fit two CTAs per
  // SM, so the next launch can start streaming on an SM while one CTA drains
  static int cap() { return num_sms() * ((SWAP && STAGES <= 4) ? small_per_sm() : 1); }
};

using KernFn = void (*)(KMaps, KArgs, KMaps, KArgs, unsigned int*);

dl_status set_smem_attr(KernFn kern, int smem, bool* done) {
  if (*done) return DL_OK;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(tc_gemm)");
  *done = true;
  return DL_OK;
}

// Kernel arguments of one GEMM problem (everything but the stream-K scheduler,
// which depends on the grid: set_sched).  bytes / flops: algorithmic work.
template <int BN, bool SWAP, int STAGES, bool PAIR>
dl_status prep_args(const GemmProblem& p, bool stream_k, KMaps& maps, KArgs& a, double* bytes, double* flops) {
  using C = Cfg<BN, SWAP, STAGES, PAIR>;
  memset(&maps, 0, sizeof(maps));
  memset(&a, 0, sizeof(a));
  a.T = static_cast<int>(p.T);
  a.tiles_tok = static_cast<int>((p.T + C::TOK_TILE - 1) / C::TOK_TILE);
  a.nseg = p.nseg;
  int tiles = 0;
  long long units = 0;
  for (int g = 0; g < p.nseg; ++g) {
    const GemmSeg& s = p.seg[g];
    KSeg& k = a.seg[g];
    k.feat_begin = static_cast<int>(s.feat_begin);
    k.feat_end = static_cast<int>(s.feat_begin + s.rows);
    k.act_koff = static_cast<int>(s.act_koff);
    k.nkb = static_cast<int>((s.klen + BK - 1) / BK);
    k.tile_first = tiles;
    k.ntiles = static_cast<int>((s.rows + C::FEAT_TILE - 1) / C::FEAT_TILE) * a.tiles_tok;
    k.unit_first = units;
    k.slab_off = p.out.seg_slab_off[g];
    k.rpr = p.out.seg_rpr[g] > 0 ? p.out.seg_rpr[g] : 1;
    k.write_end = static_cast<int>(s.feat_begin + (p.out.seg_write_rows[g] > 0 ? p.out.seg_write_rows[g] : s.rows));
    k.col_off = p.out.remap_cols ? p.out.seg_col_off[g] : s.feat_begin;
    tiles += k.ntiles;
    units += static_cast<long long>(k.ntiles) * k.nkb;
    if (s.klen > 0 && s.rows > 0) {
      if (!make_map(&maps.w[g], s.w, s.rows, s.klen, s.ldw, C::BOX_W)) {
        set_error("cuTensorMapEncodeTiled failed (weight segment %d)", g);
        return DL_ERR_CUDA;
      }
    } else {
      maps.w[g] = maps.w[0];
    }
  }
  a.glu = 0;
  if (p.glu) {
    const GemmSeg& g0 = p.seg[0];
    const GemmSeg& g1 = p.seg[1];
    if (!PAIR || stream_k || p.nseg != 2 || g0.rows != g1.rows || g0.rows % C::FEAT_TILE != 0 || g0.klen != g1.klen ||
        g0.klen <= 0 || p.out.mode != OUT_BF16 || p.out.accumulate || p.out.scatter_p || p.out.remap_cols ||
        p.out.rope_pos || p.out.fan_n || p.out.ld % 8 || (reinterpret_cast<uintptr_t>(p.out.ptr) & 15)) {
      set_error("tc_gemm: the GLU epilogue needs the prefill pair path, gate|up segments of equal rows (%% 256) "
                "and rank, a plain 16-byte-aligned bf16 output");
      return DL_ERR_INVALID_ARG;
    }
    a.glu = 1;
    tiles = a.seg[0].ntiles;   // the whole-tile schedule counts (gate, up) pairs
    static const int spol = DL_ENV("DL_GLU_ACT_POL") ? atoi(DL_ENV("DL_GLU_ACT_POL")) : 1;
    a.glu_spol = spol;
  }
  a.act_w = 0;
  a.xform = XFORM_NONE;
  if (p.xform != XFORM_NONE) {
    if (!SWAP || PAIR || !stream_k || p.fix.op != FIX_NONE || !p.xsrc || p.act_p > 1 || p.xld % 8 || p.xm % 8 ||
        p.k_act % 8) {
      set_error("tc_gemm: in-kernel activation (xform) needs the swap-AB stream-K path, 16-byte rows, no fixup");
      return DL_ERR_INVALID_ARG;
    }
    a.xform = p.xform;
    a.xsrc = p.xsrc;
    a.xld = p.xld;
    a.xm = static_cast<int>(p.xform == XFORM_SILU ? p.xm : 0);
    a.xcols = static_cast<int>(p.k_act);
    maps.act = maps.w[0];   // never read by TMA (a valid map for the descriptor prefetch)
  } else if (p.act_p > 1) {
    if (!SWAP || PAIR || p.act_w % BK || p.act_w * p.act_p != p.k_act) {
      set_error("3-D activation layout: swap-AB path with act_w %% 64 == 0 and act_p * act_w == k_act only");
      return DL_ERR_UNSUPPORTED;
    }
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(p.act_w), static_cast<cuuint64_t>(p.T),
                          static_cast<cuuint64_t>(p.act_p)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(p.act_w * 2), static_cast<cuuint64_t>(p.T * p.act_w * 2)};
    cuuint32_t box[3] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(C::BOX_A), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if (g_encode(&maps.act, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(p.act), dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled (3-D activation) failed");
      return DL_ERR_CUDA;
    }
    a.act_w = static_cast<int>(p.act_w);
  } else if (!make_map(&maps.act, p.act, p.T, p.k_act, p.ld_act, C::BOX_A)) {
    set_error("cuTensorMapEncodeTiled failed (activation)");
    return DL_ERR_CUDA;
  }
  a.total_tiles = tiles;
  a.total_units = units;
  a.stream_k = stream_k ? 1 : 0;
  a.out = p.out.ptr;
  a.ldo = p.out.ld;
  a.mode = p.out.mode;
  a.accumulate = p.out.accumulate;
  a.rope_pos = p.out.rope_pos;
  a.rope_end = static_cast<int>(p.out.rope_end);
  a.rope_l2t = p.out.rope_pos ? log2f(p.out.rope_theta) : 0.f;
  if (p.out.rope_pos) {
    // the vectorised whole-tile epilogue applies it: bf16 plain output, 32-aligned
    // feature range inside segment 0, no K-split tail, no stream-K
    // (features f < rope_end are rotated as head dim f % 128: every segment that
    // holds some of them starts on a head boundary; the K-split tail finalize
    // rotates too)
    bool heads_ok = p.seg[0].feat_begin == 0;
    for (int g = 0; g < p.nseg; ++g)
      if (p.seg[g].feat_begin < p.out.rope_end && (p.seg[g].feat_begin % 128 != 0 || p.out.remap_cols)) heads_ok = false;
    const bool ok = !stream_k && !SWAP && p.out.mode == OUT_BF16 && !p.out.accumulate && p.out.scatter_p == 0 &&
                    !p.glu && p.out.rope_end % 128 == 0 && heads_ok && p.out.rope_end <= p.n_feat && p.out.ld % 8 == 0;
    if (!ok) {
      set_error("tc_gemm: epilogue RoPE needs a whole-tile bf16 output without tail split");
      return DL_ERR_INVALID_ARG;
    }
  }
  a.scatter_p = p.out.scatter_p;
  a.slab = p.out.slab;
  a.fan_n = 0;
  if (p.out.fan_n > 0) {
    if (!SWAP || PAIR || !stream_k || p.out.mode != OUT_BF16_RED || p.fix.op != FIX_NONE || p.out.fan_n > 8) {
      set_error("tc_gemm: fused collective outputs need the swap-AB stream-K bf16 reduction path");
      return DL_ERR_INVALID_ARG;
    }
    if (p.out.scatter_p == 0 && p.out.fan_cols > 0 && p.out.fan_cols % 2) {
      set_error("tc_gemm: fused all-reduce slabs must have an even column count");
      return DL_ERR_INVALID_ARG;
    }
    a.fan_n = p.out.fan_n;
    a.fan_cols = p.out.fan_cols;
    for (int j = 0; j < 8; ++j) a.fan_delta[j] = j < p.out.fan_n ? p.out.fan_delta[j] : 0;
  }
  a.trace_slot = g_trace_host_on ? g_trace_next++ : -1;
  static const int wpol = DL_ENV("DL_PAIR_WPOL") ? atoi(DL_ENV("DL_PAIR_WPOL")) : 2;   // A/B: 0 / 1 / 2 (measured best: 2)
  a.wpol = wpol;
  static const bool tail_vec = !DL_ENV("DL_TAIL_VEC") || atoi(DL_ENV("DL_TAIL_VEC")) != 0;
  a.tail_vec = tail_vec ? 1 : 0;
  // GLU launches: weights evict_first (measured 752 vs 764 us per 70B gate|up stage 2 with evict_last, r02bg)
  static const int glu_wpol = DL_ENV("DL_GLU_WPOL") ? atoi(DL_ENV("DL_GLU_WPOL")) : 0;
  if (a.glu && glu_wpol >= 0) a.wpol = glu_wpol;
  a.dp_tiles = tiles;
  a.tail_split = 0;
  a.tail_acc = nullptr;
  a.fixup = FIX_NONE;
  static const int l2pf = DL_ENV("DL_L2PF") ? atoi(DL_ENV("DL_L2PF")) : kL2Prefetch;
  a.l2pf = l2pf;
  static const int chain_pf = DL_ENV("DL_CHAIN_PF") ? atoi(DL_ENV("DL_CHAIN_PF")) : 64;
  a.chain_pf = chain_pf;
  static const int chain_warp = DL_ENV("DL_CHAIN_WARP") ? atoi(DL_ENV("DL_CHAIN_WARP")) : 0;
  a.chain_warp = chain_warp;
  static const int acce_release = DL_ENV("DL_ACCE_RELEASE") ? atoi(DL_ENV("DL_ACCE_RELEASE")) : 0;   // A/B switch
  a.relaxed_acce = acce_release ? 0 : 1;
  static const int stage_out = DL_ENV("DL_STAGE_OUT") ? atoi(DL_ENV("DL_STAGE_OUT")) : 3;   // A/B: bit 0 plain, bit 1 accumulate
  a.stage_out = stage_out;
  if (p.fix.op != FIX_NONE) {
    bool ok = SWAP && stream_k && p.sched && p.fix.acc32 && p.fix.tile_cnt;
    for (int g = 0; g < p.nseg; ++g) ok = ok && (p.seg[g].rows == 0 || p.seg[g].klen > 0);
    if (p.fix.op == FIX_SILU) ok = ok && p.nseg == 2 && p.seg[0].rows == p.seg[1].rows && p.fix.act_out;
    if (p.fix.op == FIX_RESIDUAL) ok = ok && p.nseg == 1 && p.fix.resid;
    if (p.fix.op == FIX_ROPE_CACHE) ok = ok && p.nseg == 3 && p.out.scatter_p == 0;
    if (!ok) {
      set_error("tc_gemm: fixup %d needs swap-AB stream-K with scheduler, scratch and non-empty segments",
                p.fix.op);
      return DL_ERR_INVALID_ARG;
    }
    a.fixup = p.fix.op;
    a.acc32 = p.fix.acc32;
    a.acc_ld = p.fix.acc_ld;
    a.tile_cnt = p.fix.tile_cnt;
    a.resid = p.fix.resid;
    a.ld_resid = p.fix.ld_resid;
    a.act_out = p.fix.act_out;
    a.ld_act_out = p.fix.ld_act_out;
    a.rope = p.fix.rope;
  }
  a.sched = nullptr;
  // algorithmic work of this launch: every weight element once, the
  // activation K-range of each segment once, every output element once
  double fl = 0, by = 0;
  for (int g = 0; g < p.nseg; ++g) {
    const double rk = static_cast<double>(p.seg[g].rows) * p.seg[g].klen;
    fl += 2.0 * p.T * rk;
    by += 2.0 * rk + 2.0 * p.T * p.seg[g].klen;
  }
  by += static_cast<double>(p.T) * p.n_feat *
        (p.out.mode == OUT_BF16 ? (p.out.accumulate ? 4 : 2) : p.out.mode == OUT_BF16_RED ? 2 : 4);
  *bytes += by;
  *flops += fl;
  return DL_OK;
}

// Hybrid stream-K of a launch with `grid` CTAs: CTA c first takes its static
// range, then dynamic chunks from the work counter p.sched.
void set_sched(const GemmProblem& p, KArgs& a, int grid) {
  // Hybrid split by problem size (measured, 70B@40% decode): launches with
  // many units per CTA (TP = 1: 25-120) keep 90 % static and 8-unit dynamic
  // chunks (finer chunks cost 3-4 ms/step there: each grab is an L2 round trip
  // before its loads); launches with few (TP = 8: 4-20) balance better with
  // 85 % static and 4-unit chunks (TP = 4 / 8: 11.0 -> 10.8 / 8.73 -> 8.5 ms
  // per rank; TP = 2 15.35 -> 15.42, tools/gpu_r02am.sh).
  static const double frac_l = DL_ENV("DL_SK_STATIC") ? atof(DL_ENV("DL_SK_STATIC")) : 0.9;
  static const int chunk_l = DL_ENV("DL_SK_CHUNK") ? atoi(DL_ENV("DL_SK_CHUNK")) : 8;
  static const double frac_s = DL_ENV("DL_SK_STATIC_S") ? atof(DL_ENV("DL_SK_STATIC_S")) : 0.85;
  static const int chunk_s = DL_ENV("DL_SK_CHUNK_S") ? atoi(DL_ENV("DL_SK_CHUNK_S")) : 4;
  static const long long small_upc = DL_ENV("DL_SK_SMALL") ? atoll(DL_ENV("DL_SK_SMALL")) : 24;
  const bool small = a.total_units < small_upc * grid;
  const double frac = small ? frac_s : frac_l;
  const int chunk = small ? chunk_s : chunk_l;
  a.sched = frac >= 1.0 ? nullptr : p.sched;   // static fraction >= 1 (A/B): purely static even split
  a.static_units = static_cast<long long>(frac * static_cast<double>(a.total_units) / grid);
  a.dyn_begin = a.static_units * grid;
  a.chunk = chunk > 0 ? chunk : 1;
}

cudaError_t launch_kern(KernFn kern, int grid, int smem, const KMaps& m1, const KArgs& a1, const KMaps& m2,
                        const KArgs& a2, unsigned int* chain, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, m1, a1, m2, a2, chain);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e;
}

template <int BN, bool SWAP, int STAGES, bool PAIR = false>
dl_status launch_cfg(const GemmProblem& p, bool stream_k, cudaStream_t st) {
  using C = Cfg<BN, SWAP, STAGES, PAIR>;
  static bool attr_set[2] = {false, false};
  const bool glu = PAIR && p.glu;
  KernFn kern = PAIR ? (glu ? tc_gemm_pair_kernel<STAGES, true> : tc_gemm_pair_kernel<STAGES, false>)
                     : tc_gemm_kernel<BN, SWAP, STAGES, false>;
  DL_TRY_INTERNAL(set_smem_attr(kern, C::SMEM, &attr_set[glu ? 1 : 0]));
  KMaps maps;
  KArgs a;
  double bytes = 0, flops = 0;
  DL_TRY_INTERNAL((prep_args<BN, SWAP, STAGES, PAIR>(p, stream_k, maps, a, &bytes, &flops)));
  const long long units = a.total_units;
  const int tiles = a.total_tiles;
  const int sms = num_sms();
  int grid;
  if (stream_k) {
    const int cap = C::cap();
    grid = static_cast<int>(units < cap ? (units > 0 ? units : 1) : cap);
    if (p.sched) set_sched(p, a, grid);
  } else if (PAIR) {
    const int clusters = sms / 2;
    grid = 2 * (tiles < clusters ? (tiles > 0 ? tiles : 1) : clusters);
    // DP + stream-K tail: a last wave filled to <= 75% is split along K
    static const bool dpsk = !DL_ENV("DL_PREFILL_DPSK") || atoi(DL_ENV("DL_PREFILL_DPSK")) != 0;
    const int full = tiles / clusters, tail = tiles % clusters;
    static const double dpsk_frac = DL_ENV("DL_DPSK_FRAC") ? atof(DL_ENV("DL_DPSK_FRAC")) : 0.75;   // A/B
    if (dpsk && p.tail_acc && full >= 1 && tail > 0 && tail <= dpsk_frac * clusters) {
      const int split = clusters / tail;
      if (split >= 2 && static_cast<size_t>(tail) * (a.glu ? 2 : 1) * 256 * 256 * 4 <= p.tail_bytes) {
        a.dp_tiles = tiles - tail;
        a.tail_split = split;
        a.tail_acc = p.tail_acc;
      }
    }
  } else {
    grid = tiles < sms ? (tiles > 0 ? tiles : 1) : sms;
  }
  const int prof = prof_begin(st);
  cudaError_t e = launch_kern(kern, grid, C::SMEM, maps, a, maps, a, nullptr, st);
  prof_end(prof, st, bytes, flops, SWAP ? 1 : 0);
  launched("tc_gemm");
  if (e == cudaSuccess && a.tail_split > 0) {
    const int pf = prof_begin(st);
    const dl_status fs = launch_pdl(a.glu ? tc_tail_finalize_glu_kernel : tc_tail_finalize_kernel,
                                    dim3(a.total_tiles - a.dp_tiles, 8), dim3(256), 0, st, "tc_gemm tail finalize", a);
    prof_end(pf, st, 0.0, 0.0, 2);
    if (fs != DL_OK) return fs;
  }
  if (e != cudaSuccess) {
    set_error("tc_gemm<BN=%d,swap=%d> (T=%lld k_act=%lld nseg=%d klen=%lld/%lld/%lld koff=%lld/%lld/%lld "
              "grid=%d stream_k=%d): %s", BN, (int)SWAP, (long long)p.T, (long long)p.k_act, p.nseg,
              (long long)p.seg[0].klen, (long long)p.seg[1].klen, (long long)p.seg[2].klen,
              (long long)p.seg[0].act_koff, (long long)p.seg[1].act_koff, (long long)p.seg[2].act_koff, grid,
              (int)stream_k, cudaGetErrorString(e));
    return DL_ERR_CUDA;
  }
  return DL_OK;
}

// Fused two-stage chain (swap-AB stream-K, both problems with the same T):
// one launch, stage 2 waits on the in-kernel stage-1 arrival counter `chain`
// (2 zero-initialised uint32, reset by the kernel's last CTA).
template <int BN, int STAGES>
dl_status launch_chain(const GemmProblem& p1, const GemmProblem& p2, unsigned int* chain, cudaStream_t st) {
  using C = Cfg<BN, true, STAGES, false>;
  static bool attr_set = false;
  KernFn kern = tc_gemm_kernel<BN, true, STAGES, true>;
  DL_TRY_INTERNAL(set_smem_attr(kern, C::SMEM, &attr_set));
  KMaps m1, m2;
  KArgs a1, a2;
  double bytes = 0, flops = 0;
  DL_TRY_INTERNAL((prep_args<BN, true, STAGES, false>(p1, true, m1, a1, &bytes, &flops)));
  DL_TRY_INTERNAL((prep_args<BN, true, STAGES, false>(p2, true, m2, a2, &bytes, &flops)));
  const long long units = a1.total_units > a2.total_units ? a1.total_units : a2.total_units;
  // the in-kernel stage-1 -> stage-2 wait needs every CTA co-resident: cap the
  // grid at what the occupancy calculator says fits (e.g. BN = 256: 197 KB of
  // smem, one CTA per SM although the register budget would allow two)
  static int resident = 0;
  if (resident == 0) {
    int per_sm = 0;
    cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, C::SMEM);
    if (oe != cudaSuccess || per_sm < 1) {
      set_error("tc_gemm_chain: occupancy query failed (%s, %d CTAs/SM)", cudaGetErrorString(oe), per_sm);
      return DL_ERR_CUDA;
    }
    resident = per_sm * num_sms();
  }
  const int cap = C::cap() < resident ? C::cap() : resident;
  const int grid = static_cast<int>(units < cap ? (units > 0 ? units : 1) : cap);
  if (p1.sched) set_sched(p1, a1, grid);
  if (p2.sched) set_sched(p2, a2, grid);
  const int prof = prof_begin(st);
  cudaError_t e = launch_kern(kern, grid, C::SMEM, m1, a1, m2, a2, chain, st);
  prof_end(prof, st, bytes, flops, 1);
  launched("tc_gemm");
  if (e != cudaSuccess) {
    set_error("tc_gemm chain<BN=%d> (T=%lld grid=%d): %s", BN, (long long)p1.T, grid, cudaGetErrorString(e));
    return DL_ERR_CUDA;
  }
  return DL_OK;
}

}  // namespace

bool encode_map_bf16(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  return get_encode() && make_map(m, ptr, rows, cols, ld, box_rows);
}

unsigned long long* gemm_trace_cta_slots(int nslots) {
  if (!g_trace_host_on) return nullptr;
  unsigned long long* p = g_trace_host_buf + static_cast<long long>(g_trace_next) * 148 * 8;
  g_trace_next += nslots;
  return p;
}

dl_status set_gemm_trace(void* buf) {
  unsigned long long* p = static_cast<unsigned long long*>(buf);
  g_trace_host_on = p != nullptr;
  g_trace_next = 0;
  g_trace_host_buf = p;
  return cuda_status(cudaMemcpyToSymbol(g_trace, &p, sizeof(p)), "set trace");
}

dl_status tc_gemm(const GemmProblem& p, bool stream_k, cudaStream_t st) {
  if (p.T <= 0) return DL_OK;
  if (!get_encode()) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old or no GPU)");
    return DL_ERR_CUDA;
  }
  if (stream_k && p.out.mode != OUT_F32_RED && p.out.mode != OUT_BF16_RED && p.fix.op == FIX_NONE) {
    set_error("stream-K requires a reduction output");
    return DL_ERR_INVALID_ARG;
  }
  if (p.glu && (stream_k || p.T <= 256)) {
    set_error("tc_gemm: the GLU epilogue is a prefill (T > 256, whole-tile) configuration");
    return DL_ERR_INVALID_ARG;
  }
  static const int dec_stages = DL_ENV("DL_DECODE_STAGES") ? atoi(DL_ENV("DL_DECODE_STAGES")) : 9;
  if (p.T <= 64) return dec_stages == 4 ? launch_cfg<64, true, 4>(p, stream_k, st)
                                        : launch_cfg<64, true, 9>(p, stream_k, st);
  if (p.T <= 128) return launch_cfg<128, true, 6>(p, stream_k, st);
  if (p.T <= 256) return launch_cfg<256, true, 4>(p, stream_k, st);
  static const bool pair = !DL_ENV("DL_PREFILL_PAIR") || atoi(DL_ENV("DL_PREFILL_PAIR")) != 0;
  if (pair && !stream_k && p.out.mode == OUT_BF16) return launch_cfg<256, false, 6, true>(p, stream_k, st);
  return launch_cfg<256, false, 4>(p, stream_k, st);
}

dl_status tc_gemm_chain(const GemmProblem& p1, const GemmProblem& p2, unsigned int* chain, cudaStream_t st) {
  if (p1.T <= 0) return DL_OK;
  if (!get_encode()) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old or no GPU)");
    return DL_ERR_CUDA;
  }
  const bool red_ok = (p1.out.mode == OUT_F32_RED || p1.out.mode == OUT_BF16_RED) && p1.fix.op == FIX_NONE &&
                      (p2.out.mode == OUT_F32_RED || p2.out.mode == OUT_BF16_RED || p2.fix.op != FIX_NONE);
  if (p1.T != p2.T || p1.T > 256 || !red_ok || chain == nullptr || p2.act_p > 1) {
    set_error("tc_gemm_chain: two stream-K reduction problems with the same T <= 256 and a chain counter");
    return DL_ERR_INVALID_ARG;
  }
  if (p1.T <= 64) return launch_chain<64, 9>(p1, p2, chain, st);
  if (p1.T <= 128) return launch_chain<128, 6>(p1, p2, chain, st);
  return launch_chain<256, 4>(p1, p2, chain, st);
}

}  // namespace dl
