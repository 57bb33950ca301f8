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
constexpr int kL2Prefetch = 24; // decode: weight tiles pulled into L2 while waiting (PDL)

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
  // sched[1] counts finished CTAs (the last one resets both).  sched == null:
  // purely static stream-K.
  unsigned int* sched;
  long long static_units, dyn_begin;
  int chunk;
};

struct __align__(64) KMaps {
  CUtensorMap act;
  CUtensorMap w[3];
};

__device__ unsigned long long* g_trace = nullptr;
bool g_trace_host_on = false;   // host: assign a slot to every launch while tracing
int g_trace_next = 0;
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

struct Job {
  int seg, feat0, tok0, kb0, kb1;
};

// Job enumeration shared by the three roles (pure function of blockIdx).
struct JobIter {
  const KArgs& a;
  int cta, grid;
  int next_tile;            // whole-tile mode
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
    if (!a.stream_k) {
      if (next_tile >= a.total_tiles) return false;
      int t = next_tile;
      next_tile += grid;
      int g = 0;
      while (g + 1 < a.nseg && t >= a.seg[g + 1].tile_first) ++g;
      int local = t - a.seg[g].tile_first;
      j.seg = g;
      j.feat0 = a.seg[g].feat_begin + (local / a.tiles_tok) * FEAT_TILE;
      j.tok0 = (local % a.tiles_tok) * TOK_TILE;
      j.kb0 = 0;
      j.kb1 = a.seg[g].nkb;
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
      u += kb1 - kb0;
      return true;
    }
    return false;
  }
};

__device__ __forceinline__ long long out_index(const KArgs& a, const KSeg& s, int tok, int f) {
  if (a.scatter_p <= 0) return static_cast<long long>(tok) * a.ldo + s.col_off + (f - s.feat_begin);
  long long loc = f - s.feat_begin;
  long long owner = loc / s.rpr;
  long long col = s.slab_off + loc % s.rpr;
  return owner * static_cast<long long>(a.T) * a.slab + static_cast<long long>(tok) * a.slab + col;
}

template <int BN, bool SWAP, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ KMaps maps, const __grid_constant__ KArgs a) {
  constexpr int P_ROWS = BM;                 // MMA A operand rows
  constexpr int Q_ROWS = BN;                 // MMA B operand rows
  constexpr int P_BYTES = P_ROWS * BK * 2;
  constexpr int Q_BYTES = Q_ROWS * BK * 2;
  constexpr int STAGE_BYTES = P_BYTES + Q_BYTES;
  constexpr int FEAT_TILE = SWAP ? BM : BN;
  constexpr int TOK_TILE = SWAP ? BN : BM;
  constexpr uint32_t TMEM_COLS = 2 * BN;
  constexpr uint32_t IDESC = ptx::idesc_bf16_f32(BM, BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[STAGES];
  __shared__ __align__(8) uint64_t empty_bar[STAGES];
  __shared__ __align__(8) uint64_t accf_bar[2];
  __shared__ __align__(8) uint64_t acce_bar[2];
  __shared__ __align__(8) uint64_t jfull_bar[kJobRing];
  __shared__ __align__(8) uint64_t jempty_bar[kJobRing];
  __shared__ Job jobs[kJobRing];
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  unsigned long long* tr = (g_trace && a.trace_slot >= 0) ? g_trace + (static_cast<long long>(a.trace_slot) * 148 + blockIdx.x) * 8 : nullptr;   // debug timeline
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
  JobIter it(a, blockIdx.x, gridDim.x);
  Job j;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const uint64_t pol_w = ptx::policy_evict_first();   // weights: streamed once
      const uint64_t pol_a = ptx::policy_evict_last();    // activations: re-read
      int stage = 0;
      uint32_t phase = 0;
      // PDL: the static weight tiles of the first STAGES units are requested
      // before griddepcontrol.wait (they do not depend on the predecessor);
      // their activation halves follow once the predecessor has completed.
      int u = 0;
      bool waited = false;
      if (tr) tr[2] = gtime();
      int pend_c0[STAGES], pend_c1[STAGES];
      // Before waiting on the predecessor, also pull the weight tiles of the
      // next kL2Prefetch units (beyond the STAGES staged in smem) into L2, so
      // the dependency gap is spent streaming HBM instead of idling.
      JobIter pf_it = it;
      if (a.stream_k && a.sched)
        pf_it.set_range(blockIdx.x * a.static_units, (blockIdx.x + 1) * a.static_units);
      auto l2_prefetch = [&]() {
        int skipped = 0, issued = 0;
        Job pj;
        while (issued < kL2Prefetch && pf_it.next(pj, FEAT_TILE, TOK_TILE)) {
          const KSeg& ps = a.seg[pj.seg];
          for (int kb = pj.kb0; kb < pj.kb1 && issued < kL2Prefetch; ++kb) {
            if (skipped < STAGES) { ++skipped; continue; }   // these go to smem
            ptx::tma_prefetch_2d(&maps.w[pj.seg], kb * BK, pj.feat0 - ps.feat_begin);
            ++issued;
          }
        }
      };
      auto flush_pending = [&]() {
        if (SWAP) l2_prefetch();
        pdl_wait();
        waited = true;
        for (int i = 0; i < u && i < STAGES; ++i) {
          uint8_t* dst = smem + i * STAGE_BYTES + (SWAP ? P_BYTES : 0);
          ptx::tma_load_2d(dst, &maps.act, &full_bar[i], pend_c0[i], pend_c1[i], pol_a);
        }
      };
      int jslot = 0;
      uint32_t jphase = 0;
      auto push = [&](const Job& jb) {
        ptx::mbar_wait(&jempty_bar[jslot], jphase ^ 1);
        jobs[jslot] = jb;
        ptx::mbar_arrive(&jfull_bar[jslot]);
        if (++jslot == kJobRing) { jslot = 0; jphase ^= 1; }
      };
      auto emit = [&](const Job& jb) {
        push(jb);
        const KSeg& s = a.seg[jb.seg];
        for (int kb = jb.kb0; kb < jb.kb1; ++kb, ++u) {
          if (u >= STAGES && !waited) flush_pending();
          ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sp = smem + stage * STAGE_BYTES;
          uint8_t* sq = sp + P_BYTES;
          ptx::mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES);
          const int kx = kb * BK;
          uint8_t* sw = SWAP ? sp : sq;
          uint8_t* sa = SWAP ? sq : sp;
          ptx::tma_load_2d(sw, &maps.w[jb.seg], &full_bar[stage], kx, jb.feat0 - s.feat_begin, pol_w);
          if (waited) {
            ptx::tma_load_2d(sa, &maps.act, &full_bar[stage], s.act_koff + kx, jb.tok0, pol_a);
          } else {
            pend_c0[u] = s.act_koff + kx;
            pend_c1[u] = jb.tok0;
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      };
      if (a.stream_k && a.sched) {
        it.set_range(blockIdx.x * a.static_units, (blockIdx.x + 1) * a.static_units);
        while (it.next(j, FEAT_TILE, TOK_TILE)) emit(j);
        for (;;) {   // dynamic tail: fast SMs take more pieces
          const long long g = a.dyn_begin + static_cast<long long>(atomicAdd(a.sched, static_cast<unsigned>(a.chunk)));
          if (g >= a.total_units) break;
          it.set_range(g, g + a.chunk < a.total_units ? g + a.chunk : a.total_units);
          while (it.next(j, FEAT_TILE, TOK_TILE)) emit(j);
        }
      } else {
        while (it.next(j, FEAT_TILE, TOK_TILE)) emit(j);
      }
      Job end;
      end.seg = -1;
      push(end);
      if (!waited) flush_pending();
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
        if (j.seg < 0) break;
        ptx::mbar_wait(&acce_bar[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = j.kb0; kb < j.kb1; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          if (tr && tr[3] == 0) tr[3] = gtime();
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
      if (tr) tr[4] = gtime();
    }
  } else {
    // ===================== epilogue (warps 2..9) =====================
    // 8 warps = 2 per SM sub-partition so the per-element store latency of
    // one warp hides behind the other; warp e handles TMEM lane quarter
    // (warp & 3) and column half (e / 4) of the accumulator.
    pdl_wait();                                // outputs may alias a predecessor's buffers
    const int quarter = warp & 3;              // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;       // accumulator row (M index)
    constexpr int HALF_COLS = BN / 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    int jslot = 0;
    uint32_t jphase = 0;
    for (;;) {
      ptx::mbar_wait(&jfull_bar[jslot], jphase);
      j = jobs[jslot];
      const int my_slot = jslot;
      if (++jslot == kJobRing) { jslot = 0; jphase ^= 1; }
      if (j.seg < 0) break;
      const KSeg& s = a.seg[j.seg];
      ptx::mbar_wait(&accf_bar[acc], acc_phase);
      if (tr && warp == 2 && lane == 0) tr[5] = gtime();   // accumulator of this job ready
      ptx::tc_fence_after();
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
          if (f < s.write_end && ntok > 0) {
            const long long tstride = a.scatter_p <= 0 ? a.ldo : a.slab;
            const long long base = out_index(a, s, tok0, f);
            if (a.mode == OUT_F32_RED) {
              float* p = static_cast<float*>(a.out) + base;
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
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(&acce_bar[acc]);
        ptx::mbar_arrive(&jempty_bar[my_slot]);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (tr && warp == 2 && lane == 0) tr[6] = gtime();   // epilogue done
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc<TMEM_COLS>(tmem_base);
  if (a.sched && threadIdx.x == 0) {   // last CTA out resets the work counter for reuse
    __threadfence();
    if (atomicAdd(a.sched + 1, 1u) == gridDim.x - 1) {
      atomicExch(a.sched, 0u);
      atomicExch(a.sched + 1, 0u);
      __threadfence();
    }
  }

}


// ---------------------------------------------------------------------------
// CTA-pair prefill kernel (cta_group::2): a cluster of 2 CTAs computes a
// 256-token x 256-feature tile with M=256, N=256 MMAs issued by the leader.
// Each CTA stages only its own 128 token rows and 128 weight rows per
// k-block (32 KB / stage), halving per-SM shared-memory operand traffic
// relative to the 1-CTA 128x256 tile.  Whole tiles, bf16 (+ fused residual)
// epilogue; every CTA drains its own TMEM half (its 128 token rows).
// ---------------------------------------------------------------------------
template <int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    tc_gemm_pair_kernel(const __grid_constant__ KMaps maps, const __grid_constant__ KArgs a) {
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
      const uint64_t pol_w = ptx::policy_evict_first();
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
    int acc = 0;
    uint32_t acc_phase = 0;
    while (it.next(j, TILE, TILE)) {
      const KSeg& s = a.seg[j.seg];
      ptx::mbar_wait(&accf_bar[acc], acc_phase);
      ptx::tc_fence_after();
      const bool has_k = j.kb1 > j.kb0;
      const int tok = j.tok0 + static_cast<int>(rank) * HALF + row;
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
        if (tok < a.T && f0 < s.write_end) {
          __nv_bfloat16* o = static_cast<__nv_bfloat16*>(a.out) + out_index(a, s, tok, f0);
          if (f0 + 32 <= s.write_end && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float v[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(r[q * 8 + e]);
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
      if (lane == 0) ptx::mbar_arrive_cluster(acce0 + acc * 8);   // leader's acce_bar[acc]
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc_pair<TMEM_COLS>(tmem_base);
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

template <int BN, bool SWAP, int STAGES, bool PAIR = false>
dl_status launch_cfg(const GemmProblem& p, bool stream_k, cudaStream_t st) {
  // PAIR: cta_group::2 kernel, cluster tile 256 tokens x 256 features, each CTA
  // loads 128-row boxes of both operands.
  constexpr int FEAT_TILE = PAIR ? 256 : (SWAP ? BM : BN);
  constexpr int TOK_TILE = PAIR ? 256 : (SWAP ? BN : BM);
  constexpr int BOX_W = PAIR ? 128 : FEAT_TILE;
  constexpr int BOX_A = PAIR ? 128 : TOK_TILE;
  constexpr int SMEM = PAIR ? STAGES * 2 * 128 * BK * 2 + 1024 : STAGES * (BM + BN) * BK * 2 + 1024;
  static bool attr_set = false;
  void (*kern)(KMaps, KArgs) = PAIR ? tc_gemm_pair_kernel<STAGES> : tc_gemm_kernel<BN, SWAP, STAGES>;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(tc_gemm)");
    attr_set = true;
  }
  KMaps maps;
  memset(&maps, 0, sizeof(maps));
  KArgs a;
  memset(&a, 0, sizeof(a));
  a.T = static_cast<int>(p.T);
  a.tiles_tok = static_cast<int>((p.T + TOK_TILE - 1) / TOK_TILE);
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
    k.ntiles = static_cast<int>((s.rows + FEAT_TILE - 1) / FEAT_TILE) * a.tiles_tok;
    k.unit_first = units;
    k.slab_off = p.out.seg_slab_off[g];
    k.rpr = p.out.seg_rpr[g] > 0 ? p.out.seg_rpr[g] : 1;
    k.write_end = static_cast<int>(s.feat_begin + (p.out.seg_write_rows[g] > 0 ? p.out.seg_write_rows[g] : s.rows));
    k.col_off = p.out.remap_cols ? p.out.seg_col_off[g] : s.feat_begin;
    tiles += k.ntiles;
    units += static_cast<long long>(k.ntiles) * k.nkb;
    if (s.klen > 0 && s.rows > 0) {
      if (!make_map(&maps.w[g], s.w, s.rows, s.klen, s.ldw, BOX_W)) {
        set_error("cuTensorMapEncodeTiled failed (weight segment %d)", g);
        return DL_ERR_CUDA;
      }
    } else {
      maps.w[g] = maps.w[0];
    }
  }
  if (!make_map(&maps.act, p.act, p.T, p.k_act, p.ld_act, BOX_A)) {
    set_error("cuTensorMapEncodeTiled failed (activation)");
    return DL_ERR_CUDA;
  }
  a.total_tiles = tiles;
  a.total_units = units;
  a.stream_k = stream_k ? 1 : 0;
  a.out = p.out.ptr;
  a.ldo = p.out.ld;
  a.mode = p.out.mode;
  // debug A/B switches (timing experiments only; results are wrong with NORED)
  static const bool dbg_tile_order = getenv("DL_DEBUG_SK_TILEORDER") != nullptr;
  static const bool dbg_nored = getenv("DL_DEBUG_NORED") != nullptr;
  if (stream_k && dbg_tile_order) a.stream_k = 0;
  if (stream_k && dbg_nored) a.mode = OUT_F32_STORE;
  a.accumulate = p.out.accumulate;
  a.scatter_p = p.out.scatter_p;
  a.slab = p.out.slab;
  a.trace_slot = g_trace_host_on ? g_trace_next++ : -1;
  a.sched = nullptr;
  if (stream_k && p.sched) {
    static const double frac = getenv("DL_SK_STATIC") ? atof(getenv("DL_SK_STATIC")) : 0.9;
    static const int chunk = getenv("DL_SK_CHUNK") ? atoi(getenv("DL_SK_CHUNK")) : 8;
    const int cap = num_sms() * ((SWAP && STAGES <= 4) ? 2 : 1);   // must match the grid below
    const int g = static_cast<int>(units < cap ? (units > 0 ? units : 1) : cap);
    a.sched = p.sched;
    a.static_units = static_cast<long long>(frac * static_cast<double>(units) / g);
    a.dyn_begin = a.static_units * g;
    a.chunk = chunk > 0 ? chunk : 1;
  }
  const int sms = num_sms();
  int grid;
  if (stream_k) {
    // shallow configurations (<= 4 stages) fit two CTAs per SM: the next
    // launch can then start streaming on an SM while one CTA is still draining
    const int per_sm = (SWAP && STAGES <= 4) ? 2 : 1;
    const int cap = sms * per_sm;
    grid = static_cast<int>(units < cap ? (units > 0 ? units : 1) : cap);
  } else if (PAIR) {
    const int clusters = sms / 2;
    grid = 2 * (tiles < clusters ? (tiles > 0 ? tiles : 1) : clusters);
  } else {
    grid = tiles < sms ? (tiles > 0 ? tiles : 1) : sms;
  }
  // algorithmic work of this launch: every weight element once, the
  // activation K-range of each segment once, every output element once
  double flops = 0, bytes = 0;
  for (int g = 0; g < p.nseg; ++g) {
    const double rk = static_cast<double>(p.seg[g].rows) * p.seg[g].klen;
    flops += 2.0 * p.T * rk;
    bytes += 2.0 * rk + 2.0 * p.T * p.seg[g].klen;
  }
  bytes += static_cast<double>(p.T) * p.n_feat * (p.out.mode == OUT_BF16 ? (p.out.accumulate ? 4 : 2) : 4);
  const int prof = prof_begin(st);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, maps, a);
  prof_end(prof, st, bytes, flops, SWAP ? 1 : 0);
  launched("tc_gemm");
  if (e == cudaSuccess) e = cudaGetLastError();
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

}  // namespace

dl_status set_gemm_trace(void* buf) {
  unsigned long long* p = static_cast<unsigned long long*>(buf);
  g_trace_host_on = p != nullptr;
  g_trace_next = 0;
  return cuda_status(cudaMemcpyToSymbol(g_trace, &p, sizeof(p)), "set trace");
}

dl_status tc_gemm(const GemmProblem& p, bool stream_k, cudaStream_t st) {
  if (p.T <= 0) return DL_OK;
  if (!get_encode()) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old or no GPU)");
    return DL_ERR_CUDA;
  }
  if (stream_k && p.out.mode != OUT_F32_RED) {
    set_error("stream-K requires an fp32 reduction output");
    return DL_ERR_INVALID_ARG;
  }
  static const int dec_stages = getenv("DL_DECODE_STAGES") ? atoi(getenv("DL_DECODE_STAGES")) : 9;
  if (p.T <= 64) return dec_stages == 4 ? launch_cfg<64, true, 4>(p, stream_k, st)
                                        : launch_cfg<64, true, 9>(p, stream_k, st);
  if (p.T <= 128) return launch_cfg<128, true, 6>(p, stream_k, st);
  if (p.T <= 256) return launch_cfg<256, true, 4>(p, stream_k, st);
  static const bool pair = !getenv("DL_PREFILL_PAIR") || atoi(getenv("DL_PREFILL_PAIR")) != 0;
  if (pair && !stream_k && p.out.mode == OUT_BF16) return launch_cfg<256, false, 6, true>(p, stream_k, st);
  return launch_cfg<256, false, 4>(p, stream_k, st);
}

}  // namespace dl
