// Fused decode: a decomposed block's low-rank chains and their elementwise
// glue as ONE persistent tcgen05 kernel per half-block ("phase program").
//
// The decode step is HBM-bound on the factors (Eq. 1: every
// linear is y = A(Bx), two skinny GEMMs).  Launched as separate kernels, each
// of the ~18 per-block boundaries costs 5-16 us on B200 (kernel drain, launch,
// pipeline refill; profiles/r01_summary.md), ~30 % of a 70B layer.  Here the
// same work runs as a list of phases inside one kernel (one CTA per SM):
//
//   GEMM phase     swap-AB stream-K tile of the low-rank stage 1 or stage 2
//                  (weights = MMA M operand, <= 128 tokens = N), fp32
//                  partials red.add-ed into a zero-maintained buffer
//   elementwise    RMSNorm, fp32 -> bf16 Z, RoPE + KV-cache append,
//                  SiLU(gate) * up / ReLU, residual add -- run by the 8
//                  epilogue warps of every CTA, consume-and-clear
//
// Phases are separated by grid-wide barriers (one monotone counter per phase
// in the workspace, reset by the last CTA to exit).  The TMA producer does not
// stop at a barrier: weights are static, so it keeps streaming the next GEMM
// phase's weight tiles into the shared-memory ring while the barrier is open
// and only holds back the activation half of each stage until the phase that
// produces it has completed on every CTA.  HBM therefore stays busy across
// phase boundaries (the ring is 9 x 24 KB per SM ~ 3 us of HBM time).
//
// Co-residency (required by the grid barriers): grid = #SMs, one CTA per SM
// (216 KB of shared memory), and every CTA triggers its PDL dependents at
// entry, so a dependent grid is only launched once all CTAs of this one are
// resident.  Spin waits carry a watchdog (__trap after 2 s) so a broken
// invariant fails the launch instead of hanging the GPU.
#include <cuda.h>
#include <stdio.h>
#include <string.h>

#include "dl_internal.h"
#include "sm100_ptx.cuh"

namespace dl {
namespace {

constexpr int BK = 64;
constexpr int BM = 128;
constexpr int kThreads = 320;    // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue / elementwise
constexpr int kJobRing = 8;

struct FSeg {
  int feat_begin, feat_end, act_koff, nkb, write_end, map;
  long long unit_first, col_off;
};
struct FGemm {
  int nseg, act_map;
  FSeg seg[3];
  long long total_units;
  float* out;
  long long ldo;
};
struct FElem {
  float* acc; long long lda;
  __nv_bfloat16* x; long long ldx;
  const __nv_bfloat16* g;
  __nv_bfloat16* y; long long ldy;
  int n; float eps;
};
struct FPhase {
  int kind;   // FusedKind
  FGemm gm;
  FElem el;
};
struct FProg {
  int T, nphase;
  FPhase ph[kFusedMaxPhases];
  RopeCacheArgs rope;
  unsigned int* bar;   // kFusedMaxPhases + 1 zeroed counters (last: exit count)
  int trace_slot;      // debug timeline slot (-1: off)
};
struct __align__(64) FMaps {
  CUtensorMap m[kFusedMaxGemm * 4];
};

// debug timeline (dl_debug_fused_trace): per launch slot and CTA 48 u64 globaltimer
// stamps: [2p] / [2p+1] epilogue start / end of phase p, [28+p] producer issued
// phase p's activations, [46] entry, [47] SM id
__device__ unsigned long long* g_ftrace = nullptr;
int g_ftrace_next = -1;   // host: next launch slot (-1: tracing off)
constexpr int kTraceWords = 48;

struct FJob {
  int phase, seg, feat0, kb0, kb1;   // seg < 0: end-of-phase marker; phase < 0: end of program
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// arrive: gpu-scope fence (cumulative over the CTA's writes ordered before it
// by bar.sync) then a relaxed add, as in CUTLASS's generic barrier
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(ptx::smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// blocking wait for barrier `p` (all CTAs done with phase p), with watchdog
__device__ __forceinline__ void bar_wait(const unsigned* bar, int p, unsigned grid) {
  if (ld_acquire(bar + p) >= grid) return;
  const unsigned long long t0 = gtime();
  while (ld_acquire(bar + p) < grid) {
    if (gtime() - t0 > 2000000000ull) {
      printf("decode_fused: barrier %d timed out (%u of %u)\n", p, ld_acquire(bar + p), grid);
      __trap();
    }
  }
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

__device__ __forceinline__ float4 ldcg4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4zero(float* p) { *reinterpret_cast<float4*>(p) = make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void st_bf16x4(__nv_bfloat16* p, float a, float b, float c, float d) {
  uint2 o;
  reinterpret_cast<__nv_bfloat162*>(&o)[0] = __floats2bfloat162_rn(a, b);
  reinterpret_cast<__nv_bfloat162*>(&o)[1] = __floats2bfloat162_rn(c, d);
  *reinterpret_cast<uint2*>(p) = o;
}
__device__ __forceinline__ float4 ld_bf16x4(const __nv_bfloat16* p) {
  const uint2 v = __ldcg(reinterpret_cast<const uint2*>(p));
  const float2 a = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(&v)[0]);
  const float2 b = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(&v)[1]);
  return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ float silu_f(float g) { return g / (1.f + __expf(-g)); }

// ---------------------------------------------------------------------------
// elementwise phases: 256 epilogue threads per CTA, etid in [0, 256)
// ---------------------------------------------------------------------------
// Items of W columns over [T x n], grid-stride over all CTAs.  Each thread
// first issues the loads of U items (memory-level parallelism: these phases
// read L2-resident fp32 partials and sit on the critical path between two
// GEMM phases), then transforms and stores them.  U * sizeof(V) is sized so
// nothing spills (a spilled load result serialises the batch).
template <typename V, int W, int U, typename Ld, typename St>
__device__ __forceinline__ void for_items(int T, int n, int etid, Ld ld, St st) {
  // 32-bit index math (T * n < 2^31 on this path): a 64-bit division is a
  // subroutine call, and the calls serialise the batched loads
  const unsigned nq = static_cast<unsigned>(n) / W;
  const unsigned total = static_cast<unsigned>(T) * nq;
  const unsigned stride = gridDim.x * 256u;
  for (unsigned base = blockIdx.x * 256u + etid; base < total; base += stride * U) {
    V v[U];
    int tt[U], cc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned i = base + u * stride;
      tt[u] = -1;
      if (i < total) {
        const unsigned t = i / nq;
        tt[u] = static_cast<int>(t);
        cc[u] = static_cast<int>(i - t * nq) * W;
        v[u] = ld(tt[u], cc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (tt[u] >= 0) st(tt[u], cc[u], v[u]);
  }
}

struct F4x2 { float4 a, b; };
struct F4x4 { float4 a0, a1, b0, b1; };

__device__ __forceinline__ void el_cvt(const FElem& e, int T, int etid) {
  // n is a multiple of 64 (segment-aligned Z layout): 8 columns per item
  for_items<F4x2, 8, 4>(
      T, e.n, etid,
      [&](int t, int c) {
        const float* r = e.acc + static_cast<long long>(t) * e.lda + c;
        return F4x2{ldcg4(r), ldcg4(r + 4)};
      },
      [&](int t, int c, const F4x2& v) {
        float* r = e.acc + static_cast<long long>(t) * e.lda + c;
        st4zero(r);
        st4zero(r + 4);
        uint4 o;
        __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(&o);
        ob[0] = __floats2bfloat162_rn(v.a.x, v.a.y);
        ob[1] = __floats2bfloat162_rn(v.a.z, v.a.w);
        ob[2] = __floats2bfloat162_rn(v.b.x, v.b.y);
        ob[3] = __floats2bfloat162_rn(v.b.z, v.b.w);
        *reinterpret_cast<uint4*>(e.y + static_cast<long long>(t) * e.ldy + c) = o;
      });
}
__device__ __forceinline__ float4 silu_mul4(const float4& g, const float4& u) {
  return make_float4(silu_f(g.x) * u.x, silu_f(g.y) * u.y, silu_f(g.z) * u.z, silu_f(g.w) * u.w);
}
__device__ __forceinline__ float4 relu4(const float4& u) {
  return make_float4(fmaxf(u.x, 0.f), fmaxf(u.y, 0.f), fmaxf(u.z, 0.f), fmaxf(u.w, 0.f));
}
__device__ __forceinline__ void el_silu(const FElem& e, int T, int etid, bool glu) {
  // n = m is a multiple of 64: 8 columns of gate and up per item
  const int uoff = glu ? e.n : 0;
  for_items<F4x4, 8, 4>(
      T, e.n, etid,
      [&](int t, int c) {
        const float* r = e.acc + static_cast<long long>(t) * e.lda + c;
        F4x4 v;
        v.b0 = ldcg4(r + uoff);
        v.b1 = ldcg4(r + uoff + 4);
        if (glu) {
          v.a0 = ldcg4(r);
          v.a1 = ldcg4(r + 4);
        }
        return v;
      },
      [&](int t, int c, const F4x4& v) {
        float* r = e.acc + static_cast<long long>(t) * e.lda + c;
        st4zero(r + uoff);
        st4zero(r + uoff + 4);
        float4 o0, o1;
        if (glu) {
          st4zero(r);
          st4zero(r + 4);
          o0 = silu_mul4(v.a0, v.b0);
          o1 = silu_mul4(v.a1, v.b1);
        } else {
          o0 = relu4(v.b0);
          o1 = relu4(v.b1);
        }
        uint4 o;
        __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(&o);
        ob[0] = __floats2bfloat162_rn(o0.x, o0.y);
        ob[1] = __floats2bfloat162_rn(o0.z, o0.w);
        ob[2] = __floats2bfloat162_rn(o1.x, o1.y);
        ob[3] = __floats2bfloat162_rn(o1.z, o1.w);
        *reinterpret_cast<uint4*>(e.y + static_cast<long long>(t) * e.ldy + c) = o;
      });
}
__device__ __forceinline__ void el_resid(const FElem& e, int T, int etid) {
  for_items<F4x2, 4, 4>(
      T, e.n, etid,
      [&](int t, int c) {
        F4x2 v;
        v.a = ldcg4(e.acc + static_cast<long long>(t) * e.lda + c);
        v.b = ld_bf16x4(e.x + static_cast<long long>(t) * e.ldx + c);
        return v;
      },
      [&](int t, int c, const F4x2& v) {
        st4zero(e.acc + static_cast<long long>(t) * e.lda + c);
        st_bf16x4(e.x + static_cast<long long>(t) * e.ldx + c, v.b.x + v.a.x, v.b.y + v.a.y, v.b.z + v.a.z,
                  v.b.w + v.a.w);
      });
}
// RMSNorm of rows t = blockIdx.x, blockIdx.x + grid, ...; with acc: x += acc
// first (bf16-rounded, acc cleared), exactly as residual_rmsnorm_kernel.
// n <= 8192 (host-checked): each thread holds its <= 4 chunks of 8 in
// registers, all loads of a row issued before the reduction.
constexpr int kNormChunks = 4;
__device__ __forceinline__ void el_rmsnorm(const FElem& e, int T, int etid, bool resid, float* red) {
  const int n8 = e.n / 8;
  const uint4* gr = reinterpret_cast<const uint4*>(e.g);
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    uint4* xr = reinterpret_cast<uint4*>(e.x + static_cast<long long>(t) * e.ldx);
    float* ar = resid ? e.acc + static_cast<long long>(t) * e.lda : nullptr;
    uint4 v[kNormChunks], gv[kNormChunks];
    float4 a0[kNormChunks], a1[kNormChunks];
#pragma unroll
    for (int k = 0; k < kNormChunks; ++k) {
      const int i = etid + k * 256;
      if (i < n8) {
        v[k] = __ldcg(xr + i);
        gv[k] = gr[i];
        if (resid) {
          a0[k] = ldcg4(ar + 8 * i);
          a1[k] = ldcg4(ar + 8 * i + 4);
        }
      }
    }
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < kNormChunks; ++k) {
      const int i = etid + k * 256;
      if (i >= n8) continue;
      __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&v[k]);
      if (resid) {
        st4zero(ar + 8 * i);
        st4zero(ar + 8 * i + 4);
        const float av[8] = {a0[k].x, a0[k].y, a0[k].z, a0[k].w, a1[k].x, a1[k].y, a1[k].z, a1[k].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __bfloat1622float2(b[q]);
          b[q] = __floats2bfloat162_rn(f.x + av[2 * q], f.y + av[2 * q + 1]);
        }
        xr[i] = v[k];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(b[q]);
        ss += f.x * f.x + f.y * f.y;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((etid & 31) == 0) red[etid >> 5] = ss;
    epi_bar();
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += red[w];
    const float inv = rsqrtf(tot / static_cast<float>(e.n) + e.eps);
    uint4* yr = reinterpret_cast<uint4*>(e.y + static_cast<long long>(t) * e.ldy);
#pragma unroll
    for (int k = 0; k < kNormChunks; ++k) {
      const int i = etid + k * 256;
      if (i >= n8) continue;
      uint4 o;
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v[k]);
      const __nv_bfloat162* gb = reinterpret_cast<const __nv_bfloat162*>(&gv[k]);
      __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(b[q]);
        const float2 w = __bfloat1622float2(gb[q]);
        ob[q] = __floats2bfloat162_rn(f.x * inv * w.x, f.y * inv * w.y);
      }
      yr[i] = o;
    }
    epi_bar();   // red[] reused by the next row
  }
}
// RoPE + cache append from the fp32 q|k|v accumulator (same arithmetic as
// rope_cache_kernel in elementwise.cu); acc cleared.  The per-token position
// and cache slot are loaded with the accumulator (no dependent loads later).
struct RopeItem { float4 v; int pos, sq, cpos; };
__device__ __forceinline__ void el_rope_cache(const RopeCacheArgs& a, const FElem& e, int T, int etid) {
  const int heads = a.Hq + 2 * a.Hk;
  const float l2t = log2f(a.theta);
  for_items<RopeItem, 4, 4>(
      T, heads * a.d, etid,
      [&](int t, int col) {
        RopeItem it;
        it.v = ldcg4(e.acc + static_cast<long long>(t) * e.lda + col);
        it.pos = a.positions[t];
        if (a.decode) {
          it.sq = t;
          it.cpos = a.cache_lens[t];
        } else {
          int lo = 0, hi = a.num_seqs - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (a.cu_seqlens[mid] <= t) lo = mid; else hi = mid - 1;
          }
          it.sq = lo;
          it.cpos = a.cache_lens[lo] + (t - a.cu_seqlens[lo]);
        }
        return it;
      },
      [&](int t, int col, const RopeItem& it) {
        st4zero(e.acc + static_cast<long long>(t) * e.lda + col);
        float4 v = it.v;
        const int hd = col >> 7;            // head_dim == 128 (host-checked)
        const int c = col & 127;
        if (a.rope && hd < a.Hq + a.Hk) {
          const float pos = static_cast<float>(it.pos);
          float sn0, cs0, sn1, cs1;
          rope_sincos(pos * exp2f(-l2t * static_cast<float>(c) / a.d), &sn0, &cs0);
          rope_sincos(pos * exp2f(-l2t * static_cast<float>(c + 2) / a.d), &sn1, &cs1);
          v = make_float4(v.x * cs0 - v.y * sn0, v.x * sn0 + v.y * cs0, v.z * cs1 - v.w * sn1,
                          v.z * sn1 + v.w * cs1);
        }
        if (hd < a.Hq) {
          st_bf16x4(a.q_out + static_cast<long long>(t) * a.Hq * a.d + col, v.x, v.y, v.z, v.w);
          return;
        }
        const bool is_k = hd < a.Hq + a.Hk;
        const int kvh = is_k ? hd - a.Hq : hd - a.Hq - a.Hk;
        st_bf16x4((is_k ? a.k_cache : a.v_cache) +
                      ((static_cast<long long>(it.sq) * a.Hk + kvh) * a.max_seq + it.cpos) * a.d + c,
                  v.x, v.y, v.z, v.w);
      });
}

// stream-K job enumeration of one GEMM phase for this CTA
struct PhaseIter {
  const FGemm& g;
  long long u, u_end;
  __device__ PhaseIter(const FGemm& gm) : g(gm) {
    u = (g.total_units * blockIdx.x) / gridDim.x;
    u_end = (g.total_units * (blockIdx.x + 1)) / gridDim.x;
  }
  __device__ bool next(FJob& j) {
    while (u < u_end) {
      int s = 0;
      while (s + 1 < g.nseg && u >= g.seg[s + 1].unit_first) ++s;
      const FSeg& sg = g.seg[s];
      if (sg.nkb == 0) { u = (s + 1 < g.nseg) ? g.seg[s + 1].unit_first : u_end; continue; }
      const long long local = u - sg.unit_first;
      const int tile = static_cast<int>(local / sg.nkb);
      const int kb0 = static_cast<int>(local % sg.nkb);
      const long long rem = u_end - u;
      const int kb1 = static_cast<int>(kb0 + rem < sg.nkb ? kb0 + rem : sg.nkb);
      j.seg = s;
      j.feat0 = sg.feat_begin + tile * BM;
      j.kb0 = kb0;
      j.kb1 = kb1;
      u += kb1 - kb0;
      return true;
    }
    return false;
  }
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    fused_decode_kernel(const __grid_constant__ FMaps maps, const __grid_constant__ FProg prog) {
  constexpr int P_BYTES = BM * BK * 2;    // weight tile (MMA A operand)
  constexpr int Q_BYTES = BN * BK * 2;    // activation tile (MMA B operand)
  constexpr int STAGE_BYTES = P_BYTES + Q_BYTES;
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
  __shared__ FJob jobs[kJobRing];
  __shared__ float red[8];
  __shared__ int pend_stage[STAGES], pend_k[STAGES];   // producer: weight-only stages awaiting activations
  __shared__ uint32_t tmem_slot;

  // every CTA is resident once it runs this: dependents may launch (see header)
  pdl_trigger();
  unsigned long long* tr = (g_ftrace && prog.trace_slot >= 0)
                               ? g_ftrace + (static_cast<long long>(prog.trace_slot) * gridDim.x + blockIdx.x) * kTraceWords
                               : nullptr;
  if (tr && threadIdx.x == 0) {
    unsigned sm;
    asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
    tr[46] = gtime();
    tr[47] = sm;
  }
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const unsigned grid = gridDim.x;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < kFusedMaxGemm * 4; ++i) ptx::prefetch_tmap(&maps.m[i]);
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
      ptx::mbar_init(&jempty_bar[b], 9);   // 8 epilogue warps + the MMA thread
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(&tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const uint64_t pol_w = ptx::policy_evict_first();   // weights: streamed once
      const uint64_t pol_a = ptx::policy_evict_last();    // activations: re-read by every CTA
      int stage = 0;
      uint32_t phase = 0;
      int jslot = 0;
      uint32_t jphase = 0;
      bool pdl_done = false;
      auto push = [&](const FJob& jb) {
        ptx::mbar_wait(&jempty_bar[jslot], jphase ^ 1);
        jobs[jslot] = jb;
        ptx::mbar_arrive(&jfull_bar[jslot]);
        if (++jslot == kJobRing) { jslot = 0; jphase ^= 1; }
      };
      for (int p = 0; p < prog.nphase; ++p) {
        const FPhase& ph = prog.ph[p];
        if (ph.kind != FK_GEMM) continue;
        const FGemm& g = ph.gm;
        const CUtensorMap* amap = &maps.m[g.act_map];
        // activation of phase p is ready once phase p-1 completed everywhere
        // (p == 0: once the predecessor kernel completed)
        bool ready = false;
        int npend = 0;
        // Issue the held-back activation halves once phase p-1 completed.
#define DL_MAKE_READY()                                                                              \
  do {                                                                                               \
    if (!pdl_done) { pdl_wait(); pdl_done = true; }                                                  \
    if (p > 0) bar_wait(prog.bar, p - 1, grid);                                                      \
    fence_proxy_async_global();                                                                      \
    if (tr) tr[28 + p] = gtime();                                                                    \
    ready = true;                                                                                    \
    for (int i_ = 0; i_ < npend; ++i_)                                                               \
      ptx::tma_load_2d(smem + pend_stage[i_] * STAGE_BYTES + P_BYTES, amap, &full_bar[pend_stage[i_]], \
                       pend_k[i_], 0, pol_a);                                                        \
    npend = 0;                                                                                       \
  } while (0)
        PhaseIter it(g);
        FJob j;
        j.phase = p;
        while (it.next(j)) {
          push(j);
          const FSeg& s = g.seg[j.seg];
          for (int kb = j.kb0; kb < j.kb1; ++kb) {
            if (!ready) {
              // Keep streaming weights while the barrier is open.  Block on the
              // barrier only when the oldest ring slot is one of our own
              // weight-only stages (the MMA cannot free it without its
              // activation half); slots of the previous phase free by themselves.
              const unsigned long long t0 = gtime();
              for (;;) {
                if (mbar_test(&empty_bar[stage], phase ^ 1)) break;
                if (npend > 0 && pend_stage[0] == stage) { DL_MAKE_READY(); break; }
                if (p > 0 && pdl_done && ld_acquire(prog.bar + (p - 1)) >= grid) { DL_MAKE_READY(); break; }
                if (gtime() - t0 > 2000000000ull) {
                  printf("decode_fused: producer stalled in phase %d\n", p);
                  __trap();
                }
              }
            }
            ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
            uint8_t* sp = smem + stage * STAGE_BYTES;
            ptx::mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES);
            const int kx = kb * BK;
            ptx::tma_load_2d(sp, &maps.m[s.map], &full_bar[stage], kx, j.feat0 - s.feat_begin, pol_w);
            if (ready) {
              ptx::tma_load_2d(sp + P_BYTES, amap, &full_bar[stage], s.act_koff + kx, 0, pol_a);
            } else {
              if (npend >= STAGES) {
                printf("decode_fused: pending overflow in phase %d\n", p);
                __trap();
              }
              pend_stage[npend] = stage;
              pend_k[npend] = s.act_koff + kx;
              ++npend;
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
        if (!ready) DL_MAKE_READY();
#undef DL_MAKE_READY
        FJob m;
        m.phase = p;
        m.seg = -1;
        push(m);
      }
      FJob end;
      end.phase = -1;
      end.seg = -1;
      push(end);
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
        const FJob j = jobs[jslot];
        ptx::mbar_arrive(&jempty_bar[jslot]);
        if (++jslot == kJobRing) { jslot = 0; jphase ^= 1; }
        if (j.phase < 0) break;
        if (j.seg < 0) continue;   // end-of-phase marker
        ptx::mbar_wait(&acce_bar[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = j.kb0; kb < j.kb1; ++kb) {
          ptx::mbar_wait(&full_bar[stage], phase);
          ptx::tc_fence_after();
          const uint32_t sp = ptx::smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sq = sp + P_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = ptx::sdesc_sw128(sp + k * 32);
            const uint64_t bd = ptx::sdesc_sw128(sq + k * 32);
            ptx::umma_bf16(d_tmem, ad, bd, IDESC, (kb > j.kb0 || k > 0) ? 1u : 0u);
          }
          ptx::umma_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        ptx::umma_commit(&accf_bar[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ============ epilogue warps 2..9: GEMM epilogues + elementwise phases ============
    pdl_wait();
    const int etid = threadIdx.x - 64;
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    constexpr int HALF_COLS = BN / 2;
    const int T = prog.T;
    int acc = 0;
    uint32_t acc_phase = 0;
    int jslot = 0;
    uint32_t jphase = 0;
    for (int p = 0; p < prog.nphase; ++p) {
      const FPhase& ph = prog.ph[p];
      if (ph.kind == FK_GEMM) {
        const FGemm& g = ph.gm;
        for (;;) {
          ptx::mbar_wait(&jfull_bar[jslot], jphase);
          const FJob j = jobs[jslot];
          const int my_slot = jslot;
          if (++jslot == kJobRing) { jslot = 0; jphase ^= 1; }
          if (j.seg < 0) {
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&jempty_bar[my_slot]);
            break;
          }
          const FSeg& s = g.seg[j.seg];
          ptx::mbar_wait(&accf_bar[acc], acc_phase);
          if (tr && etid == 0 && tr[2 * p] == 0) tr[2 * p] = gtime();
          ptx::tc_fence_after();
#pragma unroll 1
          for (int c0 = half * HALF_COLS; c0 < (half + 1) * HALF_COLS; c0 += 32) {
            uint32_t r[32];
            ptx::tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN + c0, r);
            ptx::tmem_ld_wait();
            const int f = j.feat0 + row;
            const int ntok = T - c0;
            if (f < s.write_end && ntok > 0) {
              float* o = g.out + static_cast<long long>(c0) * g.ldo + s.col_off + (f - s.feat_begin);
#pragma unroll
              for (int i = 0; i < 32; ++i, o += g.ldo)
                if (i < ntok) ptx::red_add_f32(o, __uint_as_float(r[i]));
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
      } else {
        if (p > 0) {
          if (etid == 0) {
            bar_wait(prog.bar, p - 1, grid);
            __threadfence();
          }
          epi_bar();
        }
        if (tr && etid == 0) tr[2 * p] = gtime();
        const FElem& e = ph.el;
        switch (ph.kind) {
          case FK_CVT: el_cvt(e, T, etid); break;
          case FK_RMSNORM: el_rmsnorm(e, T, etid, false, red); break;
          case FK_RESID_RMSNORM: el_rmsnorm(e, T, etid, true, red); break;
          case FK_ROPE_CACHE: el_rope_cache(prog.rope, e, T, etid); break;
          case FK_SILU: el_silu(e, T, etid, true); break;
          case FK_RELU: el_silu(e, T, etid, false); break;
          case FK_RESID: el_resid(e, T, etid); break;
          default: break;
        }
      }
      // this CTA is done with phase p: publish (generic writes -> later TMA reads)
      fence_proxy_async_global();
      epi_bar();
      if (tr && etid == 0) tr[2 * p + 1] = gtime();
      if (etid == 0) red_release(prog.bar + p, 1u);
    }
    // drain the end-of-program job (the producer pushes it after the last marker)
    ptx::mbar_wait(&jfull_bar[jslot], jphase);
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(&jempty_bar[jslot]);
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc<TMEM_COLS>(tmem_base);
  if (threadIdx.x == 0) {   // last CTA out resets the phase counters for the next launch
    __threadfence();
    if (atomicAdd(prog.bar + kFusedMaxPhases, 1u) == grid - 1) {
      for (int p = 0; p < kFusedMaxPhases; ++p) atomicExch(prog.bar + p, 0u);
      atomicExch(prog.bar + kFusedMaxPhases, 0u);
      __threadfence();
    }
  }
}

template <int BN, int STAGES>
dl_status launch_fused(const FusedProgram& fp, cudaStream_t st) {
  constexpr int SMEM = STAGES * (BM + BN) * BK * 2 + 1024;
  static bool attr_set = false;
  auto kern = fused_decode_kernel<BN, STAGES>;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(fused_decode)");
    attr_set = true;
  }
  FMaps maps;
  memset(&maps, 0, sizeof(maps));
  FProg pr;
  memset(&pr, 0, sizeof(pr));
  pr.T = static_cast<int>(fp.T);
  pr.nphase = fp.n;
  pr.rope = fp.rope;
  pr.bar = fp.bar;
  pr.trace_slot = g_ftrace_next >= 0 ? g_ftrace_next++ : -1;
  int nmap = 0, ngemm = 0;
  double bytes = 0, flops = 0;
  for (int i = 0; i < fp.n; ++i) {
    const FusedStep& s = fp.step[i];
    FPhase& ph = pr.ph[i];
    ph.kind = s.kind;
    if (s.kind != FK_GEMM) {
      ph.el = FElem{s.acc, s.lda, s.x, s.ldx, s.g, s.y, s.ldy, static_cast<int>(s.n), s.eps};
      continue;
    }
    const GemmProblem& p = s.gemm;
    if (++ngemm > kFusedMaxGemm || p.out.mode != OUT_F32_RED || p.out.scatter_p != 0 || p.T != fp.T) {
      set_error("fused decode: GEMM phase %d unsupported (f32 plain reduction output only, <= %d GEMMs)", i,
                kFusedMaxGemm);
      return DL_ERR_INVALID_ARG;
    }
    FGemm& g = ph.gm;
    g.nseg = p.nseg;
    g.out = static_cast<float*>(p.out.ptr);
    g.ldo = p.out.ld;
    g.act_map = nmap;
    if (!encode_map_bf16(&maps.m[nmap++], p.act, p.T, p.k_act, p.ld_act, BN)) {
      set_error("fused decode: tensor map (activation, phase %d)", i);
      return DL_ERR_CUDA;
    }
    long long units = 0;
    for (int q = 0; q < p.nseg; ++q) {
      const GemmSeg& sg = p.seg[q];
      FSeg& f = g.seg[q];
      f.feat_begin = static_cast<int>(sg.feat_begin);
      f.feat_end = static_cast<int>(sg.feat_begin + sg.rows);
      f.act_koff = static_cast<int>(sg.act_koff);
      f.nkb = (sg.klen > 0 && sg.rows > 0) ? static_cast<int>((sg.klen + BK - 1) / BK) : 0;
      f.write_end = static_cast<int>(sg.feat_begin + (p.out.seg_write_rows[q] > 0 ? p.out.seg_write_rows[q] : sg.rows));
      f.col_off = p.out.remap_cols ? p.out.seg_col_off[q] : sg.feat_begin;
      f.unit_first = units;
      f.map = nmap;
      if (f.nkb > 0) {
        if (!encode_map_bf16(&maps.m[nmap], sg.w, sg.rows, sg.klen, sg.ldw, BM)) {
          set_error("fused decode: tensor map (weights, phase %d segment %d)", i, q);
          return DL_ERR_CUDA;
        }
      } else {
        maps.m[nmap] = maps.m[g.act_map];
      }
      ++nmap;
      units += static_cast<long long>((sg.rows + BM - 1) / BM) * f.nkb;
      const double rk = static_cast<double>(sg.rows) * sg.klen;
      flops += 2.0 * p.T * rk;
      bytes += 2.0 * rk + 2.0 * p.T * sg.klen;
    }
    g.total_units = units;
    bytes += 4.0 * p.T * p.n_feat;
  }
  for (int i = nmap; i < kFusedMaxGemm * 4; ++i) maps.m[i] = maps.m[0];
  const int prof = prof_begin(st);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_sms());
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, maps, pr);
  prof_end(prof, st, bytes, flops, 1);
  if (e != cudaSuccess) return cuda_status(e, "fused_decode launch");
  return launched("fused_decode");
}

}  // namespace

dl_status set_fused_trace(void* buf) {
  unsigned long long* p = static_cast<unsigned long long*>(buf);
  g_ftrace_next = p ? 0 : -1;
  return cuda_status(cudaMemcpyToSymbol(g_ftrace, &p, sizeof(p)), "set fused trace");
}

dl_status fused_decode(const FusedProgram& fp, cudaStream_t st) {
  if (fp.T <= 0 || fp.n <= 0) return DL_OK;
  if (fp.n > kFusedMaxPhases || !fp.bar) {
    set_error("fused decode: %d phases (max %d) or no barrier counters", fp.n, kFusedMaxPhases);
    return DL_ERR_INVALID_ARG;
  }
  if (fp.T <= 64) return launch_fused<64, 9>(fp, st);
  if (fp.T <= 128) return launch_fused<128, 6>(fp, st);
  set_error("fused decode: T=%lld > 128", (long long)fp.T);
  return DL_ERR_INVALID_ARG;
}

}  // namespace dl
