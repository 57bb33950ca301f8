// Prefill causal GQA attention on the 5th-generation tensor cores (row a6 of
// the hot path, prefill; PAPER.md:150 / :222 name FlashAttention for it):
//   out = softmax(q K^T / sqrt(d) + causal mask) V  over the head-major KV
// cache [seq][kv_head][max_seq][128] (post-RoPE keys, this chunk's keys
// already appended), query head h reading kv head floor(h * Hk / Hq)
// (SPEC.md:275), queries continuing a cached prefix of cache_lens[s] keys.
//
// One persistent CTA per SM walks work items (sequence, 128-query tile, head)
// heaviest first (causal: later query tiles see more keys).  Per item:
//   S_t = Q K_t^T    tcgen05.mma M=128 queries x N=128 keys x K=128 dims, Q and
//                    K_t K-major from TMA (128B swizzle), S in TMEM (two
//                    buffers, so S_{t+1} is computed while S_t is softmaxed)
//   P_t = exp2(S_t * log2(e)/sqrt(d) - m)      softmax warps, one query row per
//                    thread: the row max / sum never leave the thread (no
//                    shuffles); P written bf16 to shared memory (K-major,
//                    swizzled as the MMA reads it)
//   O  += P_t V_t    tcgen05.mma with V read MN-major (keys are the reduction
//                    dim, head dims contiguous), O accumulated in TMEM
// The running max m is only moved (and O, l rescaled in TMEM) when a row's
// max grows by more than 2^8: P stays <= 256, and the final O / l is the same
// normalised result (exact up to rounding).  Roles: warp 0 TMA producer,
// warp 1 MMA issuer (one thread), warps 2-9 softmax / rescale / epilogue
// (two per TMEM lane quarter, 64 key columns each).
#include <math.h>

#include <algorithm>

#include "dl_internal.h"
#include "sm100_ptx.cuh"

namespace dl {
namespace {
namespace fa {
constexpr int D = 128;                 // head dim
constexpr int BQ = 128;                // queries per tile (MMA M, TMEM lanes)
constexpr int BKV = 128;               // keys per tile (MMA N of S, K of P.V)
constexpr int kThreads = 320;                // warp 0 TMA, warp 1 MMA, warps 2-9 softmax
constexpr int TILE = 128 * D * 2;      // 32 KB: a Q, K, V or P tile
constexpr int HALF = TILE / 2;         // one 64-column TMA box (128 rows x 128 B)
constexpr int NKV = 3;                 // K / V ring stages
constexpr int XCHG = 2 * 2 * BQ * 4;   // [tile parity][column half][row] fp32 partial row maxima / sums
constexpr int BARS = 32 * 8;           // 22 mbarriers, the TMEM address slot, debug clocks
constexpr int SMEM = 7 * TILE + XCHG + BARS;   // Q, K[3], V[3], exchange, barriers (no static smem)
constexpr uint32_t TMEM_COLS = 512;    // S/P[0] cols 0-127, S/P[1] 128-255, O 256-383, Q 384-447
constexpr float kRescale = 8.f;        // log2 units
// exp2 of FMAE of every 8 scores on the FMA pipe (template argument; DL_FA_FMA_EXP
// selects it in the A/B build): 3 measured 10 % slower (the softmax is issue-bound)
constexpr uint32_t IDESC_S = ptx::idesc_bf16_f32(128, 128);                // A, B K-major
constexpr uint32_t IDESC_PV = ptx::idesc_bf16_f32(128, 128) | (1u << 16);  // B (V) MN-major
}  // namespace fa

__device__ __forceinline__ float ex2(float x) {   // 2^x, MUFU.EX2 (ex2(-inf) = 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA pipe (x <= 2^22; -inf and x < -126 give ~2^-126, negligible
// next to a row sum >= 1): x = n + f, f in [-0.5, 0.5] by the 1.5 * 2^23
// rounding trick, 2^f by its degree-4 Taylor polynomial (relative error
// < 5e-5, far below the bf16 rounding of P), 2^n added to the exponent bits.
// Used for part of each row so the softmax is not bound by the 16 / clk / SM
// MUFU.EX2 rate alone.
__device__ __forceinline__ float ex2_fma(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  float p = fmaf(f, 0.0096181291f, 0.0555041087f);
  p = fmaf(p, f, 0.2402265070f);
  p = fmaf(p, f, 0.6931471806f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

struct FaMaps {
  CUtensorMap q, k, v;
};
struct FaArgs {
  __nv_bfloat16* out;
  int64_t ldo;                 // = Hq * 128
  const int32_t* cu_seqlens;   // [num_seqs + 1]
  const int32_t* cache_lens;   // [num_seqs]
  int num_seqs, Hq, Hk, qtiles;
  int C;                       // cluster size: CTAs (query heads of one KV group) sharing each K/V tile
  int hgroups;                 // (Hq / Hk) / C head groups per KV head
  int64_t max_seq;
  float scale_log2;            // log2(e) / sqrt(d)
  int items;                   // qtiles * num_seqs * Hk * hgroups (one per cluster)
  EwTrace tr;                  // debug timeline (dl_debug_ew_trace), kind 5
  unsigned long long* ctr;     // debug per-CTA cycle breakdown (dl_debug_gemm_trace buffer), 8 u64 per CTA
};
__device__ __forceinline__ long long clk() { return clock64(); }

struct FaItem {
  int s, h, q0, nq, cl, kend, nt;
  int64_t row0, kvrow;
};

// Cluster work item i (heaviest query tiles first) for CTA `rank` of the
// cluster: the C CTAs take C query heads of one KV head (same keys, same
// causal range), so each K/V tile is read from L2 once per cluster and
// multicast.  False if the tile is past the end of its sequence.  Every role
// of every CTA of the cluster evaluates the same sequence of items.
__device__ __forceinline__ bool fa_item(const FaArgs& a, int i, FaItem& it, int rank) {
  const int per = a.num_seqs * a.Hk * a.hgroups;
  const int qt = a.qtiles - 1 - i / per;
  int rem = i - (i / per) * per;
  it.s = rem / (a.Hk * a.hgroups);
  rem -= it.s * a.Hk * a.hgroups;
  const int kvh_ = rem / a.hgroups, hg = rem - kvh_ * a.hgroups;
  it.h = kvh_ * (a.Hq / a.Hk) + hg * a.C + rank;
  const int beg = a.cu_seqlens[it.s], len = a.cu_seqlens[it.s + 1] - beg;
  it.q0 = qt * fa::BQ;
  if (it.q0 >= len) return false;
  it.nq = min(fa::BQ, len - it.q0);
  it.cl = a.cache_lens[it.s];
  it.kend = it.cl + it.q0 + it.nq;          // keys [0, kend) are visible to some row
  it.nt = (it.kend + fa::BKV - 1) / fa::BKV;
  it.row0 = beg + it.q0;
  const int kvh = it.h / (a.Hq / a.Hk);
  it.kvrow = (static_cast<int64_t>(it.s) * a.Hk + kvh) * a.max_seq;
  return true;
}

// The k-th item of this cluster: rounds of (gridDim.x / C) items, alternate
// rounds in reverse cluster order (the heaviest-first list dealt snake-wise
// balances the causal work better than round robin).
__device__ __forceinline__ int fa_snake(int k, int C) {
  const int G = gridDim.x / C, c = blockIdx.x / C;
  return k * G + ((k & 1) ? G - 1 - c : c);
}

template <int FMAE>
__global__ void __launch_bounds__(fa::kThreads, 1)
    attn_prefill_tc_kernel(const __grid_constant__ FaMaps maps, const __grid_constant__ FaArgs a) {
  using namespace fa;
  // All shared memory is dynamic (7 x 32 KB of tiles leave no room for an
  // alignment pad): with no static shared memory the window starts 1024-aligned,
  // as the 128B-swizzled TMA / UMMA tiles need -- checked, never assumed.
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((ptx::smem_u32(smem) & 1023u) != 0) __trap();
  uint8_t* sQ = smem;
  uint8_t* sK = smem + TILE;                 // [NKV]
  uint8_t* sV = smem + (1 + NKV) * TILE;     // [NKV]
  float (*xchg)[2][BQ] = reinterpret_cast<float (*)[2][BQ]>(smem + 7 * TILE);   // [parity][half][row]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 7 * TILE + XCHG);
  uint64_t& q_full = bars[0];      // Q tile landed in shared memory (TMA)
  uint64_t& q_empty = bars[1];     // Q copied to TMEM by the softmax warps (8 arrivals)
  uint64_t& q_tm = bars[2];        // Q in TMEM, ready for the S MMAs (8 arrivals)
  uint64_t& o_empty = bars[3];     // O read by the epilogue (8 arrivals)
  uint64_t* k_full = bars + 4;     // [NKV]
  uint64_t* k_empty = bars + 4 + NKV;
  uint64_t* v_full = bars + 4 + 2 * NKV;
  uint64_t* v_empty = bars + 4 + 3 * NKV;
  uint64_t* s_full = bars + 4 + 4 * NKV;        // [2]
  uint64_t* p_full = bars + 6 + 4 * NKV;        // [2] P written into the S columns (8 arrivals)
  uint64_t* p_empty = bars + 8 + 4 * NKV;       // [2] P.V of that slot retired
  uint32_t& tmem_slot = *reinterpret_cast<uint32_t*>(bars + 10 + 4 * NKV);
  volatile long long* ts_k = reinterpret_cast<volatile long long*>(bars + 24);   // debug: K issue clocks [NKV]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int rank = a.C > 1 ? static_cast<int>(ptx::cluster_ctarank()) : 0;
  const uint16_t cmask = static_cast<uint16_t>((1u << a.C) - 1u);
  ew_mark(a.tr, 1);
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&maps.q);
    ptx::prefetch_tmap(&maps.k);
    ptx::prefetch_tmap(&maps.v);
    ptx::mbar_init(&q_full, 1);
    ptx::mbar_init(&q_empty, 8);
    ptx::mbar_init(&q_tm, 8);
    ptx::mbar_init(&o_empty, 8);
    for (int i = 0; i < NKV; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], a.C);   // every CTA of the cluster has consumed the slot
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], a.C);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&p_full[i], 8);
      ptx::mbar_init(&p_empty[i], 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(&tmem_slot);
  ptx::tc_fence_before();
  if (a.C > 1) ptx::cluster_sync();   // peers' barriers are initialised before any multicast reaches them
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t tS[2] = {tmem, tmem + 128};   // fp32 S; P (bf16) overwrites cols [64h, 64h + 32)
  const uint32_t tO = tmem + 256;
  const uint32_t tQ[2] = {tmem + 384, tmem + 448};   // Q bf16, 64 columns, per item parity

  pdl_trigger();
  pdl_wait();   // q, the appended keys / values and cu_seqlens come from predecessors
  ew_mark(a.tr, 2);

  if (warp == 0) {
    // =========================== TMA producer ===========================
    if (lane == 0) {
      const uint64_t pol_kv = ptx::policy_evict_last();   // K/V re-read by the other heads of the group
      const uint64_t pol_q = ptx::policy_evict_first();
      uint32_t g = 0, n = 0;
      FaItem it;
      for (int k = 0, i; (i = fa_snake(k, a.C)) < a.items; ++k) {
        if (!fa_item(a, i, it, rank)) continue;
        ptx::mbar_wait(&q_empty, (n & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&q_full, TILE);
        ptx::tma_load_2d(sQ, &maps.q, &q_full, it.h * D, static_cast<int>(it.row0), pol_q);
        ptx::tma_load_2d(sQ + HALF, &maps.q, &q_full, it.h * D + 64, static_cast<int>(it.row0), pol_q);
        for (int t = 0; t < it.nt; ++t, ++g) {
          const int kv = g % NKV;
          const uint32_t ph = (g / NKV) & 1;
          // this CTA's slice: rows [rank * R, rank * R + R) of the K and V tiles,
          // multicast to every CTA of the cluster (each expects the whole tile)
          const int R = BKV / a.C;
          const int row = static_cast<int>(it.kvrow + t * BKV) + rank * R;
          const int so = rank * R * 128;
          ptx::mbar_wait(&k_empty[kv], ph ^ 1);
          if (a.ctr) ts_k[kv] = clk();
          ptx::mbar_arrive_expect_tx(&k_full[kv], TILE);
          if (a.C > 1) {
            ptx::tma_load_2d_mc(sK + kv * TILE + so, &maps.k, &k_full[kv], 0, row, cmask, pol_kv);
            ptx::tma_load_2d_mc(sK + kv * TILE + HALF + so, &maps.k, &k_full[kv], 64, row, cmask, pol_kv);
          } else {
            ptx::tma_load_2d(sK + kv * TILE, &maps.k, &k_full[kv], 0, row, pol_kv);
            ptx::tma_load_2d(sK + kv * TILE + HALF, &maps.k, &k_full[kv], 64, row, pol_kv);
          }
          ptx::mbar_wait(&v_empty[kv], ph ^ 1);
          ptx::mbar_arrive_expect_tx(&v_full[kv], TILE);
          if (a.C > 1) {
            ptx::tma_load_2d_mc(sV + kv * TILE + so, &maps.v, &v_full[kv], 0, row, cmask, pol_kv);
            ptx::tma_load_2d_mc(sV + kv * TILE + HALF + so, &maps.v, &v_full[kv], 64, row, cmask, pol_kv);
          } else {
            ptx::tma_load_2d(sV + kv * TILE, &maps.v, &v_full[kv], 0, row, pol_kv);
            ptx::tma_load_2d(sV + kv * TILE + HALF, &maps.v, &v_full[kv], 64, row, pol_kv);
          }
        }
        ++n;
      }
    }
  } else if (warp == 1) {
    // ====================== MMA issuer (one thread) ======================
    if (lane == 0) {
      long long w_k = 0, w_p = 0, w_o = 0;
      // S_g = Q K_g^T: A (Q) from TMEM, B (K) K-major from shared memory.  The
      // S / P columns of slot g & 1 are free: the P.V that read P_{g-2} was
      // issued (and so executes) before this MMA.
      auto issue_s = [&](uint32_t g, bool first, uint32_t n) {
        const int sl = g & 1, kv = g % NKV;
        const uint32_t ph = (g / NKV) & 1;
        long long c0 = clk();
        if (first) ptx::mbar_wait(&q_tm, n & 1);
        ptx::mbar_wait(&k_full[kv], ph);
        const long long c1 = clk();
        w_k += c1 - c0;
        if (a.ctr) w_o += c1 - ts_k[kv];   // debug: K issue -> consumed
        ptx::tc_fence_after();
        const uint32_t k_addr = ptx::smem_u32(sK + kv * TILE);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * HALF + (kk & 3) * 32;
          ptx::umma_bf16_ts(tS[sl], tQ[n & 1] + kk * 8, ptx::sdesc_sw128(k_addr + off), IDESC_S, kk > 0 ? 1u : 0u);
        }
        ptx::umma_commit(&s_full[sl]);
        if (a.C > 1) ptx::umma_commit_mc(&k_empty[kv], cmask);   // the slot is free in this CTA: tell every loader
        else ptx::umma_commit(&k_empty[kv]);
      };
      // O += P_g V_g: A (P) from the S columns in TMEM, B (V) MN-major from shared memory
      auto issue_pv = [&](uint32_t g, bool first, uint32_t n) {
        const int sl = g & 1, kv = g % NKV;
        const uint32_t ph = (g / NKV) & 1;
        if (first) ptx::mbar_wait(&o_empty, (n & 1) ^ 1);
        ptx::mbar_wait(&v_full[kv], ph);
        long long c1 = clk();
        ptx::mbar_wait(&p_full[sl], (g >> 1) & 1);
        w_p += clk() - c1;
        ptx::tc_fence_after();
        const uint32_t v_addr = ptx::smem_u32(sV + kv * TILE);
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk) {
          const uint32_t ta = tS[sl] + (kk < 4 ? kk * 8 : 64 + (kk - 4) * 8);
          ptx::umma_bf16_ts(tO, ta, ptx::sdesc_sw128_mn(v_addr + kk * 16 * 128, HALF), IDESC_PV,
                            (!first || kk > 0) ? 1u : 0u);
        }
        if (a.C > 1) ptx::umma_commit_mc(&v_empty[kv], cmask);
        else ptx::umma_commit(&v_empty[kv]);
        ptx::umma_commit(&p_empty[sl]);
      };
      uint32_t g = 0, n = 0;
      bool pend = false, pend_first = false;
      uint32_t pend_g = 0, pend_n = 0;
      FaItem it;
      for (int k = 0, i; (i = fa_snake(k, a.C)) < a.items; ++k) {
        if (!fa_item(a, i, it, rank)) continue;
        for (int t = 0; t < it.nt; ++t, ++g) {
          // at an item boundary the previous item's last P.V goes first, so its
          // epilogue does not wait for this item's Q
          if (t == 0 && pend) {
            issue_pv(pend_g, pend_first, pend_n);
            pend = false;
          }
          issue_s(g, t == 0, n);
          if (pend) issue_pv(pend_g, pend_first, pend_n);
          pend = true;
          pend_g = g;
          pend_first = t == 0;
          pend_n = n;
        }
        ++n;
      }
      if (pend) issue_pv(pend_g, pend_first, pend_n);
      if (a.ctr) {
        unsigned long long* c = a.ctr + blockIdx.x * 8;
        c[4] = w_k;
        c[5] = w_p;
        c[6] = w_o;
      }
    }
  } else {
    // ============ softmax / O rescale / epilogue (warps 2-9) ============
    // Two warps per TMEM lane quarter: warp w owns query rows 32*(w&3) + lane
    // and key columns [64*half, 64*half + 64) of each S tile (head dims
    // [64*half, +64) of O and Q); the pair combines its row maxima through
    // shared memory once per tile and its row sums once per item.
    const int quarter = warp & 3;                  // TMEM lane quarter of this warp
    const int half = (warp - 2) >> 2;              // column half
    const int row = quarter * 32 + lane;           // query row of the tile
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const int tid = threadIdx.x - 64;              // 0..255
    const int c0 = half * 64;
    uint32_t g = 0, n = 0;
    FaItem it;
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory"); };
    long long t_ws = 0, t_ld = 0, t_ex = 0, t_wp = 0;
    const long long t_beg = clk();
    // Q of item j -> TMEM buffer j & 1 (this warp's 64 dims = TMA box `half`,
    // bf16 pairs per column).  The next item's Q is copied as soon as the
    // current item's last P is out, so its S MMAs overlap this item's epilogue.
    auto copy_q = [&](uint32_t j) {
      ptx::mbar_wait(&q_full, j & 1);
      const uint8_t* qrow = sQ + half * HALF + row * 128;
      uint32_t r[32];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 v = *reinterpret_cast<const uint4*>(qrow + ((c ^ (row & 7)) << 4));
        r[c * 4 + 0] = v.x;
        r[c * 4 + 1] = v.y;
        r[c * 4 + 2] = v.z;
        r[c * 4 + 3] = v.w;
      }
      ptx::tmem_st32(tQ[j & 1] + lane_off + half * 32, r);
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(&q_tm);
        ptx::mbar_arrive(&q_empty);
      }
    };
    int kn = 0;
    FaItem nxt;
    auto find_next = [&]() -> bool {
      for (int i; (i = fa_snake(kn, a.C)) < a.items;) {
        ++kn;
        if (fa_item(a, i, nxt, rank)) return true;
      }
      return false;
    };
    bool have = find_next();
    if (have) copy_q(0);
    while (have) {
      it = nxt;
      have = find_next();
      const int qpos = it.cl + it.q0 + min(row, it.nq - 1);   // this row's position (rows past nq: not stored)
      float m = -INFINITY, l = 0.f;
      for (int t = 0; t < it.nt; ++t, ++g) {
        const int sl = g & 1;
        const uint32_t ph = (g >> 1) & 1;
        const int k0 = t * BKV + c0;                // first key of this warp's columns
        float x[64];
        long long ck0 = clk();
        ptx::mbar_wait(&s_full[sl], ph);
        long long ck1 = clk();
        t_ws += ck1 - ck0;
        ptx::tc_fence_after();
        {
          uint32_t r[2][32];   // both loads in flight, one wait
          ptx::tmem_ld32(tS[sl] + lane_off + c0, r[0]);
          ptx::tmem_ld32(tS[sl] + lane_off + c0 + 32, r[1]);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int j = 0; j < 32; ++j) x[c * 32 + j] = __uint_as_float(r[c][j]);
        }
        // causal mask (a key is visible iff its position <= the query's), row max
        // (8 independent max chains: a single fmax chain is latency-bound)
        if (k0 + 63 > it.cl + it.q0) {
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (k0 + j > qpos) x[j] = -INFINITY;
        }
        float mx8[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mx8[e] = x[e];
#pragma unroll
        for (int j = 8; j < 64; ++j) mx8[j & 7] = fmaxf(mx8[j & 7], x[j]);
        float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                         fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        // combine with the partner warp's half of the row (double-buffered by tile parity)
        xchg[t & 1][half][row] = mx;
        pair_sync();
        mx = fmaxf(mx, xchg[t & 1][half ^ 1][row]);
        const float m_new = fmaxf(m, mx * a.scale_log2);
        long long ck2 = clk();
        t_ld += ck2 - ck1;
        if (t == 0) {
          m = m_new;
        } else {
          const bool resc = m_new > m + kRescale;
          if (__any_sync(0xffffffffu, resc)) {
            // O and l move to the new max: wait for the previous P.V (the last
            // writer of O), then scale this warp's quarter-rows x 64 dims of O
            const uint32_t gp = g - 1;
            ptx::mbar_wait(&p_empty[gp & 1], (gp >> 1) & 1);
            ptx::tc_fence_after();
            const float alpha = resc ? ex2(m - m_new) : 1.f;
#pragma unroll 1
            for (int c = 0; c < 2; ++c) {
              uint32_t r[32];
              ptx::tmem_ld32(tO + lane_off + c0 + c * 32, r);
              ptx::tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) * alpha);
              ptx::tmem_st32(tO + lane_off + c0 + c * 32, r);
            }
            if (resc) {
              l *= alpha;
              m = m_new;
            }
          }
        }
        long long ck3 = clk();
        t_wp += ck3 - ck2;
        // P = exp2(S * scale - m) -> bf16 pairs into TMEM columns [64*half, +32)
        // of this slot (its own S columns, already read)
        float sum8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float p[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float xe = fmaf(x[c * 8 + e], a.scale_log2, -m);
            p[e] = e < FMAE ? ex2_fma(xe) : ex2(xe);   // FMAE of 8 on the FMA pipe
            sum8[e] += p[e];
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) pk[c * 4 + e] = pack_bf16x2(p[2 * e], p[2 * e + 1]);
        }
        ptx::tmem_st32(tS[sl] + lane_off + c0, pk);
        l += ((sum8[0] + sum8[1]) + (sum8[2] + sum8[3])) + ((sum8[4] + sum8[5]) + (sum8[6] + sum8[7]));
        if (t == it.nt - 1 && it.kend - t * BKV < BKV) {
          // keys >= kend of the last tile are masked for every row, but 0 x
          // (stale cache contents, possibly NaN) would poison O: zero those V rows
          const int kv = g % NKV;
          ptx::mbar_wait(&v_full[kv], (g / NKV) & 1);
          const int r0 = it.kend - t * BKV;
          uint8_t* vb = sV + kv * TILE;
          for (int q = tid; q < (BKV - r0) * 16; q += 256) {
            const int rr = r0 + (q >> 4), ck = q & 15;
            *reinterpret_cast<uint4*>(vb + (ck >> 3) * HALF + rr * 128 + (((ck & 7) ^ (rr & 7)) << 4)) =
                make_uint4(0u, 0u, 0u, 0u);
          }
          ptx::fence_async_smem();   // zeroed V rows before the MMA reads them
        }
        ptx::tmem_st_wait();       // P (and any O rescale) in TMEM before the P.V
        // observe every P.V retirement (the previous tile's P.V ran during this softmax,
        // so this costs nothing; it keeps each p_empty phase waited on)
        if (g > 0) ptx::mbar_wait(&p_empty[(g - 1) & 1], ((g - 1) >> 1) & 1);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&p_full[sl]);
        t_ex += clk() - ck3;
      }
      if (have) copy_q(n + 1);
      // ---- epilogue: O / l of this row (this warp's 64 dims) -> bf16 output ----
      {
        // partial sums through the exchange slot of parity nt & 1 (its last reads,
        // in tile nt - 2, are behind the pair barrier of tile nt - 1)
        xchg[it.nt & 1][half][row] = l;
        pair_sync();
        l += xchg[it.nt & 1][half ^ 1][row];
        const uint32_t gl = g - 1;
        ptx::mbar_wait(&p_empty[gl & 1], (gl >> 1) & 1);   // the item's last P.V has retired
        ptx::tc_fence_after();
        const float inv = 1.f / l;
        __nv_bfloat16* orow = a.out + (it.row0 + row) * a.ldo + static_cast<int64_t>(it.h) * D + c0;
        uint32_t r[2][32];
        ptx::tmem_ld32(tO + lane_off + c0, r[0]);
        ptx::tmem_ld32(tO + lane_off + c0 + 32, r[1]);
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&o_empty);
        if (row < it.nq) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 v;
              v.x = pack_bf16x2(__uint_as_float(r[c][q * 8 + 0]) * inv, __uint_as_float(r[c][q * 8 + 1]) * inv);
              v.y = pack_bf16x2(__uint_as_float(r[c][q * 8 + 2]) * inv, __uint_as_float(r[c][q * 8 + 3]) * inv);
              v.z = pack_bf16x2(__uint_as_float(r[c][q * 8 + 4]) * inv, __uint_as_float(r[c][q * 8 + 5]) * inv);
              v.w = pack_bf16x2(__uint_as_float(r[c][q * 8 + 6]) * inv, __uint_as_float(r[c][q * 8 + 7]) * inv);
              *reinterpret_cast<uint4*>(orow + c * 32 + q * 8) = v;
            }
        }
        pair_sync();   // the exchange slot is rewritten by the next item
      }
      ++n;
    }
    if (a.ctr && warp == 2 && lane == 0) {
      unsigned long long* c = a.ctr + blockIdx.x * 8;
      c[0] = t_ws;
      c[1] = t_ld;
      c[2] = t_ex;
      c[3] = t_wp;
      c[7] = clk() - t_beg;
    }
  }

  ptx::tc_fence_before();
  // no CTA leaves while a peer may still multicast into its shared memory or
  // arrive on its barriers
  if (a.C > 1) ptx::cluster_sync();
  else __syncthreads();
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc<TMEM_COLS>(tmem);
  ew_mark(a.tr, 3);
}

}  // namespace

dl_status launch_attention_prefill_tc(const AttnArgs& a, cudaStream_t st) {
  using namespace fa;
  if (a.d != D || a.Hk < 1 || a.Hq % a.Hk != 0) {
    set_error("attention prefill (tcgen05): head_dim %d / heads %d:%d unsupported", a.d, a.Hq, a.Hk);
    return DL_ERR_UNSUPPORTED;
  }
  // cluster size: query heads of one KV group sharing each multicast K/V tile
  // (DL_FA_CLUSTER=1/2/4/8 overrides for A/B); must divide the group size
  const int G = a.Hq / a.Hk;
  static const int c_env = DL_ENV("DL_FA_CLUSTER") ? atoi(DL_ENV("DL_FA_CLUSTER")) : 0;
  int C = c_env > 0 ? c_env : 1;   // measured: 1 and 2 equal (93-97 us / 70B layer), 4: 109, 8: 118 (8-CTA clusters leave SMs idle)
  while (C > 1 && (G % C != 0 || C > 8)) C >>= 1;
  FaMaps maps;
  const int64_t kv_rows = static_cast<int64_t>(a.num_seqs) * a.Hk * a.max_seq;
  const int64_t ldq = a.ld_q > 0 ? a.ld_q : static_cast<int64_t>(a.Hq) * D;
  if (!encode_map_bf16(&maps.q, a.q, a.T, static_cast<int64_t>(a.Hq) * D, ldq, BQ) ||
      !encode_map_bf16(&maps.k, a.k_cache, kv_rows, D, D, BKV / C) ||
      !encode_map_bf16(&maps.v, a.v_cache, kv_rows, D, D, BKV / C)) {
    set_error("attention prefill (tcgen05): cuTensorMapEncodeTiled failed");
    return DL_ERR_CUDA;
  }
  FaArgs k{};
  k.out = a.out;
  k.ldo = static_cast<int64_t>(a.Hq) * D;
  k.cu_seqlens = a.cu_seqlens;
  k.cache_lens = a.cache_lens;
  k.num_seqs = a.num_seqs;
  k.Hq = a.Hq;
  k.Hk = a.Hk;
  k.C = C;
  k.hgroups = G / C;
  k.qtiles = static_cast<int>((a.T + BQ - 1) / BQ);
  k.max_seq = a.max_seq;
  k.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
  k.items = k.qtiles * a.num_seqs * a.Hk * k.hgroups;
  k.tr = ew_trace(5);
  k.ctr = gemm_trace_cta_slots(1);
  static const int fmae = DL_ENV("DL_FA_FMA_EXP") ? atoi(DL_ENV("DL_FA_FMA_EXP")) : 0;
  void (*kern)(FaMaps, FaArgs) = fmae == 1   ? attn_prefill_tc_kernel<1>
                                 : fmae == 2 ? attn_prefill_tc_kernel<2>
                                 : fmae == 3 ? attn_prefill_tc_kernel<3>
                                             : attn_prefill_tc_kernel<0>;
  static bool attr[4] = {false, false, false, false};
  if (!attr[fmae & 3]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(attn_prefill_tc)");
    attr[fmae & 3] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = C;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  // persistent clusters: as many as can be co-resident (one CTA per SM; a
  // cluster's CTAs share a GPC, so 8-CTA clusters may leave SMs idle)
  static int max_clusters[9] = {0};
  if (max_clusters[C] == 0) {
    cfg.gridDim = dim3(C * num_sms());
    int nc = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, kern, &cfg);
    if (e != cudaSuccess || nc < 1) {
      set_error("attention prefill (tcgen05): no co-resident cluster of %d (%s)", C, cudaGetErrorString(e));
      return DL_ERR_CUDA;
    }
    max_clusters[C] = nc;
  }
  const int clusters = std::max(1, std::min(k.items, max_clusters[C]));
  cfg.gridDim = dim3(clusters * C);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, maps, k);
  if (e != cudaSuccess) return cuda_status(e, "attention prefill (tcgen05)");
  return launched("attention prefill (tcgen05)");
}

}  // namespace dl
