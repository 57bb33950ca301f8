// Causal GQA attention over the head-major KV cache (row a6 of the hot
// path): out = softmax(q K^T / sqrt(d) + causal mask) V, query head g
// reading kv head floor(g * Hk / Hq), on the rank's LOCAL
// heads only -- the duplicated self-attention of PAPER.md:141-144 is gone.
//
// Cache layout [seq][kv_head][max_seq][d=128] (bf16): one (seq, kv head) is a
// contiguous run of 256-byte key rows, staged into shared memory with
// cp.async (16-byte chunks, XOR-swizzled so ldmatrix is bank-conflict free).
// Both kernels use bf16 mma.sync.m16n8k16 tensor-core MMAs with fp32
// accumulation and an online (running max, exp2) softmax.
//
// prefill: FlashAttention-2 layout.  CTA = 64 queries x 1 head; warp w owns
//   query rows [16w, 16w+16); K/V tiles of 64 keys double-buffered; only the
//   key tiles at or below the diagonal are visited.
// decode:  one CTA per (sequence, kv head x head chunk, key split).  The
//   G = Hq/Hk query heads sharing the kv head are the MMA rows, 16 per chunk
//   (MHA: G = 1; LLaMA-3 GQA: G = 8; MQA with G > 16 takes ceil(G/16)
//   chunks), so every K/V byte is read from HBM once per 16 query heads; the 4 warps split each 64-key
//   tile 4 ways and are merged (log-sum-exp) through shared memory; key
//   splits (for small batch x heads) are merged by a second tiny kernel.
#include <math.h>
#include <stdlib.h>

#include "dl_internal.h"
#include "sm100_ptx.cuh"

namespace dl {
namespace {

constexpr int D = 128;           // head dim
constexpr int KT = 64;           // keys per tile
constexpr int QT = 64;           // queries per prefill CTA
constexpr int ROW_BYTES = D * 2; // 256
constexpr int TILE_BYTES = KT * ROW_BYTES;   // 16 KB
constexpr int kMaxSplits = 16;

__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint32_t ptx_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t swz(int row, int chunk) {   // byte offset in a [rows][128] bf16 tile
  return static_cast<uint32_t>(row * ROW_BYTES + ((chunk ^ (row & 7)) << 4));
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, bool valid) {
  const int n = valid ? 16 : 0;   // src-size 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t saddr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(saddr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t saddr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(saddr));
}
// C[16x8] += A[16x16] B[16x8], bf16 in, fp32 acc
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float ex2(float x) {   // 2^x, MUFU.EX2 (ex2(-inf) = 0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// cooperative load of `rows` rows (row r from src + r*ld elements) into a swizzled tile;
// rows >= nvalid are zero-filled.  nthr threads.
__device__ __forceinline__ void load_tile(uint32_t sbase, const __nv_bfloat16* src, int64_t ld, int rows, int nvalid,
                                          int tid, int nthr) {
  for (int i = tid; i < rows * 16; i += nthr) {
    const int r = i >> 4, c = i & 15;
    const bool v = r < nvalid;
    cp_async16(sbase + swz(r, c), v ? src + r * ld + c * 8 : src, v);
  }
}

// =============================== prefill ===================================
template <int KTP>
__global__ void __launch_bounds__(128, KTP == 32 ? 3 : 1) attn_prefill_kernel(AttnArgs a, EwTrace tr) {
  ew_mark(tr, 1);
  constexpr int PT = KTP * ROW_BYTES;   // bytes of one K or V tile
  extern __shared__ __align__(1024) uint8_t sm[];
  pdl_trigger();   // successor may launch now; it waits for us before reading
  pdl_wait();
  ew_mark(tr, 2);
  // 1-D (q tile, head) order, heaviest causal q tiles first: the light ones
  // fill the tail of the launch (blockIdx.x = (qtiles-1-qt) * Hq + h)
  const int s = blockIdx.z;
  const int h = blockIdx.x % a.Hq;
  const int q0 = (static_cast<int>(gridDim.x) / a.Hq - 1 - static_cast<int>(blockIdx.x) / a.Hq) * QT;
  const int n_new = a.cu_seqlens[s + 1] - a.cu_seqlens[s];
  if (q0 >= n_new) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t base_pos = a.cache_lens[s];
  const int kvh = static_cast<int>((static_cast<int64_t>(h) * a.Hk) / a.Hq);
  const int64_t tok0 = a.cu_seqlens[s] + q0;
  const int64_t ldq = static_cast<int64_t>(a.Hq) * D;   // output rows
  const int64_t ldqi = a.ld_q > 0 ? a.ld_q : ldq;         // q rows
  const __nv_bfloat16* Qg = a.q + tok0 * ldqi + static_cast<int64_t>(h) * D;
  const int64_t kvoff = (static_cast<int64_t>(s) * a.Hk + kvh) * a.max_seq * D;
  const __nv_bfloat16* Kg = a.k_cache + kvoff;
  const __nv_bfloat16* Vg = a.v_cache + kvoff;
  const int nq = min(QT, n_new - q0);
  const int64_t n_keys = base_pos + q0 + nq;          // keys 0 .. last query position
  const int n_kt = static_cast<int>((n_keys + KTP - 1) / KTP);

  const uint32_t sQ = ptx_smem(sm);
  const uint32_t sK0 = sQ + QT * ROW_BYTES;
  const uint32_t sV0 = sK0 + 2 * PT;

  load_tile(sQ, Qg, ldqi, QT, nq, tid, 128);
  load_tile(sK0, Kg, D, KTP, static_cast<int>(min64(KTP, n_keys)), tid, 128);
  load_tile(sV0, Vg, D, KTP, static_cast<int>(min64(KTP, n_keys)), tid, 128);
  cp_commit();

  uint32_t qf[8][4];
  float acc[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const float scale = rsqrtf(static_cast<float>(D)) * 1.4426950408889634f;
  const int64_t qpos0 = base_pos + q0 + warp * 16 + g;   // row g
  const int64_t qpos1 = qpos0 + 8;                        // row g + 8

  for (int kt = 0; kt < n_kt; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < n_kt) {
      const int64_t k1 = static_cast<int64_t>(kt + 1) * KTP;
      const int nv = static_cast<int>(min64(KTP, n_keys - k1));
      load_tile(sK0 + (buf ^ 1) * PT, Kg + k1 * D, D, KTP, nv, tid, 128);
      load_tile(sV0 + (buf ^ 1) * PT, Vg + k1 * D, D, KTP, nv, tid, 128);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int row = warp * 16 + (lane & 15);
        const int chunk = kk * 2 + (lane >> 4);
        ldsm_x4(sQ + swz(row, chunk), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    const uint32_t sK = sK0 + buf * PT, sV = sV0 + buf * PT;
    // ---- S = Q K^T (16 x KTP per warp) ----
    float sc[KTP / 8][4];
#pragma unroll
    for (int i = 0; i < KTP / 8; ++i) sc[i][0] = sc[i][1] = sc[i][2] = sc[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
      for (int np = 0; np < KTP / 16; ++np) {
        const int key = np * 16 + (lane >> 4) * 8 + (lane & 7);
        const int chunk = kk * 2 + ((lane >> 3) & 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(sK + swz(key, chunk), b0, b1, b2, b3);
        mma16816(sc[2 * np], qf[kk], b0, b1);
        mma16816(sc[2 * np + 1], qf[kk], b2, b3);
      }
    }
    // ---- causal mask, online softmax (m kept in scaled log2 units; the
    //      1/sqrt(d) * log2(e) scale is folded into one FFMA per score) ----
    const int64_t kbase = static_cast<int64_t>(kt) * KTP;
    const bool need_mask = kbase + KTP - 1 > base_pos + q0 + warp * 16 || kbase + KTP > n_keys;
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < KTP / 8; ++nt) {
      if (need_mask) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int64_t kp = kbase + nt * 8 + 2 * t4 + (e & 1);
          const int64_t qp = (e < 2) ? qpos0 : qpos1;
          if (kp > qp || kp >= n_keys) sc[nt][e] = -INFINITY;
        }
      }
      mx0 = fmaxf(mx0, fmaxf(sc[nt][0], sc[nt][1]));
      mx1 = fmaxf(mx1, fmaxf(sc[nt][2], sc[nt][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0 * scale), mn1 = fmaxf(m1, mx1 * scale);
    // rows whose every key so far is masked keep m = -inf: use 0 as the exp base
    const float b0 = mn0 == -INFINITY ? 0.f : mn0, b1 = mn1 == -INFINITY ? 0.f : mn1;
    const float c0 = ex2(m0 - b0), c1 = ex2(m1 - b1);
    m0 = mn0;
    m1 = mn1;
    l0 *= c0;
    l1 *= c1;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      acc[i][0] *= c0; acc[i][1] *= c0;
      acc[i][2] *= c1; acc[i][3] *= c1;
    }
    uint32_t pf[KTP / 16][4];
#pragma unroll
    for (int nt = 0; nt < KTP / 8; ++nt) {
      const float p0 = ex2(fmaf(sc[nt][0], scale, -b0)), p1 = ex2(fmaf(sc[nt][1], scale, -b0));
      const float p2 = ex2(fmaf(sc[nt][2], scale, -b1)), p3 = ex2(fmaf(sc[nt][3], scale, -b1));
      l0 += p0 + p1;
      l1 += p2 + p3;
      const int j = nt >> 1;
      if ((nt & 1) == 0) {
        pf[j][0] = pack_bf16(p0, p1);
        pf[j][1] = pack_bf16(p2, p3);
      } else {
        pf[j][2] = pack_bf16(p0, p1);
        pf[j][3] = pack_bf16(p2, p3);
      }
    }
    // ---- O += P V ----
#pragma unroll
    for (int j = 0; j < KTP / 16; ++j) {
#pragma unroll
      for (int dp = 0; dp < 8; ++dp) {
        const int key = j * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int chunk = dp * 2 + (lane >> 4);
        uint32_t v0, v1, v2, v3;
        ldsm_x4_t(sV + swz(key, chunk), v0, v1, v2, v3);
        mma16816(acc[2 * dp], pf[j], v0, v1);
        mma16816(acc[2 * dp + 1], pf[j], v2, v3);
      }
    }
    __syncthreads();
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float i0 = 1.f / l0, i1 = 1.f / l1;
  const int r0 = warp * 16 + g, r1 = r0 + 8;
  __nv_bfloat16* O = a.out + tok0 * ldq + static_cast<int64_t>(h) * D;
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) {
    const int col = nt * 8 + 2 * t4;
    if (r0 < nq) *reinterpret_cast<uint32_t*>(O + r0 * ldq + col) = pack_bf16(acc[nt][0] * i0, acc[nt][1] * i0);
    if (r1 < nq) *reinterpret_cast<uint32_t*>(O + r1 * ldq + col) = pack_bf16(acc[nt][2] * i1, acc[nt][3] * i1);
  }
  ew_mark(tr, 3);
}

// ================================ decode ===================================
// partial layout (splits > 1): [token][head][split] -> {m, l, acc[128]}
constexpr int PART = D + 2;

__global__ void __launch_bounds__(128) attn_decode_kernel(AttnArgs a, int splits) {
  extern __shared__ __align__(1024) uint8_t sm[];
  pdl_trigger();   // successor may launch now; it waits for us before reading
  pdl_wait();
  const int s = blockIdx.z, sp = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int Gall = a.Hq / a.Hk;
  const int nch = (Gall + 15) >> 4;                  // 16-head chunks per kv head
  const int kvh = blockIdx.y / nch, ch = blockIdx.y - kvh * nch;
  const int h0 = kvh * Gall + ch * 16;               // first query head of this CTA
  const int G = min(16, Gall - ch * 16);
  const int64_t n_keys = static_cast<int64_t>(a.cache_lens[s]) + 1;
  int64_t chunk_keys = (n_keys + splits - 1) / splits;
  chunk_keys = (chunk_keys + KT - 1) / KT * KT;
  const int64_t k_begin = sp * chunk_keys;
  const int64_t k_end = min64(n_keys, k_begin + chunk_keys);
  const int64_t ldq = static_cast<int64_t>(a.Hq) * D;
  const __nv_bfloat16* Qg = a.q + static_cast<int64_t>(s) * ldq + static_cast<int64_t>(h0) * D;
  // key row stride: head-major cache rows are D apart; the low-rank-KV
  // reconstruction buffer is token-major [row][K | V] (kv_ld), sequence s
  // starting at buffer row kv_blk0[s] * kv_bs (the remapping index list)
  const int64_t ldkv = a.kv_ld ? a.kv_ld : D;
  const int64_t kvoff = a.kv_ld ? static_cast<int64_t>(a.kv_blk0[s]) * a.kv_bs * a.kv_ld + static_cast<int64_t>(kvh) * D
                                : (static_cast<int64_t>(s) * a.Hk + kvh) * a.max_seq * D;
  const __nv_bfloat16* Kg = a.k_cache + kvoff;
  const __nv_bfloat16* Vg = a.v_cache + kvoff;

  const uint32_t sQ = ptx_smem(sm);
  const uint32_t sK0 = sQ + 16 * ROW_BYTES;
  const uint32_t sV0 = sK0 + 2 * TILE_BYTES;
  float* red = reinterpret_cast<float*>(sm + 16 * ROW_BYTES + 4 * TILE_BYTES);   // [4 warps][16][128]
  float* redm = red + 4 * 16 * D;                                                 // [4][16] m, then [4][16] l

  const int n_kt = k_end > k_begin ? static_cast<int>((k_end - k_begin + KT - 1) / KT) : 0;
  load_tile(sQ, Qg, D, 16, G, tid, 128);   // head r of the group at Qg + r*D
  if (n_kt > 0) {
    const int nv = static_cast<int>(min64(KT, k_end - k_begin));
    load_tile(sK0, Kg + k_begin * ldkv, ldkv, KT, nv, tid, 128);
    load_tile(sV0, Vg + k_begin * ldkv, ldkv, KT, nv, tid, 128);
  }
  cp_commit();

  float acc[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const float scale = rsqrtf(static_cast<float>(D)) * 1.4426950408889634f;
  uint32_t qf[8][4];

  for (int kt = 0; kt < n_kt; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < n_kt) {
      const int64_t k1 = k_begin + static_cast<int64_t>(kt + 1) * KT;
      const int nv = static_cast<int>(min64(KT, k_end - k1));
      load_tile(sK0 + (buf ^ 1) * TILE_BYTES, Kg + k1 * ldkv, ldkv, KT, nv, tid, 128);
      load_tile(sV0 + (buf ^ 1) * TILE_BYTES, Vg + k1 * ldkv, ldkv, KT, nv, tid, 128);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        ldsm_x4(sQ + swz(lane & 15, kk * 2 + (lane >> 4)), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
    }
    const uint32_t sK = sK0 + buf * TILE_BYTES, sV = sV0 + buf * TILE_BYTES;
    // this warp's 16 keys of the tile: rows [16w, 16w+16)
    float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int key = warp * 16 + (lane >> 4) * 8 + (lane & 7);
      uint32_t b0, b1, b2, b3;
      ldsm_x4(sK + swz(key, kk * 2 + ((lane >> 3) & 1)), b0, b1, b2, b3);
      mma16816(sc[0], qf[kk], b0, b1);
      mma16816(sc[1], qf[kk], b2, b3);
    }
    const int64_t kbase = k_begin + static_cast<int64_t>(kt) * KT + warp * 16;
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = sc[nt][e] * scale;
        if (kbase + nt * 8 + 2 * t4 + (e & 1) >= k_end) v = -INFINITY;
        sc[nt][e] = v;
        if (e < 2) mx0 = fmaxf(mx0, v); else mx1 = fmaxf(mx1, v);
      }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float b0 = mn0 == -INFINITY ? 0.f : mn0, b1 = mn1 == -INFINITY ? 0.f : mn1;
    const float c0 = exp2f(m0 - b0), c1 = exp2f(m1 - b1);
    m0 = mn0;
    m1 = mn1;
    l0 *= c0;
    l1 *= c1;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      acc[i][0] *= c0; acc[i][1] *= c0;
      acc[i][2] *= c1; acc[i][3] *= c1;
    }
    uint32_t pf[4];
    {
      const float p0 = exp2f(sc[0][0] - b0), p1 = exp2f(sc[0][1] - b0);
      const float p2 = exp2f(sc[0][2] - b1), p3 = exp2f(sc[0][3] - b1);
      const float p4 = exp2f(sc[1][0] - b0), p5 = exp2f(sc[1][1] - b0);
      const float p6 = exp2f(sc[1][2] - b1), p7 = exp2f(sc[1][3] - b1);
      l0 += p0 + p1 + p4 + p5;
      l1 += p2 + p3 + p6 + p7;
      pf[0] = pack_bf16(p0, p1);
      pf[1] = pack_bf16(p2, p3);
      pf[2] = pack_bf16(p4, p5);
      pf[3] = pack_bf16(p6, p7);
    }
#pragma unroll
    for (int dp = 0; dp < 8; ++dp) {
      const int key = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
      uint32_t v0, v1, v2, v3;
      ldsm_x4_t(sV + swz(key, dp * 2 + (lane >> 4)), v0, v1, v2, v3);
      mma16816(acc[2 * dp], pf, v0, v1);
      mma16816(acc[2 * dp + 1], pf, v2, v3);
    }
    __syncthreads();
  }
  cp_wait<0>();
  // ---- merge the 4 warps (log-sum-exp) ----
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  if (t4 == 0) {
    redm[warp * 16 + g] = m0;
    redm[warp * 16 + g + 8] = m1;
    redm[64 + warp * 16 + g] = l0;
    redm[64 + warp * 16 + g + 8] = l1;
  }
  __syncthreads();
  float M0 = -INFINITY, M1 = -INFINITY;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    M0 = fmaxf(M0, redm[w * 16 + g]);
    M1 = fmaxf(M1, redm[w * 16 + g + 8]);
  }
  const float B0 = M0 == -INFINITY ? 0.f : M0, B1 = M1 == -INFINITY ? 0.f : M1;
  const float f0 = exp2f(m0 - B0), f1 = exp2f(m1 - B1);
  float* myred = red + warp * 16 * D;
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) {
    const int col = nt * 8 + 2 * t4;
    myred[g * D + col] = acc[nt][0] * f0;
    myred[g * D + col + 1] = acc[nt][1] * f0;
    myred[(g + 8) * D + col] = acc[nt][2] * f1;
    myred[(g + 8) * D + col + 1] = acc[nt][3] * f1;
  }
  __syncthreads();
  // 128 threads: thread = column d, loop over the G valid rows
  for (int r = 0; r < G; ++r) {
    float Mr = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) Mr = fmaxf(Mr, redm[w * 16 + r]);
    const float Br = Mr == -INFINITY ? 0.f : Mr;
    float L = 0.f, o = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      L += redm[64 + w * 16 + r] * exp2f(redm[w * 16 + r] - Br);
      o += red[(w * 16 + r) * D + tid];
    }
    const int h = h0 + r;
    if (splits == 1) {
      a.out[static_cast<int64_t>(s) * ldq + static_cast<int64_t>(h) * D + tid] = __float2bfloat16_rn(o / L);
    } else {
      float* pp = a.partial + ((static_cast<int64_t>(s) * a.Hq + h) * splits + sp) * PART;
      pp[2 + tid] = o;
      if (tid == 0) {
        pp[0] = Mr;
        pp[1] = L;
      }
    }
  }
}

// merge key splits: one CTA (128 threads = d) per (token, head)
__global__ void __launch_bounds__(128) attn_combine_kernel(AttnArgs a, int splits) {
  pdl_trigger();   // successor may launch now; it waits for us before reading
  pdl_wait();
  const int64_t s = blockIdx.y;
  const int h = blockIdx.x, d = threadIdx.x;
  const float* pp = a.partial + (s * a.Hq + h) * splits * PART;
  float M = -INFINITY;
  for (int i = 0; i < splits; ++i) M = fmaxf(M, pp[i * PART]);
  const float B = M == -INFINITY ? 0.f : M;
  float L = 0.f, o = 0.f;
  for (int i = 0; i < splits; ++i) {
    const float f = exp2f(pp[i * PART] - B);
    L += pp[i * PART + 1] * f;
    o += pp[i * PART + 2 + d] * f;
  }
  a.out[s * a.Hq * D + static_cast<int64_t>(h) * D + d] = __float2bfloat16_rn(o / L);
}


// ============================ decode, stream-K =============================
// Flash-decoding with a balanced, persistent split (row a6 at decode).  The
// work is the list of (sequence, kv head, 16-head chunk) items, each a run of
// ceil(n_keys / 64) key tiles; the global tile list is cut into gridDim.x
// equal contiguous ranges, one per CTA (2 CTAs per SM), so every SM streams
// the same number of K/V bytes whatever the mix of context lengths.
//   warp 4      TMA producer: 64-key K and V tiles (2 x 64-column boxes each,
//               128B swizzle) into an NS-stage ring.  Tiles
//               holding only keys older than this step (head-major cache) are
//               requested before griddepcontrol.wait: they do not depend on
//               the predecessor (the RoPE + cache-append kernel writes
//               position cache_lens[s] only).
//   warps 0-3   per tile, warp w scores keys [16w, 16w+16) (mma.sync, the
//               <= 16 query heads of the group are the row block); the tile
//               row max is shared so the four P slices have one scale; the P
//               fragments are exchanged and warp w accumulates output dims
//               [32w, 32w+32) over all 64 keys.  Row sums are added once per
//               item.  An item cut by a range boundary leaves a partial
//               {m, l, o[32]} per contributing CTA and warp (slot 0: the CTA's
//               first item, slot 1: its last); the warp that completes the
//               item's (item, warp) counter last merges them and resets it.
namespace sk {
constexpr int NS = 3;                       // K|V ring stages (x 2 CTAs per SM)
constexpr int STAGE = 4 * 8192;             // K box0, K box1, V box0, V box1
constexpr int kThreads = 160;              // 4 compute warps (dim slices / key slices) + 1 producer
constexpr int SHR = 128 + 4 * 32 * 4;       // floats: tile row max [64], row sums [64]; P fragments [4][32] x 16 B
constexpr int kMaxSeqs = 1024;
constexpr int kPerSM = 2;                   // CTAs per SM (grid = kPerSM x SMs)
constexpr int kPartRow = 2 + 32;            // partial row of one warp: m, l, o[32 dims]
constexpr int kMaxGrid = 3 * 192;           // partial slots are sized for this
template <int NSx = NS>
constexpr size_t smem_bytes(int nseq) {
  return NSx * STAGE + SHR * 4 + 2 * NSx * 8 +
         static_cast<size_t>(nseq + 1) * 4;
}
}  // namespace sk

struct SkMaps {
  CUtensorMap k, v;
};
struct SkArgs {
  const __nv_bfloat16* q;
  __nv_bfloat16* out;
  const int32_t* cache_lens;
  int num_seqs, Hq, Hk, nch, Gall;
  int64_t max_seq;                // head-major cache rows per (seq, kv head)
  int token_major;                // 1: rows kv_blk0[s] * kv_bs + key, kv head at column kvh * 128
  const int32_t* kv_blk0;
  int64_t kv_bs;
  float* part;                    // [kMaxGrid][2][16][2 + D]
  unsigned* cnt;                  // [items], zero-maintained
  EwTrace tr;                     // debug timeline (dl_debug_ew_trace)
  int l2pf;                       // old-key tiles prefetched into L2 before griddepcontrol.wait
  // fused RoPE + cache append (AttnArgs::qkv)
  const __nv_bfloat16* qkv;
  int64_t ld_qkv;
  const int32_t* positions;
  float l2t;                      // log2(theta)
  int rope;
  __nv_bfloat16* kc;              // head-major caches (written: the appended key / value)
  __nv_bfloat16* vc;
  SideZero zero, zero2;
  unsigned long long* ctr;        // per-CTA debug timeline (dl_debug_gemm_trace), 8 u64 per CTA
  int reorder;                    // shared last item first (DL_ATTN_ORDER=1; default plain range order)
  int item_per;                   // > 0: CTA c takes whole items [c * item_per, (c + 1) * item_per) (never split)
};

// RoPE of the interleaved pair (dim, dim + 1) at position pos (fp32 angle
// pos * theta^(-dim/128), rope_sincos -- the rope_cache_kernel expression)
__device__ __forceinline__ uint32_t rope_pair(uint32_t v, float pos, int dim, float l2t) {
  __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&v);
  const float2 f = __bfloat1622float2(b);
  float sn, cs;
  rope_sincos(pos * exp2f(-l2t * static_cast<float>(dim) / D), &sn, &cs);
  return pack_bf16(f.x * cs - f.y * sn, f.x * sn + f.y * cs);
}

struct SkItem {
  int s, j;                       // sequence, item within the sequence (kvh * nch + ch)
  int64_t start, end;             // global tile range of the item
  int64_t g0, g1;                 // this CTA's part of it
  int n_keys;
};

__device__ __forceinline__ int64_t sk_bound(int c, int64_t N, int G) { return (static_cast<int64_t>(c) * N) / G; }
__device__ __forceinline__ int sk_owner(int64_t g, int64_t N, int G) {
  int c = static_cast<int>((g * G) / N);
  while (c + 1 < G && sk_bound(c + 1, N, G) <= g) ++c;
  while (c > 0 && sk_bound(c, N, G) > g) --c;
  return c;
}
// item containing global tile g (g < P[num_seqs]); `s` is a search hint
__device__ __forceinline__ void sk_item_at(const int32_t* P, int num_seqs, int per_seq, int64_t g, SkItem& it,
                                           const int32_t* cache_lens) {
  int lo = 0, hi = num_seqs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (P[mid] <= g) lo = mid; else hi = mid - 1;
  }
  const int s = lo;
  const int nt = (P[s + 1] - P[s]) / per_seq;
  const int j = static_cast<int>((g - P[s]) / nt);
  it.s = s;
  it.j = j;
  it.start = P[s] + static_cast<int64_t>(j) * nt;
  it.end = it.start + nt;
  it.n_keys = cache_lens[s] + 1;
}

__device__ __forceinline__ uint32_t sk_swz(uint32_t base, int key, int chunk) {   // 128B-swizzled TMA box pair
  return base + ((chunk >> 3) << 13) + key * 128 + ((((chunk & 7) ^ (key & 7))) << 4);
}

template <int NS, int PERSM>
__global__ void __launch_bounds__(sk::kThreads, PERSM)
    attn_decode_sk_kernel(const __grid_constant__ SkMaps maps, const __grid_constant__ SkArgs a) {
  using namespace sk;
  extern __shared__ __align__(1024) uint8_t sm[];   // no static shared memory: the base is 1024-aligned
  uint8_t* stages = sm;
  float* tmax = reinterpret_cast<float*>(stages + NS * STAGE);   // [4 warps][16] tile row max, then row sums
  float* pbuf = tmax + 128;                 // [4 k-slices][32 lanes] x uint4 P fragments
  uint64_t* full = reinterpret_cast<uint64_t*>(pbuf + 4 * 32 * 4);
  uint64_t* empty = full + NS;
  int32_t* P = reinterpret_cast<int32_t*>(empty + NS);

  ew_mark(a.tr, 1);
  pdl_trigger();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int per_seq = a.Hk * a.nch;
  unsigned long long* ctr = a.ctr ? a.ctr + static_cast<long long>(blockIdx.x) * 8 : nullptr;
  if (ctr && tid == 0) { ctr[0] = ew_now(); unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); ctr[7] = s; }
  // ---- prefix of tiles per sequence (cache_lens is not written inside the step) ----
  if (warp == 0) {
    // lane l owns sequences [l*per, l*per + per): their tile counts are loaded
    // once (all loads in flight together), scanned across the warp, written
    const int n = a.num_seqs, per = (n + 31) / 32, b = lane * per;
    constexpr int R = kMaxSeqs / 32;
    int cnt[R];
    int sum = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      cnt[r] = (r < per && b + r < n) ? __ldg(a.cache_lens + b + r) : -1;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      cnt[r] = cnt[r] < 0 ? 0 : per_seq * ((cnt[r] + 1 + KT - 1) / KT);
      sum += cnt[r];
    }
    int inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    int run = inc - sum;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r < per && b + r < n) P[b + r] = run;
      run += cnt[r];
    }
    if (lane == 31) P[n] = inc;
  }
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 4);   // released by the 4 compute warps
    }
    ptx::fence_barrier_init();
  }
  __syncthreads();
  if (ctr && tid == 0) ctr[1] = ew_now();
  const int G = gridDim.x, c = blockIdx.x;
  const int64_t N = P[a.num_seqs];
  // whole-item ranges (item_per > 0): the tile index of item i
  auto item_tile = [&](int64_t i) -> int64_t {
    const int64_t items = static_cast<int64_t>(a.num_seqs) * per_seq;
    if (i >= items) return N;
    const int s = static_cast<int>(i / per_seq), jj = static_cast<int>(i - static_cast<int64_t>(s) * per_seq);
    return P[s] + static_cast<int64_t>(jj) * ((P[s + 1] - P[s]) / per_seq);
  };
  const int64_t b0 = a.item_per > 0 ? item_tile(static_cast<int64_t>(c) * a.item_per) : sk_bound(c, N, G);
  const int64_t b1 = a.item_per > 0 ? item_tile(static_cast<int64_t>(c + 1) * a.item_per) : sk_bound(c + 1, N, G);
  const int64_t ldq = static_cast<int64_t>(a.Hq) * D;
  // Processing order: the range's last item (usually shared with the next
  // CTA) first, then [b0, split).  The next CTA processes that shared item
  // first too, so the merges of split items happen early, overlapped with the
  // other CTAs' streaming, instead of all piling up at the kernel's tail.
  int64_t split = b0;
  if (b1 > b0 && a.reorder) {
    SkItem li;
    sk_item_at(P, a.num_seqs, per_seq, b1 - 1, li, a.cache_lens);
    split = li.start > b0 ? li.start : b0;
  }
  const int64_t nA = b1 - split;
  auto tile_at = [&](int64_t q) -> int64_t { return q < nA ? split + q : b0 + (q - nA); };

  if (warp == 4) {
    // ============================ producer ============================
    if (lane != 0) return;
    ptx::prefetch_tmap(&maps.k);
    ptx::prefetch_tmap(&maps.v);
    const uint64_t pol = ptx::policy_evict_first();
    auto tile_coords = [&](const SkItem& it, int64_t g, int& row, int& col) {
      const int kvh = it.j / a.nch;
      const int t = static_cast<int>(g - it.start);
      if (a.token_major) {
        row = static_cast<int>(static_cast<int64_t>(a.kv_blk0[it.s]) * a.kv_bs + t * KT);
        col = kvh * D;
      } else {
        row = static_cast<int>((static_cast<int64_t>(it.s) * a.Hk + kvh) * a.max_seq + t * KT);
        col = 0;
      }
    };
    auto issue = [&](const SkItem& it, int64_t g, int64_t l) {   // l: position in the processing order
      const int st = static_cast<int>(l % NS);
      ptx::mbar_wait(&empty[st], ((l / NS) & 1) ^ 1);
      int row, col;
      tile_coords(it, g, row, col);
      uint8_t* dst = stages + st * STAGE;
      ptx::mbar_arrive_expect_tx(&full[st], STAGE);
      ptx::tma_load_2d(dst, &maps.k, &full[st], col, row, pol);
      ptx::tma_load_2d(dst + 8192, &maps.k, &full[st], col + 64, row, pol);
      ptx::tma_load_2d(dst + 16384, &maps.v, &full[st], col, row, pol);
      ptx::tma_load_2d(dst + 24576, &maps.v, &full[st], col + 64, row, pol);
    };
    const int64_t ntl = b1 - b0;
    // 1. before the predecessor completes: leading tiles of old keys only
    int64_t pre = 0;
    if (!a.token_major) {
      SkItem it;
      while (pre < ntl && pre < NS) {
        const int64_t g = tile_at(pre);
        sk_item_at(P, a.num_seqs, per_seq, g, it, a.cache_lens);
        const int t = static_cast<int>(g - it.start);
        if ((t + 1) * KT > it.n_keys - 1) break;   // tile holds the key appended by this step
        issue(it, g, pre);
        ++pre;
      }
      // ... and the next l2pf old-key tiles into L2 (HBM is otherwise idle
      // while the predecessor finishes)
      for (int64_t n = 0, q = pre; n < a.l2pf && q < ntl; ++n, ++q) {
        const int64_t g = tile_at(q);
        sk_item_at(P, a.num_seqs, per_seq, g, it, a.cache_lens);
        const int t = static_cast<int>(g - it.start);
        if ((t + 1) * KT > it.n_keys - 1) continue;
        int row, col;
        tile_coords(it, g, row, col);
        ptx::tma_prefetch_2d(&maps.k, col, row);
        ptx::tma_prefetch_2d(&maps.k, col + 64, row);
        ptx::tma_prefetch_2d(&maps.v, col, row);
        ptx::tma_prefetch_2d(&maps.v, col + 64, row);
      }
    }
    pdl_wait();
    // 2. the remaining tiles
    SkItem it{};
    it.end = -1;
    for (int64_t q = pre; q < ntl; ++q) {
      const int64_t g = tile_at(q);
      if (g < it.start || g >= it.end) sk_item_at(P, a.num_seqs, per_seq, g, it, a.cache_lens);
      issue(it, g, q);
    }
    return;
  }

  // ============================== compute ==============================
  pdl_wait();
  ew_mark(a.tr, 2);
  if (ctr && tid == 0) ctr[2] = ew_now();
  // side clears (the q|k|v group's latent buffer; at TP the reduce-scatter's
  // partial buffer), spread over every compute thread
  for (const SideZero& z : {a.zero, a.zero2}) {
    if (!z.p) continue;
    const int64_t per_row = z.row_bytes / 16, total = z.rows * per_row;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * 128 + tid; i < total; i += static_cast<int64_t>(gridDim.x) * 128) {
      const int64_t r = i / per_row;
      *reinterpret_cast<uint4*>(static_cast<uint8_t*>(z.p) + r * z.ld + (i - r * per_row) * 16) =
          make_uint4(0u, 0u, 0u, 0u);
    }
  }
  const int w = warp;
  const int g8 = lane >> 2, t4 = lane & 3;
  const float scale = rsqrtf(static_cast<float>(D)) * 1.4426950408889634f;
  int64_t lpos = 0;   // position in the processing order (ring slot / phase)
  int n_items = 0, n_merges = 0;   // debug trace
  for (int64_t g = split, send = b1; g < send || send == b1;) {
    if (g >= send) {   // segment A [split, b1) done: then [b0, split)
      if (split == b0) break;
      g = b0;
      send = split;
    }
    SkItem it;
    sk_item_at(P, a.num_seqs, per_seq, g, it, a.cache_lens);
    const int64_t e = it.end < send ? it.end : send;
    const int kvh = it.j / a.nch, ch = it.j - kvh * a.nch;
    const int h0 = kvh * a.Gall + ch * 16;
    const int Gc = min(16, a.Gall - ch * 16);
    // query fragments (rows g8, g8 + 8) straight from L2 -- written by the
    // predecessor, so after griddepcontrol.wait; rows >= Gc read as zero
    uint32_t qf[8][4];
    {
      // fused mode: raw q|k|v rows, q rotated here (pair (2i, 2i+1) = one u32)
      const uint32_t* q0 = a.qkv ? reinterpret_cast<const uint32_t*>(a.qkv + it.s * a.ld_qkv +
                                                                     static_cast<int64_t>(h0 + g8) * D)
                                 : reinterpret_cast<const uint32_t*>(a.q + it.s * ldq + static_cast<int64_t>(h0 + g8) * D);
      const uint32_t* q1 = q0 + 8 * (D / 2);
      const bool v0 = g8 < Gc, v1 = g8 + 8 < Gc;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        qf[kk][0] = v0 ? q0[kk * 8 + t4] : 0u;
        qf[kk][1] = v1 ? q1[kk * 8 + t4] : 0u;
        qf[kk][2] = v0 ? q0[kk * 8 + 4 + t4] : 0u;
        qf[kk][3] = v1 ? q1[kk * 8 + 4 + t4] : 0u;
      }
      if (a.qkv && a.rope) {
        const float pos = static_cast<float>(a.positions[it.s]);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          float sn0, cs0, sn1, cs1;
          rope_sincos(pos * exp2f(-a.l2t * static_cast<float>(kk * 16 + 2 * t4) / D), &sn0, &cs0);
          rope_sincos(pos * exp2f(-a.l2t * static_cast<float>(kk * 16 + 8 + 2 * t4) / D), &sn1, &cs1);
          auto rot = [](uint32_t v, float sn, float cs) {
            const float2 f = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&v));
            return pack_bf16(f.x * cs - f.y * sn, f.x * sn + f.y * cs);
          };
          qf[kk][0] = rot(qf[kk][0], sn0, cs0);
          qf[kk][1] = rot(qf[kk][1], sn0, cs0);
          qf[kk][2] = rot(qf[kk][2], sn1, cs1);
          qf[kk][3] = rot(qf[kk][3], sn1, cs1);
        }
      }
    }
    // fused append (a.qkv): the CTA owning the item's last tile holds the new
    // key (rotated) and value rows: lanes 0-15 one 16-byte chunk of k each,
    // lanes 16-19 this warp's 4 chunks of v.  They patch the shared-memory
    // tile (the cache slot TMA read may be stale) and are appended to the cache.
    const bool own_new = a.qkv && e == it.end;
    const int newrow = (it.n_keys - 1) & (KT - 1);
    uint4 nkv = make_uint4(0u, 0u, 0u, 0u);
    if (own_new && lane < 20) {
      const int64_t rowoff = it.s * a.ld_qkv + static_cast<int64_t>(a.Hq + kvh) * D;
      const int chunk = lane < 16 ? lane : w * 4 + (lane - 16);
      const __nv_bfloat16* srcp = a.qkv + rowoff + (lane < 16 ? 0 : static_cast<int64_t>(a.Hk) * D) + chunk * 8;
      nkv = *reinterpret_cast<const uint4*>(srcp);
      if (lane < 16 && a.rope) {
        const float pos = static_cast<float>(a.positions[it.s]);
        nkv.x = rope_pair(nkv.x, pos, chunk * 8, a.l2t);
        nkv.y = rope_pair(nkv.y, pos, chunk * 8 + 2, a.l2t);
        nkv.z = rope_pair(nkv.z, pos, chunk * 8 + 4, a.l2t);
        nkv.w = rope_pair(nkv.w, pos, chunk * 8 + 6, a.l2t);
      }
      const int64_t dst = ((static_cast<int64_t>(it.s) * a.Hk + kvh) * a.max_seq + (it.n_keys - 1)) * D + chunk * 8;
      if (lane < 16) {
        if (w == newrow / 16) *reinterpret_cast<uint4*>(a.kc + dst) = nkv;
      } else {
        *reinterpret_cast<uint4*>(a.vc + dst) = nkv;
      }
    }
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;   // m in log2 units (scaled)
    for (int64_t gt = g; gt < e; ++gt) {
      const int64_t l = lpos++;
      const int st = static_cast<int>(l % NS);
      ptx::mbar_wait(&full[st], (l / NS) & 1);
      if (ctr && tid == 0 && ctr[3] == 0) ctr[3] = ew_now();
      const uint32_t sK = ptx::smem_u32(stages + st * STAGE), sV = sK + 16384;
      const int nv = min(KT, it.n_keys - static_cast<int>(gt - it.start) * KT);   // valid keys of the tile
      if (nv < KT) {
        // keys past the end: their P is 0, but 0 * (garbage V) may be NaN;
        // zero this warp's 4 chunks (dims 32w..32w+31) of the invalid rows
        for (int i = lane; i < (KT - nv) * 4; i += 32) {
          const int key = nv + (i >> 2), chk = w * 4 + (i & 3);
          *reinterpret_cast<uint4*>(stages + st * STAGE + 16384 + sk_swz(0, key, chk)) = make_uint4(0u, 0u, 0u, 0u);
        }
      }
      const bool patch = own_new && gt == it.end - 1;
      if (patch && lane < 20) {
        if (lane < 16) {
          if (w == newrow / 16) *reinterpret_cast<uint4*>(stages + st * STAGE + sk_swz(0, newrow, lane)) = nkv;
        } else {
          *reinterpret_cast<uint4*>(stages + st * STAGE + 16384 + sk_swz(0, newrow, w * 4 + (lane - 16))) = nkv;
        }
      }
      if (nv < KT || patch) __syncwarp();
      // scores of this warp's 16 keys [16w, 16w + 16) of the tile
      float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      {
        const int key = w * 16 + (lane & 7) + ((lane >> 4) & 1) * 8;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          uint32_t b0r, b1r, b2r, b3r;
          ldsm_x4(sk_swz(sK, key, kk * 2 + ((lane >> 3) & 1)), b0r, b1r, b2r, b3r);
          mma16816(sc[0], qf[kk], b0r, b1r);
          mma16816(sc[1], qf[kk], b2r, b3r);
        }
      }
      if (w * 16 + 16 > nv) {
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (w * 16 + nt * 8 + 2 * t4 + (q & 1) >= nv) sc[nt][q] = -INFINITY;
      }
      float mx0 = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
      float mx1 = fmaxf(fmaxf(sc[0][2], sc[0][3]), fmaxf(sc[1][2], sc[1][3]));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      // tile row max over the group's 4 warps -> one scale for the whole P tile
      float* tm = tmax;
      if (t4 == 0) {
        tm[w * 16 + g8] = mx0;
        tm[w * 16 + g8 + 8] = mx1;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
      for (int ww = 0; ww < 4; ++ww) {
        mx0 = fmaxf(mx0, tm[ww * 16 + g8]);
        mx1 = fmaxf(mx1, tm[ww * 16 + g8 + 8]);
      }
      const float mn0 = fmaxf(m0, mx0 * scale), mn1 = fmaxf(m1, mx1 * scale);   // every tile has a valid key
      const float c0 = ex2(m0 - mn0), c1 = ex2(m1 - mn1);
      m0 = mn0;
      m1 = mn1;
      l0 *= c0;
      l1 *= c1;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[i][0] *= c0; acc[i][1] *= c0;
        acc[i][2] *= c1; acc[i][3] *= c1;
      }
      uint32_t pf[4];
      {
        const float p0 = ex2(fmaf(sc[0][0], scale, -mn0)), p1 = ex2(fmaf(sc[0][1], scale, -mn0));
        const float p2 = ex2(fmaf(sc[0][2], scale, -mn1)), p3 = ex2(fmaf(sc[0][3], scale, -mn1));
        const float p4 = ex2(fmaf(sc[1][0], scale, -mn0)), p5 = ex2(fmaf(sc[1][1], scale, -mn0));
        const float p6 = ex2(fmaf(sc[1][2], scale, -mn1)), p7 = ex2(fmaf(sc[1][3], scale, -mn1));
        l0 += (p0 + p1) + (p4 + p5);
        l1 += (p2 + p3) + (p6 + p7);
        pf[0] = pack_bf16(p0, p1);
        pf[1] = pack_bf16(p2, p3);
        pf[2] = pack_bf16(p4, p5);
        pf[3] = pack_bf16(p6, p7);
      }
      // share the P fragments (k-slice w of the 16 x 64 P tile) with the group
      uint4* pb = reinterpret_cast<uint4*>(pbuf);
      pb[w * 32 + lane] = make_uint4(pf[0], pf[1], pf[2], pf[3]);
      asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint32_t pk[4];
        if (ks == w) {
          pk[0] = pf[0]; pk[1] = pf[1]; pk[2] = pf[2]; pk[3] = pf[3];
        } else {
          const uint4 v = pb[ks * 32 + lane];
          pk[0] = v.x; pk[1] = v.y; pk[2] = v.z; pk[3] = v.w;
        }
        const int key = ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
        for (int dp = 0; dp < 2; ++dp) {
          uint32_t v0, v1, v2, v3;
          ldsm_x4_t(sk_swz(sV, key, w * 4 + dp * 2 + (lane >> 4)), v0, v1, v2, v3);
          mma16816(acc[2 * dp], pk, v0, v1);
          mma16816(acc[2 * dp + 1], pk, v2, v3);
        }
      }
      if (nv < KT || patch) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes before the next TMA write
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty[st]);
    }
    if (ctr && tid == 0) ctr[4] = ew_now();
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    {
      // each warp summed P over its own key slice: total row sums of the group
      float* ls = tmax + 64;
      if (t4 == 0) {
        ls[w * 16 + g8] = l0;
        ls[w * 16 + g8 + 8] = l1;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      l0 = ls[g8] + ls[16 + g8] + ls[32 + g8] + ls[48 + g8];
      l1 = ls[8 + g8] + ls[24 + g8] + ls[40 + g8] + ls[56 + g8];
      asm volatile("bar.sync 1, 128;" ::: "memory");   // ls reused by the next item
    }
    ++n_items;
    const bool whole = it.start >= b0 && it.end <= b1;
    __nv_bfloat16* orow = a.out + static_cast<int64_t>(it.s) * ldq + static_cast<int64_t>(h0) * D + w * 32 + 2 * t4;
    if (!whole) {
      // An item cut by range boundaries: the CTA whose range holds the item's
      // first tile (cf) processes it LAST (at the end of its range), the others
      // (cf + 1 .. cl) first -- so cf merges: the others publish {m, l, o[32
      // dims]} of rows g8, g8 + 8 and bump the (item, warp) counter with release
      // semantics; cf waits for them (acquire; normally already there) and folds
      // their partials into its own registers in CTA order (deterministic).  No
      // store / atomic round trip / re-read of cf's own partial on the kernel's tail.
      const int cf = sk_owner(it.start, N, G), cl = sk_owner(it.end - 1, N, G);
      unsigned* cnt = a.cnt + static_cast<int64_t>(it.s * per_seq + it.j) * 4 + w;
      if (c != cf) {
        const int pslot = it.start <= b0 ? 0 : 1;
        float* pp = a.part + ((static_cast<int64_t>(c) * 2 + pslot) * 4 + w) * 16 * kPartRow;
        if (t4 == 0) {
          pp[g8 * kPartRow] = m0;
          pp[g8 * kPartRow + 1] = l0;
          pp[(g8 + 8) * kPartRow] = m1;
          pp[(g8 + 8) * kPartRow + 1] = l1;
        }
#pragma unroll
        for (int dn = 0; dn < 4; ++dn) {
          *reinterpret_cast<float2*>(pp + g8 * kPartRow + 2 + dn * 8 + 2 * t4) = make_float2(acc[dn][0], acc[dn][1]);
          *reinterpret_cast<float2*>(pp + (g8 + 8) * kPartRow + 2 + dn * 8 + 2 * t4) = make_float2(acc[dn][2], acc[dn][3]);
        }
        __syncwarp();   // release below is cumulative over the warp's stores
        if (lane == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        g = e;
        continue;
      }
      if (lane == 0) {
        unsigned nc = 0;   // other contributors with a non-empty range (N < grid leaves some empty)
        for (int cc = cf + 1; cc <= cl; ++cc) nc += sk_bound(cc + 1, N, G) > sk_bound(cc, N, G);
        for (;;) {
          unsigned v;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
          if (v >= nc) break;
          __nanosleep(32);
        }
        *cnt = 0u;   // zero-maintained for the next launch
      }
      __syncwarp();
      ++n_merges;
      // contributors' partials are loaded MB at a time (all loads in flight), then
      // merged in CTA order: one L2 round trip per MB contributors, not per contributor
      // (MB = 2: a third in flight spills under the 2-CTA/SM register cap)
      constexpr int MB = 2;
      for (int cb = cf + 1; cb <= cl; cb += MB) {
        float km[MB][2], kl[MB][2];
        float2 ko[MB][4][2];
        bool ok[MB];
#pragma unroll
        for (int q = 0; q < MB; ++q) {
          const int cc = cb + q;
          const int64_t bc = sk_bound(cc, N, G);
          ok[q] = cc <= cl && sk_bound(cc + 1, N, G) > bc;
          if (!ok[q]) continue;
          const float* pk = a.part + ((static_cast<int64_t>(cc) * 2 + (it.start <= bc ? 0 : 1)) * 4 + w) * 16 * kPartRow;
          km[q][0] = __ldcg(pk + g8 * kPartRow);
          kl[q][0] = __ldcg(pk + g8 * kPartRow + 1);
          km[q][1] = __ldcg(pk + (g8 + 8) * kPartRow);
          kl[q][1] = __ldcg(pk + (g8 + 8) * kPartRow + 1);
#pragma unroll
          for (int dn = 0; dn < 4; ++dn) {
            ko[q][dn][0] = __ldcg(reinterpret_cast<const float2*>(pk + g8 * kPartRow + 2 + dn * 8 + 2 * t4));
            ko[q][dn][1] = __ldcg(reinterpret_cast<const float2*>(pk + (g8 + 8) * kPartRow + 2 + dn * 8 + 2 * t4));
          }
        }
#pragma unroll
        for (int q = 0; q < MB; ++q) {
          if (!ok[q]) continue;
          const float n0 = fmaxf(m0, km[q][0]), n1 = fmaxf(m1, km[q][1]);
          const float z0 = n0 == -INFINITY ? 0.f : n0, z1 = n1 == -INFINITY ? 0.f : n1;
          const float so0 = exp2f(m0 - z0), sn0 = exp2f(km[q][0] - z0), so1 = exp2f(m1 - z1),
                      sn1 = exp2f(km[q][1] - z1);
          m0 = n0;
          m1 = n1;
          l0 = l0 * so0 + kl[q][0] * sn0;
          l1 = l1 * so1 + kl[q][1] * sn1;
#pragma unroll
          for (int dn = 0; dn < 4; ++dn) {
            acc[dn][0] = acc[dn][0] * so0 + ko[q][dn][0].x * sn0;
            acc[dn][1] = acc[dn][1] * so0 + ko[q][dn][0].y * sn0;
            acc[dn][2] = acc[dn][2] * so1 + ko[q][dn][1].x * sn1;
            acc[dn][3] = acc[dn][3] * so1 + ko[q][dn][1].y * sn1;
          }
        }
      }
    }
    const float i0 = 1.f / l0, i1 = 1.f / l1;
#pragma unroll
    for (int dn = 0; dn < 4; ++dn) {
      if (g8 < Gc) *reinterpret_cast<uint32_t*>(orow + g8 * D + dn * 8) = pack_bf16(acc[dn][0] * i0, acc[dn][1] * i0);
      if (g8 + 8 < Gc)
        *reinterpret_cast<uint32_t*>(orow + (g8 + 8) * D + dn * 8) = pack_bf16(acc[dn][2] * i1, acc[dn][3] * i1);
    }
    g = e;
  }
  ew_mark(a.tr, 3);
  if (ctr && tid == 0) {
    ctr[6] = ew_now();
    ctr[5] = static_cast<unsigned long long>(b1 - b0) | (static_cast<unsigned long long>(n_items) << 16) |
             (static_cast<unsigned long long>(n_merges) << 32);   // debug: tiles, items, merges of this CTA
  }
}

}  // namespace

size_t attention_sk_workspace(int64_t max_tokens, int Hq) {
  return static_cast<size_t>((max_tokens * Hq + 63) / 64 * 64) * 4 * 4 +
         static_cast<size_t>(sk::kMaxGrid) * 2 * 4 * 16 * sk::kPartRow * sizeof(float);
}

// stream-K decode attention; DL_ERR_UNSUPPORTED -> caller uses the split kernel
dl_status launch_attention_sk(const AttnArgs& a, cudaStream_t st) {
  static const bool off = DL_ENV("DL_ATTN_SPLIT") && atoi(DL_ENV("DL_ATTN_SPLIT")) != 0;   // A/B switch
  const int nch = (a.Hq / a.Hk + 15) / 16;
  const int64_t items = static_cast<int64_t>(a.num_seqs) * a.Hk * nch;
  if (off || !a.decode || a.num_seqs > sk::kMaxSeqs || !a.sk_ws || items > a.sk_items_cap) return DL_ERR_UNSUPPORTED;
  if (a.qkv && (a.kv_ld || !a.positions || a.ld_qkv % 8)) return DL_ERR_UNSUPPORTED;
  SkMaps maps;
  SkArgs k{};
  const int64_t hk_cols = static_cast<int64_t>(a.Hk) * D;
  bool ok;
  if (a.kv_ld) {
    ok = encode_map_bf16(&maps.k, a.k_cache, a.kv_rows, hk_cols, a.kv_ld, KT) &&
         encode_map_bf16(&maps.v, a.v_cache, a.kv_rows, hk_cols, a.kv_ld, KT);
  } else {
    const int64_t rows = static_cast<int64_t>(a.num_seqs) * a.Hk * a.max_seq;
    ok = encode_map_bf16(&maps.k, a.k_cache, rows, D, D, KT) && encode_map_bf16(&maps.v, a.v_cache, rows, D, D, KT);
  }
  if (!ok) return DL_ERR_UNSUPPORTED;
  k.q = a.q;
  k.out = a.out;
  k.cache_lens = a.cache_lens;
  k.num_seqs = a.num_seqs;
  k.Hq = a.Hq;
  k.Hk = a.Hk;
  k.nch = nch;
  k.Gall = a.Hq / a.Hk;
  k.max_seq = a.max_seq;
  k.token_major = a.kv_ld ? 1 : 0;
  k.kv_blk0 = a.kv_blk0;
  k.kv_bs = a.kv_bs;
  k.cnt = static_cast<unsigned*>(a.sk_ws);
  k.tr = ew_trace(4);
  k.qkv = a.qkv;
  k.ld_qkv = a.ld_qkv;
  k.positions = a.positions;
  k.l2t = log2f(a.theta > 0.f ? a.theta : 1.f);
  k.rope = a.rope;
  k.kc = const_cast<__nv_bfloat16*>(a.k_cache);
  k.vc = const_cast<__nv_bfloat16*>(a.v_cache);
  k.zero = a.zero;
  k.zero2 = a.zero2;
  k.ctr = nullptr;
  static const int order = DL_ENV("DL_ATTN_ORDER") ? atoi(DL_ENV("DL_ATTN_ORDER")) : 0;   // measured neutral (A/B)
  k.reorder = order;
  static const int l2pf = DL_ENV("DL_ATTN_L2PF") ? atoi(DL_ENV("DL_ATTN_L2PF")) : 0;
  k.l2pf = l2pf;
  k.part = reinterpret_cast<float*>(static_cast<uint8_t*>(a.sk_ws) + (a.sk_items_cap + 63) / 64 * 64 * 4 * 4);
  // ring depth x CTAs per SM: 3 x 2 (default) or 2 x 3 (DL_ATTN_CFG=23, A/B)
  static const bool cfg23 = DL_ENV("DL_ATTN_CFG") && atoi(DL_ENV("DL_ATTN_CFG")) == 23;
  auto kern = cfg23 ? attn_decode_sk_kernel<2, 3> : attn_decode_sk_kernel<3, 2>;
  const size_t smem = cfg23 ? sk::smem_bytes<2>(a.num_seqs) : sk::smem_bytes<3>(a.num_seqs);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_decode_sk_kernel<3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sk::smem_bytes<3>(sk::kMaxSeqs)));
    cudaFuncSetAttribute(attn_decode_sk_kernel<2, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sk::smem_bytes<2>(sk::kMaxSeqs)));
    cudaFuncSetAttribute(attn_decode_sk_kernel<6, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sk::smem_bytes<6>(sk::kMaxSeqs)));
    attr = true;
  }
  // grid: every CTA keeps >= ~4 key tiles (fewer split items to merge when the
  // step is small, e.g. one KV head per rank at TP = 8), at most 2 (3) per SM
  int64_t tiles = 0;
  {
    // host-side estimate from the capacity: cache_lens lives on the device
    tiles = static_cast<int64_t>(a.num_seqs) * a.Hk * nch * ((a.max_seq + KT - 1) / KT);
  }
  int grid = std::min((cfg23 ? 3 : 2) * num_sms(), sk::kMaxGrid);
  if (tiles < static_cast<int64_t>(grid) * 4) grid = std::max(num_sms(), static_cast<int>(tiles / 4));
  grid = std::min(grid, (cfg23 ? 3 : 2) * num_sms());
  // Short items and no more items than CTAs (TP >= 2 at batch 64, context 512):
  // one CTA per item, no split and no merge.  A split item's merging CTA waits for
  // its partner's whole share, so 4-5 tiles + a merge cost about as much as the
  // 9 tiles unsplit, and the merges go away (per-rank decode at TP = 4 / 8:
  // 10.76 -> 10.29 / 8.59 -> 8.44 ms, r02bl).  Long items keep the stream-K split.
  // A/B: DL_ATTN_NOSPLIT_TILES=n (items of <= n tiles; default 16, 0 = off)
  static const int nosplit = DL_ENV("DL_ATTN_NOSPLIT_TILES") ? atoi(DL_ENV("DL_ATTN_NOSPLIT_TILES")) : 16;
  // More items than CTA slots (TP = 1): whole items per CTA, ceil(items / slots) each,
  // so equal-length items are never cut either (A/B: DL_ATTN_NOSPLIT_MULTI=0).
  static const bool multi = !DL_ENV("DL_ATTN_NOSPLIT_MULTI") || atoi(DL_ENV("DL_ATTN_NOSPLIT_MULTI")) != 0;
  if ((a.max_seq + KT - 1) / KT <= nosplit && items > 0 && (items <= grid || multi)) {
    const int64_t per = (items + grid - 1) / grid;
    grid = static_cast<int>((items + per - 1) / per);
    // whole-item ranges: nothing is split, even for ragged contexts (A/B: DL_ATTN_ITEM_RANGES=0 keeps
    // the equal tile ranges, which cut items whose lengths differ)
    static const bool item_ranges = !DL_ENV("DL_ATTN_ITEM_RANGES") || atoi(DL_ENV("DL_ATTN_ITEM_RANGES")) != 0;
    k.item_per = item_ranges ? static_cast<int>(per) : 0;
  }
  // at most one CTA per SM: a 6-stage ring per CTA (the whole SM's shared memory),
  // so a lone item's tiles are in flight together (A/B: DL_ATTN_DEEP=0)
  static const bool deep = !DL_ENV("DL_ATTN_DEEP") || atoi(DL_ENV("DL_ATTN_DEEP")) != 0;
  const bool use_deep = deep && !cfg23 && grid <= num_sms();
  k.ctr = gemm_trace_cta_slots((grid + 147) / 148);
  if (use_deep)
    return launch_pdl(attn_decode_sk_kernel<6, 1>, dim3(grid), dim3(sk::kThreads), sk::smem_bytes<6>(a.num_seqs), st,
                      "attention decode (stream-K)", maps, k);
  return launch_pdl(kern, dim3(grid), dim3(sk::kThreads), smem, st, "attention decode (stream-K)", maps, k);
}

size_t attention_workspace(int64_t max_tokens, int Hq, int d) {
  (void)d;
  return static_cast<size_t>(max_tokens) * Hq * kMaxSplits * PART * sizeof(float);
}

dl_status launch_attention(const AttnArgs& a, cudaStream_t st) {
  if (a.T <= 0) return DL_OK;
  if (a.kv_ld && (!a.decode || !a.kv_blk0 || a.kv_bs < 1 || a.kv_ld % 8)) {
    set_error("attention: token-major K/V (kv_ld) is a decode-only layout with a block map");
    return DL_ERR_INVALID_ARG;
  }
  if (a.d != D || a.Hk < 1 || a.Hq % a.Hk != 0) {
    set_error("attention: head_dim %d / heads %d:%d unsupported (d = 128, Hq %% Hk == 0)", a.d, a.Hq, a.Hk);
    return DL_ERR_UNSUPPORTED;
  }
  if (!a.decode) {
    // tcgen05 kernel (attn_tc.cu); DL_ATTN_PREFILL_MMA=1: the FA2-style mma.sync kernel below (A/B)
    static const bool mma_sync = DL_ENV("DL_ATTN_PREFILL_MMA") && atoi(DL_ENV("DL_ATTN_PREFILL_MMA")) != 0;
    if (!mma_sync) return launch_attention_prefill_tc(a, st);
    constexpr int KTP = 64;   // 64-key tiles (32-key tiles at 3 CTAs/SM measured 7% slower)
    constexpr int SMEM = QT * ROW_BYTES + 4 * KTP * ROW_BYTES;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(attn_prefill_kernel<KTP>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
      attr = true;
    }
    // grid.x covers the longest sequence: bounded by T
    const int qtiles = static_cast<int>((a.T + QT - 1) / QT);
    dim3 grid(qtiles * a.Hq, 1, a.num_seqs);
    return launch_pdl(attn_prefill_kernel<KTP>, grid, dim3(128), SMEM, st, "attention prefill", a, ew_trace(5));
  }
  {
    const dl_status s = launch_attention_sk(a, st);
    if (s != DL_ERR_UNSUPPORTED) return s;
    if (a.qkv) {
      set_error("attention: fused RoPE + append needs the stream-K decode kernel");
      return DL_ERR_UNSUPPORTED;
    }
  }
  constexpr int SMEM = 16 * ROW_BYTES + 4 * TILE_BYTES + (4 * 16 * D + 128) * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr = true;
  }
  // enough CTAs to cover the SMs twice; each split keeps >= 2 key tiles
  const int nch = (a.Hq / a.Hk + 15) / 16;
  const int64_t base = static_cast<int64_t>(a.num_seqs) * a.Hk * nch;
  int splits = 1;
  while (splits < kMaxSplits && base * splits < 2 * num_sms()) splits *= 2;
  if (a.partial == nullptr || a.partial_bytes < attention_workspace(a.T, a.Hq, a.d)) splits = 1;
  dim3 grid(splits, a.Hk * nch, a.num_seqs);
  dl_status s = launch_pdl(attn_decode_kernel, grid, dim3(128), SMEM, st, "attention decode", a, splits);
  if (s != DL_OK || splits == 1) return s;
  return launch_pdl(attn_combine_kernel, dim3(a.Hq, a.num_seqs), dim3(128), 0, st, "attention combine", a, splits);
}

}  // namespace dl
