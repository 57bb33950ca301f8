// SIMT skinny low-rank chain for T <= 16 tokens and for fp32 (true FFMA):
//   stage 1  Z[t][j] = sum_l B[j][l] X[t][l]      ("Bx")
//   stage 2  Y[t][i] (+)= sum_j A[i][j] Z[t][j]   ("A(Bx)")
// Each warp owns ROWS weight rows and streams them from HBM with 16-byte
// coalesced loads (the factors are read exactly once); the T token vectors
// ride in registers; the per-row dot products are finished with warp
// shuffles.  Z is held in fp32 storage (workspace row, L2-resident, or shared
// memory) but, for bf16 inputs, rounded to bf16 first -- the same single
// rounding the tensor-core paths apply (reading c10), so a token's output does
// not depend on which path the batch size selects.
// When the whole chain is small (k <= 1024) a single fused CTA keeps Z in
// shared memory and never writes it out.
#include <type_traits>

#include "dl_internal.h"

namespace dl {
namespace {

constexpr int kWarps = 8;
constexpr int kRows = 2;   // weight rows per warp
constexpr int kMaxT = 16;

template <typename E> struct Vec;
template <> struct Vec<float> { static constexpr int N = 4; };
template <> struct Vec<__nv_bfloat16> { static constexpr int N = 8; };

__device__ __forceinline__ void load_vec(const float* p, float* v) {
  float4 x = __ldg(reinterpret_cast<const float4*>(p));
  v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}
__device__ __forceinline__ void load_vec(const __nv_bfloat16* p, float* v) {
  uint4 x = __ldg(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&x);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(b[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
// generic-address loads for the activation operand (global or shared)
__device__ __forceinline__ void load_act(const float* p, float* v) {
  float4 x = *reinterpret_cast<const float4*>(p);
  v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}
__device__ __forceinline__ void load_act(const __nv_bfloat16* p, float* v) {
  uint4 x = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&x);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(b[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ void store_out(float* p, float v, int acc) { *p = acc ? *p + v : v; }
__device__ __forceinline__ void store_out(__nv_bfloat16* p, float v, int acc) {
  *p = __float2bfloat16_rn(acc ? __bfloat162float(*p) + v : v);
}

// in: activation rows [T x C] (type I, ld ldi); W rows [R x C] (type E).
// out[t][r] (type O, ld ldo).  Vector width follows E; I is read at the
// same column positions (I = float or E).
template <typename E, typename I, typename O, int TT>
__device__ void gemv_warp_rows(const E* __restrict__ W, int64_t ldw, int R, int C,
                               const I* __restrict__ in, int64_t ldi, int T,
                               O* __restrict__ out, int64_t ldo, int accumulate, int row0) {
  constexpr int V = Vec<E>::N;
  const int lane = threadIdx.x & 31;
  float acc[kRows][TT];
#pragma unroll
  for (int r = 0; r < kRows; ++r)
#pragma unroll
    for (int t = 0; t < TT; ++t) acc[r][t] = 0.f;
  const int Cv = C - C % V;
  for (int c = lane * V; c < Cv; c += 32 * V) {
    float w[kRows][V];
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      if (row0 + r < R) load_vec(W + static_cast<int64_t>(row0 + r) * ldw + c, w[r]);
      else
#pragma unroll
        for (int e = 0; e < V; ++e) w[r][e] = 0.f;
    }
#pragma unroll
    for (int t = 0; t < TT; ++t) {
      if (t < T) {
        float x[V];
        if constexpr (sizeof(I) == sizeof(E)) {
          load_act(reinterpret_cast<const E*>(in) + t * ldi + c, x);
        } else {
#pragma unroll
          for (int e = 0; e < V; e += 4) load_act(reinterpret_cast<const float*>(in) + t * ldi + c + e, x + e);
        }
#pragma unroll
        for (int r = 0; r < kRows; ++r)
#pragma unroll
          for (int e = 0; e < V; ++e) acc[r][t] = fmaf(w[r][e], x[e], acc[r][t]);
      }
    }
  }
  for (int c = Cv + lane; c < C; c += 32) {   // ragged tail
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      if (row0 + r >= R) continue;
      const float w = to_f(W[static_cast<int64_t>(row0 + r) * ldw + c]);
#pragma unroll
      for (int t = 0; t < TT; ++t)
        if (t < T) acc[r][t] = fmaf(w, to_f(in[t * ldi + c]), acc[r][t]);
    }
  }
#pragma unroll
  for (int r = 0; r < kRows; ++r)
#pragma unroll
    for (int t = 0; t < TT; ++t) {
      float v = acc[r][t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      acc[r][t] = v;
    }
  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      if (row0 + r >= R) continue;
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        float v = acc[r][t];
        // stage 1 of a bf16 chain (fp32 Z storage): round Z to bf16
        if constexpr (std::is_same<O, float>::value && std::is_same<E, __nv_bfloat16>::value)
          v = __bfloat162float(__float2bfloat16_rn(v));
        if (t < T) store_out(out + t * ldo + row0 + r, v, accumulate);
      }
    }
  }
}

template <typename E, typename I, typename O, int TT>
__global__ void __launch_bounds__(kWarps * 32)
    gemv_kernel(const E* __restrict__ W, int64_t ldw, int R, int C, const I* __restrict__ in, int64_t ldi,
                int T, O* __restrict__ out, int64_t ldo, int accumulate) {
  pdl_trigger();   // successor may launch now; it waits for us before reading
  pdl_wait();
  const int warp = threadIdx.x >> 5;
  const int row0 = (blockIdx.x * kWarps + warp) * kRows;
  if (row0 >= R) return;
  gemv_warp_rows<E, I, O, TT>(W, ldw, R, C, in, ldi, T, out, ldo, accumulate, row0);
}

// Fused small chain: Z in shared memory (k <= 1024, T <= 16), never written
// out.  Every CTA (32 warps) computes the whole Z = X B^T (B is small and
// L2-resident after the first CTA touches it: one pass of 64 rows at k <= 64)
// and then its own 64-row slice of Y = Z A^T, so the chain costs two dependent
// memory round trips instead of one per 16 rows (BASELINE config 1: 20 -> ~5 us).
constexpr int kSmallWarps = 32;
constexpr int kSmallRowsPerCta = kSmallWarps * kRows;
template <typename E, int TT>
__global__ void __launch_bounds__(kSmallWarps * 32)
    chain_small_kernel(const E* __restrict__ X, int64_t ldx, const E* __restrict__ A, int64_t lda,
                       const E* __restrict__ B, int64_t ldb, E* __restrict__ Y, int64_t ldy, int T,
                       int m, int n, int k, int accumulate) {
  extern __shared__ float zs[];   // [T x k_pad]
  pdl_trigger();   // successor may launch now; it waits for us before reading
  pdl_wait();
  const int kp = (k + 3) & ~3;
  const int warp = threadIdx.x >> 5;
  for (int row0 = warp * kRows; row0 < k; row0 += kSmallWarps * kRows)
    gemv_warp_rows<E, E, float, TT>(B, ldb, k, n, X, ldx, T, zs, kp, 0, row0);
  __syncthreads();
  const int row0 = blockIdx.x * kSmallRowsPerCta + warp * kRows;
  if (row0 < m) gemv_warp_rows<E, float, E, TT>(A, lda, m, k, zs, kp, T, Y, ldy, accumulate, row0);
}

template <typename E, int TT>
dl_status run(const void* X, int64_t ldx, const void* A, int64_t lda, const void* B, int64_t ldb, void* Y,
              int64_t ldy, int64_t T, int64_t m, int64_t n, int64_t k, int accumulate, void* zbuf,
              cudaStream_t st) {
  const E* x = static_cast<const E*>(X);
  const E* a = static_cast<const E*>(A);
  const E* b = static_cast<const E*>(B);
  E* y = static_cast<E*>(Y);
  const int rows_per_cta = kWarps * kRows;
  if (k <= 1024 && (m + n) * k <= (1 << 16) && T * ((k + 3) & ~3) * 4 <= 48 * 1024) {
    const int kp = static_cast<int>((k + 3) & ~3);
    size_t smem = sizeof(float) * static_cast<size_t>(T) * kp;
    return launch_pdl(chain_small_kernel<E, TT>, dim3(static_cast<int>((m + kSmallRowsPerCta - 1) / kSmallRowsPerCta)),
                      dim3(kSmallWarps * 32), smem, st, "simt chain_small", x, ldx, a, lda, b, ldb, y, ldy, (int)T,
                      (int)m, (int)n, (int)k, accumulate);
  }
  float* z = static_cast<float*>(zbuf);
  const int64_t ldz = (k + 3) & ~3;
  dl_status s = launch_pdl(gemv_kernel<E, E, float, TT>, dim3(static_cast<int>((k + rows_per_cta - 1) / rows_per_cta)),
                           dim3(kWarps * 32), 0, st, "simt stage1", b, ldb, (int)k, (int)n, x, ldx, (int)T, z, ldz, 0);
  if (s != DL_OK) return s;
  return launch_pdl(gemv_kernel<E, float, E, TT>, dim3(static_cast<int>((m + rows_per_cta - 1) / rows_per_cta)),
                    dim3(kWarps * 32), 0, st, "simt stage2", a, lda, (int)m, (int)k, z, ldz, (int)T, y, ldy, accumulate);
}

template <typename E>
dl_status dispatch(const void* X, int64_t ldx, const void* A, int64_t lda, const void* B, int64_t ldb, void* Y,
                   int64_t ldy, int64_t T, int64_t m, int64_t n, int64_t k, int acc, void* zbuf,
                   cudaStream_t st) {
  if (T <= 4) return run<E, 4>(X, ldx, A, lda, B, ldb, Y, ldy, T, m, n, k, acc, zbuf, st);
  if (T <= 8) return run<E, 8>(X, ldx, A, lda, B, ldb, Y, ldy, T, m, n, k, acc, zbuf, st);
  return run<E, 16>(X, ldx, A, lda, B, ldb, Y, ldy, T, m, n, k, acc, zbuf, st);
}

}  // namespace

dl_status simt_lowrank(const void* X, int64_t ldx, const void* A, int64_t lda, const void* B, int64_t ldb,
                       void* Y, int64_t ldy, int64_t T, int64_t m, int64_t n, int64_t k, dl_dtype dt,
                       int accumulate, void* zbuf, cudaStream_t st) {
  if (T <= 0) return DL_OK;
  if (T > kMaxT) {
    set_error("SIMT chain supports T <= %d (got %lld)", kMaxT, (long long)T);
    return DL_ERR_UNSUPPORTED;
  }
  if (dt == DL_F32) return dispatch<float>(X, ldx, A, lda, B, ldb, Y, ldy, T, m, n, k, accumulate, zbuf, st);
  return dispatch<__nv_bfloat16>(X, ldx, A, lda, B, ldb, Y, ldy, T, m, n, k, accumulate, zbuf, st);
}

}  // namespace dl
