// Memory-bound block pieces (bf16 storage, fp32 math), each one pass over
// its tensors with 8/16-byte vector accesses and 2-D grids (row = token,
// x = column group) so no per-element 64-bit index division:
//   RMSNorm (LLaMA-3 pre-norm; reading c9), the epilogues that turn the fp32
//   rank-partial accumulators into the next operand (consume-and-clear: the
//   accumulator is zeroed as it is read so the next stream-K GEMM can
//   red.add into it without a separate memset), SiLU(gate)*up, residual add,
//   RoPE + KV-cache append ("in-place rotary position
//   embedding"), embedding gather and the all-gather un-permute.
// All kernels are PDL-aware (see dl_internal.h).
#include <math.h>

#include <algorithm>
#include <stdlib.h>

#include "dl_internal.h"

namespace dl {
namespace {
unsigned long long* g_ew_buf = nullptr;   // host copy of the trace buffer pointer
int g_ew_next = 0;
}  // namespace

dl_status set_ew_trace(void* buf) {
  g_ew_buf = static_cast<unsigned long long*>(buf);
  g_ew_next = 0;
  return DL_OK;
}
EwTrace ew_trace(int kind) {
  EwTrace t{nullptr, -1, kind};
  if (g_ew_buf) {
    t.buf = g_ew_buf;
    t.slot = g_ew_next++;
  }
  return t;
}

void rn_early_init();   // A/B flag of the small kernels' load / side-clear order (below)

namespace {

// SideZero job: 16-byte zero stores spread over every thread of the grid.
__device__ __forceinline__ void side_zero(const SideZero& z) {
  if (!z.p) return;
  const int64_t per_row = z.row_bytes / 16, total = z.rows * per_row;
  const int64_t nthr = static_cast<int64_t>(gridDim.x) * gridDim.y * blockDim.x;
  for (int64_t i = (static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += nthr) {
    const int64_t r = i / per_row;
    *reinterpret_cast<uint4*>(static_cast<uint8_t*>(z.p) + r * z.ld + (i - r * per_row) * 16) = make_uint4(0, 0, 0, 0);
  }
}

// residual + RMSNorm: norm weight loaded before griddepcontrol.wait, side clears after
// the row loads (A/B: DL_RN_EARLY=0 restores the old order); set once by the host
__constant__ int g_rn_early = 1;
__device__ __forceinline__ bool rn_early() { return g_rn_early != 0; }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// one CTA (256 threads) per row; h % 8 == 0
__global__ void __launch_bounds__(256) rmsnorm_kernel(const __nv_bfloat16* __restrict__ x,
                                                      const __nv_bfloat16* __restrict__ g,
                                                      __nv_bfloat16* __restrict__ y, int h, float eps) {
  pdl_trigger();   // successor may launch now; it waits for us before reading
  pdl_wait();
  __shared__ float red[8];
  const int64_t t = blockIdx.x;
  const uint4* xr = reinterpret_cast<const uint4*>(x + t * h);
  float ss = 0.f;
  for (int i = threadIdx.x; i < h / 8; i += blockDim.x) {
    uint4 v = xr[i];
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f = __bfloat1622float2(b[e]);
      ss += f.x * f.x + f.y * f.y;
    }
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / static_cast<float>(h) + eps);
  const uint4* gr = reinterpret_cast<const uint4*>(g);
  uint4* yr = reinterpret_cast<uint4*>(y + t * h);
  for (int i = threadIdx.x; i < h / 8; i += blockDim.x) {
    uint4 v = xr[i], gv = gr[i], o;
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
    const __nv_bfloat162* gb = reinterpret_cast<const __nv_bfloat162*>(&gv);
    __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f = __bfloat1622float2(b[e]);
      float2 w = __bfloat1622float2(gb[e]);
      ob[e] = __floats2bfloat162_rn(f.x * inv * w.x, f.y * inv * w.y);
    }
    yr[i] = o;
  }
}

// x = bf16(x + acc) (acc consumed and cleared), then y = rmsnorm(x) * g: the
// o-projection residual and the MLP pre-norm in one pass (one CTA per row).
// The norm reads the bf16-rounded x, exactly as the two separate kernels did.
// 8 consecutive accumulator values, zeroed as they are read (fp32 or bf16 accumulator)
__device__ __forceinline__ void take8(float* p, float* o) {
  const float4 a0 = *reinterpret_cast<float4*>(p), a1 = *reinterpret_cast<float4*>(p + 4);
  *reinterpret_cast<float4*>(p) = make_float4(0.f, 0.f, 0.f, 0.f);
  *reinterpret_cast<float4*>(p + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
  o[0] = a0.x; o[1] = a0.y; o[2] = a0.z; o[3] = a0.w; o[4] = a1.x; o[5] = a1.y; o[6] = a1.z; o[7] = a1.w;
}
__device__ __forceinline__ void take8(__nv_bfloat16* p, float* o) {
  const uint4 v = *reinterpret_cast<uint4*>(p);
  *reinterpret_cast<uint4*>(p) = make_uint4(0u, 0u, 0u, 0u);
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(b[e]);
    o[2 * e] = f.x;
    o[2 * e + 1] = f.y;
  }
}
// One CTA (1,024 threads) per row, h <= 16,384 (h % 8 == 0): every thread
// issues all its loads (accumulator, x, gamma) before any math, so the row
// costs one memory round trip plus the block reduction; x and the norm
// input stay in registers.
constexpr int kRnThreads = 1024;
constexpr int kRnChunks = 2;   // 8-element chunks per thread
template <typename Acc>
__global__ void __launch_bounds__(kRnThreads) residual_rmsnorm_kernel(Acc* __restrict__ acc, int64_t lda,
                                                                      __nv_bfloat16* __restrict__ x,
                                                                      const __nv_bfloat16* __restrict__ g,
                                                                      __nv_bfloat16* __restrict__ y, int h, float eps,
                                                                      SideZero z, SideZero z2, EwTrace tr) {
  ew_mark(tr, 1);
  pdl_trigger();   // successor may launch now; it waits for us before reading
  __shared__ float red[32];
  const int64_t t = blockIdx.x;
  Acc* ar = acc + t * lda;
  uint4* xr = reinterpret_cast<uint4*>(x + t * h);
  const uint4* gr = reinterpret_cast<const uint4*>(g);
  const int n8 = h / 8;
  float av[kRnChunks][8];
  uint4 v[kRnChunks], gv[kRnChunks];
  const bool early = rn_early();
  if (early) {
#pragma unroll
    for (int k = 0; k < kRnChunks; ++k) {   // the norm weight is not written inside the step
      const int i = threadIdx.x + k * kRnThreads;
      if (i < n8) gv[k] = gr[i];
    }
  }
  pdl_wait();
  ew_mark(tr, 2);
  if (!early) {
    side_zero(z);
    side_zero(z2);
  }
#pragma unroll
  for (int k = 0; k < kRnChunks; ++k) {
    const int i = threadIdx.x + k * kRnThreads;
    if (i < n8) {
      if (acc) {
        take8(ar + 8 * i, av[k]);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) av[k][e] = 0.f;
      }
      v[k] = xr[i];
      if (!early) gv[k] = gr[i];
    }
  }
  if (early) {   // side clears after this row's loads are in flight (they never alias them)
    side_zero(z);
    side_zero(z2);
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kRnChunks; ++k) {
    const int i = threadIdx.x + k * kRnThreads;
    if (i >= n8) continue;
    __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&v[k]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f = __bfloat1622float2(b[e]);
      b[e] = __floats2bfloat162_rn(f.x + av[k][2 * e], f.y + av[k][2 * e + 1]);
      f = __bfloat1622float2(b[e]);   // the norm reads the bf16-rounded x
      ss += f.x * f.x + f.y * f.y;
    }
    if (acc) xr[i] = v[k];
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float s2 = red[threadIdx.x];
    s2 = warp_sum(s2);
    if (threadIdx.x == 0) red[0] = s2;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / static_cast<float>(h) + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + t * h);
#pragma unroll
  for (int k = 0; k < kRnChunks; ++k) {
    const int i = threadIdx.x + k * kRnThreads;
    if (i >= n8) continue;
    uint4 o;
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v[k]);
    const __nv_bfloat162* gb = reinterpret_cast<const __nv_bfloat162*>(&gv[k]);
    __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(b[e]);
      const float2 w = __bfloat1622float2(gb[e]);
      ob[e] = __floats2bfloat162_rn(f.x * inv * w.x, f.y * inv * w.y);
    }
    yr[i] = o;
  }
  __syncthreads();
  ew_mark(tr, 3);
}

// Plain RMSNorm for many rows (prefill): 4 rows per CTA, 256 threads per row,
// each thread holding its 4 chunks of 8 in registers (h <= 8192, h % 2048 == 0
// not required: chunks past h are skipped); all loads issued before the
// per-row reduction (named barrier per row group).
constexpr int kRrRows = 4;
constexpr int kRrThreads = 256;
constexpr int kRrChunks = 4;
__global__ void __launch_bounds__(kRrRows * kRrThreads) rmsnorm_rows_kernel(const __nv_bfloat16* __restrict__ x,
                                                                         const __nv_bfloat16* __restrict__ g,
                                                                         __nv_bfloat16* __restrict__ y, int64_t T,
                                                                         int h, float eps, EwTrace tr) {
  ew_mark(tr, 1);
  pdl_trigger();   // successor may launch now; it waits for us before reading
  pdl_wait();
  ew_mark(tr, 2);
  __shared__ float red[kRrRows][8];
  const int rg = threadIdx.x / kRrThreads, lt = threadIdx.x % kRrThreads;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kRrRows + rg;
  const bool row_ok = t < T;
  const int n8 = h / 8;
  const uint4* xr = reinterpret_cast<const uint4*>(x + (row_ok ? t : 0) * h);
  const uint4* gr = reinterpret_cast<const uint4*>(g);
  uint4 v[kRrChunks], gv[kRrChunks];
#pragma unroll
  for (int k = 0; k < kRrChunks; ++k) {
    const int i = lt + k * kRrThreads;
    if (row_ok && i < n8) {
      v[k] = xr[i];
      gv[k] = gr[i];
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kRrChunks; ++k) {
    const int i = lt + k * kRrThreads;
    if (!row_ok || i >= n8) continue;
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v[k]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(b[e]);
      ss += f.x * f.x + f.y * f.y;
    }
  }
  ss = warp_sum(ss);
  if ((lt & 31) == 0) red[rg][lt >> 5] = ss;
  asm volatile("bar.sync %0, %1;" ::"r"(1 + rg), "r"(kRrThreads) : "memory");
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < kRrThreads / 32; ++w) tot += red[rg][w];
  if (!row_ok) return;
  const float inv = rsqrtf(tot / static_cast<float>(h) + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + t * h);
#pragma unroll
  for (int k = 0; k < kRrChunks; ++k) {
    const int i = lt + k * kRrThreads;
    if (i >= n8) continue;
    uint4 o;
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v[k]);
    const __nv_bfloat162* gb = reinterpret_cast<const __nv_bfloat162*>(&gv[k]);
    __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(b[e]);
      const float2 w = __bfloat1622float2(gb[e]);
      ob[e] = __floats2bfloat162_rn(f.x * inv * w.x, f.y * inv * w.y);
    }
    yr[i] = o;
  }
  ew_mark(tr, 3);
}

// act[t][c..c+7] = bf16(silu(gate) * up) from the fp32 stage-2 accumulator
// (gate at column c, up at m + c; both consumed and cleared).  Flat item
// space (t, 8-column group), grid-stride, kSiluU items per thread with every
// load issued before any store.
constexpr int kSiluU = 4;
// 8 accumulator values at p (fp32 or bf16), then zero them
__device__ __forceinline__ void ld8(const float* p, float* o) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}
__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float* o) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(b[e]);
    o[2 * e] = f.x;
    o[2 * e + 1] = f.y;
  }
}
__device__ __forceinline__ void zero8(float* p) {
  *reinterpret_cast<float4*>(p) = make_float4(0.f, 0.f, 0.f, 0.f);
  *reinterpret_cast<float4*>(p + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
}
__device__ __forceinline__ void zero8(__nv_bfloat16* p) { *reinterpret_cast<uint4*>(p) = make_uint4(0u, 0u, 0u, 0u); }

// SiLU through one MUFU op: g * sigmoid(g) = r + r * tanh(r), r = g / 2
// (tanh.approx: relative error ~2^-11, below the bf16 rounding of the result);
// exp + reciprocal took two MUFU ops per element, which bound the 58.7 M-element
// prefill SiLU (2,048 x 28,672) as much as its 352 MB of traffic.
__device__ __forceinline__ float silu_tanh(float g) {
  const float r = 0.5f * g;
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(r));
  return fmaf(r, t, r);
}

// 2-D grid (column blocks, tokens): row t = blockIdx.y, thread items
// c = blockIdx.x * 256 + tid + u * gridDim.x * 256 (8 columns each) -- no
// per-item integer division; fast sigmoid (silu_tanh).
template <typename Acc>
__global__ void __launch_bounds__(256) silu_mul_kernel(Acc* __restrict__ acc, int64_t lda, __nv_bfloat16* __restrict__ out,
                                                       int64_t ldo, int m, int T, int relu, int clear, SideZero z,
                                                       EwTrace tr) {
  ew_mark(tr, 1);
  pdl_trigger();   // successor may launch now; it waits for us before reading
  pdl_wait();
  ew_mark(tr, 2);
  const bool early = rn_early();   // side clears after the loads are in flight (DL_RN_EARLY)
  if (!early) side_zero(z);
  const int per_row = m / 8;
  const int64_t t = blockIdx.y;
  Acc* row = acc + t * lda;
  __nv_bfloat16* orow = out + t * ldo;
  const int uoff = relu ? 0 : m;
  const int stride = gridDim.x * blockDim.x;
  float gv[kSiluU][8], uv[kSiluU][8];
#pragma unroll
  for (int u = 0; u < kSiluU; ++u) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x + u * stride;
    if (i < per_row) {
      ld8(row + uoff + i * 8, uv[u]);
      if (!relu) ld8(row + i * 8, gv[u]);
    }
  }
  if (early) side_zero(z);
#pragma unroll
  for (int u = 0; u < kSiluU; ++u) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x + u * stride;
    if (i >= per_row) continue;
    if (clear) zero8(row + uoff + i * 8);
    float o[8];
    if (relu) {
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = fmaxf(uv[u][e], 0.f);
    } else {
      if (clear) zero8(row + i * 8);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = silu_tanh(gv[u][e]) * uv[u][e];
    }
    uint4 pk;
    __nv_bfloat162* pb = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
    for (int e = 0; e < 4; ++e) pb[e] = __floats2bfloat162_rn(o[2 * e], o[2 * e + 1]);
    *reinterpret_cast<uint4*>(orow + i * 8) = pk;
  }
  __syncthreads();
  ew_mark(tr, 3);
}
template <typename Acc>
dl_status launch_silu_flat(Acc* acc, int64_t lda, __nv_bfloat16* act, int64_t ldo, int64_t T, int64_t m, int relu,
                           cudaStream_t st, const SideZero& z, int clear = 1) {
  rn_early_init();
  const int per_row = static_cast<int>(m / 8);
  const int gx = (per_row + 256 * kSiluU - 1) / (256 * kSiluU);
  return launch_pdl(silu_mul_kernel<Acc>, dim3(gx > 0 ? gx : 1, static_cast<unsigned>(T)), dim3(256), 0, st,
                    "silu_mul", acc, lda, act, ldo, static_cast<int>(m), static_cast<int>(T), relu, clear, z,
                    ew_trace(1));
}

// 2-D elementwise over [T x n] in groups of 4 columns: grid (ceil(n/4/256), T).
template <typename F>
__global__ void __launch_bounds__(256) ew4_kernel(int n4, F f, SideZero z, SideZero z2) {
  pdl_trigger();   // successor may launch now; it waits for us before reading
  pdl_wait();
  side_zero(z);
  side_zero(z2);
  const int c4 = blockIdx.x * blockDim.x + threadIdx.x;
  if (c4 < n4) f(static_cast<int64_t>(blockIdx.y), c4 * 4);
}

template <typename F>
dl_status launch_ew4(int64_t T, int64_t n, F f, cudaStream_t st, const char* what, const SideZero& z = SideZero{},
                     const SideZero& z2 = SideZero{}) {
  if (T <= 0 || n <= 0) return DL_OK;
  const int n4 = static_cast<int>(n / 4);
  dim3 grid((n4 + 255) / 256, static_cast<unsigned>(T));
  return launch_pdl(ew4_kernel<F>, grid, dim3(256), 0, st, what, n4, f, z, z2);
}

__device__ __forceinline__ float4 take4(float* p, int clear) {
  float4 v = *reinterpret_cast<float4*>(p);
  if (clear) *reinterpret_cast<float4*>(p) = make_float4(0.f, 0.f, 0.f, 0.f);
  return v;
}
__device__ __forceinline__ void store4(__nv_bfloat16* p, float a, float b, float c, float d) {
  uint2 o;
  reinterpret_cast<__nv_bfloat162*>(&o)[0] = __floats2bfloat162_rn(a, b);
  reinterpret_cast<__nv_bfloat162*>(&o)[1] = __floats2bfloat162_rn(c, d);
  *reinterpret_cast<uint2*>(p) = o;
}
__device__ __forceinline__ float4 load4(const __nv_bfloat16* p) {
  uint2 v = *reinterpret_cast<const uint2*>(p);
  float2 a = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(&v)[0]);
  float2 b = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(&v)[1]);
  return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ float silu(float g) { return g / (1.f + __expf(-g)); }

struct F32ToBf16 {
  float* acc; int64_t lda; __nv_bfloat16* out; int64_t ldo; int clear;
  __device__ void operator()(int64_t t, int c) const {
    float4 v = take4(acc + t * lda + c, clear);
    store4(out + t * ldo + c, v.x, v.y, v.z, v.w);
  }
};
struct ResidualAdd {
  float* acc; int64_t lda; __nv_bfloat16* x; int64_t ldx; int clear;
  __device__ void operator()(int64_t t, int c) const {
    float4 v = take4(acc + t * lda + c, clear);
    float4 r = load4(x + t * ldx + c);
    store4(x + t * ldx + c, r.x + v.x, r.y + v.y, r.z + v.z, r.w + v.w);
  }
};
__device__ __forceinline__ float4 take4(__nv_bfloat16* p, int clear) {
  const float4 v = load4(p);
  if (clear) *reinterpret_cast<uint2*>(p) = make_uint2(0u, 0u);
  return v;
}
struct ResidualAddBf16 {
  __nv_bfloat16* y; int64_t ldy; __nv_bfloat16* x; int64_t ldx; int clear;
  __device__ void operator()(int64_t t, int c) const {
    float4 v = take4(y + t * ldy + c, clear);
    float4 r = load4(x + t * ldx + c);
    store4(x + t * ldx + c, r.x + v.x, r.y + v.y, r.z + v.z, r.w + v.w);
  }
};
struct SiluMulF32 {
  float* acc; int64_t lda; __nv_bfloat16* out; int64_t ldo; int64_t m; int clear;
  __device__ void operator()(int64_t t, int c) const {
    float4 g = take4(acc + t * lda + c, clear);
    float4 u = take4(acc + t * lda + m + c, clear);
    store4(out + t * ldo + c, silu(g.x) * u.x, silu(g.y) * u.y, silu(g.z) * u.z, silu(g.w) * u.w);
  }
};
struct SiluMulBf16 {
  __nv_bfloat16* src; int64_t lds; __nv_bfloat16* out; int64_t ldo; int64_t m; int clear;
  __device__ void operator()(int64_t t, int c) const {
    float4 g = take4(src + t * lds + c, clear);
    float4 u = take4(src + t * lds + m + c, clear);
    store4(out + t * ldo + c, silu(g.x) * u.x, silu(g.y) * u.y, silu(g.z) * u.z, silu(g.w) * u.w);
  }
};

// Non-GLU MLP activation (OPT family): act = bf16(relu(up)).
struct ReluF32 {
  float* acc; int64_t lda; __nv_bfloat16* out; int64_t ldo; int clear;
  __device__ void operator()(int64_t t, int c) const {
    float4 u = take4(acc + t * lda + c, clear);
    store4(out + t * ldo + c, fmaxf(u.x, 0.f), fmaxf(u.y, 0.f), fmaxf(u.z, 0.f), fmaxf(u.w, 0.f));
  }
};
struct ReluBf16 {
  __nv_bfloat16* src; int64_t lds; __nv_bfloat16* out; int64_t ldo; int clear;
  __device__ void operator()(int64_t t, int c) const {
    float4 u = take4(src + t * lds + c, clear);
    store4(out + t * ldo + c, fmaxf(u.x, 0.f), fmaxf(u.y, 0.f), fmaxf(u.z, 0.f), fmaxf(u.w, 0.f));
  }
};

// RoPE + cache append.  Thread = (token, rotation pair p of the head dim):
// its angle pos * theta^(-2p/d) is computed once (before griddepcontrol.wait:
// positions, cache lengths and cu_seqlens are call inputs) and applied to
// kRopeHeads heads; grid (head groups, tokens), 128 threads = 2 x 64 pairs.
constexpr int kRopeHeads = 5;
constexpr int kRopeVec = 4;   // rotation pairs per thread (16-byte bf16 accesses; the body assumes 4)
__global__ void __launch_bounds__(128) rope_cache_kernel(RopeCacheArgs a, EwTrace tr) {
  ew_mark(tr, 1);
  pdl_trigger();   // successor may launch now; it waits for us before reading
  constexpr int TPH = 64 / kRopeVec;                    // threads per head (d = 128)
  const int heads = a.Hq + 2 * a.Hk;
  const int p0 = (threadIdx.x % TPH) * kRopeVec;        // first rotation pair of this thread
  const int hg = blockIdx.x * (128 / TPH) + threadIdx.x / TPH;
  const int h0 = (a.kv_only ? a.Hq : 0) + hg * kRopeHeads;   // kv_only: k and v heads only
  const int64_t t = blockIdx.y;
  const bool active = 2 * p0 < a.d && h0 < heads;
  float sn[kRopeVec], cs[kRopeVec];
#pragma unroll
  for (int q = 0; q < kRopeVec; ++q) {
    sn[q] = 0.f;
    cs[q] = 1.f;
  }
  if (active && a.rope && h0 < a.Hq + a.Hk) {
    // angle = pos * theta^(-2p/d) in fp32 (relative error ~1e-7, i.e. <= 3e-4 rad at
    // position 2048, far below bf16 resolution); rope_sincos (dl_internal.h)
    const float pos = static_cast<float>(a.positions[t]);
    const float l2t = log2f(a.theta);
#pragma unroll
    for (int q = 0; q < kRopeVec; ++q)
      rope_sincos(pos * exp2f(-l2t * static_cast<float>(2 * (p0 + q)) / a.d), &sn[q], &cs[q]);
  }
  int64_t slot = 0;   // cache row of this token for kv head 0: (s * Hk) * max_seq + cpos
  if (active && h0 + kRopeHeads > a.Hq) {
    int s;
    int64_t cpos;
    if (a.decode) {
      s = static_cast<int>(t);
      cpos = a.cache_lens[s];
    } else {
      int lo = 0, hi = a.num_seqs - 1;   // last s with cu[s] <= t
      while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (a.cu_seqlens[mid] <= t) lo = mid; else hi = mid - 1;
      }
      s = lo;
      cpos = a.cache_lens[s] + (t - a.cu_seqlens[s]);
    }
    // a position past the cache capacity is dropped (never written into the
    // next head's or sequence's rows; include/dl.h)
    slot = (cpos >= 0 && cpos < a.max_seq) ? static_cast<int64_t>(s) * a.Hk * a.max_seq + cpos : -1;
  }
  pdl_wait();
  ew_mark(tr, 2);
  side_zero(a.zero);
  side_zero(a.zero2);
  if (!active) return;
  constexpr int NV = 2 * kRopeVec;   // values per thread and head
  float v[kRopeHeads][NV];
#pragma unroll
  for (int j = 0; j < kRopeHeads; ++j) {
    const int hd = h0 + j;
    if (hd >= heads) break;
    const int64_t col = static_cast<int64_t>(hd) * a.d + 2 * p0;
    if (a.acc) {
      float* q = const_cast<float*>(a.acc) + t * a.ld_src + col;
#pragma unroll
      for (int e = 0; e < NV; e += 4) {
        const float4 f = *reinterpret_cast<const float4*>(q + e);
        v[j][e] = f.x; v[j][e + 1] = f.y; v[j][e + 2] = f.z; v[j][e + 3] = f.w;
        if (a.clear) *reinterpret_cast<float4*>(q + e) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    } else {
      ld8(a.src + t * a.ld_src + col, v[j]);   // NV == 8: one 16-byte load
    }
  }
#pragma unroll
  for (int j = 0; j < kRopeHeads; ++j) {
    const int hd = h0 + j;
    if (hd >= heads) break;
    float r[NV];
#pragma unroll
    for (int q = 0; q < kRopeVec; ++q) {
      const float x = v[j][2 * q], y = v[j][2 * q + 1];
      const bool rot = a.rope && hd < a.Hq + a.Hk;
      r[2 * q] = rot ? x * cs[q] - y * sn[q] : x;
      r[2 * q + 1] = rot ? x * sn[q] + y * cs[q] : y;
    }
    uint4 pk;
    __nv_bfloat162* pb = reinterpret_cast<__nv_bfloat162*>(&pk);
#pragma unroll
    for (int e = 0; e < 4; ++e) pb[e] = __floats2bfloat162_rn(r[2 * e], r[2 * e + 1]);
    if (hd < a.Hq) {
      *reinterpret_cast<uint4*>(a.q_out + t * static_cast<int64_t>(a.Hq) * a.d + static_cast<int64_t>(hd) * a.d +
                                2 * p0) = pk;
    } else if (slot >= 0) {
      const bool is_k = hd < a.Hq + a.Hk;
      const int kvh = is_k ? hd - a.Hq : hd - a.Hq - a.Hk;
      *reinterpret_cast<uint4*>((is_k ? a.k_cache : a.v_cache) +
                                (slot + static_cast<int64_t>(kvh) * a.max_seq) * a.d + 2 * p0) = pk;
    }
  }
  ew_mark(tr, 3);
}

// Decode-size variant (T <= 256): one thread per 4 dims of one token, grid
// (ceil(heads*d/4 / 128), T) -- more threads per token, shorter per-thread chains.
__global__ void __launch_bounds__(128) rope_cache_tok_kernel(RopeCacheArgs a, EwTrace tr) {
  ew_mark(tr, 1);
  pdl_trigger();   // successor may launch now; it waits for us before reading
  // Everything that depends only on the call's inputs (positions, cache
  // lengths, cu_seqlens -- never written inside the block) is done before
  // griddepcontrol.wait: the angles and the cache slot, overlapping the
  // predecessor's tail.  After the wait: one load, rotate, one store.
  const int heads = a.Hq + 2 * a.Hk;
  const int quads = a.d / 4;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = i < heads * quads;
  const int64_t t = blockIdx.y;
  const int hd = active ? i / quads : 0;
  const int e = (i - hd * quads) * 4;
  const int64_t col = static_cast<int64_t>(hd) * a.d + e;
  float sn0 = 0.f, cs0 = 1.f, sn1 = 0.f, cs1 = 1.f;
  const bool rot = active && a.rope && hd < a.Hq + a.Hk;
  if (rot) {
    // angle = pos * theta^(-2i/d) in fp32 (relative error ~1e-7, i.e. <= 3e-4 rad at
    // position 2048, far below bf16 resolution); rope_sincos (dl_internal.h)
    const float pos = static_cast<float>(a.positions[t]);
    const float l2t = log2f(a.theta);
    rope_sincos(pos * exp2f(-l2t * static_cast<float>(e) / a.d), &sn0, &cs0);
    rope_sincos(pos * exp2f(-l2t * static_cast<float>(e + 2) / a.d), &sn1, &cs1);
  }
  __nv_bfloat16* dst = nullptr;
  if (active && hd >= a.Hq) {
    int s;
    int64_t cpos;
    if (a.decode) {
      s = static_cast<int>(t);
      cpos = a.cache_lens[s];
    } else {
      int lo = 0, hi = a.num_seqs - 1;   // last s with cu[s] <= t
      while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (a.cu_seqlens[mid] <= t) lo = mid; else hi = mid - 1;
      }
      s = lo;
      cpos = a.cache_lens[s] + (t - a.cu_seqlens[s]);
    }
    const bool is_k = hd < a.Hq + a.Hk;
    const int kvh = is_k ? hd - a.Hq : hd - a.Hq - a.Hk;
    if (cpos >= 0 && cpos < a.max_seq)   // past the capacity: dropped (include/dl.h)
      dst = (is_k ? a.k_cache : a.v_cache) + ((static_cast<int64_t>(s) * a.Hk + kvh) * a.max_seq + cpos) * a.d + e;
  }
  pdl_wait();
  ew_mark(tr, 2);
  const bool early = rn_early();   // side clears after the load is in flight (DL_RN_EARLY)
  if (!early) {
    side_zero(a.zero);
    side_zero(a.zero2);
  }
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (active) {
    if (a.acc) {
      v = take4(const_cast<float*>(a.acc) + t * a.ld_src + col, a.clear);
    } else {
      v = load4(a.src + t * a.ld_src + col);
    }
  }
  if (early) {
    side_zero(a.zero);
    side_zero(a.zero2);
  }
  if (!active) return;
  if (rot) v = make_float4(v.x * cs0 - v.y * sn0, v.x * sn0 + v.y * cs0, v.z * cs1 - v.w * sn1, v.z * sn1 + v.w * cs1);
  if (hd < a.Hq) store4(a.q_out + t * static_cast<int64_t>(a.Hq) * a.d + col, v.x, v.y, v.z, v.w);
  else if (dst) store4(dst, v.x, v.y, v.z, v.w);
  ew_mark(tr, 3);
}

__global__ void __launch_bounds__(256) embedding_kernel(const __nv_bfloat16* __restrict__ table, int64_t h,
                                                        const int32_t* __restrict__ ids,
                                                        __nv_bfloat16* __restrict__ out) {
  pdl_trigger();   // successor may launch now; it waits for us before reading
  pdl_wait();
  const int64_t t = blockIdx.x;
  const uint4* src = reinterpret_cast<const uint4*>(table + static_cast<int64_t>(ids[t]) * h);
  uint4* dst = reinterpret_cast<uint4*>(out + t * h);
  for (int i = threadIdx.x; i < h / 8; i += blockDim.x) dst[i] = src[i];
}

// Greedy next token: ids[t] = argmax over the P vocab shards of
// logits[p * rank_stride + t * ld + v] (v < vloc; global id p * vloc + v).
// One CTA (512 threads) per token; ties -> the smallest id.
__global__ void __launch_bounds__(512) argmax_kernel(const __nv_bfloat16* __restrict__ logits, int64_t vloc, int P,
                                                     int64_t rank_stride, int64_t ld, int32_t* __restrict__ ids) {
  pdl_trigger();   // successor may launch now; it waits for us before reading
  pdl_wait();
  __shared__ float sv[16];
  __shared__ int si[16];
  const int64_t t = blockIdx.x;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int p = 0; p < P; ++p) {
    const __nv_bfloat16* row = logits + p * rank_stride + t * ld;
    for (int64_t v = threadIdx.x * 8; v < vloc; v += 512 * 8) {
      if (v + 8 <= vloc && ((reinterpret_cast<uintptr_t>(row + v) & 15) == 0)) {
        const uint4 u = *reinterpret_cast<const uint4*>(row + v);
        const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float f = __bfloat162float(b[e]);
          const int id = static_cast<int>(p * vloc + v + e);
          if (f > best || (f == best && id < bi)) { best = f; bi = id; }
        }
      } else {
        for (int64_t e = v; e < v + 8 && e < vloc; ++e) {
          const float f = __bfloat162float(row[e]);
          const int id = static_cast<int>(p * vloc + e);
          if (f > best || (f == best && id < bi)) { best = f; bi = id; }
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 16; ++w)
      if (sv[w] > best || (sv[w] == best && si[w] < bi)) { best = sv[w]; bi = si[w]; }
    ids[t] = bi;
  }
}

// [P][T][w] -> [T][P*w]; grid (ceil(w/8 / 128), T, P)
__global__ void __launch_bounds__(128) unpermute_kernel(const __nv_bfloat16* __restrict__ src,
                                                        __nv_bfloat16* __restrict__ dst, int P, int64_t T,
                                                        int w8) {
  pdl_trigger();   // successor may launch now; it waits for us before reading
  pdl_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= w8) return;
  const int64_t t = blockIdx.y, p = blockIdx.z;
  reinterpret_cast<uint4*>(dst)[(t * P + p) * w8 + c] = reinterpret_cast<const uint4*>(src)[(p * T + t) * w8 + c];
}

// DeInfer latent un-permute: the all-gathered slices recv [P][T][slot] (rank
// p holds latent columns [begin_p, begin_p + len_p) of the concatenated group
// rank, balanced split) -> the group's Z layout zb [T x width] (segment s at
// columns [zoff_s, zoff_s + rup(len_s, 64)), zero padded).
// grid (ceil(width / 256), T), one column per thread.
// All-gather by push into the ranks' symmetric windows (fused collective):
// row t of src [T x w] goes to dst + delta[j] + t * w (dst already offset to
// this rank's slot [rank][T][w]) for every rank j < P.  grid (ceil(w/8/128), T).
struct FanDeltas {
  long long d[8];
};
__global__ void __launch_bounds__(128) fan_copy_kernel(const __nv_bfloat16* __restrict__ src, int64_t ld_src,
                                                       __nv_bfloat16* dst, FanDeltas dl, int P, int w8,
                                                       SideZero z) {
  pdl_trigger();
  pdl_wait();
  side_zero(z);
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= w8) return;
  const int64_t t = blockIdx.y;
  const uint4 v = *reinterpret_cast<const uint4*>(src + t * ld_src + c * 8);
  for (int j = 0; j < P; ++j)
    *reinterpret_cast<uint4*>(dst + dl.d[j] + t * static_cast<int64_t>(w8) * 8 + c * 8) = v;
}

// grid (ceil(w8 / 128), T, P): rank blockIdx.z != self receives this rank's
// columns [c0, c0 + 8 * w8) of row t
__global__ void __launch_bounds__(128) fan_push_kernel(__nv_bfloat16* buf, int64_t ld, int64_t c0, int w8,
                                                       FanDeltas dl, int self, SideZero z) {
  pdl_trigger();
  pdl_wait();
  side_zero(z);
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.z;
  if (c >= w8 || j == self) return;
  const int64_t off = static_cast<int64_t>(blockIdx.y) * ld + c0 + c * 8;
  *reinterpret_cast<uint4*>(buf + dl.d[j] + off) = __ldcg(reinterpret_cast<const uint4*>(buf + off));
}

__global__ void __launch_bounds__(256) latent_unpermute_kernel(const __nv_bfloat16* __restrict__ recv,
                                                               __nv_bfloat16* __restrict__ zb, int64_t ldzb,
                                                               LatentMap mp, SideZero z) {
  pdl_trigger();   // successor may launch now; it waits for us before reading
  pdl_wait();
  side_zero(z);
  const int64_t col = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (col >= mp.width) return;
  const int64_t t = blockIdx.y;
  int s = 0;
  while (s + 1 < mp.nseg && col >= mp.zoff[s + 1]) ++s;
  const int64_t c = col - mp.zoff[s];
  __nv_bfloat16 v = __float2bfloat16_rn(0.f);
  if (c < mp.seg_len[s]) {
    const int64_t j = mp.seg_beg[s] + c;
    const int64_t big = mp.extra * (mp.base + 1);
    const int64_t p = j < big ? j / (mp.base + 1) : mp.extra + (j - big) / mp.base;
    const int64_t b = p * mp.base + (p < mp.extra ? p : mp.extra);
    v = recv[(p * mp.T + t) * mp.slot + (j - b)];
  }
  zb[t * ldzb + col] = v;
}

// ---- low-rank KV cache (N3) ------------------------------------------------
// grid T, 128 threads: one decode token per CTA, 16-byte copies.
__global__ void __launch_bounds__(128) kv_append_kernel(const __nv_bfloat16* __restrict__ zb, int64_t ldzb,
                                                        int64_t zoff, int n8, __nv_bfloat16* __restrict__ pool,
                                                        int64_t ld_slot, int32_t* __restrict__ slot_pos, int64_t bs,
                                                        const int32_t* __restrict__ tables, int64_t mbps,
                                                        const int32_t* __restrict__ cache_lens,
                                                        const int32_t* __restrict__ positions) {
  pdl_trigger();   // successor may launch now; it waits for us before reading
  pdl_wait();
  const int64_t t = blockIdx.x;
  const int64_t p = cache_lens[t];
  if (p < 0 || p / bs >= mbps) return;   // past the block table: dropped (include/dl.h)
  const int64_t slot = static_cast<int64_t>(tables[t * mbps + p / bs]) * bs + p % bs;
  const uint4* src = reinterpret_cast<const uint4*>(zb + t * ldzb + zoff);
  uint4* dst = reinterpret_cast<uint4*>(pool + slot * ld_slot);
  for (int i = threadIdx.x; i < n8; i += blockDim.x) dst[i] = src[i];
  if (threadIdx.x == 0) slot_pos[slot] = positions[t];
}

// Squeeze ("the physically contiguous KV caches are sequentially copied
// to the buffer"): buffer block b belongs to the run r with run_dst[r] <= b <
// run_dst[r] + run_len[r] (run_dst ascending); CTAs stride over buffer blocks.
__global__ void __launch_bounds__(256) kv_squeeze_kernel(const __nv_bfloat16* __restrict__ pool,
                                                         const int32_t* __restrict__ slot_pos,
                                                         __nv_bfloat16* __restrict__ squeeze,
                                                         int32_t* __restrict__ squeeze_pos, int64_t ld_slot, int64_t bs,
                                                         const int32_t* __restrict__ run_src,
                                                         const int32_t* __restrict__ run_dst,
                                                         const int32_t* __restrict__ run_len,
                                                         const int32_t* __restrict__ n_runs_p, int64_t cap_blocks) {
  pdl_trigger();   // successor may launch now; it waits for us before reading
  pdl_wait();
  const int n_runs = *n_runs_p;
  if (n_runs <= 0) return;
  const int64_t total = static_cast<int64_t>(run_dst[n_runs - 1]) + run_len[n_runs - 1];
  const int64_t blk8 = bs * ld_slot / 8;     // uint4 per block
  for (int64_t b = blockIdx.x; b < total && b < cap_blocks; b += gridDim.x) {
    int lo = 0, hi = n_runs - 1;              // last run with run_dst <= b
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (run_dst[mid] <= b) lo = mid; else hi = mid - 1;
    }
    const int64_t src_blk = run_src[lo] + (b - run_dst[lo]);
    const uint4* s4 = reinterpret_cast<const uint4*>(pool + src_blk * bs * ld_slot);
    uint4* d4 = reinterpret_cast<uint4*>(squeeze + b * bs * ld_slot);
    for (int64_t i = threadIdx.x; i < blk8; i += blockDim.x) d4[i] = s4[i];
    for (int64_t i = threadIdx.x; i < bs; i += blockDim.x) squeeze_pos[b * bs + i] = slot_pos[src_blk * bs + i];
  }
}

// in-place RoPE on reconstructed key rows ("in-place rotary position embedding
// kernel ... to the reconstruction results").  grid (ceil(heads*32/128), rows)
__global__ void __launch_bounds__(128) rope_rows_kernel(__nv_bfloat16* __restrict__ buf, int64_t ld, int heads,
                                                        const int32_t* __restrict__ pos, int64_t rows, float theta) {
  pdl_trigger();   // successor may launch now; it waits for us before reading
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= heads * 32) return;
  const int e = (i & 31) * 4;
  const float l2t = log2f(theta);
  const float f0 = exp2f(-l2t * static_cast<float>(e) / 128.f), f1 = exp2f(-l2t * static_cast<float>(e + 2) / 128.f);
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    __nv_bfloat16* p = buf + r * ld + static_cast<int64_t>(i >> 5) * 128 + e;
    const float4 v = load4(p);
    const float fp = static_cast<float>(pos[r]);
    float sn0, cs0, sn1, cs1;
    rope_sincos(fp * f0, &sn0, &cs0);
    rope_sincos(fp * f1, &sn1, &cs1);
    store4(p, v.x * cs0 - v.y * sn0, v.x * sn0 + v.y * cs0, v.z * cs1 - v.w * sn1, v.z * sn1 + v.w * cs1);
  }
}

}  // namespace

dl_status launch_kv_append(const __nv_bfloat16* zb, int64_t ldzb, int64_t zoff, int64_t ncopy, __nv_bfloat16* pool,
                           int64_t ld_slot, int32_t* slot_pos, int64_t block_size, const int32_t* block_tables,
                           int64_t max_blocks_per_seq, const int32_t* cache_lens, const int32_t* positions, int64_t T,
                           cudaStream_t st) {
  if (T <= 0) return DL_OK;
  const int n8 = static_cast<int>((ncopy + 7) / 8);
  return launch_pdl(kv_append_kernel, dim3(static_cast<unsigned>(T)), dim3(128), 0, st, "kv_append", zb, ldzb, zoff,
                    n8, pool, ld_slot, slot_pos, block_size, block_tables, max_blocks_per_seq, cache_lens, positions);
}

dl_status launch_kv_squeeze(const __nv_bfloat16* pool, const int32_t* slot_pos, __nv_bfloat16* squeeze,
                            int32_t* squeeze_pos, int64_t ld_slot, int64_t block_size, const int32_t* run_src,
                            const int32_t* run_dst, const int32_t* run_len, const int32_t* n_runs, int64_t cap_blocks,
                            cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(cap_blocks, 8LL * num_sms()));
  if (grid == 0) return DL_OK;
  return launch_pdl(kv_squeeze_kernel, dim3(grid), dim3(256), 0, st, "kv_squeeze", pool, slot_pos, squeeze,
                    squeeze_pos, ld_slot, block_size, run_src, run_dst, run_len, n_runs, cap_blocks);
}

dl_status launch_rope_rows(__nv_bfloat16* buf, int64_t ld, int heads, const int32_t* pos, int64_t rows, float theta,
                           cudaStream_t st) {
  if (rows <= 0 || heads <= 0) return DL_OK;
  dim3 grid((heads * 32 + 127) / 128, static_cast<unsigned>(std::min<int64_t>(rows, 16384)));
  return launch_pdl(rope_rows_kernel, grid, dim3(128), 0, st, "rope_rows", buf, ld, heads, pos, rows, theta);
}

dl_status launch_latent_unpermute(const __nv_bfloat16* recv, __nv_bfloat16* zb, int64_t ldzb, const LatentMap& mp,
                                  cudaStream_t st, const SideZero& z) {
  if (mp.T <= 0 || mp.width <= 0) return DL_OK;
  dim3 grid(static_cast<unsigned>((mp.width + 255) / 256), static_cast<unsigned>(mp.T));
  return launch_pdl(latent_unpermute_kernel, grid, dim3(256), 0, st, "latent_unpermute", recv, zb, ldzb, mp, z);
}

void rn_early_init() {
  static const bool done = [] {
    if (DL_ENV("DL_RN_EARLY") && atoi(DL_ENV("DL_RN_EARLY")) == 0) {
      const int zero = 0;
      cudaMemcpyToSymbol(g_rn_early, &zero, sizeof(int));
    }
    return true;
  }();
  (void)done;
}

dl_status launch_rmsnorm(const __nv_bfloat16* x, const __nv_bfloat16* g, __nv_bfloat16* y, int64_t T, int64_t h,
                         float eps, cudaStream_t st) {
  if (T <= 0) return DL_OK;
  rn_early_init();
  if (T >= 512 && h % 8 == 0 && h / 8 <= kRrThreads * kRrChunks)   // many rows: 4 rows per CTA
    return launch_pdl(rmsnorm_rows_kernel, dim3(static_cast<unsigned>((T + kRrRows - 1) / kRrRows)),
                      dim3(kRrRows * kRrThreads), 0, st, "rmsnorm", x, g, y, T, static_cast<int>(h), eps, ew_trace(2));
  if (h % 8 == 0 && h / 8 <= kRnThreads * kRnChunks)   // register-resident one-pass kernel, no accumulator
    return launch_pdl(residual_rmsnorm_kernel<float>, dim3(static_cast<unsigned>(T)), dim3(kRnThreads), 0, st,
                      "rmsnorm", static_cast<float*>(nullptr), int64_t{0}, const_cast<__nv_bfloat16*>(x), g, y,
                      static_cast<int>(h), eps, SideZero{}, SideZero{}, ew_trace(2));
  return launch_pdl(rmsnorm_kernel, dim3(static_cast<unsigned>(T)), dim3(256), 0, st, "rmsnorm", x, g, y,
                    static_cast<int>(h), eps);
}
dl_status launch_residual_rmsnorm(float* acc, int64_t lda, __nv_bfloat16* x, const __nv_bfloat16* g,
                                  __nv_bfloat16* y, int64_t T, int64_t h, float eps, cudaStream_t st,
                                  const SideZero& z, const SideZero& z2) {
  if (T <= 0) return DL_OK;
  rn_early_init();
  if (h % 8 || h / 8 > kRnThreads * kRnChunks) {
    set_error("residual_rmsnorm: h=%lld unsupported (multiple of 8, <= %d)", (long long)h, 8 * kRnThreads * kRnChunks);
    return DL_ERR_UNSUPPORTED;
  }
  return launch_pdl(residual_rmsnorm_kernel<float>, dim3(static_cast<unsigned>(T)), dim3(kRnThreads), 0, st,
                    "residual_rmsnorm", acc, lda, x, g, y, static_cast<int>(h), eps, z, z2, ew_trace(2));
}
dl_status launch_residual_rmsnorm_bf16(__nv_bfloat16* acc, int64_t lda, __nv_bfloat16* x, const __nv_bfloat16* g,
                                       __nv_bfloat16* y, int64_t T, int64_t h, float eps, cudaStream_t st,
                                       const SideZero& z, const SideZero& z2) {
  if (T <= 0) return DL_OK;
  rn_early_init();
  if (h % 8 || h / 8 > kRnThreads * kRnChunks) {
    set_error("residual_rmsnorm: h=%lld unsupported (multiple of 8, <= %d)", (long long)h, 8 * kRnThreads * kRnChunks);
    return DL_ERR_UNSUPPORTED;
  }
  return launch_pdl(residual_rmsnorm_kernel<__nv_bfloat16>, dim3(static_cast<unsigned>(T)), dim3(kRnThreads), 0, st,
                    "residual_rmsnorm_bf16", acc, lda, x, g, y, static_cast<int>(h), eps, z, z2, ew_trace(2));
}
dl_status launch_f32_to_bf16(float* acc, int64_t lda, __nv_bfloat16* out, int64_t ldo, int64_t T, int64_t n,
                             int clear, cudaStream_t st, const SideZero& z) {
  return launch_ew4(T, n, F32ToBf16{acc, lda, out, ldo, clear}, st, "f32_to_bf16", z);
}
dl_status launch_residual_add_f32(float* acc, int64_t lda, __nv_bfloat16* x, int64_t ldx, int64_t T, int64_t n,
                                  int clear, cudaStream_t st, const SideZero& z, const SideZero& z2) {
  return launch_ew4(T, n, ResidualAdd{acc, lda, x, ldx, clear}, st, "residual_add", z, z2);
}
dl_status launch_residual_add_bf16(const __nv_bfloat16* y, int64_t ldy, __nv_bfloat16* x, int64_t ldx, int64_t T,
                                   int64_t n, cudaStream_t st, int clear, const SideZero& z, const SideZero& z2) {
  return launch_ew4(T, n, ResidualAddBf16{const_cast<__nv_bfloat16*>(y), ldy, x, ldx, clear}, st, "residual_add_bf16",
                    z, z2);
}
dl_status launch_silu_mul_f32(float* acc, int64_t lda, __nv_bfloat16* act, int64_t ldo, int64_t T, int64_t m,
                              int clear, cudaStream_t st, const SideZero& z) {
  static const bool ew4 = DL_ENV("DL_SILU_EW4") != nullptr;   // A/B switch
  if (!ew4 && clear && m % 8 == 0 && lda % 4 == 0 && ldo % 8 == 0 && T > 0) {
    return launch_silu_flat(acc, lda, act, ldo, T, m, 0, st, z);
  }
  return launch_ew4(T, m, SiluMulF32{acc, lda, act, ldo, m, clear}, st, "silu_mul_f32", z);
}
dl_status launch_silu_mul_bf16(const __nv_bfloat16* src, int64_t lds, __nv_bfloat16* act, int64_t ldo, int64_t T,
                               int64_t m, cudaStream_t st, int clear, const SideZero& z) {
  if (m % 8 == 0 && lds % 8 == 0 && ldo % 8 == 0 && T > 0)
    return launch_silu_flat(const_cast<__nv_bfloat16*>(src), lds, act, ldo, T, m, 0, st, z, clear);
  return launch_ew4(T, m, SiluMulBf16{const_cast<__nv_bfloat16*>(src), lds, act, ldo, m, clear}, st, "silu_mul_bf16",
                    z);
}
dl_status launch_relu_f32(float* acc, int64_t lda, __nv_bfloat16* act, int64_t ldo, int64_t T, int64_t m,
                          int clear, cudaStream_t st, const SideZero& z) {
  return launch_ew4(T, m, ReluF32{acc, lda, act, ldo, clear}, st, "relu_f32", z);
}
dl_status launch_relu_bf16(const __nv_bfloat16* src, int64_t lds, __nv_bfloat16* act, int64_t ldo, int64_t T,
                           int64_t m, cudaStream_t st, int clear, const SideZero& z) {
  if (m % 8 == 0 && lds % 8 == 0 && ldo % 8 == 0 && T > 0)
    return launch_silu_flat(const_cast<__nv_bfloat16*>(src), lds, act, ldo, T, m, 1, st, z, clear);
  return launch_ew4(T, m, ReluBf16{const_cast<__nv_bfloat16*>(src), lds, act, ldo, clear}, st, "relu_bf16", z);
}
// Prefill append of already rotated keys and the values (RopeCacheArgs::kv_only):
// 8 tokens per CTA, one 16-byte chunk per thread (k and v rows of the q|k|v output
// -> head-major cache rows); the cache slot is found once per token (lanes of
// warp 0) before griddepcontrol.wait -- positions, cu_seqlens and cache_lens are
// not written inside the step.
constexpr int kKvTok = 8;
__global__ void __launch_bounds__(256) kv_cache_append_kernel(RopeCacheArgs a, EwTrace tr) {
  ew_mark(tr, 1);
  pdl_trigger();
  __shared__ int64_t slot_s[kKvTok];
  const int chunks = 2 * a.Hk * (a.d / 8);                 // 16-byte chunks per token
  if (threadIdx.x < kKvTok) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * kKvTok + threadIdx.x;
    int64_t slot = -1;
    if (t < a.T) {
      int lo = 0, hi = a.num_seqs - 1;   // last s with cu[s] <= t
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.cu_seqlens[mid] <= t) lo = mid; else hi = mid - 1;
      }
      const int64_t cpos = a.cache_lens[lo] + (t - a.cu_seqlens[lo]);
      if (cpos >= 0 && cpos < a.max_seq) slot = static_cast<int64_t>(lo) * a.Hk * a.max_seq + cpos;   // past capacity: dropped
    }
    slot_s[threadIdx.x] = slot;
  }
  __syncthreads();
  pdl_wait();
  ew_mark(tr, 2);
  side_zero(a.zero);
  side_zero(a.zero2);
  constexpr int PER = 8;   // chunks per thread, all loads before the stores
  for (int base = threadIdx.x; base < kKvTok * chunks; base += PER * blockDim.x) {
    uint4 v[PER];
    __nv_bfloat16* dst[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      dst[q] = nullptr;
      const int i = base + q * blockDim.x;
      if (i >= kKvTok * chunks) continue;
      const int tk = i / chunks, c = i - tk * chunks;
      const int64_t t = static_cast<int64_t>(blockIdx.x) * kKvTok + tk;
      const int64_t slot = slot_s[tk];
      if (t >= a.T || slot < 0) continue;
      const int hd = c / (a.d / 8), ck = c - hd * (a.d / 8);   // hd < Hk: key head, else value head
      const bool is_k = hd < a.Hk;
      const int kvh = is_k ? hd : hd - a.Hk;
      v[q] = *reinterpret_cast<const uint4*>(a.src + t * a.ld_src + static_cast<int64_t>(a.Hq + hd) * a.d + ck * 8);
      dst[q] = (is_k ? a.k_cache : a.v_cache) + (slot + static_cast<int64_t>(kvh) * a.max_seq) * a.d + ck * 8;
    }
#pragma unroll
    for (int q = 0; q < PER; ++q)
      if (dst[q]) *reinterpret_cast<uint4*>(dst[q]) = v[q];
  }
  ew_mark(tr, 3);
}

dl_status launch_rope_cache(const RopeCacheArgs& a, cudaStream_t st) {
  if (a.T <= 0) return DL_OK;
  rn_early_init();
  if (a.kv_only && (a.rope || a.T <= 256)) {
    set_error("rope_cache: kv_only is the prefill append of already rotated keys (rope = 0)");
    return DL_ERR_INVALID_ARG;
  }
  static const bool kv_copy = !DL_ENV("DL_KV_APPEND") || atoi(DL_ENV("DL_KV_APPEND")) != 0;   // A/B
  if (a.kv_only && kv_copy && a.src && !a.acc && a.d % 8 == 0 && a.ld_src % 8 == 0 && !a.decode)
    return launch_pdl(kv_cache_append_kernel, dim3(static_cast<unsigned>((a.T + kKvTok - 1) / kKvTok)), dim3(256), 0, st,
                      "kv_cache_append", a, ew_trace(3));
  if (a.T <= 256 && a.d % 4 == 0) {
    const int per_tok = (a.Hq + 2 * a.Hk) * (a.d / 4);
    dim3 grid((per_tok + 127) / 128, static_cast<unsigned>(a.T));
    return launch_pdl(rope_cache_tok_kernel, grid, dim3(128), 0, st, "rope_cache", a, ew_trace(3));
  }
  if (a.d != 128) {
    set_error("rope_cache: head_dim %d unsupported (128)", a.d);
    return DL_ERR_UNSUPPORTED;
  }
  const int groups = ((a.kv_only ? 0 : a.Hq) + 2 * a.Hk + kRopeHeads - 1) / kRopeHeads;
  const int per_cta = 128 / (64 / kRopeVec);
  dim3 grid((groups + per_cta - 1) / per_cta, static_cast<unsigned>(a.T));
  return launch_pdl(rope_cache_kernel, grid, dim3(128), 0, st, "rope_cache", a, ew_trace(3));
}
dl_status launch_argmax(const __nv_bfloat16* logits, int64_t T, int64_t vloc, int P, int64_t rank_stride,
                        int64_t ld, int32_t* ids, cudaStream_t st) {
  if (T <= 0) return DL_OK;
  return launch_pdl(argmax_kernel, dim3(static_cast<unsigned>(T)), dim3(512), 0, st, "argmax", logits, vloc, P,
                    rank_stride, ld, ids);
}
dl_status launch_embedding(const __nv_bfloat16* table, int64_t vocab, int64_t h, const int32_t* ids, int64_t T,
                           __nv_bfloat16* out, cudaStream_t st) {
  (void)vocab;
  if (T <= 0) return DL_OK;
  return launch_pdl(embedding_kernel, dim3(static_cast<unsigned>(T)), dim3(256), 0, st, "embedding", table, h, ids,
                    out);
}
dl_status launch_unpermute(const __nv_bfloat16* src, __nv_bfloat16* dst, int P, int64_t T, int64_t w,
                           cudaStream_t st) {
  if (T <= 0) return DL_OK;
  const int w8 = static_cast<int>(w / 8);
  dim3 grid((w8 + 127) / 128, static_cast<unsigned>(T), static_cast<unsigned>(P));
  return launch_pdl(unpermute_kernel, grid, dim3(128), 0, st, "unpermute", src, dst, P, T, w8);
}
dl_status launch_fan_copy(const __nv_bfloat16* src, int64_t ld_src, __nv_bfloat16* dst, const int64_t* delta,
                          int P, int64_t T, int64_t w, cudaStream_t st, const SideZero& z) {
  if (T <= 0 || w <= 0) return DL_OK;
  if (w % 8 || ld_src % 8 || P < 1 || P > 8) {
    set_error("fan_copy: w and ld must be multiples of 8, 1 <= P <= 8");
    return DL_ERR_UNSUPPORTED;
  }
  FanDeltas dl{};
  for (int j = 0; j < P; ++j) dl.d[j] = delta[j];
  const int w8 = static_cast<int>(w / 8);
  dim3 grid((w8 + 127) / 128, static_cast<unsigned>(T));
  return launch_pdl(fan_copy_kernel, grid, dim3(128), 0, st, "fan_copy", src, ld_src, dst, dl, P, w8, z);
}
dl_status launch_fan_push(__nv_bfloat16* buf, int64_t ld, int64_t T, int64_t c0, int64_t c1, const int64_t* delta,
                          int P, int self, cudaStream_t st, const SideZero& z) {
  if (T <= 0 || P < 1) return DL_OK;
  if ((c1 - c0) % 8 || c0 % 8 || ld % 8 || P > 8) {
    set_error("fan_push: column range and ld must be multiples of 8, P <= 8");
    return DL_ERR_UNSUPPORTED;
  }
  FanDeltas dl{};
  for (int j = 0; j < P; ++j) dl.d[j] = delta[j];
  const int w8 = static_cast<int>((c1 - c0) / 8);
  if (w8 <= 0) return DL_OK;
  dim3 grid((w8 + 127) / 128, static_cast<unsigned>(T), static_cast<unsigned>(P));
  return launch_pdl(fan_push_kernel, grid, dim3(128), 0, st, "fan_push", buf, ld, c0, w8, dl, self, z);
}
dl_status launch_copy2d(const void* src, int64_t lds, void* dst, int64_t ldd, int64_t rows, int64_t cols_bytes,
                        cudaStream_t st) {
  if (rows <= 0 || cols_bytes <= 0) return DL_OK;
  return cuda_status(cudaMemcpy2DAsync(dst, ldd, src, lds, cols_bytes, rows, cudaMemcpyDeviceToDevice, st),
                     "copy2d");
}

}  // namespace dl
