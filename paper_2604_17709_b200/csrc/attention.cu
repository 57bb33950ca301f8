// Causal GQA attention over the head-major KV cache (row a6 of the hot
// path): out = softmax(q K^T / sqrt(d) + causal mask) V, query head g
// reading kv head floor(g * Hk / Hq), on the rank's LOCAL
// heads only -- the duplicated self-attention of PAPER.md:141-144 is gone.
//
// Cache layout [seq][kv_head][max_seq][d] (bf16): one (seq, kv head) is a
// contiguous run of keys, so the key loop streams coalesced 256 B rows.
//
// attn_warp_kernel: one warp per (query token, query head); lane owns 4 of
// the d = 128 dims; keys are consumed 4 at a time (4 independent shuffle
// reductions in flight) with an online (running-max) softmax in fp32.
// Used for decode and (as the round-1 path) for prefill.
#include <math.h>

#include "dl_internal.h"

namespace dl {
namespace {

constexpr int kWarpsPerCta = 4;

__device__ __forceinline__ float4 ld_bf16x4(const __nv_bfloat16* p) {
  uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
  float2 a = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(&v)[0]);
  float2 b = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(&v)[1]);
  return make_float4(a.x, a.y, b.x, b.y);
}

__global__ void __launch_bounds__(kWarpsPerCta * 32) attn_warp_kernel(AttnArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = blockIdx.x;
  const int h = blockIdx.y * kWarpsPerCta + warp;
  if (h >= a.Hq) return;
  int s;
  int64_t qpos;   // cache position of this query (keys 0..qpos are visible)
  if (a.decode) {
    s = static_cast<int>(t);
    qpos = a.cache_lens[s];
  } else {
    int lo = 0, hi = a.num_seqs - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (a.cu_seqlens[mid] <= t) lo = mid; else hi = mid - 1;
    }
    s = lo;
    qpos = a.cache_lens[s] + (t - a.cu_seqlens[s]);
  }
  const int kvh = static_cast<int>((static_cast<int64_t>(h) * a.Hk) / a.Hq);
  const int d = a.d;   // 128
  const float scale = rsqrtf(static_cast<float>(d)) * 1.4426950408889634f;   // log2(e)/sqrt(d)
  float4 q = ld_bf16x4(a.q + t * static_cast<int64_t>(a.Hq) * d + static_cast<int64_t>(h) * d + lane * 4);
  q.x *= scale; q.y *= scale; q.z *= scale; q.w *= scale;
  const int64_t base = (static_cast<int64_t>(s) * a.Hk + kvh) * a.max_seq * d + lane * 4;
  const __nv_bfloat16* K = a.k_cache + base;
  const __nv_bfloat16* V = a.v_cache + base;
  float m = -INFINITY, l = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const int64_t nk = qpos + 1;
  int64_t u = 0;
  for (; u + 4 <= nk; u += 4) {
    float sc[4];
    float4 vv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float4 k = ld_bf16x4(K + (u + j) * d);
      vv[j] = ld_bf16x4(V + (u + j) * d);
      sc[j] = q.x * k.x + q.y * k.y + q.z * k.z + q.w * k.w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int j = 0; j < 4; ++j) sc[j] += __shfl_xor_sync(0xffffffffu, sc[j], o);
    const float mx = fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3]));
    const float mn = fmaxf(m, mx);
    const float corr = exp2f(m - mn);
    l *= corr;
    acc.x *= corr; acc.y *= corr; acc.z *= corr; acc.w *= corr;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float p = exp2f(sc[j] - mn);
      l += p;
      acc.x += p * vv[j].x; acc.y += p * vv[j].y; acc.z += p * vv[j].z; acc.w += p * vv[j].w;
    }
    m = mn;
  }
  for (; u < nk; ++u) {
    float4 k = ld_bf16x4(K + u * d);
    float4 v = ld_bf16x4(V + u * d);
    float sc = q.x * k.x + q.y * k.y + q.z * k.z + q.w * k.w;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
    const float mn = fmaxf(m, sc);
    const float corr = exp2f(m - mn);
    const float p = exp2f(sc - mn);
    l = l * corr + p;
    acc.x = acc.x * corr + p * v.x; acc.y = acc.y * corr + p * v.y;
    acc.z = acc.z * corr + p * v.z; acc.w = acc.w * corr + p * v.w;
    m = mn;
  }
  const float inv = 1.f / l;
  uint2 o;
  reinterpret_cast<__nv_bfloat162*>(&o)[0] = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
  reinterpret_cast<__nv_bfloat162*>(&o)[1] = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
  *reinterpret_cast<uint2*>(a.out + t * static_cast<int64_t>(a.Hq) * d + static_cast<int64_t>(h) * d + lane * 4) = o;
}

}  // namespace

size_t attention_workspace(int64_t max_tokens, int Hq, int d) {
  (void)max_tokens; (void)Hq; (void)d;
  return 0;
}

dl_status launch_attention(const AttnArgs& a, cudaStream_t st) {
  if (a.T <= 0) return DL_OK;
  if (a.d != 128) {
    set_error("attention: head_dim %d unsupported (128 only)", a.d);
    return DL_ERR_UNSUPPORTED;
  }
  dim3 grid(static_cast<unsigned>(a.T), static_cast<unsigned>((a.Hq + kWarpsPerCta - 1) / kWarpsPerCta));
  attn_warp_kernel<<<grid, kWarpsPerCta * 32, 0, st>>>(a);
  return cuda_status(cudaGetLastError(), "attention");
}

}  // namespace dl
