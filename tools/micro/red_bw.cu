// L2 reduction-throughput microbenchmark: red.add.f32 / red.add.v4.f32 / plain
// v4 stores over a buffer, all SMs.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 red_bw.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void red1(float* p, int n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
      asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p + i), "f"(1.f) : "memory");
}
__global__ void red4(float* p, int n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += gridDim.x * blockDim.x * 4)
      asm volatile("red.global.add.v4.f32 [%0], {%1,%1,%1,%1};" ::"l"(p + i), "f"(1.f) : "memory");
}
__global__ void red2bf(float* p, int n, int reps) {   // packed bf16x2 adds over the same bytes
  unsigned* q = reinterpret_cast<unsigned*>(p);
  for (int r = 0; r < reps; ++r)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
      asm volatile("red.global.add.noftz.bf16x2 [%0], %1;" ::"l"(q + i), "r"(0x3f803f80u) : "memory");
}
__global__ void st4(float* p, int n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += gridDim.x * blockDim.x * 4)
      *reinterpret_cast<float4*>(p + i) = make_float4(r, r, r, r);
}
__global__ void ld4(const float* p, int n, int reps, float* out) {
  float s = 0;
  for (int r = 0; r < reps; ++r)
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += gridDim.x * blockDim.x * 4) {
      float4 v = __ldcg(reinterpret_cast<const float4*>(p + i));
      s += v.x + v.y + v.z + v.w;
    }
  if (s == 12345.f) *out = s;
}
int main() {
  const int n = 4 << 20;   // 16 MB of floats (L2 resident)
  float *p, *o;
  cudaMalloc(&p, n * 4); cudaMalloc(&o, 4);
  cudaMemset(p, 0, n * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int reps = 20;
  auto run = [&](const char* name, auto fn) {
    fn(); cudaDeviceSynchronize();
    cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-8s %8.1f us for %d x 16 MB -> %7.0f GB/s\n", name, ms * 1e3, reps, 16.0 * reps * 1.048576e6 / (ms * 1e-3) / 1e9);
  };
  run("red.f32", [&] { red1<<<148 * 8, 256>>>(p, n, reps); });
  run("red.v4", [&] { red4<<<148 * 8, 256>>>(p, n, reps); });
  run("red.bf16x2", [&] { red2bf<<<148 * 8, 256>>>(p, n, reps); });
  run("st.v4", [&] { st4<<<148 * 8, 256>>>(p, n, reps); });
  run("ld.cg.v4", [&] { ld4<<<148 * 8, 256>>>(p, n, reps, o); });
  return 0;
}
