// Launch accounting and CUDA-event instrumentation of the tcgen05 GEMMs.
// bench.py uses these to count this library's kernel launches and to time
// the dominant kernel per launch with events on the launching stream (also
// inside CUDA-Graph capture, as external event-record nodes).
#include <atomic>
#include <mutex>
#include <vector>

#include "dl_internal.h"

namespace dl {
namespace {

std::atomic<long long> g_launches{0};

struct Rec {
  cudaEvent_t start = nullptr, stop = nullptr;
  double bytes = 0, flops = 0;
  int kind = 0;
};
std::mutex g_mu;
std::vector<Rec> g_recs;
int g_next = 0;
bool g_on = false;

void record(cudaEvent_t e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
  else
    cudaEventRecord(e, st);
}

}  // namespace

dl_status launched(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError(), what);
}

int prof_begin(cudaStream_t st) {
  std::lock_guard<std::mutex> l(g_mu);
  if (!g_on || g_next >= static_cast<int>(g_recs.size())) return -1;
  const int i = g_next++;
  record(g_recs[i].start, st);
  return i;
}

void prof_end(int i, cudaStream_t st, double bytes, double flops, int kind) {
  if (i < 0) return;
  std::lock_guard<std::mutex> l(g_mu);
  record(g_recs[i].stop, st);
  g_recs[i].bytes = bytes;
  g_recs[i].flops = flops;
  g_recs[i].kind = kind;
}

}  // namespace dl

using namespace dl;

extern "C" {

long long dl_launch_count(void) { return g_launches.load(); }

dl_status dl_debug_gemm_trace(void* device_buf) { return set_gemm_trace(device_buf); }
dl_status dl_debug_ew_trace(void* device_buf) { return set_ew_trace(device_buf); }


dl_status dl_profile_begin(int capacity) {
  std::lock_guard<std::mutex> l(g_mu);
  if (capacity < 0) return DL_ERR_INVALID_ARG;
  while (static_cast<int>(g_recs.size()) < capacity) {
    Rec r;
    if (cudaEventCreate(&r.start) != cudaSuccess || cudaEventCreate(&r.stop) != cudaSuccess) {
      set_error("cudaEventCreate failed");
      return DL_ERR_CUDA;
    }
    g_recs.push_back(r);
  }
  g_next = 0;
  g_on = true;
  return DL_OK;
}

dl_status dl_profile_end(void) {
  std::lock_guard<std::mutex> l(g_mu);
  g_on = false;
  return DL_OK;
}

int dl_profile_count(void) {
  std::lock_guard<std::mutex> l(g_mu);
  return g_next;
}

dl_status dl_profile_get(int i, float* ms, double* bytes, double* flops, int* kind) {
  std::lock_guard<std::mutex> l(g_mu);
  if (i < 0 || i >= g_next || !ms || !bytes || !flops || !kind) {
    set_error("dl_profile_get: bad index or null output");
    return DL_ERR_INVALID_ARG;
  }
  cudaError_t e = cudaEventElapsedTime(ms, g_recs[i].start, g_recs[i].stop);
  if (e != cudaSuccess) return cuda_status(e, "cudaEventElapsedTime");
  *bytes = g_recs[i].bytes;
  *flops = g_recs[i].flops;
  *kind = g_recs[i].kind;
  return DL_OK;
}

}  // extern "C"
