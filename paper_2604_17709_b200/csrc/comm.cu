// Tensor-parallel communicators of the C ABI (include/dl.h) and the three
// collectives the decomposed block needs (Section 2.2.1:
// partial results of the rank shards are reduce-summed; PAPER.md:174-183,
// Section 4.1: the low-rank layout all-gathers the latent):
//   all_reduce(buf)            buf = sum_r buf_r                 (in place)
//   reduce_scatter(src, dst)   dst_r = sum_j src_j[r * n, (r + 1) * n)
//   all_gather(src, dst)       dst[j * n, (j + 1) * n) = src_j
// Three kinds of communicator:
//   NCCL      the caller's ncclComm_t (one process per GPU, NVLink/NVSwitch);
//             NCCL symbols are resolved from the process that owns the comm.
//   LOOPBACK  measurement only: TP = world shapes on one GPU, the collectives
//             become local copies (results are not the sharded result).
//   GROUP     `world` ranks inside ONE process on ONE device, one host thread
//             per rank, all ranks on one shared stream (two ranks' persistent
//             kernel sequences must not run concurrently: one CTA per SM,
//             tensor-memory allocation and PDL early launch assume one
//             sequence per device).  The collectives are this library's own
//             peer-memory kernels: every rank's buffer is directly addressable
//             by the others (same device), so rank r reads the P posted
//             buffers and sums them in rank order (fp32 accumulation, one
//             rounding) -- the one-shot scheme an NVLink peer-memory
//             all-reduce uses.  Ordering between the ranks' streams is a
//             host barrier plus CUDA events: each rank records an event after
//             the producer of a collective's input, all ranks meet, then each
//             stream waits on every rank's event before the collective kernel,
//             and once more before anyone may overwrite a buffer that a peer
//             still reads.  All-reduce is in place and two-shot (reduce-
//             scatter of slabs, then all-gather), so it needs no scratch; the
//             group's symmetric window (sym_bytes per rank, one allocation)
//             belongs to the fused epilogue reductions of the decode path:
//             stage-2 epilogues red.add their partials straight into every
//             rank's window (all-reduce) or the owner's (reduce-scatter) and
//             the collective reduces to comm_barrier().  Every rank sums in the same order, so all ranks
//             receive bit-identical results (the residual stream stays
//             replicated exactly, as with NCCL).  A host barrier that is not
//             met within kBarrierTimeoutS marks the group aborted and every
//             later collective fails with DL_ERR_NCCL instead of hanging.
#include <dlfcn.h>
#include <string.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>

#include "dl_internal.h"

namespace dl {

constexpr int kMaxGroup = 8;
constexpr int kBarrierTimeoutS = 120;

struct CommGroup {
  int world = 0, device = 0;
  size_t sym_bytes = 0;
  uint8_t* sym = nullptr;   // [world][sym_bytes] device: per-rank symmetric scratch
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  bool aborted = false;
  const void* post[kMaxGroup] = {};
  cudaStream_t post_stream[kMaxGroup] = {};
  unsigned long long seq[kMaxGroup] = {};   // syncs issued by each rank (same sequence on every rank)
  cudaEvent_t ev[kMaxGroup][2] = {};
  std::atomic<int> refs{0};
};

namespace {

constexpr int kNcclSum = 0;

void* find_sym(const char* name) {
  void* p = dlsym(RTLD_DEFAULT, name);
  if (p) return p;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  return h ? dlsym(h, name) : nullptr;
}

dl_status nccl_check(const dl_comm_s* c, int r, const char* what) {
  if (r == 0) return DL_OK;
  set_error("%s failed: %s", what, c->errstr ? c->errstr(r) : "nccl error");
  return DL_ERR_NCCL;
}

size_t coll_esize(int dtype) { return dtype == kCollF32 ? 4 : 2; }

// ---------------------------------------------------------------------------
// GROUP kernels
// ---------------------------------------------------------------------------
struct PeerPtrs {
  const void* p[kMaxGroup];
};

// dst[i] = sum_{j < P} src_j[i], fp32 accumulation in rank order, one rounding.
// VEC: 16-byte accesses (all pointers 16-byte aligned, n a multiple of the
// vector width).
template <typename E, bool VEC>
__global__ void __launch_bounds__(256) peer_reduce_kernel(PeerPtrs src, int P, E* __restrict__ dst, size_t n) {
  constexpr int V = VEC ? 16 / static_cast<int>(sizeof(E)) : 1;
  const size_t nv = n / V;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nv;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float acc[V];
#pragma unroll
    for (int e = 0; e < V; ++e) acc[e] = 0.f;
    for (int j = 0; j < P; ++j) {
      const E* s = static_cast<const E*>(src.p[j]) + i * V;
      if constexpr (VEC) {
        const uint4 u = __ldcg(reinterpret_cast<const uint4*>(s));
        const E* ue = reinterpret_cast<const E*>(&u);
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] += static_cast<float>(ue[e]);
      } else {
        acc[0] += static_cast<float>(__ldcg(s));
      }
    }
    if constexpr (VEC) {
      uint4 u;
      E* ue = reinterpret_cast<E*>(&u);
#pragma unroll
      for (int e = 0; e < V; ++e) ue[e] = static_cast<E>(acc[e]);
      *reinterpret_cast<uint4*>(dst + i * V) = u;
    } else {
      dst[i] = static_cast<E>(acc[0]);
    }
  }
}

// dst[j * bytes + i] = src_j[i] for j = blockIdx.y (16-byte or byte copies)
template <bool VEC>
__global__ void __launch_bounds__(256) peer_gather_kernel(PeerPtrs src, uint8_t* __restrict__ dst, size_t bytes) {
  const int j = blockIdx.y;
  const uint8_t* s = static_cast<const uint8_t*>(src.p[j]);
  uint8_t* d = dst + static_cast<size_t>(j) * bytes;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  if constexpr (VEC) {
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < bytes / 16; i += stride)
      reinterpret_cast<uint4*>(d)[i] = __ldcg(reinterpret_cast<const uint4*>(s) + i);
  } else {
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < bytes; i += stride) d[i] = s[i];
  }
}

// dst[j * chunk .. min((j + 1) * chunk, total)) = src_j[same range] for every
// j = blockIdx.y != self (the all-gather half of the two-shot all-reduce)
template <bool VEC>
__global__ void __launch_bounds__(256) peer_slab_gather_kernel(PeerPtrs src, uint8_t* __restrict__ dst, size_t chunk,
                                                               size_t total, int self) {
  const int j = blockIdx.y;
  if (j == self) return;
  const size_t lo = static_cast<size_t>(j) * chunk;
  if (lo >= total) return;
  const size_t n = (total - lo < chunk ? total - lo : chunk);
  const uint8_t* s = static_cast<const uint8_t*>(src.p[j]) + lo;
  uint8_t* d = dst + lo;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  if constexpr (VEC) {
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n / 16; i += stride)
      reinterpret_cast<uint4*>(d)[i] = __ldcg(reinterpret_cast<const uint4*>(s) + i);
  } else {
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) d[i] = s[i];
  }
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int grid_for(size_t work) {
  const size_t g = (work + 255) / 256;
  const size_t cap = static_cast<size_t>(num_sms()) * 4;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

dl_status launch_reduce(const PeerPtrs& src, int P, void* dst, size_t n, int dtype, cudaStream_t st) {
  if (n == 0) return DL_OK;
  bool vec = al16(dst);
  for (int j = 0; j < P; ++j) vec = vec && al16(src.p[j]);
  const size_t V = 16 / coll_esize(dtype);
  vec = vec && n % V == 0;
  const int grid = grid_for(vec ? n / V : n);
  if (dtype == kCollF32) {
    if (vec) peer_reduce_kernel<float, true><<<grid, 256, 0, st>>>(src, P, static_cast<float*>(dst), n);
    else peer_reduce_kernel<float, false><<<grid, 256, 0, st>>>(src, P, static_cast<float*>(dst), n);
  } else {
    auto* d = static_cast<__nv_bfloat16*>(dst);
    if (vec) peer_reduce_kernel<__nv_bfloat16, true><<<grid, 256, 0, st>>>(src, P, d, n);
    else peer_reduce_kernel<__nv_bfloat16, false><<<grid, 256, 0, st>>>(src, P, d, n);
  }
  return launched("group reduce");
}

// ---------------------------------------------------------------------------
// GROUP host synchronisation
// ---------------------------------------------------------------------------
dl_status group_barrier(CommGroup* g) {
  std::unique_lock<std::mutex> l(g->mu);
  if (g->aborted) {
    set_error("group communicator aborted (a rank missed a collective)");
    return DL_ERR_NCCL;
  }
  const unsigned long long my = g->gen;
  if (++g->arrived == g->world) {
    g->arrived = 0;
    ++g->gen;
    g->cv.notify_all();
    return DL_OK;
  }
  const bool ok = g->cv.wait_for(l, std::chrono::seconds(kBarrierTimeoutS),
                                 [&] { return g->gen != my || g->aborted; });
  if (!ok || g->aborted) {
    g->aborted = true;
    g->cv.notify_all();
    set_error("group communicator: barrier timed out after %d s (ranks issued different collectives?)",
              kBarrierTimeoutS);
    return DL_ERR_NCCL;
  }
  return DL_OK;
}

// record this rank's event on st, meet every rank, then make st wait for
// every other rank's event of the same sync.  Events alternate between two
// slots per rank: a rank re-records a slot two syncs later, i.e. after it
// passed the next barrier, which every rank reaches only after issuing its
// waits on the slot's previous record.
dl_status group_sync(dl_comm c, cudaStream_t st) {
  CommGroup* g = c->group;
  const int slot = static_cast<int>(g->seq[c->rank]++ & 1);
  g->post_stream[c->rank] = st;
  DL_TRY_INTERNAL(cuda_status(cudaEventRecord(g->ev[c->rank][slot], st), "group: cudaEventRecord"));
  DL_TRY_INTERNAL(group_barrier(g));
  // every rank sees the same posted streams, so every rank takes the same branch
  for (int j = 0; j < g->world; ++j)
    if (g->post_stream[j] != g->post_stream[0]) {
      set_error("group communicator: all ranks must use the same stream (include/dl.h)");
      return DL_ERR_INVALID_ARG;
    }
  for (int j = 0; j < g->world; ++j)
    if (j != c->rank)
      DL_TRY_INTERNAL(cuda_status(cudaStreamWaitEvent(st, g->ev[j][slot], 0), "group: cudaStreamWaitEvent"));
  return DL_OK;
}

dl_status group_enter(dl_comm c, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs != cudaStreamCaptureStatusNone) {
    set_error("group communicator: collectives cannot be captured in a CUDA graph (host barrier)");
    return DL_ERR_UNSUPPORTED;
  }
  return cuda_status(cudaSetDevice(c->group->device), "group: cudaSetDevice");
}

PeerPtrs posted(const CommGroup* g, size_t byte_off) {
  PeerPtrs p{};
  for (int j = 0; j < g->world; ++j) p.p[j] = static_cast<const uint8_t*>(g->post[j]) + byte_off;
  return p;
}

// In-place two-shot all-reduce, no scratch: rank r sums slab r of every
// rank's buffer into its own slab r (only rank r touches slab r in this phase),
// then copies every other rank's finished slab into its buffer.  The group's
// symmetric window stays free for the fused epilogue reductions.
dl_status group_all_reduce(dl_comm c, void* buf, size_t count, int dtype, cudaStream_t st) {
  CommGroup* g = c->group;
  DL_TRY_INTERNAL(group_enter(c, st));
  const size_t es = coll_esize(dtype), P = static_cast<size_t>(g->world);
  const size_t chunk = ((count + P - 1) / P + 7) & ~static_cast<size_t>(7);   // 16-byte multiple slabs
  const size_t r = static_cast<size_t>(c->rank);
  const size_t lo = std::min(count, r * chunk), hi = std::min(count, lo + chunk);
  g->post[c->rank] = buf;
  DL_TRY_INTERNAL(group_sync(c, st));                     // every rank's input is complete
  DL_TRY_INTERNAL(launch_reduce(posted(g, lo * es), g->world, static_cast<uint8_t*>(buf) + lo * es, hi - lo, dtype,
                                st));
  DL_TRY_INTERNAL(group_sync(c, st));                     // every slab is final
  const size_t bytes = count * es, cb = chunk * es;
  bool vec = al16(buf) && cb % 16 == 0 && bytes % 16 == 0;
  for (int j = 0; j < g->world; ++j) vec = vec && al16(g->post[j]);
  const dim3 grid(grid_for(vec ? cb / 16 : cb) / g->world + 1, g->world);
  if (vec) peer_slab_gather_kernel<true><<<grid, 256, 0, st>>>(posted(g, 0), static_cast<uint8_t*>(buf), cb, bytes,
                                                               c->rank);
  else peer_slab_gather_kernel<false><<<grid, 256, 0, st>>>(posted(g, 0), static_cast<uint8_t*>(buf), cb, bytes,
                                                            c->rank);
  DL_TRY_INTERNAL(launched("group all-reduce gather"));
  return group_sync(c, st);                               // nobody reads this buffer any more
}

dl_status group_reduce_scatter(dl_comm c, const void* src, void* dst, size_t recv_count, int dtype,
                               cudaStream_t st) {
  CommGroup* g = c->group;
  DL_TRY_INTERNAL(group_enter(c, st));
  g->post[c->rank] = src;
  DL_TRY_INTERNAL(group_sync(c, st));
  DL_TRY_INTERNAL(launch_reduce(posted(g, static_cast<size_t>(c->rank) * recv_count * coll_esize(dtype)), g->world,
                                dst, recv_count, dtype, st));
  return group_sync(c, st);
}

dl_status group_all_gather(dl_comm c, const void* src, void* dst, size_t send_count, int dtype, cudaStream_t st) {
  CommGroup* g = c->group;
  DL_TRY_INTERNAL(group_enter(c, st));
  g->post[c->rank] = src;
  DL_TRY_INTERNAL(group_sync(c, st));
  const size_t bytes = send_count * coll_esize(dtype);
  if (bytes) {
    bool vec = al16(dst) && bytes % 16 == 0;
    for (int j = 0; j < g->world; ++j) vec = vec && al16(g->post[j]);
    const dim3 grid(grid_for(vec ? bytes / 16 : bytes) / g->world + 1, g->world);
    if (vec) peer_gather_kernel<true><<<grid, 256, 0, st>>>(posted(g, 0), static_cast<uint8_t*>(dst), bytes);
    else peer_gather_kernel<false><<<grid, 256, 0, st>>>(posted(g, 0), static_cast<uint8_t*>(dst), bytes);
    DL_TRY_INTERNAL(launched("group all-gather"));
  }
  return group_sync(c, st);
}

void group_release(CommGroup* g) {
  if (g->refs.fetch_sub(1) != 1) return;
  cudaSetDevice(g->device);
  for (int j = 0; j < g->world; ++j)
    for (int s = 0; s < 2; ++s)
      if (g->ev[j][s]) cudaEventDestroy(g->ev[j][s]);
  if (g->sym) cudaFree(g->sym);
  delete g;
}

}  // namespace

// ---------------------------------------------------------------------------
// symmetric window of a group communicator (fused epilogue reductions)
// ---------------------------------------------------------------------------
namespace {
// Device barrier of a multi-process window communicator (one 32-thread CTA,
// launched in plain stream order, so every earlier kernel of this rank has
// completed).  Thread 0 bumps this rank's epoch e, fences at system scope (the
// release is cumulative: the completed kernels' stores into peer windows -- the
// fused epilogue red.adds and pushes -- are ordered before it), stores e into
// slot [rank] of every peer's flag area, then lane j waits until slot [j] of
// its own area has reached e.  Epochs count barriers, so every rank must issue
// the same barrier sequence (CUDA-graph replays included: the counter lives in
// device memory).  A peer that never arrives traps after ~2^31 polls.
struct PeerFlags {
  uint32_t* slot[kMaxPeers];   // rank j's flag area (this process's mapping)
};
__global__ void __launch_bounds__(32) peer_barrier_kernel(PeerFlags f, int world, int rank) {
  uint32_t* own = f.slot[rank];
  __shared__ uint32_t e_sh;
  if (threadIdx.x == 0) {
    const uint32_t e = own[kMaxPeers] + 1;   // only this thread writes the counter
    own[kMaxPeers] = e;
    e_sh = e;
    __threadfence_system();
    for (int j = 0; j < world; ++j)
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f.slot[j] + rank), "r"(e) : "memory");
  }
  __syncwarp();
  const uint32_t e = e_sh;
  if (static_cast<int>(threadIdx.x) < world) {
    const uint32_t* p = own + threadIdx.x;
    unsigned long long polls = 0;
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
      if (static_cast<int32_t>(v - e) >= 0) break;
      if (++polls > (1ull << 31)) __trap();
      __nanosleep(64);
    }
  }
  __syncwarp();
  __threadfence_system();
}
}  // namespace

size_t comm_window_bytes(dl_comm c) {
  if (!c) return 0;
  if (c->kind == kCommGroup) return c->group->sym_bytes;
  return (c->win && c->win->connected) ? c->win->bytes : 0;
}
uint8_t* comm_window(dl_comm c, int rank) {
  if (c->kind == kCommGroup) return c->group->sym + static_cast<size_t>(rank) * c->group->sym_bytes;
  return c->win->peer[rank];
}
dl_status comm_barrier(dl_comm c, cudaStream_t st) {
  if (c->kind == kCommGroup) {
    DL_TRY_INTERNAL(group_enter(c, st));
    return group_sync(c, st);
  }
  if (!c->win || !c->win->connected) {
    set_error("comm_barrier: the communicator has no connected window");
    return DL_ERR_UNSUPPORTED;
  }
  PeerFlags f{};
  for (int j = 0; j < c->world; ++j) f.slot[j] = reinterpret_cast<uint32_t*>(c->win->peer[j] + c->win->bytes);
  peer_barrier_kernel<<<1, 32, 0, st>>>(f, c->world, c->rank);
  DL_TRY_INTERNAL(cuda_status(cudaGetLastError(), "peer barrier"));
  return launched("peer barrier");
}

// ---------------------------------------------------------------------------
// collectives used by api.cu
// ---------------------------------------------------------------------------
dl_status peer_unsupported(const char* what) {
  set_error("%s: a window-only (peer) communicator carries only the fused rank-parallel decode collectives "
            "(T <= 256, dl_block_window_bytes window); use an NCCL communicator with a window", what);
  return DL_ERR_UNSUPPORTED;
}

dl_status coll_all_reduce(dl_comm c, void* buf, size_t count, int dtype, cudaStream_t st) {
  if (count == 0) return DL_OK;
  if (c->kind == kCommPeer) return peer_unsupported("all-reduce");
  if (c->kind == kCommLoopback) return DL_OK;
  if (c->kind == kCommGroup) return group_all_reduce(c, buf, count, dtype, st);
  return nccl_check(c, c->allreduce(buf, buf, count, dtype, kNcclSum, c->nccl, st), "ncclAllReduce");
}

dl_status coll_reduce_scatter(dl_comm c, const void* src, void* dst, size_t recv_count, int dtype,
                              cudaStream_t st) {
  if (recv_count == 0) return DL_OK;
  if (c->kind == kCommPeer) return peer_unsupported("reduce-scatter");
  if (c->kind == kCommLoopback) {
    const size_t b = recv_count * coll_esize(dtype);
    return cuda_status(cudaMemcpyAsync(dst, static_cast<const uint8_t*>(src) + c->rank * b, b,
                                       cudaMemcpyDeviceToDevice, st), "loopback reduce-scatter");
  }
  if (c->kind == kCommGroup) return group_reduce_scatter(c, src, dst, recv_count, dtype, st);
  return nccl_check(c, c->reducescatter(src, dst, recv_count, dtype, kNcclSum, c->nccl, st), "ncclReduceScatter");
}

dl_status coll_all_gather(dl_comm c, const void* src, void* dst, size_t send_count, int dtype, cudaStream_t st) {
  if (send_count == 0) return DL_OK;
  if (c->kind == kCommPeer) return peer_unsupported("all-gather");
  if (c->kind == kCommLoopback) {
    const size_t b = send_count * coll_esize(dtype);
    return cuda_status(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + c->rank * b, src, b, cudaMemcpyDeviceToDevice,
                                       st), "loopback all-gather");
  }
  if (c->kind == kCommGroup) return group_all_gather(c, src, dst, send_count, dtype, st);
  return nccl_check(c, c->allgather(src, dst, send_count, dtype, c->nccl, st), "ncclAllGather");
}

}  // namespace dl

using namespace dl;

extern "C" {

dl_status dl_comm_create(void* nccl_comm, int rank, int world, dl_comm* out) {
  if (!out || !nccl_comm) {
    set_error("dl_comm_create: null argument");
    return DL_ERR_INVALID_ARG;
  }
  if (world < 1 || rank < 0 || rank >= world) {
    set_error("dl_comm_create: bad rank %d / world %d", rank, world);
    return DL_ERR_INVALID_ARG;
  }
  dl_comm_s c{};
  c.kind = kCommNccl;
  c.nccl = nccl_comm;
  c.rank = rank;
  c.world = world;
  c.allreduce = reinterpret_cast<nccl_allreduce_fn>(find_sym("ncclAllReduce"));
  c.reducescatter = reinterpret_cast<nccl_reducescatter_fn>(find_sym("ncclReduceScatter"));
  c.allgather = reinterpret_cast<nccl_allgather_fn>(find_sym("ncclAllGather"));
  c.errstr = reinterpret_cast<nccl_errstr_fn>(find_sym("ncclGetErrorString"));
  if (!c.allreduce || !c.reducescatter || !c.allgather) {
    set_error("dl_comm_create: NCCL symbols not found in the process");
    return DL_ERR_NCCL;
  }
  *out = new dl_comm_s(c);
  return DL_OK;
}

dl_status dl_comm_create_loopback(int rank, int world, dl_comm* out) {
  if (!out || world < 1 || rank < 0 || rank >= world) {
    set_error("dl_comm_create_loopback: bad arguments");
    return DL_ERR_INVALID_ARG;
  }
  dl_comm_s c{};
  c.kind = kCommLoopback;
  c.rank = rank;
  c.world = world;
  *out = new dl_comm_s(c);
  return DL_OK;
}

dl_status dl_comm_create_group(int world, size_t sym_bytes, dl_comm* comms) {
  if (!comms || world < 1 || world > kMaxGroup || sym_bytes < 256) {
    set_error("dl_comm_create_group: need 1 <= world <= %d, sym_bytes >= 256 and an output array", kMaxGroup);
    return DL_ERR_INVALID_ARG;
  }
  DL_TRY_INTERNAL(check_device_sm100());
  CommGroup* g = new CommGroup();
  g->world = world;
  g->sym_bytes = (sym_bytes + 255) & ~static_cast<size_t>(255);
  cudaError_t e = cudaGetDevice(&g->device);
  if (e == cudaSuccess) e = cudaMalloc(&g->sym, g->sym_bytes * world);
  if (e == cudaSuccess) e = cudaMemset(g->sym, 0, g->sym_bytes * world);   // window buffers are zero-maintained
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  for (int j = 0; j < world && e == cudaSuccess; ++j)
    for (int s = 0; s < 2 && e == cudaSuccess; ++s)
      e = cudaEventCreateWithFlags(&g->ev[j][s], cudaEventDisableTiming);
  if (e != cudaSuccess) {
    g->refs = 1;
    group_release(g);
    return cuda_status(e, "dl_comm_create_group");
  }
  g->refs = world;
  for (int r = 0; r < world; ++r) {
    dl_comm_s c{};
    c.kind = kCommGroup;
    c.rank = r;
    c.world = world;
    c.group = g;
    comms[r] = new dl_comm_s(c);
  }
  return DL_OK;
}

dl_status dl_comm_create_peer(int rank, int world, dl_comm* out) {
  if (!out || world < 1 || world > kMaxPeers || rank < 0 || rank >= world) {
    set_error("dl_comm_create_peer: need 1 <= world <= %d, 0 <= rank < world", kMaxPeers);
    return DL_ERR_INVALID_ARG;
  }
  dl_comm_s c{};
  c.kind = kCommPeer;
  c.rank = rank;
  c.world = world;
  *out = new dl_comm_s(c);
  return DL_OK;
}

dl_status dl_comm_window_alloc(dl_comm comm, size_t bytes) {
  if (!comm || (comm->kind != kCommNccl && comm->kind != kCommPeer) || bytes < 256 || comm->world > kMaxPeers) {
    set_error("dl_comm_window_alloc: an NCCL or peer communicator (world <= %d) and bytes >= 256", kMaxPeers);
    return DL_ERR_INVALID_ARG;
  }
  if (comm->win) {
    set_error("dl_comm_window_alloc: the communicator already has a window");
    return DL_ERR_INVALID_ARG;
  }
  DL_TRY_INTERNAL(check_device_sm100());
  PeerWindow* w = new PeerWindow();
  w->bytes = (bytes + 255) & ~static_cast<size_t>(255);
  cudaError_t e = cudaMalloc(&w->own, w->bytes + kFlagBytes);
  if (e == cudaSuccess) e = cudaMemset(w->own, 0, w->bytes + kFlagBytes);   // buffers zero-maintained, epochs 0
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (w->own) cudaFree(w->own);
    delete w;
    return cuda_status(e, "dl_comm_window_alloc");
  }
  w->peer[comm->rank] = w->own;
  comm->win = w;
  return DL_OK;
}

static_assert(sizeof(cudaIpcMemHandle_t) == DL_IPC_HANDLE_BYTES, "IPC handle size");

dl_status dl_comm_window_handle(dl_comm comm, void* handle) {
  if (!comm || !comm->win || !handle) {
    set_error("dl_comm_window_handle: no window (dl_comm_window_alloc first) or null handle");
    return DL_ERR_INVALID_ARG;
  }
  cudaIpcMemHandle_t h;
  DL_TRY_INTERNAL(cuda_status(cudaIpcGetMemHandle(&h, comm->win->own), "cudaIpcGetMemHandle"));
  memcpy(handle, &h, sizeof(h));
  return DL_OK;
}

dl_status dl_comm_window_connect(dl_comm comm, const void* handles) {
  if (!comm || !comm->win || !handles || comm->win->connected) {
    set_error("dl_comm_window_connect: needs an allocated, not yet connected window and the handles");
    return DL_ERR_INVALID_ARG;
  }
  PeerWindow* w = comm->win;
  for (int j = 0; j < comm->world; ++j) {
    if (j == comm->rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, static_cast<const uint8_t*>(handles) + static_cast<size_t>(j) * DL_IPC_HANDLE_BYTES, sizeof(h));
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (int i = 0; i < j; ++i)
        if (i != comm->rank && w->peer[i]) {
          cudaIpcCloseMemHandle(w->peer[i]);
          w->peer[i] = nullptr;
        }
      return cuda_status(e, "cudaIpcOpenMemHandle");
    }
    w->peer[j] = static_cast<uint8_t*>(p);
  }
  w->connected = true;
  return DL_OK;
}

dl_status dl_comm_destroy(dl_comm comm) {
  if (!comm) return DL_OK;
  if (comm->kind == kCommGroup && comm->group) group_release(comm->group);
  if (comm->win) {
    for (int j = 0; j < comm->world; ++j)
      if (j != comm->rank && comm->win->peer[j]) cudaIpcCloseMemHandle(comm->win->peer[j]);
    if (comm->win->own) cudaFree(comm->win->own);
    delete comm->win;
  }
  delete comm;
  return DL_OK;
}

}  // extern "C"
