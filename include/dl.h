/*
 * dl.h -- C ABI of the B200-native decomposed-LLM tensor-parallel library.
 *
 * The library computes the hot path of arxiv 2604.17709 ("DeInfer"):
 * low-rank factorised linear layers W ~= A B (Section 2.1,
 * Eq. 1; A = U_k sqrt(S_k) in R^{m x k}, B = sqrt(S_k) V_k^T in R^{k x n},
 * y = A (B x)) inside a decomposed LLaMA-3 transformer block, with the rank
 * dimension k sharded over tensor-parallel ranks (Section
 * 2.2.1, Fig. 2(b): "every process holds a small chunk of matrices", partial
 * results combined by reduce-sum).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Math convention as in the paper: W in R^{m x n}, y = W x.  Activations
 *    are token rows, row-major: X[T x n], Y[T x m], so Y = (X B^T) A^T.
 *  - Matrices are row-major with an explicit leading dimension (elements).
 *    A is [m x k] (lda >= k), B is [k x n] (ldb >= n): both are K-major,
 *    i.e. exactly the operand layout the sm_100a tensor cores consume.
 *  - All tensor arguments are DEVICE pointers owned by the caller, unless
 *    a parameter says "host".  The library never allocates device memory in
 *    dl_lowrank_linear / dl_decomposed_block_forward (CUDA-Graph capturable,
 *    PAPER.md:147-150 Section 2.2.3 "CUDA Graph requires fixed arguments");
 *    scratch comes from a caller-provided workspace sized by *_workspace().
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).  All
 *    device work is enqueued asynchronously on it; the call returns before
 *    the work completes.
 *  - Alignment: every device pointer 16-byte aligned, every leading
 *    dimension a multiple of 8 elements (bf16) / 4 elements (fp32): the TMA
 *    unit requires 16-byte row strides.  Violations -> DL_ERR_ALIGN.
 *  - Errors: arguments are validated synchronously before any launch; on a
 *    non-OK status nothing was enqueued and dl_last_error() returns a
 *    thread-local description.  Launch failures -> DL_ERR_CUDA, NCCL
 *    failures -> DL_ERR_NCCL.  Non-finite inputs are not checked.
 *  - Dtypes: DL_BF16 inputs/outputs with fp32 accumulation (tensor cores,
 *    tcgen05); DL_F32 inputs/outputs use true fp32 FFMA (SIMT path) and are
 *    limited to T <= 16 tokens per call.
 *  - There is no CPU fallback: without a usable sm_100 GPU every compute
 *    entry point returns DL_ERR_CUDA.
 */
#ifndef DL_H_
#define DL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DL_OK = 0,
  DL_ERR_INVALID_ARG = 1, /* null pointer / bad enum                          */
  DL_ERR_SHAPE = 2,       /* T < 0, m/n <= 0, ld < row length                 */
  DL_ERR_RANK = 3,        /* k < 1 or k > min(m, n)          */
  DL_ERR_PARTITION = 4,   /* k_total < world, strict split with k % world,
                             heads not divisible by world  */
  DL_ERR_DTYPE = 5,       /* dtype unsupported on the selected path          */
  DL_ERR_ALIGN = 6,       /* pointer not 16 B aligned or ld not 16 B multiple */
  DL_ERR_WORKSPACE = 7,   /* workspace NULL or smaller than *_workspace()     */
  DL_ERR_CUDA = 8,        /* no sm_100 device / launch or runtime error       */
  DL_ERR_NCCL = 9,        /* NCCL call failed or NCCL not loadable            */
  DL_ERR_UNSUPPORTED = 10 /* shape outside this version's kernels             */
} dl_status;

typedef enum { DL_F32 = 0, DL_BF16 = 1 } dl_dtype;

/* Opaque tensor-parallel communicator: wraps an ncclComm_t created by the
 * caller (e.g. torch ProcessGroupNCCL._comm_ptr()); does not own it. */
typedef struct dl_comm_s *dl_comm;

/* Thread-local message for the last non-OK status of this thread. */
const char *dl_last_error(void);
/* ABI version (major*100 + minor). */
int dl_version(void);
/* 1 if a device with compute capability 10.x is current, else 0. */
int dl_device_ok(void);

/* Reduction applied to the rank partials of dl_lowrank_linear (PAPER.md:123,
 * Fig. 2(b): the partial results of the rank shards are reduce-summed).      */
typedef enum {
  DL_REDUCE_NONE = 0,      /* no collective: Y (+)= this rank's partial A_r(B_r x) */
  DL_REDUCE_ALLREDUCE = 1, /* Y (+)= sum over ranks, [T x m] on every rank         */
  DL_REDUCE_SCATTER = 2    /* Y (+)= rank r's slab of the sum: features
                              [r m/P, (r+1) m/P), Y is [T x m/P]                 */
} dl_reduce;

/* ------------------------------------------------------------------------
 * Communicators.  Every collective has NCCL semantics and is issued on the
 * stream of the call that needs it; all ranks must issue the same sequence.
 *
 * dl_comm_create: nccl_comm is an initialised ncclComm_t (host handle) of
 *   `world` ranks in which this process is `rank` (one process per GPU over
 *   NVLink / NVSwitch).  NCCL symbols are resolved from the process (the NCCL
 *   that owns nccl_comm); DL_ERR_NCCL if absent.  The comm is not owned.
 * dl_comm_create_group: `world` (1..8) ranks inside THIS process on the
 *   current device; comms[r] (host array of `world`, filled) is rank r's
 *   communicator.  Each rank must be driven by its own host thread (the
 *   collectives meet on a host barrier), and all ranks must pass the SAME
 *   stream: the library's persistent kernels (one CTA per SM, tensor-memory
 *   allocation, programmatic early launch) are written for one kernel
 *   sequence per device, and two ranks' sequences running concurrently can
 *   starve each other; a collective whose ranks posted different streams
 *   returns DL_ERR_INVALID_ARG on every rank.  The collectives are this
 *   library's peer-memory kernels: rank r reads every rank's posted buffer
 *   directly and sums in rank order with fp32 accumulation, so every rank gets
 *   bit-identical results; the host barrier orders the ranks' enqueues (and
 *   CUDA events their streams).  sym_bytes (>= 256): per-rank symmetric scratch owned by the
 *   group (allocated once here; all-reduces larger than it run in rounds).
 *   Not capturable in a CUDA graph (DL_ERR_UNSUPPORTED during capture).  A
 *   rank that misses a collective for 120 s aborts the group: every later
 *   collective returns DL_ERR_NCCL.  Freed when all `world` comms are
 *   destroyed.  Use: TP = world on one GPU (parity of the sharded path).
 * dl_comm_create_loopback: measurement only -- `world` ranks' shapes on ONE
 *   GPU with the collectives replaced by local copies (all-gather: this
 *   rank's slice into its slot; reduce-scatter: its slot; all-reduce: no-op).
 *   Results are NOT the sharded result; the per-rank kernel work of a TP =
 *   world step is exact, so its compute time can be measured without world
 *   GPUs (tools/tp_emulate.py).
 * dl_comm_create_peer: rank `rank` of `world` (<= 8) processes whose ONLY
 *   collectives are the fused ones of the rank-parallel decode path (below):
 *   no NCCL; every other collective returns DL_ERR_UNSUPPORTED.  Needs a
 *   connected window.
 * Multi-process symmetric window (NCCL or peer communicators; the fused
 * collectives of PAPER.md:224 "communication-computation overlap and kernel
 * fusion" across processes / GPUs):
 *   dl_comm_window_alloc(comm, bytes): allocate and zero this rank's window
 *     (>= dl_block_window_bytes of the block config; owned by the comm, freed
 *     by dl_comm_destroy) plus a 256-byte flag area for the device barrier.
 *   dl_comm_window_handle(comm, handle): this window's CUDA IPC handle
 *     (DL_IPC_HANDLE_BYTES bytes written to host memory `handle`).
 *   dl_comm_window_connect(comm, handles): `handles` = world x
 *     DL_IPC_HANDLE_BYTES host bytes in rank order (exchanged by the caller,
 *     e.g. an all-gather over its process group); maps every peer's window
 *     (cudaIpcOpenMemHandle: the peers must be on GPUs with peer access --
 *     NVLink / NVSwitch -- or the same GPU).  Collective over the ranks in the
 *     sense that every rank must connect before any block call uses it.
 *   With a connected window the rank-parallel decode path (T <= 256) red.adds
 *   its stage-2 partials straight into the owners' windows over NVLink and
 *   orders the ranks with a device barrier (one 32-thread kernel: system-scope
 *   release of an epoch into every peer's flag slot, acquire-poll of its own;
 *   CUDA-graph capturable; every rank must run the same barrier sequence).
 * Any NCCL, group or peer communicator, even of world 1, selects the tensor-
 * parallel code path of the block calls; a loopback of world 1 does not.
 * ---------------------------------------------------------------------- */
#define DL_IPC_HANDLE_BYTES 64
dl_status dl_comm_create(void *nccl_comm, int rank, int world, dl_comm *out);
dl_status dl_comm_create_group(int world, size_t sym_bytes, dl_comm *comms);
dl_status dl_comm_create_loopback(int rank, int world, dl_comm *out);
dl_status dl_comm_create_peer(int rank, int world, dl_comm *out);
dl_status dl_comm_window_alloc(dl_comm comm, size_t bytes);
dl_status dl_comm_window_handle(dl_comm comm, void *handle);
dl_status dl_comm_window_connect(dl_comm comm, const void *handles);
dl_status dl_comm_destroy(dl_comm comm);

/* ------------------------------------------------------------------------
 * dl_lowrank_linear -- one decomposed linear layer
 * (Section 2.1, Eq. 1):  Y[t] (+)= A (B X[t])  for t in [0, T).
 *
 *   X [T x n] (ldx), A [m x k] (lda), B [k x n] (ldb), Y [T x m_out] (ldy),
 *   m_out = m / world for DL_REDUCE_SCATTER with a communicator, else m.
 *   comm == NULL : A, B are the full factors (reduce is irrelevant: world 1).
 *   comm != NULL : A, B are this rank's k-shards (k = k_r; the columns of A
 *                  and rows of B given by dl_tp_plan); the rank partials are
 *                  combined per `reduce`.  SCATTER needs
 *                  m % (32 * world) == 0 (DL_ERR_PARTITION).
 *   accumulate   : 0 -> Y = result;  1 -> Y = Y + result (residual fusion).
 *   The rank-k intermediate Z = X B^T is fp32-accumulated and rounded to
 *   the input dtype (bf16 for DL_BF16; fp32 stays fp32) before the second
 *   stage on every path.  Paths: T <= 16 without a bf16 collective, and all
 *   fp32 calls, run the SIMT chain (Z in shared memory when k <= 1024 and
 *   (m + n) k <= 65536, otherwise an L2-resident workspace row); larger T
 *   (or a bf16 collective) run the tcgen05 tensor-core kernels.
 *   workspace: >= dl_lowrank_linear_workspace() bytes (same T, m, n, k,
 *   dtype, comm, reduce), 256 B aligned.
 * Errors: INVALID_ARG (dtype / reduce enum), SHAPE, RANK (k < 1, or k >
 *   min(m,n) when comm == NULL), PARTITION, ALIGN, DTYPE (fp32 with T > 16),
 *   UNSUPPORTED (fp32 accumulate with a collective; m % 4 on the tensor
 *   path), WORKSPACE, CUDA, NCCL.  All checked before any launch.  T == 0 ->
 *   DL_OK no-op.
 * ---------------------------------------------------------------------- */
dl_status dl_lowrank_linear_workspace(int64_t T, int64_t m, int64_t n,
                                      int64_t k, dl_dtype dtype, dl_comm comm,
                                      dl_reduce reduce, size_t *bytes);
dl_status dl_lowrank_linear(const void *X, int64_t ldx, const void *A,
                            int64_t lda, const void *B, int64_t ldb, void *Y,
                            int64_t ldy, int64_t T, int64_t m, int64_t n,
                            int64_t k, dl_dtype dtype, int accumulate,
                            dl_comm comm, dl_reduce reduce, void *workspace,
                            size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------------
 * Rank-sharding planner, PAPER.md:183 (Section 4.1: downward factors "first
 * concatenated and then evenly split") and PAPER.md:242 (Section 4.3:
 * "appropriately partitioned and evenly distributed").
 *
 * A factor GROUP is n_seg (1..3) factor pairs that share the same input x
 * (q|k|v, gate|up, or a single matrix).  Their ranks r_0..r_{n_seg-1} are
 * concatenated into [0, R), R = sum r_g, and [0, R) is split into `world`
 * contiguous balanced ranges (rank r gets R/world, +1 for r < R % world).
 * strict != 0 reproduces SPEC.md:202: R % world != 0 -> DL_ERR_PARTITION.
 *
 * dl_tp_plan (host only): for `rank`, seg_begin[g]/seg_len[g] (host arrays
 * of n_seg) receive the rank's range inside segment g's own rank dimension
 * (len may be 0), *k_loc the rank's total.
 * ---------------------------------------------------------------------- */
dl_status dl_tp_plan(const int64_t *seg_ranks, int n_seg, int world, int rank,
                     int strict, int64_t *seg_begin, int64_t *seg_len,
                     int64_t *k_loc);

/* dl_tp_shard_factors: copy rank `rank`'s shard of a factor group on
 * `stream`.  Inputs (device): A[g] [m[g] x r[g]] (lda[g]), B[g] [r[g] x n]
 * (ldb[g]).  Outputs (device, caller-allocated): B_shard [k_loc x n]
 * (ldb_shard) = concatenation of the rank's B rows in segment order;
 * A_shard[g] [m[g] x seg_len[g]] (lda_shard[g]) = the matching columns of
 * A[g] (A_shard[g] may be NULL when seg_len[g] == 0).  seg_len_out (host,
 * optional) receives the per-segment lengths.  Host arrays: A, lda, B, ldb,
 * m, r, A_shard, lda_shard.  No collectives; runs once at load. */
dl_status dl_tp_shard_factors(int n_seg, const void *const *A,
                              const int64_t *lda, const void *const *B,
                              const int64_t *ldb, const int64_t *m,
                              const int64_t *r, int64_t n, dl_dtype dtype,
                              int world, int rank, int strict, void *B_shard,
                              int64_t ldb_shard, void *const *A_shard,
                              const int64_t *lda_shard, int64_t *seg_len_out,
                              void *stream);

/* ------------------------------------------------------------------------
 * dl_decomposed_block_forward -- one decomposed LLaMA-3 block (pipeline of
 * PAPER.md:183 Fig. 3 contents; norm/residual placement per LLaMA-3, reading
 * c9 in DESIGN.md), bf16 storage, fp32 accumulation:
 *     a = rmsnorm(x, attn_norm); q,k,v = A(B a) per matrix (one group)
 *     q,k <- RoPE(positions);  append k,v to the cache
 *     x += A_o(B_o causal_gqa_attention(q, K, V))
 *     b = rmsnorm(x, mlp_norm); x += A_down(B_down(silu(A_g(B_g b)) * A_u(B_u b)))
 * (variants via cfg->mlp_act / cfg->no_rope below; any n_heads : n_kv_heads
 * ratio -- MHA, GQA, MQA).
 * Rank sharding (comm != NULL, world P): each group's factors are the
 * rank's dl_tp_shard_factors shard; the block issues five collectives per
 * call on `stream`: reduce-scatter of the q|k|v partials by head, all-gather
 * of the attention output, all-reduce after o, gate|up and down.  Heads must
 * divide by P.  Attention runs on the rank's local heads only (removing the
 * duplicated self-attention of PAPER.md:141-144).
 * ---------------------------------------------------------------------- */
typedef struct {
  int64_t h, n_heads, n_kv_heads, head_dim, m; /* m = MLP intermediate      */
  int64_t rank_q, rank_k, rank_v, rank_o, rank_gate, rank_up, rank_down;
  float rope_theta, rms_eps;
  int64_t max_tokens; /* upper bound on T per call (workspace sizing)       */
  int64_t max_seqs;   /* upper bound on num_seqs per call                   */
  /* Model-family variants (Table 2 evaluates LLaMA-2/3
   * and OPT; "NonGLU uses ReLU").  Zero-initialised = LLaMA.   */
  int32_t mlp_act;    /* DL_MLP_SILU_GLU: x += A_down(B_down(silu(g) * u));
                         DL_MLP_RELU: x += A_down(B_down(relu(u))), no gate:
                         rank_gate must be 0 and the gu group holds the up
                         segment alone in seg[0]                            */
  int32_t no_rope;    /* 1: q, k are not rotated (positions still place the
                         cache entries)                                     */
  int32_t layout;     /* rank-sharding layout when comm != NULL (below)     */
} dl_block_config;

enum { DL_MLP_SILU_GLU = 0, DL_MLP_RELU = 1 };

/* Sharding layouts (both compute the same block; they differ in what each
 * rank stores and which collectives run, Table 1):
 * DL_LAYOUT_RANK_PARALLEL (north star, Fig. 2(b)): every factor pair split
 *   along k (dl_tp_shard_factors), partials reduced in the full space:
 *   RS(q|k|v by head), AG(attention), AR(o), AR(gate|up), AR(down).
 * DL_LAYOUT_DEINFER (Fig. 3, low-rank communication):
 *   q|k|v and gate|up ("first sub-layer"): concatenated B split by rows as
 *   above, then an all-gather of the LATENT Z [T x (l_q+l_k+l_v)], then the
 *   rank's row shard of each A (its local heads / its m/P MLP features,
 *   all l columns); o and down ("second sub-layer"): B split by input
 *   columns (the rank's local features), a reduce-sum of the LATENT
 *   partial [T x l], and the full A replicated on every rank.  Shards come
 *   from dl_deinfer_shard_factors; the weights struct then holds
 *   qkv/gu: B = concat-split rows, seg[s] = {A row shard, lda, k = l_s};
 *   o/down: B = column shard [l x n/P] (ldb), seg[0] = {full A, lda, l}.
 *   Requires m % (64 P) == 0 and h % (64 P) == 0.  Collectives per block:
 *   AG(l_q+l_k+l_v), AR(l_o), AG(l_gate+l_up), AR(l_down).                 */
enum { DL_LAYOUT_RANK_PARALLEL = 0, DL_LAYOUT_DEINFER = 1 };

/* dl_deinfer_shard_factors: copy rank `rank`'s DeInfer shard of one factor
 * group on `stream` (device memory, caller-allocated outputs).
 * sublayer 1 (q|k|v or gate|up, n_seg <= 3): B_shard [k_loc x n] is the
 *   rank's balanced share of the concatenated B rows (identical to
 *   dl_tp_shard_factors' B_shard, k_loc from dl_tp_plan); A_shard[g]
 *   [m[g]/world x r[g]] = rows [rank m[g]/world, (rank+1) m[g]/world) of
 *   A[g].  m[g] % world != 0 -> DL_ERR_PARTITION.
 * sublayer 2 (o or down, n_seg == 1): B_shard [r[0] x n/world] = columns
 *   [rank n/world, (rank+1) n/world) of B[0]; A_shard[0] [m[0] x r[0]] =
 *   a full copy of A[0].  n % world != 0 -> DL_ERR_PARTITION.
 * Leading dimensions must be multiples of 8 (bf16) / 4 (fp32).            */
dl_status dl_deinfer_shard_factors(int sublayer, int n_seg, const void *const *A,
                                   const int64_t *lda, const void *const *B,
                                   const int64_t *ldb, const int64_t *m,
                                   const int64_t *r, int64_t n, dl_dtype dtype,
                                   int world, int rank, void *B_shard,
                                   int64_t ldb_shard, void *const *A_shard,
                                   const int64_t *lda_shard, void *stream);

typedef struct {
  const void *A;  /* [m_seg x k] bf16, this rank's columns (NULL if k==0) */
  int64_t lda;    /* >= k, multiple of 8                                    */
  int64_t k;      /* this rank's rank-range length for the segment (>= 0)  */
} dl_segment;

typedef struct {
  const void *B;  /* [k_loc x n] bf16, concatenated rank rows, seg order   */
  int64_t ldb;    /* >= n, multiple of 8                                    */
  dl_segment seg[3];
} dl_factor_group;

typedef struct {
  const void *attn_norm, *mlp_norm; /* gamma, [h] bf16                     */
  dl_factor_group qkv;  /* segments q (m=h), k (m=h_kv), v (m=h_kv); n = h */
  dl_factor_group o;    /* segment o (m=h); n = h                          */
  dl_factor_group gu;   /* segments gate (m), up (m); n = h (DL_MLP_RELU:
                           seg[0] = up only)                               */
  dl_factor_group down; /* segment down (m=h); n = m                       */
} dl_block_weights;

typedef enum { DL_PREFILL = 0, DL_DECODE = 1 } dl_phase;

/* x          [T x h] bf16, residual stream, identical on every rank, updated
 *            in place.
 * positions  [T] int32 device: absolute position of each token.
 * cu_seqlens [num_seqs+1] int32 device (PREFILL): packed sequence offsets;
 *            token t of sequence s attends to tokens of s up to itself.
 * k_cache, v_cache [max_seqs x n_kv_heads/P x max_seq x head_dim] bf16:
 *            post-RoPE keys and values of this rank's kv heads.
 * cache_lens [num_seqs] int32 device: tokens already cached per sequence.
 *            PREFILL: the sequence's tokens are written at cache positions
 *            cache_lens[s] + i and attend to the cached prefix too.
 *            DECODE: T == num_seqs, token s is appended at cache_lens[s].
 *            The caller advances cache_lens after the call.  Precondition:
 *            cache_lens[s] + (tokens of s) <= max_seq; K/V of a position
 *            outside [0, max_seq) are dropped (not written), so an overrun
 *            never corrupts another head's or sequence's rows.
 * max_seq    cache capacity per sequence.
 * workspace  >= dl_block_workspace() bytes, 256 B aligned.  It must be
 *            zero-filled (cudaMemset) before its first use; every call
 *            leaves its fp32 reduction scratch zero-filled again (the
 *            epilogues consume-and-clear), so no per-call memset is needed.
 *            The workspace layout depends on the config (ranks, dims,
 *            max_tokens, layout) and world: a workspace may be shared only
 *            by calls with the same config (e.g. all layers of a model with
 *            uniform ranks); layers with different ranks need their own.
 *            Errors: SHAPE (T > max_tokens, num_seqs), PARTITION (heads %
 *            world, shard wider than the balanced split), RANK, ALIGN,
 *            UNSUPPORTED (head_dim != 128), WORKSPACE, CUDA, NCCL.       */
dl_status dl_block_workspace(const dl_block_config *cfg, int world,
                             size_t *bytes);
/* Bytes of a communicator's symmetric window (dl_comm_create_group sym_bytes,
 * or dl_comm_window_alloc) that the fused collectives of this config need:
 * with a window, the rank-parallel decode path (T <= 256) red.adds its
 * stage-2 partials straight into the ranks' windows (all-reduce into every
 * rank's copy, reduce-scatter into the owner's) and pushes the attention
 * output into every rank's all-gather slot, so each collective is a barrier
 * instead of a pass over the data.  With a smaller window (or another
 * communicator kind) the same calls run the collective kernels instead.
 * 0 for DL_LAYOUT_DEINFER (always the collective path). */
dl_status dl_block_window_bytes(const dl_block_config *cfg, int world,
                                size_t *bytes);
dl_status dl_decomposed_block_forward(
    const dl_block_config *cfg, const dl_block_weights *w, void *x, int64_t T,
    const int32_t *positions, const int32_t *cu_seqlens, int32_t num_seqs,
    dl_phase phase, void *k_cache, void *v_cache, const int32_t *cache_lens,
    int64_t max_seq, dl_comm comm, void *workspace, size_t workspace_bytes,
    void *stream);

/* dl_decomposed_stack_forward -- n_layers consecutive blocks sharing one
 * config and one workspace: exactly dl_decomposed_block_forward applied to
 * layers 0 .. n_layers-1 in order (w[l], k_caches[l], v_caches[l] per layer;
 * host arrays of device pointers), same arguments and errors otherwise.  On
 * the single-GPU decode path the residual add that ends block l is fused with
 * block l+1's attention RMSNorm (one kernel instead of two per boundary).
 * n_layers == 0 is a no-op.                                                 */
dl_status dl_decomposed_stack_forward(
    const dl_block_config *cfg, const dl_block_weights *const *w, int32_t n_layers,
    void *x, int64_t T, const int32_t *positions, const int32_t *cu_seqlens,
    int32_t num_seqs, dl_phase phase, void *const *k_caches, void *const *v_caches,
    const int32_t *cache_lens, int64_t max_seq, dl_comm comm, void *workspace,
    size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------------
 * Paged low-rank KV cache ("the low-rank
 * intermediate results between the two matrix multiplications now act as KV
 * caches", PAPER.md:219-237 two-stage reconstruction).
 *
 * Every cached token stores its latent z_k = B_k a and z_v = B_v a instead of
 * post-RoPE K / V: (l_k + l_v) / (2 h_kv) of the bytes (0.6 at 40 %).
 * Pool: num_blocks blocks of block_size slots; slot row (bf16, ld_slot
 * elements, multiple of 8) = [z_k (l_k) | zero pad to zv_off | z_v (l_v)]
 * with zv_off = rup(l_k, 64); slot_pos holds each slot's position.
 * A decode step has the paper's two stages:
 *  preparation (host, before the replay; any CPU / GPU work allowed):
 *    dl_kv_prepare scans each sequence's block table for physically
 *    contiguous runs and derives the remapping index list (the first
 *    buffer block of each sequence); the caller copies the plan to the
 *    device arrays below.
 *  replay (device, fixed buffers and shapes, CUDA-Graph capturable):
 *    dl_decomposed_block_forward_kvlr appends the new tokens' latents to the
 *    pool, copies the runs into the squeeze buffer, reconstructs K | V of the
 *    whole buffer capacity with ONE fixed-size tcgen05 GEMM ("we only need to
 *    use the GEMM kernel that has a large size"), rotates K in place
 *    with the stored positions and attends through the remapping list.
 * Works at TP = 1 and with DL_LAYOUT_DEINFER (the latent is all-gathered, so
 * every rank holds the full low-rank cache and reconstructs its local kv
 * heads); the rank-parallel layout at P > 1 has only partial latents:
 * DL_ERR_UNSUPPORTED.
 * ---------------------------------------------------------------------- */
typedef struct {
  void *pool;                  /* [num_blocks * block_size][ld_slot] bf16    */
  int32_t *slot_pos;           /* [num_blocks * block_size]                  */
  int64_t num_blocks, block_size, ld_slot;
  const int32_t *block_tables; /* device [max_seqs][max_blocks_per_seq]      */
  int64_t max_blocks_per_seq;
  /* plan (device int32, from dl_kv_prepare)                                 */
  const int32_t *run_src;      /* [max_runs] first physical block of run r   */
  const int32_t *run_dst;      /* [max_runs] first buffer block (ascending)  */
  const int32_t *run_len;      /* [max_runs] length in blocks                */
  const int32_t *n_runs;       /* [1]                                        */
  const int32_t *seq_block;    /* [max_seqs] remapping index list            */
  /* fixed buffers (caller-owned, allocated once)                            */
  void *squeeze;               /* [cap_blocks * block_size][ld_slot] bf16    */
  int32_t *squeeze_pos;        /* [cap_blocks * block_size]                  */
  void *recon;                 /* [cap_blocks * block_size][2 h_kv / P] bf16 */
  int64_t cap_blocks;
} dl_kv_lowrank;

/* dl_kv_prepare (host only): block_tables [num_seqs][max_blocks_per_seq]
 * (host), seq_tokens[s] = tokens of sequence s AFTER this step's append.
 * Outputs (host, caller-allocated): run_src / run_dst / run_len [max_runs],
 * *n_runs, seq_block [num_seqs].  Runs never cross sequences; a run starts
 * where block i+1 is not physically block i + 1.  Errors: SHAPE (bad sizes,
 * block id < 0), WORKSPACE (more than max_runs runs or cap_blocks blocks). */
dl_status dl_kv_prepare(const int32_t *block_tables, int64_t max_blocks_per_seq,
                        const int32_t *seq_tokens, int32_t num_seqs,
                        int64_t block_size, int64_t max_runs, int64_t cap_blocks,
                        int32_t *run_src, int32_t *run_dst, int32_t *run_len,
                        int32_t *n_runs, int32_t *seq_block);

/* Decode step of one block with the low-rank cache (T == num_seqs new
 * tokens, token s at position positions[s], appended at slot cache_lens[s]
 * of sequence s; attention covers cache_lens[s] + 1 keys).  Other arguments
 * as dl_decomposed_block_forward.  Extra errors: INVALID_ARG (kv fields),
 * UNSUPPORTED (rank-parallel layout at P > 1).                             */
dl_status dl_decomposed_block_forward_kvlr(
    const dl_block_config *cfg, const dl_block_weights *w, void *x, int64_t T,
    const int32_t *positions, const dl_kv_lowrank *kv, const int32_t *cache_lens,
    dl_comm comm, void *workspace, size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------------
 * Model-level helpers used by the decode / prefill step (embedding gather,
 * final norm + dense LM head).  Not part of the paper's method; provided so
 * a whole-model step runs in this library's kernels only.
 * ---------------------------------------------------------------------- */
/* Greedy next token: ids[t] = argmax_v logits (bf16) over P vocab shards,
 * element (t, global id p*vloc + v) at logits[p*rank_stride + t*ld + v]
 * (P = 1: plain [T x ld]); ties go to the smallest id.  ids: device int32 [T]. */
dl_status dl_argmax(const void *logits, int64_t T, int64_t vloc, int32_t P,
                    int64_t rank_stride, int64_t ld, int32_t *ids, void *stream);
/* out[t] = table[ids[t]]   (table [vocab x h] bf16, out [T x h] bf16)     */
dl_status dl_embedding(const void *table, int64_t vocab, int64_t h,
                       const int32_t *ids, int64_t T, void *out, void *stream);
/* out = rmsnorm(x, gamma) (bf16, fp32 math)                               */
dl_status dl_rmsnorm(const void *x, const void *gamma, void *out, int64_t T,
                     int64_t h, float eps, void *stream);
/* Dense C[T x N] = X[T x K] W[N x K]^T (bf16 in/out, fp32 acc, tcgen05),
 * used for the vocab-sharded LM head; workspace per dl_dense_workspace.   */
dl_status dl_dense_workspace(int64_t T, int64_t N, int64_t K, size_t *bytes);
dl_status dl_dense(const void *X, int64_t ldx, const void *W, int64_t ldw,
                   void *C, int64_t ldc, int64_t T, int64_t N, int64_t K,
                   void *workspace, size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------------
 * Instrumentation (used by bench.py; host-side state, not thread-safe
 * across concurrent captures).
 * dl_launch_count: kernels this library enqueued since load (a CUDA-Graph
 *   capture counts each captured launch once).
 * dl_profile_begin(capacity): from now on record a CUDA event pair around
 *   each tcgen05 GEMM launch (first `capacity` launches; inside a stream
 *   capture as external event-record nodes, so graph replays re-record).
 * dl_profile_get(i): elapsed ms of record i plus its algorithmic bytes and
 *   flops (weights + activations + outputs, each counted once) and kind
 *   (1 = swap-AB decode path, 0 = wide prefill path).
 * ---------------------------------------------------------------------- */
long long dl_launch_count(void);
dl_status dl_profile_begin(int capacity);
dl_status dl_profile_end(void);
int dl_profile_count(void);
dl_status dl_profile_get(int i, float *ms, double *bytes, double *flops,
                         int *kind);
/* Debug timeline of the tcgen05 GEMM CTAs (device_buf: >= 8 u64 per CTA of
 * the next launches, or NULL to disable): globaltimer ns at entry, setup
 * done, first TMA issued, first stage landed, last MMA issued, epilogue
 * done, exit; slot 7 = SM id. */
dl_status dl_debug_gemm_trace(void *device_buf);
/* Debug timeline of the non-GEMM decode kernels (SiLU*up, residual +
 * RMSNorm, RoPE + cache append, stream-K attention): device_buf >= 4 u64 per
 * launch of the next launches (kind 1-4, then globaltimer ns of the first CTA
 * entry, the first return from griddepcontrol.wait, the last CTA end; fill
 * entries 1-2 with ~0 and 3 with 0 before the run), or NULL to disable.     */
dl_status dl_debug_ew_trace(void *device_buf);
/* Test hook: Y[T x m] = A (B X) with X given rank-major as the attention
 * all-gather leaves it, Xg [P][T][n/P] (X[t][p*n/P + c] = Xg[p][t][c]); the
 * stage-1 TMA reads it through a 3-D map exactly as the TP o projection does.
 * bf16, 1 <= T <= 256, (n/P) % 64 == 0; workspace per dl_lowrank_linear_workspace. */
dl_status dl_debug_linear_gathered(const void *Xg, int P, const void *A, int64_t lda,
                                   const void *B, int64_t ldb, void *Y, int64_t ldy,
                                   int64_t T, int64_t m, int64_t n, int64_t k,
                                   void *workspace, size_t workspace_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DL_H_ */
