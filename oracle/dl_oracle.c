/*
 * dl_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the
 * decomposed-LLM tensor-parallel hot path of arxiv 2604.17709 ("DeInfer").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2604_17709_b200/csrc) and never includes anything from it.
 *
 * Citations: "P:<line>" = /root/reference/PAPER.md line (section / equation),
 * "S:<line>" = SPEC.md line.  Readings of silent/ambiguous points are the
 * c1..c15 readings listed in DESIGN.md ("Readings of the paper").
 *
 * Conventions (all functions):
 *   - every matrix is dense, row-major, fp64, contiguous (no leading dims);
 *   - paper math convention W in R^{m x n}, y = W x ~= A (B x) with
 *     A in R^{m x k}, B in R^{k x n}  (Section 2.1, Eq. 1);
 *   - activations are token rows: X[T x n], Y[T x m]  (Y[t] = A (B X[t]));
 *   - return value 0 = OK, negative = argument error (see ORC_E* below).
 *   - OpenMP only distributes INDEPENDENT outputs (rows / tokens) across
 *     threads; every output is computed by the plain definition, in the
 *     order the definition states.  No blocking, no fusion, no reordering.
 *
 * Parity status of each function is recorded in DESIGN.md ("Oracle pins");
 * every exported function below is pinned by a -m "not gpu" test.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ESHAPE (-1)
#define ORC_ERANK (-2)
#define ORC_EPARTITION (-3)
#define ORC_ENOMEM (-4)

/* ------------------------------------------------------------------------ */
/* Library primitive: plain matrix product C[M x N] = A[M x K] . B[K x N].    */
/* Used only as a step ("exact mathematical product").               */
/* ------------------------------------------------------------------------ */
int oracle_matmul(const double *A, const double *B, double *C, int64_t M,
                  int64_t K, int64_t N) {
  if (M < 0 || K < 0 || N < 0) return ORC_ESHAPE;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i) {
    for (int64_t j = 0; j < N; ++j) {
      double s = 0.0;
      for (int64_t l = 0; l < K; ++l) s += A[i * K + l] * B[l * N + j];
      C[i * N + j] = s;
    }
  }
  return ORC_OK;
}

/* Z[T x k] = X[T x n] B[k x n]^T: the downward projection alone (stage 1, */
/* x_v of P:168), used where the paper stores the low-rank result itself.  */
static int oracle_matmul_bt(const double *X, const double *B, double *Z,
                            int64_t T, int64_t n, int64_t k) {
  for (int64_t t = 0; t < T; ++t)
    for (int64_t j = 0; j < k; ++j) {
      double s = 0.0;
      for (int64_t l = 0; l < n; ++l) s += B[j * n + l] * X[t * n + l];
      Z[t * k + j] = s;
    }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Low-rank linear, P:103-109 (Section 2.1, Eq. 1): y = A (B x).             */
/*   Z[t][j] = sum_l B[j][l] X[t][l]        (downward projection x_v) */
/*   Y[t][i] = sum_j A[i][j] Z[t][j]        (upward projection x_u)          */
/* Stage order A(Bx) as the paper writes it; no intermediate rounding.       */
/* ------------------------------------------------------------------------ */
int oracle_lowrank_linear(const double *X, const double *A, const double *B,
                          double *Y, int64_t T, int64_t m, int64_t n,
                          int64_t k) {
  if (T < 0 || m <= 0 || n <= 0 || k < 0) return ORC_ESHAPE;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    double *z = (double *)malloc(sizeof(double) * (size_t)(k > 0 ? k : 1));
    for (int64_t j = 0; j < k; ++j) {
      double s = 0.0;
      for (int64_t l = 0; l < n; ++l) s += B[j * n + l] * X[t * n + l];
      z[j] = s;
    }
    for (int64_t i = 0; i < m; ++i) {
      double s = 0.0;
      for (int64_t j = 0; j < k; ++j) s += A[i * k + j] * z[j];
      Y[t * m + i] = s;
    }
    free(z);
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Rank-shard plan, P:123 (Section 2.2.1: "every process holds a small chunk  */
/* of matrices"), P:183 ("evenly split"), P:242 ("appropriately partitioned   */
/* and evenly distributed").  Reading c3: balanced contiguous     */
/* split of [0,k): rank r gets k/P (+1 for the first k%P ranks); align>=1    */
/* pads the shard length up to a multiple of align with zero rows/cols;      */
/* align==0 is SPEC's strict mode: k % P != 0 is an error.    */
/* Recomputed here independently of the product planner.                     */
/* ------------------------------------------------------------------------ */
int oracle_shard_range(int64_t k, int world, int rank, int64_t align,
                       int64_t *begin, int64_t *len, int64_t *len_pad) {
  if (world < 1 || rank < 0 || rank >= world || k < 0 || align < 0)
    return ORC_EPARTITION;
  if (align == 0 && (k % world) != 0) return ORC_EPARTITION;
  int64_t base = k / world, extra = k % world;
  int64_t b = 0;
  for (int r = 0; r < rank; ++r) b += base + (r < extra ? 1 : 0);
  int64_t l = base + (rank < extra ? 1 : 0);
  int64_t a = align == 0 ? 1 : align;
  *begin = b;
  *len = l;
  *len_pad = ((l + a - 1) / a) * a;
  return ORC_OK;
}

/* Sharded low-rank linear, Fig. 2(b) / P:121-123 ("for each paired low-rank */
/* matrices, there is a reduce-sum"): Y = sum_r A[:,K_r] (B[K_r,:] x), each   */
/* rank's shard zero-padded to len_pad (zero rows of B / zero columns of A).  */
int oracle_lowrank_linear_sharded(const double *X, const double *A,
                                  const double *B, double *Y, int64_t T,
                                  int64_t m, int64_t n, int64_t k, int world,
                                  int64_t align) {
  if (T < 0 || m <= 0 || n <= 0 || k < 1) return ORC_ESHAPE;
  for (int64_t i = 0; i < T * m; ++i) Y[i] = 0.0;
  for (int r = 0; r < world; ++r) {
    int64_t b0, len, lp;
    int rc = oracle_shard_range(k, world, r, align, &b0, &len, &lp);
    if (rc) return rc;
    if (lp == 0) continue;
    /* materialise this rank's padded shard: A_r [m x lp], B_r [lp x n] */
    double *Ar = (double *)calloc((size_t)(m * lp), sizeof(double));
    double *Br = (double *)calloc((size_t)(lp * n), sizeof(double));
    double *Yr = (double *)malloc(sizeof(double) * (size_t)(T * m > 0 ? T * m : 1));
    if (!Ar || !Br || !Yr) { free(Ar); free(Br); free(Yr); return ORC_ENOMEM; }
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < len; ++j) Ar[i * lp + j] = A[i * k + b0 + j];
    for (int64_t j = 0; j < len; ++j)
      for (int64_t l = 0; l < n; ++l) Br[j * n + l] = B[(b0 + j) * n + l];
    oracle_lowrank_linear(X, Ar, Br, Yr, T, m, n, lp);
    /* reduce-sum over ranks */
    for (int64_t i = 0; i < T * m; ++i) Y[i] += Yr[i];
    free(Ar); free(Br); free(Yr);
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Truncated SVD, P:103-109 (Eq. 1): W ~= A B, A = U_k sqrt(S_k) [m x k],    */
/* B = sqrt(S_k) V_k^T [k x n].  One-sided Jacobi (Hestenes) on the columns  */
/* of W (or of W^T when m < n).  sigma_all receives all       */
/* min(m,n) singular values in non-increasing order.                         */
/* ------------------------------------------------------------------------ */
static int jacobi_svd_tall(const double *W, int64_t m, int64_t n, double *U,
                           double *S, double *V) {
  /* W is m x n with m >= n.  Produces W = U diag(S) V^T, U m x n, V n x n. */
  double *G = (double *)malloc(sizeof(double) * (size_t)(m * n));
  if (!G) return ORC_ENOMEM;
  memcpy(G, W, sizeof(double) * (size_t)(m * n));
  for (int64_t i = 0; i < n * n; ++i) V[i] = 0.0;
  for (int64_t i = 0; i < n; ++i) V[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int64_t p = 0; p < n - 1; ++p) {
      for (int64_t q = p + 1; q < n; ++q) {
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        for (int64_t i = 0; i < m; ++i) {
          alpha += G[i * n + p] * G[i * n + p];
          beta += G[i * n + q] * G[i * n + q];
          gamma += G[i * n + p] * G[i * n + q];
        }
        if (gamma == 0.0) continue;
        double c_off = fabs(gamma) / sqrt(alpha * beta);
        if (c_off > off) off = c_off;
        if (c_off < 1e-15) continue;
        double zeta = (beta - alpha) / (2.0 * gamma);
        double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int64_t i = 0; i < m; ++i) {
          double gp = G[i * n + p], gq = G[i * n + q];
          G[i * n + p] = c * gp - s * gq;
          G[i * n + q] = s * gp + c * gq;
        }
        for (int64_t i = 0; i < n; ++i) {
          double vp = V[i * n + p], vq = V[i * n + q];
          V[i * n + p] = c * vp - s * vq;
          V[i * n + q] = s * vp + c * vq;
        }
      }
    }
    if (off < 1e-15) break;
  }
  for (int64_t j = 0; j < n; ++j) {
    double s = 0.0;
    for (int64_t i = 0; i < m; ++i) s += G[i * n + j] * G[i * n + j];
    s = sqrt(s);
    S[j] = s;
    for (int64_t i = 0; i < m; ++i) U[i * n + j] = s > 0 ? G[i * n + j] / s : 0.0;
  }
  free(G);
  return ORC_OK;
}

int oracle_truncated_svd(const double *W, int64_t m, int64_t n, int64_t k,
                         double *A, double *B, double *sigma_all) {
  if (m <= 0 || n <= 0) return ORC_ESHAPE;
  int64_t r = m < n ? m : n;
  if (k < 1 || k > r) return ORC_ERANK;
  int tall = m >= n;
  int64_t M = tall ? m : n, N = tall ? n : m; /* work on the tall one */
  double *Wt = (double *)malloc(sizeof(double) * (size_t)(M * N));
  double *U = (double *)malloc(sizeof(double) * (size_t)(M * N));
  double *S = (double *)malloc(sizeof(double) * (size_t)N);
  double *V = (double *)malloc(sizeof(double) * (size_t)(N * N));
  int64_t *ord = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
  if (!Wt || !U || !S || !V || !ord) {
    free(Wt); free(U); free(S); free(V); free(ord);
    return ORC_ENOMEM;
  }
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      if (tall) Wt[i * n + j] = W[i * n + j];
      else Wt[j * m + i] = W[i * n + j];
    }
  int rc = jacobi_svd_tall(Wt, M, N, U, S, V);
  if (rc) { free(Wt); free(U); free(S); free(V); free(ord); return rc; }
  /* order singular values non-increasing (selection sort, N is small) */
  for (int64_t i = 0; i < N; ++i) ord[i] = i;
  for (int64_t i = 0; i < N; ++i)
    for (int64_t j = i + 1; j < N; ++j)
      if (S[ord[j]] > S[ord[i]]) { int64_t t = ord[i]; ord[i] = ord[j]; ord[j] = t; }
  if (sigma_all)
    for (int64_t i = 0; i < N; ++i) sigma_all[i] = S[ord[i]];
  /* tall: W = U S V^T  -> left = U, right = V.
     wide: W^T = U S V^T -> W = V S U^T -> left = V, right = U. */
  for (int64_t j = 0; j < k; ++j) {
    int64_t c = ord[j];
    double rs = sqrt(S[c]);
    for (int64_t i = 0; i < m; ++i)
      A[i * k + j] = rs * (tall ? U[i * N + c] : V[i * N + c]);
    for (int64_t l = 0; l < n; ++l)
      B[j * n + l] = rs * (tall ? V[l * N + c] : U[l * N + c]);
  }
  free(Wt); free(U); free(S); free(V); free(ord);
  return ORC_OK;
}

/* Parameter count of one factor pair: "(m + n) x k". */
int64_t oracle_factor_params(int64_t m, int64_t n, int64_t k) {
  return (m + n) * k;
}

/* ------------------------------------------------------------------------ */
/* Block pieces (LLaMA-3 block; the paper is silent on norm placement, eps,  */
/* RoPE base -- readings c9 in DESIGN.md; S:300 notes the silence).          */
/* ------------------------------------------------------------------------ */

/* RMSNorm: y_i = x_i * g_i / sqrt(mean_j x_j^2 + eps). */
void oracle_rmsnorm(const double *x, const double *g, double eps, double *y,
                    int64_t T, int64_t h) {
  for (int64_t t = 0; t < T; ++t) {
    double ss = 0.0;
    for (int64_t i = 0; i < h; ++i) ss += x[t * h + i] * x[t * h + i];
    double inv = 1.0 / sqrt(ss / (double)h + eps);
    for (int64_t i = 0; i < h; ++i) y[t * h + i] = x[t * h + i] * inv * g[i];
  }
}

/* RoPE, P:222 ("in-place rotary position embedding"): each head  */
/* vector of dim d, pair (2i, 2i+1) rotated by angle pos * theta^(-2i/d).    */
/* v is [T x nh x d], rotated in place.                                      */
void oracle_rope(double *v, const int32_t *pos, int64_t T, int64_t nh,
                 int64_t d, double theta) {
  for (int64_t t = 0; t < T; ++t)
    for (int64_t hh = 0; hh < nh; ++hh)
      for (int64_t i = 0; i < d / 2; ++i) {
        double ang = (double)pos[t] * pow(theta, -2.0 * (double)i / (double)d);
        double c = cos(ang), s = sin(ang);
        double *p = v + (t * nh + hh) * d + 2 * i;
        double a = p[0], b = p[1];
        p[0] = a * c - b * s;
        p[1] = a * s + b * c;
      }
}

/* Attention for ONE query vector against a list of keys:        */
/* out = sum_u softmax_u(q.k_u / sqrt(d)) v_u, max-subtracted.  GQA: query    */
/* head g reads kv head floor(g * Hkv / H).  keys/vals are given as   */
/* arrays of row pointers (each row = Hkv*d values of one token).            */
static void attend_one(const double *q /* H*d */, const double *const *krows,
                       const double *const *vrows, int64_t nkeys, int64_t H,
                       int64_t Hkv, int64_t d, double *out /* H*d */) {
  double *sc = (double *)malloc(sizeof(double) * (size_t)(nkeys > 0 ? nkeys : 1));
  double scale = 1.0 / sqrt((double)d);
  for (int64_t g = 0; g < H; ++g) {
    int64_t j = (g * Hkv) / H;
    double mx = -INFINITY;
    for (int64_t u = 0; u < nkeys; ++u) {
      double s = 0.0;
      for (int64_t e = 0; e < d; ++e) s += q[g * d + e] * krows[u][j * d + e];
      sc[u] = s * scale;
      if (sc[u] > mx) mx = sc[u];
    }
    double den = 0.0;
    for (int64_t u = 0; u < nkeys; ++u) { sc[u] = exp(sc[u] - mx); den += sc[u]; }
    for (int64_t e = 0; e < d; ++e) {
      double s = 0.0;
      for (int64_t u = 0; u < nkeys; ++u) s += sc[u] * vrows[u][j * d + e];
      out[g * d + e] = s / den;
    }
  }
  free(sc);
}

/* Causal GQA attention over packed sequences.  q [T x H*d], k,v [T x Hkv*d]; */
/* cu_seqlens [nseq+1]; token t of sequence s attends to tokens u of s with   */
/* u <= t (packed order = position order).  out [T x H*d].                    */
int oracle_attention(const double *q, const double *k, const double *v,
                     double *out, int64_t T, const int32_t *cu_seqlens,
                     int32_t nseq, int64_t H, int64_t Hkv, int64_t d) {
  if (H <= 0 || Hkv <= 0 || H % Hkv != 0 || d <= 0) return ORC_ESHAPE;
  if (cu_seqlens[0] != 0 || cu_seqlens[nseq] != T) return ORC_ESHAPE;
  for (int32_t s = 0; s < nseq; ++s) {
    int64_t b0 = cu_seqlens[s], b1 = cu_seqlens[s + 1];
#pragma omp parallel for schedule(dynamic)
    for (int64_t t = b0; t < b1; ++t) {
      int64_t nk = t - b0 + 1;
      const double **kr = (const double **)malloc(sizeof(double *) * (size_t)nk);
      const double **vr = (const double **)malloc(sizeof(double *) * (size_t)nk);
      for (int64_t u = 0; u < nk; ++u) {
        kr[u] = k + (b0 + u) * Hkv * d;
        vr[u] = v + (b0 + u) * Hkv * d;
      }
      attend_one(q + t * H * d, kr, vr, nk, H, Hkv, d, out + t * H * d);
      free(kr); free(vr);
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Decomposed LLaMA block (P:183 pipeline contents; reading c9):              */
/*   a  = rmsnorm(x, g_attn)                                                  */
/*   q,k,v = A_q(B_q a), A_k(B_k a), A_v(B_v a)      (each Eq. 1)             */
/*   q,k <- rope(q,k, pos)                                                    */
/*   x  += A_o(B_o attention(q,k,v))                                          */
/*   b  = rmsnorm(x, g_mlp)                                                   */
/*   x  += A_down(B_down( silu(A_gate(B_gate b)) * A_up(B_up b) ))            */
/* Each factor pair may be sharded over `world` ranks (reduce-sum of partials,*/
/* Fig. 2(b) / P:123); world==1 is the plain definition.                      */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t h, n_heads, n_kv_heads, head_dim, m;
  int64_t r_q, r_k, r_v, r_o, r_gate, r_up, r_down;
  double rope_theta, rms_eps;
  /* Table 2 variants: mlp_glu 1 = SiLU(gate)*up (LLaMA), 0 = ReLU(up)
     (OPT family, "NonGLU uses ReLU"); use_rope 0 = no rotary embedding */
  int64_t mlp_glu, use_rope;
  /* layout of the rank sharding when world > 1:
     0 = rank-parallel (north star: every factor pair split along k, one
         reduce-sum per pair, Fig. 2(b));
     1 = DeInfer low-rank communication (Fig. 3): see
         deinfer_first / deinfer_second below.  Both equal world == 1.     */
  int64_t layout;
} oracle_block_cfg;

typedef struct {
  const double *g_attn, *g_mlp;             /* [h] */
  const double *A_q, *B_q, *A_k, *B_k, *A_v, *B_v, *A_o, *B_o;
  const double *A_gate, *B_gate, *A_up, *B_up, *A_down, *B_down;
} oracle_block_w;

static int lr(const double *X, const double *A, const double *B, double *Y,
              int64_t T, int64_t m, int64_t n, int64_t k, int world,
              int64_t align) {
  if (world <= 1) return oracle_lowrank_linear(X, A, B, Y, T, m, n, k);
  return oracle_lowrank_linear_sharded(X, A, B, Y, T, m, n, k, world, align);
}

static double silu(double g) { return g / (1.0 + exp(-g)); }

/* DeInfer first sub-layer, P:176 (Fig. 3): "all downward projection matrices
 * x_v in the first sub-layer are in column-wise parallel (in a split manner,
 * where all matrices are first concatenated and then evenly split), followed
 * by an all-gather operation in the low-rank latent space ... The upward
 * projection matrices x_u are also in column-parallel (but in a shard way,
 * where each process has a shard of the same matrices) ... a batched matrix
 * multiplication for the low-rank results with different upward matrix
 * shards".  Segment s: A[s] [m[s] x l[s]], B[s] [l[s] x n]; Y[s] [T x m[s]].
 *   1. B_cat = [B[0]; B[1]; ...]  (L = sum l rows), rank r holds the rows of
 *      its balanced share of [0, L) (reading c3);
 *   2. rank r: Z_r = X B_cat[rows_r]^T                     [T x len_r];
 *   3. all-gather: Z = [Z_0 | Z_1 | ...]                    [T x L];
 *   4. rank r, segment s: output rows rows_r(m[s]) (its balanced share of
 *      A[s]'s rows): Y[s][t][i] = sum_j A[s][i][j] Z[t][off_s + j].        */
static int deinfer_first(const double *X, int64_t T, int64_t n, int nseg,
                         const double *const *A, const double *const *B,
                         const int64_t *m, const int64_t *l, int world,
                         double *const *Y) {
  int64_t L = 0, off[3];
  for (int s = 0; s < nseg; ++s) { off[s] = L; L += l[s]; }
  double *Bc = (double *)malloc(sizeof(double) * (size_t)(L * n + 1));
  double *Z = (double *)malloc(sizeof(double) * (size_t)(T * L + 1));
  if (!Bc || !Z) { free(Bc); free(Z); return ORC_ENOMEM; }
  for (int s = 0; s < nseg; ++s)                                   /* step 1 */
    memcpy(Bc + off[s] * n, B[s], sizeof(double) * (size_t)(l[s] * n));
  for (int r = 0; r < world; ++r) {
    int64_t b0, len, lp;
    int rc = oracle_shard_range(L, world, r, 1, &b0, &len, &lp);
    if (rc) { free(Bc); free(Z); return rc; }
    double *Zr = (double *)malloc(sizeof(double) * (size_t)(T * len + 1));
    if (!Zr) { free(Bc); free(Z); return ORC_ENOMEM; }
    for (int64_t t = 0; t < T; ++t)                                /* step 2 */
      for (int64_t j = 0; j < len; ++j) {
        double acc = 0.0;
        for (int64_t c = 0; c < n; ++c) acc += Bc[(b0 + j) * n + c] * X[t * n + c];
        Zr[t * len + j] = acc;
      }
    for (int64_t t = 0; t < T; ++t)                                /* step 3 */
      for (int64_t j = 0; j < len; ++j) Z[t * L + b0 + j] = Zr[t * len + j];
    free(Zr);
  }
  for (int r = 0; r < world; ++r)                                  /* step 4 */
    for (int s = 0; s < nseg; ++s) {
      int64_t i0, ni, np_;
      int rc = oracle_shard_range(m[s], world, r, 1, &i0, &ni, &np_);
      if (rc) { free(Bc); free(Z); return rc; }
      for (int64_t t = 0; t < T; ++t)
        for (int64_t i = i0; i < i0 + ni; ++i) {
          double acc = 0.0;
          for (int64_t j = 0; j < l[s]; ++j) acc += A[s][i * l[s] + j] * Z[t * L + off[s] + j];
          Y[s][t * m[s] + i] = acc;
        }
    }
  free(Bc); free(Z);
  return ORC_OK;
}

/* DeInfer second sub-layer: "the downward projection matrix is in
 * row-wise parallel, and upward projection matrix is identical in each
 * process.  Therefore, after multiplying the downward matrix, each process
 * needs to have a reduce-sum ... Since every process has identical low-rank
 * data and identical upward matrix, the output would also be identical."
 * A [m x l], B [l x n]; rank r holds the columns cols_r (balanced share of
 * [0, n)) of B and sees only those features of X (its local heads / MLP
 * slice):  Z = sum_r X[:, cols_r] B[:, cols_r]^T  (reduce-sum, [T x l]);
 * Y = Z A^T on every rank.                                                 */
static int deinfer_second(const double *X, int64_t T, int64_t n,
                          const double *A, const double *B, int64_t m,
                          int64_t l, int world, double *Y) {
  double *Z = (double *)calloc((size_t)(T * l + 1), sizeof(double));
  if (!Z) return ORC_ENOMEM;
  for (int r = 0; r < world; ++r) {
    int64_t c0, nc, np_;
    int rc = oracle_shard_range(n, world, r, 1, &c0, &nc, &np_);
    if (rc) { free(Z); return rc; }
    for (int64_t t = 0; t < T; ++t)
      for (int64_t j = 0; j < l; ++j) {
        double acc = 0.0;                                  /* rank r's partial */
        for (int64_t c = c0; c < c0 + nc; ++c) acc += B[j * n + c] * X[t * n + c];
        Z[t * l + j] += acc;                               /* reduce-sum */
      }
  }
  for (int64_t t = 0; t < T; ++t)
    for (int64_t i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int64_t j = 0; j < l; ++j) acc += A[i * l + j] * Z[t * l + j];
      Y[t * m + i] = acc;
    }
  free(Z);
  return ORC_OK;
}

static int use_deinfer(const oracle_block_cfg *c, int world) { return world > 1 && c->layout == 1; }

/* q, k, v projections of the normed rows a [T x h] (q may be NULL). */
static int project_qkv(const oracle_block_cfg *c, const oracle_block_w *w,
                       const double *a, int64_t T, double *q, double *kk,
                       double *vv, int world, int64_t align) {
  int64_t h = c->h, hkv = c->n_kv_heads * c->head_dim;
  if (use_deinfer(c, world)) {
    const double *A[3] = {w->A_q, w->A_k, w->A_v}, *B[3] = {w->B_q, w->B_k, w->B_v};
    int64_t m[3] = {h, hkv, hkv}, l[3] = {c->r_q, c->r_k, c->r_v};
    double *qq = q ? q : (double *)malloc(sizeof(double) * (size_t)(T * h + 1));
    double *Y[3] = {qq, kk, vv};
    int rc = deinfer_first(a, T, h, 3, A, B, m, l, world, Y);
    if (!q) free(qq);
    return rc;
  }
  int rc = 0;
  if (q) rc |= lr(a, w->A_q, w->B_q, q, T, h, h, c->r_q, world, align);
  rc |= lr(a, w->A_k, w->B_k, kk, T, hkv, h, c->r_k, world, align);
  rc |= lr(a, w->A_v, w->B_v, vv, T, hkv, h, c->r_v, world, align);
  return rc;
}

/* MLP half + O projection are per-token; shared by prefill and decode. */
static int block_tail(const oracle_block_cfg *c, const oracle_block_w *w,
                      const double *x_in, const double *att, double *x_out,
                      int64_t T, int world, int64_t align) {
  int64_t h = c->h, m = c->m;
  double *o = (double *)malloc(sizeof(double) * (size_t)(T * h));
  double *xn = (double *)malloc(sizeof(double) * (size_t)(T * h));
  double *gt = (double *)malloc(sizeof(double) * (size_t)(T * m));
  double *up = (double *)malloc(sizeof(double) * (size_t)(T * m));
  double *dn = (double *)malloc(sizeof(double) * (size_t)(T * h));
  if (!o || !xn || !gt || !up || !dn) { free(o); free(xn); free(gt); free(up); free(dn); return ORC_ENOMEM; }
  const int di = use_deinfer(c, world);
  int rc = di ? deinfer_second(att, T, h, w->A_o, w->B_o, h, c->r_o, world, o)
              : lr(att, w->A_o, w->B_o, o, T, h, h, c->r_o, world, align);
  for (int64_t i = 0; i < T * h; ++i) x_out[i] = x_in[i] + o[i];
  oracle_rmsnorm(x_out, w->g_mlp, c->rms_eps, xn, T, h);
  if (di) {   /* gate | up concatenated and split (first sub-layer) */
    const double *A2[2] = {w->A_gate, w->A_up}, *B2[2] = {w->B_gate, w->B_up};
    int64_t m2[2] = {m, m}, l2[2] = {c->r_gate, c->r_up};
    double *Y2[2] = {gt, up};
    int g0 = c->mlp_glu ? 0 : 1;
    rc |= deinfer_first(xn, T, h, 2 - g0, A2 + g0, B2 + g0, m2 + g0, l2 + g0, world, Y2 + g0);
  } else {
    rc |= lr(xn, w->A_up, w->B_up, up, T, m, h, c->r_up, world, align);
    if (c->mlp_glu) rc |= lr(xn, w->A_gate, w->B_gate, gt, T, m, h, c->r_gate, world, align);
  }
  if (c->mlp_glu) {
    for (int64_t i = 0; i < T * m; ++i) gt[i] = silu(gt[i]) * up[i];
  } else {
    for (int64_t i = 0; i < T * m; ++i) gt[i] = up[i] > 0.0 ? up[i] : 0.0;   /* ReLU */
  }
  rc |= di ? deinfer_second(gt, T, m, w->A_down, w->B_down, h, c->r_down, world, dn)
           : lr(gt, w->A_down, w->B_down, dn, T, h, m, c->r_down, world, align);
  for (int64_t i = 0; i < T * h; ++i) x_out[i] += dn[i];
  free(o); free(xn); free(gt); free(up); free(dn);
  return rc;
}

/* Prefill over packed sequences.  x [T x h] in; outputs only the rows listed
 * in rows[0..n_rows) (all rows if rows == NULL; then n_rows must equal T)
 * into x_out [n_rows x h].  k_out, v_out (optional, [T x Hkv*d]) receive the
 * post-RoPE keys and the values of every token (what a cache stores).     */
int oracle_block_prefill(const oracle_block_cfg *c, const oracle_block_w *w,
                         const double *x, int64_t T, const int32_t *pos,
                         const int32_t *cu_seqlens, int32_t nseq,
                         const int64_t *rows, int64_t n_rows, double *x_out,
                         double *k_out, double *v_out, int world,
                         int64_t align) {
  int64_t h = c->h, H = c->n_heads, Hkv = c->n_kv_heads, d = c->head_dim;
  int64_t hkv = Hkv * d;
  if (H * d != h || H % Hkv != 0 || T < 0) return ORC_ESHAPE;
  if (!rows && n_rows != T) return ORC_ESHAPE;
  double *a = (double *)malloc(sizeof(double) * (size_t)(T * h + 1));
  double *kk = (double *)malloc(sizeof(double) * (size_t)(T * hkv + 1));
  double *vv = (double *)malloc(sizeof(double) * (size_t)(T * hkv + 1));
  double *xr = (double *)malloc(sizeof(double) * (size_t)(n_rows * h + 1));
  double *ar = (double *)malloc(sizeof(double) * (size_t)(n_rows * h + 1));
  double *qr = (double *)malloc(sizeof(double) * (size_t)(n_rows * h + 1));
  double *att = (double *)malloc(sizeof(double) * (size_t)(n_rows * h + 1));
  int32_t *pr = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n_rows + 1));
  if (!a || !kk || !vv || !xr || !ar || !qr || !att || !pr) return ORC_ENOMEM;
  int rc = 0;
  oracle_rmsnorm(x, w->g_attn, c->rms_eps, a, T, h);
  rc |= project_qkv(c, w, a, T, NULL, kk, vv, world, align);
  if (c->use_rope) oracle_rope(kk, pos, T, Hkv, d, c->rope_theta);
  for (int64_t r = 0; r < n_rows; ++r) {
    int64_t t = rows ? rows[r] : r;
    memcpy(xr + r * h, x + t * h, sizeof(double) * (size_t)h);
    memcpy(ar + r * h, a + t * h, sizeof(double) * (size_t)h);
    pr[r] = pos[t];
  }
  if (use_deinfer(c, world)) {   /* q rows from the same first sub-layer pass */
    double *kq = (double *)malloc(sizeof(double) * (size_t)(n_rows * hkv + 1));
    double *vq = (double *)malloc(sizeof(double) * (size_t)(n_rows * hkv + 1));
    rc |= project_qkv(c, w, ar, n_rows, qr, kq, vq, world, align);
    free(kq); free(vq);
  } else {
    rc |= lr(ar, w->A_q, w->B_q, qr, n_rows, h, h, c->r_q, world, align);
  }
  if (c->use_rope) oracle_rope(qr, pr, n_rows, H, d, c->rope_theta);
  /* causal attention of each requested row over its own sequence prefix */
  for (int64_t r = 0; r < n_rows; ++r) {
    int64_t t = rows ? rows[r] : r;
    int32_t s = 0;
    while (s < nseq && !(t >= cu_seqlens[s] && t < cu_seqlens[s + 1])) ++s;
    if (s == nseq) return ORC_ESHAPE;
    int64_t b0 = cu_seqlens[s], nk = t - b0 + 1;
    const double **kr = (const double **)malloc(sizeof(double *) * (size_t)nk);
    const double **vr = (const double **)malloc(sizeof(double *) * (size_t)nk);
    for (int64_t u = 0; u < nk; ++u) { kr[u] = kk + (b0 + u) * hkv; vr[u] = vv + (b0 + u) * hkv; }
    attend_one(qr + r * h, kr, vr, nk, H, Hkv, d, att + r * h);
    free(kr); free(vr);
  }
  rc |= block_tail(c, w, xr, att, x_out, n_rows, world, align);
  if (k_out) memcpy(k_out, kk, sizeof(double) * (size_t)(T * hkv));
  if (v_out) memcpy(v_out, vv, sizeof(double) * (size_t)(T * hkv));
  free(a); free(kk); free(vv); free(xr); free(ar); free(qr); free(att); free(pr);
  return rc;
}

/* Decode: one new token per sequence b (x [Bn x h]) at position cache_len[b].
 * cache_k/cache_v [Bn x max_seq x Hkv*d] hold post-RoPE keys / values of the
 * first cache_len[b] positions (cached decode == recompute).  The new
 * key/value are appended logically (k_new/v_new [Bn x Hkv*d] outputs).     */
int oracle_block_decode(const oracle_block_cfg *c, const oracle_block_w *w,
                        const double *x, int64_t Bn, const double *cache_k,
                        const double *cache_v, int64_t max_seq,
                        const int32_t *cache_len, double *x_out, double *k_new,
                        double *v_new, int world, int64_t align) {
  int64_t h = c->h, H = c->n_heads, Hkv = c->n_kv_heads, d = c->head_dim;
  int64_t hkv = Hkv * d;
  if (H * d != h || H % Hkv != 0 || Bn < 0) return ORC_ESHAPE;
  for (int64_t b = 0; b < Bn; ++b)
    if (cache_len[b] < 0 || cache_len[b] >= max_seq) return ORC_ESHAPE;
  double *a = (double *)malloc(sizeof(double) * (size_t)(Bn * h + 1));
  double *q = (double *)malloc(sizeof(double) * (size_t)(Bn * h + 1));
  double *kk = (double *)malloc(sizeof(double) * (size_t)(Bn * hkv + 1));
  double *vv = (double *)malloc(sizeof(double) * (size_t)(Bn * hkv + 1));
  double *att = (double *)malloc(sizeof(double) * (size_t)(Bn * h + 1));
  if (!a || !q || !kk || !vv || !att) return ORC_ENOMEM;
  int rc = 0;
  oracle_rmsnorm(x, w->g_attn, c->rms_eps, a, Bn, h);
  rc |= project_qkv(c, w, a, Bn, q, kk, vv, world, align);
  if (c->use_rope) {
    oracle_rope(q, cache_len, Bn, H, d, c->rope_theta);
    oracle_rope(kk, cache_len, Bn, Hkv, d, c->rope_theta);
  }
#pragma omp parallel for schedule(dynamic)
  for (int64_t b = 0; b < Bn; ++b) {
    int64_t nk = cache_len[b] + 1;
    const double **kr = (const double **)malloc(sizeof(double *) * (size_t)nk);
    const double **vr = (const double **)malloc(sizeof(double *) * (size_t)nk);
    for (int64_t u = 0; u < nk - 1; ++u) {
      kr[u] = cache_k + (b * max_seq + u) * hkv;
      vr[u] = cache_v + (b * max_seq + u) * hkv;
    }
    kr[nk - 1] = kk + b * hkv;
    vr[nk - 1] = vv + b * hkv;
    attend_one(q + b * h, kr, vr, nk, H, Hkv, d, att + b * h);
    free(kr); free(vr);
  }
  rc |= block_tail(c, w, x, att, x_out, Bn, world, align);
  if (k_new) memcpy(k_new, kk, sizeof(double) * (size_t)(Bn * hkv));
  if (v_new) memcpy(v_new, vv, sizeof(double) * (size_t)(Bn * hkv));
  free(a); free(q); free(kk); free(vv); free(att);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Low-rank KV cache (N3).  P:111: "the KV cache can be compressed as a       */
/* by-product of compressing K and V matrices in the attention layers, where  */
/* the low-rank intermediate results between the two matrix multiplications   */
/* now act as KV caches."  P:226-230 (two-stage reconstruction): the cached   */
/* low-rank rows are copied to a buffer, "the compact KV cache multiplies     */
/* upward matrices to finish the reconstruction", then "in-place rotary       */
/* position embedding" is applied to the reconstruction results.             */
/* Decode step of one block with such a cache: zk_cache [Bn x max_seq x r_k], */
/* zv_cache [Bn x max_seq x r_v] hold z_k = B_k a_j, z_v = B_v a_j of the     */
/* first cache_len[b] positions (a_j the normed input of token j).  History   */
/* keys K_j = RoPE(A_k z_k,j, j), values V_j = A_v z_v,j; the new token's     */
/* latents zk_new / zv_new are returned (what the cache appends).  world = 1  */
/* (the latent is replicated on every rank, SPEC kvcache design decision).   */
/* ------------------------------------------------------------------------ */
int oracle_block_decode_lowrank(const oracle_block_cfg *c, const oracle_block_w *w,
                                const double *x, int64_t Bn, const double *zk_cache,
                                const double *zv_cache, int64_t max_seq,
                                const int32_t *cache_len, double *x_out,
                                double *zk_new, double *zv_new) {
  int64_t h = c->h, H = c->n_heads, Hkv = c->n_kv_heads, d = c->head_dim;
  int64_t hkv = Hkv * d, lk = c->r_k, lv = c->r_v;
  if (H * d != h || H % Hkv != 0 || Bn < 0) return ORC_ESHAPE;
  for (int64_t b = 0; b < Bn; ++b)
    if (cache_len[b] < 0 || cache_len[b] >= max_seq) return ORC_ESHAPE;
  double *a = (double *)malloc(sizeof(double) * (size_t)(Bn * h + 1));
  double *q = (double *)malloc(sizeof(double) * (size_t)(Bn * h + 1));
  double *zk = (double *)malloc(sizeof(double) * (size_t)(Bn * lk + 1));
  double *zv = (double *)malloc(sizeof(double) * (size_t)(Bn * lv + 1));
  double *att = (double *)malloc(sizeof(double) * (size_t)(Bn * h + 1));
  if (!a || !q || !zk || !zv || !att) return ORC_ENOMEM;
  int rc = 0;
  oracle_rmsnorm(x, w->g_attn, c->rms_eps, a, Bn, h);
  rc |= oracle_lowrank_linear(a, w->A_q, w->B_q, q, Bn, h, h, c->r_q);
  rc |= oracle_matmul_bt(a, w->B_k, zk, Bn, h, lk);      /* z_k = B_k a (stage 1 only) */
  rc |= oracle_matmul_bt(a, w->B_v, zv, Bn, h, lv);
  if (c->use_rope) oracle_rope(q, cache_len, Bn, H, d, c->rope_theta);
#pragma omp parallel for schedule(dynamic)
  for (int64_t b = 0; b < Bn; ++b) {
    int64_t nk = cache_len[b] + 1;
    double *K = (double *)malloc(sizeof(double) * (size_t)(nk * hkv));
    double *V = (double *)malloc(sizeof(double) * (size_t)(nk * hkv));
    int32_t *pos = (int32_t *)malloc(sizeof(int32_t) * (size_t)nk);
    const double **kr = (const double **)malloc(sizeof(double *) * (size_t)nk);
    const double **vr = (const double **)malloc(sizeof(double *) * (size_t)nk);
    for (int64_t u = 0; u < nk; ++u) {
      /* compact low-rank row of token u (history from the cache, u == nk-1 the new one) */
      const double *zku = u < nk - 1 ? zk_cache + (b * max_seq + u) * lk : zk + b * lk;
      const double *zvu = u < nk - 1 ? zv_cache + (b * max_seq + u) * lv : zv + b * lv;
      for (int64_t i = 0; i < hkv; ++i) {      /* reconstruction: A_k z_k, A_v z_v */
        double sk = 0.0, sv = 0.0;
        for (int64_t j = 0; j < lk; ++j) sk += w->A_k[i * lk + j] * zku[j];
        for (int64_t j = 0; j < lv; ++j) sv += w->A_v[i * lv + j] * zvu[j];
        K[u * hkv + i] = sk;
        V[u * hkv + i] = sv;
      }
      pos[u] = (int32_t)u;
    }
    if (c->use_rope) oracle_rope(K, pos, nk, Hkv, d, c->rope_theta);   /* in place, after */
    for (int64_t u = 0; u < nk; ++u) { kr[u] = K + u * hkv; vr[u] = V + u * hkv; }
    attend_one(q + b * h, kr, vr, nk, H, Hkv, d, att + b * h);
    free(K); free(V); free(pos); free(kr); free(vr);
  }
  rc |= block_tail(c, w, x, att, x_out, Bn, 1, 1);
  if (zk_new) memcpy(zk_new, zk, sizeof(double) * (size_t)(Bn * lk));
  if (zv_new) memcpy(zv_new, zv, sizeof(double) * (size_t)(Bn * lv));
  free(a); free(q); free(zk); free(zv); free(att);
  return rc;
}

/* Preparation-stage scan: "performs a scan to find which logical block */
/* is physically contiguous".  phys[0..n) = a sequence's physical block ids in */
/* logical order; a new run starts exactly where phys[i] != phys[i-1] + 1.    */
/* Writes run starts / lengths (in blocks); returns the run count.           */
int64_t oracle_kv_runs(const int32_t *phys, int64_t n, int32_t *run_start,
                       int32_t *run_len) {
  int64_t r = -1;
  for (int64_t i = 0; i < n; ++i) {
    if (i == 0 || phys[i] != phys[i - 1] + 1) {
      ++r;
      run_start[r] = phys[i];
      run_len[r] = 0;
    }
    run_len[r] += 1;
  }
  return r + 1;
}

/* Parameter count of one decomposed block: sum over the 7 factor pairs of   */
/* (m_i + n_i) k_i  (P:109 applied per matrix; Table 1 footnote dims).  */
int64_t oracle_block_params(const oracle_block_cfg *c) {
  int64_t h = c->h, hkv = c->n_kv_heads * c->head_dim, m = c->m;
  return oracle_factor_params(h, h, c->r_q) + oracle_factor_params(hkv, h, c->r_k) +
         oracle_factor_params(hkv, h, c->r_v) + oracle_factor_params(h, h, c->r_o) +
         (c->mlp_glu ? oracle_factor_params(m, h, c->r_gate) : 0) + oracle_factor_params(m, h, c->r_up) +
         oracle_factor_params(h, m, c->r_down);
}

/* ------------------------------------------------------------------------ */
/* Communication census, P:185-216 (Section 4.1, Table 1).  Per token, per    */
/* block, in elements; all-gather costs n, reduce-sum costs 2n (Table 1 head).*/
/*  out[0]  unoptimized attention reduce-sum volume = 2(2h + 2h_kv)          */
/*  out[1]  unoptimized MLP reduce-sum volume       = 2(2m + h)              */
/*  out[2]  unoptimized block total                                          */
/*  out[3]  DeInfer attention all-gather  = l_q + l_k + l_v                  */
/*  out[4]  DeInfer MLP all-gather (printed row) = l_up + l_gate + l_down     */
/*  out[5]  DeInfer all-gather total                                         */
/*  out[6]  DeInfer block total, per-row sum (each row adds 2h)              */
/*  out[7]  DeInfer block total, printed aggregate (one 2h reduce-sum)       */
/*  out[8]  DeInfer block total, Section 4.1 text placement (2 l_o + 2 l_down,*/
/*          all-gather l_up + l_gate) -- reading c5                          */
/*  out[9]  this build's collectives (rank-sharded, reading c5/Section 8e):   */
/*          RS(h+2h_kv) + AG(h) + AR(h) + AR(2m) + AR(h), elements moved      */
/*          per token with AR counted 2n, RS/AG counted n (Table-1 units).    */
/*  out[10] number of collectives per layer in this build (5)                */
/*  out[11] number of reduce-sums per attention in Base (4)           */
/*  out[12] number of reduce-sums per GLU MLP in Base (3)                    */
/* ------------------------------------------------------------------------ */
void oracle_census(int64_t h, int64_t h_kv, int64_t m, int64_t l_q,
                   int64_t l_k, int64_t l_v, int64_t l_o, int64_t l_gate,
                   int64_t l_up, int64_t l_down, int64_t *out) {
  out[0] = 2 * (2 * h + 2 * h_kv);
  out[1] = 2 * (2 * m + h);
  out[2] = out[0] + out[1];
  out[3] = l_q + l_k + l_v;
  out[4] = l_up + l_gate + l_down;
  out[5] = out[3] + out[4];
  out[6] = out[3] + 2 * h + out[4] + 2 * h;
  out[7] = out[5] + 2 * h;
  out[8] = out[3] + 2 * l_o + (l_up + l_gate) + 2 * l_down;
  out[9] = (h + 2 * h_kv) + h + 2 * h + 2 * (2 * m) + 2 * h;
  out[10] = 5;
  /* Base: one reduce-sum per factor pair: q, k, v, o / gate, up, down */
  out[11] = 4;
  out[12] = 3;
}
