/*
 * svg2_oracle.c — plain, slow, fp64 CPU oracle for the SVG2 hot path (arXiv 2505.18875).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or constant
 * with the CUDA product path (paper_2505_18875_b200/csrc), and the product never calls it.
 *
 * Every function works on ONE (batch, head) problem, in double precision, on the exact bf16 input
 * values widened to double.  No blocking, no fusion, no reordering beyond what the paper states.
 * Citations are PAPER.md line numbers (Doc B = the paper proper) and the DESIGN.md readings R#.
 *
 *   oracle_kmeans            §4.1 Lloyd k-means on Q or K; §4.3 warm start
 *   oracle_kmeanspp_init     §4.3 k-means++ cold start (generator fixed by DESIGN R25)
 *   oracle_philox4x32_10     the counter-based generator of R25 (Salmon et al., SC'11)
 *   oracle_permute           §4.1 pi: cluster-contiguous stable ordering
 *   oracle_select_topp       §4.2 Eq.1, Eq.2, top-p
 *   oracle_attention_rows    §3.1 softmax(QK^T/sqrt d)V restricted to the selected
 *                            key clusters of the query's cluster (§4.3), renormalised
 *   oracle_dense_rows        §3.1 dense attention
 *
 * Parity pins (tests/test_oracle_*.py): closed forms, brute force on tiny inputs, numpy textbook
 * routines, invariants (argmin assignment, non-increasing objective), the permutation-equivalence
 * identity and top-p = 1 == dense.  k-means on realistic data beyond its
 * invariants is "parity unpinned" (the paper prints no worked example) — see DESIGN.md.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared (no fast-math: reductions stay sequential).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ k-means
 * X: [N, d] row-major.  C clusters.  iters Lloyd iterations, exactly (R3: no tolerance exit).
 * init: NULL => cold strided init c_j = x_{floor(j*N/C)} (R2); else warm start from init [C, d].
 * Each iteration (R4):
 *   assign : label_n = argmin_j sum_k (x_nk - c_jk)^2, direct difference, ties -> smallest j (R1, R5)
 *   update : size_j = #{n : label_n = j};  c_j = (sum_{n ascending, label_n = j} x_n) / size_j;
 *            an empty cluster keeps its previous centroid (R6)
 *   J_assign[t] = sum_n d(x_n, c_{label_n}) before the update, J_post[t] after it.
 * Outputs: labels [N] (last assign), centroids [C, d] (last update = exact means), sizes [C].
 * Returns 0, or -1 on invalid arguments (C < 1, C > N, iters < 1).
 */
static double sqdist(const double* x, const double* c, int d) {
  double acc = 0.0;
  for (int k = 0; k < d; ++k) {
    double diff = x[k] - c[k];
    acc = acc + diff * diff;
  }
  return acc;
}

int oracle_kmeans(const double* X, int64_t N, int d, int C, int iters, const double* init, int32_t* labels,
                  double* centroids, int64_t* sizes, double* J_assign, double* J_post) {
  if (C < 1 || (int64_t)C > N || iters < 1 || d < 1) return -1;
  if (init) {
    memcpy(centroids, init, sizeof(double) * (size_t)C * (size_t)d);
  } else {
    for (int j = 0; j < C; ++j) {
      int64_t src = ((int64_t)j * N) / C; /* floor(j*N/C) */
      memcpy(centroids + (size_t)j * d, X + (size_t)src * d, sizeof(double) * (size_t)d);
    }
  }
  double* sums = (double*)malloc(sizeof(double) * (size_t)C * (size_t)d);
  double* dmin = (double*)malloc(sizeof(double) * (size_t)N);
  for (int t = 0; t < iters; ++t) {
    /* assign */
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; ++n) {
      const double* x = X + (size_t)n * d;
      int best = 0;
      double bd = sqdist(x, centroids, d);
      for (int j = 1; j < C; ++j) {
        double dj = sqdist(x, centroids + (size_t)j * d, d);
        if (dj < bd) { /* strict: ties keep the smaller j */
          bd = dj;
          best = j;
        }
      }
      labels[n] = best;
      dmin[n] = bd;
    }
    double ja = 0.0;
    for (int64_t n = 0; n < N; ++n) ja += dmin[n];
    if (J_assign) J_assign[t] = ja;
    /* update: sequential sums in ascending token index */
    memset(sums, 0, sizeof(double) * (size_t)C * (size_t)d);
    for (int j = 0; j < C; ++j) sizes[j] = 0;
    for (int64_t n = 0; n < N; ++n) {
      int j = labels[n];
      sizes[j] += 1;
      double* s = sums + (size_t)j * d;
      const double* x = X + (size_t)n * d;
      for (int k = 0; k < d; ++k) s[k] = s[k] + x[k];
    }
    for (int j = 0; j < C; ++j) {
      if (sizes[j] == 0) continue; /* R6: empty cluster keeps its centroid */
      for (int k = 0; k < d; ++k) centroids[(size_t)j * d + k] = sums[(size_t)j * d + k] / (double)sizes[j];
    }
    if (J_post) {
      double jp = 0.0;
      for (int64_t n = 0; n < N; ++n) jp += sqdist(X + (size_t)n * d, centroids + (size_t)labels[n] * d, d);
      J_post[t] = jp;
    }
  }
  free(sums);
  free(dmin);
  return 0;
}

/* ------------------------------------------------------------------ k-means++ cold start
 * The paper initialises cold k-means with k-means++ (Arthur & Vassilvitskii 2007): the first centroid is a uniform
 * random point, each further centroid is point n with probability proportional to D(x_n), the squared distance to
 * the nearest centroid chosen so far.  The paper names no generator; DESIGN R25 fixes one so that the GPU and this
 * oracle pick the same points:
 *   - random numbers: Philox4x32-10 (Salmon et al., SC'11), key = (seed, stream), counter = (j, 0, 0, 0) for pick j;
 *     stream = 2 * (b * H + h) + role (role 0 = Q, 1 = K);
 *   - pick 0: n = floor(out0 * N / 2^32);
 *   - D(x_n) = sum_k (x_nk - c_k)^2 accumulated in ascending k, every operation rounded (sqdist above);
 *     after each pick D_n <- min(D_n, D(x_n, new centroid));
 *   - pick j >= 1: integer weights W_n = floor(D_n / D_ref * 2^32), D_ref = max_n D_n after pick 0 (D only
 *     decreases, so W_n <= 2^32 and the sum fits 64 bits); r = floor((out0 + 2^32 out1) * sum W / 2^64); the pick
 *     is the smallest n with W_0 + ... + W_n > r.  If every weight is 0, the pick is floor(out0 * N / 2^32).
 * Integer weights make the sampling exact and independent of summation order.  Returns 0, or -1 on bad args.
 */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n1 = (uint32_t)p1;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    const uint32_t n3 = (uint32_t)p0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

int oracle_kmeanspp_init(const double* X, int64_t N, int d, int C, uint32_t seed, uint32_t stream, int64_t* idx) {
  if (C < 1 || (int64_t)C > N || d < 1 || N > ((int64_t)1 << 31)) return -1;
  double* D = (double*)malloc(sizeof(double) * (size_t)N);
  uint64_t* W = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)N);
  const uint32_t key[2] = {seed, stream};
  double dref = 0.0;
  for (int j = 0; j < C; ++j) {
    const uint32_t ctr[4] = {(uint32_t)j, 0u, 0u, 0u};
    uint32_t out[4];
    oracle_philox4x32_10(ctr, key, out);
    int64_t pick;
    if (j == 0) {
      pick = (int64_t)(((uint64_t)out[0] * (uint64_t)N) >> 32);
    } else {
      uint64_t total = 0;
      for (int64_t n = 0; n < N; ++n) {
        W[n] = dref > 0.0 ? (uint64_t)floor(D[n] / dref * 4294967296.0) : 0u;
        total += W[n];
      }
      if (total == 0) {
        pick = (int64_t)(((uint64_t)out[0] * (uint64_t)N) >> 32);
      } else {
        const uint64_t r64 = (uint64_t)out[0] | ((uint64_t)out[1] << 32);
        const uint64_t r = (uint64_t)(((unsigned __int128)r64 * total) >> 64);
        uint64_t run = 0;
        pick = N - 1;
        for (int64_t n = 0; n < N; ++n) {
          run += W[n];
          if (run > r) {
            pick = n;
            break;
          }
        }
      }
    }
    idx[j] = pick;
    const double* c = X + (size_t)pick * d;
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; ++n) {
      const double dn = sqdist(X + (size_t)n * d, c, d);
      D[n] = (j == 0 || dn < D[n]) ? dn : D[n];
    }
    if (j == 0) {
      for (int64_t n = 0; n < N; ++n) dref = D[n] > dref ? D[n] : dref;
    }
  }
  free(D);
  free(W);
  return 0;
}

/* Assignment only (one Lloyd assign step against given centroids), with the exact distances of the
 * best and second-best centroid — used by parity tests to classify near-ties (R16). */
void oracle_assign(const double* X, int64_t N, int d, int C, const double* centroids, int32_t* labels,
                   double* d1, double* d2) {
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < N; ++n) {
    const double* x = X + (size_t)n * d;
    int best = -1;
    double b1 = INFINITY, b2 = INFINITY;
    for (int j = 0; j < C; ++j) {
      double dj = sqdist(x, centroids + (size_t)j * d, d);
      if (dj < b1) {
        b2 = b1;
        b1 = dj;
        best = j;
      } else if (dj < b2) {
        b2 = dj;
      }
    }
    labels[n] = best;
    if (d1) d1[n] = b1;
    if (d2) d2[n] = b2;
  }
}

/* ------------------------------------------------------------------ permutation
 * Stable counting sort by (label, original index) (R: SPEC.md:296).
 * perm[pos] = original index of the token at permuted position pos;  offsets[j] = start of cluster j,
 * offsets[C] = N.  Returns -1 if a label is out of range. */
int oracle_permute(const int32_t* labels, int64_t N, int C, int32_t* perm, int64_t* offsets) {
  if (C < 1) return -1;
  for (int j = 0; j <= C; ++j) offsets[j] = 0;
  for (int64_t n = 0; n < N; ++n) {
    if (labels[n] < 0 || labels[n] >= C) return -1;
    offsets[labels[n] + 1] += 1;
  }
  for (int j = 0; j < C; ++j) offsets[j + 1] += offsets[j];
  int64_t* cursor = (int64_t*)malloc(sizeof(int64_t) * (size_t)C);
  for (int j = 0; j < C; ++j) cursor[j] = offsets[j];
  for (int64_t n = 0; n < N; ++n) perm[cursor[labels[n]]++] = (int32_t)n;
  free(cursor);
  return 0;
}

/* ------------------------------------------------------------------ selection
 * cq [Cq, d], ck [Ck, d] centroids; sq [Cq], sk [Ck] cluster sizes.
 * Eq. 1: S_ij = scale * sum_k cq_ik ck_jk, accumulated as acc = fma(cq_ik, ck_jk, acc), k ascending (R8).
 * Eq. 2 (max-shifted, R9): m_i = max_{j: sk_j>0} S_ij; w_ij = sk_j exp(S_ij - m_i) (0 if sk_j = 0);
 *        Z_i = sum_j w_ij in ascending j;  P'_ij = w_ij / Z_i.
 * Top-p per query-cluster row (R10, R11): sort j by w_ij descending, ties by ascending j; walk the
 *        ranks, select rank r while (sum of selected w) < p * Z_i, skipping w = 0 entries; p == 1
 *        selects every non-empty key cluster exactly.
 * Outputs: mask [Cq, Ck] (1 = selected), *pairs = sum_i sq_i * sum_{j selected} sk_j (density numerator,
 * PAPER.md:353), optional S [Cq, Ck] and W [Cq, Ck] (= w_ij) and Z [Cq].
 * Returns -1 on p outside (0, 1]. */
typedef struct {
  double w;
  int j;
} wj_t;

static int cmp_wj(const void* a, const void* b) {
  const wj_t* x = (const wj_t*)a;
  const wj_t* y = (const wj_t*)b;
  if (x->w > y->w) return -1;
  if (x->w < y->w) return 1;
  return (x->j < y->j) ? -1 : (x->j > y->j);
}

int oracle_select_topp(const double* cq, const double* ck, const int64_t* sq, const int64_t* sk, int Cq,
                       int Ck, int d, double scale, double p, uint8_t* mask, int64_t* pairs, double* S_out,
                       double* W_out, double* Z_out) {
  if (!(p > 0.0 && p <= 1.0)) return -1;
  int64_t total = 0;
  wj_t* row = (wj_t*)malloc(sizeof(wj_t) * (size_t)Ck);
  double* S = (double*)malloc(sizeof(double) * (size_t)Ck);
  for (int i = 0; i < Cq; ++i) {
    double m = -INFINITY;
    for (int j = 0; j < Ck; ++j) {
      double acc = 0.0;
      for (int k = 0; k < d; ++k) acc = fma(cq[(size_t)i * d + k], ck[(size_t)j * d + k], acc);
      S[j] = scale * acc;
      if (sk[j] > 0 && S[j] > m) m = S[j];
    }
    double Z = 0.0;
    for (int j = 0; j < Ck; ++j) {
      double w = (sk[j] > 0) ? (double)sk[j] * exp(S[j] - m) : 0.0;
      row[j].w = w;
      row[j].j = j;
      Z = Z + w;
      if (S_out) S_out[(size_t)i * Ck + j] = S[j];
      if (W_out) W_out[(size_t)i * Ck + j] = w;
    }
    if (Z_out) Z_out[i] = Z;
    uint8_t* mrow = mask + (size_t)i * Ck;
    memset(mrow, 0, (size_t)Ck);
    int64_t keys = 0;
    if (p == 1.0) {
      for (int j = 0; j < Ck; ++j)
        if (sk[j] > 0) {
          mrow[j] = 1;
          keys += sk[j];
        }
    } else {
      qsort(row, (size_t)Ck, sizeof(wj_t), cmp_wj);
      const double target = p * Z;
      double cum = 0.0;
      for (int r = 0; r < Ck; ++r) {
        if (row[r].w == 0.0) break;
        if (!(cum < target)) break;
        mrow[row[r].j] = 1;
        keys += sk[row[r].j];
        cum = cum + row[r].w;
      }
    }
    total += sq[i] * keys;
  }
  free(row);
  free(S);
  if (pairs) *pairs = total;
  return 0;
}

/* ------------------------------------------------------------------ attention
 * For each requested query row n (original order): i = lq[n]; key set K(n) = {m : mask[i, lk[m]] = 1}.
 * s_m = scale * sum_k q_nk k_mk (k ascending);  M = max s_m;  e_m = exp(s_m - M);  l = sum e_m (m ascending);
 * o_n = (sum_m e_m v_m) / l;  lse_n = M + log(l).  Renormalised over K(n) (R12).  No permutation is used:
 * the GPU's permuted computation must agree through the identity of PAPER.md:276-281.
 * lq/lk/mask may be NULL for dense attention (every key).  Returns -1 if some row has an empty key set. */
int oracle_attention_rows(const double* Q, const double* K, const double* V, int64_t Nq, int64_t Nk, int d,
                          const int32_t* lq, const int32_t* lk, const uint8_t* mask, int Ck, double scale,
                          const int64_t* rows, int64_t nrows, double* O, double* lse) {
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(| : bad)
  for (int64_t r = 0; r < nrows; ++r) {
    const int64_t n = rows ? rows[r] : r;
    if (n < 0 || n >= Nq) {
      bad = 1;
      continue;
    }
    const double* q = Q + (size_t)n * d;
    const uint8_t* mrow = mask ? mask + (size_t)lq[n] * Ck : NULL;
    double* s = (double*)malloc(sizeof(double) * (size_t)Nk);
    double M = -INFINITY;
    int64_t cnt = 0;
    for (int64_t m = 0; m < Nk; ++m) {
      if (mrow && !mrow[lk[m]]) {
        s[m] = NAN;
        continue;
      }
      const double* kk = K + (size_t)m * d;
      double acc = 0.0;
      for (int k = 0; k < d; ++k) acc = acc + q[k] * kk[k];
      s[m] = scale * acc;
      if (s[m] > M) M = s[m];
      ++cnt;
    }
    double* o = O + (size_t)r * d;
    for (int k = 0; k < d; ++k) o[k] = 0.0;
    if (cnt == 0) {
      bad = 1;
      free(s);
      continue;
    }
    double l = 0.0;
    for (int64_t m = 0; m < Nk; ++m) {
      if (mrow && !mrow[lk[m]]) continue;
      double e = exp(s[m] - M);
      l = l + e;
      const double* vv = V + (size_t)m * d;
      for (int k = 0; k < d; ++k) o[k] = o[k] + e * vv[k];
    }
    for (int k = 0; k < d; ++k) o[k] = o[k] / l;
    if (lse) lse[r] = M + log(l);
    free(s);
  }
  return bad ? -1 : 0;
}
