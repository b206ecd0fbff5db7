/*
 * oracle/tsne_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct fp64 CPU implementation of the Barnes-Hut
 * t-SNE method of t-SNE-CUDA (Chan, Rao, Huang, Canny; arXiv 1807.11824),
 * written from /root/reference/PAPER.md.  Citations "P:Lnnn" are PAPER.md
 * lines, "S:Lnnn" SPEC.md lines, "Dnn" the readings in DESIGN.md section 3.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the CUDA path (paper_1807_11824_b200/), and the CUDA
 * path never calls it.
 *
 * Every routine here follows the paper's definition or algorithm in the
 * order the paper states it; no blocking, fusion or reordering.  OpenMP is
 * used only to run independent per-point loops on several cores (each
 * point's arithmetic is sequential and identical for any thread count).
 *
 * Pins (tests/test_oracle_*.py) and the one "parity unpinned" part (the
 * long chaotic optimiser run, pinned only by invariants) are listed in
 * DESIGN.md section 5.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_ERR_ARG 1
#define ORACLE_ERR_MEM 2

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ======================================================================
 * O1  Exact k nearest neighbours ("the K nearest neighbors of each
 * point are obtained"; tie rule S:L110: lower index wins).
 * d_ij = sum_d (x_id - x_jd)^2 in fp64, j != i; keep the K smallest by the
 * key (d_ij, j), ascending.
 * ====================================================================== */
static int key_less(double da, int32_t ja, double db, int32_t jb) {
  return (da < db) || (da == db && ja < jb);
}

static void knn_one_row(const float* X, int64_t N, int32_t D, int32_t K,
                        int64_t i, int32_t* idx_row, double* d2_row) {
  int32_t have = 0;
  const float* xi = X + (size_t)i * D;
  for (int64_t j = 0; j < N; ++j) {
    if (j == i) continue;
    const float* xj = X + (size_t)j * D;
    double d = 0.0;
    for (int32_t k = 0; k < D; ++k) {
      double t = (double)xi[k] - (double)xj[k];
      d += t * t;
    }
    /* insertion into the ascending list of the best `have` so far */
    if (have == K && !key_less(d, (int32_t)j, d2_row[K - 1], idx_row[K - 1]))
      continue;
    int32_t pos = (have < K) ? have : K - 1;
    while (pos > 0 && key_less(d, (int32_t)j, d2_row[pos - 1], idx_row[pos - 1])) {
      d2_row[pos] = d2_row[pos - 1];
      idx_row[pos] = idx_row[pos - 1];
      --pos;
    }
    d2_row[pos] = d;
    idx_row[pos] = (int32_t)j;
    if (have < K) ++have;
  }
}

int oracle_knn(const float* X, int64_t N, int32_t D, int32_t K,
               int32_t* idx, double* d2) {
  if (N < 2 || D < 1 || K < 1 || K >= N) return ORACLE_ERR_ARG;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t i = 0; i < N; ++i)
    knn_one_row(X, N, D, K, i, idx + (size_t)i * K, d2 + (size_t)i * K);
  return ORACLE_OK;
}

/* kNN for a subset of query rows (rows[r]), against all N points. */
int oracle_knn_rows(const float* X, int64_t N, int32_t D, int32_t K,
                    const int64_t* rows, int64_t nrows, int32_t* idx, double* d2) {
  if (N < 2 || D < 1 || K < 1 || K >= N) return ORACLE_ERR_ARG;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t r = 0; r < nrows; ++r)
    knn_one_row(X, N, D, K, rows[r], idx + (size_t)r * K, d2 + (size_t)r * K);
  return ORACLE_OK;
}

/* Exact squared distance of two rows (fp64), used by tests for near-tie
 * excuses. */
double oracle_sqdist(const float* X, int32_t D, int64_t i, int64_t j) {
  double d = 0.0;
  for (int32_t k = 0; k < D; ++k) {
    double t = (double)X[(size_t)i * D + k] - (double)X[(size_t)j * D + k];
    d += t * t;
  }
  return d;
}

/* ======================================================================
 * O13  Approximate kNN by IVF-PQ (Alg. 1 line 1),
 * search given an index (the training is the GPU's; its deterministic
 * k-means is checked by properties, D27):
 *   q1(y) = c_{list(y)} (coarse centroid), q2 = product quantisation of the
 *   residual y - q1(y): sub-vector j (dims [j dsub, (j+1) dsub) of the
 *   zero-padded Dp = m dsub vector) is codeword cb[j][code_j(y)];
 *   q(y) = q1(y) + q2(y - q1(y))   (the paper's "q(y) = q1(y) + q2(y - q1(y))").
 * For query x_i: the centroids in order of ||x - c||^2 (fp64, ties by index);
 * the lists are scanned in that order until tau lists are done and at least
 * Kc candidates (points other than i) were seen, or Pmax lists; each candidate
 * y by the asymmetric distance ||x - q(y)||^2, written out directly in fp64
 * (the definition, not the look-up-table expansion); the Kc smallest by
 * (distance, index); then their exact distances ||x_i - x_j||^2 (fp64, the
 * original D dimensions) and the K smallest by (d2, index).  idx = -1 / d2 =
 * +inf where fewer than K candidates were found.
 * ====================================================================== */
int oracle_ivfpq_search(const float* X, int64_t N, int32_t D, int32_t Dp, int32_t nlist,
                        int32_t m, int32_t dsub, const float* cent, const float* cb,
                        const int32_t* list_of, const uint8_t* codes, int32_t K, int32_t tau,
                        int32_t Kc, int32_t Pmax, int32_t* idx, double* d2) {
  if (N < 2 || K < 1 || Kc < K || tau < 1 || tau > nlist || m * dsub != Dp || Dp < D)
    return ORACLE_ERR_ARG;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t i = 0; i < N; ++i) {
    double* cd = (double*)malloc(sizeof(double) * (size_t)nlist);
    int32_t* co = (int32_t*)malloc(sizeof(int32_t) * (size_t)nlist);
    int32_t* cj = (int32_t*)malloc(sizeof(int32_t) * (size_t)Kc);
    double* ca = (double*)malloc(sizeof(double) * (size_t)Kc);
    const float* x = X + (size_t)i * D;
    /* coarse distances and the probe order */
    for (int32_t c = 0; c < nlist; ++c) {
      double s = 0.0;
      for (int32_t e = 0; e < Dp; ++e) {
        double t = (e < D ? (double)x[e] : 0.0) - (double)cent[(size_t)c * Dp + e];
        s += t * t;
      }
      cd[c] = s;
      co[c] = c;
    }
    for (int32_t a = 1; a < nlist; ++a) {           /* insertion sort by (distance, index) */
      int32_t v = co[a];
      int32_t b = a;
      while (b > 0 && key_less(cd[v], v, cd[co[b - 1]], co[b - 1])) { co[b] = co[b - 1]; --b; }
      co[b] = v;
    }
    /* scan the lists; keep the Kc smallest asymmetric distances */
    int32_t have = 0;
    int64_t seen = 0;
    int32_t P = nlist < Pmax ? nlist : Pmax;
    for (int32_t p = 0; p < P; ++p) {
      if (p >= tau && seen >= Kc) break;
      int32_t L = co[p];
      for (int64_t y = 0; y < N; ++y) {
        if (list_of[y] != L || y == i) continue;
        ++seen;
        double s = 0.0;
        for (int32_t e = 0; e < Dp; ++e) {
          int32_t j = e / dsub;
          double q = (double)cent[(size_t)L * Dp + e] +
                     (double)cb[((size_t)j * 256 + codes[(size_t)y * m + j]) * dsub + (e - j * dsub)];
          double t = (e < D ? (double)x[e] : 0.0) - q;
          s += t * t;
        }
        if (have == Kc && !key_less(s, (int32_t)y, ca[Kc - 1], cj[Kc - 1])) continue;
        int32_t pos = have < Kc ? have : Kc - 1;
        while (pos > 0 && key_less(s, (int32_t)y, ca[pos - 1], cj[pos - 1])) {
          ca[pos] = ca[pos - 1]; cj[pos] = cj[pos - 1]; --pos;
        }
        ca[pos] = s; cj[pos] = (int32_t)y;
        if (have < Kc) ++have;
      }
    }
    /* exact distances of the candidates, the K smallest by (d2, index) */
    int32_t* oi = idx + (size_t)i * K;
    double* od = d2 + (size_t)i * K;
    int32_t got = 0;
    for (int32_t c = 0; c < have; ++c) {
      double s = oracle_sqdist(X, D, i, cj[c]);
      if (got == K && !key_less(s, cj[c], od[K - 1], oi[K - 1])) continue;
      int32_t pos = got < K ? got : K - 1;
      while (pos > 0 && key_less(s, cj[c], od[pos - 1], oi[pos - 1])) {
        od[pos] = od[pos - 1]; oi[pos] = oi[pos - 1]; --pos;
      }
      od[pos] = s; oi[pos] = cj[c];
      if (got < K) ++got;
    }
    for (int32_t c = got; c < K; ++c) { oi[c] = -1; od[c] = 1.0 / 0.0; }
    free(cd); free(co); free(cj); free(ca);
  }
  return ORACLE_OK;
}

/* ======================================================================
 * O2  Conditional affinities p_{j|i} (Eq. 1), restricted to the K
 * neighbours (D2), bandwidth chosen so that the Shannon entropy in nats
 * equals ln(perplexity) (D3; the paper never states the rule).
 *   d'_j = d_j - min_k d_k                       (min subtraction)
 *   S(b) = sum_j exp(-b d'_j),  p_j = exp(-b d'_j) / S
 *   H(b) = ln S + b sum_j p_j d'_j
 * Bisection with bracket doubling from b0 = 1/mean(d') until
 * |H - ln perp| <= 1e-10 max(1, ln perp), at most 200 steps.
 * Degenerate rows (flag 1): all d' = 0 -> uniform over K; m >= perp ties at
 * the minimum -> uniform over the m ties (b = +inf).
 * ====================================================================== */
static double row_entropy(const double* dp, int32_t K, double beta) {
  double S = 0.0, W = 0.0;
  for (int32_t j = 0; j < K; ++j) {
    double e = exp(-beta * dp[j]);
    S += e;
    W += dp[j] * e;
  }
  return log(S) + beta * W / S;
}

int oracle_calibrate_row(const double* d, int32_t K, double perplexity,
                         double* p, double* beta_out, int32_t* iters_out) {
  double* dp = (double*)malloc(sizeof(double) * (size_t)K);
  if (!dp) return -1;
  double dmin = d[0];
  for (int32_t j = 1; j < K; ++j) if (d[j] < dmin) dmin = d[j];
  double mean = 0.0;
  int32_t ties = 0;
  for (int32_t j = 0; j < K; ++j) {
    dp[j] = d[j] - dmin;
    mean += dp[j];
    if (dp[j] == 0.0) ++ties;
  }
  mean /= (double)K;
  int flag = 0;
  int32_t it = 0;
  double beta;
  if (mean == 0.0) {                      /* all neighbours equidistant */
    for (int32_t j = 0; j < K; ++j) p[j] = 1.0 / (double)K;
    beta = 0.0;
    flag = 1;
  } else if ((double)ties >= perplexity) { /* no finite root: H(inf) = ln ties */
    for (int32_t j = 0; j < K; ++j) p[j] = (dp[j] == 0.0) ? 1.0 / (double)ties : 0.0;
    beta = INFINITY;
    flag = 1;
  } else {
    const double target = log(perplexity);
    const double tol = 1e-10 * (target > 1.0 ? target : 1.0);
    double lo = 0.0, hi = INFINITY;
    beta = 1.0 / mean;
    for (it = 0; it < 200; ++it) {
      double H = row_entropy(dp, K, beta);
      if (fabs(H - target) <= tol) break;
      if (H > target) {            /* too flat: sharpen */
        lo = beta;
        beta = isinf(hi) ? 2.0 * beta : 0.5 * (lo + hi);
      } else {
        hi = beta;
        beta = 0.5 * (lo + hi);
      }
    }
    double S = 0.0;
    for (int32_t j = 0; j < K; ++j) S += exp(-beta * dp[j]);
    for (int32_t j = 0; j < K; ++j) p[j] = exp(-beta * dp[j]) / S;
  }
  free(dp);
  if (beta_out) *beta_out = beta;
  if (iters_out) *iters_out = it;
  return flag;
}

/* all rows; returns the number of degenerate rows (>= 0) */
int64_t oracle_calibrate(const double* d2, int64_t N, int32_t K, double perplexity,
                         double* P_cond, double* beta, int32_t* flags) {
  int64_t ndeg = 0;
#pragma omp parallel for schedule(static) reduction(+ : ndeg)
  for (int64_t i = 0; i < N; ++i) {
    double b;
    int f = oracle_calibrate_row(d2 + (size_t)i * K, K, perplexity,
                                 P_cond + (size_t)i * K, &b, NULL);
    if (beta) beta[i] = b;
    if (flags) flags[i] = f;
    ndeg += (f != 0);
  }
  return ndeg;
}

/* ======================================================================
 * O3  Symmetrisation p_ij = (p_{i|j} + p_{j|i}) / 2N on the union of
 * the kNN patterns, at most 2NK nonzeros.  Emit (i,j,p_{j|i}) and
 * (j,i,p_{j|i}) for every directed edge, sort by (row, col), sum
 * duplicates, divide by 2N; round to fp32 once.  CSR, both triangles,
 * sorted columns.
 * ====================================================================== */
typedef struct { int32_t r, c; double v; } trip_t;

static int trip_cmp(const void* a, const void* b) {
  const trip_t* x = (const trip_t*)a;
  const trip_t* y = (const trip_t*)b;
  if (x->r != y->r) return x->r < y->r ? -1 : 1;
  if (x->c != y->c) return x->c < y->c ? -1 : 1;
  return 0;
}

/* col/val64/val32 need capacity 2NK; returns nnz or -1 */
int64_t oracle_symmetrize(const int32_t* idx, const double* P_cond, int64_t N, int32_t K,
                          int64_t* row_ptr, int32_t* col, double* val64, float* val32) {
  size_t m = (size_t)N * K * 2;
  trip_t* t = (trip_t*)malloc(sizeof(trip_t) * m);
  if (!t) return -1;
  size_t e = 0;
  for (int64_t i = 0; i < N; ++i)
    for (int32_t k = 0; k < K; ++k) {
      int32_t j = idx[(size_t)i * K + k];
      double p = P_cond[(size_t)i * K + k];
      t[e].r = (int32_t)i; t[e].c = j; t[e].v = p; ++e;
      t[e].r = j; t[e].c = (int32_t)i; t[e].v = p; ++e;
    }
  qsort(t, m, sizeof(trip_t), trip_cmp);
  int64_t nnz = 0;
  for (int64_t r = 0; r <= N; ++r) row_ptr[r] = 0;
  size_t a = 0;
  while (a < m) {
    size_t b = a;
    double s = 0.0;
    while (b < m && t[b].r == t[a].r && t[b].c == t[a].c) { s += t[b].v; ++b; }
    double v = s / (2.0 * (double)N);
    col[nnz] = t[a].c;
    if (val64) val64[nnz] = v;
    if (val32) val32[nnz] = (float)v;
    row_ptr[t[a].r + 1] += 1;
    ++nnz;
    a = b;
  }
  for (int64_t r = 0; r < N; ++r) row_ptr[r + 1] += row_ptr[r];
  free(t);
  return nnz;
}

/* ======================================================================
 * O4-O6  Quadtree over the 2-D embedding and the theta traversal
 * (bounding box, insertion, counts, spatial order, forces).
 *
 * O4 root box (D8): exact min/max per axis; centre c = (min+max)/2;
 *    r0 = max(span_x, span_y)/2 * (1 + 2^-20), or 1 if both spans are 0;
 *    lo = c - r0; s = 2^L / (2 r0) with L = OTREE_LEVELS = 24.  All fp64.
 * O5 cells (D7-D9): q = min(2^L-1, max(0, floor((y - lo) s))) per axis.
 *    A cell at level l holds the points sharing q >> (L-l) on both axes;
 *    it is a leaf iff it holds exactly one point or l = L (D9: the paper
 *    inserts until every leaf holds one body; L = 24 stops only
 *    points closer than ~2^-23 r0, about one fp32 ulp of the coordinates).
 *    Summary: N_c, centre of mass = mean (fp64), radius r_l = r0 2^-l
 *    (half the side of the square cell).
 * O6 traversal for point i (D10, D11): DFS from the root, children in
 *    quadrant order (2*bx + by).  Leaf: exact pairs j != i.  Non-leaf cell
 *    containing i: open.  Otherwise D^2 = |y_i - com|^2 and, if
 *    r^2 < theta^2 D^2, accept: z_i += N w, f_i += N w^2 (y_i - com),
 *    w = 1/(1 + D^2)  (P:L132 cell formula, P:L134 simultaneous Z);
 *    else open.
 * ====================================================================== */
#define OTREE_LEVELS 24

typedef struct {
  int32_t level;
  int32_t leaf;
  int64_t count;
  double comx, comy;
  uint32_t px, py;        /* cell prefix: q >> (L - level) */
  int64_t child[4];       /* node ids, -1 if empty */
  int64_t first;          /* leaf: offset of its members in `members` */
} onode_t;

typedef struct {
  onode_t* nodes;
  int64_t nnodes, cap;
  int64_t* members;       /* point ids of leaves, concatenated */
  int64_t nmembers;
  uint32_t* qx;
  uint32_t* qy;
  double r0, cx, cy;
} otree_t;

static int64_t otree_new_node(otree_t* T) {
  if (T->nnodes == T->cap) {
    T->cap = T->cap ? T->cap * 2 : 1024;
    T->nodes = (onode_t*)realloc(T->nodes, sizeof(onode_t) * (size_t)T->cap);
  }
  return T->nnodes++;
}

/* build the cell at `level` holding list[0..n) (all share the level prefix) */
static int64_t otree_build_cell(otree_t* T, const double* Y, int64_t* list, int64_t n,
                                int32_t level, int64_t* scratch) {
  int64_t id = otree_new_node(T);
  onode_t* c = &T->nodes[id];
  c->level = level;
  c->count = n;
  double sx = 0.0, sy = 0.0;
  for (int64_t a = 0; a < n; ++a) { sx += Y[2 * list[a]]; sy += Y[2 * list[a] + 1]; }
  c->comx = sx / (double)n;
  c->comy = sy / (double)n;
  c->px = T->qx[list[0]] >> (OTREE_LEVELS - level);
  c->py = T->qy[list[0]] >> (OTREE_LEVELS - level);
  for (int k = 0; k < 4; ++k) c->child[k] = -1;
  if (n == 1 || level == OTREE_LEVELS) {
    c->leaf = 1;
    c->first = T->nmembers;
    for (int64_t a = 0; a < n; ++a) T->members[T->nmembers++] = list[a];
    return id;
  }
  c->leaf = 0;
  c->first = -1;
  /* stable partition of the list into the 4 quadrants of level+1 */
  int64_t cnt[4] = {0, 0, 0, 0};
  int shift = OTREE_LEVELS - 1 - level;
  for (int64_t a = 0; a < n; ++a) {
    int q = (int)(((T->qx[list[a]] >> shift) & 1u) * 2u + ((T->qy[list[a]] >> shift) & 1u));
    cnt[q]++;
  }
  int64_t off[4] = {0, cnt[0], cnt[0] + cnt[1], cnt[0] + cnt[1] + cnt[2]};
  int64_t pos[4] = {off[0], off[1], off[2], off[3]};
  for (int64_t a = 0; a < n; ++a) {
    int q = (int)(((T->qx[list[a]] >> shift) & 1u) * 2u + ((T->qy[list[a]] >> shift) & 1u));
    scratch[pos[q]++] = list[a];
  }
  memcpy(list, scratch, sizeof(int64_t) * (size_t)n);
  for (int q = 0; q < 4; ++q) {
    if (cnt[q] == 0) continue;
    int64_t ch = otree_build_cell(T, Y, list + off[q], cnt[q], level + 1, scratch);
    T->nodes[id].child[q] = ch;   /* re-index: nodes may have moved */
  }
  return id;
}

static void otree_free(otree_t* T) {
  free(T->nodes); free(T->members); free(T->qx); free(T->qy);
  memset(T, 0, sizeof(*T));
}

static int otree_build(otree_t* T, const double* Y, int64_t N) {
  memset(T, 0, sizeof(*T));
  double minx = Y[0], maxx = Y[0], miny = Y[1], maxy = Y[1];
  for (int64_t i = 1; i < N; ++i) {
    if (Y[2 * i] < minx) minx = Y[2 * i];
    if (Y[2 * i] > maxx) maxx = Y[2 * i];
    if (Y[2 * i + 1] < miny) miny = Y[2 * i + 1];
    if (Y[2 * i + 1] > maxy) maxy = Y[2 * i + 1];
  }
  double cx = (minx + maxx) / 2.0;
  double cy = (miny + maxy) / 2.0;
  double span = (maxx - minx) > (maxy - miny) ? (maxx - minx) : (maxy - miny);
  double r0 = (span == 0.0) ? 1.0 : (span / 2.0) * (1.0 + ldexp(1.0, -20));
  double lox = cx - r0, loy = cy - r0;
  double s = ldexp(1.0, OTREE_LEVELS) / (2.0 * r0);
  T->r0 = r0; T->cx = cx; T->cy = cy;
  T->qx = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)N);
  T->qy = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)N);
  T->members = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
  int64_t* list = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
  int64_t* scratch = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
  if (!T->qx || !T->qy || !T->members || !list || !scratch) {
    free(list); free(scratch); otree_free(T); return ORACLE_ERR_MEM;
  }
  for (int64_t i = 0; i < N; ++i) {
    double fx = floor((Y[2 * i] - lox) * s);
    double fy = floor((Y[2 * i + 1] - loy) * s);
    if (fx < 0.0) fx = 0.0;
    if (fy < 0.0) fy = 0.0;
    if (fx > ldexp(1.0, OTREE_LEVELS) - 1.0) fx = ldexp(1.0, OTREE_LEVELS) - 1.0;
    if (fy > ldexp(1.0, OTREE_LEVELS) - 1.0) fy = ldexp(1.0, OTREE_LEVELS) - 1.0;
    T->qx[i] = (uint32_t)fx;
    T->qy[i] = (uint32_t)fy;
    list[i] = i;
  }
  otree_build_cell(T, Y, list, N, 0, scratch);
  free(list); free(scratch);
  return ORACLE_OK;
}

static int otree_contains(const otree_t* T, const onode_t* c, int64_t i) {
  return (T->qx[i] >> (OTREE_LEVELS - c->level)) == c->px &&
         (T->qy[i] >> (OTREE_LEVELS - c->level)) == c->py;
}

typedef struct { double fx, fy, z; int64_t visits, interactions; } oacc_t;

static void otree_visit(const otree_t* T, const double* Y, int64_t i, double theta2,
                        int64_t node, oacc_t* acc) {
  const onode_t* c = &T->nodes[node];
  acc->visits++;
  double yx = Y[2 * i], yy = Y[2 * i + 1];
  if (c->leaf) {
    for (int64_t a = 0; a < c->count; ++a) {
      int64_t j = T->members[c->first + a];
      if (j == i) continue;
      double dx = yx - Y[2 * j], dy = yy - Y[2 * j + 1];
      double w = 1.0 / (1.0 + dx * dx + dy * dy);
      acc->z += w;
      acc->fx += w * w * dx;
      acc->fy += w * w * dy;
      acc->interactions++;
    }
    return;
  }
  if (!otree_contains(T, c, i)) {
    double dx = yx - c->comx, dy = yy - c->comy;
    double D2 = dx * dx + dy * dy;
    double r = ldexp(T->r0, -c->level);
    if (r * r < theta2 * D2) {
      double w = 1.0 / (1.0 + D2);
      double n = (double)c->count;
      acc->z += n * w;
      acc->fx += n * w * w * dx;
      acc->fy += n * w * w * dy;
      acc->interactions++;
      return;
    }
  }
  for (int q = 0; q < 4; ++q)
    if (c->child[q] >= 0) otree_visit(T, Y, i, theta2, c->child[q], acc);
}

/* Repulsive numerators f_i (N x 2), z_i (N) and Z = sum_i z_i (O7, P:L82,
 * L134), for all points (pts == NULL) or the listed ones (outputs then
 * indexed by list position; Z is only returned for the full set).
 * stats (nullable): [0] nodes, [1] visits, [2] interactions. */
int oracle_repulsive_bh(const float* Yf, int64_t N, double theta,
                        const int64_t* pts, int64_t npts,
                        double* f, double* z, double* Z_out, int64_t* stats) {
  if (N < 2 || theta < 0.0) return ORACLE_ERR_ARG;
  double* Y = (double*)malloc(sizeof(double) * 2 * (size_t)N);
  if (!Y) return ORACLE_ERR_MEM;
  for (int64_t a = 0; a < 2 * N; ++a) Y[a] = (double)Yf[a];
  otree_t T;
  if (otree_build(&T, Y, N) != ORACLE_OK) { free(Y); return ORACLE_ERR_MEM; }
  int64_t n = pts ? npts : N;
  double theta2 = theta * theta;
  int64_t visits = 0, inter = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : visits, inter)
  for (int64_t a = 0; a < n; ++a) {
    int64_t i = pts ? pts[a] : a;
    oacc_t acc = {0, 0, 0, 0, 0};
    otree_visit(&T, Y, i, theta2, 0, &acc);
    f[2 * a] = acc.fx;
    f[2 * a + 1] = acc.fy;
    z[a] = acc.z;
    visits += acc.visits;
    inter += acc.interactions;
  }
  if (Z_out && !pts) {
    double Z = 0.0;
    for (int64_t a = 0; a < N; ++a) Z += z[a];   /* sequential in i (O7) */
    *Z_out = Z;
  }
  if (stats) { stats[0] = T.nnodes; stats[1] = visits; stats[2] = inter; }
  otree_free(&T);
  free(Y);
  return ORACLE_OK;
}

/* Tree introspection for the tree pins: per node (pre-order of the DFS in
 * quadrant order) level, count, leaf, com.  Returns node count; arrays may
 * be NULL to query the count.  Also returns r0, cx, cy. */
int64_t oracle_tree_dump(const float* Yf, int64_t N, int32_t* level, int64_t* count,
                         int32_t* leaf, double* com, double* box) {
  double* Y = (double*)malloc(sizeof(double) * 2 * (size_t)N);
  for (int64_t a = 0; a < 2 * N; ++a) Y[a] = (double)Yf[a];
  otree_t T;
  if (otree_build(&T, Y, N) != ORACLE_OK) { free(Y); return -1; }
  /* nodes are created in DFS pre-order by otree_build_cell */
  for (int64_t k = 0; k < T.nnodes; ++k) {
    if (level) level[k] = T.nodes[k].level;
    if (count) count[k] = T.nodes[k].count;
    if (leaf) leaf[k] = T.nodes[k].leaf;
    if (com) { com[2 * k] = T.nodes[k].comx; com[2 * k + 1] = T.nodes[k].comy; }
  }
  if (box) { box[0] = T.r0; box[1] = T.cx; box[2] = T.cy; }
  int64_t n = T.nnodes;
  otree_free(&T);
  free(Y);
  return n;
}

/* ======================================================================
 * O8  Attractive term (Eq. 5, with q_ij Z = (1+d^2)^-1):
 *     A_i = sum_{j in row i} P_ij (y_i - y_j) / (1 + |y_i - y_j|^2)
 * (the nonzero iteration of P:L115-122; the "4N" of P:L117-120 is
 * ignored, D5).
 * ====================================================================== */
static void attractive_d(const int64_t* row_ptr, const int32_t* col, const float* val,
                         int64_t N, const double* Y, double* A) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    double ax = 0.0, ay = 0.0;
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      int32_t j = col[e];
      double dx = Y[2 * i] - Y[2 * (size_t)j], dy = Y[2 * i + 1] - Y[2 * (size_t)j + 1];
      double w = 1.0 / (1.0 + dx * dx + dy * dy);
      ax += (double)val[e] * w * dx;
      ay += (double)val[e] * w * dy;
    }
    A[2 * i] = ax;
    A[2 * i + 1] = ay;
  }
}

int oracle_attractive(const int64_t* row_ptr, const int32_t* col, const float* val,
                      int64_t N, const float* Yf, double* A) {
  double* Y = (double*)malloc(sizeof(double) * 2 * (size_t)N);
  if (!Y) return ORACLE_ERR_MEM;
  for (int64_t a = 0; a < 2 * N; ++a) Y[a] = (double)Yf[a];
  attractive_d(row_ptr, col, val, N, Y, A);
  free(Y);
  return ORACLE_OK;
}

/* ======================================================================
 * Gradient, Eq. 7: dC/dy_i = 4 (F_attr + F_rep),
 * F_rep,i = -f_i / Z (Eq. 6 with the cell formula of P:L132);
 * exaggeration a multiplies the attractive term (D13, D22).
 * ====================================================================== */
static int gradient_bh_d(const int64_t* row_ptr, const int32_t* col, const float* val,
                         int64_t N, const double* Y, double theta, double exag,
                         double* dY, double* Z_out) {
  otree_t T;
  if (otree_build(&T, Y, N) != ORACLE_OK) return ORACLE_ERR_MEM;
  double* f = (double*)malloc(sizeof(double) * 2 * (size_t)N);
  double* z = (double*)malloc(sizeof(double) * (size_t)N);
  double* A = (double*)malloc(sizeof(double) * 2 * (size_t)N);
  double theta2 = theta * theta;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < N; ++i) {
    oacc_t acc = {0, 0, 0, 0, 0};
    otree_visit(&T, Y, i, theta2, 0, &acc);
    f[2 * i] = acc.fx; f[2 * i + 1] = acc.fy; z[i] = acc.z;
  }
  double Z = 0.0;
  for (int64_t i = 0; i < N; ++i) Z += z[i];
  attractive_d(row_ptr, col, val, N, Y, A);
  for (int64_t i = 0; i < N; ++i) {
    dY[2 * i] = 4.0 * (exag * A[2 * i] - f[2 * i] / Z);
    dY[2 * i + 1] = 4.0 * (exag * A[2 * i + 1] - f[2 * i + 1] / Z);
  }
  if (Z_out) *Z_out = Z;
  free(f); free(z); free(A);
  otree_free(&T);
  return ORACLE_OK;
}

int oracle_gradient_bh(const int64_t* row_ptr, const int32_t* col, const float* val,
                       int64_t N, const float* Yf, double theta, double exag,
                       double* dY, double* Z_out) {
  if (N < 2 || theta < 0.0) return ORACLE_ERR_ARG;
  double* Y = (double*)malloc(sizeof(double) * 2 * (size_t)N);
  if (!Y) return ORACLE_ERR_MEM;
  for (int64_t a = 0; a < 2 * N; ++a) Y[a] = (double)Yf[a];
  int rc = gradient_bh_d(row_ptr, col, val, N, Y, theta, exag, dY, Z_out);
  free(Y);
  return rc;
}

/* O11  Exact gradient (Eq. 3 with the Z factor restored, D1; Eq. 4):
 *   g_i = 4 sum_{j != i} (a P_ij - w_ij / Z) w_ij (y_i - y_j),
 *   w = (1 + d^2)^-1, Z = sum_{k != l} w_kl.   P given in CSR (zeros
 * elsewhere).  Y in fp64. */
int oracle_gradient_exact_d(const int64_t* row_ptr, const int32_t* col, const double* val,
                            int64_t N, const double* Y, double exag,
                            double* dY, double* Z_out) {
  double Z = 0.0;
  for (int64_t k = 0; k < N; ++k)
    for (int64_t l = 0; l < N; ++l) {
      if (k == l) continue;
      double dx = Y[2 * k] - Y[2 * l], dy = Y[2 * k + 1] - Y[2 * l + 1];
      Z += 1.0 / (1.0 + dx * dx + dy * dy);
    }
  double* prow = (double*)calloc((size_t)N, sizeof(double));
  for (int64_t i = 0; i < N; ++i) {
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) prow[col[e]] = val[e];
    double gx = 0.0, gy = 0.0;
    for (int64_t j = 0; j < N; ++j) {
      if (j == i) continue;
      double dx = Y[2 * i] - Y[2 * j], dy = Y[2 * i + 1] - Y[2 * j + 1];
      double w = 1.0 / (1.0 + dx * dx + dy * dy);
      double coef = (exag * prow[j] - w / Z) * w;
      gx += coef * dx;
      gy += coef * dy;
    }
    dY[2 * i] = 4.0 * gx;
    dY[2 * i + 1] = 4.0 * gy;
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) prow[col[e]] = 0.0;
  }
  free(prow);
  if (Z_out) *Z_out = Z;
  return ORACLE_OK;
}

/* O12  KL(P||Q) = sum_{P_ij > 0} P_ij ln(P_ij / q_ij), q_ij = w_ij / Z with the
 * exact Z (Eq. 2).  fp64 P values. */
double oracle_kl_d(const int64_t* row_ptr, const int32_t* col, const double* val,
                   int64_t N, const double* Y) {
  double Z = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : Z)
  for (int64_t k = 0; k < N; ++k) {
    double zk = 0.0;
    for (int64_t l = 0; l < N; ++l) {
      if (k == l) continue;
      double dx = Y[2 * k] - Y[2 * l], dy = Y[2 * k + 1] - Y[2 * l + 1];
      zk += 1.0 / (1.0 + dx * dx + dy * dy);
    }
    Z += zk;
  }
  double kl = 0.0;
  for (int64_t i = 0; i < N; ++i)
    for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
      double p = val[e];
      if (!(p > 0.0)) continue;
      int32_t j = col[e];
      double dx = Y[2 * i] - Y[2 * (size_t)j], dy = Y[2 * i + 1] - Y[2 * (size_t)j + 1];
      double w = 1.0 / (1.0 + dx * dx + dy * dy);
      kl += p * log(p * Z / w);
    }
  return kl;
}

double oracle_kl(const int64_t* row_ptr, const int32_t* col, const float* val,
                 int64_t N, const double* Y) {
  int64_t nnz = row_ptr[N];
  double* v = (double*)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
  for (int64_t e = 0; e < nnz; ++e) v[e] = (double)val[e];
  double kl = oracle_kl_d(row_ptr, col, v, N, Y);
  free(v);
  return kl;
}

/* ======================================================================
 * D14  Y0 = 1e-4 N(0,1): Philox4x32-10 (key = seed, counter = (i,0,0,0)),
 * uniforms u = (x + 0.5) 2^-32 from the first two words, Box-Muller in fp64.
 * ====================================================================== */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void oracle_init_y(int64_t N, uint64_t seed, double* Y) {
  const double two_pi = 6.283185307179586476925286766559;
  for (int64_t i = 0; i < N; ++i) {
    uint32_t ctr[4] = {(uint32_t)i, (uint32_t)((uint64_t)i >> 32), 0u, 0u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    oracle_philox4x32_10(ctr, key, o);
    double u1 = ((double)o[0] + 0.5) * ldexp(1.0, -32);
    double u2 = ((double)o[1] + 0.5) * ldexp(1.0, -32);
    double r = sqrt(-2.0 * log(u1));
    Y[2 * i] = 1e-4 * r * cos(two_pi * u2);
    Y[2 * i + 1] = 1e-4 * r * sin(two_pi * u2);
  }
}

/* ======================================================================
 * O9-O10  Optimiser (Algorithm 1 loop; the update rule and
 * schedule are not in the paper: D12-D16).
 *   g = 4 (a(t) A - f/Z);  per coordinate:
 *   gain <- (sign g != sign v) ? gain + 0.2 : 0.8 gain;  gain >= min_gain
 *   v <- mu(t) v - eta gain g;  y <- y + v;  then y <- y - mean(y).
 *   a(t) = exag for t < exag_iters else 1; mu(t) = mom0 for t < exag_iters
 *   else mom1.
 * Y (N x 2, fp64) is updated in place; v and gains likewise.
 * ====================================================================== */
static double sgn(double x) { return (x > 0.0) - (x < 0.0); }

int oracle_optimize(const int64_t* row_ptr, const int32_t* col, const float* val, int64_t N,
                    double* Y, double* v, double* gains, int32_t t0, int32_t n_iter,
                    double theta, double eta, double exag, int32_t exag_iters,
                    double mom0, double mom1, double min_gain) {
  double* dY = (double*)malloc(sizeof(double) * 2 * (size_t)N);
  if (!dY) return ORACLE_ERR_MEM;
  for (int32_t t = t0; t < t0 + n_iter; ++t) {
    double a = (t < exag_iters) ? exag : 1.0;
    double mu = (t < exag_iters) ? mom0 : mom1;
    int rc = gradient_bh_d(row_ptr, col, val, N, Y, theta, a, dY, NULL);
    if (rc != ORACLE_OK) { free(dY); return rc; }
    double mx = 0.0, my = 0.0;
    for (int64_t k = 0; k < 2 * N; ++k) {
      double g = dY[k];
      double gn = (sgn(g) != sgn(v[k])) ? gains[k] + 0.2 : gains[k] * 0.8;
      if (gn < min_gain) gn = min_gain;
      gains[k] = gn;
      v[k] = mu * v[k] - eta * gn * g;
      Y[k] = Y[k] + v[k];
    }
    for (int64_t i = 0; i < N; ++i) { mx += Y[2 * i]; my += Y[2 * i + 1]; }
    mx /= (double)N; my /= (double)N;
    for (int64_t i = 0; i < N; ++i) { Y[2 * i] -= mx; Y[2 * i + 1] -= my; }
  }
  free(dY);
  return ORACLE_OK;
}

/* O12  k-NN preservation: mean_i |NN_k^X(i) & NN_k^Y(i)| / k, NN^X the
 * first k of the exact high-dimensional kNN rows (stride Kx), NN^Y a brute
 * force 2-D kNN with ties by index. */
/* |NN_k^X(i) & NN_k^Y(i)| / k for one point i (the summand of O12) */
static double nn_preserved_frac(const int32_t* idx_x, int32_t Kx, int64_t N, const double* Y,
                                int32_t k, int64_t i) {
  int32_t nb[64];
  double dd[64];
  int32_t have = 0;
  for (int64_t j = 0; j < N; ++j) {
    if (j == i) continue;
    double dx = Y[2 * i] - Y[2 * j], dy = Y[2 * i + 1] - Y[2 * j + 1];
    double d = dx * dx + dy * dy;
    if (have == k && !key_less(d, (int32_t)j, dd[k - 1], nb[k - 1])) continue;
    int32_t pos = (have < k) ? have : k - 1;
    while (pos > 0 && key_less(d, (int32_t)j, dd[pos - 1], nb[pos - 1])) {
      dd[pos] = dd[pos - 1]; nb[pos] = nb[pos - 1]; --pos;
    }
    dd[pos] = d; nb[pos] = (int32_t)j;
    if (have < k) ++have;
  }
  int32_t common = 0;
  for (int32_t a = 0; a < k; ++a)
    for (int32_t b = 0; b < k; ++b)
      if (idx_x[(size_t)i * Kx + a] == nb[b]) { ++common; break; }
  return (double)common / (double)k;
}

double oracle_nn_preservation(const int32_t* idx_x, int32_t Kx, int64_t N,
                              const double* Y, int32_t k) {
  double tot = 0.0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : tot)
  for (int64_t i = 0; i < N; ++i) tot += nn_preserved_frac(idx_x, Kx, N, Y, k, i);
  return tot / (double)N;
}

/* O12 on a sample of points: the same mean over the listed rows only (for
 * N where the O(N^2) all-points form is too slow, e.g. C5). */
double oracle_nn_preservation_rows(const int32_t* idx_x, int32_t Kx, int64_t N,
                                   const double* Y, int32_t k, const int64_t* rows,
                                   int64_t nrows) {
  double tot = 0.0;
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : tot)
  for (int64_t r = 0; r < nrows; ++r) tot += nn_preserved_frac(idx_x, Kx, N, Y, k, rows[r]);
  return tot / (double)nrows;
}

/* Full pipeline (Algorithm 1): O1 -> O2 -> O3 -> init -> loop.
 * K = min(N-1, floor(3 perp)) (D4).  Y_init (fp32, nullable) overrides the
 * Philox init.  Y_out fp64 N x 2.  kl_out (nullable): exact KL at the end
 * (non-exaggerated P).  knn_idx_out (nullable, N x K) returns the kNN. */
int oracle_run(const float* X, int64_t N, int32_t D, double perplexity, double theta,
               double eta, int32_t n_iter, double exag, int32_t exag_iters,
               double mom0, double mom1, double min_gain, uint64_t seed,
               const float* Y_init, double* Y_out, double* kl_out, int32_t* knn_idx_out) {
  int32_t K = (int32_t)floor(3.0 * perplexity);
  if (K > N - 1) K = (int32_t)(N - 1);
  if (N < 2 || K < 1 || !(perplexity > 1.0) || !(perplexity < K)) return ORACLE_ERR_ARG;
  int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)N * K);
  double* d2 = (double*)malloc(sizeof(double) * (size_t)N * K);
  double* pc = (double*)malloc(sizeof(double) * (size_t)N * K);
  int64_t* rp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N + 1));
  int32_t* cl = (int32_t*)malloc(sizeof(int32_t) * (size_t)N * K * 2);
  float* vl = (float*)malloc(sizeof(float) * (size_t)N * K * 2);
  double* v = (double*)calloc((size_t)N * 2, sizeof(double));
  double* gn = (double*)malloc(sizeof(double) * (size_t)N * 2);
  oracle_knn(X, N, D, K, idx, d2);
  oracle_calibrate(d2, N, K, perplexity, pc, NULL, NULL);
  oracle_symmetrize(idx, pc, N, K, rp, cl, NULL, vl);
  if (Y_init) for (int64_t a = 0; a < 2 * N; ++a) Y_out[a] = (double)Y_init[a];
  else oracle_init_y(N, seed, Y_out);
  for (int64_t a = 0; a < 2 * N; ++a) gn[a] = 1.0;
  int rc = oracle_optimize(rp, cl, vl, N, Y_out, v, gn, 0, n_iter, theta, eta, exag,
                           exag_iters, mom0, mom1, min_gain);
  if (kl_out) *kl_out = oracle_kl(rp, cl, vl, N, Y_out);
  if (knn_idx_out) memcpy(knn_idx_out, idx, sizeof(int32_t) * (size_t)N * K);
  free(idx); free(d2); free(pc); free(rp); free(cl); free(vl); free(v); free(gn);
  return rc;
}
