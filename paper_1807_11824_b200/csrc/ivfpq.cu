// ivfpq.cu -- approximate kNN by an inverted file with product quantisation
// (SURVEY 8(f) f2): the paper's own line-1 algorithm (Alg. 1; Sec.
// III-B), FAISS's IVF-PQ:
//   * coarse quantiser q1: |C| = sqrt(N) centroids trained by k-means;
//   * residual quantiser q2: product quantisation of r = x - q1(x), m
//     sub-vectors of dsub dimensions, 256 codewords each (8-bit codes);
//   * search: the tau nearest centroids of a query x, then the K
//     nearest by the asymmetric distance ||x - q(y)||^2, q(y) = q1(y) + q2(y - q1(y)),
//     over the points y of those tau inverted lists, evaluated by look-up
//     tables: ||x - c_L - r^||^2 = ||x - c_L||^2 + sum_j (T_L[j][code_j] - 2 Q_x[j][code_j])
//     with T_L[j][k] = ||cb_jk||^2 + 2 <c_L,j, cb_jk> and Q_x[j][k] = <x_j, cb_jk>.
// This build then re-ranks the K' = K + 64 best candidates by their exact fp64
// distance (D19: P needs exact fp64 distances), so the output is the exact
// distances of approximately found neighbours.  Readings (D27):
// deterministic k-means (strided sample, strided initial centroids, fixed
// number of Lloyd iterations, empty clusters keep their centroid, means
// summed in point order in fp64), ties by index everywhere.
//
// GEMMs (distances to centroids, Q and T tables) are plain library GEMMs
// (cuBLAS SGEMM, fp32); everything else is in the kernels below.
#include <cublas_v2.h>

#include <cfloat>
#include <cmath>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace tsne {

constexpr int kKsub = 256;              // codewords per sub-quantiser (8-bit codes)
constexpr int kIvfThreads = 256;
constexpr int kIvfBlock = 16384;        // queries per search block (Q table: block x m x 256)
constexpr int kCoarseBlock = 32768;     // rows per coarse-distance GEMM block
constexpr int kMaxProbes = 64;          // probe order kept per query
constexpr int kCandCapQ = 1 << 16;      // candidate buffer per search CTA (entries)
constexpr int kMaxKc = 480;             // candidates re-ranked per query, at most

// K' candidates re-ranked: params.kprime, or K + max(64, 5K); rounded up to 32
static int ivf_kc(int K, const tsne_ivfpq_params* p) {
  int kc = (p && p->kprime > 0) ? p->kprime : K + (5 * K > 64 ? 5 * K : 64);
  if (kc < K) kc = K;
  kc = ((kc + 31) / 32) * 32;
  return kc < kMaxKc ? kc : kMaxKc;
}

struct IvfDims {
  int64_t N;
  int32_t D, Dp, nlist, m, dsub, ntrain, iters;
  uint64_t seed;
  tsne_ivfpq_params prm;
};

static IvfDims ivf_dims(int64_t N, int32_t D, const tsne_ivfpq_params* pin) {
  tsne_ivfpq_params p;
  tsne_ivfpq_params_default(&p);
  if (pin) p = *pin;
  IvfDims d;
  d.N = N;
  d.D = D;
  d.nlist = p.nlist > 0 ? p.nlist : (int32_t)std::lround(std::sqrt((double)N));
  if (d.nlist < 1) d.nlist = 1;
  d.m = p.m > 0 ? p.m : (D + 7) / 8 < 96 ? (D + 7) / 8 : 96;
  d.dsub = (D + d.m - 1) / d.m;
  d.Dp = d.m * d.dsub;
  const int64_t nt = (int64_t)d.nlist * (p.train_per_list > 0 ? p.train_per_list : 64);
  d.ntrain = (int32_t)(nt < N ? nt : N);
  d.iters = p.kmeans_iters > 0 ? p.kmeans_iters : 10;
  d.seed = p.seed;
  d.prm = p;
  return d;
}

// index layout (bytes from the index base; every part 256-aligned)
struct IvfIndex {
  float* cent;       // nlist x Dp
  float* cb;         // m x 256 x dsub
  uint8_t* codes;    // N x m, in list order
  int32_t* loff;     // nlist + 1
  int32_t* lids;     // N point of each list entry
  float* T;          // nlist x m x 256
  float* cnorm;      // nlist
};

static size_t carve_index(Carver& c, const IvfDims& d, IvfIndex& x) {
  x.cent = c.take<float>((size_t)d.nlist * d.Dp);
  x.cb = c.take<float>((size_t)d.m * kKsub * d.dsub);
  x.codes = c.take<uint8_t>((size_t)d.N * d.m);
  x.loff = c.take<int32_t>(d.nlist + 1);
  x.lids = c.take<int32_t>(d.N);
  x.T = c.take<float>((size_t)d.nlist * d.m * kKsub);
  x.cnorm = c.take<float>(d.nlist);
  return c.bytes();
}

// ---------------------------------------------------------------- workspace
struct IvfWS {
  float* Xp;          // N x Dp padded copy (only when Dp != D)
  float* xt;          // ntrain x Dp training sample (then its residuals)
  float* G;           // GEMM block: max(kCoarseBlock x nlist, ntrain x 256, kIvfBlock x m x 256)
  float* Xq;          // kIvfBlock x Dp query rows of a search block (list order)
  int32_t* assign;    // max(N, ntrain)
  int32_t* assign2;   // ntrain (sorted keys)
  int32_t* order;     // max(N, ntrain) (sort values)
  int32_t* order2;    // max(N, ntrain)
  int32_t* cnt;       // max(nlist, 256) + 1
  int32_t* off;       // max(nlist, 256) + 1
  double* sums;       // max(nlist, 256) x max(Dp, dsub)
  uint8_t* codes_pt;  // N x m codes by point
  float* norms;       // max(N, 256 m)
  int32_t* probes;    // kIvfBlock x kMaxProbes
  float* pbase;       // kIvfBlock x kMaxProbes
  uint64_t* cbuf;     // kNumSMs x kCandCapQ candidate keys
  uint64_t* cand;     // N x Kc
  void* sort_tmp;
  size_t sort_bytes;
  void* scan_tmp;
  size_t scan_bytes;
};

static size_t carve_ivf_ws(Carver& c, const IvfDims& d, int32_t Kc, IvfWS& w) {
  const int64_t nmax = d.N > d.ntrain ? d.N : d.ntrain;
  const int kmax = d.nlist > kKsub ? d.nlist : kKsub;
  w.Xp = c.take<float>(d.Dp != d.D ? (size_t)d.N * d.Dp : 0);
  w.xt = c.take<float>((size_t)d.ntrain * d.Dp);
  size_t g = (size_t)kCoarseBlock * d.nlist;
  g = std::max(g, (size_t)d.ntrain * kKsub);
  g = std::max(g, (size_t)kIvfBlock * d.m * kKsub);
  g = std::max(g, (size_t)d.ntrain * d.nlist);
  w.G = c.take<float>(g);
  w.Xq = c.take<float>((size_t)std::min<int64_t>(kIvfBlock, d.N) * d.Dp);
  w.assign = c.take<int32_t>(nmax);
  w.assign2 = c.take<int32_t>(nmax);
  w.order = c.take<int32_t>(nmax);
  w.order2 = c.take<int32_t>(nmax);
  w.cnt = c.take<int32_t>(kmax + 1);
  w.off = c.take<int32_t>(kmax + 1);
  w.sums = c.take<double>((size_t)kmax * (d.Dp > d.dsub ? d.Dp : d.dsub));
  w.codes_pt = c.take<uint8_t>((size_t)d.N * d.m);
  w.norms = c.take<float>(std::max((int64_t)d.N, (int64_t)kKsub * d.m));
  w.probes = c.take<int32_t>((size_t)kIvfBlock * kMaxProbes);
  w.pbase = c.take<float>((size_t)kIvfBlock * kMaxProbes);
  w.cbuf = c.take<uint64_t>((size_t)kNumSMs * kCandCapQ);
  w.cand = c.take<uint64_t>((size_t)d.N * (Kc > 0 ? Kc : 1));
  size_t sb = 0, cb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sb, (int32_t*)nullptr, (int32_t*)nullptr,
                                  (int32_t*)nullptr, (int32_t*)nullptr, (int)nmax);
  cub::DeviceScan::ExclusiveSum(nullptr, cb, (int32_t*)nullptr, (int32_t*)nullptr, kmax + 1);
  w.sort_tmp = c.take<char>(sb);
  w.sort_bytes = sb;
  w.scan_tmp = c.take<char>(cb);
  w.scan_bytes = cb;
  return c.bytes();
}

// ---------------------------------------------------------------- kernels
__global__ void k_pad_rows(const float* __restrict__ X, int64_t N, int D, int Dp,
                           float* __restrict__ Xp) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= N * Dp) return;
  const int64_t i = t / Dp;
  const int c = (int)(t - i * Dp);
  Xp[t] = c < D ? X[i * D + c] : 0.f;
}

// training sample: point floor(k N / ntrain) for k < ntrain
__global__ void k_take_sample(const float* __restrict__ X, int64_t N, int Dp, int ntrain,
                              float* __restrict__ xt) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)ntrain * Dp) return;
  const int64_t k = t / Dp;
  const int c = (int)(t - k * Dp);
  const int64_t i = k * N / ntrain;
  xt[t] = X[i * Dp + c];
}

// initial centroids: sample rows floor(c n / k)
__global__ void k_init_cent(const float* __restrict__ pts, int n, int dim, int ld, int k,
                            float* __restrict__ cent, int ldc) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)k * dim) return;
  const int c = (int)(t / dim), e = (int)(t - (int64_t)c * dim);
  const int64_t r = (int64_t)c * n / k;
  cent[(size_t)c * ldc + e] = pts[(size_t)r * ld + e];
}

// squared norms of k rows of dim entries (stride ld)
__global__ void k_row_norms(const float* __restrict__ a, int64_t k, int dim, int64_t ld,
                            float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (r >= k) return;
  float s = 0.f;
  for (int e = lane; e < dim; e += 32) {
    const float v = a[r * ld + e];
    s = fmaf(v, v, s);
  }
  s = warp_sum(s);
  if (lane == 0) out[r] = s;
}

// argmin_c (|c|^2 - 2 g[i][c]) per row (ties: lowest index); g row-major n x k
__global__ void k_argmin_rows(const float* __restrict__ g, int64_t n, int k,
                              const float* __restrict__ cn, int32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (r >= n) return;
  float best = FLT_MAX;
  int bi = 0x7fffffff;
  for (int c = lane; c < k; c += 32) {
    const float v = cn[c] - 2.f * g[r * k + c];
    if (v < best || (v == best && c < bi)) { best = v; bi = c; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov < best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  if (lane == 0) out[r] = bi;
}

__global__ void k_iota_i(int32_t* p, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = (int32_t)i;
}

__global__ void k_count(const int32_t* __restrict__ a, int64_t n, int32_t* __restrict__ cnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(cnt + a[i], 1);
}

// new centroid c = mean of its members, summed in point order in fp64 (the
// members of c are order[off[c] .. off[c+1]), sorted by (assignment, index));
// an empty cluster keeps its centroid
__global__ void k_centroid_means(const float* __restrict__ pts, int dim, int ld,
                                 const int32_t* __restrict__ order,
                                 const int32_t* __restrict__ off, int k,
                                 float* __restrict__ cent, int ldc) {
  const int c = blockIdx.x;
  const int a = off[c], b = off[c + 1];
  if (b <= a) return;
  for (int e = threadIdx.x; e < dim; e += blockDim.x) {
    double s = 0.0;
    for (int q = a; q < b; ++q) s += (double)pts[(size_t)order[q] * ld + e];
    cent[(size_t)c * ldc + e] = (float)(s / (double)(b - a));
  }
}

// residuals r = x - c_assign (in place on the training sample)
__global__ void k_residuals(float* __restrict__ xt, int n, int Dp, const float* __restrict__ cent,
                            const int32_t* __restrict__ assign) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * Dp) return;
  const int64_t i = t / Dp;
  const int e = (int)(t - i * Dp);
  xt[t] -= cent[(size_t)assign[i] * Dp + e];
}

// PQ codes of points [r0, r0 + n): code_j = argmin_k |r_j - cb_jk|^2 with
// r = x - c_list (one thread per point and sub-quantiser j; codebook j in
// shared memory); ties by index
__global__ void k_encode(const float* __restrict__ X, int64_t r0, int n, int Dp, int m, int dsub,
                         const float* __restrict__ cent, const int32_t* __restrict__ assign,
                         const float* __restrict__ cb, uint8_t* __restrict__ codes) {
  extern __shared__ float s_cb[];                  // 256 x dsub
  const int j = blockIdx.y;
  for (int t = threadIdx.x; t < kKsub * dsub; t += blockDim.x)
    s_cb[t] = cb[(size_t)j * kKsub * dsub + t];
  __syncthreads();
  const int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (li >= n) return;
  const int64_t i = r0 + li;
  const float* x = X + i * Dp + (size_t)j * dsub;
  const float* c = cent + (size_t)assign[i] * Dp + (size_t)j * dsub;
  float r[64];
#pragma unroll 4
  for (int e = 0; e < dsub; ++e) r[e] = x[e] - c[e];
  float best = FLT_MAX;
  int bk = 0;
  for (int k = 0; k < kKsub; ++k) {
    float d = 0.f;
    for (int e = 0; e < dsub; ++e) {
      const float t = r[e] - s_cb[k * dsub + e];
      d = fmaf(t, t, d);
    }
    if (d < best) { best = d; bk = k; }
  }
  codes[i * m + j] = (uint8_t)bk;
}

// codes of the list entries: codes_list[e] = codes_pt[lids[e]]
__global__ void k_gather_codes(const uint8_t* __restrict__ src, const int32_t* __restrict__ lids,
                               int64_t N, int m, uint8_t* __restrict__ dst) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= N * m) return;
  const int64_t e = t / m;
  const int j = (int)(t - e * m);
  dst[t] = src[(size_t)lids[e] * m + j];
}

// T[L][j][k] = |cb_jk|^2 + 2 <c_L,j, cb_jk>: the GEMM wrote <c_L,j, cb_jk> to T
__global__ void k_finish_T(float* __restrict__ T, int64_t nlist, int m,
                           const float* __restrict__ cbn) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nlist * m * kKsub) return;
  const int jk = (int)(t % ((int64_t)m * kKsub));
  T[t] = cbn[jk] + 2.f * T[t];
}

// Probe order of each query of a block: the kMaxProbes (or nlist) nearest
// centroids by |c|^2 - 2 x.c (ties by index), and ||x - c||^2 for each.
// One warp per query: repeated warp argmin over a per-lane candidate pool.
__global__ void k_probes(const float* __restrict__ g, int nb, int nlist, int P,
                         const float* __restrict__ cn, const float* __restrict__ xn,
                         const int32_t* __restrict__ qid,
                         int32_t* __restrict__ probes, float* __restrict__ pbase) {
  const int lane = threadIdx.x & 31;
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= nb) return;
  const float* gr = g + (size_t)r * nlist;
  float last = -FLT_MAX;
  int lasti = -1;
  for (int p = 0; p < P; ++p) {
    // the smallest (value, index) strictly after (last, lasti)
    float best = FLT_MAX;
    int bi = 0x7fffffff;
    for (int c = lane; c < nlist; c += 32) {
      const float v = cn[c] - 2.f * gr[c];
      const bool after = v > last || (v == last && c > lasti);
      if (after && (v < best || (v == best && c < bi))) { best = v; bi = c; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov < best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    last = best;
    lasti = bi;
    if (lane == 0) {
      probes[(size_t)r * kMaxProbes + p] = bi;
      pbase[(size_t)r * kMaxProbes + p] = xn[qid[r]] + best;
    }
  }
}

// query rows of a search block, taken in inverted-list order (queries of one
// list are neighbours: their candidates, probes and re-rank rows are shared
// in L2); norms of the rows
__global__ void k_gather_queries(const float* __restrict__ Xp, int Dp,
                                 const int32_t* __restrict__ qid, int nb,
                                 float* __restrict__ Xq) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)nb * Dp) return;
  const int64_t r = t / Dp;
  const int e = (int)(t - r * Dp);
  Xq[t] = Xp[(int64_t)qid[r] * Dp + e];
}

__device__ __forceinline__ uint64_t cand_key(float d, int32_t id) {
  uint32_t u = __float_as_uint(d);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);    // order-preserving
  return ((uint64_t)u << 32) | (uint32_t)id;
}

// The K' smallest keys of buf[0, n) (n >= K'), by an MSD radix select over the
// 64-bit keys (8-bit digits, shared histogram), written to out (any order).
__device__ void cta_select(const uint64_t* buf, int n, int Kc, uint64_t* out, int* s_hist,
                           int* s_misc) {
  uint64_t prefix = 0, pmask = 0;
  int need = Kc;                                   // still to take from the prefix bucket
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int t = threadIdx.x; t < 256; t += blockDim.x) s_hist[t] = 0;
    __syncthreads();
    // warp-aggregated increments: most keys share their leading digits, so
    // per-key shared atomics would serialise on a few bins
    for (int e0 = 0; e0 < n; e0 += blockDim.x) {
      const int e = e0 + threadIdx.x;
      uint64_t k = 0;
      const bool in = e < n && (((k = buf[e]) & pmask) == prefix);
      const int dg = in ? (int)((k >> shift) & 255) : -1;
      const unsigned grp = __match_any_sync(0xffffffffu, dg);
      if (in && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&s_hist[dg], __popc(grp));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0, d = 0;
      while (d < 256 && acc + s_hist[d] < need) { acc += s_hist[d]; ++d; }
      s_misc[0] = d;
      s_misc[1] = acc;
    }
    __syncthreads();
    const int d = s_misc[0];
    need -= s_misc[1];
    prefix |= (uint64_t)d << shift;
    pmask |= (uint64_t)255 << shift;
    __syncthreads();
  }
  // keys < prefix are all taken; prefix itself (unique keys) completes K'
  if (threadIdx.x == 0) s_misc[2] = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    const uint64_t k = buf[e];
    if (k <= prefix) out[atomicAdd(&s_misc[2], 1)] = k;
  }
  __syncthreads();
}

// Search: one CTA per query (persistent); the look-up table of each probed
// list in shared memory; every candidate's key (ADC distance, id) into this
// CTA's buffer; then the K' smallest.  Lists are probed in distance order
// until tau lists are done and at least K' candidates were seen (SPEC: more
// lists when fewer than K were found).
__global__ void __launch_bounds__(kIvfThreads)
k_ivf_scan(const int32_t* __restrict__ qid, int nb, int m, int P, int tau, int Kc,
           const float* __restrict__ Q,
           const float* __restrict__ T, const uint8_t* __restrict__ codes,
           const int32_t* __restrict__ loff, const int32_t* __restrict__ lids,
           const int32_t* __restrict__ probes, const float* __restrict__ pbase,
           uint64_t* __restrict__ cbuf, uint64_t* __restrict__ cand) {
  extern __shared__ float s_lut[];                 // m x 256
  __shared__ int s_hist[256];
  __shared__ int s_misc[4];
  uint64_t* buf = cbuf + (size_t)blockIdx.x * kCandCapQ;
  for (int r = blockIdx.x; r < nb; r += gridDim.x) {
    const int64_t qi = qid[r];
    const float* Qr = Q + (size_t)r * m * kKsub;
    if (threadIdx.x == 0) s_misc[3] = 0;
    __syncthreads();
    int p = 0;
    for (; p < P; ++p) {
      const int nseen = s_misc[3];
      if (p >= tau && nseen >= Kc) break;
      const int L = probes[(size_t)r * kMaxProbes + p];
      const float base = pbase[(size_t)r * kMaxProbes + p];
      for (int t = threadIdx.x; t < m * kKsub; t += blockDim.x)
        s_lut[t] = T[(size_t)L * m * kKsub + t] - 2.f * Qr[t];
      __syncthreads();
      const int a = loff[L], b = loff[L + 1];
      for (int e = a + threadIdx.x; e < b; e += blockDim.x) {
        const int id = lids[e];
        if (id == qi) continue;
        const uint8_t* cd = codes + (size_t)e * m;
        float d = base;
        if ((m & 15) == 0) {                     // 16 codes per vector load
          const uint4* c4 = reinterpret_cast<const uint4*>(cd);
          for (int q = 0; q < (m >> 4); ++q) {
            const uint4 v = __ldg(c4 + q);
            const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
            const float* lt = s_lut + q * 16 * kKsub;
#pragma unroll
            for (int u = 0; u < 16; ++u)
              d += lt[u * kKsub + ((w4[u >> 2] >> (8 * (u & 3))) & 255u)];
          }
        } else {
          for (int j = 0; j < m; ++j) d += s_lut[j * kKsub + cd[j]];
        }
        const int pos = atomicAdd(&s_misc[3], 1);
        if (pos < kCandCapQ) buf[pos] = cand_key(d, id);
      }
      __syncthreads();
    }
    int n = s_misc[3];
    n = n < kCandCapQ ? n : kCandCapQ;
    uint64_t* out = cand + (size_t)r * Kc;
    if (n <= Kc) {
      for (int e = threadIdx.x; e < Kc; e += blockDim.x)
        out[e] = e < n ? buf[e] : ~0ull;           // absent: the maximum key
      __syncthreads();
    } else {
      __threadfence_block();
      cta_select(buf, n, Kc, out, s_hist, s_misc);
    }
  }
}

// Exact fp64 distances of the K' candidates of each query; the K smallest by
// (d2, index) (warp per query; D18, D19)
__global__ void __launch_bounds__(256)
k_ivf_rerank(const float* __restrict__ X, const int32_t* __restrict__ qid, int nb, int D, int K,
             int Kc,
             const uint64_t* __restrict__ cand, int32_t* __restrict__ idx,
             double* __restrict__ d2) {
  __shared__ double s_d[8][512];
  __shared__ int s_j[8][512];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int r = blockIdx.x * 8 + wid;
  if (r >= nb) return;
  const int64_t i = qid[r];
  double* sd = s_d[wid];
  int* sj = s_j[wid];
  const float* xi = X + i * D;
  for (int c = 0; c < Kc; ++c) {
    const uint64_t key = cand[(size_t)r * Kc + c];
    const bool valid = key != ~0ull;
    const int j = valid ? (int)(uint32_t)key : 0x7fffffff;
    double acc = 0.0;
    if (valid) {
      const float* xj = X + (int64_t)j * D;
      for (int e = lane; e < D; e += 32) {
        const double t = (double)xi[e] - (double)xj[e];
        acc = fma(t, t, acc);
      }
      acc = warp_sum(acc);
    }
    if (lane == 0) {
      sd[c] = valid ? acc : DBL_MAX;
      sj[c] = j;
    }
  }
  int Pw = 32;
  while (Pw < Kc) Pw <<= 1;
  for (int c = Kc + lane; c < Pw; c += 32) { sd[c] = DBL_MAX; sj[c] = 0x7fffffff; }
  __syncwarp();
  for (int k = 2; k <= Pw; k <<= 1)
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int a = lane; a < Pw; a += 32) {
        const int l = a ^ jj;
        if (l > a) {
          const bool up = ((a & k) == 0);
          const double x = sd[a], y = sd[l];
          const int xa = sj[a], ya = sj[l];
          const bool gt = (x > y) || (x == y && xa > ya);
          if (gt == up) { sd[a] = y; sd[l] = x; sj[a] = ya; sj[l] = xa; }
        }
      }
      __syncwarp();
    }
  for (int c = lane; c < K; c += 32) {
    idx[i * K + c] = sj[c] == 0x7fffffff ? -1 : sj[c];
    d2[i * K + c] = sd[c];
  }
}

// ---------------------------------------------------------------- host
struct Blas {
  cublasHandle_t h = nullptr;
  ~Blas() { if (h) cublasDestroy(h); }
};

#define TSNE_BLAS_TRY(expr)                                                   \
  do {                                                                        \
    cublasStatus_t b__ = (expr);                                              \
    if (b__ != CUBLAS_STATUS_SUCCESS) {                                       \
      ::tsne::set_error("%s:%d %s -> cublas status %d", __FILE__, __LINE__,   \
                        #expr, (int)b__);                                     \
      return TSNE_ERR_CUDA;                                                   \
    }                                                                         \
  } while (0)

static inline int blk(int64_t n, int t) { return (int)((n + t - 1) / t); }

// G (row-major n x k) = A (row-major n x dim, ld lda) . B^T (B row-major k x dim, ld ldb)
static tsne_status gemm_abt(cublasHandle_t h, const float* A, int64_t n, int lda, const float* B,
                            int k, int ldb, int dim, float* G) {
  const float one = 1.f, zero = 0.f;
  TSNE_BLAS_TRY(cublasSgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, k, (int)n, dim, &one, B, ldb, A, lda,
                            &zero, G, k));
  return TSNE_OK;
}

// Lloyd iterations on pts (n x dim, ld) with k centroids (ld ldc); assignment
// of the last iteration left in w.assign
static tsne_status kmeans(cublasHandle_t h, const float* pts, int n, int dim, int ld, int k,
                          float* cent, int ldc, int iters, IvfWS& w, cudaStream_t s) {
  k_init_cent<<<blk((int64_t)k * dim, 256), 256, 0, s>>>(pts, n, dim, ld, k, cent, ldc);
  TSNE_LAUNCH_CHECK();
  tsne_status st;
  for (int it = 0; it <= iters; ++it) {
    k_row_norms<<<blk((int64_t)k * 32, 256), 256, 0, s>>>(cent, k, dim, ldc, w.norms);
    TSNE_LAUNCH_CHECK();
    if ((st = gemm_abt(h, pts, n, ld, cent, k, ldc, dim, w.G)) != TSNE_OK) return st;
    k_argmin_rows<<<blk((int64_t)n * 32, 256), 256, 0, s>>>(w.G, n, k, w.norms, w.assign);
    TSNE_LAUNCH_CHECK();
    if (it == iters) break;                      // the final assignment only
    // members of each centroid in point order: sort (assignment, index)
    k_iota_i<<<blk(n, 256), 256, 0, s>>>(w.order, n);
    TSNE_LAUNCH_CHECK();
    size_t sb = w.sort_bytes;
    int bits = 1;
    while ((1 << bits) <= k) ++bits;
    TSNE_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_tmp, sb, w.assign, w.assign2, w.order,
                                                  w.order2, n, 0, bits, s));
    TSNE_CUDA_TRY(cudaMemsetAsync(w.cnt, 0, sizeof(int32_t) * (k + 1), s));
    k_count<<<blk(n, 256), 256, 0, s>>>(w.assign, n, w.cnt);
    TSNE_LAUNCH_CHECK();
    size_t cb = w.scan_bytes;
    TSNE_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w.scan_tmp, cb, w.cnt, w.off, k + 1, s));
    k_centroid_means<<<k, 128, 0, s>>>(pts, dim, ld, w.order2, w.off, k, cent, ldc);
    TSNE_LAUNCH_CHECK();
  }
  return TSNE_OK;
}

static tsne_status ivf_build(const float* X, const IvfDims& d, IvfIndex& x, IvfWS& w,
                             cudaStream_t s) {
  Blas b;
  TSNE_BLAS_TRY(cublasCreate(&b.h));
  TSNE_BLAS_TRY(cublasSetStream(b.h, s));
  const float* Xp = X;
  if (d.Dp != d.D) {
    k_pad_rows<<<blk(d.N * d.Dp, 256), 256, 0, s>>>(X, d.N, d.D, d.Dp, w.Xp);
    TSNE_LAUNCH_CHECK();
    Xp = w.Xp;
  }
  tsne_status st;
  // 1. coarse quantiser: k-means on the training sample
  k_take_sample<<<blk((int64_t)d.ntrain * d.Dp, 256), 256, 0, s>>>(Xp, d.N, d.Dp, d.ntrain, w.xt);
  TSNE_LAUNCH_CHECK();
  if ((st = kmeans(b.h, w.xt, d.ntrain, d.Dp, d.Dp, d.nlist, x.cent, d.Dp, d.iters, w, s)) !=
      TSNE_OK)
    return st;
  // 2. residuals of the sample, one k-means of 256 codewords per sub-vector
  k_residuals<<<blk((int64_t)d.ntrain * d.Dp, 256), 256, 0, s>>>(w.xt, d.ntrain, d.Dp, x.cent,
                                                                w.assign);
  TSNE_LAUNCH_CHECK();
  for (int j = 0; j < d.m; ++j) {
    const int kk = d.ntrain < kKsub ? d.ntrain : kKsub;
    if (kk < kKsub)   // fewer training points than codewords: the unused codewords stay far
      TSNE_CUDA_TRY(cudaMemsetAsync(x.cb + (size_t)j * kKsub * d.dsub, 0x7f,
                                    sizeof(float) * kKsub * d.dsub, s));
    if ((st = kmeans(b.h, w.xt + (size_t)j * d.dsub, d.ntrain, d.dsub, d.Dp, kk,
                     x.cb + (size_t)j * kKsub * d.dsub, d.dsub, d.iters, w, s)) != TSNE_OK)
      return st;
  }
  // 3. coarse assignment of every point (blocks of rows)
  k_row_norms<<<blk((int64_t)d.nlist * 32, 256), 256, 0, s>>>(x.cent, d.nlist, d.Dp, d.Dp, x.cnorm);
  TSNE_LAUNCH_CHECK();
  for (int64_t r0 = 0; r0 < d.N; r0 += kCoarseBlock) {
    const int n = (int)std::min<int64_t>(kCoarseBlock, d.N - r0);
    if ((st = gemm_abt(b.h, Xp + r0 * d.Dp, n, d.Dp, x.cent, d.nlist, d.Dp, d.Dp, w.G)) != TSNE_OK)
      return st;
    k_argmin_rows<<<blk((int64_t)n * 32, 256), 256, 0, s>>>(w.G, n, d.nlist, x.cnorm,
                                                            w.assign + r0);
    TSNE_LAUNCH_CHECK();
  }
  // 4. PQ codes of every point
  {
    const size_t smem = sizeof(float) * kKsub * d.dsub;
    TSNE_CUDA_TRY(cudaFuncSetAttribute(k_encode, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    for (int64_t r0 = 0; r0 < d.N; r0 += (1 << 20)) {
      const int n = (int)std::min<int64_t>(1 << 20, d.N - r0);
      dim3 g(blk(n, 128), d.m);
      k_encode<<<g, 128, smem, s>>>(Xp, r0, n, d.Dp, d.m, d.dsub, x.cent, w.assign, x.cb,
                                    w.codes_pt);
      TSNE_LAUNCH_CHECK();
    }
  }
  // 5. inverted lists: points sorted by (list, index)
  k_iota_i<<<blk(d.N, 256), 256, 0, s>>>(w.order, d.N);
  TSNE_LAUNCH_CHECK();
  {
    size_t sb = w.sort_bytes;
    int bits = 1;
    while ((1 << bits) <= d.nlist) ++bits;
    TSNE_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_tmp, sb, w.assign, w.assign2, w.order,
                                                  x.lids, (int)d.N, 0, bits, s));
    TSNE_CUDA_TRY(cudaMemsetAsync(w.cnt, 0, sizeof(int32_t) * (d.nlist + 1), s));
    k_count<<<blk(d.N, 256), 256, 0, s>>>(w.assign, d.N, w.cnt);
    TSNE_LAUNCH_CHECK();
    size_t cb = w.scan_bytes;
    TSNE_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w.scan_tmp, cb, w.cnt, x.loff, d.nlist + 1, s));
  }
  k_gather_codes<<<blk(d.N * d.m, 256), 256, 0, s>>>(w.codes_pt, x.lids, d.N, d.m, x.codes);
  TSNE_LAUNCH_CHECK();
  // 6. T tables: <c_L,j, cb_jk> by one GEMM per sub-quantiser, then + |cb_jk|^2
  {
    const float one = 1.f, zero = 0.f;
    TSNE_BLAS_TRY(cublasSgemmStridedBatched(
        b.h, CUBLAS_OP_T, CUBLAS_OP_N, kKsub, d.nlist, d.dsub, &one, x.cb, d.dsub,
        (long long)kKsub * d.dsub, x.cent, d.Dp, (long long)d.dsub, &zero, x.T, d.m * kKsub,
        (long long)kKsub, d.m));
    k_row_norms<<<blk((int64_t)d.m * kKsub * 32, 256), 256, 0, s>>>(x.cb, (int64_t)d.m * kKsub,
                                                                    d.dsub, d.dsub, w.norms);
    TSNE_LAUNCH_CHECK();
    k_finish_T<<<blk((int64_t)d.nlist * d.m * kKsub, 256), 256, 0, s>>>(x.T, d.nlist, d.m, w.norms);
    TSNE_LAUNCH_CHECK();
  }
  return TSNE_OK;
}

static tsne_status ivf_search(const float* X, const IvfDims& d, const IvfIndex& x, int K, int tau,
                              int32_t* idx, double* d2, IvfWS& w, cudaStream_t s) {
  Blas b;
  TSNE_BLAS_TRY(cublasCreate(&b.h));
  TSNE_BLAS_TRY(cublasSetStream(b.h, s));
  const float* Xp = X;
  if (d.Dp != d.D) {
    k_pad_rows<<<blk(d.N * d.Dp, 256), 256, 0, s>>>(X, d.N, d.D, d.Dp, w.Xp);
    TSNE_LAUNCH_CHECK();
    Xp = w.Xp;
  }
  const int Kc = ivf_kc(K, &d.prm);
  const int P = d.nlist < kMaxProbes ? d.nlist : kMaxProbes;
  tsne_status st;
  k_row_norms<<<blk(d.N * 32, 256), 256, 0, s>>>(Xp, d.N, d.Dp, d.Dp, w.norms);
  TSNE_LAUNCH_CHECK();
  const size_t lut = sizeof(float) * d.m * kKsub;
  TSNE_CUDA_TRY(cudaFuncSetAttribute(k_ivf_scan, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)lut));
  for (int64_t q0 = 0; q0 < d.N; q0 += kIvfBlock) {
    const int nb = (int)std::min<int64_t>(kIvfBlock, d.N - q0);
    const int32_t* qid = x.lids + q0;            // the block's queries in list order
    k_gather_queries<<<blk((int64_t)nb * d.Dp, 256), 256, 0, s>>>(Xp, d.Dp, qid, nb, w.Xq);
    TSNE_LAUNCH_CHECK();
    // probe order: distances to the centroids
    if ((st = gemm_abt(b.h, w.Xq, nb, d.Dp, x.cent, d.nlist, d.Dp, d.Dp, w.G)) != TSNE_OK)
      return st;
    k_probes<<<blk((int64_t)nb * 32, 256), 256, 0, s>>>(w.G, nb, d.nlist, P, x.cnorm, w.norms,
                                                        qid, w.probes, w.pbase);
    TSNE_LAUNCH_CHECK();
    // Q tables of the block: <x_j, cb_jk>, one GEMM per sub-quantiser
    const float one = 1.f, zero = 0.f;
    TSNE_BLAS_TRY(cublasSgemmStridedBatched(
        b.h, CUBLAS_OP_T, CUBLAS_OP_N, kKsub, nb, d.dsub, &one, x.cb, d.dsub,
        (long long)kKsub * d.dsub, w.Xq, d.Dp, (long long)d.dsub, &zero, w.G,
        d.m * kKsub, (long long)kKsub, d.m));
    k_ivf_scan<<<kNumSMs, kIvfThreads, lut, s>>>(qid, nb, d.m, P, tau, Kc, w.G, x.T, x.codes,
                                                  x.loff, x.lids, w.probes, w.pbase, w.cbuf,
                                                  w.cand);
    TSNE_LAUNCH_CHECK();
    k_ivf_rerank<<<blk(nb, 8), 256, 0, s>>>(X, qid, nb, d.D, K, Kc, w.cand, idx, d2);
    TSNE_LAUNCH_CHECK();
  }
  return TSNE_OK;
}

tsne_status check_device();

}  // namespace tsne

using namespace tsne;

extern "C" {

void tsne_ivfpq_params_default(tsne_ivfpq_params* p) {
  if (!p) return;
  p->nlist = 0;
  p->m = 0;
  p->kmeans_iters = 10;
  p->train_per_list = 64;
  p->kprime = 0;
  p->seed = 0;
}

size_t tsne_ivfpq_index_size(int64_t N, int32_t D, const tsne_ivfpq_params* p) {
  if (N < 2 || D < 1) return 0;
  const IvfDims d = ivf_dims(N, D, p);
  IvfIndex x;
  Carver c(nullptr);
  return carve_index(c, d, x);
}

tsne_status tsne_ivfpq_layout(int64_t N, int32_t D, const tsne_ivfpq_params* p, int64_t* out) {
  clear_error();
  TSNE_ARG_CHECK(N >= 2 && D >= 1 && out, "bad arguments");
  const IvfDims d = ivf_dims(N, D, p);
  IvfIndex x;
  Carver c(nullptr);
  carve_index(c, d, x);
  out[0] = d.nlist; out[1] = d.m; out[2] = d.dsub; out[3] = d.Dp;
  out[4] = (int64_t)reinterpret_cast<uintptr_t>(x.cent);
  out[5] = (int64_t)reinterpret_cast<uintptr_t>(x.cb);
  out[6] = (int64_t)reinterpret_cast<uintptr_t>(x.codes);
  out[7] = (int64_t)reinterpret_cast<uintptr_t>(x.loff);
  out[8] = (int64_t)reinterpret_cast<uintptr_t>(x.lids);
  out[9] = (int64_t)reinterpret_cast<uintptr_t>(x.T);
  out[10] = d.ntrain;
  return TSNE_OK;
}

size_t tsne_ivfpq_workspace_size(int64_t N, int32_t D, int32_t K, const tsne_ivfpq_params* p) {
  if (N < 2 || D < 1) return 0;
  const IvfDims d = ivf_dims(N, D, p);
  IvfWS w;
  Carver c(nullptr);
  const int Kc = K > 0 ? ivf_kc(K, p) : 0;
  return carve_ivf_ws(c, d, Kc, w);
}

tsne_status tsne_ivfpq_build(const float* X, int64_t N, int32_t D, const tsne_ivfpq_params* p,
                             void* index, size_t index_bytes, void* ws, size_t ws_bytes,
                             tsne_stream_t stream) {
  clear_error();
  TSNE_ARG_CHECK(N >= 2 && N < (int64_t(1) << 31) - 1 && D >= 1, "need N >= 2, D >= 1");
  TSNE_ARG_CHECK(X && index, "null pointer argument");
  const IvfDims d = ivf_dims(N, D, p);
  TSNE_ARG_CHECK(d.nlist <= N && d.nlist <= (1 << 20), "nlist must be in [1, min(N, 2^20)]");
  TSNE_ARG_CHECK(d.dsub <= 64, "D / m must be <= 64 (got dsub = %d)", d.dsub);
  TSNE_ARG_CHECK(aligned(X, 4) && aligned(index, 256), "X 4-byte, index 256-byte aligned");
  IvfIndex x;
  Carver ci(nullptr);
  const size_t need_i = carve_index(ci, d, x);
  IvfWS w;
  Carver cw(nullptr);
  const size_t need_w = carve_ivf_ws(cw, d, 0, w);
  if (index_bytes < need_i || !ws || ws_bytes < need_w) {
    set_error("index needs %zu bytes (got %zu), workspace %zu (got %zu)", need_i, index_bytes,
              need_w, ws_bytes);
    return TSNE_ERR_WORKSPACE;
  }
  tsne_status st = check_device();
  if (st != TSNE_OK) return st;
  Carver c1(index);
  carve_index(c1, d, x);
  Carver c2(ws);
  carve_ivf_ws(c2, d, 0, w);
  return ivf_build(X, d, x, w, (cudaStream_t)stream);
}

tsne_status tsne_ivfpq_search(const float* X, int64_t N, int32_t D, const tsne_ivfpq_params* p,
                              const void* index, int32_t K, int32_t tau, int32_t* idx,
                              double* d2, void* ws, size_t ws_bytes, tsne_stream_t stream) {
  clear_error();
  TSNE_ARG_CHECK(N >= 2 && N < (int64_t(1) << 31) - 1 && D >= 1, "need N >= 2, D >= 1");
  TSNE_ARG_CHECK(X && index && idx && d2, "null pointer argument");
  TSNE_ARG_CHECK(K >= 1 && K < N && K <= kMaxKc, "K must be in [1, min(N-1, %d)]", kMaxKc);
  const IvfDims d = ivf_dims(N, D, p);
  TSNE_ARG_CHECK(tau >= 1 && tau <= d.nlist && tau <= kMaxProbes,
                 "tau must be in [1, min(nlist = %d, %d)]", d.nlist, kMaxProbes);
  TSNE_ARG_CHECK((int64_t)d.m * kKsub * 4 <= 227 * 1024, "m too large for the look-up table");
  const int Kc = ivf_kc(K, p);
  IvfWS w;
  Carver cw(nullptr);
  const size_t need_w = carve_ivf_ws(cw, d, Kc, w);
  if (!ws || ws_bytes < need_w) {
    set_error("workspace too small: need %zu bytes, got %zu", need_w, ws_bytes);
    return TSNE_ERR_WORKSPACE;
  }
  tsne_status st = check_device();
  if (st != TSNE_OK) return st;
  IvfIndex x;
  Carver c1(const_cast<void*>(index));
  carve_index(c1, d, x);
  Carver c2(ws);
  carve_ivf_ws(c2, d, Kc, w);
  return ivf_search(X, d, x, K, tau, idx, d2, w, (cudaStream_t)stream);
}

}  // extern "C"
