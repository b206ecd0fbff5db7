// knn.cu -- exact kNN (U1).  The paper's line 1 is approximate FAISS
// IVF-PQ; the north star asks for the exact kNN, so:
//
//  1. prep:      column mean (fp64, fixed order), X_h = fp16((x - mean) 2^e)
//                (distance-invariant centring + exact power-of-2 scaling),
//                |x_h|^2 in fp32.
//  2. candidates: expanded-form distances |x_h|^2 + |y_h|^2 - 2 x_h . y_h
//                (the row's |x_h|^2 is dropped: it does not change the order
//                within a row) for every (query, point) pair, tile by tile,
//                keeping for each query the K' = K + 64 smallest keys
//                (distance, index) -- candidate buffers in global memory,
//                compacted by a warp bitonic sort when they fill.  The N x N
//                matrix is never materialised.
//  3. re-rank:   exact fp64 sum_d (x_d - y_d)^2 of the original fp32 rows for
//                the K' candidates; sort by (d2, index) (D18); certificate
//                d2_(K) < approx_(K') - 2 e_row (D26).
#include <cfloat>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "knn.cuh"
#include "knn_select.cuh"
#include "knn_tc.cuh"

namespace tsne {

static inline int kc_of(int64_t N, int K) {
  int64_t kc = ((K + kCandExtra + 31) / 32) * 32;
  if (kc > N - 1) kc = N - 1;
  return (int)kc;
}

int knn_slots(int64_t N) {
  int64_t rb = (N + kKnnBM - 1) / kKnnBM;
  rb = (rb + 1) & ~int64_t(1);               // CTA pairs need an even count
  int64_t cap = 2 * kNumSMs;
  return (int)(rb < cap ? rb : cap);


}

void carve_knn(Carver& c, KnnWS& w, int64_t N, int32_t D, int32_t K) {
  w.N = N; w.D = D; w.K = K;
  w.Dp = ((D + 63) / 64) * 64;
  w.Kc = kc_of(N, K);
  w.slots = knn_slots(N);
  w.colsum = c.take<double>((size_t)D * 256);
  w.mean = c.take<float>(D);
  w.amax = c.take<unsigned>(4);
  w.scale = c.take<float>(4);
  w.Xh = c.take<__half>((size_t)(N + 256) * w.Dp);  // + 256 zero slack rows (tile overrun)
  w.nrm = c.take<float>(N + 256);
  w.buf = c.take<u64>((size_t)w.slots * kKnnBM * kCandCap);
  w.cand = c.take<u64>((size_t)N * w.Kc);
  w.uncert = c.take<u64>(2);
  w.rows_bad = c.take<int32_t>(N);
  {
    const size_t a = knn_tc2_sync_words(N, N), b = knn_sym_sync_words(N);
    w.sync = c.take<unsigned>(a > b ? a : b);
  }
  w.sd = c.take<double>((size_t)kScanRows * N);
  w.sd_alt = c.take<double>(N);
  w.si = c.take<int32_t>(N);
  w.si_alt = c.take<int32_t>(N);
  cub::DoubleBuffer<double> dk(nullptr, nullptr);
  cub::DoubleBuffer<int32_t> dv(nullptr, nullptr);
  w.sort_tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, w.sort_tmp_bytes, dk, dv, (int)N);
  {
    cub::DoubleBuffer<uint32_t> ck(nullptr, nullptr);
    size_t b2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b2, ck, dv, (int)N);
    if (b2 > w.sort_tmp_bytes) w.sort_tmp_bytes = b2;
  }
  w.sort_tmp = c.take<unsigned char>(w.sort_tmp_bytes);
  // symmetric search buffers (used by full-N calls with enough super-blocks)
  w.sym = N >= 4 * 256;
  if (w.sym) {
    w.C = (int32_t)(N / 64 < kSymCells ? N / 64 : kSymCells);
    w.Xs = c.take<__half>((size_t)(w.C + 256) * w.Dp);
    w.nrm_s = c.take<float>(w.C + 256);
    w.cand32 = c.take<u64>((size_t)N * 32);
    w.cell = c.take<uint32_t>(2 * (size_t)N);
    w.perm = c.take<int32_t>(2 * (size_t)N);
    w.inv = c.take<int32_t>(N);
    w.Xp = c.take<__half>((size_t)(N + 256) * w.Dp);
    w.nrm_p = c.take<float>(N + 256);
    w.tau = c.take<float>(N + 256);
    w.ntau = c.take<float>(N + 256);
    w.cnt = c.take<unsigned>(N);
    w.list = c.take<u64>((size_t)N * kSymCap);
    w.fb = c.take<int32_t>(N);
    w.Xq = c.take<__half>((size_t)(kFbRows + 256) * w.Dp);
    w.candfb = c.take<u64>((size_t)kFbRows * w.Kc);
    w.misc = c.take<unsigned>(4);
  }
}

// ---------------------------------------------------------------- prep
constexpr int kColRB = 256;  // row blocks of the fixed-order column sum

__global__ void k_colsum_part(const float* __restrict__ X, int64_t N, int D,
                              double* __restrict__ part) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= D) return;
  const int64_t r0 = (int64_t)blockIdx.y * N / kColRB, r1 = (int64_t)(blockIdx.y + 1) * N / kColRB;
  double s = 0.0;
  for (int64_t r = r0; r < r1; ++r) s += (double)X[r * D + d];
  part[(size_t)blockIdx.y * D + d] = s;
}

__global__ void k_colsum_final(const double* __restrict__ part, int64_t N, int D,
                               float* __restrict__ mean, unsigned* amax) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d == 0) { amax[0] = 0u; amax[1] = 0u; }
  if (d >= D) return;
  double s = 0.0;
  for (int b = 0; b < kColRB; ++b) s += part[(size_t)b * D + d];
  mean[d] = (float)(s / (double)N);
}

__global__ void k_absmax(const float* __restrict__ X, int64_t n, int D,
                         const float* __restrict__ mean, unsigned* amax) {
  float m = 0.f;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(X[e] - mean[e % D]));
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomicMax(amax, __float_as_uint(m));  // non-negative: int order
}

__global__ void k_scale(const unsigned* amax, float* scale) {
  const float a = __uint_as_float(*amax);
  int e = 0;
  if (a > 0.f) {
    int ex;
    frexpf(a, &ex);             // a in [2^(ex-1), 2^ex)
    e = 14 - ex;                // a 2^e < 2^14
  }
  scale[0] = ldexpf(1.f, e);
  scale[1] = ldexpf(1.f, -2 * e);
}

// warp per row: X_h row and its squared norm
__global__ void k_convert(const float* __restrict__ X, int64_t N, int D, int Dp,
                          const float* __restrict__ mean, const float* __restrict__ scale,
                          __half* __restrict__ Xh, float* __restrict__ nrm) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (row >= N + 256) return;
  const float sc = scale[0];
  double acc = 0.0;
  for (int d = lane; d < Dp; d += 32) {
    __half h = __float2half_rn(0.f);
    if (row < N && d < D) h = __float2half_rn((X[row * D + d] - mean[d]) * sc);
    Xh[row * Dp + d] = h;
    const float f = __half2float(h);
    acc += (double)(f * f);
  }
  acc = warp_sum(acc);
  if (lane == 0) nrm[row] = row < N ? (float)acc : 0.f;
}

// max_j |x_h,j|^2 over the N points (float bits into amax[1]): the norm bound
// of the D26 certificate
__global__ void k_nrm_max(const float* __restrict__ nrm, int64_t N, unsigned* amax) {
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, nrm[i]);
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomicMax(amax + 1, __float_as_uint(m));  // non-negative
}

// ---------------------------------------------------------------- re-rank
constexpr int kRR_Threads = 256;

__global__ void __launch_bounds__(kRR_Threads)
k_rerank(const float* __restrict__ X, int N, int qs, int nq, int D, int K, int Kc,
         const u64* __restrict__ cand,
         const float* __restrict__ nrm, const float* __restrict__ scale,
         int32_t* __restrict__ idx, double* __restrict__ d2, u64* __restrict__ uncert,
         int32_t* __restrict__ rows_bad, int force_mod, const int32_t* __restrict__ perm,
         const int32_t* __restrict__ inv, const unsigned* __restrict__ amax, int Dp) {
  // perm / inv (nullable): the candidates are stored by locality position
  // (symmetric search) with locality-position indices in their keys
  __shared__ double s_d[kRR_Threads / 32][256];
  __shared__ int s_j[kRR_Threads / 32][256];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int w = blockIdx.x * (kRR_Threads / 32) + wid;
  if (w >= nq) return;
  // with a locality order (symmetric search) warps take the rows in that
  // order: consecutive rows share most candidates, which then hit in L2
  const int il = perm ? perm[w] : w;                       // local query row
  const int i = qs + il;
  double* sd = s_d[wid];
  int* sj = s_j[wid];
  const float* xi = X + (size_t)i * D;
  const u64* ci = cand + (size_t)(perm ? w : il) * Kc;
  const double inv2 = (double)scale[1];
  const double nrm_i = (double)nrm[i];
  for (int c = 0; c < Kc; ++c) {
    const u64 key = ci[c];
    const int j = perm ? perm[key_idx(key)] : key_idx(key);
    const float* xj = X + (size_t)j * D;
    double acc = 0.0;
    for (int d = lane; d < D; d += 32) {
      const double t = (double)__ldg(xi + d) - (double)xj[d];
      acc = fma(t, t, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      sd[c] = acc;
      sj[c] = j;
    }
  }
  // approximate (scaled) distance of the K'-th candidate: every point that is
  // not a candidate has an approximate key >= this one
  const double tau_scaled = (double)key_val(ci[Kc - 1]) + nrm_i;
  int P = 32;
  while (P < Kc) P <<= 1;
  for (int c = Kc + lane; c < P; c += 32) { sd[c] = DBL_MAX; sj[c] = 0x7fffffff; }
  __syncwarp();
  // bitonic sort by (d2, index)
  for (int k = 2; k <= P; k <<= 1)
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int a = lane; a < P; a += 32) {
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
    idx[(size_t)il * K + c] = sj[c];
    d2[(size_t)il * K + c] = sd[c];
  }
  if (lane == 0) {
    const bool all = (Kc >= N - 1);
    // D26 certificate, an a-priori bound valid for EVERY point j (not only the
    // candidates).  In the scaled, centred units of the candidate stage
    // (c = (x - mean) 2^e real, h = fp16(c)), approx_ij = |h_j|^2 - 2 h_i.h_j +
    // |h_i|^2 with |h_k - c_k| <= u |c_k| + a per element (u = 2^-11 fp16
    // rounding + 2^-23 for the fp32 centring; a = 2^-25, fp16 subnormals), so
    //   | |h_i - h_j|^2 - |c_i - c_j|^2 | <= 2 |c_i - c_j| E1 + E1^2,
    //   E1 = u (|c_i| + |c_j|) + 2 a sqrt(Dp);
    // the computed key adds the fp32 rounding of the norms (2^-24 each), of
    // the tensor-core dot product (<= Dp 2^-22 |h_i| |h_j|, a conservative
    // model of fp32 accumulation) and of the FFMA (2^-24 |key|).  The error
    // grows with the distance, so if a non-candidate j had exact d_ij <= d_(K),
    // then approx_ij <= d_(K) + err(d_(K)) < tau: contradiction.  Hence
    // certified iff tau > d_(K) + err(d_(K)), with the norm bound M of all
    // points (amax[1]).
    const double u = 0x1p-11 + 0x1p-23, a = 0x1p-25, sqD = sqrt((double)Dp);
    const double M = (sqrt((double)__uint_as_float(amax[1]) * (1.0 + 0x1p-23)) + a * sqD) / (1.0 - u);
    const double ni = (sqrt(nrm_i * (1.0 + 0x1p-23)) + a * sqD) / (1.0 - u);
    const double E1 = u * (ni + M) + 2.0 * a * sqD;
    const double dK = sd[K - 1] / inv2 * (1.0 + 1e-12);          // scaled exact d_(K)
    const double G = 0x1p-24 * (M * M + ni * ni) + 2.0 * ((double)Dp * 0x1p-22) * ni * M +
                     0x1p-24 * (M * M + 2.0 * ni * M);
    const double bound = dK + 2.0 * sqrt(dK) * E1 + E1 * E1 + G;
    bool cert = all || (tau_scaled > bound * (1.0 + 1e-12));
    if (force_mod > 0 && i % force_mod == 0) cert = false;   // test hook (fallback coverage)
    if (!cert) {
      const u64 pos = atomicAdd(uncert, 1ull);
      rows_bad[pos] = i;
    }
  }
}

// ---------------------------------------------------------------- exact fallback (D26)
// Rows whose candidate margin could not be certified: fp64 distances to all N
// points, in the re-rank's own arithmetic (lane-strided fma, fixed butterfly),
// so a row gets the same d2 values either way; then a stable radix sort of
// (d2, index) -- ties by the lower index (D18).  Self -> +inf (sorted last).
__global__ void __launch_bounds__(256)
k_scan_dist(const float* __restrict__ X, int N, int D, const int32_t* __restrict__ rows, int nr,
            double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < N; j += nw) {
    const float* xj = X + (size_t)j * D;
    for (int r = 0; r < nr; ++r) {
      const int i = rows[r];
      const float* xi = X + (size_t)i * D;
      double acc = 0.0;
      for (int d = lane; d < D; d += 32) {
        const double t = (double)__ldg(xi + d) - (double)xj[d];
        acc = fma(t, t, acc);
      }
      acc = warp_sum(acc);
      if (lane == 0) out[(size_t)r * N + j] = (j == i) ? (double)INFINITY : acc;
    }
  }
}

__global__ void k_iota(int32_t* __restrict__ v, int n) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) v[k] = k;
}

__global__ void k_scan_emit(const double* __restrict__ dk, const int32_t* __restrict__ dv, int K,
                            int32_t* __restrict__ idx, double* __restrict__ d2) {
  for (int c = threadIdx.x; c < K; c += blockDim.x) { idx[c] = dv[c]; d2[c] = dk[c]; }
}

static tsne_status exact_fallback(const float* X, int64_t N, int32_t D, int32_t K, int64_t q0,
                                  const int32_t* rows_host, int64_t nbad, int32_t* idx, double* d2,
                                  KnnWS& w, cudaStream_t s) {
  for (int64_t r0 = 0; r0 < nbad; r0 += kScanRows) {
    const int nr = (int)((nbad - r0 < kScanRows) ? nbad - r0 : kScanRows);
    TSNE_CUDA_TRY(cudaMemcpyAsync(w.si_alt, rows_host + r0, nr * sizeof(int32_t),
                                  cudaMemcpyHostToDevice, s));
    k_scan_dist<<<8 * kNumSMs, 256, 0, s>>>(X, (int)N, D, w.si_alt, nr, w.sd);
    TSNE_LAUNCH_CHECK();
    TSNE_CUDA_TRY(cudaStreamSynchronize(s));   // si_alt is reused as a sort buffer below
    for (int r = 0; r < nr; ++r) {
      k_iota<<<2 * kNumSMs, 256, 0, s>>>(w.si, (int)N);
      TSNE_LAUNCH_CHECK();
      cub::DoubleBuffer<double> dk(w.sd + (size_t)r * N, w.sd_alt);
      cub::DoubleBuffer<int32_t> dv(w.si, w.si_alt);
      size_t tb = w.sort_tmp_bytes;
      TSNE_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_tmp, tb, dk, dv, (int)N, 0, 64, s));
      const int64_t il = rows_host[r0 + r] - q0;
      k_scan_emit<<<1, 256, 0, s>>>(dk.Current(), dv.Current(), K, idx + (size_t)il * K,
                                   d2 + (size_t)il * K);
      TSNE_LAUNCH_CHECK();
    }
  }
  return TSNE_OK;
}

// ---------------------------------------------------------------- symmetric search (knn_sym.cu)
__global__ void k_gather_rows(const __half* __restrict__ src, const float* __restrict__ nsrc,
                              const int32_t* __restrict__ idx, int64_t n, int64_t n_pad, int Dp,
                              __half* __restrict__ dst, float* __restrict__ ndst) {
  // warp per destination row; rows n .. n_pad-1 are zero (tile overrun)
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n_pad) return;
  const uint4* s4 = r < n ? reinterpret_cast<const uint4*>(src + (size_t)idx[r] * Dp) : nullptr;
  uint4* d4 = reinterpret_cast<uint4*>(dst + (size_t)r * Dp);
  for (int k = lane; k < Dp / 8; k += 32) d4[k] = s4 ? s4[k] : make_uint4(0, 0, 0, 0);
  if (lane == 0) ndst[r] = r < n ? nsrc[idx[r]] : 0.f;
}

__global__ void k_sample_idx(int32_t* __restrict__ idx, int C, int64_t N) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < C) idx[k] = (int32_t)((int64_t)k * N / C);
}

// sort key of point i: the tour rank of its cell (nearest sample)
__global__ void k_cells(const u64* __restrict__ cand32, int64_t N, int cbits,
                        const int32_t* __restrict__ group, uint32_t* __restrict__ cell,
                        int32_t* __restrict__ ids, const float* __restrict__ nrm,
                        unsigned* __restrict__ misc) {
  float m = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t cl = (uint32_t)key_idx(cand32[(size_t)i * 32]);
    cell[i] = ((uint32_t)group[cl] << cbits);   // the cell's rank in the tour
    ids[i] = (int32_t)i;
    m = fmaxf(m, nrm[i]);
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomicMax(misc, __float_as_uint(m));   // non-negative
}

__global__ void k_inv(const int32_t* __restrict__ perm, int64_t N, int32_t* __restrict__ inv) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < N;
       p += (int64_t)gridDim.x * blockDim.x)
    inv[perm[p]] = (int32_t)p;
}

// tau = the pilot's K'-th key + slack1 (rounding of the same pair in another
// tile orientation), ntau = -(tau + slack2) (the column-side fast filter)
__global__ void k_tau(const u64* __restrict__ cand, int64_t N, int Kc,
                      const unsigned* __restrict__ misc, float* __restrict__ tau,
                      float* __restrict__ ntau, unsigned* __restrict__ cnt) {
  const float mx = __uint_as_float(misc[0]);
  const float slack1 = ldexpf(mx, -11), slack2 = ldexpf(mx, -16);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N + 256;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < N) {
      const u64 k = cand[(size_t)i * Kc + Kc - 1];
      const float t = (k == kKeyMax) ? INFINITY : key_val(k) + slack1;
      tau[i] = t;
      ntau[i] = -(t + slack2);
      cnt[i] = 0u;
    } else {
      tau[i] = -INFINITY;
      ntau[i] = INFINITY;
    }
  }
}

// per point: the K' smallest keys of its list (or a fallback entry)
constexpr int kSelWarps = 4;
__global__ void __launch_bounds__(kSelWarps * 32)
k_select(const unsigned* __restrict__ cnt, u64* __restrict__ list, int64_t N, int Kc,
         u64* __restrict__ cand, int32_t* __restrict__ fb, unsigned* __restrict__ nfb) {
  __shared__ u64 scratch[kSelWarps][kSymCap];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * kSelWarps + wid;
  if (i >= N) return;
  const unsigned n = cnt[i];
  if (n > (unsigned)kSymCap || n < (unsigned)Kc) {
    if (lane == 0) fb[atomicAdd(nfb, 1u)] = (int32_t)i;
    return;
  }
  u64 t;
  compact_keys(list + (size_t)i * kSymCap, (int)n, Kc, scratch[wid], lane, cand + (size_t)i * Kc, t);
}

__global__ void k_scatter_cand(const u64* __restrict__ src, const int32_t* __restrict__ rows,
                               int n, int Kc, u64* __restrict__ cand) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)n * Kc;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / Kc, c = e % Kc;
    cand[(size_t)rows[r] * Kc + c] = src[e];
  }
}

// candidates of all N points by the symmetric search; w.cand / w.perm / w.inv
// hold the result (cand rows and key indices in locality positions)
struct StageTimer {   // TSNE_KNN_TIMING=1: per-stage times of the symmetric search (stderr)
  bool on;
  cudaStream_t s;
  cudaEvent_t ev[8];
  int n = 0;
  StageTimer(cudaStream_t st) : on(getenv("TSNE_KNN_TIMING") != nullptr), s(st) {
    if (on) for (auto& e : ev) cudaEventCreate(&e);
  }
  void mark() { if (on && n < 8) cudaEventRecord(ev[n++], s); }
  void report(const char* const* names, int64_t N, const unsigned* cnt) {
    if (!on) return;
    cudaStreamSynchronize(s);
    for (int k = 1; k < n; ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[k - 1], ev[k]);
      fprintf(stderr, "  sym %-10s %9.2f ms\n", names[k - 1], ms);
    }
    if (cnt) {
      unsigned* h = (unsigned*)malloc(N * sizeof(unsigned));
      cudaMemcpy(h, cnt, N * sizeof(unsigned), cudaMemcpyDeviceToHost);
      double sum = 0; unsigned mx = 0; int64_t over = 0;
      for (int64_t i = 0; i < N; ++i) { sum += h[i]; mx = h[i] > mx ? h[i] : mx; over += h[i] > kSymCap; }
      fprintf(stderr, "  sym lists: mean %.1f max %u overflow %lld\n", sum / N, mx, (long long)over);
      free(h);
    }
    for (auto& e : ev) cudaEventDestroy(e);
  }
};

static tsne_status sym_candidates(int64_t N, KnnWS& w, cudaStream_t s) {
  const int Dp = w.Dp, Kc = w.Kc, C = w.C;
  StageTimer tm(s);
  tm.mark();
  // 1. locality order: nearest of C sampled points (tensor-core pair kernel,
  //    K' = 32), points sorted by that cell
  k_sample_idx<<<(C + 255) / 256, 256, 0, s>>>(w.fb, C, N);
  TSNE_LAUNCH_CHECK();
  k_gather_rows<<<(int)(((int64_t)(C + 256) * 32 + 255) / 256), 256, 0, s>>>(
      w.Xh, w.nrm, w.fb, C, C + 256, Dp, w.Xs, w.nrm_s);
  TSNE_LAUNCH_CHECK();
  // cell order: a greedy nearest-neighbour tour over the samples (host, C
  // nodes, from their 32 nearest samples), so that neighbouring cells --
  // e.g. the cells of one cluster -- are adjacent in the locality order
  tsne_status st = launch_cand_pair(w.Xs, C + 256, w.Xs, C + 256, w.nrm_s, C, 0, C, Dp, 32, w.buf,
                                    w.cand32, w.slots, nullptr, s, 1, 0, nullptr);
  if (st != TSNE_OK) return st;
  {
    std::vector<u64> nb((size_t)C * 32);
    TSNE_CUDA_TRY(cudaMemcpyAsync(nb.data(), w.cand32, nb.size() * sizeof(u64),
                                  cudaMemcpyDeviceToHost, s));
    TSNE_CUDA_TRY(cudaStreamSynchronize(s));
    std::vector<int32_t> rank(C, -1);
    int next_unvisited = 0, cur = 0, r = 0;
    while (r < C) {
      rank[cur] = r++;
      int nxt = -1;
      for (int k = 0; k < 32 && k < C - 1; ++k) {           // nearest unvisited sample
        const int j = (int)(unsigned)(nb[(size_t)cur * 32 + k] & 0xffffffffull);
        if (j >= 0 && j < C && rank[j] < 0) { nxt = j; break; }
      }
      if (nxt < 0) {                                        // jump: lowest unvisited
        while (next_unvisited < C && rank[next_unvisited] >= 0) ++next_unvisited;
        nxt = next_unvisited;
      }
      cur = nxt;
      if (cur >= C) break;
    }
    TSNE_CUDA_TRY(cudaMemcpyAsync(w.inv, rank.data(), C * sizeof(int32_t), cudaMemcpyHostToDevice,
                                  s));
    TSNE_CUDA_TRY(cudaStreamSynchronize(s));   // `rank` is a host temporary
  }
  const int32_t* group = w.inv;                // cell -> tour rank (scratch until k_inv)
  st = launch_cand_pair(w.Xh, N + 256, w.Xs, C + 256, w.nrm_s, C, 0, (int)N, Dp, 32, w.buf,
                        w.cand32, w.slots, nullptr, s, 0, 0, nullptr);
  if (st != TSNE_OK) return st;
  TSNE_CUDA_TRY(cudaMemsetAsync(w.misc, 0, 4 * sizeof(unsigned), s));
  int cb = 1;
  while ((1 << cb) < C) ++cb;
  k_cells<<<4 * kNumSMs, 256, 0, s>>>(w.cand32, N, 0, group, w.cell, w.perm + N, w.nrm, w.misc);
  TSNE_LAUNCH_CHECK();
  {
    cub::DoubleBuffer<uint32_t> dk(w.cell, w.cell + N);
    cub::DoubleBuffer<int32_t> dv(w.perm + N, w.perm);
    size_t tb = w.sort_tmp_bytes;
    const int eb = cb;
    TSNE_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_tmp, tb, dk, dv, (int)N, 0, eb, s));
    if (dv.Current() != w.perm)
      TSNE_CUDA_TRY(cudaMemcpyAsync(w.perm, dv.Current(), N * sizeof(int32_t),
                                    cudaMemcpyDeviceToDevice, s));
  }
  k_inv<<<4 * kNumSMs, 256, 0, s>>>(w.perm, N, w.inv);
  TSNE_LAUNCH_CHECK();
  k_gather_rows<<<(int)(((N + 256) * 32 + 255) / 256), 256, 0, s>>>(w.Xh, w.nrm, w.perm, N, N + 256,
                                                                   Dp, w.Xp, w.nrm_p);
  TSNE_LAUNCH_CHECK();
  tm.mark();
  // 2. pilot: the K' best within kSymWindow column tiles around each point
  st = launch_cand_pair(w.Xp, N + 256, w.Xp, N + 256, w.nrm_p, (int)N, 0, (int)N, Dp, Kc, w.buf,
                        w.cand, w.slots, nullptr, s, 1, kSymWindow, nullptr);
  if (st != TSNE_OK) return st;
  k_tau<<<4 * kNumSMs, 256, 0, s>>>(w.cand, N, Kc, w.misc, w.tau, w.ntau, w.cnt);
  TSNE_LAUNCH_CHECK();
  tm.mark();
  // 3. the symmetric sweep
  st = launch_sym(w.Xp, N + 256, w.nrm_p, w.tau, w.ntau, w.cnt, w.list, kSymCap, (int)N, Dp,
                  w.sync, s);
  if (st != TSNE_OK) return st;
  tm.mark();
  // 4. selection; overflowing / underfilled points redone by the row sweep
  k_select<<<(int)((N + kSelWarps - 1) / kSelWarps), kSelWarps * 32, 0, s>>>(
      w.cnt, w.list, N, Kc, w.cand, w.fb, w.misc + 1);
  TSNE_LAUNCH_CHECK();
  unsigned nfb = 0;
  TSNE_CUDA_TRY(cudaMemcpyAsync(&nfb, w.misc + 1, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  TSNE_CUDA_TRY(cudaStreamSynchronize(s));
  tm.mark();
  w.sym_fallback = nfb;
  if (tm.on) fprintf(stderr, "  sym fallback points %u\n", nfb);
  for (unsigned r0 = 0; r0 < nfb; r0 += kFbRows) {
    const int n = (int)((nfb - r0) < (unsigned)kFbRows ? nfb - r0 : kFbRows);
    k_gather_rows<<<(int)(((int64_t)(n + 256) * 32 + 255) / 256), 256, 0, s>>>(
        w.Xp, w.nrm_p, w.fb + r0, n, n + 256, Dp, w.Xq, w.ntau);   // ntau: dead scratch now
    TSNE_LAUNCH_CHECK();
    st = launch_cand_pair(w.Xq, n + 256, w.Xp, N + 256, w.nrm_p, (int)N, 0, n, Dp, Kc, w.buf,
                          w.candfb, w.slots, nullptr, s, 1, 0, w.fb + r0);
    if (st != TSNE_OK) return st;
    k_scatter_cand<<<4 * kNumSMs, 256, 0, s>>>(w.candfb, w.fb + r0, n, Kc, w.cand);
    TSNE_LAUNCH_CHECK();
  }
  tm.mark();
  static const char* names[] = {"order", "pilot", "sweep", "select", "fallback"};
  tm.report(names, N, w.cnt);
  return TSNE_OK;
}

// ---------------------------------------------------------------- host
tsne_status run_knn(const float* X, int64_t N, int32_t D, int32_t K, int64_t q0, int64_t nq,
                    int32_t* idx, double* d2, KnnWS& w, tsne_knn_info* info, cudaStream_t s) {
  const int Dp = w.Dp, Kc = w.Kc;
  {
    dim3 g((D + 255) / 256, kColRB);
    k_colsum_part<<<g, 256, 0, s>>>(X, N, D, w.colsum);
    TSNE_LAUNCH_CHECK();
    k_colsum_final<<<(D + 255) / 256, 256, 0, s>>>(w.colsum, N, D, w.mean, w.amax);
    TSNE_LAUNCH_CHECK();
    k_absmax<<<4 * kNumSMs, 256, 0, s>>>(X, N * (int64_t)D, D, w.mean, w.amax);
    TSNE_LAUNCH_CHECK();
    k_scale<<<1, 1, 0, s>>>(w.amax, w.scale);
    TSNE_LAUNCH_CHECK();
    const int64_t rows = N + 256;
    k_convert<<<(int)((rows * 32 + 255) / 256), 256, 0, s>>>(X, N, D, Dp, w.mean, w.scale, w.Xh,
                                                            w.nrm);
    TSNE_LAUNCH_CHECK();
    k_nrm_max<<<4 * kNumSMs, 256, 0, s>>>(w.nrm, N, w.amax);
    TSNE_LAUNCH_CHECK();
  }
  TSNE_CUDA_TRY(cudaMemsetAsync(w.uncert, 0, 2 * sizeof(u64), s));
  // A full-N call uses the symmetric search (knn_sym.cu) where the tensor
  // work dominates its list appends -- large N and D (measured: C5
  // 1.28M x 2048 5.8 s -> 3.2 s; C2/C4 (D <= 784) are faster row by row);
  // otherwise the CTA-pair row sweep (knn_tc2.cu).  Test hook:
  // TSNE_KNN_PATH=tc2 / =sym forces one of the two (results are identical).
  if (!knn_tc_available()) {
    set_error("tcgen05 path unavailable (no sm_100 device or no cuTensorMapEncodeTiled)");
    return TSNE_ERR_CUDA;
  }
  const char* force = getenv("TSNE_KNN_PATH");
  const bool sym_default = N >= (int64_t(1) << 18) && Dp >= 1024;
  const bool sym = w.sym && q0 == 0 && nq == N &&
                   (force ? strcmp(force, "sym") == 0 : sym_default);
  if (sym) {
    tsne_status st = sym_candidates(N, w, s);
    if (st != TSNE_OK) return st;
  } else {
    tsne_status st = launch_cand_tc(w.Xh, w.nrm, (int)N, (int)q0, (int)nq, Dp, Kc, w.buf, w.cand, w.slots, w.sync, s);
    if (st != TSNE_OK) return st;
  }
  w.path = sym ? 2 : 1;
  const char* fm = getenv("TSNE_KNN_FORCE_FALLBACK");      // test hook: every fm-th row
  const int force_mod = fm ? atoi(fm) : 0;
  k_rerank<<<(int)((nq + 7) / 8), kRR_Threads, 0, s>>>(X, (int)N, (int)q0, (int)nq, D, K, Kc,
                                                      w.cand, w.nrm, w.scale,
                                                     idx, d2, w.uncert, w.rows_bad, force_mod,
                                                     sym ? w.perm : nullptr, sym ? w.inv : nullptr,
                                                     w.amax, Dp);
  TSNE_LAUNCH_CHECK();
  // uncertified rows (D26): exact fp64 scan of the whole data set
  u64 h = 0;
  TSNE_CUDA_TRY(cudaMemcpyAsync(&h, w.uncert, sizeof(h), cudaMemcpyDeviceToHost, s));
  TSNE_CUDA_TRY(cudaStreamSynchronize(s));
  if (h > 0) {
    int32_t* rows = (int32_t*)malloc(h * sizeof(int32_t));
    if (!rows) {
      set_error("host allocation failed");
      return TSNE_ERR_CUDA;
    }
    cudaError_t e = cudaMemcpy(rows, w.rows_bad, h * sizeof(int32_t), cudaMemcpyDeviceToHost);
    tsne_status st = (e == cudaSuccess) ? exact_fallback(X, N, D, K, q0, rows, (int64_t)h, idx,
                                                          d2, w, s)
                                        : TSNE_ERR_CUDA;
    if (e != cudaSuccess) set_error("cudaMemcpy: %s", cudaGetErrorString(e));
    if (st == TSNE_OK) {
      e = cudaStreamSynchronize(s);     // `rows` is read by the async H2D copies above
      if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); st = TSNE_ERR_CUDA; }
    }
    free(rows);
    if (st != TSNE_OK) return st;
  }
  if (info) {
    info->rows_uncertified = (int64_t)h;
    info->candidates = Kc;
    info->gemm_path = w.path;
  }
  return TSNE_OK;
}

}  // namespace tsne
