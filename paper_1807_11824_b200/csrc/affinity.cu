// affinity.cu -- the sparse joint P (U2, U3).
//
// U2 (Eq. 1; D2, D3): one warp per row, each lane holding
// ceil(K/32) of the row's squared distances.  d'_j = d_j - min d; bisection
// with bracket doubling on beta from 1/mean(d') until
// |H(beta) - ln perp| <= 1e-10 max(1, ln perp), H(beta) = ln S + beta W / S,
// S = sum exp(-beta d'), W = sum d' exp(-beta d'), at most 200 steps; fp64.
// Degenerate rows (all d' = 0, or >= perp ties at the minimum) are uniform
// (over K, resp. over the ties) and counted.
//
// U3: every directed edge (i, j, p_{j|i}) is emitted twice,
// as (i, j) and (j, i); a radix sort by (row, col) brings the (at most two)
// contributions of an unordered pair together; their sum a + b is
// commutative, so both triangles receive bitwise identical values
// (a + b) / 2N, rounded to fp32 once.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "affinity.cuh"

namespace tsne {

typedef unsigned long long u64;

static int bits_for(int64_t n) {
  int b = 1;
  while ((int64_t(1) << b) < n) ++b;
  return b;
}

void carve_p(Carver& c, PWS& w, int64_t N, int32_t K) {
  w.N = N;
  w.K = K;
  w.nb = bits_for(N);
  const int64_t E = 2 * N * (int64_t)K;
  w.pc = c.take<double>(N * K);
  w.beta = c.take<double>(N);
  w.ndeg = c.take<u64>(2);
  w.ka = c.take<u64>(E);
  w.kb = c.take<u64>(E);
  w.va = c.take<double>(E);
  w.vb = c.take<double>(E);
  size_t sb = 0, cb = 0;
  cub::DoubleBuffer<u64> dk(nullptr, nullptr);
  cub::DoubleBuffer<double> dv(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, sb, dk, dv, (int)E, 0, 2 * w.nb);
  cub::DeviceScan::ExclusiveSum(nullptr, cb, (int32_t*)nullptr, (int32_t*)nullptr, (int)(E + 1));
  w.sort_tmp = c.take<char>(sb);
  w.sort_tmp_bytes = sb;
  w.head = c.take<int32_t>(E + 1);
  w.pos = c.take<int32_t>(E + 1);
  w.scan_tmp = c.take<char>(cb);
  w.scan_tmp_bytes = cb;
}

constexpr int kMaxPer = 6;  // ceil(192 / 32)

__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ void entropy_terms(const double* dp, int n, double beta, double& S,
                                              double& W) {
  double s = 0.0, w = 0.0;
#pragma unroll
  for (int m = 0; m < kMaxPer; ++m) {
    if (m < n) {
      const double e = exp(-beta * dp[m]);
      s += e;
      w += dp[m] * e;
    }
  }
  S = warp_sum(s);
  W = warp_sum(w);
}

__global__ void k_bisect(const double* __restrict__ d2, int64_t N, int K, double perplexity,
                         double* __restrict__ pc, double* __restrict__ beta_out,
                         u64* __restrict__ ndeg) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (i >= N) return;
  const double* di = d2 + i * K;
  double dp[kMaxPer];
  int n = 0;
  double dmin = INFINITY;
#pragma unroll
  for (int m = 0; m < kMaxPer; ++m) {
    const int k = lane + 32 * m;
    dp[m] = (k < K) ? di[k] : INFINITY;
    if (k < K) { n = m + 1; dmin = fmin(dmin, dp[m]); }
  }
  dmin = warp_min_d(dmin);
  double sum = 0.0;
  int ties = 0;
#pragma unroll
  for (int m = 0; m < kMaxPer; ++m)
    if (m < n) {
      dp[m] -= dmin;
      sum += dp[m];
      ties += (dp[m] == 0.0);
    }
  sum = warp_sum(sum);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ties += __shfl_xor_sync(0xffffffffu, ties, o);
  const double mean = sum / (double)K;
  double beta;
  bool deg = false;
  double* pi = pc + i * K;
  if (mean == 0.0) {
    beta = 0.0;
    deg = true;
#pragma unroll
    for (int m = 0; m < kMaxPer; ++m)
      if (m < n) pi[lane + 32 * m] = 1.0 / (double)K;
  } else if ((double)ties >= perplexity) {
    beta = INFINITY;
    deg = true;
#pragma unroll
    for (int m = 0; m < kMaxPer; ++m)
      if (m < n) pi[lane + 32 * m] = (dp[m] == 0.0) ? 1.0 / (double)ties : 0.0;
  } else {
    const double target = log(perplexity);
    const double tol = 1e-10 * (target > 1.0 ? target : 1.0);
    double lo = 0.0, hi = INFINITY;
    beta = 1.0 / mean;
    double S, W;
    for (int it = 0; it < 200; ++it) {
      entropy_terms(dp, n, beta, S, W);
      const double H = log(S) + beta * W / S;
      if (fabs(H - target) <= tol) break;
      if (H > target) {
        lo = beta;
        beta = isinf(hi) ? 2.0 * beta : 0.5 * (lo + hi);
      } else {
        hi = beta;
        beta = 0.5 * (lo + hi);
      }
    }
    entropy_terms(dp, n, beta, S, W);
#pragma unroll
    for (int m = 0; m < kMaxPer; ++m)
      if (m < n) pi[lane + 32 * m] = exp(-beta * dp[m]) / S;
  }
  if (lane == 0) {
    if (beta_out) beta_out[i] = beta;
    if (deg) atomicAdd(ndeg, 1ull);
  }
}

__global__ void k_emit(const int32_t* __restrict__ idx, const double* __restrict__ pc, int64_t NK,
                       int K, int nb, u64* __restrict__ keys, double* __restrict__ vals) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= NK) return;
  const u64 i = (u64)(e / K);
  const u64 j = (u64)(uint32_t)idx[e];
  const double p = pc[e];
  keys[2 * e] = (i << nb) | j;
  vals[2 * e] = p;
  keys[2 * e + 1] = (j << nb) | i;
  vals[2 * e + 1] = p;
}

__global__ void k_heads(const u64* __restrict__ keys, int64_t E, int32_t* __restrict__ head) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e > E) return;
  head[e] = (e < E && (e == 0 || keys[e] != keys[e - 1])) ? 1 : 0;
}

__global__ void k_write_csr(const u64* __restrict__ keys, const double* __restrict__ vals,
                            int64_t E, int nb, int64_t N, const int32_t* __restrict__ head,
                            const int32_t* __restrict__ pos, int64_t* __restrict__ row_ptr,
                            int32_t* __restrict__ col, float* __restrict__ val) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e > E) return;
  if (e == E) { row_ptr[N] = pos[E]; return; }
  if (!head[e]) return;
  const u64 k = keys[e];
  const int64_t p = pos[e];
  const u64 mask = (1ull << nb) - 1ull;
  double s = vals[e];
  if (e + 1 < E && keys[e + 1] == k) s += vals[e + 1];   // the pair's other direction
  col[p] = (int32_t)(k & mask);
  val[p] = (float)(s / (2.0 * (double)N));
  const int64_t r = (int64_t)(k >> nb);
  if (e == 0 || (int64_t)(keys[e - 1] >> nb) != r) row_ptr[r] = p;
}

tsne_status run_compute_p(const int32_t* idx, const double* d2, int64_t N, int32_t K,
                          float perplexity, int64_t* row_ptr, int32_t* col, float* val,
                          int64_t* nnz_host, double* beta_out, PWS& w, int64_t* ndeg_host,
                          cudaStream_t s) {
  const int64_t NK = N * (int64_t)K, E = 2 * NK;
  TSNE_CUDA_TRY(cudaMemsetAsync(w.ndeg, 0, sizeof(u64), s));
  k_bisect<<<(int)((N * 32 + 255) / 256), 256, 0, s>>>(d2, N, K, (double)perplexity, w.pc,
                                                       beta_out ? beta_out : w.beta, w.ndeg);
  TSNE_LAUNCH_CHECK();
  k_emit<<<(int)((NK + 255) / 256), 256, 0, s>>>(idx, w.pc, NK, K, w.nb, w.ka, w.va);
  TSNE_LAUNCH_CHECK();
  cub::DoubleBuffer<u64> dk(w.ka, w.kb);
  cub::DoubleBuffer<double> dv(w.va, w.vb);
  size_t sb = w.sort_tmp_bytes;
  TSNE_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_tmp, sb, dk, dv, (int)E, 0, 2 * w.nb, s));
  k_heads<<<(int)((E + 256) / 256), 256, 0, s>>>(dk.Current(), E, w.head);
  TSNE_LAUNCH_CHECK();
  size_t cb = w.scan_tmp_bytes;
  TSNE_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w.scan_tmp, cb, w.head, w.pos, (int)(E + 1), s));
  k_write_csr<<<(int)((E + 256) / 256), 256, 0, s>>>(dk.Current(), dv.Current(), E, w.nb, N,
                                                     w.head, w.pos, row_ptr, col, val);
  TSNE_LAUNCH_CHECK();
  int64_t nnz = 0;
  u64 nd = 0;
  TSNE_CUDA_TRY(cudaMemcpyAsync(&nnz, row_ptr + N, sizeof(nnz), cudaMemcpyDeviceToHost, s));
  TSNE_CUDA_TRY(cudaMemcpyAsync(&nd, w.ndeg, sizeof(nd), cudaMemcpyDeviceToHost, s));
  TSNE_CUDA_TRY(cudaStreamSynchronize(s));
  *nnz_host = nnz;
  if (ndeg_host) *ndeg_host = (int64_t)nd;
  return TSNE_OK;
}

}  // namespace tsne
