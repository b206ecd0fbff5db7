// kl.cu -- the t-SNE cost of an embedding with the exact normaliser
// (SURVEY 8(f) f4): C = KL(P || Q) = sum_ij P_ij ln(P_ij / q_ij),
// q_ij = w_ij / Z, w_ij = (1 + |y_i - y_j|^2)^-1, Z = sum_{k != l} w_kl
// (Eq. 2 and the cost below it; Eq. 4).
//
// Z is the O(N^2) sum the Barnes-Hut traversal approximates; here it is taken
// exactly by a tiled pass over unordered pairs (Z = 2 sum_{k < l} w_kl):
// a block owns a 256-point row tile I and a run of column tiles J >= I staged
// in shared memory; each thread sums its point's w over a tile in fp32 (<= 256
// terms of size <= 1) and adds the tile sum to an fp64 accumulator; block and
// grid partials are reduced in a fixed order (deterministic).  The cost then
// needs one pass over the CSR:
//   KL = sum_{P_ij > 0} P_ij (ln P_ij + ln Z + ln(1 + |y_i - y_j|^2))
// in fp64 (a warp per row, fixed-order reductions).
#include <cmath>

#include "common.cuh"

namespace tsne {

constexpr int kZTile = 256;      // points per tile (= threads per block)
constexpr int kZRun = 32;        // column tiles per block
constexpr int kKlThreads = 256;

__device__ __forceinline__ float rcp_approx_kl(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ double block_sum_fixed(double v, double* s_red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_red[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_red[w];
  return t;   // valid in thread 0
}

// block b: row tile I = b / runs, column tiles J in [I + r*kZRun, ...) with
// r = b % runs; blocks whose run lies past the last tile exit at once.
__global__ void __launch_bounds__(kZTile)
k_z_pairs(const float2* __restrict__ Y, int N, int ntiles, int runs, double* __restrict__ part) {
  __shared__ float2 s_y[kZTile];
  __shared__ double s_red[kZTile / 32];
  const int I = blockIdx.x / runs, r = blockIdx.x % runs;
  const int J0 = I + r * kZRun;
  const int J1 = min(ntiles, J0 + kZRun);
  double acc = 0.0;
  if (J0 < ntiles) {
    const int i = I * kZTile + threadIdx.x;
    const float2 yi = (i < N) ? Y[i] : make_float2(0.f, 0.f);
    for (int J = J0; J < J1; ++J) {
      const int j = J * kZTile + threadIdx.x;
      __syncthreads();
      s_y[threadIdx.x] = (j < N) ? Y[j] : make_float2(0.f, 0.f);
      __syncthreads();
      const int jn = min(kZTile, N - J * kZTile);
      // diagonal tile: pairs with j > i only
      const int jb = (J == I) ? (int)threadIdx.x + 1 : 0;
      float s = 0.f;
      if (i < N) {
#pragma unroll 8
        for (int q = jb; q < jn; ++q) {
          const float dx = yi.x - s_y[q].x, dy = yi.y - s_y[q].y;
          s += rcp_approx_kl(fmaf(dy, dy, fmaf(dx, dx, 1.f)));
        }
      }
      acc += (double)s;
    }
  }
  const double t = block_sum_fixed(acc, s_red);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// one block: fixed-order sum of n partials, times `scale`, into out[0]
__global__ void __launch_bounds__(kKlThreads)
k_sum_parts(const double* __restrict__ part, int64_t n, double scale, double* __restrict__ out) {
  __shared__ double s_red[kKlThreads / 32];
  double a = 0.0;
  for (int64_t q = threadIdx.x; q < n; q += kKlThreads) a += part[q];
  const double t = block_sum_fixed(a, s_red);
  if (threadIdx.x == 0) out[0] = scale * t;
}

// warp per row: sum_e P (ln P + ln(1 + d^2)) + (sum_e P) ln Z, in fp64
__global__ void __launch_bounds__(kKlThreads)
k_kl_rows(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
          const float* __restrict__ val, const float2* __restrict__ Y, int N,
          const double* __restrict__ Zd, double* __restrict__ part) {
  __shared__ double s_red[kKlThreads / 32];
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * kKlThreads + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * kKlThreads) >> 5;
  const double lnZ = log(Zd[0]);
  double acc = 0.0;
  for (int i = warp; i < N; i += nwarps) {
    const float2 yi = Y[i];
    for (int64_t e = row_ptr[i] + lane; e < row_ptr[i + 1]; e += 32) {
      const double p = (double)val[e];
      if (!(p > 0.0)) continue;                  // zero entries contribute nothing (D20)
      const float2 yj = Y[col[e]];
      const double dx = (double)yi.x - (double)yj.x, dy = (double)yi.y - (double)yj.y;
      acc += p * (log(p) + lnZ + log1p(dx * dx + dy * dy));
    }
  }
  const double t = block_sum_fixed(acc, s_red);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

struct KlPlan {
  double* zpart = nullptr;
  double* kpart = nullptr;
  double* out = nullptr;   // [0] = Z, [1] = KL
  int64_t zblocks = 0;
  int kblocks = 0;
};

static size_t kl_plan(void* ws, int64_t N, KlPlan& p) {
  Carver c(ws);
  const int64_t ntiles = (N + kZTile - 1) / kZTile;
  const int64_t runs = (ntiles + kZRun - 1) / kZRun;
  p.zblocks = ntiles * runs;
  p.kblocks = 4 * kNumSMs;
  p.zpart = c.take<double>((size_t)p.zblocks);
  p.kpart = c.take<double>((size_t)p.kblocks);
  p.out = c.take<double>(2);
  return c.bytes();
}

size_t kl_workspace_size(int64_t N) {
  KlPlan p;
  return kl_plan(nullptr, N, p);
}

tsne_status kl_run(const int64_t* row_ptr, const int32_t* col, const float* val, int64_t N,
                   const float2* Y, void* ws, double* kl_out, double* Z_out, cudaStream_t s) {
  KlPlan p;
  kl_plan(ws, N, p);
  const int ntiles = (int)((N + kZTile - 1) / kZTile);
  const int runs = (ntiles + kZRun - 1) / kZRun;
  if (p.zblocks >= (int64_t(1) << 31)) {
    set_error("N too large for the exact-Z pass (%lld tile blocks)", (long long)p.zblocks);
    return TSNE_ERR_ARG;
  }
  k_z_pairs<<<(int)p.zblocks, kZTile, 0, s>>>(Y, (int)N, ntiles, runs, p.zpart);
  TSNE_LAUNCH_CHECK();
  k_sum_parts<<<1, kKlThreads, 0, s>>>(p.zpart, p.zblocks, 2.0, p.out);
  TSNE_LAUNCH_CHECK();
  k_kl_rows<<<p.kblocks, kKlThreads, 0, s>>>(row_ptr, col, val, Y, (int)N, p.out, p.kpart);
  TSNE_LAUNCH_CHECK();
  k_sum_parts<<<1, kKlThreads, 0, s>>>(p.kpart, p.kblocks, 1.0, p.out + 1);
  TSNE_LAUNCH_CHECK();
  double h[2];
  TSNE_CUDA_TRY(cudaMemcpyAsync(h, p.out, sizeof(h), cudaMemcpyDeviceToHost, s));
  TSNE_CUDA_TRY(cudaStreamSynchronize(s));
  *kl_out = h[1];
  if (Z_out) *Z_out = h[0];
  return TSNE_OK;
}

}  // namespace tsne
