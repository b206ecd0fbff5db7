// util.cu -- small helper kernels (input validation, fills).
#include "knn.cuh"

namespace tsne {

__global__ void k_check_finite(const float* __restrict__ X, int64_t n, int32_t* flag) {
  bool bad = false;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(X[e]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 1;
}

tsne_status check_finite(const float* X, int64_t n, int32_t* dflag, int32_t* hflag, cudaStream_t s) {
  TSNE_CUDA_TRY(cudaMemsetAsync(dflag, 0, sizeof(int32_t), s));
  k_check_finite<<<4 * kNumSMs, 256, 0, s>>>(X, n, dflag);
  TSNE_LAUNCH_CHECK();
  TSNE_CUDA_TRY(cudaMemcpyAsync(hflag, dflag, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  TSNE_CUDA_TRY(cudaStreamSynchronize(s));
  return TSNE_OK;
}

__global__ void k_fill(float* p, int64_t n, float v) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n) p[e] = v;
}

tsne_status fill_ones(float* p, int64_t n, cudaStream_t s) {
  k_fill<<<(int)((n + 255) / 256), 256, 0, s>>>(p, n, 1.f);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

}  // namespace tsne
