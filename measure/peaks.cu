// measure/peaks.cu -- microbenchmarks of the B200 peaks this build quotes
// fractions of, besides the driver's MEASURED_PEAKS.json (HBM copy, bf16 GEMM):
//   l2_read   L2 -> SM read bandwidth (ld.global.cg, 16 B per load, a 48 MB
//             buffer that stays L2-resident after the first pass)
//   l1_read   L1 hit bandwidth (ld.global.ca over a 64 KB per-CTA slice)
//   fp64_fma  DFMA throughput (8 independent chains per thread)
//   fp32_fma  FFMA throughput
//   mufu_rcp  MUFU.RCP throughput (rcp.approx.ftz.f32)
// Built and run by measure/peaks.py (CUDA events, best of several launches).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void k_l2_read(const float4* __restrict__ a, size_t n4, int reps, float* out) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
      float4 v;
      asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a + i));
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 1234.5f) out[0] = acc;
}

__global__ void k_l1_read(const float4* __restrict__ a, int slice4, int reps, float* out) {
  float acc = 0.f;
  const float4* p = a + (size_t)blockIdx.x * slice4;
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x; i < slice4; i += blockDim.x) {
      float4 v;
      asm volatile("ld.global.ca.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p + i));
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 1234.5f) out[0] = acc;
}

__global__ void k_fp64(int iters, double* out) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-9 + k;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1234.5) out[0] = s;
}

__global__ void k_fp32(int iters, float* out) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-9f + k;
  const float b = 0.999999f, c = 1e-7f;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], b, c);
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_rcp(int iters, float* out) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.f + threadIdx.x * 1e-6f + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float r;
      asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a[k]));
      a[k] = r + 1.0f;       // a dependent chain the compiler cannot fold
    }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1234.5f) out[0] = s;
}

template <class F>
static float best_ms(F launch, int trials = 7) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int t = 0; t < trials; ++t) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 64);
  // L2: 48 MB buffer, 8 passes per launch
  const size_t l2_bytes = 48ull << 20, n4 = l2_bytes / 16;
  float4* buf;
  cudaMalloc(&buf, l2_bytes);
  cudaMemset(buf, 0, l2_bytes);
  const int l2_reps = 8;
  float ms = best_ms([&] { k_l2_read<<<sms * 4, 512>>>(buf, n4, l2_reps, out); });
  printf("{\"sms\": %d, \"l2_read_gbs\": %.1f, \"l2_bytes\": %zu", sms,
         (double)l2_bytes * l2_reps / (ms * 1e-3) / 1e9, l2_bytes);
  // L1: 64 KB per CTA, one CTA per SM... 4 per SM
  const int slice4 = (64 << 10) / 16, l1_reps = 64;
  ms = best_ms([&] { k_l1_read<<<sms * 4, 512>>>(buf, slice4, l1_reps, out); });
  printf(", \"l1_read_gbs\": %.1f", (double)sms * 4 * (64 << 10) * l1_reps / (ms * 1e-3) / 1e9);
  const int iters = 4096;
  const double thr = (double)sms * 8 * 256;
  ms = best_ms([&] { k_fp64<<<sms * 8, 256>>>(iters, (double*)out); });
  printf(", \"fp64_fma_tflops\": %.2f", thr * iters * 8 * 2 / (ms * 1e-3) / 1e12);
  ms = best_ms([&] { k_fp32<<<sms * 8, 256>>>(iters, out); });
  printf(", \"fp32_fma_tflops\": %.2f", thr * iters * 8 * 2 / (ms * 1e-3) / 1e12);
  ms = best_ms([&] { k_rcp<<<sms * 8, 256>>>(iters, out); });
  printf(", \"mufu_rcp_gops\": %.1f}\n", thr * iters * 8 / (ms * 1e-3) / 1e9);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "%s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
