// knn_select.cuh -- per-row top-K' candidate selection used by both kNN
// candidate stages: (distance, index) packed into one order-preserving u64
// key (ties broken by the lower index, D18), per-row append buffers and a
// warp bitonic-sort compaction.
#pragma once
#include "common.cuh"

namespace tsne {

typedef unsigned long long u64;
constexpr u64 kKeyMax = ~0ull;

__device__ __forceinline__ u64 mkkey(float a, int j) {
  unsigned u = __float_as_uint(a);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((u64)u << 32) | (unsigned)j;
}
__device__ __forceinline__ float key_val(u64 k) {
  unsigned u = (unsigned)(k >> 32);
  u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
  return __uint_as_float(u);
}
__device__ __forceinline__ int key_idx(u64 k) { return (int)(unsigned)(k & 0xffffffffull); }

__device__ __forceinline__ void warp_bitonic_sort(u64* a, int P, int lane) {
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < P; i += 32) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = ((i & k) == 0);
          const u64 x = a[i], y = a[l];
          if ((x > y) == up) { a[i] = y; a[l] = x; }
        }
      }
      __syncwarp();
    }
}

// Warp-cooperative: sort the n keys of `rowbuf` (global) through the smem
// scratch `sm`, keep the Kc smallest (written back, and to `out` if given).
// Returns the kept count; `tau` = the Kc-th smallest key (or kKeyMax).
__device__ __forceinline__ int compact_keys(u64* __restrict__ rowbuf, int n, int Kc, u64* sm,
                                            int lane, u64* __restrict__ out, u64& tau) {
  int P = 32;
  while (P < n) P <<= 1;
  for (int i = lane; i < P; i += 32) sm[i] = (i < n) ? rowbuf[i] : kKeyMax;
  __syncwarp();
  warp_bitonic_sort(sm, P, lane);
  const int keep = n < Kc ? n : Kc;
  for (int i = lane; i < keep; i += 32) {
    rowbuf[i] = sm[i];
    if (out) out[i] = sm[i];
  }
  tau = (keep == Kc) ? sm[Kc - 1] : kKeyMax;
  __syncwarp();
  return keep;
}

}  // namespace tsne
