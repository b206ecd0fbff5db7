// knn_select.cuh -- per-row top-K' candidate selection used by both kNN
// candidate stages: (distance, index) packed into one order-preserving u64
// key (ties broken by the lower index, D18), per-row append buffers and
// warp-cooperative compaction.
//
// While the column sweep runs, a full buffer is shrunk by a pivot
// selection (32 sampled pivots sorted across lanes, a 33-bin histogram,
// keep every key <= the smallest pivot with >= K' keys below it); this keeps
// a superset of the K' best keys and lowers the threshold, at a fraction of
// the cost of sorting.  The final compaction sorts (warp bitonic in shared
// memory) and keeps exactly the K' smallest keys.
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

__device__ __forceinline__ u64 lds64(uint32_t a) {
  u64 v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts64(uint32_t a, u64 v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v));
}

// bitonic sort of P (power of 2) keys in shared memory at byte address `sa`
__device__ __forceinline__ void warp_bitonic_sort_s(uint32_t sa, int P, int lane) {
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = lane; t < (P >> 1); t += 32) {
        // t-th compare-exchange pair of this step: i has bit j clear
        const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const int l = i | j;
        const bool up = ((i & k) == 0);
        const u64 x = lds64(sa + 8u * i), y = lds64(sa + 8u * l);
        if ((x > y) == up) { sts64(sa + 8u * i, y); sts64(sa + 8u * l, x); }
      }
      __syncwarp();
    }
}

// Final compaction: sort the n keys of `rowbuf` (global) through shared
// scratch `sm` (>= next pow2 of n, >= 32 keys), keep the Kc smallest
// (written to `out`, and back to rowbuf).  Returns the kept count.
__device__ __forceinline__ int compact_keys(u64* __restrict__ rowbuf, int n, int Kc, u64* sm,
                                            int lane, u64* __restrict__ out, u64& tau) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sm);
  int P = 32;
  while (P < n) P <<= 1;
  for (int i = lane; i < P; i += 32) sts64(sa + 8u * i, (i < n) ? rowbuf[i] : kKeyMax);
  __syncwarp();
  warp_bitonic_sort_s(sa, P, lane);
  const int keep = n < Kc ? n : Kc;
  for (int i = lane; i < keep; i += 32) {
    const u64 v = lds64(sa + 8u * i);
    rowbuf[i] = v;
    if (out) out[i] = v;
  }
  tau = (keep == Kc) ? lds64(sa + 8u * (Kc - 1)) : kKeyMax;
  __syncwarp();
  return keep;
}

// Sweep-time compaction by pivot selection.  Keeps every key <= p where p is
// the smallest of 32 sampled pivots with count(<= p) >= Kc (so the K' best
// keys survive), compacting in place; tau <- p.  Falls back to the sorting
// compaction if the pivots cannot reduce the buffer below `limit`.  `scratch` is the
// shared sorting scratch (also used for pivots and the histogram).
__device__ __forceinline__ int reduce_keys(u64* __restrict__ rowbuf, int n, int Kc, int limit,
                                           u64* scratch, int lane, u64& tau) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(scratch);
  const uint32_t sh = sa + 8u * 32;          // 33 int bins after the 32 pivots
  // 1. 32 pivots sampled at evenly spaced positions, sorted across the lanes
  u64 pv = rowbuf[(int)(((long long)lane * n) >> 5)];
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const u64 o = __shfl_xor_sync(0xffffffffu, pv, j);
      const bool lower = (lane & j) == 0, asc = (lane & k) == 0;
      pv = (lower == asc) ? (pv < o ? pv : o) : (pv < o ? o : pv);
    }
  sts64(sa + 8u * lane, pv);
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(sh + 4u * lane), "r"(0));
  if (lane == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(sh + 128u), "r"(0));
  __syncwarp();
  // 2. histogram: bin(key) = number of pivots < key  (key <= piv[b] for b >= bin)
  for (int i = lane; i < n; i += 32) {
    const u64 key = rowbuf[i];
    int lo = 0, hi = 32;                      // first pivot >= key
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (lds64(sa + 8u * mid) < key) lo = mid + 1; else hi = mid;
    }
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(sh + 4u * lo));
  }
  __syncwarp();
  // 3. smallest m with count(<= piv[m]) = sum_{b <= m} hist[b] >= Kc
  int c;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(c) : "r"(sh + 4u * lane));
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, c, o);
    if (lane >= o) c += t;
  }
  const unsigned ok = __ballot_sync(0xffffffffu, c >= Kc);
  if (ok == 0) return compact_keys(rowbuf, n, Kc, scratch, lane, nullptr, tau);
  const int m = __ffs(ok) - 1;
  const int kept = __shfl_sync(0xffffffffu, c, m);
  // no reduction, or too many kept keys for the next tile: sort instead
  if (kept >= n || kept > limit) return compact_keys(rowbuf, n, Kc, scratch, lane, nullptr, tau);
  const u64 p = __shfl_sync(0xffffffffu, pv, m);
  // 4. in-place stable compaction of keys <= p (write position <= read position)
  int base = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const u64 key = (i < n) ? rowbuf[i] : kKeyMax;
    const bool keep = key <= p;
    const unsigned b = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) rowbuf[base + __popc(b & ((1u << lane) - 1u))] = key;
    base += __popc(b);
    __syncwarp();
  }
  tau = p;
  return base;
}

}  // namespace tsne
