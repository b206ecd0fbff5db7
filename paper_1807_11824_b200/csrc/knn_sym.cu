// knn_sym.cu -- the kNN candidate stage exploiting the symmetry of the
// distance matrix: every unordered pair of 256-point super-blocks {b, c} is
// multiplied ONCE (tcgen05 CTA pair, M = 256 rows of b, N = 256 columns of
// c) and the tile feeds both the rows of b (candidates j in c) and the rows of
// c (candidates i in b) -- half the tensor work of the row-by-row sweep.
//
// Selection uses static per-point thresholds instead of running top-K'
// buffers, because a point's candidates now arrive from many CTAs:
//   tau_i  = the K'-th smallest key of point i found by a cheap windowed
//            pilot sweep over the points near i in a locality order (an upper
//            bound of the K'-th smallest key over all points), plus a slack
//            that covers the rounding differences between the two sweeps;
//   list_i = every j with key_i(j) <= tau_i, appended through a global
//            atomic counter (capacity cap per point; an overflowing or
//            underfilled point is redone by the exact fallback).
// A key is (|x_j|^2 - 2 x_i.x_j, j) for point i -- the owner's own norm is
// dropped, as in the row sweep (knn_tc2.cu), so the keys of one list are
// comparable; the K' smallest of the list are then exactly the K' smallest
// keys over all points (every key <= tau_i is in the list and at least K'
// are).  The fp64 re-rank and its certificate (D26) follow unchanged.
//
// Tile schedule: the S super-blocks form waves of P consecutive super-blocks
// (P = CTA pairs in the grid; pair p owns super-row b = kP + p of wave k).
// Wave k takes the column waves l = k, k+1, ..., k + nw/2 (mod nw) -- for
// even nw the last one only if k < nw/2 -- and within its own wave only the
// columns c >= b, so each unordered pair {b, c} is computed exactly once.  At
// every step all pairs of a wave multiply the SAME column super-block, so the
// lockstep checkpoints keep it L2-resident for all of them (knn_tc.cu).  On
// the diagonal tile only the row side is used (it holds both orientations).
//
//   warp 0     TMA producer (both CTAs), as knn_tc2.cu
//   warp 1     MMA issuer (leader), as knn_tc2.cu
//   warps 2-5  epilogue: per 64 columns, a branch-free filter (2 FFMA + 2
//              FMNMX per distance); hit columns are re-read from TMEM and
//              appended to the row's / the column's list
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "knn_select.cuh"
#include "knn_tc.cuh"
#include "tc_ptx.cuh"

namespace tsne {

constexpr int S_BM = 128, S_BN = 256, S_BK = 64, S_STAGES = 6;
constexpr int S_ACC = 2;
constexpr int S_THREADS = 192;
constexpr int S_SYNC_EVERY = 8;
constexpr uint32_t S_A_BYTES = S_BM * S_BK * 2;
constexpr uint32_t S_B_BYTES = (S_BN / 2) * S_BK * 2;
constexpr uint32_t S_STAGE_BYTES = S_A_BYTES + S_B_BYTES;
constexpr uint32_t S_IDESC = (1u << 4) | ((uint32_t)(S_BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
constexpr size_t S_SMEM = 1024 + S_STAGES * S_STAGE_BYTES + 256;

struct SymArgs {
  const float* nrm;     // |x_h|^2 per point (padded with zeros)
  float* tau;           // per point threshold; -inf once the list overflowed
  float* ntau;          // -(tau + slack2): the column-side fast filter (+inf: off)
  unsigned* cnt;        // per point list length (atomic)
  u64* list;            // per point list, cap keys each
  int N, Dp, cap;
  unsigned* sync;       // lockstep checkpoints (nullable)
};

__device__ __forceinline__ int sym_steps(int S, int P) {
  const int nw = (S + P - 1) / P;
  return (nw / 2 + 1) * P;
}
// column super-block of step s for super-row b, or -1 if the step is skipped
__device__ __forceinline__ int sym_col(int b, int s, int S, int P) {
  const int nw = (S + P - 1) / P;
  const int k = b / P, d = s / P, cc = s % P;
  if ((nw & 1) == 0 && d == nw / 2 && k >= nw / 2) return -1;
  int l = k + d;
  if (l >= nw) l -= nw;
  const int c = l * P + cc;
  if (c >= S || (d == 0 && c < b)) return -1;
  return c;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(S_THREADS, 1)
k_cand_sym(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap tmap_b,
           const __grid_constant__ SymArgs a) {
  extern __shared__ unsigned char smraw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + S_STAGES * S_STAGE_BYTES);
  uint64_t* empty = full + S_STAGES;
  uint64_t* tfull = empty + S_STAGES;
  uint64_t* tempty = tfull + S_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + S_ACC);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npair_grid = gridDim.x >> 1;
  const int nkb = a.Dp / S_BK;
  const int S = (a.N + S_BN - 1) / S_BN;                // super-blocks (256 points)
  const int nsteps = sym_steps(S, npair_grid);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int q = 0; q < S_ACC; ++q) { mbar_init(&tfull[q], 1); mbar_init(&tempty[q], 2 * 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {                                             // ---- TMA producer
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_b)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      const int ncp = (nsteps + S_SYNC_EVERY - 1) / S_SYNC_EVERY;
      int wave = 0;
      for (int b = pair; b < S; b += npair_grid, ++wave) {
        for (int s = 0; s < nsteps; ++s) {
          if (a.sync && s % S_SYNC_EVERY == 0) {       // lockstep (knn_tc.cu): L2 reuse of c tiles
            const int members = 2 * min(npair_grid, S - wave * npair_grid);
            const int cp = s / S_SYNC_EVERY;
            unsigned* base_c = a.sync + (size_t)wave * ncp;
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(base_c + cp) : "memory");
            if (cp >= 2) {
              for (int spin = 0; spin < (1 << 22); ++spin) {
                unsigned v;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(base_c + cp - 2)
                             : "memory");
                if ((int)v >= members) break;
                __nanosleep(256);
              }
            }
          }
          const int c = sym_col(b, s, S, npair_grid);
          if (c < 0) continue;
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            const uint32_t full_c = mapa_shared(smem_u32(&full[stage]), 0);
            if (leader) mbar_arrive_tx(&full[stage], 2 * S_STAGE_BYTES);
            unsigned char* sa = base + stage * S_STAGE_BYTES;
            tma_load_2d_pair(sa, &tmap, full_c, kb * S_BK, b * S_BN + (int)rank * S_BM);
            tma_load_2d_pair(sa + S_A_BYTES, &tmap_b, full_c, kb * S_BK,
                             c * S_BN + (int)rank * (S_BN / 2));
            if (++stage == S_STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {                                                // ---- MMA issuer
      const uint64_t da0 = sw128_desc(smem_u32(base)), db0 = sw128_desc(smem_u32(base) + S_A_BYTES);
      int stage = 0;
      uint32_t phase = 0, aphase = 0;
      int acc = 0;
      for (int b = pair; b < S; b += npair_grid)
        for (int s = 0; s < nsteps; ++s) {
          if (sym_col(b, s, S, npair_grid) < 0) continue;
          mbar_wait(&tempty[acc], aphase ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(acc * S_BN);
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint64_t off = (uint64_t)((stage * S_STAGE_BYTES) >> 4);
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < S_BK / 16; ++k)
                mma_f16_pair(d, da0 + off + 2 * k, db0 + off + 2 * k, S_IDESC,
                             (kb | k) != 0 ? 1u : 0u);
              mma_commit_pair(&empty[stage]);
            }
            __syncwarp();
            if (++stage == S_STAGES) { stage = 0; phase ^= 1; }
          }
          if (elect_one()) mma_commit_pair(&tfull[acc]);
          __syncwarp();
          if (++acc == S_ACC) { acc = 0; aphase ^= 1; }
        }
    }
  } else {                                                        // ---- epilogue
    const int e = warp & 3;
    const int rl = e * 32 + lane;
    const uint32_t tempty_c0 = mapa_shared(smem_u32(&tempty[0]), 0);
    int acc = 0;
    uint32_t aphase = 0;
    for (int b = pair; b < S; b += npair_grid) {
      const int i = b * S_BN + (int)rank * S_BM + rl;            // this lane's row point
      const bool iok = i < a.N;
      float tau_i = -INFINITY;                                    // row side: key <= tau_i
      const float nrm_i = iok ? __ldg(a.nrm + i) : 0.f;
      const float nnrm_i = -nrm_i;                               // column side fast filter
      u64* list_i = a.list + (size_t)(iok ? i : 0) * a.cap;
      for (int s = 0; s < nsteps; ++s) {
        const int c = sym_col(b, s, S, npair_grid);
        if (c < 0) continue;
        const bool col_side = c != b;
        // re-read per tile: an overflowing list switches its point off (-inf)
        tau_i = iok ? __ldcg(a.tau + i) : -INFINITY;
        mbar_wait(&tfull[acc], aphase);
        tc_fence_after();
        const uint32_t tbase = tmem + ((uint32_t)(e * 32) << 16) + (uint32_t)(acc * S_BN);
#pragma unroll 1
        for (int ch = 0; ch < S_BN / 32; ch += 2) {              // 64 columns per TMEM wait
          const int j0 = c * S_BN + ch * 32;
          uint32_t r[64];
          tmem_ld32_nowait(tbase + ch * 32, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          tmem_ld32_nowait(tbase + ch * 32 + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
          float nv[64], nt[64];
          const float4* n4 = reinterpret_cast<const float4*>(a.nrm + j0);
          const float4* t4 = reinterpret_cast<const float4*>(a.ntau + j0);
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const float4 v = __ldg(n4 + u);
            nv[4 * u] = v.x; nv[4 * u + 1] = v.y; nv[4 * u + 2] = v.z; nv[4 * u + 3] = v.w;
            const float4 w = __ldcg(t4 + u);
            nt[4 * u] = w.x; nt[4 * u + 1] = w.y; nt[4 * u + 2] = w.z; nt[4 * u + 3] = w.w;
          }
          tmem_wait_ld();
          float mr = INFINITY, mc = INFINITY;
#pragma unroll
          for (int t = 0; t < 64; ++t) {
            const float rv = __uint_as_float(r[t]);
            mr = fminf(mr, fmaf(-2.f, rv, nv[t]));
            mc = fminf(mc, fmaf(-2.f, rv, nt[t]));
          }
          const bool hit = iok && (mr <= tau_i || (col_side && mc <= nnrm_i));
          if (!__any_sync(0xffffffffu, hit)) continue;
          // slow path: exact conditions per column (the keys' own arithmetic)
          uint64_t mrow = 0, mcol = 0;
          if (iok) {
#pragma unroll
            for (int t = 0; t < 64; ++t) {
              const float rv = __uint_as_float(r[t]);
              if (fmaf(-2.f, rv, nv[t]) <= tau_i) mrow |= 1ull << t;
              if (col_side && fmaf(-2.f, rv, nrm_i) <= -nt[t]) mcol |= 1ull << t;
            }
          }
          const uint64_t m = mrow | mcol;
          const uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)m);
          const uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(m >> 32));
          uint64_t u = ((uint64_t)hi << 32) | lo;
          while (u) {                                            // warp-uniform
            const int t = __ffsll((long long)u) - 1;
            u &= u - 1;
            const uint32_t v = tmem_ld1(tbase + ch * 32 + t);
            const int j = j0 + t;
            if (j >= a.N || j == i) continue;
            const float rv = __uint_as_float(v);
            if ((mrow >> t) & 1) {                               // j is a candidate of i
              const float d = fmaf(-2.f, rv, __ldg(a.nrm + j));
              if (d <= tau_i) {
                const unsigned pos = atomicAdd(a.cnt + i, 1u);
                if (pos < (unsigned)a.cap) list_i[pos] = mkkey(d, j);
                else if (pos == (unsigned)a.cap) { a.tau[i] = -INFINITY; a.ntau[i] = INFINITY; }
              }
            }
            if ((mcol >> t) & 1) {                               // i is a candidate of j
              const float d = fmaf(-2.f, rv, nrm_i);
              if (d <= __ldcg(a.tau + j)) {
                const unsigned pos = atomicAdd(a.cnt + j, 1u);
                if (pos < (unsigned)a.cap) a.list[(size_t)j * a.cap + pos] = mkkey(d, i);
                else if (pos == (unsigned)a.cap) { a.tau[j] = -INFINITY; a.ntau[j] = INFINITY; }
              }
            }
          }
        }
        tc_fence_before();
        if (leader) mbar_arrive(&tempty[acc]); else mbar_arrive_cluster(tempty_c0 + 8u * acc);
        if (++acc == S_ACC) { acc = 0; aphase ^= 1; }
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

size_t knn_sym_sync_words(int64_t N) {
  const int64_t S = (N + S_BN - 1) / S_BN, P = kNumSMs / 2;
  const int64_t waves = (S + P - 1) / P, nsteps = (waves / 2 + 1) * P;
  return (size_t)(waves * ((nsteps + S_SYNC_EVERY - 1) / S_SYNC_EVERY) + 1);
}

tsne_status launch_cand_sym(const CUtensorMap& map, const CUtensorMap& map_b, const float* nrm,
                            float* tau, float* ntau, unsigned* cnt,
                            unsigned long long* list, int cap, int N, int Dp, unsigned* sync,
                            cudaStream_t s) {
  TSNE_CUDA_TRY(cudaFuncSetAttribute(k_cand_sym, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)S_SMEM));
  const int S = (N + S_BN - 1) / S_BN;
  const int grid = 2 * (S < kNumSMs / 2 ? S : kNumSMs / 2);
  if (sync) TSNE_CUDA_TRY(cudaMemsetAsync(sync, 0, sizeof(unsigned) * knn_sym_sync_words(N), s));
  SymArgs a{nrm, tau, ntau, cnt, list, N, Dp, cap, grid == kNumSMs ? sync : nullptr};
  k_cand_sym<<<grid, S_THREADS, S_SMEM, s>>>(map, map_b, a);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

}  // namespace tsne
