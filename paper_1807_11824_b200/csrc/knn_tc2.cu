// knn_tc2.cu -- the kNN candidate stage on CTA pairs (tcgen05.mma.cta_group::2).
//
// Same algorithm as knn_tc.cu (expanded-form distances, per-row top-K'
// candidate buffers), but two CTAs on a TPC form a cluster and one elected
// thread of the leader issues M=256 x N=256 MMAs: each CTA stages only its
// own 128 query rows (A) and half of the 256-point column tile (B), and the
// tensor cores exchange the B halves.  Per SM this halves the shared-memory
// operand traffic of the 1-CTA M=128 kernel (TMA writes + MMA reads), which
// is what held that kernel near 50% tensor-pipe utilisation.
//
//   warp 0     TMA producer (both CTAs): A 128x64 + B 128x64 fp16 per stage,
//              128-byte swizzle; bytes complete on the LEADER's full barrier
//   warp 1     MMA issuer (leader only), fp32 accumulators: each CTA's TMEM
//              holds its 128 query rows x 256 columns, double-buffered
//   warps 2-5  epilogue (both CTAs): as knn_tc.cu; TMEM release arrives on the
//              leader's barrier (256 arrivals: both CTAs)
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "knn_select.cuh"
#include "knn_tc.cuh"
#include "tc_ptx.cuh"

namespace tsne {

constexpr int P_BM = 128, P_BN = 256, P_BK = 64, P_STAGES = 5;
constexpr int P_ACC = 2;                        // TMEM accumulator buffers (2 x 256 columns)
constexpr int P_CAP = 1024;
constexpr int P_THREADS = 192;
constexpr int P_SYNC_EVERY = 8;
constexpr uint32_t P_A_BYTES = P_BM * P_BK * 2;                 // 16 KB (this CTA's queries)
constexpr uint32_t P_B_BYTES = (P_BN / 2) * P_BK * 2;           // 16 KB (half the column tile)
constexpr uint32_t P_STAGE_BYTES = P_A_BYTES + P_B_BYTES;       // 32 KB
// kind::f16, D f32, A/B f16 K-major, N = 256, M = 256 (pair)
constexpr uint32_t P_IDESC = (1u << 4) | ((uint32_t)(P_BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
constexpr size_t P_SMEM = 1024 + P_STAGES * P_STAGE_BYTES + 256 + 4 * P_CAP * 8;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(P_THREADS, 1)
k_cand_tc2(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap tmap_b,
           const float* __restrict__ nrm, int N, int q0, int nq, int Dp,
           int Kc, u64* __restrict__ buf, u64* __restrict__ cand, unsigned* __restrict__ sync,
           int self_excl, int win_tiles, const int32_t* __restrict__ qid) {
  // rows: queries q0 .. q0+nq-1 of the A map; columns: the N points of the B
  // map with norms nrm (the same point set as the rows when self_excl != 0);
  // win_tiles > 0 restricts each CTA pair to win_tiles column tiles around
  // its own rows (the pilot of the symmetric search, knn_sym.cu)
  extern __shared__ unsigned char smraw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + P_STAGES * P_STAGE_BYTES);
  uint64_t* empty = full + P_STAGES;
  uint64_t* tfull = empty + P_STAGES;
  uint64_t* tempty = tfull + P_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + P_ACC);
  u64* sortbuf = reinterpret_cast<u64*>(base + P_STAGES * P_STAGE_BYTES + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npair_grid = gridDim.x >> 1;
  const int nkb = Dp / P_BK;
  const int nrb = (nq + P_BM - 1) / P_BM, npairs = (nrb + 1) / 2;
  const int nct_all = (N + P_BN - 1) / P_BN;
  const int nct = (win_tiles > 0 && win_tiles < nct_all) ? win_tiles : nct_all;
  // first column tile of pair pp: the window is centred on the pair's rows
  auto ct_first = [&](int pp) {
    if (nct == nct_all) return 0;
    const int c = (q0 + pp * 2 * P_BM) / P_BN - nct / 2;
    return c < 0 ? 0 : (c > nct_all - nct ? nct_all - nct : c);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < P_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < P_ACC; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 2 * 128); }
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
      const int ncp = (nct + P_SYNC_EVERY - 1) / P_SYNC_EVERY;
      int wave = 0;
      for (int pp = pair; pp < npairs; pp += npair_grid, ++wave) {
        const int rb = 2 * pp + (int)rank;
        const int ctf = ct_first(pp);
        for (int cs = 0; cs < nct; ++cs) {
          const int ct = ctf + cs;
          if (sync && ct % P_SYNC_EVERY == 0) {      // CTA lockstep for L2 reuse (knn_tc.cu)
            const int members = 2 * min(npair_grid, npairs - wave * npair_grid);
            const int cp = ct / P_SYNC_EVERY;
            unsigned* base_c = sync + (size_t)wave * ncp;
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
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            const uint32_t full_c = mapa_shared(smem_u32(&full[stage]), 0);
            if (leader) mbar_arrive_tx(&full[stage], 2 * P_STAGE_BYTES);
            unsigned char* sa = base + stage * P_STAGE_BYTES;
            tma_load_2d_pair(sa, &tmap, full_c, kb * P_BK, q0 + rb * P_BM);
            tma_load_2d_pair(sa + P_A_BYTES, &tmap_b, full_c, kb * P_BK, ct * P_BN + (int)rank * (P_BN / 2));
            if (++stage == P_STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {                                                // ---- MMA issuer
      // the whole warp walks the pipeline; one elected lane issues.  The
      // shared-memory descriptors are precomputed: a stage / K step only adds
      // its byte offset >> 4 to the start-address field.
      const uint64_t da0 = sw128_desc(smem_u32(base)), db0 = sw128_desc(smem_u32(base) + P_A_BYTES);
      int stage = 0;
      uint32_t phase = 0, aphase = 0;
      int acc = 0;
      for (int pp = pair; pp < npairs; pp += npair_grid)
        for (int cs = 0; cs < nct; ++cs) {
          mbar_wait(&tempty[acc], aphase ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(acc * P_BN);
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint64_t off = (uint64_t)((stage * P_STAGE_BYTES) >> 4);
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < P_BK / 16; ++k)
                mma_f16_pair(d, da0 + off + 2 * k, db0 + off + 2 * k, P_IDESC,
                             (kb | k) != 0 ? 1u : 0u);
              mma_commit_pair(&empty[stage]);
            }
            __syncwarp();
            if (++stage == P_STAGES) { stage = 0; phase ^= 1; }
          }
          if (elect_one()) mma_commit_pair(&tfull[acc]);
          __syncwarp();
          if (++acc == P_ACC) { acc = 0; aphase ^= 1; }
        }
    }
  } else {                                                        // ---- epilogue
    const int e = warp & 3;
    const int rl = e * 32 + lane;
    u64* mysort = sortbuf + (warp - 2) * P_CAP;
    u64* rowbuf = buf + ((size_t)blockIdx.x * P_BM + rl) * P_CAP;
    const uint32_t tempty_c0 = mapa_shared(smem_u32(&tempty[0]), 0);
    int acc = 0;
    uint32_t aphase = 0;
    for (int pp = pair; pp < npairs; pp += npair_grid) {
      const int rb = 2 * pp + (int)rank;
      const bool qok = rb * P_BM + rl < nq;
      const int q = qid ? (qok ? __ldg(qid + q0 + rb * P_BM + rl) : -1)
                        : q0 + rb * P_BM + rl;   // the query's point id
      int cnt = 0;
      u64 tau = kKeyMax;
      const int ctf = ct_first(pp);
      for (int cs = 0; cs < nct; ++cs) {
        const int ct = ctf + cs;
        mbar_wait(&tfull[acc], aphase);
        tc_fence_after();
        const int c0 = ct * P_BN;
        const uint32_t tbase = tmem + ((uint32_t)(e * 32) << 16) + (uint32_t)(acc * P_BN);
        const float tf = (tau == kKeyMax) ? INFINITY : key_val(tau);
#pragma unroll 1
        for (int ch = 0; ch < P_BN / 32; ch += 2) {    // 64 columns per TMEM wait
          const int j0 = c0 + ch * 32;
          uint32_t r[64];
          tmem_ld32_nowait(tbase + ch * 32, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          tmem_ld32_nowait(tbase + ch * 32 + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
          float nv[64];                                  // |y_j|^2: warp-uniform broadcast loads
          const float4* n4 = reinterpret_cast<const float4*>(nrm + j0);
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const float4 v = __ldg(n4 + u);
            nv[4 * u] = v.x; nv[4 * u + 1] = v.y; nv[4 * u + 2] = v.z; nv[4 * u + 3] = v.w;
          }
          tmem_wait_ld();
          // fast path: 2 instructions per distance (FFMA + FMNMX), no branches
          float mn = INFINITY;
#pragma unroll
          for (int t = 0; t < 64; ++t) mn = fminf(mn, fmaf(-2.f, __uint_as_float(r[t]), nv[t]));
          if (!__any_sync(0xffffffffu, qok && mn <= tf)) continue;
          // slow path: the columns holding a candidate for some lane of the warp
          uint64_t m = 0;
#pragma unroll
          for (int t = 0; t < 64; ++t)
            if (fmaf(-2.f, __uint_as_float(r[t]), nv[t]) <= tf) m |= 1ull << t;
          if (!qok) m = 0;
          const uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)m);
          const uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(m >> 32));
          uint64_t u = ((uint64_t)hi << 32) | lo;
          while (u) {                                    // warp-uniform loop over hit columns
            const int t = __ffsll((long long)u) - 1;
            u &= u - 1;
            const uint32_t v = tmem_ld1(tbase + ch * 32 + t);   // re-read the column from TMEM
            const float dist = fmaf(-2.f, __uint_as_float(v), __ldg(nrm + j0 + t));
            const int j = j0 + t;
            if ((m >> t) & 1) {
              const u64 key = mkkey(dist, j);
              if (j < N && (j != q || !self_excl) && key < tau) rowbuf[cnt++] = key;
            }
          }
        }
        tc_fence_before();
        if (leader) mbar_arrive(&tempty[acc]); else mbar_arrive_cluster(tempty_c0 + 8u * acc);
        if (++acc == P_ACC) { acc = 0; aphase ^= 1; }
        unsigned need = __ballot_sync(0xffffffffu, cnt > P_CAP - P_BN);
        __syncwarp();
        while (need) {
          const int l = __ffs(need) - 1;
          need &= need - 1;
          const int n = __shfl_sync(0xffffffffu, cnt, l);
          u64* rb_l = buf + ((size_t)blockIdx.x * P_BM + e * 32 + l) * P_CAP;
          u64 t;
          const int keep = reduce_keys(rb_l, n, Kc, P_CAP - P_BN, mysort, lane, t);
          if (lane == l) { cnt = keep; tau = t; }
        }
      }
      __syncwarp();
      for (int l = 0; l < 32; ++l) {
        const int ql = rb * P_BM + e * 32 + l;
        if (ql >= nq) break;
        const int n = __shfl_sync(0xffffffffu, cnt, l);
        u64* rb_l = buf + ((size_t)blockIdx.x * P_BM + e * 32 + l) * P_CAP;
        u64 t;
        int nn = n;
        if (nn > Kc + 64) nn = reduce_keys(rb_l, nn, Kc, 1 << 30, mysort, lane, t);
        compact_keys(rb_l, nn, Kc, mysort, lane, cand + (size_t)ql * Kc, t);
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

int knn_tc2_b_rows() { return P_BN / 2; }

size_t knn_tc2_sync_words(int64_t N, int64_t nq) {
  const int64_t nrb = (nq + P_BM - 1) / P_BM, npairs = (nrb + 1) / 2, nct = (N + P_BN - 1) / P_BN;
  const int64_t waves = (npairs + kNumSMs / 2 - 1) / (kNumSMs / 2);
  return (size_t)(waves * ((nct + P_SYNC_EVERY - 1) / P_SYNC_EVERY) + 1);
}

tsne_status launch_cand_tc2(const CUtensorMap& map, const CUtensorMap& map_b, const float* nrm, int N, int q0, int nq, int Dp, int Kc,
                            unsigned long long* buf, unsigned long long* cand, int slots,
                            unsigned* sync, cudaStream_t s, int self_excl, int win_tiles,
                            const int32_t* qid) {
  TSNE_CUDA_TRY(cudaFuncSetAttribute(k_cand_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)P_SMEM));
  const int nrb = (nq + P_BM - 1) / P_BM, npairs = (nrb + 1) / 2;
  int grid = 2 * (npairs < kNumSMs / 2 ? npairs : kNumSMs / 2);
  if (grid > slots) grid = slots & ~1;
  if (sync) TSNE_CUDA_TRY(cudaMemsetAsync(sync, 0, sizeof(unsigned) * knn_tc2_sync_words(N, nq), s));
  if (win_tiles > 0) sync = nullptr;          // pairs stream different tiles: no lockstep
  k_cand_tc2<<<grid, P_THREADS, P_SMEM, s>>>(map, map_b, nrm, N, q0, nq, Dp, Kc, buf, cand,
                                              grid == kNumSMs ? sync : nullptr,
                                              self_excl, win_tiles, qid);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

}  // namespace tsne
