// knn_tc.cu -- the kNN candidate stage on the 5th-generation tensor cores
// (U1; the paper's line 1 is FAISS, P:L151 -- this build's exact
// kNN needs the full N x N distance product, a dense contraction, so it runs
// on tcgen05).
//
// Persistent warp-specialised kernel, one CTA per SM (192 threads):
//   warp 0      TMA producer: 128x64 (queries) and 256x64 (points) fp16 tiles,
//               128-byte swizzle, 4-stage mbarrier ring (48 KB per stage)
//   warp 1      MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M=128 N=256
//               K=16, fp32 accumulators in TMEM, double-buffered (2 x 256 cols)
//   warps 2-5   epilogue: tcgen05.ld 32x32b (thread <-> query row), distance
//               |y|^2 - 2 x.y, per-row threshold filter, append to the row's
//               candidate buffer, warp pivot compaction (final: bitonic sort)
// The N x N matrix never exists; the only output is K' candidate keys / row.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "knn_select.cuh"
#include "knn_tc.cuh"
#include "tc_ptx.cuh"

namespace tsne {

constexpr int TC_BM = 128, TC_BN = 256, TC_BK = 64, TC_STAGES = 4;
constexpr int TC_CAP = 1024;                    // per-row candidate buffer
constexpr int TC_THREADS = 192;
constexpr int TC_SYNC_EVERY = 8;                // column tiles between CTA checkpoints
constexpr uint32_t TC_A_BYTES = TC_BM * TC_BK * 2;           // 16 KB
constexpr uint32_t TC_B_BYTES = TC_BN * TC_BK * 2;           // 32 KB
constexpr uint32_t TC_STAGE_BYTES = TC_A_BYTES + TC_B_BYTES;  // 48 KB
// instruction descriptor, kind::f16: D f32 (bits 4-5 = 1), A/B f16 (0), both
// K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28
constexpr uint32_t TC_IDESC = (1u << 4) | ((uint32_t)(TC_BN >> 3) << 17) |
                              ((uint32_t)(TC_BM >> 4) << 24);
constexpr size_t TC_SMEM = 1024 + TC_STAGES * TC_STAGE_BYTES + 256 + 4 * TC_CAP * 8;

__global__ void __launch_bounds__(TC_THREADS, 1)
k_cand_tc(const __grid_constant__ CUtensorMap tmap, const float* __restrict__ nrm, int N, int q0, int nq,
          int Dp, int Kc, u64* __restrict__ buf, u64* __restrict__ cand, unsigned* __restrict__ sync) {
  extern __shared__ unsigned char smraw[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + TC_STAGES * TC_STAGE_BYTES);
  uint64_t* empty = full + TC_STAGES;
  uint64_t* tfull = empty + TC_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  u64* sortbuf = reinterpret_cast<u64*>(base + TC_STAGES * TC_STAGE_BYTES + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = Dp / TC_BK;
  const int nrb = (nq + TC_BM - 1) / TC_BM, nct = (N + TC_BN - 1) / TC_BN;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {                                             // ---- TMA producer
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      const int ncp = (nct + TC_SYNC_EVERY - 1) / TC_SYNC_EVERY;
      int wave = 0;
      for (int rb = blockIdx.x; rb < nrb; rb += gridDim.x, ++wave)
        for (int ct = 0; ct < nct; ++ct) {
          if (sync && ct % TC_SYNC_EVERY == 0) {
            // keep all CTAs of this wave within 2 checkpoints of each other, so
            // the database tiles they stream stay L2-resident between CTAs
            const int members = min((int)gridDim.x, nrb - wave * (int)gridDim.x);
            const int cp = ct / TC_SYNC_EVERY;
            unsigned* base_c = sync + (size_t)wave * ncp;
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(base_c + cp) : "memory");
            if (cp >= 2) {
              for (int spin = 0; spin < (1 << 22); ++spin) {
                unsigned v;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(base_c + cp - 2) : "memory");
                if ((int)v >= members) break;
                __nanosleep(256);
              }
            }
          }
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_tx(&full[stage], TC_STAGE_BYTES);
            unsigned char* sa = base + stage * TC_STAGE_BYTES;
            tma_load_2d(sa, &tmap, &full[stage], kb * TC_BK, q0 + rb * TC_BM);
            tma_load_2d(sa + TC_A_BYTES, &tmap, &full[stage], kb * TC_BK, ct * TC_BN);
            tma_load_2d(sa + TC_A_BYTES + TC_A_BYTES, &tmap, &full[stage], kb * TC_BK,
                        ct * TC_BN + 128);
            if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
          }
        }
    }
  } else if (warp == 1) {
    {                                                            // ---- MMA issuer
      const uint64_t da0 = sw128_desc(smem_u32(base)), db0 = sw128_desc(smem_u32(base) + TC_A_BYTES);
      int stage = 0;
      uint32_t phase = 0, aphase = 0;
      int acc = 0;
      for (int rb = blockIdx.x; rb < nrb; rb += gridDim.x)
        for (int ct = 0; ct < nct; ++ct) {
          mbar_wait(&tempty[acc], aphase ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + (uint32_t)(acc * TC_BN);
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint64_t off = (uint64_t)((stage * TC_STAGE_BYTES) >> 4);
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < TC_BK / 16; ++k)
                mma_f16(d, da0 + off + 2 * k, db0 + off + 2 * k, TC_IDESC, (kb | k) != 0 ? 1u : 0u);
              mma_commit(&empty[stage]);
            }
            __syncwarp();
            if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
          }
          if (elect_one()) mma_commit(&tfull[acc]);
          __syncwarp();
          acc ^= 1;
          if (acc == 0) aphase ^= 1;
        }
    }
  } else {                                                        // ---- epilogue
    const int e = warp & 3;                 // TMEM lane quarter this warp may access
    const int rl = e * 32 + lane;           // local query row
    u64* mysort = sortbuf + (warp - 2) * TC_CAP;
    u64* rowbuf = buf + ((size_t)blockIdx.x * TC_BM + rl) * TC_CAP;
    int acc = 0;
    uint32_t aphase = 0;
    for (int rb = blockIdx.x; rb < nrb; rb += gridDim.x) {
      const int q = q0 + rb * TC_BM + rl;        // global query index
      const bool qok = rb * TC_BM + rl < nq;
      int cnt = 0;
      u64 tau = kKeyMax;
      for (int ct = 0; ct < nct; ++ct) {
        mbar_wait(&tfull[acc], aphase);
        tc_fence_after();
        const int c0 = ct * TC_BN;
        const uint32_t tbase = tmem + ((uint32_t)(e * 32) << 16) + (uint32_t)(acc * TC_BN);
#pragma unroll 1
        for (int ch = 0; ch < TC_BN / 32; ++ch) {
          const int j0 = c0 + ch * 32;
          const float nv = __ldg(nrm + j0 + lane);      // |y_j|^2 of this chunk, one per lane
          uint32_t r[32];
          tmem_ld32(tbase + ch * 32, r);
          // fast reject in fp32: only dist <= key_val(tau) can enter (ties by index)
          const float tf = (tau == kKeyMax) ? INFINITY : key_val(tau);
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const float dist = fmaf(-2.f, __uint_as_float(r[t]), __shfl_sync(0xffffffffu, nv, t));
            if (dist <= tf) {
              const int j = j0 + t;
              const u64 key = mkkey(dist, j);
              if (qok && j < N && j != q && key < tau) rowbuf[cnt++] = key;
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
        // compaction of this warp's rows that could overflow in the next tile
        unsigned need = __ballot_sync(0xffffffffu, cnt > TC_CAP - TC_BN);
        __syncwarp();
        while (need) {
          const int l = __ffs(need) - 1;
          need &= need - 1;
          const int n = __shfl_sync(0xffffffffu, cnt, l);
          u64* rb_l = buf + ((size_t)blockIdx.x * TC_BM + e * 32 + l) * TC_CAP;
          u64 t;
          const int keep = reduce_keys(rb_l, n, Kc, TC_CAP - TC_BN, mysort, lane, t);
          if (lane == l) { cnt = keep; tau = t; }
        }
      }
      // final compaction: the K' best keys of every row of this block
      __syncwarp();
      for (int l = 0; l < 32; ++l) {
        const int ql = rb * TC_BM + e * 32 + l;
        if (ql >= nq) break;
        const int n = __shfl_sync(0xffffffffu, cnt, l);
        u64* rb_l = buf + ((size_t)blockIdx.x * TC_BM + e * 32 + l) * TC_CAP;
        u64 t;
        int nn = n;
        if (nn > Kc + 64) nn = reduce_keys(rb_l, nn, Kc, 1 << 30, mysort, lane, t);
        compact_keys(rb_l, nn, Kc, mysort, lane, cand + (size_t)ql * Kc, t);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------- host
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool knn_tc_available() {
  static int ok = -1;
  if (ok < 0) {
    ok = 0;
    int dev = 0, major = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) == cudaSuccess &&
        major == 10) {
      cudaDriverEntryPointQueryResult q;
      void* fn = nullptr;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
              cudaSuccess &&
          q == cudaDriverEntryPointSuccess && fn) {
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        ok = 1;
      }
    }
  }
  return ok == 1;
}

size_t knn_tc_cap() { return TC_CAP; }

size_t knn_tc_sync_words(int64_t N, int64_t nq) {
  const int64_t nrb = (nq + TC_BM - 1) / TC_BM, nct = (N + TC_BN - 1) / TC_BN;
  const int64_t waves = (nrb + kNumSMs - 1) / kNumSMs;
  return (size_t)(waves * ((nct + TC_SYNC_EVERY - 1) / TC_SYNC_EVERY) + 1);
}

// 2-D fp16 tensor map over `rows` x Dp (row-major), box 64 x box_rows, 128-B swizzle
static tsne_status make_map(CUtensorMap& map, const __half* X, int64_t rows, int Dp, int box_rows) {
  if (!knn_tc_available()) {
    set_error("tcgen05 path unavailable (no sm_100 device or no cuTensorMapEncodeTiled)");
    return TSNE_ERR_CUDA;
  }
  cuuint64_t gdim[2] = {(cuuint64_t)Dp, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)Dp * 2};
  cuuint32_t box[2] = {TC_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(X), gdim,
                        gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return TSNE_ERR_CUDA;
  }
  return TSNE_OK;
}

tsne_status launch_cand_pair(const __half* A, int64_t rowsA, const __half* B, int64_t rowsB,
                             const float* nrmB, int nB, int q0, int nq, int Dp, int Kc,
                             unsigned long long* buf, unsigned long long* cand, int slots,
                             unsigned* sync, cudaStream_t s, int self_excl, int win_tiles,
                             const int32_t* qid) {
  CUtensorMap ma, mb;
  tsne_status st = make_map(ma, A, rowsA, Dp, 128);
  if (st != TSNE_OK) return st;
  st = make_map(mb, B, rowsB, Dp, knn_tc2_b_rows());
  if (st != TSNE_OK) return st;
  return launch_cand_tc2(ma, mb, nrmB, nB, q0, nq, Dp, Kc, buf, cand, slots, sync, s, self_excl,
                         win_tiles, qid);
}

tsne_status launch_sym(const __half* Xp, int64_t rows, const float* nrm, float* tau,
                       float* ntau, unsigned* cnt, unsigned long long* list, int cap, int N,
                       int Dp, unsigned* sync, cudaStream_t s) {
  CUtensorMap ma, mb;
  tsne_status st = make_map(ma, Xp, rows, Dp, 128);
  if (st != TSNE_OK) return st;
  st = make_map(mb, Xp, rows, Dp, 128);
  if (st != TSNE_OK) return st;
  return launch_cand_sym(ma, mb, nrm, tau, ntau, cnt, list, cap, N, Dp, sync, s);
}

tsne_status launch_cand_tc(const __half* Xh, const float* nrm, int N, int q0, int nq, int Dp, int Kc,
                           unsigned long long* buf, unsigned long long* cand, int slots,
                           unsigned* sync, cudaStream_t s) {
  if (!knn_tc_available()) {
    set_error("tcgen05 path unavailable (no sm_100 device or no cuTensorMapEncodeTiled)");
    return TSNE_ERR_CUDA;
  }
  CUtensorMap map;
  cuuint64_t gdim[2] = {(cuuint64_t)Dp, (cuuint64_t)N + 256};
  cuuint64_t gstride[1] = {(cuuint64_t)Dp * 2};
  cuuint32_t box[2] = {TC_BK, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(Xh), gdim,
                        gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return TSNE_ERR_CUDA;
  }
  // CTA-pair kernel by default; TSNE_KNN_PATH=tc1 selects the 1-CTA kernel
  const char* force = getenv("TSNE_KNN_PATH");
  if (!(force && strcmp(force, "tc1") == 0)) {
    CUtensorMap map_b;                                   // B half-tiles of the CTA pair
    cuuint32_t box_b[2] = {TC_BK, (cuuint32_t)knn_tc2_b_rows()};
    r = g_encode(&map_b, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(Xh), gdim,
                 gstride, box_b, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
      return TSNE_ERR_CUDA;
    }
    return launch_cand_tc2(map, map_b, nrm, N, q0, nq, Dp, Kc, buf, cand, slots, sync, s);
  }
  TSNE_CUDA_TRY(cudaFuncSetAttribute(k_cand_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)TC_SMEM));
  int nrb = (nq + TC_BM - 1) / TC_BM;
  int grid = nrb < kNumSMs ? nrb : kNumSMs;
  if (grid > slots) grid = slots;
  if (sync) TSNE_CUDA_TRY(cudaMemsetAsync(sync, 0, sizeof(unsigned) * knn_tc_sync_words(N, nq), s));
  k_cand_tc<<<grid, TC_THREADS, TC_SMEM, s>>>(map, nrm, N, q0, nq, Dp, Kc, buf, cand,
                                               grid == kNumSMs ? sync : nullptr);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

}  // namespace tsne
