// knn_tc.cu -- host side of the kNN candidate stage on the 5th-generation
// tensor cores (U1; the paper's line 1 is FAISS, P:L151 -- this
// build's exact kNN needs the full N x N distance product, a dense
// contraction, so it runs on tcgen05): TMA tensor maps (fp16, 128-byte
// swizzle) and the launches of the CTA-pair row sweep (knn_tc2.cu) and the
// symmetric search (knn_sym.cu).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "knn_select.cuh"
#include "knn_tc.cuh"
#include "tc_ptx.cuh"

namespace tsne {

constexpr int TC_BK = 64;   // K-step of the fp16 operand tiles (64 x 2 B = one 128-B swizzle row)

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
  CUtensorMap map_b;                                     // B half-tiles of the CTA pair
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

}  // namespace tsne
