// knn_tc.cuh -- tcgen05 (5th-gen tensor core) candidate stage of the kNN.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace tsne {
bool knn_tc_available();
tsne_status launch_cand_tc(const __half* Xh, const float* nrm, int N, int q0, int nq, int Dp, int Kc,
                           unsigned long long* buf, unsigned long long* cand, int slots,
                           unsigned* sync, cudaStream_t s);
size_t knn_tc_sync_words(int64_t N, int64_t nq);
size_t knn_tc2_sync_words(int64_t N, int64_t nq);
int knn_tc2_b_rows();
tsne_status launch_cand_tc2(const CUtensorMap& map, const CUtensorMap& map_b, const float* nrm, int N, int q0, int nq, int Dp, int Kc,
                            unsigned long long* buf, unsigned long long* cand, int slots,
                            unsigned* sync, cudaStream_t s);
}  // namespace tsne
