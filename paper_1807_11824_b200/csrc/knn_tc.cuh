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
size_t knn_tc2_sync_words(int64_t N, int64_t nq);
int knn_tc2_b_rows();
tsne_status launch_cand_tc2(const CUtensorMap& map, const CUtensorMap& map_b, const float* nrm, int N, int q0, int nq, int Dp, int Kc,
                            unsigned long long* buf, unsigned long long* cand, int slots,
                            unsigned* sync, cudaStream_t s, int self_excl = 1, int win_tiles = 0,
                            const int32_t* qid = nullptr);
// the pair kernel on explicit operand matrices: rows q0..q0+nq-1 of A (rowsA
// rows allocated) against the nB points of B (rowsB rows allocated, norms
// nrmB); qid (nullable): the point id of each A row (self exclusion)
tsne_status launch_cand_pair(const __half* A, int64_t rowsA, const __half* B, int64_t rowsB,
                             const float* nrmB, int nB, int q0, int nq, int Dp, int Kc,
                             unsigned long long* buf, unsigned long long* cand, int slots,
                             unsigned* sync, cudaStream_t s, int self_excl, int win_tiles,
                             const int32_t* qid);
size_t knn_sym_sync_words(int64_t N);
tsne_status launch_cand_sym(const CUtensorMap& map, const CUtensorMap& map_b, const float* nrm,
                            float* tau, float* ntau, unsigned* cnt,
                            unsigned long long* list, int cap, int N, int Dp, unsigned* sync,
                            cudaStream_t s);
tsne_status launch_sym(const __half* Xp, int64_t rows, const float* nrm, float* tau,
                       float* ntau, unsigned* cnt, unsigned long long* list, int cap, int N,
                       int Dp, unsigned* sync, cudaStream_t s);
}  // namespace tsne
