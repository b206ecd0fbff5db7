// knn.cuh -- exact k nearest neighbours (U1; Alg. 1 line 1)
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"

namespace tsne {

constexpr int kMaxK = 192;        // neighbours supported (paper: K in [32, 150])
constexpr int kCandExtra = 64;    // K' = K + 64 candidates
constexpr int kCandCap = 1024;    // per-row candidate buffer between compactions
constexpr int kKnnBM = 128;       // query rows per CTA

struct KnnWS {
  int64_t N = 0;
  int32_t D = 0, Dp = 0, K = 0, Kc = 0;
  int32_t slots = 0;              // persistent CTAs (candidate buffers)
  double* colsum = nullptr;       // D   (fp64 column sums -> mean)
  float* mean = nullptr;          // D
  unsigned* amax = nullptr;       // max |x - mean| (float bits)
  float* scale = nullptr;         // [0] = 2^e, [1] = 2^-2e
  __half* Xh = nullptr;           // N x Dp, fp16((x - mean) 2^e), zero padded
  float* nrm = nullptr;           // N   |x_h|^2 (fp32)
  unsigned long long* buf = nullptr;   // slots x 128 x kCandCap candidate keys
  unsigned long long* cand = nullptr;  // N x Kc final candidate keys (sorted)
  unsigned long long* uncert = nullptr;  // [0] count of uncertified rows
  int32_t* rows_bad = nullptr;    // list of uncertified rows (N)
  unsigned* sync = nullptr;       // CTA checkpoint counters of the tcgen05 sweep
  // exact fallback scan of uncertified rows (D26): kScanRows rows at a time
  double* sd = nullptr;           // kScanRows x N fp64 distances
  double* sd_alt = nullptr;       // N (radix-sort double buffer)
  int32_t* si = nullptr;          // N point indices
  int32_t* si_alt = nullptr;      // N
  void* sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  // symmetric candidate search (knn_sym.cu), full-N calls only
  bool sym = false;
  int32_t C = 0;                  // locality cells (sampled points)
  __half* Xs = nullptr;           // (C + 256) x Dp sampled rows
  float* nrm_s = nullptr;         // C + 256
  unsigned long long* cand32 = nullptr;          // N x 32: nearest samples
  uint32_t* cell = nullptr;       // N   cell of each point   (+ N alt)
  int32_t* perm = nullptr;        // N   locality order -> point (+ N alt)
  int32_t* inv = nullptr;         // N   point -> locality position
  __half* Xp = nullptr;           // (N + 256) x Dp rows in locality order
  float* nrm_p = nullptr;         // N + 256
  float* tau = nullptr;           // N + 256 per point thresholds
  float* ntau = nullptr;          // N + 256
  unsigned* cnt = nullptr;        // N list lengths
  unsigned long long* list = nullptr;            // N x kSymCap
  int32_t* fb = nullptr;          // N fallback points (locality positions)
  __half* Xq = nullptr;           // (kFbRows + 256) x Dp gathered fallback rows
  unsigned long long* candfb = nullptr;          // kFbRows x Kc
  unsigned* misc = nullptr;       // [0] max |x_h|^2 bits, [1] fallback count
  int64_t sym_fallback = 0;       // points redone by the row sweep (last call)
  int32_t path = 0;
};
constexpr int kScanRows = 8;
constexpr int kSymCap = 1024;     // list capacity per point
#ifndef TSNE_SYM_CELLS
#define TSNE_SYM_CELLS 8192
#endif
#ifndef TSNE_SYM_WINDOW
#define TSNE_SYM_WINDOW 6
#endif
constexpr int kSymCells = TSNE_SYM_CELLS;    // locality cells (sampled points)
constexpr int kSymWindow = TSNE_SYM_WINDOW;  // pilot window, column tiles of 256 (12: +54 ms at C5)
constexpr int kFbRows = 16384;    // fallback rows per asymmetric sweep

void carve_knn(Carver& c, KnnWS& w, int64_t N, int32_t D, int32_t K);
// Neighbours of the query rows [q0, q0 + nq) among all N points; idx / d2 are
// nq x K (row q0 + r at row r).
tsne_status run_knn(const float* X, int64_t N, int32_t D, int32_t K, int64_t q0, int64_t nq,
                    int32_t* idx, double* d2, KnnWS& w, tsne_knn_info* info, cudaStream_t s);

// util (util.cu)
tsne_status check_finite(const float* X, int64_t n, int32_t* dflag, int32_t* hflag, cudaStream_t s);
tsne_status fill_ones(float* p, int64_t n, cudaStream_t s);

}  // namespace tsne
