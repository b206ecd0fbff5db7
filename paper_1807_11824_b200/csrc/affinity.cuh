// affinity.cuh -- U2 perplexity bisection + U3 symmetrisation
#pragma once
#include "common.cuh"

namespace tsne {

struct PWS {
  int64_t N = 0;
  int32_t K = 0, nb = 0;
  double* pc = nullptr;                    // N x K conditional p_{j|i}
  double* beta = nullptr;                  // N
  unsigned long long* ndeg = nullptr;      // degenerate row count
  unsigned long long *ka = nullptr, *kb = nullptr;  // 2NK (row, col) keys
  double *va = nullptr, *vb = nullptr;     // 2NK values
  void* sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  int32_t* head = nullptr;                 // 2NK + 1 head flags -> positions
  int32_t* pos = nullptr;                  // 2NK + 1
  void* scan_tmp = nullptr;
  size_t scan_tmp_bytes = 0;
};

void carve_p(Carver& c, PWS& w, int64_t N, int32_t K);
tsne_status run_compute_p(const int32_t* idx, const double* d2, int64_t N, int32_t K,
                          float perplexity, int64_t* row_ptr, int32_t* col, float* val,
                          int64_t* nnz_host, double* beta_out, PWS& w, int64_t* ndeg_host,
                          cudaStream_t s);

}  // namespace tsne
