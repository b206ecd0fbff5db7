// knn_tc.cu -- placeholder until the tcgen05 candidate kernel lands.
#include "knn_tc.cuh"

namespace tsne {
bool knn_tc_available() { return false; }
tsne_status launch_cand_tc(const __half*, const float*, int, int, int, unsigned long long*,
                           unsigned long long*, int, cudaStream_t) {
  set_error("tcgen05 kNN path not built");
  return TSNE_ERR_CUDA;
}
}  // namespace tsne
