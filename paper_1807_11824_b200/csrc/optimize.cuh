// optimize.cuh -- the iteration loop of Algorithm 1 on one GPU.
#pragma once
#include "tree.cuh"

namespace tsne {

// attractive-pass item: consecutive nonzeros of a row, counted from the row's
// start, reduced by one warp (attract.cu); the relabelled CSR orders the
// entries of each item for the pass's window gathers (optimize.cu)
#ifndef TSNE_AT_ITEM
#define TSNE_AT_ITEM 256
#endif
constexpr int kAtItemNz = TSNE_AT_ITEM;

// schedule and optimiser constants (D12-D16; the paper states none)
struct Sched {
  int32_t exag_iters;
  float exag, mom0, mom1, eta, min_gain;
};

// Internal optimiser state.  Points are periodically relabelled into the
// Morton order of the current embedding (locality of the y_j gathers of the
// attractive pass and of the tree build); `lab[k]` is the caller's index of
// internal point k, and P is kept in internal labels (two CSR copies A/B).
// The attractive pass's batches of one CSR, cut once (attract.cu,
// k_attract_plan) and reused by every iteration until the CSR changes, so
// the pipeline's producer only streams.  grid: the pass's CTAs.
struct AtPlan {
  void* batches = nullptr;
  int4* cta = nullptr;
  int grid = 0;
};
int attract_grid_sum(int64_t N, int64_t nnz);     // CTAs of launch_attract_sum
int attract_grid_shard(int64_t n_local);          // CTAs of launch_attract_sum_shard
void carve_attract_plan(Carver& c, AtPlan& p, int64_t n_rows, int64_t nnz_cap, int grid);
tsne_status attract_plan_build(const AtPlan& p, const int64_t* row_ptr, int64_t n_rows,
                               cudaStream_t s);

struct OptWS {
  int64_t N = 0, nnz = 0;
  int32_t* t_dev = nullptr;   // iteration counter read by the update kernel
  int32_t* flag = nullptr;    // non-finite sentinel
  float2 *Ya = nullptr, *Yb = nullptr;   // embedding (double buffer of the update)
  float2 *V = nullptr, *G = nullptr;     // velocity, gains
  float2* tmp = nullptr;                 // permutation scratch
  float2* A = nullptr;                   // attractive sums (side stream)
  cudaStream_t side = nullptr;           // attractive pass runs here, concurrently
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int32_t *lab = nullptr, *lab2 = nullptr, *inv = nullptr;
  int32_t* dperm = nullptr;              // cached diffusion order of P (see enter())
  uint64_t* dtag = nullptr;              // its validity tag (device copy)
  void* ws_base = nullptr;               // the caller's workspace (cache key)
  int64_t* rp[2] = {nullptr, nullptr};
  int32_t* col[2] = {nullptr, nullptr};
  float* val[2] = {nullptr, nullptr};
  AtPlan plan[2];                        // the attractive pass's batches of P half h
  int64_t* len = nullptr;                // N+1 row lengths -> scanned row_ptr
  void* scan_tmp = nullptr;
  size_t scan_tmp_bytes = 0;
};

void carve_opt(Carver& c, OptWS& o, int64_t N, int64_t nnz);

tsne_status launch_attract_grad(const int64_t* row_ptr, const int32_t* col, const float* val,
                                const float2* Y, int64_t N, const float2* rep, const double* Z,
                                float alpha, float2* dY, cudaStream_t s);
tsne_status launch_attract_sum(const int64_t* row_ptr, const int32_t* col, const float* val,
                               const float2* Y, int64_t N, int64_t nnz, float2* A,
                               const AtPlan* plan, cudaStream_t s);
tsne_status launch_update(const float2* Yin, const float2* A, int64_t N, TreeWS& w, OptWS& o,
                          const Sched& sc, float2* Yout, float2* V, float2* G, cudaStream_t s);

// Runs n_iter iterations from the caller's state (Y, V, G) starting at t0.
// relabel_every: period of the Morton relabelling (0 = never).
tsne_status run_iterations(const int64_t* row_ptr, const int32_t* col, const float* val,
                           int64_t N, float2* Y, float2* V, float2* G, int32_t t0, int32_t n_iter,
                           float theta, const Sched& sc, bool use_graphs, int relabel_every,
                           TreeWS& w, OptWS& o, cudaStream_t s, bool cache_order,
                           bool keep_state = false);
// drops the kept state and graphs of workspace ws (tsne_optimize_release)
void release_session(const void* ws);

tsne_status profile_iterations(const int64_t* row_ptr, const int32_t* col, const float* val,
                               int64_t N, float2* Y, float2* V, float2* G, int32_t t0, int32_t reps,
                               float theta, const Sched& sc, TreeWS& w, OptWS& o, double* stage_ms,
                               int32_t* kernels, double* trav_stats, cudaStream_t s);

tsne_status launch_init_y(int64_t N, uint64_t seed, float2* Y, cudaStream_t s);

// multi-GPU run: the diffusion locality order of P (perm[N], scratch u[2N]) and
// P relabelled by a permutation (new label k <- old perm[k])
tsne_status diffusion_perm(const int64_t* row_ptr, const int32_t* col, const float* val,
                           int64_t N, TreeWS& w, float2* u, int32_t* perm, cudaStream_t s);
tsne_status permute_csr(const int32_t* perm, int64_t N, const int64_t* rp, const int32_t* col,
                        const float* val, int32_t* inv, int64_t* len, void* scan_tmp,
                        size_t scan_bytes, int64_t* rp2, int32_t* col2, float* val2,
                        cudaStream_t s);
size_t permute_csr_scan_bytes(int64_t N);

}  // namespace tsne
