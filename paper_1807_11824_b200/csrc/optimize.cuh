// optimize.cuh -- the iteration loop of Algorithm 1 on one GPU.
#pragma once
#include "tree.cuh"

namespace tsne {

// schedule and optimiser constants (D12-D16; the paper states none)
struct Sched {
  int32_t exag_iters;
  float exag, mom0, mom1, eta, min_gain;
};

struct OptWS {
  int32_t* t_dev = nullptr;   // iteration counter read by the update kernel
  int32_t* flag = nullptr;    // non-finite sentinel
  float2* Yb = nullptr;       // second embedding buffer (double buffering)
};

void carve_opt(Carver& c, OptWS& o, int64_t N);

int attract_blocks(int64_t N);
tsne_status launch_attract_grad(const int64_t* row_ptr, const int32_t* col, const float* val,
                                const float2* Y, int64_t N, const float2* rep, const double* Z,
                                float alpha, float2* dY, cudaStream_t s);
tsne_status launch_attract_update(const int64_t* row_ptr, const int32_t* col, const float* val,
                                  const float2* Yin, int64_t N, TreeWS& w, OptWS& o,
                                  const Sched& sc, float2* Yout, float2* V, float2* G,
                                  cudaStream_t s);

// Runs n_iter iterations from state (Y, V, G) starting at iteration t0.
tsne_status run_iterations(const int64_t* row_ptr, const int32_t* col, const float* val,
                           int64_t N, float2* Y, float2* V, float2* G, int32_t t0, int32_t n_iter,
                           float theta, const Sched& sc, bool use_graphs, TreeWS& w, OptWS& o,
                           cudaStream_t s);

tsne_status profile_iterations(const int64_t* row_ptr, const int32_t* col, const float* val,
                               int64_t N, float2* Y, float2* V, float2* G, int32_t t0, int32_t reps,
                               float theta, const Sched& sc, TreeWS& w, OptWS& o, double* stage_ms,
                               int32_t* kernels, cudaStream_t s);

tsne_status launch_init_y(int64_t N, uint64_t seed, float2* Y, cudaStream_t s);

}  // namespace tsne
