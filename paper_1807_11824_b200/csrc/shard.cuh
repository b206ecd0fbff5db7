// shard.cuh -- multi-GPU per-rank iteration pieces
#pragma once
#include "optimize.cuh"

namespace tsne {

struct ShardWS {
  TreeWS tree;
  int32_t *flags = nullptr, *pos = nullptr, *list = nullptr;
};

void carve_shard(Carver& c, ShardWS& w, int64_t N);
tsne_status shard_forces(ShardWS& w, const float2* Y, int64_t N, int64_t row0, int64_t row1,
                         float theta, bool recentre, float2* rep_local, double* z_partial,
                         cudaStream_t s);
tsne_status shard_recentre(ShardWS& w, float2* Y, int64_t N, cudaStream_t s);
tsne_status launch_attract_sum_shard(const int64_t* row_ptr, const int32_t* col, const float* val,
                                     const float2* Y, int64_t N, int64_t row0, int64_t n_local,
                                     float2* A, const AtPlan* plan, cudaStream_t s);
tsne_status launch_update_shard(const float2* A, const float2* Y, int64_t row0, int64_t n_local,
                                const float2* rep, const double* zp, int world, int t,
                                const Sched& sc, const BoxInfo* box, float2* V, float2* G,
                                float2* Yout, int32_t* flag, cudaStream_t s);

}  // namespace tsne
