// shard.cu -- multi-GPU building blocks (not in the paper, which
// is single-GPU).  One process per GPU; every rank keeps the full
// embedding, builds the (small) quadtree redundantly, and computes the forces
// and the update of the points it owns, rows [row0, row1).  The exchange --
// the Z partials and the all-gather of the updated Y shards -- is done by the
// caller over NCCL (torch.distributed), between the two calls below.
#include <cub/device/device_scan.cuh>

#include "shard.cuh"

namespace tsne {

void carve_shard(Carver& c, ShardWS& w, int64_t N) {
  carve_tree(c, w.tree, N);
  w.flags = c.take<int32_t>(N + 1);
  w.pos = c.take<int32_t>(N + 1);
  w.list = c.take<int32_t>(N);
  size_t sb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, sb, (int32_t*)nullptr, (int32_t*)nullptr, (int)(N + 1));
  w.scan_tmp = c.take<char>(sb);
  w.scan_tmp_bytes = sb;
}

__global__ void k_owned_flags(const int32_t* __restrict__ perm, int N, int row0, int row1,
                              int32_t* __restrict__ flags) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > N) return;
  if (k == N) { flags[N] = 0; return; }
  const int p = perm[k];
  flags[k] = (p >= row0 && p < row1) ? 1 : 0;
}

__global__ void k_owned_list(const int32_t* __restrict__ flags, const int32_t* __restrict__ pos,
                             int N, int32_t* __restrict__ list) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  if (flags[k]) list[pos[k]] = k;
}

__global__ void k_recentre(float2* Y, int N, const BoxInfo* box) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  float2 y = Y[i];
  y.x = y.x - box->shift_x;
  y.y = y.y - box->shift_y;
  Y[i] = y;
}

tsne_status shard_forces(ShardWS& w, const float2* Y, int64_t N, int64_t row0, int64_t row1,
                         float theta, bool recentre, float2* rep_local, double* z_partial,
                         cudaStream_t s) {
  // Y is read-only: the recentring shift (D15) is computed here (box->shift)
  // and applied on the fly by the tree build and by the update of the owned
  // rows (tsne_shard_update), so the attractive pass may read Y concurrently
  TreeWS& t = w.tree;
  tsne_status st = tree_ws_init(t, s);      // the workspace may be fresh (caller-owned)
  if (st != TSNE_OK) return st;
  st = recentre ? launch_bbox_mean(t, Y, s) : launch_bbox(t, Y, s);
  if (st != TSNE_OK) return st;
  if ((st = build_tree(t, Y, /*apply_shift=*/true, s)) != TSNE_OK) return st;
  const int n = (int)N;
  k_owned_flags<<<(n + 256) / 256, 256, 0, s>>>(t.perm, n, (int)row0, (int)row1, w.flags);
  TSNE_LAUNCH_CHECK();
  size_t sb = w.scan_tmp_bytes;
  TSNE_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w.scan_tmp, sb, w.flags, w.pos, n + 1, s));
  k_owned_list<<<(n + 255) / 256, 256, 0, s>>>(w.flags, w.pos, n, w.list);
  TSNE_LAUNCH_CHECK();
  return launch_traverse_list(t, theta, w.list, w.pos + n, (int)row0, rep_local, z_partial, s);
}

tsne_status shard_recentre(ShardWS& w, float2* Y, int64_t N, cudaStream_t s) {
  TSNE_CUDA_TRY(cudaMemsetAsync(w.tree.counter, 0, 8 * sizeof(unsigned), s));
  tsne_status st = launch_bbox_mean(w.tree, Y, s);
  if (st != TSNE_OK) return st;
  k_recentre<<<(int)((N + 255) / 256), 256, 0, s>>>(Y, (int)N, w.tree.box);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

}  // namespace tsne
