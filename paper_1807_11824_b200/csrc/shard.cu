// shard.cu -- multi-GPU building blocks (not in the paper, which
// is single-GPU).  One process per GPU; every rank keeps the full
// embedding, builds the (small) quadtree redundantly, and computes the forces
// and the update of the points it owns, rows [row0, row1).  The exchange --
// the Z partials and the all-gather of the updated Y shards -- is done by the
// caller over NCCL (torch.distributed), between the two calls below.
#include "shard.cuh"

namespace tsne {

void carve_shard(Carver& c, ShardWS& w, int64_t N) {
  carve_tree(c, w.tree, N);
  w.flags = c.take<int32_t>(N / 1024 + 2);   // per-block owned counts -> offsets
  w.pos = c.take<int32_t>(1);                // number of owned points
  w.list = c.take<int32_t>(N);
}

// The sorted positions k whose point perm[k] is owned ([row0, row1)), in
// sorted order: per-block counts (warp ballots), an exclusive scan of the
// block counts (one CTA), then every owned position written at its rank.
constexpr int kOwnThreads = 1024;

__device__ __forceinline__ bool owned_at(const int32_t* perm, int k, int N, int row0, int row1) {
  if (k >= N) return false;
  const int p = perm[k];
  return p >= row0 && p < row1;
}

__global__ void __launch_bounds__(kOwnThreads)
k_owned_count(const int32_t* __restrict__ perm, int N, int row0, int row1,
              int32_t* __restrict__ bcount) {
  __shared__ int s_w[kOwnThreads / 32];
  const int k = blockIdx.x * kOwnThreads + threadIdx.x;
  const unsigned b = __ballot_sync(0xffffffffu, owned_at(perm, k, N, row0, row1));
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kOwnThreads / 32; ++w) t += s_w[w];
    bcount[blockIdx.x] = t;
  }
}

// exclusive scan of nb block counts in place (one CTA), total into *ntot
__global__ void __launch_bounds__(1024) k_owned_scan(int32_t* __restrict__ bcount, int nb,
                                                     int32_t* __restrict__ ntot) {
  __shared__ int s_w[32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int per = (nb + 1023) / 1024;
  const int b0 = t * per, b1 = min(nb, b0 + per);
  int tot = 0;
  for (int b = b0; b < b1; ++b) tot += bcount[b];
  int inc = tot;
  for (int o = 1; o < 32; o <<= 1) {
    const int x = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += x;
  }
  if (lane == 31) s_w[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int v = s_w[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int x = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += x;
    }
    s_w[lane] = v;
  }
  __syncthreads();
  int off = (wid ? s_w[wid - 1] : 0) + inc - tot;
  for (int b = b0; b < b1; ++b) {
    const int c = bcount[b];
    bcount[b] = off;
    off += c;
  }
  if (t == 1023) *ntot = s_w[31];
}

__global__ void __launch_bounds__(kOwnThreads)
k_owned_write(const int32_t* __restrict__ perm, int N, int row0, int row1,
              const int32_t* __restrict__ boff, int32_t* __restrict__ list) {
  __shared__ int s_w[kOwnThreads / 32];
  const int k = blockIdx.x * kOwnThreads + threadIdx.x;
  const bool own = owned_at(perm, k, N, row0, row1);
  const unsigned b = __ballot_sync(0xffffffffu, own);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_w[wid] = __popc(b);
  __syncthreads();
  int before = boff[blockIdx.x];
  for (int w = 0; w < wid; ++w) before += s_w[w];
  if (own) list[before + __popc(b & ((1u << lane) - 1u))] = k;
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
  const int nb = (n + kOwnThreads - 1) / kOwnThreads;
  k_owned_count<<<nb, kOwnThreads, 0, s>>>(t.perm, n, (int)row0, (int)row1, w.flags);
  TSNE_LAUNCH_CHECK();
  k_owned_scan<<<1, 1024, 0, s>>>(w.flags, nb, w.pos);
  TSNE_LAUNCH_CHECK();
  k_owned_write<<<nb, kOwnThreads, 0, s>>>(t.perm, n, (int)row0, (int)row1, w.flags, w.list);
  TSNE_LAUNCH_CHECK();
  return launch_traverse_list(t, theta, w.list, w.pos, (int)row0, rep_local, z_partial, s);
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
