// tree.cu -- quadtree build over the 2-D embedding (P:L136 steps 1-4).
//
//  k_bbox        step 1: exact min/max, root box (D8)         [H1]
//  k_keys        fp64 quantisation -> 48-bit Morton key (D8, D9) [H2]
//  radix sort    (key, point id) pairs                         [H2]
//  k_gather      Y in Morton order, fixed-point coordinates, block sums,
//                split deltas (common-prefix length of sorted neighbours)
//  k_bscan       exclusive scan of the block sums (one block)
//  k_radix_build exclusive prefix sums of the fixed-point coordinates
//                (integers: exact, deterministic) [H4], and the binary
//                radix tree bottom-up: node ranges, quad-cell test,
//                start-chain counts                              [H3]
//  k_scan_cnt    quad nodes per start position -> pre-order base [H3]
//  k_quad_emit   pre-order node records, counts, centres of mass [H3, H4]
//
// The compressed quadtree is derived from the binary radix tree (Karras 2012)
// over the sorted keys: a binary node whose common prefix has length delta
// lies in the cell of level L = min(delta, 48) / 2 (48-bit keys, 24 levels,
// D9); it is a quad node iff its parent's level is smaller (otherwise it
// merges into the parent).  Keys tie-break by sorted position (delta >= 48 ->
// identical keys -> a level-24 bucket).  The binary tree is built bottom-up
// (Apetrei 2014): internal node p is the split between sorted positions p and
// p + 1; a node [l, r]'s parent is the split next to it with the longer common
// prefix (delta(r) vs delta(l - 1): never equal, so the tree is the unique
// binary radix tree).  DESIGN.md sec. 6.2.
#include <cub/device/device_radix_sort.cuh>

#include "tree.cuh"

namespace tsne {

// ---------------------------------------------------------------- workspace
struct LL2Sum {
  __host__ __device__ __forceinline__ longlong2 operator()(const longlong2& a,
                                                           const longlong2& b) const {
    return make_longlong2(a.x + b.x, a.y + b.y);
  }
};

size_t tree_cub_bytes(int64_t N) {
  size_t a = 0;
  cub::DoubleBuffer<uint64_t> dk(nullptr, nullptr);
  cub::DoubleBuffer<int32_t> dv(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, a, dk, dv, (int)N, 0, kKeyBits);
  return a;
}

void carve_tree(Carver& c, TreeWS& w, int64_t N) {
  w.N = N;
  const size_t sb = tree_cub_bytes(N);
  w.keys_a = c.take<uint64_t>(N);
  w.keys_b = c.take<uint64_t>(N);
  w.vals_a = c.take<int32_t>(N);
  w.vals_b = c.take<int32_t>(N);
  w.sort_tmp = c.take<char>(sb);
  w.sort_tmp_bytes = sb;
  w.ys = c.take<float2>(N);
  w.fq = c.take<longlong2>(N + 1);
  w.S = c.take<longlong2>(N + 1);
  w.bsum = c.take<longlong2>((N + 1 + 255) / 256 + 1);
  w.dl = c.take<uint8_t>(N);
  w.slot = c.take<unsigned long long>(N);
  w.nfo = c.take<int4>(N);
  w.cnt = c.take<int32_t>(N + 1);
  w.base = c.take<int32_t>(N + 1);
  w.tsum = c.take<int32_t>((N + 1 + kScanTile - 1) / kScanTile);
  w.ctl = c.take<uint32_t>(2);
  w.nodes = c.take<float4>(2 * N);
  w.nfirst = c.take<int32_t>(2 * N);
  w.com64 = c.take<double2>(2 * N);
  w.leafnode = c.take<int32_t>(N);
  w.box = c.take<BoxInfo>(2);
  w.has_bucket = c.take<int32_t>(1);
  w.rep = c.take<float2>(N);
  w.zpart = c.take<double>(traverse_blocks(N));
  w.ovf = c.take<int2>((size_t)traverse_blocks(N) * 256 * 12);   // traversal bucket overflow
  w.lg = c.take<int2>((size_t)traverse_blocks(N) * 256 * 16);    // traversal large buckets
  w.dlist = c.take<int2>((size_t)traverse_blocks(N) * 256);
  w.zacc = c.take<unsigned long long>(2);
  w.Z = c.take<double>(2);
  w.counter = c.take<unsigned>(8);
  w.part4 = c.take<float4>(kMaxParts);
  w.part2 = c.take<double2>(kMaxParts);
}

// ---------------------------------------------------------------- H1 bbox
constexpr int kBoxThreads = 256;

__global__ void __launch_bounds__(kBoxThreads) k_bbox(const float2* __restrict__ Y, int N,
                                                      float4* part, unsigned* counter,
                                                      BoxInfo* box) {
  float mnx = INFINITY, mxx = -INFINITY, mny = INFINITY, mxy = -INFINITY;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    float2 y = Y[i];
    mnx = fminf(mnx, y.x); mxx = fmaxf(mxx, y.x);
    mny = fminf(mny, y.y); mxy = fmaxf(mxy, y.y);
  }
  mnx = warp_min(mnx); mxx = warp_max(mxx); mny = warp_min(mny); mxy = warp_max(mxy);
  __shared__ float4 sw[kBoxThreads / 32];
  __shared__ bool last;
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sw[wid] = make_float4(mnx, mxx, mny, mxy);
  __syncthreads();
  if (threadIdx.x == 0) {
    float4 r = sw[0];
    for (int k = 1; k < kBoxThreads / 32; ++k) {
      r.x = fminf(r.x, sw[k].x); r.y = fmaxf(r.y, sw[k].y);
      r.z = fminf(r.z, sw[k].z); r.w = fmaxf(r.w, sw[k].w);
    }
    part[blockIdx.x] = r;
    __threadfence();
    unsigned t = atomicAdd(counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    float4 r = __ldcg(part);
    for (int k = 1; k < (int)gridDim.x; ++k) {
      float4 q = __ldcg(part + k);
      r.x = fminf(r.x, q.x); r.y = fmaxf(r.y, q.y);
      r.z = fminf(r.z, q.z); r.w = fmaxf(r.w, q.w);
    }
    BoxInfo b;
    make_root_box(r.x, r.y, r.z, r.w, &b);
    b.shift_x = 0.f;
    b.shift_y = 0.f;
    b.pad0 = 0.f;
    *box = b;
    *counter = 0u;
  }
}

tsne_status launch_bbox(TreeWS& w, const float2* Y, cudaStream_t s) {
  int blocks = (int)((w.N + 4 * kBoxThreads - 1) / (4 * kBoxThreads));
  if (blocks > 2 * kNumSMs) blocks = 2 * kNumSMs;
  if (blocks < 1) blocks = 1;
  k_bbox<<<blocks, kBoxThreads, 0, s>>>(Y, (int)w.N, w.part4, w.counter + 0, w.box);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

// Bounding box and recentring shift of Y (multi-GPU path: the replicated
// embedding is recentred at the start of each rank's iteration, D15).
__global__ void __launch_bounds__(kBoxThreads) k_bbox_mean(const float2* __restrict__ Y, int N,
                                                           float4* part, double2* part2,
                                                           unsigned* counter, BoxInfo* box) {
  float mnx = INFINITY, mxx = -INFINITY, mny = INFINITY, mxy = -INFINITY;
  double sx = 0.0, sy = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    float2 y = Y[i];
    mnx = fminf(mnx, y.x); mxx = fmaxf(mxx, y.x);
    mny = fminf(mny, y.y); mxy = fmaxf(mxy, y.y);
    sx += (double)y.x; sy += (double)y.y;
  }
  mnx = warp_min(mnx); mxx = warp_max(mxx); mny = warp_min(mny); mxy = warp_max(mxy);
  sx = warp_sum(sx); sy = warp_sum(sy);
  __shared__ float4 sw[kBoxThreads / 32];
  __shared__ double2 ss[kBoxThreads / 32];
  __shared__ bool last;
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { sw[wid] = make_float4(mnx, mxx, mny, mxy); ss[wid] = make_double2(sx, sy); }
  __syncthreads();
  if (threadIdx.x == 0) {
    float4 r = sw[0];
    double2 q2 = ss[0];
    for (int k = 1; k < kBoxThreads / 32; ++k) {
      r.x = fminf(r.x, sw[k].x); r.y = fmaxf(r.y, sw[k].y);
      r.z = fminf(r.z, sw[k].z); r.w = fmaxf(r.w, sw[k].w);
      q2.x += ss[k].x; q2.y += ss[k].y;
    }
    part[blockIdx.x] = r;
    part2[blockIdx.x] = q2;
    __threadfence();
    unsigned t = atomicAdd(counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    float4 r = __ldcg(part);
    double2 q2 = __ldcg(part2);
    for (int k = 1; k < (int)gridDim.x; ++k) {
      float4 q = __ldcg(part + k);
      double2 a = __ldcg(part2 + k);
      r.x = fminf(r.x, q.x); r.y = fmaxf(r.y, q.y);
      r.z = fminf(r.z, q.z); r.w = fmaxf(r.w, q.w);
      q2.x += a.x; q2.y += a.y;
    }
    const float mx = (float)(q2.x / (double)N), my = (float)(q2.y / (double)N);
    BoxInfo b;
    make_root_box(r.x - mx, r.y - mx, r.z - my, r.w - my, &b);   // monotone rounding
    b.shift_x = mx;
    b.shift_y = my;
    b.pad0 = 0.f;
    *box = b;
    *counter = 0u;
  }
}

tsne_status launch_bbox_mean(TreeWS& w, const float2* Y, cudaStream_t s) {
  int blocks = (int)((w.N + 4 * kBoxThreads - 1) / (4 * kBoxThreads));
  if (blocks > 2 * kNumSMs) blocks = 2 * kNumSMs;
  if (blocks < 1) blocks = 1;
  k_bbox_mean<<<blocks, kBoxThreads, 0, s>>>(Y, (int)w.N, w.part4, w.part2, w.counter + 3, w.box);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

// ---------------------------------------------------------------- H2 keys
// spread the kLevels bits of x to the even bit positions of a 64-bit word
__device__ __forceinline__ uint64_t spread_bits(uint32_t x32) {
  uint64_t x = x32;
  x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
  x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
  x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x << 2)) & 0x3333333333333333ull;
  x = (x | (x << 1)) & 0x5555555555555555ull;
  return x;
}

// q = min(2^L-1, max(0, floor((y - lo) * s))) in fp64 without contraction (D8, D9)
__device__ __forceinline__ uint32_t quantise(float y, double lo, double s) {
  double f = floor(__dmul_rn(__dsub_rn((double)y, lo), s));
  f = f >= 0.0 ? f : 0.0;                                           // (NaN -> 0)
  f = f <= (double)((1u << kLevels) - 1u) ? f : (double)((1u << kLevels) - 1u);
  return (uint32_t)f;
}

// Y is read-only: the pending recentring shift (D15) is applied on the fly,
// so the attractive pass may read Y concurrently.
__global__ void k_keys(const float2* __restrict__ Y, int N, const BoxInfo* __restrict__ box,
                       int apply_shift, uint64_t* __restrict__ keys, int32_t* __restrict__ vals,
                       int32_t* __restrict__ cnt, int32_t* __restrict__ has_bucket,
                       int32_t* __restrict__ tsum, int ntiles, uint32_t* __restrict__ ctl) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > N) return;
  cnt[i] = 0;
  if (i < ntiles) tsum[i] = 0;
  if (i == 0) {
    *has_bucket = 0;
    ctl[0] = ctl[0] + 1u;                               // build epoch (k_radix_build)
  }
  if (i == N) return;
  const BoxInfo b = *box;
  float2 y = Y[i];
  if (apply_shift) {
    y.x = y.x - b.shift_x;
    y.y = y.y - b.shift_y;
  }
  uint32_t qx = quantise(y.x, b.lox, b.s);
  uint32_t qy = quantise(y.y, b.loy, b.s);
  keys[i] = (spread_bits(qx) << 1) | spread_bits(qy);   // quadrant digit = 2 bx + by
  vals[i] = i;
}

tsne_status tree_ws_init(TreeWS& w, cudaStream_t s) {
  TSNE_CUDA_TRY(cudaMemsetAsync(w.counter, 0, 8 * sizeof(unsigned), s));
  TSNE_CUDA_TRY(cudaMemsetAsync(w.zacc, 0, 2 * sizeof(unsigned long long), s));
  // the radix build's node slots are tagged with a build epoch counted from 0
  TSNE_CUDA_TRY(cudaMemsetAsync(w.ctl, 0, 2 * sizeof(uint32_t), s));
  TSNE_CUDA_TRY(cudaMemsetAsync(w.slot, 0, w.N * sizeof(unsigned long long), s));
  return TSNE_OK;
}

// ---------------------------------------------------------------- gather
constexpr int kScanBlock = 256;   // k_gather / k_radix_build block = prefix-sum block

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Exclusive scan over the CTA in thread order (blockDim a multiple of 32,
// <= 1024); *tot = the CTA total.  Integer sums: exact in any association.
__device__ longlong2 cta_scan_ll2(long long x, long long y, longlong2* tot) {
  __shared__ long long wx[32], wy[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  long long ix = x, iy = y;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long ax = __shfl_up_sync(0xffffffffu, ix, o);
    const long long ay = __shfl_up_sync(0xffffffffu, iy, o);
    if (lane >= o) { ix += ax; iy += ay; }
  }
  if (lane == 31) { wx[wid] = ix; wy[wid] = iy; }
  __syncthreads();
  long long ox = 0, oy = 0, tx = 0, ty = 0;
  for (int q = 0; q < nw; ++q) {
    if (q == wid) { ox = tx; oy = ty; }
    tx += wx[q];
    ty += wy[q];
  }
  __syncthreads();                                    // wx/wy reusable
  *tot = make_longlong2(tx, ty);
  return make_longlong2(ox + ix - x, oy + iy - y);
}

__device__ int cta_scan_i32(int x, int* tot) {
  __shared__ int wv[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int ix = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, ix, o);
    if (lane >= o) ix += a;
  }
  if (lane == 31) wv[wid] = ix;
  __syncthreads();
  int o = 0, t = 0;
  for (int q = 0; q < nw; ++q) {
    if (q == wid) o = t;
    t += wv[q];
  }
  __syncthreads();
  *tot = t;
  return o + ix - x;
}

// split delta of sorted position pos (< N - 1): common-prefix length of the
// (key, position) strings at pos and pos + 1
__device__ __forceinline__ uint8_t delta_of(uint64_t a, uint64_t b, int pos) {
  return (uint8_t)(a != b ? __clzll(a ^ b) - (64 - kKeyBits)
                          : kKeyBits + __clz((uint32_t)pos ^ (uint32_t)(pos + 1)));
}

__global__ void __launch_bounds__(kScanBlock)
k_gather(const float2* __restrict__ Y, const int32_t* __restrict__ perm,
         const uint64_t* __restrict__ keys, int N, const BoxInfo* __restrict__ box,
         int apply_shift, float2* __restrict__ ys, longlong2* __restrict__ fq,
         longlong2* __restrict__ bsum, uint8_t* __restrict__ dl) {
  pdl_trigger();
  pdl_wait();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  long long qx = 0, qy = 0;
  if (k < N) {
    float2 y = Y[perm[k]];
    if (apply_shift) {
      y.x = y.x - box->shift_x;
      y.y = y.y - box->shift_y;
    }
    ys[k] = y;
    const double cx = box->cx, cy = box->cy, inv = kFixScale / box->r0;
    qx = __double2ll_rn(__dmul_rn(__dsub_rn((double)y.x, cx), inv));
    qy = __double2ll_rn(__dmul_rn(__dsub_rn((double)y.y, cy), inv));
    if (k < N - 1) dl[k] = delta_of(keys[k], keys[k + 1], k);
  }
  if (k <= N) fq[k] = make_longlong2(qx, qy);      // fq[N] = 0
  // block sum (exact integer arithmetic: the order does not matter)
  __shared__ long long sx[kScanBlock / 32], sy[kScanBlock / 32];
  qx = warp_sum_ll(qx);
  qy = warp_sum_ll(qy);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { sx[wid] = qx; sy[wid] = qy; }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tx = 0, ty = 0;
    for (int q = 0; q < kScanBlock / 32; ++q) { tx += sx[q]; ty += sy[q]; }
    bsum[blockIdx.x] = make_longlong2(tx, ty);
  }
}

// exclusive scan of the nb block sums, in place (one block): per-thread
// serial sums, warp shuffle scans, one warp over the 32 warp totals
__global__ void __launch_bounds__(1024) k_bscan(longlong2* __restrict__ bsum, int nb) {
  pdl_trigger();
  pdl_wait();
  __shared__ long long wx[32], wy[32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int per = (nb + 1023) / 1024;
  const int b0 = t * per, b1 = min(nb, b0 + per);
  long long tx = 0, ty = 0;
  for (int b = b0; b < b1; ++b) { const longlong2 v = bsum[b]; tx += v.x; ty += v.y; }
  long long ix = tx, iy = ty;                          // inclusive warp scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long ax = __shfl_up_sync(0xffffffffu, ix, o);
    const long long ay = __shfl_up_sync(0xffffffffu, iy, o);
    if (lane >= o) { ix += ax; iy += ay; }
  }
  if (lane == 31) { wx[wid] = ix; wy[wid] = iy; }
  __syncthreads();
  if (wid == 0) {
    long long vx = wx[lane], vy = wy[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long ax = __shfl_up_sync(0xffffffffu, vx, o);
      const long long ay = __shfl_up_sync(0xffffffffu, vy, o);
      if (lane >= o) { vx += ax; vy += ay; }
    }
    wx[lane] = vx;                                     // inclusive over warps
    wy[lane] = vy;
  }
  __syncthreads();
  long long ox = (wid ? wx[wid - 1] : 0) + ix - tx, oy = (wid ? wy[wid - 1] : 0) + iy - ty;
  for (int b = b0; b < b1; ++b) {
    const longlong2 v = bsum[b];
    bsum[b] = make_longlong2(ox, oy);
    ox += v.x;
    oy += v.y;
  }
}

// ---------------------------------------------------------------- H3 radix tree
__device__ __forceinline__ int qlevel(int delta) {
  return (delta < kKeyBits ? delta : kKeyBits) >> 1;
}

__device__ __forceinline__ void add_tile(int pos, int cc, int32_t* tsum, int* st, int t_hi) {
  const int t = pos / kScanTile;
  if (t_hi - t < 8) atomicAdd(&st[t_hi - t], cc);
  else atomicAdd(&tsum[t], cc);
}

__device__ void radix_climb(const uint8_t* __restrict__ dl, int N, const uint32_t* __restrict__ ctl,
                            unsigned long long* __restrict__ slot, int4* __restrict__ nfo,
                            int32_t* __restrict__ cnt, int32_t* __restrict__ tsum, int* st, int t_hi,
                            int k) {
  const unsigned long long tag = (unsigned long long)ctl[0] << 32;
  const int dprev = k > 0 ? dl[k - 1] : -1;
  const int dnext = k < N - 1 ? dl[k] : -1;
  bool left = dnext > dprev;                           // leaf k is the left child of split k
  int p = left ? k : k - 1;
  int dp = left ? dnext : dprev;
  int cc = dp < kKeyBits ? 1 : 0;                      // a leaf inside a bucket is no quad node
  if (!left) {                                         // a right child tops its start chain
    cnt[k] = cc;
    if (cc) add_tile(k, cc, tsum, st, t_hi);
  }
  int l = k, r = k;
  for (;;) {
    const uint32_t mine = left ? ((uint32_t)l | ((uint32_t)cc << 25)) : (uint32_t)r;
    const unsigned long long old = atomicExch(slot + p, tag | mine);
    if ((old & 0xffffffff00000000ull) != tag) return;  // first to arrive
    int ccl;
    if (left) {
      r = (int)(uint32_t)old;
      ccl = cc;
    } else {
      l = (int)((uint32_t)old & ((1u << 25) - 1u));
      ccl = (int)((uint32_t)old >> 25);
    }
    // node p = [l, r], delta dp; its parent
    int pp, dpp;
    bool pleft;
    const int dr = r < N - 1 ? dl[r] : -1, dlf = l > 0 ? dl[l - 1] : -1;
    if (dr < 0 && dlf < 0) {
      pp = -1; dpp = -1; pleft = false;
    } else {
      pleft = dr > dlf;
      pp = pleft ? r : l - 1;
      dpp = pleft ? dr : dlf;
    }
    const bool quad = pp < 0 || qlevel(dpp) < qlevel(dp);
    cc = ccl + (quad ? 1 : 0);
    nfo[p] = make_int4(l, r, quad ? cc : -1, dpp);
    if (!pleft) {                                      // right child or root: chain top
      cnt[l] = cc;
      if (cc) add_tile(l, cc, tsum, st, t_hi);
    }
    if (pp < 0) return;
    p = pp;
    dp = dpp;
    left = pleft;
  }
}

// (k_radix_build first writes S = the exclusive prefix sums of the fixed-point
// coordinates over its block of kScanBlock positions, offset by the block's
// scanned sum.)  One thread per leaf climbs while it is the second child to reach a node
// (atomic exchange on the node's slot, tagged with the build epoch; the first
// leaves its range end there and stops).  For the node [l, r] it resolves it
// records (l, r, cc, delta(parent)), cc = quad nodes on the chain of nodes
// starting at l from the bottom up to it (-1 if it is not a quad node), and
// at the top of a start chain cnt[l] = the chain's quad-node count (added to
// the sum of its kScanTile tile, tsum).
__global__ void __launch_bounds__(kScanBlock)
k_radix_build(const uint8_t* __restrict__ dl, int N, const uint32_t* __restrict__ ctl,
              unsigned long long* __restrict__ slot, int4* __restrict__ nfo,
              int32_t* __restrict__ cnt, int32_t* __restrict__ tsum,
              const longlong2* __restrict__ fq, const longlong2* __restrict__ boff,
              longlong2* __restrict__ S) {
  pdl_trigger();
  pdl_wait();
  // chain counts are summed per kScanTile tile: in shared memory for the 8
  // tiles ending at the CTA's own, in global memory beyond
  __shared__ int st[8];
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  {
    const longlong2 v = k <= N ? fq[k] : make_longlong2(0, 0);
    longlong2 tot;
    const longlong2 ex = cta_scan_ll2(v.x, v.y, &tot);
    const longlong2 o = boff[blockIdx.x];
    if (k <= N) S[k] = make_longlong2(o.x + ex.x, o.y + ex.y);
  }
  const int t_hi = (blockIdx.x * blockDim.x + blockDim.x - 1) / kScanTile;
  if (threadIdx.x < 8) st[threadIdx.x] = 0;
  __syncthreads();
  if (k < N) radix_climb(dl, N, ctl, slot, nfo, cnt, tsum, st, t_hi, k);
  __syncthreads();
  if (threadIdx.x < 8 && st[threadIdx.x] && t_hi - (int)threadIdx.x >= 0)
    atomicAdd(&tsum[t_hi - threadIdx.x], st[threadIdx.x]);
}

// exclusive scan of cnt[0..n) -> base[0..n) (n = N + 1: base[N] = node count);
// a tile's prefix is the sum of the tile sums before it (k_radix_build)
__global__ void __launch_bounds__(kSortThreads)
k_scan_cnt(const int32_t* __restrict__ cnt, int n, int32_t* __restrict__ base,
           const int32_t* __restrict__ tsum) {
  pdl_trigger();
  pdl_wait();
  constexpr int kPer = kScanTile / kSortThreads;      // 16, as 4 int4
  const int t = blockIdx.x;
  int pp = 0;
  for (int q = threadIdx.x; q < t; q += blockDim.x) pp += tsum[q];
  int ptot;
  (void)cta_scan_i32(pp, &ptot);                      // ptot = sum of the tiles before t
  const int i0 = t * kScanTile + threadIdx.x * kPer;
  int v[kPer], sum = 0;
  if (i0 + kPer <= n) {
#pragma unroll
    for (int q = 0; q < kPer / 4; ++q) {
      const int4 a = reinterpret_cast<const int4*>(cnt + i0)[q];
      v[4 * q] = a.x; v[4 * q + 1] = a.y; v[4 * q + 2] = a.z; v[4 * q + 3] = a.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < kPer; ++q) v[q] = i0 + q < n ? cnt[i0 + q] : 0;
  }
#pragma unroll
  for (int q = 0; q < kPer; ++q) sum += v[q];
  int tot;
  int ex = cta_scan_i32(sum, &tot) + ptot;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    if (i0 + q < n) base[i0 + q] = ex;
    ex += v[q];
  }
}

// Pre-order records: quad node x starting at s sits at base[s] + cnt[s] - cc(x)
// (the nodes starting at s come top-down after every node starting before s);
// skip = the first node after its range = base[e + 1].  Thread k emits leaf k
// and internal node (split) k.
__global__ void __launch_bounds__(kSortThreads)
k_quad_emit(int N, const uint8_t* __restrict__ dl, const int4* __restrict__ nfo,
            const int32_t* __restrict__ cnt, const int32_t* __restrict__ base,
            const float2* __restrict__ ys, const longlong2* __restrict__ S,
            const BoxInfo* __restrict__ box, float4* __restrict__ nodes,
            int32_t* __restrict__ nfirst, double2* __restrict__ com64,
            int32_t* __restrict__ leafnode, int32_t* __restrict__ has_bucket) {
  pdl_trigger();
  pdl_wait();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k == 0) {
    // sentinel after the last node (the traversal parks finished lanes there):
    // a one-point leaf of count 0 whose skip is itself
    const int nn = base[N];
    nodes[nn] = make_float4(0.f, 0.f, 0.f, __uint_as_float((uint32_t)nn | ((uint32_t)kLevelLeaf << 27)));
  }
  if (k >= N) return;
  const int dprev = k > 0 ? dl[k - 1] : -1;
  const int dnext = k < N - 1 ? dl[k] : -1;
  if (max(dprev, dnext) < kKeyBits) {                 // one-point leaf
    const int pre = base[k] + cnt[k] - 1;
    const float2 y = ys[k];
    nodes[pre] = make_float4(y.x, y.y, 1.f,
                             __uint_as_float((uint32_t)base[k + 1] | ((uint32_t)kLevelLeaf << 27)));
    nfirst[pre] = k;
    com64[pre] = make_double2((double)y.x, (double)y.y);
    leafnode[k] = pre;
  }
  if (k >= N - 1) return;
  const int4 f = nfo[k];
  if (f.z < 0) return;
  const int s = f.x, e = f.y, d = dnext;
  int level;
  if (d < kKeyBits) level = qlevel(d);
  else level = (f.w < 0 || f.w <= kKeyBits - 3) ? kLevelBucketTest : kLevelBucket;   // bucket top
  const int pre = base[s] + cnt[s] - f.z;
  const uint32_t count = (uint32_t)(e - s + 1);
  const longlong2 a = S[e + 1], b = S[s];
  const double sc = __ddiv_rn(box->r0, kFixScale);
  const double mx = __ddiv_rn(__dmul_rn((double)(a.x - b.x), sc), (double)count);
  const double my = __ddiv_rn(__dmul_rn((double)(a.y - b.y), sc), (double)count);
  const double2 c64 = make_double2(__dadd_rn(box->cx, mx), __dadd_rn(box->cy, my));
  if (level >= kLevelLeaf) {
    for (int q = s; q <= e; ++q) leafnode[q] = pre;
    atomicOr(has_bucket, 1);
  }
  nodes[pre] = make_float4((float)c64.x, (float)c64.y, (float)count,
                           __uint_as_float((uint32_t)base[e + 1] | ((uint32_t)level << 27)));
  nfirst[pre] = s;
  com64[pre] = c64;
}

// ---------------------------------------------------------------- host
static inline int cdiv(int64_t a, int b) { return (int)((a + b - 1) / b); }

tsne_status build_tree(TreeWS& w, const float2* Y, bool apply_shift, cudaStream_t s) {
  const int N = (int)w.N;
  const int T = 256;
  const int ntiles = cdiv((int64_t)N + 1, kScanTile);
  k_keys<<<cdiv(N + 1, T), T, 0, s>>>(Y, N, w.box, apply_shift ? 1 : 0, w.keys_a, w.vals_a, w.cnt,
                                      w.has_bucket, w.tsum, ntiles, w.ctl);
  TSNE_LAUNCH_CHECK();
  cub::DoubleBuffer<uint64_t> dk(w.keys_a, w.keys_b);
  cub::DoubleBuffer<int32_t> dv(w.vals_a, w.vals_b);
  size_t sb = w.sort_tmp_bytes;
  TSNE_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_tmp, sb, dk, dv, N, 0, kKeyBits, s));
  w.keys_sorted = dk.Current();
  w.perm = dv.Current();
  const int nb = cdiv(N + 1, kScanBlock);
  TSNE_CUDA_TRY(launch_pdl(k_gather, nb, kScanBlock, 0, s, Y, (const int32_t*)w.perm,
                            (const uint64_t*)w.keys_sorted, N, (const BoxInfo*)w.box,
                            apply_shift ? 1 : 0, w.ys, w.fq, w.bsum, w.dl));
  TSNE_LAUNCH_CHECK();
  TSNE_CUDA_TRY(launch_pdl(k_bscan, 1, 1024, 0, s, w.bsum, nb));
  TSNE_LAUNCH_CHECK();
  TSNE_CUDA_TRY(launch_pdl(k_radix_build, nb, kScanBlock, 0, s, (const uint8_t*)w.dl, N,
                            (const uint32_t*)w.ctl, w.slot, w.nfo, w.cnt, w.tsum,
                            (const longlong2*)w.fq, (const longlong2*)w.bsum, w.S));
  TSNE_LAUNCH_CHECK();
  TSNE_CUDA_TRY(launch_pdl(k_scan_cnt, ntiles, kSortThreads, 0, s, (const int32_t*)w.cnt, N + 1,
                            w.base, (const int32_t*)w.tsum));
  TSNE_LAUNCH_CHECK();
  TSNE_CUDA_TRY(launch_pdl(k_quad_emit, cdiv(N, T), T, 0, s, N, (const uint8_t*)w.dl,
                            (const int4*)w.nfo, (const int32_t*)w.cnt, (const int32_t*)w.base,
                            (const float2*)w.ys, (const longlong2*)w.S, (const BoxInfo*)w.box,
                            w.nodes, w.nfirst, w.com64, w.leafnode, w.has_bucket));
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

}  // namespace tsne
