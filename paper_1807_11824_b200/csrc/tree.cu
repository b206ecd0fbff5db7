// tree.cu -- quadtree build over the 2-D embedding (P:L136 steps 1-4).
//
//  k_bbox        step 1: exact min/max, root box (D8)         [H1]
//  k_keys        fp64 quantisation -> 48-bit Morton key (D8, D9) [H2]
//  radix sort    (key, point id) pairs                         [H2]
//  k_gather      Y in Morton order + fixed-point coordinates + block sums
//  k_bscan       exclusive scan of the block sums (one block)
//  k_karras      binary radix tree over the sorted keys        [H3], and the
//                exclusive prefix sums of the fixed-point coordinates
//                (integers: exact, deterministic)
//  k_quad_rank   which binary nodes are quad cells; chain rank [H3]
//  scan          quad-node count per start position -> pre-order index
//  k_quad_emit   pre-order node records, counts, centres of mass [H3, H4]
//
// The compressed quadtree is derived from a Karras (2012) binary radix tree:
// a binary node whose common prefix has length delta lies in the cell of
// level L = min(delta, 48) / 2 (48-bit keys, 24 levels, D9); it is a quad
// node iff its parent's level is smaller (otherwise it merges into the
// parent).  Keys tie-break by index (delta >= 48 -> identical keys -> a
// level-24 bucket).  DESIGN.md sec. 6.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "tree.cuh"

namespace tsne {

// ---------------------------------------------------------------- workspace
struct LL2Sum {
  __host__ __device__ __forceinline__ longlong2 operator()(const longlong2& a,
                                                           const longlong2& b) const {
    return make_longlong2(a.x + b.x, a.y + b.y);
  }
};

size_t tree_cub_bytes(int64_t N, size_t* sort_b, size_t* scan_b, size_t* scan2_b) {
  size_t a = 0, b = 0, c = 0;
  cub::DoubleBuffer<uint64_t> dk(nullptr, nullptr);
  cub::DoubleBuffer<int32_t> dv(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, a, dk, dv, (int)N, 0, kKeyBits);
  cub::DeviceScan::ExclusiveSum(nullptr, c, (int32_t*)nullptr, (int32_t*)nullptr, (int)(N + 1));
  if (sort_b) *sort_b = a;
  if (scan_b) *scan_b = b;
  if (scan2_b) *scan2_b = c;
  return a + b + c;
}

void carve_tree(Carver& c, TreeWS& w, int64_t N) {
  w.N = N;
  size_t sb, cb, c2b;
  tree_cub_bytes(N, &sb, &cb, &c2b);
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
  (void)cb;
  w.bfirst = c.take<int32_t>(N);
  w.blast = c.take<int32_t>(N);
  w.bdelta = c.take<int32_t>(N);
  w.bparent = c.take<int32_t>(N);
  w.lparent = c.take<int32_t>(N);
  w.rank = c.take<int32_t>(2 * N);
  w.cnt = c.take<int32_t>(N + 1);
  w.base = c.take<int32_t>(N + 1);
  w.scan2_tmp = c.take<char>(c2b);
  w.scan2_tmp_bytes = c2b;
  w.nodes = c.take<float4>(2 * N);
  w.nfirst = c.take<int32_t>(2 * N);
  w.com64 = c.take<double2>(2 * N);
  w.leafnode = c.take<int32_t>(N);
  w.box = c.take<BoxInfo>(2);
  w.has_bucket = c.take<int32_t>(1);
  w.rep = c.take<float2>(N);
  w.zpart = c.take<double>(traverse_blocks(N));
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
                       int32_t* __restrict__ cnt, int32_t* __restrict__ has_bucket) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > N) return;
  cnt[i] = 0;
  if (i == 0) *has_bucket = 0;
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
  return TSNE_OK;
}

// ---------------------------------------------------------------- gather
constexpr int kScanBlock = 256;   // k_gather / k_karras block = prefix-sum block

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kScanBlock)
k_gather(const float2* __restrict__ Y, const int32_t* __restrict__ perm, int N,
         const BoxInfo* __restrict__ box, int apply_shift, float2* __restrict__ ys,
         longlong2* __restrict__ fq, longlong2* __restrict__ bsum) {
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

// ---------------------------------------------------------------- H3 Karras
// common-prefix length of sorted keys a, b within the kKeyBits-bit keys;
// equal keys are told apart by their index (kKeyBits + prefix of a ^ b)
// (the key of a is passed in a register: every search step of a node compares against it)
__device__ __forceinline__ int kdelta_k(const uint64_t* __restrict__ k, int N, uint64_t ka, int a,
                                        int b) {
  if ((unsigned)b >= (unsigned)N) return -1;
  const uint64_t kb = __ldg(k + b);
  if (ka != kb) return __clzll(ka ^ kb) - (64 - kKeyBits);
  return kKeyBits + __clz((uint32_t)a ^ (uint32_t)b);
}

__global__ void __launch_bounds__(kScanBlock)
k_karras(const uint64_t* __restrict__ keys, int N, int32_t* __restrict__ bfirst,
         int32_t* __restrict__ blast, int32_t* __restrict__ bdelta, int32_t* __restrict__ bparent,
         int32_t* __restrict__ lparent, const longlong2* __restrict__ fq,
         const longlong2* __restrict__ boff, longlong2* __restrict__ S) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  {
    // S[i] = boff[block] + exclusive scan of fq within the block (i <= N)
    const longlong2 v = i <= N ? fq[i] : make_longlong2(0, 0);
    long long ix = v.x, iy = v.y;                    // inclusive warp scan
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long ax = __shfl_up_sync(0xffffffffu, ix, o);
      const long long ay = __shfl_up_sync(0xffffffffu, iy, o);
      if (lane >= o) { ix += ax; iy += ay; }
    }
    __shared__ long long wx[kScanBlock / 32], wy[kScanBlock / 32];
    if (lane == 31) { wx[wid] = ix; wy[wid] = iy; }
    __syncthreads();
    long long ox = boff[blockIdx.x].x, oy = boff[blockIdx.x].y;
    for (int q = 0; q < wid; ++q) { ox += wx[q]; oy += wy[q]; }
    if (i <= N) S[i] = make_longlong2(ox + ix - v.x, oy + iy - v.y);
  }
  if (i >= N - 1) return;
  const uint64_t ki = __ldg(keys + i);
  int d = (kdelta_k(keys, N, ki, i, i + 1) - kdelta_k(keys, N, ki, i, i - 1)) >= 0 ? 1 : -1;
  int dmin = kdelta_k(keys, N, ki, i, i - d);
  int lmax = 2;
  while (kdelta_k(keys, N, ki, i, i + lmax * d) > dmin) lmax <<= 1;
  int l = 0;
  for (int t = lmax >> 1; t >= 1; t >>= 1)
    if (kdelta_k(keys, N, ki, i, i + (l + t) * d) > dmin) l += t;
  int j = i + l * d;
  int dnode = kdelta_k(keys, N, ki, i, j);
  int s = 0, t = l;
  do {
    t = (t + 1) >> 1;
    if (kdelta_k(keys, N, ki, i, i + (s + t) * d) > dnode) s += t;
  } while (t > 1);
  int gamma = i + s * d + (d < 0 ? -1 : 0);
  int lo = min(i, j), hi = max(i, j);
  bfirst[i] = lo;
  blast[i] = hi;
  bdelta[i] = dnode;
  if (lo == gamma) lparent[gamma] = i; else bparent[gamma] = i;
  if (hi == gamma + 1) lparent[gamma + 1] = i; else bparent[gamma + 1] = i;
  if (i == 0) bparent[0] = -1;
}

__device__ __forceinline__ int qlevel(int delta) {
  return (delta < kKeyBits ? delta : kKeyBits) >> 1;
}

// binary node ids: [0, N-1) internal, [N-1, 2N-1) leaves (sorted position id-(N-1))
__device__ __forceinline__ bool internal_is_quad(const int32_t* bdelta, const int32_t* bparent,
                                                 int a) {
  int p = bparent[a];
  return p < 0 || qlevel(bdelta[p]) < qlevel(bdelta[a]);
}

__global__ void k_quad_rank(int N, const int32_t* __restrict__ bfirst,
                            const int32_t* __restrict__ bdelta, const int32_t* __restrict__ bparent,
                            const int32_t* __restrict__ lparent, int32_t* __restrict__ rank,
                            int32_t* __restrict__ cnt) {
  int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= 2 * N - 1) return;
  int s, p;
  bool quad, deepest;
  if (id < N - 1) {
    s = bfirst[id];
    p = bparent[id];
    quad = internal_is_quad(bdelta, bparent, id);
    deepest = bdelta[id] >= kKeyBits;                 // bucket top
  } else {
    int k = id - (N - 1);
    s = k;
    p = lparent[k];
    quad = qlevel(bdelta[p]) < kLevels;               // not inside a bucket
    deepest = true;
  }
  if (!quad) { rank[id] = -1; return; }
  int r = 0;
  for (int a = p; a >= 0 && bfirst[a] == s; a = bparent[a])
    if (internal_is_quad(bdelta, bparent, a)) ++r;
  rank[id] = r;
  if (deepest) cnt[s] = r + 1;
}

__global__ void k_quad_emit(int N, const int32_t* __restrict__ bfirst,
                            const int32_t* __restrict__ blast, const int32_t* __restrict__ bdelta,
                            const int32_t* __restrict__ bparent, const int32_t* __restrict__ rank,
                            const int32_t* __restrict__ base, const float2* __restrict__ ys,
                            const longlong2* __restrict__ S, const BoxInfo* __restrict__ box,
                            float4* __restrict__ nodes, int32_t* __restrict__ nfirst,
                            double2* __restrict__ com64, int32_t* __restrict__ leafnode,
                            int32_t* __restrict__ has_bucket) {
  int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= 2 * N - 1) return;
  int r = rank[id];
  if (r < 0) return;
  int s, e, level;
  if (id < N - 1) {
    s = bfirst[id];
    e = blast[id];
    int dl = bdelta[id];
    if (dl < kKeyBits) {
      level = qlevel(dl);
    } else {                                          // bucket top
      int p = bparent[id];
      level = (p < 0 || bdelta[p] <= kKeyBits - 3) ? kLevelBucketTest : kLevelBucket;
    }
  } else {
    s = e = id - (N - 1);
    level = kLevelLeaf;
  }
  int pre = base[s] + r;
  int skip = base[e + 1];
  uint32_t count = (uint32_t)(e - s + 1);
  float cxf, cyf;
  double2 c64;
  if (count == 1) {
    float2 y = ys[s];
    cxf = y.x; cyf = y.y;
    c64 = make_double2((double)y.x, (double)y.y);
    leafnode[s] = pre;
  } else {
    longlong2 a = S[e + 1], b = S[s];
    const double sc = __ddiv_rn(box->r0, kFixScale);
    double mx = __ddiv_rn(__dmul_rn((double)(a.x - b.x), sc), (double)count);
    double my = __ddiv_rn(__dmul_rn((double)(a.y - b.y), sc), (double)count);
    c64 = make_double2(__dadd_rn(box->cx, mx), __dadd_rn(box->cy, my));
    cxf = (float)c64.x; cyf = (float)c64.y;
    if (level >= kLevelLeaf) {
      for (int k = s; k <= e; ++k) leafnode[k] = pre;
      atomicOr(has_bucket, 1);
    }
  }
  nodes[pre] = make_float4(cxf, cyf, (float)count,
                           __uint_as_float((uint32_t)skip | ((uint32_t)level << 27)));
  nfirst[pre] = s;
  com64[pre] = c64;
}

// ---------------------------------------------------------------- host
static inline int cdiv(int64_t a, int b) { return (int)((a + b - 1) / b); }

tsne_status build_tree(TreeWS& w, const float2* Y, bool apply_shift, cudaStream_t s) {
  const int N = (int)w.N;
  const int T = 256;
  k_keys<<<cdiv(N + 1, T), T, 0, s>>>(Y, N, w.box, apply_shift ? 1 : 0, w.keys_a, w.vals_a, w.cnt,
                                      w.has_bucket);
  TSNE_LAUNCH_CHECK();
  cub::DoubleBuffer<uint64_t> dk(w.keys_a, w.keys_b);
  cub::DoubleBuffer<int32_t> dv(w.vals_a, w.vals_b);
  size_t sb = w.sort_tmp_bytes;
  TSNE_CUDA_TRY(cub::DeviceRadixSort::SortPairs(w.sort_tmp, sb, dk, dv, N, 0, kKeyBits, s));
  w.keys_sorted = dk.Current();
  w.perm = dv.Current();
  const int nb = cdiv(N + 1, kScanBlock);
  k_gather<<<nb, kScanBlock, 0, s>>>(Y, w.perm, N, w.box, apply_shift ? 1 : 0, w.ys, w.fq, w.bsum);
  TSNE_LAUNCH_CHECK();
  k_bscan<<<1, 1024, 0, s>>>(w.bsum, nb);
  TSNE_LAUNCH_CHECK();
  k_karras<<<nb, kScanBlock, 0, s>>>(w.keys_sorted, N, w.bfirst, w.blast, w.bdelta, w.bparent,
                                      w.lparent, w.fq, w.bsum, w.S);
  TSNE_LAUNCH_CHECK();
  k_quad_rank<<<cdiv(2 * N - 1, T), T, 0, s>>>(N, w.bfirst, w.bdelta, w.bparent, w.lparent,
                                                w.rank, w.cnt);
  TSNE_LAUNCH_CHECK();
  size_t c2 = w.scan2_tmp_bytes;
  TSNE_CUDA_TRY(cub::DeviceScan::ExclusiveSum(w.scan2_tmp, c2, w.cnt, w.base, N + 1, s));
  k_quad_emit<<<cdiv(2 * N - 1, T), T, 0, s>>>(N, w.bfirst, w.blast, w.bdelta, w.bparent, w.rank,
                                                w.base, w.ys, w.S, w.box, w.nodes, w.nfirst,
                                                w.com64, w.leafnode, w.has_bucket);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

}  // namespace tsne
