// traverse.cu -- the theta-criterion traversal (Sec. III-C;
// Algorithm 1 "R-Force Computation")                       [H5, H6]
//
// Each thread handles one point of the Morton order and walks the pre-order
// node array with its own cursor (stackless: accept or finish a leaf ->
// cursor = skip; open -> cursor + 1, the first child).  Every lane therefore
// makes exactly its own accept/open decisions (D11: no "open if any lane
// needs it" voting); lanes of a warp are Morton-consecutive, so they walk
// nearly the same nodes and their 16-byte node loads share cache lines.
//
// Criterion (D7, D10): accept iff r^2 < theta^2 D^2 with r the
// half side of the cell and D the distance to its centre of mass.  Decided
// in fp32 with a proven error margin; inside the margin the decision is
// re-taken in fp64 from the cold fp64 centre of mass (D25).
// Per-point sums: z_i += N_c w, f_i += N_c w^2 (y_i - y_c), w = 1/(1+D^2)
// (P:L132 cell formula; P:L134 simultaneous Z).  Z = sum z_i in fp64 with a
// fixed reduction order (deterministic).
#include <cstdio>
#include <cstdlib>

#include "tree.cuh"

namespace tsne {

constexpr int kTravThreads = 256;
#ifndef TSNE_TRAV_MINB
#define TSNE_TRAV_MINB 6   // 40 registers, no spills: 48 warps per SM (the lockstep walk; 5: 0.362 vs 0.343 ms at C5)
#endif

// diagnostics (traverse_stats): [0] sum of node visits, [1] sum over warps
// of the warp's max visits, [2] accepted cells + exact pairs, [3] fp64 re-tests,
// [4] bucket pairs (coincident-point cells evaluated pairwise)
__device__ unsigned long long g_trav_stats[5];

int traverse_blocks(int64_t N) { return (int)((N + kTravThreads - 1) / kTravThreads); }

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}


// Exact pairs inside each point's own bucket (a level-24 cell holding several
// points, D9): every member opens its bucket (D11) and takes all pairs with
// the other members.  Done here, before the traversal, warp-synchronously:
// the lanes of a warp that share a bucket walk its members together (one
// broadcast load per member, 32 useful pairs per step), and 64-thread blocks
// spread a large bucket's members over many SMs.  (Inside the traversal each
// lane would reach its bucket at a different step and the warp would run the
// member loop once per lane group: measured 12-21 ms per traversal at
// C2/C3 early in the run, where a few thousand points share a cell.)
// Output per sorted position: the pair sums (f, z), added by k_traverse.
struct BucketSum {
  float2 f;
  double z;
};
static_assert(sizeof(BucketSum) == sizeof(longlong2), "reuses the fixed-point scratch");
constexpr int kBucketThreads = 64;

__global__ void __launch_bounds__(kBucketThreads)
k_bucket_pairs(const float4* __restrict__ nodes, const int32_t* __restrict__ nfirst,
               const float2* __restrict__ ys, const int32_t* __restrict__ leafnode, int N,
               const int32_t* __restrict__ list, const int32_t* __restrict__ nlist,
               const int32_t* __restrict__ has_bucket, BucketSum* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  if (!*has_bucket) return;                         // no bucket in this tree (k_traverse knows)
  const int nact = list ? *nlist : N;
  // grid-stride over chunks of kBucketThreads points (a small grid, so a tree
  // without buckets costs one short launch)
  for (int base = blockIdx.x * kBucketThreads; base < nact; base += gridDim.x * kBucketThreads) {
  const int tid = base + threadIdx.x;
  const bool active = tid < nact;
  const int k = active ? (list ? list[tid] : tid) : -1;
  int s0 = -1, cnt = 0;
  float2 yi = make_float2(0.f, 0.f);
  if (active) {
    const int L = leafnode[k];
    const int c = (int)__ldg(&nodes[L].z);
    if (c > 1) {
      s0 = nfirst[L];
      cnt = c;
    }
    yi = ys[k];
  }
  float fx = 0.f, fy = 0.f;
  double z = 0.0;
  unsigned todo = __ballot_sync(0xffffffffu, s0 >= 0);
  while (todo) {                                   // one shared bucket at a time
    const int ld = __ffs(todo) - 1;
    const int sb = __shfl_sync(0xffffffffu, s0, ld);
    const int cb = __shfl_sync(0xffffffffu, cnt, ld);
    const bool mine = (s0 == sb);
    todo &= ~__ballot_sync(0xffffffffu, mine);
    int m = sb;
    const int me = sb + cb;
    for (; m + 4 <= me; m += 4) {
      float zs = 0.f;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2 yj = ys[m + u];
        const float ex = yi.x - yj.x, ey = yi.y - yj.y;
        const float wj = (mine && m + u != k) ? rcp_approx(1.f + ex * ex + ey * ey) : 0.f;
        zs += wj;
        const float ww = wj * wj;
        fx = fmaf(ww, ex, fx);
        fy = fmaf(ww, ey, fy);
      }
      z += (double)zs;
    }
    for (; m < me; ++m) {
      const float2 yj = ys[m];
      const float ex = yi.x - yj.x, ey = yi.y - yj.y;
      const float wj = (mine && m != k) ? rcp_approx(1.f + ex * ex + ey * ey) : 0.f;
      z += (double)wj;
      const float ww = wj * wj;
      fx = fmaf(ww, ex, fx);
      fy = fmaf(ww, ey, fy);
    }
  }
  if (active) {
    BucketSum b;
    b.f = make_float2(fx, fy);
    b.z = z;
    out[k] = b;
  }
  }
}

constexpr int kPend = 4;   // deferred buckets per lane (registers)
constexpr int kOvf = 12;   // and beyond, in the lane's overflow list (global memory)
constexpr int kLargeBucket = 64;   // deferred buckets this large go to k_defer_large
constexpr int kLg = 16;            // per traversal thread
constexpr int kMinLockstep = 4;   // a shorter lockstep run sends the warp to the per-lane walk
constexpr int kDeepFp32 = 16;   // deeper cells: fp64 criterion and offsets


// exact pairs of point k (y_i) with the members [s0, s0 + cnt) of a bucket;
// lanes with take == false run the loop (warp-uniform trip count) adding 0
// (members in groups of 4: their loads in flight together, z summed in fp32
// per group and added to the fp64 z once per group, as k_bucket_pairs)
__device__ __forceinline__ void bucket_pairs(const float2* __restrict__ ys, int s0, int cnt, int k,
                                             float2 yi, bool take, float& fx, float& fy,
                                             double& z) {
  int m = s0;
  const int me = s0 + cnt;
  for (; m + 4 <= me; m += 4) {
    float2 yj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) yj[u] = ys[m + u];
    float zs = 0.f;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float ex = yi.x - yj[u].x, ey = yi.y - yj[u].y;
      const float wj = (take && m + u != k) ? rcp_approx(1.f + ex * ex + ey * ey) : 0.f;
      zs += wj;
      const float ww = wj * wj;
      fx = fmaf(ww, ex, fx);
      fy = fmaf(ww, ey, fy);
    }
    z += (double)zs;
  }
  for (; m < me; ++m) {
    const float2 yj = ys[m];
    const float ex = yi.x - yj.x, ey = yi.y - yj.y;
    const float wj = (take && m != k) ? rcp_approx(1.f + ex * ex + ey * ey) : 0.f;
    z += (double)wj;
    const float ww = wj * wj;
    fx = fmaf(ww, ex, fx);
    fy = fmaf(ww, ey, fy);
  }
}

template <bool STATS>
__global__ void __launch_bounds__(kTravThreads, TSNE_TRAV_MINB)
k_traverse(const float4* __restrict__ nodes, const int32_t* __restrict__ nfirst,
           const double2* __restrict__ com64, const float2* __restrict__ ys,
           const int32_t* __restrict__ leafnode, const int32_t* __restrict__ perm,
           const int32_t* __restrict__ nnodes_p, int N, const BoxInfo* __restrict__ box,
           float theta, float2* __restrict__ rep, double* __restrict__ zpart,
           unsigned* __restrict__ counter, double* __restrict__ Zout,
           const int32_t* __restrict__ list, const int32_t* __restrict__ nlist, int row0,
           const BucketSum* __restrict__ bsum, const int32_t* __restrict__ has_bucket,
           int2* __restrict__ ovf, int2* __restrict__ lg, int2* __restrict__ dlist,
           unsigned* __restrict__ dcount) {
  pdl_trigger();
  pdl_wait();
  constexpr bool stats = STATS;
  // list (multi-GPU): the sorted positions of the points this rank owns
  // (original indices [row0, ...)); rep is then indexed by perm[k] - row0.
  // Per level code l: {thr_l = r_l^2 / theta^2, C_l} (fp32) and r_l^2 (fp64).
  // The test is
  //   diff = D^2 - thr_l  >  C_l      (accept),   |diff| <= C_l  (decide in fp64).
  // Leaves of one point (24) always "accept" (the exact pair: thr = -inf);
  // bucket leaves (26) never do (thr = +inf); cells deeper than kDeepFp32
  // and bucket tests (25, r_23) always go to fp64 (C = +inf).
  __shared__ float2 s_lv[kLevelCodes];
  __shared__ double s_r2d[kLevelCodes];
  __shared__ double s_z[kTravThreads / 32];
  __shared__ int s_done;
  const double theta2d = (double)theta * (double)theta;
  if (threadIdx.x < kLevelCodes) {
    const int l = threadIdx.x;
    const int le = (l == kLevelBucketTest) ? kLevels - 1 : (l > kLevels ? kLevels : l);
    const double r = ldexp(box->r0, -le);
    const double r2 = r * r;
    const double M = (double)box->mabs, th = (double)theta;
    // Worst-case fp32 error of theta^2 D^2 - r^2:
    //   E <= 2^-24 (2.83 theta (theta D) M + 6.83 theta^2 D^2 + r^2).
    // margin = 2^-19 (r^2 + lhs) + 2^-20 theta M (r + theta D), with the
    // AM-GM bound theta D <= (lhs / r + r) / 2, i.e. margin = A + B lhs >= 4.7 E
    // (lhs = theta^2 D^2).  Divided by theta^2 (the comparison is made on
    // diff = D^2 - r^2 / theta^2, whose fp32 error is at most E / theta^2: the
    // product by theta^2 is gone, thr is rounded once): marg = A' + B D^2 with
    // A' = A / theta^2.  With D^2 = thr + diff, |diff| > C = (A' + B thr) / (1 - B)
    // implies |diff| > marg, so one constant per level decides (B < 1/2 here).
    const double A = ldexp(1.0, -19) * r2 + ldexp(1.0, -20) * th * M * r * 1.5;
    const double B = ldexp(1.0, -19) + ldexp(1.0, -21) * th * M / r;
    float thr, C;
    if (l == kLevelLeaf) {
      thr = -INFINITY; C = 0.f;
    } else if (l == kLevelBucket || theta2d == 0.0) {
      thr = INFINITY; C = 0.f;                          // never accepted (theta = 0: exact)
    } else if (l > kDeepFp32 || !(B < 0.5)) {
      thr = (float)(r2 / theta2d); C = INFINITY;
    } else {
      thr = (float)(r2 / theta2d);
      C = (float)((A / theta2d + B * (r2 / theta2d)) / (1.0 - B) * (1.0 + ldexp(1.0, -20)));
    }
    s_lv[l] = make_float2(thr, C);
    s_r2d[l] = r2;
  }
  if (threadIdx.x == 0) s_done = 0;
  __syncthreads();
  const int nnodes = *nnodes_p;
  const int tid = blockIdx.x * kTravThreads + threadIdx.x;
  const bool active = tid < (list ? *nlist : N);
  const int k = active ? (list ? list[tid] : tid) : 0;
  int cur = active ? 0 : nnodes;
  const float2 yi = active ? ys[k] : make_float2(0.f, 0.f);
  const int Li = active ? leafnode[k] : -1;
  float fx = 0.f, fy = 0.f;
  float zf = 0.f;   // per point: ~100 terms; Z = sum over points in fp64 (A.7)
  double z = 0.0;   // bucket pairs (rare) and the final per-point value

  int pq_s[kPend], pq_c[kPend];   // deferred buckets of this lane
#pragma unroll
  for (int q = 0; q < kPend; ++q) { pq_s[q] = -1; pq_c[q] = 0; }
  int npend = 0, novf = 0, nlg = 0;
  const int nthr = gridDim.x * kTravThreads;
  const int gtid = blockIdx.x * kTravThreads + threadIdx.x;
  unsigned n_visit = 0, n_take = 0, n_f64 = 0, n_pair = 0;
  // loop-invariant addresses held in registers (the compiler would otherwise
  // rematerialise them on every visit)
  uint32_t lv_base;
  asm volatile("mov.u32 %0, %1;" : "=r"(lv_base) : "r"((uint32_t)__cvta_generic_to_shared(s_lv)));
  const float4* nodes_r;
  asm volatile("mov.b64 %0, %1;" : "=l"(nodes_r) : "l"(nodes));
  // The general treatment of one visit (node cur, fp32 quantities computed):
  // inside the fp32 band, or a deep cell (its size approaches the fp32 spacing
  // of the coordinates), the decision and the offset in fp64 (D25); accept a
  // cell / take a one-point leaf unless it contains i (D11); a bucket that is
  // not accepted is evaluated pairwise (own bucket: k_bucket_pairs).
  auto visit = [&](const float4& nd, uint32_t lvl, int skip, float2 lv, float dx, float dy,
                   float D2, float diff, bool self_in) {
    bool acc = diff > lv.y;
    if (fabsf(diff) <= lv.y && !self_in) {
      const double2 c = com64[(unsigned)cur];
      const double ex = __dsub_rn((double)yi.x, c.x), ey = __dsub_rn((double)yi.y, c.y);
      const double D2d = __dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey));
      acc = s_r2d[lvl] < __dmul_rn(theta2d, D2d);
      dx = (float)ex;
      dy = (float)ey;
      D2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
      if (stats) ++n_f64;
    }
    const bool take = acc && !self_in;
    const int node = cur;
    cur = (take || lvl >= (uint32_t)kLevelLeaf) ? skip : cur + 1;
    const float w = rcp_approx(1.f + D2);
    const float nw = take ? nd.z * w : 0.f;
    if (stats && take && nd.z > 0.f) ++n_take;
    zf += nw;
    const float nww = nw * w;
    fx = fmaf(nww, dx, fx);
    fy = fmaf(nww, dy, fy);
    if (!take && !self_in && lvl > (uint32_t)kLevelLeaf) {
      const int s0 = nfirst[node];
      const int cnt = (int)nd.z;
      if (stats) n_pair += (unsigned)cnt;
      if (cnt >= kLargeBucket && nlg < kLg) {
        // a large bucket (a collapsed cluster): walked by k_defer_large, a warp
        // per point, so the few warps that hold them do not serialise the pass
        lg[(size_t)nlg * nthr + gtid] = make_int2(s0, cnt);
        ++nlg;
      } else if (npend < kPend) {      // deferred: processed warp-synchronously after the walk
#pragma unroll
        for (int q = 0; q < kPend; ++q)
          if (q == npend) { pq_s[q] = s0; pq_c[q] = cnt; }
        ++npend;
      } else if (novf < kOvf) { // (collapsed clusters: many neighbouring buckets)
        ovf[(size_t)novf * nthr + gtid] = make_int2(s0, cnt);
        ++novf;
      } else {
        bucket_pairs(ys, s0, cnt, k, yi, true, fx, fy, z);
      }
    }
  };
  // The walk, first in warp lockstep: a fast loop over the visits the fp32
  // test settles (outside the D25 band) that are not an unaccepted bucket --
  // straight-line code, warp-uniform exits (votes), so no reconvergence per
  // visit -- and, when any lane meets another kind of visit, one round of the
  // general code in which every lane still walking finishes its current
  // visit.  A lane that is done parks on the sentinel node at index nnodes (a
  // one-point leaf of count 0 whose skip is itself, k_quad_emit): it takes
  // nothing and stays there, so the fast loop needs no per-lane predicate.
  // Where such visits are frequent (deep clusters, buckets: C2/C3 early in the
  // run) a lockstep run ends within a few visits; the warp then walks on per
  // lane.
  bool lockstep = true;
  while (lockstep && __any_sync(0xffffffffu, cur < nnodes)) {
    float4 nd;
    uint32_t lvl;
    int skip;
    float2 lv;
    float dx, dy, D2, diff;
    bool self_in;
    int nfast = 0;
    for (;;) {
      if (stats && cur < nnodes) ++n_visit;
      nd = __ldg(nodes_r + (unsigned)cur);
      const uint32_t sw = __float_as_uint(nd.w);
      lvl = sw >> 27;
      skip = (int)(sw & kSkipMask);
      asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(lv.x), "=f"(lv.y) : "r"(lv_base + 8u * lvl));
      dx = yi.x - nd.x;
      dy = yi.y - nd.y;
      D2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
      self_in = (unsigned)(Li - cur) < (unsigned)(skip - cur);   // Li in [cur, skip)
      // criterion (D10) in fp32 with the D25 margin
      diff = D2 - lv.x;
      const bool acc = diff > lv.y;
      // (bitwise, not short-circuit: no branch region per visit)
      const int rare = (int)!self_in &
                       ((int)(fabsf(diff) <= lv.y) | ((int)(lvl > (uint32_t)kLevelLeaf) & (int)!acc));
      if (__any_sync(0xffffffffu, rare)) break;
      const bool take = (int)acc & (int)!self_in;
      cur = ((int)take | (int)(lvl >= (uint32_t)kLevelLeaf)) ? skip : cur + 1;
      const float w = rcp_approx(1.f + D2);
      const float nw = take ? nd.z * w : 0.f;
      if (stats && take && nd.z > 0.f) ++n_take;
      zf += nw;
      const float nww = nw * w;
      fx = fmaf(nww, dx, fx);
      fy = fmaf(nww, dy, fy);
      ++nfast;
      if (!__any_sync(0xffffffffu, cur < nnodes)) break;
    }
    if (cur < nnodes) visit(nd, lvl, skip, lv, dx, dy, D2, diff, self_in);
    lockstep = nfast >= kMinLockstep;                  // warp-uniform
  }
  while (cur < nnodes) {
    if (stats) ++n_visit;
    const float4 nd = __ldg(nodes_r + (unsigned)cur);
    const uint32_t sw = __float_as_uint(nd.w);
    const uint32_t lvl = sw >> 27;
    const int skip = (int)(sw & kSkipMask);
    float2 lv;
    asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(lv.x), "=f"(lv.y) : "r"(lv_base + 8u * lvl));
    const float dx = yi.x - nd.x, dy = yi.y - nd.y;
    const float D2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
    const bool self_in = (unsigned)(Li - cur) < (unsigned)(skip - cur);
    visit(nd, lvl, skip, lv, dx, dy, D2, D2 - lv.x, self_in);
  }
  z += (double)zf;
  // Deferred buckets: lanes of the warp that share a bucket walk its members
  // together (a lane reaches a bucket at its own step of the walk, so doing it
  // in place would run the member loop once per lane group).
  while (true) {
    const unsigned ball = __ballot_sync(0xffffffffu, npend > 0);
    if (!ball) break;
    const int ld = __ffs(ball) - 1;
    const int sb = __shfl_sync(0xffffffffu, pq_s[0], ld);
    const int cb = __shfl_sync(0xffffffffu, pq_c[0], ld);
    bool mine = false;
#pragma unroll
    for (int q = 0; q < kPend; ++q) mine |= (q < npend) && (pq_s[q] == sb);
    bucket_pairs(ys, sb, cb, k, yi, mine, fx, fy, z);
    if (mine) {                 // drop sb from this lane's list (order kept)
      int ns = 0;
      int ts[kPend], tc[kPend];
#pragma unroll
      for (int q = 0; q < kPend; ++q) { ts[q] = 0; tc[q] = 0; }
#pragma unroll
      for (int q = 0; q < kPend; ++q) {
        if (q < npend && pq_s[q] != sb) {
#pragma unroll
          for (int r = 0; r < kPend; ++r)
            if (r == ns) { ts[r] = pq_s[q]; tc[r] = pq_c[q]; }
          ++ns;
        }
      }
#pragma unroll
      for (int q = 0; q < kPend; ++q) { pq_s[q] = ts[q]; pq_c[q] = tc[q]; }
      npend = ns;
    }
  }
  // the overflow lists, the same way (each lane's buckets are in one list or
  // the other, so each is walked once for it)
  while (true) {
    __syncwarp();
    const unsigned ball = __ballot_sync(0xffffffffu, novf > 0);
    if (!ball) break;
    const int2 e = ovf[gtid - (threadIdx.x & 31) + __ffs(ball) - 1];   // its first entry
    bool mine = false;
    for (int q = 0; q < novf; ++q) mine |= ovf[(size_t)q * nthr + gtid].x == e.x;
    bucket_pairs(ys, e.x, e.y, k, yi, mine, fx, fy, z);
    __syncwarp();
    if (mine) {
      int ns = 0;
      for (int q = 0; q < novf; ++q) {
        const int2 v = ovf[(size_t)q * nthr + gtid];
        if (v.x != e.x) ovf[(size_t)(ns++) * nthr + gtid] = v;
      }
      novf = ns;
    }
  }
  if (nlg > 0) dlist[atomicAdd(dcount, 1u)] = make_int2(gtid, nlg);
  if (active) {
    if (*has_bucket) {
      const BucketSum b = bsum[k];
      fx += b.f.x;
      fy += b.f.y;
      z += b.z;
    }
    rep[perm[k] - row0] = make_float2(fx, fy);
  }
  if (stats) {
    unsigned long long sv = n_visit, st = n_take, sf = n_f64, sp = n_pair;
    unsigned mv = n_visit;
    for (int o = 16; o > 0; o >>= 1) {
      sv += __shfl_xor_sync(0xffffffffu, sv, o);
      st += __shfl_xor_sync(0xffffffffu, st, o);
      sf += __shfl_xor_sync(0xffffffffu, sf, o);
      sp += __shfl_xor_sync(0xffffffffu, sp, o);
      mv = max(mv, __shfl_xor_sync(0xffffffffu, mv, o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(&g_trav_stats[0], sv);
      atomicAdd(&g_trav_stats[1], (unsigned long long)mv * 32ull);
      atomicAdd(&g_trav_stats[2], st);
      atomicAdd(&g_trav_stats[3], sf);
      atomicAdd(&g_trav_stats[4], sp);
    }
  }

  // Z: fixed-order fp64 reduction without a block barrier: the last warp of
  // the block to finish sums the block, the last block sums the blocks.
  const double zw = warp_sum(z);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int last_block = 0;
  if (lane == 0) {
    s_z[wid] = zw;
    __threadfence_block();
    const int prev = atomicAdd(&s_done, 1);
    if (prev == kTravThreads / 32 - 1) {
      __threadfence_block();
      double t = 0.0;
      for (int q = 0; q < kTravThreads / 32; ++q) t += ((volatile double*)s_z)[q];
      zpart[blockIdx.x] = t;
      __threadfence();
      const unsigned g = atomicAdd(counter, 1u);
      last_block = (g == gridDim.x - 1);
    }
  }
  last_block = __shfl_sync(0xffffffffu, last_block, 0);
  if (last_block) {
    __threadfence();
    double t = 0.0;
    for (int q = lane; q < (int)gridDim.x; q += 32) t += __ldcg(zpart + q);
    t = warp_sum(t);
    if (lane == 0) {
      Zout[0] = t;
      Zout[1] = 1.0 / t;
      *counter = 0u;
    }
  }
}

// The large deferred buckets of the traversal threads in the list (k_traverse
// appends them): one warp per thread, its buckets in list order, lanes over the
// members; each bucket's sums are reduced by a fixed butterfly and added in
// order, then added to the point's repulsive numerator.  The z terms enter Z
// through an exact fixed-point sum (integer part and 2^-32 units: integers, so
// the order of the warps does not matter), folded into Z and 1/Z by the last
// CTA, which also resets the list.
constexpr int kDeferThreads = 128;
__global__ void __launch_bounds__(kDeferThreads)
k_defer_large(const float2* __restrict__ ys, const int32_t* __restrict__ perm,
              const int32_t* __restrict__ list, int row0, const int2* __restrict__ lg, int nthr,
              const int2* __restrict__ dlist, unsigned* __restrict__ dcount,
              float2* __restrict__ rep, double* __restrict__ Zout,
              unsigned long long* __restrict__ zacc, unsigned* __restrict__ done) {
  pdl_trigger();
  pdl_wait();
  __shared__ bool last;
  const int lane = threadIdx.x & 31;
  const int n = (int)*dcount;
  const int wpb = kDeferThreads / 32;
  for (int it = blockIdx.x * wpb + (threadIdx.x >> 5); it < n; it += gridDim.x * wpb) {
    const int2 e = dlist[it];
    const int gtid = e.x, ne = e.y;
    const int k = list ? list[gtid] : gtid;
    const float2 yi = ys[k];
    float tx = 0.f, ty = 0.f;
    double tz = 0.0;
    for (int q = 0; q < ne; ++q) {
      const int2 b = lg[(size_t)q * nthr + gtid];
      float fx = 0.f, fy = 0.f, zs = 0.f;
      for (int m = b.x + lane; m < b.x + b.y; m += 32) {
        const float2 yj = ys[m];
        const float ex = yi.x - yj.x, ey = yi.y - yj.y;
        const float wj = m != k ? rcp_approx(1.f + ex * ex + ey * ey) : 0.f;
        zs += wj;
        const float ww = wj * wj;
        fx = fmaf(ww, ex, fx);
        fy = fmaf(ww, ey, fy);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        fx += __shfl_xor_sync(0xffffffffu, fx, o);
        fy += __shfl_xor_sync(0xffffffffu, fy, o);
        zs += __shfl_xor_sync(0xffffffffu, zs, o);
      }
      tx += fx;
      ty += fy;
      tz += (double)zs;
    }
    if (lane == 0) {
      float2* r = rep + (perm[k] - row0);
      const float2 v = *r;
      *r = make_float2(v.x + tx, v.y + ty);
      // exact in two words: the integer part (z <= 16 N per point, so the sum
      // over points stays below 2^63 for N < 2^25) and 2^-32 units of the rest
      const double zi = floor(tz);
      atomicAdd(zacc, (unsigned long long)zi);
      atomicAdd(zacc + 1, (unsigned long long)__double2ll_rn((tz - zi) * 4294967296.0));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    const unsigned long long ai = *(volatile unsigned long long*)zacc;
    const unsigned long long af = *(volatile unsigned long long*)(zacc + 1);
    if (ai | af) {
      const double Z = Zout[0] + ((double)ai + (double)af * (1.0 / 4294967296.0));
      Zout[0] = Z;
      Zout[1] = 1.0 / Z;
    }
    zacc[0] = 0ull;
    zacc[1] = 0ull;
    *dcount = 0u;
    *done = 0u;
  }
}

static tsne_status launch_defer_large(TreeWS& w, const int32_t* list, int row0, float2* rep,
                                      double* Zout, cudaStream_t s) {
  TSNE_CUDA_TRY(launch_pdl(k_defer_large, 2 * kNumSMs, kDeferThreads, 0, s, (const float2*)w.ys,
                            (const int32_t*)w.perm, list, row0, (const int2*)w.lg,
                            traverse_blocks(w.N) * kTravThreads, (const int2*)w.dlist,
                            w.counter + 5, rep, Zout, w.zacc, w.counter + 4));
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

static tsne_status launch_bucket_pairs(TreeWS& w, const int32_t* list, const int32_t* nlist,
                                       cudaStream_t s) {
  const int N = (int)w.N;
  // the fixed-point coordinates are dead after the tree build: reuse them
  const int nb = (N + kBucketThreads - 1) / kBucketThreads;
  TSNE_CUDA_TRY(launch_pdl(k_bucket_pairs, nb < 16 * kNumSMs ? nb : 16 * kNumSMs, kBucketThreads,
                            0, s, (const float4*)w.nodes, (const int32_t*)w.nfirst,
                            (const float2*)w.ys, (const int32_t*)w.leafnode, N, list, nlist,
                            (const int32_t*)w.has_bucket, reinterpret_cast<BucketSum*>(w.fq)));
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

tsne_status launch_traverse(TreeWS& w, float theta, cudaStream_t s) {
  const int N = (int)w.N;
  tsne_status st = launch_bucket_pairs(w, nullptr, nullptr, s);
  if (st != TSNE_OK) return st;
  TSNE_CUDA_TRY(launch_pdl(k_traverse<false>, traverse_blocks(N), kTravThreads, 0, s,
      w.nodes, w.nfirst, w.com64, w.ys, w.leafnode, w.perm, w.base + N, N, w.box, theta, w.rep,
      w.zpart, w.counter + 1, w.Z, nullptr, nullptr, 0,
      reinterpret_cast<const BucketSum*>(w.fq), w.has_bucket, w.ovf, w.lg, w.dlist, w.counter + 5));
  TSNE_LAUNCH_CHECK();
  return launch_defer_large(w, nullptr, 0, w.rep, w.Z, s);
}

// The same traversal with per-point counters (measurement only; synchronises s):
// out[0] node visits, [1] sum over warps of the warp's largest visit count (the
// SIMT cost), [2] interactions (accepted cells + exact pairs), [3] fp64
// re-decisions (D25 band and deep cells), [4] bucket pairs -- each per point.
tsne_status traverse_stats(TreeWS& w, float theta, double* out, cudaStream_t s) {
  const int N = (int)w.N;
  const unsigned long long zero[5] = {0, 0, 0, 0, 0};
  TSNE_CUDA_TRY(cudaMemcpyToSymbolAsync(g_trav_stats, zero, sizeof(zero), 0,
                                        cudaMemcpyHostToDevice, s));
  tsne_status st = launch_bucket_pairs(w, nullptr, nullptr, s);
  if (st != TSNE_OK) return st;
  TSNE_CUDA_TRY(launch_pdl(k_traverse<true>, traverse_blocks(N), kTravThreads, 0, s,
      w.nodes, w.nfirst, w.com64, w.ys, w.leafnode, w.perm, w.base + N, N, w.box, theta, w.rep,
      w.zpart, w.counter + 1, w.Z, nullptr, nullptr, 0,
      reinterpret_cast<const BucketSum*>(w.fq), w.has_bucket, w.ovf, w.lg, w.dlist, w.counter + 5));
  TSNE_LAUNCH_CHECK();
  if ((st = launch_defer_large(w, nullptr, 0, w.rep, w.Z, s)) != TSNE_OK) return st;
  unsigned long long h[5];
  TSNE_CUDA_TRY(cudaMemcpyFromSymbolAsync(h, g_trav_stats, sizeof(h), 0, cudaMemcpyDeviceToHost, s));
  TSNE_CUDA_TRY(cudaStreamSynchronize(s));
  for (int k = 0; k < 5; ++k) out[k] = (double)h[k] / (double)N;
  return TSNE_OK;
}

// multi-GPU: traverse only the listed sorted positions (owned points)
tsne_status launch_traverse_list(TreeWS& w, float theta, const int32_t* list, const int32_t* nlist,
                                 int row0, float2* rep_local, double* z_partial, cudaStream_t s) {
  const int N = (int)w.N;
  tsne_status st = launch_bucket_pairs(w, list, nlist, s);
  if (st != TSNE_OK) return st;
  TSNE_CUDA_TRY(launch_pdl(k_traverse<false>, traverse_blocks(N), kTravThreads, 0, s,
      w.nodes, w.nfirst, w.com64, w.ys, w.leafnode, w.perm, w.base + N, N, w.box, theta,
      rep_local, w.zpart, w.counter + 1, z_partial, list, nlist, row0,
      reinterpret_cast<const BucketSum*>(w.fq), w.has_bucket, w.ovf, w.lg, w.dlist, w.counter + 5));
  TSNE_LAUNCH_CHECK();
  return launch_defer_large(w, list, row0, rep_local, z_partial, s);
}

}  // namespace tsne
