// traverse.cu -- the theta-criterion traversal (Sec. III-C;
// Algorithm 1 "R-Force Computation")                       [H5, H6]
//
// One warp handles 32 consecutive points of the Morton order.  Each lane
// keeps its own cursor into the pre-order node array; the warp visits the
// smallest cursor of its lanes each step (one broadcast 16-byte node load),
// and only lanes whose cursor equals that node act on it.  Every lane
// therefore makes exactly its own accept/open decisions (D11: no "open if
// any lane needs it" voting), while lanes of a spatially coherent warp share
// node loads.  Accepting or finishing a leaf moves the cursor to `skip`;
// opening moves it to node + 1 (the first child).
//
// Criterion (D7, D10): accept iff r^2 < theta^2 D^2 with r the
// half side of the cell and D the distance to its centre of mass.  Decided
// in fp32 with a proven error margin; inside the margin the decision is
// re-taken in fp64 from the cold fp64 centre of mass (D25).
// Per-point sums: z_i += N_c w, f_i += N_c w^2 (y_i - y_c), w = 1/(1+D^2)
// (P:L132 cell formula; P:L134 simultaneous Z).  Z = sum z_i in fp64 with a
// fixed reduction order (deterministic).
#include "tree.cuh"

namespace tsne {

constexpr int kTravThreads = 256;

int traverse_blocks(int64_t N) { return (int)((N + kTravThreads - 1) / kTravThreads); }

__global__ void __launch_bounds__(kTravThreads)
k_traverse(const float4* __restrict__ nodes, const int32_t* __restrict__ nfirst,
           const double2* __restrict__ com64, const float2* __restrict__ ys,
           const int32_t* __restrict__ leafnode, const int32_t* __restrict__ perm,
           const int32_t* __restrict__ nnodes_p, int N, const BoxInfo* __restrict__ box,
           float theta, float2* __restrict__ rep, double* __restrict__ zpart,
           unsigned* __restrict__ counter, double* __restrict__ Zout) {
  __shared__ float s_r2[18], s_marg[18];
  __shared__ double s_r2d[18];
  __shared__ double s_z[kTravThreads / 32];
  __shared__ bool s_last;
  const float theta2 = theta * theta;
  const double theta2d = (double)theta * (double)theta;
  if (threadIdx.x < 18) {
    int l = threadIdx.x;
    int le = (l == kLevelBucketTest) ? 15 : (l > 16 ? 16 : l);
    double r = ldexp(box->r0, -le);
    double r2 = r * r;
    s_r2d[l] = r2;
    s_r2[l] = (float)r2;
    // error bound of the fp32 test:
    //   |diff_fp32 - (theta^2 D^2 - r^2)| <= 2^-24 (2.83 theta D mabs theta + 6.83 theta^2 D^2 + r^2)
    // margin = 2^-19 (r^2 + lhs) + 2^-20 theta mabs (r + theta D)  (>= 4.7x the bound)
    s_marg[l] = (float)(ldexp(1.0, -19) * r2 + ldexp(1.0, -20) * (double)theta * (double)box->mabs * r);
  }
  __syncthreads();
  const int nnodes = *nnodes_p;
  const float c2 = (float)(ldexp(1.0, -20) * (double)theta * (double)box->mabs);
  const int k = blockIdx.x * kTravThreads + threadIdx.x;
  const bool active = k < N;
  int cur = active ? 0 : nnodes;
  float2 yi = active ? ys[k] : make_float2(0.f, 0.f);
  const int Li = active ? leafnode[k] : -1;
  float fx = 0.f, fy = 0.f;
  double z = 0.0;   // fp64: Z sums up to N^2 terms of very different size

  while (true) {
    const int node = (int)__reduce_min_sync(0xffffffffu, (unsigned)cur);
    if (node >= nnodes) break;
    const float4 nd = __ldg(nodes + node);
    if (cur == node) {
      const uint32_t wv = __float_as_uint(nd.z);
      const int cnt = (int)(wv & kCountMask);
      const int lvl = (int)(wv >> 27);
      const int skip = __float_as_int(nd.w);
      int next = skip;
      bool exact = false;
      if (lvl == kLevelLeaf) {
        exact = true;
      } else if (Li >= node && Li < skip) {        // the cell contains point i (D11)
        if (lvl == kLevelBucketTest) exact = true; else next = node + 1;
      } else {
        const float dx = yi.x - nd.x, dy = yi.y - nd.y;
        const float D2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
        const float lhs = __fmul_rn(theta2, D2);
        const float diff = lhs - s_r2[lvl];
        const float marg = s_marg[lvl] + 1.9073486e-6f * lhs + c2 * sqrtf(lhs);
        bool acc;
        if (diff > marg) {
          acc = true;
        } else if (diff < -marg) {
          acc = false;
        } else {                                   // fp64 re-test (D25)
          const double2 c = com64[node];
          const double ex = __dsub_rn((double)yi.x, c.x), ey = __dsub_rn((double)yi.y, c.y);
          const double D2d = __dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey));
          acc = s_r2d[lvl] < __dmul_rn(theta2d, D2d);
        }
        if (acc) {
          const float w = __frcp_rn(1.f + D2);
          const float nw = (float)cnt * w;
          z += (double)nw;
          const float nww = nw * w;
          fx = fmaf(nww, dx, fx);
          fy = fmaf(nww, dy, fy);
        } else if (lvl == kLevelBucketTest) {
          exact = true;
        } else {
          next = node + 1;
        }
      }
      if (exact) {
        if (cnt == 1) {
          if (Li != node) {
            const float dx = yi.x - nd.x, dy = yi.y - nd.y;
            const float w = __frcp_rn(1.f + dx * dx + dy * dy);
            z += (double)w;
            const float ww = w * w;
            fx = fmaf(ww, dx, fx);
            fy = fmaf(ww, dy, fy);
          }
        } else {
          const int s0 = nfirst[node];
          for (int m = s0; m < s0 + cnt; ++m) {
            if (m == k) continue;
            const float2 yj = ys[m];
            const float dx = yi.x - yj.x, dy = yi.y - yj.y;
            const float w = __frcp_rn(1.f + dx * dx + dy * dy);
            z += (double)w;
            const float ww = w * w;
            fx = fmaf(ww, dx, fx);
            fy = fmaf(ww, dy, fy);
          }
        }
      }
      cur = next;
    }
  }
  if (active) rep[perm[k]] = make_float2(fx, fy);

  // Z partial: fixed-order fp64 reduction (deterministic)
  double zd = warp_sum(z);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_z[wid] = zd;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < kTravThreads / 32; ++q) t += s_z[q];
    zpart[blockIdx.x] = t;
    __threadfence();
    unsigned prev = atomicAdd(counter, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last && wid == 0) {
    __threadfence();
    double t = 0.0;
    for (int q = lane; q < (int)gridDim.x; q += 32) t += ((volatile double*)zpart)[q];
    t = warp_sum(t);
    if (lane == 0) {
      Zout[0] = t;
      Zout[1] = 1.0 / t;
      *counter = 0u;
    }
  }
}

tsne_status launch_traverse(TreeWS& w, float theta, cudaStream_t s) {
  const int N = (int)w.N;
  k_traverse<<<traverse_blocks(N), kTravThreads, 0, s>>>(
      w.nodes, w.nfirst, w.com64, w.ys, w.leafnode, w.perm, w.base + N, N, w.box, theta, w.rep,
      w.zpart, w.counter + 1, w.Z);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

}  // namespace tsne
