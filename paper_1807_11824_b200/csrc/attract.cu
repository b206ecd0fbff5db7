// attract.cu -- attractive forces from the sparse P (Eq. 5; the
// nonzero iteration of Sec. III-B: "P (.) Q is computed directly
// by iterating over nonzero values of P"), fused with the gradient assembly
// (Eq. 7) and, in the optimiser, with the update ("Apply Forces",
// Algorithm 1 line 8).                                      [H7, H8]
//
// One warp per CSR row: lanes stride the row's nonzeros (coalesced col/val
// stream, read once -> evict-first), gather y_j (the 8-byte-per-point
// embedding stays L2-resident), and reduce with a fixed butterfly.
//   A_i = sum_j P_ij (y_i - y_j) / (1 + |y_i - y_j|^2)      (q_ij Z, D1/D5)
//   g_i = 4 (alpha A_i - f_i / Z)
// The update kernel also produces the next iteration's recentring shift and
// bounding box (fixed-order last-block reduction), so the tree build of the
// next iteration needs no separate bbox pass.
#include "optimize.cuh"

namespace tsne {

constexpr int kAttrThreads = 256;
constexpr int kAttrWarps = kAttrThreads / 32;
constexpr int kAttrBlocksPerSM = 4;

// One warp per row.  The row's nonzeros are read as 16-byte vectors from the
// 16-byte-aligned window around [e0, e1) (lanes masked outside the row), so
// each lane has 4 independent y_j gathers in flight per vector; the row sum is
// reduced with a fixed butterfly (deterministic).
__device__ __forceinline__ float2 row_attractive(const int64_t e0, const int64_t e1,
                                                 const int64_t nnz,
                                                 const int32_t* __restrict__ col,
                                                 const float* __restrict__ val,
                                                 const float2* __restrict__ Y, int i, float2 yi,
                                                 int lane) {
  float ax = 0.f, ay = 0.f;
  for (int64_t b = (e0 & ~int64_t(3)) + 4 * lane; b < e1; b += 128) {
    int c[4];
    float p[4];
    if (b + 3 < nnz) {
      const int4 cv = __ldcs(reinterpret_cast<const int4*>(col + b));
      const float4 pv = __ldcs(reinterpret_cast<const float4*>(val + b));
      c[0] = cv.x; c[1] = cv.y; c[2] = cv.z; c[3] = cv.w;
      p[0] = pv.x; p[1] = pv.y; p[2] = pv.z; p[3] = pv.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool ok = b + q < nnz;
        c[q] = ok ? __ldcs(col + b + q) : i;
        p[q] = ok ? __ldcs(val + b + q) : 0.f;
      }
    }
    float2 yj[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool in = (b + q >= e0) && (b + q < e1);
      if (!in) { c[q] = i; p[q] = 0.f; }
      yj[q] = Y[c[q]];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float dx = yi.x - yj[q].x, dy = yi.y - yj[q].y;
      const float w = __frcp_rn(1.f + dx * dx + dy * dy);
      const float pw = p[q] * w;
      ax = fmaf(pw, dx, ax);
      ay = fmaf(pw, dy, ay);
    }
  }
  return make_float2(warp_sum(ax), warp_sum(ay));
}

// tsne_gradient: dY = 4 (alpha A - f / Z)
__global__ void __launch_bounds__(kAttrThreads)
k_attract_grad(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
               const float* __restrict__ val, const float2* __restrict__ Y, int N,
               const float2* __restrict__ rep, const double* __restrict__ Z, float alpha,
               float2* __restrict__ dY) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * kAttrThreads + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * kAttrThreads) >> 5;
  const float invZ = (float)Z[1];
  const int64_t nnz = row_ptr[N];
  for (int i = warp; i < N; i += nwarps) {
    const float2 yi = Y[i];
    const float2 a = row_attractive(row_ptr[i], row_ptr[i + 1], nnz, col, val, Y, i, yi, lane);
    if (lane == 0) {
      const float2 f = rep[i];
      dY[i] = make_float2(4.f * (alpha * a.x - f.x * invZ), 4.f * (alpha * a.y - f.y * invZ));
    }
  }
}

__device__ __forceinline__ float sgnf(float x) { return (float)((x > 0.f) - (x < 0.f)); }

// optimiser step for one coordinate (D12): gains, momentum, learning rate
__device__ __forceinline__ void update_coord(float g, float& v, float& gain, float& y, float mu,
                                             float eta, float min_gain) {
  float gn = (sgnf(g) != sgnf(v)) ? gain + 0.2f : gain * 0.8f;
  gn = fmaxf(gn, min_gain);
  gain = gn;
  v = mu * v - eta * gn * g;
  y = y + v;
}

// Attractive sums only (H7): A_i for every row, written to A.  Independent of
// the tree, the traversal and Z, so it runs concurrently with them on a side
// stream; reads the unshifted Y (differences only).
__global__ void __launch_bounds__(kAttrThreads)
k_attract_sum(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
              const float* __restrict__ val, const float2* __restrict__ Y, int N,
              float2* __restrict__ A) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * kAttrThreads + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * kAttrThreads) >> 5;
  const int64_t nnz = row_ptr[N];
  for (int i = warp; i < N; i += nwarps) {
    const float2 yi = Y[i];
    const float2 a = row_attractive(row_ptr[i], row_ptr[i + 1], nnz, col, val, Y, i, yi, lane);
    if (lane == 0) A[i] = a;
  }
}

// The update (H8): Eq. 7 with the traversal's f and Z, the D12 step, the
// pending recentring (y - shift, D15), Y' = y + v; per-block fp64 sums and
// min/max of Y' give the next iteration's shift and root box (last block).
__global__ void __launch_bounds__(kAttrThreads)
k_update(const float2* __restrict__ Yin, const float2* __restrict__ A, int N,
         const float2* __restrict__ rep, const double* __restrict__ Z, int32_t* __restrict__ t_dev,
         Sched sc, float2* __restrict__ Yout, float2* __restrict__ V, float2* __restrict__ G,
         double2* __restrict__ part2, float4* __restrict__ part4, unsigned* __restrict__ counter,
         BoxInfo* __restrict__ box, int32_t* __restrict__ flag) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int t = *t_dev;
  const float alpha = (t < sc.exag_iters) ? sc.exag : 1.f;
  const float mu = (t < sc.exag_iters) ? sc.mom0 : sc.mom1;
  const float invZ = (float)Z[1];
  const float shx = box->shift_x, shy = box->shift_y;   // read before the block arrives
  double sx = 0.0, sy = 0.0;
  float mnx = INFINITY, mxx = -INFINITY, mny = INFINITY, mxy = -INFINITY;
  bool bad = false;
  for (int i = blockIdx.x * kAttrThreads + threadIdx.x; i < N; i += gridDim.x * kAttrThreads) {
    const float2 a = A[i], f = rep[i];
    float2 v = V[i], gn = G[i], y = Yin[i];
    y.x = y.x - shx;
    y.y = y.y - shy;
    const float gx = 4.f * (alpha * a.x - f.x * invZ);
    const float gy = 4.f * (alpha * a.y - f.y * invZ);
    update_coord(gx, v.x, gn.x, y.x, mu, sc.eta, sc.min_gain);
    update_coord(gy, v.y, gn.y, y.y, mu, sc.eta, sc.min_gain);
    V[i] = v;
    G[i] = gn;
    Yout[i] = y;
    sx += (double)y.x;
    sy += (double)y.y;
    mnx = fminf(mnx, y.x); mxx = fmaxf(mxx, y.x);
    mny = fminf(mny, y.y); mxy = fmaxf(mxy, y.y);
    bad |= !(isfinite(y.x) && isfinite(y.y));
  }
  sx = warp_sum(sx);
  sy = warp_sum(sy);
  mnx = warp_min(mnx); mxx = warp_max(mxx);
  mny = warp_min(mny); mxy = warp_max(mxy);
  bad = __any_sync(0xffffffffu, bad);
  __shared__ double2 s_s[kAttrThreads];
  __shared__ float4 s_b[kAttrThreads];
  __shared__ bool s_last;
  if (lane == 0) {
    s_s[wid] = make_double2(sx, sy);
    s_b[wid] = make_float4(mnx, mxx, mny, mxy);
  }
  if (bad && lane == 0) *flag = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 ss = s_s[0];
    float4 bb = s_b[0];
    for (int q = 1; q < kAttrWarps; ++q) {
      ss.x += s_s[q].x; ss.y += s_s[q].y;
      bb.x = fminf(bb.x, s_b[q].x); bb.y = fmaxf(bb.y, s_b[q].y);
      bb.z = fminf(bb.z, s_b[q].z); bb.w = fmaxf(bb.w, s_b[q].w);
    }
    part2[blockIdx.x] = ss;
    part4[blockIdx.x] = bb;
    __threadfence();
    unsigned prev = atomicAdd(counter, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  // last block: fixed-order reduction of the per-block partials (deterministic)
  __threadfence();
  double2 ss = make_double2(0.0, 0.0);
  float4 bb = make_float4(INFINITY, -INFINITY, INFINITY, -INFINITY);
  for (int q = threadIdx.x; q < (int)gridDim.x; q += kAttrThreads) {
    const double2 a = __ldcg(part2 + q);
    const float4 b = __ldcg(part4 + q);
    ss.x += a.x; ss.y += a.y;
    bb.x = fminf(bb.x, b.x); bb.y = fmaxf(bb.y, b.y);
    bb.z = fminf(bb.z, b.z); bb.w = fmaxf(bb.w, b.w);
  }
  s_s[threadIdx.x] = ss;
  s_b[threadIdx.x] = bb;
  __syncthreads();
  for (int o = kAttrThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double2 a = s_s[threadIdx.x + o];
      const float4 b = s_b[threadIdx.x + o];
      s_s[threadIdx.x].x += a.x; s_s[threadIdx.x].y += a.y;
      float4& c = s_b[threadIdx.x];
      c.x = fminf(c.x, b.x); c.y = fmaxf(c.y, b.y); c.z = fminf(c.z, b.z); c.w = fmaxf(c.w, b.w);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ss = s_s[0];
    bb = s_b[0];
    // recentring (D15): y <- y - mean, applied by the next iteration; by the
    // monotonicity of rounding, min(fl(y - m)) = fl(min(y) - m) exactly.
    const float mx = (float)(ss.x / (double)N), my = (float)(ss.y / (double)N);
    BoxInfo b;
    make_root_box(bb.x - mx, bb.y - mx, bb.z - my, bb.w - my, &b);
    b.shift_x = mx;
    b.shift_y = my;
    b.pad0 = 0.f;
    *box = b;
    *t_dev = t + 1;
    *counter = 0u;
  }
}

int attract_blocks(int64_t N) {
  int64_t b = (N + kAttrWarps - 1) / kAttrWarps;
  int64_t cap = (int64_t)kNumSMs * kAttrBlocksPerSM;
  return (int)(b < cap ? (b < 1 ? 1 : b) : cap);
}

tsne_status launch_attract_grad(const int64_t* row_ptr, const int32_t* col, const float* val,
                                const float2* Y, int64_t N, const float2* rep, const double* Z,
                                float alpha, float2* dY, cudaStream_t s) {
  k_attract_grad<<<attract_blocks(N), kAttrThreads, 0, s>>>(row_ptr, col, val, Y, (int)N, rep, Z,
                                                            alpha, dY);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

int update_blocks(int64_t N) {
  int64_t b = (N + kAttrThreads - 1) / kAttrThreads;
  int64_t cap = (int64_t)kNumSMs * 8;
  return (int)(b < cap ? (b < 1 ? 1 : b) : cap);
}

tsne_status launch_attract_sum(const int64_t* row_ptr, const int32_t* col, const float* val,
                               const float2* Y, int64_t N, float2* A, cudaStream_t s) {
  k_attract_sum<<<attract_blocks(N), kAttrThreads, 0, s>>>(row_ptr, col, val, Y, (int)N, A);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

tsne_status launch_update(const float2* Yin, const float2* A, int64_t N, TreeWS& w, OptWS& o,
                          const Sched& sc, float2* Yout, float2* V, float2* G, cudaStream_t s) {
  k_update<<<update_blocks(N), kAttrThreads, 0, s>>>(Yin, A, (int)N, w.rep, w.Z, o.t_dev, sc, Yout,
                                                     V, G, w.part2, w.part4, w.counter + 2, w.box,
                                                     o.flag);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

}  // namespace tsne

namespace tsne {

// ---------------------------------------------------------------- multi-GPU
// Rows [row0, row0 + n_local) of this rank: attractive pass against the full
// replicated embedding, Eq. 7 with Z = the ranks' partial sums added in rank
// order (deterministic), and the D12 update into the local shard.
__global__ void __launch_bounds__(kAttrThreads)
k_attract_sum_shard(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                    const float* __restrict__ val, const float2* __restrict__ Y, int row0,
                    int n_local, float2* __restrict__ A) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * kAttrThreads + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * kAttrThreads) >> 5;
  const int64_t nnz = row_ptr[n_local];
  for (int l = warp; l < n_local; l += nwarps) {
    const int i = row0 + l;
    const float2 a = row_attractive(row_ptr[l], row_ptr[l + 1], nnz, col, val, Y, i, Y[i], lane);
    if (lane == 0) A[l] = a;
  }
}

// Eq. 7 + D12 for the owned rows, Z = the ranks' partials added in rank
// order; the pending recentring shift of this iteration (box->shift, D15) is
// applied to the owned rows on the way out, so Y itself is never modified in
// place (the attractive pass reads it concurrently)
__global__ void __launch_bounds__(kAttrThreads)
k_update_shard(const float2* __restrict__ A, const float2* __restrict__ Y, int row0, int n_local,
               const float2* __restrict__ rep, const double* __restrict__ zp, int world, int t,
               Sched sc, const BoxInfo* __restrict__ box, float2* __restrict__ V,
               float2* __restrict__ G, float2* __restrict__ Yout, int32_t* __restrict__ flag) {
  double Z = 0.0;
  for (int r = 0; r < world; ++r) Z += zp[2 * r];
  const float invZ = (float)(1.0 / Z);
  const float alpha = (t < sc.exag_iters) ? sc.exag : 1.f;
  const float mu = (t < sc.exag_iters) ? sc.mom0 : sc.mom1;
  const float shx = box->shift_x, shy = box->shift_y;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < n_local; l += gridDim.x * blockDim.x) {
    const float2 a = A[l], f = rep[l];
    const float gx = 4.f * (alpha * a.x - f.x * invZ);
    const float gy = 4.f * (alpha * a.y - f.y * invZ);
    float2 v = V[l], gn = G[l], y = Y[row0 + l];
    y.x = y.x - shx;
    y.y = y.y - shy;
    update_coord(gx, v.x, gn.x, y.x, mu, sc.eta, sc.min_gain);
    update_coord(gy, v.y, gn.y, y.y, mu, sc.eta, sc.min_gain);
    V[l] = v;
    G[l] = gn;
    Yout[l] = y;
    if (flag && !(isfinite(y.x) && isfinite(y.y))) *flag = 1;
  }
}

tsne_status launch_attract_sum_shard(const int64_t* row_ptr, const int32_t* col, const float* val,
                                     const float2* Y, int64_t row0, int64_t n_local, float2* A,
                                     cudaStream_t s) {
  if (n_local <= 0) return TSNE_OK;
  k_attract_sum_shard<<<attract_blocks(n_local), kAttrThreads, 0, s>>>(row_ptr, col, val, Y,
                                                                       (int)row0, (int)n_local, A);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

tsne_status launch_update_shard(const float2* A, const float2* Y, int64_t row0, int64_t n_local,
                                const float2* rep, const double* zp, int world, int t,
                                const Sched& sc, const BoxInfo* box, float2* V, float2* G,
                                float2* Yout, int32_t* flag, cudaStream_t s) {
  if (n_local <= 0) return TSNE_OK;
  k_update_shard<<<update_blocks(n_local), kAttrThreads, 0, s>>>(A, Y, (int)row0, (int)n_local,
                                                                 rep, zp, world, t, sc, box, V, G,
                                                                 Yout, flag);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

}  // namespace tsne
