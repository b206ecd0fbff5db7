// optimize.cu -- the per-iteration schedule (Algorithm 1 lines 3-9,
// P:L153-159): tree build -> traversal (F_rep, Z) -> fused attractive +
// update.  Two iterations (Y -> Yb -> Y) are captured once as a CUDA graph
// and replayed; the iteration-dependent constants (exaggeration, momentum)
// are read on the device from an iteration counter, so one graph serves the
// whole run.
#include <mutex>
#include <vector>

#include <cub/device/device_scan.cuh>

#include "optimize.cuh"

namespace tsne {

void carve_opt(Carver& c, OptWS& o, int64_t N, int64_t nnz) {
  o.N = N;
  o.nnz = nnz;
  o.t_dev = c.take<int32_t>(1);
  o.flag = c.take<int32_t>(1);
  o.Ya = c.take<float2>(N);
  o.Yb = c.take<float2>(N);
  o.V = c.take<float2>(N);
  o.G = c.take<float2>(N);
  o.tmp = c.take<float2>(2 * N);
  o.A = c.take<float2>(N);
  o.lab = c.take<int32_t>(N);
  o.lab2 = c.take<int32_t>(N);
  o.inv = c.take<int32_t>(N);
  o.dperm = c.take<int32_t>(N);
  o.dtag = c.take<uint64_t>(1);
  o.ws_base = reinterpret_cast<void*>(c.base);
  for (int h = 0; h < 2; ++h) {
    o.rp[h] = c.take<int64_t>(N + 1);
    o.col[h] = c.take<int32_t>(nnz + 4);
    o.val[h] = c.take<float>(nnz + 4);
    carve_attract_plan(c, o.plan[h], N, nnz, attract_grid_sum(N, nnz));
  }
  o.len = c.take<int64_t>(N + 1);
  size_t sb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, sb, (int64_t*)nullptr, (int64_t*)nullptr, (int)(N + 1));
  o.scan_tmp = c.take<char>(sb);
  o.scan_tmp_bytes = sb;
}

__global__ void k_set_state(int32_t* t_dev, int32_t t0, int32_t* flag) {
  *t_dev = t0;
  *flag = 0;
}

// the batch plan of P half h (cut by relabel(), the only writer of o.rp[h])
static const AtPlan* plan_of(const OptWS& o, const int64_t* row_ptr) {
  return row_ptr == o.rp[0] ? &o.plan[0] : row_ptr == o.rp[1] ? &o.plan[1] : nullptr;
}

// One iteration: the attractive sums run on a side stream
// concurrently with the tree build and the traversal (they only need Y);
// the update joins both.
static tsne_status one_iteration(const int64_t* row_ptr, const int32_t* col, const float* val,
                                 int64_t N, float2* Yin, float2* Yout, float2* V, float2* G,
                                 float theta, const Sched& sc, TreeWS& w, OptWS& o,
                                 cudaStream_t s) {
  TSNE_CUDA_TRY(cudaEventRecord(o.ev_fork, s));
  TSNE_CUDA_TRY(cudaStreamWaitEvent(o.side, o.ev_fork, 0));
  tsne_status st = launch_attract_sum(row_ptr, col, val, Yin, N, o.nnz, o.A, plan_of(o, row_ptr),
                                      o.side);
  if (st != TSNE_OK) return st;
  TSNE_CUDA_TRY(cudaEventRecord(o.ev_join, o.side));
  if ((st = build_tree(w, Yin, /*apply_shift=*/true, s)) != TSNE_OK) return st;
  // the traversal starts when the tree is built, beside the attractive pass's
  // tail if that is still running (joining before the traversal was measured
  // equal at C5 and 1.3x slower at C4, whose attractive pass outlasts tree +
  // traversal)
  if ((st = launch_traverse(w, theta, s)) != TSNE_OK) return st;
  TSNE_CUDA_TRY(cudaStreamWaitEvent(s, o.ev_join, 0));
  return launch_update(Yin, o.A, N, w, o, sc, Yout, V, G, s);
}

// side stream + fork/join events for the concurrent attractive pass
struct SideRes {
  OptWS& o;
  explicit SideRes(OptWS& ow) : o(ow) {
    cudaStreamCreateWithFlags(&o.side, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&o.ev_fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&o.ev_join, cudaEventDisableTiming);
  }
  ~SideRes() {
    cudaEventDestroy(o.ev_fork);
    cudaEventDestroy(o.ev_join);
    cudaStreamDestroy(o.side);
    o.side = nullptr;
  }
};

// ---------------------------------------------------------------- relabelling
// new label k <- old label perm[k]: state gathered, P rows permuted and their
// columns mapped through the inverse permutation (entry order kept).
__global__ void k_perm_state(const int32_t* __restrict__ perm, int N, const float2* __restrict__ Ys,
                             const float2* __restrict__ Vs, const float2* __restrict__ Gs,
                             const int32_t* __restrict__ lab, const int64_t* __restrict__ rp,
                             float2* __restrict__ Yd, float2* __restrict__ Vd,
                             float2* __restrict__ Gd, int32_t* __restrict__ lab2,
                             int32_t* __restrict__ inv, int64_t* __restrict__ len) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > N) return;
  if (k == N) { len[N] = 0; return; }
  const int o = perm ? perm[k] : k;
  Yd[k] = Ys[o];
  Vd[k] = Vs[o];
  Gd[k] = Gs[o];
  lab2[k] = lab ? lab[o] : o;
  inv[o] = k;
  len[k] = rp[o + 1] - rp[o];
}

// Row k of the relabelled CSR = row perm[k] of the old one, columns mapped by
// inv.  Within each attractive-pass item (kAtItem consecutive nonzeros from
// the row's start) the entries are put in bank order for the pass's window
// gathers: the window holds y_j at 8 bytes from a 16-point-aligned start, so
// entry j sits in bank pair (j mod 16); ranking each entry among the earlier
// entries of its bank pair (r) and ordering the item by (r, bank pair) puts 16
// different bank pairs in every half-warp of a gather round wherever the item
// allows (a random order: ~3-way conflicts).  The order is fixed by the CSR,
// so the row sums stay deterministic.  One warp per row.
__global__ void __launch_bounds__(256)
k_relabel_rows(const int32_t* __restrict__ perm, int N, const int64_t* __restrict__ rp_old,
               const int32_t* __restrict__ col_old, const float* __restrict__ val_old,
               const int32_t* __restrict__ inv, const int64_t* __restrict__ rp_new,
               int32_t* __restrict__ col_new, float* __restrict__ val_new) {
  constexpr int kU = kAtItemNz / 32;
  __shared__ int s_cnt[8][16];
  const int lane = threadIdx.x & 31, w = (threadIdx.x >> 5) & 7;
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (k >= N) return;
  const int o = perm ? perm[k] : k;
  const int64_t e0 = rp_old[o], e1 = rp_old[o + 1], d0 = rp_new[k];
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t q0 = 0; q0 < e1 - e0; q0 += kAtItemNz) {
    const int n = (int)min((int64_t)kAtItemNz, e1 - e0 - q0);
    if (lane < 16) s_cnt[w][lane] = 0;
    __syncwarp();
    int c[kU], r[kU];
    float v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {                   // all loads in flight first
      const int q = lane + 32 * u;
      const bool ok = q < n;
      c[u] = ok ? __ldcs(col_old + e0 + q0 + q) : 0;
      v[u] = ok ? __ldcs(val_old + e0 + q0 + q) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (lane + 32 * u < n) c[u] = inv[c[u]];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int q = lane + 32 * u;
      const bool ok = q < n;
      const int b = ok ? (c[u] & 15) : 16 + lane;
      const unsigned peers = __match_any_sync(0xffffffffu, b);
      int base = ok ? s_cnt[w][b] : 0;
      __syncwarp();
      if (ok && lane == __ffs(peers) - 1) s_cnt[w][b] = base + __popc(peers);
      __syncwarp();
      r[u] = base + __popc(peers & lt);
    }
    // rank level r holds the bank pairs with more than r entries, M[r]; an entry
    // of rank r in bank pair b lands at (entries of lower levels) + (banks
    // below b in level r): Lp[r] + popc(M[r] & ((1 << b) - 1)).  Lane r holds
    // level r < 32 (a bank pair with more than 32 entries of one item is rare:
    // those levels are counted directly).
    uint32_t M = 0;
#pragma unroll
    for (int b = 0; b < 16; ++b) M |= (s_cnt[w][b] > lane ? 1u : 0u) << b;
    const int L = __popc(M);
    int Lp = L;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, Lp, o);
      if (lane >= o) Lp += t;
    }
    Lp -= L;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int q = lane + 32 * u;
      const int rr = r[u];
      const int src = rr < 32 ? rr : 31;
      const int lp = __shfl_sync(0xffffffffu, Lp, src);
      const uint32_t m = __shfl_sync(0xffffffffu, M, src);
      if (q < n) {
        const int b = c[u] & 15;
        int pos;
        if (rr < 32) {
          pos = lp + __popc(m & ((1u << b) - 1u));
        } else {
          pos = 0;
          for (int b2 = 0; b2 < 16; ++b2) {
            const int nb2 = s_cnt[w][b2];
            pos += min(nb2, rr) + ((b2 < b && nb2 > rr) ? 1 : 0);
          }
        }
        col_new[d0 + q0 + pos] = c[u];
        val_new[d0 + q0 + pos] = v[u];
      }
    }
    __syncwarp();
  }
}

__global__ void k_scatter_out(int N, const int32_t* __restrict__ lab, const float2* __restrict__ Y,
                              const float2* __restrict__ V, const float2* __restrict__ G,
                              const BoxInfo* __restrict__ box, float2* __restrict__ Yu,
                              float2* __restrict__ Vu, float2* __restrict__ Gu) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  const int o = lab[k];
  float2 y = Y[k];
  y.x = y.x - box->shift_x;            // the last update's pending recentring
  y.y = y.y - box->shift_y;
  Yu[o] = y;
  Vu[o] = V[k];
  Gu[o] = G[k];
}

// Relabel (src P, src state, src lab) -> (P half `dst`, o.Ya/o.V/o.G, o.lab).
static tsne_status relabel(const int32_t* perm, int N, const int64_t* rp, const int32_t* col,
                           const float* val, const float2* Ys, const float2* Vs, const float2* Gs,
                           const int32_t* lab, int dst, OptWS& o, cudaStream_t s) {
  float2* Yn = o.Yb;          // free at iteration boundaries
  float2* Vn = o.tmp;
  float2* Gn = o.tmp + N;
  k_perm_state<<<(N + 256) / 256, 256, 0, s>>>(perm, N, Ys, Vs, Gs, lab, rp, Yn, Vn, Gn, o.lab2,
                                                o.inv, o.len);
  TSNE_LAUNCH_CHECK();
  size_t sb = o.scan_tmp_bytes;
  TSNE_CUDA_TRY(cub::DeviceScan::ExclusiveSum(o.scan_tmp, sb, o.len, o.rp[dst], N + 1, s));
  k_relabel_rows<<<(int)(((int64_t)N * 32 + 255) / 256), 256, 0, s>>>(
      perm, N, rp, col, val, o.inv, o.rp[dst], o.col[dst], o.val[dst]);
  TSNE_LAUNCH_CHECK();
  tsne_status st = attract_plan_build(o.plan[dst], o.rp[dst], N, s);
  if (st != TSNE_OK) return st;
  TSNE_CUDA_TRY(cudaMemcpyAsync(o.Ya, Yn, sizeof(float2) * N, cudaMemcpyDeviceToDevice, s));
  TSNE_CUDA_TRY(cudaMemcpyAsync(o.V, Vn, sizeof(float2) * N, cudaMemcpyDeviceToDevice, s));
  TSNE_CUDA_TRY(cudaMemcpyAsync(o.G, Gn, sizeof(float2) * N, cudaMemcpyDeviceToDevice, s));
  TSNE_CUDA_TRY(cudaMemcpyAsync(o.lab, o.lab2, sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, s));
  return TSNE_OK;
}

// ---------------------------------------------------------------- locality order
// Before the embedding has any structure (t < kMortonFrom: Y is still the
// 1e-4-scale random start, measured in profiles/README.md), its Morton order
// puts a row's neighbours anywhere and the attractive pass gathers y_j at
// random.  Instead the points are labelled by the Morton order of a graph
// diffusion of random coordinates, u <- D^-1 P u (kDiffuseSteps steps): the
// within-community differences decay geometrically while the communities of
// the kNN graph keep distinct means, so rows of one community become
// contiguous and their y_j fall inside the attractive pass's shared-memory
// window.  Labels only reorder rows; the method's results do not depend on it.
constexpr int kMortonFrom = 128;
constexpr int kDiffuseSteps = 8;

__global__ void __launch_bounds__(256)
k_diffuse(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
          const float* __restrict__ val, const float2* __restrict__ u, int N,
          float2* __restrict__ u2) {
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= N) return;
  float sx = 0.f, sy = 0.f, sw = 0.f;
  for (int64_t e = rp[i] + lane; e < rp[i + 1]; e += 32) {
    const float p = __ldcs(val + e);
    const float2 v = u[__ldcs(col + e)];
    sx = fmaf(p, v.x, sx);
    sy = fmaf(p, v.y, sy);
    sw += p;
  }
  sx = warp_sum(sx);
  sy = warp_sum(sy);
  sw = warp_sum(sw);
  if (lane == 0) u2[i] = (sw > 0.f) ? make_float2(sx / sw, sy / sw) : u[i];
}

// The order depends only on P, so it is kept in the caller's workspace and
// reused by later tsne_optimize calls with the same workspace and CSR.  The
// host keeps (key, fingerprint of the stored order); a hit needs the stored
// order to still hash to it (a 64-bit mix of every entry, recomputed on the
// device: ~10 us), so a workspace reused for anything else is never trusted.
struct DiffKey {
  const void* ws;
  const int64_t* rp;
  const int32_t* col;
  const float* val;
  int64_t N, nnz;
  uint64_t csr;    // fingerprint of the CSR's contents (the allocator may reuse addresses)
  uint64_t hash;
};
static std::mutex g_diff_mu;
static std::vector<DiffKey> g_diff_cache;

static bool same_key(const DiffKey& a, const DiffKey& b) {
  return a.ws == b.ws && a.rp == b.rp && a.col == b.col && a.val == b.val && a.N == b.N &&
         a.nnz == b.nnz && a.csr == b.csr;
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
  return x ^ (x >> 33);
}

// order-independent 64-bit fingerprint of (row_ptr, col, val): a sum of mixed
// (position, content) words, ~0.25 ms at C5
__global__ void k_csr_hash(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                           const float* __restrict__ val, int64_t N, int64_t nnz,
                           unsigned long long* __restrict__ out) {
  unsigned long long h = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= N; k += stride)
    h += mix64(((unsigned long long)k << 1) ^ ((unsigned long long)rp[k] * 0x9e3779b97f4a7c15ull));
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += stride)
    h += mix64(((unsigned long long)e << 1 | 1ull) ^
               (((unsigned long long)(uint32_t)__ldcs(col + e) << 32) |
                __float_as_uint(__ldcs(val + e))));
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, h);
}

static bool csr_hash(const int64_t* rp, const int32_t* col, const float* val, int64_t N,
                     int64_t nnz, const OptWS& o, uint64_t* h, cudaStream_t s) {
  if (cudaMemsetAsync(o.dtag, 0, sizeof(uint64_t), s) != cudaSuccess) return false;
  k_csr_hash<<<4 * kNumSMs, 256, 0, s>>>(rp, col, val, N, nnz, (unsigned long long*)o.dtag);
  if (cudaGetLastError() != cudaSuccess) return false;
  if (cudaMemcpyAsync(h, o.dtag, sizeof(uint64_t), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return false;
  return cudaStreamSynchronize(s) == cudaSuccess;
}

__global__ void k_perm_hash(const int32_t* __restrict__ perm, int N,
                            unsigned long long* __restrict__ out) {
  unsigned long long h = 0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
    unsigned long long x = ((unsigned long long)(uint32_t)perm[k] << 32) | (uint32_t)k;
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    h += x;                                   // a sum: independent of the order of addition
  }
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, h);
}

static bool perm_hash(const OptWS& o, int64_t N, uint64_t* h, cudaStream_t s) {
  if (cudaMemsetAsync(o.dtag, 0, sizeof(uint64_t), s) != cudaSuccess) return false;
  k_perm_hash<<<2 * kNumSMs, 256, 0, s>>>(o.dperm, (int)N, (unsigned long long*)o.dtag);
  if (cudaGetLastError() != cudaSuccess) return false;
  if (cudaMemcpyAsync(h, o.dtag, sizeof(uint64_t), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return false;
  return cudaStreamSynchronize(s) == cudaSuccess;
}

static bool diff_cached(const DiffKey& k, const OptWS& o, cudaStream_t s) {
  uint64_t want = 0;
  bool found = false;
  {
    std::lock_guard<std::mutex> g(g_diff_mu);
    for (const auto& e : g_diff_cache)
      if (same_key(e, k)) { want = e.hash; found = true; }
  }
  uint64_t h = 0;
  return found && perm_hash(o, k.N, &h, s) && h == want;
}

static tsne_status diff_remember(DiffKey k, const OptWS& o, cudaStream_t s) {
  uint64_t h = 0;
  if (!perm_hash(o, k.N, &h, s)) {
    set_error("diffusion order: fingerprint failed");
    return TSNE_ERR_CUDA;
  }
  k.hash = h;
  std::lock_guard<std::mutex> g(g_diff_mu);
  for (auto& e : g_diff_cache)
    if (e.ws == k.ws) { e = k; return TSNE_OK; }
  if (g_diff_cache.size() > 64) g_diff_cache.erase(g_diff_cache.begin());
  g_diff_cache.push_back(k);
  return TSNE_OK;
}

static tsne_status diffusion_order(const int64_t* row_ptr, const int32_t* col, const float* val,
                                   int64_t N, TreeWS& w, OptWS& o, cudaStream_t s) {
  float2* u = o.tmp;
  float2* u2 = o.tmp + N;
  tsne_status st = launch_init_y(N, 0x6c6f63616c697479ull, u, s);
  if (st != TSNE_OK) return st;
  const int blocks = (int)((N * 32 + 255) / 256);
  for (int k = 0; k < kDiffuseSteps; ++k) {
    k_diffuse<<<blocks, 256, 0, s>>>(row_ptr, col, val, u, (int)N, u2);
    TSNE_LAUNCH_CHECK();
    float2* t = u; u = u2; u2 = t;
  }
  if ((st = launch_bbox(w, u, s)) != TSNE_OK) return st;
  return build_tree(w, u, /*apply_shift=*/false, s);      // w.perm = the order
}

// ---------------------------------------------------------------- for the multi-GPU run
// The diffusion locality order of P (as above) into perm[N], on scratch u (2N).
tsne_status diffusion_perm(const int64_t* row_ptr, const int32_t* col, const float* val,
                           int64_t N, TreeWS& w, float2* u, int32_t* perm, cudaStream_t s) {
  float2* u2 = u + N;
  tsne_status st = launch_init_y(N, 0x6c6f63616c697479ull, u, s);
  if (st != TSNE_OK) return st;
  const int blocks = (int)((N * 32 + 255) / 256);
  for (int k = 0; k < kDiffuseSteps; ++k) {
    k_diffuse<<<blocks, 256, 0, s>>>(row_ptr, col, val, u, (int)N, u2);
    TSNE_LAUNCH_CHECK();
    float2* t = u; u = u2; u2 = t;
  }
  if ((st = launch_bbox(w, u, s)) != TSNE_OK) return st;
  if ((st = build_tree(w, u, /*apply_shift=*/false, s)) != TSNE_OK) return st;
  TSNE_CUDA_TRY(cudaMemcpyAsync(perm, w.perm, sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, s));
  return TSNE_OK;
}

__global__ void k_perm_lens(const int32_t* __restrict__ perm, int N, const int64_t* __restrict__ rp,
                            int32_t* __restrict__ inv, int64_t* __restrict__ len) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > N) return;
  if (k == N) { len[N] = 0; return; }
  const int o = perm[k];
  inv[o] = k;
  len[k] = rp[o + 1] - rp[o];
}

// P relabelled by perm (new label k <- old label perm[k]) into (rp2, col2, val2);
// inv [N], len [N+1] and the scan scratch are caller scratch
tsne_status permute_csr(const int32_t* perm, int64_t N, const int64_t* rp, const int32_t* col,
                        const float* val, int32_t* inv, int64_t* len, void* scan_tmp,
                        size_t scan_bytes, int64_t* rp2, int32_t* col2, float* val2,
                        cudaStream_t s) {
  k_perm_lens<<<(int)((N + 256) / 256), 256, 0, s>>>(perm, (int)N, rp, inv, len);
  TSNE_LAUNCH_CHECK();
  size_t sb = scan_bytes;
  TSNE_CUDA_TRY(cub::DeviceScan::ExclusiveSum(scan_tmp, sb, len, rp2, (int)(N + 1), s));
  k_relabel_rows<<<(int)((N * 32 + 255) / 256), 256, 0, s>>>(perm, (int)N, rp, col, val, inv, rp2,
                                                             col2, val2);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

size_t permute_csr_scan_bytes(int64_t N) {
  size_t sb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, sb, (int64_t*)nullptr, (int64_t*)nullptr, (int)(N + 1));
  return sb;
}

// Enter the internal label space: the diffusion order early in the run, the
// Morton order of the caller's Y later (or the caller's order if !morton).
static tsne_status enter(const int64_t* row_ptr, const int32_t* col, const float* val, int64_t N,
                         float2* Y, float2* V, float2* G, int32_t t0, TreeWS& w, OptWS& o,
                         bool morton, bool cache_order, cudaStream_t s) {
  k_set_state<<<1, 1, 0, s>>>(o.t_dev, t0, o.flag);
  TSNE_LAUNCH_CHECK();
  tsne_status st;
  const int32_t* perm = nullptr;
  if (morton) {
    if (t0 < kMortonFrom) {
      DiffKey key{o.ws_base, row_ptr, col, val, N, o.nnz, 0, 0};
      if (cache_order && !csr_hash(row_ptr, col, val, N, o.nnz, o, &key.csr, s)) {
        set_error("diffusion order: CSR fingerprint failed");
        return TSNE_ERR_CUDA;
      }
      if (!cache_order || !diff_cached(key, o, s)) {
        if ((st = diffusion_order(row_ptr, col, val, N, w, o, s)) != TSNE_OK) return st;
        TSNE_CUDA_TRY(cudaMemcpyAsync(o.dperm, w.perm, sizeof(int32_t) * N,
                                      cudaMemcpyDeviceToDevice, s));
        if (cache_order && (st = diff_remember(key, o, s)) != TSNE_OK) return st;
      }
      perm = o.dperm;
    } else {
      if ((st = launch_bbox(w, Y, s)) != TSNE_OK) return st;
      if ((st = build_tree(w, Y, /*apply_shift=*/false, s)) != TSNE_OK) return st;
    }
    if (!perm) perm = w.perm;
  }
  if ((st = launch_bbox(w, Y, s)) != TSNE_OK) return st;      // root box of the caller's Y
  return relabel(perm, (int)N, row_ptr, col, val, Y, V, G, nullptr, 0, o, s);
}

static tsne_status leave(int64_t N, const float2* Ycur, float2* Y, float2* V, float2* G, TreeWS& w,
                         OptWS& o, cudaStream_t s) {
  k_scatter_out<<<(int)((N + 255) / 256), 256, 0, s>>>((int)N, o.lab, Ycur, o.V, o.G, w.box, Y, V,
                                                       G);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

// Relabel only if the Morton order of the embedding puts more of P's
// nonzeros near their row than the current labels do (a sample of rows;
// "near" = within the attractive pass's half window).  On data whose kNN
// graph has no spatial structure in the embedding (C4) the diffusion order
// stays; on clustered data the Morton order wins once the clusters form.
__global__ void k_inv_perm(const int32_t* __restrict__ perm, int N, int32_t* __restrict__ inv) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < N) inv[perm[k]] = k;
}

__global__ void k_far_counts(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                             const int32_t* __restrict__ inv, int N, int stride,
                             unsigned long long* __restrict__ cnt) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) * stride;
  unsigned long long cur = 0, nw = 0;
  if (r < N) {
    const int ir = inv[r];
    for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
      const int c = col[e];
      cur += (unsigned)abs(c - r) > 6144u;
      nw += (unsigned)abs(inv[c] - ir) > 6144u;
    }
  }
  atomicAdd(cnt, cur);
  atomicAdd(cnt + 1, nw);
}

static bool morton_improves(const int64_t* rp, const int32_t* col, const int32_t* perm, int64_t N,
                            OptWS& o, cudaStream_t s) {
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(o.len);   // scratch (relabel rewrites it)
  k_inv_perm<<<(int)((N + 255) / 256), 256, 0, s>>>(perm, (int)N, o.inv);
  const int stride = N > 65536 ? (int)(N / 65536) : 1;
  const int rows = (int)((N + stride - 1) / stride);
  unsigned long long h[2] = {0, 0};
  if (cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned long long), s) != cudaSuccess) return true;
  k_far_counts<<<(rows + 255) / 256, 256, 0, s>>>(rp, col, o.inv, (int)N, stride, cnt);
  if (cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return true;
  return h[1] <= h[0];
}

struct Graph {
  cudaGraph_t g = nullptr;
  cudaGraphExec_t e = nullptr;
  ~Graph() {
    if (e) cudaGraphExecDestroy(e);
    if (g) cudaGraphDestroy(g);
  }
};

// two iterations Ya -> Yb -> Ya with P half h
static tsne_status capture_pair(Graph& gr, int h, int64_t N, float theta, const Sched& sc,
                                TreeWS& w, OptWS& o, cudaStream_t s) {
  TSNE_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  tsne_status s1 = one_iteration(o.rp[h], o.col[h], o.val[h], N, o.Ya, o.Yb, o.V, o.G, theta, sc,
                                 w, o, s);
  tsne_status s2 = (s1 == TSNE_OK) ? one_iteration(o.rp[h], o.col[h], o.val[h], N, o.Yb, o.Ya,
                                                   o.V, o.G, theta, sc, w, o, s)
                                   : s1;
  cudaError_t ce = cudaStreamEndCapture(s, &gr.g);
  if (s1 != TSNE_OK) return s1;
  if (s2 != TSNE_OK) return s2;
  TSNE_CUDA_TRY(ce);
  TSNE_CUDA_TRY(cudaGraphInstantiate(&gr.e, gr.g, 0));
  return TSNE_OK;
}

// ---------------------------------------------------------------- sessions
// With tsne_config.keep_state the workspace keeps, after a call, the internal
// state (relabelled P, Y/V/G in internal labels, the relabel phase) and the
// instantiated graphs; a later call on the same workspace with the same
// problem and constants whose t0 continues the previous call resumes from
// them -- no re-entry into the label space (k_relabel_rows re-permutes the
// 1.5 GB CSR at C5) and no graph capture -- provided the caller's Y, v,
// gains still hold exactly what the previous call wrote (a device
// fingerprint).  The caller promises not to modify P in between.
struct Session {
  const void* ws = nullptr;
  const int64_t* rp = nullptr;
  const int32_t* col = nullptr;
  const float* val = nullptr;
  int64_t N = 0, nnz = 0;
  float theta = 0.f;
  Sched sc{};
  bool use_graphs = false;
  int relabel_every = 0;
  // state after the last call
  bool live = false;          // the internal state below is valid
  int h = 0;                  // P half in use
  int since = 0;              // iterations since the last relabel checkpoint
  int32_t t_next = 0;
  uint64_t fp = 0;            // fingerprint of the caller's Y, v, gains
  int32_t* perm = nullptr;    // the tree build's output buffers (host-side selection by
  uint64_t* keys = nullptr;   // the radix sort, made when a build is enqueued eagerly)
  Graph gr[2];
  bool have_gr[2] = {false, false};
};
static std::mutex g_sess_mu;
static std::vector<Session*> g_sess;

static bool same_problem(const Session& a, const Session& b) {
  return a.ws == b.ws && a.rp == b.rp && a.col == b.col && a.val == b.val && a.N == b.N &&
         a.nnz == b.nnz && a.theta == b.theta && a.sc.exag_iters == b.sc.exag_iters &&
         a.sc.exag == b.sc.exag && a.sc.mom0 == b.sc.mom0 && a.sc.mom1 == b.sc.mom1 &&
         a.sc.eta == b.sc.eta && a.sc.min_gain == b.sc.min_gain && a.use_graphs == b.use_graphs &&
         a.relabel_every == b.relabel_every;
}

// the session of workspace `ws` (created on first use; replaced if the problem differs)
static Session* session_for(const Session& key) {
  std::lock_guard<std::mutex> g(g_sess_mu);
  for (size_t i = 0; i < g_sess.size(); ++i)
    if (g_sess[i]->ws == key.ws) {
      if (same_problem(*g_sess[i], key)) return g_sess[i];
      delete g_sess[i];
      g_sess.erase(g_sess.begin() + i);
      break;
    }
  if (g_sess.size() >= 16) {                   // bound the host memory of abandoned sessions
    delete g_sess.front();
    g_sess.erase(g_sess.begin());
  }
  Session* n = new Session();
  n->ws = key.ws; n->rp = key.rp; n->col = key.col; n->val = key.val; n->N = key.N;
  n->nnz = key.nnz; n->theta = key.theta; n->sc = key.sc; n->use_graphs = key.use_graphs;
  n->relabel_every = key.relabel_every;
  g_sess.push_back(n);
  return n;
}

void release_session(const void* ws) {
  std::lock_guard<std::mutex> g(g_sess_mu);
  for (size_t i = 0; i < g_sess.size(); ++i)
    if (g_sess[i]->ws == ws) {
      delete g_sess[i];
      g_sess.erase(g_sess.begin() + i);
      return;
    }
}

// the internal state of workspace ws is about to be overwritten by other work
static void invalidate_session(const void* ws) {
  std::lock_guard<std::mutex> g(g_sess_mu);
  for (auto* e : g_sess)
    if (e->ws == ws) e->live = false;
}

// order-dependent 64-bit fingerprint of the caller's state (Y, v, gains)
__global__ void k_state_hash(const float2* __restrict__ Y, const float2* __restrict__ V,
                             const float2* __restrict__ G, int N,
                             unsigned long long* __restrict__ out) {
  unsigned long long h = 0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
    const float2 y = Y[k], v = V[k], g = G[k];
    const unsigned long long kk = (unsigned long long)k * 0x9e3779b97f4a7c15ull;
    h += mix64(kk ^ (((unsigned long long)__float_as_uint(y.x) << 32) | __float_as_uint(y.y)));
    h += mix64((kk + 1) ^ (((unsigned long long)__float_as_uint(v.x) << 32) | __float_as_uint(v.y)));
    h += mix64((kk + 2) ^ (((unsigned long long)__float_as_uint(g.x) << 32) | __float_as_uint(g.y)));
  }
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, h);
}

static bool state_hash(const float2* Y, const float2* V, const float2* G, int64_t N,
                       const OptWS& o, uint64_t* h, cudaStream_t s) {
  if (cudaMemsetAsync(o.dtag, 0, sizeof(uint64_t), s) != cudaSuccess) return false;
  k_state_hash<<<2 * kNumSMs, 256, 0, s>>>(Y, V, G, (int)N, (unsigned long long*)o.dtag);
  if (cudaGetLastError() != cudaSuccess) return false;
  if (cudaMemcpyAsync(h, o.dtag, sizeof(uint64_t), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return false;
  return cudaStreamSynchronize(s) == cudaSuccess;
}

tsne_status run_iterations(const int64_t* row_ptr, const int32_t* col, const float* val,
                           int64_t N, float2* Y, float2* V, float2* G, int32_t t0, int32_t n_iter,
                           float theta, const Sched& sc, bool use_graphs, int relabel_every,
                           TreeWS& w, OptWS& o, cudaStream_t s, bool cache_order,
                           bool keep_state) {
  SideRes side(o);
  const bool graphs = use_graphs && s != nullptr;
  Session local;
  Session* ses = &local;
  if (keep_state) {
    Session key;
    key.ws = o.ws_base; key.rp = row_ptr; key.col = col; key.val = val; key.N = N;
    key.nnz = o.nnz; key.theta = theta; key.sc = sc; key.use_graphs = graphs;
    key.relabel_every = relabel_every;
    ses = session_for(key);
  }
  bool resume = false;
  if (keep_state && ses->live && ses->t_next == t0) {
    uint64_t h = 0;
    resume = state_hash(Y, V, G, N, o, &h, s) && h == ses->fp;
  }
  ses->live = false;
  tsne_status st;
  if (resume) {
    k_set_state<<<1, 1, 0, s>>>(o.t_dev, t0, o.flag);
    TSNE_LAUNCH_CHECK();
    w.perm = ses->perm;          // a graph replay does not set these host-side fields
    w.keys_sorted = ses->keys;
  } else {
    st = enter(row_ptr, col, val, N, Y, V, G, t0, w, o, relabel_every > 0, cache_order, s);
    if (st != TSNE_OK) return st;
    ses->h = 0;
    ses->since = 0;
  }
  int h = ses->h;
  const int period = relabel_every > 0 ? relabel_every : (1 << 30);
  int since = ses->since;
  int32_t done = 0;
  while (done < n_iter) {
    // the state is in Ya at every chunk boundary
    const int chunk = (n_iter - done) < (period - since) ? (n_iter - done) : (period - since);
    int c = 0;
    if (graphs && chunk >= 2 && (ses->have_gr[h] || n_iter >= 4)) {
      if (!ses->have_gr[h]) {
        if ((st = capture_pair(ses->gr[h], h, N, theta, sc, w, o, s)) != TSNE_OK) return st;
        ses->have_gr[h] = true;
      }
      for (; c + 2 <= chunk; c += 2) TSNE_CUDA_TRY(cudaGraphLaunch(ses->gr[h].e, s));
    }
    for (; c < chunk; ++c) {
      float2* a = (c % 2 == 0) ? o.Ya : o.Yb;
      float2* b = (c % 2 == 0) ? o.Yb : o.Ya;
      if ((st = one_iteration(o.rp[h], o.col[h], o.val[h], N, a, b, o.V, o.G, theta, sc, w, o,
                              s)) != TSNE_OK)
        return st;
    }
    if (chunk % 2)
      TSNE_CUDA_TRY(cudaMemcpyAsync(o.Ya, o.Yb, sizeof(float2) * N, cudaMemcpyDeviceToDevice, s));
    done += chunk;
    since += chunk;
    if (since == period) {
      since = 0;
      if (done < n_iter) {
        // non-finite sentinel (set by k_update), checked at every checkpoint so
        // a diverging run stops within relabel_every iterations
        int32_t bad = 0;
        TSNE_CUDA_TRY(cudaMemcpyAsync(&bad, o.flag, sizeof(bad), cudaMemcpyDeviceToHost, s));
        TSNE_CUDA_TRY(cudaStreamSynchronize(s));
        if (bad) {
          set_error("non-finite embedding during iterations [%d, %d)", t0, t0 + done);
          return TSNE_ERR_NONFINITE;
        }
      }
      // a relabel checkpoint (also at the end of a call whose state is kept)
      if ((done < n_iter || keep_state) && t0 + done >= kMortonFrom && w.perm &&
          morton_improves(o.rp[h], o.col[h], w.perm, N, o, s)) {
        // w.perm is the Morton order of the last iteration's embedding (a
        // permutation of the current labels); the pending recentring shift
        // is uniform, so it commutes with relabelling.
        if ((st = relabel(w.perm, (int)N, o.rp[h], o.col[h], o.val[h], o.Ya, o.V, o.G, o.lab,
                          1 - h, o, s)) != TSNE_OK)
          return st;
        h = 1 - h;
      }
    }
  }
  if ((st = leave(N, o.Ya, Y, V, G, w, o, s)) != TSNE_OK) return st;
  if (keep_state) {
    uint64_t hsh = 0;
    if (!state_hash(Y, V, G, N, o, &hsh, s)) {
      set_error("tsne_optimize: state fingerprint failed");
      return TSNE_ERR_CUDA;
    }
    ses->fp = hsh;
    ses->perm = w.perm;
    ses->keys = w.keys_sorted;
    ses->h = h;
    ses->since = since;
    ses->t_next = t0 + n_iter;
    ses->live = true;
  }
  return TSNE_OK;
}

tsne_status profile_iterations(const int64_t* row_ptr, const int32_t* col, const float* val,
                               int64_t N, float2* Y, float2* V, float2* G, int32_t t0, int32_t reps,
                               float theta, const Sched& sc, TreeWS& w, OptWS& o, double* stage_ms,
                               int32_t* kernels, double* trav_stats, cudaStream_t s) {
  SideRes side(o);
  invalidate_session(o.ws_base);
  tsne_status st = enter(row_ptr, col, val, N, Y, V, G, t0, w, o, true, true, s);
  if (st != TSNE_OK) return st;
  if (kernels) {  // count kernel nodes of one captured (never launched) iteration
    cudaGraph_t g = nullptr;
    TSNE_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    st = one_iteration(o.rp[0], o.col[0], o.val[0], N, o.Ya, o.Yb, o.V, o.G, theta, sc, w, o, s);
    cudaError_t ce = cudaStreamEndCapture(s, &g);
    if (st != TSNE_OK) { if (g) cudaGraphDestroy(g); return st; }
    TSNE_CUDA_TRY(ce);
    size_t n = 0;
    cudaGraphGetNodes(g, nullptr, &n);
    std::vector<cudaGraphNode_t> nodes(n);
    cudaGraphGetNodes(g, nodes.data(), &n);
    int32_t k = 0;
    for (auto nd : nodes) {
      cudaGraphNodeType t;
      cudaGraphNodeGetType(nd, &t);
      k += (t == cudaGraphNodeTypeKernel);
    }
    *kernels = k;
    cudaGraphDestroy(g);
  }
  cudaEvent_t e[5];
  for (auto& x : e) cudaEventCreate(&x);
  double acc[4] = {0, 0, 0, 0};
  float2* a = o.Ya;
  float2* b = o.Yb;
  // stages timed one after the other (no overlap), then the overlapped iteration
  for (int r = 0; r < reps && st == TSNE_OK; ++r) {
    cudaEventRecord(e[0], s);
    st = build_tree(w, a, true, s);
    cudaEventRecord(e[1], s);
    if (st == TSNE_OK) st = launch_traverse(w, theta, s);
    cudaEventRecord(e[2], s);
    if (st == TSNE_OK)
      st = launch_attract_sum(o.rp[0], o.col[0], o.val[0], a, N, o.nnz, o.A, &o.plan[0], s);
    cudaEventRecord(e[3], s);
    if (st == TSNE_OK) st = launch_update(a, o.A, N, w, o, sc, b, o.V, o.G, s);
    cudaEventRecord(e[4], s);
    cudaEventSynchronize(e[4]);
    for (int k = 0; k < 4; ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e[k], e[k + 1]);
      acc[k] += ms;
    }
    float2* t = a; a = b; b = t;
  }
  double overlapped = 0.0;
  for (int r = 0; r < reps && st == TSNE_OK; ++r) {
    cudaEventRecord(e[0], s);
    st = one_iteration(o.rp[0], o.col[0], o.val[0], N, a, b, o.V, o.G, theta, sc, w, o, s);
    cudaEventRecord(e[1], s);
    cudaEventSynchronize(e[1]);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e[0], e[1]);
    overlapped += ms;
    float2* t = a; a = b; b = t;
  }
  for (auto& x : e) cudaEventDestroy(x);
  if (st != TSNE_OK) return st;
  for (int k = 0; k < 4; ++k) stage_ms[k] = reps > 0 ? acc[k] / reps : 0.0;
  stage_ms[4] = reps > 0 ? overlapped / reps : 0.0;
  if (trav_stats) {   // counters of one more traversal of the current embedding
    if ((st = build_tree(w, a, true, s)) != TSNE_OK) return st;
    if ((st = traverse_stats(w, theta, trav_stats, s)) != TSNE_OK) return st;
  }
  if ((st = leave(N, a, Y, V, G, w, o, s)) != TSNE_OK) return st;
  TSNE_CUDA_TRY(cudaStreamSynchronize(s));
  return TSNE_OK;
}

// ---------------------------------------------------------------- D14 init
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint32_t lo0 = 0xD2511F53u * c[0], hi0 = __umulhi(0xD2511F53u, c[0]);
    const uint32_t lo1 = 0xCD9E8D57u * c[2], hi1 = __umulhi(0xCD9E8D57u, c[2]);
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
  }
}

__global__ void k_init_y(int64_t N, uint64_t seed, float2* Y) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  uint32_t c[4] = {(uint32_t)i, (uint32_t)((uint64_t)i >> 32), 0u, 0u};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  const double u1 = ((double)c[0] + 0.5) * 2.3283064365386963e-10;  // 2^-32
  const double u2 = ((double)c[1] + 0.5) * 2.3283064365386963e-10;
  const double r = sqrt(-2.0 * log(u1));
  const double two_pi = 6.283185307179586476925286766559;
  Y[i] = make_float2((float)(1e-4 * r * cos(two_pi * u2)), (float)(1e-4 * r * sin(two_pi * u2)));
}

tsne_status launch_init_y(int64_t N, uint64_t seed, float2* Y, cudaStream_t s) {
  k_init_y<<<(int)((N + 255) / 256), 256, 0, s>>>(N, seed, Y);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

}  // namespace tsne
