// optimize.cu -- the per-iteration schedule (Algorithm 1 lines 3-9,
// P:L153-159): tree build -> traversal (F_rep, Z) -> fused attractive +
// update.  Two iterations (Y -> Yb -> Y) are captured once as a CUDA graph
// and replayed; the iteration-dependent constants (exaggeration, momentum)
// are read on the device from an iteration counter, so one graph serves the
// whole run.
#include <vector>

#include "optimize.cuh"

namespace tsne {

void carve_opt(Carver& c, OptWS& o, int64_t N) {
  o.t_dev = c.take<int32_t>(1);
  o.flag = c.take<int32_t>(1);
  o.Yb = c.take<float2>(N);
}

__global__ void k_set_state(int32_t* t_dev, int32_t t0, int32_t* flag) {
  *t_dev = t0;
  *flag = 0;
}

// the first iteration's box: bbox of Y with zero shift
static tsne_status one_iteration(const int64_t* row_ptr, const int32_t* col, const float* val,
                                 int64_t N, float2* Yin, float2* Yout, float2* V, float2* G,
                                 float theta, const Sched& sc, TreeWS& w, OptWS& o,
                                 cudaStream_t s) {
  tsne_status st = build_tree(w, Yin, /*apply_shift=*/true, s);
  if (st != TSNE_OK) return st;
  st = launch_traverse(w, theta, s);
  if (st != TSNE_OK) return st;
  return launch_attract_update(row_ptr, col, val, Yin, N, w, o, sc, Yout, V, G, s);
}

__global__ void k_apply_shift(float2* Y, int N, const BoxInfo* box) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  float2 y = Y[i];
  y.x = y.x - box->shift_x;
  y.y = y.y - box->shift_y;
  Y[i] = y;
}

tsne_status run_iterations(const int64_t* row_ptr, const int32_t* col, const float* val,
                           int64_t N, float2* Y, float2* V, float2* G, int32_t t0, int32_t n_iter,
                           float theta, const Sched& sc, bool use_graphs, TreeWS& w, OptWS& o,
                           cudaStream_t s) {
  k_set_state<<<1, 1, 0, s>>>(o.t_dev, t0, o.flag);
  TSNE_LAUNCH_CHECK();
  tsne_status st = launch_bbox(w, Y, s);   // shift = 0 for the first iteration
  if (st != TSNE_OK) return st;
  int32_t done = 0;
  float2* a = Y;
  float2* b = o.Yb;
  // graphs need a non-default stream for capture
  bool graphs = use_graphs && s != nullptr && n_iter >= 4;
  if (graphs) {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    TSNE_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    tsne_status s1 = one_iteration(row_ptr, col, val, N, a, b, V, G, theta, sc, w, o, s);
    tsne_status s2 = (s1 == TSNE_OK)
                         ? one_iteration(row_ptr, col, val, N, b, a, V, G, theta, sc, w, o, s)
                         : s1;
    cudaError_t ce = cudaStreamEndCapture(s, &g);
    if (s1 != TSNE_OK || s2 != TSNE_OK) {
      if (g) cudaGraphDestroy(g);
      return s1 != TSNE_OK ? s1 : s2;
    }
    TSNE_CUDA_TRY(ce);
    TSNE_CUDA_TRY(cudaGraphInstantiate(&ge, g, 0));
    for (; done + 2 <= n_iter; done += 2) {
      cudaError_t e = cudaGraphLaunch(ge, s);
      if (e != cudaSuccess) {
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
        TSNE_CUDA_TRY(e);
      }
    }
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
  for (; done < n_iter; ++done) {
    st = one_iteration(row_ptr, col, val, N, a, b, V, G, theta, sc, w, o, s);
    if (st != TSNE_OK) return st;
    float2* t = a; a = b; b = t;
  }
  // the last update left its recentring pending: apply it
  k_apply_shift<<<(int)((N + 255) / 256), 256, 0, s>>>(a, (int)N, w.box);
  TSNE_LAUNCH_CHECK();
  if (a != Y) TSNE_CUDA_TRY(cudaMemcpyAsync(Y, a, sizeof(float2) * N, cudaMemcpyDeviceToDevice, s));
  return TSNE_OK;
}

tsne_status profile_iterations(const int64_t* row_ptr, const int32_t* col, const float* val,
                               int64_t N, float2* Y, float2* V, float2* G, int32_t t0, int32_t reps,
                               float theta, const Sched& sc, TreeWS& w, OptWS& o, double* stage_ms,
                               int32_t* kernels, cudaStream_t s) {
  if (kernels) {  // count kernel nodes of one captured (never launched) iteration
    cudaGraph_t g = nullptr;
    TSNE_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    tsne_status st = one_iteration(row_ptr, col, val, N, Y, o.Yb, V, G, theta, sc, w, o, s);
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
  k_set_state<<<1, 1, 0, s>>>(o.t_dev, t0, o.flag);
  TSNE_LAUNCH_CHECK();
  tsne_status st = launch_bbox(w, Y, s);
  if (st != TSNE_OK) return st;
  cudaEvent_t e[4];
  for (auto& x : e) cudaEventCreate(&x);
  double acc[3] = {0, 0, 0};
  float2* a = Y;
  float2* b = o.Yb;
  for (int r = 0; r < reps && st == TSNE_OK; ++r) {
    cudaEventRecord(e[0], s);
    st = build_tree(w, a, true, s);
    cudaEventRecord(e[1], s);
    if (st == TSNE_OK) st = launch_traverse(w, theta, s);
    cudaEventRecord(e[2], s);
    if (st == TSNE_OK) st = launch_attract_update(row_ptr, col, val, a, N, w, o, sc, b, V, G, s);
    cudaEventRecord(e[3], s);
    cudaEventSynchronize(e[3]);
    for (int k = 0; k < 3; ++k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e[k], e[k + 1]);
      acc[k] += ms;
    }
    float2* t = a; a = b; b = t;
  }
  for (auto& x : e) cudaEventDestroy(x);
  if (st != TSNE_OK) return st;
  for (int k = 0; k < 3; ++k) stage_ms[k] = reps > 0 ? acc[k] / reps : 0.0;
  k_apply_shift<<<(int)((N + 255) / 256), 256, 0, s>>>(a, (int)N, w.box);
  TSNE_LAUNCH_CHECK();
  if (a != Y) TSNE_CUDA_TRY(cudaMemcpyAsync(Y, a, sizeof(float2) * N, cudaMemcpyDeviceToDevice, s));
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
