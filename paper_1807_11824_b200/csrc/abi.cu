// abi.cu -- extern "C" entry points of include/tsne.h: argument validation,
// workspace carving, stream plumbing.  All compute is in the kernels of
// tree.cu, traverse.cu, attract.cu, optimize.cu, knn.cu, affinity.cu.
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "affinity.cuh"
#include "knn.cuh"
#include "optimize.cuh"
#include "shard.cuh"

namespace tsne {
size_t kl_workspace_size(int64_t N);
tsne_status kl_run(const int64_t* row_ptr, const int32_t* col, const float* val, int64_t N,
                   const float2* Y, void* ws, double* kl_out, double* Z_out, cudaStream_t s);
}  // namespace tsne

namespace tsne {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
void clear_error() { g_err[0] = 0; }

tsne_status check_device() {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    set_error("no CUDA device: %s", cudaGetErrorString(e));
    return TSNE_ERR_CUDA;
  }
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) {
    set_error("libtsne_b200 is built for sm_100a only (device %d is sm_%d.x)", dev, major);
    return TSNE_ERR_CUDA;
  }
  return TSNE_OK;
}

struct GradPlan {
  TreeWS tree;
};

static size_t grad_plan(void* base, int64_t N, GradPlan& p) {
  Carver c(base);
  carve_tree(c, p.tree, N);
  return c.bytes();
}

struct OptPlan {
  TreeWS tree;
  OptWS opt;
};

static size_t opt_plan(void* base, int64_t N, int64_t nnz, OptPlan& p) {
  Carver c(base);
  carve_tree(c, p.tree, N);
  carve_opt(c, p.opt, N, nnz);
  return c.bytes();
}

// Zeroes the last-block-done counters of a freshly carved tree workspace.
static tsne_status init_tree_ws(TreeWS& w, cudaStream_t s) { return tree_ws_init(w, s); }

// A private stream ordered after/before `s` (graphs cannot be captured on the
// legacy default stream).
struct SideStream {
  cudaStream_t user = nullptr, own = nullptr;
  cudaEvent_t ev = nullptr;
  cudaStream_t get(cudaStream_t s) {
    user = s;
    if (s != nullptr) return s;
    cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventRecord(ev, s);
    cudaStreamWaitEvent(own, ev, 0);
    return own;
  }
  void join() {
    if (!own) return;
    cudaEventRecord(ev, own);
    cudaStreamWaitEvent(user, ev, 0);
    cudaEventDestroy(ev);
    cudaStreamDestroy(own);
    own = nullptr;
  }
};

}  // namespace tsne

using namespace tsne;

extern "C" {

const char* tsne_last_error(void) { return g_err; }

int32_t tsne_abi_version(void) { return (1 << 16) | 1; }

void tsne_config_default(tsne_config* cfg) {
  if (!cfg) return;
  cfg->K = 0;
  cfg->exag_iters = 250;
  cfg->mom0 = 0.5f;
  cfg->mom1 = 0.8f;
  cfg->min_gain = 0.01f;
  cfg->seed = 42;
  cfg->Y_init = nullptr;
  cfg->use_graphs = 1;
  cfg->relabel_every = 64;
  cfg->keep_state = 0;
  cfg->knn_tau = 0;
}

// ---------------------------------------------------------------- gradient
size_t tsne_gradient_workspace_size(int64_t N) {
  if (N < 2) return 0;
  GradPlan p;
  return grad_plan(nullptr, N, p);
}

tsne_status tsne_gradient(const int64_t* row_ptr, const int32_t* col, const float* val, int64_t N,
                          const float* Y, float theta, float exaggeration, float* dY,
                          double* Z_out, void* ws, size_t ws_bytes, tsne_stream_t stream) {
  clear_error();
  TSNE_ARG_CHECK(N >= 2 && N <= kMaxTreePoints, "N must be in [2, 2^25) (got %lld)",
                 (long long)N);
  TSNE_ARG_CHECK(row_ptr && col && val && Y && dY, "null pointer argument");
  TSNE_ARG_CHECK(theta >= 0.f && std::isfinite(theta), "theta must be >= 0 (got %g)", theta);
  TSNE_ARG_CHECK(exaggeration > 0.f && std::isfinite(exaggeration), "exaggeration must be > 0");
  TSNE_ARG_CHECK(aligned(Y, 16) && aligned(dY, 8) && aligned(col, 16) && aligned(val, 16),
                 "Y, col, val need 16-byte and dY 8-byte alignment");
  GradPlan p;
  size_t need = grad_plan(nullptr, N, p);
  if (!ws || ws_bytes < need) {
    set_error("workspace too small: need %zu bytes, got %zu", need, ws_bytes);
    return TSNE_ERR_WORKSPACE;
  }
  tsne_status st = check_device();
  if (st != TSNE_OK) return st;
  grad_plan(ws, N, p);
  cudaStream_t s = (cudaStream_t)stream;
  if ((st = init_tree_ws(p.tree, s)) != TSNE_OK) return st;
  float2* Yd = const_cast<float2*>(reinterpret_cast<const float2*>(Y));
  if ((st = launch_bbox(p.tree, Yd, s)) != TSNE_OK) return st;
  if ((st = build_tree(p.tree, Yd, /*apply_shift=*/false, s)) != TSNE_OK) return st;
  if ((st = launch_traverse(p.tree, theta, s)) != TSNE_OK) return st;
  if ((st = launch_attract_grad(row_ptr, col, val, Yd, N, p.tree.rep, p.tree.Z, exaggeration,
                                reinterpret_cast<float2*>(dY), s)) != TSNE_OK)
    return st;
  if (Z_out) {
    double z[2];
    TSNE_CUDA_TRY(cudaMemcpyAsync(z, p.tree.Z, sizeof(z), cudaMemcpyDeviceToHost, s));
    TSNE_CUDA_TRY(cudaStreamSynchronize(s));
    *Z_out = z[0];
  }
  return TSNE_OK;
}

// ---------------------------------------------------------------- f4 KL
size_t tsne_kl_workspace_size(int64_t N) {
  if (N < 2) return 0;
  return kl_workspace_size(N);
}

tsne_status tsne_kl(const int64_t* row_ptr, const int32_t* col, const float* val, int64_t N,
                    const float* Y, double* kl_out, double* Z_out, void* ws, size_t ws_bytes,
                    tsne_stream_t stream) {
  clear_error();
  TSNE_ARG_CHECK(N >= 2 && N < (int64_t(1) << 27), "N must be in [2, 2^27) (got %lld)",
                 (long long)N);
  TSNE_ARG_CHECK(row_ptr && col && val && Y && kl_out, "null pointer argument");
  TSNE_ARG_CHECK(aligned(Y, 8), "Y needs 8-byte alignment");
  const size_t need = kl_workspace_size(N);
  if (!ws || ws_bytes < need) {
    set_error("workspace too small: need %zu bytes, got %zu", need, ws_bytes);
    return TSNE_ERR_WORKSPACE;
  }
  tsne_status st = check_device();
  if (st != TSNE_OK) return st;
  return kl_run(row_ptr, col, val, N, reinterpret_cast<const float2*>(Y), ws, kl_out, Z_out,
                (cudaStream_t)stream);
}

// ---------------------------------------------------------------- optimise
size_t tsne_optimize_workspace_size(int64_t N, int64_t nnz) {
  if (N < 2 || nnz < 0) return 0;
  OptPlan p;
  return opt_plan(nullptr, N, nnz, p);
}

// nnz = row_ptr[N] (one 8-byte device read; synchronises the stream)
static tsne_status read_nnz(const int64_t* row_ptr, int64_t N, int64_t* nnz, cudaStream_t s) {
  TSNE_CUDA_TRY(cudaMemcpyAsync(nnz, row_ptr + N, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  TSNE_CUDA_TRY(cudaStreamSynchronize(s));
  if (*nnz < 0) {
    set_error("row_ptr[N] = %lld < 0", (long long)*nnz);
    return TSNE_ERR_ARG;
  }
  return TSNE_OK;
}

tsne_status tsne_optimize(const int64_t* row_ptr, const int32_t* col, const float* val, int64_t N,
                          float* Y, float* v, float* gains, int32_t t0, int32_t n_iter,
                          float theta, float learning_rate, float exaggeration,
                          const tsne_config* cfg_in, void* ws, size_t ws_bytes,
                          tsne_stream_t stream) {
  clear_error();
  tsne_config cfg;
  tsne_config_default(&cfg);
  if (cfg_in) cfg = *cfg_in;
  TSNE_ARG_CHECK(N >= 2 && N <= kMaxTreePoints, "N must be in [2, 2^25) (got %lld)", (long long)N);
  TSNE_ARG_CHECK(row_ptr && col && val && Y && v && gains, "null pointer argument");
  TSNE_ARG_CHECK(theta >= 0.f && std::isfinite(theta), "theta must be >= 0");
  TSNE_ARG_CHECK(learning_rate > 0.f, "learning_rate must be > 0");
  TSNE_ARG_CHECK(exaggeration > 0.f, "exaggeration must be > 0");
  TSNE_ARG_CHECK(n_iter >= 0 && t0 >= 0, "n_iter and t0 must be >= 0");
  TSNE_ARG_CHECK(aligned(Y, 8) && aligned(v, 8) && aligned(gains, 8) && aligned(col, 16) &&
                     aligned(val, 16),
                 "Y, v, gains need 8-byte and col, val 16-byte alignment");
  tsne_status st = check_device();
  if (st != TSNE_OK) return st;
  int64_t nnz = 0;
  if ((st = read_nnz(row_ptr, N, &nnz, (cudaStream_t)stream)) != TSNE_OK) return st;
  OptPlan p;
  size_t need = opt_plan(nullptr, N, nnz, p);
  if (!ws || ws_bytes < need) {
    set_error("workspace too small: need %zu bytes, got %zu", need, ws_bytes);
    return TSNE_ERR_WORKSPACE;
  }
  if (n_iter == 0) return TSNE_OK;
  opt_plan(ws, N, nnz, p);
  SideStream ss;
  cudaStream_t s = ss.get((cudaStream_t)stream);
  if ((st = init_tree_ws(p.tree, s)) != TSNE_OK) { ss.join(); return st; }
  Sched sc{cfg.exag_iters, exaggeration, cfg.mom0, cfg.mom1, learning_rate, cfg.min_gain};
  st = run_iterations(row_ptr, col, val, N, reinterpret_cast<float2*>(Y),
                      reinterpret_cast<float2*>(v), reinterpret_cast<float2*>(gains), t0, n_iter,
                      theta, sc, cfg.use_graphs != 0, cfg.relabel_every, p.tree, p.opt, s,
                      /*cache_order=*/true, cfg.keep_state != 0);
  int32_t flag = 0;
  if (st == TSNE_OK) {
    cudaError_t e = cudaMemcpyAsync(&flag, p.opt.flag, sizeof(flag), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      set_error("tsne_optimize: %s", cudaGetErrorString(e));
      st = TSNE_ERR_CUDA;
    }
  }
  ss.join();
  if (st == TSNE_OK && flag) {
    set_error("non-finite embedding during iterations [%d, %d)", t0, t0 + n_iter);
    return TSNE_ERR_NONFINITE;
  }
  return st;
}

void tsne_optimize_release(void* ws) { release_session(ws); }

tsne_status tsne_profile_iterations(const int64_t* row_ptr, const int32_t* col, const float* val,
                                    int64_t N, float* Y, float* v, float* gains, int32_t t0,
                                    int32_t reps, float theta, float learning_rate,
                                    float exaggeration, const tsne_config* cfg_in,
                                    double* stage_ms, int32_t* kernels_per_iter,
                                    double* trav_stats, void* ws, size_t ws_bytes,
                                    tsne_stream_t stream) {
  clear_error();
  tsne_config cfg;
  tsne_config_default(&cfg);
  if (cfg_in) cfg = *cfg_in;
  TSNE_ARG_CHECK(N >= 2 && N <= kMaxTreePoints, "N must be in [2, 2^25) (got %lld)", (long long)N);
  TSNE_ARG_CHECK(row_ptr && col && val && Y && v && gains && stage_ms, "null pointer argument");
  TSNE_ARG_CHECK(reps >= 1 && t0 >= 0, "reps must be >= 1");
  tsne_status st = check_device();
  if (st != TSNE_OK) return st;
  int64_t nnz = 0;
  if ((st = read_nnz(row_ptr, N, &nnz, (cudaStream_t)stream)) != TSNE_OK) return st;
  OptPlan p;
  size_t need = opt_plan(nullptr, N, nnz, p);
  if (!ws || ws_bytes < need) {
    set_error("workspace too small: need %zu bytes, got %zu", need, ws_bytes);
    return TSNE_ERR_WORKSPACE;
  }
  opt_plan(ws, N, nnz, p);
  SideStream ss;
  cudaStream_t s = ss.get((cudaStream_t)stream);
  if ((st = init_tree_ws(p.tree, s)) != TSNE_OK) { ss.join(); return st; }
  Sched sc{cfg.exag_iters, exaggeration, cfg.mom0, cfg.mom1, learning_rate, cfg.min_gain};
  st = profile_iterations(row_ptr, col, val, N, reinterpret_cast<float2*>(Y),
                          reinterpret_cast<float2*>(v), reinterpret_cast<float2*>(gains), t0, reps,
                          theta, sc, p.tree, p.opt, stage_ms, kernels_per_iter, trav_stats, s);
  ss.join();
  return st;
}

// ---------------------------------------------------------------- multi-GPU
size_t tsne_shard_workspace_size(int64_t N) {
  if (N < 2) return 0;
  ShardWS w;
  Carver c(nullptr);
  carve_shard(c, w, N);
  return c.bytes();
}

tsne_status tsne_shard_forces(const float* Y, int64_t N, int64_t row0, int64_t row1, float theta,
                              int32_t recentre, float* rep_local, double* z_partial, void* ws,
                              size_t ws_bytes, tsne_stream_t stream) {
  clear_error();
  TSNE_ARG_CHECK(N >= 2 && N <= kMaxTreePoints, "N must be in [2, 2^25) (got %lld)", (long long)N);
  TSNE_ARG_CHECK(0 <= row0 && row0 <= row1 && row1 <= N, "bad row range [%lld, %lld)",
                 (long long)row0, (long long)row1);
  TSNE_ARG_CHECK(Y && z_partial && (rep_local || row1 == row0), "null pointer argument");
  TSNE_ARG_CHECK(theta >= 0.f && std::isfinite(theta), "theta must be >= 0");
  TSNE_ARG_CHECK(aligned(Y, 8) && (!rep_local || aligned(rep_local, 8)), "8-byte alignment needed");
  ShardWS w;
  Carver c0(nullptr);
  carve_shard(c0, w, N);
  if (!ws || ws_bytes < c0.bytes()) {
    set_error("workspace too small: need %zu bytes, got %zu", c0.bytes(), ws_bytes);
    return TSNE_ERR_WORKSPACE;
  }
  tsne_status st = check_device();
  if (st != TSNE_OK) return st;
  Carver c(ws);
  carve_shard(c, w, N);
  return shard_forces(w, reinterpret_cast<const float2*>(Y), N, row0, row1, theta, recentre != 0,
                      reinterpret_cast<float2*>(rep_local), z_partial, (cudaStream_t)stream);
}

tsne_status tsne_shard_attract(const int64_t* row_ptr_local, const int32_t* col_local,
                               const float* val_local, int64_t N, int64_t row0, int64_t row1,
                               const float* Y, float* A_local, tsne_stream_t stream) {
  clear_error();
  TSNE_ARG_CHECK(N >= 2 && N <= kMaxTreePoints, "N must be in [2, 2^25) (got %lld)", (long long)N);
  TSNE_ARG_CHECK(0 <= row0 && row0 <= row1 && row1 <= N, "bad row range");
  TSNE_ARG_CHECK(Y && (row1 == row0 || (row_ptr_local && col_local && val_local && A_local)),
                 "null pointer argument");
  TSNE_ARG_CHECK(aligned(Y, 16), "Y must be 16-byte aligned (bulk copies of its window)");
  TSNE_ARG_CHECK(row1 == row0 || (aligned(col_local, 16) && aligned(val_local, 16)),
                 "col and val must be 16-byte aligned");
  tsne_status st = check_device();
  if (st != TSNE_OK) return st;
  return launch_attract_sum_shard(row_ptr_local, col_local, val_local,
                                  reinterpret_cast<const float2*>(Y), N, row0, row1 - row0,
                                  reinterpret_cast<float2*>(A_local), nullptr,
                                  (cudaStream_t)stream);
}

tsne_status tsne_shard_update(const float* A_local, int64_t N, int64_t row0, int64_t row1,
                              const float* Y, const float* rep_local, const double* z_partials,
                              int32_t world, int32_t t, float learning_rate, float exaggeration,
                              const tsne_config* cfg_in, float* v_local, float* gains_local,
                              float* Y_local_out, int32_t* flag, void* ws, size_t ws_bytes,
                              tsne_stream_t stream) {
  clear_error();
  tsne_config cfg;
  tsne_config_default(&cfg);
  if (cfg_in) cfg = *cfg_in;
  TSNE_ARG_CHECK(N >= 2 && 0 <= row0 && row0 <= row1 && row1 <= N, "bad row range");
  TSNE_ARG_CHECK(world >= 1 && t >= 0, "world must be >= 1, t >= 0");
  TSNE_ARG_CHECK(learning_rate > 0.f && exaggeration > 0.f, "learning_rate, exaggeration > 0");
  TSNE_ARG_CHECK(Y && z_partials && (row1 == row0 || (A_local && rep_local && v_local &&
                                                     gains_local && Y_local_out)),
                 "null pointer argument");
  ShardWS w;
  Carver c0(nullptr);
  carve_shard(c0, w, N);
  if (!ws || ws_bytes < c0.bytes()) {
    set_error("workspace too small: need %zu bytes, got %zu", c0.bytes(), ws_bytes);
    return TSNE_ERR_WORKSPACE;
  }
  tsne_status st = check_device();
  if (st != TSNE_OK) return st;
  Carver c(ws);
  carve_shard(c, w, N);
  Sched sc{cfg.exag_iters, exaggeration, cfg.mom0, cfg.mom1, learning_rate, cfg.min_gain};
  return launch_update_shard(
      reinterpret_cast<const float2*>(A_local), reinterpret_cast<const float2*>(Y), row0,
      row1 - row0, reinterpret_cast<const float2*>(rep_local), z_partials, world, t, sc,
      w.tree.box, reinterpret_cast<float2*>(v_local), reinterpret_cast<float2*>(gains_local),
      reinterpret_cast<float2*>(Y_local_out), flag, (cudaStream_t)stream);
}

tsne_status tsne_recentre(float* Y, int64_t N, void* ws, size_t ws_bytes, tsne_stream_t stream) {
  clear_error();
  TSNE_ARG_CHECK(N >= 2 && Y, "bad arguments");
  ShardWS w;
  Carver c0(nullptr);
  carve_shard(c0, w, N);
  if (!ws || ws_bytes < c0.bytes()) {
    set_error("workspace too small: need %zu bytes, got %zu", c0.bytes(), ws_bytes);
    return TSNE_ERR_WORKSPACE;
  }
  tsne_status st = check_device();
  if (st != TSNE_OK) return st;
  Carver c(ws);
  carve_shard(c, w, N);
  return shard_recentre(w, reinterpret_cast<float2*>(Y), N, (cudaStream_t)stream);
}

tsne_status tsne_init_y(int64_t N, uint64_t seed, float* Y, tsne_stream_t stream) {
  clear_error();
  TSNE_ARG_CHECK(N >= 1 && Y, "bad arguments");
  tsne_status st = check_device();
  if (st != TSNE_OK) return st;
  return launch_init_y(N, seed, reinterpret_cast<float2*>(Y), (cudaStream_t)stream);
}

// ---------------------------------------------------------------- kNN
size_t tsne_knn_workspace_size(int64_t N, int32_t D, int32_t K) {
  if (N < 2 || D < 1 || K < 1) return 0;
  KnnWS w;
  Carver c(nullptr);
  carve_knn(c, w, N, D, K);
  return c.bytes();
}

tsne_status tsne_knn(const float* X, int64_t N, int32_t D, int32_t K, int32_t* idx, double* d2,
                     void* ws, size_t ws_bytes, tsne_knn_info* info, tsne_stream_t stream) {
  clear_error();
  TSNE_ARG_CHECK(N >= 2 && N < (int64_t(1) << 31) - 1, "N must be in [2, 2^31-1)");
  TSNE_ARG_CHECK(D >= 1, "D must be >= 1");
  TSNE_ARG_CHECK(K >= 1 && K < N && K <= kMaxK, "K must satisfy 1 <= K < N and K <= %d", kMaxK);
  TSNE_ARG_CHECK(X && idx && d2, "null pointer argument");
  KnnWS w;
  Carver c0(nullptr);
  carve_knn(c0, w, N, D, K);
  if (!ws || ws_bytes < c0.bytes()) {
    set_error("workspace too small: need %zu bytes, got %zu", c0.bytes(), ws_bytes);
    return TSNE_ERR_WORKSPACE;
  }
  tsne_status st = check_device();
  if (st != TSNE_OK) return st;
  Carver c(ws);
  carve_knn(c, w, N, D, K);
  return run_knn(X, N, D, K, 0, N, idx, d2, w, info, (cudaStream_t)stream);
}

tsne_status tsne_knn_rows(const float* X, int64_t N, int32_t D, int32_t K, int64_t q0, int64_t nq,
                          int32_t* idx, double* d2, void* ws, size_t ws_bytes,
                          tsne_knn_info* info, tsne_stream_t stream) {
  clear_error();
  TSNE_ARG_CHECK(N >= 2 && N < (int64_t(1) << 31) - 1, "N must be in [2, 2^31-1)");
  TSNE_ARG_CHECK(D >= 1, "D must be >= 1");
  TSNE_ARG_CHECK(K >= 1 && K < N && K <= kMaxK, "K must satisfy 1 <= K < N and K <= %d", kMaxK);
  TSNE_ARG_CHECK(q0 >= 0 && nq >= 0 && q0 + nq <= N, "query rows [q0, q0+nq) must lie in [0, N)");
  TSNE_ARG_CHECK(X && (nq == 0 || (idx && d2)), "null pointer argument");
  KnnWS w;
  Carver c0(nullptr);
  carve_knn(c0, w, N, D, K);
  if (!ws || ws_bytes < c0.bytes()) {
    set_error("workspace too small: need %zu bytes, got %zu", c0.bytes(), ws_bytes);
    return TSNE_ERR_WORKSPACE;
  }
  tsne_status st = check_device();
  if (st != TSNE_OK) return st;
  if (nq == 0) {
    if (info) { info->rows_uncertified = 0; info->candidates = w.Kc; info->gemm_path = 0; }
    return TSNE_OK;
  }
  Carver c(ws);
  carve_knn(c, w, N, D, K);
  return run_knn(X, N, D, K, q0, nq, idx, d2, w, info, (cudaStream_t)stream);
}

// ---------------------------------------------------------------- P
size_t tsne_compute_p_workspace_size(int64_t N, int32_t K) {
  if (N < 2 || K < 1) return 0;
  PWS w;
  Carver c(nullptr);
  carve_p(c, w, N, K);
  return c.bytes();
}

tsne_status tsne_compute_p(const int32_t* idx, const double* d2, int64_t N, int32_t K,
                           float perplexity, int64_t* row_ptr, int32_t* col, float* val,
                           int64_t* nnz_out, double* beta_out, void* ws, size_t ws_bytes,
                           tsne_stream_t stream) {
  clear_error();
  TSNE_ARG_CHECK(N >= 2 && N < (int64_t(1) << 31) - 1, "N must be in [2, 2^31-1)");
  TSNE_ARG_CHECK(K >= 1 && K < N && K <= kMaxK, "K must satisfy 1 <= K < N, K <= %d", kMaxK);
  TSNE_ARG_CHECK(perplexity > 1.f && perplexity < (float)K,
                 "perplexity must satisfy 1 < perplexity < K (got %g, K=%d)", perplexity, K);
  TSNE_ARG_CHECK(idx && d2 && row_ptr && col && val && nnz_out, "null pointer argument");
  TSNE_ARG_CHECK(2 * N * (int64_t)K < (int64_t(1) << 31),
                 "2 N K must be < 2^31 (directed edges of the symmetrisation, int32 positions)");
  PWS w;
  Carver c0(nullptr);
  carve_p(c0, w, N, K);
  if (!ws || ws_bytes < c0.bytes()) {
    set_error("workspace too small: need %zu bytes, got %zu", c0.bytes(), ws_bytes);
    return TSNE_ERR_WORKSPACE;
  }
  tsne_status st = check_device();
  if (st != TSNE_OK) return st;
  Carver c(ws);
  carve_p(c, w, N, K);
  int64_t ndeg = 0;
  st = run_compute_p(idx, d2, N, K, perplexity, row_ptr, col, val, nnz_out, beta_out, w, &ndeg,
                     (cudaStream_t)stream);
  if (st == TSNE_OK && ndeg > 0) {
    set_error("%lld rows had no finite bandwidth (uniform rows, D3)", (long long)ndeg);
    return TSNE_ERR_DEGENERATE;
  }
  return st;
}

// ---------------------------------------------------------------- run
tsne_status tsne_run_ex(const float* X, int64_t N, int32_t D, float perplexity, float theta,
                        float learning_rate, int32_t n_iter, float exaggeration,
                        const tsne_config* cfg_in, float* Y_out, tsne_run_info* info) {
  clear_error();
  tsne_config cfg;
  tsne_config_default(&cfg);
  if (cfg_in) cfg = *cfg_in;
  TSNE_ARG_CHECK(N >= 2 && N <= kMaxTreePoints, "N must be in [2, 2^25) (got %lld)", (long long)N);
  TSNE_ARG_CHECK(D >= 1, "D must be >= 1");
  TSNE_ARG_CHECK(X && Y_out, "null pointer argument");
  int32_t K = cfg.K > 0 ? cfg.K : (int32_t)std::floor(3.0 * (double)perplexity);
  if (K > N - 1) K = (int32_t)(N - 1);
  TSNE_ARG_CHECK(K >= 1 && K <= kMaxK, "K must be in [1, %d] (got %d)", kMaxK, K);
  TSNE_ARG_CHECK(perplexity > 1.f && perplexity < (float)K,
                 "perplexity must satisfy 1 < perplexity < K (got %g, K=%d)", perplexity, K);
  TSNE_ARG_CHECK(theta >= 0.f && std::isfinite(theta), "theta must be >= 0");
  TSNE_ARG_CHECK(learning_rate > 0.f, "learning_rate must be > 0");
  TSNE_ARG_CHECK(n_iter >= 1, "n_iter must be >= 1");
  TSNE_ARG_CHECK(exaggeration >= 1.f, "exaggeration must be >= 1");
  TSNE_ARG_CHECK(2 * N * (int64_t)K < (int64_t(1) << 31),
                 "2 N K must be < 2^31 (directed edges of the symmetrisation, int32 positions)");
  tsne_status st = check_device();
  if (st != TSNE_OK) return st;

  cudaPointerAttributes ax{}, ay{};
  TSNE_CUDA_TRY(cudaPointerGetAttributes(&ax, X));
  TSNE_CUDA_TRY(cudaPointerGetAttributes(&ay, Y_out));
  const bool x_host = ax.type != cudaMemoryTypeDevice && ax.type != cudaMemoryTypeManaged;
  const bool y_host = ay.type != cudaMemoryTypeDevice && ay.type != cudaMemoryTypeManaged;

  cudaStream_t s;
  TSNE_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t ev[6];
  for (auto& e : ev) cudaEventCreate(&e);
  const int64_t cap = 2 * N * (int64_t)K;
  size_t kb, pb, ob;
  {
    KnnWS w; Carver c(nullptr); carve_knn(c, w, N, D, K); kb = c.bytes();
  }
  {
    PWS w; Carver c(nullptr); carve_p(c, w, N, K); pb = c.bytes();
  }
  ob = tsne_optimize_workspace_size(N, cap);
  // buffers: X (if host), idx, d2, row_ptr, col, val, Y, v, gains, workspace
  Carver plan(nullptr);
  plan.take<float>(x_host ? N * D : 0);
  plan.take<int32_t>(N * K);
  plan.take<double>(N * K);
  plan.take<int64_t>(N + 1);
  plan.take<int32_t>(cap);
  plan.take<float>(cap);
  plan.take<float2>(N);
  plan.take<float2>(N);
  plan.take<float2>(N);
  plan.take<int32_t>(1);
  size_t ws_need = kb > pb ? kb : pb;
  ws_need = ws_need > ob ? ws_need : ob;
  size_t ivf_idx = 0, ivf_ws = 0;
  if (cfg.knn_tau > 0) {               // IVF-PQ: the index, then its workspace
    ivf_idx = (tsne_ivfpq_index_size(N, D, nullptr) + 255) & ~size_t(255);
    ivf_ws = tsne_ivfpq_workspace_size(N, D, K, nullptr);
    ws_need = ws_need > ivf_idx + ivf_ws ? ws_need : ivf_idx + ivf_ws;
  }
  plan.take<char>(ws_need);
  void* mem = nullptr;
  const bool timing = getenv("TSNE_RUN_TIMING") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto t0 = now();
  // plain cudaMalloc: for tens of GB it maps in milliseconds, where the
  // stream-ordered pool took 0.3-1 s to map and 0.3-5 s to release (measured)
  cudaError_t e = cudaMalloc(&mem, plan.bytes());
  if (timing) {
    cudaStreamSynchronize(s);
    fprintf(stderr, "tsne_run: alloc %.1f GB %.1f ms\n", plan.bytes() / 1e9,
            std::chrono::duration<double, std::milli>(now() - t0).count());
  }
  if (e != cudaSuccess) {
    for (auto& x : ev) cudaEventDestroy(x);
    cudaStreamDestroy(s);
    set_error("cudaMalloc(%zu): %s", plan.bytes(), cudaGetErrorString(e));
    return TSNE_ERR_CUDA;
  }
  Carver c(mem);
  float* Xd = c.take<float>(x_host ? N * D : 0);
  int32_t* idx = c.take<int32_t>(N * K);
  double* d2 = c.take<double>(N * K);
  int64_t* rp = c.take<int64_t>(N + 1);
  int32_t* col = c.take<int32_t>(cap);
  float* val = c.take<float>(cap);
  float2* Y = c.take<float2>(N);
  float2* V = c.take<float2>(N);
  float2* G = c.take<float2>(N);
  int32_t* bad = c.take<int32_t>(1);
  void* ws = c.take<char>(ws_need);

  tsne_knn_info kinfo{};
  int64_t nnz = 0, ndeg = 0;
  int32_t hbad = 0;
  cudaEventRecord(ev[0], s);
  if (x_host) e = cudaMemcpyAsync(Xd, X, sizeof(float) * N * D, cudaMemcpyHostToDevice, s);
  const float* Xuse = x_host ? Xd : X;
  cudaEventRecord(ev[1], s);
  st = (e == cudaSuccess) ? TSNE_OK : TSNE_ERR_CUDA;
  if (st == TSNE_OK) st = check_finite(Xuse, N * (int64_t)D, bad, &hbad, s);
  if (st == TSNE_OK && hbad) {
    set_error("X contains non-finite values");
    st = TSNE_ERR_ARG;
  }
  if (st == TSNE_OK && cfg.knn_tau > 0) {
    char* ib = static_cast<char*>(ws);
    st = tsne_ivfpq_build(Xuse, N, D, nullptr, ib, ivf_idx, ib + ivf_idx, ivf_ws,
                          (tsne_stream_t)s);
    if (st == TSNE_OK)
      st = tsne_ivfpq_search(Xuse, N, D, nullptr, ib, K, cfg.knn_tau, idx, d2, ib + ivf_idx,
                             ivf_ws, (tsne_stream_t)s);
  } else if (st == TSNE_OK) {
    KnnWS kw; Carver kc(ws); carve_knn(kc, kw, N, D, K);
    st = run_knn(Xuse, N, D, K, 0, N, idx, d2, kw, &kinfo, s);
  }
  cudaEventRecord(ev[2], s);
  if (st == TSNE_OK) {
    PWS pw; Carver pc(ws); carve_p(pc, pw, N, K);
    st = run_compute_p(idx, d2, N, K, perplexity, rp, col, val, &nnz, nullptr, pw, &ndeg, s);
  }
  cudaEventRecord(ev[3], s);
  if (st == TSNE_OK) {
    if (cfg.Y_init) {
      e = cudaMemcpyAsync(Y, cfg.Y_init, sizeof(float2) * N, cudaMemcpyDefault, s);
      if (e != cudaSuccess) { set_error("Y_init copy: %s", cudaGetErrorString(e)); st = TSNE_ERR_CUDA; }
    } else {
      st = launch_init_y(N, cfg.seed, Y, s);
    }
  }
  if (st == TSNE_OK) {
    cudaMemsetAsync(V, 0, sizeof(float2) * N, s);
    st = fill_ones(reinterpret_cast<float*>(G), 2 * N, s);
  }
  if (st == TSNE_OK) {
    OptPlan p;
    opt_plan(ws, N, nnz, p);
    st = init_tree_ws(p.tree, s);
    Sched sc{cfg.exag_iters, exaggeration, cfg.mom0, cfg.mom1, learning_rate, cfg.min_gain};
    if (st == TSNE_OK)
      st = run_iterations(rp, col, val, N, Y, V, G, 0, n_iter, theta, sc, cfg.use_graphs != 0,
                          cfg.relabel_every, p.tree, p.opt, s, /*cache_order=*/false);
    if (st == TSNE_OK) {
      int32_t flag = 0;
      cudaMemcpyAsync(&flag, p.opt.flag, sizeof(flag), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      if (flag) { set_error("non-finite embedding"); st = TSNE_ERR_NONFINITE; }
    }
  }
  cudaEventRecord(ev[4], s);
  if (st == TSNE_OK) {
    e = cudaMemcpyAsync(Y_out, Y, sizeof(float2) * N,
                        y_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) { set_error("Y_out copy: %s", cudaGetErrorString(e)); st = TSNE_ERR_CUDA; }
  }
  cudaEventRecord(ev[5], s);
  auto t1 = now();
  if (timing) cudaStreamSynchronize(s);
  auto t2 = now();
  e = cudaStreamSynchronize(s);
  cudaFree(mem);
  if (timing)
    fprintf(stderr, "tsne_run: tail sync %.1f ms, free %.1f ms\n",
            std::chrono::duration<double, std::milli>(t2 - t1).count(),
            std::chrono::duration<double, std::milli>(now() - t2).count());
  if (st == TSNE_OK && e != cudaSuccess) {
    set_error("tsne_run: %s", cudaGetErrorString(e));
    st = TSNE_ERR_CUDA;
  }
  if (info) {
    float ms[5] = {0, 0, 0, 0, 0};
    for (int k = 0; k < 5; ++k) cudaEventElapsedTime(&ms[k], ev[k], ev[k + 1]);
    info->ms_h2d = ms[0];
    info->ms_knn = ms[1];
    info->ms_p = ms[2];
    info->ms_loop = ms[3];
    info->ms_d2h = ms[4];
    float tot = 0;
    cudaEventElapsedTime(&tot, ev[0], ev[5]);
    info->ms_total = tot;
    info->nnz = nnz;
    info->knn_rows_uncertified = kinfo.rows_uncertified;
    info->K = K;
    info->degenerate_rows = (int32_t)ndeg;
  }
  for (auto& x : ev) cudaEventDestroy(x);
  cudaStreamDestroy(s);
  return st;
}

tsne_status tsne_run(const float* X, int64_t N, int32_t D, float perplexity, float theta,
                     float learning_rate, int32_t n_iter, float exaggeration, float* Y_out) {
  return tsne_run_ex(X, N, D, perplexity, theta, learning_rate, n_iter, exaggeration, nullptr,
                     Y_out, nullptr);
}

}  // extern "C"
