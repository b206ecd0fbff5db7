// run_sharded.cu -- Algorithm 1 end to end on G GPUs, one process per GPU
// (the paper is single-GPU), with the communicator owned
// by the library: tsne_nccl_unique_id / tsne_run_sharded / tsne_run_workspace_size.
//
// Per rank r (rows [r S, min(N, (r+1) S)) of the locality labels, S = ceil(N / G)):
//   1. X: own rows -> device (H2D if host), NCCL all-gather -> X on every rank
//   2. kNN of the own query rows against all N points (run_knn, row sweep)
//   3. NCCL all-gather of the kNN lists; P built redundantly (needs every row
//      for the symmetrisation, ~40 ms at C5); the locality labels (the
//      diffusion order of P, identical on every rank) and P relabelled by them;
//      the own rows (a contiguous label range) kept
//   4. per iteration: attractive sums of the own rows (side stream) ||
//      quadtree over the full Y (redundant) + traversal of the own points;
//      all-gather of the Z partials (rank order: every rank adds them in the
//      same order, deterministic); Eq. 7 + D12 update of the own rows;
//      all-gather of the Y shards.  One CUDA graph per schedule phase.
//   5. recentring (D15); rank 0 copies Y to Y_out.
// NCCL is loaded at run time (dlopen of libnccl.so.2: the copy PyTorch has
// already loaded, if any), so the library has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>

#include "affinity.cuh"
#include "knn.cuh"
#include "shard.cuh"

namespace tsne {

tsne_status check_device();

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi g_nccl;
std::once_flag g_nccl_once;

const NcclApi* nccl() {
  std::call_once(g_nccl_once, [] {
    NcclApi& a = g_nccl;
    a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);       // PyTorch's copy, if loaded
    if (!a.h) a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) a.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) return;
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(a.h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(a.h, "ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(a.h, "ncclCommDestroy");
    a.CommAbort = (decltype(a.CommAbort))dlsym(a.h, "ncclCommAbort");
    a.AllGather = (decltype(a.AllGather))dlsym(a.h, "ncclAllGather");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(a.h, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.CommAbort && a.AllGather &&
           a.GetErrorString;
  });
  return g_nccl.ok ? &g_nccl : nullptr;
}

#define TSNE_NCCL_TRY(expr)                                                              \
  do {                                                                                   \
    ncclResult_t r__ = (expr);                                                           \
    if (r__ != ncclSuccess) {                                                            \
      ::tsne::set_error("%s:%d %s -> %s", __FILE__, __LINE__, #expr,                     \
                        nc->GetErrorString(r__));                                        \
      return TSNE_ERR_NCCL;                                                              \
    }                                                                                    \
  } while (0)

__global__ void k_gather_y(const int32_t* __restrict__ perm, const float2* __restrict__ src,
                           int N, float2* __restrict__ dst) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < N) dst[k] = src[perm[k]];
}

__global__ void k_scatter_y(const int32_t* __restrict__ perm, const float2* __restrict__ src,
                            int N, float2* __restrict__ dst) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < N) dst[perm[k]] = src[k];
}

// rows [r0, r1) of the global CSR as a local CSR (offsets rebased)
__global__ void k_rebase(const int64_t* __restrict__ rp, int64_t r0, int64_t n,
                         int64_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i <= n) out[i] = rp[r0 + i] - rp[r0];
}

// Everything one rank allocates, carved from one buffer (sizes: plan()).
struct RankPlan {
  int64_t N, S, n_loc;
  int32_t D, K, G;
  int64_t cap;             // 2 N K: CSR capacity
  float* Xloc;             // S x D (own rows, padded)
  float* X;                // G S x D (all rows)
  int32_t* idx_l;          // S x K
  double* d2_l;            // S x K
  int32_t* idx;            // G S x K
  double* d2;              // G S x K
  int64_t* rp;             // N + 1
  int32_t* col;            // cap
  float* val;              // cap
  int64_t* rp_l;           // S + 1
  int32_t* col_l;          // cap (own rows)
  float* val_l;            // cap
  AtPlan atp;              // the attractive pass's batches of the own rows
  float2* Yfull;           // G S
  float2* Yloc;            // S
  float2 *V, *Gn, *rep, *A;  // S each
  double* zpart;           // 2
  double* zparts;          // 2 G
  int32_t* flag;           // 1 (+ non-finite X flag)
  // locality labels (the diffusion order of P): rank r owns a
  // contiguous range of labels, so its rows' neighbours fall in its window
  int32_t* perm;           // N  label -> point
  int32_t* inv;            // N
  int64_t* len;            // N + 1
  float2* u;               // 2N scratch (diffusion coordinates, Y by point)
  int64_t* rp2;            // N + 1   P in labels
  int32_t* col2;           // cap
  float* val2;             // cap
  void* scan_tmp;
  size_t scan_bytes;
  void* ws;                // max(kNN, P) scratch, then the shard workspace
  size_t ws_bytes;
};

size_t plan(RankPlan& p, void* base, int64_t N, int32_t D, int32_t K, int G) {
  p.N = N; p.D = D; p.K = K; p.G = G;
  p.S = (N + G - 1) / G;
  p.cap = 2 * N * (int64_t)K;
  const int64_t S = p.S;
  Carver c(base);
  p.Xloc = c.take<float>(S * D);
  p.X = c.take<float>(G * S * D);
  p.idx_l = c.take<int32_t>(S * K);
  p.d2_l = c.take<double>(S * K);
  p.idx = c.take<int32_t>(G * S * K);
  p.d2 = c.take<double>(G * S * K);
  p.rp = c.take<int64_t>(N + 1);
  p.col = c.take<int32_t>(p.cap + 4);
  p.val = c.take<float>(p.cap + 4);
  p.rp_l = c.take<int64_t>(S + 1);
  p.col_l = c.take<int32_t>(p.cap + 4);
  p.val_l = c.take<float>(p.cap + 4);
  carve_attract_plan(c, p.atp, S, p.cap, attract_grid_shard(S));
  p.Yfull = c.take<float2>(G * S);
  p.Yloc = c.take<float2>(S);
  p.V = c.take<float2>(S);
  p.Gn = c.take<float2>(S);
  p.rep = c.take<float2>(S);
  p.A = c.take<float2>(S);
  p.zpart = c.take<double>(2);
  p.zparts = c.take<double>(2 * G);
  p.flag = c.take<int32_t>(2);
  p.perm = c.take<int32_t>(N);
  p.inv = c.take<int32_t>(N);
  p.len = c.take<int64_t>(N + 1);
  p.u = c.take<float2>(2 * N);
  p.rp2 = c.take<int64_t>(N + 1);
  p.col2 = c.take<int32_t>(p.cap + 4);
  p.val2 = c.take<float>(p.cap + 4);
  p.scan_bytes = permute_csr_scan_bytes(N);
  p.scan_tmp = c.take<char>(p.scan_bytes);
  size_t kb, pb, sb;
  { KnnWS w; Carver q(nullptr); carve_knn(q, w, N, D, K); kb = q.bytes(); }
  { PWS w; Carver q(nullptr); carve_p(q, w, N, K); pb = q.bytes(); }
  { ShardWS w; Carver q(nullptr); carve_shard(q, w, N); sb = q.bytes(); }
  p.ws_bytes = kb > pb ? kb : pb;
  p.ws_bytes = p.ws_bytes > sb ? p.ws_bytes : sb;
  p.ws = c.take<char>(p.ws_bytes);
  return c.bytes();
}

struct Comm {
  const NcclApi* nc = nullptr;
  ncclComm_t comm = nullptr;
  bool failed = false;
  ~Comm() {
    if (!comm) return;
    if (failed) nc->CommAbort(comm);
    else nc->CommDestroy(comm);
  }
};

struct Res {
  void* mem = nullptr;
  cudaStream_t s = nullptr, side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaEvent_t ev[6] = {};
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  cudaGraph_t graph[2] = {nullptr, nullptr};
  ~Res() {
    if (s) cudaStreamSynchronize(s);
    for (int k = 0; k < 2; ++k) {
      if (gexec[k]) cudaGraphExecDestroy(gexec[k]);
      if (graph[k]) cudaGraphDestroy(graph[k]);
    }
    for (auto e : ev) if (e) cudaEventDestroy(e);
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (side) cudaStreamDestroy(side);
    if (s) cudaStreamDestroy(s);
    if (mem) cudaFree(mem);
  }
};

// one sharded iteration (t: the iteration number, for the schedule phase)
tsne_status iteration(RankPlan& p, ShardWS& w, const NcclApi* nc, ncclComm_t comm, int rank,
                      int t, bool recentre, float theta, const Sched& sc, Res& r) {
  const int64_t r0 = (int64_t)rank * p.S;
  const int64_t r1 = r0 + p.n_loc;
  cudaStream_t s = r.s;
  TSNE_CUDA_TRY(cudaEventRecord(r.fork, s));
  TSNE_CUDA_TRY(cudaStreamWaitEvent(r.side, r.fork, 0));
  tsne_status st = launch_attract_sum_shard(p.rp_l, p.col_l, p.val_l, p.Yfull, p.N, r0, p.n_loc,
                                            p.A, &p.atp, r.side);
  if (st != TSNE_OK) return st;
  TSNE_CUDA_TRY(cudaEventRecord(r.join, r.side));
  if ((st = shard_forces(w, p.Yfull, p.N, r0, r1, theta, recentre, p.rep, p.zpart, s)) != TSNE_OK)
    return st;
  TSNE_CUDA_TRY(cudaStreamWaitEvent(s, r.join, 0));
  TSNE_NCCL_TRY(nc->AllGather(p.zpart, p.zparts, 2, ncclFloat64, comm, s));
  if ((st = launch_update_shard(p.A, p.Yfull, r0, p.n_loc, p.rep, p.zparts, p.G, t, sc,
                                w.tree.box, p.V, p.Gn, p.Yloc, p.flag, s)) != TSNE_OK)
    return st;
  TSNE_NCCL_TRY(nc->AllGather(p.Yloc, p.Yfull, 2 * p.S, ncclFloat32, comm, s));
  return TSNE_OK;
}

}  // namespace
}  // namespace tsne

using namespace tsne;

extern "C" {

tsne_status tsne_nccl_unique_id(void* id_out) {
  clear_error();
  TSNE_ARG_CHECK(id_out, "null pointer argument");
  const NcclApi* nc = nccl();
  if (!nc) {
    set_error("NCCL (libnccl.so.2) could not be loaded");
    return TSNE_ERR_NCCL;
  }
  ncclUniqueId id;
  TSNE_NCCL_TRY(nc->GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == TSNE_NCCL_ID_BYTES, "ncclUniqueId size");
  memcpy(id_out, &id, sizeof(id));
  return TSNE_OK;
}

size_t tsne_run_workspace_size(int64_t N, int32_t D, int32_t K, int32_t world) {
  if (N < 2 || D < 1 || K < 1 || world < 1) return 0;
  RankPlan p;
  return plan(p, nullptr, N, D, K, world);
}

tsne_status tsne_run_sharded(const float* X_local, int64_t N_local, int64_t N, int32_t D,
                             float perplexity, float theta, float learning_rate, int32_t n_iter,
                             float exaggeration, const tsne_config* cfg_in,
                             const void* nccl_unique_id, int32_t rank, int32_t world,
                             float* Y_out, tsne_run_info* info) {
  clear_error();
  tsne_config cfg;
  tsne_config_default(&cfg);
  if (cfg_in) cfg = *cfg_in;
  TSNE_ARG_CHECK(N >= 2 && N <= kMaxTreePoints, "N must be in [2, 2^25) (got %lld)", (long long)N);
  TSNE_ARG_CHECK(D >= 1, "D must be >= 1");
  TSNE_ARG_CHECK(world >= 1 && rank >= 0 && rank < world, "need 0 <= rank < world");
  const int64_t S = (N + world - 1) / world;
  const int64_t r0 = std::min<int64_t>(N, (int64_t)rank * S);
  const int64_t n_loc = std::min<int64_t>(N, r0 + S) - r0;
  TSNE_ARG_CHECK(N_local == n_loc, "N_local must be %lld for rank %d of %d (rows [%lld, %lld))",
                 (long long)n_loc, rank, world, (long long)r0, (long long)(r0 + n_loc));
  TSNE_ARG_CHECK((X_local || n_loc == 0) && nccl_unique_id && (Y_out || rank != 0),
                 "null pointer argument");
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
  const NcclApi* nc = nccl();
  if (!nc) {
    set_error("NCCL (libnccl.so.2) could not be loaded");
    return TSNE_ERR_NCCL;
  }
  cudaPointerAttributes ax{}, ay{};
  if (X_local) TSNE_CUDA_TRY(cudaPointerGetAttributes(&ax, X_local));
  if (Y_out) TSNE_CUDA_TRY(cudaPointerGetAttributes(&ay, Y_out));
  const bool y_host = ay.type != cudaMemoryTypeDevice && ay.type != cudaMemoryTypeManaged;

  RankPlan p;
  const size_t bytes = plan(p, nullptr, N, D, K, world);
  p.n_loc = n_loc;
  Res r;
  TSNE_CUDA_TRY(cudaStreamCreateWithFlags(&r.s, cudaStreamNonBlocking));
  TSNE_CUDA_TRY(cudaStreamCreateWithFlags(&r.side, cudaStreamNonBlocking));
  TSNE_CUDA_TRY(cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming));
  TSNE_CUDA_TRY(cudaEventCreateWithFlags(&r.join, cudaEventDisableTiming));
  for (auto& e : r.ev) TSNE_CUDA_TRY(cudaEventCreate(&e));
  cudaError_t e = cudaMalloc(&r.mem, bytes);
  if (e != cudaSuccess) {
    r.mem = nullptr;
    set_error("cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
    return TSNE_ERR_CUDA;
  }
  plan(p, r.mem, N, D, K, world);
  p.n_loc = n_loc;
  cudaStream_t s = r.s;

  Comm cm;
  cm.nc = nc;
  ncclUniqueId id;
  memcpy(&id, nccl_unique_id, sizeof(id));
  {
    ncclResult_t nr = nc->CommInitRank(&cm.comm, world, id, rank);
    if (nr != ncclSuccess) {
      cm.comm = nullptr;
      set_error("ncclCommInitRank(world %d, rank %d): %s", world, rank, nc->GetErrorString(nr));
      return TSNE_ERR_NCCL;
    }
  }
  cm.failed = true;                 // until the end: abort the communicator on an early return
  tsne_knn_info kinfo{};
  int64_t nnz = 0, ndeg = 0;
  int32_t hbad = 0;

  // 1. X
  TSNE_CUDA_TRY(cudaEventRecord(r.ev[0], s));
  TSNE_CUDA_TRY(cudaMemsetAsync(p.Xloc, 0, sizeof(float) * S * D, s));
  if (n_loc > 0)
    TSNE_CUDA_TRY(cudaMemcpyAsync(p.Xloc, X_local, sizeof(float) * n_loc * D, cudaMemcpyDefault, s));
  TSNE_NCCL_TRY(nc->AllGather(p.Xloc, p.X, (size_t)S * D, ncclFloat32, cm.comm, s));
  TSNE_CUDA_TRY(cudaEventRecord(r.ev[1], s));
  if ((st = check_finite(p.X, N * (int64_t)D, p.flag + 1, &hbad, s)) != TSNE_OK) return st;
  if (hbad) {
    set_error("X contains non-finite values");
    return TSNE_ERR_ARG;
  }
  // 2. kNN of the own query rows
  TSNE_CUDA_TRY(cudaMemsetAsync(p.idx_l, 0, sizeof(int32_t) * S * K, s));
  TSNE_CUDA_TRY(cudaMemsetAsync(p.d2_l, 0, sizeof(double) * S * K, s));
  {
    KnnWS kw; Carver kc(p.ws); carve_knn(kc, kw, N, D, K);
    if (n_loc > 0 &&
        (st = run_knn(p.X, N, D, K, r0, n_loc, p.idx_l, p.d2_l, kw, &kinfo, s)) != TSNE_OK)
      return st;
  }
  // 3. the lists of every rank, P (redundant), the own rows
  TSNE_NCCL_TRY(nc->AllGather(p.idx_l, p.idx, (size_t)S * K, ncclInt32, cm.comm, s));
  TSNE_NCCL_TRY(nc->AllGather(p.d2_l, p.d2, (size_t)S * K, ncclFloat64, cm.comm, s));
  TSNE_CUDA_TRY(cudaEventRecord(r.ev[2], s));
  {
    PWS pw; Carver pc(p.ws); carve_p(pc, pw, N, K);
    if ((st = run_compute_p(p.idx, p.d2, N, K, perplexity, p.rp, p.col, p.val, &nnz, nullptr, pw,
                            &ndeg, s)) != TSNE_OK)
      return st;
  }
  ShardWS w;
  {
    Carver c(p.ws);
    carve_shard(c, w, N);
  }
  if ((st = tree_ws_init(w.tree, s)) != TSNE_OK) return st;
  // locality labels: the diffusion order of P, computed identically on every
  // rank (P and the code are identical); the ranks then own label ranges
  if ((st = diffusion_perm(p.rp, p.col, p.val, N, w.tree, p.u, p.perm, s)) != TSNE_OK) return st;
  if ((st = permute_csr(p.perm, N, p.rp, p.col, p.val, p.inv, p.len, p.scan_tmp, p.scan_bytes,
                        p.rp2, p.col2, p.val2, s)) != TSNE_OK)
    return st;
  int64_t e0 = 0, e1 = 0;
  TSNE_CUDA_TRY(cudaMemcpyAsync(&e0, p.rp2 + r0, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  TSNE_CUDA_TRY(cudaMemcpyAsync(&e1, p.rp2 + r0 + n_loc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  TSNE_CUDA_TRY(cudaStreamSynchronize(s));
  k_rebase<<<(int)((n_loc + 256) / 256), 256, 0, s>>>(p.rp2, r0, n_loc, p.rp_l);
  TSNE_LAUNCH_CHECK();
  if (e1 > e0) {                    // 16-byte aligned copies of the own rows (bulk-copy streams)
    TSNE_CUDA_TRY(cudaMemcpyAsync(p.col_l, p.col2 + e0, sizeof(int32_t) * (e1 - e0),
                                  cudaMemcpyDeviceToDevice, s));
    TSNE_CUDA_TRY(cudaMemcpyAsync(p.val_l, p.val2 + e0, sizeof(float) * (e1 - e0),
                                  cudaMemcpyDeviceToDevice, s));
  }
  p.atp.grid = attract_grid_shard(n_loc);   // <= the grid the plan was sized for
  if ((st = attract_plan_build(p.atp, p.rp_l, n_loc, s)) != TSNE_OK) return st;
  TSNE_CUDA_TRY(cudaEventRecord(r.ev[3], s));
  // 4. iterations
  TSNE_CUDA_TRY(cudaMemsetAsync(p.Yfull, 0, sizeof(float2) * world * S, s));
  if (cfg.Y_init) {                 // Y0 by point, then in labels
    TSNE_CUDA_TRY(cudaMemcpyAsync(p.u, cfg.Y_init, sizeof(float2) * N, cudaMemcpyDefault, s));
  } else if ((st = launch_init_y(N, cfg.seed, p.u, s)) != TSNE_OK) {
    return st;
  }
  k_gather_y<<<(int)((N + 255) / 256), 256, 0, s>>>(p.perm, p.u, (int)N, p.Yfull);
  TSNE_LAUNCH_CHECK();
  TSNE_CUDA_TRY(cudaMemsetAsync(p.V, 0, sizeof(float2) * S, s));
  if ((st = fill_ones(reinterpret_cast<float*>(p.Gn), 2 * S, s)) != TSNE_OK) return st;
  TSNE_CUDA_TRY(cudaMemsetAsync(p.flag, 0, sizeof(int32_t), s));
  if ((st = tree_ws_init(w.tree, s)) != TSNE_OK) return st;
  Sched sc{cfg.exag_iters, exaggeration, cfg.mom0, cfg.mom1, learning_rate, cfg.min_gain};
  const bool graphs = cfg.use_graphs != 0;
  for (int32_t t = 0; t < n_iter; ++t) {
    const int phase = t >= cfg.exag_iters ? 1 : 0;
    if (graphs && t > 0) {
      if (!r.gexec[phase]) {
        TSNE_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        st = iteration(p, w, nc, cm.comm, rank, t, true, theta, sc, r);
        cudaError_t ce = cudaStreamEndCapture(s, &r.graph[phase]);
        if (st != TSNE_OK) return st;
        TSNE_CUDA_TRY(ce);
        TSNE_CUDA_TRY(cudaGraphInstantiate(&r.gexec[phase], r.graph[phase], 0));
      }
      TSNE_CUDA_TRY(cudaGraphLaunch(r.gexec[phase], s));
    } else if ((st = iteration(p, w, nc, cm.comm, rank, t, t > 0, theta, sc, r)) != TSNE_OK) {
      return st;
    }
  }
  if ((st = shard_recentre(w, p.Yfull, N, s)) != TSNE_OK) return st;
  int32_t flag = 0;
  TSNE_CUDA_TRY(cudaMemcpyAsync(&flag, p.flag, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  TSNE_CUDA_TRY(cudaEventRecord(r.ev[4], s));
  // 5. result
  if (rank == 0) {                  // back to the caller's point order
    k_scatter_y<<<(int)((N + 255) / 256), 256, 0, s>>>(p.perm, p.Yfull, (int)N, p.u);
    TSNE_LAUNCH_CHECK();
    TSNE_CUDA_TRY(cudaMemcpyAsync(Y_out, p.u, sizeof(float2) * N,
                                  y_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
  }
  TSNE_CUDA_TRY(cudaEventRecord(r.ev[5], s));
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    set_error("tsne_run_sharded: %s", cudaGetErrorString(e));
    return TSNE_ERR_CUDA;
  }
  cm.failed = false;
  if (info) {
    float ms[5] = {0, 0, 0, 0, 0};
    for (int k = 0; k < 5; ++k) cudaEventElapsedTime(&ms[k], r.ev[k], r.ev[k + 1]);
    info->ms_h2d = ms[0];           // own rows H2D + all-gather of X
    info->ms_knn = ms[1];           // own query rows + all-gather of the lists
    info->ms_p = ms[2];
    info->ms_loop = ms[3];
    info->ms_d2h = ms[4];
    float tot = 0;
    cudaEventElapsedTime(&tot, r.ev[0], r.ev[5]);
    info->ms_total = tot;
    info->nnz = nnz;
    info->knn_rows_uncertified = kinfo.rows_uncertified;   // this rank's rows
    info->K = K;
    info->degenerate_rows = (int32_t)ndeg;
  }
  if (flag) {
    set_error("non-finite embedding");
    return TSNE_ERR_NONFINITE;
  }
  return TSNE_OK;
}

}  // extern "C"
