/*
 * include/tsne.h -- C ABI of the B200-native Barnes-Hut t-SNE library
 * (libtsne_b200.so), after t-SNE-CUDA, arXiv 1807.11824.
 *
 * Citations: "P:Lnnn" = /root/reference/PAPER.md line (section / equation
 * named beside it); "Dnn" = a reading of the paper recorded in DESIGN.md
 * section 3 (where the paper is silent, ambiguous or garbled).
 *
 * General contract (all entry points):
 *  - Arrays are row-major.  Unless an argument says HOST, pointers are
 *    DEVICE pointers on the current CUDA device, caller-owned: the library
 *    never frees caller memory and, except tsne_run / tsne_run_ex, never
 *    allocates device memory.  Scratch comes from a caller-provided
 *    workspace `ws` of `ws_bytes` bytes (query the *_workspace_size
 *    function; 256-byte aligned), so the caller's allocator (PyTorch's
 *    caching allocator) owns all device memory.
 *  - Every call is stream-ordered on `stream` (NULL = legacy default
 *    stream) and returns before the GPU work completes, unless it says it
 *    synchronises.
 *  - Inputs are read-only.  Outputs are written only when TSNE_OK is
 *    returned; on error their contents are unspecified.
 *  - Argument validation happens before any launch; a failure returns
 *    TSNE_ERR_ARG and sets the thread-local message read by
 *    tsne_last_error().  CUDA launch/runtime failures return TSNE_ERR_CUDA.
 *  - Calls are re-entrant given distinct workspaces and streams.
 *  - There is no CPU fallback: a host without a usable sm_100 device gets
 *    TSNE_ERR_CUDA from every compute entry point.
 */
#ifndef TSNE_B200_H
#define TSNE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* tsne_stream_t; /* == cudaStream_t */

typedef enum {
  TSNE_OK = 0,
  TSNE_ERR_ARG = 1,        /* invalid argument (message in tsne_last_error) */
  TSNE_ERR_CUDA = 2,       /* CUDA runtime / launch failure, or no device   */
  TSNE_ERR_WORKSPACE = 3,  /* ws == NULL or ws_bytes < required size        */
  TSNE_ERR_NONFINITE = 4,  /* NaN/Inf appeared in Y during optimisation     */
  TSNE_ERR_NCCL = 5,       /* a failed NCCL communicator or collective (tsne_run_sharded) */
  TSNE_ERR_DEGENERATE = 6  /* non-fatal: some rows had no finite beta (D3)  */
} tsne_status;

/* Thread-local, NUL-terminated message describing the last failure of a call
 * made by this thread ("" if none).  Owned by the library. */
const char* tsne_last_error(void);

/* ABI version, (major << 16) | minor. */
int32_t tsne_abi_version(void);

/* ------------------------------------------------------------------------
 * U1  Exact k nearest neighbours (Sec. III-B: "the K nearest
 * neighbors of each point are obtained"; Algorithm 1 line 1).
 * The paper uses approximate IVF-PQ; this build computes the
 * EXACT kNN: a tensor-core (tcgen05, fp16 operands, fp32
 * accumulate) distance GEMM selects K' >= K candidates per row by the
 * expanded form |x|^2 + |y|^2 - 2 x.y on column-mean-centred data, then an
 * fp64 re-rank of exact differences sum_d (x_d - y_d)^2 picks the K best.
 * For N >= 2^18 and D >= 1024 the candidate GEMM exploits the symmetry of the
 * distance matrix (each pair of 256-point blocks multiplied once, DESIGN.md
 * 6.6); the result is identical.  The call synchronises `stream` internally
 * (the host orders the locality tour and reads the fallback counts).
 *
 *   X    [N x D] float32, row-major, finite.
 *   idx  [N x K] int32 out: neighbours of row i, self excluded, ascending by
 *        (d2, index) -- ties broken by the lower index (D18).
 *   d2   [N x K] float64 out: exact squared Euclidean distances (D19).
 * Requires N >= 2, 1 <= K < N, D >= 1.
 * Exactness (D26): a row is accepted from its K' candidates only if an
 * a-priori error bound of the fp16 / fp32 candidate distances, valid for
 * EVERY point of the data set (element rounding 2^-11, norm and FFMA
 * rounding 2^-24, fp32 accumulation Dp 2^-22 |x_i||x_j|), proves that no
 * non-candidate can be nearer than the K-th re-ranked neighbour; rows it
 * cannot certify are recomputed by an exact fp64 scan of all N points.
 * `info` (HOST, nullable): when non-NULL the call synchronises `stream` and
 * reports how many rows failed the certificate and were rescanned.
 * ------------------------------------------------------------------------ */
typedef struct {
  int64_t rows_uncertified;  /* rows re-done by the exact fallback scan      */
  int32_t candidates;        /* K' used                                       */
  int32_t gemm_path;         /* 2 = tcgen05 symmetric search, 1 = tcgen05 row
                                sweep (CTA pairs), 0 = no query rows (nq = 0) */
} tsne_knn_info;

size_t tsne_knn_workspace_size(int64_t N, int32_t D, int32_t K);
tsne_status tsne_knn(const float* X, int64_t N, int32_t D, int32_t K,
                     int32_t* idx, double* d2, void* ws, size_t ws_bytes,
                     tsne_knn_info* info, tsne_stream_t stream);

/* The same search for the query rows [q0, q0 + nq) only, against all N
 * points (the multi-GPU sharding of the kNN by query point):
 * idx / d2 are nq x K, row r holding the neighbours of point q0 + r, and
 * are identical to rows q0..q0+nq-1 of tsne_knn's output (the fp16
 * centring/scaling is computed over all N rows on every call).  Workspace:
 * tsne_knn_workspace_size(N, D, K).  nq = 0 is a no-op; a range outside
 * [0, N) is TSNE_ERR_ARG. */
tsne_status tsne_knn_rows(const float* X, int64_t N, int32_t D, int32_t K,
                          int64_t q0, int64_t nq, int32_t* idx, double* d2,
                          void* ws, size_t ws_bytes, tsne_knn_info* info,
                          tsne_stream_t stream);

/* ------------------------------------------------------------------------
 * U2 + U3  Sparse joint affinities P (Eq. 1; symmetrisation
 * p_ij = (p_{i|j} + p_{j|i}) / 2N; at most 2NK nonzeros).
 * Each row's bandwidth is found by fp64 bisection so that the entropy of
 * p_{.|i} (nats) equals ln(perplexity) to 1e-10 (D3: the paper never states
 * the rule); Eq. 1 is normalised over the K neighbours (D2).
 *
 *   idx, d2   the output of tsne_knn (N x K).
 *   row_ptr   [N+1] int64 out; col [cap 2NK] int32 out; val [cap 2NK] float32
 *             out: CSR of P with both triangles, sorted unique columns, no
 *             diagonal; val[(i,j)] == val[(j,i)] bitwise; sum(val) = 1.
 *   nnz_out   HOST out: number of nonzeros (this call synchronises stream).
 *   beta_out  [N] float64 out (nullable): 1/(2 sigma_i^2).
 * Requires 1 < perplexity < K and 2 N K < 2^31 (the directed edges of the
 * symmetrisation are indexed in int32), else TSNE_ERR_ARG.  Returns TSNE_ERR_DEGENERATE (outputs valid)
 * if some row had no finite root -- all neighbours equidistant (uniform over
 * K) or >= perplexity ties at the minimum (uniform over the ties) (D3).
 * ------------------------------------------------------------------------ */
size_t tsne_compute_p_workspace_size(int64_t N, int32_t K);
tsne_status tsne_compute_p(const int32_t* idx, const double* d2, int64_t N, int32_t K,
                           float perplexity, int64_t* row_ptr, int32_t* col, float* val,
                           int64_t* nnz_out, double* beta_out, void* ws, size_t ws_bytes,
                           tsne_stream_t stream);

/* ------------------------------------------------------------------------
 * H1-H7  One Barnes-Hut t-SNE gradient at a fixed embedding
 * (Eq. 7: dC/dy_i = 4 (F_attr + F_rep)):
 *   quadtree over Y (bounding box, Morton sort, node build, counts and
 *   centres of mass; P:L136 steps 1-4), theta traversal giving the
 *   repulsive numerators and Z, CSR attractive pass (Eq. 5 via
 *   the nonzero iteration of P:L115-122).
 *   dY_i = 4 (exaggeration * A_i - f_i / Z),
 *   A_i = sum_j P_ij (y_i - y_j) / (1 + |y_i - y_j|^2)      (D1, D5)
 *   f_i = sum over accepted cells / leaves of N_c w^2 (y_i - y_c),
 *   w = 1/(1 + D^2), Z = sum_i z_i
 * Tree and criterion definitions: D7-D11 (r = half side of a square cell,
 * y_cell = centre of mass, strict r^2 < theta^2 D^2, a cell containing i is
 * always opened; leaves hold one point or are level-24 cells evaluated
 * pairwise, D9), decided as in fp64 (D25).
 *
 *   row_ptr/col/val  CSR of P as produced by tsne_compute_p; col and val
 *             must be 16-byte aligned (they are streamed by bulk copies),
 *             Y 16-byte aligned (a window of it is staged by bulk copies)
 *             and dY 8-byte aligned, else TSNE_ERR_ARG.
 *   Y     [N x 2] float32 (x,y interleaved), finite.
 *   dY    [N x 2] float32 out.
 *   Z_out HOST out (nullable): Z; when non-NULL the call synchronises.
 * Requires 2 <= N < 2^25 (the node index fits 27 bits and the fixed-point
 * centre-of-mass sums fit int64; the same limit holds for every entry point
 * that builds the quadtree), theta >= 0 (theta == 0 is the exact O(N^2) sum,
 * P:L130), exaggeration > 0.
 * ------------------------------------------------------------------------ */
size_t tsne_gradient_workspace_size(int64_t N);
tsne_status tsne_gradient(const int64_t* row_ptr, const int32_t* col, const float* val,
                          int64_t N, const float* Y, float theta, float exaggeration,
                          float* dY, double* Z_out, void* ws, size_t ws_bytes,
                          tsne_stream_t stream);

/* ------------------------------------------------------------------------
 * f4  Cost of an embedding with the EXACT normaliser:
 *   C = KL(P || Q) = sum_{P_ij > 0} P_ij ln(P_ij / q_ij),  q_ij = w_ij / Z,
 *   w_ij = (1 + |y_i - y_j|^2)^-1,  Z = sum_{k != l} w_kl
 * (Eq. 2 and the cost below it; Eq. 4).  Z is the exact
 * O(N^2) sum (each unordered pair once, fp32 pair arithmetic with fp64
 * accumulation in a fixed order: deterministic), not the Barnes-Hut
 * estimate; the cost is then one fp64 pass over the CSR.  P is used as given
 * (pass the non-exaggerated P of tsne_compute_p); zero entries contribute 0.
 *
 *   row_ptr/col/val  CSR of P (as for tsne_gradient; no alignment beyond the
 *             element size is required here).
 *   Y      [N x 2] float32, 8-byte aligned.
 *   kl_out HOST out: C.   Z_out HOST out (nullable): Z.
 * Synchronises `stream`.  Requires 2 <= N < 2^27.
 * ------------------------------------------------------------------------ */
size_t tsne_kl_workspace_size(int64_t N);
tsne_status tsne_kl(const int64_t* row_ptr, const int32_t* col, const float* val, int64_t N,
                    const float* Y, double* kl_out, double* Z_out, void* ws, size_t ws_bytes,
                    tsne_stream_t stream);

/* Schedule / optimiser constants (the paper states none of them: D12-D16). */
typedef struct {
  int32_t K;            /* neighbours; 0 -> min(N-1, floor(3 perplexity)) (D4) */
  int32_t exag_iters;   /* early-exaggeration length (250)                      */
  float mom0, mom1;     /* momentum before / after exag_iters (0.5, 0.8)        */
  float min_gain;       /* gain floor (0.01)                                    */
  uint64_t seed;        /* Philox4x32-10 key for Y0 (42) (D14)                  */
  const float* Y_init;  /* DEVICE [N x 2] initial embedding, NULL -> Philox     */
  int32_t use_graphs;   /* 1: replay the iteration as a CUDA graph (default)    */
  int32_t relabel_every; /* period (iterations) of the internal relabelling of
                           points into the Morton order of the embedding, for
                           gather locality (before iteration 128 the order of a
                           graph diffusion of P is used instead); 0 = never
                           (64).  Results differ only by floating-point
                           summation order.                                     */
  int32_t keep_state;   /* tsne_optimize only (0): 1 = keep the internal state
                           (relabelled P, embedding in internal labels, relabel
                           phase) and the instantiated CUDA graphs in the
                           workspace after the call, so that the next call on
                           the same workspace -- same P pointers, N, theta,
                           learning rate, exaggeration and schedule, t0 = the
                           previous t0 + n_iter -- continues from them instead
                           of re-entering the label space (a re-permutation of
                           P) and re-capturing the graphs.  It resumes only if
                           Y, v, gains still hold exactly what the previous call
                           wrote (checked by a device fingerprint, ~10 us);
                           otherwise it starts afresh.  The caller promises not
                           to modify row_ptr/col/val in between.  A run split
                           into such calls is bitwise identical to one call.
                           Host resources are freed by tsne_optimize_release. */
  int32_t knn_tau;      /* tsne_run_ex only (0): 0 = exact kNN (tsne_knn);
                           > 0 = approximate kNN by IVF-PQ with tau probes and
                           default index parameters (tsne_ivfpq_*, the paper's
                           FAISS path).                             */
} tsne_config;

/* Fills the defaults listed above. */
void tsne_config_default(tsne_config* cfg);

/* ------------------------------------------------------------------------
 * H1-H8  The optimisation loop of Algorithm 1 given P:
 * n_iter iterations t = t0 .. t0+n_iter-1 of
 *   tree build -> traversal (F_rep, Z) -> attractive pass fused with the
 *   update: per coordinate gain <- (sign g != sign v) ? gain + 0.2
 *   : 0.8 gain, gain >= min_gain; v <- mu(t) v - eta gain g; y <- y + v;
 *   then y <- y - mean(y)   (D12-D15).
 *   alpha(t) = exaggeration if t < exag_iters else 1; mu(t) = mom0 / mom1.
 *   Y, v, gains  [N x 2] float32 in/out (the optimiser state).
 * Returns TSNE_ERR_NONFINITE if Y became non-finite (checked at the end of
 * the call; the call synchronises stream for that check, and reads nnz =
 * row_ptr[N] at entry).  The workspace depends on nnz (the library keeps
 * two relabelled copies of P, see tsne_config.relabel_every).
 * ------------------------------------------------------------------------ */
size_t tsne_optimize_workspace_size(int64_t N, int64_t nnz);
tsne_status tsne_optimize(const int64_t* row_ptr, const int32_t* col, const float* val,
                          int64_t N, float* Y, float* v, float* gains, int32_t t0,
                          int32_t n_iter, float theta, float learning_rate,
                          float exaggeration, const tsne_config* cfg, void* ws,
                          size_t ws_bytes, tsne_stream_t stream);

/* Frees the host-side resources (kept-state record, instantiated CUDA graphs)
 * that tsne_optimize with tsne_config.keep_state attached to workspace `ws`.
 * Call it before freeing or reusing the workspace for another problem.  No
 * device work; never fails (an unknown ws is ignored). */
void tsne_optimize_release(void* ws);

/* Diagnostics for measurement (bench.py): from the optimiser state (advancing
 * it exactly like tsne_optimize by 2 * reps iterations from t0) it runs `reps`
 * eager iterations with the stages one after the other, then `reps` normal
 * (overlapped) iterations, and reports mean CUDA-event times on `stream`:
 *   stage_ms[0] tree build (H1-H4), [1] traversal (H5-H6), [2] attractive
 *   sums (H7), [3] update (H8), [4] one overlapped iteration (the attractive
 *   pass runs on a side stream concurrently with [0] and [1]).
 * kernels_per_iter (HOST out, nullable): kernel launches per iteration
 * (counted from a captured graph of one iteration).
 * trav_stats (HOST out, 5 doubles, nullable): counters of one extra traversal
 * of the final embedding, per point: [0] node visits, [1] the sum over warps
 * of the warp's largest visit count / N (SIMT steps), [2] interactions
 * (accepted cells + exact pairs), [3] fp64 re-decisions (D25), [4] bucket pairs.  It overwrites the
 * internal state of the workspace: a later keep_state tsne_optimize call on
 * it starts afresh.
 * stage_ms (HOST out, 5 doubles).  Synchronises stream. */
tsne_status tsne_profile_iterations(const int64_t* row_ptr, const int32_t* col, const float* val,
                                    int64_t N, float* Y, float* v, float* gains, int32_t t0,
                                    int32_t reps, float theta, float learning_rate,
                                    float exaggeration, const tsne_config* cfg, double* stage_ms,
                                    int32_t* kernels_per_iter, double* trav_stats, void* ws,
                                    size_t ws_bytes, tsne_stream_t stream);

/* ------------------------------------------------------------------------
 * Multi-GPU building blocks (the paper is single-GPU).
 * One process per GPU.  Every rank holds the full embedding Y [N x 2] and the
 * CSR rows [row0, row1) of P it owns (row_ptr_local: n_local + 1 offsets into
 * col_local / val_local, 16-byte aligned; columns are global point indices).
 * Per iteration:
 *   1. tsne_shard_forces: quadtree over the whole Y (built redundantly on
 *      every rank; if `recentre`, over Y - mean(Y), D15, the shift being kept
 *      in the workspace) -> the theta traversal for the owned points only:
 *      rep_local[i - row0] = f_i, z_partial[0] = sum over owned i of z_i
 *      (z_partial: 2 doubles, DEVICE).  Y is NOT modified.
 *   1'. tsne_shard_attract (may run concurrently with 1 on another stream:
 *      it only reads Y; Y 16-byte aligned): A_local[i - row0] =
 *      sum_j P_ij (y_i - y_j) q_ij Z.
 *   2. caller: all-gather the ranks' z_partial pairs (NCCL) -> z_partials
 *      [world x 2] DEVICE, in rank order.
 *   3. tsne_shard_update (same workspace as 1): Eq. 7 with Z = sum_r
 *      z_partials[2r] (added in rank order, so every rank uses the identical
 *      Z), D12 update of v_local, gains_local, and Y_local_out [n_local x 2] =
 *      the owned rows of the updated, recentred Y.
 *   4. caller: all-gather Y_local_out shards into Y (NCCL).
 * After the last iteration, tsne_recentre(Y) applies the final recentring.
 * `flag` (DEVICE int, nullable) is set to 1 on a non-finite result.
 * ------------------------------------------------------------------------ */
size_t tsne_shard_workspace_size(int64_t N);
tsne_status tsne_shard_forces(const float* Y, int64_t N, int64_t row0, int64_t row1, float theta,
                              int32_t recentre, float* rep_local, double* z_partial, void* ws,
                              size_t ws_bytes, tsne_stream_t stream);
tsne_status tsne_shard_attract(const int64_t* row_ptr_local, const int32_t* col_local,
                               const float* val_local, int64_t N, int64_t row0, int64_t row1,
                               const float* Y, float* A_local, tsne_stream_t stream);
tsne_status tsne_shard_update(const float* A_local, int64_t N, int64_t row0, int64_t row1,
                              const float* Y, const float* rep_local, const double* z_partials,
                              int32_t world, int32_t t, float learning_rate, float exaggeration,
                              const tsne_config* cfg, float* v_local, float* gains_local,
                              float* Y_local_out, int32_t* flag, void* ws, size_t ws_bytes,
                              tsne_stream_t stream);
tsne_status tsne_recentre(float* Y, int64_t N, void* ws, size_t ws_bytes, tsne_stream_t stream);

/* Y0 = 1e-4 N(0,1) from Philox4x32-10 (key = seed, counter = (i,0,0,0)),
 * Box-Muller on the first two words (D14).  Y [N x 2] float32 out. */
tsne_status tsne_init_y(int64_t N, uint64_t seed, float* Y, tsne_stream_t stream);

/* ------------------------------------------------------------------------
 * Algorithm 1 end to end: kNN -> P -> Y0 -> n_iter iterations.
 * "Input: N x d array of data; Output: N x 2 projection".
 *   X      [N x D] float32, HOST or DEVICE (detected); finite.
 *   Y_out  [N x 2] float32, HOST or DEVICE (detected).
 * The only allocating entry points: device memory for the whole pipeline
 * is allocated with one cudaMalloc (measured: it maps tens of GB in
 * milliseconds where the stream-ordered pool took seconds) and released with
 * cudaFree before return; the work runs on an internal stream.  Blocking.  Exaggeration lasts 250 iterations, momentum
 * 0.5 -> 0.8, Y0 from Philox seed 42 (see tsne_config for _ex).
 * Requires N >= 2, 1 < perplexity < K, theta >= 0, learning_rate > 0,
 * n_iter >= 1, exaggeration >= 1, 2 <= N < 2^25, 2 N K < 2^31.
 * Non-finite X -> TSNE_ERR_ARG.
 * ------------------------------------------------------------------------ */
tsne_status tsne_run(const float* X, int64_t N, int32_t D, float perplexity, float theta,
                     float learning_rate, int32_t n_iter, float exaggeration, float* Y_out);

typedef struct {
  double ms_knn, ms_p, ms_loop, ms_total;  /* CUDA-event stage times          */
  double ms_h2d, ms_d2h;                   /* host<->device copies (if HOST)  */
  int64_t nnz;                             /* nonzeros of P                   */
  int64_t knn_rows_uncertified;
  int32_t K;
  int32_t degenerate_rows;                 /* > 0: TSNE_ERR_DEGENERATE cases  */
} tsne_run_info;

tsne_status tsne_run_ex(const float* X, int64_t N, int32_t D, float perplexity, float theta,
                        float learning_rate, int32_t n_iter, float exaggeration,
                        const tsne_config* cfg, float* Y_out, tsne_run_info* info);

/* ------------------------------------------------------------------------
 * Approximate kNN by IVF-PQ: the paper's own line-1
 * algorithm, FAISS's inverted file with product quantisation (Alg. 1,
 * P:L151; Sec. III-B): |C| = sqrt(N) coarse centroids trained by
 * k-means, residuals r = x - q1(x) product-quantised into m
 * sub-vectors of 256 codewords (8-bit codes), and a search that scans the
 * inverted lists of the tau nearest centroids by the asymmetric distance
 * ||x - q(y)||^2 (look-up tables).  This build re-ranks the K' best
 * candidates of each query (kprime below) by their exact fp64 distance,
 * so d2 holds exact distances of approximately found neighbours (D19).
 * Deterministic training (D27): the training sample is the points
 * floor(k N / ntrain), initial centroids the sample rows floor(c ntrain / k),
 * a fixed number of Lloyd iterations, empty clusters keep their centroid,
 * ties by index; the seed field is reserved.
 *   nlist           0 -> round(sqrt(N))
 *   m               0 -> min(96, ceil(D / 8)); dsub = ceil(D / m) <= 64, the
 *                   vectors zero-padded to Dp = m dsub dimensions
 *   kmeans_iters    Lloyd iterations of both quantisers (10)
 *   train_per_list  ntrain = min(N, nlist * train_per_list) (64)
 *   kprime          candidates re-ranked per query, 0 -> K + max(64, 5K);
 *                   rounded up to 32, at most 480
 * The index is one caller-owned DEVICE buffer of tsne_ivfpq_index_size bytes
 * (256-byte aligned); tsne_ivfpq_layout gives its parts (byte offsets):
 *   out[0..3] nlist, m, dsub, Dp; out[4] centroids fp32 [nlist x Dp];
 *   out[5] codebooks fp32 [m x 256 x dsub]; out[6] codes u8 [N x m] in list
 *   order; out[7] list offsets int32 [nlist + 1]; out[8] list entries
 *   (point ids) int32 [N]; out[9] T tables fp32 [nlist x m x 256]
 *   (T[L][j][k] = |cb_jk|^2 + 2 <c_L,j, cb_jk>); out[10] ntrain.
 * tsne_ivfpq_search: queries = the N indexed points themselves (the kNN graph
 * of t-SNE), self excluded; tau in [1, min(nlist, 64)]; lists are probed in
 * distance order until tau lists are done and at least K' candidates were
 * seen.  idx [N x K] int32 (-1 if fewer than K were found), d2 [N x K] fp64,
 * each row ascending by (d2, idx).  X fp32 [N x D] DEVICE.  Errors: TSNE_ERR_ARG,
 * TSNE_ERR_WORKSPACE, TSNE_ERR_CUDA (also cuBLAS failures).
 * ------------------------------------------------------------------------ */
typedef struct {
  int32_t nlist, m, kmeans_iters, train_per_list, kprime;
  uint64_t seed;
} tsne_ivfpq_params;
void tsne_ivfpq_params_default(tsne_ivfpq_params* p);
size_t tsne_ivfpq_index_size(int64_t N, int32_t D, const tsne_ivfpq_params* p);
tsne_status tsne_ivfpq_layout(int64_t N, int32_t D, const tsne_ivfpq_params* p,
                              int64_t* out /* HOST, 11 */);
size_t tsne_ivfpq_workspace_size(int64_t N, int32_t D, int32_t K, const tsne_ivfpq_params* p);
tsne_status tsne_ivfpq_build(const float* X, int64_t N, int32_t D, const tsne_ivfpq_params* p,
                             void* index, size_t index_bytes, void* ws, size_t ws_bytes,
                             tsne_stream_t stream);
tsne_status tsne_ivfpq_search(const float* X, int64_t N, int32_t D, const tsne_ivfpq_params* p,
                              const void* index, int32_t K, int32_t tau, int32_t* idx,
                              double* d2, void* ws, size_t ws_bytes, tsne_stream_t stream);

/* ------------------------------------------------------------------------
 * Algorithm 1 end to end on `world` GPUs, one process per GPU (
 * the paper is single-GPU; its problem statement P:L147-148).  The
 * library owns the NCCL communicator, built from `nccl_unique_id`
 * (TSNE_NCCL_ID_BYTES bytes, identical on every rank: rank 0 obtains it with
 * tsne_nccl_unique_id and the caller broadcasts it, e.g. over
 * torch.distributed).  NCCL is loaded at run time (libnccl.so.2).
 * Rank r owns rows [r S, min(N, (r+1) S)), S = ceil(N / world):
 *   X_local [N_local x D] float32, HOST or DEVICE: this rank's rows of X;
 *           N_local must equal the size of that range.
 *   Y_out   [N x 2] float32, HOST or DEVICE: written on rank 0 (may be NULL
 *           on the other ranks).
 * Steps: X all-gathered; kNN of the own query rows against all N points
 * (row sweep + fp64 re-rank, bit-identical to tsne_knn rows); the kNN lists
 * all-gathered; P built on every rank; the points relabelled by the diffusion
 * locality order of P (identical on every rank), after which rank r iterates
 * on the contiguous label range [r S, (r+1) S) (its rows' neighbours then
 * fall in the attractive pass's window); per iteration the attractive sums and
 * the traversal of the own points, an all-gather of the Z partials (added in
 * rank order: every rank uses the identical Z), the update of the own rows,
 * an all-gather of the Y shards (CUDA graphs, one per schedule phase).
 * Allocates tsne_run_workspace_size(N, D, K, world) bytes of device memory on
 * the current device (one cudaMalloc, freed before return); blocking; every
 * rank must call it with the same arguments except X_local / N_local / rank.
 * info (HOST, nullable): stage times of this rank (ms_h2d = own rows H2D +
 * all-gather of X; ms_knn = own kNN rows + all-gather of the lists).
 * Errors: TSNE_ERR_ARG as tsne_run_ex (+ rank/world/N_local checks),
 * TSNE_ERR_NCCL for a failed communicator or collective (the communicator is
 * aborted), TSNE_ERR_NONFINITE, TSNE_ERR_CUDA.
 * ------------------------------------------------------------------------ */
#define TSNE_NCCL_ID_BYTES 128
tsne_status tsne_nccl_unique_id(void* id_out /* HOST, TSNE_NCCL_ID_BYTES */);
size_t tsne_run_workspace_size(int64_t N, int32_t D, int32_t K, int32_t world);
tsne_status tsne_run_sharded(const float* X_local, int64_t N_local, int64_t N, int32_t D,
                             float perplexity, float theta, float learning_rate, int32_t n_iter,
                             float exaggeration, const tsne_config* cfg,
                             const void* nccl_unique_id, int32_t rank, int32_t world,
                             float* Y_out, tsne_run_info* info);

#ifdef __cplusplus
}
#endif
#endif /* TSNE_B200_H */
