// tree.cuh -- the quadtree of Sec. III-C as built on the GPU:
// bounding box (step 1), Morton keys + radix sort (step 4, "sort points by
// spatial distance"), compressed quadtree from the sorted keys (steps 2-3:
// "insert", "number of points in each internal cell"), centres of mass.
//
// Node layout: one pre-order array of 16-byte hot
// records {com_x, com_y, (float) count, skip | level << 27}; the first child of
// node k is k + 1 and `skip` is the first node after k's subtree, so a
// traversal needs no stack.  Cold arrays: range start (`nfirst`, used by
// bucket leaves) and the fp64 centre of mass (`com64`, read only inside the
// fp64 decision band, D25).
//
// level field: 0..23  internal cell whose point set branches at that level
//                     (single-child chains are compressed away, D9)
//              24     leaf of one point (the exact pair)
//              25     bucket whose chain reaches level <= 23: the criterion
//                     is tested with r_23; accept -> summary, else exact pairs
//              26     bucket directly below a level-23 branching cell: exact pairs
#pragma once
#include "common.cuh"

namespace tsne {

struct BoxInfo {
  float minx, maxx, miny, maxy;  // bounding box of the (shifted) embedding
  float shift_x, shift_y;        // fp32 mean subtracted from Y before use (recentring, D15)
  float mabs;                    // max |coordinate| (shifted), bounds fp32 error (D25)
  float pad0;
  double cx, cy, r0, lox, loy, s;  // root box (D8), fp64
};

constexpr int kLevels = 24;                   // quadtree depth (D9): 2^24 cells per axis
constexpr int kKeyBits = 2 * kLevels;          // Morton key bits (48, in a 64-bit word)
constexpr int kLevelLeaf = kLevels;            // 24
constexpr int kLevelBucketTest = kLevels + 1;  // 25 (level field is 5 bits)
constexpr int kLevelBucket = kLevels + 2;      // 26: several points in a level-24 cell below a
                                               // level-23 branching cell: always exact pairs
constexpr int kLevelCodes = kLevels + 3;       // level codes 0..26
static_assert(kLevelBucket < 32, "level field");
constexpr uint32_t kSkipMask = (1u << 27) - 1u;
constexpr int kMaxParts = 4096;
constexpr int kScanTile = 4096;               // k_scan_cnt tile (16 per thread)
constexpr int kSortThreads = 256;
constexpr double kFixScale = 274877906944.0;  // 2^38: fixed-point COM sums
static_assert(2 * kMaxTreePoints < (int64_t)kSkipMask + 1, "node index must fit the skip field");
static_assert(kMaxTreePoints < (int64_t(1) << (63 - 38)), "count * 2^38 must fit int64");

struct TreeWS {
  int64_t N = 0;
  uint64_t *keys_a = nullptr, *keys_b = nullptr;
  int32_t *vals_a = nullptr, *vals_b = nullptr;
  void* sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  float2* ys = nullptr;        // Y in Morton order
  longlong2* fq = nullptr;     // fixed-point coordinates (N+1)
  longlong2* S = nullptr;      // exclusive prefix sums of fq (N+1)
  longlong2* bsum = nullptr;   // per 256-point block sums of fq, then their exclusive scan
  uint8_t* dl = nullptr;       // split deltas: common-prefix length of sorted positions i, i+1
  unsigned long long* slot = nullptr;  // per split: epoch << 32 | the first arrival's range end
  int4* nfo = nullptr;         // per split: (first, last, chain count or -1, parent delta)
  int32_t* cnt = nullptr;      // N+1: quad nodes starting at each sorted position
  int32_t* base = nullptr;     // N+1: exclusive scan of cnt (base[N] = node count)
  int32_t* tsum = nullptr;     // per kScanTile tile of cnt: its sum
  uint32_t* ctl = nullptr;     // [0] build epoch
  float4* nodes = nullptr;     // <= 2N-1 quad nodes
  int32_t* nfirst = nullptr;
  double2* com64 = nullptr;
  int32_t* leafnode = nullptr; // N, indexed by sorted position
  int32_t* has_bucket = nullptr; // 1 if the last tree has a bucket (several points in a leaf)
  BoxInfo* box = nullptr;
  float2* rep = nullptr;       // N repulsive numerators f_i (original order)
  double* zpart = nullptr;     // per traversal block
  int2* ovf = nullptr;         // per traversal thread: deferred buckets beyond the registers
  int2* lg = nullptr;          // per traversal thread: large deferred buckets (k_defer_large)
  int2* dlist = nullptr;       // traversal threads with large deferred buckets
  unsigned long long* zacc = nullptr;  // their z terms: [0] integer part, [1] 2^-32 units
  double* Z = nullptr;         // [0] = Z, [1] = 1/Z
  unsigned* counter = nullptr; // last-block-done counters (zeroed once); [4] k_defer_large
                               // done, [5] its list length
  float4* part4 = nullptr;     // per-block min/max partials (kMaxParts)
  double2* part2 = nullptr;    // per-block fp64 sum partials (kMaxParts)
  // set by build(): which double-buffer half holds the sorted result
  uint64_t* keys_sorted = nullptr;
  int32_t* perm = nullptr;
};

// Carve (or size) the tree workspace for N points.
void carve_tree(Carver& c, TreeWS& w, int64_t N);
// Zeroes the last-block-done counters of a freshly carved tree workspace.
tsne_status tree_ws_init(TreeWS& w, cudaStream_t s);
size_t tree_cub_bytes(int64_t N);

// Bounding box + root box of Y (shift = 0), written to w.box.
tsne_status launch_bbox(TreeWS& w, const float2* Y, cudaStream_t s);
// Steps 2-4 from w.box: keys (of Y - box->shift when `apply_shift`; Y itself
// is not modified), sort, build, summarise.
tsne_status build_tree(TreeWS& w, const float2* Y, bool apply_shift, cudaStream_t s);
// Repulsive pass: w.rep, w.Z
tsne_status launch_traverse(TreeWS& w, float theta, cudaStream_t s);
// measurement: per-point visit / interaction counters of one traversal (synchronises s)
tsne_status traverse_stats(TreeWS& w, float theta, double* out5, cudaStream_t s);
tsne_status launch_traverse_list(TreeWS& w, float theta, const int32_t* list, const int32_t* nlist,
                                 int row0, float2* rep_local, double* z_partial, cudaStream_t s);
// Bounding box + recentring shift (fp64 mean, fixed order) of Y, into w.box.
tsne_status launch_bbox_mean(TreeWS& w, const float2* Y, cudaStream_t s);

int traverse_blocks(int64_t N);

__host__ __device__ inline void make_root_box(float minx, float maxx, float miny, float maxy,
                                              BoxInfo* b);

}  // namespace tsne

// ---- implementation of the root box (identical arithmetic to DESIGN D8) ----
namespace tsne {
__host__ __device__ inline double dadd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
__host__ __device__ inline double dsub(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
__host__ __device__ inline double dmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
__host__ __device__ inline double ddiv(double a, double b) {
#ifdef __CUDA_ARCH__
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}

__host__ __device__ inline void make_root_box(float minx, float maxx, float miny, float maxy,
                                              BoxInfo* b) {
  b->minx = minx; b->maxx = maxx; b->miny = miny; b->maxy = maxy;
  double cx = ddiv(dadd((double)minx, (double)maxx), 2.0);
  double cy = ddiv(dadd((double)miny, (double)maxy), 2.0);
  double sx = dsub((double)maxx, (double)minx);
  double sy = dsub((double)maxy, (double)miny);
  double span = sx > sy ? sx : sy;
  double r0 = (span == 0.0) ? 1.0 : dmul(ddiv(span, 2.0), 1.0 + 9.5367431640625e-07 /*2^-20*/);
  b->cx = cx; b->cy = cy; b->r0 = r0;
  b->lox = dsub(cx, r0);
  b->loy = dsub(cy, r0);
  b->s = ddiv(16777216.0 /* 2^kLevels */, dmul(2.0, r0));
  float m = fmaxf(fmaxf(fabsf(minx), fabsf(maxx)), fmaxf(fabsf(miny), fabsf(maxy)));
  b->mabs = m;
}
}  // namespace tsne
