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
#include "tc_ptx.cuh"

namespace tsne {

constexpr int kAttrThreads = 256;
constexpr int kAttrWarps = kAttrThreads / 32;

// ---------------------------------------------------------------- H7
// Attractive pass as a persistent TMA pipeline (one CTA per SM).
// * CTA b owns the rows [f(b), f(b+1)), f(b) the first row starting at or
//   after nonzero nnz*b/G, so every CTA streams the same number of nonzeros
//   whatever the row-length distribution.
// * The rows are cut into ITEMS: consecutive pieces of kAtItem nonzeros counted
//   from the row's start (a row of n nonzeros is ceil(n / kAtItem) items, an
//   empty row one empty item).  Up to kAtItems whole items whose nonzeros fit
//   a stage buffer form a BATCH -- a batch may end inside a row, never inside
//   an item.  The batches depend only on row_ptr and the grid: the optimiser
//   and the shards cut them once per CSR (k_attract_plan, at every relabel);
//   the one-shot entry points cut them inside the kernel (same cut).
// * A producer warp streams each batch's col/val span (contiguous in the CSR)
//   and its item list into a kAtStages-deep shared-memory ring with
//   cp.async.bulk + mbarriers; the embedding window Y[wlo, wlo + kAtWin)
//   around the CTA's rows is staged once the same way.
// * Consumer warps (kAtGroups groups taking alternate batches) take the items
//   of a batch one at a time from a shared counter -- dynamic, so a long row
//   (a hub of the kNN graph: thousands of nonzeros) is spread over many warps
//   and a warp that finished early takes more of the next batch.  Lanes take
//   consecutive nonzeros of the item from shared memory, gather y_j from the
//   window (columns outside it, rare once the labels are in a locality order
//   -- come from L2 through a predicated load), and the
//   warp reduces the item with a fixed butterfly into a per-item partial.
// * A finaliser warp adds each row's partials in item order (a row continued
//   from the previous batch starts from the carried sum) and writes the rows
//   that ended.  The item cut depends only on the row, so every row is summed
//   in the same order whatever the grid, the batch cuts or the CSR around it
//   (deterministic; a shard's local CSR gives the single-GPU rows bit for bit).
#ifndef TSNE_AT_GROUPS
#define TSNE_AT_GROUPS 2
#endif
#ifndef TSNE_AT_WARPS
#define TSNE_AT_WARPS 30
#endif
#ifndef TSNE_AT_STAGES
#define TSNE_AT_STAGES 4
#endif
#ifndef TSNE_AT_CAP
#define TSNE_AT_CAP 4096
#endif
constexpr int kAtGroups = TSNE_AT_GROUPS;      // consumer groups take alternate batches
constexpr int kAtConsumers = TSNE_AT_WARPS;    // consumer warps
constexpr int kAtRows = kAtConsumers / kAtGroups;   // consumer warps per group
constexpr int kAtThreads = (kAtConsumers + 2) * 32;   // + the producer and the finaliser warp
constexpr int kAtStages = TSNE_AT_STAGES;
constexpr int kAtMetas = 2 * kAtStages;        // batch metadata slots (outlive their stage)
constexpr int kAtCap = TSNE_AT_CAP;            // nonzeros per stage buffer
constexpr int kAtBudget = kAtCap - 8;          // a batch's nonzeros (the 16-byte aligned span fits)
constexpr int kAtItem = kAtItemNz;             // nonzeros per item (optimize.cuh)
constexpr int kAtEmax = kAtItem / 32;          // 32-entry groups of an item, loaded together
constexpr int kAtItems = 32;                   // items per batch (one per producer lane)
constexpr int kAtChunk = 56;                   // rows per row_ptr prefetch chunk
constexpr int kAtLook = 3;                     // row_ptr prefetch distance (chunks)
constexpr int kAtRpSlots = kAtLook + 1;
constexpr int kAtHdrRing = 64;                 // prefetched batch headers (plan mode)
static_assert(kAtConsumers % kAtGroups == 0, "equal consumer groups");
static_assert(kAtStages % kAtGroups == 0, "a stage always serves the same consumer group");
static_assert(kAtItem % 32 == 0 && kAtEmax >= 1 && kAtEmax <= 8, "an item is 1-8 warp-wide groups");
static_assert(kAtBudget / kAtItem >= 1, "a stage holds at least one item");
static_assert(kAtCap < (1 << 13) && kAtItem < (1 << 9), "item descriptor fields");
static_assert(kAtChunk >= kAtItems + 2, "a batch's rows lie in two row_ptr chunks");

struct AtBatchHdr {
  int64_t a_lo;              // first staged nonzero (a multiple of 4)
  int32_t cnt;               // nonzeros bulk-copied from a_lo (a multiple of 4)
  int16_t n_items;           // -1: end marker
  int16_t n_tail;            // the CSR's last (< 4) nonzeros, copied after them by plain loads
};
struct AtBatch {             // one batch of the plan; copied whole into a metadata slot
  AtBatchHdr h;
  int2 item[kAtItems];       // {local row, beg | len << 13 | last << 22} (beg: offset from a_lo)
};
static_assert(sizeof(AtBatchHdr) == 16 && sizeof(AtBatch) % 16 == 0, "bulk-copy granules");
struct AtMeta {
  AtBatch b;
  float2 part[kAtItems];     // per-item partial sums (consumers -> finaliser)
  int32_t next;              // next item to take (shared counter)
  int32_t pad[3];
};
struct AtShared {            // the kernel's static shared memory
  AtMeta meta[kAtMetas];
  union {
    int64_t rpring[kAtRpSlots][kAtChunk + 1];  // row_ptr ring (batches cut in the kernel)
    AtBatchHdr hring[kAtHdrRing];              // header ring (plan mode)
  };
  uint64_t full[kAtStages], empty[kAtStages], done[kAtMetas], mfree[kAtMetas], win;
  int32_t lr0, lr1, wlo, wn;
};
// the window takes what the 227 KB per-CTA limit leaves
#ifndef TSNE_AT_SMEM_LIMIT
#define TSNE_AT_SMEM_LIMIT 232448
#endif
constexpr int kAtSmemLimit = TSNE_AT_SMEM_LIMIT;
constexpr int kAtWin =
    (int)(((kAtSmemLimit - (int)sizeof(AtShared) - 64 - kAtStages * kAtCap * 8) / 8) & ~63);
static_assert(kAtWin >= 4096, "window");
constexpr size_t kAtSmem = sizeof(float2) * kAtWin + (size_t)kAtStages * kAtCap * 8;

__device__ __forceinline__ float rcp_approx_f(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// y_j from the window when j is inside it, else from L2 (branch-free: the
// shared load is clamped into the window, the predicated global load
// overwrites it for columns outside)
__device__ __forceinline__ float2 win_y(uint32_t sbase, const float2* __restrict__ Y, int j,
                                        int wlo, int wn) {
  const unsigned o = (unsigned)(j - wlo);
  const unsigned oc = min(o, (unsigned)(wn - 1));
  float2 v;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(sbase + oc * 8u));
  asm("{\n\t.reg .pred p;\n\tsetp.ge.u32 p, %2, %3;\n\t@p ld.global.nc.v2.f32 {%0, %1}, [%4];\n\t}"
      : "+f"(v.x), "+f"(v.y)
      : "r"(o), "r"((unsigned)wn), "l"(Y + j));
  return v;
}

// (a, b) summed over the warp with 6 shuffles instead of 10: the first step
// exchanges a against b between the half-warps, so each half then reduces one
// value; fixed order, lane 0 ends with both sums (deterministic)
__device__ __forceinline__ void warp_sum2(float& a, float& b) {
  const unsigned lane = threadIdx.x & 31u;
  const bool hi = lane >= 16u;
  const float send = hi ? a : b;
  const float recv = __shfl_xor_sync(0xffffffffu, send, 16);
  float v = hi ? b + recv : a + recv;          // lanes < 16: a-sums, lanes >= 16: b-sums
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const float vb = __shfl_sync(0xffffffffu, v, 16);
  a = v;
  b = vb;
}

// (a, b, c, d) summed over the warp with 6 shuffles: the first step exchanges
// (c, d) against (a, b) between the half-warps, the second splits each half
// between its two values, then three steps reduce one value per 8 lanes.
// Fixed order (deterministic); lane 0 / 8 / 16 / 24 end with the a / b / c / d sum.
__device__ __forceinline__ float warp_sum4(float a, float b, float c, float d) {
  const unsigned lane = threadIdx.x & 31u;
  const bool hi = lane >= 16u;
  const float s1 = hi ? a : c, s2 = hi ? b : d;
  const float r1 = __shfl_xor_sync(0xffffffffu, s1, 16);
  const float r2 = __shfl_xor_sync(0xffffffffu, s2, 16);
  float x = hi ? c + r1 : a + r1;             // lanes < 16: a, b;  lanes >= 16: c, d
  float y = hi ? d + r2 : b + r2;
  const bool q = (lane & 8u) != 0u;
  const float r3 = __shfl_xor_sync(0xffffffffu, q ? x : y, 8);
  float v = q ? y + r3 : x + r3;              // lane bit 3 clear: x (a or c), set: y (b or d)
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void win_accum(float2 yi, float2 yj, float p, float& ax, float& ay) {
  const float dx = yi.x - yj.x, dy = yi.y - yj.y;
  const float w = rcp_approx_f(fmaf(dy, dy, fmaf(dx, dx, 1.f)));   // 1/(1+d^2), d^2 >= 0
  const float pw = p * w;
  ax = fmaf(pw, dx, ax);
  ay = fmaf(pw, dy, ay);
}

// E x 32 consecutive entries of a staged item (n_rem entries from cr): lane
// takes entries lane + 32u; only the last group can be partial (its absent
// entries are the point itself with p = 0).  All loads first, then the
// arithmetic: the window / L2 gathers of the item are in flight together.
template <int E>
__device__ __forceinline__ void row_block(uint32_t scr, uint32_t svr, int n_rem, int self,
                                          float2 yi, uint32_t sbase, const float2* __restrict__ Y,
                                          int wlo, int wn, int lane, float& ax, float& ay) {
  // scr / svr: shared addresses of the item's columns and values
  int c[E];
  float p[E];
#pragma unroll
  for (int u = 0; u < E; ++u) {
    const int q = lane + 32 * u;
    if (u < E - 1 || q < n_rem) {
      asm("ld.shared.b32 %0, [%1];" : "=r"(c[u]) : "r"(scr + 4u * q));
      asm("ld.shared.f32 %0, [%1];" : "=f"(p[u]) : "r"(svr + 4u * q));
    } else {
      c[u] = self;
      p[u] = 0.f;
    }
  }
  // a round whose columns all fall inside the window (the usual case once the
  // labels are in a locality order) gathers from shared memory only
  unsigned o[E];
  bool in = true;
#pragma unroll
  for (int u = 0; u < E; ++u) {
    o[u] = (unsigned)(c[u] - wlo);
    in = in && o[u] < (unsigned)wn;
  }
  float2 y[E];
  if (__all_sync(0xffffffffu, in)) {
#pragma unroll
    for (int u = 0; u < E; ++u)
      asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(y[u].x), "=f"(y[u].y) : "r"(sbase + o[u] * 8u));
  } else {
#pragma unroll
    for (int u = 0; u < E; ++u) y[u] = win_y(sbase, Y, c[u], wlo, wn);
  }
#pragma unroll
  for (int u = 0; u < E; ++u) win_accum(yi, y[u], p[u], ax, ay);
}

// spin wait (the consumers' waits are short)
__device__ __forceinline__ void mbar_wait_spin(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

// wait with a suspend-time hint: the thread sleeps until the phase completes
// (or the hint expires) instead of re-issuing try_wait -- for the producer,
// whose spinning on a full ring took a third of the SM's issue slots (ncu)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity), "r"(1000000u)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// First rows r in [0, n] with rp[r] >= T0 and with rp[r] >= T1 (rp[n] >= T0,
// T1), searched by the warp together: each round 32 lanes sample the
// remaining interval of each search, so a search over N rows takes
// ~log32(N) dependent loads.
__device__ __forceinline__ void lower_bound2_warp(const int64_t* __restrict__ rp, int n, int64_t T0,
                                                  int64_t T1, int lane, int& r0, int& r1) {
  int lo[2] = {0, 0}, hi[2] = {n, n};          // each answer lies in [lo, hi]
  const int64_t T[2] = {T0, T1};
  while (lo[0] < hi[0] || lo[1] < hi[1]) {
    int st[2];
    bool g[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      st[h] = (hi[h] - lo[h] + 31) >> 5;
      const int p = lo[h] + lane * st[h];
      g[h] = lo[h] < hi[h] ? (p >= hi[h] || rp[p] >= T[h]) : true;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const unsigned b = __ballot_sync(0xffffffffu, g[h]);
      if (lo[h] < hi[h]) {
        if (b == 0u) {
          lo[h] += 31 * st[h] + 1;
        } else {
          const int f = __ffs(b) - 1;
          if (f == 0) {
            hi[h] = lo[h];
          } else {
            hi[h] = min(hi[h], lo[h] + f * st[h]);
            lo[h] += (f - 1) * st[h] + 1;
          }
        }
      }
    }
  }
  r0 = lo[0];
  r1 = lo[1];
}

// The CTA's row range [lr0, lr1) of a grid of G CTAs over n_rows rows.
__device__ __forceinline__ void at_range(const int64_t* __restrict__ row_ptr, int n_rows, int b,
                                         int G, int lane, int& lr0, int& lr1) {
  const int64_t nnz = row_ptr[n_rows];
  lower_bound2_warp(row_ptr, n_rows, nnz * b / G, nnz * (b + 1) / G, lane, lr0, lr1);
  if (b == 0) lr0 = 0;
  if (b + 1 == G) lr1 = n_rows;
}

// row_ptr of rows [lr0, lr1] through a ring of kAtChunk-row chunks in shared
// memory, fetched kAtLook chunks ahead with cp.async (one warp)
struct RpRing {
  int64_t (*ring)[kAtChunk + 1];
  const int64_t* row_ptr;
  int lr0, lr1, nch, fetched;
  __device__ __forceinline__ void fetch(int c, int lane) {
    if (c < nch)
      for (int q = lane; q <= kAtChunk; q += 32) {
        const int r = min(lr0 + c * kAtChunk + q, lr1);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                         smem_u32(&ring[c % kAtRpSlots][q])),
                     "l"(row_ptr + r)
                     : "memory");
      }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  __device__ __forceinline__ void start(int lane) {
    nch = (lr1 - lr0 + kAtChunk - 1) / kAtChunk;
    for (int j = 0; j < kAtLook; ++j) fetch(j, lane);
    fetched = kAtLook;
  }
  // rows r .. r + 32 readable (chunks <= chunk(r) + 1 have landed)
  __device__ __forceinline__ void ready(int r, int lane) {
    const int c = (r - lr0) / kAtChunk;
    while (fetched <= c + kAtLook) fetch(fetched++, lane);
    asm volatile("cp.async.wait_group %0;" ::"n"(kAtLook - 1) : "memory");
    __syncwarp();
  }
  // (a chunk's slot holds kAtChunk + 1 entries; the end of the range at a
  // chunk boundary is the last entry of the previous chunk)
  __device__ __forceinline__ int64_t operator()(int r) const {
    const int o = r - lr0, c = o / kAtChunk, q = o - c * kAtChunk;
    if (c == nch) return ring[(c - 1) % kAtRpSlots][kAtChunk];
    return ring[c % kAtRpSlots][q];
  }
};

// Cuts the next batch at (r, e) -- e the next nonzero of row r, an item
// boundary -- (one warp): whole rows while they fit (items and nonzeros), then
// whole items of the row that does not.  Writes the item descriptors and
// returns the header; advances (r, e).
__device__ __forceinline__ AtBatchHdr pack_batch(const RpRing& rp, int lane, int lr1, int64_t nnz4,
                                                 int& r, int64_t& e, int2* __restrict__ items) {
  const int rj = r + lane;                      // lane j looks at row r + j
  const bool in = rj < lr1;
  int64_t sj = 0, tj = 0;                       // its nonzeros [sj, tj)
  int itj = 0;                                  // and items
  if (in) {
    sj = lane == 0 ? e : rp(rj);
    tj = rp(rj + 1);
    itj = max(1, (int)((tj - sj + kAtItem - 1) / kAtItem));
  }
  int I = itj;                                  // inclusive prefix of the item counts
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, I, o);
    if (lane >= o) I += v;
  }
  const bool fits = in && I <= kAtItems && tj - e <= kAtBudget;   // a prefix of the lanes
  const int f = __popc(__ballot_sync(0xffffffffu, fits));
  const int i_before = f > 0 ? __shfl_sync(0xffffffffu, I, f - 1) : 0;
  const int64_t t_before = f > 0 ? __shfl_sync(0xffffffffu, tj, f - 1) : e;
  int q = 0;                                    // whole items of row r + f
  int64_t sf = 0;
  if (f < 32) {
    sf = __shfl_sync(0xffffffffu, sj, f);
    if (r + f < lr1)
      q = (int)min((int64_t)(kAtItems - i_before), (kAtBudget - (sf - e)) / kAtItem);
  }
  const int64_t e_hi = q > 0 ? sf + (int64_t)q * kAtItem : t_before;
  const int64_t a_lo = e & ~int64_t(3);
  const int64_t a_hi = min((e_hi + 3) & ~int64_t(3), nnz4);
  if (lane < f)
    for (int u = 0; u < itj; ++u) {
      const int64_t b = sj + (int64_t)u * kAtItem;
      const int len = (int)min((int64_t)kAtItem, tj - b);
      items[I - itj + u] = make_int2(rj, (int)(b - a_lo) | (len << 13) | ((u == itj - 1) << 22));
    }
  if (lane < q)                                 // never the row's last item
    items[i_before + lane] =
        make_int2(r + f, (int)(sf + (int64_t)lane * kAtItem - a_lo) | (kAtItem << 13));
  AtBatchHdr h;
  h.a_lo = a_lo;
  h.cnt = a_hi > a_lo ? (int32_t)(a_hi - a_lo) : 0;
  h.n_items = (int16_t)(i_before + q);
  h.n_tail = (int16_t)max((int64_t)0, e_hi - max(nnz4, a_lo));
  r += f;
  e = e_hi;
  return h;
}

// Batches of CTA b are stored from plan_off(lr0(b), row_ptr[lr0(b)], b).  Every
// batch but a CTA's last holds kAtItems items or more than kAtBudget - kAtItem
// nonzeros, and a range holds at most nnz/kAtItem + rows items, so the regions
// [plan_off(b), plan_off(b + 1)) never overflow.
__host__ __device__ __forceinline__ int64_t plan_off(int64_t lr, int64_t E, int64_t b) {
  return lr / kAtItems + E / (kAtBudget - kAtItem) + E / ((int64_t)kAtItem * kAtItems) + 5 * b;
}

// One warp per pipeline CTA: its row range and its batches (the same cut as
// the in-kernel packing).  cta[b] = {lr0, lr1, first batch, batches}.
__global__ void __launch_bounds__(32) k_attract_plan(const int64_t* __restrict__ row_ptr,
                                                      int n_rows, AtBatch* __restrict__ batches,
                                                      int4* __restrict__ cta) {
  __shared__ __align__(16) int64_t ring[kAtRpSlots][kAtChunk + 1];
  const int lane = threadIdx.x, b = blockIdx.x, G = gridDim.x;
  int lr0, lr1;
  at_range(row_ptr, n_rows, b, G, lane, lr0, lr1);
  const int64_t nnz4 = row_ptr[n_rows] & ~int64_t(3);
  const int64_t e0 = row_ptr[lr0];
  const int64_t off0 = plan_off(lr0, e0, b), off1 = plan_off(lr1, row_ptr[lr1], b + 1);
  RpRing rp{ring, row_ptr, lr0, lr1, 0, 0};
  rp.start(lane);
  int r = lr0, k = 0;
  int64_t e = e0;
  while (r < lr1) {
    rp.ready(r, lane);
    if (off0 + k >= off1) __trap();             // cannot happen (plan_off's bound)
    AtBatch& B = batches[off0 + k];
    const AtBatchHdr h = pack_batch(rp, lane, lr1, nnz4, r, e, B.item);
    if (lane == 0) B.h = h;
    ++k;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (lane == 0) cta[b] = make_int4(lr0, lr1, (int)off0, k);
}

template <int MODE>
__device__ __forceinline__ void at_write(float2* __restrict__ out, const float2* __restrict__ rep,
                                         const double* __restrict__ Z, float alpha, int l,
                                         float2 a) {
  if (MODE == 0) {
    out[l] = a;
  } else {
    const float invZ = (float)Z[1];
    const float2 f = rep[l];
    out[l] = make_float2(4.f * (alpha * a.x - f.x * invZ), 4.f * (alpha * a.y - f.y * invZ));
  }
}

// MODE 0: out[l] = A_l.  MODE 1 (tsne_gradient): out[l] = 4 (alpha A_l - f_l / Z).
// Rows l in [0, n_rows) of the (local) CSR are global points row0 + l of Y.
// PLAN: the batches come from k_attract_plan (batches, cta), else the producer
// cuts them.
template <int MODE, bool PLAN>
__global__ void __launch_bounds__(kAtThreads, 1)
k_attract_tma(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
              const float* __restrict__ val, const float2* __restrict__ Y, int Ny, int row0,
              int n_rows, const AtBatch* __restrict__ batches, const int4* __restrict__ cta,
              float2* __restrict__ out, const float2* __restrict__ rep,
              const double* __restrict__ Z, float alpha) {
  extern __shared__ __align__(128) unsigned char at_smem[];
  __shared__ __align__(16) AtShared sh;
  float2* s_y = reinterpret_cast<float2*>(at_smem);
  int32_t* s_col = reinterpret_cast<int32_t*>(at_smem + sizeof(float2) * kAtWin);
  float* s_val = reinterpret_cast<float*>(s_col + kAtStages * kAtCap);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t sbase = smem_u32(s_y);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kAtStages; ++s) {
      mbar_init(&sh.full[s], 1);
      mbar_init(&sh.empty[s], kAtRows);
    }
    for (int s = 0; s < kAtMetas; ++s) {
      mbar_init(&sh.done[s], kAtRows);
      mbar_init(&sh.mfree[s], 1);
    }
    mbar_init(&sh.win, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (wid == kAtConsumers + 1) {
    // ----------------------------------------------------------- finaliser
    // Batch kk is done: add each row's partials in item order (a row continued
    // from the previous batch starts from the carried sum), write the rows
    // that ended, free the batch's metadata slot.
    float2 carry = make_float2(0.f, 0.f);
    for (int kk = 0;; ++kk) {
      const int ms = kk % kAtMetas;
      mbar_wait_sleep(&sh.done[ms], (kk / kAtMetas) & 1);
      const AtMeta& m = sh.meta[ms];
      const int ni = m.b.h.n_items;
      if (ni < 0) break;                        // the first end marker: every batch is done
      int row = -1;
      bool head = false;
      if (lane < ni) {
        row = m.b.item[lane].x;
        head = lane == 0 || m.b.item[lane - 1].x != row;
      }
      float2 acc = make_float2(0.f, 0.f);
      bool open = false;                        // the row continues in the next batch
      if (head) {
        if (lane == 0) acc = carry;
        for (int t = lane;; ++t) {
          const float2 p = m.part[t];
          acc.x += p.x;
          acc.y += p.y;
          if ((m.b.item[t].y >> 22) & 1) {
            at_write<MODE>(out, rep, Z, alpha, row, acc);
            break;
          }
          if (t == ni - 1) {
            open = true;
            break;
          }
        }
      }
      const unsigned ob = __ballot_sync(0xffffffffu, open);
      carry = make_float2(0.f, 0.f);
      if (ob) {
        const int src = __ffs(ob) - 1;
        carry.x = __shfl_sync(0xffffffffu, acc.x, src);
        carry.y = __shfl_sync(0xffffffffu, acc.y, src);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.mfree[ms]);
    }
    return;
  }

  if (wid == kAtConsumers) {
    // ------------------------------------------------------------ producer
    const int64_t nnz4 = row_ptr[n_rows] & ~int64_t(3);
    int lr0, lr1, b0 = 0, nb = 0;               // this CTA's rows: an equal share of the nonzeros
    if (PLAN) {
      const int4 ci = cta[blockIdx.x];
      lr0 = ci.x;
      lr1 = ci.y;
      b0 = ci.z;
      nb = ci.w;
    } else {
      at_range(row_ptr, n_rows, blockIdx.x, gridDim.x, lane, lr0, lr1);
    }
    int wlo = row0 + (lr0 + lr1) / 2 - kAtWin / 2;
    wlo = min(wlo, Ny - kAtWin);
    wlo = max(wlo, 0) & ~15;                     // 16-point aligned: entry j in bank pair j mod 16
    const int wn = min(kAtWin, Ny - wlo) & ~1;   // 16-byte multiple
    if (lane == 0) {
      sh.lr0 = lr0;
      sh.lr1 = lr1;
      sh.wlo = wlo;
      sh.wn = wn;
      mbar_arrive_tx(&sh.win, (uint32_t)(wn * sizeof(float2)));   // releases lr0 .. wn
      bulk_g2s(sbase, Y + wlo, (uint32_t)(wn * sizeof(float2)), &sh.win);
    }
    int k = 0;                                  // batch sequence number
    // batch k takes stage k % kAtStages once its consumers are done with batch
    // k - kAtStages, and metadata slot k % kAtMetas once the finaliser is done
    // with batch k - kAtMetas
    auto take_slot = [&]() -> AtMeta& {
      if (k >= kAtStages) mbar_wait_sleep(&sh.empty[k % kAtStages], ((k / kAtStages) - 1) & 1);
      if (k >= kAtMetas) mbar_wait_sleep(&sh.mfree[k % kAtMetas], ((k / kAtMetas) - 1) & 1);
      return sh.meta[k % kAtMetas];
    };
    // the stage's col/val: a bulk copy of [a_lo, a_lo + cnt) and the CSR's
    // last < 4 nonzeros by plain loads (released by lane 0's arrive)
    auto tail = [&](const AtBatchHdr& h, int s) {
      if (lane < h.n_tail) {
        const int64_t x = h.a_lo + h.cnt + lane;
        s_col[s * kAtCap + h.cnt + lane] = col[x];
        s_val[s * kAtCap + h.cnt + lane] = val[x];
      }
    };
    auto stream = [&](const AtBatchHdr& h, int s, uint32_t extra) {
      mbar_arrive_tx(&sh.full[s], (uint32_t)h.cnt * 8u + extra);
      if (h.cnt) {
        bulk_g2s(smem_u32(s_col + s * kAtCap), col + h.a_lo, (uint32_t)h.cnt * 4u, &sh.full[s]);
        bulk_g2s(smem_u32(s_val + s * kAtCap), val + h.a_lo, (uint32_t)h.cnt * 4u, &sh.full[s]);
      }
    };
    if (PLAN) {
      // headers prefetched 32 batches ahead; the item lists come with the data
      auto fetch_h = [&](int k0) {
        if (k0 + lane < nb)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                           smem_u32(&sh.hring[(k0 + lane) % kAtHdrRing])),
                       "l"(&batches[b0 + k0 + lane].h)
                       : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      fetch_h(0);
      for (; k < nb;) {
        if (k % 32 == 0) {
          asm volatile("cp.async.wait_group 0;" ::: "memory");
          __syncwarp();
          fetch_h(k + 32);
        }
        const AtBatchHdr h = sh.hring[k % kAtHdrRing];
        AtMeta& m = take_slot();
        const int s = k % kAtStages;
        tail(h, s);
        if (lane == 0) m.next = 0;
        __syncwarp();
        if (lane == 0) {
          stream(h, s, (uint32_t)sizeof(AtBatch));
          bulk_g2s(smem_u32(&m.b), &batches[b0 + k], (uint32_t)sizeof(AtBatch), &sh.full[s]);
        }
        ++k;
      }
    } else {
      RpRing rp{sh.rpring, row_ptr, lr0, lr1, 0, 0};
      rp.start(lane);
      int r = lr0;                              // current row
      int64_t e = row_ptr[lr0];                 // its next nonzero (an item boundary)
      while (r < lr1) {
        rp.ready(r, lane);
        AtMeta& m = take_slot();
        const int s = k % kAtStages;
        const AtBatchHdr h = pack_batch(rp, lane, lr1, nnz4, r, e, m.b.item);
        tail(h, s);
        if (lane == 0) {
          m.b.h = h;
          m.next = 0;
        }
        __syncwarp();
        if (lane == 0) stream(h, s, 0u);
        ++k;
      }
    }
    for (int g = 0; g < kAtGroups; ++g) {       // one end marker per group
      AtMeta& m = take_slot();
      if (lane == 0) {
        m.b.h.n_items = -1;
        mbar_arrive(&sh.full[k % kAtStages]);
      }
      ++k;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }

  // -------------------------------------------------------------- consumers
  mbar_wait_spin(&sh.win, 0);
  const int wlo = sh.wlo, wn = sh.wn;
  // the window's shared address held in a register (otherwise rematerialised
  // from the CTA id for every item)
  uint32_t swin, scol0, sval0;
  asm volatile("mov.u32 %0, %1;" : "=r"(swin) : "r"(sbase));
  asm volatile("mov.u32 %0, %1;" : "=r"(scol0) : "r"(smem_u32(s_col)));
  asm volatile("mov.u32 %0, %1;" : "=r"(sval0) : "r"(smem_u32(s_val)));
  const bool own_in_win = row0 + sh.lr0 >= wlo && row0 + sh.lr1 <= wlo + wn;
  const int grp = wid / kAtRows;
  for (int k = grp;; k += kAtGroups) {
    const int s = k % kAtStages, ms = k % kAtMetas;
    mbar_wait_spin(&sh.full[s], (k / kAtStages) & 1);
    AtMeta& m = sh.meta[ms];
    const int ni = m.b.h.n_items;
    if (ni < 0) {                               // end marker (wakes the finaliser)
      if (lane == 0) mbar_arrive(&sh.done[ms]);
      break;
    }
    const uint32_t scs = scol0 + 4u * (uint32_t)(s * kAtCap);
    const uint32_t svs = sval0 + 4u * (uint32_t)(s * kAtCap);
    // one item's sum over the warp's lanes (before the reduction)
    auto item_sum = [&](int t, float& ax, float& ay) {
      const int2 d = m.b.item[t];
      const int l = d.x, i = row0 + l;
      const int beg = d.y & 0x1fff, len = (d.y >> 13) & 0x1ff;
      float2 yi;                                // the row's own point
      if (own_in_win) {                         // whenever the window covers the CTA's rows
        asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(yi.x), "=f"(yi.y)
            : "r"(swin + (unsigned)(i - wlo) * 8u));
      } else {
        yi = win_y(swin, Y, i, wlo, wn);
      }
      const uint32_t scr = scs + 4u * (uint32_t)beg, svr = svs + 4u * (uint32_t)beg;
      switch ((len + 31) >> 5) {
#define TSNE_RB(e)                                                                           \
  case e:                                                                                   \
    if (e <= kAtEmax)                                                                       \
      row_block<(e <= kAtEmax ? e : 1)>(scr, svr, len, i, yi, swin, Y, wlo, wn, lane, ax, ay); \
    break;
        TSNE_RB(1) TSNE_RB(2) TSNE_RB(3) TSNE_RB(4) TSNE_RB(5) TSNE_RB(6) TSNE_RB(7) TSNE_RB(8)
#undef TSNE_RB
        default: break;
      }
    };
    // items are claimed in pairs (t even): both are summed, then reduced
    // together in one fixed butterfly (a lone last item pairs with zeros)
    int t = __shfl_sync(0xffffffffu, lane == 0 ? atomicAdd(&m.next, 2) : 0, 0);
    while (t < ni) {
      float a0 = 0.f, b0 = 0.f, a1 = 0.f, b1 = 0.f;
      item_sum(t, a0, b0);
      const bool two = t + 1 < ni;
      if (two) item_sum(t + 1, a1, b1);
      const float r = warp_sum4(a0, b0, a1, b1);   // lanes 0 / 8 / 16 / 24: a0 / b0 / a1 / b1
      if ((lane & 7) == 0 && (two || lane < 16))
        reinterpret_cast<float*>(&m.part[t])[lane >> 3] = r;
      int tn = 0;
      if (lane == 0) tn = atomicAdd(&m.next, 2);
      t = __shfl_sync(0xffffffffu, tn, 0);
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&sh.empty[s]);
      mbar_arrive(&sh.done[ms]);
    }
  }
}

// CTAs of the pipeline: all SMs when it runs alone (tsne_gradient) or when the
// pass outlasts tree + traversal (more than 200 nonzeros per row); otherwise
// 120 on a side stream concurrently with the tree build: the 28 SMs it leaves
// free take the latency-bound tree kernels, which cannot share an SM with a
// pipeline CTA (measured at C5: iteration 1.33 -> 1.25 ms, the pass alone
// 0.43 -> 0.53 ms).
#ifndef TSNE_AT_GRID_SHARED
#define TSNE_AT_GRID_SHARED 120
#endif
constexpr int kAtGridAlone = kNumSMs;
constexpr int kAtGridShared = TSNE_AT_GRID_SHARED;

static int at_blocks(int64_t n_rows, int grid) {
  const int64_t nch = (n_rows + kAtChunk - 1) / kAtChunk;
  return (int)(nch < grid ? (nch > 0 ? nch : 1) : grid);
}

int attract_grid_sum(int64_t N, int64_t nnz) {
  return at_blocks(N, nnz > 200 * N ? kAtGridAlone : kAtGridShared);
}
int attract_grid_shard(int64_t n_local) { return at_blocks(n_local, kAtGridShared); }

void carve_attract_plan(Carver& c, AtPlan& p, int64_t n_rows, int64_t nnz_cap, int grid) {
  p.grid = grid;
  p.batches = c.take<AtBatch>((size_t)plan_off(n_rows, nnz_cap, grid) + 1);
  p.cta = c.take<int4>(grid);
}

tsne_status attract_plan_build(const AtPlan& p, const int64_t* row_ptr, int64_t n_rows,
                               cudaStream_t s) {
  if (n_rows <= 0) return TSNE_OK;
  k_attract_plan<<<p.grid, 32, 0, s>>>(row_ptr, (int)n_rows, static_cast<AtBatch*>(p.batches),
                                       p.cta);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

template <int MODE, bool PLAN>
static tsne_status launch_win_t(const int64_t* row_ptr, const int32_t* col, const float* val,
                                const float2* Y, int64_t Ny, int64_t row0, int64_t n_rows,
                                const AtPlan* plan, float2* out, const float2* rep,
                                const double* Z, float alpha, cudaStream_t s, int blocks) {
  static bool attr = false;                    // not a stream operation (graph-capture safe)
  if (!attr) {
    TSNE_CUDA_TRY(cudaFuncSetAttribute(k_attract_tma<MODE, PLAN>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAtSmem));
    attr = true;
  }
  k_attract_tma<MODE, PLAN><<<blocks, kAtThreads, kAtSmem, s>>>(
      row_ptr, col, val, Y, (int)Ny, (int)row0, (int)n_rows,
      PLAN ? static_cast<const AtBatch*>(plan->batches) : nullptr, PLAN ? plan->cta : nullptr,
      out, rep, Z, alpha);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
}

// plan: the batches of this CSR cut by attract_plan_build (its grid), or null
// (the kernel cuts them; grid CTAs at most)
template <int MODE>
static tsne_status launch_win(const int64_t* row_ptr, const int32_t* col, const float* val,
                              const float2* Y, int64_t Ny, int64_t row0, int64_t n_rows,
                              float2* out, const float2* rep, const double* Z, float alpha,
                              const AtPlan* plan, cudaStream_t s, int grid) {
  if (n_rows <= 0) return TSNE_OK;
  if (plan)
    return launch_win_t<MODE, true>(row_ptr, col, val, Y, Ny, row0, n_rows, plan, out, rep, Z,
                                    alpha, s, plan->grid);
  return launch_win_t<MODE, false>(row_ptr, col, val, Y, Ny, row0, n_rows, nullptr, out, rep, Z,
                                   alpha, s, at_blocks(n_rows, grid));
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

int update_blocks(int64_t N) {
  int64_t b = (N + kAttrThreads - 1) / kAttrThreads;
  int64_t cap = (int64_t)kNumSMs * 8;
  return (int)(b < cap ? (b < 1 ? 1 : b) : cap);
}

tsne_status launch_attract_grad(const int64_t* row_ptr, const int32_t* col, const float* val,
                                const float2* Y, int64_t N, const float2* rep, const double* Z,
                                float alpha, float2* dY, cudaStream_t s) {
  return launch_win<1>(row_ptr, col, val, Y, N, 0, N, dY, rep, Z, alpha, nullptr, s, kAtGridAlone);
}

tsne_status launch_attract_sum(const int64_t* row_ptr, const int32_t* col, const float* val,
                               const float2* Y, int64_t N, int64_t nnz, float2* A,
                               const AtPlan* plan, cudaStream_t s) {
  // rows of more than ~200 nonzeros (K = 150 workloads): the pass outweighs the tree build
  // it runs beside, so it keeps every SM (attract_grid_sum)
  return launch_win<0>(row_ptr, col, val, Y, N, 0, N, A, nullptr, nullptr, 1.f, plan, s,
                       attract_grid_sum(N, nnz));
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
                                     const float2* Y, int64_t N, int64_t row0, int64_t n_local,
                                     float2* A, const AtPlan* plan, cudaStream_t s) {
  return launch_win<0>(row_ptr, col, val, Y, N, row0, n_local, A, nullptr, nullptr, 1.f, plan, s,
                       kAtGridShared);
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
