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
// Attractive pass as a persistent TMA pipeline (one CTA per SM).  The CTA
// owns a contiguous range of rows, cut into batches of at most kAtBatch rows
// whose nonzeros fit a stage buffer.  A producer warp streams each batch's
// col/val span (contiguous in the CSR) into a kAtStages-deep shared-memory
// ring with cp.async.bulk + mbarriers (the bulk copies keep ~3 batches of the
// 8-byte-per-nonzero stream in flight per SM without holding registers); the
// embedding window Y[wlo, wlo + kAtWin) around the CTA's rows is staged once
// the same way.  Two groups of kAtRows consumer warps take alternate batches
// (latency hiding for the L2 gathers); warp w of a group computes rows w and
// w + kAtRows of its batches: lanes take consecutive nonzeros from shared memory, gather y_j
// from the window (columns outside it, rare once the labels are in a locality
// order -- DESIGN.md 6.4-6.5 -- come from L2), and reduce with a fixed
// butterfly (deterministic; the result does not depend on which path an
// operand came from).  A batch whose span does not fit a stage buffer is read
// from global memory directly; rows of more than kAtLong nonzeros go to
// k_attract_long.  The sizes below are the measured best of the variants in
// DESIGN.md 6.4 (overridable at compile time for such experiments).
#ifndef TSNE_AT_ROWS
#define TSNE_AT_ROWS 15
#define TSNE_AT_GROUPS 2
#define TSNE_AT_STAGES 4
#define TSNE_AT_CAP 4096
#define TSNE_AT_WIN 12288
#endif
constexpr int kAtRows = TSNE_AT_ROWS;          // consumer warps per group
constexpr int kAtGroups = TSNE_AT_GROUPS;      // consumer groups take alternate batches
constexpr int kAtConsumers = kAtRows * kAtGroups;
constexpr int kAtThreads = (kAtConsumers + 1) * 32;
constexpr int kAtStages = TSNE_AT_STAGES;
constexpr int kAtCap = TSNE_AT_CAP;            // nonzeros per stage buffer
constexpr int kAtWin = TSNE_AT_WIN;            // window points
#ifndef TSNE_AT_BATCH
#define TSNE_AT_BATCH (2 * TSNE_AT_ROWS)
#endif
constexpr int kAtBatch = TSNE_AT_BATCH;        // rows per batch: up to 2 per consumer warp
#ifndef TSNE_AT_EMAX
#define TSNE_AT_EMAX 8
#endif
constexpr int kAtEmax = TSNE_AT_EMAX;          // 32-entry groups of a row loaded together
constexpr int kAtLong = 2048;                  // longer rows: k_attract_long
constexpr int kAtChunk = 56;                   // rows per row_ptr prefetch chunk (~2 batches)
constexpr int kAtLook = 3;                     // row_ptr prefetch distance (chunks)
constexpr int kAtRpSlots = kAtLook + 1;
static_assert(kAtStages % kAtGroups == 0, "a stage always serves the same consumer group");
constexpr size_t kAtSmem = sizeof(float2) * kAtWin + (size_t)kAtStages * kAtCap * 8;

static_assert(kAtBatch < 32, "a batch is cut by one warp ballot");
struct AtMeta {
  int64_t rp[kAtBatch + 1];  // row_ptr of the batch's rows (local CSR)
  int64_t a_lo, a_hi;        // staged nonzeros [a_lo, a_hi) (a_hi <= a_lo when not staged)
  int32_t r0, nrows;         // first local row, rows in the batch
};

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

__device__ __forceinline__ void win_accum(float2 yi, float2 yj, float p, float& ax, float& ay) {
  const float dx = yi.x - yj.x, dy = yi.y - yj.y;
  const float w = rcp_approx_f(fmaf(dy, dy, fmaf(dx, dx, 1.f)));   // 1/(1+d^2), d^2 >= 0
  const float pw = p * w;
  ax = fmaf(pw, dx, ax);
  ay = fmaf(pw, dy, ay);
}

// E x 32 consecutive entries of a staged row (n_rem entries remain from cr):
// lane takes entries lane + 32u; only the last group can be partial (its
// absent entries are the point itself with p = 0).  All loads first, then
// the arithmetic: the window / L2 gathers of the block are in flight together.
template <int E>
__device__ __forceinline__ void row_block(const int32_t* __restrict__ cr,
                                          const float* __restrict__ vr, int n_rem, int self,
                                          float2 yi, uint32_t sbase, const float2* __restrict__ Y,
                                          int wlo, int wn, int lane, float& ax, float& ay) {
  int c[E];
  float p[E];
#pragma unroll
  for (int u = 0; u < E; ++u) {
    const int q = lane + 32 * u;
    if (u < E - 1) {
      c[u] = cr[q];
      p[u] = vr[q];
    } else {
      c[u] = self;
      p[u] = 0.f;
      if (q < n_rem) {
        c[u] = cr[q];
        p[u] = vr[q];
      }
    }
  }
  float2 y[E];
#pragma unroll
  for (int u = 0; u < E; ++u) y[u] = win_y(sbase, Y, c[u], wlo, wn);
#pragma unroll
  for (int u = 0; u < E; ++u) win_accum(yi, y[u], p[u], ax, ay);
}

// spin wait (no suspend-time hint: the pipeline's waits are short and a
// sleeping producer would throttle the stream)
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

// MODE 0: out[l] = A_l.  MODE 1 (tsne_gradient): out[l] = 4 (alpha A_l - f_l / Z).
// Rows l in [0, n_rows) of the (local) CSR are global points row0 + l of Y.
template <int MODE>
__global__ void __launch_bounds__(kAtThreads, 1)
k_attract_tma(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
              const float* __restrict__ val, const float2* __restrict__ Y, int Ny, int row0,
              int n_rows, float2* __restrict__ out, const float2* __restrict__ rep,
              const double* __restrict__ Z, float alpha) {
  extern __shared__ __align__(128) unsigned char at_smem[];
  __shared__ AtMeta s_meta[kAtStages];
  __shared__ __align__(16) int64_t s_rpring[kAtRpSlots][kAtChunk + 1];
  __shared__ __align__(8) uint64_t s_full[kAtStages], s_empty[kAtStages], s_win;
  float2* s_y = reinterpret_cast<float2*>(at_smem);
  int32_t* s_col = reinterpret_cast<int32_t*>(at_smem + sizeof(float2) * kAtWin);
  float* s_val = reinterpret_cast<float*>(s_col + kAtStages * kAtCap);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // this CTA's rows [lr0, lr1): whole chunks of kAtChunk rows
  const int nch_all = (n_rows + kAtChunk - 1) / kAtChunk;
  const int c0 = (int)((int64_t)nch_all * blockIdx.x / gridDim.x);
  const int c1 = (int)((int64_t)nch_all * (blockIdx.x + 1) / gridDim.x);
  const int lr0 = c0 * kAtChunk, lr1 = min(c1 * kAtChunk, n_rows);
  int wlo = row0 + (lr0 + lr1) / 2 - kAtWin / 2;
  wlo = min(wlo, Ny - kAtWin);
  wlo = max(wlo, 0) & ~1;                      // 16-byte aligned source
  const int wn = min(kAtWin, Ny - wlo) & ~1;   // 16-byte multiple
  const bool own_in_win = row0 + lr0 >= wlo && row0 + lr1 <= wlo + wn;
  const uint32_t sbase = smem_u32(s_y);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kAtStages; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], kAtRows);
    }
    mbar_init(&s_win, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (wid == kAtConsumers) {
    // ------------------------------------------------------------ producer
    const int64_t nnz4 = row_ptr[n_rows] & ~int64_t(3);
    if (lane == 0) {
      mbar_arrive_tx(&s_win, (uint32_t)(wn * sizeof(float2)));
      bulk_g2s(sbase, Y + wlo, (uint32_t)(wn * sizeof(float2)), &s_win);
    }
    // row_ptr of chunk c + kAtLook is fetched with cp.async into a small ring
    // while chunk c is cut into batches, so the producer never waits on a
    // global load.  A batch is at most kAtBatch rows whose nonzeros fit a stage
    // (a longer single row is read from global memory by its consumer).
    auto fetch_rp = [&](int c) {
      if (c < c1)
        for (int q = lane; q <= kAtChunk; q += 32) {
          const int r = min(c * kAtChunk + q, n_rows);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                           smem_u32(&s_rpring[c % kAtRpSlots][q])),
                       "l"(row_ptr + r)
                       : "memory");
        }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // row_ptr of local row r from the ring (a chunk's slot holds kAtChunk + 1
    // entries; the end of the CTA's range at a chunk boundary is the last
    // entry of the previous chunk)
    auto rpv = [&](int r) -> int64_t {
      const int c = r / kAtChunk, o = r - c * kAtChunk;
      if (r == lr1 && o == 0) return s_rpring[(c - 1) % kAtRpSlots][kAtChunk];
      return s_rpring[c % kAtRpSlots][o];
    };
    int k = 0;                                  // batch sequence number
    auto issue = [&](int r0, int nr, bool sentinel) {
      const int s = k % kAtStages;
#ifdef TSNE_AT_SPIN
      if (k >= kAtStages) mbar_wait_spin(&s_empty[s], ((k / kAtStages) - 1) & 1);
#else
      if (k >= kAtStages) mbar_wait_sleep(&s_empty[s], ((k / kAtStages) - 1) & 1);
#endif
      AtMeta& m = s_meta[s];
      int64_t a_lo = 0, a_hi = 0;
      if (!sentinel) {
        const int64_t v = rpv(r0 + min(lane, nr));
        if (lane <= nr) m.rp[lane] = v;
        const int64_t e_lo = __shfl_sync(0xffffffffu, v, 0), e_hi = __shfl_sync(0xffffffffu, v, nr);
        a_lo = e_lo & ~int64_t(3);
        a_hi = min((e_hi + 3) & ~int64_t(3), nnz4);
        if (e_hi + 3 - a_lo > kAtCap) a_hi = a_lo;            // does not fit: read from global
      }
      if (lane == 0) {
        m.a_lo = a_lo;
        m.a_hi = a_hi;
        m.r0 = r0;
        m.nrows = sentinel ? -1 : nr;
      }
      __syncwarp();
      if (lane == 0) {
        const uint32_t cnt = (a_hi > a_lo) ? (uint32_t)(a_hi - a_lo) : 0u;
        mbar_arrive_tx(&s_full[s], cnt * 8u);
        if (cnt) {
          bulk_g2s(smem_u32(s_col + s * kAtCap), col + a_lo, cnt * 4u, &s_full[s]);
          bulk_g2s(smem_u32(s_val + s * kAtCap), val + a_lo, cnt * 4u, &s_full[s]);
        }
      }
      ++k;
    };
    // Batches are cut across chunk boundaries (a batch of at most kAtBatch <
    // kAtChunk rows spans at most two chunks), so rows of ~230 nonzeros (C4:
    // 17 per stage) do not leave a short batch at the end of every chunk.
    for (int j = 0; j < kAtLook; ++j) fetch_rp(c0 + j);
    int fetched = c0 + kAtLook;                 // next chunk to fetch
    for (int row = lr0; row < lr1;) {
      const int c = row / kAtChunk;
      while (fetched <= c + kAtLook) fetch_rp(fetched++);
      asm volatile("cp.async.wait_group %0;" ::"n"(kAtLook - 1) : "memory");   // chunks <= c + 1
      __syncwarp();
      // largest nr <= kAtBatch with rows [row, row + nr) fitting a stage (a prefix: rp grows)
      const int l = lane + 1;
      const int64_t base = rpv(row) & ~int64_t(3);
      const bool ok = l <= kAtBatch && row + l <= lr1 && rpv(min(row + l, lr1)) + 3 - base <= kAtCap;
      int nr = __popc(__ballot_sync(0xffffffffu, ok));
      nr = nr > 0 ? nr : 1;
      issue(row, nr, false);
      row += nr;
    }
    for (int g = 0; g < kAtGroups; ++g) issue(0, 0, true);   // one end marker per group
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }

  // -------------------------------------------------------------- consumers
  mbar_wait_spin(&s_win, 0);
  const int grp = wid / kAtRows, wr = wid % kAtRows;
  for (int k = grp;; k += kAtGroups) {
    const int s = k % kAtStages;
    mbar_wait_spin(&s_full[s], (k / kAtStages) & 1);
    const AtMeta& m = s_meta[s];
    if (m.nrows < 0) break;                     // end marker
    for (int br = wr; br < m.nrows; br += kAtRows) {
      const int l = m.r0 + br;
      const int i = row0 + l;
      const int64_t e0 = m.rp[br], e1 = m.rp[br + 1];
      const int64_t a_lo = m.a_lo, a_hi = m.a_hi;
      const int32_t* cs = s_col + s * kAtCap;
      const float* vs = s_val + s * kAtCap;
      float2 yi;                                  // the row's own point: in the window
      if (own_in_win) {                           // whenever the window covers the CTA's rows
        asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(yi.x), "=f"(yi.y)
            : "r"(sbase + (unsigned)(i - wlo) * 8u));
      } else {
        yi = win_y(sbase, Y, i, wlo, wn);
      }
      float ax = 0.f, ay = 0.f;
      const int n = (int)(e1 - e0);
      if (e0 >= a_lo && e1 <= a_hi) {             // the row is staged (the common case)
        const int32_t* cr = cs + (e0 - a_lo);
        const float* vr = vs + (e0 - a_lo);
        // blocks of up to 8 x 32 entries: every gather of a block is issued
        // before any arithmetic, so a row pays the L2 latency of its columns
        // outside the window about once, not once per 32 entries
        int b = 0;
        for (; n - b > kAtEmax * 32; b += kAtEmax * 32)
          row_block<kAtEmax>(cr + b, vr + b, n - b, i, yi, sbase, Y, wlo, wn, lane, ax, ay);
        switch ((n - b + 31) >> 5) {
#define TSNE_RB(e)                                                                           \
  case e:                                                                                   \
    if (e <= kAtEmax)                                                                       \
      row_block<(e <= kAtEmax ? e : 1)>(cr + b, vr + b, n - b, i, yi, sbase, Y, wlo, wn,    \
                                        lane, ax, ay);                                      \
    break;
          TSNE_RB(1) TSNE_RB(2) TSNE_RB(3) TSNE_RB(4) TSNE_RB(5) TSNE_RB(6) TSNE_RB(7) TSNE_RB(8)
#undef TSNE_RB
          default: break;
        }
      } else if (n <= kAtLong) {
        for (int q = lane; q < n; q += 32)
          win_accum(yi, win_y(sbase, Y, __ldcs(col + e0 + q), wlo, wn), __ldcs(val + e0 + q), ax,
                    ay);
      }
      warp_sum2(ax, ay);
      if (lane == 0 && n <= kAtLong) {          // longer rows: k_attract_long
        if (MODE == 0) {
          out[l] = make_float2(ax, ay);
        } else {
          const float invZ = (float)Z[1];
          const float2 f = rep[l];
          out[l] = make_float2(4.f * (alpha * ax - f.x * invZ), 4.f * (alpha * ay - f.y * invZ));
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&s_empty[s]);
  }
}

// Rows longer than kAtLong nonzeros (hubs of the kNN graph: a point that is a
// neighbour of thousands of others) would serialise one warp of the
// pipeline; a whole CTA takes each of them instead.  CTA b scans rows
// [b*n/G, (b+1)*n/G) and processes the long ones: threads stride the row, the
// sum is reduced in a fixed order (deterministic).
constexpr int kLongThreads = 512;

template <int MODE>
__global__ void __launch_bounds__(kLongThreads)
k_attract_long(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
               const float* __restrict__ val, const float2* __restrict__ Y, int row0, int n_rows,
               float2* __restrict__ out, const float2* __restrict__ rep,
               const double* __restrict__ Z, float alpha) {
  __shared__ float2 s_red[kLongThreads / 32];
  __shared__ unsigned s_ball[kLongThreads / 32];
  const int r0 = (int)((int64_t)n_rows * blockIdx.x / gridDim.x);
  const int r1 = (int)((int64_t)n_rows * (blockIdx.x + 1) / gridDim.x);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = r0; base < r1; base += kLongThreads) {
    const int r = base + (int)threadIdx.x;
    const bool lng = r < r1 && row_ptr[r + 1] - row_ptr[r] > kAtLong;
    const unsigned ball = __ballot_sync(0xffffffffu, lng);
    if (lane == 0) s_ball[wid] = ball;
    __syncthreads();
    for (int w = 0; w < kLongThreads / 32; ++w) {
      unsigned b = s_ball[w];
      while (b) {                                       // block-uniform loop
        const int l = base + w * 32 + __ffs(b) - 1;
        b &= b - 1;
        const float2 yi = Y[row0 + l];
        float ax = 0.f, ay = 0.f;
        const int64_t eb = row_ptr[l], ee = row_ptr[l + 1];
        for (int64_t e = eb + threadIdx.x; e < ee; e += 4 * kLongThreads) {   // 4 in flight
          int c[4];
          float p[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int64_t f = e + u * kLongThreads;
            c[u] = row0 + l;                           // absent: the point itself, p = 0
            p[u] = 0.f;
            if (f < ee) {
              c[u] = __ldcs(col + f);
              p[u] = __ldcs(val + f);
            }
          }
          float2 yj[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) yj[u] = __ldg(Y + c[u]);
#pragma unroll
          for (int u = 0; u < 4; ++u) win_accum(yi, yj[u], p[u], ax, ay);
        }
        ax = warp_sum(ax);
        ay = warp_sum(ay);
        if (lane == 0) s_red[wid] = make_float2(ax, ay);
        __syncthreads();
        if (threadIdx.x == 0) {
          float sx = 0.f, sy = 0.f;
          for (int q = 0; q < kLongThreads / 32; ++q) { sx += s_red[q].x; sy += s_red[q].y; }
          if (MODE == 0) {
            out[l] = make_float2(sx, sy);
          } else {
            const float invZ = (float)Z[1];
            const float2 f = rep[l];
            out[l] = make_float2(4.f * (alpha * sx - f.x * invZ), 4.f * (alpha * sy - f.y * invZ));
          }
        }
        __syncthreads();
      }
    }
    __syncthreads();
  }
}

// CTAs of the pipeline: all SMs when it runs alone (tsne_gradient); 120 when it
// runs concurrently with the tree build on a side stream (optimiser, shards):
// the 28 SMs it leaves free take the latency-bound tree kernels, which cannot
// share an SM with a pipeline CTA (measured at C5: iteration 1.33 -> 1.25 ms,
// the pass alone 0.43 -> 0.53 ms).
#ifndef TSNE_AT_GRID_SHARED
#define TSNE_AT_GRID_SHARED 120
#endif
constexpr int kAtGridAlone = kNumSMs;
constexpr int kAtGridShared = TSNE_AT_GRID_SHARED;

template <int MODE>
static tsne_status launch_win(const int64_t* row_ptr, const int32_t* col, const float* val,
                              const float2* Y, int64_t Ny, int64_t row0, int64_t n_rows,
                              float2* out, const float2* rep, const double* Z, float alpha,
                              cudaStream_t s, int grid) {
  if (n_rows <= 0) return TSNE_OK;
  static bool attr = false;                    // not a stream operation (graph-capture safe)
  if (!attr) {
    TSNE_CUDA_TRY(cudaFuncSetAttribute(k_attract_tma<MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kAtSmem));
    attr = true;
  }
  const int64_t nch = (n_rows + kAtChunk - 1) / kAtChunk;
  const int blocks = (int)(nch < grid ? nch : grid);
  k_attract_tma<MODE><<<blocks, kAtThreads, kAtSmem, s>>>(row_ptr, col, val, Y, (int)Ny,
                                                           (int)row0, (int)n_rows, out, rep, Z,
                                                           alpha);
  TSNE_LAUNCH_CHECK();
  const int64_t lb = (n_rows + kLongThreads - 1) / kLongThreads;
  const int lblocks = (int)(lb < 2 * kNumSMs ? lb : 2 * kNumSMs);
  k_attract_long<MODE><<<lblocks, kLongThreads, 0, s>>>(row_ptr, col, val, Y, (int)row0,
                                                        (int)n_rows, out, rep, Z, alpha);
  TSNE_LAUNCH_CHECK();
  return TSNE_OK;
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
  return launch_win<1>(row_ptr, col, val, Y, N, 0, N, dY, rep, Z, alpha, s, kAtGridAlone);
}

tsne_status launch_attract_sum(const int64_t* row_ptr, const int32_t* col, const float* val,
                               const float2* Y, int64_t N, int64_t nnz, float2* A, cudaStream_t s) {
  // rows of more than ~200 nonzeros (K = 150 workloads): the pass outweighs the tree build
  // it runs beside, so it keeps every SM (C4: 1.73 ms on 148 CTAs, 2.04 ms on 120)
  const int grid = nnz > 200 * N ? kAtGridAlone : kAtGridShared;
  return launch_win<0>(row_ptr, col, val, Y, N, 0, N, A, nullptr, nullptr, 1.f, s, grid);
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
                                     float2* A, cudaStream_t s) {
  return launch_win<0>(row_ptr, col, val, Y, N, row0, n_local, A, nullptr, nullptr, 1.f, s,
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
