// common.cuh -- shared plumbing of libtsne_b200 (errors, workspace carving,
// small device helpers).  Nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstddef>

#include "../../include/tsne.h"

namespace tsne {

void set_error(const char* fmt, ...);
void clear_error();

#define TSNE_CUDA_TRY(expr)                                                    \
  do {                                                                         \
    cudaError_t e__ = (expr);                                                  \
    if (e__ != cudaSuccess) {                                                  \
      ::tsne::set_error("%s:%d %s -> %s", __FILE__, __LINE__, #expr,           \
                        cudaGetErrorString(e__));                              \
      return TSNE_ERR_CUDA;                                                    \
    }                                                                          \
  } while (0)

#define TSNE_LAUNCH_CHECK() TSNE_CUDA_TRY(cudaGetLastError())

#define TSNE_ARG_CHECK(cond, ...)                                              \
  do {                                                                         \
    if (!(cond)) {                                                             \
      ::tsne::set_error(__VA_ARGS__);                                          \
      return TSNE_ERR_ARG;                                                     \
    }                                                                          \
  } while (0)

// Workspace carving: the same sequence of take() calls is run once with a
// null base (size query) and once on the caller's buffer.
struct Carver {
  uintptr_t base = 0;
  size_t off = 0;
  explicit Carver(void* b = nullptr) : base(reinterpret_cast<uintptr_t>(b)) {}
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base + off);
    off += n * sizeof(T);
    return p;
  }
  size_t bytes() const { return (off + 255) & ~size_t(255); }
};

inline bool aligned(const void* p, size_t a) {
  return (reinterpret_cast<uintptr_t>(p) % a) == 0;
}

constexpr int kNumSMs = 148;

// Largest N of the entry points that build the quadtree: the fixed-point
// centre-of-mass sums hold count * 2^38 < 2^63 (|q| < 2^38 per point) (tree.cuh kFixScale) and the
// node index (< 2N) fits the 27-bit skip field of a node record.
constexpr int64_t kMaxTreePoints = (int64_t(1) << 25) - 1;

// ---------------------------------------------------------------- device
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <class T>
__device__ __forceinline__ T ldg_stream(const T* p) {  // read-once data
  return __ldcs(p);
}

// Programmatic dependent launch: a kernel launched with launch_pdl may start
// while its predecessor on the stream is finishing; it lets its own dependents
// launch at once (pdl_trigger) and waits for the predecessor's completion and
// memory (pdl_wait) before reading anything the predecessor wrote.  (Both are
// no-ops in a kernel launched without the attribute.)
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace tsne
