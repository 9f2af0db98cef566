// Shared device/host helpers for libmqgnn (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <utility>

#include "../../include/mqgnn.h"
#include "mq_kernels.h"

namespace mq {

// ---------------------------------------------------------------------------
// error plumbing: every C-ABI entry returns MQ_OK or an error code and leaves a
// message readable through mq_last_error() (thread-local).

void set_error(const char* fmt, ...);

#define MQ_CHECK_ARG(cond, ...)                  \
  do {                                           \
    if (!(cond)) {                               \
      ::mq::set_error(__VA_ARGS__);              \
      return MQ_ERR_ARG;                         \
    }                                            \
  } while (0)

#define MQ_CUDA(call)                                                       \
  do {                                                                      \
    cudaError_t _e = (call);                                                \
    if (_e != cudaSuccess) {                                                \
      ::mq::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,            \
                      cudaGetErrorString(_e));                              \
      return MQ_ERR_CUDA;                                                   \
    }                                                                       \
  } while (0)

#define MQ_LAUNCH_CHECK(name)                                               \
  do {                                                                      \
    cudaError_t _e = cudaGetLastError();                                    \
    if (_e != cudaSuccess) {                                                \
      ::mq::set_error("launch %s: %s", name, cudaGetErrorString(_e));       \
      return MQ_ERR_CUDA;                                                   \
    }                                                                       \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// resident blocks per SM of a kernel at this block size (>= 1)
template <class K>
inline int resident_blocks(K kernel, int threads, size_t smem = 0) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) != cudaSuccess) {
    (void)cudaGetLastError();
    n = 1;
  }
  return n < 1 ? 1 : n;
}

constexpr int kNumSMs = 148;

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// ---------------------------------------------------------------------------
// per-kernel event timing (bench instrumentation; off by default, never used
// while a stream is being captured into a CUDA graph)

struct ProfScope {
  int id;
  cudaStream_t s;
  bool on;
  cudaEvent_t a, b;
  ProfScope(int kernel_id, cudaStream_t stream);
  ~ProfScope();
};

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL).  Kernels of the step's dependent chains
// are launched with programmatic stream serialisation, so kernel k+1 is
// scheduled while kernel k still runs and blocks in griddepcontrol.wait until
// k has completed and its writes are visible.  Every PDL-launched kernel
// calls MQ_PDL_ENTRY() first, unconditionally (a grid that exits without
// waiting would let its successor overtake the grid before it).  Without the
// launch attribute both instructions are no-ops.
bool pdl_enabled();

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#define MQ_PDL_ENTRY() \
  do {                 \
    ::mq::pdl_wait();  \
    ::mq::pdl_trigger(); \
  } while (0)

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------
// In-step timeline (MQ_TC_TRACE builds only): per kernel id, the earliest CTA
// entry and the latest CTA exit (%globaltimer), read by mq_debug_timeline.
#ifdef MQ_TC_TRACE
static __device__ unsigned long long g_timeline[32][2];  // one copy per translation unit
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define MQ_TL_BEGIN(id) \
  do { if (threadIdx.x == 0) atomicMin(&::mq::g_timeline[id][0], ::mq::gtimer()); } while (0)
#define MQ_TL_END(id) \
  do { if (threadIdx.x == 0) atomicMax(&::mq::g_timeline[id][1], ::mq::gtimer()); } while (0)
// reader/reset of this TU's copy: extern "C" mq_debug_timeline_<tag>
#define MQ_TL_READER(tag)                                                             \
  extern "C" int mq_debug_timeline_##tag(unsigned long long* out, int reset) {        \
    if (reset) {                                                                      \
      unsigned long long init[32][2];                                                 \
      for (int i = 0; i < 32; ++i) {                                                  \
        init[i][0] = ~0ull;                                                           \
        init[i][1] = 0ull;                                                            \
      }                                                                               \
      return cudaMemcpyToSymbol(::mq::g_timeline, init, sizeof(init)) == cudaSuccess ? 0 : 2; \
    }                                                                                 \
    return cudaMemcpyFromSymbol(out, ::mq::g_timeline, sizeof(unsigned long long) * 64) == \
                   cudaSuccess ? 0 : 2;                                               \
  }
#else
#define MQ_TL_BEGIN(id) do {} while (0)
#define MQ_TL_END(id) do {} while (0)
#define MQ_TL_READER(tag)
#endif

// ---------------------------------------------------------------------------
// Philox4x32-10 (Random123 constants), shared host/device so that host and GPU
// draws are identical by construction.

struct U4 {
  uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ void mulhilo32(uint32_t a, uint32_t b, uint32_t& hi,
                                                   uint32_t& lo) {
#ifdef __CUDA_ARCH__
  hi = __umulhi(a, b);
  lo = a * b;
#else
  uint64_t p = (uint64_t)a * (uint64_t)b;
  hi = (uint32_t)(p >> 32);
  lo = (uint32_t)p;
#endif
}

__host__ __device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo32(0xD2511F53u, c.x, hi0, lo0);
    mulhilo32(0xCD9E8D57u, c.z, hi1, lo1);
    U4 n;
    n.x = hi1 ^ c.y ^ k0;
    n.y = lo1;
    n.z = hi0 ^ c.w ^ k1;
    n.w = lo0;
    c = n;
  }
  return c;
}

// Draw x_j of the row stream (seed, epoch, batch, hop, row) — SURVEY §8c.
struct RowStream {
  uint32_t k0, k1, row, hop, batch;
  U4 cur;
  uint32_t blk;
  __host__ __device__ __forceinline__ RowStream(uint64_t seed, uint64_t epoch, uint32_t batch_,
                                                uint32_t hop_, uint32_t row_)
      : k0((uint32_t)seed), k1((uint32_t)epoch), row(row_), hop(hop_), batch(batch_),
        blk(0xFFFFFFFFu) {}
  __host__ __device__ __forceinline__ uint32_t draw(uint32_t j) {
    uint32_t b = j >> 2;
    if (b != blk) {
      U4 c{b, row, hop, batch};
      cur = philox4x32_10(c, k0, k1);
      blk = b;
    }
    switch (j & 3) {
      case 0: return cur.x;
      case 1: return cur.y;
      case 2: return cur.z;
      default: return cur.w;
    }
  }
};

// Partial Fisher-Yates over pool positions [0, n): writes k positions to pos[].
// r = j + ((x_j * (n - j)) >> 32); swap(j, r); emit element at j. The sparse map
// only ever holds the k swapped-in targets (keys >= j), kept in registers.
template <int MAXK, class IdxT>
__host__ __device__ __forceinline__ void fisher_yates(RowStream& rs, IdxT n, int k, IdxT* pos) {
  IdxT key[MAXK];
  IdxT val[MAXK];
  int used = 0;
  for (int j = 0; j < k; ++j) {
    uint64_t x = rs.draw((uint32_t)j);
    IdxT r = (IdxT)(j + (int64_t)((x * (uint64_t)(n - j)) >> 32));
    IdxT a = (IdxT)j, b = r;
    int ia = -1, ib = -1;
    for (int t = 0; t < used; ++t) {
      if (key[t] == (IdxT)j) ia = t;
      if (key[t] == r) ib = t;
    }
    if (ia >= 0) a = val[ia];
    if (ib >= 0) b = val[ib];
    pos[j] = b;
    if (ib >= 0) {
      val[ib] = a;
    } else {
      key[used] = r;
      val[used] = a;
      ++used;
    }
  }
}

// Feature store: one table, or a seed-partitioned one whose node v lives on
// shard v % n at row v / n (remote shards are peer-mapped NVLink memory).
struct StoreRef {
  const float* base[MQ_MAX_PEERS];
  int n;
  int pitch;
  __device__ __forceinline__ const float* row(int64_t id) const {
    if (n <= 1) return base[0] + id * pitch;
    const int64_t o = id % n;
    return base[o] + (id / n) * pitch;
  }
};

inline StoreRef make_store(const float* store, const float* const* shards, int n_shards,
                           int pitch) {
  StoreRef r;
  memset(&r, 0, sizeof(r));
  r.pitch = pitch;
  if (n_shards >= 2) {
    r.n = n_shards;
    for (int q = 0; q < n_shards; ++q) r.base[q] = shards[q];
  } else {
    r.n = 1;
    r.base[0] = n_shards == 1 ? shards[0] : store;
  }
  return r;
}

// Fixed-order sum p[0] + p[stride] + ... + p[(S-1)*stride] (left to right, so
// results are deterministic); the loads are issued 16 at a time so the chain
// costs ~S/16 L2 round trips instead of S (a 128-partial head gradient: 8).
#ifndef MQ_SUM_BATCH
#define MQ_SUM_BATCH 16  // partial loads in flight per batch of fixed_order_sum
#endif
__device__ __forceinline__ float fixed_order_sum(const float* __restrict__ p, int64_t stride,
                                                 int S) {
  constexpr int kB = MQ_SUM_BATCH;
  float v = 0.f;
  int s = 0;
  for (; s + kB <= S; s += kB) {
    float t[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) t[u] = __ldcg(p + (int64_t)(s + u) * stride);
#pragma unroll
    for (int u = 0; u < kB; ++u) v += t[u];
  }
  if (s < S) {
    float t[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) t[u] = s + u < S ? __ldcg(p + (int64_t)(s + u) * stride) : 0.f;
#pragma unroll
    for (int u = 0; u < kB; ++u)
      if (s + u < S) v += t[u];
  }
  return v;
}


}  // namespace mq
