// Single-pass exclusive scan with decoupled look-back (sm_100a).
//
// One launch scans n (device-resident) values: each CTA takes a dynamically
// assigned tile of THREADS*ITEMS elements, reduces it, publishes its aggregate,
// looks back over its predecessors' published aggregates/prefixes and then
// hands every element's exclusive prefix to a Store functor.  Load/Store are
// functors so the scan can compute its input on the fly (flags, bit tests)
// and emit compactions directly — the relabel and residency kernels are
// scans with custom functors.
#pragma once

#include "mq_common.cuh"

namespace mq {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

// status word: [63:62] flag (0 invalid, 1 aggregate, 2 inclusive prefix), [61:0] value
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPre = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

inline int64_t scan_tiles(int64_t n_max) { return (n_max + kScanTile - 1) / kScanTile; }

inline int64_t scan_scratch_bytes(int64_t n_max) {
  return 16 + 8 * (scan_tiles(n_max) + 1);
}

// Load:  __device__ int64_t size() const;  __device__ int64_t operator()(int64_t i) const
// Store: __device__ void operator()(int64_t i, int64_t excl, int64_t val) const;
//        __device__ void total(int64_t n, int64_t t) const
template <class Load, class Store>
__device__ __forceinline__ void scan_tile(const Load& load, const Store& store, void* scratch) {
  unsigned int* ticket = reinterpret_cast<unsigned int*>(scratch);
  unsigned long long* status = reinterpret_cast<unsigned long long*>((char*)scratch + 16);
  __shared__ int s_tile;
  __shared__ int64_t s_warp[kScanThreads / 32];
  __shared__ int64_t s_excl;

  const int tid = threadIdx.x;
  if (tid == 0) s_tile = (int)atomicAdd(ticket, 1u);
  __syncthreads();
  const int tile = s_tile;
  const int64_t n = load.size();
  const int64_t base = (int64_t)tile * kScanTile;
  if (base >= n) {
    if (tile == 0 && tid == 0) store.total(n, 0);  // n == 0
    return;
  }

  int64_t v[kScanItems];
  int64_t local = 0;
  const int64_t mine = base + (int64_t)tid * kScanItems;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = mine + k;
    v[k] = (i < n) ? load(i) : 0;
    local += v[k];
  }
  // warp inclusive scan of per-thread sums
  const int lane = tid & 31, warp = tid >> 5;
  int64_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int64_t w = (lane < kScanThreads / 32) ? s_warp[lane] : 0;
    int64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < kScanThreads / 32) s_warp[lane] = wi - w;  // exclusive warp offsets
    int64_t agg = __shfl_sync(0xffffffffu, wi, kScanThreads / 32 - 1);
    // decoupled look-back, a window of 32 predecessors per step (lane l reads
    // tile p - l): stop at the nearest published inclusive prefix, re-read
    // while a closer predecessor has published nothing yet
    int64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) st_relaxed(&status[0], kFlagPre | (unsigned long long)agg);
    } else {
      if (lane == 0) st_relaxed(&status[tile], kFlagAgg | (unsigned long long)agg);
      int p = tile - 1;
      while (true) {
        const int idx = p - lane;
        const unsigned long long w2 = idx >= 0 ? ld_relaxed(&status[idx]) : kFlagPre;
        const unsigned long long flag = w2 & ~kValMask;
        const unsigned pre = __ballot_sync(0xffffffffu, flag == kFlagPre);
        const unsigned inv = __ballot_sync(0xffffffffu, flag == 0);
        const int stop = pre ? __ffs(pre) - 1 : 32;  // nearest prefix in the window
        const unsigned closer = stop == 32 ? 0xffffffffu : ((1u << stop) - 1u);
        if (inv & closer) continue;  // a nearer tile has not published yet
        int64_t part = lane <= stop ? (int64_t)(w2 & kValMask) : 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        excl += part;
        if (stop < 32) break;
        p -= 32;
      }
      if (lane == 0) st_relaxed(&status[tile], kFlagPre | (unsigned long long)(excl + agg));
    }
    if (lane == 0) {
      s_excl = excl;
      if (base + kScanTile >= n) store.total(n, excl + agg);
    }
  }
  __syncthreads();
  int64_t run = s_excl + s_warp[warp] + (incl - local);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    int64_t i = mine + k;
    if (i < n) store(i, run, v[k]);
    run += v[k];
  }
}

template <class Load, class Store>
__global__ void __launch_bounds__(kScanThreads) scan_kernel(Load load, Store store, void* scratch) {
  scan_tile(load, store, scratch);
}

// Q independent scans in one launch: blockIdx.y selects the slot (the Load /
// Store functors read it too) and its private ticket/status region.
template <class Load, class Store>
__global__ void __launch_bounds__(kScanThreads)
    scan_q_kernel(Load load, Store store, void* scratch, int64_t scratch_stride) {
  scan_tile(load, store, reinterpret_cast<char*>(scratch) + (int64_t)blockIdx.y * scratch_stride);
}

template <class Load, class Store>
int launch_scan(const Load& load, const Store& store, int64_t n_max, void* scratch,
                cudaStream_t s, int kid = K_SCAN) {
  MQ_CUDA(cudaMemsetAsync(scratch, 0, scan_scratch_bytes(n_max), s));
  int tiles = (int)scan_tiles(n_max);
  if (tiles < 1) tiles = 1;
  {
    ProfScope ps(kid, s);
    scan_kernel<Load, Store><<<tiles, kScanThreads, 0, s>>>(load, store, scratch);
  }
  MQ_LAUNCH_CHECK("scan");
  return MQ_OK;
}

// ---- common functors
struct LoadI32 {
  const int32_t* in;
  const int32_t* n_dev;
  int64_t n_static;
  __device__ int64_t size() const { return n_dev ? (int64_t)*n_dev : n_static; }
  __device__ int64_t operator()(int64_t i) const { return in[i]; }
};

template <class OutT>
struct StoreOffsets {
  OutT* out;  // n+1 entries
  __device__ void operator()(int64_t i, int64_t excl, int64_t) const { out[i] = (OutT)excl; }
  __device__ void total(int64_t n, int64_t t) const { out[n] = (OutT)t; }
};

template <class Load, class Store>
int launch_scan_q(const Load& load, const Store& store, int64_t n_max, int nslots, void* scratch,
                  int64_t scratch_stride, cudaStream_t s, int kid) {
  MQ_CUDA(cudaMemsetAsync(scratch, 0, (size_t)scratch_stride * nslots, s));
  int tiles = (int)scan_tiles(n_max);
  if (tiles < 1) tiles = 1;
  {
    ProfScope ps(kid, s);
    scan_q_kernel<Load, Store><<<dim3(tiles, nslots), kScanThreads, 0, s>>>(load, store, scratch,
                                                                           scratch_stride);
  }
  MQ_LAUNCH_CHECK("scan_q");
  return MQ_OK;
}

}  // namespace mq
