// Feature gather: HBM GNS-cache table + (device or pinned-host) feature store.
//
// Reference: mqpipe/cache.py:111-134 (lookup, gather_features) and
// runtime.py:127-143 (transfer_stage).  Output rows are bit-identical copies.
#include "mq_common.cuh"

namespace mq {

constexpr int kGatherThreads = 256;

// One warp per output row; 16-byte vector copies.  Rows are independent, so
// each warp keeps 4 float4 loads in flight before it stores.
__global__ void __launch_bounds__(kGatherThreads) gather_kernel(
    const float* __restrict__ cache_tbl, int cache_pitch, const int32_t* __restrict__ slot_of,
    StoreRef store, const int32_t* __restrict__ ids,
    const int32_t* __restrict__ n_dev, int d4, float* __restrict__ out, int out_pitch,
    unsigned long long* __restrict__ hit_miss) {
  __shared__ unsigned int s_hits, s_miss;
  if (threadIdx.x == 0) {
    s_hits = 0;
    s_miss = 0;
  }
  __syncthreads();
  const int n = *n_dev;
  const int lane = threadIdx.x & 31;
  const int warps = kGatherThreads / 32;
  int64_t row = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5);
  const int64_t stride = (int64_t)gridDim.x * warps;
  unsigned int hits = 0, miss = 0;
  for (; row < n; row += stride) {
    const int32_t id = ids[row];
    const float4* src;
    int32_t slot = slot_of ? slot_of[id] : -1;
    if (slot >= 0) {
      src = reinterpret_cast<const float4*>(cache_tbl + (int64_t)slot * cache_pitch);
      ++hits;
    } else {
      src = reinterpret_cast<const float4*>(store.row(id));
      ++miss;
    }
    float4* dst = reinterpret_cast<float4*>(out + row * out_pitch);
    int c = lane;
    for (; c + 96 < d4; c += 128) {
      float4 a = src[c], b = src[c + 32], e = src[c + 64], f = src[c + 96];
      dst[c] = a;
      dst[c + 32] = b;
      dst[c + 64] = e;
      dst[c + 96] = f;
    }
    for (; c < d4; c += 32) dst[c] = src[c];
  }
  if (slot_of != nullptr && lane == 0) {
    atomicAdd(&s_hits, hits);
    atomicAdd(&s_miss, miss);
  }
  __syncthreads();
  if (slot_of != nullptr && threadIdx.x == 0 && (s_hits | s_miss)) {
    atomicAdd(&hit_miss[0], (unsigned long long)s_hits);
    atomicAdd(&hit_miss[1], (unsigned long long)s_miss);
  }
}

__global__ void gather_labels_kernel(const int32_t* __restrict__ all_labels,
                                     const int32_t* __restrict__ ids, const int32_t* __restrict__ n_dev,
                                     int32_t* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < *n_dev) out[i] = all_labels[ids[i]];
}

}  // namespace mq

using namespace mq;

extern "C" {

static int gather_impl(const float* cache_tbl, int32_t cache_pitch, const int32_t* slot_of,
                       StoreRef store, const int32_t* ids, const int32_t* n_dev, int32_t n_max,
                       int32_t d, float* out, int32_t out_pitch, unsigned long long* hit_miss,
                       void* stream, const char* who) {
  MQ_CHECK_ARG(ids && n_dev && out, "%s: null pointer", who);
  MQ_CHECK_ARG(d >= 1, "%s: d must be positive", who);
  const int d4 = (d + 3) / 4;
  MQ_CHECK_ARG(store.pitch % 4 == 0 && out_pitch % 4 == 0 && store.pitch >= 4 * d4 &&
                   out_pitch >= 4 * d4,
               "%s: pitches must be multiples of 4 floats covering d (d=%d, store %d, out %d)",
               who, d, store.pitch, out_pitch);
  MQ_CHECK_ARG((uintptr_t)out % 16 == 0, "%s: output must be 16B aligned", who);
  for (int q = 0; q < store.n; ++q)
    MQ_CHECK_ARG(store.base[q] && (uintptr_t)store.base[q] % 16 == 0,
                 "%s: store table %d missing or not 16B aligned", who, q);
  if (slot_of) {
    MQ_CHECK_ARG(cache_tbl && hit_miss && cache_pitch % 4 == 0 && cache_pitch >= 4 * d4 &&
                     (uintptr_t)cache_tbl % 16 == 0,
                 "%s: cache table / counters invalid", who);
  }
  if (n_max <= 0) return MQ_OK;
  cudaStream_t s = as_stream(stream);
  const int warps = kGatherThreads / 32;
  int blocks = ceil_div(n_max, warps);
  if (blocks > kNumSMs * 16) blocks = kNumSMs * 16;
  {
    ProfScope ps(K_GATHER, s);
    gather_kernel<<<blocks, kGatherThreads, 0, s>>>(cache_tbl, cache_pitch, slot_of, store, ids,
                                                    n_dev, d4, out, out_pitch, hit_miss);
  }
  MQ_LAUNCH_CHECK(who);
  return MQ_OK;
}

int mq_gather(const float* cache_tbl, int32_t cache_pitch, const int32_t* slot_of,
              const float* store, int32_t store_pitch, const int32_t* ids, const int32_t* n_dev,
              int32_t n_max, int32_t d, float* out, int32_t out_pitch,
              unsigned long long* hit_miss, void* stream) {
  MQ_CHECK_ARG(store, "mq_gather: null store");
  return gather_impl(cache_tbl, cache_pitch, slot_of, make_store(store, nullptr, 0, store_pitch),
                     ids, n_dev, n_max, d, out, out_pitch, hit_miss, stream, "mq_gather");
}

int mq_gather_sharded(const float* cache_tbl, int32_t cache_pitch, const int32_t* slot_of,
                      const float* const* shards, int32_t n_shards, int32_t store_pitch,
                      const int32_t* ids, const int32_t* n_dev, int32_t n_max, int32_t d,
                      float* out, int32_t out_pitch, unsigned long long* hit_miss,
                      void* stream) {
  MQ_CHECK_ARG(shards && n_shards >= 1 && n_shards <= MQ_MAX_PEERS,
               "mq_gather_sharded: need 1..%d shards", MQ_MAX_PEERS);
  return gather_impl(cache_tbl, cache_pitch, slot_of,
                     make_store(nullptr, shards, n_shards, store_pitch), ids, n_dev, n_max, d, out,
                     out_pitch, hit_miss, stream, "mq_gather_sharded");
}

int mq_gather_labels(const int32_t* all_labels, const int32_t* ids, const int32_t* n_dev,
                     int32_t n_max, int32_t* out, void* stream) {
  MQ_CHECK_ARG(all_labels && ids && n_dev && out, "mq_gather_labels: null pointer");
  if (n_max <= 0) return MQ_OK;
  cudaStream_t s = as_stream(stream);
  {
    ProfScope ps(K_LABELS, s);
    gather_labels_kernel<<<ceil_div(n_max, 256), 256, 0, s>>>(all_labels, ids, n_dev, out);
  }
  MQ_LAUNCH_CHECK("gather_labels");
  return MQ_OK;
}

}  // extern "C"
