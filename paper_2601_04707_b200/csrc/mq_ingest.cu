// Graph ingest on the device: the reference's build_csr
// (mqpipe/graph.py:94-139) and the column narrowing of its MQG1 container
// loader (graph.py:331-395, u64 columns -> int32 here).
//
// build_csr: key = src * n + dst per edge, np.unique (sorted, deduplicated),
// rows = key / n, cols = key % n, row_offsets by counting.  Here:
//   * an LSD radix sort of the u64 keys (8-bit digits, only the passes the
//     key range needs): per pass a digit-major tile histogram, one exclusive
//     scan over it (the decoupled look-back scan of mq_scan.cuh), and a stable
//     scatter in which each warp ranks its keys with __match_any_sync;
//   * dedup as a scan whose store functor compacts the first occurrences;
//   * row_offsets[v] = lower_bound(unique keys, v * n) (no atomics).
// Integer work: the result is bit-identical to the reference's.
#include "mq_scan.cuh"

namespace mq {
namespace ig {

constexpr int kThreads = 256;
constexpr int kPer = 16;                    // keys per thread per tile
constexpr int kTile = kThreads * kPer;      // 4096
constexpr int kWarps = kThreads / 32;
constexpr int kWarpKeys = kTile / kWarps;   // 512 contiguous keys per warp

__global__ void edge_keys_kernel(const int64_t* __restrict__ edges, int64_t m, int64_t n,
                                 unsigned long long* __restrict__ keys, int32_t* __restrict__ bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = edges[2 * i], d = edges[2 * i + 1];
    if (s < 0 || s >= n || d < 0 || d >= n) {
      *bad = 1;
      keys[i] = 0;
    } else {
      keys[i] = (unsigned long long)(s * n + d);
    }
  }
}

// counts[digit * ntiles + tile]
__global__ void __launch_bounds__(kThreads) rs_count_kernel(const unsigned long long* __restrict__ keys,
                                                            int64_t m, int shift, int64_t ntiles,
                                                            int32_t* __restrict__ counts) {
  __shared__ int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTile;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int64_t k = base + i * kThreads + threadIdx.x;
    if (k < m) atomicAdd(&h[(keys[k] >> shift) & 255u], 1);
  }
  __syncthreads();
  counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// stable scatter: warp w owns keys [base + w*512, +512), ranked 32 at a time
__global__ void __launch_bounds__(kThreads) rs_scatter_kernel(
    const unsigned long long* __restrict__ in, unsigned long long* __restrict__ out, int64_t m,
    int shift, int64_t ntiles, const int64_t* __restrict__ offsets) {
  __shared__ int wh[kWarps][256];  // per-warp digit counts, then running positions
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < kWarps * 256; d += kThreads) (&wh[0][0])[d] = 0;
  __syncthreads();
  const int64_t wbase = (int64_t)blockIdx.x * kTile + (int64_t)w * kWarpKeys;
  for (int r = 0; r < kWarpKeys; r += 32) {
    const int64_t k = wbase + r + lane;
    if (k < m) atomicAdd(&wh[w][(in[k] >> shift) & 255u], 1);
  }
  __syncthreads();
  // exclusive prefix over warps per digit, plus the tile's global base
  {
    const int d = threadIdx.x;
    int64_t run = offsets[(int64_t)d * ntiles + blockIdx.x];
    for (int ww = 0; ww < kWarps; ++ww) {
      const int c = wh[ww][d];
      wh[ww][d] = (int)(run - offsets[(int64_t)d * ntiles + blockIdx.x]);  // local start
      run += c;
    }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int r = 0; r < kWarpKeys; r += 32) {
    const int64_t k = wbase + r + lane;
    const bool ok = k < m;
    const unsigned valid = __ballot_sync(0xffffffffu, ok);
    if (valid == 0) break;
    const unsigned long long key = ok ? in[k] : 0ull;
    const int d = (int)((key >> shift) & 255u);
    const unsigned peers = __match_any_sync(0xffffffffu, ok ? d : 256 + lane) & valid;
    if (ok) {
      const int rank = __popc(peers & lt);
      const int64_t pos = offsets[(int64_t)d * ntiles + blockIdx.x] + wh[w][d] + rank;
      out[pos] = key;
    }
    __syncwarp();
    if (ok && (peers & lt) == 0) wh[w][d] += __popc(peers);  // group leader advances
    __syncwarp();
  }
}

struct LoadFirst {  // 1 where the sorted key differs from its predecessor
  const unsigned long long* keys;
  int64_t m;
  __device__ int64_t size() const { return m; }
  __device__ int64_t operator()(int64_t i) const {
    return (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
  }
};
struct StoreUnique {
  const unsigned long long* keys;
  unsigned long long* uniq;
  int64_t* count;
  __device__ void operator()(int64_t i, int64_t excl, int64_t val) const {
    if (val) uniq[excl] = keys[i];
  }
  __device__ void total(int64_t, int64_t t) const { *count = t; }
};

__global__ void csr_rows_kernel(const unsigned long long* __restrict__ uniq, int64_t e, int64_t n,
                                int64_t* __restrict__ row_off) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long target = (unsigned long long)v * (unsigned long long)n;
    int64_t lo = 0, hi = e;  // first index with key >= v * n
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (uniq[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    row_off[v] = lo;
  }
}

__global__ void csr_cols_kernel(const unsigned long long* __restrict__ uniq, int64_t e, int64_t n,
                                int32_t* __restrict__ col) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e;
       i += (int64_t)gridDim.x * blockDim.x)
    col[i] = (int32_t)(uniq[i] % (unsigned long long)n);
}

__global__ void narrow_kernel(const unsigned long long* __restrict__ in, int64_t m, int64_t n,
                              int32_t* __restrict__ out, int32_t* __restrict__ bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long v = in[i];
    if (v >= (unsigned long long)n) *bad = 1;
    out[i] = (int32_t)v;
  }
}

// graph.py:142-149: one-hot of floor(log2(deg + 1)) = bit length of deg+1 - 1
__global__ void degree_buckets_kernel(const int64_t* __restrict__ row_off, int64_t n,
                                      int32_t* __restrict__ bucket) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long x = (unsigned long long)(row_off[v + 1] - row_off[v]) + 1ull;
    bucket[v] = 63 - __clzll(x);
  }
}

inline int grid_for(int64_t n) {
  const int64_t g = (n + kThreads - 1) / kThreads;
  return (int)(g < 1 ? 1 : (g > kNumSMs * 16 ? kNumSMs * 16 : g));
}

inline int key_bits(int64_t n) {  // keys < n * n
  const unsigned long long mx = (unsigned long long)n * (unsigned long long)n;
  int b = 0;
  while (b < 64 && (mx - 1) >> b) ++b;
  return b < 1 ? 1 : b;
}

}  // namespace ig
}  // namespace mq

using namespace mq;

extern "C" {

int64_t mq_build_csr_scratch_bytes(int64_t m) {
  const int64_t ntiles = (m + ig::kTile - 1) / ig::kTile;
  const int64_t nc = 256 * (ntiles < 1 ? 1 : ntiles);
  auto r256 = [](int64_t b) { return (b + 255) / 256 * 256; };
  return r256(8 * (m < 1 ? 1 : m)) * 2 + r256(4 * nc) + r256(8 * (nc + 1)) +
         r256(scan_scratch_bytes(nc > m ? nc : (m < 1 ? 1 : m))) + 256;
}

int mq_build_csr_keys(const int64_t* edges, int64_t m, int64_t n_nodes, void* scratch,
                      unsigned long long* uniq, int64_t* n_unique_dev, int32_t* bad_dev,
                      void* stream) {
  MQ_CHECK_ARG(m >= 0 && n_nodes >= 1 && n_nodes < INT32_MAX, "mq_build_csr_keys: bad sizes");
  MQ_CHECK_ARG(scratch && uniq && n_unique_dev && bad_dev && (m == 0 || edges),
               "mq_build_csr_keys: null pointer");
  cudaStream_t s = as_stream(stream);
  MQ_CUDA(cudaMemsetAsync(bad_dev, 0, sizeof(int32_t), s));
  MQ_CUDA(cudaMemsetAsync(n_unique_dev, 0, sizeof(int64_t), s));
  if (m == 0) return MQ_OK;
  const int64_t ntiles = (m + ig::kTile - 1) / ig::kTile;
  const int64_t nc = 256 * ntiles;
  auto r256 = [](int64_t b) { return (b + 255) / 256 * 256; };
  char* p = static_cast<char*>(scratch);
  auto* ka = reinterpret_cast<unsigned long long*>(p);
  p += r256(8 * m);
  auto* kb = reinterpret_cast<unsigned long long*>(p);
  p += r256(8 * m);
  auto* counts = reinterpret_cast<int32_t*>(p);
  p += r256(4 * nc);
  auto* offsets = reinterpret_cast<int64_t*>(p);
  p += r256(8 * (nc + 1));
  void* scan_scr = p;
  {
    ProfScope ps(K_INGEST, s);
    ig::edge_keys_kernel<<<ig::grid_for(m), ig::kThreads, 0, s>>>(edges, m, n_nodes, ka, bad_dev);
  }
  MQ_LAUNCH_CHECK("edge_keys");
  const int bits = ig::key_bits(n_nodes);
  for (int shift = 0; shift < bits; shift += 8) {
    {
      ProfScope ps(K_INGEST, s);
      ig::rs_count_kernel<<<(int)ntiles, ig::kThreads, 0, s>>>(ka, m, shift, ntiles, counts);
    }
    MQ_LAUNCH_CHECK("rs_count");
    int rc = launch_scan(LoadI32{counts, nullptr, nc}, StoreOffsets<int64_t>{offsets}, nc, scan_scr,
                         s, K_INGEST);
    if (rc) return rc;
    {
      ProfScope ps(K_INGEST, s);
      ig::rs_scatter_kernel<<<(int)ntiles, ig::kThreads, 0, s>>>(ka, kb, m, shift, ntiles, offsets);
    }
    MQ_LAUNCH_CHECK("rs_scatter");
    unsigned long long* t = ka;
    ka = kb;
    kb = t;
  }
  return launch_scan(ig::LoadFirst{ka, m}, ig::StoreUnique{ka, uniq, n_unique_dev}, m, scan_scr, s,
                     K_INGEST);
}

int mq_build_csr_finish(const unsigned long long* uniq, int64_t n_unique, int64_t n_nodes,
                        int64_t* row_off, int32_t* col, void* stream) {
  MQ_CHECK_ARG(n_unique >= 0 && n_nodes >= 1 && row_off && (n_unique == 0 || (uniq && col)),
               "mq_build_csr_finish: bad arguments");
  cudaStream_t s = as_stream(stream);
  {
    ProfScope ps(K_INGEST, s);
    ig::csr_rows_kernel<<<ig::grid_for(n_nodes + 1), ig::kThreads, 0, s>>>(uniq, n_unique, n_nodes,
                                                                           row_off);
    if (n_unique)
      ig::csr_cols_kernel<<<ig::grid_for(n_unique), ig::kThreads, 0, s>>>(uniq, n_unique, n_nodes,
                                                                          col);
  }
  MQ_LAUNCH_CHECK("csr_finish");
  return MQ_OK;
}

int mq_narrow_cols(const unsigned long long* cols64, int64_t m, int64_t n_nodes, int32_t* cols32,
                   int32_t* bad_dev, void* stream) {
  MQ_CHECK_ARG(m >= 0 && n_nodes >= 1 && n_nodes <= INT32_MAX && bad_dev &&
                   (m == 0 || (cols64 && cols32)),
               "mq_narrow_cols: bad arguments");
  cudaStream_t s = as_stream(stream);
  MQ_CUDA(cudaMemsetAsync(bad_dev, 0, sizeof(int32_t), s));
  if (m == 0) return MQ_OK;
  {
    ProfScope ps(K_INGEST, s);
    ig::narrow_kernel<<<ig::grid_for(m), ig::kThreads, 0, s>>>(cols64, m, n_nodes, cols32, bad_dev);
  }
  MQ_LAUNCH_CHECK("narrow_cols");
  return MQ_OK;
}

int mq_degree_buckets(const int64_t* row_off, int64_t n_nodes, int32_t* bucket, void* stream) {
  MQ_CHECK_ARG(n_nodes >= 0 && (n_nodes == 0 || (row_off && bucket)), "mq_degree_buckets: bad arguments");
  if (n_nodes == 0) return MQ_OK;
  cudaStream_t s = as_stream(stream);
  {
    ProfScope ps(K_INGEST, s);
    ig::degree_buckets_kernel<<<ig::grid_for(n_nodes), ig::kThreads, 0, s>>>(row_off, n_nodes,
                                                                             bucket);
  }
  MQ_LAUNCH_CHECK("degree_buckets");
  return MQ_OK;
}

}  // extern "C"
