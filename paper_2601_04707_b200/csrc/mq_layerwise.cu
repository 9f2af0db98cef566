// Layer-wise samplers on the device: LADIES and FastGCN with
// the flat / debias / with-replacement forms, and the GCN arm of the
// node-wise block.
//
// Reference (mqpipe/samplers.py):
//   _restricted_rows        :247-262  rows of D^-1/2 (A+I) D^-1/2 for prev,
//                                     the loop injected at its sorted place
//   ladies_candidates       :265-271  sorted unique neighbours of prev
//   _candidate_norms        :274-283  per-candidate sum of squared entries
//                                     (np.add.at: entry order)
//   ladies/flat/fastgcn     :286-318  norms / pairwise total
//   weighted WOR            :113-135  keys u^(1/w), (key desc, index asc)
//   debias_coefficients     :353-373  sequential f64 recursion
//   _layer_wise_block       :376-440  slice, scale, row normalisation
//   sample_ladies/fastgcn   :443-495
//   node_wise_block (gcn)   :178-191
//
// Injected draws (oracle/layerwise.py, the layer contract): layer l of batch
// b draws uniforms random(n)[i] from the Philox stream (seed, epoch; ctr
// (i, 0xFFFFFFFF, l, b)); the with-replacement arm is NumPy's choice(p)
// algorithm over them: cdf = cumsum(p) (sequential), cdf /= cdf[-1],
// searchsorted(cdf, u, 'right').
//
// Bit-exactness: the f64 Laplacian entries are 1/sqrt(dh_v * dh_c) with _rn
// operations; the per-candidate sums run sequentially in entry order (a
// stable radix sort of the entries by candidate keeps np.add.at's order);
// the normalising total replays NumPy's pairwise tree (mq_refresh.cu); the
// WOR keys use the device f64 pow (one-ulp hazard as in the cache refresh).
//
// The entry points are host-orchestrated and synchronise their stream (the
// candidate count, the positive count and the unique-draw count size the
// next steps), like the reference API they replace; temporaries come from
// the stream-ordered allocator.
#include <vector>

#include <cub/cub.cuh>

#include "mq_scan.cuh"

namespace mq {

int pairwise_total(const double* a, int64_t n, double* total, cudaStream_t s);

namespace lw {

constexpr uint32_t kRow = 0xFFFFFFFFu;
constexpr int kT = 256;

__host__ __device__ __forceinline__ double layer_uniform(uint32_t seed, uint32_t epoch,
                                                         uint32_t batch, uint32_t layer,
                                                         uint32_t i) {
  const U4 x = philox4x32_10(U4{i, kRow, layer, batch}, seed, epoch);
  return ((double)(x.x >> 5) * 67108864.0 + (double)(x.y >> 6)) / 9007199254740992.0;
}

struct Graph {
  const int64_t* row_off;  // loops stripped
  const int32_t* col;
  const int32_t* loops;    // stored self loops per node (nullptr: none)
  __device__ int64_t stripped(int v) const { return row_off[v + 1] - row_off[v]; }
  __device__ int nloop(int v) const { return loops ? loops[v] : 0; }
  // loop entries of a restricted row: the stored ones, or the injected one
  __device__ int loop_copies(int v) const {
    const int k = nloop(v);
    return k > 0 ? k : 1;
  }
  // a_hat_degrees (graph.py:53-60): stored degree, +1 unless a loop is stored
  __device__ double deg_hat(int v) const { return (double)(stripped(v) + loop_copies(v)); }
  __device__ int64_t deg_hat_i(int v) const { return stripped(v) + loop_copies(v); }
};

inline int grid_for(int64_t n, int per = kT) {
  const int64_t g = (n + per - 1) / per;
  return (int)(g < 1 ? 1 : (g > kNumSMs * 16 ? kNumSMs * 16 : g));
}

// the device's default pool keeps freed blocks (the calls synchronise their
// stream; a zero release threshold would unmap the pool at every sync)
inline void keep_pool() {
  static bool done = false;
  if (done) return;
  done = true;
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  (void)cudaGetLastError();
}

// stream-ordered temporaries, freed at scope exit
struct Tmp {
  cudaStream_t s;
  std::vector<void*> ptrs;
  explicit Tmp(cudaStream_t st) : s(st) { keep_pool(); }
  ~Tmp() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
  template <class T>
  T* get(int64_t n) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, (size_t)(n < 1 ? 1 : n) * sizeof(T), s) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
};

// ---- restricted rows -----------------------------------------------------
struct LoadRowLen {
  Graph g;
  const int32_t* prev;
  int64_t n;
  __device__ int64_t size() const { return n; }
  __device__ int64_t operator()(int64_t r) const {
    const int v = prev[r];
    return g.stripped(v) + g.loop_copies(v);
  }
};

// p[r] = #stripped neighbours of prev[r] below prev[r] (rows are sorted):
// where the loop entries go
__global__ void loop_pos_kernel(Graph g, const int32_t* __restrict__ prev, int n_prev,
                                int64_t* __restrict__ lpos) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_prev; r += gridDim.x * blockDim.x) {
    const int v = prev[r];
    int64_t lo = g.row_off[v], hi = g.row_off[v + 1];
    const int64_t a = lo;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (g.col[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    lpos[r] = lo - a;
  }
}

// thread per restricted entry (hub rows spread over the grid): row by binary
// search in roff; entries in sorted column order with the loop entries at
// v's sorted place; rrow, rcol, rval (f64); candidate flags of stored entries
__global__ void restricted_kernel(Graph g, const int32_t* __restrict__ prev, int n_prev,
                                  const int64_t* __restrict__ roff, const int64_t* __restrict__ lpos,
                                  int64_t ne, int32_t* __restrict__ rrow, int32_t* __restrict__ rcol,
                                  double* __restrict__ rval, uint8_t* __restrict__ flag) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = n_prev;  // last r with roff[r] <= e
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (roff[mid] <= e) lo = mid;
      else hi = mid;
    }
    const int r = lo, v = prev[r];
    const int64_t i = e - roff[r], p = lpos[r];
    const int lc = g.loop_copies(v);
    const double dv = g.deg_hat(v);
    int c;
    if (i < p) c = g.col[g.row_off[v] + i];
    else if (i < p + lc) c = v;
    else c = g.col[g.row_off[v] + i - lc];
    rrow[e] = r;
    rcol[e] = c;
    rval[e] = __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(dv, g.deg_hat(c))));
    if (flag && (c != v || g.nloop(v) > 0)) flag[c] = 1;
  }
}

// candidates = flagged nodes in id order; pos[node] = candidate index or -1;
// the flags are cleared for the next call
struct LoadFlag {
  const uint8_t* flag;
  int64_t n;
  __device__ int64_t size() const { return n; }
  __device__ int64_t operator()(int64_t i) const { return flag[i] ? 1 : 0; }
};
struct StoreCand {
  uint8_t* flag;
  int32_t* cand;
  int32_t* pos;
  int64_t* count;
  __device__ void operator()(int64_t i, int64_t excl, int64_t val) const {
    pos[i] = val ? (int32_t)excl : -1;
    if (val) {
      cand[excl] = (int32_t)i;
      flag[i] = 0;
    }
  }
  __device__ void total(int64_t, int64_t t) const { *count = t; }
};

// ---- column norms ----------------------------------------------------------
__global__ void norm_keys_kernel(const int32_t* __restrict__ rcol, const double* __restrict__ rval,
                                 int64_t ne, const int32_t* __restrict__ pos, int32_t n_cand,
                                 uint32_t* __restrict__ key, double* __restrict__ sq) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = rcol[e];
    const int p = pos ? pos[c] : c;
    key[e] = p >= 0 ? (uint32_t)p : (uint32_t)n_cand;
    sq[e] = __dmul_rn(rval[e], rval[e]);
  }
}

__global__ void seg_bounds_kernel(const uint32_t* __restrict__ key, int64_t ne, uint32_t n_cand,
                                  int64_t* __restrict__ lo, int64_t* __restrict__ hi) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = key[e];
    if (k >= n_cand) continue;
    if (e == 0 || key[e - 1] != k) lo[k] = e;
    if (e == ne - 1 || key[e + 1] != k) hi[k] = e + 1;
  }
}

// np.add.at(col_sq, pos, vals**2): per candidate, sequential in entry order
__global__ void seg_sum_kernel(const double* __restrict__ sq, const int64_t* __restrict__ lo,
                               const int64_t* __restrict__ hi, int32_t n_cand, int flat,
                               double* __restrict__ out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n_cand;
       p += (int64_t)gridDim.x * blockDim.x) {
    // sequential in entry order (np.add.at), 16 loads in flight: a hub
    // candidate's chain costs its adds, not one memory latency per entry
    double acc = 0.0;
    int64_t e = lo[p];
    const int64_t e1 = hi[p];
    for (; e + 16 <= e1; e += 16) {
      double t[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) t[u] = __ldg(&sq[e + u]);
#pragma unroll
      for (int u = 0; u < 16; ++u) acc = __dadd_rn(acc, t[u]);
    }
    for (; e < e1; ++e) acc = __dadd_rn(acc, sq[e]);
    out[p] = flat ? __dsqrt_rn(acc) : acc;
  }
}

__global__ void normalize_kernel(const double* __restrict__ x, const double* __restrict__ total,
                                 int64_t n, double* __restrict__ probs, int32_t* __restrict__ bad) {
  const double t = *total;
  if (blockIdx.x == 0 && threadIdx.x == 0 && !(t > 0.0)) *bad = 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    probs[i] = __ddiv_rn(x[i], t);
}

// ---- draws -----------------------------------------------------------------
// WOR keys over the positive probabilities (rank among positives indexes u)
struct LoadPos {
  const double* p;
  int64_t n;
  __device__ int64_t size() const { return n; }
  __device__ int64_t operator()(int64_t i) const { return p[i] > 0.0 ? 1 : 0; }
};
struct StoreKey {
  const double* p;
  uint32_t seed, epoch, batch, layer;
  unsigned long long* skey;
  int32_t* idx;
  int64_t* positive;
  __device__ void operator()(int64_t i, int64_t excl, int64_t val) const {
    unsigned long long k = 0;
    if (val) {
      const double u = layer_uniform(seed, epoch, batch, layer, (uint32_t)excl);
      const double key = pow(u, __ddiv_rn(1.0, p[i]));
      k = (unsigned long long)__double_as_longlong(key) + 1ull;  // 0 = not eligible
    }
    skey[i] = k;
    idx[i] = (int32_t)i;
  }
  __device__ void total(int64_t, int64_t t) const { *positive = t; }
};

__global__ void iota_kernel(int32_t* __restrict__ a, int32_t n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

// cdf = cumsum(p) (sequential, as np.cumsum), then cdf /= cdf[-1]
__global__ void cumsum_kernel(const double* __restrict__ p, int64_t n, double* __restrict__ cdf) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double acc = 0.0;  // np.cumsum's sequential order; loads batched 16 ahead
  int64_t i = 0;
  for (; i + 16 <= n; i += 16) {
    double t[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) t[u] = __ldg(&p[i + u]);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      acc = __dadd_rn(acc, t[u]);
      cdf[i + u] = acc;
    }
  }
  for (; i < n; ++i) {
    acc = __dadd_rn(acc, p[i]);
    cdf[i] = acc;
  }
}
__global__ void cdf_scale_kernel(double* __restrict__ cdf, int64_t n) {
  const double last = cdf[n - 1];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n - 1;
       i += (int64_t)gridDim.x * blockDim.x)
    cdf[i] = __ddiv_rn(cdf[i], last);
}
__global__ void cdf_last_kernel(double* __restrict__ cdf, int64_t n) {
  if (blockIdx.x == 0 && threadIdx.x == 0) cdf[n - 1] = __ddiv_rn(cdf[n - 1], cdf[n - 1]);
}

// idx_j = searchsorted(cdf, u_j, 'right') = #{cdf <= u_j}
__global__ void draw_replace_kernel(const double* __restrict__ cdf, int64_t n, int32_t s,
                                    uint32_t seed, uint32_t epoch, uint32_t batch, uint32_t layer,
                                    int32_t* __restrict__ out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < s; j += gridDim.x * blockDim.x) {
    const double u = layer_uniform(seed, epoch, batch, layer, (uint32_t)j);
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (cdf[mid] <= u) lo = mid + 1;
      else hi = mid;
    }
    out[j] = (int32_t)(lo < n ? lo : n - 1);
  }
}

// debias_coefficients (samplers.py:353-373) over the draw order, one thread
__global__ void debias_kernel(const double* __restrict__ probs, const int32_t* __restrict__ order,
                              int32_t s, int64_t n, double* __restrict__ alpha,
                              double* __restrict__ beta, double* __restrict__ coef) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (int i = 0; i < s; ++i)
    alpha[i] = i == 0 ? 1.0 : __ddiv_rn((double)n, (double)((n - i) * (int64_t)(i + 1)));
  double tail = 1.0;
  for (int i = s - 1; i >= 0; --i) {
    beta[i] = __dmul_rn(alpha[i], tail);
    tail = __dmul_rn(tail, __dsub_rn(1.0, alpha[i]));
  }
  // beta_suffix[i] = beta[s-1] + ... + beta[i+1] (cumsum of the reversed betas)
  double suffix = 0.0, cs = 0.0;
  double* later = alpha;  // alpha is no longer needed: reuse it for the suffix sums
  for (int i = s - 1; i >= 0; --i) {
    later[i] = i == s - 1 ? 0.0 : suffix;
    suffix = i == s - 1 ? beta[i] : __dadd_rn(suffix, beta[i]);
  }
  for (int i = 0; i < s; ++i) {
    const double p = probs[order[i]];
    const double left = __dsub_rn(1.0, cs);  // 1 - cumsum(probs[:i])
    const double at_draw = __ddiv_rn(p, left);
    coef[i] = __dadd_rn(__ddiv_rn(beta[i], at_draw), later[i]);
    cs = i == 0 ? p : __dadd_rn(cs, p);
  }
}

// per picked column j (ascending candidate index): src id, base probability
// and the entry scale of the estimator
__global__ void scale_kernel(int mode, const int32_t* __restrict__ pick,
                             const int32_t* __restrict__ aux, int32_t n_pick, int32_t s,
                             const double* __restrict__ probs, const int32_t* __restrict__ cand,
                             const double* __restrict__ coef, int32_t* __restrict__ src_ids,
                             double* __restrict__ sample_probs, double* __restrict__ scale) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_pick; j += gridDim.x * blockDim.x) {
    const int i = pick[j];
    const double p = probs[i];
    src_ids[j] = cand ? cand[i] : i;
    sample_probs[j] = p;
    if (mode == 0)  // WOR: 1 / (s p)
      scale[j] = __ddiv_rn(1.0, __dmul_rn((double)s, p));
    else if (mode == 1)  // with replacement: count / (s p)
      scale[j] = __ddiv_rn((double)aux[j], __dmul_rn((double)s, p));
    else  // debias: the draw's coefficient
      scale[j] = coef[aux[j]];
  }
}

// ---- slice ------------------------------------------------------------------
__device__ __forceinline__ int find_sorted(const int32_t* __restrict__ a, int n, int x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < n && a[lo] == x ? lo : -1;
}
struct LoadKeep {
  const int32_t* rcol;
  const int32_t* src;
  int32_t n_src;
  int64_t n;
  __device__ int64_t size() const { return n; }
  __device__ int64_t operator()(int64_t e) const { return find_sorted(src, n_src, rcol[e]) >= 0; }
};
struct StoreSlice {
  const int32_t* rrow;
  const int32_t* rcol;
  const double* rval;
  const int64_t* roff;
  const int32_t* src;
  int32_t n_src;
  const double* scale;
  int32_t* rows;
  int32_t* cols;
  double* values;
  int32_t* row_ptr;
  int32_t n_prev;
  int64_t* nnz;
  __device__ void operator()(int64_t e, int64_t excl, int64_t val) const {
    const int r = rrow[e];
    if (roff[r] == e) row_ptr[r] = (int32_t)excl;
    if (val) {
      const int j = find_sorted(src, n_src, rcol[e]);
      rows[excl] = r;
      cols[excl] = j;
      values[excl] = __dmul_rn(rval[e], scale[j]);
    }
  }
  __device__ void total(int64_t, int64_t t) const {
    row_ptr[n_prev] = (int32_t)t;
    *nnz = t;
  }
};

// effective values: row-normalised (np.add.at row sums, entry order) or a copy
__global__ void effective_kernel(int normalize, const int32_t* __restrict__ row_ptr, int32_t n_prev,
                                 const double* __restrict__ values, double* __restrict__ eff) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_prev; r += gridDim.x * blockDim.x) {
    const int a = row_ptr[r], b = row_ptr[r + 1];
    if (!normalize) {
      for (int e = a; e < b; ++e) eff[e] = values[e];
      continue;
    }
    double sum = 0.0;
    for (int e = a; e < b; ++e) sum = __dadd_rn(sum, values[e]);
    const double div = sum > 0.0 ? sum : 1.0;
    for (int e = a; e < b; ++e) eff[e] = __ddiv_rn(values[e], div);
  }
}

// ---- LADIES target filter ------------------------------------------------
struct LoadLive {
  Graph g;
  const int32_t* t;
  int64_t n;
  __device__ int64_t size() const { return n; }
  __device__ int64_t operator()(int64_t i) const {
    const int v = t[i];
    return g.stripped(v) + g.nloop(v) > 0 ? 1 : 0;
  }
};
struct StoreLive {
  const int32_t* t;
  int32_t* out;
  int64_t* count;
  __device__ void operator()(int64_t i, int64_t excl, int64_t val) const {
    if (val) out[excl] = t[i];
  }
  __device__ void total(int64_t, int64_t tt) const { *count = tt; }
};

// ---- GCN arm of the node-wise block ------------------------------------------
// row r of the SAGE block (same draws) -> (r, r, 1/dh_v), then its sampled
// entries with (n/s) / sqrt(dh_v dh_u) (samplers.py:178-191)
__global__ void gcn_block_kernel(Graph g, const int32_t* __restrict__ dst,
                                 const int32_t* __restrict__ src_ids,
                                 const int32_t* __restrict__ row_ptr,
                                 const int32_t* __restrict__ cols, int32_t n_dst,
                                 int32_t* __restrict__ row_ptr_out, int32_t* __restrict__ rows_out,
                                 int32_t* __restrict__ cols_out, double* __restrict__ vals_out) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r <= n_dst; r += gridDim.x * blockDim.x) {
    if (r == n_dst) {
      row_ptr_out[n_dst] = row_ptr[n_dst] + n_dst;
      continue;
    }
    const int v = dst[r];
    const int a = row_ptr[r], b = row_ptr[r + 1], s = b - a;
    const int o = a + r;
    row_ptr_out[r] = o;
    const int64_t dv = g.deg_hat_i(v);
    rows_out[o] = r;
    cols_out[o] = r;
    vals_out[o] = __ddiv_rn(1.0, (double)dv);
    const double scale = s ? __ddiv_rn((double)g.stripped(v), (double)s) : 0.0;
    for (int k = 0; k < s; ++k) {
      const int c = cols[a + k];
      const int u = src_ids[c];
      rows_out[o + 1 + k] = r;
      cols_out[o + 1 + k] = c;
      vals_out[o + 1 + k] = __ddiv_rn(scale, __dsqrt_rn((double)(dv * g.deg_hat_i(u))));
    }
  }
}

inline int bits_for(uint64_t n) {
  int b = 1;
  while (b < 64 && (1ull << b) <= n) ++b;
  return b;
}

}  // namespace lw
}  // namespace mq

using namespace mq;

#define MQ_TMP(T, name, n)                                            \
  T* name = tmp.get<T>(n);                                            \
  MQ_CHECK_ARG(name != nullptr, "layer-wise sampler: out of device memory")

#define MQ_SAMPLING_ERROR(msg)                                        \
  do {                                                                \
    ::mq::set_error("%s", msg);                                       \
    return MQ_ERR_SAMPLING;                                           \
  } while (0)

extern "C" {

int mq_layer_entries(const int64_t* row_off, const int32_t* loops, const int32_t* prev,
                     int32_t n_prev, int64_t* roff, void* scratch, void* stream) {
  MQ_CHECK_ARG(row_off && prev && roff && scratch && n_prev >= 0, "mq_layer_entries: bad arguments");
  cudaStream_t s = as_stream(stream);
  lw::Graph g{row_off, nullptr, loops};
  return launch_scan(lw::LoadRowLen{g, prev, n_prev}, StoreOffsets<int64_t>{roff}, n_prev < 1 ? 1 : n_prev,
                     scratch, s, K_LAYERWISE);
}

int64_t mq_layer_scratch_bytes(int64_t n_max) { return scan_scratch_bytes(n_max < 1 ? 1 : n_max); }

int mq_layer_live_targets(const int64_t* row_off, const int32_t* loops, const int32_t* targets,
                          int32_t n, int32_t* out, int64_t* count_dev, void* scratch, void* stream) {
  MQ_CHECK_ARG(row_off && targets && out && count_dev && scratch && n >= 0,
               "mq_layer_live_targets: bad arguments");
  lw::Graph g{row_off, nullptr, loops};
  return launch_scan(lw::LoadLive{g, targets, n}, lw::StoreLive{targets, out, count_dev},
                     n < 1 ? 1 : n, scratch, as_stream(stream), K_LAYERWISE);
}

int mq_layer_fastgcn_probs(const int64_t* row_off, const int32_t* col, const int32_t* loops,
                           int64_t n_nodes, int32_t flat, double* probs, double* cdf,
                           void* stream) {
  MQ_CHECK_ARG(row_off && col && probs && n_nodes > 0 && n_nodes < INT32_MAX,
               "mq_layer_fastgcn_probs: bad arguments");
  cudaStream_t s = as_stream(stream);
  lw::Tmp tmp(s);
  lw::Graph g{row_off, col, loops};
  // every node is a row and a candidate: entries of all rows (prev = 0..n-1)
  MQ_TMP(int32_t, prev, n_nodes);
  lw::iota_kernel<<<lw::grid_for(n_nodes), lw::kT, 0, s>>>(prev, (int32_t)n_nodes);
  MQ_TMP(int64_t, roff, n_nodes + 1);
  MQ_TMP(char, scr, scan_scratch_bytes(n_nodes));
  int rc = launch_scan(lw::LoadRowLen{g, prev, n_nodes}, StoreOffsets<int64_t>{roff}, n_nodes, scr,
                       s, K_LAYERWISE);
  if (rc) return rc;
  int64_t ne = 0;
  MQ_CUDA(cudaMemcpyAsync(&ne, roff + n_nodes, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  MQ_CUDA(cudaStreamSynchronize(s));
  MQ_TMP(int32_t, rrow, ne);
  MQ_TMP(int32_t, rcol, ne);
  MQ_TMP(double, rval, ne);
  MQ_TMP(int64_t, lpos, n_nodes);
  {
    ProfScope ps(K_LAYERWISE, s);
    lw::loop_pos_kernel<<<lw::grid_for(n_nodes), lw::kT, 0, s>>>(g, prev, (int32_t)n_nodes, lpos);
    lw::restricted_kernel<<<lw::grid_for(ne), lw::kT, 0, s>>>(g, prev, (int32_t)n_nodes, roff, lpos,
                                                             ne, rrow, rcol, rval, nullptr);
  }
  MQ_LAUNCH_CHECK("restricted");
  MQ_TMP(uint32_t, key, ne);
  MQ_TMP(uint32_t, key2, ne);
  MQ_TMP(double, sq, ne);
  MQ_TMP(double, sq2, ne);
  lw::norm_keys_kernel<<<lw::grid_for(ne), lw::kT, 0, s>>>(rcol, rval, ne, nullptr, (int32_t)n_nodes,
                                                          key, sq);
  size_t tb = 0;
  MQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, sq, sq2, ne, 0,
                                          lw::bits_for((uint64_t)n_nodes), s));
  MQ_TMP(char, cubt, (int64_t)tb);
  MQ_CUDA(cub::DeviceRadixSort::SortPairs(cubt, tb, key, key2, sq, sq2, ne, 0,
                                          lw::bits_for((uint64_t)n_nodes), s));
  MQ_TMP(int64_t, lo, n_nodes);
  MQ_TMP(int64_t, hi, n_nodes);
  MQ_CUDA(cudaMemsetAsync(lo, 0, sizeof(int64_t) * n_nodes, s));
  MQ_CUDA(cudaMemsetAsync(hi, 0, sizeof(int64_t) * n_nodes, s));
  MQ_TMP(double, x, n_nodes);
  MQ_TMP(double, total, 1);
  MQ_TMP(int32_t, bad, 1);
  MQ_CUDA(cudaMemsetAsync(bad, 0, sizeof(int32_t), s));
  {
    ProfScope ps(K_LAYERWISE, s);
    lw::seg_bounds_kernel<<<lw::grid_for(ne), lw::kT, 0, s>>>(key2, ne, (uint32_t)n_nodes, lo, hi);
    lw::seg_sum_kernel<<<lw::grid_for(n_nodes), lw::kT, 0, s>>>(sq2, lo, hi, (int32_t)n_nodes, flat,
                                                               x);
  }
  MQ_LAUNCH_CHECK("fastgcn_norms");
  rc = pairwise_total(x, n_nodes, total, s);
  if (rc) return rc;
  lw::normalize_kernel<<<lw::grid_for(n_nodes), lw::kT, 0, s>>>(x, total, n_nodes, probs, bad);
  MQ_LAUNCH_CHECK("fastgcn_normalize");
  if (cdf) {
    lw::cumsum_kernel<<<1, 1, 0, s>>>(probs, n_nodes, cdf);
    lw::cdf_scale_kernel<<<lw::grid_for(n_nodes), lw::kT, 0, s>>>(cdf, n_nodes);
    lw::cdf_last_kernel<<<1, 1, 0, s>>>(cdf, n_nodes);
    MQ_LAUNCH_CHECK("fastgcn_cdf");
  }
  return MQ_OK;
}

int mq_layer_block(const int64_t* row_off, const int32_t* col, const int32_t* loops,
                   int64_t n_nodes, const int32_t* prev, int32_t n_prev, const int64_t* roff,
                   int64_t n_entries, const double* probs_global, const double* cdf_global,
                   int32_t flat, int32_t mode, int32_t budget, uint64_t seed, uint64_t epoch,
                   uint32_t batch, uint32_t layer, uint8_t* node_flags, int32_t* node_pos,
                   int32_t* rows, int32_t* cols, double* values, double* effective,
                   int32_t* row_ptr, int32_t* src_ids, double* sample_probs, int64_t* counts,
                   void* stream) {
  MQ_CHECK_ARG(row_off && col && prev && roff && rows && cols && values && effective && row_ptr &&
                   src_ids && sample_probs && counts,
               "mq_layer_block: null pointer");
  MQ_CHECK_ARG(n_nodes > 0 && n_nodes < INT32_MAX && n_prev > 0 && n_entries >= n_prev &&
                   n_entries < INT32_MAX && budget >= 0 && mode >= 0 && mode <= 2,
               "mq_layer_block: bad sizes or mode");
  MQ_CHECK_ARG(probs_global || (node_flags && node_pos),
               "mq_layer_block: LADIES needs the node flag / position tables");
  MQ_CHECK_ARG(!(mode == 1 && probs_global && !cdf_global),
               "mq_layer_block: FastGCN with replacement needs its cdf");
  cudaStream_t s = as_stream(stream);
  lw::Tmp tmp(s);
  lw::Graph g{row_off, col, loops};
  const int64_t ne = n_entries;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)epoch;
  MQ_TMP(int32_t, rrow, ne);
  MQ_TMP(int32_t, rcol, ne);
  MQ_TMP(double, rval, ne);
  MQ_TMP(char, scr, scan_scratch_bytes(n_nodes > ne ? n_nodes : ne));
  MQ_TMP(int64_t, hc, 4);  // n_cand, positive, nnz, n_uniq
  MQ_TMP(int64_t, lpos, n_prev);
  {
    ProfScope ps(K_LAYERWISE, s);
    lw::loop_pos_kernel<<<lw::grid_for(n_prev), lw::kT, 0, s>>>(g, prev, n_prev, lpos);
    lw::restricted_kernel<<<lw::grid_for(ne), lw::kT, 0, s>>>(
        g, prev, n_prev, roff, lpos, ne, rrow, rcol, rval, probs_global ? nullptr : node_flags);
  }
  MQ_LAUNCH_CHECK("restricted");

  // ---- candidates and their probabilities
  int64_t n_cand = n_nodes;
  const int32_t* cand = nullptr;
  const double* probs = probs_global;
  if (!probs_global) {
    MQ_TMP(int32_t, cbuf, ne);
    int rc = launch_scan(lw::LoadFlag{node_flags, n_nodes},
                         lw::StoreCand{node_flags, cbuf, node_pos, hc}, n_nodes, scr, s, K_LAYERWISE);
    if (rc) return rc;
    MQ_CUDA(cudaMemcpyAsync(&n_cand, hc, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MQ_CUDA(cudaStreamSynchronize(s));
    if (n_cand == 0) MQ_SAMPLING_ERROR("empty candidate set");
    cand = cbuf;
    MQ_TMP(uint32_t, key, ne);
    MQ_TMP(uint32_t, key2, ne);
    MQ_TMP(double, sq, ne);
    MQ_TMP(double, sq2, ne);
    lw::norm_keys_kernel<<<lw::grid_for(ne), lw::kT, 0, s>>>(rcol, rval, ne, node_pos,
                                                            (int32_t)n_cand, key, sq);
    size_t tb = 0;
    const int nb = lw::bits_for((uint64_t)n_cand);
    MQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, sq, sq2, ne, 0, nb, s));
    MQ_TMP(char, cubt, (int64_t)tb);
    MQ_CUDA(cub::DeviceRadixSort::SortPairs(cubt, tb, key, key2, sq, sq2, ne, 0, nb, s));
    MQ_TMP(int64_t, lo, n_cand);
    MQ_TMP(int64_t, hi, n_cand);
    MQ_CUDA(cudaMemsetAsync(lo, 0, sizeof(int64_t) * n_cand, s));
    MQ_CUDA(cudaMemsetAsync(hi, 0, sizeof(int64_t) * n_cand, s));
    MQ_TMP(double, x, n_cand);
    MQ_TMP(double, total, 1);
    MQ_TMP(int32_t, bad, 1);
    MQ_TMP(double, pbuf, n_cand);
    MQ_CUDA(cudaMemsetAsync(bad, 0, sizeof(int32_t), s));
    {
      ProfScope ps(K_LAYERWISE, s);
      lw::seg_bounds_kernel<<<lw::grid_for(ne), lw::kT, 0, s>>>(key2, ne, (uint32_t)n_cand, lo, hi);
      lw::seg_sum_kernel<<<lw::grid_for(n_cand), lw::kT, 0, s>>>(sq2, lo, hi, (int32_t)n_cand, flat, x);
    }
    MQ_LAUNCH_CHECK("layer_norms");
    rc = pairwise_total(x, n_cand, total, s);
    if (rc) return rc;
    lw::normalize_kernel<<<lw::grid_for(n_cand), lw::kT, 0, s>>>(x, total, n_cand, pbuf, bad);
    MQ_LAUNCH_CHECK("layer_normalize");
    int32_t hbad = 0;
    MQ_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    MQ_CUDA(cudaStreamSynchronize(s));
    if (hbad) MQ_SAMPLING_ERROR("all candidate columns have zero norm");
    probs = pbuf;
  }

  // ---- draws: picked candidate indices, ascending (pick), with aux =
  // draw rank (debias) or draw count (with replacement)
  int32_t n_pick = 0, s_draw = 0;
  int32_t* pick = nullptr;
  int32_t* aux = nullptr;
  double* coef = nullptr;
  if (mode == 1) {
    s_draw = budget;
    const double* cdf = cdf_global;
    if (!cdf) {
      MQ_TMP(double, cbuf, n_cand);
      lw::cumsum_kernel<<<1, 1, 0, s>>>(probs, n_cand, cbuf);
      lw::cdf_scale_kernel<<<lw::grid_for(n_cand), lw::kT, 0, s>>>(cbuf, n_cand);
      lw::cdf_last_kernel<<<1, 1, 0, s>>>(cbuf, n_cand);
      MQ_LAUNCH_CHECK("layer_cdf");
      cdf = cbuf;
    }
    MQ_TMP(int32_t, d, budget);
    MQ_TMP(int32_t, d2, budget);
    MQ_TMP(int32_t, uq, budget);
    MQ_TMP(int32_t, cnt, budget);
    MQ_TMP(int32_t, nu, 1);
    if (budget > 0) {
      lw::draw_replace_kernel<<<lw::grid_for(budget), lw::kT, 0, s>>>(cdf, n_cand, budget, k0, k1,
                                                                     batch, layer, d);
      MQ_LAUNCH_CHECK("layer_draw");
      size_t tb = 0, tb2 = 0;
      const int nb = lw::bits_for((uint64_t)n_cand);
      MQ_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, d, d2, budget, 0, nb, s));
      MQ_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tb2, d2, uq, cnt, nu, budget, s));
      MQ_TMP(char, cubt, (int64_t)(tb > tb2 ? tb : tb2));
      MQ_CUDA(cub::DeviceRadixSort::SortKeys(cubt, tb, d, d2, budget, 0, nb, s));
      MQ_CUDA(cub::DeviceRunLengthEncode::Encode(cubt, tb2, d2, uq, cnt, nu, budget, s));
      MQ_CUDA(cudaMemcpyAsync(&n_pick, nu, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      MQ_CUDA(cudaStreamSynchronize(s));
    }
    pick = uq;
    aux = cnt;
  } else {
    MQ_TMP(unsigned long long, skey, n_cand);
    MQ_TMP(unsigned long long, skey2, n_cand);
    MQ_TMP(int32_t, idx, n_cand);
    MQ_TMP(int32_t, idx2, n_cand);
    int rc = launch_scan(lw::LoadPos{probs, n_cand},
                         lw::StoreKey{probs, k0, k1, batch, layer, skey, idx, hc + 1}, n_cand, scr, s,
                         K_LAYERWISE);
    if (rc) return rc;
    size_t tb = 0;
    MQ_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, skey, skey2, idx, idx2, n_cand,
                                                      0, 64, s));
    MQ_TMP(char, cubt, (int64_t)tb);
    MQ_CUDA(cub::DeviceRadixSort::SortPairsDescending(cubt, tb, skey, skey2, idx, idx2, n_cand, 0,
                                                      64, s));
    int64_t positive = 0;
    MQ_CUDA(cudaMemcpyAsync(&positive, hc + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MQ_CUDA(cudaStreamSynchronize(s));
    s_draw = (int32_t)(budget < positive ? budget : positive);
    n_pick = s_draw;
    // idx2[0..s) = draw order; ascending candidate index with the draw rank
    MQ_TMP(int32_t, rank, s_draw);
    MQ_TMP(int32_t, pk, s_draw);
    MQ_TMP(int32_t, rk, s_draw);
    if (s_draw > 0) {
      lw::iota_kernel<<<lw::grid_for(s_draw), lw::kT, 0, s>>>(rank, s_draw);
      size_t tb2 = 0;
      const int nb = lw::bits_for((uint64_t)n_cand);
      MQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb2, idx2, pk, rank, rk, s_draw, 0, nb, s));
      MQ_TMP(char, cubt2, (int64_t)tb2);
      MQ_CUDA(cub::DeviceRadixSort::SortPairs(cubt2, tb2, idx2, pk, rank, rk, s_draw, 0, nb, s));
      if (mode == 2) {
        MQ_TMP(double, al, s_draw);
        MQ_TMP(double, be, s_draw);
        MQ_TMP(double, cf, s_draw);
        lw::debias_kernel<<<1, 1, 0, s>>>(probs, idx2, s_draw, n_cand, al, be, cf);
        MQ_LAUNCH_CHECK("debias");
        coef = cf;
      }
    }
    pick = pk;
    aux = rk;
  }
  MQ_TMP(double, scale, n_pick);
  if (n_pick > 0) {
    ProfScope ps(K_LAYERWISE, s);
    lw::scale_kernel<<<lw::grid_for(n_pick), lw::kT, 0, s>>>(mode, pick, aux, n_pick, s_draw, probs,
                                                            cand, coef, src_ids, sample_probs, scale);
  }
  MQ_LAUNCH_CHECK("layer_scale");

  // ---- slice the restricted rows to the picked columns
  int rc = launch_scan(lw::LoadKeep{rcol, src_ids, n_pick, ne},
                       lw::StoreSlice{rrow, rcol, rval, roff, src_ids, n_pick, scale, rows, cols,
                                      values, row_ptr, n_prev, hc + 2},
                       ne, scr, s, K_LAYERWISE);
  if (rc) return rc;
  {
    ProfScope ps(K_LAYERWISE, s);
    lw::effective_kernel<<<lw::grid_for(n_prev), lw::kT, 0, s>>>(mode == 0, row_ptr, n_prev, values,
                                                                effective);
  }
  MQ_LAUNCH_CHECK("layer_effective");
  int64_t h[4] = {0, n_pick, n_cand, 0};
  MQ_CUDA(cudaMemcpyAsync(&h[0], hc + 2, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  MQ_CUDA(cudaStreamSynchronize(s));
  h[3] = s_draw;
  MQ_CUDA(cudaMemcpyAsync(counts, h, sizeof(h), cudaMemcpyHostToDevice, s));
  MQ_CUDA(cudaStreamSynchronize(s));
  return MQ_OK;
}

int mq_gcn_block(const int64_t* row_off, const int32_t* loops, const int32_t* dst,
                 const int32_t* src_ids, const int32_t* row_ptr, const int32_t* cols, int32_t n_dst,
                 int32_t* row_ptr_out, int32_t* rows_out, int32_t* cols_out, double* vals_out,
                 void* stream) {
  MQ_CHECK_ARG(row_off && dst && src_ids && row_ptr && cols && row_ptr_out && rows_out &&
                   cols_out && vals_out && n_dst >= 0,
               "mq_gcn_block: bad arguments");
  cudaStream_t s = as_stream(stream);
  lw::Graph g{row_off, nullptr, loops};
  {
    ProfScope ps(K_LAYERWISE, s);
    lw::gcn_block_kernel<<<lw::grid_for(n_dst + 1), lw::kT, 0, s>>>(
        g, dst, src_ids, row_ptr, cols, n_dst, row_ptr_out, rows_out, cols_out, vals_out);
  }
  MQ_LAUNCH_CHECK("gcn_block");
  return MQ_OK;
}

int mq_layer_cdf(const double* probs, int64_t n, double* cdf, void* stream) {
  MQ_CHECK_ARG(probs && cdf && n > 0, "mq_layer_cdf: bad arguments");
  cudaStream_t s = as_stream(stream);
  lw::cumsum_kernel<<<1, 1, 0, s>>>(probs, n, cdf);
  lw::cdf_scale_kernel<<<lw::grid_for(n), lw::kT, 0, s>>>(cdf, n);
  lw::cdf_last_kernel<<<1, 1, 0, s>>>(cdf, n);
  MQ_LAUNCH_CHECK("layer_cdf");
  return MQ_OK;
}

/* host reference of the layer uniforms (tests) */
int mq_layer_uniforms_host(uint64_t seed, uint64_t epoch, uint32_t batch, uint32_t layer, int64_t n,
                           double* out) {
  MQ_CHECK_ARG(n >= 0 && (n == 0 || out), "mq_layer_uniforms_host: bad arguments");
  for (int64_t i = 0; i < n; ++i)
    out[i] = lw::layer_uniform((uint32_t)seed, (uint32_t)epoch, batch, layer, (uint32_t)i);
  return MQ_OK;
}

}  // extern "C"
