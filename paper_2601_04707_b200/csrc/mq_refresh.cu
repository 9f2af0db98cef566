// Per-epoch GNS cache refresh on the device.
//
// Reference (mqpipe):
//   cache_probs_degree  cache.py:41-48    p = in_deg / sum(in_deg)   (f64)
//   cache_probs_walk    cache.py:51-76    p <- D A p + p, `steps` times, then
//                                         p / p.sum()  (f64, numpy pairwise sum)
//   refresh_cache       cache.py:79-108   budget = ceil(f |V|) residents drawn
//                                         WOR by probs, shortfall filled by a
//                                         uniform WOR choice from the rest
//   weighted_sample_without_replacement   samplers.py:113-135: keys u^(1/w)
//                                         over positive w, top-k by (key desc,
//                                         index asc)
//
// Injected draws (oracle/philox.py, the refresh contract): random(n)[i] is the
// NumPy 53-bit double of words x_{4i}, x_{4i+1} of the Philox row stream
// (batch 0xFFFFFFFF, hop 0xFFFFFFFE, row 0); choice() is the sampling
// contract's partial Fisher-Yates on stream (batch 0xFFFFFFFF, hop 0xFFFFFFFF,
// row 0).
//
// Bit-exactness: in-degrees are integers; the walk's per-row flow is summed
// sequentially in CSR order (np.bincount's order), stored self loops re-enter
// at their sorted position, products and sums are _rn (no FMA contraction);
// the normalising total replays NumPy's pairwise summation tree.  Keys use the
// device f64 pow; glibc's pow can differ by an ulp, which changes the resident
// set only if two keys tie at the budget boundary to within an ulp.
//
// Selection without a sort: the keys' IEEE bits (non-negative doubles order
// like their bit patterns) + 1 form a u64 sort key (0 = not eligible); an
// 8-pass radix select finds the budget-th largest key T, everything above T
// is resident, and ties at T go to the lowest ids through one scan.
#include <map>
#include <mutex>
#include <vector>

#include "mq_scan.cuh"

namespace mq {
namespace rf {

constexpr int kThreads = 256;
constexpr uint32_t kBatch = 0xFFFFFFFFu;
constexpr uint32_t kHopRandom = 0xFFFFFFFEu;
constexpr uint32_t kHopChoice = 0xFFFFFFFFu;
constexpr int kPwBlock = 128;  // numpy PW_BLOCKSIZE

struct State {
  unsigned long long prefix;  // radix-select prefix of T
  unsigned long long mask;
  long long k;                // ranks still to place below the prefix
  long long positive;         // #(probs > 0)
  long long take;             // min(budget, positive)
  long long budget;
  unsigned int hist[256];
};

__host__ __device__ __forceinline__ double refresh_uniform(uint32_t seed, uint32_t epoch,
                                                           uint32_t i) {
  const U4 x = philox4x32_10(U4{i, 0u, kHopRandom, kBatch}, seed, epoch);
  return ((double)(x.x >> 5) * 67108864.0 + (double)(x.y >> 6)) / 9007199254740992.0;
}

// ---------------------------------------------------------------- degrees
__global__ void in_degree_kernel(const int32_t* __restrict__ col, int64_t E,
                                 unsigned long long* __restrict__ deg) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(deg + __ldg(col + e), 1ull);
}

__global__ void add_loops_kernel(const int32_t* __restrict__ loops, int64_t n,
                                 unsigned long long* __restrict__ deg) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    deg[v] += (unsigned long long)loops[v];
}

__global__ void degree_probs_kernel(const long long* __restrict__ deg, int64_t n, double total,
                                    double* __restrict__ probs) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    probs[v] = total == 0.0 ? 1.0 / (double)n : __ddiv_rn((double)deg[v], total);
}

// ---------------------------------------------------------------- walk
__global__ void walk_init_kernel(const uint8_t* __restrict__ train, const long long* __restrict__ deg,
                                 int64_t n, double p_train, int fanout, double* __restrict__ p,
                                 double* __restrict__ d) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    p[v] = train[v] ? p_train : 0.0;
    const double in = (double)deg[v];
    d[v] = in > 0.0 ? __ddiv_rn(in < (double)fanout ? in : (double)fanout, in) : 0.0;
  }
}

// p_out[v] = d[v] * flow[v] + p[v], flow[v] = sum over the stored arcs of row v
// of p[col] in CSR order (the stripped self loop re-inserted before the first
// neighbour > v).  One warp per row: the lanes fetch kWalkU x 32 arcs at a
// time (all gathers in flight together, so a hub row costs one memory round
// trip per 256 arcs), then the sum is carried sequentially through shuffles
// (identical in every lane) — np.bincount's exact order.
constexpr int kWalkU = 8;

__global__ void __launch_bounds__(kThreads) walk_step_kernel(
    const int64_t* __restrict__ row_off, const int32_t* __restrict__ col,
    const int32_t* __restrict__ loops, int64_t n, const double* __restrict__ p,
    const double* __restrict__ d, double* __restrict__ p_out) {
  const int lane = threadIdx.x & 31;
  const int warps = kThreads / 32;
  for (int64_t v = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5); v < n;
       v += (int64_t)gridDim.x * warps) {
    const int64_t e0 = __ldg(row_off + v), e1 = __ldg(row_off + v + 1);
    bool loop = loops != nullptr && loops[v] > 0;
    const double pv = p[v];
    double acc = 0.0;
    for (int64_t b = e0; b < e1; b += 32 * kWalkU) {
      int32_t c[kWalkU];
      double x[kWalkU];
#pragma unroll
      for (int u = 0; u < kWalkU; ++u) {
        const int64_t e = b + 32 * u + lane;
        c[u] = e < e1 ? __ldg(col + e) : 0;
      }
#pragma unroll
      for (int u = 0; u < kWalkU; ++u) x[u] = b + 32 * u + lane < e1 ? p[c[u]] : 0.0;
#pragma unroll
      for (int u = 0; u < kWalkU; ++u) {
        const int64_t bu = b + 32 * u;
        if (bu >= e1) break;
        const int m = (int)(e1 - bu < 32 ? e1 - bu : 32);
        // the stored loop enters before the group's first neighbour > v
        int ins = 32;
        if (loop) {
          const unsigned bal = __ballot_sync(0xffffffffu, lane < m && c[u] > v);
          if (bal) {
            ins = __ffs(bal) - 1;
            loop = false;
          }
        }
        if (m == 32 && ins == 32) {  // unrolled, no insertion: a bare add chain
#pragma unroll
          for (int t = 0; t < 32; ++t) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, x[u], t));
        } else {
          for (int t = 0; t < m; ++t) {
            const double xt = __shfl_sync(0xffffffffu, x[u], t);
            if (t == ins) acc = __dadd_rn(acc, pv);
            acc = __dadd_rn(acc, xt);
          }
        }
      }
    }
    if (loop) acc = __dadd_rn(acc, pv);
    if (lane == 0) p_out[v] = __dadd_rn(__dmul_rn(d[v], acc), pv);
  }
}

// ---- numpy pairwise sum (loops_utils.h.src: pairwise_sum, PW_BLOCKSIZE 128)
__device__ __forceinline__ double pw_leaf(const double* __restrict__ a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

__global__ void pw_leaves_kernel(const double* __restrict__ a, const int64_t* __restrict__ starts,
                                 int64_t nleaves, int64_t n, double* __restrict__ sums) {
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < nleaves;
       l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = starts[l], e = l + 1 < nleaves ? starts[l + 1] : n;
    sums[l] = pw_leaf(a + s, e - s);
  }
}

// The recursion's internal nodes, one height level per launch: node i of the
// level = sums[left[i]] + sums[right[i]] (the same additions, in the same
// operand order, as numpy's pairwise_sum — just evaluated level-parallel).
__global__ void pw_level_kernel(double* __restrict__ vals, const int32_t* __restrict__ left,
                                const int32_t* __restrict__ right, int64_t lo, int64_t hi,
                                int64_t base) {
  for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi;
       i += (int64_t)gridDim.x * blockDim.x)
    vals[base + i] = __dadd_rn(vals[left[i]], vals[right[i]]);
}

__global__ void pw_total_kernel(const double* __restrict__ vals, int64_t root,
                                double* __restrict__ total) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *total = __dadd_rn(0.0, vals[root]);
}

__global__ void normalize_kernel(const double* __restrict__ p, const double* __restrict__ total,
                                 int64_t n, double* __restrict__ probs, int32_t* __restrict__ bad) {
  const double t = *total;
  if (blockIdx.x == 0 && threadIdx.x == 0 && !(t > 0.0)) *bad = 1;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    probs[v] = __ddiv_rn(p[v], t);
}

// ---------------------------------------------------------------- selection
__global__ void init_state_kernel(State* st, long long budget) {
  if (threadIdx.x == 0) {
    st->prefix = 0;
    st->mask = 0;
    st->k = 0;
    st->positive = 0;
    st->take = 0;
    st->budget = budget;
  }
  st->hist[threadIdx.x] = 0;
}

// scan 1: rank positive nodes; the store writes the sort key
struct LoadPositive {
  const double* w;
  int64_t n;
  __device__ int64_t size() const { return n; }
  __device__ int64_t operator()(int64_t i) const { return w[i] > 0.0 ? 1 : 0; }
};
struct StoreKey {
  const double* w;
  uint32_t seed, epoch;
  unsigned long long* skey;
  State* st;
  __device__ void operator()(int64_t i, int64_t excl, int64_t val) const {
    unsigned long long k = 0;
    if (val) {
      const double u = refresh_uniform(seed, epoch, (uint32_t)excl);
      const double key = pow(u, __ddiv_rn(1.0, w[i]));
      k = (unsigned long long)__double_as_longlong(key) + 1ull;
    }
    skey[i] = k;
  }
  __device__ void total(int64_t, int64_t t) const {
    st->positive = t;
    st->take = t < st->budget ? t : st->budget;
    st->k = st->take;
    st->prefix = 0;
    st->mask = 0;
  }
};

__global__ void __launch_bounds__(kThreads) radix_hist_kernel(const unsigned long long* __restrict__ skey,
                                                              int64_t n, int shift, State* st) {
  __shared__ unsigned int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const unsigned long long prefix = st->prefix, mask = st->mask;
  if (st->k > 0) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
      const unsigned long long k = skey[i];
      if ((k & mask) == prefix) atomicAdd(&h[(k >> shift) & 255u], 1u);
    }
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&st->hist[threadIdx.x], h[threadIdx.x]);
}

// one block of 256: the bucket (from the top) holding the k-th largest key
__global__ void __launch_bounds__(256) radix_pick_kernel(int shift, State* st) {
  __shared__ long long c[256];
  const int t = threadIdx.x;
  const int b = 255 - t;  // descending buckets
  c[t] = st->hist[b];
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {  // inclusive scan over descending buckets
    const long long v = t >= o ? c[t - o] : 0;
    __syncthreads();
    c[t] += v;
    __syncthreads();
  }
  const long long k = st->k;
  const long long incl = c[t], excl = t ? c[t - 1] : 0;
  __syncthreads();
  if (k > 0 && excl < k && incl >= k) {
    st->prefix |= (unsigned long long)b << shift;
    st->mask |= 255ull << shift;
    st->k = k - excl;
  }
  st->hist[b] = 0;
}

// scan 2: ties at T in id order; the store writes the resident flags
struct LoadTie {
  const unsigned long long* skey;
  const State* st;
  int64_t n;
  __device__ int64_t size() const { return n; }
  __device__ int64_t operator()(int64_t i) const {
    return (st->take > 0 && skey[i] == st->prefix) ? 1 : 0;
  }
};
struct StoreChosen {
  const unsigned long long* skey;
  const State* st;
  uint8_t* chosen;
  __device__ void operator()(int64_t i, int64_t excl, int64_t val) const {
    const unsigned long long k = skey[i];
    chosen[i] = (st->take > 0 && (k > st->prefix || (val && excl < st->k))) ? 1 : 0;
  }
  __device__ void total(int64_t, int64_t) const {}
};

// scan 3 (shortfall): ids not yet resident, ascending (np.setdiff1d)
struct LoadRest {
  const uint8_t* chosen;
  int64_t n;
  __device__ int64_t size() const { return n; }
  __device__ int64_t operator()(int64_t i) const { return chosen[i] ? 0 : 1; }
};
struct StoreRest {
  int32_t* rest;
  __device__ void operator()(int64_t i, int64_t excl, int64_t val) const {
    if (val) rest[excl] = (int32_t)i;
  }
  __device__ void total(int64_t, int64_t) const {}
};

// rng.choice(rest, budget - take, replace=False): dense partial Fisher-Yates
// (equal to the contract's sparse form), one thread; rare path.
__global__ void shortfall_kernel(int32_t* __restrict__ rest, int64_t n, uint32_t seed,
                                 uint32_t epoch, const State* st, uint8_t* __restrict__ chosen) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const long long k = st->budget - st->take;
  const long long m = n - st->take;
  RowStream rs(seed, epoch, kBatch, kHopChoice, 0u);
  for (long long j = 0; j < k; ++j) {
    const uint64_t x = rs.draw((uint32_t)j);
    const long long r = j + (long long)((x * (uint64_t)(m - j)) >> 32);
    const int32_t a = rest[j];
    rest[j] = rest[r];
    rest[r] = a;
    chosen[rest[j]] = 1;
  }
}

inline int grid_for(int64_t n, int per = kThreads) {
  const int64_t g = (n + per - 1) / per;
  return (int)(g < 1 ? 1 : (g > kNumSMs * 16 ? kNumSMs * 16 : g));
}

// numpy pairwise-sum tree for a length-n array (cached per n): leaf starts in
// left-to-right order (node ids 0..L-1), internal nodes sorted by height
// (ids L.., children ids in left/right), level boundaries.
struct PwPlan {
  std::vector<int64_t> starts;
  std::vector<int32_t> left, right;
  std::vector<int64_t> level_end;  // internal-node index bounds per height 1..H
  int64_t root = 0;
};

const PwPlan& pw_plan(int64_t n) {
  static std::mutex mu;
  static std::map<int64_t, PwPlan> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(n);
  if (it != cache.end()) return it->second;
  PwPlan P;
  struct Node { int32_t l, r; int h; };
  std::vector<Node> inner;  // post-order, ids L + k after renumbering
  // iterative post-order recursion: frame (start, len, state, left id, left height)
  struct Fr { int64_t s, m; int st; int64_t lid; int lh; };
  std::vector<Fr> stk{{0, n, 0, 0, 0}};
  int64_t ret_id = 0;
  int ret_h = 0;
  std::vector<int64_t> leaf_ids;  // leaves get ids in order of creation (left to right)
  while (!stk.empty()) {
    Fr& f = stk.back();
    if (f.m <= kPwBlock) {
      ret_id = (int64_t)P.starts.size();
      ret_h = 0;
      P.starts.push_back(f.s);
      stk.pop_back();
      continue;
    }
    int64_t n2 = f.m / 2;
    n2 -= n2 % 8;
    if (f.st == 0) {
      f.st = 1;
      stk.push_back({f.s, n2, 0, 0, 0});
    } else if (f.st == 1) {
      f.lid = ret_id;
      f.lh = ret_h;
      f.st = 2;
      const int64_t s2 = f.s + n2, m2 = f.m - n2;
      stk.push_back({s2, m2, 0, 0, 0});
    } else {
      const int h = (f.lh > ret_h ? f.lh : ret_h) + 1;
      inner.push_back({(int32_t)f.lid, (int32_t)ret_id, h});
      ret_id = -(int64_t)inner.size();  // provisional: -(k+1) = internal node k
      ret_h = h;
      stk.pop_back();
    }
  }
  const int64_t L = (int64_t)P.starts.size();
  // renumber internal nodes by height (stable): final id = L + position
  int H = 0;
  for (auto& nd : inner) H = nd.h > H ? nd.h : H;
  std::vector<int64_t> cnt(H + 2, 0), pos(inner.size());
  for (auto& nd : inner) cnt[nd.h]++;
  std::vector<int64_t> off(H + 2, 0);
  for (int h = 1; h <= H; ++h) off[h + 1] = off[h] + cnt[h];
  std::vector<int64_t> fill(off);
  for (size_t k = 0; k < inner.size(); ++k) pos[k] = fill[inner[k].h]++;
  auto fin = [&](int64_t id) { return id >= 0 ? id : L + pos[-id - 1]; };
  P.left.assign(inner.size(), 0);
  P.right.assign(inner.size(), 0);
  for (size_t k = 0; k < inner.size(); ++k) {
    P.left[pos[k]] = (int32_t)fin(inner[k].l);
    P.right[pos[k]] = (int32_t)fin(inner[k].r);
  }
  for (int h = 1; h <= H; ++h) P.level_end.push_back(off[h + 1]);
  P.root = inner.empty() ? 0 : L + (int64_t)inner.size() - 1;
  (void)leaf_ids;
  return cache.emplace(n, std::move(P)).first->second;
}

}  // namespace rf

// NumPy's pairwise sum of a device f64 array of host-known length into
// *total (the refresh's level-parallel replay of the summation tree); the
// tree's temporaries come from the stream-ordered allocator.
int pairwise_total(const double* a, int64_t n, double* total, cudaStream_t s) {
  MQ_CHECK_ARG(a && total && n > 0, "pairwise_total: bad arguments");
  const rf::PwPlan& plan = rf::pw_plan(n);
  const int64_t nl = (int64_t)plan.starts.size();
  const int64_t ni = (int64_t)plan.left.size();
  void* mem = nullptr;
  const size_t bytes = 8 * (size_t)(nl + ni) + 8 * (size_t)nl + 4 * (size_t)(2 * ni) + 16;
  MQ_CUDA(cudaMallocAsync(&mem, bytes, s));
  double* sums = static_cast<double*>(mem);
  int64_t* starts = reinterpret_cast<int64_t*>(sums + nl + ni);
  int32_t* lft = reinterpret_cast<int32_t*>(starts + nl);
  int32_t* rgt = lft + ni;
  cudaError_t e = cudaMemcpyAsync(starts, plan.starts.data(), sizeof(int64_t) * nl,
                                  cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && ni)
    e = cudaMemcpyAsync(lft, plan.left.data(), sizeof(int32_t) * ni, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && ni)
    e = cudaMemcpyAsync(rgt, plan.right.data(), sizeof(int32_t) * ni, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    rf::pw_leaves_kernel<<<rf::grid_for(nl), rf::kThreads, 0, s>>>(a, starts, nl, n, sums);
    int64_t lo = 0;
    for (int64_t hi : plan.level_end) {
      rf::pw_level_kernel<<<rf::grid_for(hi - lo), rf::kThreads, 0, s>>>(sums, lft, rgt, lo, hi, nl);
      lo = hi;
    }
    rf::pw_total_kernel<<<1, 32, 0, s>>>(sums, plan.root, total);
    e = cudaGetLastError();
  }
  // the host plan vectors are read by the async copies: keep them alive (the
  // plan cache owns them) and free the device tree in stream order
  cudaFreeAsync(mem, s);
  if (e != cudaSuccess) {
    set_error("pairwise_total: %s", cudaGetErrorString(e));
    return MQ_ERR_CUDA;
  }
  return MQ_OK;
}

}  // namespace mq

using namespace mq;

extern "C" {

int mq_in_degrees(const int32_t* col, int64_t n_nodes, int64_t n_arcs, const int32_t* loops,
                  int64_t* deg, void* stream) {
  MQ_CHECK_ARG(n_nodes >= 0 && n_arcs >= 0, "mq_in_degrees: negative sizes");
  MQ_CHECK_ARG(deg && (n_arcs == 0 || col), "mq_in_degrees: null pointer");
  cudaStream_t s = as_stream(stream);
  if (n_nodes == 0) return MQ_OK;
  MQ_CUDA(cudaMemsetAsync(deg, 0, sizeof(int64_t) * n_nodes, s));
  auto* d = reinterpret_cast<unsigned long long*>(deg);
  if (n_arcs) {
    ProfScope ps(K_REFRESH_DEGREE, s);
    rf::in_degree_kernel<<<rf::grid_for(n_arcs), rf::kThreads, 0, s>>>(col, n_arcs, d);
  }
  MQ_LAUNCH_CHECK("in_degree");
  if (loops) {
    ProfScope ps(K_REFRESH_DEGREE, s);
    rf::add_loops_kernel<<<rf::grid_for(n_nodes), rf::kThreads, 0, s>>>(loops, n_nodes, d);
  }
  MQ_LAUNCH_CHECK("add_loops");
  return MQ_OK;
}

int mq_degree_probs(const int64_t* deg, int64_t n_nodes, int64_t total, double* probs,
                    void* stream) {
  MQ_CHECK_ARG(n_nodes > 0 && total >= 0 && deg && probs, "mq_degree_probs: bad arguments");
  cudaStream_t s = as_stream(stream);
  {
    ProfScope ps(K_REFRESH_PROBS, s);
    rf::degree_probs_kernel<<<rf::grid_for(n_nodes), rf::kThreads, 0, s>>>(
        reinterpret_cast<const long long*>(deg), n_nodes, (double)total, probs);
  }
  MQ_LAUNCH_CHECK("degree_probs");
  return MQ_OK;
}

int64_t mq_walk_scratch_bytes(int64_t n_nodes) {
  const int64_t leaves = n_nodes / 64 + 2;  // internal nodes < leaves
  return 8 * (3 * n_nodes + 2 * leaves) + 8 * (2 * leaves) + 8 * leaves + 64;
}

int mq_walk_probs(const int64_t* row_off, const int32_t* col, int64_t n_nodes, const int32_t* loops,
                  const int64_t* deg, const uint8_t* train_mask, int64_t n_train, int32_t fanout,
                  int32_t steps, double* probs, int32_t* bad_dev, void* scratch, void* stream) {
  MQ_CHECK_ARG(n_nodes > 0 && steps >= 0 && fanout >= 0, "mq_walk_probs: bad sizes");
  MQ_CHECK_ARG(n_train > 0, "walk probabilities need a nonempty training set");
  MQ_CHECK_ARG(row_off && deg && train_mask && probs && bad_dev && scratch,
               "mq_walk_probs: null pointer");
  cudaStream_t s = as_stream(stream);
  const rf::PwPlan& plan = rf::pw_plan(n_nodes);
  const int64_t nl = (int64_t)plan.starts.size();
  const int64_t ni = (int64_t)plan.left.size();
  double* pa = static_cast<double*>(scratch);
  double* pb = pa + n_nodes;
  double* d = pb + n_nodes;
  double* sums = d + n_nodes;                 // leaves then internal nodes
  int64_t* starts = reinterpret_cast<int64_t*>(sums + nl + ni);
  int32_t* lft = reinterpret_cast<int32_t*>(starts + nl);
  int32_t* rgt = lft + ni;
  double* total = reinterpret_cast<double*>(starts + nl + ni + 1);
  MQ_CHECK_ARG(nl <= n_nodes / 64 + 2, "mq_walk_probs: internal leaf bound");
  MQ_CUDA(cudaMemcpyAsync(starts, plan.starts.data(), sizeof(int64_t) * nl, cudaMemcpyHostToDevice,
                          s));
  if (ni) {
    MQ_CUDA(cudaMemcpyAsync(lft, plan.left.data(), sizeof(int32_t) * ni, cudaMemcpyHostToDevice, s));
    MQ_CUDA(cudaMemcpyAsync(rgt, plan.right.data(), sizeof(int32_t) * ni, cudaMemcpyHostToDevice, s));
  }
  MQ_CUDA(cudaMemsetAsync(bad_dev, 0, sizeof(int32_t), s));
  {
    ProfScope ps(K_REFRESH_PROBS, s);
    rf::walk_init_kernel<<<rf::grid_for(n_nodes), rf::kThreads, 0, s>>>(
        train_mask, reinterpret_cast<const long long*>(deg), n_nodes, 1.0 / (double)n_train, fanout,
        pa, d);
  }
  MQ_LAUNCH_CHECK("walk_init");
  for (int it = 0; it < steps; ++it) {
    {
      ProfScope ps(K_REFRESH_WALK, s);
      rf::walk_step_kernel<<<rf::grid_for(n_nodes, rf::kThreads / 32), rf::kThreads, 0, s>>>(
          row_off, col, loops, n_nodes, pa, d, pb);
    }
    MQ_LAUNCH_CHECK("walk_step");
    double* t = pa;
    pa = pb;
    pb = t;
  }
  {
    ProfScope ps(K_REFRESH_PROBS, s);
    rf::pw_leaves_kernel<<<rf::grid_for(nl), rf::kThreads, 0, s>>>(pa, starts, nl, n_nodes, sums);
    int64_t lo = 0;
    for (int64_t hi : plan.level_end) {
      rf::pw_level_kernel<<<rf::grid_for(hi - lo), rf::kThreads, 0, s>>>(sums, lft, rgt, lo, hi, nl);
      lo = hi;
    }
    rf::pw_total_kernel<<<1, 32, 0, s>>>(sums, plan.root, total);
    rf::normalize_kernel<<<rf::grid_for(n_nodes), rf::kThreads, 0, s>>>(pa, total, n_nodes, probs,
                                                                       bad_dev);
  }
  MQ_LAUNCH_CHECK("walk_normalize");
  return MQ_OK;
}

int64_t mq_refresh_scratch_bytes(int64_t n_nodes) {
  const int64_t scan = scan_scratch_bytes(n_nodes < 1 ? 1 : n_nodes);
  auto r256 = [](int64_t b) { return (b + 255) / 256 * 256; };
  return r256((int64_t)sizeof(rf::State)) + r256(8 * n_nodes) + r256(4 * n_nodes) + r256(scan);
}

int mq_refresh_select(const double* probs, int64_t n_nodes, int64_t budget, uint64_t seed,
                      uint64_t epoch, uint8_t* chosen, int64_t* counts_dev, void* scratch,
                      void* stream) {
  MQ_CHECK_ARG(n_nodes > 0 && n_nodes < INT32_MAX, "mq_refresh_select: n_nodes out of range");
  MQ_CHECK_ARG(budget >= 0 && budget <= n_nodes, "mq_refresh_select: budget out of range");
  MQ_CHECK_ARG(probs && chosen && counts_dev && scratch, "mq_refresh_select: null pointer");
  cudaStream_t s = as_stream(stream);
  char* base = static_cast<char*>(scratch);
  rf::State* st = reinterpret_cast<rf::State*>(base);
  base += ((int64_t)sizeof(rf::State) + 255) / 256 * 256;
  auto* skey = reinterpret_cast<unsigned long long*>(base);
  base += (8 * n_nodes + 255) / 256 * 256;
  auto* rest = reinterpret_cast<int32_t*>(base);
  base += (4 * n_nodes + 255) / 256 * 256;
  void* scan_scr = base;
  {
    ProfScope ps(K_REFRESH_SELECT, s);
    rf::init_state_kernel<<<1, 256, 0, s>>>(st, (long long)budget);
  }
  MQ_LAUNCH_CHECK("refresh_init");
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)epoch;
  int rc = launch_scan(rf::LoadPositive{probs, n_nodes}, rf::StoreKey{probs, k0, k1, skey, st},
                       n_nodes, scan_scr, s, K_REFRESH_SELECT);
  if (rc) return rc;
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    {
      ProfScope ps(K_REFRESH_SELECT, s);
      rf::radix_hist_kernel<<<rf::grid_for(n_nodes), rf::kThreads, 0, s>>>(skey, n_nodes, shift, st);
      rf::radix_pick_kernel<<<1, 256, 0, s>>>(shift, st);
    }
    MQ_LAUNCH_CHECK("radix_select");
  }
  rc = launch_scan(rf::LoadTie{skey, st, n_nodes}, rf::StoreChosen{skey, st, chosen}, n_nodes,
                   scan_scr, s, K_REFRESH_SELECT);
  if (rc) return rc;
  rc = launch_scan(rf::LoadRest{chosen, n_nodes}, rf::StoreRest{rest}, n_nodes, scan_scr, s,
                   K_REFRESH_SELECT);
  if (rc) return rc;
  {
    ProfScope ps(K_REFRESH_SELECT, s);
    rf::shortfall_kernel<<<1, 32, 0, s>>>(rest, n_nodes, k0, k1, st, chosen);
  }
  MQ_LAUNCH_CHECK("shortfall");
  MQ_CUDA(cudaMemcpyAsync(counts_dev, &st->positive, 2 * sizeof(long long),
                          cudaMemcpyDeviceToDevice, s));
  return MQ_OK;
}

/* host reference of the refresh uniforms (tests) */
int mq_refresh_uniforms_host(uint64_t seed, uint64_t epoch, int64_t n, double* out) {
  MQ_CHECK_ARG(n >= 0 && (n == 0 || out), "mq_refresh_uniforms_host: bad arguments");
  for (int64_t i = 0; i < n; ++i) out[i] = rf::refresh_uniform((uint32_t)seed, (uint32_t)epoch, (uint32_t)i);
  return MQ_OK;
}

}  // extern "C"
