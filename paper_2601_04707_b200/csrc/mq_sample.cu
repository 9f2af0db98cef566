// GNS-biased node-wise sampling, relabel and the per-epoch residency index.
//
// Reference semantics: mqpipe/samplers.py:142-226 (node_wise_block, SAGE arm,
// sample_node_wise) and cache.py:20-38,111-134 (residency).  Draws follow the
// injected Philox contract.
#include <climits>

#include "mq_common.cuh"
#include "mq_scan.cuh"

namespace mq {

// ------------------------------------------------------------------ Philox
__global__ void philox_fill_kernel(uint64_t seed, uint64_t epoch, uint32_t batch, uint32_t hop,
                                   uint32_t row, uint32_t count, uint32_t* out) {
  uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;  // one Philox block (4 draws)
  if ((uint64_t)b * 4 >= count) return;
  U4 c{b, row, hop, batch};
  U4 r = philox4x32_10(c, (uint32_t)seed, (uint32_t)epoch);
  uint32_t vals[4] = {r.x, r.y, r.z, r.w};
  for (int i = 0; i < 4; ++i)
    if (b * 4 + i < count) out[b * 4 + i] = vals[i];
}

// ----------------------------------------------------------- self-loop strip
__device__ __forceinline__ bool row_has(const int32_t* col, int64_t beg, int64_t end, int32_t v,
                                        int64_t* where) {
  int64_t lo = beg, hi = end;  // rows are sorted ascending (graph.py:106-116)
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (col[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  *where = lo;
  return lo < end && col[lo] == v;
}

struct LoadKeep {
  const int64_t* row_off;
  const int32_t* col;
  int64_t n;
  __device__ int64_t size() const { return n; }
  __device__ int64_t operator()(int64_t v) const {
    int64_t beg = row_off[v], end = row_off[v + 1], w;
    return (end - beg) - (row_has(col, beg, end, (int32_t)v, &w) ? 1 : 0);
  }
};

__global__ void strip_copy_kernel(const int64_t* __restrict__ row_off, const int32_t* __restrict__ col,
                                  int64_t n, const int64_t* __restrict__ out_off,
                                  int32_t* __restrict__ out_col) {
  int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (v >= n) return;
  int64_t beg = row_off[v], end = row_off[v + 1];
  int64_t ob = out_off[v];
  int64_t skip = end;  // arc index of the self loop, if any
  if (out_off[v + 1] - ob != end - beg) {
    int64_t w;
    row_has(col, beg, end, (int32_t)v, &w);
    skip = w;
  }
  for (int64_t a = beg + lane; a < end; a += 32) {
    if (a == skip) continue;
    out_col[ob + (a - beg) - (a > skip ? 1 : 0)] = col[a];
  }
}

// ------------------------------------------------------- residency index
__device__ __forceinline__ bool bit_test(const uint32_t* bits, int32_t v) {
  return (__ldg(&bits[v >> 5]) >> (v & 31)) & 1u;
}

struct LoadHotArc {
  const int32_t* col;
  const uint32_t* bits;
  int64_t n;
  __device__ int64_t size() const { return n; }
  __device__ int64_t operator()(int64_t a) const { return bit_test(bits, __ldg(&col[a])) ? 1 : 0; }
};

struct StoreHotArc {
  int64_t* hot_arc;
  int64_t* n_hot;
  __device__ void operator()(int64_t a, int64_t excl, int64_t val) const {
    if (val) hot_arc[excl] = a;
  }
  __device__ void total(int64_t, int64_t t) const { *n_hot = t; }
};

__global__ void residency_offsets_kernel(const int64_t* __restrict__ row_off, int64_t n_nodes,
                                         const int64_t* __restrict__ hot_arc,
                                         const int64_t* __restrict__ n_hot,
                                         int64_t* __restrict__ hot_off) {
  int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v > n_nodes) return;
  int64_t key = row_off[v];
  int64_t lo = 0, hi = *n_hot;  // lower_bound(hot_arc, key)
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (hot_arc[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  hot_off[v] = lo;
}

struct LoadBit {
  const uint32_t* bits;
  int64_t n;
  __device__ int64_t size() const { return n; }
  __device__ int64_t operator()(int64_t v) const { return bit_test(bits, (int32_t)v) ? 1 : 0; }
};

struct StoreSlot {
  int32_t* slot_of;
  int32_t* n_res;
  __device__ void operator()(int64_t v, int64_t excl, int64_t val) const {
    slot_of[v] = val ? (int32_t)excl : -1;
  }
  __device__ void total(int64_t, int64_t t) const { *n_res = (int32_t)t; }
};

// ------------------------------------------------------------------ sample
// One thread per dst row: every case is O(fanout) thanks to the residency
// index, so a row costs a handful of dependent loads regardless of degree.
template <int MAXK>
__global__ void __launch_bounds__(128) sample_hop_kernel(
    const int64_t* __restrict__ row_off, const int32_t* __restrict__ col,
    const int64_t* __restrict__ hot_arc, const int64_t* __restrict__ hot_off,
    const int32_t* __restrict__ dst, const int32_t* __restrict__ n_dst_dev, int fanout,
    uint64_t seed, uint64_t epoch, uint32_t batch, uint32_t hop,
    const uint32_t* __restrict__ key_dev, int32_t* __restrict__ nbr, int32_t* __restrict__ cnt) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= *n_dst_dev) return;
  if (key_dev != nullptr) {
    seed = key_dev[0];
    epoch = key_dev[1];
    batch = key_dev[2];
  }
  const int32_t v = dst[r];
  const int64_t beg = row_off[v];
  const int n = (int)(row_off[v + 1] - beg);
  int32_t* out = nbr + (int64_t)r * fanout;
  if (n <= fanout) {  // samplers.py:164-167: take every neighbour, CSR order
    for (int i = 0; i < n; ++i) out[i] = __ldg(&col[beg + i]);
    cnt[r] = n;
    return;
  }
  RowStream rs(seed, epoch, batch, hop, (uint32_t)r);
  int pos[MAXK];
  if (hot_off != nullptr) {  // samplers.py:168-175
    const int64_t hb = hot_off[v];
    const int nh = (int)(hot_off[v + 1] - hb);
    if (nh >= fanout) {
      fisher_yates<MAXK, int>(rs, nh, fanout, pos);
      for (int j = 0; j < fanout; ++j) out[j] = __ldg(&col[hot_arc[hb + pos[j]]]);
    } else {
      for (int i = 0; i < nh; ++i) out[i] = __ldg(&col[hot_arc[hb + i]]);
      const int k = fanout - nh;
      fisher_yates<MAXK, int>(rs, n - nh, k, pos);
      for (int j = 0; j < k; ++j) {
        // cold rank -> row position: skip every hot position h_i with
        // h_i - i <= rank (the hot positions are ascending)
        const int rr = pos[j];
        int c = 0;
        for (int i = 0; i < nh; ++i) c += ((int)(hot_arc[hb + i] - beg) - i <= rr) ? 1 : 0;
        out[nh + j] = __ldg(&col[beg + rr + c]);
      }
    }
  } else {  // samplers.py:176-177
    fisher_yates<MAXK, int>(rs, n, fanout, pos);
    for (int j = 0; j < fanout; ++j) out[j] = __ldg(&col[beg + pos[j]]);
  }
  cnt[r] = fanout;
}

// ------------------------------------------------------------------ relabel
struct StoreRowPtr {
  int32_t* row_ptr;
  int32_t* counts;  // counts[1] = nnz
  __device__ void operator()(int64_t i, int64_t excl, int64_t) const { row_ptr[i] = (int32_t)excl; }
  __device__ void total(int64_t n, int64_t t) const {
    row_ptr[n] = (int32_t)t;
    counts[1] = (int32_t)t;
  }
};

// dst ids lead src_ids; the node table remembers each dst id's (last) position
__global__ void relabel_mark_kernel(const int32_t* __restrict__ dst,
                                    const int32_t* __restrict__ n_dst_dev,
                                    int32_t* __restrict__ dpos, int32_t* __restrict__ src_ids) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *n_dst_dev) return;
  int32_t v = dst[i];
  src_ids[i] = v;
  atomicMax(&dpos[v], i);
}

// first occurrence (edge index) of every id that is not a dst id
__global__ void relabel_first_kernel(const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt,
                                     const int32_t* __restrict__ row_ptr,
                                     const int32_t* __restrict__ n_dst_dev, int fanout,
                                     const int32_t* __restrict__ dpos, int32_t* __restrict__ first) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int r = (int)(s / fanout), i = (int)(s % fanout);
  if (r >= *n_dst_dev || i >= cnt[r]) return;
  int32_t u = nbr[s];
  if (dpos[u] < 0) atomicMin(&first[u], row_ptr[r] + i);
}

// flags over padded slots (r, i) — same order as edges — mark first
// occurrences; the scan ranks them and the store assigns labels n_dst + rank.
struct LoadFirstFlag {
  const int32_t* nbr;
  const int32_t* cnt;
  const int32_t* row_ptr;
  const int32_t* n_dst_dev;
  const int32_t* dpos;
  const int32_t* first;
  int fanout;
  __device__ int64_t size() const { return (int64_t)(*n_dst_dev) * fanout; }
  __device__ int64_t operator()(int64_t s) const {
    int r = (int)(s / fanout), i = (int)(s % fanout);
    if (i >= cnt[r]) return 0;
    int32_t u = nbr[s];
    // a concurrent store may already have labelled u (dpos >= n_dst); only the
    // slot holding the first occurrence can ever match first[u]
    return (dpos[u] < 0 && first[u] == row_ptr[r] + i) ? 1 : 0;
  }
};

struct StoreLabel {
  const int32_t* nbr;
  const int32_t* n_dst_dev;
  int32_t* dpos;
  int32_t* src_ids;
  int32_t* counts;  // counts[0] = n_src
  __device__ void operator()(int64_t s, int64_t excl, int64_t val) const {
    if (!val) return;
    int32_t u = nbr[s];
    int32_t lab = *n_dst_dev + (int32_t)excl;
    src_ids[lab] = u;
    dpos[u] = lab;
  }
  __device__ void total(int64_t, int64_t t) const { counts[0] = *n_dst_dev + (int32_t)t; }
};

__global__ void relabel_cols_kernel(const int32_t* __restrict__ nbr, const int32_t* __restrict__ cnt,
                                    const int32_t* __restrict__ row_ptr,
                                    const int32_t* __restrict__ n_dst_dev, int fanout,
                                    const int32_t* __restrict__ dpos, int32_t* __restrict__ rows,
                                    int32_t* __restrict__ cols, float* __restrict__ vals) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int r = (int)(s / fanout), i = (int)(s % fanout);
  if (r >= *n_dst_dev) return;
  int c = cnt[r];
  if (i >= c) return;
  int e = row_ptr[r] + i;
  rows[e] = r;
  cols[e] = dpos[nbr[s]];
  vals[e] = (float)(1.0 / (double)c);  // float32(1.0 / s), samplers.py:200 + nn.py:85
}

__global__ void relabel_clean_kernel(const int32_t* __restrict__ src_ids,
                                     const int32_t* __restrict__ counts,
                                     const int32_t* __restrict__ n_dst_dev,
                                     int32_t* __restrict__ dpos, int32_t* __restrict__ first) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= counts[0]) return;
  int32_t u = src_ids[j];
  dpos[u] = -1;
  if (j >= *n_dst_dev) first[u] = INT_MAX;
}

// device-side batch plan: one thread block copies this rank's targets
__global__ void batch_setup_kernel(const int32_t* __restrict__ perm, int64_t n_perm, int batch_size,
                                   int world, int rank, int32_t* __restrict__ cursor,
                                   int32_t* __restrict__ targets, int32_t* __restrict__ n_targets,
                                   uint32_t* __restrict__ key) {
  __shared__ int64_t s_begin;
  __shared__ int s_len;
  if (threadIdx.x == 0) {
    const int64_t window = cursor[0];
    const int64_t j = window * world + rank;
    const int64_t b = j * batch_size;
    int64_t len = n_perm - b;
    len = len < 0 ? 0 : (len > batch_size ? batch_size : len);
    s_begin = b;
    s_len = (int)len;
    n_targets[0] = (int32_t)len;
    key[2] = (uint32_t)j;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < s_len; i += blockDim.x) targets[i] = perm[s_begin + i];
  __syncthreads();
  if (threadIdx.x == 0) cursor[0] += 1;
}

}  // namespace mq

using namespace mq;

extern "C" {

int mq_philox_fill_host(uint64_t seed, uint64_t epoch, uint32_t batch, uint32_t hop, uint32_t row,
                        uint32_t count, uint32_t* out) {
  MQ_CHECK_ARG(out != nullptr || count == 0, "mq_philox_fill_host: null out");
  RowStream rs(seed, epoch, batch, hop, row);
  for (uint32_t j = 0; j < count; ++j) out[j] = rs.draw(j);
  return MQ_OK;
}

int mq_philox_fill(uint64_t seed, uint64_t epoch, uint32_t batch, uint32_t hop, uint32_t row,
                   uint32_t count, uint32_t* out_dev, void* stream) {
  if (count == 0) return MQ_OK;
  MQ_CHECK_ARG(out_dev != nullptr, "mq_philox_fill: null out");
  cudaStream_t s = as_stream(stream);
  uint32_t blocks = (count + 3) / 4;
  {
    ProfScope ps(K_PHILOX, s);
    philox_fill_kernel<<<ceil_div(blocks, 256), 256, 0, s>>>(seed, epoch, batch, hop, row, count,
                                                             out_dev);
  }
  MQ_LAUNCH_CHECK("philox_fill");
  return MQ_OK;
}

int mq_fisher_yates_host(uint64_t seed, uint64_t epoch, uint32_t batch, uint32_t hop, uint32_t row,
                         int64_t n, int32_t k, int64_t* pos_out) {
  MQ_CHECK_ARG(k >= 0 && k <= MQ_MAX_FANOUT, "mq_fisher_yates_host: k=%d out of range", k);
  MQ_CHECK_ARG(k <= n, "mq_fisher_yates_host: k=%d > n=%lld", k, (long long)n);
  RowStream rs(seed, epoch, batch, hop, row);
  fisher_yates<MQ_MAX_FANOUT, int64_t>(rs, n, k, pos_out);
  return MQ_OK;
}

int64_t mq_scan_scratch_bytes(int64_t n_max) { return scan_scratch_bytes(n_max < 1 ? 1 : n_max); }

int mq_strip_self_loops(const int64_t* row_off, const int32_t* col, int64_t n_nodes, int64_t n_arcs,
                        int64_t* out_row_off, int32_t* out_col, void* scratch, void* stream) {
  MQ_CHECK_ARG(row_off && out_row_off && scratch, "mq_strip_self_loops: null pointer");
  MQ_CHECK_ARG(n_nodes >= 0 && n_arcs >= 0, "mq_strip_self_loops: negative size");
  cudaStream_t s = as_stream(stream);
  int rc = launch_scan(LoadKeep{row_off, col, n_nodes}, StoreOffsets<int64_t>{out_row_off}, n_nodes,
                       scratch, s, K_STRIP_FLAGS);
  if (rc) return rc;
  if (n_nodes == 0) return MQ_OK;
  {
    ProfScope ps(K_STRIP_FLAGS, s);
    strip_copy_kernel<<<ceil_div(n_nodes * 32, 256), 256, 0, s>>>(row_off, col, n_nodes, out_row_off,
                                                                  out_col);
  }
  MQ_LAUNCH_CHECK("strip_copy");
  return MQ_OK;
}

int mq_residency_index(const int64_t* row_off, const int32_t* col, int64_t n_nodes, int64_t n_arcs,
                       const uint32_t* resident_bits, int64_t* hot_arc, int64_t* hot_off,
                       int64_t* n_hot_dev, void* scratch, void* stream) {
  MQ_CHECK_ARG(row_off && resident_bits && hot_off && n_hot_dev && scratch,
               "mq_residency_index: null pointer");
  cudaStream_t s = as_stream(stream);
  int rc = launch_scan(LoadHotArc{col, resident_bits, n_arcs}, StoreHotArc{hot_arc, n_hot_dev},
                       n_arcs, scratch, s, K_RESIDENCY_COMPACT);
  if (rc) return rc;
  {
    ProfScope ps(K_RESIDENCY_OFFSETS, s);
    residency_offsets_kernel<<<ceil_div(n_nodes + 1, 256), 256, 0, s>>>(row_off, n_nodes, hot_arc,
                                                                        n_hot_dev, hot_off);
  }
  MQ_LAUNCH_CHECK("residency_offsets");
  return MQ_OK;
}

int mq_residency_slots(const uint32_t* resident_bits, int64_t n_nodes, int32_t* slot_of,
                       int32_t* n_resident_dev, void* scratch, void* stream) {
  MQ_CHECK_ARG(resident_bits && slot_of && n_resident_dev && scratch,
               "mq_residency_slots: null pointer");
  return launch_scan(LoadBit{resident_bits, n_nodes}, StoreSlot{slot_of, n_resident_dev}, n_nodes,
                     scratch, as_stream(stream), K_RESIDENCY_SLOTS);
}

int mq_sample_hop(const int64_t* row_off, const int32_t* col, const int64_t* hot_arc,
                  const int64_t* hot_off, const int32_t* dst, const int32_t* n_dst_dev,
                  int32_t n_dst_max, int32_t fanout, uint64_t seed, uint64_t epoch, uint32_t batch,
                  uint32_t hop, const uint32_t* key_dev, int32_t* nbr, int32_t* cnt,
                  void* stream) {
  MQ_CHECK_ARG(fanout >= 1 && fanout <= MQ_MAX_FANOUT, "mq_sample_hop: fanout %d not in [1, %d]",
               fanout, MQ_MAX_FANOUT);
  MQ_CHECK_ARG((hot_arc == nullptr) == (hot_off == nullptr),
               "mq_sample_hop: hot_arc and hot_off must both be set or both NULL");
  MQ_CHECK_ARG(row_off && dst && n_dst_dev && nbr && cnt, "mq_sample_hop: null pointer");
  if (n_dst_max <= 0) return MQ_OK;
  cudaStream_t s = as_stream(stream);
  {
    ProfScope ps(K_SAMPLE, s);
    if (fanout <= 16)
      sample_hop_kernel<16><<<ceil_div(n_dst_max, 128), 128, 0, s>>>(
          row_off, col, hot_arc, hot_off, dst, n_dst_dev, fanout, seed, epoch, batch, hop, key_dev, nbr,
          cnt);
    else
      sample_hop_kernel<MQ_MAX_FANOUT><<<ceil_div(n_dst_max, 128), 128, 0, s>>>(
          row_off, col, hot_arc, hot_off, dst, n_dst_dev, fanout, seed, epoch, batch, hop, key_dev, nbr,
          cnt);
  }
  MQ_LAUNCH_CHECK("sample_hop");
  return MQ_OK;
}

int mq_batch_setup(const int32_t* perm, int64_t n_perm, int32_t batch_size, int32_t world,
                   int32_t rank, int32_t* cursor_dev, int32_t* targets, int32_t* n_targets_dev,
                   uint32_t* key_dev, void* stream) {
  MQ_CHECK_ARG(perm && cursor_dev && targets && n_targets_dev && key_dev,
               "mq_batch_setup: null pointer");
  MQ_CHECK_ARG(batch_size >= 1 && world >= 1 && rank >= 0 && rank < world,
               "mq_batch_setup: bad batch_size/world/rank");
  cudaStream_t s = as_stream(stream);
  {
    ProfScope ps(K_BATCH_SETUP, s);
    batch_setup_kernel<<<1, 256, 0, s>>>(perm, n_perm, batch_size, world, rank, cursor_dev, targets,
                                         n_targets_dev, key_dev);
  }
  MQ_LAUNCH_CHECK("batch_setup");
  return MQ_OK;
}

int64_t mq_relabel_scratch_bytes(int32_t n_dst_max, int32_t fanout) {
  int64_t slots = (int64_t)(n_dst_max < 1 ? 1 : n_dst_max) * (fanout < 1 ? 1 : fanout);
  return scan_scratch_bytes(slots);
}

int mq_relabel(const int32_t* dst, const int32_t* n_dst_dev, int32_t n_dst_max, const int32_t* nbr,
               const int32_t* cnt, int32_t fanout, int32_t* dpos_tbl, int32_t* first_tbl,
               int32_t* row_ptr, int32_t* rows, int32_t* cols, float* vals, int32_t* src_ids,
               int32_t* counts_dev, void* scratch, void* stream) {
  MQ_CHECK_ARG(fanout >= 1 && fanout <= MQ_MAX_FANOUT, "mq_relabel: bad fanout %d", fanout);
  MQ_CHECK_ARG(dst && n_dst_dev && nbr && cnt && dpos_tbl && first_tbl && row_ptr && rows && cols &&
                   vals && src_ids && counts_dev && scratch,
               "mq_relabel: null pointer");
  cudaStream_t s = as_stream(stream);
  const int32_t nd = n_dst_max < 1 ? 1 : n_dst_max;
  const int64_t slots = (int64_t)nd * fanout;
  int rc = launch_scan(LoadI32{cnt, n_dst_dev, 0}, StoreRowPtr{row_ptr, counts_dev}, nd, scratch, s);
  if (rc) return rc;
  {
    ProfScope ps(K_RELABEL_MARK, s);
    relabel_mark_kernel<<<ceil_div(nd, 256), 256, 0, s>>>(dst, n_dst_dev, dpos_tbl, src_ids);
  }
  MQ_LAUNCH_CHECK("relabel_mark");
  {
    ProfScope ps(K_RELABEL_FIRST, s);
    relabel_first_kernel<<<ceil_div(slots, 256), 256, 0, s>>>(nbr, cnt, row_ptr, n_dst_dev, fanout,
                                                              dpos_tbl, first_tbl);
  }
  MQ_LAUNCH_CHECK("relabel_first");
  rc = launch_scan(LoadFirstFlag{nbr, cnt, row_ptr, n_dst_dev, dpos_tbl, first_tbl, fanout},
                   StoreLabel{nbr, n_dst_dev, dpos_tbl, src_ids, counts_dev}, slots, scratch, s,
                   K_RELABEL_FLAG);
  if (rc) return rc;
  {
    ProfScope ps(K_RELABEL_COLS, s);
    relabel_cols_kernel<<<ceil_div(slots, 256), 256, 0, s>>>(nbr, cnt, row_ptr, n_dst_dev, fanout,
                                                             dpos_tbl, rows, cols, vals);
  }
  MQ_LAUNCH_CHECK("relabel_cols");
  {
    ProfScope ps(K_RELABEL_CLEAN, s);
    relabel_clean_kernel<<<ceil_div(slots + nd, 256), 256, 0, s>>>(src_ids, counts_dev, n_dst_dev,
                                                                   dpos_tbl, first_tbl);
  }
  MQ_LAUNCH_CHECK("relabel_clean");
  return MQ_OK;
}

}  // extern "C"
