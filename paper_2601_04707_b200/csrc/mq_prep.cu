// Multi-queue batch preparation: sample -> relabel -> gather for Q batches in
// ONE pass (one launch per stage for all Q batches).
//
// MQ-GNN keeps a queue of prepared mini-batches ahead of the trainer
// (runtime.py:380-612, BoundedQueue pipeline.py:109-167).  Here the queue is a
// group of Q device slots filled by one pass of batched kernels: blockIdx.y
// selects the slot, so each stage's latency (dependent CSR loads, look-back
// scans) is paid once per Q batches instead of once per batch, and each
// launch has Q times the parallelism.
//
// Per slot the semantics are exactly the single-batch entry points':
// mq_batch_setup (runtime.py:95-124), mq_sample_hop (samplers.py:159-200),
// mq_relabel (samplers.py:155-156, 186-200), mq_gather (cache.py:123-134,
// runtime.py:127-143) and mq_gather_labels (samplers.py:532) — bit-identical
// blocks, ids and features for the same (seed, epoch, batch) key.
#include <climits>

#include "mq_common.cuh"
#include "mq_scan.cuh"

namespace mq {
namespace prep {

// The relabel keeps ONE int32 word per node and slot (mq_prep_desc.node_rank,
// INT32_MAX at rest), so a products-sized table (8 slots x 2.4M nodes x 4 B)
// stays L2-resident (RankTbl below: a hash of the touched nodes instead when
// the node-indexed table would not fit):
//   w[u] = -(p + 1)  u is in the current src list at position p (dst marks
//                    -(r + 1) and new labels are both stored this way);
//   w[u] = s >= 0    u's first pick slot s = r * fanout + i this hop
//                    (atomicMin: the slot order is the triplet order);
//   w[u] = INT32_MAX u untouched.
// Marks and picks are both atomicMin (order-free); a scan tile flags u iff
// w[u] == s, which no stored label (negative) can alias.  The next hop's dst
// list is this hop's src list, so its marks are already in place: only hop 0
// marks.
template <class T>
struct QP {
  T* p;
  int64_t s;  // elements between consecutive slots
  __host__ __device__ __forceinline__ T* at(int q) const { return p + (int64_t)q * s; }
};

template <class T>
inline QP<T> qp(T* p, int64_t s) {
  return QP<T>{p, s};
}

// The rank words of one slot: node-indexed (lg == 0: word of u at [u]) or,
// for graphs whose node-indexed tables would span GBs (8 slots x 111M nodes),
// an open-addressing hash of 2^lg (key, word) pairs -- key u + 1 (0 = empty)
// at [2h], its word at [2h + 1], linear probing from a multiplicative home --
// followed by hpos[position] = the entry of the src list's node at that
// position (the restore walks it: deleting entries by lookup would cut the
// probe chains of entries not yet deleted).  The same words, the same
// atomics and the same scan: only the address of a node's word changes.
struct RankTbl {
  int32_t* base;
  int64_t s;  // int32 elements between slots
  int lg;     // 0: node-indexed
  __device__ __forceinline__ int32_t* slot(int q) const { return base + (int64_t)q * s; }
  __device__ __forceinline__ uint32_t home(int32_t u) const {
    return ((uint32_t)u * 0x9E3779B1u) >> (32 - lg);
  }
  // entry of u, which some earlier access of this pass inserted
  __device__ __forceinline__ uint32_t find(int q, int32_t u) const {
    const int32_t* t = slot(q);
    const uint32_t m = (1u << lg) - 1;
    uint32_t h = home(u);
    while (__ldcg(t + 2 * h) != u + 1) h = (h + 1) & m;
    return h;
  }
  // entry of u, inserted if absent (concurrent inserts of u agree on one)
  __device__ __forceinline__ uint32_t claim(int q, int32_t u) const {
    int32_t* t = slot(q);
    const uint32_t m = (1u << lg) - 1;
    uint32_t h = home(u);
    for (;;) {
      const int32_t k = __ldcg(t + 2 * h);
      if (k == u + 1) return h;
      if (k == 0) {
        const int32_t old = atomicCAS(t + 2 * h, 0, u + 1);
        if (old == 0 || old == u + 1) return h;
      }
      h = (h + 1) & m;
    }
  }
  __device__ __forceinline__ int32_t* word(int q, int32_t u, bool insert) const {
    if (lg == 0) return slot(q) + u;
    return slot(q) + 2 * (insert ? claim(q, u) : find(q, u)) + 1;
  }
  __device__ __forceinline__ int32_t* hpos(int q) const { return slot(q) + (2ll << lg); }
  // the word of u for a node taking src position p (records hpos[p])
  __device__ __forceinline__ int32_t* word_at(int q, int32_t u, int32_t p, bool insert) const {
    if (lg == 0) return slot(q) + u;
    const uint32_t h = insert ? claim(q, u) : find(q, u);
    hpos(q)[p] = (int32_t)h;
    return slot(q) + 2 * h + 1;
  }
};

// ------------------------------------------------------------ batch setup
// slot q <- window cursor[0] + q: batch j = window*world + rank (round-robin
// deal, runtime.py:111-113), targets = perm[j*B, min(n_perm, (j+1)*B)).  The
// last block to finish advances the cursor by Q (cursor[1] = arrival count).
__global__ void setup_q_kernel(const int32_t* __restrict__ perm, int64_t n_perm, int B, int world,
                               int rank, int32_t* __restrict__ cursor, QP<int32_t> targets,
                               QP<int32_t> n_targets, QP<uint32_t> key) {
  const int q = blockIdx.y;
  __shared__ int64_t s_begin;
  __shared__ int s_len;
  if (threadIdx.x == 0) {
    const int64_t window = (int64_t)cursor[0] + q;
    const int64_t j = window * world + rank;
    const int64_t b = j * B;
    int64_t len = n_perm - b;
    len = len < 0 ? 0 : (len > B ? B : len);
    s_begin = b;
    s_len = (int)len;
    n_targets.at(q)[0] = (int32_t)len;
    key.at(q)[2] = (uint32_t)j;
  }
  __syncthreads();
  int32_t* t = targets.at(q);
  for (int i = threadIdx.x; i < s_len; i += blockDim.x) t[i] = __ldg(&perm[s_begin + i]);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&cursor[1], 1) == (int)gridDim.y - 1) {
      cursor[0] += (int)gridDim.y;
      cursor[1] = 0;
    }
  }
}

#ifndef MQ_SAMPLE_MINB
#define MQ_SAMPLE_MINB 12  // >= 12 resident 64-thread blocks per SM (register cap): products sample 27 -> 24 us/batch
#endif
#ifndef MQ_SAMPLE_MINB8
#define MQ_SAMPLE_MINB8 20  // fanout <= 8: smaller per-row arrays, more rows in flight per SM
#endif

// ------------------------------------------------------------ sample
// One thread per dst row (node_wise_block, SAGE arm).  Every case is O(fanout)
// through the per-epoch residency index; the row's gathers are issued from
// register arrays so a row costs ~4 dependent round trips
// (dst -> offsets -> hot arcs -> columns), not 2*fanout.
// With `tbl` the kernel also does the relabel's per-row bookkeeping (the
// sampled rows are independent of it): the src_ids prefix and, at hop 0,
// the dst mark (w[v] = -(max row + 1), samplers.py:155-156), and every
// pick's first-occurrence slot (w[u] = min over slots r * fanout + i: the
// slot order is the triplet order, so the minimum is the first occurrence,
// samplers.py:186-189).
struct RelabelTables {
  RankTbl w;
  QP<int32_t> src_ids;
  bool on, mark;
};

template <int MAXK>
__global__ void __launch_bounds__(64, MAXK <= 8 ? MQ_SAMPLE_MINB8 : MQ_SAMPLE_MINB) sample_q_kernel(
    const int64_t* __restrict__ row_off, const int32_t* __restrict__ col,
    const int64_t* __restrict__ hot_arc, const int64_t* __restrict__ hot_off, QP<const int32_t> dst,
    QP<const int32_t> n_dst, QP<const uint32_t> key, int fanout, uint32_t hop, QP<int32_t> nbr,
    QP<int32_t> cnt, RelabelTables tbl) {
  const int q = blockIdx.y;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= *n_dst.at(q)) return;
  const uint32_t* k = key.at(q);
  const int32_t v = dst.at(q)[r];
  if (tbl.on) {
    tbl.src_ids.at(q)[r] = v;
    if (tbl.mark) atomicMin(tbl.w.word_at(q, v, r, true), -(r + 1));
  }
  const int64_t beg = row_off[v];
  const int n = (int)(row_off[v + 1] - beg);
  int64_t hb = 0;
  int nh = 0;
  if (hot_off != nullptr) {
    hb = hot_off[v];
    nh = (int)(hot_off[v + 1] - hb);
  }
  int32_t* out = nbr.at(q) + (int64_t)r * fanout;
  int32_t x[MAXK];
  if (n <= fanout) {  // samplers.py:164-167: every neighbour, CSR order
#pragma unroll
    for (int i = 0; i < MAXK; ++i) x[i] = i < n ? __ldg(&col[beg + i]) : 0;
#pragma unroll
    for (int i = 0; i < MAXK; ++i)
      if (i < n) out[i] = x[i];
    if (tbl.on) {
#pragma unroll
      for (int i = 0; i < MAXK; ++i)
        if (i < n) atomicMin(tbl.w.word(q, x[i], true), r * fanout + i);
    }
    cnt.at(q)[r] = n;
    return;
  }
  RowStream rs(k[0], k[1], k[2], hop, (uint32_t)r);
  int pos[MAXK];
  if (hot_off != nullptr && nh >= fanout) {  // samplers.py:171-172: choice(hot, f)
    fisher_yates<MAXK, int>(rs, nh, fanout, pos);
    int64_t arc[MAXK];
#pragma unroll
    for (int j = 0; j < MAXK; ++j) arc[j] = j < fanout ? __ldg(&hot_arc[hb + pos[j]]) : 0;
#pragma unroll
    for (int j = 0; j < MAXK; ++j) x[j] = j < fanout ? __ldg(&col[arc[j]]) : 0;
#pragma unroll
    for (int j = 0; j < MAXK; ++j)
      if (j < fanout) out[j] = x[j];
    if (tbl.on) {
#pragma unroll
      for (int j = 0; j < MAXK; ++j)
        if (j < fanout) atomicMin(tbl.w.word(q, x[j], true), r * fanout + j);
    }
  } else if (hot_off != nullptr) {  // samplers.py:173-175: hot ++ choice(cold, f - |hot|)
    int64_t ha[MAXK];
#pragma unroll
    for (int i = 0; i < MAXK; ++i) ha[i] = i < nh ? __ldg(&hot_arc[hb + i]) : 0;
    const int k2 = fanout - nh;
    fisher_yates<MAXK, int>(rs, n - nh, k2, pos);
    int64_t ca[MAXK];
#pragma unroll
    for (int j = 0; j < MAXK; ++j) {
      // cold rank -> row position: skip every hot position h_i with h_i - i <= rank
      const int rr = j < k2 ? pos[j] : 0;
      int c = 0;
#pragma unroll
      for (int i = 0; i < MAXK; ++i) c += (i < nh && (int)(ha[i] - beg) - i <= rr) ? 1 : 0;
      ca[j] = beg + rr + c;
    }
    int32_t y[MAXK];
#pragma unroll
    for (int i = 0; i < MAXK; ++i) x[i] = i < nh ? __ldg(&col[ha[i]]) : 0;
#pragma unroll
    for (int j = 0; j < MAXK; ++j) y[j] = j < k2 ? __ldg(&col[ca[j]]) : 0;
#pragma unroll
    for (int i = 0; i < MAXK; ++i)
      if (i < nh) out[i] = x[i];
#pragma unroll
    for (int j = 0; j < MAXK; ++j)
      if (j < k2) out[nh + j] = y[j];
    if (tbl.on) {
#pragma unroll
      for (int i = 0; i < MAXK; ++i)
        if (i < nh) atomicMin(tbl.w.word(q, x[i], true), r * fanout + i);
#pragma unroll
      for (int j = 0; j < MAXK; ++j)
        if (j < k2) atomicMin(tbl.w.word(q, y[j], true), r * fanout + nh + j);
    }
  } else {  // samplers.py:176-177: choice(nbrs, f)
    fisher_yates<MAXK, int>(rs, n, fanout, pos);
#pragma unroll
    for (int j = 0; j < MAXK; ++j) x[j] = j < fanout ? __ldg(&col[beg + pos[j]]) : 0;
#pragma unroll
    for (int j = 0; j < MAXK; ++j)
      if (j < fanout) out[j] = x[j];
    if (tbl.on) {
#pragma unroll
      for (int j = 0; j < MAXK; ++j)
        if (j < fanout) atomicMin(tbl.w.word(q, x[j], true), r * fanout + j);
    }
  }
  cnt.at(q)[r] = fanout;
}

// ------------------------------------------------------------ relabel
__global__ void mark_q_kernel(QP<const int32_t> dst, QP<const int32_t> n_dst, RankTbl w,
                              QP<int32_t> src_ids, bool mark) {
  const int q = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *n_dst.at(q)) return;
  const int32_t v = dst.at(q)[i];
  src_ids.at(q)[i] = v;
  if (mark) atomicMin(w.word_at(q, v, i, true), -(i + 1));
}

// w[u] = min slot r * fanout + i of every pick u (sample_q_kernel does
// this inline; this kernel serves passes whose sampling ran separately)
__global__ void first_q_kernel(QP<const int32_t> nbr, QP<const int32_t> cnt,
                               QP<const int32_t> n_dst, int fanout, RankTbl w) {
  const int q = blockIdx.y;
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int r = (int)(s / fanout), i = (int)(s % fanout);
  if (r >= *n_dst.at(q) || i >= cnt.at(q)[r]) return;
  atomicMin(w.word(q, nbr.at(q)[s], true), (int32_t)s);
}

// One scan per hop over the slots r * fanout + i, two channels in one int64:
// high 32 bits = the row's triplet count at its first slot (prefix ->
// row_ptr), low 32 bits = the first-occurrence flag of a new node (prefix ->
// its label) -- the row offsets and the labels in one decoupled-look-back pass.
struct QLoadRowFlag {
  QP<const int32_t> nbr, cnt, n_dst;
  RankTbl w;
  int fanout;
  __device__ int64_t size() const { return (int64_t)(*n_dst.at(blockIdx.y)) * fanout; }
  __device__ int64_t operator()(int64_t s) const {
    const int q = blockIdx.y;
    const int r = (int)(s / fanout), i = (int)(s % fanout);
    const int c = cnt.at(q)[r];
    int64_t v = i == 0 ? ((int64_t)c << 32) : 0;
    if (i < c) {
      if (__ldcg(w.word(q, nbr.at(q)[s], false)) == (int32_t)s) v |= 1;
    }
    return v;
  }
};
struct QStoreRowLabel {
  QP<const int32_t> nbr, n_dst;
  RankTbl w;
  QP<int32_t> src_ids, counts, row_ptr;
  int fanout;
  __device__ void operator()(int64_t s, int64_t excl, int64_t val) const {
    const int q = blockIdx.y;
    if (s % fanout == 0) row_ptr.at(q)[s / fanout] = (int32_t)(excl >> 32);
    if (!(val & 1)) return;
    const int32_t u = nbr.at(q)[s];
    const int32_t lab = *n_dst.at(q) + (int32_t)(excl & 0xFFFFFFFFll);
    src_ids.at(q)[lab] = u;
    *w.word_at(q, u, lab, false) = -(lab + 1);
  }
  __device__ void total(int64_t, int64_t t) const {
    const int q = blockIdx.y;
    const int nd = *n_dst.at(q);
    row_ptr.at(q)[nd] = (int32_t)(t >> 32);
    counts.at(q)[1] = (int32_t)(t >> 32);
    counts.at(q)[0] = nd + (int32_t)(t & 0xFFFFFFFFll);
  }
};
__global__ void cols_q_kernel(QP<const int32_t> nbr, QP<const int32_t> cnt,
                              QP<const int32_t> row_ptr, QP<const int32_t> n_dst, int fanout,
                              RankTbl w, QP<int32_t> rows, QP<int32_t> cols,
                              QP<float> vals) {
  const int q = blockIdx.y;
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int r = (int)(s / fanout), i = (int)(s % fanout);
  if (r >= *n_dst.at(q)) return;
  const int c = cnt.at(q)[r];
  if (i >= c) return;
  const int e = row_ptr.at(q)[r] + i;
  rows.at(q)[e] = r;
  cols.at(q)[e] = -(*w.word(q, nbr.at(q)[s], false) + 1);
  vals.at(q)[e] = (float)(1.0 / (double)c);  // float32(1.0 / s), samplers.py:200 + nn.py:85
}

// Table restore, once per pass: every node a hop touched (dst marks, new
// labels, first-occurrence slots of any pick) is in that hop's src list, and
// each hop's src list contains the previous one's, so the last hop's src list
// covers them all.
__global__ void clean_q_kernel(QP<const int32_t> src_ids, QP<const int32_t> counts, RankTbl w) {
  const int q = blockIdx.y;
  const int n = counts.at(q)[0];
  int32_t* t = w.slot(q);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    if (w.lg == 0) {
      t[src_ids.at(q)[j]] = INT_MAX;
    } else {  // (duplicate hop-0 targets share an entry: restored twice, harmlessly)
      const int32_t h = w.hpos(q)[j];
      t[2 * h] = 0;
      t[2 * h + 1] = INT_MAX;
    }
  }
}

// ------------------------------------------------------------ gather
constexpr int kGatherThreads = 256;

__global__ void __launch_bounds__(kGatherThreads) gather_q_kernel(
    const float* __restrict__ cache_tbl, int cache_pitch, const int32_t* __restrict__ slot_of,
    StoreRef store, QP<const int32_t> ids, QP<const int32_t> n_dev,
    int d4, QP<float> out, int out_pitch, unsigned long long* __restrict__ hit_miss) {
  __shared__ unsigned int s_hits, s_miss;
  if (threadIdx.x == 0) {
    s_hits = 0;
    s_miss = 0;
  }
  __syncthreads();
  const int q = blockIdx.y;
  const int n = *n_dev.at(q);
  const int32_t* idq = ids.at(q);
  float* outq = out.at(q);
  const int lane = threadIdx.x & 31;
  const int warps = kGatherThreads / 32;
  // A warp takes 32 rows at a time: lane i resolves row i's id, cache slot
  // and source pointer (the dependent loads of all 32 rows in flight at once),
  // then the warp copies the rows kRowsInFlight at a time, lanes over the
  // row's 16-byte chunks (coalesced).
  // Rows wider than 512 B (Reddit's 602-d) keep one row per warp pass with
  // four 16-byte chunks per lane in flight.
  constexpr int kRowsInFlight = 4;
  unsigned int hits = 0, miss = 0;
  if (d4 > 32) {
    int64_t row = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5);
    const int64_t rstride = (int64_t)gridDim.x * warps;
    for (; row < n; row += rstride) {
      const int32_t id = idq[row];
      const float4* src;
      const int32_t slot = slot_of ? slot_of[id] : -1;
      if (slot >= 0) {
        src = reinterpret_cast<const float4*>(cache_tbl + (int64_t)slot * cache_pitch);
        ++hits;
      } else {
        src = reinterpret_cast<const float4*>(store.row(id));
        ++miss;
      }
      float4* dst = reinterpret_cast<float4*>(outq + row * out_pitch);
      int c = lane;
      for (; c + 96 < d4; c += 128) {
        const float4 a = src[c], b = src[c + 32], e = src[c + 64], f = src[c + 96];
        dst[c] = a;
        dst[c + 32] = b;
        dst[c + 64] = e;
        dst[c + 96] = f;
      }
      for (; c < d4; c += 32) dst[c] = src[c];
    }
  }
  int64_t row0 = ((int64_t)blockIdx.x * warps + (threadIdx.x >> 5)) * 32;
  const int64_t stride = (int64_t)gridDim.x * warps * 32;
  for (; d4 <= 32 && row0 < n; row0 += stride) {
    const int m = (int)min((int64_t)32, (int64_t)n - row0);
    const float4* my_src = nullptr;
    bool hit = false;
    if (lane < m) {
      const int32_t id = idq[row0 + lane];
      const int32_t slot = slot_of ? slot_of[id] : -1;
      hit = slot >= 0;
      my_src = hit ? reinterpret_cast<const float4*>(cache_tbl + (int64_t)slot * cache_pitch)
                   : reinterpret_cast<const float4*>(store.row(id));
    }
    // warp-uniform counts (lane 0 reports them, as on the wide path)
    const unsigned hb = __ballot_sync(0xffffffffu, hit);
    hits += __popc(hb);
    miss += (unsigned)m - __popc(hb);
    const unsigned long long my_addr = reinterpret_cast<unsigned long long>(my_src);
    for (int j = 0; j < m; j += kRowsInFlight) {
      const float4* src[kRowsInFlight];
#pragma unroll
      for (int u = 0; u < kRowsInFlight; ++u)
        src[u] = reinterpret_cast<const float4*>(__shfl_sync(0xffffffffu, my_addr, (j + u) & 31));
      for (int c = lane; c < d4; c += 32) {
        float4 v[kRowsInFlight];
#pragma unroll
        for (int u = 0; u < kRowsInFlight; ++u)
          if (j + u < m) v[u] = src[u][c];
#pragma unroll
        for (int u = 0; u < kRowsInFlight; ++u)
          if (j + u < m) reinterpret_cast<float4*>(outq + (row0 + j + u) * out_pitch)[c] = v[u];
      }
    }
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

__global__ void labels_q_kernel(const int32_t* __restrict__ all_labels, QP<const int32_t> ids,
                                QP<const int32_t> n_dev, QP<int32_t> out) {
  const int q = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < *n_dev.at(q)) out.at(q)[i] = all_labels[ids.at(q)[i]];
}

template <class T>
inline QP<const T> cq(T* p, int64_t s) {
  return QP<const T>{p, s};
}

}  // namespace prep
}  // namespace mq

using namespace mq;
using namespace mq::prep;

extern "C" {

int64_t mq_prep_scratch_bytes(int32_t n_dst_max, int32_t fanout) {
  const int64_t slots = (int64_t)(n_dst_max < 1 ? 1 : n_dst_max) * (fanout < 1 ? 1 : fanout);
  // 256-byte aligned per-slot region of the scan ticket/status words
  return (scan_scratch_bytes(slots) + 255) / 256 * 256;
}

int mq_prep_batches(const mq_prep_desc* pd, void* stream) {
  MQ_CHECK_ARG(pd != nullptr, "mq_prep_batches: null descriptor");
  const mq_prep_desc& d = *pd;
  const int Q = d.nslots;
  MQ_CHECK_ARG(Q >= 1 && Q <= 65535, "mq_prep_batches: nslots %d out of range", Q);
  MQ_CHECK_ARG(d.num_hops >= 1 && d.num_hops <= MQ_MAX_HOPS, "mq_prep_batches: num_hops %d",
               d.num_hops);
  MQ_CHECK_ARG(d.row_off && d.col && d.targets && d.n_targets && d.key && d.node_rank &&
                   d.scratch && (d.store || d.n_shards >= 1) && d.x0 && d.all_labels && d.labels,
               "mq_prep_batches: null pointer");
  MQ_CHECK_ARG(d.n_shards >= 0 && d.n_shards <= MQ_MAX_PEERS, "mq_prep_batches: n_shards %d",
               d.n_shards);
  for (int q = 0; q < d.n_shards; ++q)
    MQ_CHECK_ARG(d.store_shard[q] && (uintptr_t)d.store_shard[q] % 16 == 0,
                 "mq_prep_batches: shard %d missing or unaligned", q);
  MQ_CHECK_ARG((d.hot_arc == nullptr) == (d.hot_off == nullptr),
               "mq_prep_batches: hot_arc / hot_off must both be set or both NULL");
  MQ_CHECK_ARG(!d.slot_of || (d.cache_tbl && d.hit_miss), "mq_prep_batches: cache without table");
  const int dv4 = (d.d + 3) / 4;
  MQ_CHECK_ARG(d.d >= 1 && d.store_pitch % 4 == 0 && d.x0_pitch % 4 == 0 &&
                   d.store_pitch >= 4 * dv4 && d.x0_pitch >= 4 * dv4 &&
                   (!d.slot_of || (d.cache_pitch % 4 == 0 && d.cache_pitch >= 4 * dv4)),
               "mq_prep_batches: feature pitches must be multiples of 4 covering d");
  cudaStream_t s = as_stream(stream);
  const uint32_t mask = d.stage_mask ? d.stage_mask : 0xFFFFFFFFu;

  // 1. device batch plan (skipped when the host staged targets/keys)
  if (d.cursor != nullptr && (mask & MQ_PREP_SETUP)) {
    MQ_CHECK_ARG(d.perm && d.batch_size >= 1 && d.world >= 1 && d.rank >= 0 && d.rank < d.world,
                 "mq_prep_batches: bad batch plan");
    {
      ProfScope ps(K_BATCH_SETUP, s);
      setup_q_kernel<<<dim3(1, Q), 256, 0, s>>>(d.perm, d.n_perm, d.batch_size, d.world, d.rank,
                                                d.cursor, qp(d.targets, d.targets_s),
                                                qp(d.n_targets, d.n_targets_s),
                                                qp(d.key, d.key_s));
    }
    MQ_LAUNCH_CHECK("prep setup");
  }

  MQ_CHECK_ARG(d.hash_lg == 0 || (d.hash_lg >= 4 && d.hash_lg <= 30 &&
                                   d.table_s >= (2ll << d.hash_lg) +
                                                    d.hop[d.num_hops - 1].n_src_max),
               "mq_prep_batches: hash_lg %d does not fit table_s", d.hash_lg);
  const RankTbl rt{d.node_rank, d.table_s, d.hash_lg};

  // 2. hops: sample + relabel (samplers.py:213-226 hop chain)
  for (int h = 0; h < d.num_hops; ++h) {
    const mq_prep_hop& hp = d.hop[h];
    MQ_CHECK_ARG(hp.fanout >= 1 && hp.fanout <= MQ_MAX_FANOUT && hp.n_dst_max >= 1,
                 "mq_prep_batches: hop %d bad fanout / bound", h);
    MQ_CHECK_ARG(hp.nbr && hp.cnt && hp.row_ptr && hp.rows && hp.cols && hp.vals && hp.src_ids &&
                     hp.counts,
                 "mq_prep_batches: hop %d null buffer", h);
    const int32_t* dst = h == 0 ? d.targets : d.hop[h - 1].src_ids;
    const int64_t dst_s = h == 0 ? d.targets_s : d.hop[h - 1].src_s;
    const int32_t* nd = h == 0 ? d.n_targets : d.hop[h - 1].counts;  // counts[0] = n_src
    const int64_t nd_s = h == 0 ? d.n_targets_s : d.hop[h - 1].counts_s;
    const int f = hp.fanout;
    const int64_t slots = (int64_t)hp.n_dst_max * f;
    const bool relabel = (mask & MQ_PREP_RELABEL) != 0;
    if (mask & MQ_PREP_SAMPLE) {
      ProfScope ps(K_SAMPLE, s);
      const dim3 grid(ceil_div(hp.n_dst_max, 64), Q);
      const RelabelTables tb{rt, qp(hp.src_ids, hp.src_s), relabel, h == 0};
      if (f <= 8)
        sample_q_kernel<8><<<grid, 64, 0, s>>>(
            d.row_off, d.col, d.hot_arc, d.hot_off, cq(dst, dst_s), cq(nd, nd_s),
            cq(d.key, d.key_s), f, (uint32_t)h, qp(hp.nbr, hp.nbr_s), qp(hp.cnt, hp.cnt_s), tb);
      else if (f <= 16)
        sample_q_kernel<16><<<grid, 64, 0, s>>>(
            d.row_off, d.col, d.hot_arc, d.hot_off, cq(dst, dst_s), cq(nd, nd_s),
            cq(d.key, d.key_s), f, (uint32_t)h, qp(hp.nbr, hp.nbr_s), qp(hp.cnt, hp.cnt_s), tb);
      else
        sample_q_kernel<MQ_MAX_FANOUT><<<grid, 64, 0, s>>>(
            d.row_off, d.col, d.hot_arc, d.hot_off, cq(dst, dst_s), cq(nd, nd_s),
            cq(d.key, d.key_s), f, (uint32_t)h, qp(hp.nbr, hp.nbr_s), qp(hp.cnt, hp.cnt_s), tb);
    } else if (relabel) {  // sampled earlier: the relabel's marks and first slots alone
      ProfScope ps(K_RELABEL_MARK, s);
      mark_q_kernel<<<dim3(ceil_div(hp.n_dst_max, 256), Q), 256, 0, s>>>(
          cq(dst, dst_s), cq(nd, nd_s), rt, qp(hp.src_ids, hp.src_s), h == 0);
      first_q_kernel<<<dim3(ceil_div(slots, 256), Q), 256, 0, s>>>(
          cq(hp.nbr, hp.nbr_s), cq(hp.cnt, hp.cnt_s), cq(nd, nd_s), f, rt);
    }
    MQ_LAUNCH_CHECK("prep sample");
    if (!relabel) continue;
    int rc = launch_scan_q(
        QLoadRowFlag{cq(hp.nbr, hp.nbr_s), cq(hp.cnt, hp.cnt_s), cq(nd, nd_s), rt, f},
        QStoreRowLabel{cq(hp.nbr, hp.nbr_s), cq(nd, nd_s), rt,
                       qp(hp.src_ids, hp.src_s), qp(hp.counts, hp.counts_s),
                       qp(hp.row_ptr, hp.row_ptr_s), f},
        slots, Q, d.scratch, d.scratch_s, s, K_RELABEL_FLAG);
    if (rc) return rc;
    {
      ProfScope ps(K_RELABEL_COLS, s);
      cols_q_kernel<<<dim3(ceil_div(slots, 256), Q), 256, 0, s>>>(
          cq(hp.nbr, hp.nbr_s), cq(hp.cnt, hp.cnt_s), cq(hp.row_ptr, hp.row_ptr_s), cq(nd, nd_s), f,
          rt, qp(hp.rows, hp.edge_s), qp(hp.cols, hp.edge_s),
          qp(hp.vals, hp.edge_s));
    }
    MQ_LAUNCH_CHECK("prep cols");
    if (h == d.num_hops - 1) {
      ProfScope ps(K_RELABEL_CLEAN, s);
      int cb = ceil_div(slots + hp.n_dst_max, 256);
      const int cap = ceil_div(kNumSMs * 8, Q);
      clean_q_kernel<<<dim3(cb < cap ? cb : cap, Q), 256, 0, s>>>(
          cq(hp.src_ids, hp.src_s), cq(hp.counts, hp.counts_s), rt);
    }
    MQ_LAUNCH_CHECK("prep clean");
  }

  // 3. transfer stage: gather the input rows of every slot + target labels
  const mq_prep_hop& last = d.hop[d.num_hops - 1];
  if (mask & MQ_PREP_GATHER) {
    ProfScope ps(K_GATHER, s);
    const int warps = kGatherThreads / 32;
    // narrow rows: 32 rows per warp pass; wide rows: one row per warp pass
    int blocks = ceil_div(last.n_src_max, dv4 > 32 ? warps : warps * 32);
    // blocks per SM across the Q slots (MQ_PREP_GATHER_BPS): the pass runs
    // beside the latency-bound train chain, whose CTAs must find room
    static const int bps = getenv("MQ_PREP_GATHER_BPS") ? atoi(getenv("MQ_PREP_GATHER_BPS")) : 4;
    const int cap = ceil_div(kNumSMs * bps, Q);
    if (blocks > cap) blocks = cap;
    gather_q_kernel<<<dim3(blocks, Q), kGatherThreads, 0, s>>>(
        d.cache_tbl, d.cache_pitch, d.slot_of,
        make_store(d.store, d.store_shard, d.n_shards, d.store_pitch), cq(last.src_ids, last.src_s),
        cq(last.counts, last.counts_s), dv4, qp(d.x0, d.x0_s), d.x0_pitch, d.hit_miss);
  }
  MQ_LAUNCH_CHECK("prep gather");
  if (mask & MQ_PREP_LABELS) {
    ProfScope ps(K_LABELS, s);
    labels_q_kernel<<<dim3(ceil_div(d.batch_size, 256), Q), 256, 0, s>>>(
        d.all_labels, cq(d.targets, d.targets_s), cq(d.n_targets, d.n_targets_s),
        qp(d.labels, d.labels_s));
  }
  MQ_LAUNCH_CHECK("prep labels");
  return MQ_OK;
}

}  // extern "C"
