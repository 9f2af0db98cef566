// Full-graph SAGE evaluation: the per-epoch evaluate() of the reference
// driver (mqpipe/bench.py:82-87) over nn.full_forward (mqpipe/nn.py:218-250,
// sage arm) and nn.accuracy (nn.py:253-256).
//
// Reference, per layer l (loops stripped, nn.py:236-238):
//     agg[v] = (sum over arcs v->u in CSR order of h[u]) * inv[v],
//     inv[v] = f32(1 / deg(v)) (0 for isolated rows),
//     z      = [agg | h] W_l,  h = relu(z) except after the last layer.
// B200 form (same linear map, re-associated like the training step):
//     Y  = h [W_top | W_bot]        one tcgen05 3xTF32 GEMM over all n rows
//                                   (mq_full_transform, mq_tc.cu)
//     z[v] = inv[v] * sum_u Y_top[u] + Y_bot[v]            (mq_full_aggregate)
// so the segment sum runs at d_out (64 / classes) instead of the 602-wide
// input, and h is read once per layer.
//
// Load balance over power-law rows: the arc range [0, E) is cut into work
// items of kItem arcs, one warp per item.  A row wholly inside an item is
// summed sequentially in CSR order and written directly.  A row crossing
// item boundaries leaves one partial per item it touches (its first item's
// "tail" partial, then one "head" partial per later item); a second kernel
// sums those partials in item order.  No atomics, so evaluation is
// deterministic run to run.
#include "mq_common.cuh"

namespace mq {
namespace ev {

constexpr int kItem = 1024;   // arcs per work item
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxCols = 128;  // n_out <= 128 (4 columns per lane)

__device__ __forceinline__ int64_t last_row_at_or_before(const int64_t* __restrict__ row_off,
                                                         int64_t n, int64_t a) {
  // largest r in [0, n) with row_off[r] <= a
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (__ldg(row_off + mid) <= a) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// acc[k] (column lane + 32 k) += sum over arcs [s, e) of y[col, column], in
// arc order; the gathers are issued kU arcs at a time.
template <int NC>
__device__ __forceinline__ void seg_sum(const int32_t* __restrict__ col, int64_t s, int64_t e,
                                        const float* __restrict__ y, int ldy, int n_out, int lane,
                                        float (&acc)[NC]) {
  constexpr int kU = 8;
  for (int64_t b = s; b < e; b += 32) {
    const int m = (int)(e - b < 32 ? e - b : 32);
    const int32_t my = lane < m ? __ldg(col + b + lane) : 0;
    for (int t0 = 0; t0 < m; t0 += kU) {
      float x[kU][NC];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int32_t c = __shfl_sync(0xffffffffu, my, (t0 + u) & 31);
        const float* row = y + (int64_t)c * ldy;
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          const int j = lane + 32 * k;
          x[u][k] = (t0 + u < m && j < n_out) ? __ldg(row + j) : 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (t0 + u < m) {
#pragma unroll
          for (int k = 0; k < NC; ++k) acc[k] = __fadd_rn(acc[k], x[u][k]);
        }
    }
  }
}

// (ybot may alias out: the lean evaluate accumulates into h W_bot in place)
// (ybot NULL: no bottom term — the plain mean, agg[v] = inv * sum; `sel`
// non-NULL: only rows with sel[r] >= 0 are written, at output row sel[r])
template <int NC>
__device__ __forceinline__ void finish_row(int64_t r, int64_t deg, const float (&acc)[NC],
                                           const float* ybot, int ldb, int n_out, int relu,
                                           float* out, int ldo, int lane, const int32_t* sel) {
  // inv = where(counts > 0, 1 / counts, 0) in f32 (nn.py:239-240)
  const float inv = deg > 0 ? __fdiv_rn(1.0f, (float)deg) : 0.0f;
  const float* yb = ybot ? ybot + r * ldb : nullptr;
  const int64_t orow = sel ? (int64_t)sel[r] : r;
  if (orow < 0) return;
  float* o = out + orow * ldo;
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const int j = lane + 32 * k;
    if (j < n_out) {
      float z = __fmul_rn(acc[k], inv);
      if (yb) z = __fadd_rn(z, yb[j]);
      if (relu) z = z > 0.f ? z : 0.f;
      o[j] = z;
    } else if (j < ldo) {
      o[j] = 0.f;
    }
  }
  for (int j = 32 * NC + lane; j < ldo; j += 32) o[j] = 0.f;
}

// One warp per item: rows inside the item are finished, boundary rows leave
// partials (head[i]: row started before the item; tail[i]: row starts in the
// item and runs past its end).
template <int NC>
__global__ void __launch_bounds__(kThreads) full_agg_items_kernel(
    const int64_t* __restrict__ row_off, const int32_t* __restrict__ col, int64_t n, int64_t E,
    const float* __restrict__ y, int ldy, const float* ybot, int ldb, int n_out, int relu,
    float* out, int ldo, float* __restrict__ head, float* __restrict__ tail,
    const int32_t* __restrict__ sel) {
  const int lane = threadIdx.x & 31;
  const int64_t items = (E + kItem - 1) / kItem;
  for (int64_t i = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); i < items;
       i += (int64_t)gridDim.x * kWarps) {
    const int64_t a0 = i * kItem, a1 = (E < a0 + kItem ? E : a0 + kItem);
    int64_t r = last_row_at_or_before(row_off, n, a0);
    for (; r < n; ++r) {
      const int64_t r0 = __ldg(row_off + r), r1 = __ldg(row_off + r + 1);
      if (r0 >= a1) break;
      if (r1 == r0) continue;  // isolated rows: finished by the fix-up kernel
      if (sel && sel[r] < 0) continue;  // not requested
      float acc[NC];
#pragma unroll
      for (int k = 0; k < NC; ++k) acc[k] = 0.f;
      seg_sum<NC>(col, max(r0, a0), min(r1, a1), y, ldy, n_out, lane, acc);
      const bool before = r0 < a0, after = r1 > a1;
      if (!before && !after) {
        finish_row<NC>(r, r1 - r0, acc, ybot, ldb, n_out, relu, out, ldo, lane, sel);
      } else {
        float* p = (before ? head : tail) + i * n_out;
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          const int j = lane + 32 * k;
          if (j < n_out) p[j] = acc[k];
        }
      }
    }
  }
}

// One warp per row that crosses an item boundary or has no arcs.
template <int NC>
__global__ void __launch_bounds__(kThreads) full_agg_fixup_kernel(
    const int64_t* __restrict__ row_off, int64_t n, const float* ybot, int ldb, int n_out,
    int relu, float* out, int ldo, const float* __restrict__ head,
    const float* __restrict__ tail, const int32_t* __restrict__ sel) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); r < n;
       r += (int64_t)gridDim.x * kWarps) {
    if (sel && sel[r] < 0) continue;
    const int64_t r0 = __ldg(row_off + r), r1 = __ldg(row_off + r + 1);
    float acc[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) acc[k] = 0.f;
    if (r1 > r0) {
      const int64_t i0 = r0 / kItem, i1 = (r1 - 1) / kItem;
      if (i0 == i1) continue;  // finished by its item
      for (int64_t i = i0; i <= i1; ++i) {
        const float* p = (i == i0 ? tail : head) + i * n_out;
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          const int j = lane + 32 * k;
          acc[k] = __fadd_rn(acc[k], j < n_out ? __ldcg(p + j) : 0.f);
        }
      }
    }
    finish_row<NC>(r, r1 - r0, acc, ybot, ldb, n_out, relu, out, ldo, lane, sel);
  }
}

// numpy argmax order: the first NaN wins, else the largest value, ties to
// the lower index.  arg == C means "nothing yet".
__device__ __forceinline__ bool argmax_better(float x, int c, float best, int arg, int C) {
  if (c >= C) return false;
  if (arg >= C) return true;
  const bool xn = x != x, bn = best != best;
  if (bn) return xn && c < arg;
  if (xn) return true;
  return x > best || (x == best && c < arg);
}

// correct += #{i : argmax_c logits[ids[i], c] == labels[ids[i]]}, one warp per id.
__global__ void __launch_bounds__(kThreads) accuracy_kernel(const float* __restrict__ logits,
                                                            int ld, int C,
                                                            const int32_t* __restrict__ labels,
                                                            const int32_t* __restrict__ ids,
                                                            int64_t n_ids,
                                                            unsigned long long* correct,
                                                            int rows_are_positions) {
  const int lane = threadIdx.x & 31;
  unsigned long long mine = 0;
  for (int64_t i = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); i < n_ids;
       i += (int64_t)gridDim.x * kWarps) {
    const int64_t v = ids[i];
    const float* row = logits + (rows_are_positions ? i : v) * ld;
    float best = 0.f;
    int arg = C;
    for (int c = lane; c < C; c += 32) {
      const float x = __ldg(row + c);
      if (argmax_better(x, c, best, arg, C)) {
        best = x;
        arg = c;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
      if (argmax_better(ob, oa, best, arg, C)) {
        best = ob;
        arg = oa;
      }
    }
    if (lane == 0 && arg == __ldg(labels + v)) ++mine;
  }
  if (lane == 0 && mine) atomicAdd(correct, mine);
}

}  // namespace ev

int tc_transform_rows(const float* h, int ldh, int64_t n, int d_in, const float* W, int d_out,
                      float* y, float* part, cudaStream_t s);
int64_t tc_y_part_floats(int64_t m_max, int64_t d_out);
int tc_transform_half(const float* h, int ldh, int64_t n, int d_in, const float* W, int d_out,
                      float* y, int ldy, float* part, cudaStream_t s);
int tc_linear_cat_rows(const float* agg, int ldagg, const float* hv, int ldhv, int m, int d_in,
                       const float* W, int d_out, float* out, int ldo, int relu, float* part,
                       cudaStream_t s);
int64_t tc_af_part_floats(int64_t m_max, int64_t d_out);

}  // namespace mq

using namespace mq;

extern "C" {

int64_t mq_full_agg_scratch_bytes(int64_t n_arcs, int32_t n_out) {
  const int64_t items = (n_arcs + ev::kItem - 1) / ev::kItem;
  return 2 * (items < 1 ? 1 : items) * (int64_t)(n_out < 1 ? 1 : n_out) * 4;
}

static int full_aggregate(const int64_t* row_off, const int32_t* col, int64_t n_nodes,
                          int64_t n_arcs, const float* y, int32_t ldy, const float* ybot,
                          int32_t ldb, int32_t n_out, int32_t relu, float* out, int32_t ldo,
                          void* scratch, cudaStream_t s, const int32_t* sel = nullptr);

int mq_full_aggregate(const int64_t* row_off, const int32_t* col, int64_t n_nodes, int64_t n_arcs,
                      const float* y, int32_t ldy, int32_t n_out, int32_t relu, float* out,
                      int32_t ldo, void* scratch, void* stream) {
  MQ_CHECK_ARG(ldy >= 2 * n_out, "mq_full_aggregate: bad pitches");
  return full_aggregate(row_off, col, n_nodes, n_arcs, y, ldy, y ? y + n_out : nullptr, ldy, n_out,
                        relu, out, ldo, scratch, as_stream(stream));
}

int mq_full_aggregate_inplace(const int64_t* row_off, const int32_t* col, int64_t n_nodes,
                              int64_t n_arcs, const float* ytop, int32_t ldy, int32_t n_out,
                              int32_t relu, float* out, int32_t ldo, void* scratch, void* stream) {
  MQ_CHECK_ARG(ldy >= n_out, "mq_full_aggregate_inplace: bad pitches");
  return full_aggregate(row_off, col, n_nodes, n_arcs, ytop, ldy, out, ldo, n_out, relu, out, ldo,
                        scratch, as_stream(stream));
}

int mq_full_aggregate_rows(const int64_t* row_off, const int32_t* col, int64_t n_nodes,
                           int64_t n_arcs, const float* h, int32_t ldh, int32_t d,
                           const int32_t* sel_pos, float* agg, int32_t ldagg, void* scratch,
                           void* stream) {
  MQ_CHECK_ARG(sel_pos != nullptr, "mq_full_aggregate_rows: sel_pos is required");
  return full_aggregate(row_off, col, n_nodes, n_arcs, h, ldh, nullptr, 0, d, 0, agg, ldagg,
                        scratch, as_stream(stream), sel_pos);
}

static int full_aggregate(const int64_t* row_off, const int32_t* col, int64_t n_nodes,
                          int64_t n_arcs, const float* y, int32_t ldy, const float* ybot,
                          int32_t ldb, int32_t n_out, int32_t relu, float* out, int32_t ldo,
                          void* scratch, cudaStream_t s, const int32_t* sel) {
  MQ_CHECK_ARG(n_nodes >= 0 && n_arcs >= 0, "mq_full_aggregate: negative sizes");
  MQ_CHECK_ARG(n_out >= 1 && n_out <= ev::kMaxCols, "mq_full_aggregate: n_out must be in [1, %d]",
               ev::kMaxCols);
  MQ_CHECK_ARG(ldy >= n_out && ldo >= n_out && (!ybot || ldb >= n_out),
               "mq_full_aggregate: bad pitches");
  if (n_nodes == 0) return MQ_OK;
  MQ_CHECK_ARG(row_off && y && out && (n_arcs == 0 || (col && scratch)),
               "mq_full_aggregate: null pointer");
  const int64_t items = (n_arcs + ev::kItem - 1) / ev::kItem;
  float* head = static_cast<float*>(scratch);
  float* tail = head + (items < 1 ? 1 : items) * n_out;
  const int nc = (n_out + 31) / 32;
  const int grid_items = (int)(items < 1 ? 1 : (items + ev::kWarps - 1) / ev::kWarps > kNumSMs * 16
                                                   ? kNumSMs * 16
                                                   : (items + ev::kWarps - 1) / ev::kWarps);
  const int64_t gr = (n_nodes + ev::kWarps - 1) / ev::kWarps;
  const int grid_rows = (int)(gr > kNumSMs * 16 ? kNumSMs * 16 : gr);
#define MQ_FULL_AGG(NC)                                                                        \
  do {                                                                                         \
    if (items > 0) {                                                                           \
      ProfScope ps(K_FULL_AGG, s);                                                             \
      ev::full_agg_items_kernel<NC><<<grid_items, ev::kThreads, 0, s>>>(                       \
          row_off, col, n_nodes, n_arcs, y, ldy, ybot, ldb, n_out, relu, out, ldo, head, tail,  \
          sel);                                                                                \
    }                                                                                          \
    MQ_LAUNCH_CHECK("full_agg_items");                                                         \
    {                                                                                          \
      ProfScope ps(K_FULL_AGG_FIXUP, s);                                                       \
      ev::full_agg_fixup_kernel<NC><<<grid_rows, ev::kThreads, 0, s>>>(                        \
          row_off, n_nodes, ybot, ldb, n_out, relu, out, ldo, head, tail, sel);                \
    }                                                                                          \
    MQ_LAUNCH_CHECK("full_agg_fixup");                                                         \
  } while (0)
  switch (nc) {
    case 1: MQ_FULL_AGG(1); break;
    case 2: MQ_FULL_AGG(2); break;
    case 3: MQ_FULL_AGG(3); break;
    default: MQ_FULL_AGG(4); break;
  }
#undef MQ_FULL_AGG
  return MQ_OK;
}

int64_t mq_full_transform_part_floats(int64_t n_nodes, int32_t d_out) {
  // with at least one 128-row tile per SM the device picks a single split and
  // the GEMM writes y directly: no partial buffer
  if ((n_nodes + 127) / 128 >= kNumSMs) return 1;
  return tc_y_part_floats(n_nodes, d_out);
}

int mq_full_transform(const float* h, int32_t ldh, int64_t n_nodes, int32_t d_in, const float* W,
                      int32_t d_out, float* y, float* part, void* stream) {
  MQ_CHECK_ARG(n_nodes >= 0 && n_nodes < INT32_MAX, "mq_full_transform: n_nodes out of range");
  MQ_CHECK_ARG(d_out <= 128, "mq_full_transform: d_out must be <= 128 (UMMA N <= 256)");
  MQ_CHECK_ARG(d_in >= 1 && d_out >= 1 && ldh >= d_in && (ldh & 3) == 0,
               "mq_full_transform: bad shape (ldh must be a multiple of 4)");
  if (n_nodes == 0) return MQ_OK;
  MQ_CHECK_ARG(h && W && y && part, "mq_full_transform: null pointer");
  return tc_transform_rows(h, ldh, n_nodes, d_in, W, d_out, y, part, as_stream(stream));
}

int mq_full_transform_half(const float* h, int32_t ldh, int64_t n_nodes, int32_t d_in,
                           const float* W, int32_t d_out, float* y, int32_t ldy, float* part,
                           void* stream) {
  MQ_CHECK_ARG(n_nodes >= 0 && n_nodes < INT32_MAX && d_out >= 1 && d_out <= 256 && d_in >= 1 &&
                   ldh >= d_in && (ldh & 3) == 0 && ldy >= d_out,
               "mq_full_transform_half: bad shape");
  if (n_nodes == 0) return MQ_OK;
  MQ_CHECK_ARG(h && W && y && part, "mq_full_transform_half: null pointer");
  return tc_transform_half(h, ldh, n_nodes, d_in, W, d_out, y, ldy, part, as_stream(stream));
}

int64_t mq_full_linear_cat_part_floats(int64_t m, int32_t d_out) {
  if ((m + 127) / 128 >= kNumSMs) return 1;
  return tc_af_part_floats(m, d_out);
}

int mq_full_linear_cat(const float* agg, int32_t ldagg, const float* hv, int32_t ldhv, int64_t m,
                       int32_t d_in, const float* W, int32_t d_out, float* out, int32_t ldo,
                       int32_t relu, float* part, void* stream) {
  MQ_CHECK_ARG(m >= 0 && m < INT32_MAX && d_in >= 4 && d_in % 4 == 0 && d_out >= 1 &&
                   d_out <= 256 && ldagg % 4 == 0 && ldhv % 4 == 0 && ldo >= d_out,
               "mq_full_linear_cat: bad shape (d_in % 4 == 0, d_out <= 256)");
  if (m == 0) return MQ_OK;
  MQ_CHECK_ARG(agg && hv && W && out && part, "mq_full_linear_cat: null pointer");
  return tc_linear_cat_rows(agg, ldagg, hv, ldhv, (int)m, d_in, W, d_out, out, ldo, relu, part,
                            as_stream(stream));
}

int mq_accuracy_rows(const float* logits, int32_t ld, int32_t n_classes, const int32_t* labels,
                     const int32_t* ids, int64_t n_ids, unsigned long long* correct_dev,
                     void* stream) {
  MQ_CHECK_ARG(n_classes >= 1 && ld >= n_classes && n_ids >= 0, "mq_accuracy_rows: bad shape");
  if (n_ids == 0) return MQ_OK;
  MQ_CHECK_ARG(logits && labels && ids && correct_dev, "mq_accuracy_rows: null pointer");
  cudaStream_t s = as_stream(stream);
  const int64_t g = (n_ids + ev::kWarps - 1) / ev::kWarps;
  {
    ProfScope ps(K_ACCURACY, s);
    ev::accuracy_kernel<<<(int)(g > kNumSMs * 8 ? kNumSMs * 8 : g), ev::kThreads, 0, s>>>(
        logits, ld, n_classes, labels, ids, n_ids, correct_dev, 1);
  }
  MQ_LAUNCH_CHECK("accuracy_rows");
  return MQ_OK;
}

int mq_accuracy(const float* logits, int32_t ld, int32_t n_classes, const int32_t* labels,
                const int32_t* ids, int64_t n_ids, unsigned long long* correct_dev,
                void* stream) {
  MQ_CHECK_ARG(n_classes >= 1 && ld >= n_classes && n_ids >= 0, "mq_accuracy: bad shape");
  if (n_ids == 0) return MQ_OK;
  MQ_CHECK_ARG(logits && labels && ids && correct_dev, "mq_accuracy: null pointer");
  cudaStream_t s = as_stream(stream);
  const int64_t g = (n_ids + ev::kWarps - 1) / ev::kWarps;
  {
    ProfScope ps(K_ACCURACY, s);
    ev::accuracy_kernel<<<(int)(g > kNumSMs * 8 ? kNumSMs * 8 : g), ev::kThreads, 0, s>>>(
        logits, ld, n_classes, labels, ids, n_ids, correct_dev, 0);
  }
  MQ_LAUNCH_CHECK("accuracy");
  return MQ_OK;
}

}  // extern "C"
