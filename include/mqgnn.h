/*
 * mqgnn.h — C-ABI of libmqgnn, the B200 (sm_100a) implementation of MQ-GNN's
 * per-iteration GraphSAGE hot path.
 *
 * Conventions
 *   - every entry point is extern "C", takes plain pointers/sizes, and returns
 *     MQ_OK (0) or an MQ_ERR_* code; mq_last_error() holds the message
 *     (thread-local).  No allocation happens behind the caller's back: all
 *     device buffers are caller-owned and sized from the *_max bounds.
 *   - `stream` is a cudaStream_t passed as void*.  All work is enqueued
 *     asynchronously on it; entry points never synchronise, so a sequence of
 *     calls can be captured into a CUDA graph.
 *   - counts that are only known on the device (the frontier size of a hop,
 *     the number of sampled edges) are passed as `const int32_t* n_dev`
 *     pointers plus a host-side upper bound `n_max` that sizes the grid.
 *   - node ids are int32 (all target shapes have < 2^31 nodes); CSR row offsets
 *     and arc indices are int64.
 *   - the graph handed to the sampler is the reference CSR with stored
 *     self-loops removed (the reference drops the loop from every neighbour
 *     list before sampling, samplers.py:162, and full_forward does the same,
 *     nn.py:237-238); mq_strip_self_loops produces it.
 *
 * The reference (mqpipe, pure Python/NumPy) has no FFI; each function below
 * names the reference Python function whose semantics it implements
 * (paths relative to /root/reference/pkg/src/mqpipe/).
 */
#ifndef MQGNN_H
#define MQGNN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MQ_OK 0
#define MQ_ERR_ARG 1
#define MQ_ERR_CUDA 2
#define MQ_ERR_STATE 3
#define MQ_ERR_SAMPLING 4 /* SamplingError (samplers.py:23-24): empty candidates, zero norms */

#define MQ_MAX_FANOUT 32
/* ranks of one RaCoM exchange / shards of a partitioned feature store */
#define MQ_MAX_PEERS 8

/* Deferred split-K gradient reduction.  A flat gradient
 * element i in [offset, offset + size) is the fixed-order sum over p <
 * nparts of part[p * stride + j], with j = i - offset (kind 0) or, for
 * kind 1, the split-W layout of mq_sage_transform_bwd's partial tiles:
 * row = j / d_out, col = j % d_out, j' = row < d_in ? row * 2 d_out + col
 * : (row - d_in) * 2 d_out + d_out + col.  Elements outside every segment
 * come from the plain f32 gradient.  Passed by value into the optimizer
 * kernels, so the split-K reduction costs no launch of its own. */
#define MQ_GRAD_MAX_SEG 8
typedef struct mq_grad_seg {
  const float* part;
  const int32_t* nparts_dev; /* device-side partial count, or NULL: use nparts */
  int64_t stride;
  int64_t offset;
  int64_t size;
  int32_t nparts;
  int32_t kind;
  int32_t d_in;
  int32_t d_out;
} mq_grad_seg;
typedef struct mq_grad_src {
  int32_t nseg;
  int32_t pad_;
  mq_grad_seg seg[MQ_GRAD_MAX_SEG];
} mq_grad_src;

/* --------------------------------------------------------------- library */
int mq_version(void);
const char* mq_last_error(void);
/* Blocks until `stream` drains and reports any asynchronous kernel fault. */
int mq_stream_check(void* stream);

/* ------------------------------------------------------------ Philox draws
 * The injected-draw contract that replaces numpy's PCG64 in
 * samplers.py:172,174,177:  x_j = Philox4x32-10(key=(seed mod 2^32, epoch),
 * ctr=(j>>2, row, hop, batch))[j&3].  Host and device share one
 * implementation. */
int mq_philox_fill_host(uint64_t seed, uint64_t epoch, uint32_t batch, uint32_t hop,
                        uint32_t row, uint32_t count, uint32_t* out);
int mq_philox_fill(uint64_t seed, uint64_t epoch, uint32_t batch, uint32_t hop,
                   uint32_t row, uint32_t count, uint32_t* out_dev, void* stream);
/* Positions chosen by the partial Fisher-Yates of `choice(pool, k)` over a
 * pool of n (host reference of the device routine; k <= MQ_MAX_FANOUT). */
int mq_fisher_yates_host(uint64_t seed, uint64_t epoch, uint32_t batch, uint32_t hop,
                         uint32_t row, int64_t n, int32_t k, int64_t* pos_out);

/* ------------------------------------------------------------ graph layout
 * Replaces GraphCSR's read-only arrays (graph.py:28-91) on the device.
 * mq_strip_self_loops: out_row_off[v] counts the arcs of rows < v with
 * col != row; out_col receives them in CSR order.  `arc_flags_scratch` must
 * hold mq_scan_scratch_bytes(n_arcs) bytes. */
int64_t mq_scan_scratch_bytes(int64_t n_max);
int mq_strip_self_loops(const int64_t* row_off, const int32_t* col, int64_t n_nodes,
                        int64_t n_arcs, int64_t* out_row_off, int32_t* out_col,
                        void* scratch, void* stream);

/* ---------------------------------------------------- GNS cache residency
 * Per-epoch residency index that makes the per-row hot/cold split of
 * node_wise_block (samplers.py:168-175) O(fanout) instead of a full row scan:
 *   hot_arc[]  = indices (ascending) of every arc whose head is resident,
 *   hot_off[v] = number of hot arcs before row v (so row v's hot arcs are
 *                hot_arc[hot_off[v] .. hot_off[v+1])), length n_nodes+1.
 * resident_bits is a bitmap over node ids (CacheState.cached_mask,
 * cache.py:20-38).  *n_hot_dev receives the hot arc count.  hot_arc must hold
 * n_arcs entries (worst case). */
int mq_residency_index(const int64_t* row_off, const int32_t* col, int64_t n_nodes,
                       int64_t n_arcs, const uint32_t* resident_bits, int64_t* hot_arc,
                       int64_t* hot_off, int64_t* n_hot_dev, void* scratch, void* stream);
/* slot_of[v] = rank of v among resident nodes (ascending id) or -1; the HBM
 * cache table row of a hit (cache.py:131 searchsorted).  scratch as above
 * with n_max = n_nodes. */
int mq_residency_slots(const uint32_t* resident_bits, int64_t n_nodes, int32_t* slot_of,
                       int32_t* n_resident_dev, void* scratch, void* stream);

/* ------------------------------------------------------------- sampling
 * One hop of node_wise_block, SAGE arm (samplers.py:142-210): for dst row r,
 * v = dst[r], nbrs = row v (self loops already stripped), n = |nbrs|:
 *   n <= fanout           -> all neighbours in CSR order
 *   hot index given       -> |hot| >= fanout ? choice(hot, fanout)
 *                                            : hot ++ choice(cold, fanout-|hot|)
 *   otherwise             -> choice(nbrs, fanout)
 * with choice() the injected Philox Fisher-Yates.  Writes node ids to
 * nbr[r*fanout + i] and the count to cnt[r].  hot_arc/hot_off may be NULL
 * (no cache).  If key_dev is non-NULL the stream key is read on the device
 * (key_dev = {seed mod 2^32, epoch, batch}) instead of the by-value
 * seed/epoch/batch, so one captured CUDA graph serves every batch. */
int mq_sample_hop(const int64_t* row_off, const int32_t* col, const int64_t* hot_arc,
                  const int64_t* hot_off, const int32_t* dst, const int32_t* n_dst_dev,
                  int32_t n_dst_max, int32_t fanout, uint64_t seed, uint64_t epoch,
                  uint32_t batch, uint32_t hop, const uint32_t* key_dev, int32_t* nbr,
                  int32_t* cnt, void* stream);

/* Relabel + block emit (samplers.py:155-156, 186-200): src_ids = dst ids
 * followed by newly seen ids in first-occurrence (row, pick) order; rows/cols
 * are the block triplets, vals[e] = float32(1.0 / s_row).  row_ptr has
 * n_dst+1 entries (CSR view of the triplets).  counts_dev[0] = n_src,
 * counts_dev[1] = nnz.  dpos_tbl / first_tbl are node-indexed int32 tables
 * that must hold -1 / INT32_MAX on entry and are restored on exit.
 * scratch: mq_relabel_scratch_bytes(n_dst_max, fanout). */
int64_t mq_relabel_scratch_bytes(int32_t n_dst_max, int32_t fanout);
int mq_relabel(const int32_t* dst, const int32_t* n_dst_dev, int32_t n_dst_max,
               const int32_t* nbr, const int32_t* cnt, int32_t fanout, int32_t* dpos_tbl,
               int32_t* first_tbl, int32_t* row_ptr, int32_t* rows, int32_t* cols,
               float* vals, int32_t* src_ids, int32_t* counts_dev, void* scratch,
               void* stream);

/* ------------------------------------------------ multi-queue preparation
 * The MQ-GNN batch queue (runtime.py:380-612, pipeline.py:109-167) as ONE
 * pass of batched kernels over Q device slots: per slot exactly
 * mq_batch_setup (when cursor != NULL; else the host staged targets /
 * n_targets / key) -> [mq_sample_hop -> mq_relabel] per hop -> mq_gather +
 * mq_gather_labels, bit-identical to the single-batch entry points.  Every
 * per-slot array is given as slot 0's pointer plus a stride (elements) to the
 * next slot.  node_rank holds the relabel's rank words per slot (stride
 * table_s int32; one word per node: -(position + 1) for a node in the
 * current src list, else its first pick slot), restored on exit: with
 * hash_lg == 0 a node-indexed table [num_nodes] holding INT32_MAX; with
 * hash_lg = k > 0 an open-addressing hash of 2^k (key, word) int32 pairs
 * (key 0 / word INT32_MAX at rest) followed by the last hop's n_src_max
 * position entries, for graphs whose node-indexed tables would not fit
 * (reserved_ must be NULL); scratch holds
 * Q regions of mq_prep_scratch_bytes(max n_dst_max, its fanout) each
 * (scratch_s bytes apart).  When cursor != NULL, cursor[0] (window) advances
 * by Q and cursor[1] must be 0 at rest. */
#define MQ_MAX_HOPS 4
typedef struct mq_prep_hop {
  int32_t fanout, n_dst_max, n_src_max, pad_;
  int32_t* nbr;     int64_t nbr_s;      /* n_dst_max * fanout */
  int32_t* cnt;     int64_t cnt_s;      /* n_dst_max */
  int32_t* row_ptr; int64_t row_ptr_s;  /* n_dst_max + 1 */
  int32_t* rows;    int32_t* cols;  float* vals;  int64_t edge_s;  /* n_dst_max * fanout */
  int32_t* src_ids; int64_t src_s;      /* n_src_max */
  int32_t* counts;  int64_t counts_s;   /* [n_src, nnz] */
} mq_prep_hop;
typedef struct mq_prep_desc {
  int32_t nslots, num_hops, batch_size, world, rank, d;
  const int32_t* perm; int64_t n_perm; int32_t* cursor;
  int32_t* targets;   int64_t targets_s;
  int32_t* n_targets; int64_t n_targets_s;
  uint32_t* key;      int64_t key_s;      /* {seed mod 2^32, epoch, batch} per slot */
  mq_prep_hop hop[MQ_MAX_HOPS];
  int32_t* node_rank; void* reserved_; int64_t table_s;
  void* scratch; int64_t scratch_s;
  const int64_t* row_off; const int32_t* col; const int64_t* hot_arc; const int64_t* hot_off;
  const float* cache_tbl; int32_t cache_pitch, store_pitch;
  const int32_t* slot_of; const float* store;
  float* x0; int64_t x0_s; int32_t x0_pitch;
  uint32_t stage_mask;  /* 0 = all; else bits MQ_PREP_* select stages (profiling) */
  unsigned long long* hit_miss;
  const int32_t* all_labels; int32_t* labels; int64_t labels_s;
  /* seed-partitioned feature store (n_shards >= 2; then `store` is unused):
   * node v's row lives on shard v % n_shards at row v / n_shards, pitch
   * store_pitch — one table per rank, the others' mapped over NVLink P2P
   * (mq_ipc_open), so misses of remote rows are read peer-to-peer */
  const float* store_shard[MQ_MAX_PEERS]; int32_t n_shards, hash_lg;
} mq_prep_desc;
#define MQ_PREP_SETUP 1u
#define MQ_PREP_SAMPLE 2u
#define MQ_PREP_RELABEL 4u
#define MQ_PREP_GATHER 8u
#define MQ_PREP_LABELS 16u
int64_t mq_prep_scratch_bytes(int32_t n_dst_max, int32_t fanout);
int mq_prep_batches(const mq_prep_desc* desc, void* stream);

/* --------------------------------------------------------------- gather
 * gather_features / lookup (cache.py:111-134, runtime.py:127-143):
 *   out[i, :d] = slot_of[id] >= 0 ? cache_tbl[slot_of[id]] : store[id]
 * store may be a device table or a pinned host table (UVA pointer) — the
 * host-miss path.  slot_of may be NULL (everything served from store).
 * hit_miss[0] += hits, hit_miss[1] += misses (counted only when slot_of is
 * given).  Row pitches are in floats and must be multiples of 4. */
int mq_gather(const float* cache_tbl, int32_t cache_pitch, const int32_t* slot_of,
              const float* store, int32_t store_pitch, const int32_t* ids,
              const int32_t* n_dev, int32_t n_max, int32_t d, float* out,
              int32_t out_pitch, unsigned long long* hit_miss, void* stream);

/* mq_gather over a seed-partitioned store: misses read node v's row from
 * shards[v % n_shards] at row v / n_shards (remote shards peer-mapped over
 * NVLink).  shards is a HOST array of 1..MQ_MAX_PEERS device pointers. */
int mq_gather_sharded(const float* cache_tbl, int32_t cache_pitch, const int32_t* slot_of,
                      const float* const* shards, int32_t n_shards, int32_t store_pitch,
                      const int32_t* ids, const int32_t* n_dev, int32_t n_max, int32_t d,
                      float* out, int32_t out_pitch, unsigned long long* hit_miss,
                      void* stream);

/* ---------------------------------------------------------- SAGE numerics
 * block_apply (nn.py:79-89): agg[r] = sum over the row's triplets, in order,
 * of float32(val) * h[col] — sequential fp32 adds, bit-identical to np.add.at. */
/* y = max(x, 0) elementwise (the per-op forward's hidden activation). */
int mq_relu(const float* x, float* y, int64_t n, void* stream);
int mq_spmm_fwd(const int32_t* row_ptr, const int32_t* cols, const float* vals,
                const int32_t* n_dst_dev, int32_t n_dst_max, const float* h, int32_t ldh,
                int32_t d, float* agg, int32_t ldagg, void* stream);

/* block_apply_t + the self-path add (nn.py:92-98, 171-174):
 * dh[c] = sum_{e: col[e]=c} val[e] * dt[row[e], :d] + (c < n_dst ? dt[c, d:2d] : 0),
 * then, if mask_h != NULL, dh[c] *= (mask_h[c] > 0) (the ReLU mask of the
 * layer below, nn.py:167; mask_h is that layer's activation).
 * dh must be zeroed by this call's caller-visible semantics: the function
 * clears rows [0, n_src) itself. */
int mq_spmm_bwd(const int32_t* rows, const int32_t* cols, const float* vals,
                const int32_t* counts_dev /* [n_src, nnz] */, int32_t nnz_max,
                const int32_t* n_dst_dev, int32_t n_src_max, const float* dt, int32_t lddt,
                int32_t d, const float* mask_h, int32_t ldm, float* dh, int32_t lddh,
                void* stream);

/* sage_forward transform (nn.py:126-131): z = [agg | h_dst] @ W with W
 * (2*d_in, d_out) row-major.  z (pre-activation) and/or relu_out (max(z, 0))
 * are written when non-NULL; hidden layers only need relu_out because the
 * backward mask (pre > 0) equals (relu(pre) > 0).  agg and h share one
 * 16-byte-aligned pitch (ldagg == ldh).  Persistent split-K GEMM whose split
 * count is chosen on the device from m; the fixed-order split reduction makes
 * results deterministic.  scratch: mq_linear_scratch_bytes. */
int64_t mq_linear_scratch_bytes(int32_t m_max, int32_t d_in, int32_t d_out);
int mq_sage_linear_fwd(const float* agg, int32_t ldagg, const float* h, int32_t ldh,
                       const int32_t* m_dev, int32_t m_max, int32_t d_in, const float* W,
                       int32_t d_out, float* z, int32_t ldz, float* relu_out, int32_t ldr,
                       void* scratch, void* stream);

/* backward (nn.py:167-170): dW = [agg | h_dst]^T @ dz and, if dt != NULL,
 * dt = dz @ W^T (same kernel family and scratch as the forward). */
int mq_sage_linear_bwd(const float* agg, int32_t ldagg, const float* h, int32_t ldh,
                       const int32_t* m_dev, int32_t m_max, int32_t d_in, const float* W,
                       int32_t d_out, const float* dz, int32_t lddz, float* dW, float* dt,
                       int32_t lddt, void* scratch, void* stream);

/* ------------------------------------------------ fused training step
 * The StepRunner's SAGE step.  Hidden layers are evaluated
 * transform-first — the reference's z = [A h | h_dst] W (nn.py:126-131)
 * re-associated as Y = h [W_top | W_bot], z = A Y_top + Y_bot — so the wide
 * input features are never aggregated; the last layer is one fused kernel.
 *
 * mq_sage_transform: y (m x 2*d_out, row-major, ld 2*d_out) = h[:, :d_in] [W_top | W_bot],
 *   W (2*d_in x d_out) as in the reference.  m = *m_dev (<= m_max).
 * scratch for transform / transform_bwd: mq_sage_fused_scratch_bytes. */
int64_t mq_sage_fused_scratch_bytes(int32_t m_max, int32_t d_in, int32_t d_out);
/* Deferred output: when y_parts != NULL (requires mq_sage_y_deferred(d_out)),
 * the tensor-core split-K partial tiles part[s][m][2 d_out] (s < *y_nparts_dev,
 * m < *m_dev) are left in y_parts (mq_sage_y_parts_bytes) and y is not
 * written; mq_sage_aggregate then sums them on the fly. */
int mq_sage_y_deferred(int32_t d_out);
int64_t mq_sage_y_parts_bytes(int32_t m_max, int32_t d_out);
int mq_sage_transform(const float* h, int32_t ldh, const int32_t* m_dev, int32_t m_max,
                      int32_t d_in, const float* W, int32_t d_out, float* y, void* scratch,
                      float* y_parts, int32_t* y_nparts_dev, void* stream);
/* act[r, :d_out] = relu(sum_e val_e y[col_e, :d_out] + y[r, d_out:2 d_out]) for
 * r < *n_dst_dev (pad columns up to ldact zeroed); then zero the rows
 * [0, *zeroK_rows_dev) x zeroK_row_floats of zero0 / zero1 (either may be NULL)
 * — the backward's scatter targets, cleared here so they cost no launch.
 * With y_nparts_dev != NULL, y holds mq_sage_transform's deferred partials
 * (y_rows_dev = their m) and is reduced in fixed order on the fly. */
int mq_sage_aggregate(const int32_t* row_ptr, const int32_t* cols, const float* vals,
                      const int32_t* n_dst_dev, int32_t n_dst_max, const float* y, int32_t d_out,
                      const int32_t* y_nparts_dev, const int32_t* y_rows_dev, float* act,
                      int32_t ldact, float* zero0, const int32_t* zero0_rows_dev,
                      int32_t zero0_row_floats, float* zero1, const int32_t* zero1_rows_dev,
                      int32_t zero1_row_floats, void* stream);
/* Backward of the aggregation (nn.py:167, 171-174 re-associated):
 * dz = dh[r] * (act[r] > 0);  g[r, d_out:] = dz;  g[col_e, :d_out] += val_e dz.
 * g (n_src x 2*d_out) must be zero for rows [0, n_src) on entry. */
int mq_sage_scatter_bwd(const int32_t* row_ptr, const int32_t* cols, const float* vals,
                        const int32_t* n_dst_dev, int32_t n_dst_max, const float* dh, int32_t lddh,
                        const float* act, int32_t ldact, int32_t d_out, float* g, void* stream);
/* dW (2*d_in x d_out) = [h^T g_top ; h^T g_bot] over m = *m_dev rows and, if
 * dh != NULL, dh (m x d_in, ld lddh) = g [W_top | W_bot]^T (nn.py:168-174).
 * Deferred weight gradient: when dw_parts != NULL and mq_sage_dw_deferred(d_out)
 * is 1 (tcgen05 backend), the split-K partial tiles are left in dw_parts
 * (mq_sage_dw_parts_bytes) with their count in *dw_nparts_dev and dW is not
 * written; mq_sage_dw_grad_seg describes them for the optimizer. */
int mq_sage_dw_deferred(int32_t d_out);
int64_t mq_sage_dw_parts_bytes(int32_t d_in, int32_t d_out);
int mq_sage_transform_bwd(const float* h, int32_t ldh, const int32_t* m_dev, int32_t m_max,
                          int32_t d_in, const float* W, int32_t d_out, const float* g, float* dW,
                          float* dh, int32_t lddh, void* scratch, float* dw_parts,
                          int32_t* dw_nparts_dev, void* stream);
int mq_sage_dw_grad_seg(float* dw_parts, const int32_t* dw_nparts_dev, int32_t d_in, int32_t d_out,
                        int64_t offset, mq_grad_seg* out);
/* The last layer in one launch: agg = block_apply(h) for the *n_dst_dev target
 * rows (sequential triplet order, nn.py:79-89), logits = [agg | h_dst] W,
 * summed softmax-CE (loss_acc += loss; nonfinite |= 1 on NaN/Inf, nn.py:141-156),
 * Rows must carry <= MQ_MAX_FANOUT triplets (true of every sampled block;
 * otherwise nonfinite |= 4).
 * dlogits -> per-CTA dW partials in scratch (reduced in fixed CTA order into dW
 * when dW != NULL, else left for the optimizer: mq_sage_head_grad_seg) and,
 * if dh != NULL, dh += block_apply_t(dt[:, :d]) + self half (nn.py:167-174;
 * dh must be zero for rows [0, n_src) on entry).  With loss_ring != NULL the
 * batch loss is then moved to loss_ring[(key_dev[2]/world) % ring_len] and
 * loss_acc reset (mq_step_commit fused) by the last CTA to finish.  scratch:
 * mq_sage_head_scratch_bytes, zero-filled ONCE before first use (it holds a
 * self-resetting completion counter). */
int64_t mq_sage_head_scratch_bytes(int32_t n_dst_max, int32_t d, int32_t n_classes);
int mq_sage_head(const int32_t* row_ptr, const int32_t* cols, const float* vals,
                 const int32_t* n_dst_dev, int32_t n_dst_max, const float* h, int32_t ldh, int32_t d,
                 const float* W, int32_t n_classes, const int32_t* labels, float* dW, float* dh,
                 int32_t lddh, double* loss_acc, const uint32_t* key_dev, int32_t world,
                 double* loss_ring, int32_t ring_len, int32_t* nonfinite, void* scratch,
                 void* stream);
int mq_sage_head_grad_seg(int32_t n_dst_max, int32_t d, int32_t n_classes, void* scratch,
                          int64_t offset, mq_grad_seg* out);

/* batch_loss (nn.py:141-156): summed max-shifted softmax-CE over n rows;
 * dlogits = softmax - onehot; loss_out[0] += loss (f64);  nonfinite[0] |= 1
 * when any dlogit is NaN/Inf (FloatingPointError, nn.py:74-76). */
int mq_softmax_ce(const float* logits, int32_t ld, const int32_t* labels,
                  const int32_t* n_dev, int32_t n_max, int32_t n_classes, float* dlogits,
                  int32_t lddl, double* loss_out, int32_t* nonfinite, void* stream);

/* Device-side batch plan for graph replay (runtime.py:95-124): window
 * k = cursor[0]++, batch id j = k*world + rank (round-robin deal),
 * targets = perm[j*batch_size .. min(n_perm, (j+1)*batch_size)),
 * n_targets[0] = that length (0 when this rank has no batch in window k),
 * key_dev[2] = j.  key_dev[0..1] (seed, epoch) are left untouched. */
int mq_batch_setup(const int32_t* perm, int64_t n_perm, int32_t batch_size, int32_t world,
                   int32_t rank, int32_t* cursor_dev, int32_t* targets, int32_t* n_targets_dev,
                   uint32_t* key_dev, void* stream);

/* End-of-step bookkeeping for graph replay: with k = key_dev[2] / world (the
 * window of the batch just trained), loss_ring[k mod ring_len] = loss_acc[0];
 * loss_acc[0] = 0 (EpochStats.losses, runtime.py:72-92, read back once per
 * epoch instead of per batch). */
int mq_step_commit(double* loss_acc, const uint32_t* key_dev, int32_t world, double* loss_ring,
                   int32_t ring_len, void* stream);

/* labels[i] = all_labels[ids[i]] (build_minibatch target_labels, samplers.py:532) */
int mq_gather_labels(const int32_t* all_labels, const int32_t* ids, const int32_t* n_dev,
                     int32_t n_max, int32_t* out, void* stream);

/* adam_step (nn.py:191-206) over one flat parameter vector.  The gradient is
 * grad32 (f32) or grad64 * grad_scale cast to f32 (the RaCoM f64 window mean,
 * racom.py:47-57, 81-87); when grad_scale == 0 the scale is 1/grad64[n], the
 * all-reduced contributor count packed by mq_pack_grads (expected[k],
 * runtime.py:115-116).  step_dev is incremented on device; bias[2*(t-1)],
 * bias[2*(t-1)+1] hold float32(1 - 0.9**t), float32(1 - 0.999**t) for
 * t = 1..bias_len; steps past bias_len read the last row, which is exact
 * when the table reaches the saturated (1.0f, 1.0f) row (bias_len >= 17,400;
 * the Python side allocates 65,536 once and never reallocates it, so captured
 * graphs keep a valid pointer).  lr points at float32(learning_rate) in
 * device memory, read by every launch (a captured step follows
 * ModelState.learning_rate changes).  nonfinite[0] |= 1 on a
 * non-finite weight.  step_dev points at TWO int32: [0] the update count t,
 * [1] an arrival counter that must be 0 at rest (the launch's last CTA
 * publishes t+1 and resets it, so the bump costs no extra launch).  With
 * src != NULL (grad32 path) gradients are resolved through the deferred
 * split-K segments (mq_grad_src). */
int mq_adam(float* w, float* m, float* v, const float* grad32, const double* grad64,
            double grad_scale, int64_t n, int32_t* step_dev, const float* bias,
            int32_t bias_len, const float* lr, int32_t* nonfinite, const mq_grad_src* src,
            void* stream);
/* sgd_step (nn.py:209-215); lr as in mq_adam (device float32) */
int mq_sgd(float* w, const float* grad32, const double* grad64, double grad_scale,
           int64_t n, int32_t* step_dev, const float* lr, int32_t* nonfinite,
           const mq_grad_src* src, void* stream);
/* out64[i] = (double)grad[i] for i < n and out64[n] = (n_targets_dev[0] > 0):
 * one f64 buffer carries the window's gradient sum and contributor count
 * through a single all-reduce. */
int mq_pack_grads(const float* grad, int64_t n, const int32_t* n_targets_dev, double* out64,
                  const mq_grad_src* src, void* stream);
/* out32[i] = gradient element i resolved through src (materialises the
 * deferred reduction; tests and the eager API). */
int mq_grad_reduce(const mq_grad_src* src, const float* grad32, int64_t n, float* out32,
                   void* stream);

/* RaCoM packing for the NCCL collectives (racom.py:47-57, 118-139):
 * out64[i] = (double)in32[i];  out32[i] = (float)(in64[i] / divisor) — the
 * replica average of sync_models (sum over replicas in f64, then / n). */
int mq_f32_to_f64(const float* in32, double* out64, int64_t n, void* stream);
int mq_f64_to_f32(const double* in64, double divisor, float* out32, int64_t n, void* stream);

/* Dense-transform backend of the fused step: 1 (default) = tcgen05 3xTF32
 * (fp32-accurate split-precision on the 5th-gen tensor cores), 0 = fp32 FFMA
 * split-K on the CUDA cores.  Process-wide; for tests and A/B measurement. */
int mq_set_gemm_backend(int32_t backend);
int mq_get_gemm_backend(void);
/* Cap on the tcgen05 GEMM grid (default 148 = one CTA per SM); a smaller
 * grid means fewer, deeper split-K partitions (A/B measurement). */
int mq_set_tc_grid_cap(int32_t cap);
/* tcgen05 GEMM kernel: 2 (default) = TMA-fed, warp-specialised (operand tiles
 * by cp.async.bulk.tensor, one operand split into TMEM, double-buffered TMEM
 * accumulator) for the forward / aggregate-first / input-gradient modes, the
 * weight gradient on 1; 3 = TMA for every mode; 1 = cp.async staging with
 * register transposes everywhere.  Shapes the TMA path does not cover (N > 128,
 * unaligned pitches) run on 1.  Process-wide; A/B and tests. */
int mq_set_tc_kernel(int32_t version);
int mq_get_tc_kernel(void);
/* Programmatic dependent launch for the step's kernel chains (default on):
 * kernel k+1 is scheduled while kernel k runs and waits on the device for
 * k's completion (griddepcontrol), hiding the launch gap.  Process-wide; for
 * A/B measurement.  Takes effect for launches (and graph captures) made
 * after the call. */
int mq_set_pdl(int32_t on);
int mq_get_pdl(void);

/* Aggregate-first input layer of the fused step (the reference's own
 * association, nn.py:126-131 and 167-170), chosen when the input width is
 * narrow (d_in <= 2 d_out): the layer reads `agg` = block_apply(h)
 * (mq_spmm_fwd, bit-exact) and needs no input gradient.
 *   mq_sage_linear_af:      act = relu([agg | h[:m]] W), W (2 d_in x d_out), tcgen05
 *                           3xTF32; `part` holds mq_sage_af_parts_bytes bytes.
 *   mq_sage_linear_af_bwd:  dW partials [S][2 d_in][d_out] of
 *                           [agg | h]^T (dh * (act > 0)) over *rows_dev rows,
 *                           S -> *dw_nparts_dev (reduced by the optimizer, a
 *                           kind-0 mq_grad_seg).  d_in % 4 == 0. */
int64_t mq_sage_af_parts_bytes(int32_t m_max, int32_t d_out);
int64_t mq_sage_af_dw_parts_bytes(int32_t d_in, int32_t d_out);
int mq_sage_linear_af(const float* agg, int32_t ldagg, const float* h, int32_t ldh,
                      const int32_t* m_dev, int32_t m_max, int32_t d_in, const float* W,
                      int32_t d_out, float* act, int32_t ldact, float* part, void* stream);
int mq_sage_linear_af_bwd(const float* agg, int32_t ldagg, const float* h, int32_t ldh,
                          const int32_t* rows_dev, int32_t rows_max, int32_t d_in, const float* dh,
                          int32_t lddh, const float* act, int32_t ldact, int32_t d_out,
                          float* dw_parts, int32_t* dw_nparts_dev, void* stream);

/* ------------------------------------------------ full-graph evaluation
 * The per-epoch evaluate() of the reference driver (bench.py:82-87) over
 * nn.full_forward's sage arm (nn.py:218-250) and nn.accuracy (nn.py:253-256).
 * A layer is  Y = h [W_top | W_bot]  (mq_full_transform: n x 2 d_out, tcgen05
 * 3xTF32, `part` holds mq_full_transform_part_floats floats) followed by
 *   out[v] = relu?( f32(1/deg v) * sum_{arcs v->u, CSR order} Y_top[u] + Y_bot[v] )
 * (mq_full_aggregate; row_off/col = the loop-stripped CSR, deg 0 -> 0 * ...;
 * pad columns [n_out, ldo) are zeroed; scratch: mq_full_agg_scratch_bytes).
 * The segment sums are deterministic (no atomics).  mq_accuracy adds to
 * *correct_dev the number of ids whose first-max logit column equals the
 * label. */
int64_t mq_full_transform_part_floats(int64_t n_nodes, int32_t d_out);
int mq_full_transform(const float* h, int32_t ldh, int64_t n_nodes, int32_t d_in, const float* W,
                      int32_t d_out, float* y, float* part, void* stream);
int64_t mq_full_agg_scratch_bytes(int64_t n_arcs, int32_t n_out);
int mq_full_aggregate(const int64_t* row_off, const int32_t* col, int64_t n_nodes, int64_t n_arcs,
                      const float* y, int32_t ldy, int32_t n_out, int32_t relu, float* out,
                      int32_t ldo, void* scratch, void* stream);
int mq_accuracy(const float* logits, int32_t ld, int32_t n_classes, const int32_t* labels,
                const int32_t* ids, int64_t n_ids, unsigned long long* correct_dev,
                void* stream);
/* The lean evaluate (memory O(n d_out) instead of O(n 2 d_out) + O(n C)),
 * same reference semantics:
 *   mq_full_transform_half: y = h W over n rows, W one (d_in x d_out) half of a
 *     SAGE weight (W_top or W_bot); `part` as mq_full_transform_part_floats.
 *   mq_full_aggregate_inplace: out[v] = relu?(f32(1/deg v) * sum Y_top[u] + out[v])
 *     (out holds h W_bot on entry).
 *   mq_full_aggregate_rows: agg[sel_pos[v]] = f32(1/deg v) * sum_u h[u] (CSR
 *     order within each 1024-arc item) for the rows with sel_pos[v] >= 0 only
 *     (the last layer's mean over the evaluated rows; hubs split across
 *     warps like mq_full_aggregate, same scratch).
 *   mq_full_linear_cat: out = relu?([agg | hv] W) over m rows (tcgen05 3xTF32);
 *     `part` holds mq_full_linear_cat_part_floats floats.
 *   mq_accuracy_rows: as mq_accuracy with logits row i belonging to ids[i]. */
int mq_full_transform_half(const float* h, int32_t ldh, int64_t n_nodes, int32_t d_in,
                           const float* W, int32_t d_out, float* y, int32_t ldy, float* part,
                           void* stream);
int mq_full_aggregate_inplace(const int64_t* row_off, const int32_t* col, int64_t n_nodes,
                              int64_t n_arcs, const float* ytop, int32_t ldy, int32_t n_out,
                              int32_t relu, float* out, int32_t ldo, void* scratch, void* stream);
int mq_full_aggregate_rows(const int64_t* row_off, const int32_t* col, int64_t n_nodes,
                           int64_t n_arcs, const float* h, int32_t ldh, int32_t d,
                           const int32_t* sel_pos, float* agg, int32_t ldagg, void* scratch,
                           void* stream);
int64_t mq_full_linear_cat_part_floats(int64_t m, int32_t d_out);
int mq_full_linear_cat(const float* agg, int32_t ldagg, const float* hv, int32_t ldhv, int64_t m,
                       int32_t d_in, const float* W, int32_t d_out, float* out, int32_t ldo,
                       int32_t relu, float* part, void* stream);
int mq_accuracy_rows(const float* logits, int32_t ld, int32_t n_classes, const int32_t* labels,
                     const int32_t* ids, int64_t n_ids, unsigned long long* correct_dev,
                     void* stream);

/* ------------------------------------------------- per-epoch cache refresh
 * GNS residency on the device (cache.py:41-108, samplers.py:113-135).
 * mq_in_degrees: deg[v] = #arcs u->v of the stored CSR (graph.py in_degrees);
 *   col is the loop-stripped column array, `loops` (nullable) the per-row count
 *   of stripped self loops, which count toward their own row's in-degree.
 * mq_degree_probs: probs = deg / total (cache_probs_degree; total = stored
 *   arcs; total 0 -> uniform).
 * mq_walk_probs: cache_probs_walk — p0 = 1/|train| on train nodes, `steps`
 *   rounds of p <- D A p + p with D = min(fanout, deg)/deg, the per-row flow
 *   summed sequentially in CSR order (stored loops at their sorted position),
 *   then p / sum(p) with NumPy's pairwise summation; *bad_dev = 1 if the total
 *   is not positive.  scratch: mq_walk_scratch_bytes(n).  train_mask: u8 [n].
 * mq_refresh_select: refresh_cache's resident set as chosen[v] in {0,1}:
 *   take = min(budget, #positive) nodes by the exponential keys u^(1/w), u the
 *   refresh contract's random(#positive) (oracle/philox.py), largest first,
 *   ties to the lower id; then a WOR Fisher-Yates choice of budget - take ids
 *   from the rest (ascending).  counts_dev[0] = #positive, [1] = take.
 *   scratch: mq_refresh_scratch_bytes(n).  No host synchronisation. */
int mq_in_degrees(const int32_t* col, int64_t n_nodes, int64_t n_arcs, const int32_t* loops,
                  int64_t* deg, void* stream);
int mq_degree_probs(const int64_t* deg, int64_t n_nodes, int64_t total, double* probs,
                    void* stream);
int64_t mq_walk_scratch_bytes(int64_t n_nodes);
int mq_walk_probs(const int64_t* row_off, const int32_t* col, int64_t n_nodes, const int32_t* loops,
                  const int64_t* deg, const uint8_t* train_mask, int64_t n_train, int32_t fanout,
                  int32_t steps, double* probs, int32_t* bad_dev, void* scratch, void* stream);
int64_t mq_refresh_scratch_bytes(int64_t n_nodes);
int mq_refresh_select(const double* probs, int64_t n_nodes, int64_t budget, uint64_t seed,
                      uint64_t epoch, uint8_t* chosen, int64_t* counts_dev, void* scratch,
                      void* stream);
/* host restatement of the refresh contract's random(n) (tests) */
int mq_refresh_uniforms_host(uint64_t seed, uint64_t epoch, int64_t n, double* out);

/* ------------------------------------------------------------ graph ingest
 * build_csr (graph.py:94-139) on the device: mq_build_csr_keys sorts the
 * edge keys src * n + dst (LSD radix sort, stable warp-ranked scatter) and
 * compacts the distinct ones into `uniq` (*n_unique_dev; *bad_dev = 1 if an
 * endpoint is out of range); mq_build_csr_finish writes row_offsets (n+1,
 * int64) and int32 columns.  edges: int64 [m][2].  scratch:
 * mq_build_csr_scratch_bytes(m); uniq holds m entries.
 * mq_narrow_cols: the MQG1 loader's u64 columns (graph.py:331-395) to int32
 * (*bad_dev = 1 if a column is >= n).  mq_degree_buckets: the default
 * features' one-hot index floor(log2(deg + 1)) (graph.py:142-149). */
int64_t mq_build_csr_scratch_bytes(int64_t m);
int mq_build_csr_keys(const int64_t* edges, int64_t m, int64_t n_nodes, void* scratch,
                      unsigned long long* uniq, int64_t* n_unique_dev, int32_t* bad_dev,
                      void* stream);
int mq_build_csr_finish(const unsigned long long* uniq, int64_t n_unique, int64_t n_nodes,
                        int64_t* row_off, int32_t* col, void* stream);
int mq_narrow_cols(const unsigned long long* cols64, int64_t m, int64_t n_nodes, int32_t* cols32,
                   int32_t* bad_dev, void* stream);
int mq_degree_buckets(const int64_t* row_off, int64_t n_nodes, int32_t* bucket, void* stream);

/* ------------------------------------------------- RaCoM over peer memory
 * share_gradient + Accumulator + apply_update (racom.py:36-87, 142-184;
 * runtime.py:167-195) as two stream-ordered kernels per window, with no host
 * synchronisation and no collective library on the data path, so a
 * multi-rank window is capturable into a CUDA graph.  Every rank owns an
 * arena (mq_peer_alloc: cudaMalloc, zeroed) holding
 *   [0, 64)            flags: u64 per source rank — windows that rank has
 *                      published, written remotely by that rank
 *   [64, 128)          counters: u64 [published, applied]
 *   [256, ...)         ring x (n + 1) f32 gradient slots: [grads | contributor]
 *                      (each slot padded to 256 B; the packets are f32 as in
 *                      the reference, the f64 accumulation happens on apply)
 * exported to the other ranks with mq_ipc_export / mq_ipc_open (NVLink P2P
 * mappings across GPUs; a plain alias within one process).
 *
 * mq_racom_publish: window k = counters[published]: the resolved f32 window
 *   gradient (grad32 through the deferred split-K segments src, as mq_adam)
 *   is written to this rank's slot k % ring with the contributor flag
 *   (n_targets_dev[0] > 0), then flags[rank] = k + 1 is stored (release,
 *   system scope) into EVERY rank's arena.
 * mq_racom_apply: if published - applied > lag, window k = applied is
 *   applied: wait (acquire, system scope; bounded by timeout_ns, 0 = 30 s)
 *   until every rank has published k + 1 windows, form the Accumulator's f64
 *   running mean over the contributing ranks in rank order
 *   (mean += (g_q - mean) / count, racom.py:47-57 — the reference's serial
 *   arrival order, so the mean is bit-identical to its Accumulator), cast to
 *   f32 (nn.py:197) and run the Adam / SGD update of mq_adam / mq_sgd.
 *   lag = 0: parity schedule (apply the window just published); lag = 1:
 *   pipelined schedule (window k applied after window k+1's backward, so
 *   every gradient misses exactly one update).  A timed-out wait sets
 *   nonfinite[0] |= 8 and skips the update.
 * Both kernels size their grid to stay co-resident (<= one CTA per SM). */
#define MQ_PEER_HEADER_BYTES 256
typedef struct mq_ipc_handle { char bytes[64]; } mq_ipc_handle;
typedef struct mq_peer_exchange {
  int32_t world, rank, ring, pad_;
  int64_t n;                     /* gradient elements per slot (+1 contributor flag) */
  int64_t timeout_ns;            /* bound on the apply wait; 0 = 30 s */
  char* arena[MQ_MAX_PEERS];     /* every rank's arena, mapped into this process */
} mq_peer_exchange;
int64_t mq_peer_arena_bytes(int64_t n, int32_t ring);
int mq_peer_alloc(int64_t bytes, void** out);
int mq_peer_free(void* p);
int mq_ipc_export(void* dev_ptr, mq_ipc_handle* out);
int mq_ipc_open(const mq_ipc_handle* h, void** out);
int mq_ipc_close(void* p);
int mq_racom_publish(const mq_peer_exchange* ex, const float* grad32, const mq_grad_src* src,
                     const int32_t* n_targets_dev, void* stream);
int mq_racom_apply(const mq_peer_exchange* ex, int32_t optimizer /* 0 adam, 1 sgd */,
                   int32_t lag, float* w, float* m, float* v, int32_t* step_dev,
                   const float* bias, int32_t bias_len, const float* lr, int32_t* nonfinite,
                   void* stream);
/* counters[0..1] and the flag words of this rank's arena, read back (tests) */
int mq_peer_state(const mq_peer_exchange* ex, unsigned long long* out4 /* pub, applied, min flag, max flag */,
                  void* stream);

/* ------------------------------------------------- layer-wise samplers
 * LADIES / FastGCN (samplers.py:233-495) and the GCN node-wise arm
 * (samplers.py:178-191).  Graph = the loop-stripped CSR plus `loops` (stored
 * self loops per node, NULL when none): the restricted Laplacian rows and
 * a_hat_degrees are rebuilt from it exactly as the reference computes them
 * on the stored CSR.  Draws follow the layer contract (oracle/layerwise.py):
 * layer l of batch b reads uniforms from the Philox stream (seed, epoch;
 * ctr (i, 0xFFFFFFFF, l, b)).  These calls are host-orchestrated and
 * SYNCHRONISE their stream (the reference API they mirror returns arrays);
 * their temporaries come from the stream-ordered allocator. */

/* restricted-row offsets of prev (loop-stripped degree + loop entries),
 * roff[n_prev + 1]; roff[n_prev] = entries.  scratch: mq_layer_scratch_bytes. */
int64_t mq_layer_scratch_bytes(int64_t n_max);
int mq_layer_entries(const int64_t* row_off, const int32_t* loops, const int32_t* prev,
                     int32_t n_prev, int64_t* roff, void* scratch, void* stream);
/* sample_ladies's target filter (samplers.py:453-458): targets with a stored
 * out-degree > 0, in order; *count_dev = kept. */
int mq_layer_live_targets(const int64_t* row_off, const int32_t* loops, const int32_t* targets,
                          int32_t n, int32_t* out, int64_t* count_dev, void* scratch, void* stream);
/* fastgcn_probs (samplers.py:314-318) over all nodes (flat: unsquared
 * norms); cdf (optional, n_nodes) = the normalised cumulative sum the
 * with-replacement draw searches (NumPy's choice(p) algorithm). */
int mq_layer_fastgcn_probs(const int64_t* row_off, const int32_t* col, const int32_t* loops,
                           int64_t n_nodes, int32_t flat, double* probs, double* cdf, void* stream);
/* One layer-wise block (samplers.py:376-440).  probs_global == NULL: LADIES
 * (candidates = sorted unique neighbours of prev, probabilities = squared or,
 * with flat, unsquared restricted column norms, normalised by NumPy's
 * pairwise sum; node_flags (n bytes, zero, left zero) and node_pos (n ints)
 * are the caller's per-graph tables); else FastGCN over all nodes with the
 * given probabilities (and cdf_global for mode 1).  mode: 0 = WOR with row
 * normalisation, 1 = with replacement (counts / (s p)), 2 = debias (WOR with
 * the recursive coefficients).  Outputs: rows/cols/values/effective
 * [n_entries] (nnz used; rows nondecreasing, cols index src_ids), row_ptr
 * [n_prev + 1], src_ids / sample_probs [budget] (n_src used, ascending node
 * ids), counts[4] = {nnz, n_src, n_cand, s}.  Returns MQ_ERR_SAMPLING for an
 * empty candidate set or all-zero norms. */
int mq_layer_block(const int64_t* row_off, const int32_t* col, const int32_t* loops,
                   int64_t n_nodes, const int32_t* prev, int32_t n_prev, const int64_t* roff,
                   int64_t n_entries, const double* probs_global, const double* cdf_global,
                   int32_t flat, int32_t mode, int32_t budget, uint64_t seed, uint64_t epoch,
                   uint32_t batch, uint32_t layer, uint8_t* node_flags, int32_t* node_pos,
                   int32_t* rows, int32_t* cols, double* values, double* effective,
                   int32_t* row_ptr, int32_t* src_ids, double* sample_probs, int64_t* counts,
                   void* stream);
/* GCN arm of node_wise_block from the SAGE block of the same draws: per row
 * the self entry (r, r, 1/deg_hat[v]) then the sampled entries with
 * (n/s) / sqrt(deg_hat[v] deg_hat[u]).  Outputs sized nnz + n_dst. */
int mq_gcn_block(const int64_t* row_off, const int32_t* loops, const int32_t* dst,
                 const int32_t* src_ids, const int32_t* row_ptr, const int32_t* cols, int32_t n_dst,
                 int32_t* row_ptr_out, int32_t* rows_out, int32_t* cols_out, double* vals_out,
                 void* stream);
/* NumPy's choice(p) cdf: cumsum(p) (sequential f64) / its last element */
int mq_layer_cdf(const double* probs, int64_t n, double* cdf, void* stream);
/* host reference of the layer uniforms (tests) */
int mq_layer_uniforms_host(uint64_t seed, uint64_t epoch, uint32_t batch, uint32_t layer, int64_t n,
                           double* out);

/* dt = dz W^T alone (the per-op SAGE backward when its dW runs on the
 * tensor cores, mq_sage_linear_af_bwd); scratch: mq_linear_scratch_bytes. */
int mq_sage_linear_dt(const int32_t* m_dev, int32_t m_max, int32_t d_in, const float* W,
                      int32_t d_out, const float* dz, int32_t lddz, float* dt, int32_t lddt,
                      void* scratch, void* stream);

/* GCN layer transform (nn.py:102-113, 159-180 gcn arm): z = agg W (relu_out
 * = max(z, 0) when given); backward dW = agg^T dz and dt = dz W^T.  fp32
 * split-K, fixed-order reduction (scratch: mq_linear_scratch_bytes). */
int mq_gcn_linear_fwd(const float* agg, int32_t ldagg, const int32_t* m_dev, int32_t m_max,
                      int32_t d_in, const float* W, int32_t d_out, float* z, int32_t ldz,
                      float* relu_out, int32_t ldr, void* scratch, void* stream);
int mq_gcn_linear_bwd(const float* agg, int32_t ldagg, const int32_t* m_dev, int32_t m_max,
                      int32_t d_in, const float* W, int32_t d_out, const float* dz, int32_t lddz,
                      float* dW, float* dt, int32_t lddt, void* scratch, void* stream);

/* ------------------------------------------------------------- tracing
 * Trace / TraceEvent (pipeline.py:30-98): when the stream reaches the call,
 * append {globaltimer ns, tag << 32 | key_dev[2] (the slot's batch id) or
 * 0xFFFFFFFF} at buf[2 * i] (i = atomicAdd(cursor, 1), dropped once i >=
 * cap).  Launched dependent on its predecessor; capturable. */
int mq_trace_stamp(unsigned long long* buf, int32_t cap, unsigned int* cursor, uint32_t tag,
                   const uint32_t* key_dev, void* stream);

/* ------------------------------------------------------------- utilities */
/* cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, stream): the step's
 * pinned-host result read-back as a node of a captured graph. */
int mq_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream);
/* cudaMemsetAsync (a scatter target's clear inside a captured step). */
int mq_memset_async(void* dst, int32_t value, int64_t bytes, void* stream);
/* exclusive prefix sum of int32 counts into int32 offsets (n+1 entries). */
int mq_scan_i32(const int32_t* in, const int32_t* n_dev, int32_t n_max, int32_t* out,
                void* scratch, void* stream);

/* ---------------------------------------------------- kernel timing hooks
 * Bench instrumentation: when enabled, each kernel launch is bracketed by
 * CUDA events on its stream; mq_prof_read returns per-kernel totals (ms) and
 * launch counts.  Must be disabled while capturing a CUDA graph. */
int mq_prof_enable(int on);
int mq_prof_reset(void);
int mq_prof_num_kernels(void);
const char* mq_prof_kernel_name(int id);
int mq_prof_read(double* total_ms, int64_t* launches, int32_t n);
/* Number of kernel launches issued through this library since the last
 * reset (counted whether or not timing is enabled). */
int64_t mq_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* MQGNN_H */
