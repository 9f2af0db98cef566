// Kernel ids for the timing hooks (mq_prof_*).
#pragma once

#define MQ_KERNEL_LIST(X)                         \
  X(K_PHILOX, "philox_fill")                      \
  X(K_SCAN, "scan")                               \
  X(K_STRIP_FLAGS, "strip_self_loops")            \
  X(K_RESIDENCY_COMPACT, "residency_compact")     \
  X(K_RESIDENCY_OFFSETS, "residency_offsets")     \
  X(K_RESIDENCY_SLOTS, "residency_slots")         \
  X(K_SAMPLE, "sample_hop")                       \
  X(K_RELABEL_MARK, "relabel_mark")               \
  X(K_RELABEL_FIRST, "relabel_first")             \
  X(K_RELABEL_FLAG, "relabel_flag_scan")          \
  X(K_RELABEL_EMIT, "relabel_emit")               \
  X(K_RELABEL_COLS, "relabel_cols")               \
  X(K_RELABEL_CLEAN, "relabel_clean")             \
  X(K_GATHER, "gather")                           \
  X(K_SPMM_FWD, "spmm_fwd")                       \
  X(K_SPMM_BWD_INIT, "spmm_bwd_init")             \
  X(K_SPMM_BWD, "spmm_bwd_scatter")               \
  X(K_SPMM_BWD_MASK, "spmm_bwd_mask")             \
  X(K_LINEAR_FWD, "linear_fwd")                   \
  X(K_LINEAR_BWD_W, "linear_bwd_w")               \
  X(K_LINEAR_BWD_W_REDUCE, "linear_bwd_w_reduce") \
  X(K_LINEAR_BWD_X, "linear_bwd_x")               \
  X(K_LINEAR_FWD_REDUCE, "linear_fwd_reduce")     \
  X(K_LINEAR_BWD_X_REDUCE, "linear_bwd_x_reduce") \
  X(K_SOFTMAX_CE, "softmax_ce")                   \
  X(K_LABELS, "gather_labels")                    \
  X(K_ADAM, "adam")                               \
  X(K_SGD, "sgd")                                 \
  X(K_STEP_BUMP, "step_bump")                     \
  X(K_CONVERT, "convert")                         \
  X(K_BATCH_SETUP, "batch_setup")                \
  X(K_SAGE_TRANSFORM, "sage_transform")           \
  X(K_SAGE_TRANSFORM_REDUCE, "sage_transform_reduce") \
  X(K_SAGE_AGG, "sage_aggregate")                 \
  X(K_SAGE_HEAD, "sage_head")                     \
  X(K_SAGE_SCATTER, "sage_scatter_bwd")           \
  X(K_SAGE_DW, "sage_dw")                         \
  X(K_SAGE_DW_REDUCE, "sage_dw_reduce")           \
  X(K_SAGE_DH, "sage_dh")                         \
  X(K_SAGE_DH_REDUCE, "sage_dh_reduce")         \
  X(K_FULL_TRANSFORM, "full_transform")         \
  X(K_FULL_TRANSFORM_REDUCE, "full_transform_reduce") \
  X(K_FULL_AGG, "full_aggregate")               \
  X(K_FULL_AGG_FIXUP, "full_aggregate_fixup")   \
  X(K_ACCURACY, "accuracy")                     \
  X(K_REFRESH_DEGREE, "refresh_degree")         \
  X(K_REFRESH_PROBS, "refresh_probs")           \
  X(K_REFRESH_WALK, "refresh_walk")             \
  X(K_REFRESH_SELECT, "refresh_select")         \
  X(K_SAGE_AF, "sage_linear_af")                \
  X(K_SAGE_AF_REDUCE, "sage_linear_af_reduce")  \
  X(K_SAGE_AF_DW, "sage_linear_af_dw")          \
  X(K_INGEST, "ingest")                         \
  X(K_RACOM_PUBLISH, "racom_publish")           \
  X(K_RACOM_APPLY, "racom_apply")               \
  X(K_LAYERWISE, "layerwise")                   \
  X(K_GCN_LINEAR, "gcn_linear")                 \
  X(K_GCN_LINEAR_REDUCE, "gcn_linear_reduce")

namespace mq {
enum KernelId {
#define MQ_KENUM(e, s) e,
  MQ_KERNEL_LIST(MQ_KENUM)
#undef MQ_KENUM
      K_COUNT
};
}  // namespace mq
