// Dense SAGE layer transforms: z = [agg | h_dst] W, dW = [agg | h_dst]^T dz,
// dt = dz W^T (mqpipe/nn.py:126-131, 167-170).
//
// fp32 FMA on the CUDA cores: the reference trains in fp32 and north_star pins
// these contractions at rel 1e-5, which single-pass TF32 tensor-core math
// (10-bit mantissa) cannot meet.  The shapes are skinny (N = 41..128) with a
// row count M that only the device knows (the sampled frontier), so the
// kernel is a persistent split-K GEMM whose split factor is chosen ON THE
// DEVICE from M to fill all 148 SMs, followed by a deterministic fixed-order
// split reduction fused with the epilogue (ReLU / store / dW row scatter).
// The concat is never materialised: the K (or M) index space is padded to
// [0, P) -> agg, [P, 2P) -> h with P the 16-byte-aligned row pitch, so every
// operand load is a float4.
#include "mq_gemm.cuh"


using namespace mq;

extern "C" {

int64_t mq_linear_scratch_bytes(int32_t m_max, int32_t d_in, int32_t d_out) {
  const int64_t P2 = 2 * pitch_of(d_in);
  int64_t fwd = splitk_part_floats(m_max, d_out);
  int64_t bww = splitk_part_floats(P2, d_out);
  int64_t bwx = splitk_part_floats(m_max, 2 * d_in);
  int64_t mx = fwd > bww ? fwd : bww;
  mx = mx > bwx ? mx : bwx;
  return mx * (int64_t)sizeof(float);
}

int mq_sage_linear_fwd(const float* agg, int32_t ldagg, const float* h, int32_t ldh,
                       const int32_t* m_dev, int32_t m_max, int32_t d_in, const float* W,
                       int32_t d_out, float* z, int32_t ldz, float* relu_out, int32_t ldr,
                       void* scratch, void* stream) {
  MQ_CHECK_ARG(agg && h && m_dev && W && (z || relu_out) && scratch,
               "mq_sage_linear_fwd: null pointer");
  MQ_CHECK_ARG(d_in >= 1 && d_out >= 1 && (!z || ldz >= d_out) && (!relu_out || ldr >= d_out),
               "mq_sage_linear_fwd: bad dims");
  MQ_CHECK_ARG(ldagg == ldh && ldagg % 4 == 0 && ldagg >= d_in &&
                   ((uintptr_t)agg | (uintptr_t)h) % 16 == 0,
               "mq_sage_linear_fwd: agg and h need one 16-byte-aligned pitch >= d_in");
  if (m_max <= 0) return MQ_OK;
  cudaStream_t s = as_stream(stream);
  Dims dims{m_dev, 0, nullptr, 2 * ldagg, d_out};
  return run_gemm(ALoadConcat{agg, h, ldagg}, BLoadW{W, ldagg, d_in, d_out},
                  EpiLinearFwd{z, ldz, relu_out, ldr}, dims, m_max, 2 * ldagg, kMaxSplits,
                  reinterpret_cast<float*>(scratch), s, K_LINEAR_FWD, K_LINEAR_FWD_REDUCE);
}

int mq_sage_linear_bwd(const float* agg, int32_t ldagg, const float* h, int32_t ldh,
                       const int32_t* m_dev, int32_t m_max, int32_t d_in, const float* W,
                       int32_t d_out, const float* dz, int32_t lddz, float* dW, float* dt,
                       int32_t lddt, void* scratch, void* stream) {
  MQ_CHECK_ARG(agg && h && m_dev && W && dz && dW && scratch, "mq_sage_linear_bwd: null pointer");
  MQ_CHECK_ARG(d_in >= 1 && d_out >= 1 && lddz >= d_out && (!dt || lddt >= 2 * d_in),
               "mq_sage_linear_bwd: bad dims");
  MQ_CHECK_ARG(ldagg == ldh && ldagg % 4 == 0 && ldagg >= d_in &&
                   ((uintptr_t)agg | (uintptr_t)h) % 16 == 0,
               "mq_sage_linear_bwd: agg and h need one 16-byte-aligned pitch >= d_in");
  cudaStream_t s = as_stream(stream);
  float* part = reinterpret_cast<float*>(scratch);
  const int P = ldagg;
  {
    // dW over the padded concat rows: M = 2P (static), reduction over the m rows
    Dims dims{nullptr, 2 * P, m_dev, 0, d_out};
    int rc = run_gemm(ALoadConcatT{agg, h, P}, BLoadRow{dz, lddz, d_out},
                      EpiDW{dW, P, d_in, d_out}, dims, 2 * P, m_max, kMaxSplits, part, s,
                      K_LINEAR_BWD_W, K_LINEAR_BWD_W_REDUCE);
    if (rc) return rc;
  }
  if (dt != nullptr && m_max > 0) {
    Dims dims{m_dev, 0, nullptr, d_out, 2 * d_in};
    int rc = run_gemm(ALoadRow{dz, lddz}, BLoadWT{W, d_out, d_out, 2 * d_in}, EpiStore{dt, lddt},
                      dims, m_max, d_out, (d_out + GBK - 1) / GBK, part, s, K_LINEAR_BWD_X,
                      K_LINEAR_BWD_X_REDUCE);
    if (rc) return rc;
  }
  return MQ_OK;
}

// dt = dz W^T alone (the per-op backward when dW runs on the tensor cores)
int mq_sage_linear_dt(const int32_t* m_dev, int32_t m_max, int32_t d_in, const float* W,
                      int32_t d_out, const float* dz, int32_t lddz, float* dt, int32_t lddt,
                      void* scratch, void* stream) {
  MQ_CHECK_ARG(m_dev && W && dz && dt && scratch, "mq_sage_linear_dt: null pointer");
  MQ_CHECK_ARG(d_in >= 1 && d_out >= 1 && lddz >= d_out && lddt >= 2 * d_in,
               "mq_sage_linear_dt: bad dims");
  if (m_max <= 0) return MQ_OK;
  Dims dims{m_dev, 0, nullptr, d_out, 2 * d_in};
  return run_gemm(ALoadRow{dz, lddz}, BLoadWT{W, d_out, d_out, 2 * d_in}, EpiStore{dt, lddt}, dims,
                  m_max, d_out, (d_out + GBK - 1) / GBK, reinterpret_cast<float*>(scratch),
                  as_stream(stream), K_LINEAR_BWD_X, K_LINEAR_BWD_X_REDUCE);
}

// ---- GCN arm (nn.py:102-113, 159-180): z = agg W, dW = agg^T dz, dt = dz W^T
int mq_gcn_linear_fwd(const float* agg, int32_t ldagg, const int32_t* m_dev, int32_t m_max,
                      int32_t d_in, const float* W, int32_t d_out, float* z, int32_t ldz,
                      float* relu_out, int32_t ldr, void* scratch, void* stream) {
  MQ_CHECK_ARG(agg && m_dev && W && (z || relu_out) && scratch, "mq_gcn_linear_fwd: null pointer");
  MQ_CHECK_ARG(d_in >= 1 && d_out >= 1 && ldagg >= d_in && (!z || ldz >= d_out) &&
                   (!relu_out || ldr >= d_out),
               "mq_gcn_linear_fwd: bad dims");
  if (m_max <= 0) return MQ_OK;
  Dims dims{m_dev, 0, nullptr, d_in, d_out};
  return run_gemm(ALoadRow{agg, ldagg}, BLoadRow{W, d_out, d_out}, EpiLinearFwd{z, ldz, relu_out, ldr},
                  dims, m_max, d_in, kMaxSplits, reinterpret_cast<float*>(scratch), as_stream(stream),
                  K_GCN_LINEAR, K_GCN_LINEAR_REDUCE);
}

int mq_gcn_linear_bwd(const float* agg, int32_t ldagg, const int32_t* m_dev, int32_t m_max,
                      int32_t d_in, const float* W, int32_t d_out, const float* dz, int32_t lddz,
                      float* dW, float* dt, int32_t lddt, void* scratch, void* stream) {
  MQ_CHECK_ARG(agg && m_dev && W && dz && dW && scratch, "mq_gcn_linear_bwd: null pointer");
  MQ_CHECK_ARG(d_in >= 1 && d_out >= 1 && ldagg >= d_in && ldagg % 4 == 0 && lddz >= d_out &&
                   (uintptr_t)agg % 16 == 0 && (!dt || lddt >= d_in),
               "mq_gcn_linear_bwd: agg needs a 16-byte-aligned pitch (multiple of 4) >= d_in");
  cudaStream_t s = as_stream(stream);
  float* part = reinterpret_cast<float*>(scratch);
  {
    // dW rows over the padded pitch (pad columns of agg are zero, dropped by the epilogue)
    Dims dims{nullptr, ldagg, m_dev, 0, d_out};
    int rc = run_gemm(ALoadConcatT{agg, agg, ldagg}, BLoadRow{dz, lddz, d_out},
                      EpiDW{dW, ldagg, d_in, d_out}, dims, ldagg, m_max, kMaxSplits, part, s,
                      K_GCN_LINEAR, K_GCN_LINEAR_REDUCE);
    if (rc) return rc;
  }
  if (dt != nullptr && m_max > 0) {
    Dims dims{m_dev, 0, nullptr, d_out, d_in};
    int rc = run_gemm(ALoadRow{dz, lddz}, BLoadWT{W, d_out, d_out, d_in}, EpiStore{dt, lddt}, dims,
                      m_max, d_out, (d_out + GBK - 1) / GBK, part, s, K_GCN_LINEAR,
                      K_GCN_LINEAR_REDUCE);
    if (rc) return rc;
  }
  return MQ_OK;
}

}  // extern "C"
