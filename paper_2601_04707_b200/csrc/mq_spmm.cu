// SAGE mean aggregation as segment-reduce SpMM (forward) and its transpose.
//
// Reference: mqpipe/nn.py:79-98 (block_apply / block_apply_t) and the SAGE
// backward self-path add nn.py:171-174.
#include "mq_common.cuh"

namespace mq {

constexpr int kSpmmThreads = 256;

// Forward: one warp per dst row, lanes over 16-byte column groups.  Each
// output element is the sequential fp32 sum, in triplet order, of the
// individually rounded products float32(val) * h — exactly np.add.at's
// evaluation order (nn.py:88), so the result is bit-identical.
__global__ void __launch_bounds__(kSpmmThreads) spmm_fwd_kernel(
    const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ cols,
    const float* __restrict__ vals, const int32_t* __restrict__ n_dst_dev,
    const float* __restrict__ h, int ldh, int d4, float* __restrict__ agg, int ldagg) {
  const int lane = threadIdx.x & 31;
  const int warps = kSpmmThreads / 32;
  const int n = *n_dst_dev;
  for (int r = blockIdx.x * warps + (threadIdx.x >> 5); r < n; r += gridDim.x * warps) {
    const int e0 = row_ptr[r], e1 = row_ptr[r + 1];
    float4* out = reinterpret_cast<float4*>(agg + (int64_t)r * ldagg);
    for (int cb = 0; cb < d4; cb += 32) {
      const int c = cb + lane;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int eb = e0; eb < e1; eb += 32) {
        const int me = eb + lane;
        int32_t my_col = 0;
        float my_val = 0.f;
        if (me < e1) {
          my_col = __ldg(&cols[me]);
          my_val = __ldg(&vals[me]);
        }
        const int m = min(32, e1 - eb);
        for (int t = 0; t < m; ++t) {
          const int32_t col = __shfl_sync(0xffffffffu, my_col, t);
          const float val = __shfl_sync(0xffffffffu, my_val, t);
          if (c < d4) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(h + (int64_t)col * ldh) + c);
            acc.x = __fadd_rn(acc.x, __fmul_rn(val, x.x));
            acc.y = __fadd_rn(acc.y, __fmul_rn(val, x.y));
            acc.z = __fadd_rn(acc.z, __fmul_rn(val, x.z));
            acc.w = __fadd_rn(acc.w, __fmul_rn(val, x.w));
          }
        }
      }
      if (c < d4) out[c] = acc;
    }
  }
}

// Backward step 1: dh[c] = dt[c, d:2d] for the dst prefix (the concat's self
// half, nn.py:174), zero for the remaining src rows.
__global__ void spmm_bwd_init_kernel(const int32_t* __restrict__ counts,
                                     const int32_t* __restrict__ n_dst_dev,
                                     const float* __restrict__ dt, int lddt, int d,
                                     float* __restrict__ dh, int lddh) {
  const int n_src = counts[0], n_dst = *n_dst_dev;
  const int64_t total = (int64_t)n_src * d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / d), k = (int)(i % d);
    dh[(int64_t)c * lddh + k] = (c < n_dst) ? dt[(int64_t)c * lddt + d + k] : 0.f;
  }
}

// Backward step 2: scatter-add val * dt[row, :d] into dh[col] (block_apply_t,
// nn.py:92-98).  One warp per edge; fp32 atomics, so the summation order is
// not fixed — parity is tolerance-based.
__global__ void __launch_bounds__(kSpmmThreads) spmm_bwd_scatter_kernel(
    const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
    const float* __restrict__ vals, const int32_t* __restrict__ counts,
    const float* __restrict__ dt, int lddt, int d, float* __restrict__ dh, int lddh, int vec4) {
  const int lane = threadIdx.x & 31;
  const int warps = kSpmmThreads / 32;
  const int nnz = counts[1];
  for (int e = blockIdx.x * warps + (threadIdx.x >> 5); e < nnz; e += gridDim.x * warps) {
    const int r = rows[e], c = cols[e];
    const float val = vals[e];
    const float* src = dt + (int64_t)r * lddt;
    float* dst = dh + (int64_t)c * lddh;
    if (vec4) {
      for (int k = lane; k < d / 4; k += 32) {
        float4 x = reinterpret_cast<const float4*>(src)[k];
        float4 y = make_float4(__fmul_rn(val, x.x), __fmul_rn(val, x.y), __fmul_rn(val, x.z),
                               __fmul_rn(val, x.w));
        atomicAdd(reinterpret_cast<float4*>(dst) + k, y);
      }
    } else {
      for (int k = lane; k < d; k += 32) atomicAdd(dst + k, __fmul_rn(val, src[k]));
    }
  }
}

// Backward step 3: ReLU mask of the layer below (nn.py:167): dz = dz * (pre > 0),
// with pre > 0  <=>  relu(pre) > 0.
__global__ void spmm_bwd_mask_kernel(const int32_t* __restrict__ counts, int d,
                                     const float* __restrict__ mask_h, int ldm,
                                     float* __restrict__ dh, int lddh) {
  const int n_src = counts[0];
  const int64_t total = (int64_t)n_src * d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / d), k = (int)(i % d);
    float& x = dh[(int64_t)c * lddh + k];
    x = __fmul_rn(x, mask_h[(int64_t)c * ldm + k] > 0.f ? 1.f : 0.f);
  }
}

// y = max(x, 0) elementwise (the per-op forward's activation)
__global__ void relu_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fmaxf(x[i], 0.f);
}

}  // namespace mq

using namespace mq;

extern "C" {

int mq_relu(const float* x, float* y, int64_t n, void* stream) {
  MQ_CHECK_ARG(x && y && n >= 0, "mq_relu: bad arguments");
  if (n == 0) return MQ_OK;
  int64_t b = (n + 255) / 256;
  if (b > kNumSMs * 16) b = kNumSMs * 16;
  relu_kernel<<<(int)b, 256, 0, as_stream(stream)>>>(x, y, n);
  MQ_LAUNCH_CHECK("relu");
  return MQ_OK;
}

int mq_spmm_fwd(const int32_t* row_ptr, const int32_t* cols, const float* vals,
                const int32_t* n_dst_dev, int32_t n_dst_max, const float* h, int32_t ldh, int32_t d,
                float* agg, int32_t ldagg, void* stream) {
  MQ_CHECK_ARG(row_ptr && cols && vals && n_dst_dev && h && agg, "mq_spmm_fwd: null pointer");
  const int d4 = (d + 3) / 4;
  MQ_CHECK_ARG(d >= 1 && ldh % 4 == 0 && ldagg % 4 == 0 && ldh >= 4 * d4 && ldagg >= 4 * d4,
               "mq_spmm_fwd: leading dims must be multiples of 4 covering d");
  if (n_dst_max <= 0) return MQ_OK;
  cudaStream_t s = as_stream(stream);
  const int warps = kSpmmThreads / 32;
  int blocks = ceil_div(n_dst_max, warps);
  if (blocks > kNumSMs * 32) blocks = kNumSMs * 32;
  {
    ProfScope ps(K_SPMM_FWD, s);
    spmm_fwd_kernel<<<blocks, kSpmmThreads, 0, s>>>(row_ptr, cols, vals, n_dst_dev, h, ldh, d4, agg,
                                                    ldagg);
  }
  MQ_LAUNCH_CHECK("spmm_fwd");
  return MQ_OK;
}

int mq_spmm_bwd(const int32_t* rows, const int32_t* cols, const float* vals,
                const int32_t* counts_dev, int32_t nnz_max, const int32_t* n_dst_dev,
                int32_t n_src_max, const float* dt, int32_t lddt, int32_t d, const float* mask_h,
                int32_t ldm, float* dh, int32_t lddh, void* stream) {
  MQ_CHECK_ARG(rows && cols && vals && counts_dev && n_dst_dev && dt && dh,
               "mq_spmm_bwd: null pointer");
  MQ_CHECK_ARG(d >= 1 && lddt >= 2 * d && lddh >= d, "mq_spmm_bwd: bad leading dims");
  if (n_src_max <= 0) return MQ_OK;
  cudaStream_t s = as_stream(stream);
  const int64_t elems = (int64_t)n_src_max * d;
  int eb = ceil_div(elems, 256);
  if (eb > kNumSMs * 16) eb = kNumSMs * 16;
  {
    ProfScope ps(K_SPMM_BWD_INIT, s);
    spmm_bwd_init_kernel<<<eb, 256, 0, s>>>(counts_dev, n_dst_dev, dt, lddt, d, dh, lddh);
  }
  MQ_LAUNCH_CHECK("spmm_bwd_init");
  if (nnz_max > 0) {
    const int warps = kSpmmThreads / 32;
    int blocks = ceil_div(nnz_max, warps);
    if (blocks > kNumSMs * 32) blocks = kNumSMs * 32;
    const int vec4 = (d % 4 == 0 && lddt % 4 == 0 && lddh % 4 == 0 &&
                      ((uintptr_t)dt | (uintptr_t)dh) % 16 == 0)
                         ? 1
                         : 0;
    ProfScope ps(K_SPMM_BWD, s);
    spmm_bwd_scatter_kernel<<<blocks, kSpmmThreads, 0, s>>>(rows, cols, vals, counts_dev, dt, lddt,
                                                            d, dh, lddh, vec4);
  }
  MQ_LAUNCH_CHECK("spmm_bwd_scatter");
  if (mask_h) {
    ProfScope ps(K_SPMM_BWD_MASK, s);
    spmm_bwd_mask_kernel<<<eb, 256, 0, s>>>(counts_dev, d, mask_h, ldm, dh, lddh);
  }
  MQ_LAUNCH_CHECK("spmm_bwd_mask");
  return MQ_OK;
}

}  // extern "C"
