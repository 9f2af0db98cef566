// Optimizer building blocks shared by mq_train.cu (mq_adam / mq_sgd) and
// mq_peer.cu (the fused RaCoM apply): deferred split-K gradient resolution,
// the NumPy-2 f32 Adam element update, and the step counter bump.
#pragma once

#include "mq_common.cuh"

namespace mq {

__device__ __forceinline__ bool finite_f(float x) { return isfinite(x); }

// grad32, or the f64 window sum: * scale, or (scale == 0) / the all-reduced
// contributor count packed at g64[n] by mq_pack_grads
// step[0] = update count, step[1] = arrival counter (0 at rest): every CTA
// reads step[0] on entry; the last CTA to arrive publishes t and resets the
// counter, so the bump is fused into the optimizer launch.
__device__ __forceinline__ void step_arrive(int32_t* step, int t) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&step[1], 1) == (int)gridDim.x - 1) {
      step[0] = t;
      step[1] = 0;
    }
  }
}

// Gradient element i through the deferred split-K segments (mqgnn.h).
struct GradSrc {
  mq_grad_src s;
  bool on;
};

__device__ __forceinline__ float grad_at(const GradSrc& src, const float* g32, int64_t i) {
  if (src.on) {
    for (int k = 0; k < src.s.nseg; ++k) {
      const mq_grad_seg& sg = src.s.seg[k];
      if (i >= sg.offset && i < sg.offset + sg.size) {
        int64_t j = i - sg.offset;
        if (sg.kind == 1) {
          const int64_t row = j / sg.d_out, col = j % sg.d_out;
          j = row < sg.d_in ? row * 2 * sg.d_out + col
                            : (row - sg.d_in) * 2 * sg.d_out + sg.d_out + col;
        }
        const int np = sg.nparts_dev ? *sg.nparts_dev : sg.nparts;
        return fixed_order_sum(sg.part + j, sg.stride, np);
      }
    }
  }
  return g32[i];
}

__device__ __forceinline__ float load_grad(const GradSrc& src, const float* g32, const double* g64,
                                           double scale, double count, int64_t i) {
  if (g32) return grad_at(src, g32, i);
  return scale != 0.0 ? (float)(g64[i] * scale) : (float)(g64[i] / count);
}

__device__ __forceinline__ double grad_count(const double* g64, double scale, int64_t n) {
  return (g64 != nullptr && scale == 0.0) ? g64[n] : 1.0;
}

// Adam update of element i with gradient g (nn.py:191-206, NumPy-2 f32 op order),
// given the element's current w / m / v (loaded by the caller ahead of the
// gradient's partial sums, so their latency overlaps)
__device__ __forceinline__ bool adam_elem_v(float* __restrict__ w, float* __restrict__ m,
                                            float* __restrict__ v, int64_t i, float w0, float m0,
                                            float v0, float g, float bc1, float bc2, float lr) {
  const float b1 = (float)0.9, b2 = (float)0.999;
  const float c1 = (float)(1.0 - 0.9), c2 = (float)(1.0 - 0.999), eps = (float)1e-8;
  float mi = __fmul_rn(m0, b1);                           // m *= beta1
  mi = __fadd_rn(mi, __fmul_rn(c1, g));                   // m += (1-beta1)*g
  float vi = __fmul_rn(v0, b2);                           // v *= beta2
  vi = __fadd_rn(vi, __fmul_rn(__fmul_rn(c2, g), g));     // v += (1-beta2)*g*g
  const float mh = __fdiv_rn(mi, bc1);                    // m / (1 - beta1**t)
  const float vh = __fdiv_rn(vi, bc2);                    // v / (1 - beta2**t)
  const float upd = __fdiv_rn(__fmul_rn(lr, mh), __fadd_rn(__fsqrt_rn(vh), eps));
  const float wi = __fsub_rn(w0, upd);                    // w -= lr*mh/(sqrt(vh)+eps)
  m[i] = mi;
  v[i] = vi;
  w[i] = wi;
  return !finite_f(wi);
}
__device__ __forceinline__ bool adam_elem(float* __restrict__ w, float* __restrict__ m,
                                          float* __restrict__ v, int64_t i, float g, float bc1,
                                          float bc2, float lr) {
  return adam_elem_v(w, m, v, i, w[i], m[i], v[i], g, bc1, bc2, lr);
}

inline GradSrc make_src(const mq_grad_src* src) {
  GradSrc g;
  memset(&g, 0, sizeof(g));
  if (src != nullptr && src->nseg > 0) {
    g.s = *src;
    g.on = true;
  }
  return g;
}

inline bool src_ok(const mq_grad_src* src) {
  if (src == nullptr) return true;
  if (src->nseg < 0 || src->nseg > MQ_GRAD_MAX_SEG) return false;
  for (int k = 0; k < src->nseg; ++k) {
    const mq_grad_seg& sg = src->seg[k];
    if (!sg.part || sg.size < 0 || sg.offset < 0 || (!sg.nparts_dev && sg.nparts < 0)) return false;
    if (sg.kind == 1 && (sg.d_in < 1 || sg.d_out < 1 || sg.size != 2LL * sg.d_in * sg.d_out))
      return false;
  }
  return true;
}


}  // namespace mq
