// Loss, optimizers, RaCoM packing and the exported scan.
//
// Reference: mqpipe/nn.py:141-156 (batch_loss), nn.py:191-215 (adam_step /
// sgd_step), racom.py:47-57,118-139 (f64 accumulation).  The optimizer update
// mirrors NumPy 2's float32 arithmetic with Python-float (weak) scalars
// operation by operation, with explicit round-to-nearest intrinsics so that
// no FMA contraction changes a rounding: the update is bit-identical to the
// reference given the same gradient.
#include "mq_common.cuh"
#include "mq_scan.cuh"
#include "mq_optim.cuh"

namespace mq {

// One warp per target row; summed loss accumulated in f64.
__global__ void softmax_ce_kernel(const float* __restrict__ logits, int ld,
                                  const int32_t* __restrict__ labels,
                                  const int32_t* __restrict__ n_dev, int C, float* __restrict__ dl,
                                  int lddl, double* __restrict__ loss_out,
                                  int32_t* __restrict__ nonfinite) {
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x / 32;
  const int n = *n_dev;
  double wloss = 0.0;
  int bad = 0;
  for (int r = blockIdx.x * warps + (threadIdx.x >> 5); r < n; r += gridDim.x * warps) {
    const float* x = logits + (int64_t)r * ld;
    float m = -INFINITY;
    for (int c = lane; c < C; c += 32) m = fmaxf(m, x[c]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float s = 0.f;
    for (int c = lane; c < C; c += 32) s += expf(x[c] - m);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float logd = logf(s);
    const int lab = labels[r];
    float* g = dl + (int64_t)r * lddl;
    for (int c = lane; c < C; c += 32) {
      const float sh = x[c] - m;
      float p = expf(sh) / s;
      if (c == lab) {
        p -= 1.f;
        wloss += -(double)(sh - logd);
      }
      g[c] = p;
      bad |= !finite_f(p);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    wloss += __shfl_xor_sync(0xffffffffu, wloss, o);
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if (lane == 0) {
    if (wloss != 0.0) atomicAdd(loss_out, wloss);
    if (bad) atomicOr(nonfinite, 1);
  }
}

__global__ void step_commit_kernel(double* loss_acc, const uint32_t* key, int world, double* ring,
                                   int ring_len) {
  MQ_PDL_ENTRY();
  int k = (int)((key[2] / (uint32_t)world) % (uint32_t)ring_len);
  ring[k] = loss_acc[0];
  loss_acc[0] = 0.0;
}

// The first `coop_blocks` blocks resolve one many-partial segment (the fused
// head's per-CTA dW partials) cooperatively: a block owns 32 consecutive
// elements, warp q sums partials q, q+8, ... (all loads in flight at once),
// warp 0 adds the 8 warp sums in warp order — fixed order, deterministic, ~1
// L2 round trip instead of nparts/16.  The other blocks take every other
// element one per thread.
__global__ void adam_kernel(float* __restrict__ w, float* __restrict__ m, float* __restrict__ v,
                            const float* __restrict__ g32, const double* __restrict__ g64,
                            double scale, int64_t n, int32_t* __restrict__ step,
                            const float* __restrict__ bias, int bias_len,
                            const float* __restrict__ lr_dev,
                            int32_t* __restrict__ nonfinite, GradSrc src, int coop_seg,
                            int coop_blocks) {
  MQ_PDL_ENTRY();
  MQ_TL_BEGIN(8);
  __shared__ float red[8][33];
  const int t = step[0] + 1;  // this update's step number (nn.py:194 t += 1)
  // a wrapped counter skips the updates (flag 2); no early return, so the
  // element loads below do not wait on the step -> bias chain
  const bool wrapped = t < 1;
  // the table ends at float32(1 - beta**t) == 1.0f for both betas (t > ~17.3k),
  // so every later step reads its last row exactly (mqgnn.h mq_adam)
  const int tb = wrapped ? 1 : (t < bias_len ? t : bias_len);
  const float bc1 = bias[2 * (tb - 1)], bc2 = bias[2 * (tb - 1) + 1];
  const float lr = *lr_dev;  // float32(learning_rate), read per launch (graph replays follow it)
  const double count = grad_count(g64, scale, n);
  int bad = 0;
  int64_t c_lo = 0, c_hi = 0;  // flat range of the cooperative segment
  if (coop_blocks > 0) {
    const mq_grad_seg& sg = src.s.seg[coop_seg];
    c_lo = sg.offset;
    c_hi = sg.offset + sg.size;
  }
  if ((int)blockIdx.x < coop_blocks) {
    const mq_grad_seg& sg = src.s.seg[coop_seg];
    const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
    const int64_t j = (int64_t)blockIdx.x * 32 + lane;  // element within the segment
    const int np = sg.nparts;
    float acc = 0.f;
    if (j < sg.size) {  // warp q sums partials q, q + 8, ... in order, 16 loads in flight
      for (int base = 0; base < np; base += 128) {
        float tv[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int p = base + q + 8 * u;
          tv[u] = p < np ? __ldcg(sg.part + (int64_t)p * sg.stride + j) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (base + q + 8 * u < np) acc += tv[u];
      }
    }
    red[q][lane] = acc;
    __syncthreads();
    if (q == 0 && j < sg.size && !wrapped) {
      float g = 0.f;
#pragma unroll
      for (int r = 0; r < 8; ++r) g += red[r][lane];
      bad |= adam_elem(w, m, v, sg.offset + j, g, bc1, bc2, lr);
    }
  } else {
    const int64_t nb = (int64_t)(gridDim.x - coop_blocks);
    for (int64_t i = (int64_t)(blockIdx.x - coop_blocks) * blockDim.x + threadIdx.x; i < n;
         i += nb * blockDim.x) {
      if (i >= c_lo && i < c_hi) continue;
      const float w0 = w[i], m0 = m[i], v0 = v[i];  // in flight with the partials
      const float g = load_grad(src, g32, g64, scale, count, i);
      if (!wrapped) bad |= adam_elem_v(w, m, v, i, w0, m0, v0, g, bc1, bc2, lr);
    }
  }
  if (wrapped && blockIdx.x == 0 && threadIdx.x == 0) atomicOr(nonfinite, 2);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
  step_arrive(step, t);
  MQ_TL_END(8);
}

__global__ void sgd_kernel(float* __restrict__ w, const float* __restrict__ g32,
                           const double* __restrict__ g64, double scale, int64_t n,
                           const float* __restrict__ lr_dev,
                           int32_t* __restrict__ step, int32_t* __restrict__ nonfinite,
                           GradSrc src) {
  MQ_PDL_ENTRY();
  const int t = step[0] + 1;
  const float lr = *lr_dev;
  const double count = grad_count(g64, scale, n);
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float wi = __fsub_rn(w[i], __fmul_rn(lr, load_grad(src, g32, g64, scale, count, i)));
    w[i] = wi;
    bad |= !finite_f(wi);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
  step_arrive(step, t);
}

__global__ void f32_to_f64_kernel(const float* __restrict__ a, double* __restrict__ b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (double)a[i];
}

__global__ void pack_grads_kernel(const float* __restrict__ a, int64_t n,
                                  const int32_t* __restrict__ n_targets, double* __restrict__ b,
                                  GradSrc src) {
  MQ_PDL_ENTRY();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = i < n ? (double)grad_at(src, a, i) : (n_targets[0] > 0 ? 1.0 : 0.0);
}

__global__ void grad_reduce_kernel(GradSrc src, const float* __restrict__ a, int64_t n,
                                   float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = grad_at(src, a, i);
}

__global__ void f64_to_f32_kernel(const double* __restrict__ a, double divisor,
                                  float* __restrict__ b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (float)(a[i] / divisor);
}

inline int elem_blocks(int64_t n) {
  int b = ceil_div(n < 1 ? 1 : n, 256);
  return b > kNumSMs * 8 ? kNumSMs * 8 : b;
}

}  // namespace mq

using namespace mq;

extern "C" {

int mq_softmax_ce(const float* logits, int32_t ld, const int32_t* labels, const int32_t* n_dev,
                  int32_t n_max, int32_t n_classes, float* dlogits, int32_t lddl, double* loss_out,
                  int32_t* nonfinite, void* stream) {
  MQ_CHECK_ARG(logits && labels && n_dev && dlogits && loss_out && nonfinite,
               "mq_softmax_ce: null pointer");
  MQ_CHECK_ARG(n_classes >= 1 && ld >= n_classes && lddl >= n_classes, "mq_softmax_ce: bad dims");
  if (n_max <= 0) return MQ_OK;
  cudaStream_t s = as_stream(stream);
  int blocks = ceil_div(n_max, 8);
  if (blocks > kNumSMs * 4) blocks = kNumSMs * 4;
  {
    ProfScope ps(K_SOFTMAX_CE, s);
    softmax_ce_kernel<<<blocks, 256, 0, s>>>(logits, ld, labels, n_dev, n_classes, dlogits, lddl,
                                             loss_out, nonfinite);
  }
  MQ_LAUNCH_CHECK("softmax_ce");
  return MQ_OK;
}

int mq_adam(float* w, float* m, float* v, const float* grad32, const double* grad64,
            double grad_scale, int64_t n, int32_t* step_dev, const float* bias, int32_t bias_len,
            const float* lr, int32_t* nonfinite, const mq_grad_src* src, void* stream) {
  MQ_CHECK_ARG(w && m && v && step_dev && bias && lr && nonfinite, "mq_adam: null pointer");
  MQ_CHECK_ARG(bias_len >= 1, "mq_adam: empty bias-correction table");
  MQ_CHECK_ARG((grad32 == nullptr) != (grad64 == nullptr), "mq_adam: exactly one gradient source");
  MQ_CHECK_ARG(src_ok(src), "mq_adam: bad deferred gradient source");
  cudaStream_t s = as_stream(stream);
  // a kind-0 segment with many static partials (the head's) goes cooperative
  int coop_seg = 0, coop_blocks = 0;
  if (grad32 && src) {
    for (int k = 0; k < src->nseg; ++k) {
      const mq_grad_seg& sg = src->seg[k];
      if (sg.kind == 0 && !sg.nparts_dev && sg.nparts > 32 && sg.size > 0) {
        coop_seg = k;
        coop_blocks = (int)((sg.size + 31) / 32);
        break;
      }
    }
  }
  {
    ProfScope ps(K_ADAM, s);
    MQ_CUDA(launch_k(adam_kernel, dim3(elem_blocks(n) + coop_blocks), dim3(256), 0, s, w, m, v, grad32, grad64, grad_scale, n, step_dev,
                                               bias, bias_len, lr, nonfinite, make_src(src),
                     coop_seg, coop_blocks));
  }
  MQ_LAUNCH_CHECK("adam");
  return MQ_OK;
}

int mq_sgd(float* w, const float* grad32, const double* grad64, double grad_scale, int64_t n,
           int32_t* step_dev, const float* lr, int32_t* nonfinite, const mq_grad_src* src,
           void* stream) {
  MQ_CHECK_ARG(w && step_dev && lr && nonfinite, "mq_sgd: null pointer");
  MQ_CHECK_ARG((grad32 == nullptr) != (grad64 == nullptr), "mq_sgd: exactly one gradient source");
  MQ_CHECK_ARG(src_ok(src), "mq_sgd: bad deferred gradient source");
  cudaStream_t s = as_stream(stream);
  {
    ProfScope ps(K_SGD, s);
    MQ_CUDA(launch_k(sgd_kernel, dim3(elem_blocks(n)), dim3(256), 0, s, w, grad32, grad64, grad_scale, n, lr, step_dev,
                                              nonfinite, make_src(src)));
  }
  MQ_LAUNCH_CHECK("sgd");
  return MQ_OK;
}

int mq_step_commit(double* loss_acc, const uint32_t* key_dev, int32_t world, double* loss_ring,
                   int32_t ring_len, void* stream) {
  MQ_CHECK_ARG(loss_acc && key_dev && loss_ring && ring_len > 0 && world >= 1,
               "mq_step_commit: bad args");
  cudaStream_t s = as_stream(stream);
  {
    ProfScope ps(K_STEP_BUMP, s);
    MQ_CUDA(launch_k(step_commit_kernel, dim3(1), dim3(1), 0, s, loss_acc, key_dev, world, loss_ring, ring_len));
  }
  MQ_LAUNCH_CHECK("step_commit");
  return MQ_OK;
}

int mq_f32_to_f64(const float* in32, double* out64, int64_t n, void* stream) {
  MQ_CHECK_ARG(in32 && out64, "mq_f32_to_f64: null pointer");
  if (n <= 0) return MQ_OK;
  cudaStream_t s = as_stream(stream);
  {
    ProfScope ps(K_CONVERT, s);
    f32_to_f64_kernel<<<elem_blocks(n), 256, 0, s>>>(in32, out64, n);
  }
  MQ_LAUNCH_CHECK("f32_to_f64");
  return MQ_OK;
}

int mq_pack_grads(const float* grad, int64_t n, const int32_t* n_targets_dev, double* out64,
                  const mq_grad_src* src, void* stream) {
  MQ_CHECK_ARG(grad && n_targets_dev && out64, "mq_pack_grads: null pointer");
  MQ_CHECK_ARG(src_ok(src), "mq_pack_grads: bad gradient source");
  cudaStream_t s = as_stream(stream);
  {
    ProfScope ps(K_CONVERT, s);
    MQ_CUDA(launch_k(pack_grads_kernel, dim3(elem_blocks(n + 1)), dim3(256), 0, s, grad, n, n_targets_dev, out64,
                                                         make_src(src)));
  }
  MQ_LAUNCH_CHECK("pack_grads");
  return MQ_OK;
}

int mq_grad_reduce(const mq_grad_src* src, const float* grad32, int64_t n, float* out32,
                   void* stream) {
  MQ_CHECK_ARG(grad32 && out32 && src_ok(src), "mq_grad_reduce: bad arguments");
  if (n <= 0) return MQ_OK;
  cudaStream_t s = as_stream(stream);
  {
    ProfScope ps(K_CONVERT, s);
    grad_reduce_kernel<<<elem_blocks(n), 256, 0, s>>>(make_src(src), grad32, n, out32);
  }
  MQ_LAUNCH_CHECK("grad_reduce");
  return MQ_OK;
}

int mq_f64_to_f32(const double* in64, double divisor, float* out32, int64_t n, void* stream) {
  MQ_CHECK_ARG(in64 && out32 && divisor != 0.0, "mq_f64_to_f32: null pointer or zero divisor");
  if (n <= 0) return MQ_OK;
  cudaStream_t s = as_stream(stream);
  {
    ProfScope ps(K_CONVERT, s);
    f64_to_f32_kernel<<<elem_blocks(n), 256, 0, s>>>(in64, divisor, out32, n);
  }
  MQ_LAUNCH_CHECK("f64_to_f32");
  return MQ_OK;
}

int mq_scan_i32(const int32_t* in, const int32_t* n_dev, int32_t n_max, int32_t* out,
                void* scratch, void* stream) {
  MQ_CHECK_ARG(in && n_dev && out && scratch, "mq_scan_i32: null pointer");
  return launch_scan(LoadI32{in, n_dev, 0}, StoreOffsets<int32_t>{out}, n_max < 1 ? 1 : n_max,
                     scratch, as_stream(stream));
}

}  // extern "C"

MQ_TL_READER(train)
