// RaCoM gradient sharing over peer memory (NVLink P2P / CUDA IPC).
//
// Reference: mqpipe/racom.py:36-87 (Accumulator running mean in f64,
// apply_update), racom.py:142-184 (share_gradient: every packet goes to every
// device's inbox, self included), runtime.py:167-195 (windows applied in
// order, exactly expected[k] contributions).
//
// The reference broadcasts each device's packet to all inboxes and every
// device folds the packets of a window into a running f64 mean.  Here each
// rank writes its packet once into its own arena and raises a per-source flag
// word in every rank's arena (release, system scope); the apply kernel of
// every rank waits on its local flag words (acquire), reads all packets over
// NVLink in rank order and folds them exactly like Accumulator.accumulate in
// the serial reference's arrival order (device 0, 1, ...), then runs the
// NumPy-2 f32 Adam / SGD update.  Every rank therefore computes bit-identical
// weights without any collective call, and the window is stream-ordered on
// the device (capturable into the step's CUDA graph).
#include "mq_common.cuh"
#include "mq_optim.cuh"

namespace mq {

constexpr int kPeerThreads = 256;
constexpr int64_t kFlagsOff = 0;     // u64 [MQ_MAX_PEERS]
constexpr int64_t kCountersOff = 64; // u64 [published, applied, publish arrivals]

__host__ __device__ __forceinline__ int64_t slot_stride_bytes(int64_t n) {
  return (((n + 1) * 4 + 255) / 256) * 256;
}

__device__ __forceinline__ unsigned long long* flags_of(const mq_peer_exchange& ex, int q) {
  return reinterpret_cast<unsigned long long*>(ex.arena[q] + kFlagsOff);
}
__device__ __forceinline__ unsigned long long* counters(const mq_peer_exchange& ex) {
  return reinterpret_cast<unsigned long long*>(ex.arena[ex.rank] + kCountersOff);
}
__device__ __forceinline__ float* slot_of_rank(const mq_peer_exchange& ex, int q, uint64_t k) {
  return reinterpret_cast<float*>(ex.arena[q] + MQ_PEER_HEADER_BYTES +
                                  (int64_t)(k % (uint64_t)ex.ring) * slot_stride_bytes(ex.n));
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float ld_relaxed_sys(const float* p) {
  float v;
  asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// share_gradient: this rank's packet for window k into its own slot, then the
// flag word flags[rank] = k + 1 in every rank's arena.
__global__ void __launch_bounds__(kPeerThreads) racom_publish_kernel(
    mq_peer_exchange ex, const float* __restrict__ g32, GradSrc src,
    const int32_t* __restrict__ n_targets) {
  MQ_PDL_ENTRY();
  unsigned long long* ctr = counters(ex);
  const uint64_t k = ctr[0];
  float* dst = slot_of_rank(ex, ex.rank, k);
  const int64_t n = ex.n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = i < n ? grad_at(src, g32, i) : (n_targets[0] > 0 ? 1.f : 0.f);
  // every thread's slot stores are ordered before its CTA's arrival, and the
  // last CTA's flag stores (release, system scope) after all arrivals
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(&ctr[2], 1ull) == (unsigned long long)gridDim.x - 1) {
      __threadfence_system();
      ctr[2] = 0;
      ctr[0] = k + 1;
      for (int q = 0; q < ex.world; ++q) st_release_sys(flags_of(ex, q) + ex.rank, k + 1);
    }
  }
}

// Accumulator + apply_update: wait for every rank's packet of window k, fold
// them in rank order in f64 (racom.py:47-57), cast to f32 (nn.py:197), update.
__global__ void __launch_bounds__(kPeerThreads) racom_apply_kernel(
    mq_peer_exchange ex, int optimizer, int lag, float* __restrict__ w, float* __restrict__ m,
    float* __restrict__ v, int32_t* __restrict__ step, const float* __restrict__ bias,
    int bias_len, const float* __restrict__ lr_dev, int32_t* __restrict__ nonfinite) {
  MQ_PDL_ENTRY();
  __shared__ int s_go;
  __shared__ float s_contrib[MQ_MAX_PEERS];
  unsigned long long* ctr = counters(ex);
  const uint64_t published = ctr[0], k = ctr[1];
  // nothing (old enough) to apply: the pipelined schedule's first window
  if (published <= k + (uint64_t)lag) return;
  const int t = step[0] + 1;
  if (threadIdx.x == 0) {
    int go = 1;
    const unsigned long long t0 = global_ns();
    const unsigned long long bound =
        ex.timeout_ns > 0 ? (unsigned long long)ex.timeout_ns : 30ull * 1000000000ull;
    const unsigned long long* fl = flags_of(ex, ex.rank);
    for (int q = 0; q < ex.world && go; ++q) {
      while (ld_acquire_sys(fl + q) < k + 1) {
        if (global_ns() - t0 > bound) {
          go = 0;
          break;
        }
        __nanosleep(64);
      }
    }
    if (go) {
      for (int q = 0; q < ex.world; ++q) s_contrib[q] = ld_relaxed_sys(slot_of_rank(ex, q, k) + ex.n);
    } else if (blockIdx.x == 0) {
      atomicOr(nonfinite, 8);  // a peer never published: timeout
    }
    s_go = go;
  }
  __syncthreads();
  int bad = 0;
  if (s_go) {
    const float lr = *lr_dev;
    const int tb = t < bias_len ? t : bias_len;  // saturated table (mqgnn.h mq_adam)
    const float bc1 = bias[2 * (tb - 1)], bc2 = bias[2 * (tb - 1) + 1];
    const int64_t n = ex.n;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
      float pk[MQ_MAX_PEERS];
#pragma unroll
      for (int q = 0; q < MQ_MAX_PEERS; ++q)
        pk[q] = (q < ex.world && s_contrib[q] > 0.f) ? ld_relaxed_sys(slot_of_rank(ex, q, k) + i)
                                                     : 0.f;
      double mean = 0.0;
      int count = 0;
#pragma unroll
      for (int q = 0; q < MQ_MAX_PEERS; ++q) {
        if (q < ex.world && s_contrib[q] > 0.f) {
          ++count;
          mean = count == 1 ? (double)pk[q] : mean + ((double)pk[q] - mean) / (double)count;
        }
      }
      const float g = (float)mean;
      if (optimizer == 0) {
        bad |= adam_elem(w, m, v, i, g, bc1, bc2, lr);
      } else {
        const float wi = __fsub_rn(w[i], __fmul_rn(lr, g));
        w[i] = wi;
        bad |= !finite_f(wi);
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
  // last CTA: applied = k + 1 and the optimizer's step count (step_arrive)
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&step[1], 1) == (int)gridDim.x - 1) {
      if (s_go) {
        step[0] = t;
        ctr[1] = k + 1;
      }
      step[1] = 0;
    }
  }
}

__global__ void peer_state_kernel(mq_peer_exchange ex, unsigned long long* out) {
  unsigned long long* ctr = counters(ex);
  const unsigned long long* fl = flags_of(ex, ex.rank);
  unsigned long long lo = ~0ull, hi = 0;
  for (int q = 0; q < ex.world; ++q) {
    const unsigned long long f = ld_acquire_sys(fl + q);
    lo = f < lo ? f : lo;
    hi = f > hi ? f : hi;
  }
  out[0] = ctr[0];
  out[1] = ctr[1];
  out[2] = lo;
  out[3] = hi;
}

static bool exchange_ok(const mq_peer_exchange* ex) {
  if (!ex || ex->world < 1 || ex->world > MQ_MAX_PEERS || ex->rank < 0 ||
      ex->rank >= ex->world || ex->ring < 1 || ex->n < 1)
    return false;
  for (int q = 0; q < ex->world; ++q)
    if (!ex->arena[q] || (reinterpret_cast<uintptr_t>(ex->arena[q]) & 255)) return false;
  return true;
}

static int peer_grid(int64_t n) {
  int b = ceil_div(n + 1, kPeerThreads);
  return b > kNumSMs ? kNumSMs : (b < 1 ? 1 : b);
}

}  // namespace mq

using namespace mq;

extern "C" {

int64_t mq_peer_arena_bytes(int64_t n, int32_t ring) {
  if (n < 1 || ring < 1) return -1;
  return MQ_PEER_HEADER_BYTES + (int64_t)ring * slot_stride_bytes(n);
}

int mq_peer_alloc(int64_t bytes, void** out) {
  MQ_CHECK_ARG(out && bytes > 0, "mq_peer_alloc: bad args");
  void* p = nullptr;
  MQ_CUDA(cudaMalloc(&p, (size_t)bytes));
  MQ_CUDA(cudaMemset(p, 0, (size_t)bytes));
  MQ_CUDA(cudaDeviceSynchronize());
  *out = p;
  return MQ_OK;
}

int mq_peer_free(void* p) {
  if (p) MQ_CUDA(cudaFree(p));
  return MQ_OK;
}

int mq_ipc_export(void* dev_ptr, mq_ipc_handle* out) {
  static_assert(sizeof(mq_ipc_handle) == sizeof(cudaIpcMemHandle_t), "IPC handle size");
  MQ_CHECK_ARG(dev_ptr && out, "mq_ipc_export: bad args");
  cudaIpcMemHandle_t h;
  MQ_CUDA(cudaIpcGetMemHandle(&h, dev_ptr));
  memcpy(out, &h, sizeof(h));
  return MQ_OK;
}

int mq_ipc_open(const mq_ipc_handle* h, void** out) {
  MQ_CHECK_ARG(h && out, "mq_ipc_open: bad args");
  cudaIpcMemHandle_t hh;
  memcpy(&hh, h, sizeof(hh));
  void* p = nullptr;
  // another GPU: enable peer access lazily; the same GPU (ranks sharing a
  // device) maps the pages directly
  if (cudaIpcOpenMemHandle(&p, hh, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    MQ_CUDA(cudaIpcOpenMemHandle(&p, hh, 0));
  }
  *out = p;
  return MQ_OK;
}

int mq_ipc_close(void* p) {
  if (p) MQ_CUDA(cudaIpcCloseMemHandle(p));
  return MQ_OK;
}

int mq_racom_publish(const mq_peer_exchange* ex, const float* grad32, const mq_grad_src* src,
                     const int32_t* n_targets_dev, void* stream) {
  MQ_CHECK_ARG(exchange_ok(ex), "mq_racom_publish: bad exchange");
  MQ_CHECK_ARG(grad32 && n_targets_dev, "mq_racom_publish: null pointer");
  MQ_CHECK_ARG(src_ok(src), "mq_racom_publish: bad deferred gradient source");
  cudaStream_t s = as_stream(stream);
  {
    ProfScope ps(K_RACOM_PUBLISH, s);
    MQ_CUDA(launch_k(racom_publish_kernel, dim3(peer_grid(ex->n)), dim3(kPeerThreads), 0, s,
                     *ex, grad32, make_src(src), n_targets_dev));
  }
  MQ_LAUNCH_CHECK("racom_publish");
  return MQ_OK;
}

int mq_racom_apply(const mq_peer_exchange* ex, int32_t optimizer, int32_t lag, float* w, float* m,
                   float* v, int32_t* step_dev, const float* bias, int32_t bias_len,
                   const float* lr, int32_t* nonfinite, void* stream) {
  MQ_CHECK_ARG(exchange_ok(ex), "mq_racom_apply: bad exchange");
  MQ_CHECK_ARG(optimizer == 0 || optimizer == 1, "mq_racom_apply: optimizer 0 (adam) or 1 (sgd)");
  MQ_CHECK_ARG(lag >= 0 && lag < ex->ring - 1, "mq_racom_apply: lag must be < ring - 1");
  MQ_CHECK_ARG(w && step_dev && lr && nonfinite, "mq_racom_apply: null pointer");
  MQ_CHECK_ARG(optimizer == 1 || (m && v && bias && bias_len >= 1),
               "mq_racom_apply: Adam needs m, v and the bias table");
  cudaStream_t s = as_stream(stream);
  {
    ProfScope ps(K_RACOM_APPLY, s);
    MQ_CUDA(launch_k(racom_apply_kernel, dim3(peer_grid(ex->n)), dim3(kPeerThreads), 0, s, *ex,
                     (int)optimizer, (int)lag, w, m, v, step_dev, bias, (int)bias_len, lr,
                     nonfinite));
  }
  MQ_LAUNCH_CHECK("racom_apply");
  return MQ_OK;
}

int mq_peer_state(const mq_peer_exchange* ex, unsigned long long* out4, void* stream) {
  MQ_CHECK_ARG(exchange_ok(ex) && out4, "mq_peer_state: bad args");
  peer_state_kernel<<<1, 1, 0, as_stream(stream)>>>(*ex, out4);
  MQ_LAUNCH_CHECK("peer_state");
  return MQ_OK;
}

}  // extern "C"
