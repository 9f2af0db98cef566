// The fused SAGE training step: transform-first hidden layers and a one-launch
// head (aggregate + transform + softmax-CE + backward of the last layer).
//
// Reference: mqpipe/nn.py:116-180 (sage_forward, batch_loss, backward).  The
// reference evaluates every layer aggregate-first,
//     z = [A h | h_dst] W,          W = [W_top ; W_bot]  (2 d_in x d_out),
// which for the Reddit-shaped input layer means a 602-wide SpMM over every
// sampled edge.  A hidden layer here is evaluated transform-first (the same
// linear map, re-associated):
//     Y = h [W_top | W_bot]          (n_src x 2 d_out; one dense GEMM over the
//                                     sampled rows, h read once)
//     z[r] = sum_e val_e Y_top[col_e] + Y_bot[r]
// and its backward never needs the wide aggregate either:
//     dz = dh_out * (z > 0)
//     G  = [A^T dz | dz (dst rows, zero below)]     (n_src x 2 d_out)
//     dW = h^T G  -> rows [0, d_in) = W_top grad, [d_in, 2 d_in) = W_bot grad
//     dh = G [W_top | W_bot]^T                      (only for layers above 0)
// so the aggregation runs at d_out = 64 instead of d_in = 602.  The result is
// the reference's up to fp32 re-association (DESIGN.md §5 tolerances).
//
// The last layer (hop 0, the seeds' block) stays aggregate-first and is ONE
// kernel: each CTA owns R target rows, aggregates them (sequential fp32 in
// triplet order = np.add.at), applies W (smem-resident), runs the summed
// softmax-CE (nn.py:141-156), back-propagates dt = dl W^T straight into dh
// with vector atomics (block_apply_t + the self half, nn.py:171-174), writes
// its dW partial, and after a grid barrier the CTAs reduce the partials in a
// fixed order (deterministic dW).  CTA 0 then commits the batch loss to the
// epoch's loss ring.
#include <climits>

#include "mq_gemm.cuh"

#ifndef MQ_AGG_U
#define MQ_AGG_U 4  // neighbour rows per batch of split-partial loads in sage_aggregate_parts
#endif
#ifndef MQ_AGG_SU
#define MQ_AGG_SU 4  // split partials loaded per batch in sage_aggregate_parts
#endif

namespace mq {

// tcgen05 3xTF32 path (mq_tc.cu)
int tc_backend();
bool tc_supported(int n_out);
int tc_transform(const float* h, int ldh, const int32_t* m_dev, int m_max, int d_in, const float* W,
                 int d_out, float* y, float* part, int32_t* nparts_out, cudaStream_t s);
int64_t tc_y_part_floats(int64_t m_max, int64_t d_out);
int tc_weight_grad(const float* h, int ldh, const int32_t* rows_dev, int rows_max, int d_in,
                   int d_out, const float* g, float* dW, float* part, int32_t* nparts_out,
                   cudaStream_t s);
int64_t tc_dw_part_floats(int64_t d_in, int64_t d_out);
int64_t tc_scratch_floats(int64_t m_max, int64_t d_in, int64_t d_out);
int tc_linear_af(const float* agg, int ldagg, const float* h, int ldh, const int32_t* m_dev,
                 int m_max, int d_in, const float* W, int d_out, float* act, int ldact,
                 float* part, cudaStream_t s);
int64_t tc_af_part_floats(int64_t m_max, int64_t d_out);
int tc_linear_af_bwd(const float* agg, int ldagg, const float* h, int ldh,
                     const int32_t* rows_dev, int rows_max, int d_in, const float* dh, int lddh,
                     const float* act, int ldact, int d_out, float* part, int32_t* nparts_out,
                     cudaStream_t s);
int64_t tc_af_dw_part_floats(int64_t d_in, int64_t d_out);
int tc_dx(const float* g, const int32_t* m_dev, int m_max, int d_in, int d_out, const float* W,
          float* dh, int lddh, float* part, cudaStream_t s);


// ------------------------------------------------------------ GEMM loaders
// B(k, j) of Y = h [W_top | W_bot]: k < d_in, j < 2N
struct BLoadWSplit {
  const float* W;
  int d_in;
  int N;
  __device__ float4 load4(int k, int j) const {
    if (k >= d_in) return make_float4(0.f, 0.f, 0.f, 0.f);
    float v[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int jj = j + t;
      v[t] = jj < N ? __ldg(W + (int64_t)k * N + jj)
                    : (jj < 2 * N ? __ldg(W + (int64_t)(d_in + k) * N + (jj - N)) : 0.f);
    }
    return make_float4(v[0], v[1], v[2], v[3]);
  }
};
struct BLoadWSplitVec {  // N % 4 == 0 and W 16-byte aligned
  const float* W;
  int d_in;
  int N;
  __device__ float4 load4(int k, int j) const {
    if (k >= d_in || j >= 2 * N) return make_float4(0.f, 0.f, 0.f, 0.f);
    const float* p = j < N ? W + (int64_t)k * N + j : W + (int64_t)(d_in + k) * N + (j - N);
    return __ldg(reinterpret_cast<const float4*>(p));
  }
};
// A(o, r) = h[r, o] (dW = h^T G): o contiguous
struct ALoadT {
  static constexpr bool kKContig = false;
  const float* h;
  int ld;
  __device__ float4 load4m(int o, int r) const {
    return __ldg(reinterpret_cast<const float4*>(h + (int64_t)r * ld + o));
  }
};
// B(k, j) of dh = G [W_top | W_bot]^T: k < 2N, j < d_in
struct BLoadWSplitT {
  const float* W;
  int d_in;
  int N;
  __device__ float4 load4(int k, int j) const {
    float v[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int jj = j + t;
      float x = 0.f;
      if (jj < d_in && k < 2 * N)
        x = k < N ? __ldg(W + (int64_t)jj * N + k) : __ldg(W + (int64_t)(d_in + jj) * N + (k - N));
      v[t] = x;
    }
    return make_float4(v[0], v[1], v[2], v[3]);
  }
};
// ------------------------------------------------------------ aggregate
struct ZeroRange {
  float* p;
  const int32_t* rows_dev;
  int row_floats;
};

__device__ __forceinline__ void zero_range(ZeroRange z, int64_t tid, int64_t nthreads) {
  if (z.p == nullptr) return;
  const int64_t n = (int64_t)(*z.rows_dev) * z.row_floats;
  if ((z.row_floats & 3) == 0 && ((uintptr_t)z.p & 15) == 0) {
    float4* p4 = reinterpret_cast<float4*>(z.p);
    const float4 zz = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t i = tid; i < n / 4; i += nthreads) p4[i] = zz;
  } else {
    for (int64_t i = tid; i < n; i += nthreads) z.p[i] = 0.f;
  }
}

constexpr int kAggThreads = 256;

// Row aggregation: sum over the edges [e0, e1) of val_e * h[col_e, c .. c+1]
// (lanes own a float2 column pair).  With kExact the products are rounded
// separately and added sequentially in edge order — np.add.at's evaluation
// order (nn.py:88) — otherwise fused multiply-adds.  The row's gathers are
// issued U at a time, so a row costs about ceil(nnz / U) L2 round trips
// instead of nnz dependent ones.
template <bool kExact>
__device__ __forceinline__ float2 row_agg2(const int32_t* __restrict__ cols,
                                           const float* __restrict__ vals, int e0, int e1,
                                           const float* __restrict__ h, int ldh, int c,
                                           bool active) {
  constexpr int U = 8;
  const int lane = threadIdx.x & 31;
  float2 acc = make_float2(0.f, 0.f);
  for (int eb = e0; eb < e1; eb += 32) {
    const int me = eb + lane;
    int32_t my_col = 0;
    float my_val = 0.f;
    if (me < e1) {
      my_col = __ldg(&cols[me]);
      my_val = __ldg(&vals[me]);
    }
    const int m = min(32, e1 - eb);
    for (int t0 = 0; t0 < m; t0 += U) {
      float2 x[U];
      float v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = t0 + u;
        const int32_t col = __shfl_sync(0xffffffffu, my_col, t & 31);
        v[u] = __shfl_sync(0xffffffffu, my_val, t & 31);
        x[u] = (active && t < m)
                   ? __ldg(reinterpret_cast<const float2*>(h + (int64_t)col * ldh + c))
                   : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (t0 + u < m) {
          if (kExact) {
            acc.x = __fadd_rn(acc.x, __fmul_rn(v[u], x[u].x));
            acc.y = __fadd_rn(acc.y, __fmul_rn(v[u], x[u].y));
          } else {
            acc.x = fmaf(v[u], x[u].x, acc.x);
            acc.y = fmaf(v[u], x[u].y, acc.y);
          }
        }
      }
    }
  }
  return acc;
}

// scalar-column variant (odd widths / pitches)
template <bool kExact>
__device__ __forceinline__ float row_agg1(const int32_t* __restrict__ cols,
                                          const float* __restrict__ vals, int e0, int e1,
                                          const float* __restrict__ h, int ldh, int c,
                                          bool active) {
  constexpr int U = 8;
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  for (int eb = e0; eb < e1; eb += 32) {
    const int me = eb + lane;
    int32_t my_col = 0;
    float my_val = 0.f;
    if (me < e1) {
      my_col = __ldg(&cols[me]);
      my_val = __ldg(&vals[me]);
    }
    const int m = min(32, e1 - eb);
    for (int t0 = 0; t0 < m; t0 += U) {
      float x[U], v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = t0 + u;
        const int32_t col = __shfl_sync(0xffffffffu, my_col, t & 31);
        v[u] = __shfl_sync(0xffffffffu, my_val, t & 31);
        x[u] = (active && t < m) ? __ldg(h + (int64_t)col * ldh + c) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (t0 + u < m) acc = kExact ? __fadd_rn(acc, __fmul_rn(v[u], x[u])) : fmaf(v[u], x[u], acc);
    }
  }
  return acc;
}

// act[r, j] = relu(sum_e val_e Y[col_e, j] + Y[r, N + j]) for r < n_dst; pad
// columns [N, ldact) are written as zeros.  Then zero the requested ranges.
__global__ void __launch_bounds__(kAggThreads) sage_aggregate_kernel(
    const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ cols,
    const float* __restrict__ vals, const int32_t* __restrict__ n_dst_dev,
    const float* __restrict__ y, int N, float* __restrict__ act, int ldact, ZeroRange z0,
    ZeroRange z1) {
  MQ_PDL_ENTRY();
  const int lane = threadIdx.x & 31;
  const int warps = kAggThreads / 32;
  const int n = *n_dst_dev;
  const int ldy = 2 * N;
  const bool vec2 = (N & 1) == 0 && (ldact & 1) == 0 && (((uintptr_t)y | (uintptr_t)act) & 7) == 0;
  for (int r = blockIdx.x * warps + (threadIdx.x >> 5); r < n; r += gridDim.x * warps) {
    const int e0 = row_ptr[r], e1 = row_ptr[r + 1];
    const float* yb = y + (int64_t)r * ldy + N;
    float* out = act + (int64_t)r * ldact;
    if (vec2) {
      for (int cb = 0; cb < ldact; cb += 64) {
        const int c = cb + 2 * lane;
        const float2 acc = row_agg2<false>(cols, vals, e0, e1, y, ldy, c, c < N);
        if (c < N) {
          const float2 b = __ldg(reinterpret_cast<const float2*>(yb + c));
          const float zx = acc.x + b.x, zy = acc.y + b.y;
          *reinterpret_cast<float2*>(out + c) = make_float2(zx > 0.f ? zx : 0.f, zy > 0.f ? zy : 0.f);
        } else if (c < ldact) {
          *reinterpret_cast<float2*>(out + c) = make_float2(0.f, 0.f);
        }
      }
    } else {
      for (int cb = 0; cb < ldact; cb += 32) {
        const int c = cb + lane;
        const float acc = row_agg1<false>(cols, vals, e0, e1, y, ldy, c, c < N);
        if (c < N) {
          const float z = acc + __ldg(yb + c);
          out[c] = z > 0.f ? z : 0.f;
        } else if (c < ldact) {
          out[c] = 0.f;
        }
      }
    }
  }
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  zero_range(z0, tid, nth);
  zero_range(z1, tid, nth);
}

// Same as sage_aggregate_kernel but Y arrives as the split-K partial tiles of
// the tensor-core transform (part[s][m][2N], s < *nparts, m < *m_dev): the
// reduction over s happens on the fly in fixed order, so the transform needs
// no separate reduction pass.  (float2 columns: N even.)
__global__ void __launch_bounds__(kAggThreads) sage_aggregate_parts_kernel(
    const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ cols,
    const float* __restrict__ vals, const int32_t* __restrict__ n_dst_dev,
    const float* __restrict__ part, const int32_t* __restrict__ nparts_dev,
    const int32_t* __restrict__ m_dev, int N, float* __restrict__ act, int ldact, ZeroRange z0,
    ZeroRange z1) {
  pdl_trigger();
  MQ_TL_BEGIN(5);
  constexpr int U = MQ_AGG_U, SU = MQ_AGG_SU;
  const int lane = threadIdx.x & 31;
  const int warps = kAggThreads / 32;
  // the block (prep output) is read ahead of the wait; the partials are not
  const int n = *n_dst_dev;
  int r = blockIdx.x * warps + (threadIdx.x >> 5);
  int pe0 = 0, pe1 = 0;
  if (r < n) {
    pe0 = row_ptr[r];
    pe1 = row_ptr[r + 1];
  }
  pdl_wait();
  const int S = *nparts_dev;
  const int ldy = 2 * N;
  const int64_t stride = (int64_t)(*m_dev) * ldy;
  for (bool first = true; r < n; r += gridDim.x * warps, first = false) {
    const int e0 = first ? pe0 : row_ptr[r], e1 = first ? pe1 : row_ptr[r + 1];
    float* out = act + (int64_t)r * ldact;
    for (int cb = 0; cb < ldact; cb += 64) {
      const int c = cb + 2 * lane;
      const bool active = c < N;
      float2 acc = make_float2(0.f, 0.f);
      for (int eb = e0; eb < e1; eb += 32) {
        const int me = eb + lane;
        int32_t my_col = 0;
        float my_val = 0.f;
        if (me < e1) {
          my_col = __ldg(&cols[me]);
          my_val = __ldg(&vals[me]);
        }
        const int m = min(32, e1 - eb);
        if (S == 1) {  // one split (wide frontiers): 16 neighbour rows in flight
          constexpr int U1 = 16;
          for (int t0 = 0; t0 < m; t0 += U1) {
            float2 ld[U1];
            float val[U1];
#pragma unroll
            for (int u = 0; u < U1; ++u) {
              const int32_t cu = __shfl_sync(0xffffffffu, my_col, (t0 + u) & 31);
              val[u] = __shfl_sync(0xffffffffu, my_val, (t0 + u) & 31);
              ld[u] = (active && t0 + u < m)
                          ? __ldcg(reinterpret_cast<const float2*>(part + (int64_t)cu * ldy + c))
                          : make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < U1; ++u) {
              if (t0 + u < m) {
                acc.x = fmaf(val[u], ld[u].x, acc.x);
                acc.y = fmaf(val[u], ld[u].y, acc.y);
              }
            }
          }
          continue;
        }
        for (int t0 = 0; t0 < m; t0 += U) {
          int32_t col[U];
          float val[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            col[u] = __shfl_sync(0xffffffffu, my_col, (t0 + u) & 31);
            val[u] = __shfl_sync(0xffffffffu, my_val, (t0 + u) & 31);
          }
          float2 x[U];
#pragma unroll
          for (int u = 0; u < U; ++u) x[u] = make_float2(0.f, 0.f);
          for (int s0 = 0; s0 < S; s0 += SU) {
            float2 ld[SU][U];
#pragma unroll
            for (int ss = 0; ss < SU; ++ss)
#pragma unroll
              for (int u = 0; u < U; ++u)
                ld[ss][u] = (active && s0 + ss < S && t0 + u < m)
                                ? __ldcg(reinterpret_cast<const float2*>(
                                      part + (s0 + ss) * stride + (int64_t)col[u] * ldy + c))
                                : make_float2(0.f, 0.f);
#pragma unroll
            for (int ss = 0; ss < SU; ++ss)
#pragma unroll
              for (int u = 0; u < U; ++u) {
                x[u].x += ld[ss][u].x;
                x[u].y += ld[ss][u].y;
              }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (t0 + u < m) {
              acc.x = fmaf(val[u], x[u].x, acc.x);
              acc.y = fmaf(val[u], x[u].y, acc.y);
            }
          }
        }
      }
      if (active) {
        float2 b = make_float2(0.f, 0.f);
        for (int s0 = 0; s0 < S; s0 += 8) {
          float2 p[8];
#pragma unroll
          for (int ss = 0; ss < 8; ++ss)
            p[ss] = s0 + ss < S ? __ldcg(reinterpret_cast<const float2*>(
                                      part + (s0 + ss) * stride + (int64_t)r * ldy + N + c))
                                : make_float2(0.f, 0.f);
#pragma unroll
          for (int ss = 0; ss < 8; ++ss) {
            b.x += p[ss].x;
            b.y += p[ss].y;
          }
        }
        const float zx = acc.x + b.x, zy = acc.y + b.y;
        *reinterpret_cast<float2*>(out + c) = make_float2(zx > 0.f ? zx : 0.f, zy > 0.f ? zy : 0.f);
      } else if (c < ldact) {
        *reinterpret_cast<float2*>(out + c) = make_float2(0.f, 0.f);
      }
    }
  }
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  zero_range(z0, tid, nth);
  zero_range(z1, tid, nth);
  MQ_TL_END(5);
}

// ------------------------------------------------------------ scatter bwd
// dz = dh[r] * (act[r] > 0);  G[r, N:2N] = dz;  G[col_e, 0:N] += val_e dz
// (G zeroed beforehand for rows [0, n_src)).
__global__ void __launch_bounds__(kAggThreads) sage_scatter_bwd_kernel(
    const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ cols,
    const float* __restrict__ vals, const int32_t* __restrict__ n_dst_dev,
    const float* __restrict__ dh, int lddh, const float* __restrict__ act, int ldact, int N,
    float* __restrict__ G) {
  pdl_trigger();
  MQ_TL_BEGIN(7);
  const int lane = threadIdx.x & 31;
  const int warps = kAggThreads / 32;
  const int n = *n_dst_dev;  // the block (prep output) ahead of the wait; dh / act / G after
  int r = blockIdx.x * warps + (threadIdx.x >> 5);
  int pe0 = 0, pe1 = 0;
  int32_t pcol = 0;  // the first row's first 32 triplets, also ahead of the wait
  float pval = 0.f;
  if (r < n) {
    pe0 = row_ptr[r];
    pe1 = row_ptr[r + 1];
    if (pe0 + lane < pe1) {
      pcol = __ldg(&cols[pe0 + lane]);
      pval = __ldg(&vals[pe0 + lane]);
    }
  }
  pdl_wait();
  const int ldg = 2 * N;
  const bool vec2 = (N & 1) == 0 && (lddh & 1) == 0 && (ldact & 1) == 0 &&
                    (((uintptr_t)dh | (uintptr_t)act | (uintptr_t)G) & 7) == 0;
  for (bool first = true; r < n; r += gridDim.x * warps, first = false) {
    const int e0 = first ? pe0 : row_ptr[r], e1 = first ? pe1 : row_ptr[r + 1];
    if (vec2) {
      const int n2 = N / 2;
      for (int cb = 0; cb < n2; cb += 32) {
        const int c = cb + lane;
        const bool active = c < n2;
        float2 dz = make_float2(0.f, 0.f);
        if (active) {
          const float2 g = *reinterpret_cast<const float2*>(dh + (int64_t)r * lddh + 2 * c);
          const float2 a = *reinterpret_cast<const float2*>(act + (int64_t)r * ldact + 2 * c);
          dz = make_float2(a.x > 0.f ? g.x : 0.f, a.y > 0.f ? g.y : 0.f);
          *reinterpret_cast<float2*>(G + (int64_t)r * ldg + N + 2 * c) = dz;
        }
        for (int eb = e0; eb < e1; eb += 32) {
          const int me = eb + lane;
          int32_t my_col = 0;
          float my_val = 0.f;
          if (first && eb == e0) {
            my_col = pcol;
            my_val = pval;
          } else if (me < e1) {
            my_col = __ldg(&cols[me]);
            my_val = __ldg(&vals[me]);
          }
          const int m = min(32, e1 - eb);
          for (int t = 0; t < m; ++t) {
            const int32_t col = __shfl_sync(0xffffffffu, my_col, t);
            const float val = __shfl_sync(0xffffffffu, my_val, t);
            if (active)
              atomicAdd(reinterpret_cast<float2*>(G + (int64_t)col * ldg + 2 * c),
                        make_float2(val * dz.x, val * dz.y));
          }
        }
      }
    } else {
      for (int c = lane; c < N; c += 32) {
        const float g = dh[(int64_t)r * lddh + c];
        const float dz = act[(int64_t)r * ldact + c] > 0.f ? g : 0.f;
        G[(int64_t)r * ldg + N + c] = dz;
        for (int e = e0; e < e1; ++e)
          atomicAdd(G + (int64_t)__ldg(&cols[e]) * ldg + c, __ldg(&vals[e]) * dz);
      }
    }
  }
  MQ_TL_END(7);
}

// ------------------------------------------------------------ head
struct HeadArgs {
  const int32_t* row_ptr;
  const int32_t* cols;
  const float* vals;
  const int32_t* n_dst_dev;
  const float* h;
  int ldh;
  int d;
  const float* W;
  int C;
  int Cp;  // smem row stride of W (odd: conflict-free column walks)
  const int32_t* labels;
  float* dW;
  float* dh;
  int lddh;
  float* part;
  int32_t* done;
  double* loss_acc;
  const uint32_t* key;
  int world;
  double* ring;
  int ring_len;
  int32_t* nonfinite;
  int R;
};

#ifdef MQ_TC_TRACE
__device__ unsigned long long g_head_trace[16];
__device__ unsigned long long g_head_cta[256][8];  // every CTA's phase times
__device__ __forceinline__ void htrace(int i) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x == 0) g_head_trace[i] = t;
    if (blockIdx.x < 256 && i < 8) g_head_cta[blockIdx.x][i] = t;
  }
}
#else
__device__ __forceinline__ void htrace(int) {}
#endif

// Two CTA shapes, both 512 threads: 4 target rows x 4 warps (256 CTAs at a
// batch of 1024, two per SM) when two CTAs' shared memory fits on an SM,
// else 8 rows x 2 warps (one wave of 128 CTAs; papers' 172 classes need
// ~120 KB per CTA).  The row phases (aggregation, CE) use the first R
// warps, the dense phases (logits, dt, dW partial) and the dt scatter all of
// them.  Measured on the Reddit step: 8 x 2 50.2 us/step, 4 x 4 49.3,
// 8 x 4 52.2, 4 x 2 55.1 (an earlier build).
#if defined(MQ_HEAD_LATE_TRIGGER)
#error "MQ_HEAD_LATE_TRIGGER with the multi-warp head faulted intermittently (DESIGN.md 7b): unsupported"
#endif
constexpr int kHeadKq = 8;  // k slices of the logits product
constexpr int kHeadCq = 4;  // class slices of the dt product

__host__ __device__ inline int head_red_floats(int R, int d, int C) {
  const int a = kHeadKq * R * C, b = kHeadCq * R * 2 * d;
  return ((a > b ? a : b) + 3) & ~3;
}
constexpr int kHeadMaxEdges = MQ_MAX_FANOUT;  // a seeds-block row has <= fanout triplets

template <int R, int WPR>
__global__ void __launch_bounds__(32 * WPR * R, 2) sage_head_kernel(HeadArgs a) {
  static_assert(R % 4 == 0, "the dt product reads dlT as float4 per class");
  constexpr int kHeadWarps = WPR * R;
  constexpr int kHeadThreads = 32 * kHeadWarps;
// The scatter that follows launches at the head's trigger.  With 8-warp CTAs
// a trigger after the dW partials was faster (60.2 -> 58.8 us/step); with the
// 16-warp head the entry trigger is (58.1 vs 59.3 us/step), and the late
// trigger combined with 16 warps faulted / hung at products-shape epoch
// boundaries (unresolved), so the entry trigger is the default.
// -DMQ_HEAD_LATE_TRIGGER moves it after the dW partials.
#ifndef MQ_HEAD_LATE_TRIGGER
  pdl_trigger();
#endif
  MQ_TL_BEGIN(6);
  htrace(0);
  extern __shared__ __align__(16) float smem[];
  const int d = a.d, d2 = 2 * a.d, d2p = (d2 + 3) & ~3, C = a.C, Cp = a.Cp;
  float* Ws = smem;                 // [d2p][Cp]  (rows >= d2 zero)
  float* both = Ws + d2p * Cp;      // [R][d2p]   = [agg | h_dst | 0 pad]
  float* dl = both + R * d2p;       // [R][C]     logits, then dlogits
  float* dlT = dl + R * C;          // [C][R]     dlogits, class-major (dt operand)
  float* red = dlT + R * C;         // slice sums of the logits / dt products
  float* dts = red + head_red_floats(R, d, C);  // [R][d2p] dt = dl W^T
  __shared__ int32_t s_col[R][kHeadMaxEdges];
  __shared__ float s_val[R][kHeadMaxEdges];
  __shared__ int s_ne[R];
  __shared__ double s_loss[R];
  __shared__ int s_bad;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;  // warp <-> row (warp < R)
  const int n = *a.n_dst_dev;
  const bool row_warp = warp < R;
  const int r = blockIdx.x * R + (row_warp ? warp : 0);
  const bool live = row_warp && r < n;
  if (tid == 0) s_bad = 0;
  // this row's edges and label first: their latency overlaps the W copy
  int e0 = 0, ne = 0, lab = -1;
  if (live) {
    e0 = a.row_ptr[r];
    ne = a.row_ptr[r + 1] - e0;
    if (lane == 0) lab = a.labels[r];
    if (ne > kHeadMaxEdges) {  // not a sampled block (rows carry <= fanout triplets)
      if (lane == 0) atomicOr(a.nonfinite, 4);
      ne = kHeadMaxEdges;
    }
  }
  if (row_warp && lane < ne) {
    s_col[warp][lane] = __ldg(&a.cols[e0 + lane]);
    s_val[warp][lane] = __ldg(&a.vals[e0 + lane]);
  }
  if (row_warp && lane == 0) s_ne[warp] = ne;
  pdl_wait();  // W, h and dh come from the preceding kernels
  const bool w_async = Cp == C && ((uintptr_t)a.W & 15) == 0 && ((d2 * C) & 3) == 0;
  if (w_async) {  // same layout: 16-byte cp.async, landing while phase 1 aggregates
    const float4* src = reinterpret_cast<const float4*>(a.W);
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(Ws));
    for (int i = tid; i < d2 * C / 4; i += kHeadThreads)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 16u * (uint32_t)i),
                   "l"(src + i)
                   : "memory");
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    for (int i = d2 * C + tid; i < d2p * Cp; i += kHeadThreads) Ws[i] = 0.f;
  } else {
    for (int i = tid; i < d2p * C; i += kHeadThreads) {
      const int k = i / C, c = i % C;
      Ws[k * Cp + c] = k < d2 ? __ldg(a.W + i) : 0.f;
    }
  }


  htrace(1);
  // 1. both[row] = [agg | h_dst]: agg bit-exact (sequential triplet order,
  //    nn.py:79-89); the row's gathers issued together
  {
    float* brow = both + warp * d2p;
    if (!row_warp) {
    } else if (!live) {
      for (int c = lane; c < d2p; c += 32) brow[c] = 0.f;
    } else {
      __syncwarp();
      const float* self = a.h + (int64_t)r * a.ldh;
      const bool vec2 = (d & 1) == 0 && (a.ldh & 1) == 0 && ((uintptr_t)a.h & 7) == 0;
      if (vec2) {
        for (int cb = 0; cb < d; cb += 64) {
          const int c = cb + 2 * lane;
          float2 acc = make_float2(0.f, 0.f);
          for (int e0b = 0; e0b < ne; e0b += 8) {
            float2 x[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
              x[u] = (c < d && e0b + u < ne)
                         ? __ldg(reinterpret_cast<const float2*>(
                               a.h + (int64_t)s_col[warp][e0b + u] * a.ldh + c))
                         : make_float2(0.f, 0.f);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              if (e0b + u < ne) {
                const float v = s_val[warp][e0b + u];
                acc.x = __fadd_rn(acc.x, __fmul_rn(v, x[u].x));
                acc.y = __fadd_rn(acc.y, __fmul_rn(v, x[u].y));
              }
            }
          }
          if (c < d) {
            const float2 hv = __ldg(reinterpret_cast<const float2*>(self + c));
            brow[c] = acc.x;
            brow[c + 1] = acc.y;
            brow[d + c] = hv.x;
            brow[d + c + 1] = hv.y;
          }
        }
      } else {
        for (int cb = 0; cb < d; cb += 32) {
          const int c = cb + lane;
          float acc = 0.f;
          for (int e = 0; e < ne; ++e)
            if (c < d)
              acc = __fadd_rn(acc, __fmul_rn(s_val[warp][e],
                                             __ldg(a.h + (int64_t)s_col[warp][e] * a.ldh + c)));
          if (c < d) {
            brow[c] = acc;
            brow[d + c] = __ldg(self + c);
          }
        }
      }
      for (int c = d2 + lane; c < d2p; c += 32) brow[c] = 0.f;
    }
  }
  if (w_async) asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();

  htrace(2);
  // 2. logits = both W, register-blocked over the CTA's R rows: thread
  //    (class c, k slice kq) reads each W element once and the R rows' k slice
  //    as broadcasts; the kHeadKq slice sums are combined in slice order.
  {
    const int kr = ((d2p / 4 + kHeadKq - 1) / kHeadKq) * 4;
    for (int item = tid; item < C * kHeadKq; item += kHeadThreads) {
      const int c = item % C, kq = item / C;
      const int k0 = kq * kr, k1 = min(d2p, k0 + kr);
      float acc[R];
#pragma unroll
      for (int i = 0; i < R; ++i) acc[i] = 0.f;
      for (int k = k0; k < k1; k += 4) {
        const float w0 = Ws[(k + 0) * Cp + c], w1 = Ws[(k + 1) * Cp + c];
        const float w2 = Ws[(k + 2) * Cp + c], w3 = Ws[(k + 3) * Cp + c];
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const float4 x = *reinterpret_cast<const float4*>(both + i * d2p + k);
          acc[i] = fmaf(x.w, w3, fmaf(x.z, w2, fmaf(x.y, w1, fmaf(x.x, w0, acc[i]))));
        }
      }
#pragma unroll
      for (int i = 0; i < R; ++i) red[(kq * R + i) * C + c] = acc[i];
    }
    __syncthreads();
    for (int item = tid; item < R * C; item += kHeadThreads) {
      float v = 0.f;
#pragma unroll
      for (int kq = 0; kq < kHeadKq; ++kq) v += red[kq * R * C + item];
      dl[item] = v;
    }
  }
  __syncthreads();

  htrace(3);
  // 3. summed softmax-CE (nn.py:141-156), dl <- softmax - onehot (row-major
  //    for the dW partial, class-major in dlT for dt)
  if (row_warp) {
    float* x = dl + warp * C;
    double wloss = 0.0;
    int bad = 0;
    if (!live) {
      for (int c = lane; c < C; c += 32) {
        x[c] = 0.f;
        dlT[c * R + warp] = 0.f;
      }
    } else {
      lab = __shfl_sync(0xffffffffu, lab, 0);
      float m = -INFINITY;
      for (int c = lane; c < C; c += 32) m = fmaxf(m, x[c]);
#pragma unroll
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      float s = 0.f, shl = 0.f;
      for (int c = lane; c < C; c += 32) {
        const float sh = x[c] - m;
        const float e = expf(sh);
        if (c == lab) shl = sh;
        s += e;
        x[c] = e;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      const float logd = logf(s);
      for (int c = lane; c < C; c += 32) {
        float p = x[c] / s;
        if (c == lab) {
          p -= 1.f;
          wloss += -(double)(shl - logd);
        }
        x[c] = p;
        dlT[c * R + warp] = p;
        bad |= !isfinite(p);
      }
    }
    const unsigned any_loss = __ballot_sync(0xffffffffu, wloss != 0.0);
    if (any_loss) wloss = __shfl_sync(0xffffffffu, wloss, __ffs(any_loss) - 1);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      s_loss[warp] = wloss;
      if (bad) s_bad = 1;
    }
  }
  __syncthreads();
  // the batch loss and this CTA's completion count, right after the CE: no
  // global write of the thread is pending yet, so its fence is cheap (at the
  // kernel's end it waited on the dt atomics and dW stores: ~1 us per CTA).
  // The last CTA to get here commits the loss to the epoch's loss ring.
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < R; ++w) t += s_loss[w];
    if (t != 0.0) atomicAdd(a.loss_acc, t);
    if (s_bad) atomicOr(a.nonfinite, 1);
    if (a.ring != nullptr) {
      __threadfence();
      if (atomicAdd(a.done, 1) == (int)gridDim.x - 1) {
        __threadfence();
        const int k = (int)((a.key[2] / (uint32_t)a.world) % (uint32_t)a.ring_len);
        volatile double* la = a.loss_acc;
        a.ring[k] = *la;
        *la = 0.0;
        *a.done = 0;
      }
    }
  }

  htrace(4);
  // 4. dt = dl W^T (register-blocked like the logits: thread (k, class slice))
  //    into dts, then dh += dt: the self half to the dst row, the top half
  //    scattered over the row's edges (dh zeroed for rows [0, n_src)
  //    beforehand) by both warps of each row.
  if (a.dh != nullptr) {
    const int cr = (C + kHeadCq - 1) / kHeadCq;
    for (int item = tid; item < d2 * kHeadCq; item += kHeadThreads) {
      const int k = item % d2, cq = item / d2;
      const int c0 = cq * cr, c1 = min(C, c0 + cr);
      float acc[R];
#pragma unroll
      for (int i = 0; i < R; ++i) acc[i] = 0.f;
      for (int c = c0; c < c1; ++c) {
        const float w = Ws[k * Cp + c];
#pragma unroll
        for (int i4 = 0; i4 < R / 4; ++i4) {
          const float4 p = *reinterpret_cast<const float4*>(dlT + c * R + 4 * i4);
          acc[4 * i4 + 0] = fmaf(p.x, w, acc[4 * i4 + 0]);
          acc[4 * i4 + 1] = fmaf(p.y, w, acc[4 * i4 + 1]);
          acc[4 * i4 + 2] = fmaf(p.z, w, acc[4 * i4 + 2]);
          acc[4 * i4 + 3] = fmaf(p.w, w, acc[4 * i4 + 3]);
        }
      }
#pragma unroll
      for (int i = 0; i < R; ++i) red[(cq * R + i) * d2 + k] = acc[i];
    }
    __syncthreads();
    for (int item = tid; item < R * d2; item += kHeadThreads) {
      float v = 0.f;
#pragma unroll
      for (int cq = 0; cq < kHeadCq; ++cq) v += red[cq * R * d2 + item];
      dts[(item / d2) * d2p + item % d2] = v;
    }
    __syncthreads();
    const int rw = warp % R;  // this warp's row; warps rw and rw + R share it
    const int rr = blockIdx.x * R + rw;
    if (rr < n) {
      const int nrow = s_ne[rw];
      const float* dtr = dts + rw * d2p;
      const int t64 = (warp / R) * 32 + lane, nt = 32 * (kHeadWarps / R);
      const bool v4 = (d & 3) == 0 && (a.lddh & 3) == 0 && ((uintptr_t)a.dh & 15) == 0;
      if (v4) {
        const int d4 = d >> 2;
        for (int i = t64; i < (nrow + 1) * d4; i += nt) {
          const int e = i / d4, j = 4 * (i % d4);
          if (e == nrow) {
            atomicAdd(reinterpret_cast<float4*>(a.dh + (int64_t)rr * a.lddh + j),
                      *reinterpret_cast<const float4*>(dtr + d + j));
          } else {
            const float v = s_val[rw][e];
            const float4 t = *reinterpret_cast<const float4*>(dtr + j);
            atomicAdd(reinterpret_cast<float4*>(a.dh + (int64_t)s_col[rw][e] * a.lddh + j),
                      make_float4(v * t.x, v * t.y, v * t.z, v * t.w));
          }
        }
      } else {
        for (int i = t64; i < (nrow + 1) * d; i += nt) {
          const int e = i / d, j = i % d;
          if (e == nrow) atomicAdd(a.dh + (int64_t)rr * a.lddh + j, dtr[d + j]);
          else atomicAdd(a.dh + (int64_t)s_col[rw][e] * a.lddh + j, s_val[rw][e] * dtr[j]);
        }
      }
    }
  }
  __syncthreads();

  htrace(5);
  // 5. this CTA's dW partial = both^T dl: thread (k octet, class), 8 k per item
  {
    float* part = a.part + (int64_t)blockIdx.x * d2 * C;
    const int n8 = (d2p + 7) / 8;
    for (int item = tid; item < n8 * C; item += kHeadThreads) {
      const int k0 = 8 * (item / C), c = item % C;
      float acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.f;
#pragma unroll 4
      for (int i = 0; i < R; ++i) {
        const float v = dl[i * C + c];
        const float4 b0 = *reinterpret_cast<const float4*>(both + i * d2p + k0);
        const float4 b1 = k0 + 4 < d2p ? *reinterpret_cast<const float4*>(both + i * d2p + k0 + 4)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
        acc[0] = fmaf(b0.x, v, acc[0]);
        acc[1] = fmaf(b0.y, v, acc[1]);
        acc[2] = fmaf(b0.z, v, acc[2]);
        acc[3] = fmaf(b0.w, v, acc[3]);
        acc[4] = fmaf(b1.x, v, acc[4]);
        acc[5] = fmaf(b1.y, v, acc[5]);
        acc[6] = fmaf(b1.z, v, acc[6]);
        acc[7] = fmaf(b1.w, v, acc[7]);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (k0 + q < d2) part[(k0 + q) * C + c] = acc[q];
    }
  }

  htrace(6);
#ifdef MQ_HEAD_LATE_TRIGGER
  pdl_trigger();
#endif
  // 6. dW stays as per-CTA partials: the optimizer reduces them in fixed CTA
  //    order (mq_grad_src), so no grid-wide barrier is needed here.
  htrace(7);
  MQ_TL_END(6);
}

// dW = fixed-order sum of the head's per-CTA partials (materialising API)
__global__ void head_dw_reduce_kernel(const float* __restrict__ part, int nparts, int total,
                                      float* __restrict__ dW) {
  MQ_PDL_ENTRY();
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < total; o += gridDim.x * blockDim.x)
    dW[o] = fixed_order_sum(part + o, total, nparts);
}

inline int64_t head_smem_bytes(int R, int d, int C) {
  const int Cp = C | 1, d2p = (2 * d + 3) & ~3;
  // W, both, dl, dlT, slice sums, dt (+ the static edge stash)
  return (int64_t)(d2p * Cp + R * d2p + 2 * R * C + head_red_floats(R, d, C) + R * d2p) *
         (int64_t)sizeof(float);
}

// target rows per CTA: 4 while two CTAs (+ their static stash and the
// per-CTA reservation) fit in an SM's 228 KB, else 8
inline int head_rows(int d, int C) {
  return 2 * (head_smem_bytes(4, d, C) + 4096) <= 228 * 1024 ? 4 : 8;
}

}  // namespace mq

using namespace mq;

extern "C" {

int64_t mq_sage_fused_scratch_bytes(int32_t m_max, int32_t d_in, int32_t d_out) {
  const int64_t K4 = pitch_of(d_in);
  int64_t a = splitk_part_floats(m_max, 2 * d_out);  // transform
  int64_t b = splitk_part_floats(K4, 2 * d_out);     // dW
  int64_t c = splitk_part_floats(m_max, d_in);       // dh
  int64_t mx = a > b ? a : b;
  mx = mx > c ? mx : c;
  const int64_t t = tc_scratch_floats(m_max, d_in, d_out);
  mx = mx > t ? mx : t;
  return mx * (int64_t)sizeof(float);
}

int mq_sage_y_deferred(int32_t d_out) {
  return (tc_backend() == 1 && tc_supported(2 * d_out) && (d_out % 2) == 0) ? 1 : 0;
}

int64_t mq_sage_y_parts_bytes(int32_t m_max, int32_t d_out) {
  return tc_y_part_floats(m_max, d_out) * (int64_t)sizeof(float);
}

int mq_sage_transform(const float* h, int32_t ldh, const int32_t* m_dev, int32_t m_max,
                      int32_t d_in, const float* W, int32_t d_out, float* y, void* scratch,
                      float* y_parts, int32_t* y_nparts_dev, void* stream) {
  MQ_CHECK_ARG(h && m_dev && W && scratch && (y || y_parts), "mq_sage_transform: null pointer");
  MQ_CHECK_ARG((y_parts == nullptr) == (y_nparts_dev == nullptr),
               "mq_sage_transform: y_parts and y_nparts_dev go together");
  MQ_CHECK_ARG(!y_parts || mq_sage_y_deferred(d_out),
               "mq_sage_transform: deferred partials need the tcgen05 backend and even d_out");
  MQ_CHECK_ARG(d_in >= 1 && d_out >= 1 && ldh >= d_in && ldh % 4 == 0 && (uintptr_t)h % 16 == 0,
               "mq_sage_transform: h needs a 16-byte-aligned pitch (multiple of 4) >= d_in");
  if (m_max <= 0) return MQ_OK;
  cudaStream_t s = as_stream(stream);
  Dims dims{m_dev, 0, nullptr, d_in, 2 * d_out};
  float* part = reinterpret_cast<float*>(scratch);
  if (y_parts != nullptr)  // deferred: the aggregation sums the partial tiles
    return tc_transform(h, ldh, m_dev, m_max, d_in, W, d_out, nullptr, y_parts, y_nparts_dev, s);
  if (tc_backend() == 1 && tc_supported(2 * d_out))
    return tc_transform(h, ldh, m_dev, m_max, d_in, W, d_out, y, part, nullptr, s);
  EpiStore epi{y, 2 * d_out};
  if (d_out % 4 == 0 && (uintptr_t)W % 16 == 0)
    return run_gemm(ALoadRow{h, ldh}, BLoadWSplitVec{W, d_in, d_out}, epi, dims, m_max, d_in,
                    kMaxSplits, part, s, K_SAGE_TRANSFORM, K_SAGE_TRANSFORM_REDUCE);
  return run_gemm(ALoadRow{h, ldh}, BLoadWSplit{W, d_in, d_out}, epi, dims, m_max, d_in, kMaxSplits,
                  part, s, K_SAGE_TRANSFORM, K_SAGE_TRANSFORM_REDUCE);
}

int mq_sage_aggregate(const int32_t* row_ptr, const int32_t* cols, const float* vals,
                      const int32_t* n_dst_dev, int32_t n_dst_max, const float* y, int32_t d_out,
                      const int32_t* y_nparts_dev, const int32_t* y_rows_dev, float* act,
                      int32_t ldact, float* zero0, const int32_t* zero0_rows_dev,
                      int32_t zero0_row_floats, float* zero1, const int32_t* zero1_rows_dev,
                      int32_t zero1_row_floats, void* stream) {
  MQ_CHECK_ARG(row_ptr && cols && vals && n_dst_dev && y && act, "mq_sage_aggregate: null pointer");
  MQ_CHECK_ARG(d_out >= 1 && ldact >= d_out, "mq_sage_aggregate: bad dims");
  MQ_CHECK_ARG((!zero0 || zero0_rows_dev) && (!zero1 || zero1_rows_dev),
               "mq_sage_aggregate: zero range without a row count");
  cudaStream_t s = as_stream(stream);
  const int warps = kAggThreads / 32;
  int blocks = ceil_div(n_dst_max < 1 ? 1 : n_dst_max, warps);
  // one wave: the row bound is far above the live rows (Reddit: 11,264 vs
  // ~2,000), and surplus blocks only queue behind the resident ones
  {
    static const bool one_wave = getenv("MQ_AGG_ONE_WAVE") == nullptr || atoi(getenv("MQ_AGG_ONE_WAVE"));
    static const int cap_parts = kNumSMs * resident_blocks(sage_aggregate_parts_kernel, kAggThreads);
    static const int cap_plain = kNumSMs * resident_blocks(sage_aggregate_kernel, kAggThreads);
    const int cap = one_wave ? (y_nparts_dev ? cap_parts : cap_plain) : kNumSMs * 8;
    if (blocks > cap) blocks = cap;
  }
  MQ_CHECK_ARG(!y_nparts_dev || (y_rows_dev && d_out % 2 == 0 && ldact % 2 == 0 &&
                                  ((uintptr_t)y & 7) == 0 && ((uintptr_t)act & 7) == 0),
               "mq_sage_aggregate: partial input needs y_rows_dev and even, aligned widths");
  {
    ProfScope ps(K_SAGE_AGG, s);
    if (y_nparts_dev)
      MQ_CUDA(launch_k(sage_aggregate_parts_kernel, dim3(blocks), dim3(kAggThreads), 0, s, 
          row_ptr, cols, vals, n_dst_dev, y, y_nparts_dev, y_rows_dev, d_out, act, ldact,
          ZeroRange{zero0, zero0_rows_dev, zero0_row_floats},
          ZeroRange{zero1, zero1_rows_dev, zero1_row_floats}));
    else
      MQ_CUDA(launch_k(sage_aggregate_kernel, dim3(blocks), dim3(kAggThreads), 0, s, 
          row_ptr, cols, vals, n_dst_dev, y, d_out, act, ldact,
          ZeroRange{zero0, zero0_rows_dev, zero0_row_floats},
          ZeroRange{zero1, zero1_rows_dev, zero1_row_floats}));
  }
  MQ_LAUNCH_CHECK("sage_aggregate");
  return MQ_OK;
}

int mq_sage_scatter_bwd(const int32_t* row_ptr, const int32_t* cols, const float* vals,
                        const int32_t* n_dst_dev, int32_t n_dst_max, const float* dh, int32_t lddh,
                        const float* act, int32_t ldact, int32_t d_out, float* g, void* stream) {
  MQ_CHECK_ARG(row_ptr && cols && vals && n_dst_dev && dh && act && g,
               "mq_sage_scatter_bwd: null pointer");
  MQ_CHECK_ARG(d_out >= 1 && lddh >= d_out && ldact >= d_out, "mq_sage_scatter_bwd: bad dims");
  if (n_dst_max <= 0) return MQ_OK;
  cudaStream_t s = as_stream(stream);
  const int warps = kAggThreads / 32;
  int blocks = ceil_div(n_dst_max, warps);
  {
    static const bool one_wave = getenv("MQ_AGG_ONE_WAVE") == nullptr || atoi(getenv("MQ_AGG_ONE_WAVE"));
    static const int cap = one_wave ? kNumSMs * resident_blocks(sage_scatter_bwd_kernel, kAggThreads)
                                    : kNumSMs * 8;
    if (blocks > cap) blocks = cap;
  }
  {
    ProfScope ps(K_SAGE_SCATTER, s);
    MQ_CUDA(launch_k(sage_scatter_bwd_kernel, dim3(blocks), dim3(kAggThreads), 0, s, row_ptr, cols, vals, n_dst_dev, dh, lddh,
                                                           act, ldact, d_out, g));
  }
  MQ_LAUNCH_CHECK("sage_scatter_bwd");
  return MQ_OK;
}

int mq_sage_dw_deferred(int32_t d_out) {
  return (tc_backend() == 1 && tc_supported(2 * d_out)) ? 1 : 0;
}

int64_t mq_sage_af_parts_bytes(int32_t m_max, int32_t d_out) {
  return tc_af_part_floats(m_max, d_out) * (int64_t)sizeof(float);
}

int64_t mq_sage_af_dw_parts_bytes(int32_t d_in, int32_t d_out) {
  return tc_af_dw_part_floats(d_in, d_out) * (int64_t)sizeof(float);
}

int mq_sage_linear_af(const float* agg, int32_t ldagg, const float* h, int32_t ldh,
                      const int32_t* m_dev, int32_t m_max, int32_t d_in, const float* W,
                      int32_t d_out, float* act, int32_t ldact, float* part, void* stream) {
  MQ_CHECK_ARG(agg && h && m_dev && W && act && part, "mq_sage_linear_af: null pointer");
  MQ_CHECK_ARG(d_in >= 4 && d_in % 4 == 0 && d_out >= 1 && d_out <= 256 && ldagg >= d_in &&
                   ldh >= d_in && ldagg % 4 == 0 && ldh % 4 == 0 && ldact >= d_out &&
                   ((uintptr_t)agg | (uintptr_t)h) % 16 == 0,
               "mq_sage_linear_af: bad dims / alignment (d_in % 4 == 0, d_out <= 256)");
  if (m_max <= 0) return MQ_OK;
  return tc_linear_af(agg, ldagg, h, ldh, m_dev, m_max, d_in, W, d_out, act, ldact, part,
                      as_stream(stream));
}

int mq_sage_linear_af_bwd(const float* agg, int32_t ldagg, const float* h, int32_t ldh,
                          const int32_t* rows_dev, int32_t rows_max, int32_t d_in, const float* dh,
                          int32_t lddh, const float* act, int32_t ldact, int32_t d_out,
                          float* dw_parts, int32_t* dw_nparts_dev, void* stream) {
  MQ_CHECK_ARG(agg && h && rows_dev && dh && act && dw_parts && dw_nparts_dev,
               "mq_sage_linear_af_bwd: null pointer");
  MQ_CHECK_ARG(d_in >= 4 && d_in % 4 == 0 && d_out >= 1 && d_out <= 256 && ldagg % 4 == 0 &&
                   ldh % 4 == 0 && lddh >= d_out && ldact >= d_out &&
                   ((uintptr_t)agg | (uintptr_t)h) % 16 == 0,
               "mq_sage_linear_af_bwd: bad dims / alignment");
  return tc_linear_af_bwd(agg, ldagg, h, ldh, rows_dev, rows_max, d_in, dh, lddh, act, ldact,
                          d_out, dw_parts, dw_nparts_dev, as_stream(stream));
}

int64_t mq_sage_dw_parts_bytes(int32_t d_in, int32_t d_out) {
  return tc_dw_part_floats(d_in, d_out) * (int64_t)sizeof(float);
}

int mq_sage_transform_bwd(const float* h, int32_t ldh, const int32_t* m_dev, int32_t m_max,
                          int32_t d_in, const float* W, int32_t d_out, const float* g, float* dW,
                          float* dh, int32_t lddh, void* scratch, float* dw_parts,
                          int32_t* dw_nparts_dev, void* stream) {
  MQ_CHECK_ARG(h && m_dev && W && g && scratch, "mq_sage_transform_bwd: null pointer");
  MQ_CHECK_ARG((dw_parts == nullptr) == (dw_nparts_dev == nullptr),
               "mq_sage_transform_bwd: dw_parts and dw_nparts_dev go together");
  MQ_CHECK_ARG(dW || (dw_parts && mq_sage_dw_deferred(d_out)),
               "mq_sage_transform_bwd: dW is required unless the weight gradient is deferred");
  MQ_CHECK_ARG(d_in >= 1 && d_out >= 1 && ldh >= d_in && ldh % 4 == 0 && (uintptr_t)h % 16 == 0 &&
                   (!dh || lddh >= d_in),
               "mq_sage_transform_bwd: bad dims / alignment");
  cudaStream_t s = as_stream(stream);
  float* part = reinterpret_cast<float*>(scratch);
  if (tc_backend() == 1 && tc_supported(2 * d_out)) {
    // deferred: the partial tiles stay in dw_parts for the optimizer to reduce
    int rc = dw_parts ? tc_weight_grad(h, ldh, m_dev, m_max, d_in, d_out, g, nullptr, dw_parts,
                                       dw_nparts_dev, s)
                      : tc_weight_grad(h, ldh, m_dev, m_max, d_in, d_out, g, dW, part, nullptr, s);
    if (rc) return rc;
  } else {
    Dims dims{nullptr, pitch_of(d_in), m_dev, 0, 2 * d_out};
    int rc = run_gemm(ALoadT{h, ldh}, BLoadRow{g, 2 * d_out, 2 * d_out}, EpiDWSplit{dW, d_in, d_out},
                      dims, pitch_of(d_in), m_max, kMaxSplits, part, s, K_SAGE_DW,
                      K_SAGE_DW_REDUCE);
    if (rc) return rc;
  }
  if (dh != nullptr && m_max > 0 && tc_backend() == 1 && d_in <= 256 && (2 * d_out) % 4 == 0 &&
      ((uintptr_t)g & 15) == 0) {
    int rc = tc_dx(g, m_dev, m_max, d_in, d_out, W, dh, lddh, part, s);
    if (rc) return rc;
  } else if (dh != nullptr && m_max > 0) {
    Dims dims{m_dev, 0, nullptr, 2 * d_out, d_in};
    int rc = run_gemm(ALoadRow{g, 2 * d_out}, BLoadWSplitT{W, d_in, d_out}, EpiStore{dh, lddh}, dims,
                      m_max, 2 * d_out, (2 * d_out + GBK - 1) / GBK, part, s, K_SAGE_DH,
                      K_SAGE_DH_REDUCE);
    if (rc) return rc;
  }
  return MQ_OK;
}

int64_t mq_sage_head_scratch_bytes(int32_t n_dst_max, int32_t d, int32_t n_classes) {
  const int R = head_rows(d, n_classes);
  const int64_t G = (n_dst_max + R - 1) / R;
  return 256 + G * 2 * d * (int64_t)n_classes * (int64_t)sizeof(float);
}

int mq_sage_head(const int32_t* row_ptr, const int32_t* cols, const float* vals,
                 const int32_t* n_dst_dev, int32_t n_dst_max, const float* h, int32_t ldh, int32_t d,
                 const float* W, int32_t n_classes, const int32_t* labels, float* dW, float* dh,
                 int32_t lddh, double* loss_acc, const uint32_t* key_dev, int32_t world,
                 double* loss_ring, int32_t ring_len, int32_t* nonfinite, void* scratch,
                 void* stream) {
  MQ_CHECK_ARG(row_ptr && cols && vals && n_dst_dev && h && W && labels && loss_acc && nonfinite &&
                   scratch,
               "mq_sage_head: null pointer");
  MQ_CHECK_ARG(d >= 1 && n_classes >= 1 && ldh >= d && (!dh || lddh >= d),
               "mq_sage_head: bad dims");
  MQ_CHECK_ARG(!loss_ring || (key_dev && ring_len > 0 && world >= 1), "mq_sage_head: bad ring");
  if (n_dst_max <= 0) return MQ_OK;
  const int R = head_rows(d, n_classes);
  const int G = ceil_div(n_dst_max, R);
  const int64_t smem = head_smem_bytes(R, d, n_classes);
  MQ_CHECK_ARG(smem <= 220 * 1024, "mq_sage_head: d=%d, classes=%d need %lld B of shared memory", d,
               n_classes, (long long)smem);
  cudaStream_t s = as_stream(stream);
  auto kern = R == 4 ? sage_head_kernel<4, 4> : sage_head_kernel<8, 2>;
  static thread_local int64_t configured[2] = {0, 0};
  if (smem > configured[R == 8]) {  // (static smem counts against the 48 KB default too)
    MQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured[R == 8] = smem;
  }
  HeadArgs a;
  a.row_ptr = row_ptr;
  a.cols = cols;
  a.vals = vals;
  a.n_dst_dev = n_dst_dev;
  a.h = h;
  a.ldh = ldh;
  a.d = d;
  a.W = W;
  a.C = n_classes;
  a.Cp = n_classes | 1;
  a.labels = labels;
  a.dW = dW;
  a.dh = dh;
  a.lddh = lddh;
  a.done = reinterpret_cast<int32_t*>(scratch);
  a.part = reinterpret_cast<float*>(reinterpret_cast<char*>(scratch) + 256);
  a.loss_acc = loss_acc;
  a.key = key_dev;
  a.world = world;
  a.ring = loss_ring;
  a.ring_len = ring_len;
  a.nonfinite = nonfinite;
  a.R = R;
  {
    ProfScope ps(K_SAGE_HEAD, s);
    MQ_CUDA(launch_k(kern, dim3(G), dim3(512), smem, s, a));
  }
  MQ_LAUNCH_CHECK("sage_head");
  if (dW != nullptr) {
    const int total = 2 * d * n_classes;
    ProfScope ps(K_SAGE_DW_REDUCE, s);
    MQ_CUDA(launch_k(head_dw_reduce_kernel, dim3(ceil_div(total, 256)), dim3(256), 0, s, a.part, G, total, dW));
  }
  MQ_LAUNCH_CHECK("head_dw_reduce");
  return MQ_OK;
}

#ifdef MQ_TC_TRACE
extern "C" int mq_debug_head_trace(unsigned long long* out) {
  MQ_CUDA(cudaMemcpyFromSymbol(out, g_head_trace, sizeof(unsigned long long) * 16));
  return MQ_OK;
}
extern "C" int mq_debug_head_cta(unsigned long long* out) {  // [256][8] phase times
  MQ_CUDA(cudaMemcpyFromSymbol(out, g_head_cta, sizeof(unsigned long long) * 256 * 8));
  return MQ_OK;
}
#endif

int mq_sage_head_grad_seg(int32_t n_dst_max, int32_t d, int32_t n_classes, void* scratch,
                          int64_t offset, mq_grad_seg* out) {
  MQ_CHECK_ARG(scratch && out && n_dst_max >= 1 && d >= 1 && n_classes >= 1,
               "mq_sage_head_grad_seg: bad arguments");
  const int R = head_rows(d, n_classes);
  memset(out, 0, sizeof(*out));
  out->part = reinterpret_cast<const float*>(reinterpret_cast<char*>(scratch) + 256);
  out->nparts = ceil_div(n_dst_max, R);
  out->stride = 2LL * d * n_classes;
  out->offset = offset;
  out->size = 2LL * d * n_classes;
  out->kind = 0;
  return MQ_OK;
}

int mq_sage_dw_grad_seg(float* dw_parts, const int32_t* dw_nparts_dev, int32_t d_in, int32_t d_out,
                        int64_t offset, mq_grad_seg* out) {
  MQ_CHECK_ARG(dw_parts && dw_nparts_dev && out && d_in >= 1 && d_out >= 1,
               "mq_sage_dw_grad_seg: bad arguments");
  memset(out, 0, sizeof(*out));
  out->part = dw_parts;
  out->nparts_dev = dw_nparts_dev;
  out->stride = (int64_t)d_in * 2 * d_out;
  out->offset = offset;
  out->size = 2LL * d_in * d_out;
  out->kind = 1;
  out->d_in = d_in;
  out->d_out = d_out;
  return MQ_OK;
}

}  // extern "C"

MQ_TL_READER(fused)
