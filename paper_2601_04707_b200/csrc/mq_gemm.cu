// Dense SAGE layer transforms: z = [agg | h_dst] W, dW = [agg | h_dst]^T dz,
// dt = dz W^T (mqpipe/nn.py:126-131, 167-170).
//
// fp32 SIMT tiles with FMA accumulation.  The reference trains in fp32 and
// north_star pins these contractions at rel 1e-5, which TF32 tensor-core math
// (10-bit mantissa) cannot meet; the concat is never materialised — the A
// loader reads the agg and self halves from their own buffers.
#include "mq_common.cuh"

namespace mq {

constexpr int BM = 64, BN = 64, BK = 16, kGemmThreads = 256;

struct Dims {
  const int32_t* m_dev;  // if set, M = *m_dev (else m)
  int m;
  const int32_t* k_dev;  // if set, K = *k_dev (else k)
  int k;
  int n;
  __device__ int M() const { return m_dev ? *m_dev : m; }
  __device__ int K() const { return k_dev ? *k_dev : k; }
};

// A(i, k) of z = [agg | h] W: k contiguous
struct ALoadConcat {
  static constexpr bool kKContig = true;
  const float* agg;
  int lda;
  const float* h;
  int ldh;
  int d_in;
  __device__ float operator()(int i, int k) const {
    return k < d_in ? __ldg(&agg[(int64_t)i * lda + k]) : __ldg(&h[(int64_t)i * ldh + (k - d_in)]);
  }
};
// A(o, r) = [agg | h](r, o) for dW (output row o over 2*d_in, reduction r over rows): o contiguous
struct ALoadConcatT {
  static constexpr bool kKContig = false;
  const float* agg;
  int lda;
  const float* h;
  int ldh;
  int d_in;
  __device__ float operator()(int o, int r) const {
    return o < d_in ? __ldg(&agg[(int64_t)r * lda + o]) : __ldg(&h[(int64_t)r * ldh + (o - d_in)]);
  }
};
// plain row-major matrix, element (i, k) at p[i*ld + k]
struct ALoadRow {
  static constexpr bool kKContig = true;
  const float* p;
  int ld;
  __device__ float operator()(int i, int k) const { return __ldg(&p[(int64_t)i * ld + k]); }
};
// B(k, j) = p[k*ld + j]: j contiguous
struct BLoadRow {
  static constexpr bool kKContig = false;
  const float* p;
  int ld;
  __device__ float operator()(int k, int j) const { return __ldg(&p[(int64_t)k * ld + j]); }
};
// B(k, j) = p[j*ld + k] (transposed weight): k contiguous
struct BLoadT {
  static constexpr bool kKContig = true;
  const float* p;
  int ld;
  __device__ float operator()(int k, int j) const { return __ldg(&p[(int64_t)j * ld + k]); }
};

struct EpiLinearFwd {
  float* z;
  int ldz;
  float* relu;
  int ldr;
  __device__ void operator()(int i, int j, float v, int) const {
    if (z) z[(int64_t)i * ldz + j] = v;
    if (relu) relu[(int64_t)i * ldr + j] = v > 0.f ? v : 0.f;
  }
};
struct EpiStore {
  float* c;
  int ldc;
  __device__ void operator()(int i, int j, float v, int) const { c[(int64_t)i * ldc + j] = v; }
};
struct EpiPartial {
  float* part;  // [splits][M][N]
  int M, N;
  __device__ void operator()(int i, int j, float v, int z) const {
    part[((int64_t)z * M + i) * N + j] = v;
  }
};

// C[M, N] = sum_k A(i,k) B(k,j) over the k-range of split blockIdx.z.
template <class AL, class BL, class Epi>
__global__ void __launch_bounds__(kGemmThreads) sgemm_kernel(AL A, BL B, Epi epi, Dims dims,
                                                             int k_chunk) {
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN + 4];
  const int M = dims.M(), N = dims.n, K = dims.K();
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kb = blockIdx.z * k_chunk;
  const int ke = min(K, kb + k_chunk);
  const bool live = m0 < M;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  if (live) {
    for (int k0 = kb; k0 < ke; k0 += BK) {
#pragma unroll
      for (int q = 0; q < (BM * BK) / kGemmThreads; ++q) {
        const int idx = tid + q * kGemmThreads;
        int mi, ki;
        if (AL::kKContig) {
          mi = idx / BK;
          ki = idx % BK;
        } else {
          mi = idx % BM;
          ki = idx / BM;
        }
        const int gm = m0 + mi, gk = k0 + ki;
        As[ki][mi] = (gm < M && gk < ke) ? A(gm, gk) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < (BN * BK) / kGemmThreads; ++q) {
        const int idx = tid + q * kGemmThreads;
        int ni, ki;
        if (BL::kKContig) {
          ni = idx / BK;
          ki = idx % BK;
        } else {
          ni = idx % BN;
          ki = idx / BN;
        }
        const int gn = n0 + ni, gk = k0 + ki;
        Bs[ki][ni] = (gn < N && gk < ke) ? B(gk, gn) : 0.f;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < BK; ++k) {
        const float4 a = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
        const float4 b = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
  }
  if (!live) return;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn < N) epi(gm, gn, acc[i][j], blockIdx.z);
    }
  }
}

// dW[i] = sum over splits, in split order (deterministic)
__global__ void reduce_splits_kernel(const float* __restrict__ part, int splits, int64_t mn,
                                     float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < mn;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += part[(int64_t)z * mn + i];
    out[i] = s;
  }
}

constexpr int kBwdWSplitRows = 256;  // reduction rows per split of the dW GEMM

inline int bwd_w_splits(int m_max) {
  int s = ceil_div(m_max < 1 ? 1 : m_max, kBwdWSplitRows);
  return s < 1 ? 1 : s;
}

}  // namespace mq

using namespace mq;

extern "C" {

int mq_sage_linear_fwd(const float* agg, int32_t ldagg, const float* h, int32_t ldh,
                       const int32_t* m_dev, int32_t m_max, int32_t d_in, const float* W,
                       int32_t d_out, float* z, int32_t ldz, float* relu_out, int32_t ldr,
                       void* stream) {
  MQ_CHECK_ARG(agg && h && m_dev && W && (z || relu_out), "mq_sage_linear_fwd: null pointer");
  MQ_CHECK_ARG(d_in >= 1 && d_out >= 1 && (!z || ldz >= d_out) && (!relu_out || ldr >= d_out),
               "mq_sage_linear_fwd: bad dims");
  if (m_max <= 0) return MQ_OK;
  cudaStream_t s = as_stream(stream);
  Dims dims{m_dev, 0, nullptr, 2 * d_in, d_out};
  dim3 grid(ceil_div(m_max, BM), ceil_div(d_out, BN), 1);
  {
    ProfScope ps(K_LINEAR_FWD, s);
    sgemm_kernel<<<grid, kGemmThreads, 0, s>>>(ALoadConcat{agg, ldagg, h, ldh, d_in},
                                               BLoadRow{W, d_out},
                                               EpiLinearFwd{z, ldz, relu_out, ldr}, dims, 2 * d_in);
  }
  MQ_LAUNCH_CHECK("linear_fwd");
  return MQ_OK;
}

int64_t mq_linear_bwd_w_scratch_bytes(int32_t m_max, int32_t d_in, int32_t d_out) {
  return (int64_t)bwd_w_splits(m_max) * 2 * d_in * d_out * sizeof(float);
}

int mq_sage_linear_bwd(const float* agg, int32_t ldagg, const float* h, int32_t ldh,
                       const int32_t* m_dev, int32_t m_max, int32_t d_in, const float* W,
                       int32_t d_out, const float* dz, int32_t lddz, float* dW, float* dt,
                       int32_t lddt, void* scratch, void* stream) {
  MQ_CHECK_ARG(agg && h && m_dev && W && dz && dW && scratch, "mq_sage_linear_bwd: null pointer");
  MQ_CHECK_ARG(d_in >= 1 && d_out >= 1 && lddz >= d_out && (!dt || lddt >= 2 * d_in),
               "mq_sage_linear_bwd: bad dims");
  cudaStream_t s = as_stream(stream);
  const int mo = 2 * d_in;
  const int splits = bwd_w_splits(m_max);
  float* part = reinterpret_cast<float*>(scratch);
  {
    // dW partials: output (2*d_in x d_out), reduction over the m rows in splits
    Dims dims{nullptr, mo, m_dev, 0, d_out};
    dim3 grid(ceil_div(mo, BM), ceil_div(d_out, BN), splits);
    ProfScope ps(K_LINEAR_BWD_W, s);
    sgemm_kernel<<<grid, kGemmThreads, 0, s>>>(ALoadConcatT{agg, ldagg, h, ldh, d_in},
                                               BLoadRow{dz, lddz}, EpiPartial{part, mo, d_out},
                                               dims, kBwdWSplitRows);
  }
  MQ_LAUNCH_CHECK("linear_bwd_w");
  {
    int64_t mn = (int64_t)mo * d_out;
    int blocks = ceil_div(mn, 256);
    if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
    ProfScope ps(K_LINEAR_BWD_W_REDUCE, s);
    reduce_splits_kernel<<<blocks, 256, 0, s>>>(part, splits, mn, dW);
  }
  MQ_LAUNCH_CHECK("linear_bwd_w_reduce");
  if (dt != nullptr && m_max > 0) {
    Dims dims{m_dev, 0, nullptr, d_out, mo};
    dim3 grid(ceil_div(m_max, BM), ceil_div(mo, BN), 1);
    ProfScope ps(K_LINEAR_BWD_X, s);
    sgemm_kernel<<<grid, kGemmThreads, 0, s>>>(ALoadRow{dz, lddz}, BLoadT{W, d_out},
                                               EpiStore{dt, lddt}, dims, d_out);
  }
  MQ_LAUNCH_CHECK("linear_bwd_x");
  return MQ_OK;
}

}  // extern "C"
