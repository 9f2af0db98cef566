// Persistent split-K fp32 GEMM machinery shared by the SAGE transforms
// (mq_gemm.cu: aggregate-first layer transforms; mq_fused.cu: the fused
// transform-first step).  See mq_gemm.cu for the design notes.
#pragma once

#include "mq_common.cuh"

namespace mq {

constexpr int GBM = 64, GBN = 64, GBK = 16, GTHREADS = 256;
constexpr int kMaxSplits = 16;

struct Dims {
  const int32_t* m_dev;  // if set, M = *m_dev (else m)
  int m;
  const int32_t* k_dev;  // if set, K = *k_dev (else k)
  int k;
  int n;
  __device__ int M() const { return m_dev ? *m_dev : m; }
  __device__ int K() const { return k_dev ? *k_dev : k; }
};

__device__ __forceinline__ float4 ld4_guard(const float* p, int n_valid) {
  // n_valid in [0, 4]: elements beyond are zero
  if (n_valid >= 4 && ((uintptr_t)p & 15) == 0) return __ldg(reinterpret_cast<const float4*>(p));
  float v[4] = {0.f, 0.f, 0.f, 0.f};
  for (int i = 0; i < 4 && i < n_valid; ++i) v[i] = __ldg(p + i);
  return make_float4(v[0], v[1], v[2], v[3]);
}

// ---- operand loaders: load4(i, k) returns A(i, k..k+3) / B(k.., j) as float4
// A(i, k) of z = [agg | h] W over the padded k space (k contiguous)
struct ALoadConcat {
  static constexpr bool kKContig = true;
  const float* agg;
  const float* h;
  int ld;  // common pitch P of agg and h (multiple of 4)
  __device__ float4 load4(int i, int k, int K) const {  // K = 2P
    if (k >= K) return make_float4(0.f, 0.f, 0.f, 0.f);
    const float* p = k < ld ? agg + (int64_t)i * ld + k : h + (int64_t)i * ld + (k - ld);
    return __ldg(reinterpret_cast<const float4*>(p));
  }
};
// A(o, r) = [agg | h](r, o) for dW (o over the padded 2P, r over rows): o contiguous
struct ALoadConcatT {
  static constexpr bool kKContig = false;
  const float* agg;
  const float* h;
  int ld;
  __device__ float4 load4m(int o, int r) const {  // o..o+3 at row r
    const float* p = o < ld ? agg + (int64_t)r * ld + o : h + (int64_t)r * ld + (o - ld);
    return __ldg(reinterpret_cast<const float4*>(p));
  }
};
// row-major A (i, k) = p[i*ld + k], k contiguous, K columns valid
struct ALoadRow {
  static constexpr bool kKContig = true;
  const float* p;
  int ld;
  __device__ float4 load4(int i, int k, int K) const {
    return ld4_guard(p + (int64_t)i * ld + k, K - k);
  }
};
// B(k, j) of z = [agg | h] W: padded k -> W row, j contiguous, N columns
struct BLoadW {
  const float* W;
  int ld;    // pitch P of the concat halves
  int d_in;  // real rows per half
  int N;
  __device__ float4 load4(int k, int j) const {
    int row;
    if (k < ld) {
      if (k >= d_in) return make_float4(0.f, 0.f, 0.f, 0.f);
      row = k;
    } else {
      if (k - ld >= d_in) return make_float4(0.f, 0.f, 0.f, 0.f);
      row = d_in + (k - ld);
    }
    return ld4_guard(W + (int64_t)row * N + j, N - j);
  }
};
// B(r, j) = dz[r*ld + j] for dW: j contiguous
struct BLoadRow {
  const float* p;
  int ld;
  int N;
  __device__ float4 load4(int k, int j) const { return ld4_guard(p + (int64_t)k * ld + j, N - j); }
};
// B(k, j) = W[j*ld + k] (dt = dz W^T: k over d_out, j over 2*d_in)
struct BLoadWT {
  const float* W;
  int ld;  // d_out
  int K;   // d_out
  int N;   // 2*d_in
  __device__ float4 load4(int k, int j) const {
    float v[4];
    for (int t = 0; t < 4; ++t)
      v[t] = (j + t < N && k < K) ? __ldg(W + (int64_t)(j + t) * ld + k) : 0.f;
    return make_float4(v[0], v[1], v[2], v[3]);
  }
};

struct Split {
  int tiles_m, tiles_n, S, k_chunk;
};

__device__ __forceinline__ Split choose_split(int M, int N, int K, int grid, int s_cap) {
  Split s;
  s.tiles_m = (M + GBM - 1) / GBM;
  s.tiles_n = (N + GBN - 1) / GBN;
  const int tiles = max(1, s.tiles_m * s.tiles_n);
  const int kb = max(1, (K + GBK - 1) / GBK);
  int S = (grid + tiles - 1) / tiles;
  S = max(1, min(S, min(s_cap, kb)));
  const int per = (kb + S - 1) / S;  // k blocks per split
  s.k_chunk = per * GBK;
  s.S = (K + s.k_chunk - 1) / s.k_chunk;
  if (s.S < 1) s.S = 1;
  return s;
}

// Persistent split-K tile loop; partial tile sums go to part[s][M_ld][N].
template <class AL, class BL>
__global__ void __launch_bounds__(GTHREADS, 2)
    sgemm_splitk_kernel(AL A, BL B, Dims dims, int s_cap, float* __restrict__ part) {
  __shared__ __align__(16) float As[2][GBK][GBM + 4];
  __shared__ __align__(16) float Bs[2][GBK][GBN + 4];
  const int M = dims.M(), N = dims.n, K = dims.K();
  const Split sp = choose_split(M, N, K, gridDim.x, s_cap);
  const int items = sp.tiles_m * sp.tiles_n * sp.S;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;

  for (int w = blockIdx.x; w < items; w += gridDim.x) {
    const int s = w % sp.S;
    const int t = w / sp.S;
    const int m0 = (t / sp.tiles_n) * GBM, n0 = (t % sp.tiles_n) * GBN;
    const int kb = s * sp.k_chunk, ke = min(K, kb + sp.k_chunk);
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

    // per-thread load slots: one float4 of A and one of B per BK step
    float4 ra, rb;
    auto load_tiles = [&](int k0) {
      if constexpr (AL::kKContig) {
        const int mi = tid >> 2, kq = (tid & 3) * 4;
        const int gm = m0 + mi, gk = k0 + kq;
        ra = (gm < M && gk < ke) ? A.load4(gm, gk, ke) : make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        const int ki = tid >> 4, mq4 = (tid & 15) * 4;
        const int gk = k0 + ki, gm = m0 + mq4;
        ra = (gk < ke && gm < M) ? A.load4m(gm, gk) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      {
        const int ki = tid >> 4, nq = (tid & 15) * 4;
        const int gk = k0 + ki, gn = n0 + nq;
        rb = (gk < ke && gn < N) ? B.load4(gk, gn) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    auto store_tiles = [&](int buf) {
      if constexpr (AL::kKContig) {
        const int mi = tid >> 2, kq = (tid & 3) * 4;
        As[buf][kq + 0][mi] = ra.x;
        As[buf][kq + 1][mi] = ra.y;
        As[buf][kq + 2][mi] = ra.z;
        As[buf][kq + 3][mi] = ra.w;
      } else {
        const int ki = tid >> 4, mq4 = (tid & 15) * 4;
        *reinterpret_cast<float4*>(&As[buf][ki][mq4]) = ra;
      }
      const int ki = tid >> 4, nq = (tid & 15) * 4;
      *reinterpret_cast<float4*>(&Bs[buf][ki][nq]) = rb;
    };

    int buf = 0;
    load_tiles(kb);
    store_tiles(0);
    __syncthreads();
    for (int k0 = kb; k0 < ke; k0 += GBK) {
      const bool more = k0 + GBK < ke;
      if (more) load_tiles(k0 + GBK);
#pragma unroll
      for (int k = 0; k < GBK; ++k) {
        const float4 a = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
        const float4 b = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4]);
        const float av[4] = {a.x, a.y, a.z, a.w};
        const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      if (more) store_tiles(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
    float* out = part + (int64_t)s * M * N;  // partials packed by the live M
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int gm = m0 + ty * 4 + i;
      if (gm >= M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int gn = n0 + tx * 4 + j;
        if (gn < N) out[(int64_t)gm * N + gn] = acc[i][j];
      }
    }
    __syncthreads();
  }
}

// ---- split reduction + epilogues (fixed split order: deterministic)
struct EpiLinearFwd {
  float* z;
  int ldz;
  float* relu;
  int ldr;
  __device__ void operator()(int i, int j, float v) const {
    if (z) z[(int64_t)i * ldz + j] = v;
    if (relu) relu[(int64_t)i * ldr + j] = v > 0.f ? v : 0.f;
  }
};
struct EpiStore {
  float* c;
  int ldc;
  __device__ void operator()(int i, int j, float v) const { c[(int64_t)i * ldc + j] = v; }
};
// padded concat row o -> dW row (skip the pad rows)
struct EpiDW {
  float* dW;
  int ld;  // pitch P
  int d_in;
  int N;
  __device__ void operator()(int o, int j, float v) const {
    int row;
    if (o < ld) {
      if (o >= d_in) return;
      row = o;
    } else {
      if (o - ld >= d_in) return;
      row = d_in + (o - ld);
    }
    dW[(int64_t)row * N + j] = v;
  }
};

// (o, j) of h^T G -> dW row o (W_top grad) or d_in + o (W_bot grad)
struct EpiDWSplit {
  float* dW;
  int d_in;
  int N;
  __device__ void operator()(int o, int j, float v) const {
    if (o >= d_in) return;
    if (j < N)
      dW[(int64_t)o * N + j] = v;
    else
      dW[(int64_t)(d_in + o) * N + (j - N)] = v;
  }
};

template <class Epi>
__global__ void splitk_reduce_kernel(const float* __restrict__ part, Dims dims, int grid_gemm,
                                     int s_cap, Epi epi) {
  const int M = dims.M(), N = dims.n, K = dims.K();
  const Split sp = choose_split(M, N, K, grid_gemm, s_cap);
  const int64_t total = (int64_t)M * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / N), j = (int)(e % N);
    epi(i, j, fixed_order_sum(part + (int64_t)i * N + j, (int64_t)M * N, sp.S));
  }
}

constexpr int kGemmGrid = kNumSMs * 2;

template <class AL, class BL, class Epi>
int run_gemm(const AL& A, const BL& B, const Epi& epi, Dims dims, int m_max, int k_max, int s_cap,
             float* part, cudaStream_t s, int kid_gemm, int kid_red) {
  const int tiles_max = ceil_div(m_max < 1 ? 1 : m_max, GBM) * ceil_div(dims.n, GBN);
  (void)k_max;
  int grid = kGemmGrid;
  if (grid > tiles_max * s_cap) grid = tiles_max * s_cap;
  if (grid < 1) grid = 1;
  {
    ProfScope ps(kid_gemm, s);
    sgemm_splitk_kernel<AL, BL><<<grid, GTHREADS, 0, s>>>(A, B, dims, s_cap, part);
  }
  MQ_LAUNCH_CHECK("sgemm_splitk");
  int64_t mn = (int64_t)(m_max < 1 ? 1 : m_max) * dims.n;
  int rb = ceil_div(mn, 256);
  if (rb > kNumSMs * 4) rb = kNumSMs * 4;
  {
    ProfScope ps(kid_red, s);
    splitk_reduce_kernel<Epi><<<rb, 256, 0, s>>>(part, dims, grid, s_cap, epi);
  }
  MQ_LAUNCH_CHECK("splitk_reduce");
  return MQ_OK;
}

inline int pitch_of(int d) { return (d + 3) / 4 * 4; }

// floats of split-K partials for an (m_max x n) output: S*M <= min(kMaxSplits*M,
// grid*GBM/tiles_n + M) because the device picks S = ceil(grid / tiles).
inline int64_t splitk_part_floats(int64_t m_max, int64_t n) {
  if (m_max < 1) m_max = 1;
  int64_t a = (int64_t)kMaxSplits * m_max;
  int64_t b = (int64_t)kGemmGrid * GBM + m_max;
  return (a < b ? a : b) * n;
}

}  // namespace mq
