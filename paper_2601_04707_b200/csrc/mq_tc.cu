// fp32-accurate GEMMs on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// The two dense contractions of the transform-first SAGE layer (mq_fused.cu):
//   FWD:  Y (M x N)  = X (M x K) . B        X = sampled input rows (K-major),
//                                           B = [W_top | W_bot] (N contiguous)
//   DW:   P (M x N)  = X^T (M x K) . G      M = features, K = sampled rows,
//                                           X and G row-major (MN-major)
// (mqpipe/nn.py:126-131 forward transform and nn.py:168-170 weight gradient.)
//
// Precision: the reference trains in fp32 and north_star pins these
// contractions at rel 1e-5, which one TF32 pass (10-bit mantissa) misses.
// Each operand is split on the fly into x = hi + lo with hi = tf32_rn(x),
// lo = tf32_rn(x - hi), and the tile product is accumulated in fp32 TMEM as
// A_hi B_hi + A_hi B_lo + A_lo B_hi ("3xTF32"): error ~2^-21 per product.
//
// Structure (one CTA per SM, 256 threads, persistent over (m-tile, k-split)
// work items chosen on the device from the live M / K):
//   * all threads stage the next 128x32 A block and 32xN B block from global
//     memory (float4 loads, register double-buffered), split hi/lo and store
//     them in the canonical no-swizzle UMMA layouts (8x16B core matrices);
//   * one elected thread issues 3 x 4 tcgen05.mma.kind::tf32 (M=128, K=8)
//     per 32-wide k block into a TMEM accumulator and tcgen05.commit's to the
//     stage's mbarrier, which releases the stage for the next refill;
//   * warps 0-3 drain TMEM (tcgen05.ld 32x32b) and store the fp32 partial
//     tile; a fixed-order split reduction applies the layer epilogue.
#include "mq_gemm.cuh"

namespace mq {
namespace tc {

constexpr int BM = 128;        // UMMA M (TMEM lanes)
constexpr int BK = 32;         // k block per stage (4 MMAs of K = 8)
constexpr int kThreads = 256;
constexpr int kStages = 2;
constexpr int kMaxN = 256;
constexpr int kMaxSplitsTc = 32;

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

// D[tmem] (+)= A[smem] . B[smem], kind::tf32
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 32 lanes x 32 consecutive 32-bit TMEM columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// no-swizzle UMMA shared-memory descriptor (version 1, base offset 0)
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, M = 128, N = n
__host__ __device__ constexpr uint32_t instr_desc(int n, bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void split4(float4 v, float4& hi, float4& lo) {
  hi.x = tf32_rn(v.x);
  hi.y = tf32_rn(v.y);
  hi.z = tf32_rn(v.z);
  hi.w = tf32_rn(v.w);
  lo.x = tf32_rn(v.x - hi.x);
  lo.y = tf32_rn(v.y - hi.y);
  lo.z = tf32_rn(v.z - hi.z);
  lo.w = tf32_rn(v.w - hi.w);
}

// ---- optional per-phase timeline of CTA 0 (build with -DMQ_TC_TRACE)
#ifdef MQ_TC_TRACE
__device__ unsigned long long g_tc_trace[32];
__device__ __forceinline__ void trace(int i) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && i < 32) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tc_trace[i] = t;
  }
}
#else
__device__ __forceinline__ void trace(int) {}
#endif

// ------------------------------------------------------------ work split
struct Work {
  int tiles_m, S, kb_per;  // m tiles, k splits, k blocks per split
};

__host__ __device__ inline Work choose_work(int M, int K, int grid) {
  Work w;
  w.tiles_m = (M + BM - 1) / BM;
  if (w.tiles_m < 1) w.tiles_m = 1;
  const int nkb = K > 0 ? (K + BK - 1) / BK : 1;
  int S = (grid + w.tiles_m - 1) / w.tiles_m;
  if (S > nkb) S = nkb;
  if (S > kMaxSplitsTc) S = kMaxSplitsTc;
  if (S < 1) S = 1;
  w.kb_per = (nkb + S - 1) / S;
  w.S = (nkb + w.kb_per - 1) / w.kb_per;
  return w;
}

// ------------------------------------------------------------ operands
// Both operands are staged K-major in the canonical no-swizzle layout
// (bytes; core matrix = 8 rows x 16 B = 4 consecutive k of 8 rows):
//     [k/4][row/8][row%8][k%4]   LBO (next 4-k chunk) = ROWS*16, SBO (next 8 rows) = 128
// (a probe on B200 showed kind::tf32 with MN-major operands returning zeros,
// so row-major-in-k sources are transposed in registers, 4x4 at a time).
// FWD: A = X rows (already K-major), B(n, k) = [W_top | W_bot][k][n].
// DW:  A(m, k) = X[k][m] (m = feature), B(n, k) = G[k][n]   (k = sampled row).
enum Mode { kFwd = 0, kDw = 1 };

struct Operands {
  const float* x;  // X (rows x ldx)
  int ldx;
  int d_in;        // valid X columns
  const float* w;  // FWD: W (2 d_in x n_half)
  int n_half;      // FWD: d_out
  const float* g;  // DW: G (rows x N)
  int N;           // output columns (2 d_out)
  int Np;          // padded to a multiple of 16 (UMMA N)
};

// four consecutive columns [c, c+4) of a row, zero beyond `valid`
__device__ __forceinline__ float4 ld_row4(const float* p, int c, int valid, bool vec_ok) {
  if (vec_ok && c + 4 <= valid) return __ldg(reinterpret_cast<const float4*>(p + c));
  float t[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int u = 0; u < 4; ++u)
    if (c + u < valid) t[u] = __ldg(p + c + u);
  return make_float4(t[0], t[1], t[2], t[3]);
}

// A block registers: FWD 4 row chunks, DW one 4x4 block (4 rows of X)
// FWD chunk i: q = warp + 8 i -> (m/8 = q>>1, k4 = (q&1)*4 + lane>>3), m%8 = lane&7
// DW: thread -> (m4 = tid & 31, k4 = tid >> 5): rows k0+4k4+r, features m0+4m4..+3
template <int MODE>
__device__ __forceinline__ void load_a(const Operands& op, int M, int K, int m0, int k0, int tid,
                                       float4 (&ra)[4]) {
  const int lane = tid & 31, w = tid >> 5;
  if (MODE == kFwd) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = w + 8 * i;
      const int m = (q >> 1) * 8 + (lane & 7);
      const int k = k0 + ((q & 1) * 4 + (lane >> 3)) * 4;
      const int gm = m0 + m;
      ra[i] = (gm < M && k < K) ? ld_row4(op.x + (int64_t)gm * op.ldx, k, op.d_in, true)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else {
    const int gm = m0 + 4 * lane;
    const int kr = k0 + 4 * w;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int k = kr + r;
      ra[r] = (k < K && gm < op.d_in) ? ld_row4(op.x + (int64_t)k * op.ldx, gm, op.d_in, true)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

__device__ __forceinline__ void st_split(uint8_t* hi_base, uint8_t* lo_base, uint32_t off, float4 v) {
  float4 hi, lo;
  split4(v, hi, lo);
  *reinterpret_cast<float4*>(hi_base + off) = hi;
  *reinterpret_cast<float4*>(lo_base + off) = lo;
}

// store a 4x4 block given as 4 rows (k = 0..3) x 4 columns (row index c = 0..3)
// as 4 K-major chunks: chunk c = (rows[0][c], rows[1][c], rows[2][c], rows[3][c])
__device__ __forceinline__ void st_transposed(uint8_t* hi_base, uint8_t* lo_base, uint32_t off0,
                                              const float4 (&r)[4]) {
  st_split(hi_base, lo_base, off0 + 0, make_float4(r[0].x, r[1].x, r[2].x, r[3].x));
  st_split(hi_base, lo_base, off0 + 16, make_float4(r[0].y, r[1].y, r[2].y, r[3].y));
  st_split(hi_base, lo_base, off0 + 32, make_float4(r[0].z, r[1].z, r[2].z, r[3].z));
  st_split(hi_base, lo_base, off0 + 48, make_float4(r[0].w, r[1].w, r[2].w, r[3].w));
}

template <int MODE>
__device__ __forceinline__ void store_a(uint8_t* hi, uint8_t* lo, int tid, const float4 (&ra)[4]) {
  const int lane = tid & 31, w = tid >> 5;
  if (MODE == kFwd) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = w + 8 * i;
      const int m = (q >> 1) * 8 + (lane & 7);
      const int k4 = (q & 1) * 4 + (lane >> 3);
      st_split(hi, lo, (uint32_t)(k4 * (BM * 16) + m * 16), ra[i]);
    }
  } else {
    // rows m = 4 lane .. +3 (features), k chunk k4 = w
    st_transposed(hi, lo, (uint32_t)(w * (BM * 16) + (4 * lane) * 16), ra);
  }
}

// B block: (k0..k0+31) x (n 0..Np): 8 k4 x Np/4 n4 blocks of 4x4, at most
// kMaxN/128 = 2 blocks per thread, register double-buffered like A
constexpr int kBPerThread = (8 * (kMaxN / 4) + kThreads - 1) / kThreads;

template <int MODE>
__device__ __forceinline__ float4 load_b4(const Operands& op, int K, int k, int n) {
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (k >= K || n >= op.N) return v;
  if (MODE == kFwd) {
    if (k >= op.d_in) return v;
    const int h = op.n_half;
    if ((h & 3) == 0)
      return n < h ? __ldg(reinterpret_cast<const float4*>(op.w + (int64_t)k * h + n))
                   : __ldg(reinterpret_cast<const float4*>(op.w + (int64_t)(op.d_in + k) * h +
                                                           (n - h)));
    float t4[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int nn = n + e;
      t4[e] = nn < h ? __ldg(op.w + (int64_t)k * h + nn)
                     : (nn < op.N ? __ldg(op.w + (int64_t)(op.d_in + k) * h + (nn - h)) : 0.f);
    }
    return make_float4(t4[0], t4[1], t4[2], t4[3]);
  }
  return ld_row4(op.g + (int64_t)k * op.N, n, op.N, (op.N & 3) == 0);
}

template <int MODE>
__device__ __forceinline__ void load_b(const Operands& op, int K, int k0, int tid,
                                       float4 (&rb)[kBPerThread][4]) {
  const int n4s = op.Np / 4;
#pragma unroll
  for (int i = 0; i < kBPerThread; ++i) {
    const int c = tid + i * kThreads;
    const int n4 = c % n4s, k4 = c / n4s;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      rb[i][u] = c < 8 * n4s ? load_b4<MODE>(op, K, k0 + 4 * k4 + u, 4 * n4)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

__device__ __forceinline__ void store_b(const Operands& op, uint8_t* hi, uint8_t* lo, int tid,
                                        const float4 (&rb)[kBPerThread][4]) {
  const int n4s = op.Np / 4;
#pragma unroll
  for (int i = 0; i < kBPerThread; ++i) {
    const int c = tid + i * kThreads;
    if (c < 8 * n4s) {
      const int n4 = c % n4s, k4 = c / n4s;
      st_transposed(hi, lo, (uint32_t)(k4 * (op.Np * 16) + 4 * n4 * 16), rb[i]);
    }
  }
}

struct Smem {
  // per stage: A_hi, A_lo (BM*BK floats), B_hi, B_lo (BK*kMaxN floats max)
  static constexpr int kA = BM * BK * 4;  // bytes
  __host__ __device__ static int b_bytes(int Np) { return BK * Np * 4; }
  __host__ __device__ static int stage_bytes(int Np) { return 2 * kA + 2 * b_bytes(Np); }
  __host__ __device__ static int total(int Np) { return kStages * stage_bytes(Np) + 1024; }
};

// ------------------------------------------------------------ kernel
template <int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(Operands op, const int32_t* m_dev, int m_static, const int32_t* k_dev,
                   int k_static, float* __restrict__ part, int32_t* __restrict__ nparts_out) {
  MQ_PDL_ENTRY();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bars[kStages + 1];
  __shared__ uint32_t s_tmem;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int M = m_dev ? *m_dev : m_static;
  const int K = k_dev ? *k_dev : k_static;
  const int Np = op.Np;
  const Work wk = choose_work(M, K, gridDim.x);
  const int items = wk.tiles_m * wk.S;
  if (nparts_out != nullptr && blockIdx.x == 0 && tid == 0) *nparts_out = wk.S;
  if ((int)blockIdx.x >= items || M <= 0) return;

  trace(0);
  const uint32_t tmem_cols = Np <= 32 ? 32 : Np <= 64 ? 64 : Np <= 128 ? 128 : 256;
  if (warp == 0) tmem_alloc(&s_tmem, tmem_cols);
  if (tid == 0) {
    for (int i = 0; i <= kStages; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const int stage_bytes = Smem::stage_bytes(Np);
  const uint32_t smem_base = smem_u32(smem);
  const uint32_t idesc = instr_desc(Np, false, false);
  trace(1);

  uint32_t it = 0;  // global k-block counter (stage/phase bookkeeping)
  uint32_t acc_phase = 0;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int s = item % wk.S;
    const int tile = item / wk.S;
    const int m0 = tile * BM;
    const int kb0 = s * wk.kb_per;
    const int nkb_total = (K + BK - 1) / BK;
    const int kb1 = min(nkb_total, kb0 + wk.kb_per);

    if (kb0 >= kb1) {  // no rows to reduce over (K == 0): the partial is zero
      if (warp < 4 && m0 + warp * 32 + lane < M) {
        float* out = part + ((int64_t)s * M + m0 + warp * 32 + lane) * op.N;
        for (int c = 0; c < op.N; ++c) out[c] = 0.f;
      }
      continue;
    }
    float4 ra[4];
    float4 rb[kBPerThread][4];
    load_a<MODE>(op, M, K, m0, kb0 * BK, tid, ra);
    load_b<MODE>(op, K, kb0 * BK, tid, rb);
    trace(2);
    for (int kb = kb0; kb < kb1; ++kb, ++it) {
      const int stage = it % kStages;
      uint8_t* st = smem + stage * stage_bytes;
      // the MMAs that last read this stage must have completed
      if (it >= (uint32_t)kStages) mbar_wait(&bars[stage], ((it / kStages) - 1) & 1);
      // ---- stage A and B (split hi/lo)
      store_a<MODE>(st, st + Smem::kA, tid, ra);
      store_b(op, st + 2 * Smem::kA, st + 2 * Smem::kA + Smem::b_bytes(Np), tid, rb);
      fence_async_smem();
      tc_fence_before();
      __syncthreads();
      trace(3 + 2 * (kb - kb0));
      // prefetch the next A block while the tensor core works on this one
      if (kb + 1 < kb1) {
        load_a<MODE>(op, M, K, m0, (kb + 1) * BK, tid, ra);
        load_b<MODE>(op, K, (kb + 1) * BK, tid, rb);
      }
      if (tid == 0) {
        tc_fence_after();
        const uint32_t a_hi = smem_base + stage * stage_bytes;
        const uint32_t a_lo = a_hi + Smem::kA;
        const uint32_t b_hi = a_hi + 2 * Smem::kA;
        const uint32_t b_lo = b_hi + Smem::b_bytes(Np);
#pragma unroll
        for (int j = 0; j < BK / 8; ++j) {  // K = 8 per MMA = two 4-wide k chunks
          const uint32_t a_off = (uint32_t)(2 * j) * (BM * 16);
          const uint32_t b_off = (uint32_t)(2 * j) * (Np * 16);
          const uint64_t dah = smem_desc(a_hi + a_off, BM * 16, 128);
          const uint64_t dal = smem_desc(a_lo + a_off, BM * 16, 128);
          const uint64_t dbh = smem_desc(b_hi + b_off, Np * 16, 128);
          const uint64_t dbl = smem_desc(b_lo + b_off, Np * 16, 128);
          const uint32_t first = (kb == kb0 && j == 0) ? 0u : 1u;
          mma_tf32(tmem, dal, dbh, idesc, first);  // small terms first
          mma_tf32(tmem, dah, dbl, idesc, 1u);
          mma_tf32(tmem, dah, dbh, idesc, 1u);
        }
        mma_commit(&bars[stage]);
      }
      trace(4 + 2 * (kb - kb0));
    }
    // ---- accumulator ready -> partial tile
    if (tid == 0) mma_commit(&bars[kStages]);
    mbar_wait(&bars[kStages], acc_phase & 1);
    ++acc_phase;
    tc_fence_after();
    trace(20);
    if (warp < 4) {
      const int m = warp * 32 + lane;
      const int gm = m0 + m;
      float* out = part + ((int64_t)s * M + gm) * op.N;
      for (int cb = 0; cb < Np; cb += 32) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)cb, v);
        if (gm < M) {
          if ((op.N & 3) == 0 && cb + 32 <= op.N) {
#pragma unroll
            for (int u = 0; u < 32; u += 4)
              *reinterpret_cast<float4*>(out + cb + u) = make_float4(v[u], v[u + 1], v[u + 2], v[u + 3]);
          } else {
#pragma unroll
            for (int u = 0; u < 32; ++u)
              if (cb + u < op.N) out[cb + u] = v[u];
          }
        }
      }
    }
    tc_fence_before();
    __syncthreads();
    trace(21);
  }
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols);
  }
  trace(22);
}

// fixed-order split reduction + layer epilogue (same decomposition as the GEMM)
template <class Epi>
__global__ void tc_reduce_kernel(const float* __restrict__ part, const int32_t* m_dev, int m_static,
                                 const int32_t* k_dev, int k_static, int N, int grid_gemm, Epi epi) {
  MQ_PDL_ENTRY();
  const int M = m_dev ? *m_dev : m_static;
  const int K = k_dev ? *k_dev : k_static;
  const Work wk = choose_work(M, K, grid_gemm);
  const int64_t total = (int64_t)M * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / N), j = (int)(e % N);
    epi(i, j, fixed_order_sum(part + e, total, wk.S));
  }
}

}  // namespace tc

// ------------------------------------------------------------ host side
static int g_gemm_backend = 1;  // 1 = tcgen05 3xTF32, 0 = fp32 FFMA split-K

inline int tc_grid(int m_max, int k_max) {
  const int tiles = (m_max + tc::BM - 1) / tc::BM;
  const int nkb = (k_max + tc::BK - 1) / tc::BK;
  long long cap = (long long)(tiles < 1 ? 1 : tiles) *
                  (nkb < 1 ? 1 : (nkb > tc::kMaxSplitsTc ? tc::kMaxSplitsTc : nkb));
  return (int)(cap < kNumSMs ? cap : kNumSMs);
}

template <int MODE, class Epi>
int run_tc_gemm(const tc::Operands& op, const int32_t* m_dev, int m_static, int m_max,
                const int32_t* k_dev, int k_static, int k_max, float* part, const Epi& epi,
                cudaStream_t s, int kid, int kid_red, bool skip_reduce = false,
                int32_t* nparts_out = nullptr) {
  const int smem = tc::Smem::total(op.Np);
  static thread_local bool configured[2] = {false, false};
  if (!configured[MODE]) {
    MQ_CUDA(cudaFuncSetAttribute(tc::tc_gemm_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 tc::Smem::total(tc::kMaxN)));
    configured[MODE] = true;
  }
  const int grid = tc_grid(m_max, k_max);
  {
    ProfScope ps(kid, s);
    MQ_CUDA(launch_k(tc::tc_gemm_kernel<MODE>, dim3(grid), dim3(tc::kThreads), smem, s, op, m_dev, m_static, k_dev, k_static,
                                                             part, nparts_out));
  }
  MQ_LAUNCH_CHECK("tc_gemm");
  if (skip_reduce) return MQ_OK;
  int64_t mn = (int64_t)(m_max < 1 ? 1 : m_max) * op.N;
  int rb = ceil_div(mn, 256);
  if (rb > kNumSMs * 4) rb = kNumSMs * 4;
  {
    ProfScope ps(kid_red, s);
    MQ_CUDA(launch_k(tc::tc_reduce_kernel<Epi>, dim3(rb), dim3(256), 0, s, part, m_dev, m_static, k_dev, k_static, op.N, grid,
                                                 epi));
  }
  MQ_LAUNCH_CHECK("tc_reduce");
  return MQ_OK;
}

// floats of partials the tc path may write for an (m_max x n) output: the
// device picks S <= ceil(grid / tiles_m), so S*M <= grid*BM + M.
inline int64_t tc_part_floats(int64_t m_max, int64_t n) {
  if (m_max < 1) m_max = 1;
  const int64_t a = (int64_t)tc::kMaxSplitsTc * m_max;
  const int64_t b = (int64_t)kNumSMs * tc::BM + m_max;
  return (a < b ? a : b) * n;
}

}  // namespace mq

using namespace mq;

// Entry points used by mq_fused.cu (C++ linkage inside the library).
namespace mq {

int tc_backend() { return g_gemm_backend; }

bool tc_supported(int n_out) {
  const int Np = (n_out + 15) / 16 * 16;
  return Np <= tc::kMaxN;
}

int tc_transform(const float* h, int ldh, const int32_t* m_dev, int m_max, int d_in, const float* W,
                 int d_out, float* y, float* part, int32_t* nparts_out, cudaStream_t s) {
  tc::Operands op{h, ldh, d_in, W, d_out, nullptr, 2 * d_out, (2 * d_out + 15) / 16 * 16};
  // y == NULL: leave the partial tiles (count -> *nparts_out) for the aggregation
  return run_tc_gemm<tc::kFwd>(op, m_dev, 0, m_max, nullptr, d_in, d_in, part,
                               EpiStore{y, 2 * d_out}, s, K_SAGE_TRANSFORM,
                               K_SAGE_TRANSFORM_REDUCE, y == nullptr, nparts_out);
}

int64_t tc_y_part_floats(int64_t m_max, int64_t d_out) { return tc_part_floats(m_max, 2 * d_out); }

// Y = h [W_top | W_bot] over a host-known row count (full-graph evaluation)
int tc_transform_rows(const float* h, int ldh, int64_t n, int d_in, const float* W, int d_out,
                      float* y, float* part, cudaStream_t s) {
  tc::Operands op{h, ldh, d_in, W, d_out, nullptr, 2 * d_out, (2 * d_out + 15) / 16 * 16};
  return run_tc_gemm<tc::kFwd>(op, nullptr, (int)n, (int)n, nullptr, d_in, d_in, part,
                               EpiStore{y, 2 * d_out}, s, K_FULL_TRANSFORM,
                               K_FULL_TRANSFORM_REDUCE);
}

int tc_weight_grad(const float* h, int ldh, const int32_t* rows_dev, int rows_max, int d_in,
                   int d_out, const float* g, float* dW, float* part, int32_t* nparts_out,
                   cudaStream_t s) {
  tc::Operands op{h, ldh, d_in, nullptr, d_out, g, 2 * d_out, (2 * d_out + 15) / 16 * 16};
  // dW == NULL: leave the partial tiles (count -> *nparts_out) for the consumer
  return run_tc_gemm<tc::kDw>(op, nullptr, d_in, d_in, rows_dev, 0, rows_max, part,
                              EpiDWSplit{dW, d_in, d_out}, s, K_SAGE_DW, K_SAGE_DW_REDUCE,
                              dW == nullptr, nparts_out);
}

int64_t tc_dw_part_floats(int64_t d_in, int64_t d_out) { return tc_part_floats(d_in, 2 * d_out); }

int64_t tc_scratch_floats(int64_t m_max, int64_t d_in, int64_t d_out) {
  int64_t a = tc_part_floats(m_max, 2 * d_out);
  int64_t b = tc_part_floats(d_in, 2 * d_out);
  return a > b ? a : b;
}

}  // namespace mq

extern "C" {

int mq_set_gemm_backend(int32_t backend) {
  MQ_CHECK_ARG(backend == 0 || backend == 1, "mq_set_gemm_backend: 0 (fp32 FFMA) or 1 (tcgen05)");
  g_gemm_backend = backend;
  return MQ_OK;
}

int mq_get_gemm_backend(void) { return g_gemm_backend; }

#ifdef MQ_TC_TRACE
int mq_debug_tc_trace(unsigned long long* out) {
  MQ_CUDA(cudaMemcpyFromSymbol(out, tc::g_tc_trace, sizeof(unsigned long long) * 32));
  return MQ_OK;
}
#endif

}  // extern "C"
