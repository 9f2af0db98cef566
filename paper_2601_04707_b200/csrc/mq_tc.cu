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
#include <cuda.h>
#include <stdlib.h>  // CUtensorMap (the encoder comes from the runtime's driver entry point)

#include "mq_gemm.cuh"

namespace mq {
namespace tc {

constexpr int BM = 128;        // UMMA M (TMEM lanes)
constexpr int BK = 32;         // k block per stage (4 MMAs of K = 8)
constexpr int kThreads = 256;           // staging / epilogue warps 0-7
constexpr int kBlock = kThreads + 32;    // + warp 8: TMEM owner and MMA issuer
constexpr int kStages = 2;
constexpr int kMaxN = 256;
constexpr int kCoopTiles = 512;     // tiles covered by the cooperative split reduction
constexpr int kMaxSplitsTc = 148;  // = SMs: a one-tile DW (d_in <= 128) still fills the GPU

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

// v2 split: hi = tf32_rn(x) by integer rounding (2 ops), lo = x - hi exactly;
// lo is left in fp32 and the tensor core's own tf32 read of it costs at most
// 2^-10 |lo| <= 2^-21 |x| (v1 rounds lo explicitly: same bound, 6 more ops)
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
__device__ __forceinline__ void split4f(float4 v, float4& hi, float4& lo) {
  hi = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
  lo = make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
}

// ---- optional per-phase timeline of CTA 0 (build with -DMQ_TC_TRACE)
#ifdef MQ_TC_TRACE
__device__ unsigned long long g_tc_trace[64];
__device__ __forceinline__ void trace(int i) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && i < 32) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tc_trace[i] = t;
  }
}
__device__ unsigned long long g_tc_cta[256][2];
__device__ __forceinline__ void cta_mark(int i) {
  if (threadIdx.x == 0 && blockIdx.x < 256) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tc_cta[blockIdx.x][i] = t;
  }
}
__device__ __forceinline__ void ktrace(bool on, uint32_t it, int p) {
  if (on && it < 3) trace(3 + 8 * (int)it + p);
}
__device__ __forceinline__ void trace_at(int i) {  // caller picks the thread
  if (blockIdx.x == 0 && i < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tc_trace[i] = t;
  }
}
#else
__device__ __forceinline__ void trace_at(int) {}
__device__ __forceinline__ void trace(int) {}
__device__ __forceinline__ void ktrace(bool, uint32_t, int) {}
__device__ __forceinline__ void cta_mark(int) {}
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
// Aggregate-first layer (mq_sage_linear_af, the reference's own association,
// nn.py:126-131 / 167-170) — used for the input layer when d_in is narrow:
//   FCAT: Z (M x N) = [agg | h] (M x 2 d_in) . W (2 d_in x N)   M = dst rows
//   DCAT: P (2 d_in x N) = [agg | h]^T . (dh * (act > 0))      K = dst rows
//   DX:   dh (M x d_in) = G (M x 2 d_out) . [W_top | W_bot]^T  (nn.py:171-174,
//         the input gradient of a transform-first hidden layer; B is K-major
//         straight from W's rows)
enum Mode { kFwd = 0, kDw = 1, kFwdCat = 2, kDwCat = 3, kDx = 4 };
__host__ __device__ constexpr bool rowA(int mode) {  // A = rows of a row-major matrix (K-major)
  return mode == kFwd || mode == kFwdCat || mode == kDx;
}

struct Operands {
  const float* x;  // X (rows x ldx)                      CAT: agg
  int ldx;
  int d_in;        // valid X columns
  const float* w;  // FWD: W (2 d_in x n_half)            FCAT: W (2 d_in x N)
  int n_half;      // FWD: d_out
  const float* g;  // DW: G (rows x N)                    DCAT: dh (rows x ldg)
  int N;           // output columns (2 d_out; CAT: d_out)
  int Np;          // padded to a multiple of 16 (UMMA N)
  const float* x2 = nullptr;  // CAT: h (second K / M half)
  int ldx2 = 0;
  int ldg = 0;                // DCAT: dh pitch
  const float* act = nullptr; // DCAT: relu output (mask), pitch ldact
  int ldact = 0;
  int wd_in = 0, wd_out = 0;  // DX: W is (2 wd_in x wd_out); N = wd_in, K = 2 wd_out
  float* out = nullptr;       // when the device picks S = 1: write the tile here directly
  int ldo = 0;
  int relu = 0;               // ... through max(., 0) (the FCAT layer's activation)
};

// DX operand B(n, k..k+3): row n of W_top (k < wd_out) or W_bot, K-major
__device__ __forceinline__ const float* dx_src(const Operands& op, int n, int k) {
  return k < op.wd_out ? op.w + (int64_t)n * op.wd_out + k
                       : op.w + (int64_t)(op.wd_in + n) * op.wd_out + (k - op.wd_out);
}

// CAT operand A: four consecutive columns c of row r of [agg | h] (d_in % 4 == 0)
__device__ __forceinline__ float4 ld_cat4(const Operands& op, int64_t r, int c) {
  if (c < op.d_in) return __ldg(reinterpret_cast<const float4*>(op.x + r * op.ldx + c));
  if (c < 2 * op.d_in)
    return __ldg(reinterpret_cast<const float4*>(op.x2 + r * op.ldx2 + (c - op.d_in)));
  return make_float4(0.f, 0.f, 0.f, 0.f);
}

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
  if (rowA(MODE)) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = w + 8 * i;
      const int m = (q >> 1) * 8 + (lane & 7);
      const int k = k0 + ((q & 1) * 4 + (lane >> 3)) * 4;
      const int gm = m0 + m;
      if (MODE != kFwdCat)
        ra[i] = (gm < M && k < K) ? ld_row4(op.x + (int64_t)gm * op.ldx, k, op.d_in, true)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
      else
        ra[i] = (gm < M && k < K) ? ld_cat4(op, gm, k) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else {
    const int gm = m0 + 4 * lane;
    const int kr = k0 + 4 * w;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int k = kr + r;
      if (MODE == kDw)
        ra[r] = (k < K && gm < op.d_in) ? ld_row4(op.x + (int64_t)k * op.ldx, gm, op.d_in, true)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
      else
        ra[r] = (k < K && gm < 2 * op.d_in) ? ld_cat4(op, k, gm) : make_float4(0.f, 0.f, 0.f, 0.f);
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
// at off0 + 16 c.  Neighbouring threads' blocks are 64 B apart, so the four
// stores go out in a thread-dependent rotation (`rot`): the 8 lanes of a
// store phase then hit 8 distinct 16-byte bank groups (no bank conflicts).
__device__ __forceinline__ float4 col4(const float4 (&r)[4], int c) {
  return c == 0 ? make_float4(r[0].x, r[1].x, r[2].x, r[3].x)
       : c == 1 ? make_float4(r[0].y, r[1].y, r[2].y, r[3].y)
       : c == 2 ? make_float4(r[0].z, r[1].z, r[2].z, r[3].z)
                : make_float4(r[0].w, r[1].w, r[2].w, r[3].w);
}
__device__ __forceinline__ void st_transposed(uint8_t* hi_base, uint8_t* lo_base, uint32_t off0,
                                              const float4 (&r)[4], int rot) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = (j + rot) & 3;
    st_split(hi_base, lo_base, off0 + 16 * c, col4(r, c));
  }
}

template <int MODE>
__device__ __forceinline__ void store_a(uint8_t* hi, uint8_t* lo, int tid, const float4 (&ra)[4]) {
  const int lane = tid & 31, w = tid >> 5;
  if (rowA(MODE)) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = w + 8 * i;
      const int m = (q >> 1) * 8 + (lane & 7);
      const int k4 = (q & 1) * 4 + (lane >> 3);
      st_split(hi, lo, (uint32_t)(k4 * (BM * 16) + m * 16), ra[i]);
    }
  } else {
    // rows m = 4 lane .. +3 (features), k chunk k4 = w
    st_transposed(hi, lo, (uint32_t)(w * (BM * 16) + (4 * lane) * 16), ra, lane >> 1);
  }
}

// B block: (k0..k0+31) x (n 0..Np): 8 k4 x Np/4 n4 blocks of 4x4, at most
// kMaxN/128 = 2 blocks per thread, register double-buffered like A
constexpr int kBPerThread = (8 * (kMaxN / 4) + kThreads - 1) / kThreads;

template <int MODE>
__device__ __forceinline__ float4 load_b4(const Operands& op, int K, int k, int n) {
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (k >= K || n >= op.N) return v;
  if (MODE == kFwdCat) {  // W (2 d_in x N), row k
    if (k >= 2 * op.d_in) return v;
    return ld_row4(op.w + (int64_t)k * op.N, n, op.N, (op.N & 3) == 0);
  }
  if (MODE == kDwCat) {  // dz = dh * (act > 0), row k
    const float4 g = ld_row4(op.g + (int64_t)k * op.ldg, n, op.N, (op.N & 3) == 0);
    const float4 a = ld_row4(op.act + (int64_t)k * op.ldact, n, op.N, (op.N & 3) == 0);
    return make_float4(a.x > 0.f ? g.x : 0.f, a.y > 0.f ? g.y : 0.f, a.z > 0.f ? g.z : 0.f,
                       a.w > 0.f ? g.w : 0.f);
  }
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

// DX B chunk j of a thread: g = j * kThreads + tid, n = g % Np, k4 = g / Np
// (consecutive lanes -> consecutive n: conflict-free K-major smem stores)
template <int MODE>
__device__ __forceinline__ void load_b(const Operands& op, int K, int k0, int tid,
                                       float4 (&rb)[kBPerThread][4]) {
  if (MODE == kDx) {
#pragma unroll
    for (int j = 0; j < 4 * kBPerThread; ++j) {
      const int g = j * kThreads + tid;
      const int n = g % op.Np, k = k0 + 4 * (g / op.Np);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (g < 8 * op.Np && n < op.N && k < K) {
        const float* p = dx_src(op, n, k);
        if ((op.wd_out & 3) == 0) {
          v = __ldg(reinterpret_cast<const float4*>(p));
        } else {
          float t[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) t[e] = k + e < K ? __ldg(dx_src(op, n, k + e)) : 0.f;
          v = make_float4(t[0], t[1], t[2], t[3]);
        }
      }
      rb[j >> 2][j & 3] = v;
    }
    return;
  }
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

template <int MODE>
__device__ __forceinline__ void store_b(const Operands& op, uint8_t* hi, uint8_t* lo, int tid,
                                        const float4 (&rb)[kBPerThread][4]) {
  if (MODE == kDx) {
#pragma unroll
    for (int j = 0; j < 4 * kBPerThread; ++j) {
      const int g = j * kThreads + tid;
      if (g < 8 * op.Np)
        st_split(hi, lo, (uint32_t)((g / op.Np) * (op.Np * 16) + (g % op.Np) * 16), rb[j >> 2][j & 3]);
    }
    return;
  }
  const int n4s = op.Np / 4;
#pragma unroll
  for (int i = 0; i < kBPerThread; ++i) {
    const int c = tid + i * kThreads;
    if (c < 8 * n4s) {
      const int n4 = c % n4s, k4 = c / n4s;
      st_transposed(hi, lo, (uint32_t)(k4 * (op.Np * 16) + 4 * n4 * 16), rb[i], n4 >> 1);
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

// ------------------------------------------------------------ async staging
// Deep prefetch for the vectorisable shapes: each thread's A / B chunks of a
// k block land by cp.async (16 B, zero-filled past the valid columns) in a
// THREAD-PRIVATE slot of an R-deep raw ring, so R - 1 k blocks are in flight
// per CTA (the register path holds one) and no barrier is needed between a
// chunk's arrival and its hi/lo split: the thread that loaded it converts it.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_dyn(int n) {  // wait_group needs an immediate
  switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;\n" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;\n" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;\n" ::: "memory"); break;
    case 3: asm volatile("cp.async.wait_group 3;\n" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 4;\n" ::: "memory"); break;
  }
}
constexpr int kMaxRaw = 6;  // raw ring depth cap (wait_group <= 4)

__host__ __device__ inline int raw_chunks(int mode, int Np) {
  const int nb = (Np + 127) / 128;  // B chunk groups per thread (kBPerThread in use)
  return 4 + 4 * nb + (mode == kDwCat ? 4 * nb : 0);
}
__host__ __device__ inline int raw_bytes(int mode, int Np) { return raw_chunks(mode, Np) * kThreads * 16; }

__device__ __forceinline__ int vbytes(int valid_cols) {  // 4-float chunk, `valid_cols` valid
  return valid_cols <= 0 ? 0 : (valid_cols >= 4 ? 16 : 4 * valid_cols);
}

// cat source of columns [c, c+4) of row r of [x | x2] (d_in % 4 == 0)
__device__ __forceinline__ const float* cat_src(const Operands& op, int64_t r, int c, int& bytes) {
  if (c < op.d_in) {
    bytes = 16;
    return op.x + r * op.ldx + c;
  }
  if (c < 2 * op.d_in) {
    bytes = 16;
    return op.x2 + r * op.ldx2 + (c - op.d_in);
  }
  bytes = 0;
  return op.x;
}

template <int MODE>
__device__ __forceinline__ void issue_async(const Operands& op, int M, int K, int m0, int k0,
                                            int tid, uint32_t slot) {
  const int lane = tid & 31, w = tid >> 5;
  auto dst = [&](int j) { return slot + (uint32_t)((j * kThreads + tid) * 16); };
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float* src = op.x;
    int bytes = 0;
    if (rowA(MODE)) {
      // coalesced: 8 consecutive lanes fetch one row's 32 k (128 B); the
      // chunk lands at the XOR-swizzled slot [row][k4 ^ (row & 7)], so both
      // this write and the converter's column-wise read are conflict-free
      const int g = i * kThreads + tid;
      const int row = g >> 3, k4 = g & 7;
      const int gm = m0 + row;
      const int k = k0 + 4 * k4;
      if (gm < M && k < K) {
        if (MODE != kFwdCat) {
          src = op.x + (int64_t)gm * op.ldx + k;
          bytes = vbytes(op.d_in - k);
        } else {
          src = cat_src(op, gm, k, bytes);
        }
      }
      cp_async16(slot + (uint32_t)((row * 8 + (k4 ^ (row & 7))) * 16), bytes ? src : op.x, bytes);
      continue;
    } else {
      const int gm = m0 + 4 * lane;
      const int k = k0 + 4 * w + i;
      if (k < K) {
        if (MODE == kDw) {
          src = op.x + (int64_t)k * op.ldx + gm;
          bytes = vbytes(op.d_in - gm);
        } else {
          src = cat_src(op, k, gm, bytes);
        }
      }
    }
    cp_async16(dst(i), bytes ? src : op.x, bytes);
  }
  const int n4s = op.Np / 4;
  const int nb = (op.Np + 127) / 128;
  if (MODE == kDx) {
    for (int j = 0; j < 4 * nb; ++j) {
      const int g = j * kThreads + tid;
      const int n = g % op.Np, k = k0 + 4 * (g / op.Np);
      const bool ok = g < 8 * op.Np && n < op.N && k < K;
      cp_async16(dst(4 + j), ok ? dx_src(op, n, k) : op.x, ok ? 16 : 0);
    }
    return;
  }
  for (int i = 0; i < nb; ++i) {
    const int c = tid + i * kThreads;
    const int n4 = c % n4s, k4 = c / n4s;
    const int n = 4 * n4;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + 4 * k4 + u;
      const float* src = op.x;
      const float* msk = op.x;
      int bytes = 0;
      if (c < 8 * n4s && k < K && n < op.N) {
        if (MODE == kFwd) {
          if (k < op.d_in) {
            const int h = op.n_half;
            src = n < h ? op.w + (int64_t)k * h + n : op.w + (int64_t)(op.d_in + k) * h + (n - h);
            bytes = vbytes(op.N - n);
          }
        } else if (MODE == kFwdCat) {
          if (k < 2 * op.d_in) {
            src = op.w + (int64_t)k * op.N + n;
            bytes = vbytes(op.N - n);
          }
        } else if (MODE == kDw) {
          src = op.g + (int64_t)k * op.N + n;
          bytes = vbytes(op.N - n);
        } else {
          src = op.g + (int64_t)k * op.ldg + n;
          msk = op.act + (int64_t)k * op.ldact + n;
          bytes = vbytes(op.N - n);
        }
      }
      cp_async16(dst(4 + 4 * i + u), bytes ? src : op.x, bytes);
      if (MODE == kDwCat) cp_async16(dst(4 + 4 * nb + 4 * i + u), bytes ? msk : op.x, bytes);
    }
  }
}

template <int MODE>
__device__ __forceinline__ void read_raw(const Operands& op, const uint8_t* slot, int tid,
                                         float4 (&ra)[4], float4 (&rb)[kBPerThread][4]) {
  auto at = [&](int j) {
    return *reinterpret_cast<const float4*>(slot + (size_t)(j * kThreads + tid) * 16);
  };
  if (rowA(MODE)) {  // the shared, swizzled A tile (see issue_async)
    const int lane = tid & 31, w = tid >> 5;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q = w + 8 * i;
      const int m = (q >> 1) * 8 + (lane & 7);
      const int k4 = (q & 1) * 4 + (lane >> 3);
      ra[i] = *reinterpret_cast<const float4*>(slot + (size_t)(m * 8 + (k4 ^ (m & 7))) * 16);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) ra[i] = at(i);
  }
  const int nb = (op.Np + 127) / 128;
#pragma unroll
  for (int i = 0; i < kBPerThread; ++i)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (i < nb) {
        float4 g = at(4 + 4 * i + u);
        if (MODE == kDwCat) {
          const float4 a = at(4 + 4 * nb + 4 * i + u);
          g = make_float4(a.x > 0.f ? g.x : 0.f, a.y > 0.f ? g.y : 0.f, a.z > 0.f ? g.z : 0.f,
                          a.w > 0.f ? g.w : 0.f);
        }
        rb[i][u] = g;
      } else {
        rb[i][u] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
}

// ------------------------------------------------------------ kernel
template <int MODE, bool ASYNC>
__global__ void __launch_bounds__(kBlock, 1)
    tc_gemm_kernel(Operands op, const int32_t* m_dev, int m_static, const int32_t* k_dev,
                   int k_static, float* __restrict__ part, int32_t* __restrict__ nparts_out,
                   int R) {
  // PDL: TMEM allocation and barrier setup overlap the predecessor's tail;
  // every operand read waits (pdl_wait) — the frontier counts (m_dev / k_dev)
  // come from the prep pass, which completed before this graph segment
  pdl_trigger();
  MQ_TL_BEGIN(MODE);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned, derived from smem_raw by an integer offset so the
  // compiler keeps the shared address space (LDS / STS, not generic LD / ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bars[kStages + 1];
  __shared__ uint32_t s_tmem;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int M = m_dev ? *m_dev : m_static;
  const int K = k_dev ? *k_dev : k_static;
  const int Np = op.Np;
  const Work wk = choose_work(M, K, gridDim.x);
  const int items = wk.tiles_m * wk.S;
  // the split count is published only after the wait: with programmatic
  // dependent launch this grid may start while the previous window's optimizer
  // still reads the same counter
  auto publish_nparts = [&]() {
    if (nparts_out != nullptr && blockIdx.x == 0 && tid == 0) *nparts_out = wk.S;
  };
  if ((int)blockIdx.x >= items || M <= 0) {
    pdl_wait();
    publish_nparts();
    return;
  }

  trace(0);
  cta_mark(0);
  const bool worker = warp < kThreads / 32;
  const bool issuer = tid == kThreads;  // warp 8, lane 0
  const uint32_t tmem_cols = Np <= 32 ? 32 : Np <= 64 ? 64 : Np <= 128 ? 128 : 256;
  if (!worker) tmem_alloc(&s_tmem, tmem_cols);
  if (tid == 0) {
    for (int i = 0; i <= kStages; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  publish_nparts();
  const uint32_t tmem = s_tmem;
  const int stage_bytes = Smem::stage_bytes(Np);
  const uint32_t smem_base = smem_u32(smem);
  const uint32_t idesc = instr_desc(Np, false, false);
  trace(1);

  uint32_t it = 0;  // global k-block counter (stage/phase bookkeeping)
  uint32_t acc_phase = 0;
  const int nkb_total = (K + BK - 1) / BK;
  float4 ra[4];
  float4 rb[kBPerThread][4];
  bool have = false;  // ra/rb already hold this item's first k block
  // async ring: the load cursor runs R - 1 k blocks ahead of the MMAs, across items
  uint8_t* raw = smem + kStages * stage_bytes;
  const uint32_t raw_base = smem_u32(raw);
  const int rbytes = raw_bytes(MODE, Np);
  int l_item = blockIdx.x, l_kb = 0, l_kb1 = 0;
  auto l_begin = [&]() {
    while (l_item < items) {
      l_kb = (l_item % wk.S) * wk.kb_per;
      l_kb1 = min(nkb_total, l_kb + wk.kb_per);
      if (l_kb < l_kb1) return;
      l_item += gridDim.x;
    }
  };
  auto l_issue = [&](uint32_t seq) {  // the cursor's k block into slot seq % R, then advance
    if (l_item < items) {
      issue_async<MODE>(op, M, K, (l_item / wk.S) * BM, l_kb * BK, tid,
                        raw_base + (uint32_t)((seq % (uint32_t)R) * rbytes));
      if (++l_kb >= l_kb1) {
        l_item += gridDim.x;
        l_begin();
      }
    }
    cp_commit();
  };
  if (ASYNC && worker) {
    l_begin();
    for (int r = 0; r < R - 1; ++r) l_issue((uint32_t)r);
  }
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int s = item % wk.S;
    const int tile = item / wk.S;
    const int m0 = tile * BM;
    const int kb0 = s * wk.kb_per;
    const int kb1 = min(nkb_total, kb0 + wk.kb_per);

    if (kb0 >= kb1) {  // no rows to reduce over (K == 0): the partial is zero
      if (warp < 4 && m0 + warp * 32 + lane < M) {  // (all threads skip alike)
        float* out = part + ((int64_t)s * M + m0 + warp * 32 + lane) * op.N;
        for (int c = 0; c < op.N; ++c) out[c] = 0.f;
      }
      have = false;
      continue;
    }
    if (!ASYNC && !have && worker) {
      load_a<MODE>(op, M, K, m0, kb0 * BK, tid, ra);
      load_b<MODE>(op, K, kb0 * BK, tid, rb);
    }
    have = false;
    const bool first_item = item == (int)blockIdx.x;
    if (first_item) trace(2);
    for (int kb = kb0; kb < kb1; ++kb, ++it) {
      const int stage = it % kStages;
      uint8_t* st = smem + stage * stage_bytes;
      ktrace(first_item, it, 0);
      if (worker) {
        if (ASYNC) {  // this k block's chunks have landed
          cp_wait_dyn(R - 2);
          // the forward A tile is shared between the staging threads
          if (rowA(MODE)) asm volatile("bar.sync 2, %0;" ::"n"(kThreads));
          ktrace(first_item, it, 1);
          read_raw<MODE>(op, raw + (size_t)(it % (uint32_t)R) * rbytes, tid, ra, rb);
          l_issue(it + (uint32_t)R - 1);
          ktrace(first_item, it, 2);
        }
        // the MMAs that last read this stage must have completed
        if (it >= (uint32_t)kStages) mbar_wait(&bars[stage], ((it / kStages) - 1) & 1);
        ktrace(first_item, it, 3);
        // ---- stage A and B (split hi/lo)
        store_a<MODE>(st, st + Smem::kA, tid, ra);
        ktrace(first_item, it, 4);
        store_b<MODE>(op, st + 2 * Smem::kA, st + 2 * Smem::kA + Smem::b_bytes(Np), tid, rb);
        ktrace(first_item, it, 5);
      }
      fence_async_smem();
      tc_fence_before();
      __syncthreads();
      ktrace(first_item, it, 6);
      // prefetch the next A block while the tensor core works on this one;
      // after the last block, the next item's first block, so its load
      // latency hides behind this item's accumulator drain
      if (ASYNC || !worker) {
      } else if (kb + 1 < kb1) {
        load_a<MODE>(op, M, K, m0, (kb + 1) * BK, tid, ra);
        load_b<MODE>(op, K, (kb + 1) * BK, tid, rb);
      } else if (item + (int)gridDim.x < items) {
        const int nitem = item + (int)gridDim.x;
        const int nkb0 = (nitem % wk.S) * wk.kb_per;
        if (nkb0 < nkb_total) {
          load_a<MODE>(op, M, K, (nitem / wk.S) * BM, nkb0 * BK, tid, ra);
          load_b<MODE>(op, K, nkb0 * BK, tid, rb);
          have = true;
        }
      }
      if (issuer) {  // off the staging warps' critical path
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
      ktrace(first_item, it, 7);
    }
    // ---- accumulator ready -> partial tile (all 8 staging warps: warp w
    // drains TMEM lanes 32 (w % 4).. and every other 32-column block)
    if (issuer) mma_commit(&bars[kStages]);
    mbar_wait(&bars[kStages], acc_phase & 1);
    ++acc_phase;
    tc_fence_after();
    if (first_item) trace(27);
    if (worker) {
      // TMEM -> smem tile [BM][Np + 4] (the stage buffers are idle: this
      // item's MMAs have completed) -> coalesced row stores: a warp writes
      // whole rows instead of 32 rows x 16 B per instruction
      float* tile = reinterpret_cast<float*>(smem);
      const int ldt = (Np + 31) / 32 * 32 + 4;  // whole 32-column TMEM loads fit
      const int m = (warp & 3) * 32 + lane;
      for (int cb = 32 * (warp >> 2); cb < Np; cb += 64) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)cb, v);
#pragma unroll
        for (int u = 0; u < 32; u += 4)
          *reinterpret_cast<float4*>(tile + m * ldt + cb + u) =
              make_float4(v[u], v[u + 1], v[u + 2], v[u + 3]);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kThreads));  // staging warps only
      const int rows = min(BM, M - m0);
      // a single split is already the result: straight to op.out when given
      float* dst = (wk.S == 1 && op.out) ? op.out : part + (int64_t)s * M * op.N;
      const int ldd = (wk.S == 1 && op.out) ? op.ldo : op.N;
      const bool relu = wk.S == 1 && op.out && op.relu;
      if ((op.N & 3) == 0 && (ldd & 3) == 0 && ((uintptr_t)dst & 15) == 0) {
        const int n4 = op.N / 4;
        for (int e = tid; e < rows * n4; e += kThreads) {
          const int r = e / n4, c = 4 * (e % n4);
          float4 v = *reinterpret_cast<const float4*>(tile + r * ldt + c);
          if (relu) v = make_float4(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f), fmaxf(v.z, 0.f), fmaxf(v.w, 0.f));
          *reinterpret_cast<float4*>(dst + (int64_t)(m0 + r) * ldd + c) = v;
        }
      } else {
        for (int e = tid; e < rows * op.N; e += kThreads) {
          const int r = e / op.N, c = e % op.N;
          const float v = tile[r * ldt + c];
          dst[(int64_t)(m0 + r) * ldd + c] = relu ? fmaxf(v, 0.f) : v;
        }
      }
    }
    tc_fence_before();
    __syncthreads();
    if (first_item) trace(28);
  }
  if (ASYNC && worker) cp_wait_dyn(0);
  if (!worker) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols);
  }
  trace(29);
  cta_mark(1);
  MQ_TL_END(MODE);
}

// fixed-order split reduction + layer epilogue (same decomposition as the GEMM)
template <class Epi>
__global__ void tc_reduce_kernel(const float* __restrict__ part, const int32_t* m_dev, int m_static,
                                 const int32_t* k_dev, int k_static, int N, int grid_gemm, Epi epi,
                                 bool direct) {
  MQ_PDL_ENTRY();
  const int M = m_dev ? *m_dev : m_static;
  const int K = k_dev ? *k_dev : k_static;
  const Work wk = choose_work(M, K, grid_gemm);
  if (direct && wk.S == 1) return;  // the GEMM wrote the result (op.out)
  const int64_t total = (int64_t)M * N;
  const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < M; i += gridDim.x * wpb)  // warp per row
    for (int j = lane; j < N; j += 32) epi(i, j, fixed_order_sum(part + (int64_t)i * N + j, total, wk.S));
}


// ============================================================================
// v2: TMA-fed, warp-specialised 3xTF32 GEMM (all five modes).
//
// Operand tiles arrive by TMA (cp.async.bulk.tensor, 128-byte swizzle) as
// they are stored: K-major row blocks (FWD / FCAT / DX A, DX B) or 32 x 32
// MN-major blocks (W / G / dh columns, and X^T for the weight gradients).
// Converter warps split each landed tile into hi = tf32_rn(x) and
// lo = tf32_rn(x - hi).  A goes to TENSOR MEMORY (tcgen05.st; each thread one
// tile row, the MMA reads A from TMEM), so the shared-memory port carries only
// the TMA writes, one read of A and the B traffic -- staging A hi / lo in
// smem and reading it three times per k block made the converters, not the
// tensor core, the bound.  B stays in smem, K-major with a 128-byte swizzle:
// MN-major tiles are transposed through registers (a probe of kind::tf32 with
// MN-major descriptors returned zeros on this part), DX's K-major W rows are
// split in place.  The MMA warp issues the 3 x 4 tcgen05.mma per 32-wide k
// block; epilogue warps drain a double-buffered TMEM accumulator while the
// next tile's MMAs run.  Roles (448 threads):
//   warp 0        TMA producer (one lane)
//   warps 1..8    converters (256 threads)
//   warp 9        TMEM owner + MMA issuer (one lane)
//   warps 10..13  epilogue (TMEM lane quarter = warp % 4)
// Pipelines: full[s] (TMA bytes) -> conv[s] (8 converter warps) -> MMA ->
// empty[s] (tcgen05.commit) back to the producer; accf[b] / acce[b] between
// the MMA warp and the epilogue per accumulator buffer.
// Work split (split-K over k blocks, S from the live M / K as in v1) with a
// CTA keeping ONE split for all its tiles: CTA b -> split b % S, tiles
// b / S, b / S + G, ... (G = grid / S).  The numerics equal v1's (same hi/lo
// split, same MMA order per k block); the aggregate-first modes run over a
// padded concat (each K / M half rounded up to 32) so TMA boxes never
// straddle the two sources.
struct Maps {
  CUtensorMap a, a2, b, b2;
};

struct Geo {
  int kbA;     // FCAT / DX: k blocks of the first K source (ceil(d / 32))
  int p1;      // DCAT: padded rows of the agg half of the output (ceil32(d_in))
  int nf = 0;  // DW: feature columns per tile (the MMA N of the swapped product)
};

__host__ __device__ constexpr bool a_mn(int mode) { return mode == kDw || mode == kDwCat; }
__host__ __device__ constexpr bool b_mn(int mode) { return mode != kDx; }

__host__ __device__ inline Work work2(int mode, const Geo& g, int M, int K, int grid) {
  Work w;
  const int mpad = mode == kDwCat ? 2 * g.p1 : M;
  const int nkb = (mode == kFwdCat || mode == kDx) ? 2 * g.kbA : (K > 0 ? (K + BK - 1) / BK : 0);
  w.tiles_m = (mpad + BM - 1) / BM;
  if (w.tiles_m < 1) w.tiles_m = 1;
  int S = (grid + w.tiles_m - 1) / w.tiles_m;
  if (S > nkb) S = nkb;
  if (S > kMaxSplitsTc) S = kMaxSplitsTc;
  if (S < 1) S = 1;
  w.kb_per = nkb > 0 ? (nkb + S - 1) / S : 0;
  w.S = nkb > 0 ? (nkb + w.kb_per - 1) / w.kb_per : 1;
  return w;
}

constexpr int kThreads2 = 448;
constexpr int kMaxN2 = 128;                      // v2 covers N <= 128 (wider: v1)
constexpr int kMaxBChunks = kMaxN2 * 8 / 128;  // B chunks per converter thread (group of 128)
constexpr int kConvThreads = 256;
constexpr int kConvGroups = 2;  // converter groups of 4 warps (alternate k blocks)
constexpr int kMaxStages2 = 8;

__host__ __device__ inline int b_tile_bytes(int mode, int Np) {
  return b_mn(mode) ? 4096 * ((Np + 31) / 32) : 128 * Np;
}
// FWD / FCAT run transposed ("swapped"): Y^T = W^T X^T, so the weights are
// the TMEM operand (A' = W^T: 32 scalar reads down a W column per thread, no
// smem transpose) and the sampled rows the smem operand (B' = X rows, K-major
// straight from TMA, split in place); the accumulator is features x rows.
// The weight gradient P = X^T G runs swapped too (P^T = G^T X): G's columns
// go to TMEM by scalar reads, X^T (d_in <= 128 features) is the transposed
// smem operand -- half the transposition of the unswapped order at 2 d_out =
// 128 > d_in.
__host__ __device__ constexpr bool swapped(int mode) {
  return mode == kFwd || mode == kFwdCat || mode == kDw;
}
__host__ __device__ inline int stage2_bytes(int mode, int Np) {
  if (swapped(mode)) return b_tile_bytes(mode, Np) + 2 * 16384;  // W raw + X hi / lo
  return 16384 + (mode == kDwCat ? 3 : 2) * b_tile_bytes(mode, Np);  // raw A + B hi/lo (+ mask)
}
// TMEM columns: accumulators 2 x cstride, then per stage A hi (32) | A lo (32)
__host__ __device__ inline int tmem_cstride(int mode, int Np) {
  return swapped(mode) ? BM : (Np + 31) / 32 * 32;
}
__host__ __device__ inline int max_stages_tmem(int mode, int Np) {
  return (512 - 2 * tmem_cstride(mode, Np)) / 64;
}

// D[tmem] (+)= A[tmem] . B[smem], kind::tf32 (A: 128 lanes x 8 columns per K = 8)
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// 32 lanes x 32 consecutive 32-bit columns (two x16 stores)
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]);
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  tmem_st16(taddr, *reinterpret_cast<const float(*)[16]>(&v[0]));
  tmem_st16(taddr + 16, *reinterpret_cast<const float(*)[16]>(&v[16]));
}
// 32 lanes x 16 consecutive 32-bit columns from 16 registers per thread
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                      uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// 128-byte-swizzle K-major UMMA descriptor: 8-row groups 1024 B apart (SBO);
// a K = 8 step advances the start by 32 B inside the swizzle atom.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr, uint32_t lbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

// Cooperative split reduction (deferred FWD / DW, S > 1): after a tile's S
// split CTAs have stored their partials, each of them sums a 1/S row slice of
// the tile over the S partials (fixed order p = 0..S-1, as fixed_order_sum)
// and writes it into partial slot 0, and the kernel publishes nparts = 1: the
// consumer (aggregation / optimizer) then reads ONE copy instead of S.  The S
// CTAs of a tile meet on a per-tile arrival counter (all CTAs of the
// persistent grid are co-resident: one per SM); the last to finish resets it.
// coop[2 t] = arrivals, coop[2 t + 1] = departures; zero at rest.
__device__ __forceinline__ int ld_acquire_gpu(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void coop_reduce_tile(float* __restrict__ part, int32_t* __restrict__ coop,
                                                 int t, int s, int S, int Mout, int N, int etid) {
  asm volatile("bar.sync 3, 128;" ::: "memory");  // the 4 epilogue warps stored this tile
  if (etid == 0) {
    __threadfence();
    atomicAdd(&coop[2 * t], 1);
    while (ld_acquire_gpu(&coop[2 * t]) < S) __nanosleep(40);
    __threadfence();
  }
  asm volatile("bar.sync 3, 128;" ::: "memory");
  const int r0 = t * BM, nr = min(BM, Mout - r0);
  const int lo = r0 + (s * nr) / S, hi = r0 + ((s + 1) * nr) / S;
  const int64_t stride = (int64_t)Mout * N;
  if ((N & 3) == 0) {
    const int n4 = N >> 2;
    for (int e = etid; e < (hi - lo) * n4; e += 128) {
      const int64_t o = (int64_t)(lo + e / n4) * N + 4 * (e % n4);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      int p = 0;
      for (; p + 8 <= S; p += 8) {
        float4 x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = __ldcg(reinterpret_cast<const float4*>(part + (p + u) * stride + o));
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          v.x += x[u].x;
          v.y += x[u].y;
          v.z += x[u].z;
          v.w += x[u].w;
        }
      }
      for (; p < S; ++p) {
        const float4 x = __ldcg(reinterpret_cast<const float4*>(part + p * stride + o));
        v.x += x.x;
        v.y += x.y;
        v.z += x.z;
        v.w += x.w;
      }
      *reinterpret_cast<float4*>(part + o) = v;
    }
  } else {
    for (int e = etid; e < (hi - lo) * N; e += 128) {
      const int64_t o = (int64_t)(lo + e / N) * N + e % N;
      part[o] = fixed_order_sum(part + o, stride, S);
    }
  }
  asm volatile("bar.sync 3, 128;" ::: "memory");
  if (etid == 0) {
    __threadfence();
    if (atomicAdd(&coop[2 * t + 1], 1) == S - 1) {
      coop[2 * t + 1] = 0;
      atomicExch(&coop[2 * t], 0);
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads2, 1)
    tc2_kernel(const __grid_constant__ Maps maps, Operands op, Geo geo, const int32_t* m_dev,
               int m_static, const int32_t* k_dev, int k_static, float* __restrict__ part,
               int32_t* __restrict__ nparts_out, int ST, int32_t* __restrict__ coop,
               int stage_on) {
  pdl_trigger();
  MQ_TL_BEGIN(MODE);
  if (threadIdx.x == 0) trace_at(0);
  if (threadIdx.x == 0) {  // the descriptors are kernel parameters: fetch them
    // while the barriers / TMEM are set up and the predecessor drains
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.a2)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.b)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.b2)) : "memory");
  }
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps LDS / STS
  __shared__ __align__(8) uint64_t full[kMaxStages2], conv[kMaxStages2], empty[kMaxStages2];
  __shared__ __align__(8) uint64_t accf[2], acce[2];
  __shared__ uint32_t s_tmem;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int M = m_dev ? *m_dev : m_static;
  const int K = k_dev ? *k_dev : k_static;
  const int Np = op.Np;
  const Work wk = work2(MODE, geo, M, K, gridDim.x);
  // the S partials of a tile are summed in place (coop_reduce_tile)
  const bool coop_on = coop != nullptr && wk.S > 1 && swapped(MODE);
  // published after the wait (see tc_gemm_kernel): the previous window's
  // optimizer may still read this counter when the grid starts
  auto publish_nparts = [&]() {
    if (nparts_out != nullptr && blockIdx.x == 0 && tid == 0) *nparts_out = coop_on ? 1 : wk.S;
  };
  const int G = (int)gridDim.x / wk.S;  // CTAs per split
  const int b = blockIdx.x;
  if (M <= 0 || b >= G * wk.S) {
    pdl_wait();
    publish_nparts();
    return;
  }
  const int s = b % wk.S;
  const int nkb = (MODE == kFwdCat || MODE == kDx) ? 2 * geo.kbA : (K + BK - 1) / BK;
  const int kb0 = s * wk.kb_per, kb1 = min(nkb, kb0 + wk.kb_per);
  const int Mout = MODE == kDwCat ? 2 * op.d_in : M;  // rows of the stored result
  float* dst = (wk.S == 1 && op.out) ? op.out : part + (int64_t)s * Mout * op.N;
  const int ldd = (wk.S == 1 && op.out) ? op.ldo : op.N;
  const bool relu = wk.S == 1 && op.out && op.relu;

  if (kb0 >= kb1) {  // K == 0: the partial is zero
    pdl_wait();
    publish_nparts();
    for (int t = b / wk.S; t < wk.tiles_m; t += G)
      for (int e = tid; e < BM * op.N; e += kThreads2) {
        const int r = t * BM + e / op.N;
        if (r < Mout) dst[(int64_t)r * ldd + e % op.N] = 0.f;
      }
    return;
  }

  constexpr bool SW = swapped(MODE);
  const int cstride = tmem_cstride(MODE, Np);
  const uint32_t tmem_cols = 512;  // accumulators + the A operand stages (one CTA per SM)
  if (warp == 9) tmem_alloc(&s_tmem, tmem_cols);
  if (tid == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&conv[i], 4);  // the 4 warps of the converter group
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&accf[i], 1);
      mbar_init(&acce[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  publish_nparts();
  const uint32_t tmem = s_tmem;
  const int BB = b_tile_bytes(MODE, Np);
  const int SB = stage2_bytes(MODE, Np);
  const uint32_t sbase = smem_u32(smem);
  // smem stage: [A raw 16K | B hi | B lo | (DCAT) act mask]; A hi / lo go to TMEM
  // swapped (FWD / FCAT): [W raw (BB) | X hi 16K | X lo 16K]; W^T hi / lo go to TMEM
  const int t_first = b / wk.S;
  if (tid == 0) trace_at(1);

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const int nbox_b = (Np + 31) / 32;
      uint32_t it = 0;
      for (int t = t_first; t < wk.tiles_m; t += G) {
        const int m0 = t * BM;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int st = it % ST;
          if (it >= (uint32_t)ST) mbar_wait(&empty[st], ((it / ST) - 1) & 1);
          if (it < 8) trace_at(2 + (int)it);
          mbar_expect_tx(&full[st], 16384u + (uint32_t)BB * (MODE == kDwCat ? 2u : 1u));
          // (swapped: the X rows land at sa, the W boxes at sb)
          const uint32_t sa = SW ? sbase + st * SB + BB : sbase + st * SB;
          const uint32_t sb = SW ? sbase + st * SB : sa + 16384, sm = sb + 2 * BB;
          // ---- A
          if (MODE == kFwd) {
            tma2d(sa, &maps.a, kb * BK, m0, &full[st]);
          } else if (MODE == kFwdCat || MODE == kDx) {
            if (kb < geo.kbA) tma2d(sa, &maps.a, kb * BK, m0, &full[st]);
            else tma2d(sa, &maps.a2, (kb - geo.kbA) * BK, m0, &full[st]);
          } else if (MODE == kDw) {
            for (int j = 0; j < 4; ++j) tma2d(sa + 4096 * j, &maps.a, m0 + 32 * j, kb * BK, &full[st]);
          } else {  // kDwCat: padded rows [agg | h]
            for (int j = 0; j < 4; ++j) {
              const int m = m0 + 32 * j;
              if (m < geo.p1) tma2d(sa + 4096 * j, &maps.a, m, kb * BK, &full[st]);
              else tma2d(sa + 4096 * j, &maps.a2, m - geo.p1, kb * BK, &full[st]);
            }
          }
          // ---- B
          if (MODE == kFwd) {  // box j: 32 columns of W_top (n < h) or W_bot (N may be h alone)
            for (int j = 0; j < nbox_b; ++j) {
              const int n0 = 32 * j;
              if (n0 < op.n_half) tma2d(sb + 4096 * j, &maps.b, n0, kb * BK, &full[st]);
              else tma2d(sb + 4096 * j, &maps.b, n0 - op.n_half, op.d_in + kb * BK, &full[st]);
            }
          } else if (MODE == kFwdCat) {
            const int row = kb < geo.kbA ? kb * BK : op.d_in + (kb - geo.kbA) * BK;
            for (int j = 0; j < nbox_b; ++j) tma2d(sb + 4096 * j, &maps.b, 32 * j, row, &full[st]);
          } else if (MODE == kDx) {
            if (kb < geo.kbA) tma2d(sb, &maps.b, kb * BK, 0, &full[st]);
            else tma2d(sb, &maps.b, (kb - geo.kbA) * BK, op.wd_in, &full[st]);
          } else {
            for (int j = 0; j < nbox_b; ++j) {
              tma2d(sb + 4096 * j, &maps.b, 32 * j, kb * BK, &full[st]);
              if (MODE == kDwCat) tma2d(sm + 4096 * j, &maps.b2, 32 * j, kb * BK, &full[st]);
            }
          }
        }
      }
    }
  } else if (warp <= 8) {
    // ------------------------------------------------------------ converters
    // kConvGroups groups of 4 warps take alternate k blocks, so the
    // latency chain of one block (TMA wait, LDS, TMEM store, B transpose,
    // fences) overlaps the next block's
    const int g = (warp - 1) >> 2;
    const int gt = tid - 32 - 128 * g;  // 0..127 within the group
    const int q = warp & 3;             // TMEM lane quarter of this warp
    const int m = 32 * q + lane;        // the A tile row this thread splits
    // B transposition items of this thread: chunk (row n, k4) for item gt + 128 i
    const int Nt = MODE == kDw ? geo.nf : Np;  // rows of the transposed smem operand
    const int nit = (Nt * 8 - gt + 127) / 128;  // items this thread owns (<= kMaxBChunks)
    int cn[kMaxBChunks], ck[kMaxBChunks];
    {
      const int q128 = 128 / Nt, r128 = 128 % Nt;
      int n = gt % Nt, k4 = gt / Nt;
#pragma unroll
      for (int i = 0; i < kMaxBChunks; ++i) {
        cn[i] = n;
        ck[i] = k4;
        n += r128;
        k4 += q128;
        if (n >= Nt) {
          n -= Nt;
          ++k4;
        }
      }
    }
    // MN-major 32 x 32 boxes at `raw` -> K-major 128-byte-swizzled rows (hi over
    // the raw tile, lo at raw + lo_off): four 32-bit reads down the tile per
    // 16-byte chunk (consecutive lanes = consecutive rows: conflict-free), all
    // reads issued first, the converter group synced, then swizzled stores
    auto transpose_mn = [&](uint8_t* raw, int lo_off, const uint8_t* mask, int krow0) {
      float rvv[kMaxBChunks][4];
#pragma unroll
      for (int i = 0; i < kMaxBChunks; ++i) {
        const int n = i < nit ? cn[i] : cn[0], k4 = i < nit ? ck[i] : ck[0];
        const int base = (n >> 5) * 4096 + (n & 3) * 4, c = (n & 31) >> 2;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = 4 * k4 + u;
          rvv[i][u] = *reinterpret_cast<const float*>(raw + base + k * 128 + ((c ^ (k & 7)) << 4));
        }
      }
      if (mask != nullptr) {  // DCAT: dz = dh * (act > 0)
#pragma unroll
        for (int i = 0; i < kMaxBChunks; ++i) {
          const int n = i < nit ? cn[i] : cn[0], k4 = i < nit ? ck[i] : ck[0];
          const int base = (n >> 5) * 4096 + (n & 3) * 4, c = (n & 31) >> 2;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int k = 4 * k4 + u;
            if (!(*reinterpret_cast<const float*>(mask + base + k * 128 + ((c ^ (k & 7)) << 4)) > 0.f))
              rvv[i][u] = 0.f;
          }
        }
      }
      if (a_mn(MODE) && krow0 + BK > K) {  // the last k block: rows past the live K
#pragma unroll
        for (int i = 0; i < kMaxBChunks; ++i)
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (krow0 + 4 * ck[i] + u >= K) rvv[i][u] = 0.f;
      }
      asm volatile("bar.sync %0, 128;" ::"r"(1 + g));
#pragma unroll
      for (int i = 0; i < kMaxBChunks; ++i) {
        if (i < nit) {
          const int n = cn[i], k4 = ck[i];
          const uint32_t o = (uint32_t)n * 128u + (uint32_t)((k4 ^ (n & 7)) << 4);
          float4 hi, lo;
          split4f(make_float4(rvv[i][0], rvv[i][1], rvv[i][2], rvv[i][3]), hi, lo);
          *reinterpret_cast<float4*>(raw + o) = hi;
          *reinterpret_cast<float4*>(raw + lo_off + o) = lo;
        }
      }
    };
    uint32_t it = 0;
    for (int t = t_first; t < wk.tiles_m; t += G) {
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        if ((int)(it % kConvGroups) != g) continue;
        const int st = it % ST;
        mbar_wait(&full[st], (it / ST) & 1);
        if (gt == 0 && it < 8) trace_at(10 + (int)it);
        const int krow0 = kb * BK;
        if (SW) {
          uint8_t* sw = smem + st * SB;  // W boxes (MN-major, 32 features x 32 k each)
          uint8_t* sx = sw + BB;         // X rows (K-major), split in place
          // ---- A' = W^T -> TMEM: thread = feature n = 32 q + lane, its 32 k
          {
            float hi[32], lo[32];
            const bool live = 32 * q < Np;  // warp-uniform: features past Np stay zero
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              float v = live ? *reinterpret_cast<const float*>(
                  sw + q * 4096 + k * 128 + ((((lane >> 2) ^ (k & 7)) << 4) | ((lane & 3) << 2))) : 0.f;
              if (MODE == kDw && krow0 + k >= K) v = 0.f;  // rows past the live K
              hi[k] = tf32_hi(v);
              lo[k] = v - hi[k];
            }
            const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(2 * cstride + 64 * st);
            tmem_st32(ta, hi);
            tmem_st32(ta + 32, lo);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          }
          if (gt == 0 && it == 1) trace_at(33);
          if (MODE == kDw) {  // ---- B' = X^T (feature boxes): transposed
            transpose_mn(sx, 16384, nullptr, krow0);
          } else {  // ---- B' = X rows: in-place hi, lo beside (elementwise, conflict-free)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int o = (gt + 128 * i) * 16;
              float4 hi, lo;
              split4f(*reinterpret_cast<const float4*>(sx + o), hi, lo);
              *reinterpret_cast<float4*>(sx + o) = hi;
              *reinterpret_cast<float4*>(sx + 16384 + o) = lo;
            }
          }
          if (gt == 0 && it == 1) trace_at(36);
          tc_fence_before();
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&conv[st]);
          if (gt == 0 && it < 2) trace_at(30 + (int)it);
          continue;
        }
        uint8_t* sa = smem + st * SB;
        uint8_t* sb = sa + 16384;
        // ---- A -> TMEM: thread = tile row m, all 32 k (two halves of 16),
        // split hi / lo into the stage's 32 + 32 TMEM columns (the MMA reads A
        // from TMEM)
        {
          const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(2 * cstride + 64 * st);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            float hi[16], lo[16];
            if (!a_mn(MODE)) {  // K-major rows (128-byte swizzle: chunk c at c ^ (m & 7))
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4) {
                const int c = 4 * hh + c4;
                float4 h4, l4;
                split4f(*reinterpret_cast<const float4*>(sa + m * 128 + ((c ^ (m & 7)) << 4)), h4, l4);
                hi[4 * c4] = h4.x; hi[4 * c4 + 1] = h4.y; hi[4 * c4 + 2] = h4.z; hi[4 * c4 + 3] = h4.w;
                lo[4 * c4] = l4.x; lo[4 * c4 + 1] = l4.y; lo[4 * c4 + 2] = l4.z; lo[4 * c4 + 3] = l4.w;
              }
            } else {  // MN-major 32 x 32 box q: k row at k * 128, chunk (m % 32) / 4 at ^ (k & 7)
#pragma unroll
              for (int kk = 0; kk < 16; ++kk) {
                const int k = 16 * hh + kk;
                float v = *reinterpret_cast<const float*>(
                    sa + q * 4096 + k * 128 + ((((lane >> 2) ^ (k & 7)) << 4) | ((lane & 3) << 2)));
                if (krow0 + k >= K) v = 0.f;
                hi[kk] = tf32_hi(v);
                lo[kk] = v - hi[kk];
              }
            }
            tmem_st16(ta + 16 * hh, hi);
            tmem_st16(ta + 32 + 16 * hh, lo);
          }
          if (gt == 0 && it == 1) trace_at(32);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          if (gt == 0 && it == 1) trace_at(33);
        }
        // ---- B (smem): MN-major tiles transposed to K-major through
        // registers (read, sync the group, write hi over the raw tile and lo
        // beside it); DX's W rows are K-major already
        if (b_mn(MODE)) {
          transpose_mn(sb, BB, MODE == kDwCat ? sb + 2 * BB : nullptr, krow0);
          if (gt == 0 && it == 1) trace_at(36);
        } else {
          for (int o = gt * 16; o < BB; o += 128 * 16) {
            float4 hi, lo;
            split4f(*reinterpret_cast<const float4*>(sb + o), hi, lo);
            *reinterpret_cast<float4*>(sb + o) = hi;
            *reinterpret_cast<float4*>(sb + BB + o) = lo;
          }
        }
        tc_fence_before();
        fence_async_smem();
        __syncwarp();
        if (gt == 0 && it == 1) trace_at(37);
        if (lane == 0) mbar_arrive(&conv[st]);
        if (gt == 0 && it < 2) trace_at(30 + (int)it);
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      // both operands K-major; swapped: N = the 128-row tile of X
      const uint32_t idesc = instr_desc(SW ? (MODE == kDw ? geo.nf : BM) : Np, false, false);
      uint32_t it = 0, ti = 0;
      for (int t = t_first; t < wk.tiles_m; t += G, ++ti) {
        const uint32_t ab = ti & 1;
        if (ti >= 2) mbar_wait(&acce[ab], ((ti >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + ab * (uint32_t)cstride;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int st = it % ST;
          mbar_wait(&conv[st], (it / ST) & 1);
          if (it < 8) trace_at(18 + (int)it);
          tc_fence_after();
          const uint32_t a_hi = tmem + (uint32_t)(2 * cstride + 64 * st), a_lo = a_hi + 32;
          const uint32_t b_hi = SW ? sbase + st * SB + BB : sbase + st * SB + 16384;
          const uint32_t b_lo = b_hi + (SW ? 16384 : BB);
#pragma unroll
          for (int j = 0; j < BK / 8; ++j) {
            const uint32_t ko = 32u * j;  // K = 8 step inside the 128-byte swizzle atom
            const uint64_t dbh = sw128_desc(b_hi + ko, 16), dbl = sw128_desc(b_lo + ko, 16);
            const uint32_t acc = (kb == kb0 && j == 0) ? 0u : 1u;
            mma_tf32_ts(d, a_lo + 8 * j, dbh, idesc, acc);  // small terms first (as v1)
            mma_tf32_ts(d, a_hi + 8 * j, dbl, idesc, 1u);
            mma_tf32_ts(d, a_hi + 8 * j, dbh, idesc, 1u);
          }
          mma_commit(&empty[st]);
        }
        mma_commit(&accf[ab]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quarter
    const int etid = tid - 320;  // 0..127 over the four epilogue warps
    uint32_t ti = 0;
    const bool vec = (op.N & 3) == 0 && (ldd & 3) == 0 && ((uintptr_t)dst & 15) == 0;
    // swapped modes storing whole rows (partial tiles, or an output whose
    // pitch is N): each 32-row chunk goes TMEM -> registers -> a shared
    // staging buffer (double-buffered, conflict-free: lanes are consecutive
    // features) -> ONE bulk async copy of its contiguous rows.  The
    // per-thread 4-byte global stores this replaces were bound by the SM's
    // store path (~0.9 us per 16 KB chunk with all CTAs storing).
    // (only CTAs that loop over several tiles: there the next tile's MMAs
    // overlap the copies; a one-tile split-K CTA measured no gain in-step)
    // staging: the reserved area (stage_on & 3), or -- for a CTA's LAST tile,
    // whose MMAs have consumed every pipeline stage (stage_on & 4) -- the
    // pipeline's own stage memory, so no extra shared memory is reserved
    const bool bulk_ok = SW && ldd == op.N && vec;
    const bool bulk_res = bulk_ok && (stage_on & 3) && ((stage_on & 3) > 1 || wk.tiles_m > G);
    const bool bulk_last = bulk_ok && (stage_on & 4);
    int chunk = 0;
    for (int t = t_first; t < wk.tiles_m; t += G, ++ti) {
      const uint32_t ab = ti & 1;
      mbar_wait(&accf[ab], (ti >> 1) & 1);
      if (warp == 10 && lane == 0 && ti < 2) trace_at(26 + 2 * (int)ti);
      tc_fence_after();
      const bool bulk = bulk_res || (bulk_last && t + G >= wk.tiles_m);
      float* stage = reinterpret_cast<float*>(bulk_res ? smem + ST * SB : smem);
      if (bulk) {
        const int n = q * 32 + lane;
        for (int cb = 0; cb < BM; cb += 32) {
          const int r0 = t * BM + cb;
          const int nr = min(32, M - r0);
          // chunks past the last row issue no copy and must not take a
          // buffer turn: the read-wait below lets the most recent copy run
          // on, which must be the OTHER buffer's
          if (nr <= 0) continue;
          float v[32];
          tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + ab * (uint32_t)cstride + (uint32_t)cb, v);
          float* sb = stage + (chunk & 1) * (32 * op.N);
          ++chunk;
          // the copy that read this buffer two chunks ago has finished reading
          if (etid == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          asm volatile("bar.sync 3, 128;" ::: "memory");
          if (n < op.N) {
#pragma unroll
            for (int u = 0; u < 32; ++u) sb[u * op.N + n] = relu ? fmaxf(v[u], 0.f) : v[u];
          }
          fence_async_smem();
          asm volatile("bar.sync 3, 128;" ::: "memory");
          if (etid == 0) {
            asm volatile(
                "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                "cp.async.bulk.commit_group;" ::"l"(dst + (int64_t)r0 * ldd),
                "r"(smem_u32(sb)), "r"((uint32_t)(nr * op.N * 4))
                : "memory");
          }
        }
        tc_fence_before();
        __syncwarp();
        if (warp == 10 && lane == 0 && ti < 1) trace_at(27);
        if (lane == 0) mbar_arrive(&acce[ab]);
        if (coop_on) coop_reduce_tile(part, coop, t, s, wk.S, Mout, op.N, tid - 320);
        continue;
      }
      if (SW) {  // TMEM lane = output feature n, column = row of the tile
        const int n = q * 32 + lane;
        if (32 * q < op.N) {  // warp-uniform
          for (int cb = 0; cb < BM; cb += 32) {
            float v[32];
            tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + ab * (uint32_t)cstride + (uint32_t)cb, v);
            const int r0 = t * BM + cb;
            if (n < op.N) {
#pragma unroll
              for (int u = 0; u < 32; ++u)
                if (r0 + u < M) dst[(int64_t)(r0 + u) * ldd + n] = relu ? fmaxf(v[u], 0.f) : v[u];
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (warp == 10 && lane == 0 && ti < 1) trace_at(27);
        if (lane == 0) mbar_arrive(&acce[ab]);
        if (coop_on) coop_reduce_tile(part, coop, t, s, wk.S, Mout, op.N, tid - 320);
        continue;
      }
      const int p = t * BM + q * 32 + lane;  // row in the (padded) M space
      int r = p;
      if (MODE == kDwCat) r = p < geo.p1 ? (p < op.d_in ? p : -1)
                                         : (p - geo.p1 < op.d_in ? op.d_in + p - geo.p1 : -1);
      const bool ok = r >= 0 && r < Mout;
      float* row = dst + (int64_t)(ok ? r : 0) * ldd;
      for (int cb = 0; cb < Np; cb += 32) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + ab * (uint32_t)cstride + (uint32_t)cb, v);
        if (!ok) continue;
        if (relu) {
#pragma unroll
          for (int u = 0; u < 32; ++u) v[u] = fmaxf(v[u], 0.f);
        }
        if (vec && cb + 32 <= op.N) {
#pragma unroll
          for (int u = 0; u < 32; u += 4)
            *reinterpret_cast<float4*>(row + cb + u) = make_float4(v[u], v[u + 1], v[u + 2], v[u + 3]);
        } else {
#pragma unroll
          for (int u = 0; u < 32; ++u)
            if (cb + u < op.N) row[cb + u] = v[u];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (warp == 10 && lane == 0 && ti < 1) trace_at(27);
      if (lane == 0) mbar_arrive(&acce[ab]);
    }
  }
  // the bulk copies' global writes, complete and ordered for the generic
  // proxy before the grid signals completion (a programmatic dependent
  // launch reads them right after its griddepcontrol.wait)
  if (tid == 320) {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc(tmem, tmem_cols);
  }
  if (tid == 0) trace_at(29);
  MQ_TL_END(MODE);
}

template <class Epi>
__global__ void tc2_reduce_kernel(const float* __restrict__ part, int mode, Geo geo,
                                  const int32_t* m_dev, int m_static, const int32_t* k_dev,
                                  int k_static, int N, int grid_gemm, Epi epi, bool direct) {
  MQ_PDL_ENTRY();
  const int M = m_dev ? *m_dev : m_static;
  const int K = k_dev ? *k_dev : k_static;
  const Work wk = work2(mode, geo, M, K, grid_gemm);
  if (direct && wk.S == 1) return;
  const int64_t total = (int64_t)M * N;
  const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < M; i += gridDim.x * wpb)
    for (int j = lane; j < N; j += 32) epi(i, j, fixed_order_sum(part + (int64_t)i * N + j, total, wk.S));
}

}  // namespace tc

// ------------------------------------------------------------ host side
static int g_gemm_backend = 1;  // 1 = tcgen05 3xTF32, 0 = fp32 FFMA split-K

static int g_tc_grid_cap = kNumSMs;  // experiments: fewer CTAs -> fewer, deeper splits

inline int tc_grid(int m_max, int k_max) {
  const int tiles = (m_max + tc::BM - 1) / tc::BM;
  const int nkb = (k_max + tc::BK - 1) / tc::BK;
  long long cap = (long long)(tiles < 1 ? 1 : tiles) *
                  (nkb < 1 ? 1 : (nkb > tc::kMaxSplitsTc ? tc::kMaxSplitsTc : nkb));
  return (int)(cap < g_tc_grid_cap ? cap : g_tc_grid_cap);
}

inline bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// the cp.async ring needs every operand row chunk 16-byte aligned
template <int MODE>
bool tc_async_ok(const tc::Operands& op) {
  if (!al16(op.x) || (op.ldx & 3)) return false;
  if (MODE == tc::kFwd) return al16(op.w) && (op.n_half & 3) == 0;
  if (MODE == tc::kDw) return al16(op.g) && (op.N & 3) == 0;
  if (MODE == tc::kDx) return al16(op.w) && (op.wd_out & 3) == 0;
  if (MODE == tc::kFwdCat)
    return al16(op.x2) && (op.ldx2 & 3) == 0 && (op.d_in & 3) == 0 && al16(op.w) && (op.N & 3) == 0;
  return al16(op.x2) && (op.ldx2 & 3) == 0 && (op.d_in & 3) == 0 && al16(op.g) &&
         (op.ldg & 3) == 0 && al16(op.act) && (op.ldact & 3) == 0 && (op.N & 3) == 0;
}

constexpr int kSmemBudget = 226 * 1024;  // 227 KB opt-in minus the static barriers

// ---- v2 launch: tensor maps over the operands, or -1 when a shape / pointer
// falls outside what the TMA path covers (then v1 runs)
static int g_tc_v2 = 2;  // 0: v1 everywhere, 2: TMA (DW by rule), 3: TMA for every mode

typedef CUresult (*PFN_tmapEncode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_tmapEncode tmap_encoder() {
  static PFN_tmapEncode fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_tmapEncode>(p);
  }
  return fn;
}

// row-major fp32 matrix (rows x cols, pitch ld floats), 128-byte swizzled boxes
static bool tmap2d(CUtensorMap* m, const float* base, int64_t cols, int64_t rows, int64_t ld,
                   int box_c, int box_r) {
  PFN_tmapEncode enc = tmap_encoder();
  if (!enc || !base || cols < 1 || rows < 1 || !al16(base) || (ld & 3) || ld < cols) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_c, (cuuint32_t)box_r};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline int64_t tc_part_floats_base(int64_t m_max, int64_t n);
static int g_tc_coop = -1;  // cooperative split reduction of the deferred FWD / DW (MQ_TC2_COOP)
// bulk (async-copy engine) epilogue stores of the swapped modes, MQ_TC2_BULK bits:
//   8  a CTA's last tile stages through the pipeline's own stage memory
//      (default: Reddit 54.4 -> 49.4 us/step, products 429 -> 421 us/step)
//   1  FWD: a reserved 32 KB staging area for every tile of many-tile CTAs
//   2  the same for DW;  4  reserve it whatever the tile count
// (bits 1/2/4 cost more than they save in-step: the larger shared-memory
// footprint alone slowed the Reddit step ~4 us and products ~3 %)
static const int g_tc_bulk = getenv("MQ_TC2_BULK") ? atoi(getenv("MQ_TC2_BULK")) : 8;

template <int MODE, class Epi>
int run_tc2(const tc::Operands& op, const int32_t* m_dev, int m_static, int m_max,
            const int32_t* k_dev, int k_static, int k_max, float* part, const Epi& epi,
            cudaStream_t s, int kid, int kid_red, bool skip_reduce, int32_t* nparts_out) {
  using namespace tc;
  if (g_tc_coop < 0) {
    const char* e = getenv("MQ_TC2_COOP");
    g_tc_coop = e ? atoi(e) : 0;
  }
  if (!g_tc_v2 || op.Np > kMaxN2) return -1;
  // DW (X^T G, both operands MN-major) runs swapped, transposing X^T.  In the
  // fused step (deferred partials) it wins at every width (Reddit's 602-d
  // layer: 12.6 -> 11.6 us); the materialising per-op call with d_in > 128
  // measures faster on v1 (21 vs 29 us with its split reduction)
  if (MODE == kDw && op.d_in > 128 && !skip_reduce && g_tc_v2 < 3) return -1;
  const int SB = stage2_bytes(MODE, op.Np);
  // swapped modes: an optional double-buffered 32-row staging area for the
  // bulk epilogue of every tile (MQ_TC2_BULK bits 1/2/4), reserved only
  // where CTAs loop over many tiles (a host-known row count above one tile
  // per CTA, or a short K that leaves the product unsplit)
  const bool many_tiles = (m_dev == nullptr && (m_static + BM - 1) / BM > kNumSMs) || k_max <= 256;
  const int stage_bytes =
      swapped(MODE) && (g_tc_bulk & (MODE == kDw ? 2 : 1)) && (many_tiles || (g_tc_bulk & 4))
          ? 2 * 32 * op.Np * 4
          : 0;
  int ST = (kSmemBudget - 1024 - stage_bytes) / SB;
  if (ST > kMaxStages2) ST = kMaxStages2;
  if (ST > max_stages_tmem(MODE, op.Np)) ST = max_stages_tmem(MODE, op.Np);
  {  // experiment knob: fewer stages = a smaller shared-memory footprint
    static const int cap_st = getenv("MQ_TC2_MAX_STAGES") ? atoi(getenv("MQ_TC2_MAX_STAGES")) : 0;
    if (cap_st >= 2 && ST > cap_st) ST = cap_st;
  }
  ST &= ~1;  // an odd stage count hung the products step (MQ_TC2_MAX_STAGES=3): even only
  if (ST < 2) return -1;
  Maps mp;
  Geo geo{0, 0};
  bool ok = false;
  const int mrows = m_max < 1 ? 1 : m_max, krows = k_max < 1 ? 1 : k_max;
  if (MODE == kFwd) {
    // W rows past d_in exist only when the bottom half is part of the product
    ok = op.n_half % 32 == 0 && tmap2d(&mp.a, op.x, op.d_in, mrows, op.ldx, 32, BM) &&
         tmap2d(&mp.b, op.w, op.n_half, (op.N > op.n_half ? 2 : 1) * op.d_in, op.n_half, 32, 32);
    mp.a2 = mp.a;
    mp.b2 = mp.b;
  } else if (MODE == kFwdCat) {
    geo.kbA = (op.d_in + BK - 1) / BK;
    ok = tmap2d(&mp.a, op.x, op.d_in, mrows, op.ldx, 32, BM) &&
         tmap2d(&mp.a2, op.x2, op.d_in, mrows, op.ldx2, 32, BM) &&
         tmap2d(&mp.b, op.w, op.N, 2 * op.d_in, op.N, 32, 32);
    mp.b2 = mp.b;
  } else if (MODE == kDx) {
    geo.kbA = (op.wd_out + BK - 1) / BK;
    ok = (op.wd_out & 3) == 0 && tmap2d(&mp.a, op.x, op.wd_out, mrows, 2 * op.wd_out, 32, BM) &&
         tmap2d(&mp.a2, op.x + op.wd_out, op.wd_out, mrows, 2 * op.wd_out, 32, BM) &&
         tmap2d(&mp.b, op.w, op.wd_out, 2 * op.wd_in, op.wd_out, 32, op.Np);
    mp.b2 = mp.b;
  } else if (MODE == kDw) {
    geo.nf = op.d_in >= 128 ? 128 : (op.d_in + 15) / 16 * 16;
    ok = tmap2d(&mp.a, op.x, op.d_in, krows, op.ldx, 32, 32) &&
         tmap2d(&mp.b, op.g, op.N, krows, op.N, 32, 32);
    mp.a2 = mp.a;
    mp.b2 = mp.b;
  } else {
    geo.p1 = (op.d_in + 31) / 32 * 32;
    ok = tmap2d(&mp.a, op.x, op.d_in, krows, op.ldx, 32, 32) &&
         tmap2d(&mp.a2, op.x2, op.d_in, krows, op.ldx2, 32, 32) &&
         tmap2d(&mp.b, op.g, op.N, krows, op.ldg, 32, 32) &&
         tmap2d(&mp.b2, op.act, op.N, krows, op.ldact, 32, 32);
  }
  if (!ok) return -1;
  static thread_local bool configured[5] = {};
  if (!configured[MODE]) {
    MQ_CUDA(cudaFuncSetAttribute(tc2_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSmemBudget));
    configured[MODE] = true;
  }
  int grid = tc_grid(m_max, k_max);
  {  // experiment knob: cap the v2 grid (fewer, deeper k splits -> less partial traffic)
    static const int cap2 = [] {
      const char* e = getenv("MQ_TC2_GRID_CAP");
      return e ? atoi(e) : 0;
    }();
    if (cap2 > 0 && grid > cap2) grid = cap2;
  }
  // deferred swapped products (FWD Y parts, DW parts): the split CTAs of a
  // tile sum their partials in place; counters live in the buffer's tail
  int32_t* coop = nullptr;
  const int64_t mrow = MODE == kDwCat ? 2 * ((m_max + 31) / 32 * 32) : (m_max < 1 ? 1 : m_max);
  if (g_tc_coop && skip_reduce && nparts_out != nullptr && swapped(MODE) &&
      (mrow + BM - 1) / BM <= kCoopTiles)
    coop = reinterpret_cast<int32_t*>(part + tc_part_floats_base(m_max, op.N));
  {
    ProfScope ps(kid, s);
    MQ_CUDA(launch_k(tc2_kernel<MODE>, dim3(grid), dim3(kThreads2),
                     (size_t)(ST * SB + 1024 + stage_bytes), s, mp, op, geo, m_dev, m_static, k_dev,
                     k_static, part, nparts_out, ST, coop,
                     (stage_bytes > 0 ? (g_tc_bulk & 4 ? 2 : 1) : 0) |
                         (swapped(MODE) && (g_tc_bulk & 8) ? 4 : 0)));
  }
  MQ_LAUNCH_CHECK("tc2_gemm");
  if (skip_reduce) return MQ_OK;
  int64_t mn = (int64_t)(m_max < 1 ? 1 : m_max) * op.N;
  int rb = ceil_div(mn, 256);
  if (rb > kNumSMs * 4) rb = kNumSMs * 4;
  {
    ProfScope ps(kid_red, s);
    MQ_CUDA(launch_k(tc2_reduce_kernel<Epi>, dim3(rb), dim3(256), 0, s, part, (int)MODE, geo, m_dev,
                     m_static, k_dev, k_static, op.N, grid, epi, op.out != nullptr));
  }
  MQ_LAUNCH_CHECK("tc2_reduce");
  return MQ_OK;
}

template <int MODE, class Epi>
int run_tc_gemm(const tc::Operands& op, const int32_t* m_dev, int m_static, int m_max,
                const int32_t* k_dev, int k_static, int k_max, float* part, const Epi& epi,
                cudaStream_t s, int kid, int kid_red, bool skip_reduce = false,
                int32_t* nparts_out = nullptr) {
  {
    const int r = run_tc2<MODE>(op, m_dev, m_static, m_max, k_dev, k_static, k_max, part, epi, s,
                                kid, kid_red, skip_reduce, nparts_out);
    if (r >= 0) return r;
  }
  static thread_local bool configured[5][2] = {};
  const int base = tc::Smem::total(op.Np);
  int R = (kSmemBudget - base) / tc::raw_bytes(MODE, op.Np);
  if (R > tc::kMaxRaw) R = tc::kMaxRaw;
  const bool async = R >= 2 && tc_async_ok<MODE>(op);
  const int smem = async ? base + R * tc::raw_bytes(MODE, op.Np) : base;
  if (!configured[MODE][async]) {
    if (async)
      MQ_CUDA(cudaFuncSetAttribute(tc::tc_gemm_kernel<MODE, true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
    else
      MQ_CUDA(cudaFuncSetAttribute(tc::tc_gemm_kernel<MODE, false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   tc::Smem::total(tc::kMaxN)));
    configured[MODE][async] = true;
  }
  const int grid = tc_grid(m_max, k_max);
  {
    ProfScope ps(kid, s);
    if (async)
      MQ_CUDA(launch_k(tc::tc_gemm_kernel<MODE, true>, dim3(grid), dim3(tc::kBlock), smem, s, op,
                       m_dev, m_static, k_dev, k_static, part, nparts_out, R));
    else
      MQ_CUDA(launch_k(tc::tc_gemm_kernel<MODE, false>, dim3(grid), dim3(tc::kBlock), smem, s,
                       op, m_dev, m_static, k_dev, k_static, part, nparts_out, 0));
  }
  MQ_LAUNCH_CHECK("tc_gemm");
  if (skip_reduce) return MQ_OK;
  int64_t mn = (int64_t)(m_max < 1 ? 1 : m_max) * op.N;
  int rb = ceil_div(mn, 256);
  if (rb > kNumSMs * 4) rb = kNumSMs * 4;
  {
    ProfScope ps(kid_red, s);
    MQ_CUDA(launch_k(tc::tc_reduce_kernel<Epi>, dim3(rb), dim3(256), 0, s, part, m_dev, m_static, k_dev, k_static, op.N, grid,
                                                 epi, op.out != nullptr));
  }
  MQ_LAUNCH_CHECK("tc_reduce");
  return MQ_OK;
}

// floats of partials the tc path may write for an (m_max x n) output: the
// device picks S <= ceil(grid / tiles_m), so S*M <= grid*BM + M.
inline int64_t tc_part_floats_base(int64_t m_max, int64_t n) {
  if (m_max < 1) m_max = 1;
  const int64_t a = (int64_t)tc::kMaxSplitsTc * m_max;
  const int64_t b = (int64_t)kNumSMs * tc::BM + m_max;
  return (a < b ? a : b) * n;
}
// + the cooperative reduction's per-tile counters (zeroed with the buffer,
// left at zero by every launch)
inline int64_t tc_part_floats(int64_t m_max, int64_t n) {
  return tc_part_floats_base(m_max, n) + 2 * tc::kCoopTiles;
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
  op.out = y;
  op.ldo = 2 * d_out;
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

// aggregate-first input layer: act = relu([agg | h] W) over the live dst rows
int tc_linear_af(const float* agg, int ldagg, const float* h, int ldh, const int32_t* m_dev,
                 int m_max, int d_in, const float* W, int d_out, float* act, int ldact,
                 float* part, cudaStream_t s) {
  tc::Operands op{agg, ldagg, d_in, W, d_out, nullptr, d_out, (d_out + 15) / 16 * 16};
  op.x2 = h;
  op.ldx2 = ldh;
  op.out = act;
  op.ldo = ldact;
  op.relu = 1;
  return run_tc_gemm<tc::kFwdCat>(op, m_dev, 0, m_max, nullptr, 2 * d_in, 2 * d_in, part,
                                  EpiLinearFwd{nullptr, 0, act, ldact}, s, K_SAGE_AF,
                                  K_SAGE_AF_REDUCE);
}

int64_t tc_af_part_floats(int64_t m_max, int64_t d_out) { return tc_part_floats(m_max, d_out); }

// y = h W (one d_in x d_out half of a SAGE weight), host-known rows
int tc_transform_half(const float* h, int ldh, int64_t n, int d_in, const float* W, int d_out,
                      float* y, int ldy, float* part, cudaStream_t s) {
  tc::Operands op{h, ldh, d_in, W, d_out, nullptr, d_out, (d_out + 15) / 16 * 16};
  op.out = y;
  op.ldo = ldy;
  return run_tc_gemm<tc::kFwd>(op, nullptr, (int)n, (int)n, nullptr, d_in, d_in, part,
                               EpiStore{y, ldy}, s, K_FULL_TRANSFORM, K_FULL_TRANSFORM_REDUCE);
}

// out = [relu] ([agg | hv] W) over m host-known rows (the lean evaluate's last layer)
int tc_linear_cat_rows(const float* agg, int ldagg, const float* hv, int ldhv, int m, int d_in,
                       const float* W, int d_out, float* out, int ldo, int relu, float* part,
                       cudaStream_t s) {
  tc::Operands op{agg, ldagg, d_in, W, d_out, nullptr, d_out, (d_out + 15) / 16 * 16};
  op.x2 = hv;
  op.ldx2 = ldhv;
  op.out = out;
  op.ldo = ldo;
  op.relu = relu;
  if (relu)
    return run_tc_gemm<tc::kFwdCat>(op, nullptr, m, m, nullptr, 2 * d_in, 2 * d_in, part,
                                    EpiLinearFwd{nullptr, 0, out, ldo}, s, K_FULL_TRANSFORM,
                                    K_FULL_TRANSFORM_REDUCE);
  return run_tc_gemm<tc::kFwdCat>(op, nullptr, m, m, nullptr, 2 * d_in, 2 * d_in, part,
                                  EpiStore{out, ldo}, s, K_FULL_TRANSFORM, K_FULL_TRANSFORM_REDUCE);
}

// its weight gradient as deferred split-K partials [S][2 d_in][d_out]
int tc_linear_af_bwd(const float* agg, int ldagg, const float* h, int ldh,
                     const int32_t* rows_dev, int rows_max, int d_in, const float* dh, int lddh,
                     const float* act, int ldact, int d_out, float* part, int32_t* nparts_out,
                     cudaStream_t s) {
  tc::Operands op{agg, ldagg, d_in, nullptr, d_out, dh, d_out, (d_out + 15) / 16 * 16};
  op.x2 = h;
  op.ldx2 = ldh;
  op.ldg = lddh;
  op.act = act;
  op.ldact = ldact;
  return run_tc_gemm<tc::kDwCat>(op, nullptr, 2 * d_in, 2 * d_in, rows_dev, 0, rows_max, part,
                                 EpiStore{nullptr, 0}, s, K_SAGE_AF_DW, K_SAGE_AF_DW, true,
                                 nparts_out);
}

int64_t tc_af_dw_part_floats(int64_t d_in, int64_t d_out) { return tc_part_floats(2 * d_in, d_out); }

// input gradient of a transform-first layer: dh = G [W_top | W_bot]^T over the
// live rows; a single split writes dh directly (no reduction pass)
int tc_dx(const float* g, const int32_t* m_dev, int m_max, int d_in, int d_out, const float* W,
          float* dh, int lddh, float* part, cudaStream_t s) {
  tc::Operands op{g, 2 * d_out, 2 * d_out, W, 0, nullptr, d_in, (d_in + 15) / 16 * 16};
  op.wd_in = d_in;
  op.wd_out = d_out;
  op.out = dh;
  op.ldo = lddh;
  return run_tc_gemm<tc::kDx>(op, m_dev, 0, m_max, nullptr, 2 * d_out, 2 * d_out, part,
                              EpiStore{dh, lddh}, s, K_SAGE_DH, K_SAGE_DH_REDUCE);
}

int64_t tc_scratch_floats(int64_t m_max, int64_t d_in, int64_t d_out) {
  int64_t a = tc_part_floats(m_max, 2 * d_out);
  int64_t b = tc_part_floats(d_in, 2 * d_out);
  int64_t c = tc_part_floats(m_max, d_in);  // dh (tc_dx)
  a = a > b ? a : b;
  return a > c ? a : c;
}

}  // namespace mq

extern "C" {

int mq_set_gemm_backend(int32_t backend) {
  MQ_CHECK_ARG(backend == 0 || backend == 1, "mq_set_gemm_backend: 0 (fp32 FFMA) or 1 (tcgen05)");
  g_gemm_backend = backend;
  return MQ_OK;
}

int mq_get_gemm_backend(void) { return g_gemm_backend; }

int mq_set_tc_kernel(int32_t version) {
  MQ_CHECK_ARG(version >= 1 && version <= 3,
               "mq_set_tc_kernel: 1 (cp.async staging), 2 (TMA; DW stays on 1) or 3 (TMA for all)");
  g_tc_v2 = version == 1 ? 0 : version;
  return MQ_OK;
}

int mq_get_tc_kernel(void) { return g_tc_v2 ? g_tc_v2 : 1; }

int mq_set_tc_grid_cap(int32_t cap) {
  MQ_CHECK_ARG(cap >= 1 && cap <= kNumSMs, "mq_set_tc_grid_cap: 1..%d", kNumSMs);
  g_tc_grid_cap = cap;
  return MQ_OK;
}

#ifdef MQ_TC_TRACE
int mq_debug_tc_cta(unsigned long long* out) {
  MQ_CUDA(cudaMemcpyFromSymbol(out, tc::g_tc_cta, sizeof(unsigned long long) * 512));
  return MQ_OK;
}

int mq_debug_tc_trace(unsigned long long* out) {
  MQ_CUDA(cudaMemcpyFromSymbol(out, tc::g_tc_trace, sizeof(unsigned long long) * 64));
  return MQ_OK;
}
#endif

}  // extern "C"

MQ_TL_READER(tc)
