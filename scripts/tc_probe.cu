// Standalone probe of tcgen05.mma kind::tf32 operand layouts (no-swizzle
// canonical layouts, K-major and MN-major).  Build and run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tc_probe scripts/tc_probe.cu && /tmp/tc_probe
// One CTA, one MMA (M=128, N=128, K=8) per variant; prints max error vs CPU.
// Result on B200 (2026-10-17): K-major A and B exact; any MN-major tf32
// operand returned zeros -> mq_tc.cu stages everything K-major.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// A: 128 x 8 (m, k), B: 128 x 8 (n, k); D = A B^T (128 x 128)
// a_mn / b_mn select the layout of each operand in smem.
__global__ void probe(const float* A, const float* B, float* D, int a_mn, int b_mn, int variant,
                      uint32_t* dbg) {
  __shared__ __align__(1024) float sa[128 * 8];
  __shared__ __align__(1024) float sb[128 * 8];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // stage
  for (int i = tid; i < 128 * 8; i += blockDim.x) {
    const int m = i / 8, k = i % 8;
    uint32_t off;  // float index
    // K-major: [k4][m/8][m%8][k%4]  (LBO = 128*16 B, SBO = 128 B)
    // MN-major: [k8][m/4][k%8][m%4] (SBO = 128 B, LBO = 32*128 B)
    if (!a_mn) off = (k / 4) * (128 * 4) + (m / 8) * 32 + (m % 8) * 4 + (k % 4);
    else off = (m / 4) * 32 + (k % 8) * 4 + (m % 4);
    sa[off] = A[m * 8 + k];
    if (!b_mn) off = (k / 4) * (128 * 4) + (m / 8) * 32 + (m % 8) * 4 + (k % 4);
    else off = (m / 4) * 32 + (k % 8) * 4 + (m % 4);
    sb[off] = B[m * 8 + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s_tmem)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  if (tid == 0) dbg[0] = tmem;
  if (tid == 0) {
    uint32_t a_lbo = a_mn ? 32 * 128 : 128 * 16, a_sbo = 128;
    uint32_t b_lbo = b_mn ? 32 * 128 : 128 * 16, b_sbo = 128;
    if (variant == 1) {  // swapped lbo/sbo
      uint32_t t = a_lbo; a_lbo = a_sbo; a_sbo = t;
      t = b_lbo; b_lbo = b_sbo; b_sbo = t;
    }
    const uint64_t da = smem_desc(smem_u32(sa), a_lbo, a_sbo);
    const uint64_t db = smem_desc(smem_u32(sb), b_lbo, b_sbo);
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) |
                           ((uint32_t)b_mn << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    dbg[1] = idesc;
    dbg[2] = (uint32_t)da;
    dbg[3] = (uint32_t)(da >> 32);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&bar)) : "memory");
  }
  {
    const uint32_t addr = smem_u32(&bar);
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(addr), "r"(0u) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    for (int cb = 0; cb < 128; cb += 32) {
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
          : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)cb));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const int m = warp * 32 + lane;
      for (int u = 0; u < 32; ++u) D[m * 128 + cb + u] = __uint_as_float(r[u]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
  }
}

int main() {
  const int n = 128 * 8;
  float *hA = (float*)malloc(n * 4), *hB = (float*)malloc(n * 4), *hD = (float*)malloc(128 * 128 * 4);
  for (int i = 0; i < n; ++i) {
    hA[i] = (float)((i * 37) % 17 - 8) / 4.0f;  // exactly representable in tf32
    hB[i] = (float)((i * 11) % 13 - 6) / 2.0f;
  }
  float *A, *B, *D;
  uint32_t* dbg;
  cudaMalloc(&A, n * 4);
  cudaMalloc(&B, n * 4);
  cudaMalloc(&D, 128 * 128 * 4);
  cudaMalloc(&dbg, 64);
  cudaMemcpy(A, hA, n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, n * 4, cudaMemcpyHostToDevice);
  for (int variant = 0; variant < 1; ++variant)  // variant 1 (lbo<->sbo swapped) faults
    for (int a_mn = 0; a_mn < 2; ++a_mn)
      for (int b_mn = 0; b_mn < 2; ++b_mn) {
        cudaMemset(D, 0, 128 * 128 * 4);
        probe<<<1, 128>>>(A, B, D, a_mn, b_mn, variant, dbg);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(hD, D, 128 * 128 * 4, cudaMemcpyDeviceToHost);
        uint32_t hd[4];
        cudaMemcpy(hd, dbg, 16, cudaMemcpyDeviceToHost);
        double err = 0, mx = 0;
        for (int m = 0; m < 128; ++m)
          for (int j = 0; j < 128; ++j) {
            double ref = 0;
            for (int k = 0; k < 8; ++k) ref += (double)hA[m * 8 + k] * hB[j * 8 + k];
            err = fmax(err, fabs(ref - hD[m * 128 + j]));
            mx = fmax(mx, fabs(ref));
          }
        printf("variant %d a_mn %d b_mn %d: err %s max_err %.4g (max |ref| %.4g) D[0..3] %g %g %g %g tmem %u idesc %08x descA %08x%08x\n",
               variant, a_mn, b_mn, cudaGetErrorString(e), err, mx, hD[0], hD[1], hD[2], hD[3],
               hd[0], hd[1], hd[3], hd[2]);
        if (e != cudaSuccess) return 1;
      }
  return 0;
}
