// tcgen05 self-test: one CTA computes D = A * B^T (fp16 in, fp32 accumulate
// in TMEM) with operands staged in the canonical no-swizzle core-matrix
// layout, K-major or MN-major, and dumps all 128 TMEM lanes.  Used by
// tests/test_gpu_tcgen05.py to pin the descriptor conventions the fused
// edge kernels rely on.
#include "common.cuh"
#include "tc.cuh"

namespace fcg {

struct StOperand {
  int mn_major;   // 0: physical rows = MN, contiguous = K; 1: rows = K, contiguous = MN
  int core_rows_fastest;  // core placement order
  int swap;       // swap the LBO/SBO field assignment
};

__device__ __forceinline__ void st_offsets(const StOperand &o, int MN, int K, uint32_t &Si,
                                           uint32_t &Sj) {
  int PR = o.mn_major ? K : MN, PC = o.mn_major ? MN : K;
  if (o.core_rows_fastest) { Si = 128; Sj = (PR / 8) * 128; }
  else { Sj = 128; Si = (PC / 8) * 128; }
}

__device__ void st_fill(const StOperand &o, const uint16_t *src, int MN, int K, uint8_t *dst) {
  uint32_t Si, Sj;
  st_offsets(o, MN, K, Si, Sj);
  for (int q = threadIdx.x; q < MN * K; q += blockDim.x) {
    int mn = q / K, k = q % K;
    int r = o.mn_major ? k : mn, c = o.mn_major ? mn : k;
    uint32_t off = (r / 8) * Si + (c / 8) * Sj + (r % 8) * 16 + (c % 8) * 2;
    *(uint16_t *)(dst + off) = src[q];
  }
}

__device__ uint64_t st_desc(const StOperand &o, const uint8_t *base, int MN, int K, int k0) {
  uint32_t Si, Sj;
  st_offsets(o, MN, K, Si, Sj);
  uint32_t kstride = o.mn_major ? Si : Sj, mnstride = o.mn_major ? Sj : Si;
  uint32_t start = tc::smem_u32(base) + (k0 / 8) * kstride;
  // canonical assumption: K-major LBO = K stride, SBO = MN stride;
  //                       MN-major LBO = MN stride, SBO = K stride
  uint32_t lbo = o.mn_major ? mnstride : kstride, sbo = o.mn_major ? kstride : mnstride;
  if (o.swap) { uint32_t t = lbo; lbo = sbo; sbo = t; }
  return tc::smem_desc(start, lbo, sbo);
}

__global__ void __launch_bounds__(128)
k_selftest_mma(const uint16_t *A, const uint16_t *B, float *dump, int M, int N, int K,
               StOperand oa, StOperand ob) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  uint8_t *As = sm, *Bs = sm + M * K * 2;
  const bool a_tmem = oa.core_rows_fastest == 2;  // A operand from TMEM (M = 128)
  if (!a_tmem) st_fill(oa, A, M, K, As);
  st_fill(ob, B, N, K, Bs);
  tc::fence_async_smem();
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc<256>(&tmem_base);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  uint32_t tbase = tmem_base;
  const uint32_t a_col = 128;  // A in TMEM columns [128, 128 + K/2)
  if (a_tmem) {
    // lane m = row m; column j packs (A[m][2j], A[m][2j+1])
    const int m = threadIdx.x;
    for (int j0 = 0; j0 < K / 2; j0 += 16) {
      float v[16];
      for (int j = 0; j < 16; ++j) {
        uint32_t lo = A[m * K + 2 * (j0 + j)], hi = A[m * K + 2 * (j0 + j) + 1];
        v[j] = __uint_as_float(lo | (hi << 16));
      }
      tc::tmem_st16(tbase + ((uint32_t)(32 * (threadIdx.x >> 5)) << 16) + a_col + j0, v);
    }
    tc::tmem_st_wait();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
  }
  if (threadIdx.x == 0) {
    uint32_t idesc = tc::idesc_f16(M, N, a_tmem ? 0 : oa.mn_major, ob.mn_major);
    for (int k0 = 0; k0 < K; k0 += 16) {
      if (a_tmem)
        tc::mma_f16_ts(tbase, tbase + a_col + k0 / 2, st_desc(ob, Bs, N, K, k0), idesc, k0 > 0);
      else
        tc::mma_f16_ss(tbase, st_desc(oa, As, M, K, k0), st_desc(ob, Bs, N, K, k0), idesc,
                       k0 > 0);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tc::tmem_ld16(tbase + ((uint32_t)(32 * warp) << 16) + c0, v);
    tc::tmem_ld_wait();
    for (int i = 0; i < 16; ++i) dump[(32 * warp + lane) * N + c0 + i] = v[i];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<256>(tbase);
}

}  // namespace fcg

extern "C" int fcg_selftest_mma(const uint16_t *A, const uint16_t *B, float *dump, int M, int N,
                                int K, int a_mn, int a_order, int a_swap, int b_mn, int b_order,
                                int b_swap, void *stream) {
  using namespace fcg;
  if ((M != 64 && M != 128) || N % 16 || N < 16 || N > 256 || K % 16 || K > 256 ||
      (a_order == 2 && (M != 128 || N > 128 || K > 256))) {
    set_error("selftest_mma: unsupported shape");
    return FCG_ERR_ARG;
  }
  size_t smem = (size_t)(M + N) * K * 2;
  cudaFuncSetAttribute(k_selftest_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  StOperand oa{a_mn, a_order, a_swap}, ob{b_mn, b_order, b_swap};
  k_selftest_mma<<<1, 128, smem, (cudaStream_t)stream>>>(A, B, dump, M, N, K, oa, ob);
  return cuda_status("selftest_mma");
}
