// Device helpers shared by the tcgen05 edge and node kernels: power-of-two
// scaling, block max, fp16 hi/lo operand packing, descriptors, GEMM issue.
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"
#include "tc.cuh"

namespace fcg {

__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }

// Power-of-two scale s with max*2^s in [2^14, 2^15); 1 for an all-zero tile.
__device__ __forceinline__ int scale_exp(float m) {
  if (!(m > 0.f) || !isfinite(m)) return 0;
  int e;
  frexpf(m, &e);  // m = f * 2^e, f in [0.5, 1)
  return 15 - e;
}

// Block-wide max of non-negative values (every thread of the CTA calls it).
__device__ __forceinline__ float block_amax(float v, unsigned int *slot) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMax(slot, __float_as_uint(v));
  __syncthreads();
  return __uint_as_float(*slot);
}

// Named barrier over a subset of the CTA (id 1.. ; id 0 is __syncthreads).
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Max over the threads of one named-barrier group.
__device__ __forceinline__ float group_amax(float v, unsigned int *slot, int bar_id, int nthreads) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMax(slot, __float_as_uint(v));
  named_sync(bar_id, nthreads);
  return __uint_as_float(*slot);
}

// Store 8 consecutive columns e0..e0+7 of K-row r of an MN-major B operand
// with N columns (kstride = bytes per 8 K-rows = 16*N; hi image at act, lo
// image at act + K*kstride/8), values pre-scaled.
__device__ __forceinline__ void put_b8n(uint8_t *act, int K, uint32_t kstride, int r, int e0,
                                        const float *v, float scale, bool with_lo) {
  uint32_t off = (uint32_t)(r >> 3) * kstride + (uint32_t)(e0 >> 3) * 128u + (uint32_t)(r & 7) * 16u;
  __half2 hi[4], lo[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float a = v[2 * i] * scale, b = v[2 * i + 1] * scale;
    hi[i] = __floats2half2_rn(a, b);
    float2 hf = __half22float2(hi[i]);
    lo[i] = __floats2half2_rn(a - hf.x, b - hf.y);
  }
  *(uint4 *)(act + off) = *(uint4 *)hi;
  if (with_lo) *(uint4 *)(act + (uint32_t)K * (kstride >> 3) + off) = *(uint4 *)lo;
}

// N=128 variant (kstride 2048).
__device__ __forceinline__ void put_b8(uint8_t *act, int K, int r, int e0, const float *v,
                                       float scale, bool with_lo) {
  uint32_t off = (uint32_t)(r >> 3) * 2048u + (uint32_t)(e0 >> 3) * 128u + (uint32_t)(r & 7) * 16u;
  __half2 hi[4], lo[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float a = v[2 * i] * scale, b = v[2 * i + 1] * scale;
    hi[i] = __floats2half2_rn(a, b);
    float2 hf = __half22float2(hi[i]);
    lo[i] = __floats2half2_rn(a - hf.x, b - hf.y);
  }
  *(uint4 *)(act + off) = *(uint4 *)hi;
  if (with_lo) *(uint4 *)(act + (uint32_t)K * 256u + off) = *(uint4 *)lo;
}

// Descriptors (SWIZZLE_NONE, LBO = core stride along K, SBO = along M/N;
// pinned on hardware by tests/test_gpu_tcgen05.py).
__device__ __forceinline__ uint64_t desc_w_kmajor(uint32_t base, int in_dim, int k0) {
  return tc::smem_desc(base + (uint32_t)(k0 >> 3) * 128u, 128u, (uint32_t)(in_dim >> 3) * 128u);
}
__device__ __forceinline__ uint64_t desc_w_mnmajor(uint32_t base, int in_dim, int k0) {
  uint32_t rowstride = (uint32_t)(in_dim >> 3) * 128u;
  return tc::smem_desc(base + (uint32_t)(k0 >> 3) * rowstride, rowstride, 128u);
}
__device__ __forceinline__ uint64_t desc_act(uint32_t base, int k0, uint32_t kstride = 2048u) {
  return tc::smem_desc(base + (uint32_t)(k0 >> 3) * kstride, kstride, 128u);
}

// Issue one GEMM D(tmem) = A(weights) x B(act) over K, with the product set
// {hi*hi, hi*lo, lo*hi} (nprod=3), {hi*hi, hi*lo} (2) or {hi*hi} (1).
__device__ __forceinline__ void issue_gemm(uint32_t d, uint32_t w_base, uint32_t w_lo_off,
                                           int in_dim, bool w_mn, uint32_t act_base, int K,
                                           uint32_t idesc, int nprod,
                                           uint32_t kstride = 2048u) {
  uint32_t act_lo = act_base + (uint32_t)K * (kstride >> 3);
#pragma unroll 1
  for (int k0 = 0; k0 < K; k0 += 16) {
    uint64_t ah = w_mn ? desc_w_mnmajor(w_base, in_dim, k0) : desc_w_kmajor(w_base, in_dim, k0);
    uint64_t bh = desc_act(act_base, k0, kstride);
    tc::mma_f16_ss(d, ah, bh, idesc, k0 > 0);
    if (nprod >= 2) tc::mma_f16_ss(d, ah, desc_act(act_lo, k0, kstride), idesc, 1);
    if (nprod >= 3) {
      uint64_t al = w_mn ? desc_w_mnmajor(w_base + w_lo_off, in_dim, k0)
                         : desc_w_kmajor(w_base + w_lo_off, in_dim, k0);
      tc::mma_f16_ss(d, al, bh, idesc, 1);
    }
  }
}

// MUFU approximations with denormals flushed (the library is built without
// -ftz, which would make __expf/__logf carry range fix-ups); used only by the
// tensor-core epilogues, whose parity is tolerance-based.
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2_ftz(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// shifted softplus max(x,0) + log1p(exp(-|x|)) - ln2 (model.py:93-100) and
// its derivative sigmoid(x) (model.py:103-107) on MUFU ex2/lg2/rcp (abs.
// error ~1e-7).  Used by the W16 path as well: its fp16 activation rounding
// turns the ~1e-7 difference from NumPy's expf/log1pf into occasional
// rounding flips (~1e-4 relative energy on tiny systems), far inside the
// reference's own W16 contract (1e-2 vs fp32, tests/test_quantize.py:169),
// while CUDA's accurate expf/log1pf cost 37% of the W16 step.
// ln2 * (lg2(1 + t) - 1) = ln2 * lg2(0.5 t + 0.5): the -1 folds into one FFMA.
__device__ __forceinline__ float ssp_fast(float x) {
  return fmaf(kLn2, lg2_ftz(fmaf(ex2_ftz(fabsf(x) * -kLog2e), 0.5f, 0.5f)), fmaxf(x, 0.f));
}
// s * ssp(x) for a power-of-two s > 0 from xs = s * x (exact): the scale rides
// in the constants, c_ln2 = s ln2 and c_e = -log2(e) / s.
__device__ __forceinline__ float ssp_scaled(float xs, float c_ln2, float c_e) {
#ifdef FCG_ACCURATE_EPI  // diagnostic builds: libm transcendentals (precision A/B)
  const float s = c_ln2 / kLn2;  // the power-of-two scale
  const float x = xs / s;
  return s * (fmaxf(x, 0.f) + log1pf(expf(-fabsf(x))) - kLn2);
#else
  return fmaf(c_ln2, lg2_ftz(fmaf(ex2_ftz(fabsf(xs) * c_e), 0.5f, 0.5f)), fmaxf(xs, 0.f));
#endif
}
__device__ __forceinline__ float sigmoid_fast(float x) {
  return rcp_ftz(1.f + ex2_ftz(x * -kLog2e));
}

// ---- packed fp32x2 (sm_100 FFMA2 / FMUL2 / FADD2) ----------------------------
// The edge epilogues are issue-bound; every elementwise step on a pair of
// values is one instruction.  Round-to-nearest per element, so results are
// bitwise those of the scalar forms.
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
// c_ln2 * lg2(0.5 t + 0.5) + max(x, 0) with t = 2^(|x| c_e): ssp_scaled on a pair
__device__ __forceinline__ float2 ssp_scaled2(float2 xs, float c_ln2, float c_e) {
  const float2 t = make_float2(ex2_ftz(fabsf(xs.x) * c_e), ex2_ftz(fabsf(xs.y) * c_e));
  const float2 u = fma2(t, f2(0.5f), f2(0.5f));
  const float2 l = make_float2(lg2_ftz(u.x), lg2_ftz(u.y));
  return fma2(f2(c_ln2), l, make_float2(fmaxf(xs.x, 0.f), fmaxf(xs.y, 0.f)));
}
__device__ __forceinline__ float2 ssp_fast2(float2 x) {
  return ssp_scaled2(x, kLn2, -kLog2e);
}
__device__ __forceinline__ float2 ex2_2(float2 x) {
  return make_float2(ex2_ftz(x.x), ex2_ftz(x.y));
}

}  // namespace fcg
