// Harmonic bond prior (md.py:109-124) device code, shared by k_prior
// (md.cu) and the force assembly of the fused MD step (model.cu), which
// evaluates the prior forces inline instead of reading them back.
#pragma once
#include "common.cuh"

namespace fcg {

// ---- harmonic prior, md.py:109-124 -----------------------------------------
struct BondVec { float fx, fy, fz, e; };
__device__ __forceinline__ BondVec bond_eval(const fcg_prior &pr, const float *P, int b) {
  int i = pr.bond_i[b], j = pr.bond_j[b];
  float x = __fsub_rn(P[3 * i], P[3 * j]), y = __fsub_rn(P[3 * i + 1], P[3 * j + 1]),
        z = __fsub_rn(P[3 * i + 2], P[3 * j + 2]);
  float d = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y)), __fmul_rn(z, z)));
  float k = pr.k[b];
  float st = __fsub_rn(d, pr.r0[b]);
  float safe = d > 0.f ? d : 1.f;
  float coef = __fdiv_rn(__fmul_rn(-k, st), safe);
  BondVec o;
  o.fx = __fmul_rn(coef, x);
  o.fy = __fmul_rn(coef, y);
  o.fz = __fmul_rn(coef, z);
  o.e = __fmul_rn(__fmul_rn(k, st), st);
  return o;
}

// One thread per bead: it applies its incident bonds in np.add.at order (all
// "+fvec" for bonds where it is atom i, then "-fvec" where it is atom j), so
// the per-bead sums are bitwise the reference's.
__device__ __forceinline__ float3 prior_bead_force(const fcg_prior &pr, const float *pos, int N,
                                                   int g) {
  const int r = g / N, i = g % N;
  const float *P = pos + (size_t)r * N * 3;
  float fx = 0.f, fy = 0.f, fz = 0.f;
  if (pr.num_bonds > 0) {
    for (int q = pr.inc_ptr[i]; q < pr.inc_ptr[i + 1]; ++q) {
      BondVec v = bond_eval(pr, P, pr.inc_bond[q]);
      if (pr.inc_sign[q] > 0) {
        fx = __fadd_rn(fx, v.fx); fy = __fadd_rn(fy, v.fy); fz = __fadd_rn(fz, v.fz);
      } else {
        fx = __fadd_rn(fx, -v.fx); fy = __fadd_rn(fy, -v.fy); fz = __fadd_rn(fz, -v.fz);
      }
    }
  }
  return make_float3(fx, fy, fz);
}
__device__ __forceinline__ void prior_bead(const fcg_prior &pr, const float *pos, int N, int RN,
                                           float *f_prior, int g) {
  if (g >= RN) return;
  const float3 f3 = prior_bead_force(pr, pos, N, g);
  float *f = f_prior + (size_t)g * 3;
  f[0] = f3.x; f[1] = f3.y; f[2] = f3.z;
}

// Prior energy 0.5 * sum k*s^2 per replica (md.py:118), one CTA per replica.
__device__ __forceinline__ void prior_energy(const fcg_prior &pr, const float *pos, int N,
                                             float *e_prior, int r) {
  const float *P = pos + (size_t)r * N * 3;
  __shared__ float red[256];
  float acc = 0.f;
  for (int b = threadIdx.x; b < pr.num_bonds; b += blockDim.x) acc += bond_eval(pr, P, b).e;
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) e_prior[r] = 0.5f * red[0];
}

}  // namespace fcg
