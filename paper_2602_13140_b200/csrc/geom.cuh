// Per-edge geometry, the edge-balanced work-unit row boundaries of the fused
// edge kernels and the embedding lookup: the work of k_edge_geom
// (edge_tc.cu), also run inside the fused neighbour assembly of fcg_md_step
// (nbr.cu), so both produce the same bits.
#pragma once
#include "common.cuh"

namespace fcg {

// Edge k = (own -> nbr): u = r_own - r_nbr, d = |u| in the reference's _rn
// order (flash.py:279), and cutoff_envelope(_grad) (model.py:110-120).
__device__ __forceinline__ void edge_geom_one(const float *pos, int own, int nbr, float cutoff,
                                              float4 *geo, float2 *env, long long k) {
  const float *po = pos + (size_t)own * 3, *pn = pos + (size_t)nbr * 3;
  const float ux = __fsub_rn(po[0], pn[0]), uy = __fsub_rn(po[1], pn[1]),
              uz = __fsub_rn(po[2], pn[2]);
  const float d =
      __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(ux, ux), __fmul_rn(uy, uy)), __fmul_rn(uz, uz)));
  float c = 0.f, dc = 0.f;
  if (d < cutoff) {
    float sn, cs;
    sincosf((3.14159265358979f * d) / cutoff, &sn, &cs);
    c = 0.5f * (cs + 1.f);
    dc = (float)(-0.5 * 3.141592653589793 / (double)cutoff) * sn;
  }
  geo[k] = make_float4(ux, uy, uz, d);
  env[k] = make_float2(c, dc);
}

// Boundary index r of the CSR (lo = ptr[r-1], or -1 for r = 0; hi = ptr[r]):
// work unit u of G starts at row r for every u with lo < e_tot*u/G <= hi,
// so the G units split the edges evenly and every row has one owner.
__device__ __forceinline__ void unit_rows_at(long long r, long long lo, long long hi,
                                             long long e_tot, int32_t *ur, long long G,
                                             int nrows) {
  if (!ur) return;
  if (r == 0) {
    ur[0] = 0;
    ur[G] = nrows;
  }
  if (hi <= lo) return;  // empty row: no boundary maps to it
  long long u = lo < 0 ? 1 : (e_tot > 0 ? ((lo + 1) * G + e_tot - 1) / e_tot : G);
  if (u < 1) u = 1;
  for (; u < G && e_tot * u / G <= hi; ++u) ur[u] = (int32_t)r;
}

// X = embedding[types] (flash.py:201), block 0's pre-linear from the
// per-type table, and the operand-bound words reset (thread t of nt; `first`
// = the first CTA).
__device__ __forceinline__ void embed_rows(const EmbedJob &ej, int nrows, long long t,
                                           long long nt, bool first) {
  if (!ej.X) return;
  if (first && (int)threadIdx.x < ej.namax)
    ej.amax[threadIdx.x] = (threadIdx.x == 0 && ej.P0) ? __float_as_uint(ej.p0_amax) : 0u;
  for (long long q = t; q < (long long)nrows * (D / 4); q += nt) {
    const long long g = q / (D / 4);
    const int c4 = (int)(q % (D / 4));
    const int ty = ld_dep(&ej.types[g % ej.N]);
    *(float4 *)&ej.X[g * D + c4 * 4] = ld_dep((const float4 *)&ej.emb[(size_t)ty * D + c4 * 4]);
    if (ej.P0)
      *(float4 *)&ej.P0[g * D + c4 * 4] =
          ld_dep((const float4 *)&ej.p0_table[(size_t)ty * D + c4 * 4]);
  }
}

}  // namespace fcg
