// (b)(c)(d) SchNet energy + forces for all replicas, fp32.
//
// Replaces flash_energy_forces (flash.py:446-501): embedding gather, T fused
// interaction blocks (flash_block_forward, flash.py:192-245), readout
// (model.py:297-318 on params.readout), ones-seeded backward, T fused
// backward blocks (flash_block_backward, flash.py:248-307) and forces=-grad_r.
//
// Layout in HBM (g = r*N + i, rows of FCG_D floats):
//   X [RN][D]        node features, updated in place block by block
//   P_t [RN][D]      pre-linear output of block t (kept for backward)
//   Zp_t [RN][D]     post-MLP hidden pre-activation of block t (backward)
//   H [RN][D]        destination segment sums (one store per row)
//   G [RN][D]        dE/dX, updated in place backwards
//   GH, GP [RN][D]   dE/dH, dE/dP of the current block
//   gsum [cap_e]     float4 per CSR slot: sum over blocks of the per-edge
//                    position gradient g_e (flash.py:294) of the edge whose
//                    src is the slot's row (owner-indexed, single writer)
// Edge tensors (basis, filters, messages) never leave shared memory.
//
// Edge kernels own whole CSR rows (cta_row_range): the forward walks dst
// rows (messages reduced into H rows), the backward walks the same rows as
// src segments (grad_P rows) — identical because the graph is symmetric and
// the reference's src-grouped perm is the rev[] map.  No atomics.
#include <cuda_fp16.h>
#include <stdlib.h>

#include "common.cuh"
#include "prior.cuh"

namespace fcg {

constexpr int TE = 64;          // edges (or node rows) per tile
constexpr int NT = 256;         // threads per CTA
constexpr int LDR = DR + 4;     // padded row stride of [TE][DR] tiles
constexpr int LDH = D + 4;      // padded row stride of [TE][D] tiles

// ---------------------------------------------------------------------------
// 64-row register-tiled SIMT GEMM: acc[4][NC] += A[64][K] (smem, row-major,
// stride lda) x Bt[K][NOUT] (global, k-major).  Thread (ty,tx) = (tid/16,
// tid%16) owns rows ty*4..ty*4+3 and columns col(j).
template <int NOUT>
__device__ __forceinline__ int gcol(int tx, int j) {
  if (NOUT == 128) return j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4);
  return tx * 4 + j;
}

template <int K, int NOUT>
__device__ __forceinline__ void gemm64(const float *As, int lda, const float *__restrict__ Bt,
                                       float (&acc)[4][NOUT / 16]) {
  constexpr int NC = NOUT / 16;
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[i][j] = 0.f;
#pragma unroll 2
  for (int k = 0; k < K; k += 4) {
    float4 a[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = *(const float4 *)&As[(ty * 4 + i) * lda + k];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const float *brow = Bt + (size_t)(k + kk) * NOUT;
      float4 b0 = __ldg((const float4 *)&brow[tx * 4]);
      float4 b1 = b0;
      if (NC == 8) b1 = __ldg((const float4 *)&brow[64 + tx * 4]);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float av = kk == 0 ? a[i].x : kk == 1 ? a[i].y : kk == 2 ? a[i].z : a[i].w;
        acc[i][0] = fmaf(av, b0.x, acc[i][0]);
        acc[i][1] = fmaf(av, b0.y, acc[i][1]);
        acc[i][2] = fmaf(av, b0.z, acc[i][2]);
        acc[i][3] = fmaf(av, b0.w, acc[i][3]);
        if (NC == 8) {
          acc[i][4] = fmaf(av, b1.x, acc[i][4]);
          acc[i][5] = fmaf(av, b1.y, acc[i][5]);
          acc[i][6] = fmaf(av, b1.z, acc[i][6]);
          acc[i][7] = fmaf(av, b1.w, acc[i][7]);
        }
      }
    }
  }
}

// W16 forward semantics (quantize.py:68-71, :86): every linear layer of the
// forward sees its input rounded to fp16 (then widened back to fp32).
__device__ __forceinline__ float q16(float x) { return __half2float(__float2half_rn(x)); }
__device__ __forceinline__ float maybe_q16(float x, int quant) { return quant ? q16(x) : x; }

// Load rows [row0, row0+64) of a [nrows][D] global matrix into a padded smem
// tile (optionally fp16-rounding the values: forward input of a W16 layer).
__device__ __forceinline__ void load_rows(float *As, const float *__restrict__ src, int row0,
                                          int nrows, int quant = 0) {
  for (int q = threadIdx.x; q < TE * (D / 4); q += NT) {
    int r = q / (D / 4), c4 = q % (D / 4);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row0 + r < nrows) v = __ldg((const float4 *)&src[(size_t)(row0 + r) * D + c4 * 4]);
    if (quant) { v.x = q16(v.x); v.y = q16(v.y); v.z = q16(v.z); v.w = q16(v.w); }
    *(float4 *)&As[r * LDH + c4 * 4] = v;
  }
}

// ---------------------------------------------------------------------------
// node kernels
__global__ void k_embed(const float *emb, const int32_t *types, int N,
                        int RN, float *X, unsigned int *amax, int namax) {
  pdl_trigger();
  pdl_wait();
  if (blockIdx.x == 0 && (int)threadIdx.x < namax) amax[threadIdx.x] = 0u;  // scale maxima
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= RN * (D / 4)) return;
  int g = q / (D / 4), c4 = q % (D / 4);
  int t = types[g % N];
  *(float4 *)&X[(size_t)g * D + c4 * 4] = ld_dep((const float4 *)&emb[(size_t)t * D + c4 * 4]);
}

// Y = A W^T + b (pre-linear, flash.py:207), or with kAccumulate: Y += A W
// (grad_X += grad_P @ W_pre, flash.py:300; Bt = W itself).
template <bool kBias, bool kAccumulate>
__global__ void __launch_bounds__(NT)
k_node_linear(const float *__restrict__ A, const float *__restrict__ Bt,
              const float *__restrict__ bias, float *__restrict__ Y, int nrows, int quant) {
  extern __shared__ float smem[];
  float *As = smem;
  const int row0 = blockIdx.x * TE;
  load_rows(As, A, row0, nrows, quant);
  __syncthreads();
  float acc[4][8];
  gemm64<D, D>(As, LDH, Bt, acc);
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int row = row0 + ty * 4 + i;
    if (row >= nrows) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int c = h * 64 + tx * 4;
      float4 o = make_float4(acc[i][4 * h], acc[i][4 * h + 1], acc[i][4 * h + 2], acc[i][4 * h + 3]);
      if (kBias) {
        float4 b = __ldg((const float4 *)&bias[c]);
        o.x += b.x; o.y += b.y; o.z += b.z; o.w += b.w;
      }
      float4 *dst = (float4 *)&Y[(size_t)row * D + c];
      if (kAccumulate) {
        float4 y = *dst;
        o.x += y.x; o.y += y.y; o.z += y.z; o.w += y.w;
      }
      *dst = o;
    }
  }
}

// post MLP + residual (flash.py:240-241): Zp = H Wp0^T + b0 (kept), U =
// ssp(Zp) Wp1^T + b1, X += U.
__global__ void __launch_bounds__(NT)
k_node_post(const float *__restrict__ H, const fcg_block blk, float *__restrict__ Zp,
            float *__restrict__ X, int nrows, int quant) {
  extern __shared__ float smem[];
  float *As = smem, *Bs = smem + TE * LDH;
  const int row0 = blockIdx.x * TE;
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  load_rows(As, H, row0, nrows, quant);
  __syncthreads();
  float acc[4][8];
  gemm64<D, D>(As, LDH, blk.p0_wt, acc);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int r = ty * 4 + i, row = row0 + r;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int c = gcol<128>(tx, j);
      float z = acc[i][j] + __ldg(&blk.p0_b[c]);
      if (row < nrows) Zp[(size_t)row * D + c] = z;
      Bs[r * LDH + c] = maybe_q16(ssp(z), quant);
    }
  }
  __syncthreads();
  gemm64<D, D>(Bs, LDH, blk.p1_wt, acc);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int row = row0 + ty * 4 + i;
    if (row >= nrows) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int c = gcol<128>(tx, j);
      X[(size_t)row * D + c] += acc[i][j] + __ldg(&blk.p1_b[c]);
    }
  }
}

// Backward of the post MLP (mlp_backward_input, model.py:321-332, called at
// flash.py:264): GH = ((G Wp1) * ssp'(Zp)) Wp0.
__global__ void __launch_bounds__(NT)
k_node_post_bwd(const float *__restrict__ G, const fcg_block blk, const float *__restrict__ Zp,
                float *__restrict__ GH, int nrows) {
  extern __shared__ float smem[];
  float *As = smem, *Bs = smem + TE * LDH;
  const int row0 = blockIdx.x * TE;
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  load_rows(As, G, row0, nrows);
  __syncthreads();
  float acc[4][8];
  gemm64<D, D>(As, LDH, blk.p1_w, acc);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int r = ty * 4 + i, row = row0 + r;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int c = gcol<128>(tx, j);
      float z = row < nrows ? Zp[(size_t)row * D + c] : 0.f;
      Bs[r * LDH + c] = acc[i][j] * ssp_grad(z);
    }
  }
  __syncthreads();
  gemm64<D, D>(Bs, LDH, blk.p0_w, acc);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int row = row0 + ty * 4 + i;
    if (row >= nrows) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) GH[(size_t)row * D + gcol<128>(tx, j)] = acc[i][j];
  }
}

// Readout (flash.py:487-492): per_atom = ssp(X Wr0^T + br0) . wr1 + br1, and
// the ones-seeded backward G = (wr1 * ssp'(zr)) Wr0.
__global__ void __launch_bounds__(NT)
k_readout(const float *__restrict__ X, const fcg_model m, float *__restrict__ per_atom,
          float *__restrict__ G, int nrows) {
  extern __shared__ float smem[];
  float *As = smem, *Bs = smem + TE * LDH;  // Bs: [TE][LDR]
  const int row0 = blockIdx.x * TE;
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  const int quant = m.format == FCG_FMT_W16;
  load_rows(As, X, row0, nrows, quant);
  __syncthreads();
  float acc[4][4];
  gemm64<D, RH>(As, LDH, m.r0_wt, acc);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int r = ty * 4 + i;
    float part = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int c = tx * 4 + j;
      float z = acc[i][j] + __ldg(&m.r0_b[c]);
      float w1 = __ldg(&m.r1_w[c]);
      part += maybe_q16(ssp(z), quant) * w1;
      Bs[r * LDR + c] = w1 * ssp_grad(z);
    }
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    int row = row0 + r;
    if (tx == 0 && row < nrows) per_atom[row] = part + m.r1_b;
  }
  __syncthreads();
  float acc2[4][8];
  gemm64<RH, D>(Bs, LDR, m.r0_w, acc2);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int row = row0 + ty * 4 + i;
    if (row >= nrows) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) G[(size_t)row * D + gcol<128>(tx, j)] = acc2[i][j];
  }
}

// ---------------------------------------------------------------------------
// edge kernels
// Envelope C(d) and C'(d) (model.py:242-252), fp32 as numpy evaluates them.
__device__ __forceinline__ void envelope(float d, float cutoff, float &c, float &dc) {
  const float pi = 3.14159265358979f;
  if (d < cutoff) {
    float a = (pi * d) / cutoff;
    float sn, cs;
    sincosf(a, &sn, &cs);
    c = 0.5f * (cs + 1.f);
    dc = (float)(-0.5 * 3.141592653589793 / (double)cutoff) * sn;
  } else {
    c = 0.f;
    dc = 0.f;
  }
}

// Per-tile edge geometry into smem; returns nothing, fills s_* arrays.
__device__ __forceinline__ void tile_geometry(const EdgeArgs &a, int t0, int n_e, bool src_owned,
                                              int *s_own, int *s_nbr, float *s_d, float4 *s_u) {
  int t = threadIdx.x;
  if (t < TE) {
    int o = -1, n = 0;
    float d = 0.f;
    float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
    if (t < n_e) {
      int k = t0 + t;
      o = a.own[k];
      n = a.nbr[k];
      const float *po = a.pos + (size_t)o * 3, *pn = a.pos + (size_t)n * 3;
      // forward edge (dst=o, src=n): u = r_dst - r_src = r_o - r_n;
      // backward edge (dst=n, src=o): u = r_n - r_o (flash.py:221, :279)
      float ux = __fsub_rn(po[0], pn[0]), uy = __fsub_rn(po[1], pn[1]), uz = __fsub_rn(po[2], pn[2]);
      if (src_owned) { ux = -ux; uy = -uy; uz = -uz; }
      d = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(ux, ux), __fmul_rn(uy, uy)), __fmul_rn(uz, uz)));
      u = make_float4(ux, uy, uz, 0.f);
    }
    s_own[t] = o;
    s_nbr[t] = n;
    s_d[t] = d;
    s_u[t] = u;
  }
}

// Basis b[e][k] = exp((-g*dk)*dk) * C(d) into a [TE][LDR] tile (model.py:255-265).
__device__ __forceinline__ void tile_basis(const EdgeArgs &a, const float *s_d, float *rb) {
  for (int q = threadIdx.x; q < TE * DR; q += NT) {
    int e = q / DR, k = q % DR;
    float d = s_d[e];
    float c, dc;
    envelope(d, a.cutoff, c, dc);
    float dl = d - __ldg(&a.centers[k]);
    rb[e * LDR + k] = maybe_q16(__expf((-a.gamma * dl) * dl) * c, a.quant);
  }
}

// Segmented reduce of a [TE][LDH] tile along CSR rows: thread c (<128) keeps
// the running sum of channel c for row `cur`, flushing each completed row
// exactly once and writing zeros for empty rows.
struct RowReducer {
  int cur;
  float acc;
  __device__ __forceinline__ void init(int rb) { cur = rb; acc = 0.f; }
  __device__ __forceinline__ void tile(const float *tileb, const int *s_own, int n_e,
                                       float *__restrict__ out) {
    int c = threadIdx.x;
    for (int e = 0; e < n_e; ++e) {
      int row = s_own[e];
      if (row != cur) {
        out[(size_t)cur * D + c] = acc;
        for (int z = cur + 1; z < row; ++z) out[(size_t)z * D + c] = 0.f;
        cur = row;
        acc = 0.f;
      }
      acc += tileb[e * LDH + c];
    }
  }
  __device__ __forceinline__ void finish(int re, float *__restrict__ out) {
    int c = threadIdx.x;
    if (cur < re) {
      out[(size_t)cur * D + c] = acc;
      for (int z = cur + 1; z < re; ++z) out[(size_t)z * D + c] = 0.f;
    }
  }
};

// Fused forward edge pass (flash_block_forward tile loop, flash.py:215-236):
// d -> basis -> filter MLP -> message P[src]*w -> dst segment sums H.
__global__ void __launch_bounds__(NT, 2)
k_edge_fwd(const EdgeArgs a, const float *__restrict__ P, float *__restrict__ H) {
  extern __shared__ float smem[];
  float *rb = smem;                 // [TE][LDR] basis
  float *hb = rb + TE * LDR;        // [TE][LDH] hidden, then messages
  __shared__ int s_own[TE], s_nbr[TE];
  __shared__ float s_d[TE];
  __shared__ float4 s_u[TE];
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;

  int e_tot = a.ptr[a.nrows];
  long long eff = e_tot > a.cap_e ? a.cap_e : e_tot;
  int rbeg, rend;
  cta_row_range(a.ptr, a.nrows, eff, blockIdx.x, gridDim.x, rbeg, rend);
  int eb = a.ptr[rbeg], ee = a.ptr[rend];
  if (ee > eff) ee = (int)eff;
  if (eb > ee) eb = ee;
  RowReducer red;
  red.init(rbeg);

  for (int t0 = eb; t0 < ee; t0 += TE) {
    int n_e = min(TE, ee - t0);
    __syncthreads();
    tile_geometry(a, t0, n_e, false, s_own, s_nbr, s_d, s_u);
    __syncthreads();
    tile_basis(a, s_d, rb);
    __syncthreads();
    float acc[4][8];
    gemm64<DR, D>(rb, LDR, a.blk.f0_wt, acc);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        int c = gcol<128>(tx, j);
        hb[(ty * 4 + i) * LDH + c] = maybe_q16(ssp(acc[i][j] + __ldg(&a.blk.f0_b[c])), a.quant);
      }
    __syncthreads();
    gemm64<D, D>(hb, LDH, a.blk.f1_wt, acc);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int e = ty * 4 + i;
      const float *prow = P + (size_t)s_nbr[e] * D;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        int c = gcol<128>(tx, j);
        float w = acc[i][j] + __ldg(&a.blk.f1_b[c]);
        hb[e * LDH + c] = __ldg(&prow[c]) * w;
      }
    }
    __syncthreads();
    if (threadIdx.x < D) red.tile(hb, s_own, n_e, H);
  }
  if (threadIdx.x < D) red.finish(rend, H);
}

// Fused backward edge pass over src-owned segments (flash_block_backward
// tile loop, flash.py:272-295): recompute basis/filter, gH = grad_H[dst],
// grad_P rows = src-segment sums of gH*w, grad_w = gH*P[src] -> filter
// backward -> grad_d -> g_e, accumulated into the owner-indexed gsum.
__global__ void __launch_bounds__(NT, 2)
k_edge_bwd(const EdgeArgs a, const float *__restrict__ P, const float *__restrict__ GH,
           float *__restrict__ GP, float4 *__restrict__ gsum, int accumulate) {
  extern __shared__ float smem[];
  float *xb = smem;                 // [TE][LDH] basis (stride LDR), then contrib
  float *hb = xb + TE * LDH;        // [TE][LDH] hidden, then grad_w
  float *zb = hb + TE * LDH;        // [TE][LDH] z0, then grad_z0
  __shared__ int s_own[TE], s_nbr[TE];
  __shared__ float s_d[TE];
  __shared__ float4 s_u[TE];
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;

  int e_tot = a.ptr[a.nrows];
  long long eff = e_tot > a.cap_e ? a.cap_e : e_tot;
  int rbeg, rend;
  cta_row_range(a.ptr, a.nrows, eff, blockIdx.x, gridDim.x, rbeg, rend);
  int eb = a.ptr[rbeg], ee = a.ptr[rend];
  if (ee > eff) ee = (int)eff;
  if (eb > ee) eb = ee;
  RowReducer red;
  red.init(rbeg);

  for (int t0 = eb; t0 < ee; t0 += TE) {
    int n_e = min(TE, ee - t0);
    __syncthreads();
    tile_geometry(a, t0, n_e, true, s_own, s_nbr, s_d, s_u);
    __syncthreads();
    tile_basis(a, s_d, xb);
    __syncthreads();
    float acc[4][8];
    gemm64<DR, D>(xb, LDR, a.blk.f0_wt, acc);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        int c = gcol<128>(tx, j);
        float z = acc[i][j] + __ldg(&a.blk.f0_b[c]);
        zb[(ty * 4 + i) * LDH + c] = z;
        hb[(ty * 4 + i) * LDH + c] = maybe_q16(ssp(z), a.quant);
      }
    __syncthreads();
    gemm64<D, D>(hb, LDH, a.blk.f1_wt, acc);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int e = ty * 4 + i;
      const float *ghrow = GH + (size_t)s_nbr[e] * D;
      const float *prow = P + (size_t)max(s_own[e], 0) * D;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        int c = gcol<128>(tx, j);
        float w = acc[i][j] + __ldg(&a.blk.f1_b[c]);
        float gh = e < n_e ? __ldg(&ghrow[c]) : 0.f;
        xb[e * LDH + c] = gh * w;              // contribution to grad_P[src]
        hb[e * LDH + c] = gh * __ldg(&prow[c]); // grad_w
      }
    }
    __syncthreads();
    if (threadIdx.x < D) red.tile(xb, s_own, n_e, GP);
    // grad_h = grad_w @ W1, then * ssp'(z0)   (mlp_backward_input, model.py:326-331)
    gemm64<D, D>(hb, LDH, a.blk.f1_w, acc);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        int c = gcol<128>(tx, j);
        float *zp = &zb[(ty * 4 + i) * LDH + c];
        *zp = acc[i][j] * ssp_grad(*zp);
      }
    __syncthreads();
    // grad_b = grad_z0 @ W0; grad_d = sum_k grad_b * db (flash.py:292-293)
    float acc4[4][4];
    gemm64<D, DR>(zb, LDH, a.blk.f0_w, acc4);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int e = ty * 4 + i;
      float d = s_d[e];
      float c, dc;
      envelope(d, a.cutoff, c, dc);
      float part = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int k = tx * 4 + j;
        float dl = d - __ldg(&a.centers[k]);
        float gs = __expf((-a.gamma * dl) * dl);
        float db = gs * ((-2.f * a.gamma) * dl * c + dc);  // model.py:289
        part += acc4[i][j] * db;
      }
#pragma unroll
      for (int o = 8; o >= 1; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (tx == 0 && e < n_e) {
        float inv = d > TINY_DISTANCE ? 1.f / d : 0.f;  // _safe_inv, flash.py:176-178
        float s = part * inv;
        float4 u = s_u[e];
        float4 g = make_float4(s * u.x, s * u.y, s * u.z, 0.f);
        float4 *dst = &gsum[t0 + e];
        if (accumulate) {
          float4 o = *dst;
          g.x += o.x; g.y += o.y; g.z += o.z;
        }
        *dst = g;
      }
    }
  }
  if (threadIdx.x < D) red.finish(rend, GP);
}

// grad_r[x] = sum_{k in row x} (gsum[rev[k]] - gsum[k])  (flash.py:298-299,
// dst-segment sum minus src-segment sum), forces = -grad_r (+ f_extra), then
// optionally the trailing half-kick (md.py:134-138) and the blow-up check
// (md.py:183-185).  FF_LPN lanes per node; single writer per output.
constexpr int FF_LPN = 8;  // lanes per node in k_forces_finish

__device__ __forceinline__ void forces_node(const int32_t *ptr, const int32_t *rev,
                                            const float4 *gsum, const float4 *gr, int N,
                                            int RN, int64_t cap_e,
                                            const float *f_extra, const fcg_prior &pr,
                                            int use_prior, const float *pos, float *forces,
                                            const fcg_md_params &kick, int do_kick,
                                            const float *mass, float *vel, int64_t *status,
                                            const int64_t *step) {
  // FF_LPN lanes per node: each lane gathers up to four of the node's CSR
  // slots per pass with all loads issued before use, then a fixed-order
  // butterfly over the node's lanes (deterministic; replaces a serial
  // per-thread walk, then a warp per node that left lanes and SMs idle)
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int g = (int)(tid / FF_LPN);
  const int lane = threadIdx.x & (FF_LPN - 1);
  float gx = 0.f, gy = 0.f, gz = 0.f;
  if (gr) {  // scatter schedule: grad_r accumulated by atomics in the edge kernels
    if (g < RN && lane == 0) {
      const float4 v = gr[g];
      gx = v.x; gy = v.y; gz = v.z;
    }
  } else if (g < RN && (long long)ptr[RN] <= cap_e) {
    const int k1 = ptr[g + 1];
    for (int k0 = ptr[g] + lane; k0 < k1; k0 += 4 * FF_LPN) {
      int r[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) r[j] = k0 + j * FF_LPN < k1 ? rev[k0 + j * FF_LPN] : -1;
      float4 av[4], bv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        av[j] = r[j] >= 0 ? gsum[r[j]] : make_float4(0.f, 0.f, 0.f, 0.f);
        bv[j] = r[j] >= 0 ? gsum[k0 + j * FF_LPN] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        gx += av[j].x - bv[j].x;
        gy += av[j].y - bv[j].y;
        gz += av[j].z - bv[j].z;
      }
    }
  }
#pragma unroll
  for (int o = FF_LPN / 2; o; o >>= 1) {
    gx += __shfl_xor_sync(0xffffffffu, gx, o);
    gy += __shfl_xor_sync(0xffffffffu, gy, o);
    gz += __shfl_xor_sync(0xffffffffu, gz, o);
  }
  if (lane != 0 || g >= RN) return;
  float f[3] = {-gx, -gy, -gz};
  bool bad = false;
  const int i = g % N;
  float fp[3] = {0.f, 0.f, 0.f};
  if (use_prior) {  // the prior forces of this bead, as k_prior computes them
    const float3 v = prior_bead_force(pr, pos, N, g);
    fp[0] = v.x; fp[1] = v.y; fp[2] = v.z;
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    if (use_prior) f[q] = __fadd_rn(f[q], fp[q]);                    // out.forces + f_prior
    else if (f_extra) f[q] = __fadd_rn(f[q], f_extra[(size_t)g * 3 + q]);
    forces[(size_t)g * 3 + q] = f[q];
    bad |= !(fabsf(f[q]) <= FORCE_BLOWUP_LIMIT);  // catches NaN too
    if (do_kick) {
      float dv = __fdiv_rn(__fmul_rn(kick.half_dt, f[q]), mass[i]);
      vel[(size_t)g * 3 + q] = __fadd_rn(vel[(size_t)g * 3 + q], dv);
    }
  }
  if (bad && status) {
    if (atomicCAS((unsigned long long *)&status[FCG_ST_BLOWUP], 0ull, 1ull) == 0ull)
      status[FCG_ST_BLOWUP_STEP] = step ? *step : 0;
  }
}

// energy[r] = sum_i per_atom[r*N + i] (flash.py:489), fixed tree order.
__device__ __forceinline__ void replica_energy(const float *per_atom, int N, float *energy,
                                               int r) {
  __shared__ float red[256];
  float acc = 0.f;
  for (int i = threadIdx.x; i < N; i += blockDim.x) acc += per_atom[(size_t)r * N + i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) energy[r] = red[0];
}

// Forces and replica energies in one launch (independent outputs): blocks
// [0, nff) run forces_node, the next R blocks replica_energy, and with a
// prior (the fused MD step) the last R blocks the prior energies — the
// prior forces are evaluated inline by forces_node, so the step has no
// separate prior launch.
__global__ void __launch_bounds__(256)
k_forces_finish(const int32_t *ptr, const int32_t *rev, const float4 *gsum, const float4 *gr,
                int N, int RN,
                int64_t cap_e, const float *f_extra, const fcg_prior pr, int use_prior,
                const float *pos, float *e_prior, float *forces, fcg_md_params kick,
                int do_kick, const float *mass, float *vel, int64_t *status, const int64_t *step,
                int nff, int R, const float *per_atom, float *energy) {
  pdl_trigger();
  pdl_wait();
  if ((int)blockIdx.x < nff)
    forces_node(ptr, rev, gsum, gr, N, RN, cap_e, f_extra, pr, use_prior, pos, forces, kick,
                do_kick, mass, vel, status, step);
  else if ((int)blockIdx.x < nff + R)
    replica_energy(per_atom, N, energy, blockIdx.x - nff);
  else
    prior_energy(pr, pos, N, e_prior, blockIdx.x - nff - R);
}

// ---------------------------------------------------------------------------
static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// Edge-kernel implementation: the tcgen05 kernels (edge_tc.cu) are the
// product path; FCG_EDGE_IMPL=simt selects the fp32 FFMA kernels above as a
// diagnostic A/B reference (same results within fp32 round-off).
static bool use_simt_edges() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("FCG_EDGE_IMPL");
    v = (e && e[0] == 's') ? 1 : 0;
  }
  return v == 1;
}

struct EfBuffers {
  float *X, *H, *G, *GH, *GP;
  float *P[FCG_MAX_BLOCKS], *Zp[FCG_MAX_BLOCKS];
  float4 *gsum;
  float4 *gr;  // [RN] grad_r of the scatter schedule
  float4 *geo;
  float2 *env;
  int32_t *unit_rows;
  unsigned int *amax;  // [2*T]: max |P_t|, max |GH_t| (edge-kernel operand bounds)
};

static EfBuffers carve_ef(Carver &c, int T, size_t RN, int64_t cap_e) {
  EfBuffers b;
  size_t rows = (RN + TE - 1) / TE * TE;
  b.X = c.take<float>(rows * D);
  b.H = c.take<float>(rows * D);
  b.G = c.take<float>(rows * D);
  b.GH = c.take<float>(rows * D);
  b.GP = c.take<float>(rows * D);
  for (int t = 0; t < T; ++t) {
    b.P[t] = c.take<float>(rows * D);
    b.Zp[t] = c.take<float>(rows * D);
  }
  b.gsum = c.take<float4>((size_t)cap_e + 1);
  b.gr = c.take<float4>(rows);
  b.geo = c.take<float4>((size_t)cap_e + 1);
  b.env = c.take<float2>((size_t)cap_e + 1);
  b.unit_rows = c.take<int32_t>(4096);  // backward partition at 0, forward at 2048
  b.amax = c.take<unsigned int>(2 * FCG_MAX_BLOCKS);
  return b;
}

size_t ef_ws_bytes(const fcg_model *m, int R, int N, int64_t cap_e) {
  Carver c(nullptr, 0);
  carve_ef(c, m ? m->num_blocks : FCG_MAX_BLOCKS, (size_t)R * N, cap_e);
  return c.off + 256;
}

static bool smem_configured = false;
static void configure_smem() {
  if (smem_configured) return;
  size_t big = 3 * TE * LDH * sizeof(float);
  cudaFuncSetAttribute(k_edge_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)big);
  cudaFuncSetAttribute(k_edge_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)((TE * LDR + TE * LDH) * sizeof(float)));
  cudaFuncSetAttribute(k_node_post, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(2 * TE * LDH * sizeof(float)));
  cudaFuncSetAttribute(k_node_post_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(2 * TE * LDH * sizeof(float)));
  cudaFuncSetAttribute(k_readout, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)((TE * LDH + TE * LDR) * sizeof(float)));
  cudaFuncSetAttribute(k_node_linear<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(TE * LDH * sizeof(float)));
  cudaFuncSetAttribute(k_node_linear<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(TE * LDH * sizeof(float)));
  smem_configured = true;
}

// FCG_NODE_FUSE=0: one launch per node stage (A/B)
static bool node_fuse_enabled() {
  static const bool on = [] {
    const char *v = getenv("FCG_NODE_FUSE");
    return !(v && v[0] == '0');
  }();
  return on;
}

int energy_forces(const fcg_model *m, const float *pos, const int32_t *types, int R, int N,
                  const int32_t *ptr, const int32_t *nbr, const int32_t *rev,
                  const int32_t *own, int64_t cap_e, float *per_atom, float *energy,
                  float *forces, void *ws, size_t ws_bytes, cudaStream_t s,
                  const float *f_extra, const fcg_md_params *kick, const float *mass,
                  float *vel, int64_t *status, const int64_t *step, int schedule,
                  const fcg_prior *prior, float *prior_e, const NbrDefer *defer) {
  if (!m || m->num_blocks < 0 || m->num_blocks > FCG_MAX_BLOCKS) {
    set_error("energy_forces: bad model descriptor");
    return FCG_ERR_ARG;
  }
  if (m->format != FCG_FMT_FP32 && m->format != FCG_FMT_W16) {
    set_error("energy_forces: unknown weight format");
    return FCG_ERR_ARG;
  }
  const int T = m->num_blocks;
  const int RN = R * N;
  Carver c(ws, ws_bytes);
  EfBuffers b = carve_ef(c, T, (size_t)RN, cap_e);
  if (!c.ok()) { set_error("energy_forces: workspace too small"); return FCG_ERR_ARG; }
  configure_smem();

  const int node_grid = ceil_div(RN, TE);
  const size_t sm1 = TE * LDH * sizeof(float), sm2 = 2 * sm1;

  EdgeArgs ea;
  ea.pos = pos; ea.ptr = ptr; ea.nbr = nbr; ea.own = own; ea.nrows = RN; ea.cap_e = cap_e;
  ea.cutoff = m->cutoff; ea.gamma = m->gamma; ea.centers = m->centers;
  const int quant = m->format == FCG_FMT_W16;
  ea.quant = quant;
  ea.dbg = g_dbg_phase;
  if (schedule != FCG_SCHED_SEGRED && schedule != FCG_SCHED_SCATTER) {
    set_error("energy_forces: unknown schedule");
    return FCG_ERR_ARG;
  }
  // the fused-scatter ablation (flash.py:373-443) runs the 64-edge tcgen05 kernels
  const bool scatter = schedule == FCG_SCHED_SCATTER;
  const bool simt = !scatter && use_simt_edges();
  if (scatter) cudaMemsetAsync(b.gr, 0, sizeof(float4) * (size_t)RN, s);
  const int eg = simt ? 2 * sm_count() : sm_count();
  // block 0's pre-linear comes from the per-type table when the model has
  // one (tcgen05 path: k_edge_geom gathers it with the embedding)
  const bool p0_tab = m->pre0_table != nullptr && T > 0;
  const EmbedJob ej{m->embedding, types, N, b.X, b.amax, 2 * FCG_MAX_BLOCKS,
                    m->pre0_table, p0_tab ? b.P[0] : nullptr, m->pre0_amax};
  const bool deferred = defer && defer->active;  // nbr_build left its assembly to us
  if (deferred && simt) {
    FCG_PROF(P_NBR_FILL, s);
    launch_nbr_assemble(*defer, GeomJob{}, s);
  }
  if (simt) {  // the tcgen05 path does the lookup inside k_edge_geom
    FCG_PROF(P_EMBED, s);
    launch_pdl(PDL_SMALL, k_embed, ceil_div((long long)RN * (D / 4), 256), 256, 0, s, m->embedding,
               types, N, RN, b.X, b.amax, 2 * FCG_MAX_BLOCKS);
  }
  if (!simt) {
    edge_tc_configure();
    node_tc_configure();
    if (deferred) {  // one launch: CSR assembly + geometry + unit rows + embedding
      FCG_PROF(P_NBR_FILL, s);
      const GeomJob gj{pos, m->cutoff, b.geo, b.env, {b.unit_rows, b.unit_rows + 2048},
                       {edge_tc_units(eg), edge_tc_units_fwd(eg)}, ej};
      launch_nbr_assemble(*defer, gj, s);
    } else {
      FCG_PROF(P_EDGE_GEOM, s);
      launch_edge_geom(ea, b.geo, b.env, b.unit_rows, edge_tc_units(eg), b.unit_rows + 2048,
                       edge_tc_units_fwd(eg), ej, s);
    }
  }

  // fused node launches (tcgen05 path): post(t) + pre(t+1), post(T-1) +
  // readout + post_bwd(T-1), pre_bwd(t) + post_bwd(t-1)
  const bool nfuse = !simt && node_fuse_enabled() && T > 0;
  for (int t = 0; t < T; ++t) {
    const fcg_block &blk = m->blocks[t];
    ea.blk = blk;
    ea.amax_pg = b.amax + 2 * t;
    if (!(t == 0 && p0_tab && !simt) && !(nfuse && t > 0)) {
      FCG_PROF(P_NODE_PRE, s);
      if (simt)
        k_node_linear<true, false><<<node_grid, NT, sm1, s>>>(b.X, blk.pre_wt, blk.pre_b, b.P[t],
                                                             RN, quant);
      else
        launch_node_pre_tc(b.X, blk, quant, b.P[t], RN, b.amax + 2 * t, s);
    }
    {
      FCG_PROF(P_EDGE_FWD, s);
      if (simt)
        k_edge_fwd<<<eg, NT, (TE * LDR + TE * LDH) * sizeof(float), s>>>(ea, b.P[t], b.H);
      else
      {
        if (scatter) cudaMemsetAsync(b.H, 0, sizeof(float) * (size_t)RN * D, s);
        launch_edge_fwd_tc(ea, b.geo, b.env, b.unit_rows + 2048, b.P[t], b.H, eg, s, scatter);
      }
    }
    if (nfuse && t + 1 < T) {
      FCG_PROF(P_NODE_POST, s);
      launch_node_post_pre_tc(b.H, blk, m->blocks[t + 1], quant, b.Zp[t], b.X, b.P[t + 1], RN,
                              ptr, b.amax + 2 * (t + 1), s);
    } else if (nfuse) {
      FCG_PROF(P_NODE_POST, s);
      launch_node_post_readout_tc(b.H, blk, *m, quant, b.Zp[t], b.X, per_atom, b.G, b.GH, RN,
                                  ptr, b.amax + 2 * t + 1, s);
    } else {
      FCG_PROF(P_NODE_POST, s);
      if (simt)
        k_node_post<<<node_grid, NT, sm2, s>>>(b.H, blk, b.Zp[t], b.X, RN, quant);
      else
        launch_node_post_tc(b.H, blk, quant, b.Zp[t], b.X, RN, ptr, s);
    }
  }
  if (!nfuse) {
    FCG_PROF(P_READOUT, s);
    if (simt)
      k_readout<<<node_grid, NT, (TE * LDH + TE * LDR) * sizeof(float), s>>>(b.X, *m, per_atom,
                                                                             b.G, RN);
    else
      launch_readout_tc(b.X, *m, per_atom, b.G, RN, s);
  }
  for (int t = T - 1; t >= 0; --t) {
    const fcg_block &blk = m->blocks[t];
    ea.blk = blk;
    ea.amax_pg = b.amax + 2 * t;
    if (!nfuse) {  // (fused: done by the launch before)
      FCG_PROF(P_NODE_POST_BWD, s);
      if (simt)
        k_node_post_bwd<<<node_grid, NT, sm2, s>>>(b.G, blk, b.Zp[t], b.GH, RN);
      else
        launch_node_post_bwd_tc(b.G, blk, quant, b.Zp[t], b.GH, RN, b.amax + 2 * t + 1, s);
    }
    {
      FCG_PROF(P_EDGE_BWD, s);
      if (simt)
        k_edge_bwd<<<eg, NT, 3 * TE * LDH * sizeof(float), s>>>(ea, b.P[t], b.GH, b.GP, b.gsum,
                                                               t != T - 1);
      else
      {
        if (scatter) cudaMemsetAsync(b.GP, 0, sizeof(float) * (size_t)RN * D, s);
        launch_edge_bwd_tc(ea, b.geo, b.env, b.unit_rows, b.P[t], b.GH, b.GP, b.gsum, t != T - 1,
                           eg, s, scatter ? b.gr : nullptr);
      }
    }
    // grad_X of block 0 (flash.py:300) is the gradient with respect to the
    // embedding output, which has no position dependence: forces never read
    // it, so the last pre-linear backward is skipped
    if (t > 0 && nfuse) {
      FCG_PROF(P_NODE_PRE_BWD, s);
      const fcg_block &prv = m->blocks[t - 1];
      launch_node_prebwd_postbwd_tc(b.GP, blk, prv, quant, b.G, b.Zp[t - 1], b.GH, RN, ptr,
                                    b.amax + 2 * (t - 1) + 1, s);
    } else if (t > 0) {
      FCG_PROF(P_NODE_PRE_BWD, s);
      if (simt)
        k_node_linear<false, true><<<node_grid, NT, sm1, s>>>(b.GP, blk.pre_w, nullptr, b.G, RN, 0);
      else
        launch_node_pre_bwd_tc(b.GP, blk, quant, b.G, RN, ptr, s);
    }
  }
  if (T == 0) cudaMemsetAsync(b.gsum, 0, sizeof(float4) * (size_t)(cap_e + 1), s);
  fcg_md_params kp{};
  if (kick) kp = *kick;
  FCG_PROF(P_FORCES, s);
  const int nff = (int)ceil_div((long long)RN * FF_LPN, 256);
  fcg_prior pr{};
  if (prior) pr = *prior;
  const int use_prior = prior != nullptr;
  launch_pdl(PDL_SMALL, k_forces_finish, nff + R + (use_prior ? R : 0), 256, 0, s, ptr, rev,
             b.gsum, (const float4 *)(scatter ? b.gr : nullptr), N, RN, cap_e, f_extra, pr,
             use_prior, pos, prior_e, forces, kp, (int)(kick != nullptr), mass, vel, status, step,
             nff, R, per_atom, energy);
  return cuda_status("energy_forces");
}

}  // namespace fcg
