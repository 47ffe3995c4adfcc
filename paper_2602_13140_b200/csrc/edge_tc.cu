// (b)(c)(d) Fused edge passes on the 5th-generation tensor cores.
//
// Same contract as the fused edge loop of the reference (flash.py:215-236
// forward, :272-295 backward) — edge tensors never reach HBM — with the
// per-edge filter-MLP GEMMs on tcgen05.mma (kind::f16, fp32 accumulate in
// TMEM).
//
// Formulation ("transposed"): D[channel][edge] = W[channel][k] * X[k][edge].
//   A = weights, resident in SMEM for the whole kernel (K-major in the
//       forward; the SAME bytes read MN-major give W^T for the backward);
//   B = per-tile edge activations written by the epilogue threads
//       (MN-major: row = channel, contiguous edges);
//   D = TMEM, lane = channel, column = edge.
//
// Work decomposition: a CTA (one per SM, 16 warps) hosts four independent
// groups of 4 warps (one warp per TMEM lane quarter).  All groups read the
// same resident weights; each owns a range of whole CSR rows (balanced by
// edge count), walks it in 32-edge tiles, and has its own B-operand
// buffers, 128 TMEM columns and mbarriers, so the MMA and gather latency of
// one group hides under the epilogues of the other three.  Inside a group
// every thread owns one channel across all 32 edges of a tile, so the
// destination (forward) / source (backward) segment reduction is a running
// sum per thread with a single store per CSR row — no atomics, no
// cross-thread merge.
//
// No barriers inside a group: every warp keeps a private copy of the tile
// metadata, and when a warp has written its quarter of a GEMM's B operand it
// bumps that GEMM kind's arrival counter; the LAST of the four warps to
// arrive issues the tcgen05.mma chain and commits it to the kind's
// mbarrier, on which each warp waits on its own.  Same-kind requests are
// ordered by those completion waits, so a counter per kind (mod 4) suffices.
//
// fp32 parity (SURVEY §7 hard part 2): plain fp16/TF32 operands lose ~1e-3;
// both operands are split as x*2^s = hi + lo (fp16 each, ~22 significant
// bits) and we accumulate hi*hi + hi*lo + lo*hi.  Weights carry a
// host-chosen power-of-two prescale.  Activation scales are static too —
// chosen from bounds (host: h from the filter-0 weights, db from gamma and
// r_cut; device: grad_w from max|GH| * max|P| written by the node kernels) —
// so no tile needs a max-reduction barrier; the absolute split error stays
// <= bound * 2^-39.  W16 weights (quantize.py) use the stored fp16 weights
// directly: one MMA in the forward (inputs rounded to fp16 as the reference
// does), two in the backward, dequant scales applied per channel.
//
// Backward (flash_block_backward): grad_d = sum_k grad_b[k] db[k] with
// grad_b = W0^T gz is evaluated in forward mode as grad_d = sum_c gz[c] *
// dz0[c] with dz0 = W0 db (one more K=64 GEMM, G1'), so gz never becomes a
// tensor-core operand and the reduction over channels is a warp transpose-sum.
#include <cuda_fp16.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc.cuh"
#include "tc_ops.cuh"
#include "geom.cuh"

namespace fcg {

constexpr int TT = 32;           // edges per tile (MMA N)
constexpr int NGRP = 4;          // independent warp groups per CTA (backward)
// The forward's TMEM map and aliased smem layout also fit a fifth group
// (-DFCG_FWD_GROUPS=5: 640 threads at 96 registers), measured slower
// (1.136 vs 1.111 ms/step: the spills cost more than the extra warps hide).
#ifndef FCG_FWD_GROUPS
#define FCG_FWD_GROUPS 4
#endif
constexpr int FWD_NGRP = FCG_FWD_GROUPS;
constexpr int MAX_NGRP = FWD_NGRP > NGRP ? FWD_NGRP : NGRP;
constexpr int GT = 128;          // threads per group: one warp per TMEM lane quarter
constexpr int TC_THREADS = NGRP * GT;
constexpr int FWD_THREADS = FWD_NGRP * GT;
constexpr uint32_t KSTR = (TT / 8) * 128;  // B operand bytes per 8 K-rows
constexpr uint32_t SM_W0 = 0;          // W0 hi|lo: 2 x 128x64 fp16
constexpr uint32_t SM_W1 = 32768;      // W1 hi|lo: 2 x 128x128 fp16
constexpr uint32_t SM_BUF = 98304;     // per group: basis buffer (K=64) + act buffer (K=128)
constexpr uint32_t BB_BYTES = 2 * DR * TT * 2;  // basis / db hi|lo: 8 KB
constexpr uint32_t HB_BYTES = 2 * D * TT * 2;   // h / grad_w hi|lo: 16 KB
constexpr uint32_t GBUF_BYTES = BB_BYTES + HB_BYTES;
constexpr uint32_t SM_META = SM_BUF + NGRP * GBUF_BYTES;
constexpr uint32_t W0_BYTES = D * DR * 2, W1_BYTES = D * D * 2;
// forward TMEM slots inside a group's columns: z0 | w
constexpr uint32_t S0 = 0, S1 = 32;
enum { BAR_G1 = 0, BAR_G2 = 1, BAR_G3 = 2, BAR_G1P = 3 };

constexpr int NWARP = MAX_NGRP * GT / 32;
struct WarpMeta {  // one tile, private to a warp (double-buffered)
  int own[TT], nbr[TT];  // nbr holds row offsets nbr * D
  float d[TT], env[TT], denv[TT];
};
struct TcShared {
  WarpMeta wm[NWARP][2];
  float xg[MAX_NGRP][2][4][TT];   // per-quarter partial grad_d (double-buffered)
  uint64_t bar[MAX_NGRP][4];      // GEMM completion, per kind
  uint64_t xbar[MAX_NGRP];        // the four partial grad_d rows of a tile are written
  uint64_t wbar;                  // filter weight images landed (bulk copy)
  unsigned int req[MAX_NGRP][4];  // operand arrivals per GEMM kind (mod 4)
  uint32_t tmem;
};
constexpr uint32_t SM_TOTAL = SM_META + sizeof(TcShared);
static_assert(SM_TOTAL + 1024 <= 232448, "shared memory budget");
// Forward layout: group buffers from offset 0; the weight images are staged
// over them (SM_W0/SM_W1 < FWD_SM_META) and moved to TMEM before any group
// writes its buffers.
constexpr uint32_t FWD_SM_BUF = 0;
constexpr uint32_t FWD_SM_META = FWD_SM_BUF + FWD_NGRP * GBUF_BYTES;
constexpr uint32_t FWD_SM_TOTAL = FWD_SM_META + sizeof(TcShared);
static_assert(SM_W1 + 2 * W1_BYTES <= FWD_SM_META, "forward staging aliases the group buffers");
static_assert(FWD_SM_TOTAL + 1024 <= 232448, "forward shared memory budget");

// ---- CSR segment sums -------------------------------------------------------
// Running sum of one channel over edges in CSR order; each completed row is
// stored once.  Rows are warp-uniform (all lanes walk the same edges).  Rows
// without edges are never written: the node kernel that consumes the sums
// reads them as zero through the CSR degree (an empty segment sums to 0,
// flash.py:109-135), so the walk needs no zero-fill branches.
struct SegSum {
  int row;       // row of the open segment (-1: the unit has no edges)
  float acc;
  float *outc;   // out + channel
  // Tile of TT edges in CSR order with rows own[] (padding edges repeat the
  // last valid row and carry m = 0).
  __device__ __forceinline__ void tile(const int *own, const float (&m)[TT]) {
    // All lanes walk the same edges, so the edges that start a new row form
    // one warp-uniform mask (a ballot): halves without a row start are a
    // tree sum, others test a uniform bit per edge instead of comparing rows.
    const int lane = threadIdx.x & 31;
    const int cur = own[lane];
    const unsigned starts = __ballot_sync(0xffffffffu, cur != (lane ? own[lane - 1] : row));
#pragma unroll
    for (int h = 0; h < TT; h += 16) {
      const unsigned hb = (starts >> h) & 0xffffu;
      if (hb == 0u) {  // the open row continues through all 16 edges
        float s[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] = m[h + i] + m[h + i + 8];
#pragma unroll
        for (int i = 0; i < 4; ++i) s[i] += s[i + 4];
        acc += (s[0] + s[2]) + (s[1] + s[3]);
      } else {
        block8(own, &m[h], h, hb & 0xffu);
        block8(own, &m[h + 8], h + 8, hb >> 8);
      }
    }
  }
  // Eight edges h0.. with row-start bits b8: a tree sum when no row starts
  // among them (most 8-edge blocks at ~23 edges per row), else the walk.
  __device__ __forceinline__ void block8(const int *own, const float *m, int h0, unsigned b8) {
    if (b8 == 0u) {
      acc += ((m[0] + m[4]) + (m[2] + m[6])) + ((m[1] + m[5]) + (m[3] + m[7]));
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if ((b8 >> i) & 1u) {  // edge h0+i starts a row (warp-uniform)
          if (row >= 0) outc[(uint32_t)row * D] = acc;
          row = own[h0 + i];
          acc = 0.f;
        }
        acc += m[i];
      }
    }
  }
  // The same walk split in two: starts(own) once per tile, then half(h)
  // for edges h..h+15 (h = 0, 16) with only those 16 values live.
  __device__ __forceinline__ unsigned starts(const int *own) const {
    const int lane = threadIdx.x & 31;
    const int cur = own[lane];
    return __ballot_sync(0xffffffffu, cur != (lane ? own[lane - 1] : row));
  }
  // starts() for a tile whose slots from n_e on are padding: they never
  // start a row (their messages are zero).
  __device__ __forceinline__ unsigned starts_n(const int *own, int n_e) const {
    const int lane = threadIdx.x & 31;
    const int cur = own[lane];
    return __ballot_sync(0xffffffffu,
                         lane < n_e && cur != (lane ? own[lane - 1] : row));
  }
  __device__ __forceinline__ void half(const int *own, const float (&m)[16], int h,
                                       unsigned st) {
    const unsigned hb = (st >> h) & 0xffffu;
    if (hb == 0u) {
      float s[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) s[i] = m[i] + m[i + 8];
#pragma unroll
      for (int i = 0; i < 4; ++i) s[i] += s[i + 4];
      acc += (s[0] + s[2]) + (s[1] + s[3]);
    } else {
      block8(own, &m[0], h, hb & 0xffu);
      block8(own, &m[8], h + 8, hb >> 8);
    }
  }
  __device__ __forceinline__ void finish() {
    if (row >= 0) outc[(uint32_t)row * D] = acc;
  }
};

// Atomic scatter of one tile (the "fused but scatter" ablation schedule,
// flash.py:373-443: np.add.at per tile instead of segment sums): every valid
// edge adds its message to its row with a red.global.add; the 32 lanes of a
// warp hold 32 consecutive channels of one row, so each instruction is one
// coalesced 128-byte reduction.  Summation order is the arrival order.
__device__ __forceinline__ void scatter_tile(float *outc, const int *own, const float (&m)[TT],
                                             int n_e) {
#pragma unroll
  for (int i = 0; i < TT; ++i)
    if (i < n_e) atomicAdd(outc + (uint32_t)own[i] * D, m[i]);
}

// ---- per-step edge geometry (the reference's d cache, flash.py:221-223) ------
// geo[k] = (u, d) with u = r[own] - r[nbr] for CSR slot k; env[k] = (C, C').
// Also the row range of every work unit, balanced by edge count, for the
// edge launches that follow: unit u starts at the first row r with
// ptr[r] >= t_u = e_tot * u / G (cta_row_range's split).  Each row writes the
// boundaries t_u in (ptr[r-1], ptr[r]] — one coalesced pass instead of G
// dependent binary searches.
__global__ void __launch_bounds__(256)
k_edge_geom(const float *pos, const int32_t *ptr, const int32_t *nbr, const int32_t *own,
            int nrows, int64_t cap_e, float cutoff, float4 *geo, float2 *env,
            int32_t *unit_rows, int nunits, int32_t *unit_rows2, int nunits2, const EmbedJob ej) {
  pdl_trigger();
  pdl_wait();
  __syncthreads();  // keeps ptxas from hoisting loads above the wait
  long long e_tot = ld_dep(&ptr[nrows]);
  if (e_tot > cap_e) e_tot = cap_e;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x,
                  nt = (long long)gridDim.x * blockDim.x;
  for (long long r = t; r <= nrows; r += nt) {
    const long long lo = r == 0 ? -1 : ld_dep(&ptr[r - 1]), hi = ld_dep(&ptr[r]);
    unit_rows_at(r, lo, hi, e_tot, unit_rows, nunits, nrows);    // backward (4 groups)
    unit_rows_at(r, lo, hi, e_tot, unit_rows2, nunits2, nrows);  // forward partition
  }
  for (long long k = t; k < e_tot; k += nt) edge_geom_one(pos, own[k], nbr[k], cutoff, geo, env, k);
  embed_rows(ej, nrows, t, nt, blockIdx.x == 0);
}

// ---- descriptors and MMA chains ------------------------------------------------
// A descriptor pair (hi image, lo image) and its advance per 16 K-values, in
// the 16-byte units of the descriptor's address field (smem < 256 KB, so the
// field never carries into LBO).
struct Desc {
  uint64_t hi, lo;
  uint32_t step;
};
__device__ __forceinline__ Desc wdesc_k(uint32_t base, int in_dim, uint32_t lo_off) {
  return {desc_w_kmajor(base, in_dim, 0), desc_w_kmajor(base + lo_off, in_dim, 0), 16u};
}
__device__ __forceinline__ Desc wdesc_mn(uint32_t base, int in_dim, uint32_t lo_off) {
  return {desc_w_mnmajor(base, in_dim, 0), desc_w_mnmajor(base + lo_off, in_dim, 0),
          (uint32_t)(in_dim >> 3) * 128u * 2u / 16u};
}
template <uint32_t KS = KSTR>
__device__ __forceinline__ Desc adesc(uint32_t base, int K) {
  return {desc_act(base, 0, KS), desc_act(base + (uint32_t)K * (KS >> 3), 0, KS), 2u * KS / 16u};
}
// D (+)= A x B over KS k-steps with the product set {hi*hi, hi*lo, lo*hi}
// truncated to NP terms.  Issued by one lane; the k loop stays rolled to keep
// the kernel's code (and i-cache footprint) small.
template <int KS, int NP>
__device__ __forceinline__ void mma_chain(uint32_t d, Desc a, Desc b, uint32_t idesc) {
#pragma unroll 1
  for (int k = 0; k < KS; ++k) {
    tc::mma_f16_ss_warp(d, a.hi, b.hi, idesc, k > 0);
    if (NP >= 2) tc::mma_f16_ss_warp(d, a.hi, b.lo, idesc, 1);
    if (NP >= 3) tc::mma_f16_ss_warp(d, a.lo, b.hi, idesc, 1);
    a.hi += a.step; a.lo += a.step;
    b.hi += b.step; b.lo += b.step;
  }
}

// Store 8 consecutive edges e0.. of K-row r of a B operand (hi image, and
// the lo image K*KSTR/8 bytes further when LO), values times `scale`.
// PK: the lo residual of a pair in one packed FADD (the WS kernels; the
// older kernels keep the scalar form, whose register allocation it upsets).
template <bool LO, uint32_t KS = KSTR, bool PK = false>
__device__ __forceinline__ void put8(uint8_t *act, int K, int r, int e0, const float *v,
                                     float scale) {
  const uint32_t off = (uint32_t)(r >> 3) * KS + (uint32_t)(e0 >> 3) * 128u + (uint32_t)(r & 7) * 16u;
  __half2 hi[4], lo[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float a = v[2 * i] * scale, b = v[2 * i + 1] * scale;
    hi[i] = __floats2half2_rn(a, b);
    if (LO && PK) {  // x - hi is exact: same bits as the scalar form
      const float2 l = fma2(__half22float2(hi[i]), f2(-1.f), make_float2(a, b));
      lo[i] = __floats2half2_rn(l.x, l.y);
    } else if (LO) {
      const float2 hf = __half22float2(hi[i]);
      lo[i] = __floats2half2_rn(a - hf.x, b - hf.y);
    }
  }
  *(uint4 *)(act + off) = *(uint4 *)hi;
  if (LO) *(uint4 *)(act + (uint32_t)K * (KS >> 3) + off) = *(uint4 *)lo;
}

// ---- per-warp context ----------------------------------------------------------
struct Wctx {
  int w, g, q, lane, ch;
  int eo;          // first edge column of this warp's tile part in the B operand
  unsigned amask;  // arrivals per GEMM request - 1 (warps of a group - 1)
  uint32_t tl;      // TMEM address of this warp's lane quarter at the group's columns
  uint32_t tmem_g;  // TMEM address of the group's columns, lane 0
  uint8_t *bb, *hb;
  uint32_t sbb, shb;
  TcShared *sh;
  __device__ __forceinline__ WarpMeta *meta(int it) const { return &sh->wm[w][it & 1]; }
  __device__ __forceinline__ void wait(int which, int it) const {
    tc::mbar_wait(&sh->bar[g][which], (uint32_t)(it & 1));
    tc::fence_after_sync();
  }
  // This warp's part of a GEMM's operands is written (smem) and its TMEM
  // reads of the columns the GEMM overwrites are done.  True (warp-uniform)
  // for the last of the group's four warps to arrive: that warp issues (one
  // elected lane per instruction).
  // arrive() with the request counters passed explicitly (kernels whose
  // shared layout is not TcShared)
  __device__ __forceinline__ bool arrive_fm(unsigned int *req, int kind) const {
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncwarp();
    unsigned int old = 0u;
    if (lane == 0) {
      __threadfence_block();
      old = atomicAdd(&req[kind], 1u);
    }
    const bool last = (__shfl_sync(0xffffffffu, old, 0) & amask) == amask;  // warp-uniform
    if (last) {
      __threadfence_block();
      tc::fence_after_sync();
    }
    return last;
  }
  __device__ __forceinline__ bool arrive(int kind) const {
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncwarp();
    unsigned int old = 0u;
    if (lane == 0) {
      __threadfence_block();
      old = atomicAdd(&sh->req[g][kind], 1u);
    }
    const bool last = (__shfl_sync(0xffffffffu, old, 0) & amask) == amask;  // warp-uniform
    if (last) {
      __threadfence_block();
      tc::fence_after_sync();
    }
    return last;
  }
};

#define REQ(kind, CHAIN)                              \
  do {                                                \
    if (W.arrive(kind)) {                             \
      CHAIN;                                          \
      tc::mma_commit_warp(&W.sh->bar[W.g][kind]);     \
    }                                                 \
    __syncwarp();                                     \
  } while (0)

__device__ __forceinline__ Wctx make_wctx(uint8_t *sm, TcShared *sh, uint32_t gcols,
                                          uint32_t buf_base) {
  Wctx W;
  // warp index through a shuffle: the compiler then knows it (and every
  // address derived from it) is warp-uniform, so MMA descriptors stay in
  // uniform registers instead of an R2UR waterfall per tcgen05.mma
  W.w = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  W.g = W.w >> 2;
  W.q = W.w & 3;
  W.lane = threadIdx.x & 31;
  W.ch = 32 * W.q + W.lane;
  W.eo = 0;
  W.amask = 3u;
  W.sh = sh;
  W.bb = sm + buf_base + W.g * GBUF_BYTES;
  W.hb = W.bb + BB_BYTES;
  W.sbb = tc::smem_u32(W.bb);
  W.shb = tc::smem_u32(W.hb);
  W.tmem_g = sh->tmem + gcols * W.g;
  W.tl = W.tmem_g + ((uint32_t)(32 * W.q) << 16);
  return W;
}

// The filter weight images are staged by the TMA engine (cp.async.bulk);
// every thread waits on wbar before reading them.
__device__ __forceinline__ void kernel_prologue(uint8_t *sm, TcShared *sh, const fcg_block &b,
                                                int ngrp) {
  if (threadIdx.x == 0) {
    tc::mbar_init(&sh->wbar, 1);
    tc::fence_mbar_init();
    tc::mbar_expect_tx(&sh->wbar, 2 * W0_BYTES + 2 * W1_BYTES);
    tc::bulk_g2s(sm + SM_W0, b.f0_img, 2 * W0_BYTES, &sh->wbar);
    tc::bulk_g2s(sm + SM_W1, b.f1_img, 2 * W1_BYTES, &sh->wbar);
  }
  if ((int)threadIdx.x < ngrp) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      tc::mbar_init(&sh->bar[threadIdx.x][i], 1);
      sh->req[threadIdx.x][i] = 0u;
    }
    tc::mbar_init(&sh->xbar[threadIdx.x], 4);
    tc::fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&sh->tmem);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
}

// ---- weights as the TMEM-resident A operand ----------------------------------------
// Row m of a weight lives in lane m, element k in column k/2 (pinned by
// tests/test_gpu_tcgen05.py::test_a_operand_in_tmem), so an MMA reads its A
// slice from TMEM and only B (1 KB per MMA) from shared memory, instead of
// 4 KB of A + 1 KB of B.  The images are staged in shared memory by the bulk
// copy of kernel_prologue and moved to TMEM by the lanes that own the rows.
// Forward columns: [TW0, TW0+64) W0 hi | lo (K=64: 32 columns each),
// [TW1, TW1+128) W1 hi | lo (K=128).
constexpr uint32_t FWD_GCOLS = 64;  // forward groups: slots S0, S1 only
constexpr uint32_t TW0 = FWD_NGRP * FWD_GCOLS, TW1 = TW0 + 64;
static_assert(TW1 + 128 <= 512, "TMEM budget");

// Row m of a staged core-matrix image with K inputs (element (r,c) at
// ((r/8)*(K/8)+c/8)*64 + (r%8)*8 + c%8) -> TMEM columns from taddr; TRANS
// moves row m of W^T (column m of a square image) instead.
template <bool TRANS>
__device__ __forceinline__ void image_row_to_tmem(const uint16_t *img, int K, int m,
                                                  uint32_t taddr) {
#pragma unroll 1
  for (int c0 = 0; c0 < K / 2; c0 += 16) {  // 16 columns = 32 K-values
    float v[16];
    if (!TRANS) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint4 u = *(const uint4 *)(img + ((m / 8) * (K / 8) + c0 / 4 + j) * 64 + (m % 8) * 8);
        v[4 * j] = __uint_as_float(u.x); v[4 * j + 1] = __uint_as_float(u.y);
        v[4 * j + 2] = __uint_as_float(u.z); v[4 * j + 3] = __uint_as_float(u.w);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int k = 2 * (c0 + j);  // W^T[m][k] = W[k][m], k and k+1 in one column
        const uint32_t e0 = img[((k / 8) * (K / 8) + m / 8) * 64 + (k % 8) * 8 + m % 8];
        const uint32_t e1 = img[(((k + 1) / 8) * (K / 8) + m / 8) * 64 + ((k + 1) % 8) * 8 + m % 8];
        v[j] = __uint_as_float(e0 | (e1 << 16));
      }
    }
    tc::tmem_st16(taddr + c0, v);
  }
}

// End of the static prologue: TMEM stores done, then the PDL wait right
// before a block barrier (ptxas does not hoist loads across bar.sync, while
// it does move ld.global.nc across griddepcontrol.wait alone;
// tools/check_pdl.py / tests/test_host.py check the SASS).
__device__ __forceinline__ void prologue_done() {
  tc::tmem_st_wait();
  tc::fence_before_sync();
  pdl_wait();
  __syncthreads();
  tc::fence_after_sync();
}

// Forward: warp w moves image (w / 4) % 4 (W0 hi, W0 lo, W1 hi, W1 lo) for
// its lane quarter.
__device__ __forceinline__ void load_fwd_weights_tmem(const uint8_t *sm, uint32_t tmem) {
  const int w = threadIdx.x >> 5, q = w & 3, m = 32 * q + (threadIdx.x & 31);
  const int img = (w >> 2) & 3;
  const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
  if (w >= 16) {
    // a fifth group has nothing to move
  } else if (img < 2)
    image_row_to_tmem<false>((const uint16_t *)(sm + SM_W0 + (img & 1) * W0_BYTES), DR, m,
                             lane_base + TW0 + (img & 1) * (DR / 2));
  else
    image_row_to_tmem<false>((const uint16_t *)(sm + SM_W1 + (img & 1) * W1_BYTES), D, m,
                             lane_base + TW1 + (img & 1) * (D / 2));
  prologue_done();
}

// D (+)= A(TMEM columns a_hi / a_lo) x B over KS k-steps (8 A columns each)
template <int KS, int NP>
__device__ __forceinline__ void mma_chain_ts(uint32_t d, uint32_t a_hi, uint32_t a_lo, Desc b,
                                             uint32_t idesc) {
#pragma unroll 1
  for (int k = 0; k < KS; ++k) {
    tc::mma_f16_ts_warp(d, a_hi + 8 * k, b.hi, idesc, k > 0);
    if (NP >= 2) tc::mma_f16_ts_warp(d, a_hi + 8 * k, b.lo, idesc, 1);
    if (NP >= 3) tc::mma_f16_ts_warp(d, a_lo + 8 * k, b.hi, idesc, 1);
    b.hi += b.step; b.lo += b.step;
  }
}

// Raw per-edge metadata of one tile, one lane per edge, held in registers a
// tile ahead of use so the global-load latency stays off the critical path.
struct MetaRegs {
  int o, n, n_e;
  float4 g;
  float2 c;
  __device__ __forceinline__ void load(const EdgeArgs &a, const float4 *geo,
                                       const float2 *env, int t0, int count,
                                       int lane) {
    n_e = count;
    o = -1; n = 0;
    g = make_float4(0.f, 0.f, 0.f, 0.f);
    c = make_float2(0.f, 0.f);
    if (lane < count) {
      o = a.own[t0 + lane];
      n = a.nbr[t0 + lane];
      g = geo[t0 + lane];
      c = env[t0 + lane];
    }
  }
  // Into the warp's private metadata.  Padding edges get nbr = 0, zero
  // geometry and the last valid edge's row.  Returns the lane's (u, d) for
  // the g_e epilogue (u flipped for src-owned rows: the backward edge has
  // dst = nbr, src = own, u = r_nbr - r_own, flash.py:279); `rows2` tells
  // whether the tile's edges fall in at most two CSR rows (first and last).
  __device__ __forceinline__ float4 store(WarpMeta *m, bool src_owned, int lane,
                                          bool &rows2) const {
    const int first = __shfl_sync(0xffffffffu, o, 0);
    const int last = __shfl_sync(0xffffffffu, o, max(n_e - 1, 0));
    rows2 = __all_sync(0xffffffffu, lane >= n_e || o == first || o == last);
    m->own[lane] = lane < n_e ? o : last;  // padding edges extend the last row (m = 0)
    m->nbr[lane] = n * D;  // row offset of the gathered operand (P[src] / GH[dst])
    m->d[lane] = g.w;
    m->env[lane] = c.x;
    m->denv[lane] = c.y;
    __syncwarp();
    return src_owned ? make_float4(-g.x, -g.y, -g.z, g.w) : g;
  }
  // As store(), plus whether the tile's edges fall in at most three CSR
  // rows (first, `mid`, last): 95% of coil-269 tiles; their P[src] values
  // are then three loads per thread instead of 32 gathers.
  __device__ __forceinline__ float4 store3(WarpMeta *m, bool src_owned, int lane, bool &rows3,
                                           int &mid) const {
    bool r2;
    const float4 u = store(m, src_owned, lane, r2);
    const int first = __shfl_sync(0xffffffffu, o, 0);
    const int last = __shfl_sync(0xffffffffu, o, max(n_e - 1, 0));
    const unsigned other = __ballot_sync(0xffffffffu, lane < n_e && o != first && o != last);
    mid = other ? __shfl_sync(0xffffffffu, o, __ffs(other) - 1) : first;
    rows3 = __all_sync(0xffffffffu, lane >= n_e || o == first || o == last || o == mid);
    return u;
  }
};

// Gaussian basis b[k][e] = exp((-g*dk)*dk) * C(d) (model.py:123-133) or, with
// DERIV, its derivative db = exp(..) * (-2 g dk C + C') (model.py:148-157),
// as the K=64 B operand.  Each warp writes 16 of the 64 K-rows: thread
// (q, lane) covers k = 16q + lane%16 for edges 16*(lane/16)..+15.  The fp32
// forward basis is scaled 2^14 and split; the W16 forward basis is rounded
// to fp16 unscaled (quantize.py:68-71); db is always split (fp32 backward).
// Padding edges carry C = C' = 0, so their columns are zero without a mask.
template <bool DERIV, bool Q, uint32_t KS = KSTR, bool PK = false>
__device__ __forceinline__ void tile_basis(const EdgeArgs &a, const Wctx &W, const WarpMeta *m,
                                           float log2_scale) {
  const int k = 16 * W.q + (W.lane & 15), e0 = (W.lane >> 4) * 16;  // edges within the tile
  const float mu = ld_dep(&a.centers[k]);
  const float ngl = -a.gamma * kLog2e, g2 = -2.f * a.gamma;
  float v[16];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float4 d4 = *(const float4 *)&m->d[e0 + 4 * j];
    const float4 c4 = *(const float4 *)&m->env[e0 + 4 * j];
    const float dd[4] = {d4.x, d4.y, d4.z, d4.w}, cc[4] = {c4.x, c4.y, c4.z, c4.w};
    float pp[4] = {0.f, 0.f, 0.f, 0.f};
    if (DERIV) {
      const float4 p4 = *(const float4 *)&m->denv[e0 + 4 * j];
      pp[0] = p4.x; pp[1] = p4.y; pp[2] = p4.z; pp[3] = p4.w;
    }
#pragma unroll
    for (int i = 0; i < 4; i += 2) {
      const float2 dl = add2(make_float2(dd[i], dd[i + 1]), f2(-mu));
      // exp(-g dl^2) * 2^log2_scale in one ex2: the operand scale is free
      const float2 gs = ex2_2(fma2(mul2(f2(ngl), dl), dl, f2(log2_scale)));
      const float2 c = make_float2(cc[i], cc[i + 1]);
      const float2 r = DERIV ? mul2(gs, fma2(mul2(f2(g2), dl), c, make_float2(pp[i], pp[i + 1])))
                             : mul2(gs, c);
      v[4 * j + i] = r.x;
      v[4 * j + i + 1] = r.y;
    }
  }
  constexpr bool LO = DERIV || !Q;
  put8<LO, KS, PK>(W.bb, DR, k, W.eo + e0, &v[0], 1.f);
  put8<LO, KS, PK>(W.bb, DR, k, W.eo + e0 + 8, &v[8], 1.f);
}

// h = ssp(z0) for this thread's channel over the tile (z0 = TMEM S0 scaled),
// as the K=128 B operand (act buffer).  Padding columns carry finite values
// that no valid edge reads.
// The fp32 split needs h * 2^f_hexp: the power-of-two scale is folded into
// z's constants and ssp's (HScale), so no separate multiply per element.
struct HScale {
  float rs, b, c_ln2, c_e;  // z*hs = acc*rs + b; ssp_scaled constants
  __device__ __forceinline__ HScale(float rs0, float b0c, float hs)
      : rs(rs0 * hs), b(b0c * hs), c_ln2(kLn2 * hs), c_e(-kLog2e / hs) {}
};

template <bool Q, uint32_t KS = KSTR, bool PK = false>
__device__ __forceinline__ void tile_h(const Wctx &W, float rs0, float b0c, const HScale &hk) {
  float v[TT];
  tc::tmem_ld32w(W.tl + S0, v);
  // fp32: hs * ssp(z); W16: ssp(z), rounded to fp16 (quantize.py:80-88) by
  // put8's hi-only pack (RN).  A pair of edges per instruction.
  const float rs = Q ? rs0 : hk.rs, bb = Q ? b0c : hk.b;
  const float cl = Q ? kLn2 : hk.c_ln2, ce = Q ? -kLog2e : hk.c_e;
#pragma unroll
  for (int i = 0; i < TT; i += 2) {
    const float2 h = ssp_scaled2(fma2(make_float2(v[i], v[i + 1]), f2(rs), f2(bb)), cl, ce);
    v[i] = h.x;
    v[i + 1] = h.y;
  }
#pragma unroll
  for (int j = 0; j < TT / 8; ++j) put8<!Q, KS, PK>(W.hb, D, W.ch, W.eo + 8 * j, &v[8 * j], 1.f);
}

// Sum of p over the 32 lanes of the warp for every edge: a butterfly
// reduce-scatter leaves edge `lane`'s sum in lane `lane`.
__device__ __forceinline__ float warp_edge_sum(float (&p)[TT], int lane) {
#pragma unroll
  for (int o = 16; o >= 2; o >>= 1) {  // the adds a pair per instruction (same sums)
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; i += 2) {
      const float r0 = __shfl_xor_sync(0xffffffffu, upper ? p[i] : p[i + o], o);
      const float r1 = __shfl_xor_sync(0xffffffffu, upper ? p[i + 1] : p[i + 1 + o], o);
      const float2 s = add2(make_float2(upper ? p[i + o] : p[i], upper ? p[i + 1 + o] : p[i + 1]),
                            make_float2(r0, r1));
      p[i] = s.x;
      p[i + 1] = s.y;
    }
  }
  const bool upper = (lane & 1) != 0;
  return (upper ? p[1] : p[0]) + __shfl_xor_sync(0xffffffffu, upper ? p[0] : p[1], 1);
}

// phase timestamps for diagnosis: CTA 0, warp 0, first 16 tiles
#define PHASE(kind, it, ph)                                                          \
  do {                                                                             \
    if (a.dbg && blockIdx.x == 0 && threadIdx.x == 0 && (it) >= 0 && (it) < 16)    \
      a.dbg[((kind) * 16 + (it)) * 64 + (ph)] = clock64();                         \
  } while (0)

// Timeline stamps of the 64-edge forward and the forward-mode backward
// (diagnostic builds only, -DFCG_EDGE_STAMPS; tools/diag_edge_timeline.py):
// lane 0 of the first warp of each group in CTA 0 records clock64() at phase
// `ph` of iteration `it` (< 32) into dbg[((kind*2 + group)*32 + it)*16 + ph].
#ifdef FCG_EDGE_STAMPS
#define STAMP(kind, grp_first, g, it, ph)                                                  \
  do {                                                                                    \
    if (a.dbg && blockIdx.x == 0 && (grp_first) && (threadIdx.x & 31) == 0 && (it) >= 0 && \
        (it) < 32)                                                                         \
      a.dbg[(((kind) * 2 + (g)) * 32 + (it)) * 16 + (ph)] = clock64();                     \
  } while (0)
#else
#define STAMP(kind, grp_first, g, it, ph) do { } while (0)
#endif

struct UnitRange {
  int rbeg, rend, eb, ee;
};
__device__ __forceinline__ UnitRange unit_range(const EdgeArgs &a, const int32_t *unit_rows,
                                                int unit) {
  UnitRange t;
  const int e_tot = a.ptr[a.nrows];
  const long long eff = e_tot > a.cap_e ? a.cap_e : e_tot;
  t.rbeg = unit_rows[unit];
  t.rend = unit_rows[unit + 1];
  t.eb = a.ptr[t.rbeg];
  t.ee = a.ptr[t.rend];
  if (t.ee > eff) t.ee = (int)eff;
  if (t.eb > t.ee) t.eb = t.ee;
  return t;
}

// ---------------------------------------------------------------------------
// Forward: per 32-edge tile of dst rows
//   b -> [G1] z0 -> h = ssp(z0) -> [G2] w -> m = P[src]*w -> H rows.
// While G2(i) runs the warp builds its part of the basis of tile i+1 and
// requests G1(i+1); the gathers P[src] of tile i+1 are in flight during
// G1(i+1).  Iteration -1 only prepares tile 0.
template <bool Q>
__global__ void __launch_bounds__(FWD_THREADS, 1)
k_edge_fwd_tc(const EdgeArgs a, const float4 *geo, const float2 *env,
              const int32_t *unit_rows, const float *P,
              float *H) {
  extern __shared__ __align__(1024) uint8_t sm[];
  TcShared *sh = (TcShared *)(sm + FWD_SM_META);
  const fcg_block &B = a.blk;
  pdl_trigger();
  kernel_prologue(sm, sh, B, FWD_NGRP);
  tc::mbar_wait(&sh->wbar, 0);
  load_fwd_weights_tmem(sm, sh->tmem);  // ends with the PDL wait
  const Wctx W = make_wctx(sm, sh, FWD_GCOLS, FWD_SM_BUF);
  const uint32_t idesc = tc::idesc_f16(128, TT, 0, 1);
  constexpr int NP = Q ? 1 : 3;
  const uint32_t w0h = sh->tmem + TW0, w0l = w0h + DR / 2, w1h = sh->tmem + TW1, w1l = w1h + D / 2;
  const Desc bb = adesc(W.sbb, DR), hb = adesc(W.shb, D);

  const UnitRange tr = unit_range(a, unit_rows, FWD_NGRP * blockIdx.x + W.g);
  const int ntiles = (tr.ee - tr.eb + TT - 1) / TT;
  const int ch = W.ch;
  const float *Pch = opaque_ptr(P + ch);  // gathers: Pch + nbr row offset
  SegSum seg;
  seg.row = ntiles > 0 ? a.own[tr.eb] : -1;
  seg.acc = 0.f;
  seg.outc = opaque_ptr(H + ch);

  const float b0c = ld_dep(&B.f0_b[ch]), b1c = ld_dep(&B.f1_b[ch]);
  const float rs0 = Q ? ld_dep(&B.f0_s[ch]) : pow2f(-(B.f0_exp + 14));
  const float hs = Q ? 1.f : pow2f(B.f_hexp);
  const HScale hk(rs0, b0c, hs);
  const float s1 = Q ? ld_dep(&B.f1_s[ch]) : pow2f(-(B.f1_exp + B.f_hexp));
  const float bsc = Q ? 0.f : 14.f;  // log2 of the forward basis scale

  float pv[TT];  // P[src][ch] of the current tile
  MetaRegs mr;   // raw metadata of the tile after next
  for (int it = -1; it < ntiles; ++it) {
    const int t0 = tr.eb + it * TT;
    const bool more = it + 1 < ntiles;
    const int n_n = min(TT, tr.ee - t0 - TT);
    PHASE(0, it, 0);
    if (it < 0) {
      bool r2;
      mr.load(a, geo, env, tr.eb, n_n, W.lane);
      mr.store(W.meta(0), false, W.lane, r2);
      if (more) mr.load(a, geo, env, tr.eb + TT, min(TT, tr.ee - tr.eb - TT), W.lane);
    } else {
      W.wait(BAR_G1, it);
      PHASE(0, it, 1);
      tile_h<Q>(W, rs0, b0c, hk);
      REQ(BAR_G2, (mma_chain_ts<D / 16, NP>(W.tmem_g + S1, w1h, w1l, hb, idesc)));
      PHASE(0, it, 2);
      if (more) {
        bool r2;
        mr.store(W.meta(it + 1), false, W.lane, r2);
        if (it + 2 < ntiles) mr.load(a, geo, env, t0 + 2 * TT, min(TT, tr.ee - t0 - 2 * TT), W.lane);
      }
    }
    if (more) {  // basis + G1 of the next tile overlap G2
      tile_basis<false, Q>(a, W, W.meta(it + 1), bsc);
      REQ(BAR_G1, (mma_chain_ts<DR / 16, NP>(W.tmem_g + S0, w0h, w0l, bb, idesc)));
    }
    PHASE(0, it, 3);
    if (it >= 0) {
      W.wait(BAR_G2, it);
      PHASE(0, it, 4);
      // m = (W1 h + b1) * P[src] (flash.py:229), dst segment sums (flash.py:232-234)
      float v[TT];
      tc::tmem_ld32w(W.tl + S1, v);
#pragma unroll
      for (int i = 0; i < TT; ++i) v[i] = (v[i] * s1 + b1c) * pv[i];
      if (tr.ee - t0 < TT) {
#pragma unroll
        for (int i = 0; i < TT; ++i) v[i] = i < tr.ee - t0 ? v[i] : 0.f;
      }
      seg.tile(W.meta(it)->own, v);
      PHASE(0, it, 5);
    }
    if (more) {
      const WarpMeta *Mn = W.meta(it + 1);
#pragma unroll
      for (int i = 0; i < TT; ++i) pv[i] = ld_gather(Pch + (uint32_t)Mn->nbr[i]);
    }
  }
  seg.finish();
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(sh->tmem);
}

// ---------------------------------------------------------------------------
// Backward over src-owned rows (flash_block_backward, flash.py:272-295), per
// 32-edge tile:
//   gH = GH[dst]; [G1] z0 (recompute) -> h, ssp'(z0) -> [G2] w;
//   grad_w = gH*P[src] -> [G3, W1^T] grad_h;
//   grad_P rows = src-segment sums of gH*w (while G3 runs);
//   db -> [G1'] dz0 = W0 db;  gz = grad_h * ssp'(z0);
//   grad_d = sum_c gz*dz0 (= sum_k grad_b*db, flash.py:293) -> g_e = grad_d/d*u.
//
// With N = 32 edges per MMA the A operand dominates the tensor core's
// shared-memory reads (4 KB of weights per 1 KB of edges), so W1 and W1^T —
// the A operands of G2 and G3, two thirds of the MMAs — are TMEM-resident
// (columns [TB1, 512)), and W0 stays in shared memory.  That leaves each group
// two 32-column slots: SA holds z0, then w, then dz0; SB holds grad_h, then
// gz.  ssp'(z0) is stashed in the shared memory W1 was staged through.  G1 of
// tile i+1 is issued as soon as the grad_d operands of tile i are in registers
// and overlaps the reduction.
constexpr uint32_t BWD_GCOLS = 64, SA = 0, SB = 32;
constexpr uint32_t TB1 = NGRP * BWD_GCOLS, TB1T = TB1 + 128;
static_assert(TB1T + 128 <= 512, "TMEM budget");
constexpr uint32_t STASH_BYTES = D * TT * 4;
static_assert(NGRP * STASH_BYTES <= 2 * W1_BYTES, "stash fits in the W1 staging area");

// W1 (K-major rows) and W1^T (row m = column m of W1) hi | lo from the staged
// shared-memory images into TMEM; warp w moves image w / 4 for its lane
// quarter.  The W1 staging area becomes the ssp' stash afterwards.
__device__ __forceinline__ void load_w1_tmem(const uint8_t *sm, uint32_t tmem) {
  const int w = threadIdx.x >> 5, q = w & 3, m = 32 * q + (threadIdx.x & 31);
  const int img = (w >> 2) & 3;  // 0: W1 hi, 1: W1 lo, 2: W1^T hi, 3: W1^T lo
  const uint16_t *base = (const uint16_t *)(sm + SM_W1 + (img & 1) * W1_BYTES);
  const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (img < 2 ? TB1 : TB1T) + (img & 1) * (D / 2);
  if (img < 2) image_row_to_tmem<false>(base, D, m, taddr);
  else image_row_to_tmem<true>(base, D, m, taddr);
  prologue_done();
}

// h = ssp(z0) as the K=128 B operand (act buffer) and ssp'(z0) into the
// thread's stash entries ([edge/4][channel] float4s, conflict-free).  fp32:
// ssp'(z) = sigmoid(z) = 1 - exp(-ssp(z))/2 from h; W16: from z0 itself (h is
// rounded to fp16).
// The stash holds ssp'(z0) * kz, kz = the scales of grad_h (sg3) and dz0
// (sdz), so gz and the grad_d product need no separate multiplies.
template <bool Q, uint32_t KS = KSTR>
__device__ __forceinline__ void tile_h_bwd(const Wctx &W, float rs0, float b0c, const HScale &hk,
                                           float kz, float4 *stash) {
  float v[TT];
  tc::tmem_ld32w(W.tl + SA, v);
#pragma unroll
  for (int i = 0; i < TT; i += 4) {
    float s[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (Q) {
        const float z = v[i + j] * rs0 + b0c;
        s[j] = sigmoid_fast(z) * kz;
        v[i + j] = ssp_fast(z);  // rounded to fp16 by put8's hi-only pack
      } else {
        v[i + j] = ssp_scaled(v[i + j] * hk.rs + hk.b, hk.c_ln2, hk.c_e);  // hs * h
        s[j] = fmaf(-0.5f * kz, ex2_ftz(v[i + j] * hk.c_e), kz);        // kz (1 - e^-h / 2)
      }
    }
    stash[(i / 4) * D + W.ch] = make_float4(s[0], s[1], s[2], s[3]);
  }
#pragma unroll
  for (int j = 0; j < TT / 8; ++j) put8<!Q, KS>(W.hb, D, W.ch, W.eo + 8 * j, &v[8 * j], 1.f);
}

template <bool Q>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_edge_bwd_tc(const EdgeArgs a, const float4 *geo, const float2 *env,
              const int32_t *unit_rows, const float *P,
              const float *GH, float *GP, float4 *gsum,
              int accumulate) {
  extern __shared__ __align__(1024) uint8_t sm[];
  TcShared *sh = (TcShared *)(sm + SM_META);
  const fcg_block &B = a.blk;
  pdl_trigger();
  kernel_prologue(sm, sh, B, NGRP);
  tc::mbar_wait(&sh->wbar, 0);
  load_w1_tmem(sm, sh->tmem);  // ends with the PDL wait
  const Wctx W = make_wctx(sm, sh, BWD_GCOLS, SM_BUF);
  float4 *stash = (float4 *)(sm + SM_W1 + W.g * STASH_BYTES);
  const uint32_t sbase = tc::smem_u32(sm);
  const uint32_t id_f = tc::idesc_f16(128, TT, 0, 1);
  constexpr int NPF = Q ? 1 : 3, NPB = Q ? 2 : 3;
  const Desc w0 = wdesc_k(sbase + SM_W0, DR, W0_BYTES);
  const uint32_t w1h = sh->tmem + TB1, w1l = w1h + D / 2, w1th = sh->tmem + TB1T, w1tl = w1th + D / 2;
  const Desc bb = adesc(W.sbb, DR), hb = adesc(W.shb, D);

  const UnitRange tr = unit_range(a, unit_rows, NGRP * blockIdx.x + W.g);
  const int ntiles = (tr.ee - tr.eb + TT - 1) / TT;
  const int ch = W.ch;
  const float *GHch = opaque_ptr(GH + ch);  // gathers: GHch + dst row offset
  const float *Pch = opaque_ptr(P + ch);    // P[src] rows of the tile
  SegSum seg;
  seg.row = ntiles > 0 ? a.own[tr.eb] : -1;
  seg.acc = 0.f;
  seg.outc = opaque_ptr(GP + ch);

  const float b0c = ld_dep(&B.f0_b[ch]), b1c = ld_dep(&B.f1_b[ch]);
  const float rs0 = Q ? ld_dep(&B.f0_s[ch]) : pow2f(-(B.f0_exp + 14));
  const float hs = Q ? 1.f : pow2f(B.f_hexp);
  const HScale hk(rs0, b0c, hs);
  const float s1 = Q ? ld_dep(&B.f1_s[ch]) : pow2f(-(B.f1_exp + B.f_hexp));
  const float bsc = Q ? 0.f : 14.f;  // log2 of the forward basis scale
  // backward GEMMs against the stored fp16 weights fold the W16 dequant
  // scale of the contracted index into the operand: g @ (s*w16) == (g*s) @ w16
  const float q1 = Q ? ld_dep(&B.f1_s[ch]) : 1.f;
  const float pmax = __uint_as_float(a.amax_pg[0]), ghmax = __uint_as_float(a.amax_pg[1]);
  const int sg = scale_exp(pmax * ghmax * B.f1_qmax);
  const float gws = pow2f(sg) * q1;
  const float sg3 = pow2f(-((Q ? 0 : B.f1_exp) + sg));
  const float sdz = (Q ? ld_dep(&B.f0_s[ch]) : pow2f(-B.f0_exp)) * pow2f(-B.f_dbexp);
  const float kz = sg3 * sdz;

  float4 ue = make_float4(0.f, 0.f, 0.f, 0.f), ue_n = ue;  // this lane's edge: (u, d)
  bool rows2 = true, rows2_n = true;
  MetaRegs mr;  // raw metadata of the tile after next
  if (ntiles > 0) {  // tile 0: metadata, basis, G1
    mr.load(a, geo, env, tr.eb, min(TT, tr.ee - tr.eb), W.lane);
    ue_n = mr.store(W.meta(0), true, W.lane, rows2_n);
    if (ntiles > 1) mr.load(a, geo, env, tr.eb + TT, min(TT, tr.ee - tr.eb - TT), W.lane);
    tile_basis<false, Q>(a, W, W.meta(0), bsc);
    REQ(BAR_G1, (mma_chain<DR / 16, NPF>(W.tmem_g + SA, w0, bb, id_f)));
  }
  for (int it = 0; it < ntiles; ++it) {
    ue = ue_n;
    rows2 = rows2_n;
    const int t0 = tr.eb + it * TT;
    const bool more = it + 1 < ntiles;
    PHASE(1, it, 0);
    const WarpMeta *M = W.meta(it);
    const int n_e = min(TT, tr.ee - t0);
    float gh[TT];  // grad_H[dst][ch] (flash.py:281)
#pragma unroll
    for (int i = 0; i < TT; ++i) gh[i] = ld_gather(GHch + (uint32_t)M->nbr[i]);
    // P[src][ch] (flash.py:291): src = the tile's CSR rows, usually its
    // first and last only
    const int o_f = M->own[0], o_l = M->own[n_e - 1];
    const float p_f = ld_gather(Pch + (uint32_t)o_f * D), p_l = ld_gather(Pch + (uint32_t)o_l * D);
    const float pf_s = p_f * gws, pl_s = p_l * gws;  // grad_w operand scale folded in
    W.wait(BAR_G1, it);
    PHASE(1, it, 1);
    tile_h_bwd<Q>(W, rs0, b0c, hk, kz, stash);
    REQ(BAR_G2, (mma_chain_ts<D / 16, NPF>(W.tmem_g + SA, w1h, w1l, hb, id_f)));
    PHASE(1, it, 2);
    if (more) {
      ue_n = mr.store(W.meta(it + 1), true, W.lane, rows2_n);
      if (it + 2 < ntiles) mr.load(a, geo, env, t0 + 2 * TT, min(TT, tr.ee - t0 - 2 * TT), W.lane);
    }
    W.wait(BAR_G2, it);
    PHASE(1, it, 3);
    // grad_w = gH * P[src] (flash.py:291) -> B operand of G3 (W1^T)
#pragma unroll
    for (int j = 0; j < TT / 8; ++j) {
      const int4 oa = *(const int4 *)&M->own[8 * j], ob = *(const int4 *)&M->own[8 * j + 4];
      const int oo[8] = {oa.x, oa.y, oa.z, oa.w, ob.x, ob.y, ob.z, ob.w};
      float v[8];
      if (rows2) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = gh[8 * j + i] * (oo[i] == o_l ? pl_s : pf_s);
        put8<true>(W.hb, D, ch, 8 * j, v, 1.f);
      } else {  // a tile spanning 3+ rows: per-edge loads
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = gh[8 * j + i] * ld_gather(Pch + (uint32_t)max(oo[i], 0) * D);
        put8<true>(W.hb, D, ch, 8 * j, v, gws);
      }
    }
    REQ(BAR_G3, (mma_chain_ts<D / 16, NPB>(W.tmem_g + SB, w1th, w1tl, hb, id_f)));
    PHASE(1, it, 4);
    // while G3 runs: grad_P rows = src-segment sums of gH * w (flash.py:283-288)
    {
      float v[TT];
      tc::tmem_ld32w(W.tl + SA, v);
#pragma unroll
      for (int i = 0; i < TT; ++i) v[i] = gh[i] * (v[i] * s1 + b1c);
      if (n_e < TT) {
#pragma unroll
        for (int i = 0; i < TT; ++i) v[i] = i < n_e ? v[i] : 0.f;
      }
      seg.tile(M->own, v);
    }
    PHASE(1, it, 5);
    // db -> basis buffer (G1 is done), G1': dz0 = W0 db into SA (w consumed)
    tile_basis<true, Q>(a, W, M, (float)B.f_dbexp);
    REQ(BAR_G1P, (mma_chain<DR / 16, NPB>(W.tmem_g + SA, w0, bb, id_f)));
    PHASE(1, it, 6);
    W.wait(BAR_G3, it);
    // gz = grad_h * ssp'(z0) (mlp_backward_input, model.py:189-200), kept in SB
    {
      float gz[TT];
      tc::tmem_ld32w(W.tl + SB, gz);
#pragma unroll
      for (int i = 0; i < TT; i += 4) {
        const float4 s = stash[(i / 4) * D + ch];
        gz[i] *= s.x; gz[i + 1] *= s.y; gz[i + 2] *= s.z; gz[i + 3] *= s.w;
      }
      tc::tmem_st32(W.tl + SB, gz);
      tc::tmem_st_wait();
    }
    PHASE(1, it, 7);
    W.wait(BAR_G1P, it);
    PHASE(1, it, 8);
    // grad_d[e] = sum_c gz[c][e] * dz0[c][e]: per-warp transpose-sum, then
    // the four lane quarters in fixed order (warp 0 of the group)
    float p[TT];
    {
      float dz[TT];
      tc::tmem_ld32w(W.tl + SB, p);
      tc::tmem_ld32w(W.tl + SA, dz);
#pragma unroll
      for (int i = 0; i < TT; ++i) p[i] *= dz[i];  // sdz rides in the stash
    }
    if (more) {  // basis + G1 of the next tile (SA is read) overlap the reduction
      tile_basis<false, Q>(a, W, W.meta(it + 1), bsc);
      REQ(BAR_G1, (mma_chain<DR / 16, NPF>(W.tmem_g + SA, w0, bb, id_f)));
    }
    PHASE(1, it, 9);
    float *xg = &sh->xg[W.g][it & 1][0][0];
    xg[W.q * TT + W.lane] = warp_edge_sum(p, W.lane);
    __syncwarp();
    if (W.lane == 0) tc::mbar_arrive(&sh->xbar[W.g]);
    if (W.q == 0) {
      tc::mbar_wait(&sh->xbar[W.g], (uint32_t)(it & 1));
      const int e = W.lane;
      if (e < n_e) {
        const float gd = ((xg[e] + xg[TT + e]) + xg[2 * TT + e]) + xg[3 * TT + e];
        const float inv = ue.w > TINY_DISTANCE ? 1.f / ue.w : 0.f;  // _safe_inv, flash.py:176-178
        const float s = gd * inv;
        float4 g = make_float4(s * ue.x, s * ue.y, s * ue.z, 0.f);  // flash.py:294
        float4 *dst = &gsum[t0 + e];
        if (accumulate) {
          const float4 o = *dst;
          g.x += o.x; g.y += o.y; g.z += o.z;
        }
        *dst = g;
      }
    }
    PHASE(1, it, 10);
  }
  seg.finish();
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(sh->tmem);
}

constexpr uint32_t KSTR64 = (64 / 8) * 128;  // B operand bytes per 8 K-rows, 64 edges

// ---------------------------------------------------------------------------
// Forward with 64-edge MMAs (the default; FCG_FWD64=0 selects k_edge_fwd_tc):
// 2 groups x 8 warps, each group's tile = 32 edges of each of its two work
// units, as in k_edge_bwd64.  TMEM: 2 x 128 group columns (z0 | w, 64 wide)
// + W0 | W1 at TW0; shared memory: the forward layout (buffers 2 x 48 KB).
template <bool Q, bool SC>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_edge_fwd64(const EdgeArgs a, const float4 *geo, const float2 *env,
             const int32_t *unit_rows, const float *P, float *H) {
  extern __shared__ __align__(1024) uint8_t sm[];
  TcShared *sh = (TcShared *)(sm + FWD_SM_META);
  const fcg_block &B = a.blk;
  pdl_trigger();
  kernel_prologue(sm, sh, B, FWD_NGRP);
  tc::mbar_wait(&sh->wbar, 0);
  load_fwd_weights_tmem(sm, sh->tmem);  // ends with the PDL wait
  Wctx W;
  W.w = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  W.g = W.w >> 3;
  const int hf = (W.w >> 2) & 1;
  const int u = 2 * W.g + hf;
  W.q = W.w & 3;
  W.lane = threadIdx.x & 31;
  W.ch = 32 * W.q + W.lane;
  W.eo = 32 * hf;
  W.amask = 7u;
  W.sh = sh;
  W.bb = sm + FWD_SM_BUF + W.g * 2 * GBUF_BYTES;
  W.hb = W.bb + 2 * BB_BYTES;
  W.sbb = tc::smem_u32(W.bb);
  W.shb = tc::smem_u32(W.hb);
  W.tmem_g = sh->tmem + 128u * W.g;
  W.tl = W.tmem_g + ((uint32_t)(32 * W.q) << 16) + 32u * hf;
  const uint32_t idesc = tc::idesc_f16(128, 64, 0, 1);
  constexpr int NP = Q ? 1 : 3;
  constexpr uint32_t Z0 = 0, WS = 64;  // TMEM slots: z0 | w, 64 columns each
  const uint32_t w0h = sh->tmem + TW0, w0l = w0h + DR / 2, w1h = sh->tmem + TW1, w1l = w1h + D / 2;
  const Desc bb = adesc<KSTR64>(W.sbb, DR), hb = adesc<KSTR64>(W.shb, D);

  const UnitRange tr = unit_range(a, unit_rows, FWD_NGRP * blockIdx.x + u);
  const UnitRange to = unit_range(a, unit_rows, FWD_NGRP * blockIdx.x + (u ^ 1));
  const int ntiles = (tr.ee - tr.eb + TT - 1) / TT;
  const int nt_all = max(ntiles, (to.ee - to.eb + TT - 1) / TT);
  const int ch = W.ch;
  const float *Pch = opaque_ptr(P + ch);
  SegSum seg;
  seg.row = ntiles > 0 ? a.own[tr.eb] : -1;
  seg.acc = 0.f;
  seg.outc = opaque_ptr(H + ch);

  const float b0c = ld_dep(&B.f0_b[ch]), b1c = ld_dep(&B.f1_b[ch]);
  const float rs0 = Q ? ld_dep(&B.f0_s[ch]) : pow2f(-(B.f0_exp + 14));
  const float hs = Q ? 1.f : pow2f(B.f_hexp);
  const HScale hk(rs0, b0c, hs);
  const float s1 = Q ? ld_dep(&B.f1_s[ch]) : pow2f(-(B.f1_exp + B.f_hexp));
  const float bsc = Q ? 0.f : 14.f;

  float pv[TT];
  MetaRegs mr;
  for (int it = -1; it < nt_all; ++it) {
    const int t0 = tr.eb + it * TT;
    const bool more = it + 1 < nt_all;
    if (it < 0) {
      bool r2;
      mr.load(a, geo, env, tr.eb, min(TT, tr.ee - tr.eb), W.lane);
      mr.store(W.meta(0), false, W.lane, r2);
      mr.load(a, geo, env, tr.eb + TT, min(TT, tr.ee - tr.eb - TT), W.lane);
    } else {
      STAMP(0, (W.w & 7) == 0, W.g, it, 0);
      W.wait(BAR_G1, it);
      STAMP(0, (W.w & 7) == 0, W.g, it, 1);
      tile_h<Q, KSTR64>(W, rs0, b0c, hk);
      STAMP(0, (W.w & 7) == 0, W.g, it, 2);
      REQ(BAR_G2, (mma_chain_ts<D / 16, NP>(W.tmem_g + WS, w1h, w1l, hb, idesc)));
      STAMP(0, (W.w & 7) == 0, W.g, it, 3);
      if (more) {
        bool r2;
        mr.store(W.meta(it + 1), false, W.lane, r2);
        mr.load(a, geo, env, t0 + 2 * TT, min(TT, tr.ee - t0 - 2 * TT), W.lane);
      }
    }
    if (more) {  // basis + G1 of the next tile overlap G2
      tile_basis<false, Q, KSTR64>(a, W, W.meta(it + 1), bsc);
      REQ(BAR_G1, (mma_chain_ts<DR / 16, NP>(W.tmem_g + Z0, w0h, w0l, bb, idesc)));
    }
    STAMP(0, (W.w & 7) == 0, W.g, it, 4);
    if (it >= 0) {
      W.wait(BAR_G2, it);
      STAMP(0, (W.w & 7) == 0, W.g, it, 5);
      float v[TT];
      tc::tmem_ld32w(W.tl + WS, v);
      const int n_e = min(TT, tr.ee - t0);
      if (n_e > 0) {  // m = (W1 h + b1) * P[src], dst segment sums
#pragma unroll
        for (int i = 0; i < TT; i += 2) {
          const float2 m = mul2(fma2(make_float2(v[i], v[i + 1]), f2(s1), f2(b1c)),
                                make_float2(pv[i], pv[i + 1]));
          v[i] = m.x;
          v[i + 1] = m.y;
        }
        if (SC) {
          scatter_tile(seg.outc, W.meta(it)->own, v, n_e);
        } else {
          if (n_e < TT) {
#pragma unroll
            for (int i = 0; i < TT; ++i) v[i] = i < n_e ? v[i] : 0.f;
          }
          seg.tile(W.meta(it)->own, v);
        }
      }
    }
    STAMP(0, (W.w & 7) == 0, W.g, it, 6);
    if (more) {
      const WarpMeta *Mn = W.meta(it + 1);
      if (tr.ee - (t0 + TT) > 0) {
#pragma unroll
        for (int i = 0; i < TT; ++i) pv[i] = ld_gather(Pch + (uint32_t)Mn->nbr[i]);
      }
    }
    STAMP(0, (W.w & 7) == 0, W.g, it, 7);
  }
  if (!SC) seg.finish();
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(sh->tmem);
}

// ---------------------------------------------------------------------------
// Forward with a dedicated MMA warp (the default; FCG_FWD_WS=0 selects
// k_edge_fwd64).  With last-arriver issue, the warp that issues a chain
// stays blocked in tcgen05.mma for about the chain's duration, and the
// group's next request waits for that warp's share of the epilogue
// (timeline stamps: ~1k cycles per G2 chain, tools/diag_edge_timeline.py).
// Here a fifth warpgroup issues every chain: the 16 epilogue warps only
// arrive on a per-group "operands ready" mbarrier (8 arrivals) and never
// block on the tensor pipe.  Registers: the CTA holds 640 x 96; the issuer
// warpgroup drops to 24 and the four epilogue warpgroups grow to 112
// (setmaxnreg; 112 is the most the pool released by the issuer covers).
constexpr int WS_THREADS = TC_THREADS + 128;
struct FwdWsShared {
  TcShared t;
  uint64_t ready[2][4];  // operands of a group's chain written (8 warp arrivals)
};
static_assert(FWD_SM_META + sizeof(FwdWsShared) + 1024 <= 232448, "forward WS smem budget");

__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(tc::smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
// An epilogue warp's operands for a chain are in shared memory (generic
// proxy writes made visible to the tensor core) and its TMEM reads of the
// columns the chain overwrites are complete: one arrival per warp.
__device__ __forceinline__ void ws_ready(uint64_t *bar) {
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) tc::mbar_arrive(bar);
}

template <bool Q, bool SC>
__global__ void __launch_bounds__(WS_THREADS, 1)
k_edge_fwd_ws(const EdgeArgs a, const float4 *geo, const float2 *env,
              const int32_t *unit_rows, const float *P, float *H) {
  extern __shared__ __align__(1024) uint8_t sm[];
  FwdWsShared *ws = (FwdWsShared *)(sm + FWD_SM_META);
  TcShared *sh = &ws->t;
  const fcg_block &B = a.blk;
  pdl_trigger();
  if (threadIdx.x < 2) {
#pragma unroll
    for (int i = 0; i < 4; ++i) tc::mbar_init(&ws->ready[threadIdx.x][i], 8);
  }
  kernel_prologue(sm, sh, B, FWD_NGRP);
  tc::mbar_wait(&sh->wbar, 0);
  load_fwd_weights_tmem(sm, sh->tmem);  // ends with the PDL wait
  const uint32_t idesc = tc::idesc_f16(128, 64, 0, 1);
  constexpr int NP = Q ? 1 : 3;
  constexpr uint32_t Z0 = 0, WS = 64;  // TMEM slots: z0 | w, 64 columns each
  const uint32_t w0h = sh->tmem + TW0, w0l = w0h + DR / 2, w1h = sh->tmem + TW1, w1l = w1h + D / 2;
  if (threadIdx.x >= TC_THREADS) {
    // ---- the MMA warpgroup: warp 16 issues every chain of both groups --------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 24;\n" ::: "memory");
    if (threadIdx.x >= TC_THREADS + 32) return;
    int nt[2], c[2] = {0, 0};
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const UnitRange r0 = unit_range(a, unit_rows, FWD_NGRP * blockIdx.x + 2 * g);
      const UnitRange r1 = unit_range(a, unit_rows, FWD_NGRP * blockIdx.x + 2 * g + 1);
      nt[g] = max((r0.ee - r0.eb + TT - 1) / TT, (r1.ee - r1.eb + TT - 1) / TT);
    }
    while (c[0] < 2 * nt[0] || c[1] < 2 * nt[1]) {
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        if (c[g] >= 2 * nt[g]) continue;
        const int kind = (c[g] & 1) ? BAR_G2 : BAR_G1;
        if (!mbar_try(&ws->ready[g][kind], (uint32_t)((c[g] >> 1) & 1))) continue;
        tc::fence_after_sync();
        const uint32_t sb = tc::smem_u32(sm + FWD_SM_BUF + g * 2 * GBUF_BYTES);
        const uint32_t tg = sh->tmem + 128u * g;
        if (kind == BAR_G1)
          mma_chain_ts<DR / 16, NP>(tg + Z0, w0h, w0l, adesc<KSTR64>(sb, DR), idesc);
        else
          mma_chain_ts<D / 16, NP>(tg + WS, w1h, w1l, adesc<KSTR64>(sb + 2 * BB_BYTES, D), idesc);
        tc::mma_commit_warp(&sh->bar[g][kind]);
        ++c[g];
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 112;\n" ::: "memory");
  Wctx W;
  W.w = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  W.g = W.w >> 3;
  const int hf = (W.w >> 2) & 1;
  const int u = 2 * W.g + hf;
  W.q = W.w & 3;
  W.lane = threadIdx.x & 31;
  W.ch = 32 * W.q + W.lane;
  W.eo = 32 * hf;
  W.amask = 7u;
  W.sh = sh;
  W.bb = sm + FWD_SM_BUF + W.g * 2 * GBUF_BYTES;
  W.hb = W.bb + 2 * BB_BYTES;
  W.sbb = tc::smem_u32(W.bb);
  W.shb = tc::smem_u32(W.hb);
  W.tmem_g = sh->tmem + 128u * W.g;
  W.tl = W.tmem_g + ((uint32_t)(32 * W.q) << 16) + 32u * hf;

  const UnitRange tr = unit_range(a, unit_rows, FWD_NGRP * blockIdx.x + u);
  const UnitRange to = unit_range(a, unit_rows, FWD_NGRP * blockIdx.x + (u ^ 1));
  const int ntiles = (tr.ee - tr.eb + TT - 1) / TT;
  const int nt_all = max(ntiles, (to.ee - to.eb + TT - 1) / TT);
  const int ch = W.ch;
  const float *Pch = opaque_ptr(P + ch);
  SegSum seg;
  seg.row = ntiles > 0 ? a.own[tr.eb] : -1;
  seg.acc = 0.f;
  seg.outc = opaque_ptr(H + ch);

  const float b0c = ld_dep(&B.f0_b[ch]), b1c = ld_dep(&B.f1_b[ch]);
  const float rs0 = Q ? ld_dep(&B.f0_s[ch]) : pow2f(-(B.f0_exp + 14));
  const float hs = Q ? 1.f : pow2f(B.f_hexp);
  const HScale hk(rs0, b0c, hs);
  const float s1 = Q ? ld_dep(&B.f1_s[ch]) : pow2f(-(B.f1_exp + B.f_hexp));
  const float bsc = Q ? 0.f : 14.f;

  float pv[TT];
  MetaRegs mr;
  for (int it = -1; it < nt_all; ++it) {
    const int t0 = tr.eb + it * TT;
    const bool more = it + 1 < nt_all;
    if (it < 0) {
      bool r2;
      mr.load(a, geo, env, tr.eb, min(TT, tr.ee - tr.eb), W.lane);
      mr.store(W.meta(0), false, W.lane, r2);
      mr.load(a, geo, env, tr.eb + TT, min(TT, tr.ee - tr.eb - TT), W.lane);
    } else {
      STAMP(0, (W.w & 7) == 0, W.g, it, 0);
      W.wait(BAR_G1, it);
      STAMP(0, (W.w & 7) == 0, W.g, it, 1);
      tile_h<Q, KSTR64, true>(W, rs0, b0c, hk);
      STAMP(0, (W.w & 7) == 0, W.g, it, 2);
      ws_ready(&ws->ready[W.g][BAR_G2]);
      STAMP(0, (W.w & 7) == 0, W.g, it, 3);
      if (more) {
        bool r2;
        mr.store(W.meta(it + 1), false, W.lane, r2);
        mr.load(a, geo, env, t0 + 2 * TT, min(TT, tr.ee - t0 - 2 * TT), W.lane);
      }
    }
    if (more) {  // basis + G1 of the next tile overlap G2
      tile_basis<false, Q, KSTR64, true>(a, W, W.meta(it + 1), bsc);
      ws_ready(&ws->ready[W.g][BAR_G1]);
    }
    STAMP(0, (W.w & 7) == 0, W.g, it, 4);
    if (it >= 0) {
      W.wait(BAR_G2, it);
      STAMP(0, (W.w & 7) == 0, W.g, it, 5);
      float v[TT];
      tc::tmem_ld32w(W.tl + WS, v);
      const int n_e = min(TT, tr.ee - t0);
      if (n_e > 0) {  // m = (W1 h + b1) * P[src], dst segment sums
#pragma unroll
        for (int i = 0; i < TT; i += 2) {
          const float2 m = mul2(fma2(make_float2(v[i], v[i + 1]), f2(s1), f2(b1c)),
                                make_float2(pv[i], pv[i + 1]));
          v[i] = m.x;
          v[i + 1] = m.y;
        }
        if (SC) {
          scatter_tile(seg.outc, W.meta(it)->own, v, n_e);
        } else {
          if (n_e < TT) {
#pragma unroll
            for (int i = 0; i < TT; ++i) v[i] = i < n_e ? v[i] : 0.f;
          }
          seg.tile(W.meta(it)->own, v);
        }
      }
    }
    STAMP(0, (W.w & 7) == 0, W.g, it, 6);
    if (more) {
      const WarpMeta *Mn = W.meta(it + 1);
      if (tr.ee - (t0 + TT) > 0) {
#pragma unroll
        for (int i = 0; i < TT; ++i) pv[i] = ld_gather(Pch + (uint32_t)Mn->nbr[i]);
      }
    }
    STAMP(0, (W.w & 7) == 0, W.g, it, 7);
  }
  if (!SC) seg.finish();
  tc::fence_before_sync();
  // the issuer warpgroup has returned: sync the epilogue threads only
  asm volatile("bar.sync 1, %0;" ::"r"(TC_THREADS) : "memory");
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(sh->tmem);
}


static bool fwd_ws_enabled() {
  static const bool on = [] {
    const char *v = getenv("FCG_FWD_WS");
    return !(v && v[0] == '0');
  }();
  return on;
}

static bool fwd64_enabled() {
  static const bool on = [] {
    const char *v = getenv("FCG_FWD64");
    return !(v && v[0] == '0');
  }();
  return on;
}

// ---------------------------------------------------------------------------
// Backward with 64-edge MMAs (the default; FCG_BWD64=0 selects k_edge_bwd_tc):
// 2 groups x 8 warps.
// A group's tile is 32 edges from each of its two work units (warps 0-3:
// unit 2g, warps 4-7: unit 2g+1, every CSR row still has one walker), so
// each GEMM is N = 64 and a group issues half the MMAs per edge.  TMEM: 2 x
// 128 accumulator columns (SA, SB 64 wide) + W1 | W1^T; the shared-memory
// layout is the 4-group one (buffers 2 x 48 KB, stash per unit).
// SC (the fused-scatter ablation, flash.py:373-443): grad_P rows and the
// position gradient are accumulated with atomics — grad_P[src] += gH*w per
// channel, grad_r[dst] += g_e, grad_r[src] -= g_e (gr, float4 per node) —
// instead of segment sums and the per-slot gsum the force assembly gathers.
template <bool Q, bool SC>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_edge_bwd64(const EdgeArgs a, const float4 *geo, const float2 *env,
             const int32_t *unit_rows, const float *P,
             const float *GH, float *GP, float4 *gsum,
             int accumulate, float4 *gr) {
  extern __shared__ __align__(1024) uint8_t sm[];
  TcShared *sh = (TcShared *)(sm + SM_META);
  const fcg_block &B = a.blk;
  pdl_trigger();
  kernel_prologue(sm, sh, B, NGRP);  // bar[0..1] per group, xbar[0..3] per unit
  tc::mbar_wait(&sh->wbar, 0);
  load_w1_tmem(sm, sh->tmem);  // ends with the PDL wait
  Wctx W;
  W.w = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  W.g = W.w >> 3;
  const int hf = (W.w >> 2) & 1;
  const int u = 2 * W.g + hf;  // work unit / stash / grad_d partials of this warp
  W.q = W.w & 3;
  W.lane = threadIdx.x & 31;
  W.ch = 32 * W.q + W.lane;
  W.eo = 32 * hf;
  W.amask = 7u;
  W.sh = sh;
  W.bb = sm + SM_BUF + W.g * 2 * GBUF_BYTES;
  W.hb = W.bb + 2 * BB_BYTES;
  W.sbb = tc::smem_u32(W.bb);
  W.shb = tc::smem_u32(W.hb);
  W.tmem_g = sh->tmem + 128u * W.g;
  W.tl = W.tmem_g + ((uint32_t)(32 * W.q) << 16) + 32u * hf;
  float4 *stash = (float4 *)(sm + SM_W1 + u * STASH_BYTES);
  const uint32_t sbase = tc::smem_u32(sm);
  const uint32_t id_f = tc::idesc_f16(128, 64, 0, 1);
  constexpr int NPF = Q ? 1 : 3, NPB = Q ? 2 : 3;
  constexpr uint32_t SA64 = 0, SB64 = 64;
  const Desc w0 = wdesc_k(sbase + SM_W0, DR, W0_BYTES);
  const uint32_t w1h = sh->tmem + TB1, w1l = w1h + D / 2, w1th = sh->tmem + TB1T, w1tl = w1th + D / 2;
  const Desc bb = adesc<KSTR64>(W.sbb, DR), hb = adesc<KSTR64>(W.shb, D);

  const UnitRange tr = unit_range(a, unit_rows, NGRP * blockIdx.x + u);
  const UnitRange to = unit_range(a, unit_rows, NGRP * blockIdx.x + (u ^ 1));
  const int ntiles = (tr.ee - tr.eb + TT - 1) / TT;
  const int nt_all = max(ntiles, (to.ee - to.eb + TT - 1) / TT);  // the group's iterations
  const int ch = W.ch;
  const float *GHch = opaque_ptr(GH + ch);
  const float *Pch = opaque_ptr(P + ch);
  SegSum seg;
  seg.row = ntiles > 0 ? a.own[tr.eb] : -1;
  seg.acc = 0.f;
  seg.outc = opaque_ptr(GP + ch);

  const float b0c = ld_dep(&B.f0_b[ch]), b1c = ld_dep(&B.f1_b[ch]);
  const float rs0 = Q ? ld_dep(&B.f0_s[ch]) : pow2f(-(B.f0_exp + 14));
  const float hs = Q ? 1.f : pow2f(B.f_hexp);
  const HScale hk(rs0, b0c, hs);
  const float s1 = Q ? ld_dep(&B.f1_s[ch]) : pow2f(-(B.f1_exp + B.f_hexp));
  const float bsc = Q ? 0.f : 14.f;
  const float q1 = Q ? ld_dep(&B.f1_s[ch]) : 1.f;
  const float pmax = __uint_as_float(a.amax_pg[0]), ghmax = __uint_as_float(a.amax_pg[1]);
  const int sg = scale_exp(pmax * ghmax * B.f1_qmax);
  const float gws = pow2f(sg) * q1;
  const float sg3 = pow2f(-((Q ? 0 : B.f1_exp) + sg));
  const float sdz = (Q ? ld_dep(&B.f0_s[ch]) : pow2f(-B.f0_exp)) * pow2f(-B.f_dbexp);
  const float kz = sg3 * sdz;

  float4 ue = make_float4(0.f, 0.f, 0.f, 0.f), ue_n = ue;
  bool rows2 = true, rows2_n = true;
  MetaRegs mr;
  if (nt_all > 0) {  // tile 0 (possibly empty for this half): metadata, basis, G1
    mr.load(a, geo, env, tr.eb, min(TT, tr.ee - tr.eb), W.lane);
    ue_n = mr.store(W.meta(0), true, W.lane, rows2_n);
    mr.load(a, geo, env, tr.eb + TT, min(TT, tr.ee - tr.eb - TT), W.lane);
    tile_basis<false, Q, KSTR64>(a, W, W.meta(0), bsc);
    REQ(BAR_G1, (mma_chain<DR / 16, NPF>(W.tmem_g + SA64, w0, bb, id_f)));
  }
  for (int it = 0; it < nt_all; ++it) {
    ue = ue_n;
    rows2 = rows2_n;
    const int t0 = tr.eb + it * TT;
    const bool more = it + 1 < nt_all;
    const WarpMeta *M = W.meta(it);
    const int n_e = min(TT, tr.ee - t0);  // <= 0: this half has no tile this iteration
    float gh[TT];
    float pf_s = 0.f, pl_s = 0.f;
    int o_l = -1;
    if (n_e > 0) {
#pragma unroll
      for (int i = 0; i < TT; ++i) gh[i] = ld_gather(GHch + (uint32_t)M->nbr[i]);
      const int o_f = M->own[0];
      o_l = M->own[n_e - 1];
      pf_s = ld_gather(Pch + (uint32_t)o_f * D) * gws;
      pl_s = ld_gather(Pch + (uint32_t)o_l * D) * gws;
    } else {
#pragma unroll
      for (int i = 0; i < TT; ++i) gh[i] = 0.f;
    }
    W.wait(BAR_G1, it);
    tile_h_bwd<Q, KSTR64>(W, rs0, b0c, hk, kz, stash);
    REQ(BAR_G2, (mma_chain_ts<D / 16, NPF>(W.tmem_g + SA64, w1h, w1l, hb, id_f)));
    if (more) {
      ue_n = mr.store(W.meta(it + 1), true, W.lane, rows2_n);
      mr.load(a, geo, env, t0 + 2 * TT, min(TT, tr.ee - t0 - 2 * TT), W.lane);
    }
    W.wait(BAR_G2, it);
#pragma unroll
    for (int j = 0; j < TT / 8; ++j) {
      const int4 oa = *(const int4 *)&M->own[8 * j], ob = *(const int4 *)&M->own[8 * j + 4];
      const int oo[8] = {oa.x, oa.y, oa.z, oa.w, ob.x, ob.y, ob.z, ob.w};
      float v[8];
      if (rows2) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = gh[8 * j + i] * (oo[i] == o_l ? pl_s : pf_s);
        put8<true, KSTR64>(W.hb, D, ch, W.eo + 8 * j, v, 1.f);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = gh[8 * j + i] * ld_gather(Pch + (uint32_t)max(oo[i], 0) * D);
        put8<true, KSTR64>(W.hb, D, ch, W.eo + 8 * j, v, gws);
      }
    }
    REQ(BAR_G3, (mma_chain_ts<D / 16, NPB>(W.tmem_g + SB64, w1th, w1tl, hb, id_f)));
    if (n_e > 0) {  // grad_P rows = src-segment sums of gH * w
      float v[TT];
      tc::tmem_ld32w(W.tl + SA64, v);
#pragma unroll
      for (int i = 0; i < TT; ++i) v[i] = gh[i] * (v[i] * s1 + b1c);
      if (SC) {
        scatter_tile(seg.outc, M->own, v, n_e);
      } else {
        if (n_e < TT) {
#pragma unroll
          for (int i = 0; i < TT; ++i) v[i] = i < n_e ? v[i] : 0.f;
        }
        seg.tile(M->own, v);
      }
    } else {
      float v[TT];
      tc::tmem_ld32w(W.tl + SA64, v);  // warp-collective order kept; values unused
      (void)v;
    }
    tile_basis<true, Q, KSTR64>(a, W, M, (float)B.f_dbexp);
    REQ(BAR_G1P, (mma_chain<DR / 16, NPB>(W.tmem_g + SA64, w0, bb, id_f)));
    W.wait(BAR_G3, it);
    {
      float gz[TT];
      tc::tmem_ld32w(W.tl + SB64, gz);
#pragma unroll
      for (int i = 0; i < TT; i += 4) {
        const float4 sv = stash[(i / 4) * D + ch];
        gz[i] *= sv.x; gz[i + 1] *= sv.y; gz[i + 2] *= sv.z; gz[i + 3] *= sv.w;
      }
      tc::tmem_st32(W.tl + SB64, gz);
      tc::tmem_st_wait();
    }
    W.wait(BAR_G1P, it);
    float p[TT];
    {
      float dz[TT];
      tc::tmem_ld32w(W.tl + SB64, p);
      tc::tmem_ld32w(W.tl + SA64, dz);
#pragma unroll
      for (int i = 0; i < TT; ++i) p[i] *= dz[i];
    }
    if (more) {
      tile_basis<false, Q, KSTR64>(a, W, W.meta(it + 1), bsc);
      REQ(BAR_G1, (mma_chain<DR / 16, NPF>(W.tmem_g + SA64, w0, bb, id_f)));
    }
    float *xg = &sh->xg[u][it & 1][0][0];
    xg[W.q * TT + W.lane] = warp_edge_sum(p, W.lane);
    __syncwarp();
    if (W.lane == 0) tc::mbar_arrive(&sh->xbar[u]);
    if (W.q == 0) {
      tc::mbar_wait(&sh->xbar[u], (uint32_t)(it & 1));
      const int e = W.lane;
      if (e < n_e) {
        const float gd = ((xg[e] + xg[TT + e]) + xg[2 * TT + e]) + xg[3 * TT + e];
        const float inv = ue.w > TINY_DISTANCE ? 1.f / ue.w : 0.f;
        const float sc = gd * inv;
        float4 g = make_float4(sc * ue.x, sc * ue.y, sc * ue.z, 0.f);
        if (SC) {  // np.add.at(grad_r, dst, gu); np.add.at(grad_r, src, -gu)
          float *gd_ = (float *)&gr[(uint32_t)M->nbr[e] / D];
          float *gs_ = (float *)&gr[M->own[e]];
          atomicAdd(gd_, g.x); atomicAdd(gd_ + 1, g.y); atomicAdd(gd_ + 2, g.z);
          atomicAdd(gs_, -g.x); atomicAdd(gs_ + 1, -g.y); atomicAdd(gs_ + 2, -g.z);
        } else {
          float4 *dst = &gsum[t0 + e];
          if (accumulate) {
            const float4 o = *dst;
            g.x += o.x; g.y += o.y; g.z += o.z;
          }
          *dst = g;
        }
      }
    }
  }
  if (!SC) seg.finish();
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(sh->tmem);
}

// ---------------------------------------------------------------------------
// Backward in forward mode (the default; FCG_BWD_FM=0 selects k_edge_bwd64).
//
// flash_block_backward (flash.py:272-295) needs, per edge, grad_P rows
// (src-segment sums of gH*w) and grad_d = sum_c grad_w[c] dw[c]/dd with
// grad_w = gH[dst] * P[src].  The reference reaches grad_d in reverse mode
// (grad_b = filter backward of grad_w, then grad_b . db); here the
// derivative of the filter output is propagated forward instead:
//   dw/dd = W1 (ssp'(z0) * (W0 db)) = W1 v,
// so one tile needs two MMA chains, both with weights as the A operand:
//   [G1 | G1'] = W0 [b | db]  -> z0 | dz0    (K = 64, N = 2 x 64 edges)
//   [G2 | G3 ] = W1 [h | v ]  -> w  | u      (K = 128, N = 2 x 64 edges)
// with h = ssp(z0), v = ssp'(z0) dz0; then grad_P += gH*(w + b1) and
// grad_d = sum_c gH[c] P[src][c] u[c].  Compared with k_edge_bwd64 that is
// the same number of MMAs (72 per tile, fp32), but two completion waits per
// tile instead of four, no W1^T (TMEM holds W1 and W0, 192 columns), no
// ssp' stash and no TMEM store; grad_w never becomes an MMA operand.
//
// Work decomposition as k_edge_bwd64: 2 groups x 8 warps, a group tile = 32
// edges of each of its two work units (warps 0-3 / 4-7), one walker per CSR
// row.  TMEM: group g owns columns [128g, 128g+128): [0, 64) z0 then w,
// [64, 128) dz0 then u (unit half hf at +32 hf); W1 hi|lo at 256, W0 hi|lo at
// 384.  Shared memory per group: the K=64 basis operand [b | db] (N = 128)
// and the K=128 operand [h | v] (N = 128), hi and lo images.
constexpr uint32_t FM_TW1 = 256, FM_TW0 = 384;
// Group shape: UPG work units per group (2: two groups of 8 warps, N = 128
// operands; 1: four groups of 4 warps, N = 64).  Per group: the basis
// operand [b | db] (K = 64) and [h | v] (K = 128), N = 64 UPG, hi|lo.
template <int UPG>
struct FmCfg {
  static constexpr int NGRP = 4 / UPG;
  static constexpr uint32_t N = 64u * UPG;          // operand columns: 32 UPG edges x 2
  static constexpr uint32_t RH = 32u * UPG;         // right half: dz0 / u columns
  static constexpr uint32_t KS = (N / 8) * 128;     // bytes per 8 K-rows
  static constexpr uint32_t BB = 2 * DR * N * 2;
  static constexpr uint32_t HV = 2 * D * N * 2;
  static constexpr uint32_t GBUF = BB + HV;
};
constexpr uint32_t FM_SM_META = 4 * (2 * DR * 64 * 2 + 2 * D * 64 * 2);  // 192 KB either shape
constexpr int FM_MBUF = 3;  // metadata buffers per work unit (tiles it, it+1, it+2)

// Tile metadata of one work unit, shared by its four warps and filled by
// cp.async (no registers in flight): raw CSR columns of the tile's edges.
// Slots past the unit's edge count keep values of an earlier tile (zero at
// start) — valid indices and finite geometry; every consumer masks them.
struct UnitMeta {
  int own[TT], nbr[TT];
  float d[TT], env[TT], denv[TT];
};
struct FmShared {
  UnitMeta um[4][FM_MBUF];
  float xg[4][2][4][TT];     // per-quarter partial grad_d (double-buffered)
  uint64_t bar[4][4];        // GEMM completion per group, per kind
  uint64_t xbar[4];          // the four partial grad_d rows of a unit's tile are written
  uint64_t mbar[4][FM_MBUF]; // a metadata buffer's copies landed (128 noinc arrivals)
  uint64_t wbar;             // weight images landed
  unsigned int req[4][4];    // operand arrivals per GEMM kind
  uint32_t tmem;
};
constexpr uint32_t FM_SM_TOTAL = FM_SM_META + sizeof(FmShared);
static_assert(SM_W1 + 2 * W1_BYTES <= FM_SM_META, "weight staging aliases the group buffers");
static_assert(FM_SM_TOTAL + 1024 <= 232448, "forward-mode backward shared memory budget");
static_assert(FM_TW0 + DR <= 512, "TMEM budget");

__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tc::smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(bar))
               : "memory");
}

// Copies of tile columns [t0, t0+count) into a unit buffer: warp quarter q
// moves one or two of the five columns, one element per lane; every thread
// of the unit's four warps then arrives (noinc) on the buffer's mbarrier.
__device__ __forceinline__ void meta_issue(const EdgeArgs &a, const float4 *geo, const float2 *env,
                                           UnitMeta *m, uint64_t *bar, int t0, int count, int q,
                                           int lane) {
  if (lane < count) {
    const int k = t0 + lane;
    if (q == 0) cp_async4(&m->own[lane], &a.own[k]);
    else if (q == 1) cp_async4(&m->nbr[lane], &a.nbr[k]);
    else if (q == 2) cp_async4(&m->d[lane], &geo[k].w);
    else {
      cp_async4(&m->env[lane], &env[k].x);
      cp_async4(&m->denv[lane], &env[k].y);
    }
  }
  cp_async_arrive_noinc(bar);
}

// W1 hi | lo and W0 hi | lo from the staged images into TMEM: warp w moves
// image (w / 4) % 4 for its lane quarter.
// Threads from TC_THREADS on (the MMA warpgroup of the WS kernels) only join
// the closing barrier: every thread reaches the same bar.sync.
__device__ __forceinline__ void load_fm_weights_tmem(const uint8_t *sm, uint32_t tmem) {
  const int w = threadIdx.x >> 5, q = w & 3, m = 32 * q + (threadIdx.x & 31);
  const int img = (w >> 2) & 3;  // 0: W1 hi, 1: W1 lo, 2: W0 hi, 3: W0 lo
  const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
  if (threadIdx.x < TC_THREADS) {
    if (img < 2)
      image_row_to_tmem<false>((const uint16_t *)(sm + SM_W1 + (img & 1) * W1_BYTES), D, m,
                               lane_base + FM_TW1 + (img & 1) * (D / 2));
    else
      image_row_to_tmem<false>((const uint16_t *)(sm + SM_W0 + (img & 1) * W0_BYTES), DR, m,
                               lane_base + FM_TW0 + (img & 1) * (DR / 2));
  }
  prologue_done();
}

// One tile's pair of chains into the group's columns: the left half (z0 /
// w, NPL products) and the right half (dz0 / u, NPR products), N/2 columns
// each.  Equal product counts issue one chain over both halves.
template <int KS, int NPL, int NPR, int N>
__device__ __forceinline__ void mma_pair_ts(uint32_t d, uint32_t a_hi, uint32_t a_lo, Desc b) {
  if (NPL == NPR) {
    mma_chain_ts<KS, NPL>(d, a_hi, a_lo, b, tc::idesc_f16(128, N, 0, 1));
  } else {
    const uint32_t idh = tc::idesc_f16(128, N / 2, 0, 1);
    mma_chain_ts<KS, NPL>(d, a_hi, a_lo, b, idh);
    Desc br = b;
    br.hi += (N / 2 / 8) * 128u / 16u;  // columns N/2.. of the operand (core rows of 128 B)
    br.lo += (N / 2 / 8) * 128u / 16u;
    mma_chain_ts<KS, NPR>(d + N / 2, a_hi, a_lo, br, idh);
  }
}

// Basis [b | db] of one tile from a unit buffer into the group's K=64 operand.
template <bool Q, int UPG, bool PK = false>
__device__ __forceinline__ void tile_basis_pair(const EdgeArgs &a, Wctx &W, const UnitMeta *m,
                                                float bsc, float dbsc) {
  using C = FmCfg<UPG>;
  tile_basis<false, Q, C::KS, PK>(a, W, (const WarpMeta *)m, bsc);
  W.eo += C::RH;
  tile_basis<true, Q, C::KS, PK>(a, W, (const WarpMeta *)m, dbsc);
  W.eo -= C::RH;
}

template <bool Q, int UPG>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_edge_bwd_fm(const EdgeArgs a, const float4 *geo, const float2 *env,
              const int32_t *unit_rows, const float *P,
              const float *GH, float *GP, float4 *gsum,
              int accumulate) {
  extern __shared__ __align__(1024) uint8_t sm[];
  FmShared *sh = (FmShared *)(sm + FM_SM_META);
  const fcg_block &B = a.blk;
  pdl_trigger();
  if (threadIdx.x == 0) {
    tc::mbar_init(&sh->wbar, 1);
    tc::fence_mbar_init();
    tc::mbar_expect_tx(&sh->wbar, 2 * W0_BYTES + 2 * W1_BYTES);
    tc::bulk_g2s(sm + SM_W0, B.f0_img, 2 * W0_BYTES, &sh->wbar);
    tc::bulk_g2s(sm + SM_W1, B.f1_img, 2 * W1_BYTES, &sh->wbar);
  }
  using C = FmCfg<UPG>;
  if (threadIdx.x < 4) {
    const int u0 = threadIdx.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      tc::mbar_init(&sh->bar[u0][i], 1);
      sh->req[u0][i] = 0u;
    }
    tc::mbar_init(&sh->xbar[u0], 4);
#pragma unroll
    for (int b = 0; b < FM_MBUF; ++b) tc::mbar_init(&sh->mbar[u0][b], 128);
    tc::fence_mbar_init();
  }
  for (int i = threadIdx.x; i < (int)(sizeof(sh->um) / 4); i += blockDim.x)
    ((int *)sh->um)[i] = 0;
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&sh->tmem);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  tc::mbar_wait(&sh->wbar, 0);
  load_fm_weights_tmem(sm, sh->tmem);  // ends with the PDL wait

  Wctx W;
  W.w = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  W.g = W.w / (4 * UPG);
  const int hf = UPG == 2 ? (W.w >> 2) & 1 : 0;
  const int u = UPG * W.g + hf;  // work unit / metadata / grad_d partials of this warp
  W.q = W.w & 3;
  W.lane = threadIdx.x & 31;
  W.ch = 32 * W.q + W.lane;
  W.eo = 32 * hf;
  W.amask = 4u * UPG - 1u;
  W.sh = (TcShared *)nullptr;
  W.bb = sm + W.g * C::GBUF;
  W.hb = W.bb + C::BB;
  W.sbb = tc::smem_u32(W.bb);
  W.shb = tc::smem_u32(W.hb);
  W.tmem_g = sh->tmem + 2u * C::RH * W.g;
  W.tl = W.tmem_g + ((uint32_t)(32 * W.q) << 16) + 32u * hf;
  constexpr int NB = Q ? 1 : 3, NDB = Q ? 2 : 3, NH = Q ? 1 : 3, NV = Q ? 2 : 3;
  const uint32_t w0h = sh->tmem + FM_TW0, w0l = w0h + DR / 2;
  const uint32_t w1h = sh->tmem + FM_TW1, w1l = w1h + D / 2;
  const Desc bb = adesc<C::KS>(W.sbb, DR), hb = adesc<C::KS>(W.shb, D);

  const UnitRange tr = unit_range(a, unit_rows, NGRP * blockIdx.x + u);
  const int ntiles = (tr.ee - tr.eb + TT - 1) / TT;
  int nt_all = ntiles;  // the group's iterations
  if (UPG == 2) {
    const UnitRange to = unit_range(a, unit_rows, NGRP * blockIdx.x + (u ^ 1));
    nt_all = max(ntiles, (to.ee - to.eb + TT - 1) / TT);
  }
  const int ch = W.ch;
  const int lane = W.lane;
  const float *GHch = opaque_ptr(GH + ch);
  const float *Pch = opaque_ptr(P + ch);
  SegSum seg;
  seg.row = ntiles > 0 ? a.own[tr.eb] : -1;
  seg.acc = 0.f;
  seg.outc = opaque_ptr(GP + ch);

  // E1 constants (this thread's channel = hidden unit k of filter layer 0)
  // (the W16 row scales are re-read from L1 where they are used: held
  // across the loop they cost the kernel its last registers)
  const float b0c = ld_dep(&B.f0_b[ch]);
  const float hs = Q ? 1.f : pow2f(B.f_hexp);
  const HScale hk(Q ? 1.f : pow2f(-(B.f0_exp + 14)), b0c, hs);
  // E2 constants (this thread's channel = output channel c of filter layer 1)
  const float b1c = ld_dep(&B.f1_b[ch]);
  const float bsc = Q ? 0.f : 14.f, dbsc = (float)B.f_dbexp;
  auto count_of = [&](int t) { return min(TT, tr.ee - (tr.eb + t * TT)); };
  auto um = [&](int t) { return &sh->um[u][t % FM_MBUF]; };
  auto meta_wait = [&](int t) {
    tc::mbar_wait(&sh->mbar[u][t % FM_MBUF], (uint32_t)((t / FM_MBUF) & 1));
  };

  if (nt_all > 0) {  // tiles 0 and 1 in flight; tile 0's [b | db] and G1 | G1'
    meta_issue(a, geo, env, um(0), &sh->mbar[u][0], tr.eb, count_of(0), W.q, lane);
    if (nt_all > 1)
      meta_issue(a, geo, env, um(1), &sh->mbar[u][1], tr.eb + TT, count_of(1), W.q, lane);
    meta_wait(0);
    tile_basis_pair<Q, UPG>(a, W, um(0), bsc, dbsc);
    if (W.arrive_fm(sh->req[W.g], BAR_G1)) {
      mma_pair_ts<DR / 16, NB, NDB, C::N>(W.tmem_g, w0h, w0l, bb);
      tc::mma_commit_warp(&sh->bar[W.g][BAR_G1]);
    }
    __syncwarp();
  }
  for (int it = 0; it < nt_all; ++it) {
    const int t0 = tr.eb + it * TT;
    const bool more = it + 1 < nt_all;
    const UnitMeta *M = um(it);
    const int n_e = count_of(it);  // <= 0: this half has no tile this iteration

    // ---- E1: h = ssp(z0), v = ssp'(z0) dz0 -> [h | v] -----------------------
    // z0 = acc * rs0 + b0; v * 2^f_vexp from the dz0 accumulator (W0 *
    // 2^f0_exp (fp32) or w16 (W16, row scale s0) times db * 2^f_dbexp)
    const float rs0 = Q ? ld_dep(&B.f0_s[ch]) : pow2f(-(B.f0_exp + 14));
    const float kv = Q ? rs0 * pow2f(B.f_vexp - B.f_dbexp)
                       : pow2f(B.f_vexp - B.f0_exp - B.f_dbexp);
    STAMP(1, (W.w & 7) == 0, W.g, it, 0);
    tc::mbar_wait(&sh->bar[W.g][BAR_G1], (uint32_t)(it & 1));
    tc::fence_after_sync();
    STAMP(1, (W.w & 7) == 0, W.g, it, 1);
#pragma unroll
    for (int c0 = 0; c0 < TT; c0 += 16) {
      float z[16], dz[16];
      tc::tmem_ld16w(W.tl + c0, z);
      tc::tmem_ld16w(W.tl + C::RH + c0, dz);
#pragma unroll
      for (int i = 0; i < 16; i += Q ? 1 : 2) {
        if (Q) {  // scalar: pairing the W16 loop costs that kernel a spill
          const float zz = z[i] * rs0 + b0c;
          dz[i] *= sigmoid_fast(zz) * kv;  // kv * ssp'(z0)
          z[i] = ssp_fast(zz);  // rounded to fp16 by put8's hi-only pack (quantize.py:80-88)
        } else {  // a pair of edges per instruction
          const float2 h = ssp_scaled2(fma2(make_float2(z[i], z[i + 1]), f2(hk.rs), f2(hk.b)),
                                       hk.c_ln2, hk.c_e);                       // hs * h
          const float2 sp = fma2(f2(-0.5f * kv), ex2_2(mul2(h, f2(hk.c_e))), f2(kv));  // kv ssp'
          const float2 d = mul2(make_float2(dz[i], dz[i + 1]), sp);
          z[i] = h.x; z[i + 1] = h.y;
          dz[i] = d.x; dz[i + 1] = d.y;
        }
      }
#pragma unroll
      for (int j = 0; j < 16; j += 8) {
        put8<!Q, C::KS>(W.hb, D, ch, W.eo + c0 + j, &z[j], 1.f);
        put8<true, C::KS>(W.hb, D, ch, C::RH + W.eo + c0 + j, &dz[j], 1.f);
      }
    }
    STAMP(1, (W.w & 7) == 0, W.g, it, 2);
    if (W.arrive_fm(sh->req[W.g], BAR_G2)) {
      mma_pair_ts<D / 16, NH, NV, C::N>(W.tmem_g, w1h, w1l, hb);
      tc::mma_commit_warp(&sh->bar[W.g][BAR_G2]);
    }
    __syncwarp();
    STAMP(1, (W.w & 7) == 0, W.g, it, 3);

    // ---- gathers of this tile (consumed after the [G2 | G3] wait) ------------
    float gh[TT];
    float pf = 0.f, pm = 0.f, pl = 0.f;  // P[src] of the first, middle and last row
    int o_f = -1, o_l = -1;
    bool rows3 = true;
    float4 ue = make_float4(0.f, 0.f, 0.f, 0.f);
    if (n_e > 0) {
      const int o = M->own[lane];
      o_f = M->own[0];
      o_l = M->own[n_e - 1];
      const unsigned other = __ballot_sync(0xffffffffu, lane < n_e && o != o_f && o != o_l);
      const int mid = other ? __shfl_sync(0xffffffffu, o, __ffs(other) - 1) : o_f;
      rows3 = __all_sync(0xffffffffu, lane >= n_e || o == o_f || o == o_l || o == mid);
#pragma unroll
      for (int i = 0; i < TT; ++i) gh[i] = ld_gather(GHch + ((uint32_t)M->nbr[i] << 7));
      pf = ld_gather(Pch + (uint32_t)o_f * D);  // scaled by ku where used
      pm = ld_gather(Pch + (uint32_t)mid * D);
      pl = ld_gather(Pch + (uint32_t)o_l * D);
      if (W.q == 0 && lane < n_e) ue = ld_dep(&geo[t0 + lane]);
    } else {
#pragma unroll
      for (int i = 0; i < TT; ++i) gh[i] = 0.f;
    }
    if (more) {  // next tile's [b | db] (the basis buffer is free: G1 done)
      meta_wait(it + 1);
      tile_basis_pair<Q, UPG>(a, W, um(it + 1), bsc, dbsc);
    }

    // ---- E2: grad_P segment sums, grad_d partials --------------------------
    const float s1 = Q ? ld_dep(&B.f1_s[ch]) : pow2f(-(B.f1_exp + B.f_hexp));
    const float ku = Q ? s1 * pow2f(-B.f_vexp) : pow2f(-(B.f1_exp + B.f_vexp));
    STAMP(1, (W.w & 7) == 0, W.g, it, 4);
    tc::mbar_wait(&sh->bar[W.g][BAR_G2], (uint32_t)(it & 1));
    tc::fence_after_sync();
    STAMP(1, (W.w & 7) == 0, W.g, it, 5);
    // every warp of the group is past iteration it-1: tile it+2's copies may
    // reuse the buffer of tile it-1
    if (it + 2 < nt_all)
      meta_issue(a, geo, env, um(it + 2), &sh->mbar[u][(it + 2) % FM_MBUF], t0 + 2 * TT,
                 count_of(it + 2), W.q, lane);
    float q[TT];
    {
      const unsigned st = n_e > 0 ? seg.starts_n(M->own, n_e) : 0u;
#pragma unroll
      for (int h = 0; h < TT; h += 16) {
        float v[16];
        tc::tmem_ld16w(W.tl + h, v);  // w accumulator
        if (n_e > 0) {
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const float2 m = mul2(make_float2(gh[h + i], gh[h + i + 1]),
                                  fma2(make_float2(v[i], v[i + 1]), f2(s1), f2(b1c)));
            v[i] = h + i < n_e ? m.x : 0.f;
            v[i + 1] = h + i + 1 < n_e ? m.y : 0.f;
          }
          seg.half(M->own, v, h, st);
        }
      }
      tc::tmem_ld32w(W.tl + C::RH, q);  // u accumulator
    }
    STAMP(1, (W.w & 7) == 0, W.g, it, 6);
    if (more) {  // TMEM columns read: the next tile's G1 | G1' may overwrite them
      if (W.arrive_fm(sh->req[W.g], BAR_G1)) {
        mma_pair_ts<DR / 16, NB, NDB, C::N>(W.tmem_g, w0h, w0l, bb);
        tc::mma_commit_warp(&sh->bar[W.g][BAR_G1]);
      }
      __syncwarp();
    }
    if (rows3) {
      pf *= ku; pm *= ku; pl *= ku;
#pragma unroll
      for (int j = 0; j < TT; j += 4) {
        const int4 o4 = *(const int4 *)&M->own[j];
        const int oo[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
          q[j + i] *= gh[j + i] * (oo[i] == o_l ? pl : (oo[i] == o_f ? pf : pm));
      }
    } else {  // four or more rows (~5% of coil-269 tiles): per-edge gathers
#pragma unroll
      for (int i = 0; i < TT; ++i)
        q[i] *= gh[i] * ld_gather(Pch + (uint32_t)M->own[i] * D) * ku;
    }
    STAMP(1, (W.w & 7) == 0, W.g, it, 7);
    float *xg = &sh->xg[u][it & 1][0][0];
    xg[W.q * TT + lane] = warp_edge_sum(q, lane);
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&sh->xbar[u]);
    if (W.q == 0) {
      tc::mbar_wait(&sh->xbar[u], (uint32_t)(it & 1));
      const int e = lane;
      if (e < n_e) {
        const float gd = ((xg[e] + xg[TT + e]) + xg[2 * TT + e]) + xg[3 * TT + e];
        // backward edge: dst = nbr, src = own, u = r_nbr - r_own (flash.py:279)
        const float inv = ue.w > TINY_DISTANCE ? 1.f / ue.w : 0.f;
        const float sc = -gd * inv;
        float4 g = make_float4(sc * ue.x, sc * ue.y, sc * ue.z, 0.f);
        float4 *dst = &gsum[t0 + e];
        if (accumulate) {
          const float4 o = *dst;
          g.x += o.x; g.y += o.y; g.z += o.z;
        }
        *dst = g;
      }
    }
    STAMP(1, (W.w & 7) == 0, W.g, it, 8);
  }
  seg.finish();
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(sh->tmem);
}

// Forward-mode backward with the dedicated MMA warpgroup of k_edge_fwd_ws
// (the default; FCG_BWD_WS=0 selects k_edge_bwd_fm with last-arriver issue).
// Without the MMA issue code the epilogue fits the 112 registers with no
// spills: 0.848 -> 0.814 ms/step at C2.
struct BwdWsShared {
  FmShared fm;
  uint64_t ready[2][4];
};
static_assert(FM_SM_META + sizeof(BwdWsShared) + 1024 <= 232448, "backward WS smem budget");

template <bool Q, int UPG>
__global__ void __launch_bounds__(WS_THREADS, 1)
k_edge_bwd_fmws(const EdgeArgs a, const float4 *geo, const float2 *env,
                const int32_t *unit_rows, const float *P,
                const float *GH, float *GP, float4 *gsum,
                int accumulate) {
  static_assert(UPG == 2, "two groups of 8 warps");
  extern __shared__ __align__(1024) uint8_t sm[];
  BwdWsShared *wsh = (BwdWsShared *)(sm + FM_SM_META);
  FmShared *sh = &wsh->fm;
  const fcg_block &B = a.blk;
  pdl_trigger();
  if (threadIdx.x == 0) {
    tc::mbar_init(&sh->wbar, 1);
    tc::fence_mbar_init();
    tc::mbar_expect_tx(&sh->wbar, 2 * W0_BYTES + 2 * W1_BYTES);
    tc::bulk_g2s(sm + SM_W0, B.f0_img, 2 * W0_BYTES, &sh->wbar);
    tc::bulk_g2s(sm + SM_W1, B.f1_img, 2 * W1_BYTES, &sh->wbar);
  }
  using C = FmCfg<UPG>;
  if (threadIdx.x < 4) {
    const int u0 = threadIdx.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      tc::mbar_init(&sh->bar[u0][i], 1);
      sh->req[u0][i] = 0u;
    }
    tc::mbar_init(&sh->xbar[u0], 4);
#pragma unroll
    for (int b = 0; b < FM_MBUF; ++b) tc::mbar_init(&sh->mbar[u0][b], 128);
    if (u0 < 2) {
#pragma unroll
      for (int i = 0; i < 4; ++i) tc::mbar_init(&wsh->ready[u0][i], 8);
    }
    tc::fence_mbar_init();
  }
  for (int i = threadIdx.x; i < (int)(sizeof(sh->um) / 4); i += blockDim.x)
    ((int *)sh->um)[i] = 0;
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&sh->tmem);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  tc::mbar_wait(&sh->wbar, 0);
  load_fm_weights_tmem(sm, sh->tmem);  // ends with the PDL wait + block barrier
  constexpr int NB = Q ? 1 : 3, NDB = Q ? 2 : 3, NH = Q ? 1 : 3, NV = Q ? 2 : 3;
  const uint32_t w0h = sh->tmem + FM_TW0, w0l = w0h + DR / 2;
  const uint32_t w1h = sh->tmem + FM_TW1, w1l = w1h + D / 2;
  if (threadIdx.x >= TC_THREADS) {  // the MMA warpgroup (see k_edge_fwd_ws)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 24;\n" ::: "memory");
    if (threadIdx.x >= TC_THREADS + 32) return;
    int nt[2], c[2] = {0, 0};
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const UnitRange r0 = unit_range(a, unit_rows, NGRP * blockIdx.x + 2 * g);
      const UnitRange r1 = unit_range(a, unit_rows, NGRP * blockIdx.x + 2 * g + 1);
      nt[g] = max((r0.ee - r0.eb + TT - 1) / TT, (r1.ee - r1.eb + TT - 1) / TT);
    }
    while (c[0] < 2 * nt[0] || c[1] < 2 * nt[1]) {
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        if (c[g] >= 2 * nt[g]) continue;
        const int kind = (c[g] & 1) ? BAR_G2 : BAR_G1;
        if (!mbar_try(&wsh->ready[g][kind], (uint32_t)((c[g] >> 1) & 1))) continue;
        tc::fence_after_sync();
        const uint8_t *bbp = sm + g * C::GBUF;
        const uint32_t tg = sh->tmem + 2u * C::RH * g;
        if (kind == BAR_G1)
          mma_pair_ts<DR / 16, NB, NDB, C::N>(tg, w0h, w0l, adesc<C::KS>(tc::smem_u32(bbp), DR));
        else
          mma_pair_ts<D / 16, NH, NV, C::N>(tg, w1h, w1l,
                                            adesc<C::KS>(tc::smem_u32(bbp + C::BB), D));
        tc::mma_commit_warp(&sh->bar[g][kind]);
        ++c[g];
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 112;\n" ::: "memory");

  Wctx W;
  W.w = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  W.g = W.w / (4 * UPG);
  const int hf = UPG == 2 ? (W.w >> 2) & 1 : 0;
  const int u = UPG * W.g + hf;  // work unit / metadata / grad_d partials of this warp
  W.q = W.w & 3;
  W.lane = threadIdx.x & 31;
  W.ch = 32 * W.q + W.lane;
  W.eo = 32 * hf;
  W.amask = 4u * UPG - 1u;
  W.sh = (TcShared *)nullptr;
  W.bb = sm + W.g * C::GBUF;
  W.hb = W.bb + C::BB;
  W.sbb = tc::smem_u32(W.bb);
  W.shb = tc::smem_u32(W.hb);
  W.tmem_g = sh->tmem + 2u * C::RH * W.g;
  W.tl = W.tmem_g + ((uint32_t)(32 * W.q) << 16) + 32u * hf;

  const UnitRange tr = unit_range(a, unit_rows, NGRP * blockIdx.x + u);
  const int ntiles = (tr.ee - tr.eb + TT - 1) / TT;
  int nt_all = ntiles;  // the group's iterations
  if (UPG == 2) {
    const UnitRange to = unit_range(a, unit_rows, NGRP * blockIdx.x + (u ^ 1));
    nt_all = max(ntiles, (to.ee - to.eb + TT - 1) / TT);
  }
  const int ch = W.ch;
  const int lane = W.lane;
  const float *GHch = opaque_ptr(GH + ch);
  const float *Pch = opaque_ptr(P + ch);
  SegSum seg;
  seg.row = ntiles > 0 ? a.own[tr.eb] : -1;
  seg.acc = 0.f;
  seg.outc = opaque_ptr(GP + ch);

  // E1 constants (this thread's channel = hidden unit k of filter layer 0)
  // (the W16 row scales are re-read from L1 where they are used: held
  // across the loop they cost the kernel its last registers)
  const float b0c = ld_dep(&B.f0_b[ch]);
  const float hs = Q ? 1.f : pow2f(B.f_hexp);
  const HScale hk(Q ? 1.f : pow2f(-(B.f0_exp + 14)), b0c, hs);
  // E2 constants (this thread's channel = output channel c of filter layer 1)
  const float b1c = ld_dep(&B.f1_b[ch]);
  const float bsc = Q ? 0.f : 14.f, dbsc = (float)B.f_dbexp;
  auto count_of = [&](int t) { return min(TT, tr.ee - (tr.eb + t * TT)); };
  auto um = [&](int t) { return &sh->um[u][t % FM_MBUF]; };
  auto meta_wait = [&](int t) {
    tc::mbar_wait(&sh->mbar[u][t % FM_MBUF], (uint32_t)((t / FM_MBUF) & 1));
  };

  if (nt_all > 0) {  // tiles 0 and 1 in flight; tile 0's [b | db] and G1 | G1'
    meta_issue(a, geo, env, um(0), &sh->mbar[u][0], tr.eb, count_of(0), W.q, lane);
    if (nt_all > 1)
      meta_issue(a, geo, env, um(1), &sh->mbar[u][1], tr.eb + TT, count_of(1), W.q, lane);
    meta_wait(0);
    tile_basis_pair<Q, UPG>(a, W, um(0), bsc, dbsc);
    ws_ready(&wsh->ready[W.g][BAR_G1]);
  }
  for (int it = 0; it < nt_all; ++it) {
    const int t0 = tr.eb + it * TT;
    const bool more = it + 1 < nt_all;
    const UnitMeta *M = um(it);
    const int n_e = count_of(it);  // <= 0: this half has no tile this iteration

    // ---- E1: h = ssp(z0), v = ssp'(z0) dz0 -> [h | v] -----------------------
    // z0 = acc * rs0 + b0; v * 2^f_vexp from the dz0 accumulator (W0 *
    // 2^f0_exp (fp32) or w16 (W16, row scale s0) times db * 2^f_dbexp)
    const float rs0 = Q ? ld_dep(&B.f0_s[ch]) : pow2f(-(B.f0_exp + 14));
    const float kv = Q ? rs0 * pow2f(B.f_vexp - B.f_dbexp)
                       : pow2f(B.f_vexp - B.f0_exp - B.f_dbexp);
    const float e1rs = Q ? rs0 : hk.rs, e1b = Q ? b0c : hk.b;
    const float e1cl = Q ? kLn2 : hk.c_ln2, e1ce = Q ? -kLog2e : hk.c_e;
    STAMP(1, (W.w & 7) == 0, W.g, it, 0);
    tc::mbar_wait(&sh->bar[W.g][BAR_G1], (uint32_t)(it & 1));
    tc::fence_after_sync();
    STAMP(1, (W.w & 7) == 0, W.g, it, 1);
#pragma unroll
    for (int c0 = 0; c0 < TT; c0 += 16) {
      float z[16], dz[16];
      tc::tmem_ld16w(W.tl + c0, z);
      tc::tmem_ld16w(W.tl + C::RH + c0, dz);
#pragma unroll
      for (int i = 0; i < 16; i += 2) {  // a pair of edges per instruction
        // fp32: hs * h = hs * ssp(z0); W16: ssp(z0), rounded to fp16 by put8's
        // hi-only pack (quantize.py:80-88).  kv * ssp'(z0) = kv (1 - e^-ssp / 2)
        // from the unrounded value.
        const float2 h = ssp_scaled2(fma2(make_float2(z[i], z[i + 1]), f2(e1rs), f2(e1b)),
                                     e1cl, e1ce);
        const float2 sp = fma2(f2(-0.5f * kv), ex2_2(mul2(h, f2(e1ce))), f2(kv));
        const float2 d = mul2(make_float2(dz[i], dz[i + 1]), sp);
        z[i] = h.x; z[i + 1] = h.y;
        dz[i] = d.x; dz[i + 1] = d.y;
      }
#pragma unroll
      for (int j = 0; j < 16; j += 8) {
        put8<!Q, C::KS, !Q>(W.hb, D, ch, W.eo + c0 + j, &z[j], 1.f);
        put8<true, C::KS, !Q>(W.hb, D, ch, C::RH + W.eo + c0 + j, &dz[j], 1.f);
      }
    }
    STAMP(1, (W.w & 7) == 0, W.g, it, 2);
    ws_ready(&wsh->ready[W.g][BAR_G2]);
    STAMP(1, (W.w & 7) == 0, W.g, it, 3);

    // ---- gathers of this tile (consumed after the [G2 | G3] wait) ------------
    float gh[TT];
    float pf = 0.f, pm = 0.f, pl = 0.f;  // P[src] of the first, middle and last row
    int o_f = -1, o_l = -1;
    int ia = TT, ib = TT;  // tile edges [0, ia): first row, [ia, ib): middle, [ib, n_e): last
    bool rows3 = true;
    float4 ue = make_float4(0.f, 0.f, 0.f, 0.f);
    float3 acc = make_float3(0.f, 0.f, 0.f);  // the slot's grad from the later blocks
    if (n_e > 0) {
      const int o = M->own[lane];
      o_f = M->own[0];
      o_l = M->own[n_e - 1];
      const unsigned other = __ballot_sync(0xffffffffu, lane < n_e && o != o_f && o != o_l);
      const int mid = other ? __shfl_sync(0xffffffffu, o, __ffs(other) - 1) : o_f;
      rows3 = __all_sync(0xffffffffu, lane >= n_e || o == o_f || o == o_l || o == mid);
      {  // the rows are runs (CSR order): edge i's P[src] is a select on i
        ia = __popc(__ballot_sync(0xffffffffu, lane < n_e && o == o_f));
        ib = n_e - __popc(__ballot_sync(0xffffffffu, lane < n_e && o == o_l));
      }
#pragma unroll
      for (int i = 0; i < TT; ++i) gh[i] = ld_gather(GHch + ((uint32_t)M->nbr[i] << 7));
      if (n_e < TT) {  // the unit's last tile (warp-uniform): padding edges carry
                       // gH = 0, so their messages and q terms vanish unmasked
#pragma unroll
        for (int i = 0; i < TT; ++i) gh[i] = i < n_e ? gh[i] : 0.f;
      }
      pf = ld_gather(Pch + (uint32_t)o_f * D);  // scaled by ku where used
      pm = ld_gather(Pch + (uint32_t)mid * D);
      pl = ld_gather(Pch + (uint32_t)o_l * D);
      if (W.q == 0 && lane < n_e) {
        ue = ld_dep(&geo[t0 + lane]);
        if (accumulate) {  // issued a tile ahead of its use: off the iteration's tail
          const float4 o = gsum[t0 + lane];
          acc = make_float3(o.x, o.y, o.z);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < TT; ++i) gh[i] = 0.f;
    }
    if (more) {  // next tile's [b | db] (the basis buffer is free: G1 done)
      meta_wait(it + 1);
      tile_basis_pair<Q, UPG>(a, W, um(it + 1), bsc, dbsc);
    }

    // ---- E2: grad_P segment sums, grad_d partials --------------------------
    const float s1 = Q ? ld_dep(&B.f1_s[ch]) : pow2f(-(B.f1_exp + B.f_hexp));
    const float ku = Q ? s1 * pow2f(-B.f_vexp) : pow2f(-(B.f1_exp + B.f_vexp));
    STAMP(1, (W.w & 7) == 0, W.g, it, 4);
    tc::mbar_wait(&sh->bar[W.g][BAR_G2], (uint32_t)(it & 1));
    tc::fence_after_sync();
    STAMP(1, (W.w & 7) == 0, W.g, it, 5);
    // every warp of the group is past iteration it-1: tile it+2's copies may
    // reuse the buffer of tile it-1
    if (it + 2 < nt_all)
      meta_issue(a, geo, env, um(it + 2), &sh->mbar[u][(it + 2) % FM_MBUF], t0 + 2 * TT,
                 count_of(it + 2), W.q, lane);
    float q[TT];
    {
      tc::tmem_ld32w(W.tl + C::RH, q);  // u accumulator
      const unsigned st = n_e > 0 ? seg.starts_n(M->own, n_e) : 0u;
#pragma unroll
      for (int h = 0; h < TT; h += 16) {
        float v[16];
        tc::tmem_ld16w(W.tl + h, v);  // w accumulator
        // the tile's TMEM is read: the next G1 | G1' may write it while the
        // segment sums run
        if (h + 16 == TT && more) ws_ready(&wsh->ready[W.g][BAR_G1]);
        if (n_e > 0) {
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const float2 m = mul2(make_float2(gh[h + i], gh[h + i + 1]),
                                  fma2(make_float2(v[i], v[i + 1]), f2(s1), f2(b1c)));
            v[i] = m.x;  // zero past n_e (gH = 0 there)
            v[i + 1] = m.y;
          }
          seg.half(M->own, v, h, st);
        }
      }
    }
    STAMP(1, (W.w & 7) == 0, W.g, it, 6);
    if (rows3 && ia >= ib) {  // one or two rows (~60% of C2 tiles): a 2-way select
      pf *= ku; pl *= ku;
#pragma unroll
      for (int i = 0; i < TT; i += 2) {
        const float2 pp = make_float2(i < ia ? pf : pl, i + 1 < ia ? pf : pl);
        const float2 r = mul2(mul2(make_float2(q[i], q[i + 1]), make_float2(gh[i], gh[i + 1])), pp);
        q[i] = r.x;
        q[i + 1] = r.y;
      }
    } else if (rows3 && !Q) {
      pf *= ku; pm *= ku; pl *= ku;
#pragma unroll
      for (int i = 0; i < TT; i += 2) {
        const float2 pp = make_float2(i < ia ? pf : (i < ib ? pm : pl),
                                      i + 1 < ia ? pf : (i + 1 < ib ? pm : pl));
        const float2 r = mul2(mul2(make_float2(q[i], q[i + 1]), make_float2(gh[i], gh[i + 1])), pp);
        q[i] = r.x;
        q[i + 1] = r.y;
      }
    } else if (rows3) {  // W16: by row id (the index form costs that kernel a spill)
      pf *= ku; pm *= ku; pl *= ku;
#pragma unroll
      for (int j = 0; j < TT; j += 4) {
        const int4 o4 = *(const int4 *)&M->own[j];
        const int oo[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
        for (int i = 0; i < 4; i += 2) {
          const float2 pp = make_float2(oo[i] == o_l ? pl : (oo[i] == o_f ? pf : pm),
                                        oo[i + 1] == o_l ? pl : (oo[i + 1] == o_f ? pf : pm));
          const float2 r = mul2(mul2(make_float2(q[j + i], q[j + i + 1]),
                                     make_float2(gh[j + i], gh[j + i + 1])), pp);
          q[j + i] = r.x;
          q[j + i + 1] = r.y;
        }
      }
    } else {  // four or more rows (~5% of coil-269 tiles): per-edge gathers
#pragma unroll
      for (int i = 0; i < TT; ++i)
        q[i] *= gh[i] * ld_gather(Pch + (uint32_t)M->own[i] * D) * ku;
    }
    STAMP(1, (W.w & 7) == 0, W.g, it, 7);
    // the unit's four partial grad_d rows -> its first warp: a named barrier
    // per unit (id 2 + u, 128 threads), arrive-only for the producers.  A
    // producer cannot arrive for tile it+1 before the consumer has synced
    // for tile it: that needs G2 | G3 of tile it+1, i.e. the consumer's E1.
    float *xg = &sh->xg[u][it & 1][0][0];
    xg[W.q * TT + lane] = warp_edge_sum(q, lane);
    if (W.q != 0) asm volatile("bar.arrive %0, 128;" ::"r"(2 + u) : "memory");
    if (W.q == 0) {
      asm volatile("bar.sync %0, 128;" ::"r"(2 + u) : "memory");
      const int e = lane;
      if (e < n_e) {
        const float gd = ((xg[e] + xg[TT + e]) + xg[2 * TT + e]) + xg[3 * TT + e];
        // backward edge: dst = nbr, src = own, u = r_nbr - r_own (flash.py:279)
        const float inv = ue.w > TINY_DISTANCE ? 1.f / ue.w : 0.f;
        const float sc = -gd * inv;
        float4 g = make_float4(sc * ue.x, sc * ue.y, sc * ue.z, 0.f);
        if (accumulate) {
          g.x += acc.x; g.y += acc.y; g.z += acc.z;
        }
        gsum[t0 + e] = g;
      }
    }
    STAMP(1, (W.w & 7) == 0, W.g, it, 8);
  }
  seg.finish();
  tc::fence_before_sync();
  asm volatile("bar.sync 1, %0;" ::"r"(TC_THREADS) : "memory");
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(sh->tmem);
}


static bool bwd_ws_enabled() {  // default on; FCG_BWD_WS=0 selects k_edge_bwd_fm
  static const bool on = [] {
    const char *v = getenv("FCG_BWD_WS");
    return !(v && v[0] == '0');
  }();
  return on;
}

// FCG_BWD_UPG=1: four groups of 4 warps (one work unit each) instead of two of 8
static int bwd_fm_upg() {
  static const int v = [] {
    const char *e = getenv("FCG_BWD_UPG");
    return (e && e[0] == '1') ? 1 : 2;
  }();
  return v;
}

static bool bwd_fm_enabled() {
  static const bool on = [] {
    const char *v = getenv("FCG_BWD_FM");
    return !(v && v[0] == '0');
  }();
  return on;
}

// Default on (1.0415 -> 1.0251 ms/step at C2); FCG_BWD64=0 runs the 4-group
// 32-edge kernel above (A/B).
static bool bwd64_enabled() {
  static const bool on = [] {
    const char *v = getenv("FCG_BWD64");
    return !(v && v[0] == '0');
  }();
  return on;
}

void edge_tc_configure() {
  static bool done = false;
  if (done) return;
  const int smem = (int)(SM_TOTAL + 1024), fsmem = (int)(FWD_SM_TOTAL + 1024);
  cudaFuncSetAttribute(k_edge_fwd_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, fsmem);
  cudaFuncSetAttribute(k_edge_fwd_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, fsmem);
  for (auto k : {k_edge_fwd_ws<false, false>, k_edge_fwd_ws<true, false>,
                 k_edge_fwd_ws<false, true>, k_edge_fwd_ws<true, true>})
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(FWD_SM_META + sizeof(FwdWsShared) + 1024));
  cudaFuncSetAttribute(k_edge_fwd64<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, fsmem);
  cudaFuncSetAttribute(k_edge_fwd64<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, fsmem);
  cudaFuncSetAttribute(k_edge_fwd64<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, fsmem);
  cudaFuncSetAttribute(k_edge_fwd64<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, fsmem);
  cudaFuncSetAttribute(k_edge_bwd_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_edge_bwd_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_edge_bwd_fmws<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(FM_SM_META + sizeof(BwdWsShared) + 1024));
  cudaFuncSetAttribute(k_edge_bwd_fmws<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(FM_SM_META + sizeof(BwdWsShared) + 1024));
  cudaFuncSetAttribute(k_edge_bwd_fm<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(FM_SM_TOTAL + 1024));
  cudaFuncSetAttribute(k_edge_bwd_fm<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(FM_SM_TOTAL + 1024));
  cudaFuncSetAttribute(k_edge_bwd_fm<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(FM_SM_TOTAL + 1024));
  cudaFuncSetAttribute(k_edge_bwd_fm<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(FM_SM_TOTAL + 1024));
  cudaFuncSetAttribute(k_edge_bwd64<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_edge_bwd64<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_edge_bwd64<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_edge_bwd64<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  done = true;
}

int edge_tc_units(int grid) { return NGRP * grid; }
int edge_tc_units_fwd(int grid) { return FWD_NGRP * grid; }

void launch_edge_geom(const EdgeArgs &a, float4 *geo, float2 *env, int32_t *unit_rows,
                      int nunits, int32_t *unit_rows_fwd, int nunits_fwd, const EmbedJob &ej,
                      cudaStream_t s) {
  launch_pdl(PDL_GEOM, k_edge_geom, 1184, 256, 0, s, a.pos, a.ptr, a.nbr, a.own, a.nrows, a.cap_e,
             a.cutoff, geo, env, unit_rows, nunits, unit_rows_fwd, nunits_fwd, ej);
}

void launch_edge_fwd_tc(const EdgeArgs &a, const float4 *geo, const float2 *env,
                        const int32_t *unit_rows, const float *P, float *H, int grid,
                        cudaStream_t s, bool scatter) {
  if (fwd_ws_enabled() && fwd64_enabled() && FWD_NGRP == 4) {  // H zeroed by the caller (scatter)
    const uint32_t wsm = (uint32_t)(FWD_SM_META + sizeof(FwdWsShared) + 1024);
    if (scatter)
      launch_pdl(PDL_EDGE_FWD, a.quant ? k_edge_fwd_ws<true, true> : k_edge_fwd_ws<false, true>,
                 grid, WS_THREADS, wsm, s, a, geo, env, unit_rows, P, H);
    else
      launch_pdl(PDL_EDGE_FWD, a.quant ? k_edge_fwd_ws<true, false> : k_edge_fwd_ws<false, false>,
                 grid, WS_THREADS, wsm, s, a, geo, env, unit_rows, P, H);
  } else if (scatter)
    launch_pdl(PDL_EDGE_FWD, a.quant ? k_edge_fwd64<true, true> : k_edge_fwd64<false, true>,
               grid, TC_THREADS, FWD_SM_TOTAL + 1024, s, a, geo, env, unit_rows, P, H);
  else if (fwd64_enabled() && FWD_NGRP == 4)  // the 64-edge kernel uses the 4-unit partition
    launch_pdl(PDL_EDGE_FWD, a.quant ? k_edge_fwd64<true, false> : k_edge_fwd64<false, false>,
               grid, TC_THREADS, FWD_SM_TOTAL + 1024, s, a, geo, env, unit_rows, P, H);
  else
    launch_pdl(PDL_EDGE_FWD, a.quant ? k_edge_fwd_tc<true> : k_edge_fwd_tc<false>, grid,
               FWD_THREADS, FWD_SM_TOTAL + 1024, s, a, geo, env, unit_rows, P, H);
}

void launch_edge_bwd_tc(const EdgeArgs &a, const float4 *geo, const float2 *env,
                        const int32_t *unit_rows, const float *P, const float *GH, float *GP,
                        float4 *gsum, int accumulate, int grid, cudaStream_t s, float4 *gr) {
  if (gr)  // scatter schedule: GP and gr zeroed by the caller
    launch_pdl(PDL_EDGE_BWD, a.quant ? k_edge_bwd64<true, true> : k_edge_bwd64<false, true>,
               grid, TC_THREADS, SM_TOTAL + 1024, s, a, geo, env, unit_rows, P, GH, GP, gsum,
               accumulate, gr);
  else if (bwd_fm_enabled() && bwd_ws_enabled())
    launch_pdl(PDL_EDGE_BWD, a.quant ? k_edge_bwd_fmws<true, 2> : k_edge_bwd_fmws<false, 2>, grid,
               WS_THREADS, (uint32_t)(FM_SM_META + sizeof(BwdWsShared) + 1024), s, a, geo, env,
               unit_rows, P, GH, GP, gsum, accumulate);
  else if (bwd_fm_enabled() && bwd_fm_upg() == 1)
    launch_pdl(PDL_EDGE_BWD, a.quant ? k_edge_bwd_fm<true, 1> : k_edge_bwd_fm<false, 1>, grid,
               TC_THREADS, FM_SM_TOTAL + 1024, s, a, geo, env, unit_rows, P, GH, GP, gsum,
               accumulate);
  else if (bwd_fm_enabled())
    launch_pdl(PDL_EDGE_BWD, a.quant ? k_edge_bwd_fm<true, 2> : k_edge_bwd_fm<false, 2>, grid,
               TC_THREADS, FM_SM_TOTAL + 1024, s, a, geo, env, unit_rows, P, GH, GP, gsum,
               accumulate);
  else if (bwd64_enabled())
    launch_pdl(PDL_EDGE_BWD, a.quant ? k_edge_bwd64<true, false> : k_edge_bwd64<false, false>,
               grid, TC_THREADS, SM_TOTAL + 1024, s, a, geo, env, unit_rows, P, GH, GP, gsum,
               accumulate, (float4 *)nullptr);
  else
    launch_pdl(PDL_EDGE_BWD, a.quant ? k_edge_bwd_tc<true> : k_edge_bwd_tc<false>, grid,
               TC_THREADS, SM_TOTAL + 1024, s, a, geo, env, unit_rows, P, GH, GP, gsum, accumulate);
}

}  // namespace fcg
