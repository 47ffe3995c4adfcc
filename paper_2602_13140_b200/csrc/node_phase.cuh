// Atom-wise MLP stages on the tensor cores: pre-linear, post MLP + residual,
// readout with its ones-seeded backward, and the two node-side backward
// GEMMs (model.py:297-332 as used by flash.py:207, :240-241, :264, :300,
// :487-492), as device functions over one chunk of NN node rows.
//
// The standalone node kernels (node_tc.cu) run one chunk per CTA.  The
// stages take their barrier, shared-memory slots and TMEM base from the
// context, so they can also run inside another kernel over a range of rows
// (several chunks, node_chunk_reset between them): running them in the
// tails of the fused edge kernels, on the CSR rows each CTA's work units
// own, was measured and dropped (0.866 vs 0.814 ms/step at C2 — the tails
// serialise load -> GEMM -> epilogue on one CTA per SM, where separate
// PDL-overlapped launches with two CTAs per SM hide it).
//
// Same transposed formulation as the edge kernels: D[out][node] = W x^T with
// the weight image as the A operand (K-major forward, MN-major = W^T
// backward, same bytes) and NN node rows as the MN-major B operand (row =
// input channel).  Thread (warp w, lane l) owns channel 32(w%4)+l for nodes
// [32(w/4), +32), so every global load/store is a coalesced 128-byte row
// segment.  fp32 parity uses the fp16 hi/lo split of edge_tc.cu; W16
// weights run hi-only in the forward (inputs rounded to fp16 like
// quantize.py:68-71) and fold the dequant scale into the operand backward.
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"
#include "tc.cuh"
#include "tc_ops.cuh"

namespace fcg {

constexpr int NPT = 32;  // nodes per thread (one channel each)
constexpr uint32_t IMG128 = 128 * 128 * 2;  // bytes of one 128x128 fp16 image half
constexpr uint32_t IMG64 = 64 * 128 * 2;
constexpr uint32_t NTM_D0 = 0, NTM_D1 = 128;
constexpr uint32_t NSM_WA = 0, NSM_WB = 65536;  // weight image slots (hi|lo, <= 64 KB each)

// Diagnostic phase stamps (tools/diag_node_phase.py, -DFCG_NODE_STAMPS): with
// fcg_debug_phase_buffer set, thread 0 of every CTA records clock64() at
// phase `ph` of launch kind `kind` (the last launch of a kind wins) and
// %globaltimer at slots 6 and 7.
__device__ unsigned long long *d_node_dbg = nullptr;
__device__ __forceinline__ void node_stamp(int kind, int ph) {
#ifdef FCG_NODE_STAMPS  // diagnostic builds only: reads d_node_dbg before the PDL wait
  unsigned long long *b = d_node_dbg;
  if (b && threadIdx.x == 0) {
    unsigned long long t;
    if (ph >= 6) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    else t = clock64();
    b[4096 + ((size_t)kind * 1024 + blockIdx.x) * 8 + ph] = t;
  }
#endif
}

struct NodeMeta {
  unsigned int amax[4];
  uint64_t bar;   // MMA completion
  uint64_t wbar[2];  // weight slot A / B landed (bulk copy), one barrier per slot
  uint32_t tmem;
};

struct NodeCtx {
  int warp, lane, quarter, part, ch, ec;
  uint32_t tm, tl, sbase;   // TMEM base, this warp's lane quarter, weight slots' smem base
  uint32_t phase;           // MMA barrier phase
  uint32_t wph[2];          // weight-slot barrier phases
  int sync_id, sync_n;      // named barrier of the participating threads
  uint8_t *act;             // B operand (K = 128 x NN, hi | lo)
  NodeMeta *meta;
};

__device__ __forceinline__ void nsync(const NodeCtx &c) {
  asm volatile("bar.sync %0, %1;" ::"r"(c.sync_id), "r"(c.sync_n) : "memory");
}

__device__ __forceinline__ NodeCtx node_ctx(uint8_t *sm_w, uint8_t *act, NodeMeta *meta,
                                            uint32_t tmem, int sync_id, int sync_n) {
  NodeCtx c;
  c.warp = threadIdx.x >> 5;
  c.lane = threadIdx.x & 31;
  c.quarter = c.warp & 3;
  c.part = c.warp >> 2;
  c.ch = 32 * c.quarter + c.lane;
  c.ec = NPT * c.part;
  c.tm = tmem;
  c.tl = tmem + ((uint32_t)(32 * c.quarter) << 16);
  c.sbase = tc::smem_u32(sm_w);
  c.phase = 0;
  c.wph[0] = c.wph[1] = 0;
  c.sync_id = sync_id;
  c.sync_n = sync_n;
  c.act = act;
  c.meta = meta;
  return c;
}

// Max of non-negative values over the participating threads (slot zeroed by
// the caller before the chunk).
__device__ __forceinline__ float node_amax(float v, unsigned int *slot, const NodeCtx &c) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMax(slot, __float_as_uint(v));
  nsync(c);
  return __uint_as_float(*slot);
}

// max |v| over the chunk into a global slot (float bits of a non-negative
// value as uint: order-independent, so deterministic).  The fused edge
// kernels derive their operand scales from these maxima.
__device__ __forceinline__ void node_global_amax(float v, unsigned int *slot, const NodeCtx &c) {
  if (!slot) return;
  unsigned int *cta_slot = &c.meta->amax[3];
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMax(cta_slot, __float_as_uint(v));
  nsync(c);
  if (threadIdx.x == 0 && *cta_slot) atomicMax(slot, *cta_slot);
}

// Zero the chunk-local maxima (between chunks: every thread is past its
// last read of them).
__device__ __forceinline__ void node_chunk_reset(const NodeCtx &c) {
  nsync(c);
  if (threadIdx.x < 4) c.meta->amax[threadIdx.x] = 0u;
  nsync(c);
}

// Rows [node0, node0+NN) of a [*][128] fp32 matrix (times a per-channel
// factor) -> MN-major B operand (row = channel); rows from `rlim` on read as
// zero.  Forward W16 operands are fp16-rounded and unscaled; otherwise split
// hi/lo with a chunk-max scale.  With a CSR row pointer, rows of nodes
// without edges read as zero: the fused edge kernels write segment sums
// only for non-empty CSR rows (an empty segment sums to zero,
// flash.py:109-135).  Returns the scale exponent.
template <uint32_t KSTR>
__device__ __forceinline__ int rows_to_act(const float *src, int node0, int rlim,
                                           const NodeCtx &c, float colscale, bool q16_only,
                                           unsigned int *slot,
                                           const int32_t *csr_ptr = nullptr) {
  // empty-row mask of the warp's NPT (= 32) nodes: lane l reads ptr[n0+l],
  // its neighbour's value is ptr[n0+l+1]
  uint32_t empty = 0u;
  if (csr_ptr) {
    const int n0 = node0 + c.ec, nl = n0 + c.lane;
    const int a = ld_dep(&csr_ptr[min(nl, rlim)]);
    const int b31 = ld_dep(&csr_ptr[min(n0 + 32, rlim)]);
    const int up = __shfl_down_sync(0xffffffffu, a, 1);
    empty = __ballot_sync(0xffffffffu, nl < rlim && (c.lane == 31 ? b31 : up) == a);
  }
  static_assert(NPT == 32, "one warp lane per node of the thread's range");
  float v[NPT];
  float mx = 0.f;
  // the thread's rows are consecutive: one base, immediate offsets i * D
  const float *rb = opaque_ptr(src + (size_t)(node0 + c.ec) * D + c.ch);
  if (node0 + c.ec + NPT <= rlim && empty == 0u) {  // warp-uniform: no checks needed
#pragma unroll
    for (int i = 0; i < NPT; ++i) v[i] = ld_dep(rb + i * D) * colscale;
  } else {
#pragma unroll
    for (int i = 0; i < NPT; ++i) {
      const bool in = node0 + c.ec + i < rlim && !((empty >> i) & 1u);
      v[i] = in ? ld_dep(rb + i * D) * colscale : 0.f;
    }
  }
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    if (q16_only) v[i] = __half2float(__float2half_rn(v[i]));
    mx = fmaxf(mx, fabsf(v[i]));
  }
  int s = 0;
  if (!q16_only) s = scale_exp(node_amax(mx, slot, c));
  const float sc = pow2f(s);
#pragma unroll
  for (int g = 0; g < NPT / 8; ++g)
    put_b8n(c.act, D, KSTR, c.ch, c.ec + 8 * g, &v[8 * g], sc, !q16_only);
  return s;
}

// TMEM block [ch][32 nodes] -> B operand rows (K = rows of act).  The TMEM
// loads are warp-collective, so every lane runs them; `active` lanes store.
template <uint32_t KSTR>
__device__ __forceinline__ void tmem_rows_to_act(uint32_t tcol, uint8_t *act, int K, int row,
                                                 int ec, float scale, bool with_lo,
                                                 bool active = true) {
#pragma unroll
  for (int c0 = 0; c0 < NPT; c0 += 16) {
    float v[16];
    tc::tmem_ld16(tcol + ec + c0, v);
    tc::tmem_ld_wait();
    if (active) {
      put_b8n(act, K, KSTR, row, ec + c0, &v[0], scale, with_lo);
      put_b8n(act, K, KSTR, row, ec + c0 + 8, &v[8], scale, with_lo);
    }
  }
}

// D(tmem) = W(slot) x act: every participating thread's operand writes are
// fenced and synchronised, thread 0 waits for the weight images and issues.
template <uint32_t KSTR>
__device__ __forceinline__ void node_issue(const NodeCtx &c, uint32_t d, uint32_t w_slot,
                                           uint32_t w_lo_off, int in_dim, bool w_mn, int K,
                                           uint32_t idesc, int nprod) {
  tc::fence_async_smem();
  tc::fence_before_sync();
  nsync(c);
  if (threadIdx.x == 0) {
    const int ws = w_slot == NSM_WA ? 0 : 1;  // a GEMM waits for its own slot only
    tc::mbar_wait(&c.meta->wbar[ws], c.wph[ws]);
    tc::fence_after_sync();
    issue_gemm(d, c.sbase + w_slot, w_lo_off, in_dim, w_mn, tc::smem_u32(c.act), K, idesc, nprod,
               KSTR);
    tc::mma_commit(&c.meta->bar);
  }
}
__device__ __forceinline__ void node_wait(NodeCtx &c) {
  tc::mbar_wait(&c.meta->bar, c.phase);
  c.phase ^= 1;
  tc::fence_after_sync();
}

// The readout weights a stage reads (a view of fcg_model).
struct ReadoutW {
  int format;
  const uint16_t *r0_img;
  int r0_exp;
  const float *r0_s, *r0_b, *r1_w;
  float r1_b;
};
__host__ __device__ inline ReadoutW readout_view(const fcg_model &m) {
  return ReadoutW{m.format, m.r0_img, m.r0_exp, m.r0_s, m.r0_b, m.r1_w, m.r1_b};
}

// Stage weight images into the slots (thread 0; one barrier per slot).
__device__ __forceinline__ void node_stage_weights(const NodeCtx &c, const uint16_t *img_a,
                                                   uint32_t bytes_a, const uint16_t *img_b,
                                                   uint32_t bytes_b) {
  if (threadIdx.x == 0) {
    uint8_t *base = (uint8_t *)__cvta_shared_to_generic(c.sbase);
    tc::mbar_expect_tx(&c.meta->wbar[0], bytes_a);
    tc::bulk_g2s(base + NSM_WA, img_a, bytes_a, &c.meta->wbar[0]);
    if (img_b) {
      tc::mbar_expect_tx(&c.meta->wbar[1], bytes_b);
      tc::bulk_g2s(base + NSM_WB, img_b, bytes_b, &c.meta->wbar[1]);
    }
  }
}

// A weight slot reloaded once the GEMM reading it has completed, so that a
// chain of stages in one kernel (the fused node launches of node_tc.cu) has
// its next image in place by the time it needs it.  The copy completes the
// next phase of that slot's barrier, which the slot's next GEMM waits for
// (a GEMM on the other slot does not).  The slot must have been staged by
// the prologue: its phase 0 is that first image.
struct Restage {
  uint32_t slot;
  const uint16_t *img;
  uint32_t bytes;
};
__device__ __forceinline__ void node_restage(NodeCtx &c, const Restage *r) {
  if (!r) return;
  const int ws = r->slot == NSM_WA ? 0 : 1;
  if (threadIdx.x == 0) {  // thread 0 has seen the GEMM's completion barrier
    uint8_t *base = (uint8_t *)__cvta_shared_to_generic(c.sbase);
    tc::mbar_expect_tx(&c.meta->wbar[ws], r->bytes);
    tc::bulk_g2s(base + r->slot, r->img, r->bytes, &c.meta->wbar[ws]);
  }
  c.wph[ws] ^= 1u;
}

// ---------------------------------------------------------------------------
// Y = X W^T + b (pre-linear, flash.py:207)                      [mode 0]
// Y += G_in W   (grad_X += grad_P @ W_pre, flash.py:300)        [mode 1]
// Weights: the pre image in slot A.
template <int kMode, uint32_t KSTR, int NN>
__device__ __forceinline__ void stage_linear(NodeCtx &c, const float *X, int wexp,
                                             const float *bias, const float *rowscale, int quant,
                                             float *Y, int node0, int rlim,
                                             unsigned int *amax_out, const int32_t *csr_ptr,
                                             const Restage *after = nullptr, int stk = -1) {
  const size_t r0 = (size_t)(node0 + c.ec) * D + c.ch;  // this thread: rows r0 + i*D
  float *Yr = opaque_ptr(Y + r0);
  const bool fwd = kMode == 0;
  // backward folds the W16 row scale of the K index (output channel) into X
  const float fold = (!fwd && quant) ? ld_dep(&rowscale[c.ch]) : 1.f;
  const int s = rows_to_act<KSTR>(X, node0, rlim, c, fold, fwd && quant, &c.meta->amax[0],
                                  csr_ptr);
  if (stk >= 0) node_stamp(stk, 1);
  node_issue<KSTR>(c, c.tm + NTM_D0, NSM_WA, IMG128, D, !fwd, D,
                   tc::idesc_f16(128, NN, fwd ? 0 : 1, 1), quant ? (fwd ? 1 : 2) : 3);
  // the accumulated operand (backward) is fetched while the GEMM runs
  float yv[NPT];
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const int n = node0 + c.ec + i;
    yv[i] = (!fwd && n < rlim) ? Yr[i * D] : 0.f;
  }
  node_wait(c);
  node_restage(c, after);
  if (stk >= 0) node_stamp(stk, 2);
  const float un = pow2f(-((quant ? 0 : wexp) + s)) * ((fwd && quant) ? ld_dep(&rowscale[c.ch]) : 1.f);
  const float b = fwd ? ld_dep(&bias[c.ch]) : 0.f;
  float mx = 0.f;
#pragma unroll
  for (int c0 = 0; c0 < NPT; c0 += 16) {
    float v[16];
    tc::tmem_ld16w(c.tl + NTM_D0 + c.ec + c0, v);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      int n = node0 + c.ec + c0 + i;
      if (n < rlim) {
        float r = v[i] * un + b;
        r = fwd ? r : yv[c0 + i] + r;
        Yr[(c0 + i) * D] = r;
        mx = fmaxf(mx, fabsf(r));
      }
    }
  }
  node_global_amax(mx, amax_out, c);
}

// post MLP + residual (flash.py:240-241): Zp = H Wp0^T + b0 (kept for the
// backward), U = ssp(Zp) Wp1^T + b1, X += U.  Weights: p0 in slot A, p1 in B.
template <uint32_t KSTR, int NN>
__device__ __forceinline__ void stage_post(NodeCtx &c, const float *H, const fcg_block &blk,
                                           int quant, float *Zp, float *X, int node0, int rlim,
                                           const int32_t *csr_ptr,
                                           const Restage *after1 = nullptr,
                                           const Restage *after2 = nullptr, int stk = -1) {
  const size_t r0 = (size_t)(node0 + c.ec) * D + c.ch;  // this thread: rows r0 + i*D
  float *Zpr = opaque_ptr(Zp + r0), *Xr = opaque_ptr(X + r0);
  const int np = quant ? 1 : 3;
  const uint32_t idesc = tc::idesc_f16(128, NN, 0, 1);
  const int s0 = rows_to_act<KSTR>(H, node0, rlim, c, 1.f, quant, &c.meta->amax[0], csr_ptr);
  if (stk >= 0) node_stamp(stk, 2);
  node_issue<KSTR>(c, c.tm + NTM_D0, NSM_WA, IMG128, D, false, D, idesc, np);
  node_wait(c);
  node_restage(c, after1);
  if (stk >= 0) node_stamp(stk, 3);
  const float un0 = quant ? ld_dep(&blk.p0_s[c.ch]) : pow2f(-(blk.p0_exp + s0));
  const float b0 = ld_dep(&blk.p0_b[c.ch]);
  float mx = 0.f;
#pragma unroll
  for (int c0 = 0; c0 < NPT; c0 += 16) {
    float v[16];
    tc::tmem_ld16(c.tl + NTM_D0 + c.ec + c0, v);
    tc::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      int n = node0 + c.ec + c0 + i;
      float z = v[i] * un0 + b0;
      if (n < rlim) Zpr[(c0 + i) * D] = z;
      const float a = quant ? __half2float(__float2half_rn(ssp_fast(z))) : ssp_fast(z);
      v[i] = n < rlim ? a : 0.f;
      mx = fmaxf(mx, fabsf(v[i]));
    }
    tc::tmem_st16(c.tl + NTM_D0 + c.ec + c0, v);
  }
  tc::tmem_st_wait();
  int s1 = 0;
  if (!quant) s1 = scale_exp(node_amax(mx, &c.meta->amax[1], c));
  tmem_rows_to_act<KSTR>(c.tl + NTM_D0, c.act, D, c.ch, c.ec, pow2f(s1), !quant);
  if (stk >= 0) node_stamp(stk, 4);
  node_issue<KSTR>(c, c.tm + NTM_D1, NSM_WB, IMG128, D, false, D, idesc, np);
  // the residual stream is fetched while the GEMM runs
  float xv[NPT];
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const int n = node0 + c.ec + i;
    xv[i] = n < rlim ? Xr[i * D] : 0.f;
  }
  node_wait(c);
  node_restage(c, after2);
  if (stk >= 0) node_stamp(stk, 5);
  const float un1 = quant ? ld_dep(&blk.p1_s[c.ch]) : pow2f(-(blk.p1_exp + s1));
  const float b1 = ld_dep(&blk.p1_b[c.ch]);
#pragma unroll
  for (int c0 = 0; c0 < NPT; c0 += 16) {
    float v[16];
    tc::tmem_ld16w(c.tl + NTM_D1 + c.ec + c0, v);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      int n = node0 + c.ec + c0 + i;
      if (n < rlim) Xr[(c0 + i) * D] = xv[c0 + i] + (v[i] * un1 + b1);
    }
  }
}

// Backward of the post MLP (mlp_backward_input, model.py:321-332; called at
// flash.py:264): GH = ((G Wp1) * ssp'(Zp)) Wp0, on dequantised weights.
// Weights: p1 in slot A, p0 in slot B.
template <uint32_t KSTR, int NN>
__device__ __forceinline__ void stage_post_bwd(NodeCtx &c, const float *G, const fcg_block &blk,
                                               int quant, const float *Zp, float *GH, int node0,
                                               int rlim, unsigned int *amax_out) {
  const size_t r0 = (size_t)(node0 + c.ec) * D + c.ch;  // this thread: rows r0 + i*D
  const float *Zpr = opaque_ptr(Zp + r0);
  float *GHr = opaque_ptr(GH + r0);
  const int np = quant ? 2 : 3;
  const uint32_t idesc = tc::idesc_f16(128, NN, 1, 1);
  const float f1 = quant ? ld_dep(&blk.p1_s[c.ch]) : 1.f;
  const int sg = rows_to_act<KSTR>(G, node0, rlim, c, f1, false, &c.meta->amax[0]);
  node_issue<KSTR>(c, c.tm + NTM_D0, NSM_WA, IMG128, D, true, D, idesc, np);
  // ssp'(Zp) operands are fetched while the GEMM runs
  float zv[NPT];
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const int n = node0 + c.ec + i;
    zv[i] = n < rlim ? ld_dep(Zpr + i * D) : 0.f;
  }
  node_wait(c);
  const float un = pow2f(-((quant ? 0 : blk.p1_exp) + sg));
  const float f0 = quant ? ld_dep(&blk.p0_s[c.ch]) : 1.f;
  float mx = 0.f;
#pragma unroll
  for (int c0 = 0; c0 < NPT; c0 += 16) {
    float v[16];
    tc::tmem_ld16w(c.tl + NTM_D0 + c.ec + c0, v);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      int n = node0 + c.ec + c0 + i;
      v[i] = n < rlim ? v[i] * un * sigmoid_fast(zv[c0 + i]) * f0 : 0.f;
      mx = fmaxf(mx, fabsf(v[i]));
    }
    tc::tmem_st16(c.tl + NTM_D0 + c.ec + c0, v);
  }
  tc::tmem_st_wait();
  const int sz = scale_exp(node_amax(mx, &c.meta->amax[1], c));
  tmem_rows_to_act<KSTR>(c.tl + NTM_D0, c.act, D, c.ch, c.ec, pow2f(sz), true);
  node_issue<KSTR>(c, c.tm + NTM_D1, NSM_WB, IMG128, D, true, D, idesc, np);
  node_wait(c);
  const float un1 = pow2f(-((quant ? 0 : blk.p0_exp) + sz));
  mx = 0.f;
#pragma unroll
  for (int c0 = 0; c0 < NPT; c0 += 16) {
    float v[16];
    tc::tmem_ld16(c.tl + NTM_D1 + c.ec + c0, v);
    tc::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      int n = node0 + c.ec + c0 + i;
      if (n < rlim) {
        GHr[(c0 + i) * D] = v[i] * un1;
        mx = fmaxf(mx, fabsf(v[i] * un1));
      }
    }
  }
  node_global_amax(mx, amax_out, c);
}

// Readout (flash.py:487-492): per_atom = ssp(X Wr0^T + br0) . wr1 + br1 and
// the ones-seeded backward G = (wr1 * ssp'(zr)) Wr0.  Layer 0 has 64
// outputs: an M=64 GEMM whose row k lives in TMEM lane 32(k/16) + k%16.
// Weights: r0 in slot A.  Scratch [NN][65] floats in the act area.
template <uint32_t KSTR, int NN>
__device__ __forceinline__ void stage_readout(NodeCtx &c, const float *X, const ReadoutW &m,
                                              float *per_atom, float *G, int node0, int rlim,
                                              const Restage *after = nullptr) {
  float *red = (float *)c.act;  // [NN nodes][65] after G1 completes
  const bool quant = m.format == FCG_FMT_W16;
  const size_t r0 = (size_t)(node0 + c.ec) * D + c.ch;  // this thread: rows r0 + i*D
  float *Gr = opaque_ptr(G + r0);
  const int sx = rows_to_act<KSTR>(X, node0, rlim, c, 1.f, quant, &c.meta->amax[0]);
  node_issue<KSTR>(c, c.tm + NTM_D0, NSM_WA, IMG64, D, false, D, tc::idesc_f16(64, NN, 0, 1),
                   quant ? 1 : 3);
  node_wait(c);
  const int k = 16 * c.quarter + (c.lane & 15);
  const bool row_lane = c.lane < 16;
  const float un = quant ? ld_dep(&m.r0_s[k]) : pow2f(-(m.r0_exp + sx));
  const float b0 = ld_dep(&m.r0_b[k]);
  const float w1 = ld_dep(&m.r1_w[k]);
  const float fold = quant ? ld_dep(&m.r0_s[k]) : 1.f;
  float mx = 0.f;
#pragma unroll
  for (int c0 = 0; c0 < NPT; c0 += 16) {
    float v[16];
    tc::tmem_ld16(c.tl + NTM_D0 + c.ec + c0, v);
    tc::tmem_ld_wait();
    if (row_lane) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        int e = c.ec + c0 + i;
        bool ok = node0 + e < rlim;
        float z = v[i] * un + b0;
        const float a = quant ? __half2float(__float2half_rn(ssp_fast(z))) : ssp_fast(z);
        red[e * 65 + k] = ok ? a * w1 : 0.f;
        v[i] = ok ? w1 * sigmoid_fast(z) * fold : 0.f;
        mx = fmaxf(mx, fabsf(v[i]));
      }
    }
    tc::tmem_st16(c.tl + NTM_D0 + c.ec + c0, v);
  }
  tc::tmem_st_wait();
  const int sz = scale_exp(node_amax(mx, &c.meta->amax[1], c));
  const int t = threadIdx.x;
  if (t < NN && node0 + t < rlim) {
    float s = 0.f;
#pragma unroll 8
    for (int q = 0; q < RH; ++q) s += red[t * 65 + q];
    per_atom[node0 + t] = s + m.r1_b;
  }
  nsync(c);  // red is dead before the B operand overwrites it
  tmem_rows_to_act<KSTR>(c.tl + NTM_D0, c.act, RH, k, c.ec, pow2f(sz), true, row_lane);
  node_issue<KSTR>(c, c.tm + NTM_D1, NSM_WA, IMG64, D, true, RH, tc::idesc_f16(128, NN, 1, 1),
                   quant ? 2 : 3);
  node_wait(c);
  node_restage(c, after);
  const float un1 = pow2f(-((quant ? 0 : m.r0_exp) + sz));
#pragma unroll
  for (int c0 = 0; c0 < NPT; c0 += 16) {
    float v[16];
    tc::tmem_ld16(c.tl + NTM_D1 + c.ec + c0, v);
    tc::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      int n = node0 + c.ec + c0 + i;
      if (n < rlim) Gr[(c0 + i) * D] = v[i] * un1;
    }
  }
}

}  // namespace fcg
