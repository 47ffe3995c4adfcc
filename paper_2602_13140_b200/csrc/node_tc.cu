// Atom-wise MLPs on the tensor cores: pre-linear, post MLP + residual,
// readout with its ones-seeded backward, and the two node-side backward
// GEMMs (model.py:297-332 as used by flash.py:207, :240-241, :264, :300,
// :487-492).
//
// Same transposed formulation as the edge kernels: D[out][node] = W x^T with
// the weight image as the A operand (K-major forward, MN-major = W^T
// backward, same bytes) and 128 node rows per CTA as the MN-major B operand
// (row = input channel).  Thread (warp w, lane l) owns channel 32(w%4)+l for
// nodes [32(w/4), +32), so every global load/store is a coalesced 128-byte
// row segment.  fp32 parity uses the fp16 hi/lo split of edge_tc.cu; W16
// weights run hi-only in the forward (inputs rounded to fp16 like
// quantize.py:68-71) and fold the dequant scale into the operand backward.
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

struct NodeMeta {
  unsigned int amax[4];
  uint64_t bar;   // MMA completion
  uint64_t wbar;  // weight images landed (bulk copy)
  uint32_t tmem;
};

// Tile shape and shared-memory layout of a node kernel: kNN node rows per
// CTA (MMA N) with 128 channels x kNN/NPT node parts = 4 kNN threads, kNW
// staged weight images (64 KB slots), then the B operand (K=128 x kNN,
// hi|lo).  The one-image kernels run 64-node CTAs so two fit per SM (smem
// ~99 KB, 256 threads x 128 registers): one CTA's row loads then overlap
// the other's GEMM and epilogue.  The two-image post kernels need 160 KB
// even at 64 nodes and keep 128-node CTAs.
#ifndef FCG_NN_ONE
#define FCG_NN_ONE 64
#endif
template <int kNN, int kNW>
struct NodeCfg {
  static constexpr int NN = kNN;
  static constexpr int NTH = 4 * kNN;
  static constexpr int MIN_CTAS = 512 / NTH;
  static constexpr uint32_t KSTR = (uint32_t)(kNN / 8) * 128u;  // B bytes per 8 K-rows
  static constexpr uint32_t WA = NSM_WA, WB = NSM_WB;
  static constexpr uint32_t ACT = (uint32_t)kNW * 65536u;
  static constexpr uint32_t ACT_BYTES = 2u * 128u * (uint32_t)kNN * 2u;
  static constexpr uint32_t META = ACT + ACT_BYTES;
  static constexpr uint32_t SMEM = META + (uint32_t)sizeof(NodeMeta) + 1024u;
  static_assert(RH * 65 * 4 <= ACT_BYTES * 2, "readout scratch fits the B operand area");
};
using CfgLin = NodeCfg<FCG_NN_ONE, 1>;
using CfgRo = NodeCfg<FCG_NN_ONE, 1>;
using CfgPost = NodeCfg<128, 2>;

// Diagnostic phase stamps (tools/diag_node_phase.py, -DFCG_NODE_STAMPS): with
// fcg_debug_phase_buffer set, thread 0 of every CTA records clock64() at
// phase `ph` of launch kind `kind` (the last launch of a kind wins) and
// %globaltimer at entry (slot 6) and exit (slot 7).
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
static void node_dbg_sync() {
  static unsigned long long *cur = nullptr;
  if (g_dbg_phase != cur) {
    cur = g_dbg_phase;
    cudaMemcpyToSymbol(d_node_dbg, &cur, sizeof(cur));
  }
}

struct NodeCtx {
  int warp, lane, quarter, part, ch, ec;
  uint32_t tm, tl, sbase;
  uint32_t phase;
};

// Weight images are staged by the TMA engine (cp.async.bulk) while the
// threads load their activation rows; the issuing thread waits on wbar
// before the first MMA.
__device__ __forceinline__ NodeCtx node_prologue(uint8_t *sm, NodeMeta *meta,
                                                 const uint16_t *img_a, uint32_t bytes_a,
                                                 const uint16_t *img_b = nullptr,
                                                 uint32_t bytes_b = 0) {
  pdl_trigger();
  NodeCtx c;
  c.warp = threadIdx.x >> 5;
  c.lane = threadIdx.x & 31;
  c.quarter = c.warp & 3;
  c.part = c.warp >> 2;
  c.ch = 32 * c.quarter + c.lane;
  c.ec = NPT * c.part;
  if (threadIdx.x == 0) {
    tc::mbar_init(&meta->bar, 1);
    tc::mbar_init(&meta->wbar, 1);
    tc::fence_mbar_init();
    tc::mbar_expect_tx(&meta->wbar, bytes_a + bytes_b);
    tc::bulk_g2s(sm + NSM_WA, img_a, bytes_a, &meta->wbar);
    if (img_b) tc::bulk_g2s(sm + NSM_WB, img_b, bytes_b, &meta->wbar);
  }
  if (threadIdx.x < 4) meta->amax[threadIdx.x] = 0u;
  if (threadIdx.x < 32) tc::tmem_alloc<256>(&meta->tmem);
  // PDL wait right before the block barrier: ptxas moves ld.global.nc
  // above griddepcontrol.wait alone, but not above bar.sync
  // (tools/check_pdl.py); the weight images are in flight meanwhile.
  pdl_wait();
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  c.tm = meta->tmem;
  c.tl = c.tm + ((uint32_t)(32 * c.quarter) << 16);
  c.sbase = tc::smem_u32(sm);
  c.phase = 0;
  return c;
}

// max |v| over the launch into a global slot (float bits of a non-negative
// value as uint: order-independent, so deterministic).  The fused edge
// kernels derive their operand scales from these maxima.
__device__ __forceinline__ void global_amax(float v, unsigned int *slot, unsigned int *cta_slot) {
  if (!slot) return;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMax(cta_slot, __float_as_uint(v));
  __syncthreads();
  if (threadIdx.x == 0 && *cta_slot) atomicMax(slot, *cta_slot);
}

__device__ __forceinline__ void node_epilogue_end(NodeMeta *meta, const NodeCtx &c) {
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<256>(c.tm);
}

// Rows [node0, node0+NN) of a [nrows][128] fp32 matrix (times a per-channel
// factor) -> MN-major B operand (row = channel).  Forward W16 operands are
// fp16-rounded and unscaled; otherwise split hi/lo with a block-max scale.
// With a CSR row pointer, rows of nodes without edges read as zero: the
// fused edge kernels write segment sums only for non-empty CSR rows (an
// empty segment sums to zero, flash.py:109-135).  Returns the scale exponent.
template <uint32_t KSTR>
__device__ __forceinline__ int rows_to_act(const float *src, int node0, int nrows,
                                           const NodeCtx &c, float colscale, bool q16_only,
                                           unsigned int *slot, uint8_t *act,
                                           const int32_t *csr_ptr = nullptr) {
  // empty-row mask of the warp's NPT (= 32) nodes: lane l reads ptr[n0+l],
  // its neighbour's value is ptr[n0+l+1]
  uint32_t empty = 0u;
  if (csr_ptr) {
    const int n0 = node0 + c.ec, nl = n0 + c.lane;
    const int a = ld_dep(&csr_ptr[min(nl, nrows)]);
    const int b31 = ld_dep(&csr_ptr[min(n0 + 32, nrows)]);
    const int up = __shfl_down_sync(0xffffffffu, a, 1);
    empty = __ballot_sync(0xffffffffu, nl < nrows && (c.lane == 31 ? b31 : up) == a);
  }
  static_assert(NPT == 32, "one warp lane per node of the thread's range");
  float v[NPT];
  float mx = 0.f;
  // the thread's rows are consecutive: one base, immediate offsets i * D
  const float *rb = opaque_ptr(src + (size_t)(node0 + c.ec) * D + c.ch);
  if (node0 + c.ec + NPT <= nrows && empty == 0u) {  // warp-uniform: no checks needed
#pragma unroll
    for (int i = 0; i < NPT; ++i) v[i] = ld_dep(rb + i * D) * colscale;
  } else {
#pragma unroll
    for (int i = 0; i < NPT; ++i) {
      const bool in = node0 + c.ec + i < nrows && !((empty >> i) & 1u);
      v[i] = in ? ld_dep(rb + i * D) * colscale : 0.f;
    }
  }
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    if (q16_only) v[i] = __half2float(__float2half_rn(v[i]));
    mx = fmaxf(mx, fabsf(v[i]));
  }
  int s = 0;
  if (!q16_only) s = scale_exp(block_amax(mx, slot));
  const float sc = pow2f(s);
#pragma unroll
  for (int g = 0; g < NPT / 8; ++g)
    put_b8n(act, D, KSTR, c.ch, c.ec + 8 * g, &v[8 * g], sc, !q16_only);
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

#define NODE_ISSUE(...)                 \
  do {                                  \
    tc::fence_async_smem();             \
    tc::fence_before_sync();            \
    __syncthreads();                    \
    if (threadIdx.x == 0) {             \
      tc::mbar_wait(&meta->wbar, 0);    \
      tc::fence_after_sync();           \
      issue_gemm(__VA_ARGS__, Cfg::KSTR);\
      tc::mma_commit(&meta->bar);       \
    }                                   \
  } while (0)

#define NODE_WAIT()                     \
  do {                                  \
    tc::mbar_wait(&meta->bar, c.phase); \
    c.phase ^= 1;                       \
    tc::fence_after_sync();             \
  } while (0)

// ---------------------------------------------------------------------------
// Y = X W^T + b (pre-linear, flash.py:207)                      [mode 0]
// Y += G_in W   (grad_X += grad_P @ W_pre, flash.py:300)        [mode 1]
template <int kMode>
__global__ void __launch_bounds__(CfgLin::NTH, CfgLin::MIN_CTAS)
k_node_linear_tc(const float *X, const uint16_t *img, int wexp,
                 const float *bias, const float *rowscale, int quant,
                 float *Y, int nrows, unsigned int *amax_out,
                 const int32_t *csr_ptr) {
  using Cfg = CfgLin;
  node_stamp(kMode, 6);
  node_stamp(kMode, 0);
  extern __shared__ __align__(1024) uint8_t sm[];
  NodeMeta *meta = (NodeMeta *)(sm + Cfg::META);
  uint8_t *act = sm + Cfg::ACT;
  NodeCtx c = node_prologue(sm, meta, img, 2 * IMG128);
  node_stamp(kMode, 1);
  const int node0 = blockIdx.x * Cfg::NN;
  const size_t r0 = (size_t)(node0 + c.ec) * D + c.ch;  // this thread: rows r0 + i*D
  float *Yr = opaque_ptr(Y + r0);
  const bool fwd = kMode == 0;
  // backward folds the W16 row scale of the K index (output channel) into X
  const float fold = (!fwd && quant) ? ld_dep(&rowscale[c.ch]) : 1.f;
  const int s = rows_to_act<Cfg::KSTR>(X, node0, nrows, c, fold, fwd && quant, &meta->amax[0], act, csr_ptr);
  node_stamp(kMode, 2);
  NODE_ISSUE(c.tm + NTM_D0, c.sbase + Cfg::WA, IMG128, D, !fwd, c.sbase + Cfg::ACT, D,
             tc::idesc_f16(128, Cfg::NN, fwd ? 0 : 1, 1), quant ? (fwd ? 1 : 2) : 3);
  // the accumulated operand (backward) is fetched while the GEMM runs
  float yv[NPT];
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const int n = node0 + c.ec + i;
    yv[i] = (!fwd && n < nrows) ? Yr[i * D] : 0.f;
  }
  NODE_WAIT();
  node_stamp(kMode, 3);
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
      if (n < nrows) {
        float r = v[i] * un + b;
        r = fwd ? r : yv[c0 + i] + r;
        Yr[(c0 + i) * D] = r;
        mx = fmaxf(mx, fabsf(r));
      }
    }
  }
  global_amax(mx, amax_out, &meta->amax[3]);
  node_stamp(kMode, 4);
  node_epilogue_end(meta, c);
  node_stamp(kMode, 7);
}

// post MLP + residual (flash.py:240-241): Zp = H Wp0^T + b0 (kept for the
// backward), U = ssp(Zp) Wp1^T + b1, X += U.
__global__ void __launch_bounds__(CfgPost::NTH, CfgPost::MIN_CTAS)
k_node_post_tc(const float *H, const fcg_block blk, int quant,
               float *Zp, float *X, int nrows,
               const int32_t *csr_ptr) {
  using Cfg = CfgPost;
  node_stamp(2, 6);
  node_stamp(2, 0);
  extern __shared__ __align__(1024) uint8_t sm[];
  NodeMeta *meta = (NodeMeta *)(sm + Cfg::META);
  uint8_t *act = sm + Cfg::ACT;
  NodeCtx c = node_prologue(sm, meta, blk.p0_img, 2 * IMG128, blk.p1_img, 2 * IMG128);
  node_stamp(2, 1);
  const int node0 = blockIdx.x * Cfg::NN;
  const size_t r0 = (size_t)(node0 + c.ec) * D + c.ch;  // this thread: rows r0 + i*D
  float *Zpr = opaque_ptr(Zp + r0), *Xr = opaque_ptr(X + r0);
  const int np = quant ? 1 : 3;
  const uint32_t idesc = tc::idesc_f16(128, Cfg::NN, 0, 1);
  const int s0 = rows_to_act<Cfg::KSTR>(H, node0, nrows, c, 1.f, quant, &meta->amax[0], act, csr_ptr);
  node_stamp(2, 2);
  NODE_ISSUE(c.tm + NTM_D0, c.sbase + Cfg::WA, IMG128, D, false, c.sbase + Cfg::ACT, D, idesc, np);
  NODE_WAIT();
  node_stamp(2, 3);
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
      if (n < nrows) Zpr[(c0 + i) * D] = z;
      const float a = quant ? __half2float(__float2half_rn(ssp_fast(z))) : ssp_fast(z);
      v[i] = n < nrows ? a : 0.f;
      mx = fmaxf(mx, fabsf(v[i]));
    }
    tc::tmem_st16(c.tl + NTM_D0 + c.ec + c0, v);
  }
  tc::tmem_st_wait();
  int s1 = 0;
  if (!quant) s1 = scale_exp(block_amax(mx, &meta->amax[1]));
  tmem_rows_to_act<Cfg::KSTR>(c.tl + NTM_D0, act, D, c.ch, c.ec, pow2f(s1), !quant);
  NODE_ISSUE(c.tm + NTM_D1, c.sbase + Cfg::WB, IMG128, D, false, c.sbase + Cfg::ACT, D, idesc, np);
  node_stamp(2, 4);
  // the residual stream is fetched while the GEMM runs
  float xv[NPT];
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const int n = node0 + c.ec + i;
    xv[i] = n < nrows ? Xr[i * D] : 0.f;
  }
  NODE_WAIT();
  const float un1 = quant ? ld_dep(&blk.p1_s[c.ch]) : pow2f(-(blk.p1_exp + s1));
  const float b1 = ld_dep(&blk.p1_b[c.ch]);
#pragma unroll
  for (int c0 = 0; c0 < NPT; c0 += 16) {
    float v[16];
    tc::tmem_ld16w(c.tl + NTM_D1 + c.ec + c0, v);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      int n = node0 + c.ec + c0 + i;
      if (n < nrows) Xr[(c0 + i) * D] = xv[c0 + i] + (v[i] * un1 + b1);
    }
  }
  node_stamp(2, 5);
  node_epilogue_end(meta, c);
  node_stamp(2, 7);
}

// Backward of the post MLP (mlp_backward_input, model.py:321-332; called at
// flash.py:264): GH = ((G Wp1) * ssp'(Zp)) Wp0, on dequantised weights.
__global__ void __launch_bounds__(CfgPost::NTH, CfgPost::MIN_CTAS)
k_node_post_bwd_tc(const float *G, const fcg_block blk, int quant,
                   const float *Zp, float *GH, int nrows,
                   unsigned int *amax_out) {
  using Cfg = CfgPost;
  node_stamp(3, 6);
  node_stamp(3, 0);
  extern __shared__ __align__(1024) uint8_t sm[];
  NodeMeta *meta = (NodeMeta *)(sm + Cfg::META);
  uint8_t *act = sm + Cfg::ACT;
  NodeCtx c = node_prologue(sm, meta, blk.p1_img, 2 * IMG128, blk.p0_img, 2 * IMG128);
  node_stamp(3, 1);
  const int node0 = blockIdx.x * Cfg::NN;
  const size_t r0 = (size_t)(node0 + c.ec) * D + c.ch;  // this thread: rows r0 + i*D
  const float *Zpr = opaque_ptr(Zp + r0);
  float *GHr = opaque_ptr(GH + r0);
  const int np = quant ? 2 : 3;
  const uint32_t idesc = tc::idesc_f16(128, Cfg::NN, 1, 1);
  const float f1 = quant ? ld_dep(&blk.p1_s[c.ch]) : 1.f;
  const int sg = rows_to_act<Cfg::KSTR>(G, node0, nrows, c, f1, false, &meta->amax[0], act);
  node_stamp(3, 2);
  NODE_ISSUE(c.tm + NTM_D0, c.sbase + Cfg::WA, IMG128, D, true, c.sbase + Cfg::ACT, D, idesc, np);
  // ssp'(Zp) operands are fetched while the GEMM runs
  float zv[NPT];
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const int n = node0 + c.ec + i;
    zv[i] = n < nrows ? ld_dep(Zpr + i * D) : 0.f;
  }
  NODE_WAIT();
  node_stamp(3, 3);
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
      v[i] = n < nrows ? v[i] * un * sigmoid_fast(zv[c0 + i]) * f0 : 0.f;
      mx = fmaxf(mx, fabsf(v[i]));
    }
    tc::tmem_st16(c.tl + NTM_D0 + c.ec + c0, v);
  }
  tc::tmem_st_wait();
  const int sz = scale_exp(block_amax(mx, &meta->amax[1]));
  tmem_rows_to_act<Cfg::KSTR>(c.tl + NTM_D0, act, D, c.ch, c.ec, pow2f(sz), true);
  NODE_ISSUE(c.tm + NTM_D1, c.sbase + Cfg::WB, IMG128, D, true, c.sbase + Cfg::ACT, D, idesc, np);
  NODE_WAIT();
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
      if (n < nrows) {
        GHr[(c0 + i) * D] = v[i] * un1;
        mx = fmaxf(mx, fabsf(v[i] * un1));
      }
    }
  }
  global_amax(mx, amax_out, &meta->amax[3]);
  node_stamp(3, 5);
  node_epilogue_end(meta, c);
  node_stamp(3, 7);
}

// Readout (flash.py:487-492): per_atom = ssp(X Wr0^T + br0) . wr1 + br1 and
// the ones-seeded backward G = (wr1 * ssp'(zr)) Wr0.  Layer 0 has 64
// outputs: an M=64 GEMM whose row k lives in TMEM lane 32(k/16) + k%16.
__global__ void __launch_bounds__(CfgRo::NTH, CfgRo::MIN_CTAS)
k_readout_tc(const float *X, const fcg_model m, float *per_atom,
             float *G, int nrows) {
  using Cfg = CfgRo;
  node_stamp(4, 6);
  node_stamp(4, 0);
  extern __shared__ __align__(1024) uint8_t sm[];
  NodeMeta *meta = (NodeMeta *)(sm + Cfg::META);
  uint8_t *act = sm + Cfg::ACT;
  float *red = (float *)(sm + Cfg::ACT);  // [128 nodes][65] after G1 completes
  NodeCtx c = node_prologue(sm, meta, m.r0_img, 2 * IMG64);
  node_stamp(4, 1);
  const bool quant = m.format == FCG_FMT_W16;
  const int node0 = blockIdx.x * Cfg::NN;
  const size_t r0 = (size_t)(node0 + c.ec) * D + c.ch;  // this thread: rows r0 + i*D
  float *Gr = opaque_ptr(G + r0);
  const int sx = rows_to_act<Cfg::KSTR>(X, node0, nrows, c, 1.f, quant, &meta->amax[0], act);
  node_stamp(4, 2);
  NODE_ISSUE(c.tm + NTM_D0, c.sbase + Cfg::WA, IMG64, D, false, c.sbase + Cfg::ACT, D,
             tc::idesc_f16(64, Cfg::NN, 0, 1), quant ? 1 : 3);
  NODE_WAIT();
  node_stamp(4, 3);
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
        bool ok = node0 + e < nrows;
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
  const int sz = scale_exp(block_amax(mx, &meta->amax[1]));
  if (threadIdx.x < Cfg::NN && node0 + (int)threadIdx.x < nrows) {
    float s = 0.f;
#pragma unroll 8
    for (int q = 0; q < RH; ++q) s += red[threadIdx.x * 65 + q];
    per_atom[node0 + threadIdx.x] = s + m.r1_b;
  }
  __syncthreads();  // red is dead before the B operand overwrites it
  tmem_rows_to_act<Cfg::KSTR>(c.tl + NTM_D0, act, RH, k, c.ec, pow2f(sz), true, row_lane);
  NODE_ISSUE(c.tm + NTM_D1, c.sbase + Cfg::WA, IMG64, D, true, c.sbase + Cfg::ACT, RH,
             tc::idesc_f16(128, Cfg::NN, 1, 1), quant ? 2 : 3);
  NODE_WAIT();
  const float un1 = pow2f(-((quant ? 0 : m.r0_exp) + sz));
#pragma unroll
  for (int c0 = 0; c0 < NPT; c0 += 16) {
    float v[16];
    tc::tmem_ld16(c.tl + NTM_D1 + c.ec + c0, v);
    tc::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      int n = node0 + c.ec + c0 + i;
      if (n < nrows) Gr[(c0 + i) * D] = v[i] * un1;
    }
  }
  node_stamp(4, 5);
  node_epilogue_end(meta, c);
  node_stamp(4, 7);
}

// ---------------------------------------------------------------------------
void node_tc_configure() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(k_node_linear_tc<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, CfgLin::SMEM);
  cudaFuncSetAttribute(k_node_linear_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, CfgLin::SMEM);
  cudaFuncSetAttribute(k_node_post_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, CfgPost::SMEM);
  cudaFuncSetAttribute(k_node_post_bwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, CfgPost::SMEM);
  cudaFuncSetAttribute(k_readout_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, CfgRo::SMEM);
  done = true;
}

template <class Cfg>
static inline int node_grid(int nrows) { return (nrows + Cfg::NN - 1) / Cfg::NN; }

void launch_node_pre_tc(const float *X, const fcg_block &b, int quant, float *P, int nrows,
                        unsigned int *amax_p, cudaStream_t s) {
  node_dbg_sync();
  launch_pdl(PDL_NODE_PRE, k_node_linear_tc<0>, node_grid<CfgLin>(nrows), CfgLin::NTH,
             CfgLin::SMEM, s, X, b.pre_img, b.pre_exp, b.pre_b, b.pre_s, quant, P, nrows, amax_p,
             nullptr);
}
void launch_node_pre_bwd_tc(const float *GP, const fcg_block &b, int quant, float *G, int nrows,
                            const int32_t *csr_ptr, cudaStream_t s) {
  launch_pdl(PDL_NODE_PRE_BWD, k_node_linear_tc<1>, node_grid<CfgLin>(nrows), CfgLin::NTH,
             CfgLin::SMEM, s, GP, b.pre_img, b.pre_exp, nullptr, b.pre_s, quant, G, nrows, nullptr,
             csr_ptr);
}
void launch_node_post_tc(const float *H, const fcg_block &b, int quant, float *Zp, float *X,
                         int nrows, const int32_t *csr_ptr, cudaStream_t s) {
  launch_pdl(PDL_NODE_POST, k_node_post_tc, node_grid<CfgPost>(nrows), CfgPost::NTH,
             CfgPost::SMEM, s, H, b, quant, Zp, X, nrows, csr_ptr);
}
void launch_node_post_bwd_tc(const float *G, const fcg_block &b, int quant, const float *Zp,
                             float *GH, int nrows, unsigned int *amax_gh, cudaStream_t s) {
  launch_pdl(PDL_NODE_POST_BWD, k_node_post_bwd_tc, node_grid<CfgPost>(nrows), CfgPost::NTH,
             CfgPost::SMEM, s, G, b, quant, Zp, GH, nrows, amax_gh);
}
void launch_readout_tc(const float *X, const fcg_model &m, float *per_atom, float *G, int nrows,
                       cudaStream_t s) {
  launch_pdl(PDL_READOUT, k_readout_tc, node_grid<CfgRo>(nrows), CfgRo::NTH, CfgRo::SMEM, s, X,
             m, per_atom, G, nrows);
}

}  // namespace fcg
