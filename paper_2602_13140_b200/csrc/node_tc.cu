// Atom-wise MLP kernels (one chunk of node rows per CTA) over the stages of
// node_phase.cuh: one stage per launch, or consecutive stages fused.
#include "node_phase.cuh"

namespace fcg {

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
static void node_dbg_sync() {
  static unsigned long long *cur = nullptr;
  if (g_dbg_phase != cur) {
    cur = g_dbg_phase;
    cudaMemcpyToSymbol(d_node_dbg, &cur, sizeof(cur));
  }
}

// Prologue of a standalone node kernel: barriers, TMEM, the weight images
// staged by the TMA engine while the threads load their activation rows.
template <class Cfg>
__device__ __forceinline__ NodeCtx node_prologue(uint8_t *sm, const uint16_t *img_a,
                                                 uint32_t bytes_a,
                                                 const uint16_t *img_b = nullptr,
                                                 uint32_t bytes_b = 0) {
  pdl_trigger();
  NodeMeta *meta = (NodeMeta *)(sm + Cfg::META);
  if (threadIdx.x == 0) {
    tc::mbar_init(&meta->bar, 1);
    tc::mbar_init(&meta->wbar[0], 1);
    tc::mbar_init(&meta->wbar[1], 1);
    tc::fence_mbar_init();
  }
  if (threadIdx.x < 4) meta->amax[threadIdx.x] = 0u;
  if (threadIdx.x < 32) tc::tmem_alloc<256>(&meta->tmem);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  NodeCtx c = node_ctx(sm, sm + Cfg::ACT, meta, meta->tmem, 0, Cfg::NTH);
  node_stage_weights(c, img_a, bytes_a, img_b, bytes_b);
  // PDL wait right before the block barrier: ptxas moves ld.global.nc
  // above griddepcontrol.wait alone, but not above bar.sync
  // (tools/check_pdl.py); the weight images are in flight meanwhile.
  pdl_wait();
  __syncthreads();
  return c;
}

__device__ __forceinline__ void node_epilogue_end(const NodeCtx &c) {
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<256>(c.tm);
}

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
  NodeCtx c = node_prologue<Cfg>(sm, img, 2 * IMG128);
  node_stamp(kMode, 1);
  stage_linear<kMode, Cfg::KSTR, Cfg::NN>(c, X, wexp, bias, rowscale, quant, Y,
                                          blockIdx.x * Cfg::NN, nrows, amax_out, csr_ptr);
  node_stamp(kMode, 4);
  node_epilogue_end(c);
  node_stamp(kMode, 7);
}

// post MLP + residual (flash.py:240-241)
__global__ void __launch_bounds__(CfgPost::NTH, CfgPost::MIN_CTAS)
k_node_post_tc(const float *H, const fcg_block blk, int quant,
               float *Zp, float *X, int nrows,
               const int32_t *csr_ptr) {
  using Cfg = CfgPost;
  node_stamp(2, 6);
  node_stamp(2, 0);
  extern __shared__ __align__(1024) uint8_t sm[];
  NodeCtx c = node_prologue<Cfg>(sm, blk.p0_img, 2 * IMG128, blk.p1_img, 2 * IMG128);
  node_stamp(2, 1);
  stage_post<Cfg::KSTR, Cfg::NN>(c, H, blk, quant, Zp, X, blockIdx.x * Cfg::NN, nrows, csr_ptr);
  node_stamp(2, 5);
  node_epilogue_end(c);
  node_stamp(2, 7);
}

// Backward of the post MLP (model.py:321-332; flash.py:264)
__global__ void __launch_bounds__(CfgPost::NTH, CfgPost::MIN_CTAS)
k_node_post_bwd_tc(const float *G, const fcg_block blk, int quant,
                   const float *Zp, float *GH, int nrows,
                   unsigned int *amax_out) {
  using Cfg = CfgPost;
  node_stamp(3, 6);
  node_stamp(3, 0);
  extern __shared__ __align__(1024) uint8_t sm[];
  NodeCtx c = node_prologue<Cfg>(sm, blk.p1_img, 2 * IMG128, blk.p0_img, 2 * IMG128);
  node_stamp(3, 1);
  stage_post_bwd<Cfg::KSTR, Cfg::NN>(c, G, blk, quant, Zp, GH, blockIdx.x * Cfg::NN, nrows,
                                     amax_out);
  node_stamp(3, 5);
  node_epilogue_end(c);
  node_stamp(3, 7);
}

// Readout (flash.py:487-492) and its ones-seeded backward
__global__ void __launch_bounds__(CfgRo::NTH, CfgRo::MIN_CTAS)
k_readout_tc(const float *X, const fcg_model m, float *per_atom,
             float *G, int nrows) {
  using Cfg = CfgRo;
  node_stamp(4, 6);
  node_stamp(4, 0);
  extern __shared__ __align__(1024) uint8_t sm[];
  NodeCtx c = node_prologue<Cfg>(sm, m.r0_img, 2 * IMG64);
  node_stamp(4, 1);
  stage_readout<Cfg::KSTR, Cfg::NN>(c, X, readout_view(m), per_atom, G, blockIdx.x * Cfg::NN,
                                    nrows);
  node_stamp(4, 5);
  node_epilogue_end(c);
  node_stamp(4, 7);
}

// ---- fused node launches ---------------------------------------------------
// Consecutive row-local stages on the same chunk of node rows in one launch
// (each thread reads back only rows it wrote itself, so no barrier is
// needed between the stages beyond the ones inside them).  The weight slot
// a stage no longer reads is reloaded with the next stage's image as soon as
// its GEMM completes (Restage), overlapping the epilogue.

// post(t) + pre(t+1): X(t+1) = X + post MLP, P(t+1) = X(t+1) W_pre^T + b
__global__ void __launch_bounds__(CfgPost::NTH, CfgPost::MIN_CTAS)
k_node_post_pre_tc(const float *H, const fcg_block blk, const fcg_block nxt, int quant,
                   float *Zp, float *X, float *Pn, int nrows, const int32_t *csr_ptr,
                   unsigned int *amax_p) {
  using Cfg = CfgPost;
  extern __shared__ __align__(1024) uint8_t sm[];
  node_stamp(2, 0);
  NodeCtx c = node_prologue<Cfg>(sm, blk.p0_img, 2 * IMG128, blk.p1_img, 2 * IMG128);
  const int node0 = blockIdx.x * Cfg::NN;
  const Restage pre{NSM_WA, nxt.pre_img, 2 * IMG128};
  node_stamp(2, 6);
  node_stamp(2, 1);
  stage_post<Cfg::KSTR, Cfg::NN>(c, H, blk, quant, Zp, X, node0, nrows, csr_ptr, &pre, nullptr, 2);
  node_stamp(2, 7);
  node_chunk_reset(c);
  node_stamp(0, 6);
  node_stamp(0, 0);
  stage_linear<0, Cfg::KSTR, Cfg::NN>(c, X, nxt.pre_exp, nxt.pre_b, nxt.pre_s, quant, Pn, node0,
                                      nrows, amax_p, nullptr, nullptr, 0);
  node_stamp(0, 3);
  node_epilogue_end(c);
  node_stamp(0, 7);
}

// post(T-1) + readout + post_bwd(T-1): the last block's forward tail and
// the head of the backward
__global__ void __launch_bounds__(CfgPost::NTH, CfgPost::MIN_CTAS)
k_node_post_readout_tc(const float *H, const fcg_block blk, const ReadoutW ro, int quant,
                       float *Zp, float *X, float *per_atom, float *G, float *GH, int nrows,
                       const int32_t *csr_ptr, unsigned int *amax_gh) {
  using Cfg = CfgPost;
  extern __shared__ __align__(1024) uint8_t sm[];
  NodeCtx c = node_prologue<Cfg>(sm, blk.p0_img, 2 * IMG128, blk.p1_img, 2 * IMG128);
  const int node0 = blockIdx.x * Cfg::NN;
  const Restage r0{NSM_WA, ro.r0_img, 2 * IMG64}, p0{NSM_WB, blk.p0_img, 2 * IMG128};
  stage_post<Cfg::KSTR, Cfg::NN>(c, H, blk, quant, Zp, X, node0, nrows, csr_ptr, &r0, &p0);
  node_chunk_reset(c);
  const Restage p1{NSM_WA, blk.p1_img, 2 * IMG128};
  stage_readout<Cfg::KSTR, Cfg::NN>(c, X, ro, per_atom, G, node0, nrows, &p1);
  node_chunk_reset(c);
  stage_post_bwd<Cfg::KSTR, Cfg::NN>(c, G, blk, quant, Zp, GH, node0, nrows, amax_gh);
  node_epilogue_end(c);
}

// pre_bwd(t) + post_bwd(t-1): G += GP(t) W_pre(t), GH(t-1) from G
__global__ void __launch_bounds__(CfgPost::NTH, CfgPost::MIN_CTAS)
k_node_prebwd_postbwd_tc(const float *GP, const fcg_block blk, const fcg_block prv, int quant,
                         float *G, const float *Zp, float *GH, int nrows,
                         const int32_t *csr_ptr, unsigned int *amax_gh) {
  using Cfg = CfgPost;
  extern __shared__ __align__(1024) uint8_t sm[];
  NodeCtx c = node_prologue<Cfg>(sm, blk.pre_img, 2 * IMG128, prv.p0_img, 2 * IMG128);
  const int node0 = blockIdx.x * Cfg::NN;
  const Restage p1{NSM_WA, prv.p1_img, 2 * IMG128};
  stage_linear<1, Cfg::KSTR, Cfg::NN>(c, GP, blk.pre_exp, nullptr, blk.pre_s, quant, G, node0,
                                      nrows, nullptr, csr_ptr, &p1);
  node_chunk_reset(c);
  stage_post_bwd<Cfg::KSTR, Cfg::NN>(c, G, prv, quant, Zp, GH, node0, nrows, amax_gh);
  node_epilogue_end(c);
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
  cudaFuncSetAttribute(k_node_post_pre_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       CfgPost::SMEM);
  cudaFuncSetAttribute(k_node_post_readout_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       CfgPost::SMEM);
  cudaFuncSetAttribute(k_node_prebwd_postbwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       CfgPost::SMEM);
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
void launch_node_post_pre_tc(const float *H, const fcg_block &b, const fcg_block &nxt, int quant,
                             float *Zp, float *X, float *Pn, int nrows, const int32_t *csr_ptr,
                             unsigned int *amax_p, cudaStream_t s) {
  node_dbg_sync();
  launch_pdl(PDL_NODE_POST, k_node_post_pre_tc, node_grid<CfgPost>(nrows), CfgPost::NTH,
             CfgPost::SMEM, s, H, b, nxt, quant, Zp, X, Pn, nrows, csr_ptr, amax_p);
}
void launch_node_post_readout_tc(const float *H, const fcg_block &b, const fcg_model &m,
                                 int quant, float *Zp, float *X, float *per_atom, float *G,
                                 float *GH, int nrows, const int32_t *csr_ptr,
                                 unsigned int *amax_gh, cudaStream_t s) {
  launch_pdl(PDL_NODE_POST, k_node_post_readout_tc, node_grid<CfgPost>(nrows), CfgPost::NTH,
             CfgPost::SMEM, s, H, b, readout_view(m), quant, Zp, X, per_atom, G, GH, nrows,
             csr_ptr, amax_gh);
}
void launch_node_prebwd_postbwd_tc(const float *GP, const fcg_block &b, const fcg_block &prv,
                                   int quant, float *G, const float *Zp, float *GH, int nrows,
                                   const int32_t *csr_ptr, unsigned int *amax_gh,
                                   cudaStream_t s) {
  launch_pdl(PDL_NODE_POST_BWD, k_node_prebwd_postbwd_tc, node_grid<CfgPost>(nrows),
             CfgPost::NTH, CfgPost::SMEM, s, GP, b, prv, quant, G, Zp, GH, nrows, csr_ptr,
             amax_gh);
}
void launch_readout_tc(const float *X, const fcg_model &m, float *per_atom, float *G, int nrows,
                       cudaStream_t s) {
  launch_pdl(PDL_READOUT, k_readout_tc, node_grid<CfgRo>(nrows), CfgRo::NTH, CfgRo::SMEM, s, X,
             m, per_atom, G, nrows);
}

}  // namespace fcg
