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

constexpr int NN = 128;           // node rows per CTA (MMA N)
constexpr int NTH = 512;          // 16 warps
constexpr int NPT = NN / 4;       // nodes per thread
constexpr uint32_t NSM_WA = 0;         // first weight image (hi|lo, <= 64 KB)
constexpr uint32_t NSM_WB = 65536;     // second weight image
constexpr uint32_t NSM_ACT = 131072;   // B operand hi|lo / fp32 scratch (64 KB)
constexpr uint32_t NSM_META = 196608;
constexpr uint32_t IMG128 = 128 * 128 * 2;  // bytes of one 128x128 fp16 image half
constexpr uint32_t IMG64 = 64 * 128 * 2;
constexpr uint32_t NTM_D0 = 0, NTM_D1 = 128;

struct NodeMeta {
  unsigned int amax[4];
  uint64_t bar;   // MMA completion
  uint64_t wbar;  // weight images landed (bulk copy)
  uint32_t tmem;
};
constexpr uint32_t NSM_TOTAL = NSM_META + sizeof(NodeMeta);

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

// Rows [node0, node0+128) of a [nrows][128] fp32 matrix (times a per-channel
// factor) -> MN-major B operand (row = channel).  Forward W16 operands are
// fp16-rounded and unscaled; otherwise split hi/lo with a block-max scale.
// With a CSR row pointer, rows of nodes without edges read as zero: the
// fused edge kernels write segment sums only for non-empty CSR rows (an
// empty segment sums to zero, flash.py:109-135).  Returns the scale exponent.
__device__ __forceinline__ int rows_to_act(const float *src, int node0, int nrows,
                                           const NodeCtx &c, float colscale, bool q16_only,
                                           unsigned int *slot, uint8_t *act,
                                           const int32_t *csr_ptr = nullptr) {
  float v[NPT];
  float mx = 0.f;
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    int n = node0 + c.ec + i;
    const bool in = n < nrows;
    float x = in ? ld_dep(&src[(size_t)n * D + c.ch]) * colscale : 0.f;
    if (csr_ptr && in && ld_dep(&csr_ptr[n + 1]) == ld_dep(&csr_ptr[n])) x = 0.f;
    if (q16_only) x = __half2float(__float2half_rn(x));
    v[i] = x;
    mx = fmaxf(mx, fabsf(x));
  }
  int s = 0;
  if (!q16_only) s = scale_exp(block_amax(mx, slot));
  const float sc = pow2f(s);
#pragma unroll
  for (int g = 0; g < NPT / 8; ++g) put_b8(act, D, c.ch, c.ec + 8 * g, &v[8 * g], sc, !q16_only);
  return s;
}

// TMEM block [ch][32 nodes] -> B operand rows (K = rows of act).  The TMEM
// loads are warp-collective, so every lane runs them; `active` lanes store.
__device__ __forceinline__ void tmem_rows_to_act(uint32_t tcol, uint8_t *act, int K, int row,
                                                 int ec, float scale, bool with_lo,
                                                 bool active = true) {
#pragma unroll
  for (int c0 = 0; c0 < NPT; c0 += 16) {
    float v[16];
    tc::tmem_ld16(tcol + ec + c0, v);
    tc::tmem_ld_wait();
    if (active) {
      put_b8(act, K, row, ec + c0, &v[0], scale, with_lo);
      put_b8(act, K, row, ec + c0 + 8, &v[8], scale, with_lo);
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
      issue_gemm(__VA_ARGS__);          \
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
__global__ void __launch_bounds__(NTH, 1)
k_node_linear_tc(const float *X, const uint16_t *img, int wexp,
                 const float *bias, const float *rowscale, int quant,
                 float *Y, int nrows, unsigned int *amax_out,
                 const int32_t *csr_ptr) {
  extern __shared__ __align__(1024) uint8_t sm[];
  NodeMeta *meta = (NodeMeta *)(sm + NSM_META);
  uint8_t *act = sm + NSM_ACT;
  NodeCtx c = node_prologue(sm, meta, img, 2 * IMG128);
  const int node0 = blockIdx.x * NN;
  const bool fwd = kMode == 0;
  // backward folds the W16 row scale of the K index (output channel) into X
  const float fold = (!fwd && quant) ? ld_dep(&rowscale[c.ch]) : 1.f;
  const int s = rows_to_act(X, node0, nrows, c, fold, fwd && quant, &meta->amax[0], act, csr_ptr);
  NODE_ISSUE(c.tm + NTM_D0, c.sbase + NSM_WA, IMG128, D, !fwd, c.sbase + NSM_ACT, D,
             tc::idesc_f16(128, NN, fwd ? 0 : 1, 1), quant ? (fwd ? 1 : 2) : 3);
  // the accumulated operand (backward) is fetched while the GEMM runs
  float yv[NPT];
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const int n = node0 + c.ec + i;
    yv[i] = (!fwd && n < nrows) ? Y[(size_t)n * D + c.ch] : 0.f;
  }
  NODE_WAIT();
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
        Y[(size_t)n * D + c.ch] = r;
        mx = fmaxf(mx, fabsf(r));
      }
    }
  }
  global_amax(mx, amax_out, &meta->amax[3]);
  node_epilogue_end(meta, c);
}

// post MLP + residual (flash.py:240-241): Zp = H Wp0^T + b0 (kept for the
// backward), U = ssp(Zp) Wp1^T + b1, X += U.
__global__ void __launch_bounds__(NTH, 1)
k_node_post_tc(const float *H, const fcg_block blk, int quant,
               float *Zp, float *X, int nrows,
               const int32_t *csr_ptr) {
  extern __shared__ __align__(1024) uint8_t sm[];
  NodeMeta *meta = (NodeMeta *)(sm + NSM_META);
  uint8_t *act = sm + NSM_ACT;
  NodeCtx c = node_prologue(sm, meta, blk.p0_img, 2 * IMG128, blk.p1_img, 2 * IMG128);
  const int node0 = blockIdx.x * NN;
  const int np = quant ? 1 : 3;
  const uint32_t idesc = tc::idesc_f16(128, NN, 0, 1);
  const int s0 = rows_to_act(H, node0, nrows, c, 1.f, quant, &meta->amax[0], act, csr_ptr);
  NODE_ISSUE(c.tm + NTM_D0, c.sbase + NSM_WA, IMG128, D, false, c.sbase + NSM_ACT, D, idesc, np);
  NODE_WAIT();
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
      if (n < nrows) Zp[(size_t)n * D + c.ch] = z;
      const float a = quant ? __half2float(__float2half_rn(ssp_fast(z))) : ssp_fast(z);
      v[i] = n < nrows ? a : 0.f;
      mx = fmaxf(mx, fabsf(v[i]));
    }
    tc::tmem_st16(c.tl + NTM_D0 + c.ec + c0, v);
  }
  tc::tmem_st_wait();
  int s1 = 0;
  if (!quant) s1 = scale_exp(block_amax(mx, &meta->amax[1]));
  tmem_rows_to_act(c.tl + NTM_D0, act, D, c.ch, c.ec, pow2f(s1), !quant);
  NODE_ISSUE(c.tm + NTM_D1, c.sbase + NSM_WB, IMG128, D, false, c.sbase + NSM_ACT, D, idesc, np);
  // the residual stream is fetched while the GEMM runs
  float xv[NPT];
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const int n = node0 + c.ec + i;
    xv[i] = n < nrows ? X[(size_t)n * D + c.ch] : 0.f;
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
      if (n < nrows) X[(size_t)n * D + c.ch] = xv[c0 + i] + (v[i] * un1 + b1);
    }
  }
  node_epilogue_end(meta, c);
}

// Backward of the post MLP (mlp_backward_input, model.py:321-332; called at
// flash.py:264): GH = ((G Wp1) * ssp'(Zp)) Wp0, on dequantised weights.
__global__ void __launch_bounds__(NTH, 1)
k_node_post_bwd_tc(const float *G, const fcg_block blk, int quant,
                   const float *Zp, float *GH, int nrows,
                   unsigned int *amax_out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  NodeMeta *meta = (NodeMeta *)(sm + NSM_META);
  uint8_t *act = sm + NSM_ACT;
  NodeCtx c = node_prologue(sm, meta, blk.p1_img, 2 * IMG128, blk.p0_img, 2 * IMG128);
  const int node0 = blockIdx.x * NN;
  const int np = quant ? 2 : 3;
  const uint32_t idesc = tc::idesc_f16(128, NN, 1, 1);
  const float f1 = quant ? ld_dep(&blk.p1_s[c.ch]) : 1.f;
  const int sg = rows_to_act(G, node0, nrows, c, f1, false, &meta->amax[0], act);
  NODE_ISSUE(c.tm + NTM_D0, c.sbase + NSM_WA, IMG128, D, true, c.sbase + NSM_ACT, D, idesc, np);
  // ssp'(Zp) operands are fetched while the GEMM runs
  float zv[NPT];
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const int n = node0 + c.ec + i;
    zv[i] = n < nrows ? ld_dep(&Zp[(size_t)n * D + c.ch]) : 0.f;
  }
  NODE_WAIT();
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
  tmem_rows_to_act(c.tl + NTM_D0, act, D, c.ch, c.ec, pow2f(sz), true);
  NODE_ISSUE(c.tm + NTM_D1, c.sbase + NSM_WB, IMG128, D, true, c.sbase + NSM_ACT, D, idesc, np);
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
        GH[(size_t)n * D + c.ch] = v[i] * un1;
        mx = fmaxf(mx, fabsf(v[i] * un1));
      }
    }
  }
  global_amax(mx, amax_out, &meta->amax[3]);
  node_epilogue_end(meta, c);
}

// Readout (flash.py:487-492): per_atom = ssp(X Wr0^T + br0) . wr1 + br1 and
// the ones-seeded backward G = (wr1 * ssp'(zr)) Wr0.  Layer 0 has 64
// outputs: an M=64 GEMM whose row k lives in TMEM lane 32(k/16) + k%16.
__global__ void __launch_bounds__(NTH, 1)
k_readout_tc(const float *X, const fcg_model m, float *per_atom,
             float *G, int nrows) {
  extern __shared__ __align__(1024) uint8_t sm[];
  NodeMeta *meta = (NodeMeta *)(sm + NSM_META);
  uint8_t *act = sm + NSM_ACT;
  float *red = (float *)(sm + NSM_ACT);  // [128 nodes][65] after G1 completes
  NodeCtx c = node_prologue(sm, meta, m.r0_img, 2 * IMG64);
  const bool quant = m.format == FCG_FMT_W16;
  const int node0 = blockIdx.x * NN;
  const int sx = rows_to_act(X, node0, nrows, c, 1.f, quant, &meta->amax[0], act);
  NODE_ISSUE(c.tm + NTM_D0, c.sbase + NSM_WA, IMG64, D, false, c.sbase + NSM_ACT, D,
             tc::idesc_f16(64, NN, 0, 1), quant ? 1 : 3);
  NODE_WAIT();
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
  if (threadIdx.x < NN && node0 + (int)threadIdx.x < nrows) {
    float s = 0.f;
#pragma unroll 8
    for (int q = 0; q < RH; ++q) s += red[threadIdx.x * 65 + q];
    per_atom[node0 + threadIdx.x] = s + m.r1_b;
  }
  __syncthreads();  // red is dead before the B operand overwrites it
  tmem_rows_to_act(c.tl + NTM_D0, act, RH, k, c.ec, pow2f(sz), true, row_lane);
  NODE_ISSUE(c.tm + NTM_D1, c.sbase + NSM_WA, IMG64, D, true, c.sbase + NSM_ACT, RH,
             tc::idesc_f16(128, NN, 1, 1), quant ? 2 : 3);
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
      if (n < nrows) G[(size_t)n * D + c.ch] = v[i] * un1;
    }
  }
  node_epilogue_end(meta, c);
}

// ---------------------------------------------------------------------------
void node_tc_configure() {
  static bool done = false;
  if (done) return;
  const int sm = (int)NSM_TOTAL + 1024;
  cudaFuncSetAttribute(k_node_linear_tc<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k_node_linear_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k_node_post_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k_node_post_bwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k_readout_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  done = true;
}

static inline int node_grid(int nrows) { return (nrows + NN - 1) / NN; }

void launch_node_pre_tc(const float *X, const fcg_block &b, int quant, float *P, int nrows,
                        unsigned int *amax_p, cudaStream_t s) {
  launch_pdl(PDL_NODE_PRE, k_node_linear_tc<0>, node_grid(nrows), NTH, NSM_TOTAL + 1024, s,
      X, b.pre_img, b.pre_exp, b.pre_b, b.pre_s, quant, P, nrows, amax_p, nullptr);
}
void launch_node_pre_bwd_tc(const float *GP, const fcg_block &b, int quant, float *G, int nrows,
                            const int32_t *csr_ptr, cudaStream_t s) {
  launch_pdl(PDL_NODE_PRE_BWD, k_node_linear_tc<1>, node_grid(nrows), NTH, NSM_TOTAL + 1024, s,
      GP, b.pre_img, b.pre_exp, nullptr, b.pre_s, quant, G, nrows, nullptr, csr_ptr);
}
void launch_node_post_tc(const float *H, const fcg_block &b, int quant, float *Zp, float *X,
                         int nrows, const int32_t *csr_ptr, cudaStream_t s) {
  launch_pdl(PDL_NODE_POST, k_node_post_tc, node_grid(nrows), NTH, NSM_TOTAL + 1024, s, H, b, quant, Zp, X,
             nrows, csr_ptr);
}
void launch_node_post_bwd_tc(const float *G, const fcg_block &b, int quant, const float *Zp,
                             float *GH, int nrows, unsigned int *amax_gh, cudaStream_t s) {
  launch_pdl(PDL_NODE_POST_BWD, k_node_post_bwd_tc, node_grid(nrows), NTH, NSM_TOTAL + 1024, s, G, b, quant, Zp, GH,
             nrows, amax_gh);
}
void launch_readout_tc(const float *X, const fcg_model &m, float *per_atom, float *G, int nrows,
                       cudaStream_t s) {
  launch_pdl(PDL_READOUT, k_readout_tc, node_grid(nrows), NTH, NSM_TOTAL + 1024, s, X, m, per_atom, G, nrows);
}

}  // namespace fcg
