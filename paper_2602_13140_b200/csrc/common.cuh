// Shared internals of libfcg.so (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/fcg.h"

namespace fcg {

constexpr int D = FCG_D;
constexpr int DR = FCG_DR;
constexpr int RH = FCG_RH;
constexpr float FORCE_BLOWUP_LIMIT = 1.0e6f;  // md.py:30
constexpr float TINY_DISTANCE = 1e-12f;       // reference.py:36 (compared in fp32)

void set_error(const std::string &msg);
int cuda_status(const char *where);  // FCG_OK or FCG_ERR_CUDA (sets message)

inline int ceil_div(long long a, long long b) { return int((a + b - 1) / b); }

// ---- programmatic dependent launch (PDL) ------------------------------------
// The step's kernels are a serial chain.  Launched with PDL, a kernel's CTAs
// may start while its predecessor drains: each kernel lets its dependents
// launch at entry (pdl_trigger) and runs only its static prologue — TMEM
// allocation, weight staging from the immutable model images — before
// pdl_wait, which returns once the predecessor grid has completed and its
// writes are visible.  Every CTA of a PDL-launched kernel passes pdl_wait
// before touching step data and before exiting, so completion stays
// transitive along the chain.  Both are no-ops without the launch attribute.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Loads in PDL-launched kernels are coherent (ld.global), never
// ld.global.nc: ptxas treats .nc data as read-only for the kernel's whole
// lifetime and hoists such loads above griddepcontrol.wait and even bar.sync,
// i.e. before the predecessor's writes are visible.  So those kernels use
// ld_dep instead of __ldg and no const __restrict__ pointers (checked on the
// SASS by tools/check_pdl.py, run by tests/test_host.py).
template <class T>
__device__ __forceinline__ T ld_dep(const T *p) {
  return __ldca(p);  // ld.global.ca: coherent, L1-cached
}
// Gathers whose ADDRESS derives from data loaded after the wait (CSR
// metadata staged in shared memory) cannot be hoisted above it, so they keep
// the read-only path.
template <class T>
__device__ __forceinline__ T ld_gather(const T *p) {
  return __ldg(p);
}
// A per-thread base pointer the compiler cannot re-associate with the
// offsets added to it: base + (uint32_t)off then compiles to a single
// IMAD.WIDE.U32 per gather instead of a 64-bit sign-extended add chain.
template <class T>
__device__ __forceinline__ T *opaque_ptr(T *p) {
  T *q;
  asm("mov.b64 %0, %1;" : "=l"(q) : "l"(p));
  return q;
}
enum PdlSite { PDL_GEOM, PDL_EDGE_FWD, PDL_EDGE_BWD, PDL_NODE_PRE, PDL_NODE_PRE_BWD,
               PDL_NODE_POST, PDL_NODE_POST_BWD, PDL_READOUT,
               PDL_SMALL };  // integrator, prior, neighbour, embed and finish kernels
bool pdl_enabled(int site);  // FCG_PDL=<bitmask of sites> in the environment (A/B)
template <typename... KArgs, typename... Args>
inline void launch_pdl(int site, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled(site) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// Workspace carving: bump allocator over a caller buffer, 256-byte aligned.
struct Carver {
  char *base;
  size_t cap, off = 0;
  Carver(void *b, size_t c) : base((char *)b), cap(c) {}
  template <class T>
  T *take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T *p = (T *)(base ? base + off : nullptr);
    off += n * sizeof(T);
    return p;
  }
  bool ok() const { return off <= cap; }
};

// ---- device math shared by the edge and node kernels ----------------------

// shifted softplus max(x,0) + log1p(exp(-|x|)) - ln2, model.py:93-100
__device__ __forceinline__ float ssp(float x) {
  return fmaxf(x, 0.f) + log1pf(__expf(-fabsf(x))) - 0.6931471805599453f;
}
// its derivative 0.5*(1+tanh(x/2)), model.py:103-107
__device__ __forceinline__ float ssp_grad(float x) {
  return 0.5f * (1.f + tanhf(0.5f * x));
}

// Lower bound over a nondecreasing int32 array: first idx in [0, n] with a[idx] >= v.
__device__ __forceinline__ int lower_bound_i32(const int32_t *a, int n, long long v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if ((long long)ld_dep(&a[mid]) < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Rows [row_begin, row_end) of the flattened CSR owned by CTA `c` of `G`,
// balanced by edge count.  Every row is owned by exactly one CTA, so every
// segment sum has a single writer (no atomics anywhere).
__device__ __forceinline__ void cta_row_range(const int32_t *ptr, int nrows, long long e_total,
                                              int c, int G, int &rb, int &re) {
  long long t0 = e_total * c / G, t1 = e_total * (c + 1) / G;
  rb = (c == 0) ? 0 : lower_bound_i32(ptr, nrows + 1, t0);
  re = (c == G - 1) ? nrows : lower_bound_i32(ptr, nrows + 1, t1);
  if (rb > nrows) rb = nrows;
  if (re > nrows) re = nrows;
}

// Arguments shared by the fused edge kernels (SIMT and tcgen05).
struct EdgeArgs {
  const float *pos;
  const int32_t *ptr, *nbr, *own;
  int nrows;
  int64_t cap_e;
  float cutoff, gamma;
  const float *centers;
  fcg_block blk;
  int quant;
  // device maxima of |P| and |GH| of the current block (written by the node
  // kernels that produce them): the bound of grad_w = GH[dst] * P[src]
  const unsigned int *amax_pg;
  unsigned long long *dbg;  // optional phase timestamps (fcg_debug_phase_buffer)
};
extern unsigned long long *g_dbg_phase;

}  // namespace fcg

// ---- built-in kernel profiler (CUDA events per kernel class) -----------------
namespace fcg {
enum ProfId {
  P_NBR_COUNT, P_NBR_SCAN, P_NBR_FILL, P_NBR_REV, P_EMBED, P_NODE_PRE, P_EDGE_FWD, P_NODE_POST,
  P_READOUT, P_NODE_POST_BWD, P_EDGE_BWD, P_NODE_PRE_BWD, P_FORCES, P_NOISE, P_BAOA, P_PRIOR,
  P_STEP, P_EDGE_GEOM, P_COUNT
};
extern bool g_prof_on;
void prof_mark(int id, bool begin, cudaStream_t s);
struct ProfScope {
  int id;
  cudaStream_t s;
  ProfScope(int i, cudaStream_t st) : id(i), s(st) { if (g_prof_on) prof_mark(id, true, s); }
  ~ProfScope() { if (g_prof_on) prof_mark(id, false, s); }
};
}  // namespace fcg
#define FCG_PROF_CAT2(a, b) a##b
#define FCG_PROF_CAT(a, b) FCG_PROF_CAT2(a, b)
#define FCG_PROF(id, s) ::fcg::ProfScope FCG_PROF_CAT(_prof_, __LINE__)((id), (s))

// ---- launchers implemented across the .cu files -----------------------------
namespace fcg {
struct NbrDefer;
struct GeomJob;
// nbr.cu
size_t nbr_ws_bytes(int R, int N);
int nbr_build(const float *pos, int R, int N, double r_cut, int64_t cap_e, int32_t *ptr,
              int32_t *nbr, int32_t *rev, int32_t *own, int64_t *status, void *ws,
              size_t ws_bytes, cudaStream_t s, const int64_t *gate = nullptr, int stride = 1,
              NbrDefer *defer = nullptr);
int nbr_build_f64(const double *pos, int R, int N, double r_cut, int64_t cap_e, int32_t *ptr,
                  int32_t *nbr, int32_t *rev, int32_t *own, int64_t *status, void *ws,
                  size_t ws_bytes, cudaStream_t s);
size_t group_ws_bytes(int64_t E, int n);
int group_by(const int64_t *key, int64_t E, int n, int64_t *ptr, int64_t *perm, void *ws,
             size_t ws_bytes, cudaStream_t s);
size_t segment_reduce_ws_bytes(int64_t E, int k, int nseg, size_t elem);
int segment_reduce(const float *values, int64_t E, int k, const int64_t *ptr, int nseg,
                   float *out, void *ws, size_t ws_bytes, cudaStream_t s);
int segment_reduce_f64(const double *values, int64_t E, int k, const int64_t *ptr, int nseg,
                       double *out, void *ws, size_t ws_bytes, cudaStream_t s);
// model.cu
size_t ef_ws_bytes(const fcg_model *m, int R, int N, int64_t cap_e);
int energy_forces(const fcg_model *m, const float *pos, const int32_t *types, int R, int N,
                  const int32_t *ptr, const int32_t *nbr, const int32_t *rev,
                  const int32_t *own, int64_t cap_e, float *per_atom, float *energy,
                  float *forces, void *ws, size_t ws_bytes, cudaStream_t s,
                  const float *f_extra, const fcg_md_params *kick, const float *mass,
                  float *vel, int64_t *status, const int64_t *step, int schedule = 0,
                  const fcg_prior *prior = nullptr, float *prior_e = nullptr,
                  const NbrDefer *defer = nullptr);
// md.cu
int normal_noise(uint64_t seed, int rep_offset, const int64_t *step, int R, int N, float *out,
                 cudaStream_t s);
int langevin_baoa(const fcg_md_params *p, const float *mass, int R, int N, const float *forces,
                  const float *noise, float *pos, float *vel, cudaStream_t s);
int half_kick(const fcg_md_params *p, const float *mass, int R, int N, const float *forces,
              float *vel, cudaStream_t s);
int prior_forces(const fcg_prior *pr, const float *pos, int R, int N, float *e_prior,
                 float *f_prior, cudaStream_t s);
int step_advance(int64_t *step, cudaStream_t s);
size_t noise_ring_bytes(int R, int N);
int langevin_leading(const fcg_md_params *p, const float *mass, int R, int N,
                     const float *forces, int64_t *step, float *pos, float *vel, void *ring_ws,
                     int64_t *status, cudaStream_t s);
// node_tc.cu
void node_tc_configure();
void launch_node_pre_tc(const float *X, const fcg_block &b, int quant, float *P, int nrows,
                        unsigned int *amax_p, cudaStream_t s);
void launch_node_pre_bwd_tc(const float *GP, const fcg_block &b, int quant, float *G, int nrows,
                            const int32_t *csr_ptr, cudaStream_t s);
void launch_node_post_tc(const float *H, const fcg_block &b, int quant, float *Zp, float *X,
                         int nrows, const int32_t *csr_ptr, cudaStream_t s);
void launch_node_post_bwd_tc(const float *G, const fcg_block &b, int quant, const float *Zp,
                             float *GH, int nrows, unsigned int *amax_gh, cudaStream_t s);
void launch_readout_tc(const float *X, const fcg_model &m, float *per_atom, float *G, int nrows,
                       cudaStream_t s);
// fused node launches (FCG_NODE_FUSE=0: the separate kernels above)
void launch_node_post_pre_tc(const float *H, const fcg_block &b, const fcg_block &nxt, int quant,
                             float *Zp, float *X, float *Pn, int nrows, const int32_t *csr_ptr,
                             unsigned int *amax_p, cudaStream_t s);
void launch_node_post_readout_tc(const float *H, const fcg_block &b, const fcg_model &m,
                                 int quant, float *Zp, float *X, float *per_atom, float *G,
                                 float *GH, int nrows, const int32_t *csr_ptr,
                                 unsigned int *amax_gh, cudaStream_t s);
void launch_node_prebwd_postbwd_tc(const float *GP, const fcg_block &b, const fcg_block &prv,
                                   int quant, float *G, const float *Zp, float *GH, int nrows,
                                   const int32_t *csr_ptr, unsigned int *amax_gh,
                                   cudaStream_t s);
// edge_tc.cu
void edge_tc_configure();
int edge_tc_units(int grid);      // work units of the backward edge kernel
int edge_tc_units_fwd(int grid);  // work units of the forward edge kernel
// Optional embedding lookup riding on k_edge_geom's launch (X == nullptr: none).
struct EmbedJob {
  const float *emb;
  const int32_t *types;
  int N;
  float *X;
  unsigned int *amax;
  int namax;
  const float *p0_table;  // optional: block 0's pre-linear per type -> P0
  float *P0;
  float p0_amax;
};
void launch_edge_geom(const EdgeArgs &a, float4 *geo, float2 *env, int32_t *unit_rows,
                      int nunits, int32_t *unit_rows_fwd, int nunits_fwd, const EmbedJob &ej,
                      cudaStream_t s);
// k_edge_geom's work (geometry, work-unit row boundaries, embedding) for a
// kernel that writes or owns the CSR rows (geo == nullptr: none).
struct GeomJob {
  const float *pos;
  float cutoff;
  float4 *geo;
  float2 *env;
  int32_t *ur[2];
  int nu[2];
  EmbedJob ej;
};
// The fused neighbour assembly (N <= 512) handed by nbr_build to the force
// evaluation, which launches it together with the edge geometry (fcg_md_step).
struct NbrDefer {
  bool active;
  const uint32_t *masks;
  const int32_t *rep_total;
  int R, N;
  int64_t cap_e;
  int32_t *ptr, *nbr, *rev, *own;
  int64_t *status;
  const int64_t *gate;
  int stride;
};
void launch_nbr_assemble(const NbrDefer &d, const GeomJob &gj, cudaStream_t s);
void launch_edge_fwd_tc(const EdgeArgs &a, const float4 *geo, const float2 *env,
                        const int32_t *unit_rows, const float *P, float *H, int grid,
                        cudaStream_t s, bool scatter = false);
void launch_edge_bwd_tc(const EdgeArgs &a, const float4 *geo, const float2 *env,
                        const int32_t *unit_rows, const float *P, const float *GH, float *GP,
                        float4 *gsum, int accumulate, int grid, cudaStream_t s,
                        float4 *gr = nullptr);
}  // namespace fcg
