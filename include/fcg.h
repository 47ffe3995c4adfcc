/*
 * fcg.h — C ABI of the B200-native FlashSchNet MD step (libfcg.so).
 *
 * This is the drop-in boundary for the reference package `flashcg`
 * (/root/reference/pkg/src/flashcg).  Every entry point below replaces one
 * NumPy call site of the reference hot path; the reference symbol it stands
 * in for is cited beside it as file:line.  The Python host layer
 * (paper_2602_13140_b200/) binds these with ctypes and mirrors the
 * reference's Python API on top of them.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers, caller-owned (torch tensors on
 *    the Python side).  The library never allocates device memory; scratch
 *    space is a caller-provided workspace sized by the *_workspace_bytes
 *    queries.
 *  - `stream` is a cudaStream_t passed as void*.  Every call only enqueues
 *    work on that stream and never synchronises the host, so a sequence of
 *    calls can be captured into a CUDA graph.
 *  - Replicas are batched as a block-diagonal graph: bead i of replica r is
 *    global node g = r*N + i.  Neighbour lists are one flattened CSR over
 *    all R*N nodes, edges in canonical (replica, dst, src) order, so a
 *    replica's slice equals the reference's canonical per-replica list
 *    (neighbors.py:47-50) shifted by r*N.
 *  - Return value: FCG_OK or an FCG_ERR_* code; fcg_last_error() gives the
 *    message of the last failure on the calling thread.
 */
#ifndef FCG_H
#define FCG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FCG_ABI_VERSION 1

/* Compiled feature widths.  Smaller model configs are zero-padded to these,
 * which is exact: padded filter/update channels carry ssp(0)=0 and padded
 * weights are 0 (model.py:93-107). */
#define FCG_D 128    /* hidden_dim and filter_hidden_dim, padded   */
#define FCG_DR 64    /* rbf_dim, padded                            */
#define FCG_RH 64    /* readout_hidden_dim, padded                 */
#define FCG_MAX_BLOCKS 8

enum {
  FCG_OK = 0,
  FCG_ERR_CAPACITY = 1, /* edge capacity too small: grow buffers, retry   */
  FCG_ERR_ARG = 2,      /* bad argument / layout mismatch (-> ValueError) */
  FCG_ERR_CUDA = 3      /* CUDA launch or runtime error                   */
};

/* Status words (int64 device array of FCG_STATUS_WORDS).  The host zeroes
 * it once; OVERFLOW, MAXDEG and BLOWUP are sticky so a flag raised at any
 * step of a captured multi-step graph survives until the host reads it. */
#define FCG_STATUS_WORDS 8
enum {
  FCG_ST_EDGES = 0,       /* total edges over all replicas, last build     */
  FCG_ST_OVERFLOW = 1,    /* sticky: an edge total exceeded cap_e          */
  FCG_ST_MAXDEG = 2,      /* sticky max row length                         */
  FCG_ST_BLOWUP = 3,      /* sticky: |F| > 1e6 or non-finite (md.py:183)   */
  FCG_ST_BLOWUP_STEP = 4, /* first step index at which BLOWUP was raised   */
  FCG_ST_EDGE_SUM = 5,    /* running sum of EDGES over builds              */
  FCG_ST_BUILDS = 6,      /* number of neighbour builds                    */
  FCG_ST_ARRIVE = 7       /* internal: arrivals of the MD step's BAOA CTAs
                             (self-resetting; zero between steps)          */
};

/* Weight formats of fcg_model.format. */
enum {
  FCG_FMT_FP32 = 0, /* ModelParams, fp32 (model.py:232-327)                  */
  FCG_FMT_W16 = 1   /* QuantizedParams, fp16 weights + fp32 per-row scale
                       (quantize.py:55-123)                                  */
};

/* One interaction block (model.py:365-370: pre_linear, filter_mlp, post_mlp).
 * Weights are stored twice: `*_w` row-major (out, in) exactly as the
 * reference holds them, `*_wt` transposed (in, out).  All fp32, padded.
 * For FCG_FMT_W16 the fp32 arrays hold the dequantised weights
 * (scale[:,None]*fp32(w16), quantize.py:51) used by the backward pass, and
 * the `*_h` arrays hold the stored fp16 weights with `*_s` the fp32 scales. */
typedef struct {
  const float *pre_w, *pre_wt, *pre_b;    /* [D][D], [D][D], [D]   */
  const float *f0_w, *f0_wt, *f0_b;       /* [D][DR], [DR][D], [D] */
  const float *f1_w, *f1_wt, *f1_b;       /* [D][D], [D][D], [D]   */
  const float *p0_w, *p0_wt, *p0_b;       /* [D][D], [D][D], [D]   */
  const float *p1_w, *p1_wt, *p1_b;       /* [D][D], [D][D], [D]   */
  /* FCG_FMT_W16 only (else NULL): fp16 stored weights (out,in) + scales   */
  const uint16_t *pre_h, *f0_h, *f1_h, *p0_h, *p1_h;
  const float *pre_s, *f0_s, *f1_s, *p0_s, *p1_s;
  /* tcgen05 operand images of the filter MLP for the fused edge kernels:
   * fp16, canonical no-swizzle core-matrix layout of the (out, in) matrix
   * (element (r,c) at ((r/8)*(in/8) + c/8)*64 + (r%8)*8 + c%8), the "hi"
   * image followed by the "lo" image.  FCG_FMT_FP32: hi+lo = W * 2^exp
   * to ~22 bits; FCG_FMT_W16: hi = stored fp16 weights, lo = 0, exp = 0
   * (the per-row scales *_s are applied in the epilogue). */
  const uint16_t *f0_img, *f1_img; /* [2][D][DR], [2][D][D] */
  int f0_exp, f1_exp;
  /* same images for the node MLPs (pre_linear, post0, post1), [2][D][D] */
  const uint16_t *pre_img, *p0_img, *p1_img;
  int pre_exp, p0_exp, p1_exp;
  /* Static power-of-two operand scales of the fused edge kernels, chosen on
   * the host from weight/basis bounds so the kernels need no per-tile max:
   * f_hexp for h = ssp(filter0(b)) (|h| <= max_c sum_k |W0[c][k]| + |b0[c]|
   * since 0 <= b <= 1), f_dbexp for the basis derivative db (|db| <=
   * sqrt(2*gamma/e) + pi/(2*r_cut)); f1_qmax = max W16 row scale of filter
   * layer 1 (1 for fp32), folded into grad_w's bound; f_vexp for
   * v = ssp'(z0) * (W0 db), the operand of the forward-mode backward
   * (|v[c]| <= max_d sum_k |W0[c][k]| |db_k(d)|, evaluated on the host). */
  int f_hexp, f_dbexp;
  float f1_qmax;
  int f_vexp;
} fcg_block;

typedef struct {
  int format;           /* FCG_FMT_*                                        */
  int num_blocks;       /* ModelConfig.num_blocks (<= FCG_MAX_BLOCKS)       */
  int num_types;        /* ModelConfig.num_atom_types                       */
  float cutoff;         /* fp32(ModelConfig.cutoff) (model.py:242-246)      */
  float gamma;          /* fp32(RbfSpec.gamma) (model.py:262-264)           */
  const float *centers; /* [DR] fp32(RbfSpec.centers), zero-padded          */
  const float *embedding; /* [num_types][D]                                 */
  fcg_block blocks[FCG_MAX_BLOCKS];
  const float *r0_w, *r0_wt, *r0_b; /* readout layer 0: [RH][D],[D][RH],[RH] */
  const float *r1_w;                /* readout layer 1 weight row [RH]       */
  float r1_b;                       /* readout layer 1 bias                  */
  const uint16_t *r0_h; const float *r0_s; /* W16 only */
  const uint16_t *r1_h; float r1_s;        /* W16 only */
  const uint16_t *r0_img;                  /* readout layer 0 image, [2][RH][D] */
  int r0_exp;
  /* Optional (NULL: computed every step by the pre-linear kernel): block 0's
   * pre-linear P = X W_pre^T + b of every embedding row, [num_types][D].
   * X of block 0 is embedding[types] (flash.py:201), which does not depend
   * on positions, so P_0 is a per-model table the geometry kernel gathers;
   * pre0_amax = max |table| (an upper bound of max |P_0| for the edge
   * kernels' operand scales). */
  const float *pre0_table;
  float pre0_amax;
} fcg_model;

/* Library identity. */
int fcg_abi_version(void);
const char *fcg_last_error(void);

/* Built-in profiler: with profiling on, every kernel launch of the entry
 * points below is bracketed by CUDA events on its stream (eager use only,
 * not under graph capture).  fcg_profile_read synchronises the device and
 * returns, per kernel class, the summed device time and launch count; names
 * are 32-byte NUL-padded records.  Returns the number of classes written. */
int fcg_profile_enable(int on);
/* Diagnostics: when set (device buffer of >= 2*64*16 uint64), the tcgen05
 * edge kernels record clock64() at phase boundaries of CTA 0 / group 0 for
 * the first 16 tiles ([kernel 0=fwd,1=bwd][tile][phase]); NULL disables. */
int fcg_debug_phase_buffer(void *dev_ptr);
int fcg_profile_read(int max_classes, char *names, double *total_ms,
                     int *launches);

/* ---------------------------------------------------------------------
 * (a) neighbour list + CSR
 * Replaces build_neighbors_cells (neighbors.py:67-110) + _canonical (:47-50)
 * + group_by_destination / group_by_source (neighbors.py:113-132) for all
 * replicas at once.  Edge (j -> i) exists iff fp64 dist2 < r_cut*r_cut with
 * dist2 = (dx*dx + dz*dz) + dy*dy on fp32->fp64 positions (strict <, no self
 * edges).  Outputs:
 *   ptr[R*N+1]  dst-CSR row pointer == reference group_by_destination.ptr
 *               (flattened; per replica subtract ptr[r*N]); ptr_src == ptr.
 *   nbr[cap_e]  global src node of each edge, rows sorted ascending
 *               (== reference NeighborList.src + r*N); the dst perm is the
 *               identity.
 *   rev[cap_e]  id of the reverse edge; equals group_by_source.perm.
 *   own[cap_e]  dst (row) node of each edge (== NeighborList.dst + r*N).
 *   status[]    FCG_ST_* words.
 * ------------------------------------------------------------------- */
size_t fcg_nbr_workspace_bytes(int R, int N);
int fcg_nbr_build(const float *pos, int R, int N, double r_cut, int64_t cap_e,
                  int32_t *ptr, int32_t *nbr, int32_t *rev, int32_t *own,
                  int64_t *status, void *ws, size_t ws_bytes, void *stream);

/* Same as fcg_nbr_build for float64 positions (64-bit mode inputs). */
int fcg_nbr_build_f64(const double *pos, int R, int N, double r_cut,
                      int64_t cap_e, int32_t *ptr, int32_t *nbr, int32_t *rev,
                      int32_t *own, int64_t *status, void *ws, size_t ws_bytes,
                      void *stream);

/* General stable grouping of an arbitrary edge key list (the reference's
 * _group_by, neighbors.py:113-120): ptr[n+1] = exclusive cumsum of
 * bincount(key), perm = argsort(key, kind="stable"). */
size_t fcg_group_workspace_bytes(int64_t E, int n);
int fcg_group_by(const int64_t *key, int64_t E, int n, int64_t *ptr,
                 int64_t *perm, void *ws, size_t ws_bytes, void *stream);

/* (d) CSR segment reduce, flash.py:109-135: out[s] = sum values[ptr[s]:ptr[s+1]]
 * (rows of width k), empty segments -> 0, no atomics, fixed summation order.
 * Segments are cut into chunks of <= 256 rows reduced by separate CTAs and
 * combined in chunk order (the reference's segment_split partials), so the
 * cost does not depend on the degree distribution (bench.py:91-118).
 * Workspace: fcg_segment_reduce_workspace_bytes (valid for both widths). */
size_t fcg_segment_reduce_workspace_bytes(int64_t E, int k, int nseg);
int fcg_segment_reduce(const float *values, int64_t E, int k,
                       const int64_t *ptr, int nseg, float *out, void *ws,
                       size_t ws_bytes, void *stream);

int fcg_segment_reduce_f64(const double *values, int64_t E, int k,
                           const int64_t *ptr, int nseg, double *out, void *ws,
                           size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------
 * (b)(c)(d)(e) energy and forces of the SchNet model, flash.py:446-501.
 * Consumes the CSR of fcg_nbr_build.  Outputs per_atom[R*N] (readout
 * epsilon, flash.py:488), energy[R] (per-replica sum, flash.py:489) and
 * forces[R*N*3] = -dE/dr (flash.py:501).  No prior term.
 * ------------------------------------------------------------------- */
size_t fcg_ef_workspace_bytes(const fcg_model *m, int R, int N, int64_t cap_e);
int fcg_energy_forces(const fcg_model *m, const float *pos,
                      const int32_t *types, int R, int N, const int32_t *ptr,
                      const int32_t *nbr, const int32_t *rev,
                      const int32_t *own, int64_t cap_e, float *per_atom,
                      float *energy, float *forces, void *ws, size_t ws_bytes,
                      void *stream);

/* The same evaluation under an explicit aggregation schedule
 * (PipelineMode(fused=True, segred=...), flash.py:446-501):
 *   FCG_SCHED_SEGRED  the contention-free CSR segment sums (the product
 *                     path, flash.py:192-307; = fcg_energy_forces);
 *   FCG_SCHED_SCATTER the "fused but scatter" ablation (flash.py:373-443):
 *                     the same fused tcgen05 edge kernels, but messages,
 *                     grad_P rows and the position gradient are aggregated
 *                     with atomic adds (np.add.at per tile in the
 *                     reference), so sums are order-dependent at fp32
 *                     round-off. */
enum { FCG_SCHED_SEGRED = 0, FCG_SCHED_SCATTER = 1 };
int fcg_energy_forces_sched(const fcg_model *m, const float *pos,
                            const int32_t *types, int R, int N,
                            const int32_t *ptr, const int32_t *nbr,
                            const int32_t *rev, const int32_t *own,
                            int64_t cap_e, float *per_atom, float *energy,
                            float *forces, void *ws, size_t ws_bytes,
                            int schedule, void *stream);

/* ---------------------------------------------------------------------
 * (f) batched Langevin integrator, md.py:109-208.
 * ------------------------------------------------------------------- */

/* Harmonic bond prior (md.py:109-124) in node-incidence form: for bead i,
 * bonds inc_bond[inc_ptr[i]:inc_ptr[i+1]] with sign inc_sign (+1 when i is
 * the bond's first atom, -1 when second), ordered as np.add.at applies them
 * (all "+", then all "-", each in bond order). */
typedef struct {
  int num_bonds;
  const int32_t *bond_i, *bond_j; /* [M]                        */
  const float *k, *r0;            /* [M] fp32(spring_k), fp32(rest_length) */
  const int32_t *inc_ptr;         /* [N+1]                      */
  const int32_t *inc_bond;        /* [2M]                       */
  const int32_t *inc_sign;        /* [2M]                       */
} fcg_prior;

typedef struct {
  float half_dt;   /* fp32(0.5 * dt_ps)                       (md.py:137,162) */
  float c1;        /* fp32(exp(-friction*dt_ps))              (md.py:165)     */
  float c2_num;    /* fp32((1 - c1*c1) * KB * temperature)    (md.py:166)     */
  uint64_t seed;   /* SimConfig.seed                          (md.py:127-131) */
  int rep_offset;  /* global index of replica 0 of this shard                 */
  int neighbor_stride;
  int schedule;    /* FCG_SCHED_* of the force evaluation in fcg_md_step      */
} fcg_md_params;

/* numpy-exact noise: out[r][k] = float32(Generator(Philox(key=[seed, rep],
 * counter=[0,0,0,step])).standard_normal((N,3)).ravel()[k]) with
 * rep = rep_offset + r and step = *step (device int64), md.py:127-131,167-168. */
int fcg_normal_noise(uint64_t seed, int rep_offset, const int64_t *step,
                     int R, int N, float *out, void *stream);

/* B + A + O + A of langevin_step (md.py:150-172) with the given noise;
 * fp32 semantics as numpy 2 (NEP 50) evaluates them. */
int fcg_langevin_baoa(const fcg_md_params *p, const float *mass, int R,
                      int N, const float *forces,
                      const float *noise, float *pos, float *vel, void *stream);

/* half_kick, md.py:134-138: vel += (half_dt * F) / m. */
int fcg_half_kick(const fcg_md_params *p, const float *mass, int R, int N,
                  const float *forces, float *vel, void *stream);

/* Prior energy + forces for all replicas (md.py:109-124): e_prior[R],
 * f_prior[R*N*3]. */
int fcg_prior_forces(const fcg_prior *pr, const float *pos, int R, int N,
                     float *e_prior, float *f_prior, void *stream);

/* One full MD step for all replicas: noise, BAOA, neighbour rebuild,
 * energy/forces, prior, trailing half-kick, blow-up flag, step += 1
 * (md.py:199-207 with _ReplicaForces, md.py:231-273).  `forces` holds the
 * forces of the current state on entry and of the new state on exit.
 * potential[R] / prior[R] receive the info dict of the new state. */
size_t fcg_md_workspace_bytes(const fcg_model *m, int R, int N, int64_t cap_e);
int fcg_md_step(const fcg_model *m, const fcg_prior *pr,
                const fcg_md_params *p, const float *mass,
                const int32_t *types, int R, int N, double r_cut,
                int64_t cap_e, int64_t *step, float *pos, float *vel,
                float *forces, float *potential, float *prior,
                int32_t *ptr, int32_t *nbr, int32_t *rev, int32_t *own,
                int64_t *status, void *ws, size_t ws_bytes, void *stream);

/* Asynchronous copy of `bytes` between any two of host (pinned) and device
 * memory on `stream` (cudaMemcpyDefault): the host I/O of an MD step in the
 * same stream — and CUDA graph — as fcg_md_step, so a host-buffer step is
 * one graph launch (paper_2602_13140_b200.MDEngine.step_host). */
int fcg_memcpy_async(void *dst, const void *src, size_t bytes, void *stream);

/* ---------------------------------------------------------------------
 * (f) output pipeline, md.py:224-228 / :312-326.  HOST pointers.
 * Formats R trajectory frames (replica indices replica0..replica0+R-1) of
 * float32 positions[R][N][3] exactly as the reference's _format_frame
 * ("%.9f" coordinates) into out[cap]; returns the byte count, or minus the
 * required size when out is NULL or too small.  nthreads <= 0: all cores.
 * ------------------------------------------------------------------- */
int64_t fcg_format_xyz(const float *pos, const int32_t *types, int R, int N,
                       int64_t step, int replica0, char *out, int64_t cap,
                       int nthreads);

/* ---- trajectory analysis (analysis.py) ----------
 * Batched over F frames x[F][N][3] (fp64, device) against one reference
 * structure ref[N][3].  Replaces the per-frame numpy loops of
 * analysis.py:56-143 / :260-276.
 *
 * fcg_kabsch: optimal proper superposition of every frame onto ref
 * (kabsch_align, analysis.py:56-81): rmsd[F]; rot[F][3][3] and trans[F][3]
 * (nullable) with moved = R x + t; degenerate[F] = 1 where the reference
 * raises DegenerateStructureError (fewer than 3 beads or s1 <= 1e-12 s0). */
int fcg_kabsch(const double *x, const double *ref, int F, int N, double *rmsd,
               double *rot, double *trans, int32_t *degenerate, void *stream);
/* fcg_gdt_counts: the GDT-TS seed search of gdt_ts (analysis.py:115-143):
 * windows[W][2] = (start, length) seeds; best[F][4] = the largest number of
 * beads within cutoffs[c] (<=) over all non-degenerate seeds.  GDT-TS of a
 * frame = mean_c(best[c] / N) (done by the caller). */
int fcg_gdt_counts(const double *x, const double *ref, int F, int N,
                   const int32_t *windows, int W, const double *cutoffs,
                   int32_t *best, void *stream);
/* fcg_native_q: fraction of native contacts (fraction_native_contacts,
 * analysis.py:100-108): q[f] = mean_c 1/(1+exp(beta (r_c - lam r0_c))) over
 * pairs[C][2]; C >= 1 (an empty contact set is a ValueError upstream). */
int fcg_native_q(const double *x, int F, int N, const int32_t *pairs,
                 const double *ref_dist, int C, double beta, double lam, double *q,
                 void *stream);

/* ---- quantize_model calibration (quantize.py:126-178)
 * err[r][c] = dw^T gram dw, dw = fp64(fp16(w[r] / cand[r][c])) * cand[r][c]
 * - w[r] (non-finite entries -> 1e30), all fp64 on the device: w[rows][k],
 * cand[rows][ncand], gram[k][k] (k <= 256).  The caller takes the argmin
 * per row (w16.quantize_model(device="cuda"), which re-scores near-ties on
 * the host so the scales stay bit-identical to the reference's). */
int fcg_calib_errors(const double *w, int rows, int k, const double *cand, int ncand,
                     const double *gram, double *err, void *stream);

/* Diagnostics: tcgen05 (kind::f16) GEMM self-test.  dump[128][N] receives
 * the raw TMEM accumulator lanes of D = A * B^T for A[M][K], B[N][K] fp16
 * staged in the canonical no-swizzle core-matrix layout (K-major or
 * MN-major, two core orders, LBO/SBO assignment optionally swapped). */
int fcg_selftest_mma(const uint16_t *A, const uint16_t *B, float *dump, int M,
                     int N, int K, int a_mn, int a_order, int a_swap, int b_mn,
                     int b_order, int b_swap, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FCG_H */
