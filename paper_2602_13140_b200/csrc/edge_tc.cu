// (b)(c)(d) Fused edge passes on the 5th-generation tensor cores.
//
// Same contract as the fused edge loop of the reference (flash.py:215-236
// forward, :272-295 backward) — edge tensors never reach HBM — but the four
// per-edge filter-MLP GEMMs run as tcgen05.mma (kind::f16, fp32 accumulate
// in TMEM).
//
// Formulation ("transposed"): D[channel][edge] = W[channel][k] * X[k][edge].
//   A = weights, resident in SMEM for the whole kernel (K-major in the
//       forward; the SAME bytes read MN-major give W^T for the backward);
//   B = per-tile edge activations written by the epilogue threads
//       (MN-major: row = channel, contiguous edges);
//   D = TMEM, lane = channel, column = edge.
//
// Work decomposition: a CTA (one per SM, 16 warps) hosts two independent
// groups of 8 warps.  Both groups read the same resident weights but own a
// separate range of CSR rows, 64-edge tiles, B-operand buffer, TMEM columns,
// mbarrier and named barrier, so one group's MMA and gather latency hides
// under the other group's epilogue.  Inside a group every thread owns one
// channel across 32 consecutive edges of the tile (2 threads per channel),
// so the destination (forward) / source (backward) segment reduction is a
// running sum per thread plus an ordered 2-way merge, with a single store
// per CSR row — no atomics.
//
// fp32 parity (SURVEY §7 hard part 2): plain fp16/TF32 operands lose ~1e-3;
// we split both operands as x*2^s = hi + lo (fp16 each, ~22 significant
// bits) and accumulate hi*hi + hi*lo + lo*hi.  Weights carry a host-chosen
// power-of-two prescale; activations get a per-tile power-of-two scale from
// a group max, removed exactly in the epilogue.  W16 weights (quantize.py)
// use the stored fp16 weights directly: one MMA in the forward (inputs
// rounded to fp16 as the reference does), two in the backward.
#include <cuda_fp16.h>

#include "common.cuh"
#include "tc.cuh"
#include "tc_ops.cuh"

namespace fcg {

constexpr int TT = 64;           // edges per tile (MMA N)
constexpr int NGRP = 2;          // independent warp groups per CTA
constexpr int GT = 256;          // threads per group (8 warps, 2 per lane quarter)
constexpr int TC_THREADS = NGRP * GT;
constexpr int NPART = 2;         // edge parts per channel within a group
constexpr int EPT = TT / NPART;  // edges per thread (32)
constexpr uint32_t KSTR = (TT / 8) * 128;  // B operand bytes per 8 K-rows
constexpr uint32_t SM_W0 = 0;          // W0 hi|lo: 2 x 128x64 fp16
constexpr uint32_t SM_W1 = 32768;      // W1 hi|lo: 2 x 128x128 fp16
constexpr uint32_t SM_BUF = 98304;     // per group: basis buffer (K=64) + act buffer (K=128)
constexpr uint32_t BB_BYTES = 2 * 64 * TT * 2;   // basis hi|lo: 16 KB
constexpr uint32_t HB_BYTES = 2 * 128 * TT * 2;  // h / grad_w / gz hi|lo, or fp32 scratch: 32 KB
constexpr uint32_t GBUF_BYTES = BB_BYTES + HB_BYTES;
constexpr uint32_t SM_META = SM_BUF + NGRP * GBUF_BYTES;
constexpr uint32_t W0_BYTES = 128 * 64 * 2, W1_BYTES = 128 * 128 * 2;
constexpr int RED_LD = 65;       // padded stride of the [edge][k] fp32 scratch

struct TcMeta {  // per tile (double-buffered per group)
  int own[TT], nbr[TT];
  float d[TT], env[TT], denv[TT];
  float4 u[TT];
  unsigned int amax[4];
  float xch[NPART - 1][3][128];  // part 1 -> part 0 segment boundary partials
};
struct TcShared {
  TcMeta meta[NGRP][2];
  uint64_t bar[NGRP][2];  // [0]: GEMM1 commits, [1]: other GEMM commits
  uint32_t tmem;
};
constexpr uint32_t SM_TOTAL = SM_META + sizeof(TcShared);

// ---- CSR segment sums across the edge parts of a tile -------------------------
// Each (channel, part) thread feeds its 32 edges in order: runs that start
// and end inside the part are complete and written directly (one store per
// row, empty rows between them zeroed); the first and last run of the part
// go to an ordered merge done by the part-0 thread.
struct Runs {
  int row, nruns;
  float acc, head;
  __device__ __forceinline__ void init() { row = -1; nruns = 0; acc = 0.f; head = 0.f; }
  __device__ __forceinline__ void begin(int o, int c, float *__restrict__ out) {
    if (row >= 0) {
      if (nruns == 0) head = acc; else out[(size_t)row * D + c] = acc;
#pragma unroll 1
      for (int z = row + 1; z < o; ++z) out[(size_t)z * D + c] = 0.f;
      ++nruns;
    }
    row = o;
    acc = 0.f;
  }
  // 16 consecutive edges e0.. with values m (first `cnt` valid).  Rows are
  // warp-uniform; a chunk with one row or one row change avoids per-edge
  // branches.
  __device__ __forceinline__ void chunk(const int *own, int e0, int cnt, const float (&m)[16], int c,
                                        float *__restrict__ out) {
    if (cnt == 16) {
      const int o0 = own[e0], o15 = own[e0 + 15];
      if (o0 == o15) {
        if (o0 != row) begin(o0, c, out);
        float s[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] = m[i] + m[i + 8];
#pragma unroll
        for (int i = 0; i < 4; ++i) s[i] += s[i + 4];
        acc += (s[0] + s[2]) + (s[1] + s[3]);
        return;
      }
      // first index whose row equals the chunk's last row
      int b = 15;
      while (b > 0 && own[e0 + b - 1] == o15) --b;
      bool single_change = true;
#pragma unroll 1
      for (int i = 1; i < b; ++i) single_change &= own[e0 + i] == o0;
      if (single_change) {
        float lo = 0.f, hi = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (i < b) lo += m[i]; else hi += m[i];
        }
        if (o0 != row) begin(o0, c, out);
        acc += lo;
        begin(o15, c, out);
        acc += hi;
        return;
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < cnt) {
        int o = own[e0 + i];
        if (o != row) begin(o, c, out);
        acc += m[i];
      }
    }
  }
  __device__ __forceinline__ void close() {
    if (row >= 0) {
      if (nruns == 0) head = acc;
      ++nruns;
    }
  }
};

// Ordered merge of one part's boundary runs into the open carry segment.
__device__ __forceinline__ void merge_part(int &crow, float &cacc, int nruns, float head,
                                           float tail, int head_row, int tail_row, int c,
                                           float *__restrict__ out) {
  if (nruns == 0) return;
  if (head_row == crow) {
    cacc += head;
  } else {
    out[(size_t)crow * D + c] = cacc;
#pragma unroll 1
    for (int z = crow + 1; z < head_row; ++z) out[(size_t)z * D + c] = 0.f;
    crow = head_row;
    cacc = head;
  }
  if (nruns > 1) {  // head run complete; rows up to the tail were written by the part
    out[(size_t)crow * D + c] = cacc;
    crow = tail_row;
    cacc = tail;
  }
}

__device__ __forceinline__ void finish_rows(int crow, float cacc, int rend, int c,
                                            float *__restrict__ out) {
  if (crow < rend) {
    out[(size_t)crow * D + c] = cacc;
#pragma unroll 1
    for (int z = crow + 1; z < rend; ++z) out[(size_t)z * D + c] = 0.f;
  }
}

// ---- per-step edge geometry (the reference's d cache, flash.py:221-223) ------
// geo[k] = (u, d) with u = r[own] - r[nbr] for CSR slot k; env[k] = (C, C').
// Block 0 also computes the row range of every work unit (balanced by edge
// count) once per step for the six edge launches that follow.
__global__ void __launch_bounds__(256)
k_edge_geom(const float *__restrict__ pos, const int32_t *__restrict__ ptr,
            const int32_t *__restrict__ nbr, const int32_t *__restrict__ own, int nrows,
            int64_t cap_e, float cutoff, float4 *__restrict__ geo, float2 *__restrict__ env,
            int32_t *__restrict__ unit_rows, int nunits) {
  long long e_tot = ptr[nrows];
  if (e_tot > cap_e) e_tot = cap_e;
  if (blockIdx.x == 0) {
    for (int u = threadIdx.x; u <= nunits; u += blockDim.x) {
      int rb, re;
      cta_row_range(ptr, nrows, e_tot, u < nunits ? u : nunits - 1, nunits, rb, re);
      unit_rows[u] = u < nunits ? rb : re;
    }
  }
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < e_tot;
       k += (long long)gridDim.x * blockDim.x) {
    const float *po = pos + (size_t)own[k] * 3, *pn = pos + (size_t)nbr[k] * 3;
    float ux = __fsub_rn(po[0], pn[0]), uy = __fsub_rn(po[1], pn[1]), uz = __fsub_rn(po[2], pn[2]);
    float d = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(ux, ux), __fmul_rn(uy, uy)), __fmul_rn(uz, uz)));
    float c = 0.f, dc = 0.f;
    if (d < cutoff) {  // cutoff_envelope(_grad), model.py:242-252
      float sn, cs;
      sincosf((3.14159265358979f * d) / cutoff, &sn, &cs);
      c = 0.5f * (cs + 1.f);
      dc = (float)(-0.5 * 3.141592653589793 / (double)cutoff) * sn;
    }
    geo[k] = make_float4(ux, uy, uz, d);
    env[k] = make_float2(c, dc);
  }
}

// ---- per-group context ---------------------------------------------------------
struct Grp {
  int g;              // group index
  int gt;             // thread index within the group
  int warp, lane, quarter, part, ch, ec;
  int bar_id;         // named barrier of the group
  uint32_t tl;        // TMEM address of this lane quarter + group column base
  uint32_t tmem_g;    // TMEM base of the group (lane 0)
  uint8_t *bb, *hb;   // basis buffer, act buffer
  uint32_t sbb, shb;  // their shared addresses
  TcShared *sh;
  uint32_t ph[2];
  __device__ __forceinline__ void sync() const { named_sync(bar_id, GT); }
  __device__ __forceinline__ TcMeta *meta(int i) const { return &sh->meta[g][i & 1]; }
  __device__ __forceinline__ void wait(int which) {
    tc::mbar_wait(&sh->bar[g][which], ph[which]);
    ph[which] ^= 1;
    tc::fence_after_sync();
  }
};

__device__ __forceinline__ Grp make_group(uint8_t *sm, TcShared *sh) {
  Grp G;
  G.g = threadIdx.x / GT;
  G.gt = threadIdx.x % GT;
  G.warp = G.gt >> 5;
  G.lane = threadIdx.x & 31;
  G.quarter = G.warp & 3;
  G.part = G.warp >> 2;
  G.ch = 32 * G.quarter + G.lane;
  G.ec = EPT * G.part;
  G.bar_id = 1 + G.g;
  G.sh = sh;
  G.bb = sm + SM_BUF + G.g * GBUF_BYTES;
  G.hb = G.bb + BB_BYTES;
  G.sbb = tc::smem_u32(G.bb);
  G.shb = tc::smem_u32(G.hb);
  G.tmem_g = sh->tmem + 256u * G.g;
  G.tl = G.tmem_g + ((uint32_t)(32 * G.quarter) << 16);
  G.ph[0] = G.ph[1] = 0;
  return G;
}

__device__ __forceinline__ void stage_weights(uint8_t *sm, const fcg_block &b) {
  const uint4 *s0 = (const uint4 *)b.f0_img, *s1 = (const uint4 *)b.f1_img;
  uint4 *d0 = (uint4 *)(sm + SM_W0), *d1 = (uint4 *)(sm + SM_W1);
  for (int q = threadIdx.x; q < (int)(2 * W0_BYTES / 16); q += TC_THREADS) d0[q] = __ldg(s0 + q);
  for (int q = threadIdx.x; q < (int)(2 * W1_BYTES / 16); q += TC_THREADS) d1[q] = __ldg(s1 + q);
}

__device__ __forceinline__ void kernel_prologue(uint8_t *sm, TcShared *sh, const fcg_block &B) {
  stage_weights(sm, B);
  if (threadIdx.x % GT == 0) {
    tc::mbar_init(&sh->bar[threadIdx.x / GT][0], 1);
    tc::mbar_init(&sh->bar[threadIdx.x / GT][1], 1);
    tc::fence_mbar_init();
  }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&sh->tmem);
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
}

__device__ __forceinline__ void tile_meta(const EdgeArgs &a, const float4 *__restrict__ geo,
                                          const float2 *__restrict__ env, const Grp &G,
                                          TcMeta *m, int t0, int n_e, bool src_owned) {
  int t = G.gt;
  if (t < TT) {
    int o = -1, n = 0;
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    float2 c = make_float2(0.f, 0.f);
    if (t < n_e) {
      o = a.own[t0 + t];
      n = a.nbr[t0 + t];
      g = geo[t0 + t];
      c = env[t0 + t];
    }
    // backward edge (dst=nbr, src=own): u = r_nbr - r_own (flash.py:279)
    if (src_owned) { g.x = -g.x; g.y = -g.y; g.z = -g.z; }
    m->own[t] = o;
    m->nbr[t] = n;
    m->d[t] = g.w;
    m->env[t] = c.x;
    m->denv[t] = c.y;
    m->u[t] = make_float4(g.x, g.y, g.z, 0.f);
  }
  if (t < 4) m->amax[t] = 0u;
}

// Basis b[k][e] (model.py:255-265) as the K=64 B operand (basis buffer):
// fp32 path scaled by 2^14 and split; W16 path rounded to fp16 unscaled
// (quantize.py:68-71).
__device__ __forceinline__ void tile_basis_tc(const EdgeArgs &a, const Grp &G, const TcMeta *m,
                                              int n_e, bool quant) {
#pragma unroll 2
  for (int q = G.gt; q < DR * (TT / 8); q += GT) {
    int k = q % DR, e0 = (q / DR) * 8;
    float mu = __ldg(&a.centers[k]);
    float4 d0 = *(const float4 *)&m->d[e0], d1 = *(const float4 *)&m->d[e0 + 4];
    float4 c0 = *(const float4 *)&m->env[e0], c1 = *(const float4 *)&m->env[e0 + 4];
    float dd[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
    float cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float dl = dd[i] - mu;
      v[i] = (e0 + i) < n_e ? __expf((-a.gamma * dl) * dl) * cc[i] : 0.f;
    }
    put_b8n(G.bb, DR, KSTR, k, e0, v, quant ? 1.f : 16384.f, !quant);
  }
}

// Segment reduction of a [128 ch][64 e] fp32 tile held in TMEM columns
// starting at tcol: both parts scan, part 1 publishes boundary partials, part
// 0 merges them into the carry.  Called by every thread of the group.
__device__ __forceinline__ void reduce_tile(uint32_t tcol, const Grp &G, TcMeta *meta, int n_e,
                                            int &crow, float &cacc, float *__restrict__ out) {
  const int lo = EPT * G.part, hi = min(lo + EPT, n_e);
  Runs r;
  r.init();
#pragma unroll 1
  for (int c0 = 0; c0 < EPT; c0 += 16) {
    float m[16];
    tc::tmem_ld16(tcol + lo + c0, m);
    tc::tmem_ld_wait();
    r.chunk(meta->own, lo + c0, min(16, hi - lo - c0), m, G.ch, out);
  }
  r.close();
  if (G.part == 1) {
    meta->xch[0][0][G.ch] = r.head;
    meta->xch[0][1][G.ch] = r.acc;
    meta->xch[0][2][G.ch] = __int_as_float(r.nruns);
  }
  G.sync();
  if (G.part == 0) {
    merge_part(crow, cacc, r.nruns, r.head, r.acc, meta->own[0], meta->own[max(hi - 1, 0)], G.ch,
               out);
    merge_part(crow, cacc, __float_as_int(meta->xch[0][2][G.ch]), meta->xch[0][0][G.ch],
               meta->xch[0][1][G.ch], meta->own[EPT], meta->own[max(n_e - 1, EPT)], G.ch, out);
  }
}

// Write this thread's [ch][32 edges] fp32 TMEM block as the hi/lo fp16 B
// operand (K = 128 rows, act buffer) of the next GEMM with the given scale.
__device__ __forceinline__ void tmem_to_act(uint32_t tcol, const Grp &G, float scale,
                                            bool with_lo) {
#pragma unroll 1
  for (int c0 = 0; c0 < EPT; c0 += 16) {
    float v[16];
    tc::tmem_ld16(tcol + G.ec + c0, v);
    tc::tmem_ld_wait();
    put_b8n(G.hb, D, KSTR, G.ch, G.ec + c0, &v[0], scale, with_lo);
    put_b8n(G.hb, D, KSTR, G.ch, G.ec + c0 + 8, &v[8], scale, with_lo);
  }
}

// all threads of the group: make the smem operand writes visible to the
// tensor core, then the group's first thread issues the GEMM and commits it
// to barrier `which`
#define GRP_ISSUE(which, ...)           \
  do {                                  \
    tc::fence_async_smem();             \
    tc::fence_before_sync();            \
    G.sync();                           \
    if (G.gt == 0) {                    \
      tc::fence_after_sync();           \
      issue_gemm(__VA_ARGS__, KSTR);    \
      tc::mma_commit(&G.sh->bar[G.g][which]); \
    }                                   \
  } while (0)

// phase timestamps for diagnosis: CTA 0, group 0, first 16 tiles
#define PHASE(kind, it, ph)                                                          \
  do {                                                                             \
    if (a.dbg && blockIdx.x == 0 && threadIdx.x == 0 && (it) < 16)                 \
      a.dbg[((kind) * 16 + (it)) * 64 + (ph)] = clock64();                         \
  } while (0)

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
// Forward: per 64-edge tile of dst rows
//   b -> [G1] z0 -> h=ssp(z0) -> [G2] w -> m = P[src]*w -> H rows.
// Software-pipelined per group: while G2(i) runs the group builds the basis
// of tile i+1 and issues G1(i+1); while G1(i+1) runs it finishes tile i
// (messages + segment sums).  TMEM per group: D0[2] = cols 0/64 (z0, h),
// D1[2] = 128/192 (w, m), by tile parity.
__global__ void __launch_bounds__(TC_THREADS, 1)
k_edge_fwd_tc(const EdgeArgs a, const float4 *__restrict__ geo, const float2 *__restrict__ env,
              const int32_t *__restrict__ unit_rows, const float *__restrict__ P,
              float *__restrict__ H) {
  extern __shared__ __align__(1024) uint8_t sm[];
  TcShared *sh = (TcShared *)(sm + SM_META);
  const bool quant = a.quant != 0;
  const fcg_block &B = a.blk;
  kernel_prologue(sm, sh, B);
  Grp G = make_group(sm, sh);
  const uint32_t sbase = tc::smem_u32(sm);
  const uint32_t idesc = tc::idesc_f16(128, TT, 0, 1);
  const int nprod = quant ? 1 : 3;

  const UnitRange tr = unit_range(a, unit_rows, NGRP * blockIdx.x + G.g);
  const int ntiles = (tr.ee - tr.eb + TT - 1) / TT;
  int crow = tr.rbeg;
  float cacc = 0.f;

  const int ch = G.ch, ec = G.ec;
  const float b0c = __ldg(&B.f0_b[ch]), b1c = __ldg(&B.f1_b[ch]);
  const float rs0 = quant ? __ldg(&B.f0_s[ch]) : pow2f(-(B.f0_exp + 14));
  const float rs1 = quant ? __ldg(&B.f1_s[ch]) : 1.f;

  float pv[EPT];  // P[src][ch] of this thread's edges of the current tile
  if (ntiles > 0) {
    TcMeta *m0 = G.meta(0);
    tile_meta(a, geo, env, G, m0, tr.eb, min(TT, tr.ee - tr.eb), false);
    G.sync();
    tile_basis_tc(a, G, m0, min(TT, tr.ee - tr.eb), quant);
    GRP_ISSUE(0, G.tmem_g + 0, sbase + SM_W0, W0_BYTES, DR, false, G.sbb, DR, idesc, nprod);
#pragma unroll
    for (int i = 0; i < EPT; ++i) pv[i] = __ldg(&P[(size_t)m0->nbr[ec + i] * D + ch]);
  }
  for (int it = 0; it < ntiles; ++it) {
    const int t0 = tr.eb + it * TT;
    const int n_e = min(TT, tr.ee - t0);
    TcMeta *M = G.meta(it);
    const uint32_t d0 = 64u * (it & 1), d1 = 128u + 64u * (it & 1);
    PHASE(0, it, 0);
    G.wait(0);  // G1(it)
    PHASE(0, it, 1);

    // epilogue 1: h = ssp(W0 b + b0), staged in place in D0, then -> act buffer
    float mx = 0.f;
#pragma unroll
    for (int c0 = 0; c0 < EPT; c0 += 16) {
      float v[16];
      tc::tmem_ld16(G.tl + d0 + ec + c0, v);
      tc::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float h = ssp_fast(v[i] * rs0 + b0c);
        if (quant) h = __half2float(__float2half_rn(h));
        v[i] = (ec + c0 + i) < n_e ? h : 0.f;
        mx = fmaxf(mx, fabsf(v[i]));
      }
      tc::tmem_st16(G.tl + d0 + ec + c0, v);
    }
    tc::tmem_st_wait();
    PHASE(0, it, 2);
    int sh_ = 0;
    if (!quant) sh_ = scale_exp(group_amax(mx, &M->amax[0], G.bar_id, GT));
    PHASE(0, it, 3);
    tmem_to_act(G.tl + d0, G, pow2f(sh_), !quant);
    PHASE(0, it, 4);
    GRP_ISSUE(1, G.tmem_g + d1, sbase + SM_W1, W1_BYTES, D, false, G.shb, D, idesc, nprod);
    PHASE(0, it, 5);

    // overlap with G2(it): basis of the next tile and its G1
    if (it + 1 < ntiles) {
      TcMeta *Mn = G.meta(it + 1);
      const int n_n = min(TT, tr.ee - (t0 + TT));
      tile_meta(a, geo, env, G, Mn, t0 + TT, n_n, false);
      G.sync();
      PHASE(0, it, 6);
      tile_basis_tc(a, G, Mn, n_n, quant);
      PHASE(0, it, 7);
      GRP_ISSUE(0, G.tmem_g + (64u * ((it + 1) & 1)), sbase + SM_W0, W0_BYTES, DR, false, G.sbb,
                DR, idesc, nprod);
    }
    PHASE(0, it, 8);
    G.wait(1);  // G2(it)
    PHASE(0, it, 9);

    // epilogue 2: m = (W1 h + b1) * P[src] (flash.py:229), in place in D1,
    // then dst segment sums (flash.py:232-234)
    const float s1 = quant ? rs1 : pow2f(-(B.f1_exp + sh_));
#pragma unroll
    for (int c = 0; c < EPT / 16; ++c) {
      float v[16];
      tc::tmem_ld16(G.tl + d1 + ec + 16 * c, v);
      tc::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = (v[i] * s1 + b1c) * pv[16 * c + i];
      tc::tmem_st16(G.tl + d1 + ec + 16 * c, v);
    }
    tc::tmem_st_wait();
    PHASE(0, it, 10);
    reduce_tile(G.tl + d1, G, M, n_e, crow, cacc, H);
    PHASE(0, it, 11);
    if (it + 1 < ntiles) {
      const TcMeta *Mn = G.meta(it + 1);
#pragma unroll
      for (int i = 0; i < EPT; ++i) pv[i] = __ldg(&P[(size_t)Mn->nbr[ec + i] * D + ch]);
    }
    tc::fence_before_sync();
    G.sync();
    PHASE(0, it, 12);
  }
  if (G.part == 0) finish_rows(crow, cacc, tr.rend, ch, H);
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(sh->tmem);
}

// ---------------------------------------------------------------------------
// Backward over src-owned rows (flash_block_backward, flash.py:272-295):
//   b -> [G1] z0 -> h -> [G2] w;  gH = GH[dst], grad_w = gH*P[src] ->
//   [G3] grad_h = grad_w W1 -> gz = grad_h*ssp'(z0) -> [G4] grad_b = gz W0
//   -> grad_d = sum_k grad_b*db -> g_e = grad_d/d * u  (gsum, owner slot);
//   grad_P rows = src-segment sums of gH*w (computed while G3 runs).  The
//   basis and G1 of tile i+1 overlap G4 of tile i.
// TMEM per group: D0 = 0 z0, D1 = 64 w (then gH*w), D2 = 128 h (then
// grad_h, then gz), D3 = 192 grad_w stash (then grad_b from G4).
__global__ void __launch_bounds__(TC_THREADS, 1)
k_edge_bwd_tc(const EdgeArgs a, const float4 *__restrict__ geo, const float2 *__restrict__ env,
              const int32_t *__restrict__ unit_rows, const float *__restrict__ P,
              const float *__restrict__ GH, float *__restrict__ GP, float4 *__restrict__ gsum,
              int accumulate) {
  extern __shared__ __align__(1024) uint8_t sm[];
  TcShared *sh = (TcShared *)(sm + SM_META);
  const bool quant = a.quant != 0;
  const fcg_block &B = a.blk;
  kernel_prologue(sm, sh, B);
  Grp G = make_group(sm, sh);
  float *red_s = (float *)G.hb;
  const uint32_t sbase = tc::smem_u32(sm);
  const uint32_t idesc_fwd = tc::idesc_f16(128, TT, 0, 1);
  const uint32_t idesc_g3 = tc::idesc_f16(128, TT, 1, 1);
  const uint32_t idesc_g4 = tc::idesc_f16(64, TT, 1, 1);
  const int nprod_f = quant ? 1 : 3, nprod_b = quant ? 2 : 3;
  constexpr uint32_t D0 = 0, D1 = 64, D2 = 128, D3 = 192;

  const UnitRange tr = unit_range(a, unit_rows, NGRP * blockIdx.x + G.g);
  const int ntiles = (tr.ee - tr.eb + TT - 1) / TT;
  int crow = tr.rbeg;
  float cacc = 0.f;

  const int ch = G.ch, ec = G.ec;
  const float b0c = __ldg(&B.f0_b[ch]), b1c = __ldg(&B.f1_b[ch]);
  const float rs0 = quant ? __ldg(&B.f0_s[ch]) : pow2f(-(B.f0_exp + 14));
  const float rs1 = quant ? __ldg(&B.f1_s[ch]) : 1.f;
  // backward GEMMs against the stored fp16 weights fold the W16 dequant
  // scale into the operand: g @ (s*w16) == (g*s) @ w16
  const float q1 = quant ? __ldg(&B.f1_s[ch]) : 1.f;
  const float q0 = quant ? __ldg(&B.f0_s[ch]) : 1.f;
  const int ew0 = quant ? 0 : B.f0_exp, ew1 = quant ? 0 : B.f1_exp;

  if (ntiles > 0) {
    TcMeta *m0 = G.meta(0);
    tile_meta(a, geo, env, G, m0, tr.eb, min(TT, tr.ee - tr.eb), true);
    G.sync();
    tile_basis_tc(a, G, m0, min(TT, tr.ee - tr.eb), quant);
    GRP_ISSUE(0, G.tmem_g + D0, sbase + SM_W0, W0_BYTES, DR, false, G.sbb, DR, idesc_fwd,
              nprod_f);
  }
  for (int it = 0; it < ntiles; ++it) {
    const int t0 = tr.eb + it * TT;
    const int n_e = min(TT, tr.ee - t0);
    TcMeta *M = G.meta(it);
    PHASE(1, it, 0);
    // while G1 runs: grad_w[c][e] = gH * P[src][c] (flash.py:291) into the
    // D3 stash + tile max
    float mx = 0.f;
#pragma unroll
    for (int c0 = 0; c0 < EPT; c0 += 16) {
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        int e = ec + c0 + i;
        float g = 0.f;
        if (e < n_e)
          g = __ldg(&GH[(size_t)M->nbr[e] * D + ch]) * __ldg(&P[(size_t)M->own[e] * D + ch]);
        v[i] = g * q1;
        mx = fmaxf(mx, fabsf(v[i]));
      }
      tc::tmem_st16(G.tl + D3 + ec + c0, v);
    }
    tc::tmem_st_wait();
    PHASE(1, it, 1);
    const int sg = scale_exp(group_amax(mx, &M->amax[1], G.bar_id, GT));
    PHASE(1, it, 2);
    G.wait(0);  // G1(it)
    PHASE(1, it, 3);

    // recompute h = ssp(z0) into D2; z0 stays in D0
    mx = 0.f;
#pragma unroll
    for (int c0 = 0; c0 < EPT; c0 += 16) {
      float v[16];
      tc::tmem_ld16(G.tl + D0 + ec + c0, v);
      tc::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float h = ssp_fast(v[i] * rs0 + b0c);
        if (quant) h = __half2float(__float2half_rn(h));
        v[i] = (ec + c0 + i) < n_e ? h : 0.f;
        mx = fmaxf(mx, fabsf(v[i]));
      }
      tc::tmem_st16(G.tl + D2 + ec + c0, v);
    }
    tc::tmem_st_wait();
    int sh_ = 0;
    if (!quant) sh_ = scale_exp(group_amax(mx, &M->amax[0], G.bar_id, GT));
    tmem_to_act(G.tl + D2, G, pow2f(sh_), !quant);
    PHASE(1, it, 4);
    GRP_ISSUE(1, G.tmem_g + D1, sbase + SM_W1, W1_BYTES, D, false, G.shb, D, idesc_fwd, nprod_f);
    PHASE(1, it, 5);
    G.wait(1);  // G2
    PHASE(1, it, 6);

    // grad_w (stashed in D3) -> B operand of G3
    tmem_to_act(G.tl + D3, G, pow2f(sg), true);
    GRP_ISSUE(1, G.tmem_g + D2, sbase + SM_W1, W1_BYTES, D, true, G.shb, D, idesc_g3, nprod_b);
    PHASE(1, it, 7);
    // while G3 runs: grad_P rows = src-segment sums of gH * w (flash.py:283-288)
    {
      const float s1 = quant ? rs1 : pow2f(-(B.f1_exp + sh_));
#pragma unroll
      for (int c0 = 0; c0 < EPT; c0 += 16) {
        float v[16], g[16];
        tc::tmem_ld16(G.tl + D1 + ec + c0, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) g[i] = __ldg(&GH[(size_t)M->nbr[ec + c0 + i] * D + ch]);
        tc::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = g[i] * (v[i] * s1 + b1c);
        tc::tmem_st16(G.tl + D1 + ec + c0, v);
      }
      tc::tmem_st_wait();
      PHASE(1, it, 8);
      reduce_tile(G.tl + D1, G, M, n_e, crow, cacc, GP);
    }
    PHASE(1, it, 9);
    G.wait(1);  // G3
    PHASE(1, it, 10);

    // gz = grad_h * ssp'(z0) (mlp_backward_input, model.py:326-331), in place in D2
    {
      const float sg3 = pow2f(-(ew1 + sg));
      mx = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < EPT; c0 += 16) {
        float gh[16], z[16];
        tc::tmem_ld16(G.tl + D2 + ec + c0, gh);
        tc::tmem_ld16(G.tl + D0 + ec + c0, z);
        tc::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float z0 = z[i] * rs0 + b0c;
          float g = (ec + c0 + i) < n_e ? gh[i] * sg3 * sigmoid_fast(z0) * q0 : 0.f;
          gh[i] = g;
          mx = fmaxf(mx, fabsf(g));
        }
        tc::tmem_st16(G.tl + D2 + ec + c0, gh);
      }
      tc::tmem_st_wait();
      PHASE(1, it, 11);
      sh_ = scale_exp(group_amax(mx, &M->amax[2], G.bar_id, GT));
      tmem_to_act(G.tl + D2, G, pow2f(sh_), true);
      GRP_ISSUE(1, G.tmem_g + D3, sbase + SM_W0, W0_BYTES, DR, true, G.shb, D, idesc_g4,
                nprod_b);
    }
    PHASE(1, it, 12);
    // overlap with G4(it): basis of the next tile and its G1 (D0 is free now)
    if (it + 1 < ntiles) {
      TcMeta *Mn = G.meta(it + 1);
      const int n_n = min(TT, tr.ee - (t0 + TT));
      tile_meta(a, geo, env, G, Mn, t0 + TT, n_n, true);
      G.sync();
      tile_basis_tc(a, G, Mn, n_n, quant);
      GRP_ISSUE(0, G.tmem_g + D0, sbase + SM_W0, W0_BYTES, DR, false, G.sbb, DR, idesc_fwd,
                nprod_f);
    }
    PHASE(1, it, 13);
    G.wait(1);  // G4
    PHASE(1, it, 14);

    // grad_d[e] = sum_k grad_b[k][e] * db[k][e] (flash.py:293).  M=64 D lives
    // in lanes 32q + (0..15) of each quarter: row k = 16q + lane.
    {
      const int k = 16 * G.quarter + (G.lane & 15);
      const float mu = __ldg(&a.centers[k]);
      const float s4 = pow2f(-(ew0 + sh_));
      const float g2 = -2.f * a.gamma;
#pragma unroll
      for (int c0 = 0; c0 < EPT; c0 += 16) {
        float gb[16];
        tc::tmem_ld16(G.tl + D3 + ec + c0, gb);
        tc::tmem_ld_wait();
        if (G.lane < 16) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            int e = ec + c0 + i;
            float dl = M->d[e] - mu;
            float gs = __expf((-a.gamma * dl) * dl);
            float db = gs * (g2 * dl * M->env[e] + M->denv[e]);  // model.py:289
            red_s[e * RED_LD + k] = gb[i] * s4 * db;
          }
        }
      }
    }
    G.sync();
    PHASE(1, it, 15);
    if (G.gt < TT && G.gt < n_e) {
      const int e = G.gt;
      float gd = 0.f;
#pragma unroll 8
      for (int k = 0; k < DR; ++k) gd += red_s[e * RED_LD + k];
      float d = M->d[e];
      float inv = d > TINY_DISTANCE ? 1.f / d : 0.f;  // _safe_inv, flash.py:176-178
      float s = gd * inv;
      float4 u = M->u[e];
      float4 g = make_float4(s * u.x, s * u.y, s * u.z, 0.f);
      float4 *dst = &gsum[t0 + e];
      if (accumulate) {
        float4 o = *dst;
        g.x += o.x; g.y += o.y; g.z += o.z;
      }
      *dst = g;
    }
    tc::fence_before_sync();
    G.sync();
    PHASE(1, it, 16);
  }
  if (G.part == 0) finish_rows(crow, cacc, tr.rend, ch, GP);
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(sh->tmem);
}

void edge_tc_configure() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(k_edge_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(SM_TOTAL + 1024));
  cudaFuncSetAttribute(k_edge_bwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(SM_TOTAL + 1024));
  done = true;
}

int edge_tc_units(int grid) { return NGRP * grid; }

void launch_edge_geom(const EdgeArgs &a, float4 *geo, float2 *env, int32_t *unit_rows,
                      int nunits, cudaStream_t s) {
  k_edge_geom<<<1184, 256, 0, s>>>(a.pos, a.ptr, a.nbr, a.own, a.nrows, a.cap_e, a.cutoff, geo,
                                   env, unit_rows, nunits);
}

void launch_edge_fwd_tc(const EdgeArgs &a, const float4 *geo, const float2 *env,
                        const int32_t *unit_rows, const float *P, float *H, int grid,
                        cudaStream_t s) {
  k_edge_fwd_tc<<<grid, TC_THREADS, SM_TOTAL + 1024, s>>>(a, geo, env, unit_rows, P, H);
}

void launch_edge_bwd_tc(const EdgeArgs &a, const float4 *geo, const float2 *env,
                        const int32_t *unit_rows, const float *P, const float *GH, float *GP,
                        float4 *gsum, int accumulate, int grid, cudaStream_t s) {
  k_edge_bwd_tc<<<grid, TC_THREADS, SM_TOTAL + 1024, s>>>(a, geo, env, unit_rows, P, GH, GP,
                                                         gsum, accumulate);
}

}  // namespace fcg
