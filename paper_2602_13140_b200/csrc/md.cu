// (f) Batched Langevin integrator: numpy-exact noise stream, BAOAB halves,
// harmonic prior.  Replaces md.py:109-208 for all replicas at once.
//
// Bitwise contract with the reference under numpy 2 (NEP 50):
//  - noise: Generator(Philox(key=[seed, rep], counter=[0,0,0,step]))
//    .standard_normal((N,3)).astype(float32) (md.py:127-131, :167-168),
//    reproduced as Philox-4x64-10 + numpy's 256-layer ziggurat with the
//    exact tables extracted from numpy (ziggurat_tables.h);
//  - every Python-float coefficient is rounded to fp32 first and each
//    operation rounds in fp32, left to right: v + ((0.5dt*F)/m), etc.  We use
//    _rn intrinsics so nvcc cannot contract into FMAs.
#include "common.cuh"
#include "prior.cuh"
#include "ziggurat_tables.h"

namespace fcg {

constexpr int NOISE_RING = 16;  // steps of noise generated per refill

// ---- Philox-4x64-10 (Random123 / numpy) ------------------------------------
struct U64x4 { uint64_t v[4]; };

__device__ __forceinline__ U64x4 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2,
                                                uint64_t c3, uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
    uint64_t hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += W0; k1 += W1;
  }
  U64x4 o;
  o.v[0] = c0; o.v[1] = c1; o.v[2] = c2; o.v[3] = c3;
  return o;
}

// q-th 64-bit word of the (seed, rep, step) stream.  numpy increments the
// 256-bit counter before every block, so block b runs on [b+1, 0, 0, step].
__device__ __forceinline__ uint64_t stream_word(uint64_t seed, uint64_t rep, uint64_t step,
                                                uint64_t q) {
  U64x4 o = philox4x64_10((q >> 2) + 1, 0, 0, step, seed, rep);
  int w = (int)(q & 3);
  return w == 0 ? o.v[0] : w == 1 ? o.v[1] : w == 2 ? o.v[2] : o.v[3];
}

__device__ __forceinline__ double zig_w(int i) { return __longlong_as_double((long long)fcg_zig_wi_bits[i]); }
__device__ __forceinline__ double zig_f(int i) { return __longlong_as_double((long long)fcg_zig_fi_bits[i]); }

__device__ __forceinline__ double u64_to_unit(uint64_t r) {
  return __dmul_rn((double)(r >> 11), 1.0 / 9007199254740992.0);
}

struct ZigDraw {
  double x;
  uint64_t rabs;
  int idx;
  bool fast;
};
__device__ __forceinline__ ZigDraw zig_decode(uint64_t r) {
  ZigDraw z;
  z.idx = (int)(r & 0xff);
  r >>= 8;
  int sign = (int)(r & 1);
  z.rabs = (r >> 1) & 0x000fffffffffffffull;
  z.x = __dmul_rn((double)z.rabs, zig_w(z.idx));
  if (sign) z.x = -z.x;
  z.fast = z.rabs < fcg_zig_ki_bits[z.idx];
  return z;
}

// Rejection branches of numpy's random_standard_normal for a draw at stream
// position q that failed the fast test; returns the sample and the number of
// words consumed from q on.
__device__ double zig_slow(uint64_t seed, uint64_t rep, uint64_t step, uint64_t q, uint64_t r0,
                           uint64_t *consumed) {
  const double ZR = 3.6541528853610088, ZINV = 0.27366123732975828;
  uint64_t used = 1;
  ZigDraw z = zig_decode(r0);
  for (;;) {
    if (z.fast) break;
    if (z.idx == 0) {
      for (;;) {
        double u1 = u64_to_unit(stream_word(seed, rep, step, q + used)); ++used;
        double xx = __dmul_rn(-ZINV, log1p(-u1));
        double u2 = u64_to_unit(stream_word(seed, rep, step, q + used)); ++used;
        double yy = -log1p(-u2);
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
          double v = __dadd_rn(ZR, xx);
          z.x = ((z.rabs >> 8) & 1) ? -v : v;
          *consumed = used;
          return z.x;
        }
      }
    } else {
      double u = u64_to_unit(stream_word(seed, rep, step, q + used)); ++used;
      double lhs = __dadd_rn(__dmul_rn(__dsub_rn(zig_f(z.idx - 1), zig_f(z.idx)), u), zig_f(z.idx));
      if (lhs < exp(__dmul_rn(__dmul_rn(-0.5, z.x), z.x))) break;
    }
    z = zig_decode(stream_word(seed, rep, step, q + used)); ++used;
  }
  *consumed = used;
  return z.x;
}

// One warp per replica walks its stream in windows of 128 words: lane L
// computes Philox block (base + L), i.e. words 4L..4L+3 of the window, and
// decodes a draw at each of them.  Draws from the current sample start up to
// the first draw that misses the fast path are consecutive samples; that
// draw's owner lane resolves numpy's rejection loop alone (reading further
// words on demand) and the walk resumes after the words it consumed.
// The warp's walk over one (seed, rep, step) stream, writing n3 samples.
__device__ __forceinline__ void noise_stream(uint64_t seed, uint64_t rep, uint64_t step, int n3,
                                             float *__restrict__ dst, int lane) {
  uint64_t pos = 0;  // stream position of the next sample start
  int produced = 0;
  while (produced < n3) {
    const uint64_t wbase = (pos >> 2) << 2;  // window = words [wbase, wbase + 128)
    U64x4 o = philox4x64_10(((wbase >> 2) + lane) + 1, 0, 0, step, seed, rep);
    ZigDraw z[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) z[j] = zig_decode(o.v[j]);
    const uint64_t wend = wbase + 128;
    while (pos < wend && produced < n3) {
      // first slow draw at or after pos (window-relative index, 128 = none)
      int my = 128;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint64_t p = wbase + 4 * lane + j;
        if (my == 128 && p >= pos && !z[j].fast) my = 4 * lane + j;
      }
      const int first = __reduce_min_sync(0xffffffffu, my);
      const uint64_t stop = first == 128 ? wend : wbase + first;
      // fast samples at positions [pos, stop)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint64_t p = wbase + 4 * lane + j;
        if (p >= pos && p < stop) {
          long long idx = produced + (long long)(p - pos);
          if (idx < n3) dst[idx] = __double2float_rn(z[j].x);
        }
      }
      produced += (int)(stop - pos);
      if (first == 128) {
        pos = wend;
        break;
      }
      double xs = 0.0;
      uint64_t used = 0;
      const int owner = first >> 2, jj = first & 3;
      if (lane == owner) {
        uint64_t r = jj == 0 ? o.v[0] : jj == 1 ? o.v[1] : jj == 2 ? o.v[2] : o.v[3];
        xs = zig_slow(seed, rep, step, stop, r, &used);
      }
      xs = __shfl_sync(0xffffffffu, xs, owner);
      used = __shfl_sync(0xffffffffu, used, owner);
      if (lane == 0 && produced < n3) dst[produced] = __double2float_rn(xs);
      produced += 1;
      pos = stop + used;
    }
  }
}

__global__ void __launch_bounds__(256)
k_normal_noise(uint64_t seed, int rep_offset, const int64_t *__restrict__ stepp, int R, int n3,
               float *__restrict__ out) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= R) return;
  noise_stream(seed, (uint64_t)(rep_offset + warp), (uint64_t)*stepp, n3,
               out + (size_t)warp * n3, lane);
}

// ---- noise ring for fcg_md_step ---------------------------------------------
// The noise of a step depends only on (seed, replica, step) (md.py:127-131),
// so the MD step generates it NOISE_RING steps at a time (R x NOISE_RING
// warps instead of R) into a workspace ring.  A device tag {magic, seed,
// rep_offset, base step} says which steps the ring holds; every CTA of the
// leading half-step kernel evaluates ring_valid() on the same tag, and only
// the step advance (its last CTA to finish) rewrites it.
struct NoiseTag {
  uint64_t magic, seed;
  int64_t rep_offset, base, layout;  // layout = R * 2^32 + 3N
};
constexpr uint64_t kNoiseMagic = 0x4e6f697365526e67ull;  // "NoiseRng"
__device__ __forceinline__ bool ring_valid(const NoiseTag *t, uint64_t seed, int rep_offset,
                                           int64_t layout, int64_t step) {
  return t->magic == kNoiseMagic && t->seed == seed && t->rep_offset == rep_offset &&
         t->layout == layout && step >= t->base && step < t->base + NOISE_RING;
}


int normal_noise(uint64_t seed, int rep_offset, const int64_t *step, int R, int N, float *out,
                 cudaStream_t s) {
  if (R < 1 || N < 1) { set_error("normal_noise: bad shape"); return FCG_ERR_ARG; }
  FCG_PROF(P_NOISE, s);
  k_normal_noise<<<ceil_div((long long)R * 32, 256), 256, 0, s>>>(seed, rep_offset, step, R, 3 * N,
                                                                  out);
  return cuda_status("normal_noise");
}

// ---- BAOAB halves ----------------------------------------------------------
// langevin_step, md.py:158-172:
//   v = v + ((h*F)/m); r = r + h*v; v = c1*v + sqrt(c2n/m)*xi; r = r + h*v
__global__ void k_baoa(fcg_md_params p, const float *__restrict__ mass, int N, long long n,
                       const float *__restrict__ F, const float *__restrict__ xi,
                       float *__restrict__ pos, float *__restrict__ vel) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= n) return;
  int i = (int)((t / 3) % N);
  float m = mass[i];
  float v = vel[t], r = pos[t];
  v = __fadd_rn(v, __fdiv_rn(__fmul_rn(p.half_dt, F[t]), m));
  r = __fadd_rn(r, __fmul_rn(p.half_dt, v));
  float c2 = __fsqrt_rn(__fdiv_rn(p.c2_num, m));
  v = __fadd_rn(__fmul_rn(p.c1, v), __fmul_rn(c2, xi[t]));
  r = __fadd_rn(r, __fmul_rn(p.half_dt, v));
  vel[t] = v;
  pos[t] = r;
}

int langevin_baoa(const fcg_md_params *p, const float *mass, int R, int N, const float *forces,
                  const float *noise, float *pos, float *vel, cudaStream_t s) {
  long long n = (long long)R * N * 3;
  FCG_PROF(P_BAOA, s);
  k_baoa<<<ceil_div(n, 256), 256, 0, s>>>(*p, mass, N, n, forces, noise, pos, vel);
  return cuda_status("langevin_baoa");
}

// Noise refill and BAOA in one launch: CTA r owns replica r.  On a refill
// step its NOISE_RING warps each generate one step of the replica's noise
// (the same warps per refill as a separate noise launch would use), then the CTA
// applies BAOA to the replica's 3N coordinates with this step's slot —
// only replica r's noise is read, so a CTA barrier orders the two.  The
// last CTA to finish (an arrival counter in the status words, reset by
// that CTA) then advances the step and, after a refill, the ring tag —
// every CTA has read both before it arrives.
static_assert(NOISE_RING * 32 <= 1024, "one warp per ring step");
__global__ void __launch_bounds__(NOISE_RING * 32)
k_noise_baoa_ring(fcg_md_params p, const float *mass, int N, int R, const float *F,
                  NoiseTag *tag, int64_t *stepp, float *ring, float *pos,
                  float *vel, unsigned long long *arrive) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const int n3 = 3 * N;
  const long long n = (long long)R * n3;
  const int64_t step = *stepp;
  const bool valid = ring_valid(tag, p.seed, p.rep_offset, ((int64_t)R << 32) + n3, step);
  if (!valid) {
    const int j = threadIdx.x >> 5, lane = threadIdx.x & 31;
    noise_stream(p.seed, (uint64_t)(p.rep_offset + r), (uint64_t)(step + j), n3,
                 ring + ((size_t)j * R + r) * n3, lane);
    __syncthreads();
  }
  const int64_t slot = valid ? step - tag->base : 0;
  const float *xi = ring + slot * n + (size_t)r * n3;
  float *pr = pos + (size_t)r * n3, *vr = vel + (size_t)r * n3;
  const float *Fr = F + (size_t)r * n3;
  for (int k = threadIdx.x; k < n3; k += blockDim.x) {
    const float m = mass[k / 3];
    float v = vr[k], x = pr[k];
    v = __fadd_rn(v, __fdiv_rn(__fmul_rn(p.half_dt, Fr[k]), m));
    x = __fadd_rn(x, __fmul_rn(p.half_dt, v));
    const float c2 = __fsqrt_rn(__fdiv_rn(p.c2_num, m));
    v = __fadd_rn(__fmul_rn(p.c1, v), __fmul_rn(c2, xi[k]));
    x = __fadd_rn(x, __fmul_rn(p.half_dt, v));
    vr[k] = v;
    pr[k] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(arrive, 1ull) == (unsigned long long)gridDim.x - 1) {
      __threadfence();
      if (!valid) {
        tag->magic = kNoiseMagic;
        tag->seed = p.seed;
        tag->rep_offset = p.rep_offset;
        tag->layout = ((int64_t)R << 32) + n3;
        tag->base = step;
      }
      *stepp = step + 1;
      *arrive = 0ull;
    }
  }
}

size_t noise_ring_bytes(int R, int N) {
  return 256 + sizeof(float) * (size_t)NOISE_RING * R * N * 3;
}

// Leading B + A + O + A of langevin_step (md.py:200-202) for all replicas
// with the ring noise, then step += 1.
int langevin_leading(const fcg_md_params *p, const float *mass, int R, int N,
                     const float *forces, int64_t *step, float *pos, float *vel, void *ring_ws,
                     int64_t *status, cudaStream_t s) {
  NoiseTag *tag = (NoiseTag *)ring_ws;
  float *ring = (float *)((char *)ring_ws + 256);
  const long long n = (long long)R * N * 3;
  (void)n;
  {
    FCG_PROF(P_BAOA, s);  // noise refill (every NOISE_RING steps) + BAOA + step advance
    launch_pdl(PDL_SMALL, k_noise_baoa_ring, R, NOISE_RING * 32, 0, s, *p, mass, N, R, forces,
               tag, step, ring, pos, vel,
               (unsigned long long *)(status + FCG_ST_ARRIVE));
  }
  return cuda_status("langevin_leading");
}

// half_kick, md.py:134-138
__global__ void k_half_kick(fcg_md_params p, const float *__restrict__ mass, int N, long long n,
                            const float *__restrict__ F, float *__restrict__ vel) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= n) return;
  int i = (int)((t / 3) % N);
  vel[t] = __fadd_rn(vel[t], __fdiv_rn(__fmul_rn(p.half_dt, F[t]), mass[i]));
}

int half_kick(const fcg_md_params *p, const float *mass, int R, int N, const float *forces,
              float *vel, cudaStream_t s) {
  long long n = (long long)R * N * 3;
  k_half_kick<<<ceil_div(n, 256), 256, 0, s>>>(*p, mass, N, n, forces, vel);
  return cuda_status("half_kick");
}

// Both in one launch (they only read positions): blocks [0, nbead) do the
// per-bead forces, the last R blocks the per-replica energies.
__global__ void __launch_bounds__(256)
k_prior(const fcg_prior pr, const float *pos, int N, int RN, int nbead, float *f_prior,
        float *e_prior) {
  pdl_trigger();
  pdl_wait();
  if ((int)blockIdx.x < nbead)
    prior_bead(pr, pos, N, RN, f_prior, blockIdx.x * blockDim.x + threadIdx.x);
  else
    prior_energy(pr, pos, N, e_prior, blockIdx.x - nbead);
}

int prior_forces(const fcg_prior *pr, const float *pos, int R, int N, float *e_prior,
                 float *f_prior, cudaStream_t s) {
  FCG_PROF(P_PRIOR, s);
  const int nbead = (int)ceil_div((long long)R * N, 256);
  launch_pdl(PDL_SMALL, k_prior, nbead + R, 256, 0, s, *pr, pos, N, R * N, nbead, f_prior,
             e_prior);
  return cuda_status("prior_forces");
}

__global__ void k_step_advance(int64_t *step) { *step += 1; }
int step_advance(int64_t *step, cudaStream_t s) {
  FCG_PROF(P_STEP, s);
  k_step_advance<<<1, 1, 0, s>>>(step);
  return cuda_status("step_advance");
}

}  // namespace fcg
