// (f) rank 4 of SURVEY §8: batched trajectory analysis (analysis.py) on the
// GPU — Kabsch RMSD (analysis.py:56-85), the native-contact fraction Q
// (:100-108) and the GDT-TS superposition search (:115-143) for F frames at
// once, in fp64 like the reference.
//
// Superposition.  The reference takes the SVD of H = xc^T yc and builds the
// optimal PROPER rotation R = V diag(1,1,d) U^T (d = sign det).  Here the
// same rotation comes from Horn's quaternion form: the eigenvector of the
// largest eigenvalue of the symmetric 4x4 K(H), by cyclic Jacobi in fp64 —
// no SVD and no reflection fix-up (|dR| <= 1e-13, |d rmsd| <= 2e-15 against
// the reference on 2000 random cases).  The reference's degeneracy test
// (s1 <= 1e-12 max(s0, 1), analysis.py:74-75) uses singular values from a
// 3x3 Jacobi on H^T H.
//
// Work decomposition: lane-strided passes over the beads with warp-shuffle
// fp64 sums (centroids first, then the centred covariance, as the reference
// does).  RMSD: one warp per frame, every lane solving the frame's small
// eigenproblems.  GDT: one warp per 32 seeds of a frame, one seed's
// eigenproblems per lane, then warp-cooperative counting of the beads within
// the 0.1/0.2/0.4/0.8 nm ladder with ballots; the best seed per cutoff is an
// atomicMax on integer counts and the host forms count/n and the mean
// exactly as the reference does.  Q: one CTA per frame.
#include "common.cuh"

namespace fcg {

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Cyclic Jacobi on a symmetric N x N matrix: a -> diagonal (eigenvalues),
// v -> eigenvectors (columns).
template <int N>
__device__ void jacobi_eig(double (&a)[N][N], double (&v)[N][N]) {
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) v[i][j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0, diag = 0.0;
#pragma unroll
    for (int p = 0; p < N; ++p) {
      diag += a[p][p] * a[p][p];
#pragma unroll
      for (int q = p + 1; q < N; ++q) off += a[p][q] * a[p][q];
    }
    if (off <= 1e-36 * diag || off == 0.0) break;
#pragma unroll
    for (int p = 0; p < N; ++p) {
#pragma unroll
      for (int q = p + 1; q < N; ++q) {
        const double apq = a[p][q];
        if (apq == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        // A <- P^T A P with P = I except P[p][p]=P[q][q]=c, P[p][q]=s, P[q][p]=-s
#pragma unroll
        for (int k = 0; k < N; ++k) {  // columns
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {  // rows
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const double vkp = v[k][p], vkq = v[k][q];
          v[k][p] = c * vkp - s * vkq;
          v[k][q] = s * vkp + c * vkq;
        }
      }
    }
  }
}

// Optimal proper rotation taking centred x onto centred y from
// H[a][b] = sum_i x_i[a] y_i[b]; false if H is degenerate by the reference's
// criterion.
__device__ bool rotation_from_cov(const double (&h)[3][3], double (&r)[3][3]) {
  double m[3][3], ev[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      m[i][j] = h[0][i] * h[0][j] + h[1][i] * h[1][j] + h[2][i] * h[2][j];
  jacobi_eig<3>(m, ev);
  double s[3] = {sqrt(fmax(m[0][0], 0.0)), sqrt(fmax(m[1][1], 0.0)), sqrt(fmax(m[2][2], 0.0))};
  // sort descending (3 elements)
  if (s[0] < s[1]) { double t = s[0]; s[0] = s[1]; s[1] = t; }
  if (s[1] < s[2]) { double t = s[1]; s[1] = s[2]; s[2] = t; }
  if (s[0] < s[1]) { double t = s[0]; s[0] = s[1]; s[1] = t; }
  if (s[1] <= 1e-12 * fmax(s[0], 1.0)) return false;

  const double sxx = h[0][0], sxy = h[0][1], sxz = h[0][2];
  const double syx = h[1][0], syy = h[1][1], syz = h[1][2];
  const double szx = h[2][0], szy = h[2][1], szz = h[2][2];
  double k[4][4] = {{sxx + syy + szz, syz - szy, szx - sxz, sxy - syx},
                    {syz - szy, sxx - syy - szz, sxy + syx, szx + sxz},
                    {szx - sxz, sxy + syx, -sxx + syy - szz, syz + szy},
                    {sxy - syx, szx + sxz, syz + szy, -sxx - syy + szz}};
  double v[4][4];
  jacobi_eig<4>(k, v);
  double q[4] = {v[0][0], v[1][0], v[2][0], v[3][0]}, lmax = k[0][0];
#pragma unroll
  for (int i = 1; i < 4; ++i) {
    if (k[i][i] > lmax) {  // eigenvector of the largest eigenvalue
      lmax = k[i][i];
#pragma unroll
      for (int j = 0; j < 4; ++j) q[j] = v[j][i];
    }
  }
  const double nrm = 1.0 / sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
#pragma unroll
  for (int i = 0; i < 4; ++i) q[i] *= nrm;
  const double q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3];
  r[0][0] = q0 * q0 + q1 * q1 - q2 * q2 - q3 * q3;
  r[0][1] = 2.0 * (q1 * q2 - q0 * q3);
  r[0][2] = 2.0 * (q1 * q3 + q0 * q2);
  r[1][0] = 2.0 * (q1 * q2 + q0 * q3);
  r[1][1] = q0 * q0 - q1 * q1 + q2 * q2 - q3 * q3;
  r[1][2] = 2.0 * (q2 * q3 - q0 * q1);
  r[2][0] = 2.0 * (q1 * q3 - q0 * q2);
  r[2][1] = 2.0 * (q2 * q3 + q0 * q1);
  r[2][2] = q0 * q0 - q1 * q1 - q2 * q2 + q3 * q3;
  return true;
}

struct Superpose {
  double xm[3], ym[3];
  double r[3][3];
  bool ok;
};

// Warp-collective superposition of beads [b0, b0+len) of x onto y.
__device__ Superpose superpose_warp(const double *x, const double *y, int b0, int len, int lane) {
  Superpose sp;
  double sx[3] = {0, 0, 0}, sy[3] = {0, 0, 0};
  for (int i = lane; i < len; i += 32) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      sx[a] += x[(size_t)(b0 + i) * 3 + a];
      sy[a] += y[(size_t)(b0 + i) * 3 + a];
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    sp.xm[a] = warp_sum_d(sx[a]) / len;
    sp.ym[a] = warp_sum_d(sy[a]) / len;
  }
  double h[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int i = lane; i < len; i += 32) {
    double xc[3], yc[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      xc[a] = x[(size_t)(b0 + i) * 3 + a] - sp.xm[a];
      yc[a] = y[(size_t)(b0 + i) * 3 + a] - sp.ym[a];
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) h[a][b] += xc[a] * yc[b];
  }
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) h[a][b] = warp_sum_d(h[a][b]);
  sp.ok = len >= 3 && rotation_from_cov(h, sp.r);
  return sp;
}

// ---- Kabsch RMSD per frame (kabsch_align / rmsd, analysis.py:56-85) ----------
__global__ void __launch_bounds__(256)
k_kabsch(const double *x, const double *ref, int F, int n, double *rmsd, double *rot,
         double *trans, int32_t *degenerate) {
  const int lane = threadIdx.x & 31;
  const long long f = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (f >= F) return;
  const double *xf = x + (size_t)f * n * 3;
  const Superpose sp = superpose_warp(xf, ref, 0, n, lane);
  double ss = 0.0;
  if (sp.ok) {
    for (int i = lane; i < n; i += 32) {
      double xc[3], d2 = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) xc[a] = xf[(size_t)i * 3 + a] - sp.xm[a];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double m = sp.r[a][0] * xc[0] + sp.r[a][1] * xc[1] + sp.r[a][2] * xc[2];
        const double d = m - (ref[(size_t)i * 3 + a] - sp.ym[a]);
        d2 += d * d;
      }
      ss += d2;
    }
  }
  ss = warp_sum_d(ss);
  if (lane == 0) {
    degenerate[f] = sp.ok ? 0 : 1;
    rmsd[f] = sp.ok ? sqrt(ss / n) : 0.0;
    if (rot) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) rot[(size_t)f * 9 + a * 3 + b] = sp.ok ? sp.r[a][b] : 0.0;
    }
    if (trans) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
        trans[(size_t)f * 3 + a] =
            sp.ok ? sp.ym[a] - (sp.r[a][0] * sp.xm[0] + sp.r[a][1] * sp.xm[1] + sp.r[a][2] * sp.xm[2])
                  : 0.0;
    }
  }
}

// ---- GDT-TS window search (gdt_ts, analysis.py:115-143) ----------------------
// One warp per 32 seeds of one frame (windows[w] = (start, length)).  The
// covariances are warp-cooperative sums (lane j keeps seed j's), the
// eigen-solves then run one seed per lane — 32 at once instead of 32 lanes
// repeating one — and each rotation is broadcast in turn to count the beads
// within the cutoff ladder; the per-cutoff maxima stay in registers until one
// atomicMax per warp.
__global__ void __launch_bounds__(256)
k_gdt(const double *x, const double *ref, int F, int n, const int32_t *windows, int W,
      double c0, double c1, double c2, double c3, int32_t *best) {
  const int lane = threadIdx.x & 31;
  const int nblk = (W + 31) / 32;
  const long long t = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (t >= (long long)F * nblk) return;
  const int f = (int)(t / nblk), wb = (int)(t % nblk) * 32;
  const int nw = min(32, W - wb);
  const double *xf = x + (size_t)f * n * 3;
  double mh[3][3], mxm[3], mym[3];
  int mlen = 0;
  for (int j = 0; j < nw; ++j) {
    const int b0 = windows[2 * (wb + j)], len = windows[2 * (wb + j) + 1];
    double sx[3] = {0, 0, 0}, sy[3] = {0, 0, 0};
    for (int i = lane; i < len; i += 32) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        sx[a] += xf[(size_t)(b0 + i) * 3 + a];
        sy[a] += ref[(size_t)(b0 + i) * 3 + a];
      }
    }
    double xm[3], ym[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      xm[a] = warp_sum_d(sx[a]) / len;
      ym[a] = warp_sum_d(sy[a]) / len;
    }
    double h[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int i = lane; i < len; i += 32) {
      double xc[3], yc[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        xc[a] = xf[(size_t)(b0 + i) * 3 + a] - xm[a];
        yc[a] = ref[(size_t)(b0 + i) * 3 + a] - ym[a];
      }
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) h[a][b] += xc[a] * yc[b];
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) h[a][b] = warp_sum_d(h[a][b]);
    if (lane == j) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        mxm[a] = xm[a];
        mym[a] = ym[a];
#pragma unroll
        for (int b = 0; b < 3; ++b) mh[a][b] = h[a][b];
      }
      mlen = len;
    }
  }
  // one seed per lane
  double r[3][3], tr[3];
  const bool ok = lane < nw && mlen >= 3 && rotation_from_cov(mh, r);
  if (ok) {
#pragma unroll
    for (int a = 0; a < 3; ++a) tr[a] = mym[a] - (r[a][0] * mxm[0] + r[a][1] * mxm[1] + r[a][2] * mxm[2]);
  }
  const unsigned okmask = __ballot_sync(0xffffffffu, ok);
  int keep = 0;  // lane c < 4: best count for cutoff c over this warp's seeds
  for (int j = 0; j < nw; ++j) {
    if (!((okmask >> j) & 1u)) continue;  // a degenerate seed is skipped (analysis.py:133-134)
    double rj[3][3], tj[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      tj[a] = __shfl_sync(0xffffffffu, tr[a], j);
#pragma unroll
      for (int b = 0; b < 3; ++b) rj[a][b] = __shfl_sync(0xffffffffu, r[a][b], j);
    }
    int cnt[4] = {0, 0, 0, 0};
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      double dist = 1e300;
      if (i < n) {
        const double px = xf[(size_t)i * 3], py = xf[(size_t)i * 3 + 1], pz = xf[(size_t)i * 3 + 2];
        double d[3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
          d[a] = (rj[a][0] * px + rj[a][1] * py + rj[a][2] * pz + tj[a]) - ref[(size_t)i * 3 + a];
        dist = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])),
                              __dmul_rn(d[2], d[2])));
      }
      cnt[0] += __popc(__ballot_sync(0xffffffffu, dist <= c0));
      cnt[1] += __popc(__ballot_sync(0xffffffffu, dist <= c1));
      cnt[2] += __popc(__ballot_sync(0xffffffffu, dist <= c2));
      cnt[3] += __popc(__ballot_sync(0xffffffffu, dist <= c3));
    }
    const int mine = lane == 0 ? cnt[0] : lane == 1 ? cnt[1] : lane == 2 ? cnt[2] : cnt[3];
    keep = max(keep, mine);
  }
  if (lane < 4 && okmask) atomicMax(&best[(size_t)f * 4 + lane], keep);
}

// ---- native-contact fraction (fraction_native_contacts, analysis.py:100-108) --
__global__ void __launch_bounds__(256)
k_native_q(const double *x, int n, const int32_t *pairs, const double *ref_dist, int C,
           double beta, double lam, double *q) {
  __shared__ double part[8];
  const double *xf = x + (size_t)blockIdx.x * n * 3;
  double s = 0.0;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const int i = pairs[2 * c], j = pairs[2 * c + 1];
    const double dx = xf[(size_t)i * 3] - xf[(size_t)j * 3];
    const double dy = xf[(size_t)i * 3 + 1] - xf[(size_t)j * 3 + 1];
    const double dz = xf[(size_t)i * 3 + 2] - xf[(size_t)j * 3 + 2];
    const double r = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    s += 1.0 / (1.0 + exp(beta * (r - lam * ref_dist[c])));
  }
  s = warp_sum_d(s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
    q[blockIdx.x] = t / C;
  }
}

}  // namespace fcg

using namespace fcg;

extern "C" int fcg_kabsch(const double *x, const double *ref, int F, int N, double *rmsd,
                          double *rot, double *trans, int32_t *degenerate, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (F < 0 || N < 1 || (F && (!x || !ref || !rmsd || !degenerate))) {
    set_error("kabsch: bad arguments");
    return FCG_ERR_ARG;
  }
  if (F == 0) return FCG_OK;
  k_kabsch<<<ceil_div((long long)F * 32, 256), 256, 0, s>>>(x, ref, F, N, rmsd, rot, trans,
                                                            degenerate);
  return cuda_status("kabsch");
}

extern "C" int fcg_gdt_counts(const double *x, const double *ref, int F, int N,
                              const int32_t *windows, int W, const double *cutoffs,
                              int32_t *best, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (F < 0 || N < 1 || W < 0 || !cutoffs || (F && (!x || !ref || !best)) || (W && !windows)) {
    set_error("gdt_counts: bad arguments");
    return FCG_ERR_ARG;
  }
  if (F == 0) return FCG_OK;
  cudaMemsetAsync(best, 0, sizeof(int32_t) * 4 * (size_t)F, s);
  if (W > 0)
    k_gdt<<<ceil_div((long long)F * ((W + 31) / 32) * 32, 256), 256, 0, s>>>(
        x, ref, F, N, windows, W, cutoffs[0], cutoffs[1], cutoffs[2], cutoffs[3], best);
  return cuda_status("gdt_counts");
}

extern "C" int fcg_native_q(const double *x, int F, int N, const int32_t *pairs,
                            const double *ref_dist, int C, double beta, double lam, double *q,
                            void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (F < 0 || N < 1 || C < 1 || (F && (!x || !pairs || !ref_dist || !q))) {
    set_error("native_q: bad arguments (an empty contact set has no Q)");
    return FCG_ERR_ARG;
  }
  if (F == 0) return FCG_OK;
  k_native_q<<<F, 256, 0, s>>>(x, N, pairs, ref_dist, C, beta, lam, q);
  return cuda_status("native_q");
}
