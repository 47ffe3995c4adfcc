// quantize_model's scale calibration on the GPU (
// quantize.py:126-178, :224-299).
//
// For every output row of a linear layer and every candidate scale s, the
// reference rounds the row to fp16 at that scale, q = fp16(w / s), and
// scores the candidate by the output error the rounding causes on the
// calibration inputs: err = dw^T G dw with dw = q s - w and G = X^T X the
// Gram matrix of the inputs.  One CTA scores one (row, candidate) pair in
// fp64: thread i forms dw_i, the CTA keeps dw in shared memory, thread i
// computes (G dw)_i and the products are summed in a fixed tree order.
// Rounding follows numpy: the quotient in fp64, then fp64 -> fp16 round to
// nearest even (__double2half).  The host picks the argmin; the summation
// order differs from numpy's BLAS, so rows whose best two candidates are
// within a relative 1e-9 are re-scored on the host with the reference's
// own operations (w16.quantize_model), which keeps the chosen scales — and
// so the stored fp16 weights — bit-identical to the reference.
#include <cuda_fp16.h>

#include "common.cuh"

namespace fcg {

constexpr int CAL_MAXK = 256;

__global__ void __launch_bounds__(256)
k_calib_errors(const double *__restrict__ w, int k, const double *__restrict__ cand, int ncand,
               const double *__restrict__ gram, double *__restrict__ err) {
  __shared__ double dw[CAL_MAXK];
  __shared__ double red[256];
  const int row = blockIdx.x / ncand, c = blockIdx.x % ncand;
  const double s = cand[(size_t)row * ncand + c];
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const double wi = w[(size_t)row * k + i];
    const double q = (double)__half2float(__double2half(wi / s));
    double d = q * s - wi;
    if (!isfinite(d)) d = 1e30;  // np.where(np.isfinite(dw), dw, 1e30)
    dw[i] = d;
  }
  __syncthreads();
  double acc = 0.0;
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const double *g = gram + (size_t)i * k;
    double gi = 0.0;
    for (int j = 0; j < k; ++j) gi = fma(g[j], dw[j], gi);
    acc = fma(dw[i], gi, acc);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) err[blockIdx.x] = red[0];
}

}  // namespace fcg

extern "C" int fcg_calib_errors(const double *w, int rows, int k, const double *cand, int ncand,
                                const double *gram, double *err, void *stream) {
  if (rows < 0 || k < 1 || k > fcg::CAL_MAXK || ncand < 1) {
    fcg::set_error("calib_errors: bad shape (1 <= k <= 256, ncand >= 1)");
    return FCG_ERR_ARG;
  }
  if (rows == 0) return FCG_OK;
  fcg::k_calib_errors<<<rows * ncand, 256, 0, (cudaStream_t)stream>>>(w, k, cand, ncand, gram,
                                                                      err);
  return fcg::cuda_status("calib_errors");
}
