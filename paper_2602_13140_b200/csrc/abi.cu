// extern "C" entry points of libfcg.so (declared in include/fcg.h).
#include <stdlib.h>

#include <string>

#include "common.cuh"

namespace fcg {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int cuda_status(const char *where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(where) + ": " + cudaGetErrorString(e));
    return FCG_ERR_CUDA;
  }
  return FCG_OK;
}

// FCG_PDL: bitmask of launch sites using PDL (PdlSite); default all, 0 = off.
bool pdl_enabled(int site) {
  static const unsigned mask = [] {
    const char *v = getenv("FCG_PDL");
    return v ? (unsigned)strtoul(v, nullptr, 0) : ~0u;
  }();
  return (mask >> site) & 1u;
}

// ---- profiler ----------------------------------------------------------
bool g_prof_on = false;
unsigned long long *g_dbg_phase = nullptr;
static const char *kProfNames[P_COUNT] = {
    "nbr_count", "nbr_scan", "nbr_fill", "nbr_rev", "embed", "node_pre", "edge_fwd",
    "node_post", "readout", "node_post_bwd", "edge_bwd", "node_pre_bwd", "forces_finish",
    "noise", "baoa", "prior", "step_advance", "edge_geom"};
constexpr int kProfMax = 8192;
struct ProfClass {
  cudaEvent_t ev[2 * kProfMax];
  int n = 0;
  bool made = false;
};
static ProfClass g_prof[P_COUNT];

void prof_mark(int id, bool begin, cudaStream_t s) {
  ProfClass &c = g_prof[id];
  if (!c.made) {
    for (int i = 0; i < 2 * kProfMax; ++i) cudaEventCreate(&c.ev[i]);
    c.made = true;
  }
  if (c.n >= kProfMax) return;
  cudaEventRecord(c.ev[2 * c.n + (begin ? 0 : 1)], s);
  if (!begin) c.n++;
}

static size_t md_extra_bytes(int R, int N) {
  Carver c(nullptr, 0);
  c.take<char>(noise_ring_bytes(R, N));  // noise ring + tag
  c.take<float>((size_t)R * N * 3);  // prior forces
  c.take<float>((size_t)R * N);      // per-atom energies
  return c.off + 256;
}

}  // namespace fcg

using namespace fcg;

extern "C" {

int fcg_abi_version(void) { return FCG_ABI_VERSION; }

const char *fcg_last_error(void) { return g_last_error.c_str(); }

int fcg_profile_enable(int on) {
  cudaDeviceSynchronize();
  for (auto &c : g_prof) c.n = 0;
  g_prof_on = on != 0;
  return cuda_status("profile_enable");
}

int fcg_profile_read(int max_classes, char *names, double *total_ms, int *launches) {
  if (cudaDeviceSynchronize() != cudaSuccess) return cuda_status("profile_read");
  int k = 0;
  for (int id = 0; id < P_COUNT && k < max_classes; ++id) {
    ProfClass &c = g_prof[id];
    if (!c.n) continue;
    double tot = 0;
    for (int i = 0; i < c.n; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c.ev[2 * i], c.ev[2 * i + 1]);
      tot += ms;
    }
    snprintf(names + 32 * k, 32, "%s", kProfNames[id]);
    total_ms[k] = tot;
    launches[k] = c.n;
    ++k;
  }
  return k;
}

int fcg_debug_phase_buffer(void *dev_ptr) {
  g_dbg_phase = (unsigned long long *)dev_ptr;
  return FCG_OK;
}

size_t fcg_nbr_workspace_bytes(int R, int N) { return nbr_ws_bytes(R, N); }

int fcg_nbr_build(const float *pos, int R, int N, double r_cut, int64_t cap_e, int32_t *ptr,
                  int32_t *nbr, int32_t *rev, int32_t *own, int64_t *status, void *ws,
                  size_t ws_bytes, void *stream) {
  return nbr_build(pos, R, N, r_cut, cap_e, ptr, nbr, rev, own, status, ws, ws_bytes,
                   (cudaStream_t)stream);
}

int fcg_nbr_build_f64(const double *pos, int R, int N, double r_cut, int64_t cap_e, int32_t *ptr,
                      int32_t *nbr, int32_t *rev, int32_t *own, int64_t *status, void *ws,
                      size_t ws_bytes, void *stream) {
  return nbr_build_f64(pos, R, N, r_cut, cap_e, ptr, nbr, rev, own, status, ws, ws_bytes,
                       (cudaStream_t)stream);
}

size_t fcg_group_workspace_bytes(int64_t E, int n) { return group_ws_bytes(E, n); }

int fcg_group_by(const int64_t *key, int64_t E, int n, int64_t *ptr, int64_t *perm, void *ws,
                 size_t ws_bytes, void *stream) {
  return group_by(key, E, n, ptr, perm, ws, ws_bytes, (cudaStream_t)stream);
}

size_t fcg_segment_reduce_workspace_bytes(int64_t E, int k, int nseg) {
  return segment_reduce_ws_bytes(E, k, nseg, sizeof(double));
}

int fcg_segment_reduce(const float *values, int64_t E, int k, const int64_t *ptr, int nseg,
                       float *out, void *ws, size_t ws_bytes, void *stream) {
  return segment_reduce(values, E, k, ptr, nseg, out, ws, ws_bytes, (cudaStream_t)stream);
}

int fcg_segment_reduce_f64(const double *values, int64_t E, int k, const int64_t *ptr, int nseg,
                           double *out, void *ws, size_t ws_bytes, void *stream) {
  return segment_reduce_f64(values, E, k, ptr, nseg, out, ws, ws_bytes, (cudaStream_t)stream);
}

size_t fcg_ef_workspace_bytes(const fcg_model *m, int R, int N, int64_t cap_e) {
  return ef_ws_bytes(m, R, N, cap_e);
}

int fcg_energy_forces(const fcg_model *m, const float *pos, const int32_t *types, int R, int N,
                      const int32_t *ptr, const int32_t *nbr, const int32_t *rev,
                      const int32_t *own, int64_t cap_e, float *per_atom, float *energy,
                      float *forces, void *ws, size_t ws_bytes, void *stream) {
  return energy_forces(m, pos, types, R, N, ptr, nbr, rev, own, cap_e, per_atom, energy, forces,
                       ws, ws_bytes, (cudaStream_t)stream, nullptr, nullptr, nullptr, nullptr,
                       nullptr, nullptr);
}

int fcg_energy_forces_sched(const fcg_model *m, const float *pos, const int32_t *types, int R,
                            int N, const int32_t *ptr, const int32_t *nbr, const int32_t *rev,
                            const int32_t *own, int64_t cap_e, float *per_atom, float *energy,
                            float *forces, void *ws, size_t ws_bytes, int schedule,
                            void *stream) {
  return energy_forces(m, pos, types, R, N, ptr, nbr, rev, own, cap_e, per_atom, energy, forces,
                       ws, ws_bytes, (cudaStream_t)stream, nullptr, nullptr, nullptr, nullptr,
                       nullptr, nullptr, schedule);
}

int fcg_normal_noise(uint64_t seed, int rep_offset, const int64_t *step, int R, int N, float *out,
                     void *stream) {
  return normal_noise(seed, rep_offset, step, R, N, out, (cudaStream_t)stream);
}

int fcg_langevin_baoa(const fcg_md_params *p, const float *mass, int R, int N,
                      const float *forces, const float *noise, float *pos, float *vel,
                      void *stream) {
  return langevin_baoa(p, mass, R, N, forces, noise, pos, vel, (cudaStream_t)stream);
}

int fcg_half_kick(const fcg_md_params *p, const float *mass, int R, int N, const float *forces,
                  float *vel, void *stream) {
  return half_kick(p, mass, R, N, forces, vel, (cudaStream_t)stream);
}

int fcg_prior_forces(const fcg_prior *pr, const float *pos, int R, int N, float *e_prior,
                     float *f_prior, void *stream) {
  return prior_forces(pr, pos, R, N, e_prior, f_prior, (cudaStream_t)stream);
}

size_t fcg_md_workspace_bytes(const fcg_model *m, int R, int N, int64_t cap_e) {
  return nbr_ws_bytes(R, N) + ef_ws_bytes(m, R, N, cap_e) + md_extra_bytes(R, N) + 1024;
}

int fcg_md_step(const fcg_model *m, const fcg_prior *pr, const fcg_md_params *p,
                const float *mass, const int32_t *types, int R, int N, double r_cut,
                int64_t cap_e, int64_t *step, float *pos, float *vel, float *forces,
                float *potential, float *prior, int32_t *ptr, int32_t *nbr, int32_t *rev,
                int32_t *own, int64_t *status, void *ws, size_t ws_bytes, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (ws_bytes < fcg_md_workspace_bytes(m, R, N, cap_e)) {
    set_error("md_step: workspace too small");
    return FCG_ERR_ARG;
  }
  char *w = (char *)ws;
  size_t nb = nbr_ws_bytes(R, N), eb = ef_ws_bytes(m, R, N, cap_e);
  void *ws_nbr = w;
  void *ws_ef = w + ((nb + 255) & ~size_t(255));
  Carver c(w + ((nb + 255) & ~size_t(255)) + ((eb + 255) & ~size_t(255)), md_extra_bytes(R, N));
  void *ring = c.take<char>(noise_ring_bytes(R, N));
  float *fprior = c.take<float>((size_t)R * N * 3);
  float *per_atom = c.take<float>((size_t)R * N);

  int rc;
  // leading B + A + O + A with the forces of the current state (md.py:200-202)
  if ((rc = langevin_leading(p, mass, R, N, forces, step, pos, vel, ring, status, s))) return rc;
  // force evaluation at the new positions (md.py:203, _ReplicaForces)
  // (the fused assembly for N <= 512 is launched by the force evaluation,
  // together with the edge geometry)
  NbrDefer defer{};
  if ((rc = nbr_build(pos, R, N, r_cut, cap_e, ptr, nbr, rev, own, status, ws_nbr, nb, s, step,
                      p->neighbor_stride, &defer)))
    return rc;
  (void)fprior;
  // model forces + prior (evaluated inline by the force assembly, which also
  // sums the prior energies), blow-up check and the trailing half-kick
  // (md.py:204-205)
  return energy_forces(m, pos, types, R, N, ptr, nbr, rev, own, cap_e, per_atom, potential,
                       forces, ws_ef, eb, s, nullptr, p, mass, vel, status, step, p->schedule,
                       pr, prior, &defer);
}

int fcg_memcpy_async(void *dst, const void *src, size_t bytes, void *stream) {
  if (bytes == 0) return FCG_OK;
  if (!dst || !src) {
    set_error("memcpy_async: null pointer");
    return FCG_ERR_ARG;
  }
  cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream);
  return cuda_status("memcpy_async");
}

}  // extern "C"
