// (f) Host-side output formatting for run_simulation (md.py:224-228,
// :312-326): trajectory.xyz frames in the reference's exact bytes.
//
// The reference formats every bead with Python f"{x:.9f}" on float32 values,
// i.e. "%.9f" of the value widened to double, which the C library's
// correctly rounded conversion reproduces byte for byte (Python spells
// non-finite values "nan"/"inf"/"-inf" whatever the NaN sign, handled here).
// Formatting 64 replicas x 269 beads in Python takes ~70 ms; this runs
// replicas on worker threads and is called from run_simulation's writer
// thread with the GIL released, so output overlaps the GPU steps.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace fcg {

static inline void put_coord(std::string &s, float v) {
  char b[64];
  const double x = (double)v;
  if (isnan(x)) {
    s += "nan";
  } else if (isinf(x)) {
    s += x > 0 ? "inf" : "-inf";
  } else {
    int n = snprintf(b, sizeof b, "%.9f", x);
    if (n >= (int)sizeof b) {  // |x| >= 1e54: widen
      std::vector<char> big((size_t)n + 1);
      snprintf(big.data(), big.size(), "%.9f", x);
      s.append(big.data(), (size_t)n);
    } else {
      s.append(b, (size_t)n);
    }
  }
}

// One frame: "N\nstep=S replica=R\nB<t> x y z\n..." (md.py:224-228).
static void format_frame(std::string &s, const float *pos, const int32_t *types, int N,
                         long long step, long long replica) {
  char b[64];
  int n = snprintf(b, sizeof b, "%d\nstep=%lld replica=%lld\n", N, step, replica);
  s.append(b, (size_t)n);
  for (int i = 0; i < N; ++i) {
    n = snprintf(b, sizeof b, "B%d ", (int)types[i]);
    s.append(b, (size_t)n);
    put_coord(s, pos[3 * i]);
    s += ' ';
    put_coord(s, pos[3 * i + 1]);
    s += ' ';
    put_coord(s, pos[3 * i + 2]);
    s += '\n';
  }
}

}  // namespace fcg

using namespace fcg;

extern "C" int64_t fcg_format_xyz(const float *pos, const int32_t *types, int R, int N,
                                  int64_t step, int replica0, char *out, int64_t cap,
                                  int nthreads) {
  if (R < 0 || N < 0 || (!pos && R * N) || (!types && N)) {
    set_error("format_xyz: bad arguments");
    return -1;
  }
  std::vector<std::string> parts((size_t)R);
  int T = nthreads > 0 ? nthreads : (int)std::thread::hardware_concurrency();
  if (T < 1) T = 1;
  if (T > R) T = R > 0 ? R : 1;
  auto work = [&](int t) {
    for (int r = t; r < R; r += T) {
      parts[(size_t)r].reserve((size_t)N * 48 + 64);
      format_frame(parts[(size_t)r], pos + (size_t)r * N * 3, types, N, (long long)step,
                   (long long)replica0 + r);
    }
  };
  if (T == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back(work, t);
    for (auto &x : th) x.join();
  }
  int64_t total = 0;
  for (auto &p : parts) total += (int64_t)p.size();
  if (!out || cap < total) return -total;
  char *o = out;
  for (auto &p : parts) {
    memcpy(o, p.data(), p.size());
    o += p.size();
  }
  return total;
}
