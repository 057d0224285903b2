// Internal helpers shared by the pbg CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "pbg.h"

namespace pbg {

constexpr int kOff = PBG_OFFSET;

// Pitched field layout (see include/pbg.h).  Element (i, j, k) at i*s0 + j*pitch + k + kOff.
struct Layout {
  int n0, n1, n2;
  long long pitch;
  long long s0;
  __host__ __device__ __forceinline__ long long at(int i, int j, int k) const {
    return (long long)i * s0 + (long long)j * pitch + k + kOff;
  }
};

inline Layout make_layout(const pbg_grid* g) {
  Layout L;
  L.n0 = g->n[0];
  L.n1 = g->n[1];
  L.n2 = g->n[2];
  L.pitch = g->pitch;
  L.s0 = (long long)g->n[1] * g->pitch;
  return L;
}

// Error plumbing -----------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_cuda(cudaError_t e, const char* what);
int validate_grid(const pbg_grid* g);

#define PBG_CUDA(call)                                 \
  do {                                                 \
    int _rc = ::pbg::check_cuda((call), #call);        \
    if (_rc != PBG_OK) return _rc;                     \
  } while (0)

#define PBG_LAUNCH_CHECK(what)                                    \
  do {                                                            \
    int _rc = ::pbg::check_cuda(cudaGetLastError(), what);        \
    if (_rc != PBG_OK) return _rc;                                \
  } while (0)

// NaN-propagating clip (np.clip semantics, schemes.py:96).
__device__ __forceinline__ double clip_nan(double t, double c) {
  return t > c ? c : (t < -c ? -c : t);
}

// _apply_flow (schemes.py:88-103): pm * (decay >= 1 ? w : 2*artanh(clip(decay*tanh(w/2)))).
__device__ __forceinline__ double sinh_flow(double w, double decay, double pm) {
  const double kClip = __longlong_as_double(0x3FEFFFFFFFFFFFFFLL);  // nextafter(1, 0)
  double out;
  if (decay >= 1.0) {
    out = w;
  } else {
    double t = __dmul_rn(tanh(__dmul_rn(0.5, w)), decay);
    t = clip_nan(t, kClip);
    out = __dmul_rn(2.0, atanh(t));
  }
  return pm != 1.0 ? __dmul_rn(pm, out) : out;
}

// Same map as sinh_flow, evaluated as log(((1+d)E + (1-d)) / ((1-d)E + (1+d))), E = exp(w):
// one exp, one division and one log instead of tanh + atanh (~2x fewer instructions).  For
// |w| > 38, tanh(w/2) rounds to +-1 in fp64 and the reference returns +-2*atanh(d) (`sat`,
// precomputed on the host).  Agrees with sinh_flow to ~1e-16 absolute.
__device__ __forceinline__ double sinh_flow_fast(double w, double d, double sat, double pm) {
  double out;
  if (d >= 1.0) {
    out = w;
  } else if (fabs(w) > 38.0) {
    out = copysign(sat, w);
  } else {
    const double E = exp(w);
    const double opd = 1.0 + d, omd = 1.0 - d;
    out = log(fma(opd, E, omd) / fma(omd, E, opd));
  }
  return pm != 1.0 ? pm * out : out;
}

}  // namespace pbg
