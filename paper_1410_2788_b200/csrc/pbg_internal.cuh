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

}  // namespace pbg
