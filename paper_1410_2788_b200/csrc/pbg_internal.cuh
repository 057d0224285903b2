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

// Polynomial coefficients live in constant memory: as c[][] operands of DFMA they cost
// nothing extra, while 64-bit literals would each need two uniform moves per use.
static __constant__ double kExpPoly[13] = {
    2.08767569878680989792e-09, 2.50521083854417187751e-08, 2.75573192239858906526e-07,
    2.75573192239858906526e-06, 2.48015873015873015873e-05, 1.98412698412698412698e-04,
    1.38888888888888888889e-03, 8.33333333333333333333e-03, 4.16666666666666666667e-02,
    1.66666666666666666667e-01, 0.5, 1.0, 1.0};
// 1/19, 1/17, ..., 1/3, then ln2 split (hi, lo) and 1/ln2, sqrt2.
static __constant__ double kLogPoly[13] = {
    1.0 / 19.0, 1.0 / 17.0, 1.0 / 15.0, 1.0 / 13.0, 1.0 / 11.0, 1.0 / 9.0, 1.0 / 7.0,
    1.0 / 5.0,  1.0 / 3.0,  6.93147180369123816490e-01, 1.90821492927058770002e-10,
    1.4426950408889634, 1.41421356237309504880};

// exp(w) for |w| <= 40: Cody-Waite reduction by ln 2 (k by the 1.5*2^52 rounding trick, no
// conversion instructions), degree-12 Taylor polynomial on |r| <= ln2/2 (truncation < 2e-16
// relative), exponent added directly (no range checks).
__device__ __forceinline__ double exp_small(double w) {
  const double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  const double t = fma(w, kLogPoly[11], kMagic);
  const double k = t - kMagic;
  const int ki = __double2loint(t);  // k (two's complement in the low word)
  double r = fma(-k, kLogPoly[9], w);
  r = fma(-k, kLogPoly[10], r);
  double p = kExpPoly[0];
#pragma unroll
  for (int q = 1; q < 13; ++q) p = fma(p, r, kExpPoly[q]);
  return __hiloint2double(__double2hiint(p) + (ki << 20), __double2loint(p));
}

// log(N / D) for positive normal N, D with one division: N = 2^eN mN, D = 2^eD mD,
// mN/mD reduced into [1/sqrt2, sqrt2] (selects, no branches), log m = 2 atanh(s),
// s = (mN - mD)/(mN + mD), |s| <= 0.1716, odd series to s^19 (truncation < 3e-17 relative).
__device__ __forceinline__ double log_ratio(double N, double D) {
  const int hn = __double2hiint(N), hd = __double2hiint(D);
  int k = (hn >> 20) - (hd >> 20);
  double mn = __hiloint2double((hn & 0x000FFFFF) | 0x3FF00000, __double2loint(N));
  double md = __hiloint2double((hd & 0x000FFFFF) | 0x3FF00000, __double2loint(D));
  const bool up = mn > kLogPoly[12] * md;
  const bool dn = md > kLogPoly[12] * mn;
  md = up ? md + md : md;
  mn = dn ? mn + mn : mn;
  k += (int)up - (int)dn;
  const double den = mn + md;
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(den));
  double e = fma(-den, y, 1.0);
  y = fma(y, e, y);
  e = fma(-den, y, 1.0);
  y = fma(y, e, y);
  const double sn = (mn - md) * y;
  const double s2 = sn * sn;
  double p = kLogPoly[0];
#pragma unroll
  for (int q = 1; q < 9; ++q) p = fma(p, s2, kLogPoly[q]);
  const double lm = 2.0 * fma(p * s2, sn, sn);
  const double kd = (double)k;
  return fma(kd, kLogPoly[9], fma(kd, kLogPoly[10], lm));
}

// Same map as sinh_flow, evaluated as log(((1+d)E + (1-d)) / ((1-d)E + (1+d))), E = exp(w),
// with the reduced-range exp/log above.  For |w| > 38, tanh(w/2) rounds to +-1 in fp64 and
// the reference returns +-2*atanh(d) (`sat`, precomputed on the host); decay >= 1 and NaN
// pass w through.  Agrees with sinh_flow to ~1e-16 absolute.
__device__ __forceinline__ double sinh_flow_fast(double w, double d, double sat, double pm) {
  double out;
  if (d >= 1.0 || !(fabs(w) <= 38.0)) {  // rare: identity palette, saturation, NaN
    out = (d >= 1.0 || w != w) ? w : copysign(sat, w);
  } else {
    const double E = exp_small(w);
    const double opd = 1.0 + d, omd = 1.0 - d;
    out = log_ratio(fma(opd, E, omd), fma(omd, E, opd));
  }
  return pm != 1.0 ? pm * out : out;
}

}  // namespace pbg
