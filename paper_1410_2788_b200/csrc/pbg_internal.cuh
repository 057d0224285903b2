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

// ---------------------------------------------------------------------------------------
// Table-driven flow for the sweep kernels (tables staged in shared memory per block):
//   exp:  w = (64 e + j) ln2/64 + r, |r| <= ln2/128, E = 2^e * T[j] * (1 + expm1_5(r))
//   log:  x = 2^e m, m = c_i (1 + t) with c_i = 1/invc_i the centre of the i-th of 128
//         mantissa bins, |t| <= 2^-8, log x = e ln2 - log(invc_i) + log1p_6(t)
// log(N/D) = log N - log D: no division, absolute error ~3e-16 independent of w.
constexpr int kExpTab = 64, kLogTab = 128;
constexpr int kFlowTabDoubles = kExpTab + 2 * kLogTab;  // T[64] | (invc, -log invc)[128]

static __constant__ double kFlowTabC[8] = {
    92.332482616893656768,             // 64/ln2
    6.93147180369123816490e-01 / 64.0,  // ln2/64, Cody-Waite high part (exact k*hi)
    1.90821492927058770002e-10 / 64.0,  // ln2/64, low part
    1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0,
    6.93147180369123816490e-01, 1.90821492927058770002e-10};

__device__ __forceinline__ double exp_tab(double w, const double* T) {
  const double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  const double t = fma(w, kFlowTabC[0], kMagic);
  const double kd = t - kMagic;
  const int kk = __double2loint(t);
  double r = fma(-kd, kFlowTabC[1], w);
  r = fma(-kd, kFlowTabC[2], r);
  double q = fma(r, kFlowTabC[3], kFlowTabC[4]);
  q = fma(q, r, kFlowTabC[5]);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = q * r;  // expm1(r)
  const double Tj = T[kk & (kExpTab - 1)];
  const double E = fma(Tj, q, Tj);
  return __hiloint2double(__double2hiint(E) + ((kk >> 6) << 20), __double2loint(E));
}

// log of the mantissa of a positive normal x; adds the unbiased exponent to e.
__device__ __forceinline__ double log_mant(double x, int& e, const double2* LT) {
  const int hx = __double2hiint(x);
  e += (hx >> 20) - 1023;
  const double m = __hiloint2double((hx & 0x000FFFFF) | 0x3FF00000, __double2loint(x));
  const double2 c = LT[(hx >> 13) & (kLogTab - 1)];
  const double t = fma(m, c.x, -1.0);
  double p = fma(t, -1.0 / 6.0, 0.2);
  p = fma(p, t, -0.25);
  p = fma(p, t, 1.0 / 3.0);
  p = fma(p, t, -0.5);
  return c.y + fma(t * p, t, t);
}

__device__ __forceinline__ double sinh_flow_tab(double w, double d, double sat, double pm,
                                                const double* FT) {
  double out;
  if (d >= 1.0 || !(fabs(w) <= 38.0)) {  // rare: identity palette, saturation, NaN
    out = (d >= 1.0 || w != w) ? w : copysign(sat, w);
  } else {
    const double E = exp_tab(w, FT);
    const double opd = 1.0 + d, omd = 1.0 - d;
    int en = 0, ed = 0;
    const double2* LT = reinterpret_cast<const double2*>(FT + kExpTab);
    const double ln = log_mant(fma(opd, E, omd), en, LT);
    const double ld = log_mant(fma(omd, E, opd), ed, LT);
    const double kd = (double)(en - ed);
    out = fma(kd, kFlowTabC[6], fma(kd, kFlowTabC[7], ln - ld));
  }
  return pm != 1.0 ? pm * out : out;
}

}  // namespace pbg
