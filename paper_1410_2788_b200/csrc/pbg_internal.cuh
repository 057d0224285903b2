// Internal helpers shared by the pbg CUDA translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>

#include "pbg.h"

namespace pbg {

constexpr int kOff = PBG_OFFSET;

// Pitched field layout (see include/pbg.h).  Element (i, j, k) at i*s0 + j*pitch + k + kOff.
struct Layout {
  int n0, n1, n2;
  long long pitch;
  long long s0;
  // Batched marches (config 5): nb grids of this shape, bs elements apart in every buffer
  // (nb = 1, bs = 0 for one grid).  at() addresses grid 0; kernels add b * bs.
  int nb;
  long long bs;
  __host__ __device__ __forceinline__ long long at(int i, int j, int k) const {
    return (long long)i * s0 + (long long)j * pitch + k + kOff;
  }
};

// The march's per-axis scratch comes from cudaMallocAsync on the device's default pool,
// whose release threshold is 0: every stream synchronisation would hand the pool's memory
// back to the driver and the next march would map it again (measured as host-side cost of
// concurrent config-5 marches).  Keep it cached, once per device.
inline void keep_pool_memory() {
  static std::once_flag flags[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::call_once(flags[dev], [dev] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

inline Layout make_layout(const pbg_grid* g) {
  Layout L;
  L.n0 = g->n[0];
  L.n1 = g->n[1];
  L.n2 = g->n[2];
  L.pitch = g->pitch;
  L.s0 = (long long)g->n[1] * g->pitch;
  L.nb = 1;
  L.bs = 0;
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

// Piecewise-polynomial sinh flow for the sweep kernels: F(x) = 2 artanh(d tanh(x/2)) on
// x = |w| in [0, 38], cut at x + 1 = 2^e (1 + s/16), e = 0..5, s = 0..15 (84 intervals,
// finer where F bends), each interval a degree-9 polynomial in t = x - c about its centre c
// (Chebyshev interpolation at 10 nodes, built on the host in extended precision per decay,
// sweep.cu build_flow_poly).  Interval layout: 12 doubles [c, a0, ..., a9, 0].  Absolute
// error <= ~4e-16 for 0 < d <= 0.99 (the reference's own tanh/atanh evaluation carries
// 4e-16 .. 1e-14 there): one index computation, 10 fp64 operations, 6 shared-memory loads.
constexpr int kFPolyIv = 84, kFPolyStride = 12, kFPolyDoubles = kFPolyIv * kFPolyStride;

__device__ __forceinline__ double flow_poly(double x, const double* P) {
  const int idx = (__double2hiint(x + 1.0) >> 16) - 0x3FF0;  // exponent * 16 + top 4 bits
  const double2* Q = reinterpret_cast<const double2*>(P + idx * kFPolyStride);
  const double2 q0 = Q[0], q1 = Q[1], q2 = Q[2], q3 = Q[3], q4 = Q[4], q5 = Q[5];
  const double t = x - q0.x;
  double p = fma(q5.x, t, q4.y);
  p = fma(p, t, q4.x);
  p = fma(p, t, q3.y);
  p = fma(p, t, q3.x);
  p = fma(p, t, q2.y);
  p = fma(p, t, q2.x);
  p = fma(p, t, q1.y);
  p = fma(p, t, q1.x);
  return fma(p, t, q0.y);
}

// Small-argument flow: for |w| <= kFSmallX, F(w) = w * G(w^2) with G analytic in y = w^2
// (nearest singularity at y = -pi^2), so one degree-15 polynomial in t = y - kFSmallX^2 / 2
// (Chebyshev interpolation on y in [0, kFSmallX^2], built per decay on the host in extended
// precision, sweep.cu build_flow_small) gives F to ~1 ulp relative.  Its 16 coefficients are
// kernel parameters (constant-bank operands, the same for every lane): no table loads, so the
// solvent far field -- most of the grid -- costs 17 fp64 operations and no shared memory.
constexpr int kFSmallN = 16;
constexpr double kFSmallX = 2.0;

__host__ __device__ __forceinline__ double flow_small(double w, const double* g) {
  const double t = fma(w, w, -0.5 * kFSmallX * kFSmallX);
  double p = g[kFSmallN - 1];
#pragma unroll
  for (int q = kFSmallN - 2; q >= 0; --q) p = fma(p, t, g[q]);
  return w * p;
}

// Tiny-argument tier: |w| <= kFTinyX (~93% of all nodes in the protein configs), the same
// construction on y in [0, kFTinyX^2] needs only degree 7 (8 coefficients, 10 fp64 operations;
// B200 issues 64 DFMA per SM-clock, so the flow's fp64 work bounds the LODIE2 epilogue).
constexpr int kFTinyN = 8;
constexpr double kFTinyX = 0.5;

__host__ __device__ __forceinline__ double flow_tiny(double w, const double* g) {
  const double t = fma(w, w, -0.5 * kFTinyX * kFTinyX);
  double p = g[kFTinyN - 1];
#pragma unroll
  for (int q = kFTinyN - 2; q >= 0; --q) p = fma(p, t, g[q]);
  return w * p;
}

// pm * flow(w) with the interval table P of decay d: d >= 1 passes w through, |w| > 38
// (tanh(w/2) rounds to +-1 in the reference) gives +-sat = +-2 atanh(d), NaN propagates.
__device__ __forceinline__ double sinh_flow_poly(double w, double d, double sat, double pm,
                                                 const double* P) {
  double out;
  const double x = fabs(w);
  if (d >= 1.0 || !(x <= 38.0)) {  // rare: identity palette, saturation, NaN
    out = (d >= 1.0 || w != w) ? w : copysign(sat, w);
  } else {
    out = copysign(flow_poly(x, P), w);
  }
  return pm != 1.0 ? pm * out : out;
}

}  // namespace pbg
