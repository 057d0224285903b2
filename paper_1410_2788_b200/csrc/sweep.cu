// Implicit line sweeps and the fused LOD/AOS/MAOS time step for sm_100a.
//
// Reference: pbsplit/tridiag.py:120-219 (prefactored batched Thomas), pbsplit/schemes.py:
// 88-103 (sinh flow), 123-143 (delta2_block), 274-329 (Stepper sweeps/steps), 399-425 (march).
//
// Every implicit sweep solves (1 - f*d2_a) x = rhs on all interior lines of axis a, where
// the tridiagonal rows are  sub = -f*e_minus, diag = 1 + f*(e_plus + e_minus),
// sup = -f*e_plus  (tridiag.py:165, 179-181), with the static Dirichlet fold-ins on the
// first/last row (tridiag.py:193-202).  Instead of the reference's single serial Thomas per
// line with stored LU factors (3 x 8 B/node of coefficient traffic per sweep), each line is
// split into P segments of S rows handled by P threads:
//
//   * rows j < S-1 of a segment are "inner"; row S-1 is a separator t_k.  Inner unknowns are
//     x_j = y_j + alpha_j * t_{k-1} + beta_j * t_k (three Thomas solves of the segment block
//     sharing one elimination, coefficients recomputed from the 1-byte node codes);
//   * the separators obey a diagonally dominant tridiagonal "reduced" system, solved by
//     parallel cyclic reduction (warp shuffles for the contiguous axis, shared memory for the
//     strided axes);
//   * inner values are then reconstructed in registers.
//
// The result equals the reference's Thomas solution up to fp64 reassociation (the system is
// strictly diagonally dominant; see DESIGN.md for the measured 1e-15-level agreement).
//
// Strided axes (0 and 1): block = LB adjacent k columns x P segments.  Each warp row reads
// LB consecutive doubles of one grid row (coalesced 64-256 B), no transposition.
// Contiguous axis (2): one warp per line; the row is staged in shared memory with a padded
// (bank-conflict-free) segment layout, lane = segment, PCR via shuffles.
//
// Prologue / epilogue fusions (all per node, in registers):
//   PRO_FLOW  w = pm*flow(u)         LODIE1/LODCN1 first sweep, MAOS branches
//   PRO_SRC   w = u + dta*rho        LODIE2/LODCN2 first sweep
//   CN        rhs += (cn_f/h^2)*delta2(w) along the sweep axis
//   extra     rhs += coef*dta*rho    AOS/MAOS branch source
//   EPI_*     LODIE1 source, LODIE2 flow, AOS/MAOS accumulate/combine, divergence flag.

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <vector>

#include "pbg_internal.cuh"

namespace pbg {

enum { PRO_NONE = 0, PRO_FLOW = 1, PRO_SRC = 2 };
enum {
  EPI_STORE = 0,
  EPI_SRC = 1,
  EPI_FLOW = 2,
  EPI_AOS0 = 3,
  EPI_AOS1 = 4,
  EPI_AOS2 = 5,
  EPI_MAOS0 = 6,
  EPI_MAOS1 = 7,
  EPI_MAOS2 = 8
};

struct AxisCoef {
  double diag[4];  // [em*2 + ep]  1 + f*(e_plus + e_minus)
  double sub[2];   // [em]         -f*e_minus
  double sup[2];   // [ep]         -f*e_plus
  double flo[2];   // [em]         f*e_minus   (low fold, times the face value)
  double fhi[2];   // [ep]         f*e_plus    (high fold)
  double eps[2];   // palette (CN stencil)
};

struct SweepArgs {
  Layout L;
  int m;  // interior nodes along the sweep axis
  const double* src;
  const double* bnd;
  const uint8_t* codes;
  const double* rho;
  double* dst;
  const double* acc;
  AxisCoef co;
  int cn;
  double cnc;  // cn_f / h^2
  int pro;
  double pro_coef;
  int has_extra;
  double extra;
  double decay0, decay1;  // flow decay for solute-bit 0 / 1
  double pm;
  int epi;
  double epi_coef;
  int* div_step;
  int step;
  double thr;
  int check;
};

__device__ __forceinline__ double pro_val(const SweepArgs& a, double v, uint32_t c,
                                          long long off) {
  if (a.pro == PRO_FLOW) return sinh_flow(v, (c & 1u) ? a.decay1 : a.decay0, a.pm);
  if (a.pro == PRO_SRC && (c & 16u)) return __dadd_rn(v, __dmul_rn(a.pro_coef, a.rho[off]));
  return v;
}

// Face value seen by the CN stencil: after a flow stage the reference re-applies the
// boundary (schemes.py:280-283), otherwise the running field's own faces are read.
__device__ __forceinline__ double face_val(const SweepArgs& a, long long off) {
  return a.pro == PRO_FLOW ? a.bnd[off] : a.src[off];
}

__device__ __forceinline__ void row_coefs(const AxisCoef& co, int i, int m, uint32_t em,
                                          uint32_t ep, double& av, double& bv, double& cv) {
  if (i >= m) {  // padding rows: identity, decoupled
    av = 0.0;
    bv = 1.0;
    cv = 0.0;
    return;
  }
  av = (i == 0) ? 0.0 : (em ? co.sub[1] : co.sub[0]);
  cv = (i == m - 1) ? 0.0 : (ep ? co.sup[1] : co.sup[0]);
  bv = em ? (ep ? co.diag[3] : co.diag[2]) : (ep ? co.diag[1] : co.diag[0]);
}

// rhs of row i from the stage field w (wm, wc, wp = w at rows i-1, i, i+1).
__device__ __forceinline__ double row_rhs(const SweepArgs& a, int i, uint32_t c, uint32_t em,
                                          uint32_t ep, double wm, double wc, double wp,
                                          long long off, double blo, double bhi) {
  double r = wc;
  if (a.cn) {
    const double epv = ep ? a.co.eps[1] : a.co.eps[0];
    const double emv = em ? a.co.eps[1] : a.co.eps[0];
    const double d2 =
        __dadd_rn(__dmul_rn(epv, __dsub_rn(wp, wc)), __dmul_rn(emv, __dsub_rn(wm, wc)));
    r = __dadd_rn(r, __dmul_rn(a.cnc, d2));
  }
  if (a.has_extra && (c & 16u)) r = __dadd_rn(r, __dmul_rn(a.extra, a.rho[off]));
  if (i == 0) r = __dadd_rn(r, __dmul_rn(em ? a.co.flo[1] : a.co.flo[0], blo));
  if (i == a.m - 1) r = __dadd_rn(r, __dmul_rn(ep ? a.co.fhi[1] : a.co.fhi[0], bhi));
  return r;
}

// Epilogue for the final value x at a node (AOS0's flow(u) term is added by the caller).
__device__ __forceinline__ double epi_val(const SweepArgs& a, double x, uint32_t c,
                                          long long off) {
  switch (a.epi) {
    case EPI_SRC:
      return (c & 16u) ? __dadd_rn(x, __dmul_rn(a.epi_coef, a.rho[off])) : x;
    case EPI_FLOW:
      return sinh_flow(x, (c & 1u) ? a.decay1 : a.decay0, 1.0);
    case EPI_AOS1:
    case EPI_MAOS1:
      return __dadd_rn(a.acc[off], x);
    case EPI_AOS2:
      return __dmul_rn(0.25, __dadd_rn(a.acc[off], x));
    case EPI_MAOS2:
      return __ddiv_rn(__dadd_rn(a.acc[off], x), 3.0);
    default:
      return x;
  }
}

__device__ __forceinline__ bool is_bad(double v, double thr) {
  return !isfinite(v) || fabs(v) > thr;
}

// Segment elimination.  On entry r[j] = rhs of row i0+j, cd[j] = code of node of row i0+j
// (cd[S] = code of the following node).  On exit, for inner rows j < S-1:
//   r[j] = y_j, da[j] = alpha_j, cb[j] = beta_j;  separator coefficients in as/bs/cs.
template <int S>
__device__ __forceinline__ void seg_solve(double (&r)[S], double (&cb)[S], double (&da)[S],
                                          const uint32_t (&cd)[S + 1], int i0, int m, int sh,
                                          const AxisCoef& co, double& as, double& bs,
                                          double& cs) {
  double cpp = 0.0, dyp = 0.0, dap = 1.0, lastinv = 0.0, lastc = 0.0;
#pragma unroll
  for (int j = 0; j < S - 1; ++j) {
    const uint32_t em = (cd[j] >> sh) & 1u, ep = (cd[j + 1] >> sh) & 1u;
    double av, bv, cv;
    row_coefs(co, i0 + j, m, em, ep, av, bv, cv);
    const double inv = __drcp_rn(fma(-av, cpp, bv));
    const double cpj = cv * inv;
    const double dy = fma(-av, dyp, r[j]) * inv;
    const double dA = -(av * dap) * inv;
    r[j] = dy;
    da[j] = dA;
    cb[j] = cpj;
    cpp = cpj;
    dyp = dy;
    dap = dA;
    lastinv = inv;
    lastc = cv;
  }
  double be = -lastc * lastinv;
  double y = r[S - 2], al = da[S - 2];
  cb[S - 2] = be;
#pragma unroll
  for (int j = S - 3; j >= 0; --j) {
    const double c = cb[j];
    y = fma(-c, y, r[j]);
    al = fma(-c, al, da[j]);
    be = -c * be;
    r[j] = y;
    da[j] = al;
    cb[j] = be;
  }
  const uint32_t em = (cd[S - 1] >> sh) & 1u, ep = (cd[S] >> sh) & 1u;
  row_coefs(co, i0 + S - 1, m, em, ep, as, bs, cs);
}

// ---------------------------------------------------------------------------------------
// Strided axes (0, 1).  blockDim = (LB, P); block (x = k group, y = outer interior index).
template <int S>
__global__ void __launch_bounds__(512) k_sweep_strided(const SweepArgs a, const int axis) {
  extern __shared__ double sm[];
  if (a.div_step && *((volatile int*)a.div_step) < a.step) return;
  const int LB = blockDim.x, P = blockDim.y;
  const int lane = threadIdx.x, seg = threadIdx.y;
  const int tid = seg * LB + lane, NT = LB * P;
  const Layout& L = a.L;
  const int m = a.m;
  const int kcol = 1 + blockIdx.x * LB + lane;
  const int outer = 1 + blockIdx.y;
  const bool active = kcol <= L.n2 - 2;
  long long base, stride;
  if (axis == 0) {
    base = L.at(0, outer, kcol);
    stride = L.s0;
  } else {
    base = L.at(outer, 0, kcol);
    stride = L.pitch;
  }
  const int sh = 1 + axis;
  const int i0 = seg * S;

  double r[S], cb[S], da[S];
  uint32_t cd[S + 1];
#pragma unroll
  for (int j = 0; j <= S; ++j) {
    const int i = i0 + j;
    cd[j] = (active && i <= m) ? (uint32_t)a.codes[base + (long long)(i + 1) * stride] : 0u;
  }
#pragma unroll
  for (int j = 0; j < S; ++j) {
    const int i = i0 + j;
    r[j] = (active && i < m) ? a.src[base + (long long)(i + 1) * stride] : 0.0;
  }
  double blo = 0.0, bhi = 0.0;
  if (active && i0 == 0) blo = a.bnd[base];
  if (active && i0 <= m - 1 && m - 1 < i0 + S) bhi = a.bnd[base + (long long)(m + 1) * stride];

  // stage field w (prologue) for own rows; rows == m hold the far face (CN neighbour)
#pragma unroll
  for (int j = 0; j < S; ++j) {
    const int i = i0 + j;
    const long long off = base + (long long)(i + 1) * stride;
    if (!active || i > m) {
      r[j] = 0.0;
    } else if (i == m) {
      r[j] = a.cn ? face_val(a, off) : 0.0;
    } else {
      r[j] = pro_val(a, r[j], cd[j], off);
    }
  }
  double wprev = 0.0, wnext = 0.0;
  if (a.cn && active) {
    if (i0 == 0) {
      wprev = face_val(a, base);
    } else if (i0 - 1 < m) {
      const long long off = base + (long long)i0 * stride;
      wprev = pro_val(a, a.src[off], a.codes[off], off);
    }
    const int inx = i0 + S;
    const long long off = base + (long long)(inx + 1) * stride;
    if (inx < m) {
      wnext = pro_val(a, a.src[off], a.codes[off], off);
    } else if (inx == m) {
      wnext = face_val(a, off);
    }
  }
  // rhs (in place, keeping the previous stage value for the stencil)
  {
    double wm = wprev;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const int i = i0 + j;
      const double wc = r[j];
      const double wp = (j + 1 < S) ? r[j + 1] : wnext;
      if (active && i < m) {
        const uint32_t sh2 = (uint32_t)sh;
        const uint32_t em = (cd[j] >> sh2) & 1u, ep = (cd[j + 1] >> sh2) & 1u;
        r[j] = row_rhs(a, i, cd[j], em, ep, wm, wc, wp, base + (long long)(i + 1) * stride,
                       blo, bhi);
      } else {
        r[j] = 0.0;
      }
      wm = wc;
    }
  }

  double as, bs, cs;
  seg_solve<S>(r, cb, da, cd, i0, m, sh, a.co, as, bs, cs);
  const double rs = r[S - 1];

  double* sA = sm;
  double* sB = sm + NT;
  double* sC = sm + 2 * NT;
  double* sR = sm + 3 * NT;
  sA[tid] = r[0];
  sB[tid] = da[0];
  sC[tid] = cb[0];
  __syncthreads();
  double yFn = 0.0, aFn = 0.0, bFn = 0.0;
  if (seg + 1 < P) {
    yFn = sA[tid + LB];
    aFn = sB[tid + LB];
    bFn = sC[tid + LB];
  }
  __syncthreads();
  const double yL = r[S - 2], aL = da[S - 2], bL = cb[S - 2];
  double A = as * aL;
  double B = bs + as * bL + cs * aFn;
  double C = cs * bFn;
  double R = rs - as * yL - cs * yFn;
  for (int d = 1; d < P; d <<= 1) {
    sA[tid] = A;
    sB[tid] = __drcp_rn(B);
    sC[tid] = C;
    sR[tid] = R;
    __syncthreads();
    double Am = 0.0, iBm = 1.0, Cm = 0.0, Rm = 0.0, Ap = 0.0, iBp = 1.0, Cp = 0.0, Rp = 0.0;
    if (seg >= d) {
      const int o = tid - d * LB;
      Am = sA[o];
      iBm = sB[o];
      Cm = sC[o];
      Rm = sR[o];
    }
    if (seg + d < P) {
      const int o = tid + d * LB;
      Ap = sA[o];
      iBp = sB[o];
      Cp = sC[o];
      Rp = sR[o];
    }
    __syncthreads();
    const double k1 = -A * iBm, k2 = -C * iBp;
    A = k1 * Am;
    C = k2 * Cp;
    B = B + k1 * Cm + k2 * Ap;
    R = R + k1 * Rm + k2 * Rp;
  }
  const double t = R / B;
  sA[tid] = t;
  __syncthreads();
  const double tm = (seg > 0) ? sA[tid - LB] : 0.0;

  bool bad = false;
#pragma unroll
  for (int j = 0; j < S; ++j) {
    const int i = i0 + j;
    if (!active || i >= m) continue;
    const long long off = base + (long long)(i + 1) * stride;
    double x = (j < S - 1) ? fma(cb[j], t, fma(da[j], tm, r[j])) : t;
    if (a.epi == EPI_AOS0) {
      x = __dadd_rn(sinh_flow(a.src[off], (cd[j] & 1u) ? a.decay1 : a.decay0, a.pm), x);
    } else {
      x = epi_val(a, x, cd[j], off);
    }
    a.dst[off] = x;
    bad |= is_bad(x, a.thr);
  }
  if (a.check) {
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x + threadIdx.y * blockDim.x) % 32 == 0)
      atomicMin(a.div_step, a.step);
  }
}

// ---------------------------------------------------------------------------------------
// Contiguous axis (2): one warp per (i, j) line, lane = segment of S rows.
template <int S>
__host__ __device__ constexpr int cpos(int p) {
  return (S % 2 == 0) ? p + p / S : p;
}

template <int S>
__host__ __device__ constexpr int contig_buf_doubles() {
  return ((cpos<S>(32 * S + 2) + 2) + 1) & ~1;
}

template <int S>
__global__ void __launch_bounds__(256) k_sweep_contig(const SweepArgs a, const int nlines) {
  extern __shared__ double sm[];
  if (a.div_step && *((volatile int*)a.div_step) < a.step) return;
  constexpr int BUF = contig_buf_doubles<S>();
  constexpr int CBUF = 32 * S + 8;
  const int W = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int line = blockIdx.x * W + warp;
  if (line >= nlines) return;
  const Layout& L = a.L;
  const int m = a.m, n2 = L.n2;
  const int ii = 1 + line / (L.n1 - 2), jj = 1 + line % (L.n1 - 2);
  const long long rb = L.at(ii, jj, 0);
  double* buf = sm + warp * BUF;
  uint8_t* cbuf = reinterpret_cast<uint8_t*>(sm + W * BUF) + warp * CBUF;

  for (int e = lane; e < n2; e += 32) {
    buf[cpos<S>(e)] = a.src[rb + e];
    cbuf[e] = a.codes[rb + e];
  }
  __syncwarp();

  const int i0 = lane * S;
  double r[S], cb[S], da[S];
  uint32_t cd[S + 1];
#pragma unroll
  for (int j = 0; j <= S; ++j) {
    const int p = i0 + j + 1;
    cd[j] = (p <= n2 - 1) ? (uint32_t)cbuf[p] : 0u;
  }
#pragma unroll
  for (int j = 0; j < S; ++j) {
    const int i = i0 + j, p = i + 1;
    if (i < m) {
      r[j] = pro_val(a, buf[cpos<S>(p)], cd[j], rb + p);
    } else if (i == m) {
      r[j] = a.cn ? face_val(a, rb + p) : 0.0;
    } else {
      r[j] = 0.0;
    }
  }
  double wprev = __shfl_up_sync(0xffffffffu, r[S - 1], 1);
  double wnext = __shfl_down_sync(0xffffffffu, r[0], 1);
  if (lane == 0) wprev = a.cn ? face_val(a, rb) : 0.0;
  if (lane == 31) wnext = (a.cn && 32 * S == m) ? face_val(a, rb + m + 1) : 0.0;
  double blo = 0.0, bhi = 0.0;
  if (i0 == 0) blo = a.bnd[rb];
  if (i0 <= m - 1 && m - 1 < i0 + S) bhi = a.bnd[rb + m + 1];
  {
    double wm = wprev;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const int i = i0 + j;
      const double wc = r[j];
      const double wp = (j + 1 < S) ? r[j + 1] : wnext;
      if (i < m) {
        const uint32_t em = (cd[j] >> 3) & 1u, ep = (cd[j + 1] >> 3) & 1u;
        r[j] = row_rhs(a, i, cd[j], em, ep, wm, wc, wp, rb + i + 1, blo, bhi);
      } else {
        r[j] = 0.0;
      }
      wm = wc;
    }
  }
  double as, bs, cs;
  seg_solve<S>(r, cb, da, cd, i0, m, 3, a.co, as, bs, cs);
  const double rs = r[S - 1];
  double yFn = __shfl_down_sync(0xffffffffu, r[0], 1);
  double aFn = __shfl_down_sync(0xffffffffu, da[0], 1);
  double bFn = __shfl_down_sync(0xffffffffu, cb[0], 1);
  if (lane == 31) yFn = aFn = bFn = 0.0;
  double A = as * da[S - 2];
  double B = bs + as * cb[S - 2] + cs * aFn;
  double C = cs * bFn;
  double R = rs - as * r[S - 2] - cs * yFn;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double iB = __drcp_rn(B);
    double Am = __shfl_up_sync(0xffffffffu, A, d);
    double iBm = __shfl_up_sync(0xffffffffu, iB, d);
    double Cm = __shfl_up_sync(0xffffffffu, C, d);
    double Rm = __shfl_up_sync(0xffffffffu, R, d);
    double Ap = __shfl_down_sync(0xffffffffu, A, d);
    double iBp = __shfl_down_sync(0xffffffffu, iB, d);
    double Cp = __shfl_down_sync(0xffffffffu, C, d);
    double Rp = __shfl_down_sync(0xffffffffu, R, d);
    if (lane < d) {
      Am = 0.0;
      iBm = 1.0;
      Cm = 0.0;
      Rm = 0.0;
    }
    if (lane + d >= 32) {
      Ap = 0.0;
      iBp = 1.0;
      Cp = 0.0;
      Rp = 0.0;
    }
    const double k1 = -A * iBm, k2 = -C * iBp;
    A = k1 * Am;
    C = k2 * Cp;
    B = B + k1 * Cm + k2 * Ap;
    R = R + k1 * Rm + k2 * Rp;
  }
  const double t = R / B;
  double tm = __shfl_up_sync(0xffffffffu, t, 1);
  if (lane == 0) tm = 0.0;

#pragma unroll
  for (int j = 0; j < S; ++j) {
    const int i = i0 + j, p = i + 1;
    if (i >= m) continue;
    double x = (j < S - 1) ? fma(cb[j], t, fma(da[j], tm, r[j])) : t;
    if (a.epi == EPI_AOS0)
      x = __dadd_rn(sinh_flow(buf[cpos<S>(p)], (cd[j] & 1u) ? a.decay1 : a.decay0, a.pm), x);
    buf[cpos<S>(p)] = x;
  }
  __syncwarp();
  bool bad = false;
  for (int p = lane + 1; p <= m; p += 32) {
    double x = buf[cpos<S>(p)];
    if (a.epi != EPI_AOS0) x = epi_val(a, x, cbuf[p], rb + p);
    a.dst[rb + p] = x;
    bad |= is_bad(x, a.thr);
  }
  if (a.check) {
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(a.div_step, a.step);
  }
}

// ---------------------------------------------------------------------------------------
// Host-side launch helpers.

static int strided_S(int m) { return m <= 128 ? 4 : (m <= 512 ? 8 : 16); }

template <int S>
static void launch_strided_S(const SweepArgs& a, int axis, cudaStream_t st) {
  const int m = a.m;
  const int P = (m + S - 1) / S;
  const int LB = P <= 16 ? 32 : (P <= 32 ? 16 : 8);
  const int nouter = (axis == 0 ? a.L.n1 : a.L.n0) - 2;
  dim3 grid((a.L.n2 - 2 + LB - 1) / LB, nouter);
  dim3 block(LB, P);
  const size_t smem = sizeof(double) * 4 * LB * P;
  k_sweep_strided<S><<<grid, block, smem, st>>>(a, axis);
}

static int launch_strided(const SweepArgs& a, int axis, cudaStream_t st) {
  const int m = a.m;
  if (m > 1024) return fail(PBG_E_UNSUPPORTED, "line too long for strided sweep (m > 1024)");
  switch (strided_S(m)) {
    case 4: launch_strided_S<4>(a, axis, st); break;
    case 8: launch_strided_S<8>(a, axis, st); break;
    default: launch_strided_S<16>(a, axis, st); break;
  }
  PBG_LAUNCH_CHECK("k_sweep_strided");
  return PBG_OK;
}

template <int S>
static void launch_contig_S(const SweepArgs& a, cudaStream_t st) {
  const int W = 8;
  const int nlines = (a.L.n0 - 2) * (a.L.n1 - 2);
  const size_t smem = (size_t)W * (contig_buf_doubles<S>() * sizeof(double) + (32 * S + 8));
  k_sweep_contig<S><<<(nlines + W - 1) / W, 32 * W, smem, st>>>(a, nlines);
}

static int launch_contig(const SweepArgs& a, cudaStream_t st) {
  const int m = a.m;
  if (m <= 64) launch_contig_S<2>(a, st);
  else if (m <= 96) launch_contig_S<3>(a, st);
  else if (m <= 128) launch_contig_S<4>(a, st);
  else if (m <= 192) launch_contig_S<6>(a, st);
  else if (m <= 256) launch_contig_S<8>(a, st);
  else if (m <= 384) launch_contig_S<12>(a, st);
  else if (m <= 512) launch_contig_S<16>(a, st);
  else if (m <= 768) launch_contig_S<24>(a, st);
  else if (m <= 1024) launch_contig_S<32>(a, st);
  else return fail(PBG_E_UNSUPPORTED, "line too long for contiguous sweep (m > 1024)");
  PBG_LAUNCH_CHECK("k_sweep_contig");
  return PBG_OK;
}

static int launch_sweep(const SweepArgs& a, int axis, cudaStream_t st) {
  return axis == 2 ? launch_contig(a, st) : launch_strided(a, axis, st);
}

// Tridiagonal row tables for one axis: f = factor / h^2 (tridiag.py:165, 179-181, 199-202).
static AxisCoef make_axis_coef(const double eps[2], double factor, double h) {
  AxisCoef c;
  const double f = factor / (h * h);
  for (int em = 0; em < 2; ++em)
    for (int ep = 0; ep < 2; ++ep) c.diag[em * 2 + ep] = 1.0 + f * (eps[ep] + eps[em]);
  for (int b = 0; b < 2; ++b) {
    c.sub[b] = -f * eps[b];
    c.sup[b] = -f * eps[b];
    c.flo[b] = f * eps[b];
    c.fhi[b] = f * eps[b];
    c.eps[b] = eps[b];
  }
  return c;
}

static SweepArgs base_args(const pbg_grid* g, const pbg_palette* pal, int axis, double factor) {
  SweepArgs a;
  memset(&a, 0, sizeof(a));
  a.L = make_layout(g);
  a.m = g->n[axis] - 2;
  a.co = make_axis_coef(pal->eps[axis], factor, g->h);
  a.decay0 = a.decay1 = 1.0;
  a.pm = 1.0;
  a.pro = PRO_NONE;
  a.epi = EPI_STORE;
  a.thr = INFINITY;
  return a;
}

// Variant table (schemes.py:209-262).
struct Plan {
  int family;  // 0: LOD flow-first (IE1/CN1), 1: LOD source-first (IE2/CN2), 2: AOS, 3: MAOS
  double mult;  // sweep factor = mult * dta
  int cn;
  double src[3];
};

static bool plan_for(int v, Plan& p) {
  p.src[0] = p.src[1] = p.src[2] = 0.0;
  switch (v) {
    case PBG_LODIE1: p = {0, 1.0, 0, {0, 0, 0}}; return true;
    case PBG_LODIE2: p = {1, 1.0, 0, {0, 0, 0}}; return true;
    case PBG_LODCN1: p = {0, 0.5, 1, {0, 0, 0}}; return true;
    case PBG_LODCN2: p = {1, 0.5, 1, {0, 0, 0}}; return true;
    case PBG_AOSIE1: p = {2, 4.0, 0, {4.0, 0.0, 0.0}}; return true;
    case PBG_AOSIE2: p = {2, 4.0, 0, {4.0 / 3.0, 4.0 / 3.0, 4.0 / 3.0}}; return true;
    case PBG_AOSCN1: p = {2, 2.0, 1, {4.0, 0.0, 0.0}}; return true;
    case PBG_AOSCN2: p = {2, 2.0, 1, {4.0 / 3.0, 4.0 / 3.0, 4.0 / 3.0}}; return true;
    case PBG_MAOSIE: p = {3, 3.0, 0, {1.0, 1.0, 1.0}}; return true;
    case PBG_MAOSCN: p = {3, 1.5, 1, {1.0, 1.0, 1.0}}; return true;
    default: return false;
  }
}

__global__ void k_faces_bad(const Layout L, const double* x, double thr, int* flag) {
  // One thread per node of the six faces.  Faces equal the Dirichlet data after step 1, so a
  // bad face means march() stops at step 1 (max|u| includes faces, schemes.py:417-421).
  const long long n01 = (long long)L.n0 * L.n1, n02 = (long long)L.n0 * L.n2,
                  n12 = (long long)L.n1 * L.n2;
  const long long total = 2 * (n01 + n02 + n12);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long u = t;
    int i, j, k;
    if (u < 2 * n12) {
      i = (u < n12) ? 0 : L.n0 - 1;
      u %= n12;
      j = (int)(u / L.n2);
      k = (int)(u % L.n2);
    } else if ((u -= 2 * n12) < 2 * n02) {
      j = (u < n02) ? 0 : L.n1 - 1;
      u %= n02;
      i = (int)(u / L.n2);
      k = (int)(u % L.n2);
    } else {
      u -= 2 * n02;
      k = (u < n01) ? 0 : L.n2 - 1;
      u %= n01;
      i = (int)(u / L.n1);
      j = (int)(u % L.n1);
    }
    const double v = x[L.at(i, j, k)];
    if (!isfinite(v) || fabs(v) > thr) atomicMin(flag, 1);
  }
}

static bool g_profile = false;
static double g_prof_ms[3] = {0, 0, 0};
static long long g_prof_n[3] = {0, 0, 0};

}  // namespace pbg

using namespace pbg;

extern "C" PBG_API int pbg_set_profiling(int32_t on) {
  g_profile = on != 0;
  for (int a = 0; a < 3; ++a) {
    g_prof_ms[a] = 0.0;
    g_prof_n[a] = 0;
  }
  return PBG_OK;
}

extern "C" PBG_API int pbg_get_profile(double axis_ms[3], int64_t launches[3]) {
  for (int a = 0; a < 3; ++a) {
    if (axis_ms) axis_ms[a] = g_prof_ms[a];
    if (launches) launches[a] = g_prof_n[a];
  }
  return PBG_OK;
}

extern "C" PBG_API int pbg_march(const pbg_march_desc* d, int32_t* steps_taken,
                                 int32_t* diverged_step, int32_t* result_slot,
                                 float* device_ms, void* stream) {
  if (!d) return fail(PBG_E_INVALID, "null descriptor");
  int rc = validate_grid(&d->grid);
  if (rc) return rc;
  Plan plan;
  if (!plan_for(d->variant, plan))
    return fail(PBG_E_UNSUPPORTED, "variant not supported by the device march");
  if (!(d->dt > 0) || !(d->alpha > 0) || d->nsteps < 1)
    return fail(PBG_E_INVALID, "dt, alpha must be positive and nsteps >= 1");
  if (!d->codes || !d->rho || !d->initial || !d->work[0] || !d->work[1])
    return fail(PBG_E_INVALID, "null device buffer");
  cudaStream_t st = (cudaStream_t)stream;
  const pbg_grid* g = &d->grid;
  const double dta = d->dt / d->alpha;
  const double factor = plan.mult * dta;
  const double h2 = g->h * g->h;

  // Flow decays (schemes.py:212, 264-270): LOD/MAOS exp(-k2*dta); AOS exact exp(-4*k2*dta),
  // literal exp(-k2*dta) with premultiplier 4.
  double dec_lod[2], dec_aos[2];
  for (int b = 0; b < 2; ++b) {
    const double k2 = d->pal.kappa2[b];
    dec_lod[b] = std::exp(-k2 * dta);
    dec_aos[b] = d->aos_literal ? std::exp(-k2 * dta) : std::exp(-4.0 * k2 * dta);
  }
  const double aos_pm = d->aos_literal ? 4.0 : 1.0;

  SweepArgs ax[3];
  for (int axis = 0; axis < 3; ++axis) {
    SweepArgs a = base_args(g, &d->pal, axis, factor);
    a.codes = d->codes;
    a.rho = d->rho;
    a.bnd = d->work[0];
    a.cn = plan.cn;
    a.cnc = plan.cn ? (plan.mult * dta) / h2 : 0.0;
    a.thr = d->divergence_threshold;
    switch (plan.family) {
      case 0:  // LODIE1 / LODCN1: flow -> sweeps -> + dta*rho
        if (axis == 0) {
          a.pro = PRO_FLOW;
          a.decay0 = dec_lod[0];
          a.decay1 = dec_lod[1];
        }
        if (axis == 2) {
          a.epi = EPI_SRC;
          a.epi_coef = dta;
        }
        break;
      case 1:  // LODIE2 / LODCN2: + dta*rho -> sweeps -> flow
        if (axis == 0) {
          a.pro = PRO_SRC;
          a.pro_coef = dta;
        }
        if (axis == 2) {
          a.epi = EPI_FLOW;
          a.decay0 = dec_lod[0];
          a.decay1 = dec_lod[1];
        }
        break;
      case 2:  // AOS: 0.25*(((pm*flow(u) + b0) + b1) + b2), branches from u
        a.epi = axis == 0 ? EPI_AOS0 : (axis == 1 ? EPI_AOS1 : EPI_AOS2);
        if (axis == 0) {
          a.decay0 = dec_aos[0];
          a.decay1 = dec_aos[1];
          a.pm = aos_pm;
        }
        a.has_extra = plan.src[axis] != 0.0;
        a.extra = plan.src[axis] * dta;
        break;
      case 3:  // MAOS: ((b0 + b1) + b2)/3, branches from flow(u)
        a.pro = PRO_FLOW;
        a.decay0 = dec_lod[0];
        a.decay1 = dec_lod[1];
        a.epi = axis == 0 ? EPI_MAOS0 : (axis == 1 ? EPI_MAOS1 : EPI_MAOS2);
        a.has_extra = 1;
        a.extra = plan.src[axis] * dta;
        break;
    }
    a.check = (axis == 2) && d->check_divergence;
    ax[axis] = a;
  }

  int* dflag = nullptr;
  PBG_CUDA(cudaMallocAsync(&dflag, sizeof(int), st));
  const int init = INT_MAX;
  PBG_CUDA(cudaMemcpyAsync(dflag, &init, sizeof(init), cudaMemcpyHostToDevice, st));
  if (d->check_divergence) {
    k_faces_bad<<<148, 256, 0, st>>>(make_layout(g), d->work[0], d->divergence_threshold,
                                     dflag);
    PBG_LAUNCH_CHECK("k_faces_bad");
  }

  int st_idx = -1;
  if (d->initial == d->work[0]) st_idx = 0;
  else if (d->initial == d->work[1]) st_idx = 1;
  const int st0 = st_idx;

  cudaEvent_t e0, e1;
  PBG_CUDA(cudaEventCreate(&e0));
  PBG_CUDA(cudaEventCreate(&e1));
  std::vector<cudaEvent_t> kev;  // per-launch events when profiling is on
  PBG_CUDA(cudaEventRecord(e0, st));
  for (int s = 1; s <= d->nsteps; ++s) {
    const double* X = st_idx < 0 ? d->initial : d->work[st_idx];
    const int other = st_idx < 0 ? 0 : 1 - st_idx;
    double* A = d->work[other];
    double* Bf = st_idx < 0 ? d->work[1] : d->work[st_idx];
    for (int axis = 0; axis < 3; ++axis) {
      SweepArgs a = ax[axis];
      a.step = s;
      a.div_step = d->check_divergence ? dflag : nullptr;
      if (plan.family <= 1) {
        a.src = axis == 0 ? X : (axis == 1 ? A : Bf);
        a.dst = axis == 0 ? A : (axis == 1 ? Bf : A);
      } else {
        a.src = X;
        a.acc = A;
        a.dst = A;
      }
      if (g_profile) {
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        cudaEventRecord(ev, st);
        kev.push_back(ev);
      }
      rc = launch_sweep(a, axis, st);
      if (g_profile) {
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        cudaEventRecord(ev, st);
        kev.push_back(ev);
      }
      if (rc) {
        cudaFreeAsync(dflag, st);
        return rc;
      }
    }
    st_idx = other;
  }
  PBG_CUDA(cudaEventRecord(e1, st));
  int dstep = INT_MAX;
  PBG_CUDA(cudaMemcpyAsync(&dstep, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
  PBG_CUDA(cudaFreeAsync(dflag, st));
  PBG_CUDA(cudaStreamSynchronize(st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  for (size_t q = 0; q + 1 < kev.size(); q += 2) {
    float kms = 0.f;
    cudaEventElapsedTime(&kms, kev[q], kev[q + 1]);
    const int axis = (int)((q / 2) % 3);
    g_prof_ms[axis] += kms;
    g_prof_n[axis] += 1;
  }
  for (auto ev : kev) cudaEventDestroy(ev);
  int taken = d->nsteps;
  if (d->check_divergence && dstep != INT_MAX) {
    taken = dstep;
    if (diverged_step) *diverged_step = dstep;
  } else if (diverged_step) {
    *diverged_step = 0;
  }
  // state slot after `taken` steps
  int slot;
  if (st0 < 0) slot = (taken - 1) % 2;
  else slot = (st0 + taken) % 2;
  if (steps_taken) *steps_taken = taken;
  if (result_slot) *result_slot = slot;
  if (device_ms) *device_ms = ms;
  return PBG_OK;
}

extern "C" PBG_API int pbg_sweep(const pbg_grid* g, const pbg_palette* pal,
                                 const uint8_t* codes, int32_t axis, double factor, int32_t cn,
                                 const double* src, const double* bnd, double* dst,
                                 void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  if (axis < 0 || axis > 2) return fail(PBG_E_INVALID, "axis must be 0, 1 or 2");
  if (!pal || !codes || !src || !bnd || !dst) return fail(PBG_E_INVALID, "null pointer");
  SweepArgs a = base_args(g, pal, axis, factor);
  a.codes = codes;
  a.src = src;
  a.bnd = bnd;
  a.dst = dst;
  a.rho = src;  // never read (no source terms)
  a.cn = cn ? 1 : 0;
  a.cnc = cn ? factor / (g->h * g->h) : 0.0;
  return launch_sweep(a, axis, (cudaStream_t)stream);
}
