// Implicit line sweeps and the fused LOD/AOS/MAOS time step for sm_100a.
//
// Reference: pbsplit/tridiag.py:120-219 (prefactored batched Thomas), pbsplit/schemes.py:
// 88-103 (sinh flow), 123-143 (delta2_block), 274-329 (Stepper sweeps/steps), 399-425 (march).
//
// Every implicit sweep solves (1 - f*d2_a) x = rhs on all interior lines of axis a, where
// the tridiagonal rows are  sub = -f*e_minus, diag = 1 + f*(e_plus + e_minus),
// sup = -f*e_plus  (tridiag.py:165, 179-181), with the static Dirichlet fold-ins on the
// first/last row (tridiag.py:193-202).  The reference runs one serial Thomas per line with
// stored LU factors.  Here each line is split into P segments of S rows (S = 16, P = 8/16/32;
// S = 32 for lines longer than 512), one thread per segment:
//
//   * rows j < S-1 of a segment are "inner", row S-1 is a separator t_k; inner unknowns are
//     x_j = y_j + alpha_j * t_{k-1} + beta_j * t_k  (one elimination, three right-hand sides);
//   * the P separators of a line satisfy a diagonally dominant tridiagonal "reduced" system,
//     solved with a precomputed dense inverse on lines of one dielectric ("clean"), by
//     parallel cyclic reduction in shared memory otherwise;
//   * alpha/beta and the LU factors of a segment depend only on the coefficient codes: a
//     segment whose nodes carry one dielectric ("uniform", >90% in the protein configs) reads
//     them from per-axis tables (the dominant kind from kernel parameters = constant bank),
//     other segments from factors precomputed once per march (k_seg_factors).
//
// Data movement: every block stages a tile of LB lines x the whole line through shared memory
// with asynchronous copies (LDGSTS).  Axes 0/1 ("column tiles"): LB adjacent k columns, each
// row of the tile one 64/128-byte run.  Axis 2 ("row tiles"): LB adjacent (i, j) lines, each
// a contiguous row.  The prologue is applied in the staging pass, the line is solved from
// shared memory / registers, and the epilogue runs in the coalesced store pass.
//
// Prologue / epilogue fusions:
//   PRO_FLOW  w = pm*flow(u)         LODIE1/LODCN1 first sweep, MAOS branches
//   PRO_SRC   w = u + dta*rho        LODIE2/LODCN2 first sweep
//   CN        rhs += (cn_f/h^2)*delta2(w) along the sweep axis
//   extra     rhs += coef*dta*rho    AOS/MAOS branch source
//   EPI_*     LODIE1 source, LODIE2 flow, AOS/MAOS accumulate/combine, divergence flag.

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include <cub/cub.cuh>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "sweep.cuh"

namespace pbg {

// Asynchronous global->shared copies (LDGSTS): issued back to back, no register round trip.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Which second tile the epilogue needs: 0 none, 1 the raw field (AOS0), 2 the accumulator.
__host__ __device__ __forceinline__ int epi_needs(int epi) {
  return epi == EPI_AOS0 ? 1
                         : ((epi == EPI_AOS1 || epi == EPI_AOS2 || epi == EPI_MAOS1 ||
                             epi == EPI_MAOS2)
                                ? 2
                                : 0);
}

// Flow interval tables staged in shared memory at FP + kFlowHdr (kFlowHdr: alignment slack).
constexpr int kFlowHdr = 6;
// Palette constants come from the kernel parameters (constant bank, selected by the solute
// bit), the interval tables from shared memory.
__device__ __forceinline__ double flow_sm(const SweepArgs& a, const double* FP, double w,
                                          uint32_t s, double pm) {
  if (s) {  // solute palette: usually no ions (decay 1, the flow is the identity)
    if (a.decay1 >= 1.0 || w != w) return pm != 1.0 ? pm * w : w;
    return sinh_flow_poly(w, a.decay1, a.sat1, pm, FP + kFlowHdr + a.foff[1]);
  }
  if (a.fsmall_on && fabs(w) <= kFSmallX) {  // solvent far field: no table loads
    const double out = fabs(w) <= kFTinyX ? flow_tiny(w, a.ftiny) : flow_small(w, a.fsmall);
    return pm != 1.0 ? pm * out : out;
  }
  return sinh_flow_poly(w, a.decay0, a.sat0, pm, FP + kFlowHdr + a.foff[0]);
}

// pm * flow of four independent nodes in place: the tiny-argument polynomial for all of
// them first (branch-free, so the four Horner chains interleave), then flow_sm for the rarer
// others (solute palette, |w| > kFTinyX, no small form).  Same results as flow_sm per node.
__device__ __forceinline__ void flow_group(const SweepArgs& a, const double* FP, double& w0,
                                           double& w1, double& w2, double& w3, uint32_t s0,
                                           uint32_t s1, uint32_t s2, uint32_t s3, double pm) {
  const double x0 = flow_tiny(w0, a.ftiny), x1 = flow_tiny(w1, a.ftiny);
  const double x2 = flow_tiny(w2, a.ftiny), x3 = flow_tiny(w3, a.ftiny);
  // branch-free: solute palette, |w| above the tiny range (NaN included), no small form
  const unsigned big = (fabs(w0) <= kFTinyX ? 0u : 1u) | (fabs(w1) <= kFTinyX ? 0u : 2u) |
                       (fabs(w2) <= kFTinyX ? 0u : 4u) | (fabs(w3) <= kFTinyX ? 0u : 8u);
  const unsigned need = a.fsmall_on ? (big | s0 | (s1 << 1) | (s2 << 2) | (s3 << 3)) : 15u;
  const double in0 = w0, in1 = w1, in2 = w2, in3 = w3;
  w0 = pm != 1.0 ? pm * x0 : x0;
  w1 = pm != 1.0 ? pm * x1 : x1;
  w2 = pm != 1.0 ? pm * x2 : x2;
  w3 = pm != 1.0 ? pm * x3 : x3;
  if (!need) return;
  // the others one at a time through ONE inlined copy of flow_sm (a per-node copy made the
  // row kernels' code 4x larger and their instruction fetch a top stall)
#pragma unroll 1
  for (unsigned m = need; m; m &= m - 1) {
    const int u = __ffs(m) - 1;
    const double w = u == 0 ? in0 : (u == 1 ? in1 : (u == 2 ? in2 : in3));
    const uint32_t s = u == 0 ? s0 : (u == 1 ? s1 : (u == 2 ? s2 : s3));
    const double r = flow_sm(a, FP, w, s, pm);
    if (u == 0) w0 = r;
    else if (u == 1) w1 = r;
    else if (u == 2) w2 = r;
    else w3 = r;
  }
}

// pm * flow of four independent nodes in place, the small-argument polynomial (|w| <= 2: all
// solvent nodes of the protein configs) for all of them, branch-free with the identity of an
// ion-free solute palette selected per node; flow_sm only for the rare others (|w| > 2, NaN,
// a solute palette with ions, no small form).  Seven more DFMA per node than the tiny tier
// but no divergent fallback near the molecule (k_sweep_rowlean: the lanes of a warp sit 16
// rows apart on the same line).
__device__ __forceinline__ void flow_group_small(const SweepArgs& a, const double* FP,
                                                 double& w0, double& w1, double& w2, double& w3,
                                                 uint32_t s0, uint32_t s1, uint32_t s2,
                                                 uint32_t s3, double pm) {
  const double x0 = flow_small(w0, a.fsmall), x1 = flow_small(w1, a.fsmall);
  const double x2 = flow_small(w2, a.fsmall), x3 = flow_small(w3, a.fsmall);
  const unsigned big = (fabs(w0) <= kFSmallX ? 0u : 1u) | (fabs(w1) <= kFSmallX ? 0u : 2u) |
                       (fabs(w2) <= kFSmallX ? 0u : 4u) | (fabs(w3) <= kFSmallX ? 0u : 8u);
  const unsigned sol = s0 | (s1 << 1) | (s2 << 2) | (s3 << 3);
  const bool sol_id = a.decay1 >= 1.0;  // launch-uniform
  const unsigned need = a.fsmall_on ? (sol_id ? (big & ~sol) : (big | sol)) : 15u;
  const double in0 = w0, in1 = w1, in2 = w2, in3 = w3;
  w0 = (sol_id && s0) ? w0 : x0;
  w1 = (sol_id && s1) ? w1 : x1;
  w2 = (sol_id && s2) ? w2 : x2;
  w3 = (sol_id && s3) ? w3 : x3;
  if (pm != 1.0) {
    w0 *= pm;
    w1 *= pm;
    w2 *= pm;
    w3 *= pm;
  }
  if (!need) return;
#pragma unroll 1
  for (unsigned m = need; m; m &= m - 1) {
    const int u = __ffs(m) - 1;
    const double w = u == 0 ? in0 : (u == 1 ? in1 : (u == 2 ? in2 : in3));
    const uint32_t s = u == 0 ? s0 : (u == 1 ? s1 : (u == 2 ? s2 : s3));
    const double r = flow_sm(a, FP, w, s, pm);
    if (u == 0) w0 = r;
    else if (u == 1) w1 = r;
    else if (u == 2) w2 = r;
    else w3 = r;
  }
}

__host__ __device__ __forceinline__ bool uses_flow(int pro, int epi) {
  return pro == PRO_FLOW || epi == EPI_FLOW || epi == EPI_AOS0;
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

// Reciprocal of a well-conditioned positive pivot: MUFU seed + two Newton steps (~1 ulp,
// no special-case paths).
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

__device__ __forceinline__ bool is_bad(double v, double thr) {
  // non-finite or above the threshold; thr is clamped to DBL_MAX so that +-inf and NaN fail
  // the single comparison
  return !(fabs(v) <= fmin(thr, 1.7976931348623157e308));
}

// CN explicit half for row values (wm, wc, wp) with the row's eps bits (em, ep).
__device__ __forceinline__ double cn_term(const SweepArgs& a, uint32_t em, uint32_t ep,
                                          double wm, double wc, double wp) {
  const double epv = ep ? a.co.eps[1] : a.co.eps[0];
  const double emv = em ? a.co.eps[1] : a.co.eps[0];
  const double d2 =
      __dadd_rn(__dmul_rn(epv, __dsub_rn(wp, wc)), __dmul_rn(emv, __dsub_rn(wm, wc)));
  return __dadd_rn(wc, __dmul_rn(a.cnc, d2));
}

// Per-thread segment state after the local elimination.
struct SegOut {
  double yF, aF, bF, yL, aL, bL;  // first / last inner row: y, alpha, beta
  double as, bs, cs, rs;          // separator row coefficients and rhs
};

// Node bits for the pointwise prologue / epilogue in the layout of the old 1-byte codes
// (bit 0 solute, bit 4 charged), taken from a segment descriptor.
__device__ __forceinline__ uint32_t node_bits(unsigned long long w1, int bit) {
  return (uint32_t)((w1 >> bit) & 1ull) | ((uint32_t)((w1 >> (32 + bit)) & 1ull) << 4);
}

// Table-driven elimination of a uniform segment (5 fp64 ops per row, no reciprocal).
template <int S, typename Tab>
__device__ __forceinline__ void uni_eliminate(double (&r)[S], Tab tab, SegOut& o) {
  double dyp = 0.0;
#pragma unroll
  for (int j = 0; j < S - 1; ++j) {
    const double dy = fma(-tab(TQ_G, j), dyp, r[j] * tab(TQ_INV, j));
    r[j] = dy;
    dyp = dy;
  }
  double y = r[S - 2];
#pragma unroll
  for (int j = S - 3; j >= 0; --j) {
    y = fma(-tab(TQ_CP, j), y, r[j]);
    r[j] = y;
  }
  o.yF = r[0];
  o.yL = r[S - 2];
  o.aF = tab(TQ_AL, 0);
  o.bF = tab(TQ_BE, 0);
  o.aL = tab(TQ_AL, S - 2);
  o.bL = tab(TQ_BE, S - 2);
}

template <int S, int WS, typename Tab>
__device__ __forceinline__ void uni_finish(const double (&r)[S], Tab tab, double tm, double t,
                                           double* w0) {
#pragma unroll
  for (int j = 0; j < S - 1; ++j) w0[j * WS] = fma(tab(TQ_BE, j), t, fma(tab(TQ_AL, j), tm, r[j]));
}

// Table type of a segment whose S nodes carry the same eps bit; -1 if it must use its own
// precomputed factors.  The first segment and a last segment whose separator is the padding
// row m both use the interior tables (type 0): the first segment's missing left separator is
// zero, which makes the interior table's extra sub-diagonal term vanish exactly, and the
// padding separator's right-hand side is zeroed (seg_eliminate) so its coupling to row m-1
// multiplies zero.  Results are bit-identical to the dedicated first / last tables, and
// warps made only of solvent segments take the parameter-table path wherever they sit.
template <int S>
__device__ __forceinline__ int seg_type(unsigned long long amask, int i0, int m, int first) {
  const unsigned long long allm = (1ull << S) - 1ull, bits = amask & allm;
  if (bits != 0ull && bits != allm) return -1;
  if (i0 + S <= m) return 0;
  if (i0 + S - 1 == m && !first) return 0;
  return -1;
}

// Descriptor word 0: bits 0..S eps bits, bits 34.. (slot + 1) of a general segment's
// precomputed factors (0 = uniform segment, tables).
constexpr int kSlotShift = 34;
__host__ __device__ __forceinline__ unsigned long long eps_bits(unsigned long long w0, int S) {
  return w0 & ((2ull << S) - 1ull);
}

// Elimination of one segment, always table driven: the dominant kind (interior segment,
// palette 0) reads kernel-parameter tables when the whole warp is of that kind; otherwise
// each lane reads its own table (shared-memory uniform tables, or the per-segment factors a
// general segment got at march setup, k_seg_factors).  Returns the table pointer for the
// finish step (nullptr = parameter tables).
template <int S>
__device__ __forceinline__ const double* seg_eliminate(const SweepArgs& a, double (&r)[S],
                                                       unsigned long long amask, int i0,
                                                       int first, const double* T, SegOut& o) {
  const int m = a.m;
  const int ttype = seg_type<S>(amask, i0, m, first);
  o.rs = i0 + S - 1 < m ? r[S - 1] : 0.0;  // a padding separator carries zero
  row_coefs(a.co, i0 + S - 1, m, (uint32_t)(amask >> (S - 1)) & 1u,
            (uint32_t)(amask >> S) & 1u, o.as, o.bs, o.cs);
  if (__all_sync(0xffffffffu, ttype == 0 && !(amask & 1ull))) {
    uni_eliminate<S>(r, [&](int q, int j) { return a.tmid[q * kTabRows + j]; }, o);
    return nullptr;
  }
  const double* Tv =
      ttype >= 0 ? T + (ttype * 2 + (int)(amask & 1ull)) * 5 * kTabRows
                 : a.gfac + (long long)((amask >> kSlotShift) - 1ull) * 5 * kTabRows;
  uni_eliminate<S>(r, [&](int q, int j) { return Tv[q * kTabRows + j]; }, o);
  return Tv;
}

// x_j = y_j + alpha_j*tm + beta_j*t for the inner rows, written to w0[j*WS].
template <int S, int WS>
__device__ __forceinline__ void seg_finish(const SweepArgs& a, const double* Tv,
                                           const double (&r)[S], double tm, double t,
                                           double* w0) {
  if (Tv == nullptr)
    uni_finish<S, WS>(r, [&](int q, int j) { return a.tmid[q * kTabRows + j]; }, tm, t, w0);
  else
    uni_finish<S, WS>(r, [&](int q, int j) { return Tv[q * kTabRows + j]; }, tm, t, w0);
}

// ---------------------------------------------------------------------------------------
// Strided axes (0, 1).  blockDim = (LB columns, 32 segments); block (x = k group, y = outer).
// Shared memory: tables | reduced inverse | W[NR][LB] stage/solution | Y[NR][LB] (AOS/MAOS)
// | 4x(LB*32) scratch | descriptors D[32][LB][2].
template <int S, int P>
__host__ __device__ constexpr int strided_rows() {
  return P * S + 2;
}

// Row stride (doubles) of one line in the shared tile of a row-tile launch (axis 2): room
// for rows 0..NR-1 plus one leading slot so that row 1 (global k = 1, 256-byte aligned) is
// 16-byte aligned, rounded to 2 mod 4 (2-way bank aliasing at most across lines).
template <int S, int P>
__host__ __device__ constexpr int rt_stride() {
  return (((P * S + 2 + 1) + 3) & ~3) + 2;
}

template <int LB, bool RT>
__host__ __device__ constexpr size_t tile_doubles(int S, int kSegS) {
  return RT ? (size_t)LB * ((((kSegS * S + 3) + 3) & ~3) + 2) : (size_t)(kSegS * S + 2) * LB;
}

template <int LB, bool RT>
__host__ __device__ constexpr size_t strided_smem(int S, int kSegS, bool needY, int fpoly_n) {
  return sizeof(double) * (kTabDoubles + kSegS * (kSegS + 2) + (needY ? 2 : 1) * tile_doubles<LB, RT>(S, kSegS) +
                           4 * LB * kSegS) +
         sizeof(unsigned long long) * 2 * kSegS * LB + (kFlowHdr + fpoly_n) * sizeof(double);
}

// Shared-memory flow doubles of a launch: the interval tables only where the flow runs.
__host__ __forceinline__ int flow_stage_n(const SweepArgs& a) {
  return uses_flow(a.pro, a.epi) ? a.fpoly_n : 0;
}

// Reduced system over the P separators of each line of a tile (block-wide, all threads):
// a precomputed dense inverse when every line of the tile is one dielectric end to end
// ("clean"), parallel cyclic reduction otherwise.  Returns the thread's separator t and its
// left neighbour's tm.  Scratch X: 4 * LB * kSegS doubles.
template <int S, int kSegS, int LB>
__device__ __forceinline__ void reduced_solve(const SweepArgs& a, const SegOut& o,
                                              const double* Mi, double* X, bool active,
                                              unsigned long long amask, double& t, double& tm) {
  constexpr int NT = LB * kSegS;
  const int lane = threadIdx.x, seg = threadIdx.y, tid = seg * LB + lane;
  double* sA = X;
  double* sB = X + NT;
  double* sC = X + 2 * NT;
  double* sR = X + 3 * NT;
  sA[tid] = o.yF;
  sB[tid] = o.aF;
  sC[tid] = o.bF;
  // clean tile: every line of the tile is one dielectric (palette 0) end to end
  const bool clean = __syncthreads_and(!active || eps_bits(amask, S) == 0ull) && a.static_ok;
  if (clean) {  // static inverse: separator rhs per line, one dot product, one exchange
    constexpr int RP = kSegS + 2;  // padded rows: conflict-free 16-byte loads
    double* sRl = X + 2 * NT;      // [line][separator] (spans sC, sR; sC unused here)
    const double yFn = (seg + 1 < kSegS) ? sA[tid + LB] : 0.0;
    sRl[lane * RP + seg] = o.rs - o.as * o.yL - o.cs * yFn;
    __syncthreads();
    const double2* Rr = reinterpret_cast<const double2*>(sRl + lane * RP);
    const double2* Mr = reinterpret_cast<const double2*>(Mi + seg * RP);  // row seg
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int q = 0; q < kSegS / 2; q += 2) {
      const double2 r0 = Rr[q], m0 = Mr[q], r1 = Rr[q + 1], m1 = Mr[q + 1];
      s0 = fma(m0.x, r0.x, s0);
      s1 = fma(m0.y, r0.y, s1);
      s2 = fma(m1.x, r1.x, s2);
      s3 = fma(m1.y, r1.y, s3);
    }
    t = (s0 + s1) + (s2 + s3);
    sB[tid] = t;
    __syncthreads();
    tm = (seg > 0) ? sB[tid - LB] : 0.0;
  } else {  // parallel cyclic reduction
    double yFn = 0.0, aFn = 0.0, bFn = 0.0;
    if (seg + 1 < kSegS) {
      yFn = sA[tid + LB];
      aFn = sB[tid + LB];
      bFn = sC[tid + LB];
    }
    __syncthreads();
    double A = o.as * o.aL, B = o.bs + o.as * o.bL + o.cs * aFn, Cc = o.cs * bFn,
           R = o.rs - o.as * o.yL - o.cs * yFn;
#pragma unroll
    for (int d = 1; d < kSegS; d <<= 1) {
      sA[tid] = A;
      sB[tid] = fast_rcp(B);
      sC[tid] = Cc;
      sR[tid] = R;
      __syncthreads();
      double Am = 0.0, iBm = 1.0, Cm = 0.0, Rm = 0.0, Ap = 0.0, iBp = 1.0, Cp = 0.0, Rp = 0.0;
      if (seg >= d) {
        const int q = tid - d * LB;
        Am = sA[q];
        iBm = sB[q];
        Cm = sC[q];
        Rm = sR[q];
      }
      if (seg + d < kSegS) {
        const int q = tid + d * LB;
        Ap = sA[q];
        iBp = sB[q];
        Cp = sC[q];
        Rp = sR[q];
      }
      __syncthreads();
      const double k1 = -A * iBm, k2 = -Cc * iBp;
      A = k1 * Am;
      Cc = k2 * Cp;
      B = B + k1 * Cm + k2 * Ap;
      R = R + k1 * Rm + k2 * Rp;
    }
    t = R * fast_rcp(B);
    sA[tid] = t;
    __syncthreads();
    tm = (seg > 0) ? sA[tid - LB] : 0.0;
  }
}

// High Dirichlet fold of row m-1 (tridiag.py:217): owned by segment (m-1)/S at row (m-1)%S,
// both launch-uniform, so the static-index select below runs in one thread per line.
template <int S>
__device__ __forceinline__ void fold_high(const SweepArgs& a, double (&r)[S],
                                          unsigned long long amask, double bhi) {
  const int jl = (a.m - 1) % S;
#pragma unroll
  for (int j = 0; j < S; ++j)
    if (j == jl)
      r[j] = __dadd_rn(r[j], __dmul_rn(((amask >> (j + 1)) & 1ull) ? a.co.fhi[1] : a.co.fhi[0],
                                       bhi));
}

// Sparse per-owner fix-up at the charged nodes of a segment: *slot(j) += coef * rho(j).
template <typename Slot, typename RhoAt>
__device__ __forceinline__ void charged_fixup(unsigned cmask, double coef, Slot slot,
                                              RhoAt rho_row) {
  while (cmask) {
    const int j = __ffs(cmask) - 1;
    cmask &= cmask - 1;
    double* v = slot(j);
    *v = __dadd_rn(*v, __dmul_rn(coef, *rho_row(j)));
  }
}

// One tile = LB lines x kSegS segments (thread (lane, seg) = segment seg of line lane).
//   RT = false (axes 0, 1): the LB lines are adjacent k columns; the tile is stored row-major
//        W[p][l] and staged / stored in 16-byte chunks of adjacent columns;
//   RT = true  (axis 2, "row tiles"): the LB lines are adjacent j rows, each contiguous in
//        global memory; the tile is stored line-major W[l][p] (stride rt_stride) and staged /
//        stored as contiguous rows.
template <int S, int kSegS, int LB, bool RT>
struct TileShape {
  static constexpr int NT = LB * kSegS, NR = strided_rows<S, kSegS>();
  static constexpr int RS = rt_stride<S, kSegS>();
  static constexpr int WS = RT ? 1 : LB;  // shared-memory step between consecutive rows
  static constexpr int CPR = LB / 2, RPP = NT / CPR;  // 16-byte chunks per row, rows per pass
  static constexpr int TD = RT ? LB * RS : NR * LB;   // doubles of one staged tile
};

// Where a tile sits: tile (tx, ty) of a launch with nty outer indices.
struct TileGeo {
  int b;        // grid of a batched march (0 otherwise); base includes b * L.bs
  int c0;       // first line of the tile (k for column tiles, j for row tiles)
  int outer;    // outer index (j for axis 0, i for axes 1 and 2)
  int ncols;    // active lines
  int stride;   // global step between consecutive rows of a line
  long long base;  // global offset of row 0 of tile line 0
};

// Slab phase A (axis-0 column tiles): the compact index (j-1)*(n2-2) + (k-1) of line (j, k)
// in the exchanged end-row planes (only interior lines travel, no pitch padding or faces).
__device__ __forceinline__ long long ends_index(const SweepArgs& a, const TileGeo& g, int l) {
  return (long long)(g.outer - 1) * (a.L.n2 - 2) + (g.c0 - 1 + l);
}

template <int LB, bool RT>
__device__ __forceinline__ TileGeo tile_geo(const SweepArgs& a, int axis, int tx, int ty,
                                            int nty, int b = 0) {
  const Layout& L = a.L;
  TileGeo g;
  g.b = b;
  g.c0 = 1 + tx * LB;
  // Row tiles walk the planes in reverse: the axis-1 sweep before them wrote the last planes
  // last, so those are still in L2 when this launch starts.
  g.outer = RT ? a.o0 + nty - ty : 1 + ty + a.o0;  // a.o0: first outer index of a chunk launch
  const int K = (RT ? L.n1 : L.n2) - 2;  // lines per outer index
  g.ncols = min(LB, K + 1 - g.c0);
  if (RT) {
    g.base = L.at(g.outer, g.c0, 0);
    g.stride = 1;
  } else if (axis == 0) {
    g.base = L.at(0, g.outer, g.c0);
    g.stride = (int)L.s0;
  } else {
    g.base = L.at(g.outer, 0, g.c0);
    g.stride = (int)L.pitch;
  }
  g.base += (long long)b * L.bs;
  return g;
}

// Asynchronous staging of one tile (own descriptor, field rows, epilogue operand); rows past
// the far face are zeroed.  The caller commits the group.
template <int S, int kSegS, int LB, bool RT>
__device__ __forceinline__ void stage_tile(const SweepArgs& a, const TileGeo& g, double* W,
                                           double* Yt, unsigned long long* D, int needY) {
  using TS = TileShape<S, kSegS, LB, RT>;
  constexpr int NT = TS::NT, NR = TS::NR, RS = TS::RS, CPR = TS::CPR, RPP = TS::RPP;
  const int lane = threadIdx.x, seg = threadIdx.y, tid = seg * LB + lane;
  const Layout& L = a.L;
  const int m = a.m, nl = m + 2;
  const int K = (RT ? L.n1 : L.n2) - 2;
  const double* gy_all = needY == 1 ? a.src : a.acc;
  if (D)
    cp_async16(D + 2 * tid,
               a.desc + g.b * a.dstride +
                   2 * (((long long)(g.outer - 1) * kSegS + seg) * K + (g.c0 - 1 + lane)));
  if (RT) {
    // rows 1..m+1 of each line in 16-byte chunks (row 1 is 256-byte aligned), row 0 alone
    const int nch = (m + 1) / 2;  // full chunks; an odd last row goes alone
    const long long gstep = L.pitch;
    for (int c = tid; c < nch; c += NT) {
      const double* gp = a.src + g.base + 1 + 2 * c;
      unsigned w = (unsigned)__cvta_generic_to_shared(W + 2 + 2 * c);
      for (int l = 0; l < g.ncols; ++l, gp += gstep, w += RS * 8)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(w), "l"(gp));
      if (needY) {
        const double* gy = gy_all + g.base + 1 + 2 * c;
        unsigned y = (unsigned)__cvta_generic_to_shared(Yt + 2 + 2 * c);
        for (int l = 0; l < g.ncols; ++l, gy += gstep, y += RS * 8)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(y), "l"(gy));
      }
    }
    if (tid < g.ncols) {
      const long long lbt = g.base + (long long)tid * L.pitch;
      cp_async8(W + tid * RS + 1, a.src + lbt);
      if ((m + 1) & 1) cp_async8(W + tid * RS + 1 + m + 1, a.src + lbt + m + 1);
      if (needY) {
        cp_async8(Yt + tid * RS + 1, gy_all + lbt);
        if ((m + 1) & 1) cp_async8(Yt + tid * RS + 1 + m + 1, gy_all + lbt + m + 1);
      }
    }
    for (int c = tid; c < LB * (NR - nl); c += NT) {  // rows past the far face
      const int l = c / (NR - nl), p = nl + c % (NR - nl);
      W[l * RS + 1 + p] = 0.0;
    }
  } else {
    const int q = (tid % CPR) * 2, p0 = tid / CPR;
    const long long gstep = (long long)RPP * g.stride;
    const double* gp = a.src + g.base + p0 * (long long)g.stride + q;
    double* w = W + p0 * LB + q;
#pragma unroll 4
    for (int p = p0; p < nl; p += RPP, gp += gstep, w += RPP * LB) cp_async16(w, gp);
    if (needY) {
      const double* gyp = gy_all + g.base + p0 * (long long)g.stride + q;
      double* yp = Yt + p0 * LB + q;
#pragma unroll 4
      for (int p = p0; p < nl; p += RPP, gyp += gstep, yp += RPP * LB) cp_async16(yp, gyp);
    }
    for (int c = nl * LB + tid; c < NR * LB; c += NT) W[c] = 0.0;  // rows past the far face
  }
}

// Once the own descriptor has landed: a general segment reads its precomputed factors from
// global memory, so bring the five rows of its table towards L1; same for the source at
// charged nodes.  Returns the Dirichlet value the thread folds into its first / last row.
template <int S, int kSegS, int LB, bool RT>
__device__ __forceinline__ double tile_prefetch(const SweepArgs& a, const TileGeo& g,
                                                const unsigned long long* D) {
  const int lane = threadIdx.x, seg = threadIdx.y, tid = seg * LB + lane;
  double bfold = 0.0;
  if (lane < g.ncols) {
    const long long gl = g.base + (RT ? (long long)lane * a.L.pitch : (long long)lane);
    const unsigned long long slot = D[2 * tid] >> kSlotShift;
    if (slot) {
      const double* f = a.gfac + (long long)(slot - 1) * 5 * kTabRows;
#pragma unroll
      for (int q = 0; q < 5; ++q) asm volatile("prefetch.global.L1 [%0];" ::"l"(f + q * kTabRows));
    }
    unsigned cm = (unsigned)(D[2 * tid + 1] >> 32);
    const double* rr = a.rho + gl + (long long)(seg * S + 1) * g.stride;
    while (cm) {
      const int j = __ffs(cm) - 1;
      cm &= cm - 1;
      asm volatile("prefetch.global.L1 [%0];" ::"l"(rr + (long long)j * g.stride));
    }
    if (seg == 0) bfold = a.bnd[gl];
    else if (seg == (a.m - 1) / S) bfold = a.bnd[gl + a.hi_off];
  }
  return bfold;
}

// Everything after staging: prologue, local elimination, reduced system, reconstruction,
// epilogue and coalesced store of one tile.  Block-uniform control flow (all barriers are
// reached by every thread).
template <int S, int kSegS, bool CN, int LB, bool RT>
__device__ __forceinline__ void tile_body(const SweepArgs& a, const TileGeo& g, const double* T,
                                          const double* Mi, double* W, const double* Yt,
                                          double* X, const unsigned long long* D,
                                          const double* FP, double bfold) {
  using TS = TileShape<S, kSegS, LB, RT>;
  constexpr int NT = TS::NT, RS = TS::RS, WS = TS::WS, CPR = TS::CPR, RPP = TS::RPP;
  const int lane = threadIdx.x, seg = threadIdx.y, tid = seg * LB + lane;
  const Layout& L = a.L;
  const int m = a.m, nl = m + 2;
  const int ncols = g.ncols, stride = g.stride;
  const long long base = g.base;
  auto lb = [&](int l) { return base + (RT ? (long long)l * L.pitch : (long long)l); };
  auto sidx = [&](int p, int l) { return RT ? l * RS + 1 + p : p * LB + l; };
  const uint32_t* D32 = reinterpret_cast<const uint32_t*>(D);
  // solute bit of row p of tile line l (low word of descriptor word 1)
  auto solute = [&](int sg, int sb, int l) { return (D32[4 * (sg * LB + l) + 2] >> sb) & 1u; };

  const int i0 = seg * S;
  // lines past the last interior one read unrelated descriptor words: neutralise them
  const bool act = lane < ncols;
  const unsigned long long amask = act ? D[2 * tid] : 0ull;
  const unsigned cmask = act ? (unsigned)(D[2 * tid + 1] >> 32) : 0u;
  const long long gl = lb(lane);  // this thread's line
  const double* rrow = a.rho + gl + (long long)(i0 + 1) * stride;
  auto rho_row = [&](int j) { return rrow + (long long)j * stride; };
  double* w0 = W + sidx(i0 + 1, lane);
  if (a.pro == PRO_FLOW) {  // flow stage: interior rows transformed, faces = Dirichlet data
    if (tid < 2 * LB) {
      const int l = tid % LB;
      const bool hi = tid >= LB;
      if (l < ncols) W[sidx(hi ? nl - 1 : 0, l)] = a.bnd[lb(l) + (hi ? a.hi_off : 0ll)];
    }
    const double pm = a.pm;
    if (RT) {
      for (int p = 1 + tid; p < nl - 1; p += NT) {
        const int sg = (p - 1) / S, sb = (p - 1) - sg * S;
        for (int l = 0; l < ncols; ++l)
          W[l * RS + 1 + p] = flow_sm(a, FP, W[l * RS + 1 + p], solute(sg, sb, l), pm);
      }
    } else {
      const int l = tid % LB;
      for (int p = 1 + tid / LB; p < nl - 1; p += NT / LB) {
        const int sg = (p - 1) / S;
        W[p * LB + l] = flow_sm(a, FP, W[p * LB + l], solute(sg, (p - 1) - sg * S, l), pm);
      }
    }
    __syncthreads();
  } else if (a.pro == PRO_SRC) {  // w = u + dta*rho at the charged nodes only
    if (cmask) charged_fixup(cmask, a.pro_coef, [&](int j) { return w0 + j * WS; }, rho_row);
    __syncthreads();
  }

  {
    // Phase 2: rhs of the own rows (registers), local elimination.
    const bool active = lane < ncols;
    double r[S];
    if (RT && !CN && S % 2 == 0) {  // rows i0+1.. of a row tile: 16-byte aligned pairs
#pragma unroll
      for (int j = 0; j < S; j += 2) {
        const double2 v = *reinterpret_cast<const double2*>(w0 + j);
        r[j] = v.x;
        r[j + 1] = v.y;
      }
    } else {
      const double* wrow = w0;
#pragma unroll
      for (int j = 0; j < S; ++j) {
        const double wc = wrow[j * WS];
        r[j] = CN ? cn_term(a, (uint32_t)(amask >> j) & 1u, (uint32_t)(amask >> (j + 1)) & 1u,
                            wrow[(j - 1) * WS], wc, wrow[(j + 1) * WS])
                  : wc;
      }
    }
    if (a.has_extra && cmask) {
#pragma unroll
      for (int j = 0; j < S; ++j)
        if ((cmask >> j) & 1u) r[j] = __dadd_rn(r[j], __dmul_rn(a.extra, *rho_row(j)));
    }
    if (seg == 0 && active)
      r[0] = __dadd_rn(r[0], __dmul_rn((amask & 1ull) ? a.co.flo[1] : a.co.flo[0], bfold));
    if (seg == (m - 1) / S && active)
      fold_high<S>(a, r, amask, seg == 0 ? a.bnd[gl + a.hi_off] : bfold);
    SegOut o;
    const double* Tv = seg_eliminate<S>(a, r, amask, i0, seg == 0, T, o);

    // Phase 3: reduced system over the separators of each line.
    double t, tm;
    reduced_solve<S, kSegS, LB>(a, o, Mi, X, active, amask, t, tm);

    // Phase 4: reconstruct the inner rows, separator = t; sparse source epilogue (LODIE1).
    if (RT && S % 2 == 0) {
      // Row tiles: the separator slot of the last segment lies past row m (inside the line's
      // stride, never stored), so whole 16-byte pairs are written.
      if (Tv == nullptr) {
#pragma unroll
        for (int j = 0; j < S - 1; ++j)
          r[j] = fma(a.tmid[TQ_BE * kTabRows + j], t, fma(a.tmid[TQ_AL * kTabRows + j], tm, r[j]));
      } else {
#pragma unroll
        for (int j = 0; j < S - 1; ++j)
          r[j] = fma(Tv[TQ_BE * kTabRows + j], t, fma(Tv[TQ_AL * kTabRows + j], tm, r[j]));
      }
      r[S - 1] = t;
#pragma unroll
      for (int j = 0; j < S; j += 2)
        *reinterpret_cast<double2*>(w0 + j) = make_double2(r[j], r[j + 1]);
    } else {
      if (!a.ends || seg == 0 || seg == (m - 1) / S)  // ends-only: rows 1 and m
        seg_finish<S, WS>(a, Tv, r, tm, t, w0);
      if (i0 + S - 1 < m) w0[(S - 1) * WS] = t;
    }
    if (a.epi == EPI_SRC && cmask)
      charged_fixup(cmask, a.epi_coef, [&](int j) { return w0 + j * WS; }, rho_row);
    __syncthreads();
  }
  if (a.ends) {  // slab phase A (axis 0): only the chunk's end rows leave the block
    if (tid < 2 * LB) {
      const int l = tid % LB;
      const bool hi = tid >= LB;
      if (l < ncols)  // compact (j-1)*(n2-2) + (k-1) planes
        a.ends[ends_index(a, g, l) + (hi ? a.ends_off : 0ll)] = W[sidx(hi ? m : 1, l)];
    }
    return;
  }
  // Phase 5: epilogue + coalesced store of the interior rows.
  {
    bool bad = false;
    const int epi = a.epi;
    const bool plain = (epi == EPI_STORE || epi == EPI_SRC || epi == EPI_MAOS0) && !a.check;
    // per-node epilogue loop (one rolled copy per epilogue kind)
    auto loop = [&](auto f) {
      if (RT) {
        for (int p = 1 + tid; p <= m; p += NT) {
          double* g = a.dst + base + p;
          const int sg = (p - 1) / S, sb = (p - 1) - sg * S;
          for (int l = 0; l < ncols; ++l, g += L.pitch) {
            const double x = f(l * RS + 1 + p, solute(sg, sb, l));
            *g = x;
            bad |= is_bad(x, a.thr);
          }
        }
      } else {
        const int l = tid % LB;
        if (l >= ncols) return;
        double* g = a.dst + base + l;
        for (int p = 1 + tid / LB; p <= m; p += NT / LB) {
          const int sg = (p - 1) / S;
          const double x = f(p * LB + l, solute(sg, (p - 1) - sg * S, l));
          g[(long long)p * stride] = x;
          bad |= is_bad(x, a.thr);
        }
      }
    };
    if (RT && !CN && epi == EPI_FLOW) {  // LODIE2 flow: four lines at a time
      for (int p = 1 + tid; p <= m; p += NT) {
        double* gp = a.dst + base + p;
        const int sg = (p - 1) / S, sb = (p - 1) - sg * S;
        int l = 0;
        for (; l + 4 <= ncols; l += 4) {
          double x[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) x[u] = W[(l + u) * RS + 1 + p];
          flow_group(a, FP, x[0], x[1], x[2], x[3], solute(sg, sb, l), solute(sg, sb, l + 1),
                     solute(sg, sb, l + 2), solute(sg, sb, l + 3), 1.0);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            gp[(long long)(l + u) * L.pitch] = x[u];
            bad |= is_bad(x[u], a.thr);
          }
        }
        for (; l < ncols; ++l) {
          const double x = flow_sm(a, FP, W[l * RS + 1 + p], solute(sg, sb, l), 1.0);
          gp[(long long)l * L.pitch] = x;
          bad |= is_bad(x, a.thr);
        }
      }
    } else if (plain && RT) {  // rows 1..m: 16-byte chunks (1,2), (3,4), ...; an odd last row alone
      const int nch = m / 2;
      for (int c = tid; c < nch; c += NT) {
        double* g = a.dst + base + 1 + 2 * c;
        const double* w = W + 2 + 2 * c;
        for (int l = 0; l < ncols; ++l, g += L.pitch, w += RS)
          *reinterpret_cast<double2*>(g) = *reinterpret_cast<const double2*>(w);
      }
      if ((m & 1) && tid < ncols) a.dst[lb(tid) + m] = W[sidx(m, tid)];
    } else if (plain) {
      const int q = (tid % CPR) * 2, p0 = 1 + tid / CPR;  // 16-byte chunks
      const long long gstep = (long long)RPP * stride;
      double* g = a.dst + base + p0 * (long long)stride + q;
      const double* w = W + p0 * LB + q;
      if (q + 1 < ncols) {
#pragma unroll 4
        for (int p = p0; p <= m; p += RPP, g += gstep, w += RPP * LB)
          *reinterpret_cast<double2*>(g) = *reinterpret_cast<const double2*>(w);
      } else if (q < ncols) {
        for (int p = p0; p <= m; p += RPP, g += gstep, w += RPP * LB) *g = *w;
      }
    } else {
      const double pm = a.pm;
      switch (epi) {
        case EPI_FLOW:
          loop([&](int c, uint32_t b) { return flow_sm(a, FP, W[c], b, 1.0); });
          break;
        case EPI_AOS0:
          loop([&](int c, uint32_t b) { return __dadd_rn(flow_sm(a, FP, Yt[c], b, pm), W[c]); });
          break;
        case EPI_AOS1:
        case EPI_MAOS1: loop([&](int c, uint32_t) { return __dadd_rn(Yt[c], W[c]); }); break;
        case EPI_AOS2:
          loop([&](int c, uint32_t) { return __dmul_rn(0.25, __dadd_rn(Yt[c], W[c])); });
          break;
        case EPI_MAOS2:
          loop([&](int c, uint32_t) { return __ddiv_rn(__dadd_rn(Yt[c], W[c]), 3.0); });
          break;
        default: loop([&](int c, uint32_t) { return W[c]; }); break;
      }
    }
    if (a.check) {
      if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0) atomicMin(a.div_step + g.b, a.step);
    }
  }
}


// r[j] += v for a runtime j (unrolled selects keep r in registers).
template <int S>
__device__ __forceinline__ void add_at(double (&r)[S], int j, double v) {
#pragma unroll
  for (int k = 0; k < S; ++k)
    if (k == j) r[k] = __dadd_rn(r[k], v);
}

// Sparse charged-node fix-up on register rows: r[j] += coef * rr[j * st] for the set bits of
// cmask (a rolled loop, so the rare source loads are not hoisted into registers).
template <int S>
__device__ __forceinline__ void fix_regs(double (&r)[S], unsigned cmask, double coef,
                                         const double* rr, int st) {
  while (cmask) {
    const int j = __ffs(cmask) - 1;
    cmask &= cmask - 1;
    add_at<S>(r, j, __dmul_rn(coef, rr[j * st]));
  }
}

// Next row of a strided line: the pointer advances by one 64-bit add per row (two integer
// instructions); left to itself the compiler rebuilds every row address from j * stride with
// uniform multiplies, sign extensions and carries (~5.5 instructions per row, 24% of the
// column kernels' instructions, profiles/ncu_r02b).  The empty asm keeps the running pointer
// opaque.
template <typename T>
__device__ __forceinline__ T* next_row(T* p, long long st) {
  p += st;
  asm volatile("" : "+l"(p));
  return p;
}

// Per-tile work of the column kernels once the thread's rows are in registers: r[j] = row
// i0+1+j of the line (rows past m+1 zero), wl / wr = raw rows i0 and i0+S+1 (CN only).
// Prologue, CN explicit half, folds, elimination, reduced system (block-wide barriers: every
// thread of the block calls this), reconstruction, epilogue and the store of rows 1..m.
// MODE 1 ("plain"): no flow and no accumulator operand anywhere (prologue none / source,
// epilogue store / source / MAOS first branch, no divergence test) -- the LOD column sweeps,
// compiled without the other stages so that those do not cost the common path registers.
// MODE 2: the AOS first branch with its grouped flow epilogue.  MODE 0: everything else.
template <int S, int kSegS, bool CN, int LB, int MODE = 0>
__device__ __forceinline__ void col_body(const SweepArgs& a, const TileGeo& g, double (&r)[S],
                                         double wl, double wr, unsigned long long amask,
                                         unsigned long long w1, double bfold, const double* T,
                                         const double* Mi, double* X, const double* FP) {
  constexpr bool PLAIN = MODE == 1;
  const int lane = threadIdx.x, seg = threadIdx.y;
  const int m = a.m, i0 = seg * S;
  const bool act = lane < g.ncols;
  const int st = g.stride;  // 32-bit row offsets: one IMAD.WIDE per address
  const long long gl = g.base + lane;
  const uint32_t sbits = (uint32_t)w1, cmask = (uint32_t)(w1 >> 32);
  const double* rr = a.rho + gl + (long long)(i0 + 1) * st;  // source of row j: rr[j * st]
  // Prologue on the own rows: w = pm*flow(u) or w = u + dta*rho (charged nodes).
  if (!PLAIN && a.pro == PRO_FLOW) {
    const double pm = a.pm;
#pragma unroll
    for (int j = 0; j < S; ++j)
      if (i0 + 1 + j <= m) r[j] = flow_sm(a, FP, r[j], (sbits >> j) & 1u, pm);
    const int jf = m - i0;  // the far face row m+1, if inside this segment: Dirichlet data
    if (CN && act && jf >= 0 && jf < S) {
      const double bh = a.bnd[gl + a.hi_off];
#pragma unroll
      for (int j = 0; j < S; ++j)
        if (j == jf) r[j] = bh;
    }
  } else if (a.pro == PRO_SRC && cmask) {
    fix_regs<S>(r, cmask, a.pro_coef, rr, st);
  }
  if (CN) {  // explicit half along the axis; the rows just outside the segment, prologue applied
    auto outside = [&](int p, double w) {  // w = raw value of row p (0..m+1) of this line
      if (p > m + 1 || !act) return 0.0;
      if (p == 0 || p == m + 1) return a.pro == PRO_FLOW ? a.bnd[gl + (p ? a.hi_off : 0ll)] : w;
      const uint32_t c = a.codes[gl + (long long)p * st];
      if (a.pro == PRO_FLOW) w = flow_sm(a, FP, w, c & 1u, a.pm);
      else if (a.pro == PRO_SRC && ((c >> 4) & 1u))
        w = __dadd_rn(w, __dmul_rn(a.pro_coef, a.rho[gl + (long long)p * st]));
      return w;
    };
    wl = outside(i0, wl);
    wr = outside(i0 + S + 1, wr);
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const double wc = r[j], wn = j + 1 < S ? r[j + 1] : wr;
      r[j] = cn_term(a, (uint32_t)(amask >> j) & 1u, (uint32_t)(amask >> (j + 1)) & 1u, wl, wc,
                     wn);
      wl = wc;
    }
  }
  if (a.has_extra && cmask) fix_regs<S>(r, cmask, a.extra, rr, st);
  if (seg == 0 && act)
    r[0] = __dadd_rn(r[0], __dmul_rn((amask & 1ull) ? a.co.flo[1] : a.co.flo[0], bfold));
  if (seg == (m - 1) / S && act)
    fold_high<S>(a, r, amask, seg == 0 ? a.bnd[gl + a.hi_off] : bfold);

  SegOut o;
  const double* Tv = seg_eliminate<S>(a, r, amask, i0, seg == 0, T, o);
  double t, tm;
  reduced_solve<S, kSegS, LB>(a, o, Mi, X, act, amask, t, tm);
  // Reconstruction in registers: x_j = y_j + alpha_j tm + beta_j t, separator = t.
  if (Tv == nullptr) {
#pragma unroll
    for (int j = 0; j < S - 1; ++j)
      r[j] = fma(a.tmid[TQ_BE * kTabRows + j], t, fma(a.tmid[TQ_AL * kTabRows + j], tm, r[j]));
  } else {
#pragma unroll
    for (int j = 0; j < S - 1; ++j)
      r[j] = fma(Tv[TQ_BE * kTabRows + j], t, fma(Tv[TQ_AL * kTabRows + j], tm, r[j]));
  }
  r[S - 1] = t;
  if (a.epi == EPI_SRC && cmask) fix_regs<S>(r, cmask, a.epi_coef, rr, st);
  if (!act) return;
  if (a.ends) {  // slab phase A (axis 0): only the chunk's end rows 1 and m leave the block
    const long long ei = ends_index(a, g, threadIdx.x);
    if (seg == 0) a.ends[ei] = r[0];
    const int jl = (m - 1) - i0;
#pragma unroll
    for (int j = 0; j < S; ++j)
      if (j == jl) a.ends[ei + a.ends_off] = r[j];
    return;
  }
  // Epilogue and store of the own rows 1..m.
  double* drow = a.dst + gl + (long long)(i0 + 1) * st;
  const int epi = a.epi;
  bool bad = false;
  if (PLAIN || ((epi == EPI_STORE || epi == EPI_SRC || epi == EPI_MAOS0) && !a.check)) {
    if (i0 + S <= m) {  // whole segment inside the line: no per-row predicates
      double* dp = drow;
#pragma unroll
      for (int j = 0; j < S; ++j) {
        *dp = r[j];
        if (j + 1 < S) dp = next_row(dp, st);
      }
    } else {
#pragma unroll
      for (int j = 0; j < S; ++j)
        if (i0 + 1 + j <= m) drow[j * st] = r[j];
    }
  } else if (MODE == 2 && epi == EPI_AOS0) {
    // AOS first branch: pm * flow(u) + b0 (schemes.py:313-323), the flow of four rows at a
    // time (tiny-argument tier interleaved and branch-free, the others one by one) instead of
    // sixteen inlined per-node tier selections
    const double* yrow = a.src + gl + (long long)(i0 + 1) * st;
    const double pm = a.pm;
#pragma unroll
    for (int q = 0; q < S; q += 4) {
      double y[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) y[u] = i0 + 1 + q + u <= m ? yrow[(q + u) * st] : 0.0;
      flow_group(a, FP, y[0], y[1], y[2], y[3], (sbits >> q) & 1u, (sbits >> (q + 1)) & 1u,
                 (sbits >> (q + 2)) & 1u, (sbits >> (q + 3)) & 1u, pm);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (i0 + 1 + q + u > m) continue;
        const double x = __dadd_rn(y[u], r[q + u]);
        drow[(q + u) * st] = x;
        bad |= is_bad(x, a.thr);
      }
    }
  } else {
    const double* yrow = (epi == EPI_AOS0 ? a.src : a.acc) + gl + (long long)(i0 + 1) * st;
    const bool needY = epi_needs(epi) != 0;
    const double pm = a.pm;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      if (i0 + 1 + j > m) continue;
      const uint32_t sb = (sbits >> j) & 1u;
      const double yv = needY ? yrow[j * st] : 0.0;
      double x;
      switch (epi) {
        case EPI_FLOW: x = flow_sm(a, FP, r[j], sb, 1.0); break;
        case EPI_AOS0: x = __dadd_rn(flow_sm(a, FP, yv, sb, pm), r[j]); break;
        case EPI_AOS1:
        case EPI_MAOS1: x = __dadd_rn(yv, r[j]); break;
        case EPI_AOS2: x = __dmul_rn(0.25, __dadd_rn(yv, r[j])); break;
        case EPI_MAOS2: x = __ddiv_rn(__dadd_rn(yv, r[j]), 3.0); break;
        default: x = r[j]; break;
      }
      drow[j * st] = x;
      bad |= is_bad(x, a.thr);
    }
  }
  if (!PLAIN && a.check && bad) atomicMin(a.div_step + g.b, a.step);
}

// Stage the block's tables (uniform-segment LU tables, clean-line inverse, flow palette and
// interval tables) with cp.async; the caller commits.
template <int kSegS>
__device__ __forceinline__ void stage_tables(const SweepArgs& a, double* T, double* Mi,
                                             double* FP, int tid, int NT) {
  for (int c = tid; c < kTabDoubles / 2; c += NT) cp_async16(T + 2 * c, a.tab + 2 * c);
  if (a.static_ok)
    for (int c = tid; c < kSegS * (kSegS + 2) / 2; c += NT) cp_async16(Mi + 2 * c, a.minv + 2 * c);
  if (uses_flow(a.pro, a.epi))
    for (int c = tid; c < a.fpoly_n / 2; c += NT) cp_async16(FP + kFlowHdr + 2 * c, a.fpoly + 2 * c);
}

template <int kSegS>
__device__ __forceinline__ const unsigned long long* col_desc(const SweepArgs& a,
                                                              const TileGeo& g) {
  return a.desc + g.b * a.dstride +
         2 * (((long long)(g.outer - 1) * kSegS + threadIdx.y) * (a.L.n2 - 2) +
                       (g.c0 - 1 + threadIdx.x));
}

// Column sweeps without a staged tile (axes 0 and 1).  Thread (lane, seg) loads the S rows
// of its segment straight into registers -- one warp-wide load covers two 128-byte row
// chunks of 16 adjacent columns -- eliminates, joins the block-wide reduced system, and
// stores its rows back from registers.  Shared memory holds only the tables and the
// reduced-system scratch.  Block (LB columns, kSegS segments), grid (column groups, outer).
template <int S, int kSegS, bool CN, int LB, int MODE>
__global__ void __launch_bounds__(LB * kSegS, S >= 32 ? 1 : 1024 / (LB * kSegS))
    k_sweep_col(const SweepArgs a, const int axis) {
  constexpr bool PLAIN = MODE == 1;
  extern __shared__ double sm[];
  constexpr int NT = LB * kSegS;
  const int dstep = a.div_step ? *((volatile int*)(a.div_step + blockIdx.z)) : INT_MAX;
  const int tid = threadIdx.y * LB + threadIdx.x;
  const TileGeo g = tile_geo<LB, false>(a, axis, blockIdx.x, blockIdx.y, gridDim.y, blockIdx.z);
  const int m = a.m, i0 = threadIdx.y * S;
  const bool act = threadIdx.x < g.ncols;
  const int st = g.stride;
  const long long gl = g.base + threadIdx.x;
  unsigned long long amask = 0ull, w1 = 0ull;
  if (act) {  // word 1 (solute / charged bits) only where a prologue or epilogue needs it
    const unsigned long long* dp = col_desc<kSegS>(a, g);
    if (a.pro != PRO_NONE || a.has_extra || a.epi != EPI_STORE) {
      const ulonglong2 dd = *reinterpret_cast<const ulonglong2*>(dp);
      amask = dd.x;
      w1 = dd.y;
    } else {
      amask = *dp;
    }
  }
  double r[S];
  const double* srow = a.src + gl + (long long)(i0 + 1) * st;
  if (act && i0 + S <= m + 1) {  // whole segment inside rows 1..m+1: no per-row predicates
    const double* sp = srow;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      r[j] = *sp;
      if (j + 1 < S) sp = next_row(sp, st);
    }
  } else {
#pragma unroll
    for (int j = 0; j < S; ++j) r[j] = (act && i0 + 1 + j <= m + 1) ? srow[j * st] : 0.0;
  }
  double wl = 0.0, wr = 0.0;
  if (CN && act) {
    if (i0 <= m + 1) wl = a.src[gl + (long long)i0 * st];
    if (i0 + S + 1 <= m + 1) wr = a.src[gl + (long long)(i0 + S + 1) * st];
  }
  double bfold = 0.0;
  if (act) {
    if (threadIdx.y == 0) bfold = a.bnd[gl];
    else if ((int)threadIdx.y == (m - 1) / S) bfold = a.bnd[gl + a.hi_off];
  }
  if (act) {
    // A general segment's factor tables (five 120-byte rows, L2 resident) start towards L1
    // while the rows load: the elimination reads them on its dependent chain.  After the other
    // loads in program order: the test waits for the descriptor, and ahead of them it held
    // the row loads back by that latency (slab phase A +10%, config 5 +3%).
    if (const unsigned long long slot = amask >> kSlotShift) {
      const double* tp = a.gfac + (long long)(slot - 1ull) * 5 * kTabRows;
#pragma unroll
      for (int q = 0; q < 5; ++q) asm volatile("prefetch.global.L1 [%0];" ::"l"(tp + q * kTabRows));
    }
  }
  if (!PLAIN && epi_needs(a.epi) == 2 && act) {  // accumulator rows of the AOS / MAOS epilogue: on their
                                       // way to L1 while the line is solved
    const double* yp = a.acc + gl + (long long)(i0 + 1) * st;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      if (i0 + 1 + j <= m) asm volatile("prefetch.global.L1 [%0];" ::"l"(yp));
      if (j + 1 < S) yp = next_row(yp, st);
    }
  }
  // The uniform-segment tables stay in global memory (7.7 KB, L1-resident): only warps
  // with a non-solvent or general segment read them, the dominant kind comes from the
  // kernel parameters, and staging them per block cost 7% of the kernel's instructions.
  double* Mi = sm;
  double* X = Mi + kSegS * (kSegS + 2);
  double* FP = X + 4 * NT;
  if (a.static_ok)
    for (int c = tid; c < kSegS * (kSegS + 2) / 2; c += NT) cp_async16(Mi + 2 * c, a.minv + 2 * c);
  if (!PLAIN && uses_flow(a.pro, a.epi))
    for (int c = tid; c < a.fpoly_n / 2; c += NT) cp_async16(FP + kFlowHdr + 2 * c, a.fpoly + 2 * c);
  cp_async_wait_all();
  __syncthreads();
  if (dstep < a.step) return;  // an earlier step diverged: nothing more to compute
  col_body<S, kSegS, CN, LB, MODE>(a, g, r, wl, wr, amask, w1, bfold, a.tab, Mi, X, FP);
}

// ---------------------------------------------------------------------------------------
// Fused axis-0 + axis-1 column sweeps of a LOD step (schemes.py:301-311, order kept).  The
// lines of both families lie inside a k-slab (a group of adjacent k columns, all i and j),
// and a slab of 16-64 columns is a few tens of MB: one persistent launch runs the axis-0
// tiles of slab x and, `lag` slabs later, the axis-1 tiles of slab x, which find the axis-0
// output in L2 and store in place over it, so that the intermediate field never travels to
// HBM and back.  Both parts are the register-direct column tile of k_sweep_col (same block
// shape, same 64 registers, four blocks per SM), so the fusion costs no occupancy.  Blocks
// take items from a global queue whose order is the dependency order (an item only waits
// for earlier items, all held by running blocks: no deadlock); an axis-0 tile publishes its
// slab with a fence + counter increment, an axis-1 tile spins (one thread, acquire loads)
// until its slab's counter reaches the tiles per slab.  Within a slab the tiles run with the
// column group fastest, so concurrently running tiles read adjacent 128-byte row chunks.
struct Fuse01Ctl {
  int* q;       // q[0] next item, q[1] blocks that left, q[2 + x] finished axis-0 tiles of slab x
  int nslab;    // slabs
  int tw;       // column groups (of LB columns) per slab
  int ntx;      // column groups in all
  int n0i, n1i; // outer indices: axis-0 tiles per column group (n1 - 2), axis-1 (n0 - 2)
  int lag;      // slabs of axis-0 tiles queued ahead of the axis-1 tiles (1 <= lag <= nslab)
};

template <int S, int kSegS, int LB>
__device__ __forceinline__ void col_tile_run(const SweepArgs& a, int axis, int tx, int outer,
                                             const double* Mi, double* X, const double* FP) {
  TileGeo g;
  g.b = 0;
  g.c0 = 1 + tx * LB;
  g.outer = outer;
  g.ncols = min(LB, (a.L.n2 - 2) + 1 - g.c0);
  if (axis == 0) {
    g.base = a.L.at(0, outer, g.c0);
    g.stride = (int)a.L.s0;
  } else {
    g.base = a.L.at(outer, 0, g.c0);
    g.stride = (int)a.L.pitch;
  }
  const int m = a.m, i0 = threadIdx.y * S, st = g.stride;
  const bool act = (int)threadIdx.x < g.ncols;
  const long long gl = g.base + threadIdx.x;
  unsigned long long amask = 0ull, w1 = 0ull;
  if (act) {
    const unsigned long long* dp = col_desc<kSegS>(a, g);
    if (a.pro != PRO_NONE || a.has_extra || a.epi != EPI_STORE) {
      const ulonglong2 dd = *reinterpret_cast<const ulonglong2*>(dp);
      amask = dd.x;
      w1 = dd.y;
    } else {
      amask = *dp;
    }
  }
  double r[S];
  const double* srow = a.src + gl + (long long)(i0 + 1) * st;
  if (act && i0 + S <= m + 1) {
    const double* sp = srow;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      r[j] = *sp;
      if (j + 1 < S) sp = next_row(sp, st);
    }
  } else {
#pragma unroll
    for (int j = 0; j < S; ++j) r[j] = (act && i0 + 1 + j <= m + 1) ? srow[j * st] : 0.0;
  }
  double bfold = 0.0;
  if (act) {
    if (threadIdx.y == 0) bfold = a.bnd[gl];
    else if ((int)threadIdx.y == (m - 1) / S) bfold = a.bnd[gl + a.hi_off];
  }
  col_body<S, kSegS, false, LB>(a, g, r, 0.0, 0.0, amask, w1, bfold, a.tab, Mi, X, FP);
}

template <int S, int kSegS, int LB>
__global__ void __launch_bounds__(LB * kSegS, S >= 32 ? 1 : 1024 / (LB * kSegS))
    k_sweep_fused01(const SweepArgs a0, const SweepArgs a1, const Fuse01Ctl c) {
  extern __shared__ double sm[];
  constexpr int NT = LB * kSegS, MD = kSegS * (kSegS + 2);
  __shared__ int s_item;
  const int tid = threadIdx.y * LB + threadIdx.x;
  const int dstep = a0.div_step ? *((volatile int*)a0.div_step) : INT_MAX;
  double* Mi0 = sm;
  double* Mi1 = Mi0 + MD;
  double* X = Mi1 + MD;
  double* FP = X + 4 * NT;
  if (a0.static_ok)
    for (int t = tid; t < MD / 2; t += NT) cp_async16(Mi0 + 2 * t, a0.minv + 2 * t);
  if (a1.static_ok)
    for (int t = tid; t < MD / 2; t += NT) cp_async16(Mi1 + 2 * t, a1.minv + 2 * t);
  if (uses_flow(a0.pro, a0.epi))
    for (int t = tid; t < a0.fpoly_n / 2; t += NT) cp_async16(FP + kFlowHdr + 2 * t, a0.fpoly + 2 * t);
  if (dstep < a0.step) {  // an earlier step diverged: nothing more to compute
    cp_async_wait_all();
    return;
  }
  if (tid == 0) s_item = atomicAdd(c.q, 1);
  cp_async_wait_all();
  __syncthreads();

  const int per0 = c.tw * c.n0i, per1 = c.tw * c.n1i, per = per0 + per1;
  const int nitems = c.nslab * per;  // laid out as if every slab had c.tw column groups
  const int head = c.lag * per0, full = c.nslab - c.lag;
  int item = s_item;
  while (item < nitems) {
    int nxt = 0;
    if (tid == 0) nxt = atomicAdd(c.q, 1);  // claimed now, taken up when this item is done
    // queue order: axis-0 tiles of slabs 0..lag-1, then for slab x: its axis-1 tiles, the
    // axis-0 tiles of slab x+lag.  The last slab may be narrower: the queue is laid out as if
    // every slab had c.tw groups and items of missing groups are skipped.
    int kind, slab, w;
    if (item < head) {
      kind = 0;
      slab = item / per0;
      w = item - slab * per0;
    } else {
      const int r = item - head;
      if (r < full * per) {
        const int grp = r / per, v = r - grp * per;
        kind = v < per1 ? 1 : 0;
        slab = v < per1 ? grp : grp + c.lag;
        w = v < per1 ? v : v - per1;
      } else {
        const int r2 = r - full * per;
        kind = 1;
        slab = full + r2 / per1;
        w = r2 - (slab - full) * per1;
      }
    }
    const int outer = 1 + w / c.tw, tx = slab * c.tw + (w - (outer - 1) * c.tw);
    const bool exists = tx < c.ntx;
    if (kind == 0) {
      if (exists) col_tile_run<S, kSegS, LB>(a0, 0, tx, outer, Mi0, X, FP);
      if (tid == 0) s_item = nxt;
      __syncthreads();  // every store of the tile is issued; the scratch is free again
      if (tid == 0) {
        __threadfence();
        atomicAdd(c.q + 2 + slab, 1);
      }
    } else {
      if (tid == 0) {
        const int* d = c.q + 2 + slab;
        while (ld_acquire(d) < per0) __nanosleep(64);
      }
      __syncthreads();
      if (exists) col_tile_run<S, kSegS, LB>(a1, 1, tx, outer, Mi1, X, FP);
      if (tid == 0) s_item = nxt;
      __syncthreads();
    }
    item = s_item;
  }
  // The last block to leave resets the queue for the next launch.
  __syncthreads();
  if (tid == 0) s_item = atomicAdd(c.q + 1, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (s_item)
    for (int t = tid; t < 2 + c.nslab; t += NT) c.q[t] = 0;
}

// Staged-tile kernel: block (x = column / row group, y = outer index).  Serves the row
// sweeps (axis 2) and, with PBG_COL=0, the column sweeps.
template <int S, int kSegS, bool CN, int LB, bool RT>
__global__ void __launch_bounds__(LB * kSegS, LB * kSegS <= 128 ? 6 : (LB * kSegS <= 256 ? 3 : 2))
    k_sweep_strided(const SweepArgs a, const int axis, const int ntx, const int nty) {
  extern __shared__ double sm[];
  using TS = TileShape<S, kSegS, LB, RT>;
  constexpr int NT = TS::NT, TD = TS::TD;
  const int dstep = a.div_step ? *((volatile int*)a.div_step) : INT_MAX;
  const int tid = threadIdx.y * LB + threadIdx.x;
  const int needY = epi_needs(a.epi);
  double* T = sm;
  double* Mi = T + kTabDoubles;
  double* W = Mi + kSegS * (kSegS + 2);
  double* Yt = W + TD;
  double* X = Yt + (needY ? TD : 0);
  unsigned long long* D = reinterpret_cast<unsigned long long*>(X + 4 * NT);
  double* FP = reinterpret_cast<double*>(D + 2 * NT);  // flow tables at FP + kFlowHdr
  // The tables once per block; the block then walks tiles blockIdx.x, + gridDim.x, ...
  for (int c = tid; c < kTabDoubles / 2; c += NT) cp_async16(T + 2 * c, a.tab + 2 * c);
  if (a.static_ok)
    for (int c = tid; c < kSegS * (kSegS + 2) / 2; c += NT) cp_async16(Mi + 2 * c, a.minv + 2 * c);
  if (uses_flow(a.pro, a.epi))
    for (int c = tid; c < a.fpoly_n / 2; c += NT) cp_async16(FP + kFlowHdr + 2 * c, a.fpoly + 2 * c);
  asm volatile("cp.async.commit_group;\n" ::);
  if (a.L.nb == 1 && dstep < a.step) {  // an earlier step diverged: nothing more to compute
    cp_async_wait_all();
    return;
  }
  const int per = ntx * nty, ntiles = per * a.L.nb;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int b = tile / per, tl = tile - b * per;
    if (a.L.nb > 1 && a.div_step && a.div_step[b] < a.step) continue;  // grid b stopped
    const TileGeo g = tile_geo<LB, RT>(a, axis, tl % ntx, tl / ntx, nty, b);
    stage_tile<S, kSegS, LB, RT>(a, g, W, Yt, D, needY);
    asm volatile("cp.async.commit_group;\n" ::);
    cp_async_wait_all();
    const double bfold = tile_prefetch<S, kSegS, LB, RT>(a, g, D);
    __syncthreads();
    tile_body<S, kSegS, CN, LB, RT>(a, g, T, Mi, W, Yt, X, D, FP, bfold);
    __syncthreads();  // the tile buffers are restaged by the next iteration
  }
  cp_async_wait_all();  // a block whose tiles all belonged to stopped grids
}

// ---------------------------------------------------------------------------------------
// Row sweeps (axis 2) with G = 32 or 16 lanes per line, for lines of m = G*S - 1 interior
// rows (n2 = 65, 129, 257, 513) and the LOD epilogues (store, LODIE1 source, LODIE2 flow).
// Lane `seg` of a line owns segment seg (rows seg*S+1 .. seg*S+S; the last separator is the
// far face, a padding row), so the reduced system over the G separators is solved inside the
// warp (clean lines: the static inverse, one dot product; others: PCR with shuffles).  Warps
// never wait for one another: after the block stages its tables, each warp stages its own
// 32/G lines (cp.async, 16-byte chunks, segments padded by two doubles so that the lanes'
// 16-byte row loads are conflict-free), solves them, and stores them in coalesced 256-byte
// row runs, then takes the next lines.  Descriptors are line-major here (G per line).
constexpr int kRWarps = 8;

// Line-major descriptor index of axis-2 line (i, j).
__device__ __forceinline__ long long line_desc(const Layout& L, int i, int j) {
  return (long long)(i - 1) * (L.n1 - 2) + (j - 1);
}

template <int S, int G>
struct RowWarp {
  static constexpr int NL = 32 / G;         // lines per warp
  static constexpr int SP = S + 2;          // padded segment stride (doubles)
  static constexpr int LW = G * SP + 2;     // one line buffer (rows 1..G*S at pos(p))
  static constexpr int RW = G + 2;          // separator scratch of one line
  static constexpr int WD = NL * (LW + RW); // per-warp doubles
  __device__ static __forceinline__ int pos(int p) {  // p = 1..G*S
    return 2 + (p - 1) + 2 * ((p - 1) / S);
  }
};

__host__ __device__ constexpr size_t rowwarp_smem(int S, int G, int fpoly_n) {
  return sizeof(double) * (kTabDoubles + G * (G + 2) +
                           (size_t)kRWarps * (32 / G) * (G * (S + 2) + 2 + G + 2) + kFlowHdr +
                           fpoly_n);
}

// Line solve of the row-warp sweeps once lane `seg` holds rows seg*S+1 .. seg*S+S of its line
// in r[]: Dirichlet folds, segment elimination, the reduced system over the G separators of
// the line inside the warp (clean lines: the static inverse, one dot product; others: PCR with
// shuffles), reconstruction (separator = t) and the LODIE1 sparse source.  sR: G + 2 doubles
// of per-line scratch.
template <int S, int G>
__device__ __forceinline__ void rw_solve(const SweepArgs& a, double (&r)[S],
                                         unsigned long long amask, uint32_t cmask, double bfold,
                                         bool valid, int seg, const double* T, const double* Mi,
                                         double* sR, long long base) {
  constexpr unsigned FULL = 0xffffffffu;
  const int m = a.m, i0 = seg * S;
  if (seg == 0 && valid)
    r[0] = __dadd_rn(r[0], __dmul_rn((amask & 1ull) ? a.co.flo[1] : a.co.flo[0], bfold));
  if (seg == (m - 1) / S && valid)
    fold_high<S>(a, r, amask, seg == 0 ? a.bnd[base + a.hi_off] : bfold);
  SegOut o;
  const double* Tv = seg_eliminate<S>(a, r, amask, i0, seg == 0, T, o);

  // reduced system over the G separators of each line
  double t, tm;
  const bool nx = seg + 1 < G;
  const double yFn = __shfl_down_sync(FULL, o.yF, 1, G);
  const bool clean = __all_sync(FULL, eps_bits(amask, S) == 0ull) && a.static_ok;
  if (clean) {
    sR[seg] = o.rs - o.as * o.yL - o.cs * (nx ? yFn : 0.0);
    __syncwarp();
    const double2* Rr = reinterpret_cast<const double2*>(sR);
    const double2* Mr = reinterpret_cast<const double2*>(Mi + seg * (G + 2));
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int q = 0; q < G / 2; q += 2) {
      const double2 r0 = Rr[q], m0 = Mr[q], r1 = Rr[q + 1], m1 = Mr[q + 1];
      s0 = fma(m0.x, r0.x, s0);
      s1 = fma(m0.y, r0.y, s1);
      s2 = fma(m1.x, r1.x, s2);
      s3 = fma(m1.y, r1.y, s3);
    }
    t = (s0 + s1) + (s2 + s3);
  } else {  // parallel cyclic reduction with shuffles
    const double aFn = __shfl_down_sync(FULL, o.aF, 1, G);
    const double bFn = __shfl_down_sync(FULL, o.bF, 1, G);
    double A = o.as * o.aL, B = o.bs + o.as * o.bL + o.cs * (nx ? aFn : 0.0),
           Cc = o.cs * (nx ? bFn : 0.0), R = o.rs - o.as * o.yL - o.cs * (nx ? yFn : 0.0);
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
      const double iB = fast_rcp(B);
      const double Am = __shfl_up_sync(FULL, A, d, G), iBm = __shfl_up_sync(FULL, iB, d, G),
                   Cm = __shfl_up_sync(FULL, Cc, d, G), Rm = __shfl_up_sync(FULL, R, d, G);
      const double Ap = __shfl_down_sync(FULL, A, d, G), iBp = __shfl_down_sync(FULL, iB, d, G),
                   Cp = __shfl_down_sync(FULL, Cc, d, G), Rp = __shfl_down_sync(FULL, R, d, G);
      const bool lo = seg >= d, hi = seg + d < G;
      const double k1 = lo ? -A * iBm : 0.0, k2 = hi ? -Cc * iBp : 0.0;
      A = lo ? k1 * Am : 0.0;
      Cc = hi ? k2 * Cp : 0.0;
      B = B + (lo ? k1 * Cm : 0.0) + (hi ? k2 * Ap : 0.0);
      R = R + (lo ? k1 * Rm : 0.0) + (hi ? k2 * Rp : 0.0);
    }
    t = R * fast_rcp(B);
  }
  tm = __shfl_up_sync(FULL, t, 1, G);
  if (seg == 0) tm = 0.0;

  // reconstruct the own rows (separator = t) and put them back into the line buffer
  if (Tv == nullptr) {
#pragma unroll
    for (int q = 0; q < S - 1; ++q)
      r[q] = fma(a.tmid[TQ_BE * kTabRows + q], t, fma(a.tmid[TQ_AL * kTabRows + q], tm, r[q]));
  } else {
#pragma unroll
    for (int q = 0; q < S - 1; ++q)
      r[q] = fma(Tv[TQ_BE * kTabRows + q], t, fma(Tv[TQ_AL * kTabRows + q], tm, r[q]));
  }
  r[S - 1] = t;
  if (a.epi == EPI_SRC && cmask) fix_regs<S>(r, cmask, a.epi_coef, a.rho + base + i0 + 1, 1);
}

// Epilogue + coalesced store of rows 1..m of the warp's lines from the line buffer (at(p) =
// row p): the G lanes of a line take consecutive rows (G * 8 = 128- or 256-byte runs), each
// lane S of them; an idle sub-warp (odd line count) joins the shuffles but stores nothing.
// Divergence test of the row-warp store pass (non-finite, or |x| above the threshold,
// schemes.py:417-421): one compare with the hoisted clamped threshold per node (an fmax
// accumulator measured 9% of the kernel's instructions: fp64 fmax is a compare-select chain).
struct DivAcc {
  double thr;       // threshold clamped to DBL_MAX: +-inf and NaN fail the one comparison
  bool b = false;
  __device__ __forceinline__ explicit DivAcc(double t) : thr(fmin(t, 1.7976931348623157e308)) {}
  __device__ __forceinline__ void add(double x) { b |= !(fabs(x) <= thr); }
  __device__ __forceinline__ bool bad(double) const { return b; }
};

// Epilogue + coalesced store of rows 1..m of the warp's lines from the line buffer (at(p) =
// row p): the G lanes of a line take consecutive rows (G * 8 = 128- or 256-byte runs), each
// lane S of them; an idle sub-warp (odd line count) stores nothing.  Row-warp lines have
// m + 1 = G*S rows, so only the last lane's last row (the far face) is skipped.  sbits: the
// lane's solute bits in store order (row-warp descriptors, k_build_desc).
template <int S, int G, typename At>
__device__ __forceinline__ void rw_store(const SweepArgs& a, At at, bool valid, int seg,
                                         uint32_t sbits, const double* FP, long long base,
                                         DivAcc& acc) {
  double* gdst = a.dst + base;
  auto inside = [&](int q) { return q < S - 1 || seg < G - 1; };  // p <= m = G*S - 1
  if (a.epi == EPI_FLOW) {  // the tiny-argument form for almost every node
    constexpr int S4 = S & ~3;
#pragma unroll
    for (int q = S4; q < S; ++q) {  // rows past the last group of four
      double x = at(1 + seg + G * q);
      x = flow_sm(a, FP, x, (sbits >> q) & 1u, 1.0);
      if (valid && inside(q)) {
        gdst[1 + seg + G * q] = x;
        acc.add(x);
      }
    }
#pragma unroll 1
    for (int q = 0; q < S4; q += 4) {
      double x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = at(1 + seg + G * (q + u));
      flow_group(a, FP, x[0], x[1], x[2], x[3], (sbits >> q) & 1u, (sbits >> (q + 1)) & 1u,
                 (sbits >> (q + 2)) & 1u, (sbits >> (q + 3)) & 1u, 1.0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (valid && inside(q + u)) {
          gdst[1 + seg + G * (q + u)] = x[u];
          acc.add(x[u]);
        }
      }
    }
  } else if (a.epi == EPI_AOS2) {  // AOS: 0.25 * (accumulated branches + this branch),
                                   // read and written in place, same rounding as tiles
    const double* gy = a.acc + base;
#pragma unroll
    for (int q = 0; q < S; ++q) {
      const int p = 1 + seg + G * q;
      if (valid && inside(q)) {
        const double x = __dmul_rn(0.25, __dadd_rn(gy[p], at(p)));
        gdst[p] = x;
        if (a.check) acc.add(x);
      }
    }
  } else {
#pragma unroll
    for (int q = 0; q < S; ++q) {
      const int p = 1 + seg + G * q;
      if (valid && inside(q)) {
        const double x = at(p);
        gdst[p] = x;
        if (a.check) acc.add(x);
      }
    }
  }
}

template <int S, int G, bool BATCH>
__global__ void __launch_bounds__(kRWarps * 32, 3)
    k_sweep_rowwarp(const SweepArgs a, const int nlines) {
  extern __shared__ double sm[];
  using RW = RowWarp<S, G>;
  constexpr int NL = RW::NL;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int NT = kRWarps * 32;
  const int dstep = a.div_step ? *((volatile int*)a.div_step) : INT_MAX;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sub = lane / G, seg = lane % G;
  double* T = sm;
  double* Mi = T + kTabDoubles;             // G x (G + 2) (rows padded)
  double* Wb = Mi + G * (G + 2);
  double* FP = Wb + kRWarps * RW::WD;       // flow tables at FP + kFlowHdr
  for (int c = tid; c < kTabDoubles / 2; c += NT) cp_async16(T + 2 * c, a.tab + 2 * c);
  if (a.static_ok)
    for (int c = tid; c < G * (G + 2) / 2; c += NT) cp_async16(Mi + 2 * c, a.minv + 2 * c);
  if (uses_flow(a.pro, a.epi))
    for (int c = tid; c < a.fpoly_n / 2; c += NT) cp_async16(FP + kFlowHdr + 2 * c, a.fpoly + 2 * c);
  asm volatile("cp.async.commit_group;\n" ::);
  cp_async_wait_all();
  __syncthreads();
  if (a.L.nb == 1 && dstep < a.step) return;  // an earlier step diverged: nothing more to compute

  const Layout& L = a.L;
  const int m = a.m, K = L.n1 - 2, i0 = seg * S;
  const int itop = a.on ? a.o0 + a.on : L.n0 - 2;  // planes itop, itop-1, ... (reverse)
  double* W = Wb + warp * RW::WD + sub * RW::LW;          // this lane's line
  double* sR = Wb + warp * RW::WD + NL * RW::LW + sub * RW::RW;
  DivAcc acc(a.thr);
  const int nlp = BATCH ? nlines / L.nb : nlines;  // lines per grid (batched: nb grids)
  for (int wl = blockIdx.x * kRWarps + warp; wl * NL < nlines; wl += gridDim.x * kRWarps) {
    const int line = wl * NL + sub;
    const int b = BATCH && line < nlines ? line / nlp : 0, ln = line - b * nlp;
    // NL == 1: the loop condition; batched: grids that stopped at an earlier step are skipped
    const bool valid = (NL == 1 || line < nlines) &&
                       (!BATCH || !a.div_step || a.div_step[b] >= a.step);
    // planes in reverse (the axis-1 sweep before this one wrote the last planes last)
    const int i = valid ? itop - ln / K : 1, j = valid ? 1 + ln % K : 1;
    const long long base = L.at(i, j, 0) + (long long)b * L.bs;
    unsigned long long amask = 0ull;
    uint32_t sbits = 0u, cmask = 0u;
    double bfold = 0.0;
    if (valid) {
      // stage rows 1..G*S (row G*S = m+1, the far face) in 16-byte chunks
      const double* gsrc = a.src + base + 1;
#pragma unroll
      for (int q = 0; q < S / 2; ++q) {
        const int c = seg + G * q;  // chunk c: rows 2c+1, 2c+2 (one segment, S even)
        cp_async16(W + RW::pos(2 * c + 1), gsrc + 2 * c);
      }
      const ulonglong2 dd = *reinterpret_cast<const ulonglong2*>(
          a.desc + b * a.dstride + 2 * (line_desc(L, i, j) * G + seg));
      amask = dd.x;
      sbits = (uint32_t)dd.y;
      cmask = (uint32_t)(dd.y >> 32);
      if (seg == 0) bfold = a.bnd[base];
      else if (seg == (m - 1) / S) bfold = a.bnd[base + a.hi_off];
      if (a.epi == EPI_AOS2)  // the accumulated branches of this line, read by the store pass
        for (int c = seg; c < G * S / 16; c += G)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(a.acc + base + 1 + 16 * c));
    }
    asm volatile("cp.async.commit_group;\n" ::);
    {  // the warp's next lines towards L2 while this one is solved (LODIE1 c4: 533 -> 498 us)
      const int nl = (wl + gridDim.x * kRWarps) * NL + sub;
      if (nl < nlines) {
        const int nb2 = BATCH ? nl / nlp : 0, nn = nl - nb2 * nlp;
        const double* np = a.src + L.at(itop - nn / K, 1 + nn % K, 0) + (long long)nb2 * L.bs + 1;
        for (int c = seg; c < G * S / 16; c += G)  // 128-byte lines
          asm volatile("prefetch.global.L2 [%0];" ::"l"(np + 16 * c));
      }
    }
    cp_async_wait_all();
    __syncwarp();

    double r[S];
#pragma unroll
    for (int q = 0; q < S; q += 2) {
      const double2 v = valid ? *reinterpret_cast<const double2*>(W + 2 + seg * RW::SP + q)
                              : make_double2(0.0, 0.0);
      r[q] = v.x;
      r[q + 1] = v.y;
    }
    rw_solve<S, G>(a, r, amask, cmask, bfold, valid, seg, T, Mi, sR, base);
    if (valid) {
#pragma unroll
      for (int q = 0; q < S; q += 2)
        *reinterpret_cast<double2*>(W + 2 + seg * RW::SP + q) = make_double2(r[q], r[q + 1]);
    }
    __syncwarp();

    if (G % S == 0) {  // rows 1 + seg + G*k sit at pos(1 + seg) + k*(G + 2G/S): no division
      const int p0 = RW::pos(1 + seg);
      rw_store<S, G>(a, [&](int p) { return W[p0 + ((p - 1 - seg) / G) * (G + 2 * G / S)]; },
                     valid, seg, sbits, FP, base, acc);
    } else {
      rw_store<S, G>(a, [&](int p) { return W[RW::pos(p)]; }, valid, seg, sbits, FP, base, acc);
    }
    if (BATCH && a.check) {  // batched: the line's own grid (lines of a warp may differ)
      if (acc.bad(a.thr)) atomicMin(a.div_step + b, a.step);
      acc = DivAcc(a.thr);
    }
    __syncwarp();  // the line buffers are restaged by the next lines
  }
  if (!BATCH && a.check && __any_sync(FULL, acc.bad(a.thr)) && lane == 0)
    atomicMin(a.div_step, a.step);
}

// ---------------------------------------------------------------------------------------
// Row sweeps (axis 2) with TMA staging: the same per-warp line solve as k_sweep_rowwarp, but
// each line is brought into shared memory by ONE tensor copy (cp.async.bulk.tensor, a box of
// G*S/16 128-byte chunks of the line, 128-byte swizzle) completing on an mbarrier, and every
// warp keeps two line buffers: the copy of its next line is in flight while the current one
// is solved and stored.  The swizzle (16-byte unit u of 128-byte chunk c lands at unit
// u ^ (c & 7)) keeps the lanes' 16-byte segment-row reads and the coalesced store pass free
// of bank conflicts without padding, so one contiguous copy per line suffices.
// Shared memory: [NW warps x 2 buffers x NL lines x G*S doubles, 1024-aligned] | tables |
// reduced inverse | per-line separator scratch | flow tables | mbarriers.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1,
                                            int c2, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(tm)), "r"(c0), "r"(c1), "r"(c2),
      "r"(smem_u32(bar))
      : "memory");
}

// Swizzled position of row e (0-based, e = p - 1) in a line buffer of 16-double chunks.
__device__ __forceinline__ int swz(int e) {
  const int c = e >> 4;
  return (c << 4) | ((((e >> 1) & 7) ^ (c & 7)) << 1) | (e & 1);
}

template <int S, int G, int NW>
struct RowTma {
  static constexpr int NL = 32 / G;        // lines per warp
  static constexpr int LD = G * S;         // doubles per line buffer (rows 1..m+1)
  static constexpr int WB = NL * LD;       // doubles per warp buffer
  static constexpr size_t lines_bytes = (size_t)NW * 2 * WB * sizeof(double);
  static constexpr size_t smem(int fpoly_n) {
    return 1024 + lines_bytes +
           sizeof(double) * (kTabDoubles + G * (G + 2) + NW * NL * (G + 2) + kFlowHdr + fpoly_n) +
           sizeof(unsigned long long) * NW * 2;
  }
};

template <int S, int G, int NW, bool BATCH>
__global__ void __launch_bounds__(NW * 32, 1)
    k_sweep_rowtma(const SweepArgs a, const int nlines, const __grid_constant__ CUtensorMap tm) {
  static_assert(S == 16, "one 128-byte chunk per segment");
  extern __shared__ unsigned char smraw[];
  using RT = RowTma<S, G, NW>;
  constexpr int NL = RT::NL, LD = RT::LD, WB = RT::WB;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int NT = NW * 32;
  const int dstep = a.div_step ? *((volatile int*)a.div_step) : INT_MAX;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sub = lane / G, seg = lane % G;
  double* Lb = reinterpret_cast<double*>(
      smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u));  // 1024-aligned line buffers
  double* T = Lb + NW * 2 * WB;
  double* Mi = T + kTabDoubles;         // G x (G + 2)
  double* sRb = Mi + G * (G + 2);       // NW * NL * (G + 2)
  double* FP = sRb + NW * NL * (G + 2);  // flow tables at FP + kFlowHdr
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(FP + kFlowHdr + a.fpoly_n + (a.fpoly_n & 1));
  for (int c = tid; c < kTabDoubles / 2; c += NT) cp_async16(T + 2 * c, a.tab + 2 * c);
  if (a.static_ok)
    for (int c = tid; c < G * (G + 2) / 2; c += NT) cp_async16(Mi + 2 * c, a.minv + 2 * c);
  if (uses_flow(a.pro, a.epi))
    for (int c = tid; c < a.fpoly_n / 2; c += NT) cp_async16(FP + kFlowHdr + 2 * c, a.fpoly + 2 * c);
  asm volatile("cp.async.commit_group;\n" ::);
  if (tid < NW * 2) mbar_init(bars + tid, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  cp_async_wait_all();
  __syncthreads();
  if (a.L.nb == 1 && dstep < a.step) return;  // an earlier step diverged: nothing more to compute

  const Layout& L = a.L;
  const int m = a.m, K = L.n1 - 2;
  const int itop = a.on ? a.o0 + a.on : L.n0 - 2;  // planes itop, itop-1, ... (reverse)
  double* sR = sRb + (warp * NL + sub) * (G + 2);
  unsigned long long* bar = bars + warp * 2;
  const int stride = gridDim.x * NW;
  const int wl0 = blockIdx.x * NW + warp;
  // lane 0: one tensor copy per valid line of warp-iteration wl into buffer b
  const int nlp = BATCH ? nlines / L.nb : nlines;  // lines per grid (batched: nb grids)
  const long long grid_lines = BATCH ? L.bs / L.pitch : 0;  // tensor-map lines between grids
  auto issue = [&](int wl, int b) {
    int nv = 0;
#pragma unroll
    for (int l = 0; l < NL; ++l) nv += wl * NL + l < nlines;
    mbar_expect_tx(bar + b, (unsigned)(nv * LD * sizeof(double)));
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      const int line = wl * NL + l;
      if (line < nlines) {
        const int gb = BATCH ? line / nlp : 0, ln = line - gb * nlp;
        const int i = itop - ln / K, j = 1 + ln % K;
        tma_load_3d(Lb + (warp * 2 + b) * WB + l * LD, &tm, 0, 0,
                    (int)(gb * grid_lines) + i * L.n1 + j, bar + b);
      }
    }
  };
  if (lane == 0) {
    if (wl0 * NL < nlines) issue(wl0, 0);
    if ((wl0 + stride) * NL < nlines) issue(wl0 + stride, 1);
  }
  // descriptor words and Dirichlet fold value of warp-iteration wl's line, loaded one
  // iteration ahead (their latency was the kernel's top stall when loaded in place)
  auto line_of = [&](int wl, int& i, int& j, int& gb) {
    const int line = wl * NL + sub;
    const bool v = NL == 1 || line < nlines;
    gb = BATCH && v ? line / nlp : 0;
    const int ln = line - gb * nlp;
    i = v ? itop - ln / K : 1;
    j = v ? 1 + ln % K : 1;
    return v && wl * NL < nlines;
  };
  auto fetch = [&](int wl, ulonglong2& dd, double& bf) {
    int i, j, gb;
    dd = make_ulonglong2(0ull, 0ull);
    bf = 0.0;
    if (line_of(wl, i, j, gb)) {
      dd = *reinterpret_cast<const ulonglong2*>(a.desc + gb * a.dstride +
                                                2 * (line_desc(L, i, j) * G + seg));
      const long long bs = L.at(i, j, 0) + gb * L.bs;
      if (seg == 0) bf = a.bnd[bs];
      else if (seg == (m - 1) / S) bf = a.bnd[bs + a.hi_off];
    }
  };
  ulonglong2 ddn;
  double bfn;
  fetch(wl0, ddn, bfn);
  DivAcc acc(a.thr);
  int it = 0;
  for (int wl = wl0; wl * NL < nlines; wl += stride, ++it) {
    const int b = it & 1;
    int i, j, gb;
    const bool inl = line_of(wl, i, j, gb);
    // batched: grids that stopped at an earlier step are skipped (their copy still lands)
    const bool valid = inl && (!BATCH || !a.div_step || a.div_step[gb] >= a.step);
    const long long base = L.at(i, j, 0) + gb * L.bs;
    const unsigned long long amask = ddn.x;
    const uint32_t sbits = (uint32_t)ddn.y, cmask = (uint32_t)(ddn.y >> 32);
    const double bfold = bfn;
    fetch(wl + stride, ddn, bfn);
    double* W = Lb + (warp * 2 + b) * WB + sub * LD;
    mbar_wait(bar + b, (unsigned)(it >> 1) & 1u);

    double r[S];
#pragma unroll
    for (int q = 0; q < S; q += 2) {  // chunk `seg`, 16-byte unit q/2 at its swizzled place
      const double2 v = valid ? *reinterpret_cast<const double2*>(
                                    W + seg * 16 + ((((q >> 1) ^ (seg & 7))) << 1))
                              : make_double2(0.0, 0.0);
      r[q] = v.x;
      r[q + 1] = v.y;
    }
    rw_solve<S, G>(a, r, amask, cmask, bfold, valid, seg, T, Mi, sR, base);
    if (valid) {
#pragma unroll
      for (int q = 0; q < S; q += 2)
        *reinterpret_cast<double2*>(W + seg * 16 + ((((q >> 1) ^ (seg & 7))) << 1)) =
            make_double2(r[q], r[q + 1]);
    }
    __syncwarp();
    rw_store<S, G>(a, [&](int p) { return W[swz(p - 1)]; }, valid, seg, sbits, FP, base, acc);
    if (BATCH && a.check) {  // batched: the line's own grid (lines of a warp may differ)
      if (acc.bad(a.thr)) atomicMin(a.div_step + gb, a.step);
      acc = DivAcc(a.thr);
    }
    // the buffer's generic-proxy reads/writes are ordered before the next tensor copy into it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0 && (wl + 2 * stride) * NL < nlines) issue(wl + 2 * stride, b);
  }
  if (!BATCH && a.check && __any_sync(FULL, acc.bad(a.thr)) && lane == 0)
    atomicMin(a.div_step, a.step);
}

// ---------------------------------------------------------------------------------------
// Row sweeps (axis 2), TMA in and TMA out: every warp owns three line buffers in shared
// memory.  A line arrives by one tensor copy (128-byte swizzle, mbarrier), lane `seg` takes
// its 16 rows into registers, the line is solved inside the warp (rw_solve), the LODIE2 flow
// and the divergence test run on those registers, the rows go back to the same buffer and one
// tensor store writes the line out.  The lanes never address global memory for the field, no
// transposing store pass, no per-node predicates: the far face row m+1 travels with the line
// and is written back unchanged.  Copies of the lines two iterations ahead are in flight while
// a line is solved; the store of a buffer has a whole iteration to drain before the buffer is
// refilled.  One block of NW warps per SM, so every lane may keep its rows and the flow's
// temporaries in up to 128 registers.  Lines of 16 x G rows (m + 1 = 256, 512), single grid,
// LOD epilogues (store, LODIE1 source, LODIE2 flow); source and destination faces must agree
// (march buffers, or in place).  Descriptors: line-major, solute bits in row order (lm = 2).
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tm, int c0, int c1, int c2,
                                             const void* src) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
          reinterpret_cast<unsigned long long>(tm)),
      "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int S_, int G, int NW, int NB_>
struct RowLean {
  static constexpr int S = S_, NL = 32 / G, LD = G * S, NB = NB_;
  static constexpr int LDP = (LD + 127) & ~127;  // line buffers 1024-byte aligned (swizzle)
  static constexpr int WB = NL * LDP;
  static constexpr size_t lines_bytes = (size_t)NW * NB * WB * sizeof(double);
  static constexpr size_t smem(int fpoly_n) {
    return 1024 + lines_bytes +
           sizeof(double) * (kTabDoubles + G * (G + 2) + NW * NL * (G + 2) + kFlowHdr + fpoly_n + 2) +
           sizeof(unsigned long long) * NW * NB;
  }
};

// Offset (doubles) of 16-byte unit u of a line inside its swizzled buffer: chunk u / 8, unit
// (u % 8) ^ (chunk % 8).
__device__ __forceinline__ int lean_unit(int u) {
  const int c = u >> 3;
  return (c << 4) | (((u & 7) ^ (c & 7)) << 1);
}

// BATCH: nb stacked grids (config 5): a line belongs to grid b = line / (lines per grid),
// divergence flags per grid, a stopped grid's lines are skipped.  AOS epilogue
// (a.epi == EPI_AOS2, FLOWK == 0): 0.25 * (accumulated branches + this branch), the
// accumulator rows read from global memory (prefetched to L1 an iteration ahead).
template <int S_, int G, int NW, int NB_, int FLOWK, bool BATCH>
__global__ void __launch_bounds__(NW * 32, 1)
    k_sweep_rowlean(const SweepArgs a, const int nlines, const __grid_constant__ CUtensorMap tms,
                    const __grid_constant__ CUtensorMap tmd) {
  extern __shared__ unsigned char smraw[];
  using RL = RowLean<S_, G, NW, NB_>;
  constexpr int S = RL::S, NL = RL::NL, LD = RL::LD, LDP = RL::LDP, WB = RL::WB, NB = RL::NB;
  constexpr int HG = S % 8 == 0 ? 8 : 4;  // rows per interleaved flow group
  static_assert(NB == 2 || NB == 3, "two or three line buffers per warp");
  static_assert(S % 4 == 0 && LD % 16 == 0, "whole 128-byte chunks per line");
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int NT = NW * 32;
  constexpr bool FLOW = FLOWK != 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sub = lane / G, seg = lane % G;
  double* Lb = reinterpret_cast<double*>(
      smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u));  // 1024-aligned line buffers
  double* T = Lb + NW * NB * WB;         // uniform-segment tables
  double* Mi = T + kTabDoubles;          // G x (G + 2)
  double* sRb = Mi + G * (G + 2);        // NW * NL * (G + 2)
  double* FP = sRb + NW * NL * (G + 2);  // flow tables at FP + kFlowHdr
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(
      FP + kFlowHdr + (FLOW ? a.fpoly_n + (a.fpoly_n & 1) : 0));
  for (int c = tid; c < kTabDoubles / 2; c += NT) cp_async16(T + 2 * c, a.tab + 2 * c);
  if (a.static_ok)
    for (int c = tid; c < G * (G + 2) / 2; c += NT) cp_async16(Mi + 2 * c, a.minv + 2 * c);
  if (FLOW)
    for (int c = tid; c < a.fpoly_n / 2; c += NT) cp_async16(FP + kFlowHdr + 2 * c, a.fpoly + 2 * c);
  asm volatile("cp.async.commit_group;\n" ::);
  if (tid < NW * NB) mbar_init(bars + tid, NL);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  cp_async_wait_all();
  __syncthreads();
  if (!BATCH) {  // an earlier step diverged: nothing more to compute
    const int dstep = a.div_step ? *((volatile int*)a.div_step) : INT_MAX;
    if (dstep < a.step) return;
  }

  const Layout& L = a.L;
  const int K = L.n1 - 2;
  const int npl = a.on ? a.on : L.n0 - 2;          // planes per grid
  const int itop = a.on ? a.o0 + a.on : L.n0 - 2;  // planes itop, itop-1, ... (reverse)
  const int nlp = npl * K;                         // lines per grid
  const int glines = BATCH ? (int)(L.bs / L.pitch) : 0;  // field lines between grids
  const bool aos = FLOWK == 0 && a.epi == EPI_AOS2;
  double* sR = sRb + (warp * NL + sub) * (G + 2);
  unsigned long long* bar = bars + warp * NB;
  double* Wq = Lb + warp * NB * WB + sub * LDP;  // buffer b of this lane's line: Wq + b * WB
  // Line cursor of a lane: line = (warp-iteration) * NL + sub walks by `dl` lines per
  // iteration; grid, plane and row follow without divisions.
  struct Cur {
    int ln, b, i, j;
  };
  const int dl = gridDim.x * NW * NL;
  const int db = BATCH ? dl / nlp : 0, dlr = dl - db * nlp, dq = dlr / K, dr = dlr - dq * K;
  Cur c0;
  c0.ln = (blockIdx.x * NW + warp) * NL + sub;
  c0.b = BATCH ? c0.ln / nlp : 0;
  {
    const int l = c0.ln - c0.b * nlp;
    c0.i = itop - l / K;
    c0.j = 1 + l % K;
  }
  auto advance = [&](Cur& c) {
    c.ln += dl;
    c.b += db;
    c.i -= dq;
    c.j += dr;
    if (c.j > K) {
      c.j -= K;
      c.i -= 1;
    }
    if (BATCH && c.i <= itop - npl) {
      c.i += npl;
      c.b += 1;
    }
  };
  auto fline = [&](const Cur& c) { return c.b * glines + c.i * L.n1 + c.j; };  // field line
  // seg == 0 lanes: tensor copy of the line into buffer b (every sub-line arrives once per
  // phase, a line past the end with no bytes)
  auto issue = [&](const Cur& c, int b) {
    if (c.ln < nlines) {
      mbar_expect_tx(bar + b, (unsigned)(LD * sizeof(double)));
      tma_load_3d(Wq + b * WB, &tms, 0, 0, fline(c), bar + b);
    } else {
      mbar_arrive(bar + b);
    }
  };
  // descriptor words, fold value and (batch) the grid's flag of a line, fetched one
  // iteration ahead; the AOS accumulator rows start towards L1
  auto fetch = [&](const Cur& c, ulonglong2& dd, double& bf, int& ds) {
    dd = make_ulonglong2(0ull, 0ull);
    bf = 0.0;
    ds = INT_MAX;
    if (c.ln < nlines) {
      // 32-bit line arithmetic: a line is `pitch` doubles
      dd = *reinterpret_cast<const ulonglong2*>(
          a.desc + (BATCH ? c.b * a.dstride : 0ll) +
          2 * (long long)(((c.i - 1) * K + (c.j - 1)) * G + seg));
      const long long off = (long long)fline(c) * L.pitch + kOff;
      if (seg == 0) bf = a.bnd[off];
      else if (seg == G - 1) bf = a.bnd[off + a.hi_off];
      if (BATCH && a.div_step) ds = a.div_step[c.b];
      if (aos) {
        const double* ap = a.acc + off + seg * S + 1;
        asm volatile("prefetch.global.L1 [%0];" ::"l"(ap));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(ap + S - 1));
      }
    }
  };
  Cur c1 = c0;  // one iteration ahead
  advance(c1);
  Cur c2 = c1;  // two iterations ahead
  advance(c2);
  if (seg == 0) {
    issue(c0, 0);
    issue(c1, 1);
  }
  ulonglong2 ddn;
  double bfn;
  int dsn;
  fetch(c0, ddn, bfn, dsn);
  const double thrc = fmin(a.thr, 1.7976931348623157e308);
  const int thrH = thrc >= 0.0 ? __double2hiint(thrc) : -1;
  bool bad = false;
  // offsets of the lane's S / 2 16-byte units in its line buffer (S = 16: one chunk per lane)
  const int u0 = seg * (S / 2);
  auto uoff = [&](int k) {
    return S == 16 ? (seg << 4) | ((k ^ (seg & 7)) << 1) : lean_unit(u0 + k);
  };
  int it = 0;
  for (int w0 = blockIdx.x * NW + warp; w0 * NL < nlines; w0 += gridDim.x * NW, ++it) {
    const int b = it % NB;
    const bool valid = c0.ln < nlines && (!BATCH || dsn >= a.step);
    const long long base = (valid ? (long long)fline(c0) * L.pitch : 0ll) + kOff;
    const unsigned long long amask = ddn.x;
    const uint32_t sbits = (uint32_t)ddn.y, cmask = (uint32_t)(ddn.y >> 32);
    const double bfold = bfn;
    fetch(c1, ddn, bfn, dsn);
    double* W = Wq + b * WB;  // this lane's line
    mbar_wait(bar + b, (unsigned)(it / NB) & 1u);

    double r[S];
#pragma unroll
    for (int q = 0; q < S; q += 2) {
      // (an idle sub-line solves whatever its buffer holds; nothing of it is stored or tested)
      const double2 v = *reinterpret_cast<const double2*>(W + uoff(q >> 1));
      r[q] = v.x;
      r[q + 1] = v.y;
    }
    rw_solve<S, G>(a, r, amask, cmask, bfold, valid, seg, T, Mi, sR, base);
    unsigned need = 0u;  // FLOWK == 3: rows whose flow is evaluated from the buffer below
    int mx = 0;  // divergence test: largest high word of |x| over the lane's final rows
    if (FLOWK == 3) {
      // Flow on the lane's rows, HG interleaved Horner chains at a time, the tier chosen per
      // warp and group (no divergence): the tiny-argument polynomial when every row of the
      // warp's group is solvent with |w| <= 0.5 (the far field, most of the grid), else the
      // small-argument polynomial (|w| <= 2) with the solute rows keeping w.  Rows outside
      // both (|w| > 2, NaN, a solute palette with ions, no small form) are redone from the
      // buffer below (need).
      const unsigned force = a.fsmall_on ? sbits : 0xffffu;
      const unsigned ident = a.decay1 >= 1.0 ? sbits : 0u;  // ion-free solute: w is final
#pragma unroll
      for (int h = 0; h < S; h += HG) {
        bool tiny = ((force >> h) & ((1u << HG) - 1u)) == 0u;
#pragma unroll
        for (int u = 0; u < HG; ++u) tiny = tiny && fabs(r[h + u]) <= kFTinyX;
        double t[HG], p[HG];
        // (an idle sub-line holds stale data: it must not decide the tier of the others)
        if (__all_sync(FULL, tiny || !valid)) {
#pragma unroll
          for (int u = 0; u < HG; ++u) {
            t[u] = fma(r[h + u], r[h + u], -0.5 * kFTinyX * kFTinyX);
            p[u] = a.ftiny[kFTinyN - 1];
          }
#pragma unroll
          for (int c = kFTinyN - 2; c >= 0; --c)
#pragma unroll
            for (int u = 0; u < HG; ++u) p[u] = fma(p[u], t[u], a.ftiny[c]);
#pragma unroll
          for (int u = 0; u < HG; ++u) {
            r[h + u] *= p[u];
            mx = max(mx, __double2hiint(r[h + u]) & 0x7fffffff);
          }
        } else {
#pragma unroll
          for (int u = 0; u < HG; ++u) {
            t[u] = fma(r[h + u], r[h + u], -0.5 * kFSmallX * kFSmallX);
            p[u] = a.fsmall[kFSmallN - 1];
          }
#pragma unroll
          for (int c = kFSmallN - 2; c >= 0; --c)
#pragma unroll
            for (int u = 0; u < HG; ++u) p[u] = fma(p[u], t[u], a.fsmall[c]);
#pragma unroll
          for (int u = 0; u < HG; ++u) {
            const bool keep = !(fabs(r[h + u]) <= kFSmallX) || ((force >> (h + u)) & 1u);
            need |= keep ? (1u << (h + u)) : 0u;
            r[h + u] = keep ? r[h + u] : r[h + u] * p[u];
            // final unless it is redone from the buffer (tested there)
            if (!keep || ((ident >> (h + u)) & 1u))
              mx = max(mx, __double2hiint(r[h + u]) & 0x7fffffff);
          }
        }
      }
      need &= ~ident;
      if (seg == G - 1) need &= (1u << (S - 1)) - 1u;  // the face row
    } else if (FLOW) {
#pragma unroll
      for (int q = 0; q < S; q += 4)
        flow_group(a, FP, r[q], r[q + 1], r[q + 2], r[q + 3], (sbits >> q) & 1u,
                   (sbits >> (q + 1)) & 1u, (sbits >> (q + 2)) & 1u, (sbits >> (q + 3)) & 1u,
                   1.0);
    } else if (aos) {  // 0.25 * (accumulated branches + this branch), rounding as the tiles
      const double2* ap = reinterpret_cast<const double2*>(a.acc + base + seg * S + 1);
#pragma unroll
      for (int q = 0; q < S; q += 2) {
        const double2 y = valid ? ap[q >> 1] : make_double2(0.0, 0.0);
        r[q] = __dmul_rn(0.25, __dadd_rn(y.x, r[q]));
        r[q + 1] = __dmul_rn(0.25, __dadd_rn(y.y, r[q + 1]));
      }
    }
    if (seg == G - 1) r[S - 1] = 0.0;
    // divergence test (schemes.py:417-421) on the high words: |x| > thr for sure when the
    // high word is above the threshold's, undecided only when equal (exact compare then)
    if (FLOWK != 3) {  // (FLOWK == 3 tests its rows where the flow leaves them)
#pragma unroll
      for (int q = 0; q < S; ++q) mx = max(mx, __double2hiint(r[q]) & 0x7fffffff);
    }
    bool lbad = false;
    if (mx >= thrH && valid) {
      if (mx > thrH) {
        lbad = true;
      } else {
#pragma unroll
        for (int q = 0; q < S; ++q) lbad |= !((need >> q) & 1u) && !(fabs(r[q]) <= thrc);
      }
    }
    if (seg == G - 1) r[S - 1] = bfold;  // row m + 1: the far face keeps its Dirichlet value
    if (valid) {
#pragma unroll
      for (int q = 0; q < S; q += 2)
        *reinterpret_cast<double2*>(W + uoff(q >> 1)) = make_double2(r[q], r[q + 1]);
    }
    if (FLOWK == 3) {
      // The other rows, from the buffer, spread over the whole warp: they cluster in the few
      // lanes whose segment lies in a pocket of the molecule (|w| > 2 next to the charges), and
      // a lane-private loop ran as long as the fullest lane while the others idled.  Lane
      // counts are prefix-summed, item i belongs to the lane whose running count first
      // exceeds i (binary search in the warp's scratch) and is that lane's (i - before)-th
      // needed row; any lane can reach it because the rows sit in shared memory.
      const unsigned nd = valid ? need : 0u;
      if (__any_sync(FULL, nd != 0u)) {
        unsigned short* sc = reinterpret_cast<unsigned short*>(sRb + warp * NL * (G + 2));
        int incl = __popc(nd);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int v = __shfl_up_sync(FULL, incl, d);
          if (lane >= d) incl += v;
        }
        const int total = __shfl_sync(FULL, incl, 31);
        sc[lane] = (unsigned short)incl;
        sc[32 + lane] = (unsigned short)nd;
        sc[64 + lane] = (unsigned short)sbits;
        if (BATCH) sc[96 + lane] = (unsigned short)c0.b;  // the owner's grid (divergence flag)
        __syncwarp();
#pragma unroll 1
        for (int i = lane; i < total; i += 32) {
          int o = 0;
#pragma unroll
          for (int step = 16; step; step >>= 1)
            if ((int)sc[o + step - 1] <= i) o += step;
          const int before = o ? (int)sc[o - 1] : 0;
          const int u = __fns((unsigned)sc[32 + o], 0, i - before + 1);
          const int oseg = o % G;
          const int uo = S == 16 ? (oseg << 4) | (((u >> 1) ^ (oseg & 7)) << 1)
                                 : lean_unit(oseg * (S / 2) + (u >> 1));
          double* slot = Lb + warp * NB * WB + (o / G) * LDP + b * WB + (uo | (u & 1));
          const double x = flow_sm(a, FP, *slot, ((unsigned)sc[64 + o] >> u) & 1u, 1.0);
          *slot = x;
          if (BATCH) {
            if (a.check && !(fabs(x) <= thrc)) atomicMin(a.div_step + sc[96 + o], a.step);
          } else {
            lbad |= !(fabs(x) <= thrc);
          }
        }
      }
    }
    if (BATCH) {  // the line's own grid (the lines of a warp may belong to different grids)
      if (a.check && lbad) atomicMin(a.div_step + c0.b, a.step);
    } else {
      bad |= lbad;
    }
    // the lanes' writes are ordered before the tensor store reads the buffer
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (seg == 0) {
      if (valid) tma_store_3d(&tmd, 0, 0, fline(c0), Wq + b * WB);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      // the buffer refilled next was stored one iteration ago (three buffers: all but the
      // newest group done) or just now (two buffers)
      if (NB == 3) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      if ((w0 + 2 * gridDim.x * NW) * NL < nlines) issue(c2, (it + 2) % NB);
    }
    c0 = c1;
    c1 = c2;
    advance(c2);
  }
  if (seg == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (!BATCH && a.check && __any_sync(FULL, bad) && lane == 0) atomicMin(a.div_step, a.step);
}

// ---------------------------------------------------------------------------------------
// Fused axis-1 + axis-2 sweeps of a LOD step (schemes.py:301-311, order 0 -> 1 -> 2 kept).
// The lines of both families lie inside one i-plane, so one persistent launch runs the
// axis-1 column tiles of plane p and, a few planes later, the axis-2 lines of plane p, which
// read the axis-1 output from L2 and store in place over it: the intermediate field never
// travels to HBM and back (step traffic 48 -> 32 B per node).  Blocks take work items from
// one global queue (atomic counter, the next item claimed while the current one runs).  The
// queue order IS the dependency order -- `lag` planes of column tiles, then for every plane
// its line groups followed by the column tiles of plane p + lag -- and an item only ever
// waits for earlier items, all of which are held by running blocks, so the launch cannot
// deadlock whatever the number of resident blocks.  A column tile publishes its plane with a
// fence + counter increment; a line group spins (one thread, acquire loads) until its plane's
// counter reaches the tiles per plane.  Both sweeps use the kernels' own bodies: col_body
// (register-direct column tiles) and the row-warp line solve (rw_solve / rw_store), with the
// reduced-system scratch of the one and the line buffers of the other sharing shared memory.
// Requires square planes and equal axis coefficients (one table set, P = G separators).
struct FuseCtl {
  int* q;      // q[0] next item, q[1] blocks that left, q[2 + p] finished column tiles of plane p
  int np;      // interior planes
  int n1, n2;  // items per plane: axis-1 column tiles, axis-2 line groups
  int lag;     // planes of column tiles queued ahead of the line groups (1 <= lag <= np)
};

template <int S, int P, int LB, int G>
struct Fused12 {
  static constexpr int NT = LB * P, NW = NT / 32;
  using RW = RowWarp<S, G>;
  static constexpr int XD = 4 * NT, WD = NW * RW::WD;
  static constexpr int UD = ((XD > WD ? XD : WD) + 1) & ~1;  // scratch union, doubles
  static constexpr size_t smem(int fpoly_n) {
    return sizeof(double) * (kTabDoubles + P * (P + 2) + UD + kFlowHdr + fpoly_n + 2);
  }
};

template <int S, int P, int LB, int G>
__global__ void __launch_bounds__(LB * P, 3)
    k_sweep_fused12(const SweepArgs a1, const SweepArgs a2, const FuseCtl c) {
  static_assert(P == G, "one reduced-system shape for both axes");
  extern __shared__ double sm[];
  using F = Fused12<S, P, LB, G>;
  using RW = RowWarp<S, G>;
  constexpr int NT = F::NT, NW = F::NW, NL = RW::NL;
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ int s_item;
  const int tid = threadIdx.y * LB + threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int dstep = a2.div_step ? *((volatile int*)a2.div_step) : INT_MAX;
  double* T = sm;
  double* Mi = T + kTabDoubles;
  double* U = Mi + P * (P + 2);  // column tiles: reduced-system scratch; line groups: buffers
  double* FP = U + F::UD;
  stage_tables<P>(a2, T, Mi, FP, tid, NT);
  asm volatile("cp.async.commit_group;\n" ::);
  if (dstep < a2.step) {  // an earlier step diverged: nothing more to compute
    cp_async_wait_all();
    return;
  }
  if (tid == 0) s_item = atomicAdd(c.q, 1);
  cp_async_wait_all();
  __syncthreads();

  const Layout& L = a2.L;
  const int K = L.n1 - 2;  // lines per plane (either family: square planes)
  const int nitems = c.np * (c.n1 + c.n2), per = c.n1 + c.n2;
  const int head = c.lag * c.n1, full = c.np - c.lag;
  const int sub = lane / G, seg = lane % G;
  double* W = U + warp * RW::WD + sub * RW::LW;  // this lane's line buffer
  double* sR = U + warp * RW::WD + NL * RW::LW + sub * RW::RW;
  DivAcc acc(a2.thr);
  int item = s_item;
  while (item < nitems) {
    int nxt = 0;
    if (tid == 0) nxt = atomicAdd(c.q, 1);  // claimed now, taken up when this item is done
    int kind, plane, si;  // kind 1: column tile si of plane, 2: line group si of plane
    if (item < head) {
      kind = 1;
      plane = item / c.n1;
      si = item - plane * c.n1;
    } else {
      const int r = item - head;
      if (r < full * per) {
        const int grp = r / per, w = r - grp * per;
        kind = w < c.n2 ? 2 : 1;
        plane = w < c.n2 ? grp : grp + c.lag;
        si = w < c.n2 ? w : w - c.n2;
      } else {
        const int r2 = r - full * per;
        kind = 2;
        plane = full + r2 / c.n2;
        si = r2 % c.n2;
      }
    }
    if (kind == 1) {  // ---- axis-1 column tile (as k_sweep_col) ----
      TileGeo g;
      g.b = 0;
      g.c0 = 1 + si * LB;
      g.outer = plane + 1;
      g.ncols = min(LB, (L.n2 - 2) + 1 - g.c0);
      g.base = L.at(g.outer, 0, g.c0);
      g.stride = (int)L.pitch;
      const int m = a1.m, i0 = threadIdx.y * S, st = g.stride;
      const bool act = (int)threadIdx.x < g.ncols;
      const long long gl = g.base + threadIdx.x;
      unsigned long long amask = 0ull;
      if (act) amask = *col_desc<P>(a1, g);
      double r[S];
      const double* srow = a1.src + gl + (long long)(i0 + 1) * st;
      if (act && i0 + S <= m + 1) {
#pragma unroll
        for (int j = 0; j < S; ++j) r[j] = srow[j * st];
      } else {
#pragma unroll
        for (int j = 0; j < S; ++j) r[j] = (act && i0 + 1 + j <= m + 1) ? srow[j * st] : 0.0;
      }
      double bfold = 0.0;
      if (act) {
        if (threadIdx.y == 0) bfold = a1.bnd[gl];
        else if ((int)threadIdx.y == (m - 1) / S) bfold = a1.bnd[gl + a1.hi_off];
      }
      col_body<S, P, false, LB, 1>(a1, g, r, 0.0, 0.0, amask, 0ull, bfold, T, Mi, U, FP);
      if (tid == 0) s_item = nxt;
      __syncthreads();  // every store of the tile is issued; the scratch is free again
      if (tid == 0) {
        __threadfence();
        atomicAdd(c.q + 2 + plane, 1);
      }
    } else {  // ---- axis-2 line group: NW warps x NL lines of plane `plane` ----
      if (tid == 0) {
        const int* d = c.q + 2 + plane;
        while (ld_acquire(d) < c.n1) __nanosleep(64);
      }
      __syncthreads();
      const int m = a2.m;
      const int ln = (si * NW + warp) * NL + sub;
      const bool valid = ln < K;
      const int i = plane + 1, j = valid ? 1 + ln : 1;
      const long long base = L.at(i, j, 0);
      unsigned long long amask = 0ull;
      uint32_t sbits = 0u, cmask = 0u;
      double bfold = 0.0;
      if (valid) {
        const double* gsrc = a2.src + base + 1;
#pragma unroll
        for (int q = 0; q < S / 2; ++q) {
          const int ch = seg + G * q;  // chunk: rows 2ch+1, 2ch+2 (one segment, S even)
          cp_async16(W + RW::pos(2 * ch + 1), gsrc + 2 * ch);
        }
        const ulonglong2 dd = *reinterpret_cast<const ulonglong2*>(
            a2.desc + 2 * (line_desc(L, i, j) * G + seg));
        amask = dd.x;
        sbits = (uint32_t)dd.y;
        cmask = (uint32_t)(dd.y >> 32);
        if (seg == 0) bfold = a2.bnd[base];
        else if (seg == (m - 1) / S) bfold = a2.bnd[base + a2.hi_off];
      }
      asm volatile("cp.async.commit_group;\n" ::);
      cp_async_wait_all();
      __syncwarp();
      double r[S];
#pragma unroll
      for (int q = 0; q < S; q += 2) {
        const double2 v = valid ? *reinterpret_cast<const double2*>(W + 2 + seg * RW::SP + q)
                                : make_double2(0.0, 0.0);
        r[q] = v.x;
        r[q + 1] = v.y;
      }
      rw_solve<S, G>(a2, r, amask, cmask, bfold, valid, seg, T, Mi, sR, base);
      if (valid) {
#pragma unroll
        for (int q = 0; q < S; q += 2)
          *reinterpret_cast<double2*>(W + 2 + seg * RW::SP + q) = make_double2(r[q], r[q + 1]);
      }
      __syncwarp();
      if (G % S == 0) {
        const int p0 = RW::pos(1 + seg);
        rw_store<S, G>(a2, [&](int p) { return W[p0 + ((p - 1 - seg) / G) * (G + 2 * G / S)]; },
                       valid, seg, sbits, FP, base, acc);
      } else {
        rw_store<S, G>(a2, [&](int p) { return W[RW::pos(p)]; }, valid, seg, sbits, FP, base,
                       acc);
      }
      if (tid == 0) s_item = nxt;
      __syncthreads();  // line buffers and the item slot are reused
    }
    item = s_item;
  }
  if (a2.check && __any_sync(FULL, acc.bad(a2.thr)) && lane == 0)
    atomicMin(a2.div_step, a2.step);
  // The last block to leave resets the queue for the next launch.
  __syncthreads();
  if (tid == 0) s_item = atomicAdd(c.q + 1, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (s_item)
    for (int t = tid; t < 2 + c.np; t += NT) c.q[t] = 0;
}

// ---------------------------------------------------------------------------------------
// Segment descriptors, built once per march and axis from the 1-byte node codes:
//   word 0: bit j = eps bit (axis) of the node of row i0+j, j = 0..S (zero past node m+1)
//   word 1: bits 0..S-1 solute bit of the nodes of rows i0..i0+S-1; bits 32.. charged bits
// Layout: ((outer-1)*P + seg)*K + (line-1); line-major ((outer-1)*K + line-1)*P + seg for the
// row-warp sweeps (lm = 1: solute bits in the store-pass order of k_sweep_rowwarp / rowtma;
// lm = 2: in row order, k_sweep_rowlean).
__global__ void k_build_desc(const Layout L, int axis, int S, int P, int lm,
                             const uint8_t* __restrict__ codes,
                             unsigned long long* __restrict__ desc) {
  const int m = (axis == 0 ? L.n0 : (axis == 1 ? L.n1 : L.n2)) - 2;
  const int K = (axis == 2 ? L.n1 : L.n2) - 2;  // lines per outer index
  const long long nseg = (long long)((axis == 0 ? L.n1 : L.n0) - 2) * P * K;
  const int sh = 1 + axis;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nseg;
       t += (long long)gridDim.x * blockDim.x) {
    int c, seg, outer;
    if (lm) {  // line-major (row-warp sweeps): t = (line * P + seg)
      seg = (int)(t % P);
      const long long line = t / P;
      c = 1 + (int)(line % K);
      outer = 1 + (int)(line / K);
    } else {
      c = 1 + (int)(t % K);
      const long long os = t / K;
      seg = (int)(os % P);
      outer = 1 + (int)(os / P);
    }
    const long long base =
        axis == 0 ? L.at(0, outer, c) : (axis == 1 ? L.at(outer, 0, c) : L.at(outer, c, 0));
    const long long stride = axis == 0 ? L.s0 : (axis == 1 ? L.pitch : 1);
    const int i0 = seg * S;
    unsigned long long w0 = 0, w1 = 0;
    for (int j = 0; j <= S; ++j) {
      const int p = i0 + j + 1;
      if (p > m + 1) break;
      const uint32_t c = codes[base + p * stride];
      w0 |= (unsigned long long)((c >> sh) & 1u) << j;
      if (j < S && p <= m) {
        if (lm != 1) w1 |= (unsigned long long)(c & 1u) << j;
        w1 |= (unsigned long long)((c >> 4) & 1u) << (32 + j);
      }
    }
    if (lm == 1)  // row-warp store pass: lane `seg` stores rows 1 + seg + P*q, q = 0..S-1; its
             // solute bits in that order (no per-node shuffle in the LODIE2 flow epilogue)
      for (int q = 0; q < S; ++q) {
        const int p = 1 + seg + P * q;
        if (p <= m) w1 |= (unsigned long long)(codes[base + p * stride] & 1u) << q;
      }
    desc[2 * t] = w0;
    desc[2 * t + 1] = w1;
  }
}

// LU factors, alpha and beta of one general segment (5 x kTabRows doubles at F): rows j of
// the segment are rows i0+j of the line; `first` = the segment starts the line (row 0 has no
// sub-diagonal), d = m - i0 (row j >= d is a decoupled padding row, row d-1 has no
// super-diagonal).  Same recurrences as the uniform tables (make_tables).
__device__ void seg_factors(const AxisCoef& co, unsigned long long eb, int first, int d, int S,
                            double* F) {
  double cpp = 0.0, dap = 1.0, lastinv = 0.0, lastc = 0.0;
  for (int j = 0; j < S - 1; ++j) {
    const uint32_t em = (uint32_t)(eb >> j) & 1u, ep = (uint32_t)(eb >> (j + 1)) & 1u;
    double av, bv, cv;
    if (j >= d) {
      av = 0.0;
      bv = 1.0;
      cv = 0.0;
    } else {
      av = (first && j == 0) ? 0.0 : (em ? co.sub[1] : co.sub[0]);
      cv = (j == d - 1) ? 0.0 : (ep ? co.sup[1] : co.sup[0]);
      bv = em ? (ep ? co.diag[3] : co.diag[2]) : (ep ? co.diag[1] : co.diag[0]);
    }
    const double inv = 1.0 / (bv - av * cpp);
    const double cpj = cv * inv;
    const double da = -(av * dap) * inv;
    F[TQ_INV * kTabRows + j] = inv;
    F[TQ_G * kTabRows + j] = av * inv;
    F[TQ_CP * kTabRows + j] = cpj;
    F[TQ_AL * kTabRows + j] = da;  // forward values, replaced by alpha below
    cpp = cpj;
    dap = da;
    lastinv = inv;
    lastc = cv;
  }
  double bb = -lastc * lastinv, aa = F[TQ_AL * kTabRows + S - 2];
  F[TQ_BE * kTabRows + S - 2] = bb;
  for (int j = S - 3; j >= 0; --j) {
    const double c = F[TQ_CP * kTabRows + j];
    aa = F[TQ_AL * kTabRows + j] - c * aa;
    bb = -c * bb;
    F[TQ_AL * kTabRows + j] = aa;
    F[TQ_BE * kTabRows + j] = bb;
  }
}

// General-segment factors depend only on (eps bits, first, min(m - i0, S)): segments that
// share that key share one table.  The key space (S <= 16: 24 bits) is marked in a bitmap,
// ranked by a prefix count, and each distinct key gets its factors once -- a few MB that stay
// in L2 instead of 1.3 KB per segment streamed from HBM by every sweep.
constexpr int kDedupMaxS = 16;
__host__ __device__ __forceinline__ int key_bits(int S) { return S + 1 + 1 + 5; }

__device__ __forceinline__ bool seg_general(unsigned long long w0, int S, int i0, int m,
                                            int first, unsigned& key) {
  const unsigned long long eb = eps_bits(w0, S);
  const unsigned long long allm = (1ull << S) - 1ull, bits = eb & allm;
  if (bits == 0ull || bits == allm) {
    if (i0 + S <= m) return false;
    if (i0 + S - 1 == m && !first) return false;
  }
  const int d = min(max(m - i0, 0), S);
  key = (unsigned)eb | ((unsigned)first << (S + 1)) | ((unsigned)d << (S + 2));
  return true;
}

__global__ void k_mark_keys(const Layout L, int axis, int S, int P, int lm,
                            const unsigned long long* __restrict__ desc,
                            unsigned* __restrict__ bitmap) {
  const int m = (axis == 0 ? L.n0 : (axis == 1 ? L.n1 : L.n2)) - 2;
  const int K = (axis == 2 ? L.n1 : L.n2) - 2;
  const long long nseg = (long long)((axis == 0 ? L.n1 : L.n0) - 2) * P * K;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nseg;
       t += (long long)gridDim.x * blockDim.x) {
    const int seg = lm ? (int)(t % P) : (int)((t / K) % P);
    unsigned key;
    if (seg_general(desc[2 * t], S, seg * S, m, seg == 0, key))
      if (!((bitmap[key >> 5] >> (key & 31)) & 1u)) atomicOr(bitmap + (key >> 5), 1u << (key & 31));
  }
}

__global__ void k_popc_words(const unsigned* __restrict__ bitmap, int nw, int* __restrict__ cnt) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x)
    cnt[w] = __popc(bitmap[w]);
}

// One thread per bitmap word: the factors of every distinct key, at its rank.
__global__ void k_key_factors(AxisCoef co, int S, const unsigned* __restrict__ bitmap,
                              const int* __restrict__ base, int nw, double* __restrict__ gfac) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x) {
    unsigned bits = bitmap[w];
    int rank = base[w];
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const unsigned key = ((unsigned)w << 5) | (unsigned)b;
      const unsigned long long eb = key & ((2u << S) - 1u);
      const int first = (key >> (S + 1)) & 1u, d = (int)(key >> (S + 2));
      seg_factors(co, eb, first, d, S, gfac + (long long)rank * 5 * kTabRows);
      ++rank;
    }
  }
}

__global__ void k_assign_slots(const Layout L, int axis, int S, int P, int lm,
                               unsigned long long* __restrict__ desc,
                               const unsigned* __restrict__ bitmap, const int* __restrict__ base) {
  const int m = (axis == 0 ? L.n0 : (axis == 1 ? L.n1 : L.n2)) - 2;
  const int K = (axis == 2 ? L.n1 : L.n2) - 2;
  const long long nseg = (long long)((axis == 0 ? L.n1 : L.n0) - 2) * P * K;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nseg;
       t += (long long)gridDim.x * blockDim.x) {
    const int seg = lm ? (int)(t % P) : (int)((t / K) % P);
    const unsigned long long w0 = desc[2 * t];
    unsigned key;
    if (!seg_general(w0, S, seg * S, m, seg == 0, key)) continue;
    const unsigned w = key >> 5, below = bitmap[w] & ((1u << (key & 31)) - 1u);
    const int rank = base[w] + __popc(below);
    desc[2 * t] = w0 | ((unsigned long long)(rank + 1) << kSlotShift);
  }
}

// General segments (not one dielectric, or partial at the line end): their LU factors,
// alpha and beta are static for the march, so they are computed once here (same
// recurrences as the uniform tables, per-row coefficients) and read like a table by the
// sweeps.  Pass 0 counts, pass 1 assigns slots (atomic; values do not depend on the slot)
// and writes factors + slot into descriptor word 0.
__global__ void k_seg_factors(const Layout L, int axis, int S, int P, int lm, AxisCoef co, int pass,
                              unsigned long long* __restrict__ desc, int* __restrict__ counter,
                              double* __restrict__ gfac) {
  const int m = (axis == 0 ? L.n0 : (axis == 1 ? L.n1 : L.n2)) - 2;
  const int K = (axis == 2 ? L.n1 : L.n2) - 2;
  const long long nseg = (long long)((axis == 0 ? L.n1 : L.n0) - 2) * P * K;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nseg;
       t += (long long)gridDim.x * blockDim.x) {
    const int seg = lm ? (int)(t % P) : (int)((t / K) % P);
    const int i0 = seg * S, first = seg == 0;
    const unsigned long long w0 = desc[2 * t];
    const unsigned long long eb = eps_bits(w0, S);
    const unsigned long long allm = (1ull << S) - 1ull, bits = eb & allm;
    bool general = true;
    if (bits == 0ull || bits == allm) {
      if (i0 + S <= m) general = false;
      else if (i0 + S - 1 == m && !first) general = false;
    }
    if (!general) continue;
    if (pass == 0) {
      atomicAdd(counter, 1);
      continue;
    }
    const int slot = atomicAdd(counter, 1);
    seg_factors(co, eb, first, min(max(m - i0, 0), S), S, gfac + (long long)slot * 5 * kTabRows);
    desc[2 * t] = w0 | ((unsigned long long)(slot + 1) << kSlotShift);
  }
}

// ---------------------------------------------------------------------------------------
// Host-side launch helpers.

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

static bool col_enabled();
static int seg_S(int m, int P, int axis) {
  if (P == 4) return m > 48 ? 16 : 12;
  // 65..80-row lines of the strided axes (cost-weighted slab chunks): eight segments of 10
  // rows instead of 12 (two idle segments per line); column sweeps only
  if (P == 8 && axis < 2 && m > 64 && m <= 80 && col_enabled()) return 10;
  // 129..192-row lines of the strided axes (cost-weighted slab chunks at four ranks): sixteen
  // segments of 10 or 12 rows instead of 16 (up to seven idle segments per line); column
  // sweeps only
  if (P == 16 && axis < 2 && m > 128 && m <= 192 && col_enabled()) return m <= 160 ? 10 : 12;
  if (P == 16) return m <= 256 ? 16 : 0;  // instantiated: P = 8 with any S, 16/32 with 16/32
  if (P == 32) return m <= 512 ? 16 : (m <= 1024 ? 32 : 0);
  const int opts[] = {2, 3, 4, 6, 8, 12, 16, 24, 32};
  for (int s : opts)
    if (P * s >= m) return s;
  return 0;
}
// Strided axes: segments of ~16 rows (registers and occupancy balance, measured); the
// contiguous axis always uses the 32 lanes of a warp.
static int seg_P(int axis, int m) {
  // 33..64-row lines of the strided axes (the axis-0 chunks of an 8-rank slab march at 513
  // planes): four segments of 12 or 16 rows, sixteen 64-thread blocks per SM, instead of
  // eight segments of 6 or 8 rows -- twice the rows in flight per thread and half the
  // separators per line (PBG_P4=0 keeps the old shape, for comparison).
  static const bool p4 = env_int("PBG_P4", 1) != 0;
  if (p4 && axis < 2 && m > 32 && m <= 64 && col_enabled()) return 4;
  return m <= 128 ? 8 : (m <= 256 ? 16 : 32);
}

// Row-warp sweeps (k_sweep_rowwarp) for axis 2: lines of G*S - 1 interior rows where they
// measured faster than the row tiles, and the LOD epilogues; PBG_ROWWARP=0 keeps the row-tile
// kernel, for comparison.
static int rowwarp_G(int m) {
  if (m + 1 == 512) return 32;  // S = 16 (c4: 734 -> 645 us with the LODIE2 flow)
  if (m + 1 == 256) return 16;  // S = 16 (c3: 100 -> 95 us; two lines per warp)
  if (m + 1 == 128) return 16;  // S = 8  (c2: 25 -> 22 us)
  if (m + 1 == 96) {            // c5 97^3 lines: S = 12, four lines per warp, or (PBG_RW96G)
    static const int g = [] {   // S = 6, two lines per warp
      const char* e = getenv("PBG_RW96G");
      return e && atoi(e) == 16 ? 16 : 8;
    }();
    return g;
  }
  return 0;
}
static int rowwarp_S(int m) {
  const int G = rowwarp_G(m);
  return G ? (m + 1) / G : 0;
}
// PBG_FUSED12=1: axis-1 and axis-2 sweeps of a LOD step in one launch (k_sweep_fused12).
static bool fused12_enabled() {
  static const bool on = [] {
    const char* e = getenv("PBG_FUSED12");
    return e && e[0] == '1';
  }();
  return on;
}

static bool rowwarp_ok(const SweepArgs& a, int axis) {
  static const bool on = [] {
    const char* e = getenv("PBG_ROWWARP");
    return !(e && e[0] == '0');
  }();
  return on && axis == 2 && !a.cn && a.pro == PRO_NONE && !a.has_extra && !a.ends &&
         (a.epi == EPI_STORE || a.epi == EPI_FLOW || a.epi == EPI_SRC || a.epi == EPI_AOS2) &&
         rowwarp_S(a.m) != 0;
}

// Column sweeps run register-direct (k_sweep_col) unless PBG_COL=0 selects the staged-tile
// kernels, for comparison.
static bool col_enabled() {
  static const bool on = [] {
    const char* e = getenv("PBG_COL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Per (kernel, dynamic shared memory, device): raise the shared-memory limit once and cache
// the resident blocks per SM x SM count, so launches issue no attribute / occupancy queries
// (the config-5 batch issues ~40k launches from 8 host threads).
static int resident_blocks(const void* fn, int nthreads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, size_t, int>, int> cache;
  static std::map<std::pair<const void*, int>, size_t> limit;  // attribute set per kernel
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(fn, smem, dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  // The limit only ever grows: lowering it for a smaller launch would make a later, cached
  // larger launch of the same kernel fail.
  size_t& lim = limit[std::make_pair(fn, dev)];
  if (smem > 48 * 1024 && smem > lim) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    lim = smem;
  }
  int nsm = 148, bps = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, nthreads, smem);
  const int r = nsm * std::max(bps, 1);
  cache[key] = r;
  return r;
}

template <int S, int P, bool CN, int LB, bool RT>
static void launch_strided_SCL(const SweepArgs& a, int axis, cudaStream_t st) {
  const int nouter = a.on ? a.on : (axis == 0 ? a.L.n1 : a.L.n0) - 2;
  const int nlines = (RT ? a.L.n1 : a.L.n2) - 2;
  const int ntx = (nlines + LB - 1) / LB;
  dim3 block(LB, P);
  const size_t smem = strided_smem<LB, RT>(S, P, epi_needs(a.epi) != 0, flow_stage_n(a));
  auto kern = k_sweep_strided<S, P, CN, LB, RT>;
  // persistent blocks: as many as fit at once (the tables are staged once per block)
  const int grid =
      std::min(ntx * nouter * a.L.nb, resident_blocks((const void*)kern, LB * P, smem));
  kern<<<grid, block, smem, st>>>(a, axis, ntx, nouter);
}

// Axis 0 rows are one field plane apart (MB strides): 128-byte row chunks keep DRAM pages
// and TLB entries busy (64-byte chunks run at ~55% of copy bandwidth there, measured).
template <int S, int P, bool CN>
static void launch_col(const SweepArgs& a, int axis, cudaStream_t st) {
  constexpr int LB = 16;
  const int nouter = a.on ? a.on : (axis == 0 ? a.L.n1 : a.L.n0) - 2;
  const int ntx = (a.L.n2 - 2 + LB - 1) / LB;
  const size_t smem = sizeof(double) * (P * (P + 2) + 4 * LB * P + kFlowHdr + flow_stage_n(a));
  const bool plain = !CN && (a.pro == PRO_NONE || a.pro == PRO_SRC) && !a.check &&
                     (a.epi == EPI_STORE || a.epi == EPI_SRC || a.epi == EPI_MAOS0);
  const bool aos0 = !CN && S % 4 == 0 && a.epi == EPI_AOS0 && a.pro == PRO_NONE;
  auto kern = plain ? k_sweep_col<S, P, false, LB, 1>
                    : (aos0 ? k_sweep_col<S, P, false, LB, 2> : k_sweep_col<S, P, CN, LB, 0>);
  resident_blocks((const void*)kern, LB * P, smem);  // shared-memory limit, once
  kern<<<dim3(ntx, nouter, a.L.nb), dim3(LB, P), smem, st>>>(a, axis);
}

// Row tiles of 16 lines for lines of <= 256 rows (256 threads per block: fewer duplicated
// per-block tables per SM than 8-line tiles); PBG_RT16=0 keeps 8-line tiles, for comparison.
static bool rt16_enabled() {
  static const bool on = [] {
    const char* e = getenv("PBG_RT16");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int S, int P, bool CN>
static void launch_strided_SC(const SweepArgs& a, int axis, cudaStream_t st) {
  if (axis < 2 && col_enabled()) return launch_col<S, P, CN>(a, axis, st);
  // 16-column tiles (128-byte row chunks) unless a second staged tile (AOS/MAOS epilogue
  // operand) would halve the resident blocks.
  // Tiles must also fit the 227 KB of shared memory per block (long lines with AOS/MAOS).
  const bool needY = epi_needs(a.epi) != 0;
  const bool wide = !needY;
  const bool fits16 = strided_smem<16, false>(S, P, needY, flow_stage_n(a)) <= 232448;
  if (axis == 0 && fits16) launch_strided_SCL<S, P, CN, 16, false>(a, axis, st);
  else if (axis == 0) launch_strided_SCL<S, P, CN, 8, false>(a, axis, st);
  else if (axis == 1 && wide) launch_strided_SCL<S, P, CN, 16, false>(a, axis, st);
  else if (axis == 1) launch_strided_SCL<S, P, CN, 8, false>(a, axis, st);
  else if (P <= 16 && rt16_enabled()) launch_strided_SCL<S, P, CN, 16, true>(a, axis, st);
  else launch_strided_SCL<S, P, CN, 8, true>(a, axis, st);
}

template <int S, int P>
static void launch_strided_SP(const SweepArgs& a, int axis, cudaStream_t st) {
  if (a.cn) launch_strided_SC<S, P, true>(a, axis, st);
  else launch_strided_SC<S, P, false>(a, axis, st);
}

#define PBG_DISPATCH_S(S_, CALL)                                                        \
  switch (S_) {                                                                         \
    case 2: CALL(2); break;                                                             \
    case 3: CALL(3); break;                                                             \
    case 4: CALL(4); break;                                                             \
    case 6: CALL(6); break;                                                             \
    case 8: CALL(8); break;                                                             \
    case 12: CALL(12); break;                                                           \
    case 16: CALL(16); break;                                                           \
    case 24: CALL(24); break;                                                           \
    case 32: CALL(32); break;                                                           \
    default: return fail(PBG_E_UNSUPPORTED, "line too long for the device sweep (m > 768)"); \
  }

template <int S, int G>
static void launch_rowwarp_SG(const SweepArgs& a, cudaStream_t st) {
  const int nlines = (a.on ? a.on : a.L.n0 - 2) * (a.L.n1 - 2) * a.L.nb;
  const size_t smem = rowwarp_smem(S, G, flow_stage_n(a));
  auto kern = a.L.nb > 1 ? k_sweep_rowwarp<S, G, true> : k_sweep_rowwarp<S, G, false>;
  const int per_block = kRWarps * (32 / G);
  const int grid = std::min((nlines + per_block - 1) / per_block,
                            resident_blocks((const void*)kern, kRWarps * 32, smem));
  kern<<<grid, kRWarps * 32, smem, st>>>(a, nlines);
}

// TMA row-warp sweeps (k_sweep_rowtma) for 16-row segments (m + 1 = 512, 256); PBG_ROWTMA=0
// keeps the cp.async row-warp kernel, for comparison.  PBG_ROWTMA_NW: warps per block.
static int rowtma_mode() {
  static const int v = [] {
    const char* e = getenv("PBG_ROWTMA");
    return e && *e ? atoi(e) : 1;
  }();
  return v;
}
static int rowtma_nw() {
  static const int v = [] {
    const char* e = getenv("PBG_ROWTMA_NW");
    return e && *e ? atoi(e) : 20;
  }();
  return v;
}

using EncodeTiled = PFN_cuTensorMapEncodeTiled_v12000;
static EncodeTiled encode_tiled() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  });
  return fn;
}

// Tensor map of the axis-2 lines of a field: (16 doubles, chunk, line) with the line index
// i*n1 + j, based at row 1 (k = 1, 256-byte aligned), 128-byte swizzle.
static bool line_tensor_map(const SweepArgs& a, int box_chunks, CUtensorMap* tm,
                            const double* field = nullptr) {
  EncodeTiled fn = encode_tiled();
  if (!fn) return false;
  const Layout& L = a.L;
  cuuint64_t dims[3] = {16, (cuuint64_t)((L.pitch - kOff - 1) / 16),
                        L.nb > 1 ? (cuuint64_t)L.nb * (cuuint64_t)(L.bs / L.pitch)
                                 : (cuuint64_t)L.n0 * (cuuint64_t)L.n1};
  cuuint64_t strides[2] = {128, (cuuint64_t)L.pitch * sizeof(double)};
  cuuint32_t box[3] = {16, (cuuint32_t)box_chunks, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)((field ? field : a.src) + kOff + 1),
            dims, strides,
            box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int S, int G, int NW>
static bool launch_rowtma_SGN(const SweepArgs& a, cudaStream_t st) {
  CUtensorMap tm;
  if (!line_tensor_map(a, G * S / 16, &tm)) return false;
  const int nlines = (a.on ? a.on : a.L.n0 - 2) * (a.L.n1 - 2) * a.L.nb;
  const size_t smem = RowTma<S, G, NW>::smem(flow_stage_n(a));
  auto kern = a.L.nb > 1 ? k_sweep_rowtma<S, G, NW, true> : k_sweep_rowtma<S, G, NW, false>;
  const int per_block = NW * (32 / G);
  const int grid = std::min((nlines + per_block - 1) / per_block,
                            resident_blocks((const void*)kern, NW * 32, smem));
  kern<<<grid, NW * 32, smem, st>>>(a, nlines, tm);
  return true;
}

template <int S, int G>
static bool launch_rowtma_SG(const SweepArgs& a, cudaStream_t st) {
  // 20 warps per block measured best (8 / 12 / 16: +7..19%, profiles/rowtma_ab_r02.txt)
  if (rowtma_nw() == 16) return launch_rowtma_SGN<S, G, 16>(a, st);
  return launch_rowtma_SGN<S, G, 20>(a, st);
}

// TMA-in / TMA-out row sweeps (k_sweep_rowlean): the default for 256- and 512-row lines of a
// single grid with the LOD epilogues; PBG_ROWLEAN=0 keeps k_sweep_rowwarp / k_sweep_rowtma,
// PBG_ROWLEAN_NW = warps per block (16; 12, 20, 24 for comparison).
static bool rowlean_enabled() {
  static const bool on = [] {
    const char* e = getenv("PBG_ROWLEAN");
    return !(e && e[0] == '0');
  }();
  return on;
}
static bool rowlean_ok(const SweepArgs& a) {
  if (!rowlean_enabled()) return false;
  const int S = rowwarp_S(a.m), G = rowwarp_G(a.m);
  if (S == 16 && a.L.nb == 1)  // 256- and 512-row lines of a single grid, LOD epilogues
    return a.epi == EPI_STORE || a.epi == EPI_FLOW || a.epi == EPI_SRC;
  if (S == 12 && G == 8)  // 96-row lines (config 5), single or batched, LOD and AOS epilogues
    return a.epi == EPI_STORE || a.epi == EPI_FLOW || a.epi == EPI_SRC || a.epi == EPI_AOS2;
  return false;
}

template <int S, int G, int NW, int NB>
static bool launch_rowlean_T(const SweepArgs& a, cudaStream_t st) {
  CUtensorMap tms, tmd;
  if (!line_tensor_map(a, G * S / 16, &tms, a.src) || !line_tensor_map(a, G * S / 16, &tmd, a.dst))
    return false;
  const int nlines = (a.on ? a.on : a.L.n0 - 2) * (a.L.n1 - 2) * a.L.nb;
  const bool flow = a.epi == EPI_FLOW;
  const size_t smem = RowLean<S, G, NW, NB>::smem(flow ? a.fpoly_n : 0);
  // PBG_FLOWK=1: flow_group (tiny tier + per-node fallback) instead of the per-warp tier
  // choice on all rows, for comparison
  static const int fk = env_int("PBG_FLOWK", 3) == 1 ? 1 : 3;
  constexpr bool BATCH = S == 12;  // the batched form also serves a single 97^3 grid
  auto kern = !flow ? k_sweep_rowlean<S, G, NW, NB, 0, BATCH>
                    : (fk == 3 ? k_sweep_rowlean<S, G, NW, NB, 3, BATCH>
                               : k_sweep_rowlean<S, G, NW, NB, 1, BATCH>);
  const int per_block = NW * (32 / G);
  const int grid = std::min((nlines + per_block - 1) / per_block,
                            resident_blocks((const void*)kern, NW * 32, smem));
  kern<<<grid, NW * 32, smem, st>>>(a, nlines, tms, tmd);
  return true;
}

static bool launch_rowlean(const SweepArgs& a, cudaStream_t st) {
  // 16 warps x 3 buffers measured best or equal (20 x 2: c4 -2%, c3 equal; 12 and 24 slower:
  // profiles/rowlean_ab_r02.txt); PBG_ROWLEAN_NW=20 selects 20 x 2
  static const int nw = env_int("PBG_ROWLEAN_NW", 16);
  const int S = rowwarp_S(a.m), G = rowwarp_G(a.m);
  if (S == 12) return launch_rowlean_T<12, 8, 16, 3>(a, st);
  if (G == 32) return nw == 20 ? launch_rowlean_T<16, 32, 20, 2>(a, st)
                               : launch_rowlean_T<16, 32, 16, 3>(a, st);
  return nw == 20 ? launch_rowlean_T<16, 16, 20, 2>(a, st) : launch_rowlean_T<16, 16, 16, 3>(a, st);
}

static int launch_strided(const SweepArgs& a, int axis, cudaStream_t st) {
  if (a.rw == 2) {
    if (!a.faces_ok && a.src != a.dst)
      return fail(PBG_E_INVALID, "row sweep: source and destination faces must agree");
    if (!launch_rowlean(a, st)) return fail(PBG_E_CUDA, "tensor map encoding failed");
    PBG_LAUNCH_CHECK("k_sweep_rowlean");
    return PBG_OK;
  }
  // TMA staging measured faster for 256-row lines (c3), slower for 512-row lines (c4:
  // 1.62 vs 1.59 ms/step; profiles/rowtma_ab_r02.txt); PBG_ROWTMA=0/1/2: off / auto / on.
  if (a.rw && rowwarp_S(a.m) == 16 &&
      (rowtma_mode() == 2 || (rowtma_mode() == 1 && rowwarp_G(a.m) == 16))) {
    const bool ok = rowwarp_G(a.m) == 32 ? launch_rowtma_SG<16, 32>(a, st)
                                         : launch_rowtma_SG<16, 16>(a, st);
    if (ok) {
      PBG_LAUNCH_CHECK("k_sweep_rowtma");
      return PBG_OK;
    }
  }
  if (a.rw) {
    switch (rowwarp_G(a.m) * 100 + rowwarp_S(a.m)) {
      case 3216: launch_rowwarp_SG<16, 32>(a, st); break;
      case 1616: launch_rowwarp_SG<16, 16>(a, st); break;
      case 1608: launch_rowwarp_SG<8, 16>(a, st); break;
      case 812: launch_rowwarp_SG<12, 8>(a, st); break;
      case 1606: launch_rowwarp_SG<6, 16>(a, st); break;
      default: return fail(PBG_E_UNSUPPORTED, "row-warp sweep without a segment length");
    }
    PBG_LAUNCH_CHECK("k_sweep_rowwarp");
    return PBG_OK;
  }
  const int P = seg_P(axis, a.m), S = seg_S(a.m, P, axis);
  if (P == 4) {  // column sweeps only (seg_P)
    if (S == 16) {
      if (a.cn) launch_col<16, 4, true>(a, axis, st);
      else launch_col<16, 4, false>(a, axis, st);
    } else {
      if (a.cn) launch_col<12, 4, true>(a, axis, st);
      else launch_col<12, 4, false>(a, axis, st);
    }
    PBG_LAUNCH_CHECK("k_sweep_col");
    return PBG_OK;
  }
  if (P == 8 && S == 10) {  // column sweeps only (seg_S)
    if (a.cn) launch_col<10, 8, true>(a, axis, st);
    else launch_col<10, 8, false>(a, axis, st);
    PBG_LAUNCH_CHECK("k_sweep_col");
    return PBG_OK;
  }
  if (P == 8) {
#define PBG_STRIDED8(S) launch_strided_SP<S, 8>(a, axis, st)
    PBG_DISPATCH_S(S, PBG_STRIDED8)
#undef PBG_STRIDED8
  } else if (P == 16 && S == 10) {  // column sweeps only (seg_S)
    if (a.cn) launch_col<10, 16, true>(a, axis, st);
    else launch_col<10, 16, false>(a, axis, st);
    PBG_LAUNCH_CHECK("k_sweep_col");
    return PBG_OK;
  } else if (P == 16 && S == 12) {
    if (a.cn) launch_col<12, 16, true>(a, axis, st);
    else launch_col<12, 16, false>(a, axis, st);
    PBG_LAUNCH_CHECK("k_sweep_col");
    return PBG_OK;
  } else if (P == 16 && S == 16) {
    launch_strided_SP<16, 16>(a, axis, st);
  } else if (P == 32 && S == 16) {
    launch_strided_SP<16, 32>(a, axis, st);
  } else if (P == 32 && S == 32) {
    launch_strided_SP<32, 32>(a, axis, st);
  } else {
    return fail(PBG_E_UNSUPPORTED, "line too long for the device sweep (m > 1024)");
  }
  PBG_LAUNCH_CHECK("k_sweep_strided");
  return PBG_OK;
}


// Fused axis-1 + axis-2 launch (k_sweep_fused12): LOD steps on square planes whose two axes
// share their coefficient tables and whose axis-2 sweep is a row-warp sweep with as many
// separators per line as the axis-1 column tiles (n1 = n2 = 257: 16 x 16; 513: 32 x 16).
// Measured slower than the separate launches (c3 265 vs 208 us/step, c4 1.97 vs 1.50 ms,
// profiles/fused12_ab_r02.txt: three blocks of 8 warps per SM, one work item at a time each,
// hide less latency than the separate kernels' free-running warps), so PBG_FUSED12=1 only
// selects it for comparison.
static int fused12_shape(const SweepArgs& a1, const SweepArgs& a2) {
  if (!fused12_enabled() || a2.rw != 1 || a1.cn || a2.cn || a1.L.nb != 1 || a1.L.n1 != a1.L.n2) return 0;
  if (a1.pro != PRO_NONE || a1.epi != EPI_STORE || a1.has_extra || a1.ends || a1.check) return 0;
  if (memcmp(&a1.co, &a2.co, sizeof(AxisCoef)) || memcmp(a1.tmid, a2.tmid, sizeof(a1.tmid)) ||
      a1.static_ok != a2.static_ok)
    return 0;
  const int P = seg_P(1, a1.m), S = seg_S(a1.m, P, 1);
  if (P != rowwarp_G(a2.m) || S != rowwarp_S(a2.m) || S != 16) return 0;
  return P == 16 || P == 32 ? P : 0;
}

template <int S, int P, int LB, int G>
static void launch_fused12_T(const SweepArgs& a1, const SweepArgs& a2, int* q, cudaStream_t st) {
  using F = Fused12<S, P, LB, G>;
  const size_t smem = F::smem(flow_stage_n(a2));
  auto kern = k_sweep_fused12<S, P, LB, G>;
  const int resident = resident_blocks((const void*)kern, F::NT, smem);
  FuseCtl c;
  c.q = q;
  c.np = a1.L.n0 - 2;
  c.n1 = (a1.L.n2 - 2 + LB - 1) / LB;
  c.n2 = (a2.L.n1 - 2 + F::NW * (32 / G) - 1) / (F::NW * (32 / G));
  // every column tile of plane p is claimed at least `resident` items before the line groups
  // of plane p, so those rarely have to wait
  static const int lag_env = [] {
    const char* e = getenv("PBG_FUSED12_LAG");
    return e && *e ? atoi(e) : 0;
  }();
  const int lag = lag_env > 0 ? lag_env : resident / (c.n1 + c.n2) + 2;
  c.lag = std::max(1, std::min(lag, c.np));
  const int grid = std::min(c.np * (c.n1 + c.n2), resident);
  kern<<<grid, dim3(LB, P), smem, st>>>(a1, a2, c);
}

static int launch_fused12(const SweepArgs& a1, const SweepArgs& a2, int* q, cudaStream_t st) {
  if (!a2.fpoly) return fail(PBG_E_CUDA, "flow table allocation failed");
  switch (fused12_shape(a1, a2)) {
    case 16: launch_fused12_T<16, 16, 16, 16>(a1, a2, q, st); break;
    case 32: launch_fused12_T<16, 32, 8, 32>(a1, a2, q, st); break;
    default: return fail(PBG_E_UNSUPPORTED, "fused axis-1/axis-2 sweep: unsupported shape");
  }
  PBG_LAUNCH_CHECK("k_sweep_fused12");
  return PBG_OK;
}


// Fused axis-0 + axis-1 launch (k_sweep_fused01): LOD steps of a single grid whose first two
// axes use the same segmentation.  Measured slower than the separate launches (c3 126-129 vs
// 124 us for the two sweeps, c4 1119 vs 982 us, profiles/fused01_ab_r02.txt: the column tiles
// are not bound by DRAM latency, and the slab order costs DRAM locality), so PBG_FUSED01=1
// only selects it for comparison; PBG_FUSED01_TW = column groups per slab, PBG_FUSED01_LAG =
// slabs of lead.
static bool fused01_ok(const SweepArgs& a0, const SweepArgs& a1) {
  static const bool on = env_int("PBG_FUSED01", 0) != 0;
  if (!on || !col_enabled() || a0.cn || a1.cn || a0.L.nb != 1 || a0.ends || a1.ends) return false;
  if (a0.epi != EPI_STORE || a0.has_extra || a0.check) return false;
  if (a1.pro != PRO_NONE || a1.epi != EPI_STORE || a1.has_extra || a1.check) return false;
  const int P0 = seg_P(0, a0.m), P1 = seg_P(1, a1.m);
  if (P0 != P1 || seg_S(a0.m, P0, 0) != 16 || seg_S(a1.m, P1, 1) != 16) return false;
  return P0 == 16 || P0 == 32;
}

template <int S, int P>
static void launch_fused01_T(const SweepArgs& a0, const SweepArgs& a1, int* q, cudaStream_t st) {
  constexpr int LB = 16;
  const size_t smem =
      sizeof(double) * (2 * P * (P + 2) + 4 * LB * P + kFlowHdr + flow_stage_n(a0));
  auto kern = k_sweep_fused01<S, P, LB>;
  const int resident = resident_blocks((const void*)kern, LB * P, smem);
  static const int tw_env = env_int("PBG_FUSED01_TW", 0), lag_env = env_int("PBG_FUSED01_LAG", 0);
  Fuse01Ctl c;
  c.q = q;
  c.ntx = (a0.L.n2 - 2 + LB - 1) / LB;
  c.n0i = a0.L.n1 - 2;
  c.n1i = a0.L.n0 - 2;
  // slabs of at most ~18 MB: the axis-0 output of `lag` + 1 slabs and the in-place axis-1
  // output of the slab before them stay in L2 together
  const double group_mb = (double)a0.L.n0 * a0.L.n1 * LB * 8.0 / 1e6;
  c.tw = tw_env > 0 ? tw_env : std::max(1, std::min(4, (int)(18.0 / group_mb)));
  c.tw = std::min(c.tw, c.ntx);
  c.nslab = (c.ntx + c.tw - 1) / c.tw;
  // every axis-0 tile of slab x is claimed at least `resident` items before the axis-1 tiles
  // of slab x
  const int per0 = c.tw * c.n0i;
  const int lag = lag_env > 0 ? lag_env : (resident + per0 - 1) / per0 + 1;
  c.lag = std::max(1, std::min(lag, c.nslab));
  const int grid = std::min(c.nslab * c.tw * (c.n0i + c.n1i), resident);
  kern<<<grid, dim3(LB, P), smem, st>>>(a0, a1, c);
}

static int launch_fused01(const SweepArgs& a0, const SweepArgs& a1, int* q, cudaStream_t st) {
  if (!a0.fpoly) return fail(PBG_E_CUDA, "flow table allocation failed");
  if (seg_P(0, a0.m) == 16) launch_fused01_T<16, 16>(a0, a1, q, st);
  else launch_fused01_T<16, 32>(a0, a1, q, st);
  PBG_LAUNCH_CHECK("k_sweep_fused01");
  return PBG_OK;
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

// Uniform-segment tables (same recurrences as the general device path).
static void make_tables(const AxisCoef& co, int S, double* out) {
  for (int i = 0; i < kTabDoubles; ++i) out[i] = 0.0;
  for (int type = 0; type < 3; ++type) {
    for (int v = 0; v < 2; ++v) {
      double* T = out + (type * 2 + v) * 5 * kTabRows;
      const double b = co.diag[v * 2 + v];
      double cpp = 0.0, dap = 1.0, lastinv = 0.0, c = 0.0;
      double da[kTabRows], cp[kTabRows];
      for (int j = 0; j < S - 1; ++j) {
        const double aj = (type == 1 && j == 0) ? 0.0 : co.sub[v];
        c = (type == 2 && j == S - 2) ? 0.0 : co.sup[v];
        const double inv = 1.0 / (b - aj * cpp);
        cp[j] = c * inv;
        da[j] = -(aj * dap) * inv;
        T[TQ_INV * kTabRows + j] = inv;
        T[TQ_G * kTabRows + j] = aj * inv;
        T[TQ_CP * kTabRows + j] = cp[j];
        cpp = cp[j];
        dap = da[j];
        lastinv = inv;
      }
      double bb = -c * lastinv, aa = da[S - 2];
      T[TQ_AL * kTabRows + S - 2] = aa;
      T[TQ_BE * kTabRows + S - 2] = bb;
      for (int j = S - 3; j >= 0; --j) {
        aa = da[j] - cp[j] * aa;
        bb = -cp[j] * bb;
        T[TQ_AL * kTabRows + j] = aa;
        T[TQ_BE * kTabRows + j] = bb;
      }
    }
  }
}

// Dense inverse of the reduced (separator) system of a clean line: every node carries eps
// palette 0, segment k uses table type first / interior / last.  Valid when 32*S is m or
// m + 1 (the last separator is row m-1 or the padding row m).
static bool make_reduced_inverse(const AxisCoef& co, const double* tab, int S, int m, int P,
                                 double* minv) {
  if (!(P * S == m || P * S == m + 1)) return false;
  auto T = [&](int type, int q, int j) { return tab[(type * 2) * 5 * kTabRows + q * kTabRows + j]; };
  auto type_of = [&](int k) { return k == 0 ? 1 : ((k == P - 1 && P * S == m + 1) ? 2 : 0); };
  double A[kSeg], B[kSeg], C[kSeg];
  for (int k = 0; k < P; ++k) {
    const int ty = type_of(k), i = k * S + S - 1;
    if (i >= m) {
      A[k] = 0.0;
      B[k] = 1.0;
      C[k] = 0.0;
      continue;
    }
    const double as = co.sub[0], bs = co.diag[0], cs = (i == m - 1) ? 0.0 : co.sup[0];
    double aFn = 0.0, bFn = 0.0;
    if (k + 1 < P) {
      aFn = T(type_of(k + 1), TQ_AL, 0);
      bFn = T(type_of(k + 1), TQ_BE, 0);
    }
    A[k] = as * T(ty, TQ_AL, S - 2);
    B[k] = bs + as * T(ty, TQ_BE, S - 2) + cs * aFn;
    C[k] = cs * bFn;
  }
  static thread_local double M[kSeg][2 * kSeg];
  for (int r = 0; r < P; ++r)
    for (int c = 0; c < 2 * P; ++c) M[r][c] = 0.0;
  for (int r = 0; r < P; ++r) {
    if (r > 0) M[r][r - 1] = A[r];
    M[r][r] = B[r];
    if (r + 1 < P) M[r][r + 1] = C[r];
    M[r][P + r] = 1.0;
  }
  for (int c = 0; c < P; ++c) {  // Gauss-Jordan, diagonally dominant: no pivoting
    const double piv = M[c][c];
    for (int q = 0; q < 2 * P; ++q) M[c][q] /= piv;
    for (int r = 0; r < P; ++r) {
      if (r == c || M[r][c] == 0.0) continue;
      const double f = M[r][c];
      for (int q = 0; q < 2 * P; ++q) M[r][q] -= f * M[c][q];
    }
  }
  for (int r = 0; r < P; ++r)  // row-major, rows padded to P + 2 (conflict-free loads)
    for (int c = 0; c < P; ++c) minv[r * (P + 2) + c] = M[r][P + c];
  return true;
}

// Interpolates f at the n Chebyshev nodes of [c - r, c + r] in extended precision and
// re-expands the Chebyshev series in powers of t = x - c: out[q] = coefficient of t^q.
template <int n, typename F>
static void cheb_powers(F f, long double c, long double r, double* out) {
  const long double pi = 3.141592653589793238462643383279502884L;
  long double y[n], g[n];
  for (int k = 0; k < n; ++k) y[k] = f(c + r * std::cos(pi * (k + 0.5L) / n));
  for (int j = 0; j < n; ++j) {
    long double acc = 0.0L;
    for (int k = 0; k < n; ++k) acc += y[k] * std::cos(pi * j * (k + 0.5L) / n);
    g[j] = (j == 0 ? 1.0L : 2.0L) * acc / n;
  }
  // sum_j g_j T_j(u), u = t / r, in powers of u (T_{j+1} = 2u T_j - T_{j-1})
  long double Tp[n] = {0}, Tc[n] = {0}, b[n] = {0};
  Tp[0] = 1.0L;
  Tc[1] = 1.0L;
  b[0] = g[0];
  b[1] = g[1];
  for (int j = 2; j < n; ++j) {
    long double Tn[n] = {0};
    for (int q = 0; q + 1 < n; ++q) Tn[q + 1] = 2.0L * Tc[q];
    for (int q = 0; q < n; ++q) {
      Tn[q] -= Tp[q];
      b[q] += g[j] * Tn[q];
      Tp[q] = Tc[q];
      Tc[q] = Tn[q];
    }
  }
  long double rp = 1.0L;
  for (int q = 0; q < n; ++q, rp *= r) out[q] = (double)(b[q] / rp);
}

// Flow interval table of decay d (pbg_internal.cuh, flow_poly): on interval [lo, hi] the
// map F(x) = 2 artanh(d tanh(x/2)) is interpolated at the 10 Chebyshev nodes in extended
// precision, and the Chebyshev series is re-expanded in powers of t = x - c.
static void build_flow_poly(double d, double* out) {
  for (int iv = 0; iv < kFPolyIv; ++iv) {
    const int e = iv / 16, s = iv % 16;
    const double lo = std::ldexp(1.0 + s / 16.0, e) - 1.0;
    const double hi = std::ldexp(1.0 + (s + 1) / 16.0, e) - 1.0;
    const double c = 0.5 * (lo + hi);
    const long double r = 0.5L * ((long double)hi - (long double)lo);
    double* o = out + iv * kFPolyStride;
    o[0] = c;
    cheb_powers<10>(
        [&](long double x) { return 2.0L * std::atanh((long double)d * std::tanh(0.5L * x)); },
        (long double)c, r, o + 1);
    o[kFPolyStride - 1] = 0.0;
  }
}

// Small-argument flow of decay d (pbg_internal.cuh, flow_small): G(y) = F(sqrt y) / sqrt y on
// y in [0, kFSmallX^2] (G(0) = d), in powers of t = y - kFSmallX^2 / 2.
template <int n>
static void build_flow_even(double d, double X, double* out) {
  const long double Y = (long double)X * X;
  cheb_powers<n>(
      [&](long double y) {
        const long double x = std::sqrt(y);
        return 2.0L * std::atanh((long double)d * std::tanh(0.5L * x)) / x;
      },
      0.5L * Y, 0.5L * Y, out);
}

static void build_flow_small(double d, double* out) { build_flow_even<kFSmallN>(d, kFSmallX, out); }
static void build_flow_tiny(double d, double* out) { build_flow_even<kFTinyN>(d, kFTinyX, out); }

// Host cache of the small- and tiny-argument coefficients per decay (set_decays runs per
// launch).
static void flow_small_coefs(double d, double* small, double* tiny) {
  static std::mutex mu;
  static std::map<double, std::vector<double>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(d);
  if (it == cache.end()) {
    std::vector<double> g(kFSmallN + kFTinyN);
    build_flow_small(d, g.data());
    build_flow_tiny(d, g.data() + kFSmallN);
    it = cache.emplace(d, std::move(g)).first;
  }
  std::copy(it->second.begin(), it->second.begin() + kFSmallN, small);
  std::copy(it->second.begin() + kFSmallN, it->second.end(), tiny);
}

// Device copy of the interval tables of a decay pair, [palette slot][kFPolyDoubles], cached
// per device for the process (a march uses at most two pairs).
static const double* flow_poly_table(double d0, double d1, int& ntab) {
  static std::mutex mu;
  static std::map<std::tuple<int, double, double>, std::pair<double*, int>> cache;
  int dev = 0;
  ntab = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(dev, d0, d1);
  auto it = cache.find(key);
  if (it != cache.end()) {
    ntab = it->second.second;
    return it->second.first;
  }
  std::vector<double> h;
  for (double d : {d0, d1}) {
    if (!(d < 1.0) || (ntab == 1 && d == d0)) continue;
    h.resize((size_t)(ntab + 1) * kFPolyDoubles);
    build_flow_poly(d, h.data() + (size_t)ntab * kFPolyDoubles);
    ++ntab;
  }
  if (h.empty()) h.assign(2, 0.0);
  double* p = nullptr;
  if (cudaMalloc(&p, h.size() * sizeof(double)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
    return nullptr;
  cache[key] = {p, ntab};
  return p;
}

void set_decays(SweepArgs& a, double d0, double d1) {
  a.decay0 = d0;
  a.decay1 = d1;
  a.sat0 = d0 < 1.0 ? 2.0 * std::atanh(d0) : 0.0;
  a.sat1 = d1 < 1.0 ? 2.0 * std::atanh(d1) : 0.0;
  int ntab = 0;
  a.fpoly = flow_poly_table(d0, d1, ntab);
  a.fpoly_n = ntab * kFPolyDoubles;
  a.foff[0] = 0;  // palette 0 has slot 0 when it needs one
  a.foff[1] = (d0 < 1.0 && d1 < 1.0 && d1 != d0) ? kFPolyDoubles : 0;
  a.fsmall_on = d0 >= 0.0 && d0 < 1.0;
  if (a.fsmall_on) flow_small_coefs(d0, a.fsmall, a.ftiny);
}

SweepArgs base_args(const pbg_grid* g, const pbg_palette* pal, int axis, double factor) {
  SweepArgs a;
  memset(&a, 0, sizeof(a));
  a.L = make_layout(g);
  a.m = g->n[axis] - 2;
  a.co = make_axis_coef(pal->eps[axis], factor, g->h);
  set_decays(a, 1.0, 1.0);
  a.pm = 1.0;
  a.pro = PRO_NONE;
  a.epi = EPI_STORE;
  a.thr = INFINITY;
  a.hi_off = (long long)(a.m + 1) * (axis == 0 ? a.L.s0 : (axis == 1 ? a.L.pitch : 1));
  return a;
}


static long long desc_segments(const Layout& L, int axis, int P) {
  return (long long)((axis == 0 ? L.n1 : L.n0) - 2) * P * ((axis == 2 ? L.n1 : L.n2) - 2);
}

int prepare_axis(SweepArgs& a, int axis, const uint8_t* codes, AxisAux& aux,
                        cudaStream_t st) {
  a.rw = rowwarp_ok(a, axis) ? 1 : 0;
  if (a.rw && a.faces_ok && rowlean_ok(a) && !fused12_enabled()) a.rw = 2;
  const int P = a.rw ? rowwarp_G(a.m) : seg_P(axis, a.m);
  const int S = a.rw ? rowwarp_S(a.m) : seg_S(a.m, P, axis);
  const int lm = a.rw;
  if (S < 2) return fail(PBG_E_UNSUPPORTED, "line too long for the device sweep (m > 768)");
  std::vector<double> host(kTabDoubles + kSeg * (kSeg + 2), 0.0);
  make_tables(a.co, S, host.data());
  memcpy(a.tmid, host.data(), sizeof(a.tmid));  // type 0 (interior), palette 0
  a.static_ok =
      make_reduced_inverse(a.co, host.data(), S, a.m, P, host.data() + kTabDoubles) ? 1 : 0;
  PBG_CUDA(cudaMallocAsync(&aux.buf, host.size() * sizeof(double), st));
  PBG_CUDA(cudaMemcpyAsync(aux.buf, host.data(), host.size() * sizeof(double),
                           cudaMemcpyHostToDevice, st));
  const long long nseg = desc_segments(a.L, axis, P);
  // +64 words of slack: tiles past the last interior column read (unused) descriptors; a
  // batched march keeps one such block per grid (a.dstride words apart)
  const int nb = a.L.nb;
  a.dstride = 2 * nseg + 64;
  PBG_CUDA(cudaMallocAsync(&aux.desc, nb * a.dstride * sizeof(unsigned long long), st));
  for (int b = 0; b < nb; ++b) {
    k_build_desc<<<148 * 8, 256, 0, st>>>(a.L, axis, S, P, lm, codes + b * a.L.bs,
                                           aux.desc + b * a.dstride);
    PBG_LAUNCH_CHECK("k_build_desc");
  }
  if (S <= kDedupMaxS) {
    const int nw = 1 << (key_bits(S) - 5);
    unsigned* bitmap = nullptr;
    int *cnt = nullptr, *base = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, base, nw, st);
    PBG_CUDA(cudaMallocAsync(&bitmap, (size_t)nw * sizeof(unsigned), st));
    PBG_CUDA(cudaMallocAsync(&cnt, (size_t)nw * sizeof(int), st));
    PBG_CUDA(cudaMallocAsync(&base, (size_t)nw * sizeof(int), st));
    PBG_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    PBG_CUDA(cudaMemsetAsync(bitmap, 0, (size_t)nw * sizeof(unsigned), st));
    for (int b = 0; b < nb; ++b) {
      k_mark_keys<<<148 * 8, 256, 0, st>>>(a.L, axis, S, P, lm, aux.desc + b * a.dstride,
                                           bitmap);
      PBG_LAUNCH_CHECK("k_mark_keys");
    }
    k_popc_words<<<(nw + 255) / 256, 256, 0, st>>>(bitmap, nw, cnt);
    PBG_LAUNCH_CHECK("k_popc_words");
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, base, nw, st);
    PBG_LAUNCH_CHECK("cub::DeviceScan");
    int last[2] = {0, 0};
    PBG_CUDA(cudaMemcpyAsync(&last[0], base + nw - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    PBG_CUDA(cudaMemcpyAsync(&last[1], cnt + nw - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    PBG_CUDA(cudaStreamSynchronize(st));  // also: the host staging vector dies here
    const int ndist = last[0] + last[1];
    PBG_CUDA(cudaMallocAsync(&aux.gfac, ((size_t)ndist + 1) * 5 * kTabRows * sizeof(double), st));
    if (ndist > 0) {
      k_key_factors<<<(nw + 255) / 256, 256, 0, st>>>(a.co, S, bitmap, base, nw, aux.gfac);
      PBG_LAUNCH_CHECK("k_key_factors");
      for (int b = 0; b < nb; ++b) {
        k_assign_slots<<<148 * 8, 256, 0, st>>>(a.L, axis, S, P, lm, aux.desc + b * a.dstride,
                                                bitmap, base);
        PBG_LAUNCH_CHECK("k_assign_slots");
      }
    }
    PBG_CUDA(cudaFreeAsync(bitmap, st));
    PBG_CUDA(cudaFreeAsync(cnt, st));
    PBG_CUDA(cudaFreeAsync(base, st));
    PBG_CUDA(cudaFreeAsync(tmp, st));
  } else {  // long segments: one table per general segment
    int* counter = nullptr;
    PBG_CUDA(cudaMallocAsync(&counter, sizeof(int), st));
    PBG_CUDA(cudaMemsetAsync(counter, 0, sizeof(int), st));
    for (int b = 0; b < nb; ++b) {
      k_seg_factors<<<148 * 8, 256, 0, st>>>(a.L, axis, S, P, lm, a.co, 0,
                                              aux.desc + b * a.dstride, counter, nullptr);
      PBG_LAUNCH_CHECK("k_seg_factors");
    }
    int ngen = 0;
    PBG_CUDA(cudaMemcpyAsync(&ngen, counter, sizeof(int), cudaMemcpyDeviceToHost, st));
    PBG_CUDA(cudaStreamSynchronize(st));  // also: the host staging vector dies here
    PBG_CUDA(cudaMallocAsync(&aux.gfac, ((size_t)ngen + 1) * 5 * kTabRows * sizeof(double), st));
    if (ngen > 0) {
      PBG_CUDA(cudaMemsetAsync(counter, 0, sizeof(int), st));
      for (int b = 0; b < nb; ++b) {
        k_seg_factors<<<148 * 8, 256, 0, st>>>(a.L, axis, S, P, lm, a.co, 1,
                                               aux.desc + b * a.dstride, counter, aux.gfac);
        PBG_LAUNCH_CHECK("k_seg_factors");
      }
    }
    PBG_CUDA(cudaFreeAsync(counter, st));
  }
  a.gfac = aux.gfac;
  a.tab = aux.buf;
  a.minv = aux.buf + kTabDoubles;
  a.desc = aux.desc;
  return PBG_OK;
}

void release_axis(AxisAux& aux, cudaStream_t st) {
  if (aux.buf) cudaFreeAsync(aux.buf, st);
  if (aux.desc) cudaFreeAsync(aux.desc, st);
  if (aux.gfac) cudaFreeAsync(aux.gfac, st);
  aux.buf = nullptr;
  aux.desc = nullptr;
  aux.gfac = nullptr;
}

int launch_sweep(const SweepArgs& a, int axis, cudaStream_t st) {
  if (!a.fpoly) return fail(PBG_E_CUDA, "flow table allocation failed");
  return launch_strided(a, axis, st);
}


bool plan_for(int v, Plan& p) {
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

__global__ void k_faces_bad(const Layout L, const double* x, double thr, int* flag,
                            int skip_lo, int skip_hi) {
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
    if ((skip_lo && i == 0) || (skip_hi && i == L.n0 - 1)) continue;  // slab ghost planes
    const double v = x[L.at(i, j, k)];
    if (!isfinite(v) || fabs(v) > thr) atomicMin(flag, 1);
  }
}

// Per-axis launch arguments of one march (variant plan, flow decays, fusions).
void march_axes(const pbg_march_desc* d, const Plan& plan, SweepArgs ax[3]) {
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
  // No ions anywhere (the vacuum marches of the energy pipeline): the LOD flow is the identity
  // (_apply_flow returns w for decay >= 1, schemes.py:88-103), so those steps carry no flow stage.
  const bool flow_id = dec_lod[0] >= 1.0 && dec_lod[1] >= 1.0;

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
        if (axis == 0 && !flow_id) {
          a.pro = PRO_FLOW;
          set_decays(a, dec_lod[0], dec_lod[1]);
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
        if (axis == 2 && !flow_id) {
          a.epi = EPI_FLOW;
          set_decays(a, dec_lod[0], dec_lod[1]);
        }
        break;
      case 2:  // AOS: 0.25*(((pm*flow(u) + b0) + b1) + b2), branches from u
        a.epi = axis == 0 ? EPI_AOS0 : (axis == 1 ? EPI_AOS1 : EPI_AOS2);
        if (axis == 0) {
          set_decays(a, dec_aos[0], dec_aos[1]);
          a.pm = aos_pm;
        }
        a.has_extra = plan.src[axis] != 0.0;
        a.extra = plan.src[axis] * dta;
        break;
      case 3:  // MAOS: ((b0 + b1) + b2)/3, branches from flow(u)
        a.pro = PRO_FLOW;
        set_decays(a, dec_lod[0], dec_lod[1]);
        a.epi = axis == 0 ? EPI_MAOS0 : (axis == 1 ? EPI_MAOS1 : EPI_MAOS2);
        a.has_extra = 1;
        a.extra = plan.src[axis] * dta;
        break;
    }
    a.check = (axis == 2) && d->check_divergence;
    ax[axis] = a;
  }
}

static bool g_profile = false;
static double g_prof_ms[3] = {0, 0, 0};
static long long g_prof_n[3] = {0, 0, 0};

}  // namespace pbg

using namespace pbg;

extern "C" PBG_API int pbg_flow_table(double decay, double* out) {
  static_assert(kFPolyDoubles == PBG_FLOW_TABLE_DOUBLES, "flow table size");
  if (!out) return fail(PBG_E_INVALID, "null pointer");
  if (!(decay >= 0.0 && decay < 1.0)) return fail(PBG_E_INVALID, "decay must be in [0, 1)");
  build_flow_poly(decay, out);
  return PBG_OK;
}

extern "C" PBG_API int pbg_flow_small(double decay, double* out) {
  static_assert(kFSmallN == PBG_FLOW_SMALL_DOUBLES, "small-argument flow size");
  if (!out) return fail(PBG_E_INVALID, "null pointer");
  if (!(decay >= 0.0 && decay < 1.0)) return fail(PBG_E_INVALID, "decay must be in [0, 1)");
  build_flow_small(decay, out);
  return PBG_OK;
}

extern "C" PBG_API int pbg_flow_tiny(double decay, double* out) {
  static_assert(kFTinyN == PBG_FLOW_TINY_DOUBLES, "tiny-argument flow size");
  if (!out) return fail(PBG_E_INVALID, "null pointer");
  if (!(decay >= 0.0 && decay < 1.0)) return fail(PBG_E_INVALID, "decay must be in [0, 1)");
  build_flow_tiny(decay, out);
  return PBG_OK;
}

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

// A prepared march (pbg_plan_*): the per-axis tables, segment descriptors and deduplicated
// general-segment factors of one (problem codes, variant, dt, alpha) are built once -- the
// reference's Stepper.__init__ (schemes.py:188-262) -- and every run only launches the step
// kernels, with one host synchronisation at its end (reading the divergence flag).
struct pbg_plan {
  pbg_march_desc d;  // codes / rho pointers stay the caller's
  int nb = 1;        // batched march: nb grids, bs elements apart in every buffer
  long long bs = 0;
  Plan plan;
  SweepArgs ax[3];
  AxisAux aux[3];
  bool extra = false;  // ADI / explicit Euler: march_extra per run
  int* dflag = nullptr;
  int* hflag = nullptr;  // pinned
  int* fq = nullptr;     // work queue of the fused axis-1/axis-2 launch (zero between launches)
  int* fq01 = nullptr;   // work queue of the fused axis-0/axis-1 launch
  cudaEvent_t e0 = nullptr, e1 = nullptr;
};

namespace pbg {
__global__ void k_set_int(int* p, int n, int v) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) p[t] = v;
}
static std::mutex g_prof_mu;

static void plan_free(pbg_plan* p, cudaStream_t st) {
  for (int q = 0; q < 3; ++q) release_axis(p->aux[q], st);
  if (p->dflag) cudaFreeAsync(p->dflag, st);
  if (p->fq) cudaFreeAsync(p->fq, st);
  if (p->fq01) cudaFreeAsync(p->fq01, st);
  if (p->hflag) cudaFreeHost(p->hflag);
  if (p->e0) cudaEventDestroy(p->e0);
  if (p->e1) cudaEventDestroy(p->e1);
  delete p;
}
}  // namespace pbg

static int check_desc(const pbg_march_desc* d) {
  if (!d) return fail(PBG_E_INVALID, "null descriptor");
  int rc = validate_grid(&d->grid);
  if (rc) return rc;
  if (!(d->dt > 0) || !(d->alpha > 0))
    return fail(PBG_E_INVALID, "dt, alpha must be positive");
  if (!d->codes || !d->rho) return fail(PBG_E_INVALID, "null device buffer");
  return PBG_OK;
}

extern "C" PBG_API int pbg_plan_create_batch(const pbg_march_desc* d, int32_t nbatch,
                                             int64_t batch_stride, pbg_plan** out,
                                             void* stream) {
  if (!out) return fail(PBG_E_INVALID, "null output handle");
  *out = nullptr;
  int rc = check_desc(d);
  if (rc) return rc;
  if (nbatch < 1) return fail(PBG_E_INVALID, "nbatch must be >= 1");
  const Layout L0 = make_layout(&d->grid);
  if (nbatch > 1 && (batch_stride < L0.n0 * L0.s0 || batch_stride % L0.pitch))
    return fail(PBG_E_INVALID,
                "batch_stride must cover one pitched grid and be a multiple of the pitch");
  if (nbatch > 1 &&
      (d->variant == PBG_ADI1 || d->variant == PBG_ADI2 || d->variant == PBG_EULER))
    return fail(PBG_E_UNSUPPORTED, "batched marches support the splitting schemes");
  if (!d->work[0]) return fail(PBG_E_INVALID, "null device buffer");
  keep_pool_memory();
  cudaStream_t st = (cudaStream_t)stream;
  pbg_plan* p = new pbg_plan();
  p->d = *d;
  p->nb = nbatch;
  p->bs = nbatch > 1 ? batch_stride : 0;
  auto bail = [&](int code) {
    plan_free(p, st);
    return code;
  };
  if (cudaMallocHost(&p->hflag, nbatch * sizeof(int)) != cudaSuccess ||
      cudaEventCreate(&p->e0) != cudaSuccess || cudaEventCreate(&p->e1) != cudaSuccess)
    return bail(fail(PBG_E_CUDA, "plan allocation failed"));
  if (d->variant == PBG_ADI1 || d->variant == PBG_ADI2 || d->variant == PBG_EULER) {
    p->extra = true;
    *out = p;
    return PBG_OK;
  }
  if (!plan_for(d->variant, p->plan))
    return bail(fail(PBG_E_UNSUPPORTED, "variant not supported by the device march"));
  march_axes(d, p->plan, p->ax);
  for (int axis = 0; axis < 3; ++axis) {
    p->ax[axis].L.nb = p->nb;
    p->ax[axis].L.bs = p->bs;
    p->ax[axis].faces_ok = 1;  // both work buffers' faces hold the Dirichlet data (pbg.h)
    rc = prepare_axis(p->ax[axis], axis, d->codes, p->aux[axis], st);
    if (rc) return bail(rc);
  }
  if (cudaMallocAsync(&p->dflag, p->nb * sizeof(int), st) != cudaSuccess)
    return bail(fail(PBG_E_CUDA, "plan allocation failed"));
  if (p->plan.family <= 1 && fused01_ok(p->ax[0], p->ax[1])) {
    const size_t qb = (size_t)(2 + d->grid.n[2]) * sizeof(int);
    if (cudaMallocAsync(&p->fq01, qb, st) != cudaSuccess ||
        cudaMemsetAsync(p->fq01, 0, qb, st) != cudaSuccess)
      return bail(fail(PBG_E_CUDA, "plan allocation failed"));
  }
  if (p->plan.family <= 1 && fused12_shape(p->ax[1], p->ax[2])) {
    const size_t qb = (size_t)(2 + d->grid.n[0]) * sizeof(int);
    if (cudaMallocAsync(&p->fq, qb, st) != cudaSuccess ||
        cudaMemsetAsync(p->fq, 0, qb, st) != cudaSuccess)
      return bail(fail(PBG_E_CUDA, "plan allocation failed"));
  }
  if (cudaStreamSynchronize(st) != cudaSuccess)  // the plan may run on any stream
    return bail(fail(PBG_E_CUDA, "plan setup failed"));
  *out = p;
  return PBG_OK;
}

extern "C" PBG_API int pbg_plan_create(const pbg_march_desc* d, pbg_plan** out, void* stream) {
  return pbg_plan_create_batch(d, 1, 0, out, stream);
}

extern "C" PBG_API int pbg_plan_destroy(pbg_plan* p, void* stream) {
  if (p) plan_free(p, (cudaStream_t)stream);
  return PBG_OK;
}

extern "C" PBG_API int pbg_plan_run_batch(pbg_plan* p, const double* initial, double* work0,
                                          double* work1, int32_t nsteps,
                                          int32_t check_divergence, int32_t* steps_taken,
                                          int32_t* diverged_step, int32_t* result_slot,
                                          float* device_ms, void* stream) {
  if (!p) return fail(PBG_E_INVALID, "null plan");
  if (!initial || !work0 || !work1) return fail(PBG_E_INVALID, "null device buffer");
  if (nsteps < 1) return fail(PBG_E_INVALID, "nsteps must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  if (p->extra) {
    pbg_march_desc d = p->d;
    d.initial = initial;
    d.work[0] = work0;
    d.work[1] = work1;
    d.nsteps = nsteps;
    d.check_divergence = check_divergence;
    return march_extra(&d, steps_taken, diverged_step, result_slot, device_ms, st);
  }
  const pbg_grid* g = &p->d.grid;
  const Plan& plan = p->plan;
  double* work[2] = {work0, work1};
  int* dflag = p->dflag;
  int rc = PBG_OK;
  const int nb = p->nb;
  k_set_int<<<1, 256, 0, st>>>(dflag, nb, INT_MAX);
  PBG_LAUNCH_CHECK("k_set_int");
  if (check_divergence) {
    for (int b = 0; b < nb; ++b) {
      k_faces_bad<<<148, 256, 0, st>>>(make_layout(g), work0 + b * p->bs,
                                       p->d.divergence_threshold, dflag + b);
      PBG_LAUNCH_CHECK("k_faces_bad");
    }
  }

  int st_idx = -1;
  if (initial == work0) st_idx = 0;
  else if (initial == work1) st_idx = 1;
  const int st0 = st_idx;
  // LOD steps whose axis-2 sweep runs the row-warp kernel may write it in place over the
  // axis-1 output (its lines are staged whole before they are stored), so the step's state
  // stays in one buffer; PBG_FUSE12 = plane chunk of an axis-1/axis-2 interleave (measured
  // slower: launch tails).
  const bool lod_rw = plan.family <= 1 && p->ax[2].rw;
  const int chunk = lod_rw ? env_int("PBG_FUSE12", 0) : 0;
  // LOD sweeps in place on one state buffer when a field is about the L2 size or smaller
  // (c3 257^3: 216 -> 211 us/step, the next sweep re-reads what the previous one left in L2);
  // at 513^3 (8.7x L2) in place measured 2-4% slower, so the ping-pong stays there.
  // PBG_INPLACE=0/1 forces either (profiles/inplace_ab_r02.txt).
  const double field_mb = (double)nb * g->n[0] * g->n[1] * g->pitch * 8.0 / 1e6;
  const bool inpl_all =
      plan.family <= 1 && env_int("PBG_INPLACE", field_mb <= 256.0 ? 1 : 0) != 0;
  // One launch for the axis-1 and axis-2 sweeps (k_sweep_fused12), axis 2 in place over the
  // axis-1 output while it is still in L2.
  const bool fused = p->fq != nullptr && chunk == 0;
  // One launch for the axis-0 and axis-1 sweeps (k_sweep_fused01), axis 1 in place over the
  // axis-0 output while it is still in L2; the axis-2 sweep then runs in place too.
  const bool fused01 = p->fq01 != nullptr && chunk == 0 && !fused;
  const bool inpl =
      inpl_all || fused || (lod_rw && (chunk > 0 || env_int("PBG_INPLACE2", 0) != 0));
  const int nplanes = g->n[0] - 2;

  std::vector<cudaEvent_t> kev;  // per-launch events when profiling is on
  auto mark = [&]() {
    if (!g_profile) return;
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    cudaEventRecord(ev, st);
    kev.push_back(ev);
  };
  PBG_CUDA(cudaEventRecord(p->e0, st));
  for (int s = 1; s <= nsteps && !rc; ++s) {
    const double* X = st_idx < 0 ? initial : work[st_idx];
    const int other = st_idx < 0 ? 0 : 1 - st_idx;
    double* A = work[other];
    double* Bf = st_idx < 0 ? work[1] : work[st_idx];
    SweepArgs as[3];
    for (int axis = 0; axis < 3; ++axis) {
      SweepArgs& a = as[axis];
      a = p->ax[axis];
      a.bnd = work0;  // faces hold the Dirichlet data
      a.step = s;
      a.div_step = check_divergence ? dflag : nullptr;
      a.check = (axis == 2) && check_divergence;
      if (plan.family <= 1) {
        a.src = axis == 0 ? X : (axis == 1 ? A : Bf);
        a.dst = axis == 0 ? A : (axis == 1 ? Bf : (inpl ? Bf : A));
        if (inpl_all) {  // every sweep in place on the state buffer (one field per step)
          a.src = axis == 0 ? X : Bf;
          a.dst = Bf;
        } else if (fused01) {  // axis 0 into the other buffer, axes 1 and 2 in place there
          a.src = axis == 0 ? X : A;
          a.dst = A;
        }
      } else {
        a.src = X;
        a.acc = A;
        a.dst = A;
      }
    }
    for (int axis = 0; axis < 3 && !rc; ++axis) {
      mark();
      if (chunk > 0 && axis == 1) {  // axes 1 and 2 interleaved over plane chunks
        for (int c0 = 0; c0 < nplanes && !rc; c0 += chunk) {
          for (int q = 1; q <= 2 && !rc; ++q) {
            SweepArgs a = as[q];
            a.o0 = c0;
            a.on = std::min(chunk, nplanes - c0);
            rc = launch_sweep(a, q, st);
          }
        }
      } else if (fused01 && axis <= 1) {
        if (axis == 0) rc = launch_fused01(as[0], as[1], p->fq01, st);
      } else if (fused && axis >= 1) {
        if (axis == 1) rc = launch_fused12(as[1], as[2], p->fq, st);
      } else if (!(chunk > 0 && axis == 2)) {
        rc = launch_sweep(as[axis], axis, st);
      }
      mark();
    }
    st_idx = inpl ? (st_idx < 0 ? 1 : st_idx) : other;
  }
  if (rc) {
    cudaStreamSynchronize(st);
    for (auto ev : kev) cudaEventDestroy(ev);
    return rc;
  }
  PBG_CUDA(cudaEventRecord(p->e1, st));
  PBG_CUDA(cudaMemcpyAsync(p->hflag, dflag, nb * sizeof(int), cudaMemcpyDeviceToHost, st));
  PBG_CUDA(cudaStreamSynchronize(st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, p->e0, p->e1);
  if (!kev.empty()) {
    std::lock_guard<std::mutex> lock(g_prof_mu);  // marches may run on several host threads
    for (size_t q = 0; q + 1 < kev.size(); q += 2) {
      float kms = 0.f;
      cudaEventElapsedTime(&kms, kev[q], kev[q + 1]);
      const int axis = (int)((q / 2) % 3);
      g_prof_ms[axis] += kms;
      g_prof_n[axis] += 1;
    }
  }
  for (auto ev : kev) cudaEventDestroy(ev);
  for (int b = 0; b < nb; ++b) {  // per grid: steps taken, divergence, state slot
    const int dstep = p->hflag[b];
    int taken = nsteps;
    if (check_divergence && dstep != INT_MAX) {
      taken = dstep;
      if (diverged_step) diverged_step[b] = dstep;
    } else if (diverged_step) {
      diverged_step[b] = 0;
    }
    int slot;
    if (inpl) slot = st0 < 0 ? 1 : st0;
    else if (st0 < 0) slot = (taken - 1) % 2;
    else slot = (st0 + taken) % 2;
    if (steps_taken) steps_taken[b] = taken;
    if (result_slot) result_slot[b] = slot;
  }
  if (device_ms) *device_ms = ms;
  return PBG_OK;
}

extern "C" PBG_API int pbg_plan_run(pbg_plan* p, const double* initial, double* work0,
                                    double* work1, int32_t nsteps, int32_t check_divergence,
                                    int32_t* steps_taken, int32_t* diverged_step,
                                    int32_t* result_slot, float* device_ms, void* stream) {
  if (p && p->nb != 1) return fail(PBG_E_INVALID, "batched plan: use pbg_plan_run_batch");
  return pbg_plan_run_batch(p, initial, work0, work1, nsteps, check_divergence, steps_taken,
                            diverged_step, result_slot, device_ms, stream);
}

extern "C" PBG_API int pbg_march(const pbg_march_desc* d, int32_t* steps_taken,
                                 int32_t* diverged_step, int32_t* result_slot,
                                 float* device_ms, void* stream) {
  int rc = check_desc(d);
  if (rc) return rc;
  if (d->nsteps < 1) return fail(PBG_E_INVALID, "nsteps must be >= 1");
  if (!d->initial || !d->work[0] || !d->work[1]) return fail(PBG_E_INVALID, "null device buffer");
  pbg_plan* p = nullptr;
  rc = pbg_plan_create(d, &p, stream);
  if (rc) return rc;
  rc = pbg_plan_run(p, d->initial, d->work[0], d->work[1], d->nsteps, d->check_divergence,
                    steps_taken, diverged_step, result_slot, device_ms, stream);
  pbg_plan_destroy(p, stream);
  return rc;
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
  cudaStream_t st = (cudaStream_t)stream;
  AxisAux aux;
  rc = prepare_axis(a, axis, codes, aux, st);
  if (rc) return rc;
  rc = launch_sweep(a, axis, st);
  release_axis(aux, st);
  return rc;
}

