// Shared declarations of the sweep engine (sweep.cu) for the other march drivers
// (slab.cu: multi-GPU slab march, schemes_extra.cu: ADI / explicit Euler).
#pragma once

#include <cstdint>

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

constexpr int kSeg = 32;   // segments per line, contiguous axis (one warp lane each)

struct AxisCoef {
  double diag[4];  // [em*2 + ep]  1 + f*(e_plus + e_minus)
  double sub[2];   // [em]         -f*e_minus
  double sup[2];   // [ep]         -f*e_plus
  double flo[2];   // [em]         f*e_minus   (low fold, times the face value)
  double fhi[2];   // [ep]         f*e_plus    (high fold)
  double eps[2];   // palette (CN stencil)
};

// Uniform-segment tables: tab[((type*2 + v)*5 + q)*kTabRows + j], type 0 = interior segment,
// 1 = first segment of a line (row 0 has no sub-diagonal), 2 = last segment whose separator is
// the padding row m (its last inner row is row m-1, no super-diagonal); q = inv, g = a*inv,
// cp, alpha, beta.
constexpr int kTabRows = 32;
constexpr int kTabDoubles = 3 * 2 * 5 * kTabRows;
enum { TQ_INV = 0, TQ_G = 1, TQ_CP = 2, TQ_AL = 3, TQ_BE = 4 };

struct SweepArgs {
  Layout L;
  int m;  // interior nodes along the sweep axis
  const double* src;
  const double* bnd;
  const uint8_t* codes;
  const double* rho;
  double* dst;
  const double* acc;
  const double* tab;   // uniform-segment tables (kTabDoubles)
  const double* minv;  // 32x32 inverse of the clean-line reduced system
  const unsigned long long* desc;  // per-segment descriptors (2 words), see k_build_desc
  const double* gfac;  // precomputed factors of general segments (5 x kTabRows each)
  int static_ok;       // the clean-line reduced inverse applies to this axis (32*S in {m, m+1})
  AxisCoef co;
  // Table of the dominant segment kind (interior, palette 0 = solvent) as kernel parameters:
  // with unrolled rows the compiler folds these into constant-bank operands (no loads).
  double tmid[5 * kTabRows];
  int cn;
  double cnc;  // cn_f / h^2
  int pro;
  double pro_coef;
  int has_extra;
  double extra;
  double decay0, decay1;  // flow decay for solute-bit 0 / 1
  double sat0, sat1;      // 2*atanh(decay)
  double pm;
  int epi;
  double epi_coef;
  int* div_step;
  int step;
  double thr;
  int check;
  // Flow interval tables (kFPolyDoubles per palette with decay < 1, sweep.cu flow_poly_table),
  // staged into shared memory by launches that apply the flow; foff[b] = offset of palette
  // b's table, fpoly_n = doubles to stage.
  const double* fpoly;
  int foff[2];
  int fpoly_n;
  // Axis 2 runs a row-warp kernel (line-major descriptors, P = lanes per line), set by
  // prepare_axis: 1 = k_sweep_rowwarp / k_sweep_rowtma (solute bits in store-pass order),
  // 2 = k_sweep_rowlean (solute bits in row order).
  int rw;
  // The far faces (k = n2 - 1) of src and dst hold the same values (march work buffers, or
  // src == dst): k_sweep_rowlean writes the face row back with the line.
  int faces_ok;
  // Small-argument flow of palette 0 (pbg_internal.cuh flow_small), when decay0 < 1.
  int fsmall_on;
  double fsmall[kFSmallN];
  double ftiny[kFTinyN];
  // Strided axes: offset (from the line base) of the high boundary value in bnd; normally
  // plane m+1 of a field, one plane for the two-plane ghost buffers of the slab march.
  long long hi_off;
  // Slab march phase A (ends-only mode): store rows 1 and m of every line into ends[base] /
  // ends[base + ends_off] instead of the field (axis 0 only).
  double* ends;
  long long ends_off;
  // Outer-index range of a launch (axis 1 column tiles: planes i; axis 2 row-warp lines:
  // planes i): planes o0+1 .. o0+on; on = 0 means all interior planes.
  int o0, on;
  // Batched marches: descriptor words per grid (desc + b * dstride is grid b's block);
  // div_step holds one flag per grid.
  long long dstride;
};


// Per-launch-sequence device data of one axis: tables, reduced inverse, segment descriptors.
struct AxisAux {
  double* buf = nullptr;
  unsigned long long* desc = nullptr;
  double* gfac = nullptr;
};

// Variant table (schemes.py:209-262).
struct Plan {
  int family;  // 0: LOD flow-first (IE1/CN1), 1: LOD source-first (IE2/CN2), 2: AOS, 3: MAOS
  double mult;  // sweep factor = mult * dta
  int cn;
  double src[3];
};

SweepArgs base_args(const pbg_grid* g, const pbg_palette* pal, int axis, double factor);
void set_decays(SweepArgs& a, double d0, double d1);
int prepare_axis(SweepArgs& a, int axis, const uint8_t* codes, AxisAux& aux, cudaStream_t st);
void release_axis(AxisAux& aux, cudaStream_t st);
int launch_sweep(const SweepArgs& a, int axis, cudaStream_t st);
bool plan_for(int v, Plan& p);
void march_axes(const pbg_march_desc* d, const Plan& plan, SweepArgs ax[3]);
__global__ void k_faces_bad(const Layout L, const double* x, double thr, int* flag,
                            int skip_lo = 0, int skip_hi = 0);
// ADI1 / ADI2 / explicit Euler marches (schemes_extra.cu), same contract as pbg_march.
int march_extra(const pbg_march_desc* d, int32_t* steps_taken, int32_t* diverged_step,
                int32_t* result_slot, float* device_ms, cudaStream_t st);

}  // namespace pbg
