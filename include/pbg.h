/*
 * pbg.h — C ABI of the B200-native pseudo-transient Poisson–Boltzmann LOD/AOS step.
 *
 * This is the drop-in boundary for the hot path of the reference package `pbsplit`
 * (arXiv 1410.2788).  The reference has no FFI of its own: its boundary is the Python
 * API re-exported by pkg/src/pbsplit/__init__.py:4-21 and the single backend switch
 * `_solve_batch(sub, cp, inv, rhs, dp, out)` (pkg/src/pbsplit/tridiag.py:144-147).
 * Each entry point below names the reference function it replaces.  Python binds these
 * symbols with ctypes (paper_1410_2788_b200/_native.py); INTEGRATION.md shows the stub a
 * pbsplit maintainer would add.
 *
 * Conventions
 *  - All fields are fp64 on the device in the "pitched" layout of pbg_layout():
 *      element (i, j, k) lives at  base[(i*n1 + j)*pitch + k + PBG_OFFSET]
 *    i.e. the reference's C order data[i, j, k] (pbsplit/grid.py:16-22) with the contiguous
 *    k rows padded so that interior node k = 1 starts on a 256-byte boundary.
 *  - Per-node coefficient codes are one uint8 per node in the same layout:
 *      bit 0        node is solute (kappa2 palette index; eps_node == eps_m)
 *      bit 1+a      the half-edge between node p-e_a and p along axis a uses eps palette 1
 *      bit 4        node carries a nonzero deposited source (rho != 0)
 *  - Every call returns 0 on success, a negative PBG_E* code on failure; the message is in
 *    pbg_last_error() (thread-local).  Invalid inputs map to ValueError in Python, exactly
 *    where the reference raises ValueError.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are asynchronous
 *    unless documented otherwise.
 */
#ifndef PBG_H
#define PBG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PBG_API __attribute__((visibility("default")))

#define PBG_OFFSET 31

enum {
  PBG_OK = 0,
  PBG_E_INVALID = -1, /* invalid argument (reference: ValueError) */
  PBG_E_CUDA = -2,    /* CUDA runtime error */
  PBG_E_UNSUPPORTED = -3
};

/* Scheme ids, same order as pbsplit.schemes.SchemeVariant (pbsplit/schemes.py:20-33). */
enum {
  PBG_LODIE1 = 0, PBG_LODIE2 = 1, PBG_LODCN1 = 2, PBG_LODCN2 = 3,
  PBG_AOSIE1 = 4, PBG_AOSIE2 = 5, PBG_AOSCN1 = 6, PBG_AOSCN2 = 7,
  PBG_MAOSIE = 8, PBG_MAOSCN = 9, PBG_ADI1 = 10, PBG_ADI2 = 11, PBG_EULER = 12
};

/* Uniform grid (pbsplit/grid.py:14-35): node coordinate along axis a is lo[a] + h*idx. */
typedef struct pbg_grid {
  int32_t n[3];   /* nodes per axis, boundary included (nx, ny, nz) */
  int64_t pitch;  /* elements per (i, j) row, from pbg_layout() */
  double lo[3];
  double h;
} pbg_grid;

/* Coefficient palettes: the two values a half-edge eps / a node kappa2 can take. */
typedef struct pbg_palette {
  double eps[3][2];  /* eps[a][bit] for half-edges along axis a */
  double kappa2[2];  /* kappa2[bit0] */
} pbg_palette;

/* Pitched layout for an (n0, n1, n2) grid: pitch (elements per row) and total element
 * count to allocate per field.  Pure arithmetic, no device access. */
PBG_API int pbg_layout(int32_t n0, int32_t n1, int32_t n2, int64_t* pitch, int64_t* nelem);

PBG_API const char* pbg_last_error(void);
PBG_API int pbg_version(void);

/* ---------------------------------------------------------------------------------------
 * Layout movement (replaces the reference's np.ascontiguousarray / moveaxis copies).
 * dense: C-contiguous (n0, n1, n2) fp64 array; pitched: pbg_layout buffer.  Device ptrs.
 */
PBG_API int pbg_pitch_from_dense(const pbg_grid* g, const double* dense, double* pitched,
                                 void* stream);
PBG_API int pbg_dense_from_pitched(const pbg_grid* g, const double* pitched, double* dense,
                                   void* stream);
/* Copy only the six boundary faces of src into dst (BoundarySpec.apply, problem.py:63-69). */
PBG_API int pbg_copy_faces(const pbg_grid* g, const double* src, double* dst, void* stream);

/* ---------------------------------------------------------------------------------------
 * Coefficient assembly (north_star item 1).
 *
 * pbg_pack_region: dense RegionMap arrays -> codes + palettes.  Replaces the consumption of
 * RegionMap.eps_half_{x,y,z} / kappa2 by LineSweepSolver.__init__ (tridiag.py:167-181) and
 * Stepper.__init__ (schemes.py:203-212).  eps_half_a has the reference shape (n with n_a-1),
 * C-contiguous; kappa2 and rho are (n0, n1, n2).  Fails with PBG_E_UNSUPPORTED if an array
 * holds more than two distinct values.  Synchronous (reads back the palette).
 */
PBG_API int pbg_pack_region(const pbg_grid* g, const double* eps_half_x,
                            const double* eps_half_y, const double* eps_half_z,
                            const double* kappa2, const double* rho_dense, uint8_t* codes,
                            pbg_palette* palette, void* stream);

/* Inverse of pack: codes + palette -> dense RegionMap arrays (any output may be NULL).
 * eps_node_pal gives the node dielectric for solute-bit 0 / 1 (eps_s, eps_m). */
PBG_API int pbg_expand_region(const pbg_grid* g, const uint8_t* codes, const pbg_palette* pal,
                              const double eps_node_pal[2], double* eps_node,
                              double* eps_half_x, double* eps_half_y, double* eps_half_z,
                              double* kappa2, void* stream);

/* Union-of-spheres classification + kappa2 mask (geometry.py:78-85, 117-156) written
 * straight into codes (bits 0-3).  atoms: device array of natoms x 5 doubles
 * (x, y, z, charge, radius) in generation order.  palette receives the values
 * build_region_maps would use.  codes must be zeroed by the caller or by this call
 * (zero_first != 0). */
PBG_API int pbg_classify_spheres(const pbg_grid* g, const double* atoms, int32_t natoms,
                                 double probe_inflation, double eps_m, double eps_s,
                                 double kappa2_solvent, int32_t zero_first, uint8_t* codes,
                                 pbg_palette* palette, void* stream);

/* Analytic sphere classification (AnalyticSphere.solute_mask, geometry.py:58-60). */
PBG_API int pbg_classify_sphere(const pbg_grid* g, double R, double eps_m, double eps_s,
                                double kappa2_solvent, uint8_t* codes, pbg_palette* palette,
                                void* stream);

/* Trilinear charge deposit (grid.py:205-252), bit-identical and deterministic: qfrac and
 * rho are pitched fp64 (zeroed by this call); if codes is non-NULL it gets bit 4 where
 * rho != 0.
 * Synchronous: validates atom placement, returns PBG_E_INVALID with the reference's
 * message if an atom is not strictly inside the interior. */
PBG_API int pbg_deposit(const pbg_grid* g, const double* atoms, int32_t natoms,
                        double prefactor, double* qfrac, double* rho, uint8_t* codes,
                        void* stream);

/* Set code bit 4 exactly where the pitched source rho is nonzero (clears it elsewhere). */
PBG_API int pbg_mark_charged(const pbg_grid* g, const double* rho_pitched, uint8_t* codes,
                             void* stream);

/* Screened-Coulomb Dirichlet data on the six faces (problem.py:44-61, 106-117), written
 * into the faces of dst (interior untouched).  Synchronous (checks d == 0). */
PBG_API int pbg_coulomb_faces(const pbg_grid* g, const double* atoms, int32_t natoms,
                              double eps_s, double kappa_bar, double* dst, void* stream);

/* ---------------------------------------------------------------------------------------
 * The time step (north_star items 2-4).
 */
typedef struct pbg_march_desc {
  pbg_grid grid;
  pbg_palette pal;
  int32_t variant;          /* PBG_LODIE1 .. PBG_EULER */
  int32_t aos_literal;      /* MarchConfig.aos_nonlinear == "literal" */
  double dt;
  double alpha;             /* already resolved: config.alpha or problem.alpha */
  double divergence_threshold;
  int32_t nsteps;           /* int(round(T/dt)), >= 1 (schemes.py:406-408) */
  int32_t check_divergence; /* 1: march semantics (stop at first bad step); 0: step() */
  const uint8_t* codes;     /* device, pitched */
  const double* rho;        /* device, pitched dense source */
  const double* initial;    /* device, pitched; may alias work[0] when its faces already
                               equal the boundary values */
  double* work[2];          /* device, pitched, faces hold the Dirichlet values */
} pbg_march_desc;

/* march() (schemes.py:399-425) / Stepper.step (schemes.py:365-380) on device.
 * Synchronous at the end (reads the divergence flag once).  *result_slot = index into
 * work[] holding the final field; *steps_taken, *diverged_step (0 = none) as MarchReport.
 * *device_ms = CUDA-event time of the step loop (setup excluded, like wall_time). */
PBG_API int pbg_march(const pbg_march_desc* d, int32_t* steps_taken, int32_t* diverged_step,
                      int32_t* result_slot, float* device_ms, void* stream);

/* A prepared march (the reference's Stepper: schemes.py:188-262 factor once, then step):
 * pbg_plan_create builds the per-axis tables, segment descriptors and deduplicated segment
 * factors for d's codes / variant / dt / alpha (d->codes and d->rho must stay valid for the
 * plan's lifetime; d->work[0] is used for setup only; synchronous).  pbg_plan_run marches
 * nsteps from `initial` with the two work buffers (faces = Dirichlet data, as pbg_march),
 * launching only the step kernels and synchronising once at the end; check_divergence 1 =
 * march semantics, 0 = Stepper.step / step() (schemes.py:365-396).  Outputs as pbg_march.
 * pbg_march == create + run + destroy.  A plan may run on any stream, one run at a time. */
typedef struct pbg_plan pbg_plan;
PBG_API int pbg_plan_create(const pbg_march_desc* d, pbg_plan** out, void* stream);
PBG_API int pbg_plan_run(pbg_plan* p, const double* initial, double* work0, double* work1,
                         int32_t nsteps, int32_t check_divergence, int32_t* steps_taken,
                         int32_t* diverged_step, int32_t* result_slot, float* device_ms,
                         void* stream);
PBG_API int pbg_plan_destroy(pbg_plan* p, void* stream);

/* Batched plans (config 5: many independent grids of one shape; SURVEY.md §8e "batched into
 * one launch per sweep"): d->grid describes ONE grid; codes, rho, initial and work[] hold
 * nbatch such grids batch_stride elements apart (batch_stride >= the pitched grid size and a
 * multiple of the pitch); all grids share d->pal.  Every sweep is one launch over the lines
 * of all grids; divergence is tracked per grid (a grid that stops is skipped by the later
 * steps).  steps_taken / diverged_step / result_slot are arrays of nbatch.  Splitting
 * schemes only.  pbg_plan_create == create_batch with nbatch 1. */
PBG_API int pbg_plan_create_batch(const pbg_march_desc* d, int32_t nbatch,
                                  int64_t batch_stride, pbg_plan** out, void* stream);
PBG_API int pbg_plan_run_batch(pbg_plan* p, const double* initial, double* work0,
                               double* work1, int32_t nsteps, int32_t check_divergence,
                               int32_t* steps_taken, int32_t* diverged_step,
                               int32_t* result_slot, float* device_ms, void* stream);

/* Per-sweep-kernel timing (CUDA events around every launch inside pbg_march, on the
 * launching stream).  pbg_set_profiling(1) enables and resets the accumulators;
 * pbg_get_profile returns the summed milliseconds and launch counts per sweep axis. */
PBG_API int pbg_set_profiling(int32_t on);
PBG_API int pbg_get_profile(double axis_ms[3], int64_t launches[3]);

/* Same march from HOST buffers: uploads the inputs, marches, downloads the final field.
 *   codes_pitched_host  uint8 codes in the pitched layout (pbg_layout nelem bytes)
 *   rho_nnz/idx/val     the deposited source as (flat C-order node index, value) pairs
 *   faces_host          Dirichlet data packed face by face: x-lo (n1*n2), x-hi, y-lo (n0*n2),
 *                       y-hi, z-lo (n0*n1), z-hi, each row-major in its remaining axes
 *   initial_dense_host  C-contiguous (n0,n1,n2) initial field, or NULL for the reference's
 *                       protein default (zero interior, Dirichlet faces; problem.py:227-228)
 *   final_dense_host    receives the final field, C-contiguous (n0,n1,n2)
 * Pointers inside d_template (codes, rho, initial, work) are ignored.  This is the call a
 * reference-side FFI binding makes; pinned host memory is fastest. */
PBG_API int pbg_march_host(const pbg_march_desc* d_template, const uint8_t* codes_pitched_host,
                           int64_t rho_nnz, const int64_t* rho_idx, const double* rho_val,
                           const double* faces_host, const double* initial_dense_host,
                           double* final_dense_host, int32_t* steps_taken,
                           int32_t* diverged_step, float* device_ms, void* stream);

/* Scatter packed faces (layout as in pbg_march_host) into the faces of dst0 (and dst1 if
 * non-NULL). */
PBG_API int pbg_unpack_faces(const pbg_grid* g, const double* packed, double* dst0,
                             double* dst1, void* stream);

/* One implicit sweep (ie_sweep / cn_sweep, schemes.py:146-176): solves
 * (1 - factor*d2_axis) out = rhs (+ CN explicit half when cn != 0) on every interior line.
 * src: field whose interior is the rhs (and whose faces feed the CN stencil); bnd: field
 * whose faces hold the Dirichlet data; dst interior receives the solution. */
PBG_API int pbg_sweep(const pbg_grid* g, const pbg_palette* pal, const uint8_t* codes,
                      int32_t axis, double factor, int32_t cn, const double* src,
                      const double* bnd, double* dst, void* stream);

/* ---------------------------------------------------------------------------------------
 * Slab-decomposed march (no reference counterpart -- the reference is
 * single-process).  The grid is split along axis 0; rank r owns a contiguous range of
 * interior planes and describes its LOCAL grid in d: n[0] = owned planes + 2, plane 0 and
 * plane n[0]-1 are the global faces on the first / last rank and ghost planes otherwise
 * (their initial contents: the neighbours' initial values).  codes, rho, initial and work[]
 * are the local slabs of the global pitched buffers (planes [first-1, last+1]), which share
 * the global layout.  Variants: LODIE1, LODIE2, LODCN2.
 *
 * Exchange buffers (device, owned by the caller): send holds pbg_slab_exchange_elems(local)
 * doubles, recv nranks times that; after every *pack / step_a(_chunk) call the caller
 * all-gathers the phase's part of send (pbg_slab_phase) into recv in rank order
 * (ncclAllGather, or a device copy when all partitions live on one GPU) before step_b.
 *
 *   create            computes this rank's static responses into send  -> all-gather
 *   setup             keeps the gathered responses
 *   per step:  [halo_pack -> all-gather -> halo_unpack]   (CN only)
 *              step_a  (chunk solve, end rows + divergence flag into send) -> all-gather
 *              step_b  (interface solve, axis-0 chunk sweep, axis-1, axis-2 sweeps)
 *   flag_pack -> all-gather -> finish  (steps taken / divergence agreed over all ranks;
 *                                       *result_slot indexes work[] as in pbg_march)
 * Results equal pbg_march on the whole grid up to reassociation (parity tests). */
typedef struct pbg_slab pbg_slab;
/* Doubles of the send buffer (recv: nranks times that) for a local grid. */
PBG_API int64_t pbg_slab_exchange_elems(const pbg_grid* local);
/* Exchange phases: which part of send travels (offset, count in doubles); the gathered
 * blocks land rank-major at recv + nranks*offset.  SETUP: the static responses (once);
 * HALO: the state's end planes (LODCN2, per step); STEP: chunk `chunk` of the end rows of
 * phase A + the divergence flag (per step, one all-gather per chunk so that the exchange of
 * chunk c overlaps phase A of chunk c+1).  Only interior lines travel (compact planes of
 * (n1-2)*(n2-2) values).  PBG_SLAB_CHUNKS (env, default 4) sets the chunk count; it must be
 * the same on every rank. */
enum { PBG_SLAB_SETUP = 0, PBG_SLAB_HALO = 1, PBG_SLAB_STEP = 2 };
PBG_API int32_t pbg_slab_nchunks(const pbg_slab* h);
PBG_API int pbg_slab_phase(const pbg_slab* h, int32_t phase, int32_t chunk, int64_t* offset,
                           int64_t* count);
/* Phase A of one chunk (axis-0 lines with j in the chunk); pbg_slab_step_a = all chunks. */
PBG_API int pbg_slab_step_a_chunk(pbg_slab* h, int32_t chunk, void* stream);
PBG_API int pbg_slab_create(const pbg_march_desc* d, int32_t rank, int32_t nranks,
                            double* send, double* recv, pbg_slab** out, void* stream);
PBG_API int pbg_slab_setup(pbg_slab* h, void* stream);
PBG_API int pbg_slab_halo_pack(pbg_slab* h, void* stream);
PBG_API int pbg_slab_halo_unpack(pbg_slab* h, void* stream);
PBG_API int pbg_slab_step_a(pbg_slab* h, void* stream);
PBG_API int pbg_slab_step_b(pbg_slab* h, void* stream);
PBG_API int pbg_slab_flag_pack(pbg_slab* h, void* stream);
PBG_API int pbg_slab_finish(pbg_slab* h, int32_t* steps_taken, int32_t* diverged_step,
                            int32_t* result_slot, void* stream);
PBG_API int pbg_slab_destroy(pbg_slab* h, void* stream);

/* nonlinear_step (schemes.py:106-120) on n contiguous elements with per-element kappa2:
 * out = pm * flow(w; decay = exp(-coef * kappa2)), coef = rate*dt/alpha. */
PBG_API int pbg_flow_dense(int64_t n, const double* w, const double* kappa2, double coef,
                           double premultiplier, double* out, void* stream);

/* Host only (no device needed): the interval table the sweep kernels evaluate the flow
 * 2*artanh(decay*tanh(w/2)) with (|w| <= 38, 0 <= decay < 1): PBG_FLOW_TABLE_DOUBLES
 * doubles, 84 intervals of 12 [centre, a0..a9, 0], interval index = (hi word of |w|+1 >> 16)
 * - 0x3FF0, value = sum a_q (|w| - centre)^q with the sign of w.  Replaces the per-node
 * tanh/atanh of _apply_flow (schemes.py:88-103) on the hot path; exported for testing. */
#define PBG_FLOW_TABLE_DOUBLES 1008
PBG_API int pbg_flow_table(double decay, double* out);

/* Host only: the small-argument form the sweep kernels use for solvent nodes with
 * |w| <= 2 (before the table): flow = w * sum g_q t^q, t = fma(w, w, -2), q = 0..15
 * (PBG_FLOW_SMALL_DOUBLES coefficients g_q, Horner with fma).  Same replaced reference
 * code as pbg_flow_table; exported for testing. */
#define PBG_FLOW_SMALL_DOUBLES 16
PBG_API int pbg_flow_small(double decay, double* out);

/* Host only: the tier used first, for |w| <= 0.5: flow = w * sum g_q t^q,
 * t = fma(w, w, -0.125), q = 0..7 (PBG_FLOW_TINY_DOUBLES coefficients).  Exported for
 * testing. */
#define PBG_FLOW_TINY_DOUBLES 8
PBG_API int pbg_flow_tiny(double decay, double* out);

/* Direct vacuum Poisson solve (vacuum_potential_fast, energy.py:59-85): -eps_m * d2(out) =
 * rho on the interior with out = bnd on the faces (bnd: pitched field whose faces hold the
 * Dirichlet data).  Boundary lifting, type-I DST along each axis (cuFFT D2Z of the odd
 * extension), eigenvalue divide, inverse DST.  Synchronous; scratch ~5 interior-sized
 * fp64 arrays. */
PBG_API int pbg_vacuum_dst(const pbg_grid* g, double eps_m, const double* rho,
                           const double* bnd, double* out, void* stream);

/* ---------------------------------------------------------------------------------------
 * Energy (north_star item 5).
 *
 * pbg_energy_atoms: 0.5 * KCAL * sum_a q_a * sum_corners w * dphi, where
 *   dphi = (ca*phi_m_a + cb*phi_m_b) - (cc*phi_0_a + cd*phi_0_b)
 * (ca, cb) = (2, -1) fuses richardson() (energy.py:99-106); (1, 0) is the plain field.
 * Null phi_*_b pointers are treated as zero.  Deterministic fixed-order reduction.
 * Equals solvation_energy(qfrac, phi_m, phi_0) (energy.py:31-43) up to summation order.
 * Synchronous. */
PBG_API int pbg_energy_atoms(const pbg_grid* g, const double* atoms, int32_t natoms,
                             const double* phi_m_a, const double* phi_m_b, double ca,
                             double cb, const double* phi_0_a, const double* phi_0_b,
                             double cc, double cd, double kcal, double* delta_g,
                             void* stream);

/* Dense form of solvation_energy: sum over all nodes of qfrac*(phi_m - phi_0) (pitched
 * inputs), times 0.5*kcal.  Synchronous. */
PBG_API int pbg_energy_dense(const pbg_grid* g, const double* qfrac, const double* phi_m,
                             const double* phi_0, double kcal, double* delta_g, void* stream);

/* out = ca*a + cb*b on every node (richardson: ca=2 on phi(dt/2), cb=-1 on phi(dt)). */
PBG_API int pbg_axpby(const pbg_grid* g, double ca, const double* a, double cb,
                      const double* b, double* out, void* stream);

/* max |x| over all nodes (NaN-propagating) -- used by step() / tests.  Synchronous. */
PBG_API int pbg_maxabs(const pbg_grid* g, const double* x, double* result, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PBG_H */
