// Slab-decomposed march across ranks; see the section comment below.

#include <algorithm>
#include <climits>
#include <vector>

#include "sweep.cuh"

using namespace pbg;

// ---------------------------------------------------------------------------------------
// Slab-decomposed march: the grid is split along axis 0 into contiguous
// slabs of interior planes, one per rank.  A rank's local grid carries one extra plane on
// each side: the global face on the first / last rank, otherwise a ghost plane.  Axes 1 and
// 2, the flow and the source are rank-local.  The axis-0 sweep couples the ranks; it is
// solved exactly by a two-level partitioned (SPIKE-style) scheme:
//
//   phase A   each rank solves its chunk of every axis-0 line with zero values in the
//             internal ghost planes (true faces kept) and keeps only the chunk's first and
//             last rows g_f, g_l (ends-only mode of k_sweep_strided: 8 B/node read);
//   exchange  all ranks all-gather (g_f, g_l) planes + their divergence flag;
//   interface every rank solves, per line, the 2N-unknown system of chunk end values
//               F_r = g_f + p_f L_{r-1} + q_f F_{r+1},  L_r = g_l + p_l L_{r-1} + q_l F_{r+1}
//             whose responses p, q (the chunk's end rows for a unit ghost value) are static
//             and gathered once at setup; the neighbours' end values become the rank's
//             ghost (Dirichlet) values;
//   phase B   the ordinary axis-0 sweep of the chunk with those ghost values, then the
//             rank-local axis-1 and axis-2 sweeps.
//
// The chunk system with the exact neighbour values is the global system restricted to the
// chunk, so the result equals the single-device march up to reassociation.  CN variants
// also exchange the state's end planes before phase A (the explicit half reads the ghost
// planes).  The caller moves the exchange buffers (NCCL all-gather, or a device copy when
// all partitions live on one GPU).

namespace pbg {

constexpr int kMaxRanks = 16;
constexpr long long kExchTail = 32;  // flag + padding, keeps rank blocks 256-byte aligned

static long long slab_plane(const Layout& L) { return L.s0; }

// x += c*rho on n elements (LODCN2 halo: the ghost planes carry w = u + dta*rho).
__global__ void k_slab_add_source(double* x, const double* rho, double c, long long n) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const double r = rho[t];
    if (r != 0.0) x[t] = __dadd_rn(x[t], __dmul_rn(c, r));
  }
}
static long long slab_elems(const Layout& L) { return 4 * slab_plane(L) + kExchTail; }

// Per line (j, k): block Thomas over the ranks' chunk end values.  recv/coef hold one
// exchange block of E doubles per rank: planes [g_f | g_l | .. ] and [p_f | p_l | q_f | q_l].
__global__ void k_slab_interface(const Layout L, int rank, int nranks, const double* recv,
                                 const double* coef, long long E, double* gb, int* dflag) {
  const long long plane = L.s0;
  if (blockIdx.x == 0 && (int)threadIdx.x < nranks) {
    const int f = *reinterpret_cast<const int*>(recv + threadIdx.x * E + 4 * plane);
    if (f != INT_MAX) atomicMin(dflag, f);
  }
  const int nj = L.n1 - 2, nk = L.n2 - 2;
  const long long nl = (long long)nj * nk;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nl;
       t += (long long)gridDim.x * blockDim.x) {
    const int j = 1 + (int)(t / nk), k = 1 + (int)(t % nk);
    const long long o = L.at(0, j, k);
    double e[kMaxRanks], hh[kMaxRanks], cc[kMaxRanks], dd[kMaxRanks];
    double c = 0.0, d = 0.0;
    for (int r = 0; r < nranks; ++r) {
      const double* G = recv + r * E;
      const double* Q = coef + r * E;
      const double gf = G[o], gl = G[plane + o];
      const double pf = r > 0 ? Q[o] : 0.0, pl = r > 0 ? Q[plane + o] : 0.0;
      const double qf = r + 1 < nranks ? Q[2 * plane + o] : 0.0;
      const double ql = r + 1 < nranks ? Q[3 * plane + o] : 0.0;
      const double inv = 1.0 / (1.0 - pf * d);
      e[r] = (gf + pf * c) * inv;
      hh[r] = qf * inv;
      const double cn = gl + pl * c + pl * d * e[r];
      const double dn = pl * d * hh[r] + ql;
      cc[r] = c = cn;
      dd[r] = d = dn;
    }
    double F = 0.0, Lprev = 0.0, Fnext = 0.0;
    for (int r = nranks - 1; r >= 0; --r) {
      const double Fr = e[r] + hh[r] * F;
      if (r == rank + 1) Fnext = Fr;
      if (r == rank - 1) Lprev = cc[r] + dd[r] * F;
      F = Fr;
    }
    if (rank > 0) gb[o] = Lprev;
    if (rank + 1 < nranks) gb[plane + o] = Fnext;
  }
}

}  // namespace pbg

struct pbg_slab {
  pbg_march_desc d;
  int rank, nranks;
  Plan plan;
  SweepArgs ax[3];
  AxisAux aux[3];
  double* send;
  double* recv;
  double* coef = nullptr;  // nranks exchange blocks: the gathered responses
  double* gbA = nullptr;   // ghost values of phase A: zeros (faces on the outer ranks)
  double* gbB = nullptr;   // ghost values of phase B: the neighbours' chunk end values
  int* dflag = nullptr;
  int st_idx, st0, step;
  long long plane, E;
};

static int slab_state(const pbg_slab* h, const double** X, double** A, double** Bf) {
  const pbg_march_desc* d = &h->d;
  *X = h->st_idx < 0 ? d->initial : d->work[h->st_idx];
  const int other = h->st_idx < 0 ? 0 : 1 - h->st_idx;
  *A = d->work[other];
  *Bf = h->st_idx < 0 ? d->work[1] : d->work[h->st_idx];
  return other;
}

extern "C" PBG_API int64_t pbg_slab_exchange_elems(const pbg_grid* local) {
  if (!local) return -1;
  return slab_elems(make_layout(local));
}

extern "C" PBG_API int pbg_slab_destroy(pbg_slab* h, void* stream) {
  if (!h) return PBG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  for (int q = 0; q < 3; ++q) release_axis(h->aux[q], st);
  if (h->coef) cudaFreeAsync(h->coef, st);
  if (h->gbA) cudaFreeAsync(h->gbA, st);
  if (h->gbB) cudaFreeAsync(h->gbB, st);
  if (h->dflag) cudaFreeAsync(h->dflag, st);
  cudaStreamSynchronize(st);
  delete h;
  return PBG_OK;
}

extern "C" PBG_API int pbg_slab_create(const pbg_march_desc* d, int32_t rank, int32_t nranks,
                                       double* send, double* recv, pbg_slab** out,
                                       void* stream) {
  if (!d || !out) return fail(PBG_E_INVALID, "null descriptor");
  *out = nullptr;
  int rc = validate_grid(&d->grid);
  if (rc) return rc;
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks)
    return fail(PBG_E_INVALID, "rank / nranks out of range (1 <= nranks <= 16)");
  if (!send || !recv) return fail(PBG_E_INVALID, "null exchange buffer");
  Plan plan;
  if (!plan_for(d->variant, plan))
    return fail(PBG_E_UNSUPPORTED, "variant not supported by the device march");
  if (plan.family > 1 || d->variant == PBG_LODCN1)
    return fail(PBG_E_UNSUPPORTED,
                "slab march supports LODIE1, LODIE2 and LODCN2 (AOS/MAOS/LODCN1: single device)");
  if (!(d->dt > 0) || !(d->alpha > 0) || d->nsteps < 1)
    return fail(PBG_E_INVALID, "dt, alpha must be positive and nsteps >= 1");
  if (!d->codes || !d->rho || !d->initial || !d->work[0] || !d->work[1])
    return fail(PBG_E_INVALID, "null device buffer");
  cudaStream_t st = (cudaStream_t)stream;
  pbg_slab* h = new pbg_slab();
  h->d = *d;
  h->rank = rank;
  h->nranks = nranks;
  h->plan = plan;
  h->send = send;
  h->recv = recv;
  march_axes(d, plan, h->ax);
  for (int axis = 0; axis < 3; ++axis) {
    rc = prepare_axis(h->ax[axis], axis, d->codes, h->aux[axis], st);
    if (rc) {
      pbg_slab_destroy(h, stream);
      return rc;
    }
  }
  const Layout L = make_layout(&d->grid);
  h->plane = slab_plane(L);
  h->E = slab_elems(L);
  const size_t pb = h->plane * sizeof(double);
  const bool first = rank == 0, last = rank == nranks - 1;
  auto cu = [&](cudaError_t e) {
    if (e != cudaSuccess) {
      fail(PBG_E_CUDA, cudaGetErrorString(e));
      return false;
    }
    return true;
  };
  double* zeros = nullptr;
  double* unit = nullptr;
  const long long nelem = (long long)L.n0 * L.s0 + 64;
  bool ok = cu(cudaMallocAsync(&h->coef, nranks * h->E * sizeof(double), st)) &&
            cu(cudaMallocAsync(&h->gbA, 2 * pb, st)) && cu(cudaMallocAsync(&h->gbB, 2 * pb, st)) &&
            cu(cudaMallocAsync(&h->dflag, sizeof(int), st)) &&
            cu(cudaMallocAsync(&zeros, nelem * sizeof(double), st)) &&
            cu(cudaMallocAsync(&unit, 2 * pb, st)) &&
            cu(cudaMemsetAsync(zeros, 0, nelem * sizeof(double), st)) &&
            cu(cudaMemsetAsync(h->gbA, 0, 2 * pb, st));
  if (ok) {  // outer ranks keep the true faces as their fixed Dirichlet values
    const double* w = d->work[0];
    if (first) ok = cu(cudaMemcpyAsync(h->gbA, w, pb, cudaMemcpyDeviceToDevice, st));
    if (ok && last)
      ok = cu(cudaMemcpyAsync(h->gbA + h->plane, w + (L.n0 - 1) * h->plane, pb,
                              cudaMemcpyDeviceToDevice, st));
    if (ok) ok = cu(cudaMemcpyAsync(h->gbB, h->gbA, 2 * pb, cudaMemcpyDeviceToDevice, st));
  }
  if (ok) {
    const int init = INT_MAX;
    ok = cu(cudaMemcpyAsync(h->dflag, &init, sizeof(init), cudaMemcpyHostToDevice, st));
  }
  // Static responses of the chunk's end rows to a unit low / high ghost value: the same
  // kernel on a zero field without prologue, so the arithmetic matches phase A.
  for (int side = 0; ok && side < 2; ++side) {
    std::vector<double> hv(2 * h->plane, 0.0);
    for (long long q = 0; q < h->plane; ++q) hv[side * h->plane + q] = 1.0;
    ok = cu(cudaMemcpyAsync(unit, hv.data(), 2 * pb, cudaMemcpyHostToDevice, st)) &&
         cu(cudaStreamSynchronize(st));
    if (!ok) break;
    SweepArgs a = h->ax[0];
    a.pro = PRO_NONE;
    a.has_extra = 0;
    a.epi = EPI_STORE;
    a.check = 0;
    a.src = zeros;
    a.rho = zeros;
    a.dst = zeros;
    a.bnd = unit;
    a.hi_off = h->plane;
    a.ends = send + 2 * side * h->plane;
    a.ends_off = h->plane;
    a.step = 1;
    a.div_step = nullptr;
    if (launch_sweep(a, 0, st)) ok = false;
  }
  if (ok) {
    const int init = INT_MAX;
    ok = cu(cudaMemcpyAsync(send + 4 * h->plane, &init, sizeof(init), cudaMemcpyHostToDevice,
                            st));
  }
  if (ok && d->check_divergence) {
    k_faces_bad<<<148, 256, 0, st>>>(L, d->work[0], d->divergence_threshold, h->dflag,
                                     first ? 0 : 1, last ? 0 : 1);
    ok = cudaGetLastError() == cudaSuccess || (fail(PBG_E_CUDA, "k_faces_bad"), false);
  }
  if (zeros) cudaFreeAsync(zeros, st);
  if (unit) cudaFreeAsync(unit, st);
  if (ok) ok = cu(cudaStreamSynchronize(st));
  if (!ok) {
    pbg_slab_destroy(h, stream);
    return PBG_E_CUDA;
  }
  h->st_idx = -1;
  if (d->initial == d->work[0]) h->st_idx = 0;
  else if (d->initial == d->work[1]) h->st_idx = 1;
  h->st0 = h->st_idx;
  h->step = 0;
  *out = h;
  return PBG_OK;
}

extern "C" PBG_API int pbg_slab_setup(pbg_slab* h, void* stream) {
  if (!h) return fail(PBG_E_INVALID, "null slab");
  cudaStream_t st = (cudaStream_t)stream;
  PBG_CUDA(cudaMemcpyAsync(h->coef, h->recv, h->nranks * h->E * sizeof(double),
                           cudaMemcpyDeviceToDevice, st));
  return PBG_OK;
}

extern "C" PBG_API int pbg_slab_halo_pack(pbg_slab* h, void* stream) {
  if (!h) return fail(PBG_E_INVALID, "null slab");
  cudaStream_t st = (cudaStream_t)stream;
  const double *X;
  double *A, *Bf;
  slab_state(h, &X, &A, &Bf);
  const int n0 = h->d.grid.n[0];
  const size_t pb = h->plane * sizeof(double);
  PBG_CUDA(cudaMemcpyAsync(h->send, X + h->plane, pb, cudaMemcpyDeviceToDevice, st));
  PBG_CUDA(cudaMemcpyAsync(h->send + h->plane, X + (n0 - 2) * h->plane, pb,
                           cudaMemcpyDeviceToDevice, st));
  if (h->ax[0].pro == PRO_SRC) {  // the CN stencil of the first sweep reads w = u + dta*rho
    const double* rho = h->d.rho;
    k_slab_add_source<<<148, 256, 0, st>>>(h->send, rho + h->plane, h->ax[0].pro_coef,
                                           h->plane);
    k_slab_add_source<<<148, 256, 0, st>>>(h->send + h->plane, rho + (n0 - 2) * h->plane,
                                           h->ax[0].pro_coef, h->plane);
    PBG_LAUNCH_CHECK("k_slab_add_source");
  }
  return PBG_OK;
}

extern "C" PBG_API int pbg_slab_halo_unpack(pbg_slab* h, void* stream) {
  if (!h) return fail(PBG_E_INVALID, "null slab");
  cudaStream_t st = (cudaStream_t)stream;
  const double *X;
  double *A, *Bf;
  slab_state(h, &X, &A, &Bf);
  double* Xw = const_cast<double*>(X);  // ghost planes only; never the owned planes
  const int n0 = h->d.grid.n[0];
  const size_t pb = h->plane * sizeof(double);
  if (h->rank > 0)
    PBG_CUDA(cudaMemcpyAsync(Xw, h->recv + (h->rank - 1) * h->E + h->plane, pb,
                             cudaMemcpyDeviceToDevice, st));
  if (h->rank + 1 < h->nranks)
    PBG_CUDA(cudaMemcpyAsync(Xw + (n0 - 1) * h->plane, h->recv + (h->rank + 1) * h->E, pb,
                             cudaMemcpyDeviceToDevice, st));
  return PBG_OK;
}

extern "C" PBG_API int pbg_slab_step_a(pbg_slab* h, void* stream) {
  if (!h) return fail(PBG_E_INVALID, "null slab");
  cudaStream_t st = (cudaStream_t)stream;
  const double *X;
  double *A, *Bf;
  slab_state(h, &X, &A, &Bf);
  SweepArgs a = h->ax[0];
  a.step = h->step + 1;
  a.div_step = h->d.check_divergence ? h->dflag : nullptr;
  a.src = X;
  a.dst = A;  // not written in ends-only mode
  a.bnd = h->gbA;
  a.hi_off = h->plane;
  a.ends = h->send;
  a.ends_off = h->plane;
  int rc = launch_sweep(a, 0, st);
  if (rc) return rc;
  PBG_CUDA(cudaMemcpyAsync(h->send + 4 * h->plane, h->dflag, sizeof(int),
                           cudaMemcpyDeviceToDevice, st));
  return PBG_OK;
}

extern "C" PBG_API int pbg_slab_step_b(pbg_slab* h, void* stream) {
  if (!h) return fail(PBG_E_INVALID, "null slab");
  cudaStream_t st = (cudaStream_t)stream;
  const double *X;
  double *A, *Bf;
  const int other = slab_state(h, &X, &A, &Bf);
  const Layout L = make_layout(&h->d.grid);
  k_slab_interface<<<148 * 4, 256, 0, st>>>(L, h->rank, h->nranks, h->recv, h->coef, h->E,
                                            h->gbB, h->dflag);
  PBG_LAUNCH_CHECK("k_slab_interface");
  const int s = h->step + 1;
  for (int axis = 0; axis < 3; ++axis) {
    SweepArgs a = h->ax[axis];
    a.step = s;
    a.div_step = h->d.check_divergence ? h->dflag : nullptr;
    a.src = axis == 0 ? X : (axis == 1 ? A : Bf);
    a.dst = axis == 0 ? A : (axis == 1 ? Bf : A);
    if (axis == 0) {
      a.bnd = h->gbB;
      a.hi_off = h->plane;
    }
    int rc = launch_sweep(a, axis, st);
    if (rc) return rc;
  }
  h->st_idx = other;
  h->step = s;
  return PBG_OK;
}

extern "C" PBG_API int pbg_slab_flag_pack(pbg_slab* h, void* stream) {
  if (!h) return fail(PBG_E_INVALID, "null slab");
  PBG_CUDA(cudaMemcpyAsync(h->send + 4 * h->plane, h->dflag, sizeof(int),
                           cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return PBG_OK;
}

extern "C" PBG_API int pbg_slab_finish(pbg_slab* h, int32_t* steps_taken,
                                       int32_t* diverged_step, int32_t* result_slot,
                                       void* stream) {
  if (!h) return fail(PBG_E_INVALID, "null slab");
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int> flags(h->nranks);
  for (int r = 0; r < h->nranks; ++r)
    PBG_CUDA(cudaMemcpyAsync(&flags[r], h->recv + r * h->E + 4 * h->plane, sizeof(int),
                             cudaMemcpyDeviceToHost, st));
  int local = INT_MAX;
  PBG_CUDA(cudaMemcpyAsync(&local, h->dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
  PBG_CUDA(cudaStreamSynchronize(st));
  int dstep = local;
  for (int f : flags) dstep = std::min(dstep, f);
  const int nsteps = h->step;
  int taken = nsteps;
  if (h->d.check_divergence && dstep != INT_MAX) taken = std::min(dstep, nsteps);
  if (diverged_step) *diverged_step = (h->d.check_divergence && dstep != INT_MAX) ? taken : 0;
  int slot;
  if (h->st0 < 0) slot = (taken - 1) % 2;
  else slot = (h->st0 + taken) % 2;
  if (steps_taken) *steps_taken = taken;
  if (result_slot) *result_slot = slot;
  return PBG_OK;
}
