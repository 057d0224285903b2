// Slab-decomposed march across ranks; see the section comment below.

#include <algorithm>
#include <climits>
#include <cstdlib>
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
// Exchange layouts (doubles; every block a multiple of 32 so rank blocks stay 256-byte
// aligned).  Only interior lines travel, in the compact order c(j, k) = (j-1)*(n2-2) + (k-1)
// (C of them per plane):
//   setup  [p_f | p_l | q_f | q_l] (4C)                       static responses, once
//   halo   [state plane 1 | state plane n0-2] (pitched planes) LODCN2 only, per step
//   step   nchunks blocks, chunk c = interior rows j in [1 + c*J, 1 + (c+1)*J):
//          [header 32: divergence flag | g_f of the chunk's lines | g_l of them]
//          all-gathered chunk by chunk, so the exchange of chunk c overlaps phase A of c+1.
__host__ __device__ static long long rup32(long long n) { return (n + 31) / 32 * 32; }
__host__ __device__ static long long compact_plane(const Layout& L) { return (long long)(L.n1 - 2) * (L.n2 - 2); }
static int chunk_rows(const Layout& L, int nchunks) { return (L.n1 - 2 + nchunks - 1) / nchunks; }
static int n_chunks(const Layout& L, int want) {
  const int J = chunk_rows(L, want);
  return (L.n1 - 2 + J - 1) / J;  // no empty chunk
}
__host__ __device__ static long long chunk_block(const Layout& L, int J, int c) {
  const int rows = min(J, L.n1 - 2 - c * J);
  return kExchTail + rup32(2LL * rows * (L.n2 - 2));
}
static long long setup_elems(const Layout& L) { return rup32(4 * compact_plane(L)) + kExchTail; }
static long long halo_elems(const Layout& L) { return 2 * slab_plane(L) + kExchTail; }
static long long step_elems(const Layout& L, int nchunks) {
  const int J = chunk_rows(L, nchunks), nc = n_chunks(L, nchunks);
  long long t = 0;
  for (int c = 0; c < nc; ++c) t += chunk_block(L, J, c);
  return t;
}
static long long slab_elems(const Layout& L, int nchunks) {
  return std::max(std::max(setup_elems(L), halo_elems(L)), step_elems(L, nchunks));
}
static int slab_chunks_env() {
  const char* e = getenv("PBG_SLAB_CHUNKS");
  const int v = e && *e ? atoi(e) : 4;
  return std::max(1, std::min(v, 64));
}

// Static half of the interface elimination for one line's responses: per rank
//   inv = 1 / (1 - pf d),  hh = qf inv,  d' = pl d hh + ql
// (d = 0 before rank 0).  st[r] = {pf, pl, inv, hh, pl d, d'}.
struct SlabStatic {
  double pf, pl, inv, hh, pld, dd;
};
__device__ __forceinline__ SlabStatic slab_static(int r, int nranks, const double* Q,
                                                  long long C, long long t, double d) {
  SlabStatic s;
  s.pf = r > 0 ? Q[t] : 0.0;
  s.pl = r > 0 ? Q[C + t] : 0.0;
  const double qf = r + 1 < nranks ? Q[2 * C + t] : 0.0;
  const double ql = r + 1 < nranks ? Q[3 * C + t] : 0.0;
  s.inv = 1.0 / (1.0 - s.pf * d);
  s.hh = qf * s.inv;
  s.pld = s.pl * d;
  s.dd = s.pld * s.hh + ql;
  return s;
}

// Lines whose responses equal line 0's on every rank (uni[t] = 1): in a protein problem
// most axis-0 lines are solvent end to end, so their p, q are the same few constants and
// the interface solve reads them from shared memory instead of 4 * nranks doubles per line.
// (Whatever line 0 is, the flag only says "same coefficients as line 0".)
__global__ void k_slab_classify(long long C, int nranks, const double* coef, long long Es,
                                unsigned char* uni, SlabStatic* s0) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // line 0's static elimination, once
    double d = 0.0;
    for (int r = 0; r < nranks; ++r) {
      s0[r] = slab_static(r, nranks, coef + r * Es, C, 0, d);
      d = s0[r].dd;
    }
  }
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < C;
       t += (long long)gridDim.x * blockDim.x) {
    bool same = true;
    for (int r = 0; r < nranks; ++r) {
      const double* Q = coef + r * Es;
      for (int q = 0; q < 4; ++q) same = same && Q[q * C + t] == Q[q * C];
    }
    uni[t] = same ? 1 : 0;
  }
}

// Per line (j, k): block Thomas over the ranks' chunk end values.  recv holds the step
// exchange (chunk blocks, rank-major inside each chunk), coef the gathered setup blocks.
// NR = nranks (compile time: the recurrence lives in registers).  Only the rank's two
// neighbour values leave the kernel: L_{rank-1} and F_{rank+1}.
template <int NR>
__global__ void __launch_bounds__(128, 4)
    k_slab_interface(const Layout L, int rank, const double* recv, const double* coef,
                     long long Es, int J, const unsigned char* uni, const SlabStatic* g0,
                     double* gb, int* dflag) {
  const long long plane = L.s0, C = compact_plane(L);
  const long long B0 = chunk_block(L, J, 0);
  __shared__ SlabStatic s0[NR];
  if ((int)threadIdx.x < NR) s0[threadIdx.x] = g0[threadIdx.x];  // line 0's (k_slab_classify)
  if (blockIdx.x == 0 && blockIdx.y == 0 && (int)threadIdx.x < NR) {
    const int f = *reinterpret_cast<const int*>(recv + threadIdx.x * B0);
    if (f != INT_MAX) atomicMin(dflag, f);
  }
  __syncthreads();
  // grid (k groups, interior rows j): the chunk and its block are uniform per block
  const int nj = L.n1 - 2, nk = L.n2 - 2;
  const int j = 1 + blockIdx.y;
  const int c = (j - 1) / J;
  const long long Bc = chunk_block(L, J, c);
  const long long len = (long long)min(J, nj - c * J) * nk;
  const double* chunk = recv + (long long)NR * c * B0;  // all earlier chunks are full
  for (int k = 1 + blockIdx.x * blockDim.x + threadIdx.x; k <= nk; k += gridDim.x * blockDim.x) {
    const long long t = (long long)(j - 1) * nk + (k - 1);
    const long long o = L.at(0, j, k);
    const long long local = t - (long long)c * J * nk;
    const bool same = uni[t] != 0;
    double gf[NR], gl[NR];  // all loads in flight before the recurrence starts
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const double* G = chunk + r * Bc + kExchTail;
      gf[r] = G[local];
      gl[r] = G[len + local];
    }
    double e[NR], hh[NR];
    double cv = 0.0, cprev = 0.0, dprev = 0.0;  // (c, d) of rank - 1
    auto fwd = [&](int r, const SlabStatic& s) {
      e[r] = (gf[r] + s.pf * cv) * s.inv;
      hh[r] = s.hh;
      cv = gl[r] + s.pl * cv + s.pld * e[r];
      if (r == rank - 1) {
        cprev = cv;
        dprev = s.dd;
      }
    };
    if (same) {
#pragma unroll
      for (int r = 0; r < NR; ++r) fwd(r, s0[r]);
    } else {
      double d = 0.0;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const SlabStatic s = slab_static(r, NR, coef + r * Es, C, t, d);
        d = s.dd;
        fwd(r, s);
      }
    }
    double F = 0.0, Frank = 0.0, Fnext = 0.0;
#pragma unroll
    for (int r = NR - 1; r >= 0; --r) {
      F = e[r] + hh[r] * F;
      if (r == rank + 1) Fnext = F;
      if (r == rank) Frank = F;
    }
    if (rank > 0) gb[o] = cprev + dprev * Frank;
    if (rank + 1 < NR) gb[plane + o] = Fnext;
  }
}

template <int NR>
static void launch_interface_N(const Layout& L, int rank, const double* recv,
                               const double* coef, long long Es, int J,
                               const unsigned char* uni, const SlabStatic* g0, double* gb,
                               int* dflag, cudaStream_t st) {
  const dim3 grid((L.n2 - 2 + 127) / 128, L.n1 - 2);  // 128 registers: four blocks per SM
  k_slab_interface<NR><<<grid, 128, 0, st>>>(L, rank, recv, coef, Es, J, uni, g0, gb, dflag);
}

static void launch_interface(int nranks, const Layout& L, int rank, const double* recv,
                             const double* coef, long long Es, int J, const unsigned char* uni,
                             const SlabStatic* g0, double* gb, int* dflag, cudaStream_t st) {
#define PBG_IFACE(N) \
  case N: launch_interface_N<N>(L, rank, recv, coef, Es, J, uni, g0, gb, dflag, st); break;
  switch (nranks) {
    PBG_IFACE(1) PBG_IFACE(2) PBG_IFACE(3) PBG_IFACE(4) PBG_IFACE(5) PBG_IFACE(6) PBG_IFACE(7)
    PBG_IFACE(8) PBG_IFACE(9) PBG_IFACE(10) PBG_IFACE(11) PBG_IFACE(12) PBG_IFACE(13)
    PBG_IFACE(14) PBG_IFACE(15) PBG_IFACE(16)
  }
#undef PBG_IFACE
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
  unsigned char* uni = nullptr;  // per interior line: responses equal line 0's on every rank
  SlabStatic* s0 = nullptr;      // line 0's static interface elimination, per rank
  int* dflag = nullptr;
  int st_idx, st0, step;
  long long plane, C, Es, Eh;
  int J, nchunks;  // step exchange: chunks of J interior rows j
};

static long long chunk_offset(const pbg_slab* h, int c) {
  return (long long)c * chunk_block(make_layout(&h->d.grid), h->J, 0);
}

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
  return slab_elems(make_layout(local), slab_chunks_env());
}

extern "C" PBG_API int32_t pbg_slab_nchunks(const pbg_slab* h) { return h ? h->nchunks : -1; }

extern "C" PBG_API int pbg_slab_phase(const pbg_slab* h, int32_t phase, int32_t chunk,
                                      int64_t* offset, int64_t* count) {
  if (!h || !offset || !count) return fail(PBG_E_INVALID, "null argument");
  const Layout L = make_layout(&h->d.grid);
  switch (phase) {
    case PBG_SLAB_SETUP: *offset = 0; *count = h->Es; return PBG_OK;
    case PBG_SLAB_HALO: *offset = 0; *count = h->Eh; return PBG_OK;
    case PBG_SLAB_STEP:
      if (chunk < 0 || chunk >= h->nchunks) return fail(PBG_E_INVALID, "chunk out of range");
      *offset = chunk_offset(h, chunk);
      *count = chunk_block(L, h->J, chunk);
      return PBG_OK;
    default: return fail(PBG_E_INVALID, "unknown exchange phase");
  }
}

extern "C" PBG_API int pbg_slab_destroy(pbg_slab* h, void* stream) {
  if (!h) return PBG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  for (int q = 0; q < 3; ++q) release_axis(h->aux[q], st);
  if (h->coef) cudaFreeAsync(h->coef, st);
  if (h->gbA) cudaFreeAsync(h->gbA, st);
  if (h->gbB) cudaFreeAsync(h->gbB, st);
  if (h->uni) cudaFreeAsync(h->uni, st);
  if (h->s0) cudaFreeAsync(h->s0, st);
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
    h->ax[axis].faces_ok = 1;  // both work buffers' faces hold the Dirichlet data (pbg.h)
    rc = prepare_axis(h->ax[axis], axis, d->codes, h->aux[axis], st);
    if (rc) {
      pbg_slab_destroy(h, stream);
      return rc;
    }
  }
  const Layout L = make_layout(&d->grid);
  h->plane = slab_plane(L);
  h->C = compact_plane(L);
  h->Es = setup_elems(L);
  h->Eh = halo_elems(L);
  h->J = chunk_rows(L, slab_chunks_env());
  h->nchunks = n_chunks(L, slab_chunks_env());
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
  bool ok = cu(cudaMallocAsync(&h->coef, nranks * h->Es * sizeof(double), st)) &&
            cu(cudaMallocAsync(&h->gbA, 2 * pb, st)) && cu(cudaMallocAsync(&h->gbB, 2 * pb, st)) &&
            cu(cudaMallocAsync(&h->dflag, sizeof(int), st)) &&
            cu(cudaMallocAsync(&h->uni, (size_t)h->C, st)) &&
            cu(cudaMallocAsync(&h->s0, kMaxRanks * sizeof(SlabStatic), st)) &&
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
    a.ends = send + 2 * side * h->C;
    a.ends_off = h->C;
    a.step = 1;
    a.div_step = nullptr;
    if (launch_sweep(a, 0, st)) ok = false;
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
  PBG_CUDA(cudaMemcpyAsync(h->coef, h->recv, h->nranks * h->Es * sizeof(double),
                           cudaMemcpyDeviceToDevice, st));
  k_slab_classify<<<148 * 4, 256, 0, st>>>(h->C, h->nranks, h->coef, h->Es, h->uni, h->s0);
  PBG_LAUNCH_CHECK("k_slab_classify");
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
    PBG_CUDA(cudaMemcpyAsync(Xw, h->recv + (h->rank - 1) * h->Eh + h->plane, pb,
                             cudaMemcpyDeviceToDevice, st));
  if (h->rank + 1 < h->nranks)
    PBG_CUDA(cudaMemcpyAsync(Xw + (n0 - 1) * h->plane, h->recv + (h->rank + 1) * h->Eh, pb,
                             cudaMemcpyDeviceToDevice, st));
  return PBG_OK;
}

extern "C" PBG_API int pbg_slab_step_a_chunk(pbg_slab* h, int32_t chunk, void* stream) {
  if (!h) return fail(PBG_E_INVALID, "null slab");
  if (chunk < 0 || chunk >= h->nchunks) return fail(PBG_E_INVALID, "chunk out of range");
  cudaStream_t st = (cudaStream_t)stream;
  const double *X;
  double *A, *Bf;
  slab_state(h, &X, &A, &Bf);
  const Layout L = make_layout(&h->d.grid);
  const long long off = chunk_offset(h, chunk);
  const int j0 = chunk * h->J, rows = std::min(h->J, L.n1 - 2 - j0);
  SweepArgs a = h->ax[0];
  a.step = h->step + 1;
  a.div_step = h->d.check_divergence ? h->dflag : nullptr;
  a.src = X;
  a.dst = A;  // not written in ends-only mode
  a.bnd = h->gbA;
  a.hi_off = h->plane;
  a.o0 = j0;  // axis-0 lines (j, k) with j in this chunk
  a.on = rows;
  // the kernel writes ends[c(j, k)] and ends[c(j, k) + ends_off] (compact c): shift the base
  // so the chunk's g_f / g_l land right after its header
  a.ends = h->send + off + kExchTail - (long long)j0 * (L.n2 - 2);
  a.ends_off = (long long)rows * (L.n2 - 2);
  int rc = launch_sweep(a, 0, st);
  if (rc) return rc;
  if (chunk == 0)  // the flag after the previous step rides in chunk 0's header
    PBG_CUDA(cudaMemcpyAsync(h->send, h->dflag, sizeof(int), cudaMemcpyDeviceToDevice, st));
  return PBG_OK;
}

extern "C" PBG_API int pbg_slab_step_a(pbg_slab* h, void* stream) {
  if (!h) return fail(PBG_E_INVALID, "null slab");
  for (int c = 0; c < h->nchunks; ++c) {
    int rc = pbg_slab_step_a_chunk(h, c, stream);
    if (rc) return rc;
  }
  return PBG_OK;
}

extern "C" PBG_API int pbg_slab_step_b(pbg_slab* h, void* stream) {
  if (!h) return fail(PBG_E_INVALID, "null slab");
  cudaStream_t st = (cudaStream_t)stream;
  const double *X;
  double *A, *Bf;
  const int other = slab_state(h, &X, &A, &Bf);
  const Layout L = make_layout(&h->d.grid);
  launch_interface(h->nranks, L, h->rank, h->recv, h->coef, h->Es, h->J, h->uni, h->s0,
                   h->gbB, h->dflag, st);
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
  PBG_CUDA(cudaMemcpyAsync(h->send, h->dflag, sizeof(int), cudaMemcpyDeviceToDevice,
                           (cudaStream_t)stream));
  return PBG_OK;
}

extern "C" PBG_API int pbg_slab_finish(pbg_slab* h, int32_t* steps_taken,
                                       int32_t* diverged_step, int32_t* result_slot,
                                       void* stream) {
  if (!h) return fail(PBG_E_INVALID, "null slab");
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int> flags(h->nranks);
  for (int r = 0; r < h->nranks; ++r)
    PBG_CUDA(cudaMemcpyAsync(&flags[r], h->recv + r * chunk_block(make_layout(&h->d.grid), h->J, 0),
                             sizeof(int), cudaMemcpyDeviceToHost, st));
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
