// Comparison schemes of the reference on the device:
//   ADI1 / ADI2  (pbsplit/schemes.py:240-247, 331-353): flow, explicit delta2 terms of the
//                other axes, three implicit line sweeps (the tile kernel of sweep.cu);
//   ExplicitEuler (schemes.py:248-253, 355-363): one fused 7-point stencil + masked sinh
//                reaction per step.
// Same march contract as pbg_march (ping-pong work buffers whose faces hold the Dirichlet
// data, device divergence flag = first bad step, kernels of later steps exit at once).
// Arithmetic follows the reference expression order (numpy evaluation order) so results
// agree to rounding of the individual operations.

#include <climits>
#include <cmath>
#include <vector>

#include "sweep.cuh"

namespace pbg {

struct PalDev {
  double eps[3][2];
  double k2[2];
  double decay[2], sat[2];
};

// Interior node t -> (i, j, k), k fastest.
__device__ __forceinline__ void node_of(const Layout& L, long long t, int& i, int& j, int& k) {
  const int nk = L.n2 - 2, nj = L.n1 - 2;
  k = 1 + (int)(t % nk);
  const long long r = t / nk;
  j = 1 + (int)(r % nj);
  i = 1 + (int)(r / nj);
}

__device__ __forceinline__ long long interior_count(const Layout& L) {
  return (long long)(L.n0 - 2) * (L.n1 - 2) * (L.n2 - 2);
}

// delta2_block (schemes.py:123-143) at node o along axis a (stride st): the half-edge eps
// bit of edge (p-1, p) lives at node p (bit 1 + a of the code).
__device__ __forceinline__ double delta2_at(const PalDev& P, const uint8_t* codes,
                                            const double* u, long long o, long long st, int a) {
  const uint32_t em = (codes[o] >> (1 + a)) & 1u, ep = (codes[o + st] >> (1 + a)) & 1u;
  const double c = u[o];
  return __dadd_rn(__dmul_rn(P.eps[a][ep], __dsub_rn(u[o + st], c)),
                   __dmul_rn(P.eps[a][em], __dsub_rn(u[o - st], c)));
}

__device__ __forceinline__ bool bad(double v, double thr) { return !isfinite(v) || fabs(v) > thr; }

// u_new = u + dta * ((lap - react) + rho), lap = (d0 + d1 + d2) / h^2, react = k2 sinh(u)
// where k2 > 0 (schemes.py:355-363).
__global__ void k_euler(const Layout L, PalDev P, const uint8_t* __restrict__ codes,
                        const double* __restrict__ x, const double* __restrict__ rho,
                        double dta, double h2, double* __restrict__ out, int* flag, int step,
                        double thr, int check) {
  if (flag && *((volatile int*)flag) < step) return;
  bool b = false;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < interior_count(L);
       t += (long long)gridDim.x * blockDim.x) {
    int i, j, k;
    node_of(L, t, i, j, k);
    const long long o = L.at(i, j, k);
    const double d0 = delta2_at(P, codes, x, o, L.s0, 0);
    const double d1 = delta2_at(P, codes, x, o, L.pitch, 1);
    const double d2 = delta2_at(P, codes, x, o, 1, 2);
    const double lap = __ddiv_rn(__dadd_rn(__dadd_rn(d0, d1), d2), h2);
    const double u = x[o];
    const double k2 = P.k2[codes[o] & 1u];
    const double react = k2 > 0.0 ? __dmul_rn(k2, sinh(u)) : 0.0;
    const double v = __dadd_rn(u, __dmul_rn(dta, __dadd_rn(__dsub_rn(lap, react), rho[o])));
    out[o] = v;
    b |= check && bad(v, thr);
  }
  if (check && __any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicMin(flag, step);
}

// out = pm * flow(src) on the interior (exact reference map, tanh / atanh).
__global__ void k_flow_field(const Layout L, PalDev P, const uint8_t* __restrict__ codes,
                             const double* __restrict__ src, double* __restrict__ out,
                             int* flag, int step, double thr, int check) {
  if (flag && *((volatile int*)flag) < step) return;
  bool b = false;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < interior_count(L);
       t += (long long)gridDim.x * blockDim.x) {
    int i, j, k;
    node_of(L, t, i, j, k);
    const long long o = L.at(i, j, k);
    const double v = sinh_flow(src[o], P.decay[codes[o] & 1u], 1.0);
    out[o] = v;
    b |= check && bad(v, thr);
  }
  if (check && __any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicMin(flag, step);
}

// ADI right-hand side from the flowed field w: sy = delta2_y(w)/h^2, sz = delta2_z(w)/h^2,
// rhs = w + dta*((sy + sz) + rho)                  (ADI1, schemes.py:331-342)
// rhs = w + dta*(((0.5 sx + sy) + sz) + rho)       (ADI2, schemes.py:344-353)
__global__ void k_adi_rhs(const Layout L, PalDev P, const uint8_t* __restrict__ codes,
                          const double* __restrict__ w, const double* __restrict__ rho,
                          double dta, double h2, int adi2, double* __restrict__ rhs,
                          double* __restrict__ sy, double* __restrict__ sz, int* flag,
                          int step) {
  if (flag && *((volatile int*)flag) < step) return;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < interior_count(L);
       t += (long long)gridDim.x * blockDim.x) {
    int i, j, k;
    node_of(L, t, i, j, k);
    const long long o = L.at(i, j, k);
    const double y = __ddiv_rn(delta2_at(P, codes, w, o, L.pitch, 1), h2);
    const double z = __ddiv_rn(delta2_at(P, codes, w, o, 1, 2), h2);
    double s;
    if (adi2) {
      const double x = __ddiv_rn(delta2_at(P, codes, w, o, L.s0, 0), h2);
      s = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(0.5, x), y), z), rho[o]);
    } else {
      s = __dadd_rn(__dadd_rn(y, z), rho[o]);
    }
    rhs[o] = __dadd_rn(w[o], __dmul_rn(dta, s));
    sy[o] = y;
    sz[o] = z;
  }
}

// r = u - coef * s on the interior.
__global__ void k_adi_sub(const Layout L, const double* __restrict__ u,
                          const double* __restrict__ s, double coef, double* __restrict__ r,
                          int* flag, int step) {
  if (flag && *((volatile int*)flag) < step) return;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < interior_count(L);
       t += (long long)gridDim.x * blockDim.x) {
    int i, j, k;
    node_of(L, t, i, j, k);
    const long long o = L.at(i, j, k);
    r[o] = __dsub_rn(u[o], __dmul_rn(coef, s[o]));
  }
}

int march_extra(const pbg_march_desc* d, int32_t* steps_taken, int32_t* diverged_step,
                int32_t* result_slot, float* device_ms, cudaStream_t st) {
  const pbg_grid* g = &d->grid;
  const Layout L = make_layout(g);
  const int v = d->variant;
  const double dta = d->dt / d->alpha, h2 = g->h * g->h;
  const bool adi2 = v == PBG_ADI2;
  PalDev P;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 2; ++b) P.eps[a][b] = d->pal.eps[a][b];
  for (int b = 0; b < 2; ++b) {
    P.k2[b] = d->pal.kappa2[b];
    P.decay[b] = std::exp(-(adi2 ? 0.5 : 1.0) * P.k2[b] * dta);  // schemes.py:240-247
    P.sat[b] = 0.0;
  }
  const size_t bytes = ((size_t)L.n0 * L.s0 + 64) * sizeof(double);
  const int nb = 148 * 8, nt = 256;
  const int check = d->check_divergence ? 1 : 0;
  const double thr = d->divergence_threshold;

  // scratch fields (faces = Dirichlet data): w, rhs, u, sy, sz
  double* tmp[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  const int ntmp = v == PBG_EULER ? 0 : 5;
  AxisAux aux[3];
  SweepArgs ax[3];
  int* dflag = nullptr;
  auto cleanup = [&]() {
    for (int q = 0; q < 5; ++q)
      if (tmp[q]) cudaFreeAsync(tmp[q], st);
    for (int q = 0; q < 3; ++q) release_axis(aux[q], st);
    if (dflag) cudaFreeAsync(dflag, st);
  };
  int rc = PBG_OK;
  auto cu = [&](cudaError_t e) {
    if (e != cudaSuccess) rc = fail(PBG_E_CUDA, cudaGetErrorString(e));
    return e == cudaSuccess;
  };
  bool ok = cu(cudaMallocAsync(&dflag, sizeof(int), st));
  const int init = INT_MAX;
  if (ok) ok = cu(cudaMemcpyAsync(dflag, &init, sizeof(int), cudaMemcpyHostToDevice, st));
  for (int q = 0; ok && q < ntmp; ++q)
    ok = cu(cudaMallocAsync(&tmp[q], bytes, st)) &&
         cu(cudaMemcpyAsync(tmp[q], d->work[0], bytes, cudaMemcpyDeviceToDevice, st));
  if (ok && v != PBG_EULER) {
    const double factor = adi2 ? 0.5 * dta : dta;
    for (int a = 0; ok && a < 3; ++a) {
      ax[a] = base_args(g, &d->pal, a, factor);
      ax[a].codes = d->codes;
      ax[a].rho = d->rho;
      ax[a].bnd = d->work[0];
      ax[a].thr = thr;
      rc = prepare_axis(ax[a], a, d->codes, aux[a], st);
      ok = rc == PBG_OK;
    }
  }
  if (ok && check) {
    k_faces_bad<<<148, 256, 0, st>>>(L, d->work[0], thr, dflag, 0, 0);
    ok = cu(cudaGetLastError());
  }
  int st_idx = -1;
  if (d->initial == d->work[0]) st_idx = 0;
  else if (d->initial == d->work[1]) st_idx = 1;
  const int st0 = st_idx;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  int* fl = check ? dflag : nullptr;
  for (int s = 1; ok && s <= d->nsteps; ++s) {
    const double* X = st_idx < 0 ? d->initial : d->work[st_idx];
    const int other = st_idx < 0 ? 0 : 1 - st_idx;
    double* A = d->work[other];
    if (v == PBG_EULER) {
      k_euler<<<nb, nt, 0, st>>>(L, P, d->codes, X, d->rho, dta, h2, A, fl, s, thr, check);
      ok = cu(cudaGetLastError());
    } else {
      double *W = tmp[0], *R = tmp[1], *U = tmp[2], *SY = tmp[3], *SZ = tmp[4];
      const double sub = adi2 ? 0.5 * dta : dta;
      k_flow_field<<<nb, nt, 0, st>>>(L, P, d->codes, X, W, fl, s, thr, 0);
      k_adi_rhs<<<nb, nt, 0, st>>>(L, P, d->codes, W, d->rho, dta, h2, adi2 ? 1 : 0, R, SY, SZ,
                                   fl, s);
      ok = cu(cudaGetLastError());
      for (int a = 0; ok && a < 3; ++a) {
        SweepArgs sa = ax[a];
        sa.step = s;
        sa.div_step = fl;
        sa.src = R;
        sa.dst = (a == 2 && !adi2) ? A : U;
        sa.check = (a == 2 && !adi2) ? check : 0;
        rc = launch_sweep(sa, a, st);
        ok = rc == PBG_OK;
        if (ok && a < 2) {
          k_adi_sub<<<nb, nt, 0, st>>>(L, U, a == 0 ? SY : SZ, sub, R, fl, s);
          ok = cu(cudaGetLastError());
        }
      }
      if (ok && adi2) {
        k_flow_field<<<nb, nt, 0, st>>>(L, P, d->codes, U, A, fl, s, thr, check);
        ok = cu(cudaGetLastError());
      }
    }
    st_idx = other;
  }
  cudaEventRecord(e1, st);
  int dstep = INT_MAX;
  if (ok) ok = cu(cudaMemcpyAsync(&dstep, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
  cleanup();
  if (ok) ok = cu(cudaStreamSynchronize(st));
  float ms = 0.f;
  if (ok) cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (!ok) return rc != PBG_OK ? rc : PBG_E_CUDA;
  int taken = d->nsteps;
  if (check && dstep != INT_MAX) taken = dstep;
  if (diverged_step) *diverged_step = (check && dstep != INT_MAX) ? dstep : 0;
  if (steps_taken) *steps_taken = taken;
  if (result_slot) *result_slot = st0 < 0 ? (taken - 1) % 2 : (st0 + taken) % 2;
  if (device_ms) *device_ms = ms;
  return PBG_OK;
}

}  // namespace pbg
