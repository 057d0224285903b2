// Direct vacuum Poisson solver: -eps_m * d2(phi) = rho with Dirichlet faces
// (pbsplit/energy.py:59-85, vacuum_potential_fast).
//
// Boundary lifting (the face values enter the right-hand side of the nodes next to the
// faces), type-I discrete sine transform along each axis, division by the 7-point
// eigenvalues lambda = (eps/h^2) * sum_d 4 sin^2(pi m_d / (2 (n_d - 1))), inverse DST.
// Each 1-D DST-I of length N is a real FFT of length M = 2(N + 1) of the odd extension
// (0, x, 0, -reverse(x)): y_k = -Im F_{k+1} (scipy's unnormalised type-I), and the inverse
// divides by M.  FFTs are cuFFT D2Z plans; the odd extension is packed line-interleaved
// (transform index slowest, line fastest) for the axes whose lines are strided in the
// interior array, so packing and unpacking stay coalesced.

#include <cufft.h>

#include <cmath>
#include <vector>

#include "pbg_internal.cuh"

namespace pbg {

// Interior array A: (N0, N1, N2), k fastest.
struct Dims {
  int n[3];
  __host__ __device__ long long count() const { return (long long)n[0] * n[1] * n[2]; }
};

// rhs = rho + (eps/h^2) * lap(g), g = the Dirichlet faces with a zero interior; the
// neighbour sum follows energy.py:46-56 (x+, x-, y+, y-, z+, z-).
__global__ void k_vac_rhs(const Layout L, Dims D, const double* __restrict__ rho,
                          const double* __restrict__ bnd, double c, double* __restrict__ A) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < D.count();
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t % D.n[2]) + 1;
    const long long r = t / D.n[2];
    const int j = (int)(r % D.n[1]) + 1;
    const int i = (int)(r / D.n[1]) + 1;
    auto g = [&](int a, int b, int cc) {
      const bool face = a == 0 || a == L.n0 - 1 || b == 0 || b == L.n1 - 1 || cc == 0 ||
                        cc == L.n2 - 1;
      return face ? bnd[L.at(a, b, cc)] : 0.0;
    };
    double lap = -0.0;
    lap = __dadd_rn(lap, g(i + 1, j, k));
    lap = __dadd_rn(lap, g(i - 1, j, k));
    lap = __dadd_rn(lap, g(i, j + 1, k));
    lap = __dadd_rn(lap, g(i, j - 1, k));
    lap = __dadd_rn(lap, g(i, j, k + 1));
    lap = __dadd_rn(lap, g(i, j, k - 1));
    A[t] = __dadd_rn(rho[L.at(i, j, k)], __dmul_rn(c, lap));
  }
}

// Element (line, p) of the lines along `axis` inside A (line enumerates the other two axes
// in A order, the faster one fastest).
__device__ __forceinline__ long long line_elem(const Dims& D, int axis, long long line,
                                               int p) {
  if (axis == 2) return line * D.n[2] + p;
  if (axis == 1) {
    const long long i = line / D.n[2], k = line % D.n[2];
    return (i * D.n[1] + p) * D.n[2] + k;
  }
  return (long long)p * D.n[1] * D.n[2] + line;
}

// Odd extension of every line into v.  interleaved: v[n * nlines + line]; else
// v[line * M + n].
__global__ void k_vac_pack(Dims D, int axis, const double* __restrict__ A,
                           double* __restrict__ v, int interleaved) {
  const int N = D.n[axis], M = 2 * (N + 1);
  const long long nlines = D.count() / N;
  const long long total = nlines * M;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long line;
    int n;
    if (interleaved) {
      n = (int)(t / nlines);
      line = t % nlines;
    } else {
      line = t / M;
      n = (int)(t % M);
    }
    double x = 0.0;
    if (n >= 1 && n <= N) x = A[line_elem(D, axis, line, n - 1)];
    else if (n >= N + 2) x = -A[line_elem(D, axis, line, M - n - 1)];
    v[t] = x;
  }
}

// y_k = -Im F_{k+1} * scale back into A.
__global__ void k_vac_unpack(Dims D, int axis, const cufftDoubleComplex* __restrict__ F,
                             double* __restrict__ A, double scale, int interleaved) {
  const int N = D.n[axis], M = 2 * (N + 1), H = M / 2 + 1;
  const long long nlines = D.count() / N;
  const long long total = nlines * N;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long line;
    int k;
    if (interleaved) {
      k = (int)(t / nlines);
      line = t % nlines;
    } else {
      line = t / N;
      k = (int)(t % N);
    }
    const long long f = interleaved ? (long long)(k + 1) * nlines + line : line * H + k + 1;
    const double y = -F[f].y;
    A[line_elem(D, axis, line, k)] = scale == 1.0 ? y : __dmul_rn(y, scale);
  }
}

__global__ void k_vac_divide(Dims D, const double* __restrict__ lam, double c,
                             double* __restrict__ A) {
  const double* l0 = lam;
  const double* l1 = lam + D.n[0];
  const double* l2 = l1 + D.n[1];
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < D.count();
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t % D.n[2]);
    const long long r = t / D.n[2];
    const int j = (int)(r % D.n[1]);
    const int i = (int)(r / D.n[1]);
    const double l = __dmul_rn(c, __dadd_rn(__dadd_rn(l0[i], l1[j]), l2[k]));
    A[t] = __ddiv_rn(A[t], l);
  }
}

__global__ void k_vac_store(const Layout L, Dims D, const double* __restrict__ A,
                            double* __restrict__ out) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < D.count();
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t % D.n[2]) + 1;
    const long long r = t / D.n[2];
    const int j = (int)(r % D.n[1]) + 1;
    const int i = (int)(r / D.n[1]) + 1;
    out[L.at(i, j, k)] = A[t];
  }
}

}  // namespace pbg

using namespace pbg;

extern "C" PBG_API int pbg_vacuum_dst(const pbg_grid* g, double eps_m, const double* rho,
                                      const double* bnd, double* out, void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  if (!rho || !bnd || !out) return fail(PBG_E_INVALID, "null pointer");
  if (!(eps_m > 0)) return fail(PBG_E_INVALID, "eps_m must be positive");
  cudaStream_t st = (cudaStream_t)stream;
  const Layout L = make_layout(g);
  Dims D{{g->n[0] - 2, g->n[1] - 2, g->n[2] - 2}};
  const double c = eps_m / (g->h * g->h);

  // per-axis eigenvalues 4 sin^2(pi m / (2(n-1))), m = 1..n-2 (host libm, like numpy)
  std::vector<double> lam;
  for (int a = 0; a < 3; ++a) {
    const int n = g->n[a];
    for (int m = 1; m <= n - 2; ++m) {
      const double s = std::sin(M_PI * m / (2.0 * (n - 1)));
      lam.push_back(4.0 * (s * s));
    }
  }
  size_t vmax = 0, fmax = 0;
  for (int a = 0; a < 3; ++a) {
    const long long nl = D.count() / D.n[a];
    const long long M = 2LL * (D.n[a] + 1);
    vmax = std::max(vmax, (size_t)(nl * M));
    fmax = std::max(fmax, (size_t)(nl * (M / 2 + 1)));
  }
  double *A = nullptr, *v = nullptr, *dlam = nullptr;
  cufftDoubleComplex* F = nullptr;
  cufftHandle plans[3] = {0, 0, 0};
  bool made[3] = {false, false, false};
  auto cleanup = [&]() {
    for (int a = 0; a < 3; ++a)
      if (made[a]) cufftDestroy(plans[a]);
    if (A) cudaFreeAsync(A, st);
    if (v) cudaFreeAsync(v, st);
    if (F) cudaFreeAsync(F, st);
    if (dlam) cudaFreeAsync(dlam, st);
  };
  auto cu = [&](cudaError_t e) {
    if (e == cudaSuccess) return true;
    fail(PBG_E_CUDA, cudaGetErrorString(e));
    return false;
  };
  bool ok = cu(cudaMallocAsync(&A, D.count() * sizeof(double), st)) &&
            cu(cudaMallocAsync(&v, vmax * sizeof(double), st)) &&
            cu(cudaMallocAsync(&F, fmax * sizeof(cufftDoubleComplex), st)) &&
            cu(cudaMallocAsync(&dlam, lam.size() * sizeof(double), st)) &&
            cu(cudaMemcpyAsync(dlam, lam.data(), lam.size() * sizeof(double),
                               cudaMemcpyHostToDevice, st));
  for (int a = 0; ok && a < 3; ++a) {
    int M = 2 * (D.n[a] + 1);
    const long long nl = D.count() / D.n[a];
    const int inter = a < 2;
    int inembed[1] = {M}, onembed[1] = {M / 2 + 1};
    cufftResult r = cufftPlanMany(&plans[a], 1, &M, inembed, inter ? (int)nl : 1,
                                  inter ? 1 : M, onembed, inter ? (int)nl : 1,
                                  inter ? 1 : M / 2 + 1, CUFFT_D2Z, (int)nl);
    if (r != CUFFT_SUCCESS) {
      fail(PBG_E_CUDA, "cufftPlanMany failed");
      ok = false;
      break;
    }
    made[a] = true;
    if (cufftSetStream(plans[a], st) != CUFFT_SUCCESS) {
      fail(PBG_E_CUDA, "cufftSetStream failed");
      ok = false;
    }
  }
  const int nb = 148 * 8, nt = 256;
  if (ok) {
    k_vac_rhs<<<nb, nt, 0, st>>>(L, D, rho, bnd, c, A);
    ok = cu(cudaGetLastError());
  }
  for (int pass = 0; ok && pass < 2; ++pass) {  // forward DST, divide, inverse DST
    for (int a = 0; ok && a < 3; ++a) {
      const int inter = a < 2;
      const double scale = pass == 0 ? 1.0 : 1.0 / (2.0 * (D.n[a] + 1));
      k_vac_pack<<<nb, nt, 0, st>>>(D, a, A, v, inter);
      ok = cu(cudaGetLastError());
      if (ok && cufftExecD2Z(plans[a], v, F) != CUFFT_SUCCESS) {
        fail(PBG_E_CUDA, "cufftExecD2Z failed");
        ok = false;
      }
      if (ok) {
        k_vac_unpack<<<nb, nt, 0, st>>>(D, a, F, A, scale, inter);
        ok = cu(cudaGetLastError());
      }
    }
    if (ok && pass == 0) {
      k_vac_divide<<<nb, nt, 0, st>>>(D, dlam, c, A);
      ok = cu(cudaGetLastError());
    }
  }
  if (ok)
    ok = cu(cudaMemcpyAsync(out, bnd, ((size_t)L.n0 * L.s0 + 64) * sizeof(double),
                            cudaMemcpyDeviceToDevice, st));
  if (ok) {
    k_vac_store<<<nb, nt, 0, st>>>(L, D, A, out);
    ok = cu(cudaGetLastError());
  }
  if (ok) ok = cu(cudaStreamSynchronize(st));  // plans and buffers die here
  cleanup();
  return ok ? PBG_OK : PBG_E_CUDA;
}
