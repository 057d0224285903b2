// C ABI plumbing: errors, layout, layout conversion, pointwise ops, reductions, host march.
//
// References: pbsplit/grid.py:128-152 (ScalarField fp64 C order), problem.py:63-69
// (BoundarySpec.apply), schemes.py:106-120 (nonlinear_step), energy.py:31-43, 99-106
// (solvation_energy, richardson).

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "pbg_internal.cuh"

namespace pbg {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return PBG_OK;
  std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
  return fail(PBG_E_CUDA, msg);
}

int validate_grid(const pbg_grid* g) {
  if (!g) return fail(PBG_E_INVALID, "null grid");
  for (int a = 0; a < 3; ++a)
    if (g->n[a] < 3) return fail(PBG_E_INVALID, "every axis needs at least 3 nodes");
  if (g->pitch < (int64_t)g->n[2] + kOff) return fail(PBG_E_INVALID, "pitch too small");
  if (g->pitch % 32)  // 256-byte aligned rows: the row sweeps' 16-byte and tensor copies
    return fail(PBG_E_INVALID, "pitch must be a multiple of 32 (use pbg_layout)");
  if (!(g->h > 0)) return fail(PBG_E_INVALID, "spacing must be positive");
  return PBG_OK;
}

// ---------------------------------------------------------------------------------------
__global__ void k_pitch_from_dense(const Layout L, const double* __restrict__ dense,
                                   double* __restrict__ pitched) {
  const long long total = (long long)L.n0 * L.n1 * L.n2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t % L.n2);
    const long long ij = t / L.n2;
    pitched[ij * L.pitch + k + kOff] = dense[t];
  }
}

__global__ void k_dense_from_pitched(const Layout L, const double* __restrict__ pitched,
                                     double* __restrict__ dense) {
  const long long total = (long long)L.n0 * L.n1 * L.n2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t % L.n2);
    const long long ij = t / L.n2;
    dense[t] = pitched[ij * L.pitch + k + kOff];
  }
}

// Face node enumeration: t in [0, 2*(n1*n2 + n0*n2 + n0*n1)) -> (i, j, k), in the packed
// face order x-lo, x-hi, y-lo, y-hi, z-lo, z-hi (each face row-major in its two axes).
__device__ __forceinline__ void face_node(const Layout& L, long long t, int& i, int& j,
                                          int& k) {
  const long long n12 = (long long)L.n1 * L.n2, n02 = (long long)L.n0 * L.n2,
                  n01 = (long long)L.n0 * L.n1;
  if (t < 2 * n12) {
    i = t < n12 ? 0 : L.n0 - 1;
    t %= n12;
    j = (int)(t / L.n2);
    k = (int)(t % L.n2);
  } else if ((t -= 2 * n12) < 2 * n02) {
    j = t < n02 ? 0 : L.n1 - 1;
    t %= n02;
    i = (int)(t / L.n2);
    k = (int)(t % L.n2);
  } else {
    t -= 2 * n02;
    k = t < n01 ? 0 : L.n2 - 1;
    t %= n01;
    i = (int)(t / L.n1);
    j = (int)(t % L.n1);
  }
}

__host__ __device__ inline long long face_count(const Layout& L) {
  return 2 * ((long long)L.n1 * L.n2 + (long long)L.n0 * L.n2 + (long long)L.n0 * L.n1);
}

__global__ void k_copy_faces(const Layout L, const double* __restrict__ src,
                             double* __restrict__ dst) {
  const long long total = face_count(L);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int i, j, k;
    face_node(L, t, i, j, k);
    const long long o = L.at(i, j, k);
    dst[o] = src[o];
  }
}

__global__ void k_unpack_faces(const Layout L, const double* __restrict__ packed,
                               double* __restrict__ dst0, double* __restrict__ dst1) {
  const long long total = face_count(L);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int i, j, k;
    face_node(L, t, i, j, k);
    const long long o = L.at(i, j, k);
    const double v = packed[t];
    dst0[o] = v;
    if (dst1) dst1[o] = v;
  }
}

// nonlinear_step on a dense array with per-element kappa2 (schemes.py:106-120).
__global__ void k_flow_dense(long long n, const double* __restrict__ w,
                             const double* __restrict__ k2, double coef, double pm,
                             double* __restrict__ out) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const double decay = exp(__dmul_rn(-coef, k2[t]));
    out[t] = sinh_flow(w[t], decay, pm);
  }
}

__global__ void k_axpby(const Layout L, double ca, const double* __restrict__ a, double cb,
                        const double* __restrict__ b, double* __restrict__ out) {
  const long long total = (long long)L.n0 * L.n1 * L.n2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t % L.n2);
    const long long o = (t / L.n2) * L.pitch + k + kOff;
    out[o] = __dadd_rn(__dmul_rn(ca, a[o]), __dmul_rn(cb, b[o]));
  }
}

// Deterministic two-level reductions: block b reduces the fixed index range
// [b*chunk, (b+1)*chunk) with a fixed tree; the host-side second pass sums partials in order.
constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 1184;  // 8 x 148 SMs

template <typename Op>
__device__ double block_reduce(double v, Op op) {
  __shared__ double sh[kRedThreads / 32];
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_down_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (l < kRedThreads / 32) ? sh[l] : op.identity();
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_down_sync(0xffffffffu, v, o));
  }
  return v;
}

struct SumOp {
  __device__ double operator()(double a, double b) const { return a + b; }
  __device__ double identity() const { return 0.0; }
};
struct MaxAbsOp {  // NaN-propagating max
  __device__ double operator()(double a, double b) const {
    return (a != a || b != b) ? (a + b) : fmax(a, b);
  }
  __device__ double identity() const { return 0.0; }
};

__global__ void k_energy_dense(const Layout L, const double* __restrict__ q,
                               const double* __restrict__ pm, const double* __restrict__ p0,
                               double* __restrict__ partial) {
  const long long total = (long long)L.n0 * L.n1 * L.n2;
  const long long chunk = (total + gridDim.x - 1) / gridDim.x;
  const long long beg = blockIdx.x * chunk, end = min(total, beg + chunk);
  double acc = 0.0;
  for (long long t = beg + threadIdx.x; t < end; t += blockDim.x) {
    const int k = (int)(t % L.n2);
    const long long o = (t / L.n2) * L.pitch + k + kOff;
    const double qv = q[o];
    if (qv != 0.0) acc += qv * (pm[o] - p0[o]);
  }
  acc = block_reduce(acc, SumOp());
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

__global__ void k_maxabs(const Layout L, const double* __restrict__ x,
                         double* __restrict__ partial) {
  const long long total = (long long)L.n0 * L.n1 * L.n2;
  const long long chunk = (total + gridDim.x - 1) / gridDim.x;
  const long long beg = blockIdx.x * chunk, end = min(total, beg + chunk);
  MaxAbsOp op;
  double acc = 0.0;
  for (long long t = beg + threadIdx.x; t < end; t += blockDim.x) {
    const int k = (int)(t % L.n2);
    const long long o = (t / L.n2) * L.pitch + k + kOff;
    acc = op(acc, fabs(x[o]));
  }
  acc = block_reduce(acc, op);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

// Energy by trilinear gather at the atoms: per atom the deposit cell/weights of
// grid.py:219-236 and trilinear_weights (grid.py:189-202), dphi fused with richardson.
__global__ void k_energy_atoms(const Layout L, double lo0, double lo1, double lo2, double h,
                               const double* __restrict__ atoms, int natoms,
                               const double* __restrict__ pma, const double* __restrict__ pmb,
                               double ca, double cb, const double* __restrict__ p0a,
                               const double* __restrict__ p0b, double cc, double cd,
                               double* __restrict__ out) {
  double acc = 0.0;
  for (int a = threadIdx.x; a < natoms; a += blockDim.x) {
    const double* at = atoms + 5 * a;
    const double lo[3] = {lo0, lo1, lo2};
    int cell[3];
    double fr[3];
    for (int d = 0; d < 3; ++d) {
      const double t = __ddiv_rn(__dsub_rn(at[d], lo[d]), h);
      double c = floor(t);
      double f = __dsub_rn(t, c);
      if (f >= 1.0 - 1e-12) {
        c += 1.0;
        f = 0.0;
      }
      cell[d] = (int)c;
      fr[d] = f;
    }
    double s = 0.0;
    for (int di = 0; di < 2; ++di) {
      const double wx = di ? fr[0] : 1.0 - fr[0];
      for (int dj = 0; dj < 2; ++dj) {
        const double wy = dj ? fr[1] : 1.0 - fr[1];
        for (int dk = 0; dk < 2; ++dk) {
          const double wz = dk ? fr[2] : 1.0 - fr[2];
          const double w = __dmul_rn(__dmul_rn(wx, wy), wz);
          if (w == 0.0) continue;
          const long long o = L.at(cell[0] + di, cell[1] + dj, cell[2] + dk);
          double phm = ca * pma[o];
          if (pmb) phm += cb * pmb[o];
          double ph0 = cc * p0a[o];
          if (p0b) ph0 += cd * p0b[o];
          s += __dmul_rn(at[3], w) * (phm - ph0);
        }
      }
    }
    acc += s;
  }
  acc = block_reduce(acc, SumOp());
  if (threadIdx.x == 0) out[0] = acc;
}

// Palette discovery for pack_region: slot[0] <- element 0 (by the host), slot[1] the second
// distinct value, flag set on a third value or a NaN.
__global__ void k_palette(long long n, const double* __restrict__ x,
                          unsigned long long* slots, int* flag) {
  const double p0 = x[0];
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    const double v = x[t];
    if (v != v) {
      *flag = 1;
      continue;
    }
    if (v == p0) continue;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    unsigned long long cur = slots[1];
    if (cur == ~0ull) cur = atomicCAS(&slots[1], ~0ull, bits);
    if (cur != ~0ull && __longlong_as_double((long long)cur) != v) *flag = 1;
  }
}

__global__ void k_pack(const Layout L, const double* __restrict__ ex,
                       const double* __restrict__ ey, const double* __restrict__ ez,
                       const double* __restrict__ k2, const double* __restrict__ rho,
                       double ex1, double ey1, double ez1, double k21, int hx, int hy, int hz,
                       int hk, uint8_t* __restrict__ codes) {
  const long long total = (long long)L.n0 * L.n1 * L.n2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t % L.n2);
    const int j = (int)((t / L.n2) % L.n1);
    const int i = (int)(t / ((long long)L.n1 * L.n2));
    uint32_t c = 0;
    if (hk && k2[t] == k21) c |= 1u;
    if (hx && i >= 1 && ex[((long long)(i - 1) * L.n1 + j) * L.n2 + k] == ex1) c |= 2u;
    if (hy && j >= 1 && ey[((long long)i * (L.n1 - 1) + (j - 1)) * L.n2 + k] == ey1) c |= 4u;
    if (hz && k >= 1 && ez[((long long)i * L.n1 + j) * (L.n2 - 1) + (k - 1)] == ez1) c |= 8u;
    if (rho && rho[t] != 0.0) c |= 16u;
    codes[L.at(i, j, k)] = (uint8_t)c;
  }
}

static int grid_blocks(long long n, int threads = 256) {
  long long b = (n + threads - 1) / threads;
  return (int)std::max(1LL, std::min(b, 148LL * 16));
}

static int discover_palette(const double* x, long long n, double out[2], bool& two,
                            cudaStream_t st, unsigned long long* slots, int* flag) {
  const unsigned long long init[2] = {0ull, ~0ull};
  PBG_CUDA(cudaMemcpyAsync(slots, init, sizeof(init), cudaMemcpyHostToDevice, st));
  PBG_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
  k_palette<<<grid_blocks(n), 256, 0, st>>>(n, x, slots, flag);
  PBG_LAUNCH_CHECK("k_palette");
  unsigned long long got[2];
  int f = 0;
  PBG_CUDA(cudaMemcpyAsync(&got[1], slots + 1, sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, st));
  PBG_CUDA(cudaMemcpyAsync(&got[0], x, sizeof(double), cudaMemcpyDeviceToHost, st));
  PBG_CUDA(cudaMemcpyAsync(&f, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  PBG_CUDA(cudaStreamSynchronize(st));
  if (f) return fail(PBG_E_UNSUPPORTED,
                     "coefficient map holds more than two distinct values (or NaN); the "
                     "device solver encodes at most two per map");
  double v0;
  memcpy(&v0, &got[0], sizeof(double));
  out[0] = v0;
  if (got[1] == ~0ull) {
    out[1] = v0;
    two = false;
  } else {
    double v1;
    memcpy(&v1, &got[1], sizeof(double));
    out[1] = v1;
    two = true;
  }
  return PBG_OK;
}

}  // namespace pbg

using namespace pbg;

extern "C" {

PBG_API const char* pbg_last_error(void) { return g_last_error.c_str(); }

PBG_API int pbg_version(void) { return 1; }

PBG_API int pbg_layout(int32_t n0, int32_t n1, int32_t n2, int64_t* pitch, int64_t* nelem) {
  if (n0 < 3 || n1 < 3 || n2 < 3) return fail(PBG_E_INVALID, "every axis needs >= 3 nodes");
  const int64_t p = ((int64_t)n2 + kOff + 31) / 32 * 32;
  if (pitch) *pitch = p;
  // +64 elements of slack: tile loads may read a few padding columns past the last row
  if (nelem) *nelem = (int64_t)n0 * n1 * p + 64;
  return PBG_OK;
}

PBG_API int pbg_pitch_from_dense(const pbg_grid* g, const double* dense, double* pitched,
                                 void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  Layout L = make_layout(g);
  k_pitch_from_dense<<<grid_blocks((long long)L.n0 * L.n1 * L.n2), 256, 0,
                       (cudaStream_t)stream>>>(L, dense, pitched);
  PBG_LAUNCH_CHECK("k_pitch_from_dense");
  return PBG_OK;
}

PBG_API int pbg_dense_from_pitched(const pbg_grid* g, const double* pitched, double* dense,
                                   void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  Layout L = make_layout(g);
  k_dense_from_pitched<<<grid_blocks((long long)L.n0 * L.n1 * L.n2), 256, 0,
                         (cudaStream_t)stream>>>(L, pitched, dense);
  PBG_LAUNCH_CHECK("k_dense_from_pitched");
  return PBG_OK;
}

PBG_API int pbg_copy_faces(const pbg_grid* g, const double* src, double* dst, void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  Layout L = make_layout(g);
  k_copy_faces<<<grid_blocks(face_count(L)), 256, 0, (cudaStream_t)stream>>>(L, src, dst);
  PBG_LAUNCH_CHECK("k_copy_faces");
  return PBG_OK;
}

PBG_API int pbg_unpack_faces(const pbg_grid* g, const double* packed, double* dst0,
                             double* dst1, void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  Layout L = make_layout(g);
  k_unpack_faces<<<grid_blocks(face_count(L)), 256, 0, (cudaStream_t)stream>>>(L, packed,
                                                                               dst0, dst1);
  PBG_LAUNCH_CHECK("k_unpack_faces");
  return PBG_OK;
}

PBG_API int pbg_flow_dense(int64_t n, const double* w, const double* kappa2, double coef,
                           double premultiplier, double* out, void* stream) {
  if (n <= 0) return PBG_OK;
  k_flow_dense<<<grid_blocks(n), 256, 0, (cudaStream_t)stream>>>(n, w, kappa2, coef,
                                                                  premultiplier, out);
  PBG_LAUNCH_CHECK("k_flow_dense");
  return PBG_OK;
}

PBG_API int pbg_axpby(const pbg_grid* g, double ca, const double* a, double cb,
                      const double* b, double* out, void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  Layout L = make_layout(g);
  k_axpby<<<grid_blocks((long long)L.n0 * L.n1 * L.n2), 256, 0, (cudaStream_t)stream>>>(
      L, ca, a, cb, b, out);
  PBG_LAUNCH_CHECK("k_axpby");
  return PBG_OK;
}

static int finish_partials(double* partial, int nb, bool is_max, double* result,
                           cudaStream_t st) {
  double host[kRedBlocks];
  PBG_CUDA(cudaMemcpyAsync(host, partial, sizeof(double) * nb, cudaMemcpyDeviceToHost, st));
  PBG_CUDA(cudaFreeAsync(partial, st));
  PBG_CUDA(cudaStreamSynchronize(st));
  double acc = 0.0;
  for (int b = 0; b < nb; ++b) {
    if (is_max) acc = (acc != acc || host[b] != host[b]) ? NAN : std::max(acc, host[b]);
    else acc += host[b];
  }
  *result = acc;
  return PBG_OK;
}

PBG_API int pbg_energy_dense(const pbg_grid* g, const double* qfrac, const double* phi_m,
                             const double* phi_0, double kcal, double* delta_g,
                             void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  Layout L = make_layout(g);
  double* partial = nullptr;
  PBG_CUDA(cudaMallocAsync(&partial, sizeof(double) * kRedBlocks, st));
  k_energy_dense<<<kRedBlocks, kRedThreads, 0, st>>>(L, qfrac, phi_m, phi_0, partial);
  PBG_LAUNCH_CHECK("k_energy_dense");
  double total = 0.0;
  rc = finish_partials(partial, kRedBlocks, false, &total, st);
  if (rc) return rc;
  *delta_g = 0.5 * total * kcal;
  return PBG_OK;
}

PBG_API int pbg_maxabs(const pbg_grid* g, const double* x, double* result, void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  Layout L = make_layout(g);
  double* partial = nullptr;
  PBG_CUDA(cudaMallocAsync(&partial, sizeof(double) * kRedBlocks, st));
  k_maxabs<<<kRedBlocks, kRedThreads, 0, st>>>(L, x, partial);
  PBG_LAUNCH_CHECK("k_maxabs");
  return finish_partials(partial, kRedBlocks, true, result, st);
}

PBG_API int pbg_energy_atoms(const pbg_grid* g, const double* atoms, int32_t natoms,
                             const double* phi_m_a, const double* phi_m_b, double ca,
                             double cb, const double* phi_0_a, const double* phi_0_b,
                             double cc, double cd, double kcal, double* delta_g,
                             void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  if (natoms < 1 || !atoms || !phi_m_a || !phi_0_a) return fail(PBG_E_INVALID, "bad args");
  cudaStream_t st = (cudaStream_t)stream;
  Layout L = make_layout(g);
  double* out = nullptr;
  PBG_CUDA(cudaMallocAsync(&out, sizeof(double), st));
  k_energy_atoms<<<1, kRedThreads, 0, st>>>(L, g->lo[0], g->lo[1], g->lo[2], g->h, atoms, natoms,
                                     phi_m_a, phi_m_b, ca, cb, phi_0_a, phi_0_b, cc, cd,
                                     out);
  PBG_LAUNCH_CHECK("k_energy_atoms");
  double total = 0.0;
  PBG_CUDA(cudaMemcpyAsync(&total, out, sizeof(double), cudaMemcpyDeviceToHost, st));
  PBG_CUDA(cudaFreeAsync(out, st));
  PBG_CUDA(cudaStreamSynchronize(st));
  *delta_g = 0.5 * total * kcal;
  return PBG_OK;
}

PBG_API int pbg_pack_region(const pbg_grid* g, const double* eps_half_x,
                            const double* eps_half_y, const double* eps_half_z,
                            const double* kappa2, const double* rho_dense, uint8_t* codes,
                            pbg_palette* palette, void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  if (!eps_half_x || !eps_half_y || !eps_half_z || !kappa2 || !codes || !palette)
    return fail(PBG_E_INVALID, "null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  Layout L = make_layout(g);
  const long long n0 = L.n0, n1 = L.n1, n2 = L.n2;
  unsigned long long* slots = nullptr;
  int* flag = nullptr;
  PBG_CUDA(cudaMallocAsync(&slots, 2 * sizeof(unsigned long long), st));
  PBG_CUDA(cudaMallocAsync(&flag, sizeof(int), st));
  const double* arrs[4] = {eps_half_x, eps_half_y, eps_half_z, kappa2};
  const long long sizes[4] = {(n0 - 1) * n1 * n2, n0 * (n1 - 1) * n2, n0 * n1 * (n2 - 1),
                              n0 * n1 * n2};
  double pal[4][2];
  bool two[4];
  for (int q = 0; q < 4; ++q) {
    rc = discover_palette(arrs[q], sizes[q], pal[q], two[q], st, slots, flag);
    if (rc) {
      cudaFreeAsync(slots, st);
      cudaFreeAsync(flag, st);
      return rc;
    }
  }
  PBG_CUDA(cudaFreeAsync(slots, st));
  PBG_CUDA(cudaFreeAsync(flag, st));
  PBG_CUDA(cudaMemsetAsync(codes, 0, (size_t)(n0 * n1 * L.pitch), st));
  k_pack<<<grid_blocks(n0 * n1 * n2), 256, 0, st>>>(
      L, eps_half_x, eps_half_y, eps_half_z, kappa2, rho_dense, pal[0][1], pal[1][1],
      pal[2][1], pal[3][1], two[0], two[1], two[2], two[3], codes);
  PBG_LAUNCH_CHECK("k_pack");
  for (int a = 0; a < 3; ++a) {
    palette->eps[a][0] = pal[a][0];
    palette->eps[a][1] = pal[a][1];
  }
  palette->kappa2[0] = pal[3][0];
  palette->kappa2[1] = pal[3][1];
  return PBG_OK;
}

// March from HOST buffers (the reference-facing FFI call).
//   codes_pitched_host : uint8 in the pitched layout (pbg_layout nelem bytes)
//   rho_dense_host     : dense (n0,n1,n2) source, or NULL with rho_nnz/rho_idx/rho_val
//   faces_host         : packed faces (x-lo, x-hi, y-lo, y-hi, z-lo, z-hi)
//   initial_dense_host : dense initial field, or NULL = zero interior + boundary faces
//   final_dense_host   : receives the final dense field
PBG_API int pbg_march_host(const pbg_march_desc* t, const uint8_t* codes_pitched_host,
                            int64_t rho_nnz, const int64_t* rho_idx, const double* rho_val,
                            const double* faces_host, const double* initial_dense_host,
                            double* final_dense_host, int32_t* steps_taken,
                            int32_t* diverged_step, float* device_ms, void* stream);

}  // extern "C"

__global__ void k_scatter_sparse(const Layout L, long long nnz, const long long* __restrict__ idx,
                                 const double* __restrict__ val, double* __restrict__ dst) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nnz;
       t += (long long)gridDim.x * blockDim.x) {
    const long long f = idx[t];
    const int k = (int)(f % L.n2);
    dst[(f / L.n2) * L.pitch + k + kOff] = val[t];
  }
}

extern "C" PBG_API int pbg_march_host(const pbg_march_desc* t, const uint8_t* codes_h,
                                       int64_t rho_nnz, const int64_t* rho_idx,
                                       const double* rho_val, const double* faces_h,
                                       const double* init_h, double* final_h,
                                       int32_t* steps_taken, int32_t* diverged_step,
                                       float* device_ms, void* stream) {
  if (!t) return fail(PBG_E_INVALID, "null descriptor");
  int rc = validate_grid(&t->grid);
  if (rc) return rc;
  if (!codes_h || !faces_h || !final_h) return fail(PBG_E_INVALID, "null host buffer");
  cudaStream_t st = (cudaStream_t)stream;
  keep_pool_memory();
  Layout L = make_layout(&t->grid);
  const size_t nelem = (size_t)L.n0 * L.n1 * L.pitch + 64;  // pbg_layout's nelem
  const size_t nf = (size_t)face_count(L);
  uint8_t* codes = nullptr;
  double *rho = nullptr, *w0 = nullptr, *w1 = nullptr, *init = nullptr, *faces = nullptr;
  long long* idx = nullptr;
  double* val = nullptr;
  PBG_CUDA(cudaMallocAsync(&codes, nelem, st));
  PBG_CUDA(cudaMallocAsync(&rho, nelem * sizeof(double), st));
  PBG_CUDA(cudaMallocAsync(&w0, nelem * sizeof(double), st));
  PBG_CUDA(cudaMallocAsync(&w1, nelem * sizeof(double), st));
  PBG_CUDA(cudaMallocAsync(&faces, nf * sizeof(double), st));
  PBG_CUDA(cudaMemcpyAsync(codes, codes_h, nelem, cudaMemcpyHostToDevice, st));
  PBG_CUDA(cudaMemcpyAsync(faces, faces_h, nf * sizeof(double), cudaMemcpyHostToDevice, st));
  PBG_CUDA(cudaMemsetAsync(rho, 0, nelem * sizeof(double), st));
  if (rho_nnz > 0) {
    PBG_CUDA(cudaMallocAsync(&idx, rho_nnz * sizeof(long long), st));
    PBG_CUDA(cudaMallocAsync(&val, rho_nnz * sizeof(double), st));
    PBG_CUDA(cudaMemcpyAsync(idx, rho_idx, rho_nnz * sizeof(long long), cudaMemcpyHostToDevice,
                             st));
    PBG_CUDA(cudaMemcpyAsync(val, rho_val, rho_nnz * sizeof(double), cudaMemcpyHostToDevice,
                             st));
    k_scatter_sparse<<<grid_blocks(rho_nnz), 256, 0, st>>>(L, rho_nnz, idx, val, rho);
    PBG_LAUNCH_CHECK("k_scatter_sparse");
  }
  const size_t row = (size_t)L.n2 * sizeof(double);
  if (init_h) {
    PBG_CUDA(cudaMallocAsync(&init, nelem * sizeof(double), st));
    PBG_CUDA(cudaMemcpy2DAsync(init + kOff, L.pitch * sizeof(double), init_h, row, row,
                               (size_t)L.n0 * L.n1, cudaMemcpyHostToDevice, st));
  } else {
    PBG_CUDA(cudaMemsetAsync(w0, 0, nelem * sizeof(double), st));
  }
  k_unpack_faces<<<grid_blocks((long long)nf), 256, 0, st>>>(L, faces, w0, w1);
  PBG_LAUNCH_CHECK("k_unpack_faces");
  pbg_march_desc d = *t;
  d.codes = codes;
  d.rho = rho;
  d.work[0] = w0;
  d.work[1] = w1;
  d.initial = init_h ? init : w0;
  int32_t taken = 0, dstep = 0, slot = 0;
  float ms = 0.f;
  rc = pbg_march(&d, &taken, &dstep, &slot, &ms, stream);
  if (rc == PBG_OK) {
    const double* res = slot == 0 ? w0 : w1;
    rc = check_cuda(cudaMemcpy2DAsync(final_h, row, res + kOff, L.pitch * sizeof(double), row,
                                      (size_t)L.n0 * L.n1, cudaMemcpyDeviceToHost, st),
                    "download final");
  }
  cudaFreeAsync(codes, st);
  cudaFreeAsync(rho, st);
  cudaFreeAsync(w0, st);
  cudaFreeAsync(w1, st);
  cudaFreeAsync(faces, st);
  if (init) cudaFreeAsync(init, st);
  if (idx) cudaFreeAsync(idx, st);
  if (val) cudaFreeAsync(val, st);
  if (rc) return rc;
  PBG_CUDA(cudaStreamSynchronize(st));
  if (steps_taken) *steps_taken = taken;
  if (diverged_step) *diverged_step = dstep;
  if (device_ms) *device_ms = ms;
  return PBG_OK;
}

// codes -> dense RegionMap arrays (used when a device-assembled RegionMap is read on the host).
__global__ void k_expand_region(const Layout L, const uint8_t* __restrict__ codes, double en0,
                                double en1, double ex0, double ex1, double ey0, double ey1,
                                double ez0, double ez1, double k20, double k21,
                                double* __restrict__ eps_node, double* __restrict__ ex,
                                double* __restrict__ ey, double* __restrict__ ez,
                                double* __restrict__ k2) {
  const long long total = (long long)L.n0 * L.n1 * L.n2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t % L.n2);
    const int j = (int)((t / L.n2) % L.n1);
    const int i = (int)(t / ((long long)L.n1 * L.n2));
    const uint32_t c = codes[L.at(i, j, k)];
    if (eps_node) eps_node[t] = (c & 1u) ? en1 : en0;
    if (k2) k2[t] = (c & 1u) ? k21 : k20;
    if (ex && i >= 1) ex[((long long)(i - 1) * L.n1 + j) * L.n2 + k] = (c & 2u) ? ex1 : ex0;
    if (ey && j >= 1) ey[((long long)i * (L.n1 - 1) + (j - 1)) * L.n2 + k] = (c & 4u) ? ey1 : ey0;
    if (ez && k >= 1) ez[((long long)i * L.n1 + j) * (L.n2 - 1) + (k - 1)] = (c & 8u) ? ez1 : ez0;
  }
}

extern "C" PBG_API int pbg_expand_region(const pbg_grid* g, const uint8_t* codes,
                                         const pbg_palette* pal, const double eps_node_pal[2],
                                         double* eps_node, double* eps_half_x,
                                         double* eps_half_y, double* eps_half_z,
                                         double* kappa2, void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  if (!codes || !pal || !eps_node_pal) return fail(PBG_E_INVALID, "null pointer");
  Layout L = make_layout(g);
  k_expand_region<<<grid_blocks((long long)L.n0 * L.n1 * L.n2), 256, 0,
                    (cudaStream_t)stream>>>(
      L, codes, eps_node_pal[0], eps_node_pal[1], pal->eps[0][0], pal->eps[0][1],
      pal->eps[1][0], pal->eps[1][1], pal->eps[2][0], pal->eps[2][1], pal->kappa2[0],
      pal->kappa2[1], eps_node, eps_half_x, eps_half_y, eps_half_z, kappa2);
  PBG_LAUNCH_CHECK("k_expand_region");
  return PBG_OK;
}

__global__ void k_mark_charged(const Layout L, const double* __restrict__ rho,
                               uint8_t* __restrict__ codes) {
  const long long total = (long long)L.n0 * L.n1 * L.n2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t % L.n2);
    const long long o = (t / L.n2) * L.pitch + k + kOff;
    codes[o] = (uint8_t)((codes[o] & 15u) | (rho[o] != 0.0 ? 16u : 0u));
  }
}

extern "C" PBG_API int pbg_mark_charged(const pbg_grid* g, const double* rho_pitched,
                                        uint8_t* codes, void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  Layout L = make_layout(g);
  k_mark_charged<<<grid_blocks((long long)L.n0 * L.n1 * L.n2), 256, 0,
                   (cudaStream_t)stream>>>(L, rho_pitched, codes);
  PBG_LAUNCH_CHECK("k_mark_charged");
  return PBG_OK;
}
