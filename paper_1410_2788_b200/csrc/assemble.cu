// Coefficient assembly on the device (north_star item 1).
//
//   classify_spheres  UnionOfSpheres.solute_mask over the node mesh and the three half-edge
//                     meshes (geometry.py:78-85, 117-156), per-atom bounding-box scatter with
//                     the reference's exact coordinate and distance arithmetic (bit-exact).
//   classify_sphere   AnalyticSphere (geometry.py:58-60).
//   deposit           deposit_charges (grid.py:205-252): trilinear weights, snap rule,
//                     interior check; node sums in the reference's np.add.at order
//                     (corner-major, atom-minor) via a stable radix sort -> bit-exact and
//                     deterministic.
//   coulomb_faces     coulomb_screened_values on the six faces (problem.py:44-61, 106-117).

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

#include "pbg_internal.cuh"

namespace pbg {

__device__ __forceinline__ double node_coord(double lo, double h, int i) {
  return __dadd_rn(lo, __dmul_rn(h, (double)i));  // grid.py:39-41
}

__device__ __forceinline__ double half_coord(double lo, double h, int i) {
  return __dadd_rn(node_coord(lo, h, i), __dmul_rn(0.5, h));  // geometry.py:117-119
}

__device__ __forceinline__ void or_code(uint8_t* codes, long long off, uint32_t bits) {
  const uintptr_t addr = reinterpret_cast<uintptr_t>(codes + off);
  unsigned int* word = reinterpret_cast<unsigned int*>(addr & ~(uintptr_t)3);
  atomicOr(word, bits << (8 * (addr & 3)));
}

// One block per atom.  mesh 0: nodes (bit 0); mesh 1+a: half-edges along axis a, the edge
// between node p and p+1 sets bit (1+a) of node p+1.
__global__ void k_classify_spheres(const Layout L, double lo0, double lo1, double lo2, double h,
                                   const double* __restrict__ atoms, double probe,
                                   uint8_t* codes) {
  const double* at = atoms + 5 * blockIdx.x;
  const double c[3] = {at[0], at[1], at[2]};
  const double rr = __dadd_rn(at[4], probe);
  const double rr2 = __dmul_rn(rr, rr);
  const double lo[3] = {lo0, lo1, lo2};
  const int n[3] = {L.n0, L.n1, L.n2};
  int b0[3], b1[3];
  for (int d = 0; d < 3; ++d) {
    b0[d] = max(0, (int)floor((c[d] - rr - lo[d]) / h) - 2);
    b1[d] = min(n[d] - 1, (int)ceil((c[d] + rr - lo[d]) / h) + 2);
  }
  const int e0 = b1[0] - b0[0] + 1, e1 = b1[1] - b0[1] + 1, e2 = b1[2] - b0[2] + 1;
  const long long vol = (long long)e0 * e1 * e2;
  for (int mesh = 0; mesh < 4; ++mesh) {
    const int ha = mesh - 1;  // half axis, -1 for nodes
    for (long long t = threadIdx.x; t < vol; t += blockDim.x) {
      int idx[3];
      idx[2] = b0[2] + (int)(t % e2);
      idx[1] = b0[1] + (int)((t / e2) % e1);
      idx[0] = b0[0] + (int)(t / ((long long)e1 * e2));
      if (ha >= 0 && idx[ha] > n[ha] - 2) continue;
      double d2 = 0.0;
      for (int d = 0; d < 3; ++d) {
        const double p = (d == ha) ? half_coord(lo[d], h, idx[d]) : node_coord(lo[d], h, idx[d]);
        const double dx = __dsub_rn(p, c[d]);
        d2 = d == 0 ? __dmul_rn(dx, dx) : __dadd_rn(d2, __dmul_rn(dx, dx));
      }
      if (d2 <= rr2) {
        if (ha >= 0) idx[ha] += 1;
        or_code(codes, L.at(idx[0], idx[1], idx[2]), ha < 0 ? 1u : (2u << ha));
      }
    }
  }
}

__global__ void k_classify_sphere(const Layout L, double lo0, double lo1, double lo2, double h,
                                  double R2, uint8_t* codes) {
  const long long total = (long long)L.n0 * L.n1 * L.n2;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t % L.n2);
    const int j = (int)((t / L.n2) % L.n1);
    const int i = (int)(t / ((long long)L.n1 * L.n2));
    const int idx[3] = {i, j, k};
    const double lo[3] = {lo0, lo1, lo2};
    uint32_t c = 0;
    for (int mesh = 0; mesh < 4; ++mesh) {
      const int ha = mesh - 1;
      if (ha >= 0 && idx[ha] == 0) continue;  // node p carries the edge (p-1, p)
      double r2 = 0.0;
      for (int d = 0; d < 3; ++d) {
        const double p =
            (d == ha) ? half_coord(lo[d], h, idx[d] - 1) : node_coord(lo[d], h, idx[d]);
        r2 = d == 0 ? __dmul_rn(p, p) : __dadd_rn(r2, __dmul_rn(p, p));
      }
      if (r2 <= R2) c |= ha < 0 ? 1u : (2u << ha);
    }
    codes[L.at(i, j, k)] = (uint8_t)(codes[L.at(i, j, k)] | c);
  }
}

// Per atom: cell, fractional offsets and the snap rule (grid.py:226-236).
__device__ __forceinline__ void atom_cell(const double* at, const double lo[3], double h,
                                          int cell[3], double fr[3]) {
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
}

// Contribution e = corner*N + atom (the np.add.at order of grid.py:247-249).
__global__ void k_deposit_contrib(const Layout L, double lo0, double lo1, double lo2, double h,
                                  const double* __restrict__ atoms, int natoms,
                                  long long* __restrict__ keys, int* __restrict__ vals,
                                  double* __restrict__ contrib, int* __restrict__ bad) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= natoms) return;
  const double* at = atoms + 5 * a;
  const double lo[3] = {lo0, lo1, lo2};
  const int n[3] = {L.n0, L.n1, L.n2};
  int cell[3];
  double fr[3];
  atom_cell(at, lo, h, cell, fr);
  bool isbad = false;
  for (int d = 0; d < 3; ++d) {
    const bool low = cell[d] < 1;
    const bool high = (cell[d] > n[d] - 3) && !((cell[d] == n[d] - 2) && (fr[d] == 0.0));
    isbad |= low || high;
  }
  if (isbad) {
    atomicMin(bad, a);
    for (int c = 0; c < 8; ++c) {
      keys[(long long)c * natoms + a] = LLONG_MAX;
      vals[(long long)c * natoms + a] = c * natoms + a;
      contrib[(long long)c * natoms + a] = 0.0;
    }
    return;
  }
  const double q = at[3];
  int c = 0;
  for (int di = 0; di < 2; ++di) {
    const double wx = di ? fr[0] : 1.0 - fr[0];
    for (int dj = 0; dj < 2; ++dj) {
      const double wy = dj ? fr[1] : 1.0 - fr[1];
      for (int dk = 0; dk < 2; ++dk, ++c) {
        const double wz = dk ? fr[2] : 1.0 - fr[2];
        const double w = __dmul_rn(__dmul_rn(wx, wy), wz);
        const long long e = (long long)c * natoms + a;
        const long long node =
            ((long long)(cell[0] + di) * L.n1 + (cell[1] + dj)) * L.n2 + (cell[2] + dk);
        keys[e] = (w == 0.0) ? LLONG_MAX : node;
        vals[e] = (int)e;
        contrib[e] = __dmul_rn(q, w);
      }
    }
  }
}

__global__ void k_deposit_sum(const Layout L, long long ne, const long long* __restrict__ keys,
                              const int* __restrict__ order, const double* __restrict__ contrib,
                              double factor, double* __restrict__ qfrac,
                              double* __restrict__ rho, uint8_t* __restrict__ codes) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= ne) return;
  const long long key = keys[p];
  if (key == LLONG_MAX) return;
  if (p > 0 && keys[p - 1] == key) return;  // not a segment head
  double s = 0.0;
  for (long long q = p; q < ne && keys[q] == key; ++q) s = __dadd_rn(s, contrib[order[q]]);
  const int k = (int)(key % L.n2);
  const long long o = (key / L.n2) * L.pitch + k + kOff;
  qfrac[o] = s;
  const double r = __dmul_rn(factor, s);
  rho[o] = r;
  if (codes && r != 0.0) codes[o] = (uint8_t)(codes[o] | 16u);
}

// Screened Coulomb sum at each face node; atoms staged through shared memory in order.
__global__ void k_coulomb_faces(const Layout L, double lo0, double lo1, double lo2, double h,
                                const double* __restrict__ atoms, int natoms, double damp,
                                double scale, double* __restrict__ dst, int* __restrict__ bad) {
  __shared__ double sa[256 * 4];
  const long long total = 2 * ((long long)L.n1 * L.n2 + (long long)L.n0 * L.n2 +
                               (long long)L.n0 * L.n1);
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int i = 0, j = 0, k = 0;
  const bool live = t < total;
  if (live) {
    long long u = t;
    const long long n12 = (long long)L.n1 * L.n2, n02 = (long long)L.n0 * L.n2,
                    n01 = (long long)L.n0 * L.n1;
    if (u < 2 * n12) {
      i = u < n12 ? 0 : L.n0 - 1;
      u %= n12;
      j = (int)(u / L.n2);
      k = (int)(u % L.n2);
    } else if ((u -= 2 * n12) < 2 * n02) {
      j = u < n02 ? 0 : L.n1 - 1;
      u %= n02;
      i = (int)(u / L.n2);
      k = (int)(u % L.n2);
    } else {
      u -= 2 * n02;
      k = u < n01 ? 0 : L.n2 - 1;
      u %= n01;
      i = (int)(u / L.n1);
      j = (int)(u % L.n1);
    }
  }
  const double px = __dadd_rn(lo0, __dmul_rn(h, (double)i));
  const double py = __dadd_rn(lo1, __dmul_rn(h, (double)j));
  const double pz = __dadd_rn(lo2, __dmul_rn(h, (double)k));
  double total_v = 0.0;
  bool hit = false;
  for (int base = 0; base < natoms; base += 256) {
    const int cnt = min(256, natoms - base);
    __syncthreads();
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
      const double* at = atoms + 5 * (base + q);
      sa[4 * q + 0] = at[0];
      sa[4 * q + 1] = at[1];
      sa[4 * q + 2] = at[2];
      sa[4 * q + 3] = at[3];
    }
    __syncthreads();
    if (live) {
      for (int q = 0; q < cnt; ++q) {
        const double dx = __dsub_rn(px, sa[4 * q + 0]);
        const double dy = __dsub_rn(py, sa[4 * q + 1]);
        const double dz = __dsub_rn(pz, sa[4 * q + 2]);
        const double d2 =
            __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
        const double d = __dsqrt_rn(d2);
        hit |= (d == 0.0);
        total_v = __dadd_rn(total_v,
                            __dmul_rn(__ddiv_rn(sa[4 * q + 3], d), exp(__dmul_rn(-damp, d))));
      }
    }
  }
  if (live) {
    if (hit) atomicExch(bad, 1);
    dst[L.at(i, j, k)] = __dmul_rn(scale, total_v);
  }
}

}  // namespace pbg

using namespace pbg;

extern "C" PBG_API int pbg_classify_spheres(const pbg_grid* g, const double* atoms,
                                            int32_t natoms, double probe, double eps_m,
                                            double eps_s, double kappa2_solvent,
                                            int32_t zero_first, uint8_t* codes,
                                            pbg_palette* palette, void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  if (!(eps_m > 0) || !(eps_s > 0)) return fail(PBG_E_INVALID, "dielectric constants must be positive");
  if (kappa2_solvent < 0) return fail(PBG_E_INVALID, "kappa2_solvent must be >= 0");
  if (probe < 0) return fail(PBG_E_INVALID, "probe_inflation must be >= 0");
  cudaStream_t st = (cudaStream_t)stream;
  Layout L = make_layout(g);
  if (zero_first) PBG_CUDA(cudaMemsetAsync(codes, 0, (size_t)L.n0 * L.n1 * L.pitch, st));
  if (natoms > 0) {
    k_classify_spheres<<<natoms, 256, 0, st>>>(L, g->lo[0], g->lo[1], g->lo[2], g->h, atoms,
                                               probe, codes);
    PBG_LAUNCH_CHECK("k_classify_spheres");
  }
  if (palette) {
    for (int a = 0; a < 3; ++a) {
      palette->eps[a][0] = eps_s;
      palette->eps[a][1] = eps_m;
    }
    palette->kappa2[0] = (eps_s == eps_m) ? 0.0 : kappa2_solvent;  // geometry.py:148
    palette->kappa2[1] = 0.0;
  }
  return PBG_OK;
}

extern "C" PBG_API int pbg_classify_sphere(const pbg_grid* g, double R, double eps_m,
                                           double eps_s, double kappa2_solvent, uint8_t* codes,
                                           pbg_palette* palette, void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  if (!(R > 0)) return fail(PBG_E_INVALID, "sphere radius must be positive");
  if (!(eps_m > 0) || !(eps_s > 0)) return fail(PBG_E_INVALID, "dielectric constants must be positive");
  if (kappa2_solvent < 0) return fail(PBG_E_INVALID, "kappa2_solvent must be >= 0");
  cudaStream_t st = (cudaStream_t)stream;
  Layout L = make_layout(g);
  PBG_CUDA(cudaMemsetAsync(codes, 0, (size_t)L.n0 * L.n1 * L.pitch, st));
  const long long total = (long long)L.n0 * L.n1 * L.n2;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
  k_classify_sphere<<<blocks, 256, 0, st>>>(L, g->lo[0], g->lo[1], g->lo[2], g->h, R * R,
                                            codes);
  PBG_LAUNCH_CHECK("k_classify_sphere");
  if (palette) {
    for (int a = 0; a < 3; ++a) {
      palette->eps[a][0] = eps_s;
      palette->eps[a][1] = eps_m;
    }
    palette->kappa2[0] = (eps_s == eps_m) ? 0.0 : kappa2_solvent;
    palette->kappa2[1] = 0.0;
  }
  return PBG_OK;
}

extern "C" PBG_API int pbg_deposit(const pbg_grid* g, const double* atoms, int32_t natoms,
                                   double prefactor, double* qfrac, double* rho,
                                   uint8_t* codes, void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  if (natoms < 1) return fail(PBG_E_INVALID, "system has no atoms");
  cudaStream_t st = (cudaStream_t)stream;
  Layout L = make_layout(g);
  const size_t nel = (size_t)L.n0 * L.n1 * L.pitch;
  PBG_CUDA(cudaMemsetAsync(qfrac, 0, nel * sizeof(double), st));
  PBG_CUDA(cudaMemsetAsync(rho, 0, nel * sizeof(double), st));
  const long long ne = 8LL * natoms;
  long long *keys = nullptr, *keys2 = nullptr;
  int *vals = nullptr, *vals2 = nullptr, *bad = nullptr;
  double* contrib = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, vals, vals2, (int)ne, 0, 64,
                                  st);
  PBG_CUDA(cudaMallocAsync(&keys, ne * sizeof(long long), st));
  PBG_CUDA(cudaMallocAsync(&keys2, ne * sizeof(long long), st));
  PBG_CUDA(cudaMallocAsync(&vals, ne * sizeof(int), st));
  PBG_CUDA(cudaMallocAsync(&vals2, ne * sizeof(int), st));
  PBG_CUDA(cudaMallocAsync(&contrib, ne * sizeof(double), st));
  PBG_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
  PBG_CUDA(cudaMallocAsync(&tmp, tmp_bytes + 16, st));
  const int big = INT_MAX;
  PBG_CUDA(cudaMemcpyAsync(bad, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  k_deposit_contrib<<<(natoms + 127) / 128, 128, 0, st>>>(L, g->lo[0], g->lo[1], g->lo[2],
                                                          g->h, atoms, natoms, keys, vals,
                                                          contrib, bad);
  PBG_LAUNCH_CHECK("k_deposit_contrib");
  cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, vals, vals2, (int)ne, 0, 64, st);
  PBG_LAUNCH_CHECK("cub::DeviceRadixSort");
  const double factor = prefactor / std::pow(g->h, 3.0);  // grid.py:251
  k_deposit_sum<<<(int)((ne + 255) / 256), 256, 0, st>>>(L, ne, keys2, vals2, contrib, factor,
                                                         qfrac, rho, codes);
  PBG_LAUNCH_CHECK("k_deposit_sum");
  int badh = INT_MAX;
  PBG_CUDA(cudaMemcpyAsync(&badh, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  cudaFreeAsync(keys, st);
  cudaFreeAsync(keys2, st);
  cudaFreeAsync(vals, st);
  cudaFreeAsync(vals2, st);
  cudaFreeAsync(contrib, st);
  cudaFreeAsync(bad, st);
  cudaFreeAsync(tmp, st);
  PBG_CUDA(cudaStreamSynchronize(st));
  if (badh != INT_MAX) {
    char buf[160];
    snprintf(buf, sizeof(buf), "atom %d is not strictly inside the grid interior", badh);
    return fail(PBG_E_INVALID, buf);
  }
  return PBG_OK;
}

extern "C" PBG_API int pbg_coulomb_faces(const pbg_grid* g, const double* atoms,
                                         int32_t natoms, double eps_s, double kappa_bar,
                                         double* dst, void* stream) {
  int rc = validate_grid(g);
  if (rc) return rc;
  if (!(eps_s > 0)) return fail(PBG_E_INVALID, "eps_s must be positive");
  cudaStream_t st = (cudaStream_t)stream;
  Layout L = make_layout(g);
  const long long total = 2 * ((long long)L.n1 * L.n2 + (long long)L.n0 * L.n2 +
                               (long long)L.n0 * L.n1);
  int* bad = nullptr;
  PBG_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
  PBG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
  const double c_es = 332.0636 / 0.592183;  // constants.py:12-17
  const double damp = kappa_bar / std::sqrt(eps_s);
  const double scale = c_es / eps_s;
  k_coulomb_faces<<<(int)((total + 255) / 256), 256, 0, st>>>(
      L, g->lo[0], g->lo[1], g->lo[2], g->h, atoms, natoms, damp, scale, dst, bad);
  PBG_LAUNCH_CHECK("k_coulomb_faces");
  int badh = 0;
  PBG_CUDA(cudaMemcpyAsync(&badh, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  cudaFreeAsync(bad, st);
  PBG_CUDA(cudaStreamSynchronize(st));
  if (badh) return fail(PBG_E_INVALID, "boundary point coincides with an atom center");
  return PBG_OK;
}
