#include <cstdio>
#include <cmath>
#include "pbg_internal.cuh"
__global__ void k(const double* w, int n, double d, double sat, double* a, double* b) {
  int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
  a[i] = pbg::sinh_flow(w[i], d, 1.0); b[i] = pbg::sinh_flow_fast(w[i], d, sat, 1.0);
}
int main() {
  const int n = 1 << 20; double *w, *a, *b; cudaMallocManaged(&w, n*8); cudaMallocManaged(&a, n*8); cudaMallocManaged(&b, n*8);
  for (int i = 0; i < n; ++i) { double t = (i + 0.5) / n; w[i] = (t - 0.5) * 90.0; if (i % 7 == 0) w[i] *= 1e-6; if (i % 11 == 0) w[i] *= 1e-12; }
  double ds[] = {0.99999, 0.9, 0.53, 0.1, 1e-3};
  for (double d : ds) {
    double sat = 2.0 * std::atanh(d);
    k<<<(n + 255) / 256, 256>>>(w, n, d, sat, a, b); cudaDeviceSynchronize();
    double maxabs = 0, maxrel = 0; for (int i = 0; i < n; ++i) { double e = fabs(a[i] - b[i]); maxabs = fmax(maxabs, e); if (fabs(a[i]) > 1e-3) maxrel = fmax(maxrel, e / fabs(a[i])); }
    printf("d=%g max abs diff %.3e  max rel diff (|out|>1e-3) %.3e\n", d, maxabs, maxrel);
  }
}
