// Microbenchmark: stage [rows x W bytes] tiles at a large row stride through shared memory
// (cp.async) and write them back -- the access pattern of the axis-0 / axis-1 sweeps.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void cp16(void* s, const void* g) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g));
}
template <int W>  // doubles per row chunk
__global__ void k_tiles(const double* src, double* dst, int rows, long long stride, int ncol_groups, long long outer_stride) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, NT = blockDim.x;
  const long long base = (long long)blockIdx.y * outer_stride + (long long)blockIdx.x * W;
  const int cpr = W / 2;
  for (int c = tid; c < rows * cpr; c += NT) {
    int p = c / cpr, q = (c % cpr) * 2;
    cp16(sm + p * W + q, src + base + p * stride + q);
  }
  asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();
  for (int c = tid; c < rows * cpr; c += NT) {
    int p = c / cpr, q = (c % cpr) * 2;
    *(double2*)(dst + base + p * stride + q) = *(double2*)(sm + p * W + q);
  }
}
template <int W>
void run(double* a, double* b, int n, long long pitch, bool axis0) {
  long long s0 = (long long)n * pitch;
  long long stride = axis0 ? s0 : pitch;
  long long outer = axis0 ? pitch : s0;
  dim3 grid(512 / W, n);
  size_t smem = (size_t)n * W * 8;
  cudaFuncSetAttribute(k_tiles<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nt = 256;
  for (int w = 0; w < 2; ++w) k_tiles<W><<<grid, nt, smem>>>(a, b, n, stride, 512 / W, outer);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k_tiles<W><<<grid, nt, smem>>>(a, b, n, stride, 512 / W, outer);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
  double bytes = 2.0 * n * (double)n * 512 * 8;
  printf("axis%d W=%3d doubles (%4d B/row) smem %6zu: %.1f us  %.0f GB/s  %s\n", axis0 ? 0 : 1, W, W * 8, smem, ms * 1e3, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  int n = 513; long long pitch = 544;
  size_t bytes = (size_t)n * n * pitch * 8 + 4096;
  double *a, *b; cudaMalloc(&a, bytes); cudaMalloc(&b, bytes);
  cudaMemset(a, 0, bytes); cudaMemset(b, 0, bytes);
  for (int ax = 0; ax < 2; ++ax) {
    run<8>(a, b, n, pitch, ax == 0);
    run<16>(a, b, n, pitch, ax == 0);
    run<32>(a, b, n, pitch, ax == 0);

  }
  return 0;
}
