// Microbenchmark: the column-tile staging pattern of the axis-0 / axis-1 sweeps (LB = 16
// adjacent doubles x 515 rows at a large row stride, staged through shared memory and written
// back), moved three ways:
//   (a) cp.async 16-byte chunks (LDGSTS) + STG.128 from shared memory (current sweeps);
//   (b) one cp.async.bulk (TMA, non-tensor) per 128-byte row chunk, mbarrier completion, and
//       cp.async.bulk shared->global stores;
//   (c) cp.async.bulk.tensor.3d boxes {16, 1, 256} (tensor map) both ways.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 bulk_tiles.cu -lcuda -o bulk_tiles
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

constexpr int LB = 16;

__device__ __forceinline__ unsigned smaddr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smaddr(b)), "r"(n));
  asm volatile("fence.mbarrier_init.release.cluster;" ::);
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smaddr(b)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}" ::"r"(smaddr(b)),
      "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* s, const void* g, unsigned bytes,
                                         unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smaddr(s)),
      "l"(g), "r"(bytes), "r"(smaddr(b))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* g, const void* s, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g),
               "r"(smaddr(s)), "r"(bytes)
               : "memory");
}

struct Geo {
  long long stride, outer;
  int rows;
};

__global__ void k_cpasync(const double* src, double* dst, Geo G) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, NT = blockDim.x;
  const long long base = (long long)blockIdx.y * G.outer + (long long)blockIdx.x * LB;
  for (int c = tid; c < G.rows * 8; c += NT) {
    const int p = c / 8, q = (c % 8) * 2;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smaddr(sm + p * LB + q)),
                 "l"(src + base + p * G.stride + q));
  }
  asm volatile("cp.async.wait_all;\n" ::);
  __syncthreads();
  for (int c = tid; c < G.rows * 8; c += NT) {
    const int p = c / 8, q = (c % 8) * 2;
    *(double2*)(dst + base + p * G.stride + q) = *(double2*)(sm + p * LB + q);
  }
}

__global__ void k_bulk(const double* src, double* dst, Geo G) {
  extern __shared__ double sm[];
  __shared__ unsigned long long mbar;
  const int tid = threadIdx.x, NT = blockDim.x;
  const long long base = (long long)blockIdx.y * G.outer + (long long)blockIdx.x * LB;
  if (tid == 0) mbar_init(&mbar, 1);
  __syncthreads();
  if (tid == 0) mbar_expect(&mbar, G.rows * LB * 8);
  for (int p = tid; p < G.rows; p += NT) bulk_g2s(sm + p * LB, src + base + p * G.stride, LB * 8, &mbar);
  mbar_wait(&mbar, 0);
  __syncthreads();
  for (int p = tid; p < G.rows; p += NT) bulk_s2g(dst + base + p * G.stride, sm + p * LB, LB * 8);
  asm volatile("cp.async.bulk.commit_group;" ::);
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__global__ void k_tensor(const __grid_constant__ CUtensorMap tm, Geo G, int axis0) {
  extern __shared__ __align__(1024) double smt[];
  double* sm = smt;
  __shared__ unsigned long long mbar;
  const int tid = threadIdx.x;
  // coordinates (k, j, i): axis 0 tiles run along i at fixed j, axis 1 along j at fixed i
  const int k0 = blockIdx.x * LB;
  if (tid == 0) {
    mbar_init(&mbar, 1);
    mbar_expect(&mbar, G.rows * LB * 8);
    for (int r0 = 0; r0 < G.rows; r0 += 256) {
      const int j = axis0 ? blockIdx.y : r0, i = axis0 ? r0 : blockIdx.y;
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smaddr(sm + r0 * LB)),
          "l"(&tm), "r"(k0), "r"(j), "r"(i), "r"(smaddr(&mbar))
          : "memory");
    }
  }
  __syncthreads();
  mbar_wait(&mbar, 0);
  if (tid == 0) {
    for (int r0 = 0; r0 < G.rows; r0 += 256) {
      const int j = axis0 ? blockIdx.y : r0, i = axis0 ? r0 : blockIdx.y;
      asm volatile(
          "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::
              "l"(&tm),
          "r"(k0), "r"(j), "r"(i), "r"(smaddr(sm + r0 * LB))
          : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::);
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

int main() {
  const int n = 513;
  const long long pitch = 544;
  const size_t elems = (size_t)n * n * pitch + 4096;
  double *a, *b, *c;
  cudaMalloc(&a, elems * 8);
  cudaMalloc(&b, elems * 8);
  cudaMalloc(&c, elems * 8);
  cudaMemset(a, 0, elems * 8);
  cudaMemset(b, 0, elems * 8);
  // fill a with a pattern, check both methods agree
  double* h = (double*)malloc(elems * 8);
  for (size_t i = 0; i < elems; ++i) h[i] = (double)(i % 1000003);
  cudaMemcpy(a, h, elems * 8, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)n, (cuuint64_t)n};
  cuuint64_t strides[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)pitch * n * 8};
  cuuint32_t box[3] = {LB, 1, 256}, es[3] = {1, 1, 1};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int ax = 0; ax < 2; ++ax) {
    const bool axis0 = ax == 0;
    Geo G;
    G.rows = n + 2 > 512 ? 512 : n;  // tensor boxes of 256 rows: 512 rows per tile
    G.stride = axis0 ? (long long)n * pitch : pitch;
    G.outer = axis0 ? pitch : (long long)n * pitch;
    dim3 grid(512 / LB, n - 2);
    const size_t smem = (size_t)G.rows * LB * 8;
    cudaFuncSetAttribute(k_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_tensor, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (axis0) { box[1] = 1; box[2] = 256; } else { box[1] = 256; box[2] = 1; }
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a, dims, strides,
                                        box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("tensor map encode failed %d\n", (int)r);
    for (int v = 0; v < 3; ++v) {
      for (int nt : {128, 256, 512}) {
        auto launch = [&]() {
          if (v == 0) k_cpasync<<<grid, nt, smem>>>(a, b, G);
          else if (v == 1) k_bulk<<<grid, nt, smem>>>(a, b, G);
          else k_tensor<<<grid, nt, smem>>>(tm, G, axis0);
        };
        launch();
        launch();
        cudaEventRecord(e0);
        for (int it = 0; it < 5; ++it) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 5;
        const double bytes = 2.0 * G.rows * (double)(n - 2) * 512 * 8;
        printf("axis%d %-8s nt=%3d smem %6zu: %7.1f us  %6.0f GB/s  %s\n", ax,
               v == 0 ? "cp.async" : (v == 1 ? "bulk" : "tensor"), nt, smem, ms * 1e3,
               bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        if (v == 2) break;  // one thread issues everything
      }
    }
  }
  return 0;
}
