// FP64 tensor-core (DMMA) throughput by mma.sync shape on sm_100a: m8n8k4 (two per
// m16n8k4), m16n8k4, m16n8k8, m16n8k16, register operands only, 8 independent
// accumulators per warp, 148 x 8 warps.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_shapes dmma_shapes.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__device__ __forceinline__ void mma16x8(double (&c)[4], const double* a, const double* b);

template <>
__device__ __forceinline__ void mma16x8<4>(double (&c)[4], const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(b[0]));
}
template <>
__device__ __forceinline__ void mma16x8<8>(double (&c)[4], const double* a, const double* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
template <>
__device__ __forceinline__ void mma16x8<16>(double (&c)[4], const double* a, const double* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int K>
__global__ void __launch_bounds__(256) bench(int iters, double* out) {
  double a[8], b[4], c[8][4];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-3 * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - 1e-3 * (threadIdx.x + i);
  for (int q = 0; q < 8; ++q)
    for (int e = 0; e < 4; ++e) c[q][e] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) mma16x8<K>(c[q], a, b);
  }
  double s = 0;
  for (int q = 0; q < 8; ++q)
    for (int e = 0; e < 4; ++e) s += c[q][e];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  const int iters = 20000;
  auto run = [&](auto kern, int K) {
    kern<<<148, 256>>>(100, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<148, 256>>>(iters, d);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 16 * 8 * K * 8.0 * iters * 8 /*warps*/ * 148;
    printf("m16n8k%d: %.2f TF/s (%s)\n", K, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
  };
  for (int rep = 0; rep < 2; ++rep) {
    run(bench<4>, 4);
    run(bench<8>, 8);
    run(bench<16>, 16);
  }
  return 0;
}
