// Microbenchmark: FP64 tensor-core (DMMA) peak on sm_100a, register-only
// (no memory traffic), to pin the roofline denominator MEASURED_PEAKS lacks.
#include <cstdio>
#include <cuda_runtime.h>

template <int ITERS>
__global__ void dmma_m16n8k16(double* out) {
  double a[8], b[4], c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0};
  for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
        "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
        : "+d"(c0[0]), "+d"(c0[1]), "+d"(c0[2]), "+d"(c0[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
          "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
        "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
        : "+d"(c1[0]), "+d"(c1[1]), "+d"(c1[2]), "+d"(c1[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
          "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) s += c0[i] + c1[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int ITERS>
__global__ void dmma_m8n8k4(double* out) {
  double a = 1e-3 * threadIdx.x, b = 2e-3 * threadIdx.x;
  double c[4][2] = {};
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  double* out; cudaMalloc(&out, 4096 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int ITERS = 4096;
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int bps = 1; bps <= 4; bps *= 2) {
      int grid = p.multiProcessorCount * bps;
      dmma_m16n8k16<ITERS><<<grid, warps * 32>>>(out);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) dmma_m16n8k16<ITERS><<<grid, warps * 32>>>(out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 5.0 * grid * warps * (double)ITERS * 2 * (2.0 * 16 * 8 * 16);
      printf("m16n8k16 warps/blk %2d blk/SM %d: %.2f TF/s\n", warps, bps, flops / ms / 1e9);
      dmma_m8n8k4<ITERS><<<grid, warps * 32>>>(out);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) dmma_m8n8k4<ITERS><<<grid, warps * 32>>>(out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 5.0 * grid * warps * (double)ITERS * 4 * (2.0 * 8 * 8 * 4);
      printf("m8n8k4   warps/blk %2d blk/SM %d: %.2f TF/s\n", warps, bps, flops / ms / 1e9);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
