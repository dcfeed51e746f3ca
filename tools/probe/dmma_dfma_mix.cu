// Probe: (1) is one m8n8k4 f64 DMMA bitwise an fma chain over k = 0..3 (or the reverse)?
// (2) do non-tensor DFMAs issue on a pipe separate from DMMA, i.e. does running both in
// the same warps add throughput?  nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_dfma_mix.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

__global__ void dmma_once(const double* A, const double* B, const double* Cin, double* D) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a = A[g * 4 + t], b = B[t * 8 + g];
  double c0 = Cin[g * 8 + 2 * t], c1 = Cin[g * 8 + 2 * t + 1];
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  D[g * 8 + 2 * t] = c0;
  D[g * 8 + 2 * t + 1] = c1;
}

template <bool MMA, bool FMA, int ITERS>
__global__ void mix(double* out, double s) {
  double a = 1e-3 * threadIdx.x, b = 2e-3 * threadIdx.x;
  double c[4][2] = {};
  double f[8];
  for (int i = 0; i < 8; ++i) f[i] = 1e-4 * (threadIdx.x + i);
#pragma unroll 2
  for (int it = 0; it < ITERS; ++it) {
    if (MMA) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
    if (FMA) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = fma(f[i], s, a);
    }
  }
  double acc = 0;
  for (int j = 0; j < 4; ++j) acc += c[j][0] + c[j][1];
  for (int i = 0; i < 8; ++i) acc += f[i];
  if (acc == 12345.678) out[threadIdx.x] = acc;
}

template <bool MMA, bool FMA>
float timeit(double* out, int grid, int threads) {
  const int IT = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mix<MMA, FMA, IT><<<grid, threads>>>(out, 0.999);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) mix<MMA, FMA, IT><<<grid, threads>>>(out, 0.999);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  // (1) rounding of one DMMA
  double hA[32], hB[32], hC[64], hD[64];
  srand(7);
  int same_fwd = 0, same_rev = 0, total = 0;
  double *A, *B, *C, *D;
  cudaMalloc(&A, 32 * 8); cudaMalloc(&B, 32 * 8); cudaMalloc(&C, 64 * 8); cudaMalloc(&D, 64 * 8);
  for (int trial = 0; trial < 200; ++trial) {
    for (int i = 0; i < 32; ++i) hA[i] = (rand() / (double)RAND_MAX - 0.5) * pow(2.0, rand() % 40 - 20);
    for (int i = 0; i < 32; ++i) hB[i] = (rand() / (double)RAND_MAX - 0.5) * pow(2.0, rand() % 40 - 20);
    for (int i = 0; i < 64; ++i) hC[i] = (rand() / (double)RAND_MAX - 0.5) * pow(2.0, rand() % 40 - 20);
    cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
    cudaMemcpy(C, hC, 512, cudaMemcpyHostToDevice);
    dmma_once<<<1, 32>>>(A, B, C, D);
    cudaMemcpy(hD, D, 512, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) {
        double fw = hC[i * 8 + j], rv = hC[i * 8 + j];
        for (int k = 0; k < 4; ++k) fw = fma(hA[i * 4 + k], hB[k * 8 + j], fw);
        for (int k = 3; k >= 0; --k) rv = fma(hA[i * 4 + k], hB[k * 8 + j], rv);
        same_fwd += hD[i * 8 + j] == fw;
        same_rev += hD[i * 8 + j] == rv;
        ++total;
      }
  }
  printf("DMMA m8n8k4 vs fma chain k=0..3: %d/%d equal; k=3..0: %d/%d equal\n", same_fwd, total, same_rev, total);
  // (2) throughput
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* out;
  cudaMalloc(&out, 4096 * 8);
  for (int warps = 4; warps <= 16; warps *= 2) {
    const int grid = p.multiProcessorCount * 2, th = warps * 32;
    const double n = (double)grid * th / 32 * 4096;  // warp-iterations
    float tm = timeit<true, false>(out, grid, th), tf = timeit<false, true>(out, grid, th),
          tb = timeit<true, true>(out, grid, th);
    // per warp-iteration: 4 DMMA m8n8k4 = 4 * 256 FMA; 32 DFMA x 32 lanes = 1024 FMA
    printf("warps/CTA %2d: DMMA only %.3f ms (%.1f TF/s) | DFMA only %.3f ms (%.1f TF/s) | both %.3f ms (%.1f TF/s)\n",
           warps, tm, n * 1024 * 2 / (tm * 1e-3) / 1e12, tf, n * 1024 * 2 / (tf * 1e-3) / 1e12, tb,
           n * 2048 * 2 / (tb * 1e-3) / 1e12);
  }
  return 0;
}
