// Microbenchmark: inter-CTA exchange latency through L2 on B200.
// (1) ping-pong between CTA 0 and CTA G-1 via volatile flags
// (2) all-to-all "publish + poll G flags" rounds (the panel's exchange pattern)
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void stv(unsigned* p, unsigned v) { asm volatile("st.volatile.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ unsigned ldv(const unsigned* p) { unsigned v; asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned ldr(const unsigned* p) { unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }

__global__ void pingpong(unsigned* flags, int iters, long long* out) {
  int c = blockIdx.x, G = gridDim.x;
  if (threadIdx.x != 0) return;
  if (c != 0 && c != G - 1) return;
  long long t0 = clock64();
  for (int i = 1; i <= iters; ++i) {
    if (c == 0) { stv(&flags[0], i); while (ldv(&flags[64]) != (unsigned)i) {} }
    else { while (ldv(&flags[0]) != (unsigned)i) {} stv(&flags[64], i); }
  }
  if (c == 0) out[0] = (clock64() - t0) / iters;
}

__global__ void alltoall(unsigned* flags, int iters, long long* out, int relaxed) {
  int c = blockIdx.x, G = gridDim.x;
  int lane = threadIdx.x;
  long long t0 = clock64();
  for (int i = 1; i <= iters; ++i) {
    if (lane == 0) stv(&flags[c * 32], i);
    for (int q = lane; q < G; q += 32) {
      if (relaxed) while (ldr(&flags[q * 32]) < (unsigned)i) {}
      else while (ldv(&flags[q * 32]) < (unsigned)i) {}
    }
    __syncwarp();
  }
  if (c == 0 && lane == 0) out[1] = (clock64() - t0) / iters;
}

int main() {
  unsigned* flags; long long* out; cudaMalloc(&flags, 1 << 20); cudaMalloc(&out, 64);
  for (int G : {2, 16, 74, 148}) {
    cudaMemset(flags, 0, 1 << 20);
    pingpong<<<G, 32>>>(flags, 1000, out);
    long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    cudaMemset(flags, 0, 1 << 20);
    alltoall<<<G, 32>>>(flags, 1000, out, 0);
    cudaMemcpy(h + 1, out + 1, 8, cudaMemcpyDeviceToHost);
    long long r; cudaMemset(flags, 0, 1 << 20);
    alltoall<<<G, 32>>>(flags, 1000, out, 1);
    cudaMemcpy(&r, out + 1, 8, cudaMemcpyDeviceToHost);
    printf("G=%3d pingpong round trip %lld cyc, all-to-all round %lld cyc (relaxed %lld)  err=%s\n", G, h[0], h[1], r,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
