// Panel-exchange replica: all-to-all LL records (+ optional row data), one
// step per iteration, to find what makes a record round slow.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/sync_latency3.cu -o tools/sync_latency3
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
struct WS { uint4 rec[2][256][8]; uint4 row[2][256][64]; };
__device__ __forceinline__ void st4(uint4* p, unsigned a, unsigned b, unsigned c, unsigned d) {
  asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ uint4 ld4(const uint4* p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__global__ void xchg(WS* ws, int iters, long long* out, int rowdata, int smem_touch, int mode) {
  extern __shared__ double sm[];
  const int G = gridDim.x, cta = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (smem_touch) for (int i = threadIdx.x; i < smem_touch; i += blockDim.x) sm[i] = i;
  __syncthreads();
  long long t0 = clock64(), tpoll = 0;
  for (int j = 0; j < iters; ++j) {
    const int par = j & 1;
    const unsigned f = 1000u + j;
    if (warp == 0) {
      if (lane == 0) { st4(&ws->rec[par][cta][0], cta, f, 0, f); st4(&ws->rec[par][cta][1], cta, f, cta + 1, f); }
      if (rowdata) for (int c = lane; c < 64; c += 32) st4(&ws->row[par][cta][c], c, f, cta, f);
      long long tp = clock64();
      constexpr int QMAX = 8;
      const int nq = (G - lane + 31) / 32;
      unsigned pending = nq >= 32 ? 0xffffffffu : ((1u << nq) - 1u);
      int best = -1;
      while (pending) {
        uint4 a[QMAX], b[QMAX];
#pragma unroll
        for (int i = 0; i < QMAX; ++i)
          if ((pending >> i) & 1u) { a[i] = ld4(&ws->rec[par][lane + 32 * i][0]); b[i] = ld4(&ws->rec[par][lane + 32 * i][1]); }
#pragma unroll
        for (int i = 0; i < QMAX; ++i) {
          if (!((pending >> i) & 1u)) continue;
          if (a[i].y != f || a[i].w != f || b[i].y != f || b[i].w != f) continue;
          pending &= ~(1u << i);
          best = max(best, (int)((a[i].x * 2654435761u + j) % 1000003u));
        }
      }
      for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(~0u, best, o));
      tpoll += clock64() - tp;
      const int win = best % G;
      if (rowdata) for (int c = lane; c < 64; c += 32) { uint4 x; do { x = ld4(&ws->row[par][win][c]); } while (x.y != f || x.w != f); }
    } else if ((mode & 8) && smem_touch >= 128 * 64) {  // late-update-like smem rank-1 (warps 1..7)
      for (int i = warp - 1; i < 128; i += 7)
        for (int c = (j % 60) + 2 + lane; c < 64; c += 32) sm[i * 64 + c] = __dsub_rn(sm[i * 64 + c], __dmul_rn(sm[i * 64], 0.5));
    }
    __syncthreads();
    if ((mode & 1) && smem_touch >= 128 * 64) {  // early-update-like: one row per thread
      for (int i = threadIdx.x; i < 128; i += blockDim.x) {
        const double l = __ddiv_rn(sm[i * 64 + (j % 64)], 1.25);
        sm[i * 64 + (j % 64)] = l;
        sm[i * 64 + ((j + 1) % 64)] = __dsub_rn(sm[i * 64 + ((j + 1) % 64)], __dmul_rn(l, 0.75));
      }
    }
    if (mode & 2) { __syncthreads(); __syncthreads(); }
  }
  if (cta == 0 && threadIdx.x == 0) { out[0] = (clock64() - t0) / iters; out[1] = tpoll / iters; }
}
int main() {
  WS* ws; long long* out; cudaMalloc(&ws, sizeof(WS)); cudaMalloc(&out, 64);
  cudaFuncSetAttribute(xchg, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int G : {16, 148}) for (int coop : {1}) for (int smem : {70 * 1024}) for (int rows : {1}) for (int mode : {0, 1, 2, 8, 11}) {
    long long h[2];
    cudaMemset(ws, 0, sizeof(WS));
    int iters = 400, touch = smem / 8;
    if (coop) {
      void* args[] = {&ws, &iters, &out, &rows, &touch, &mode};
      cudaLaunchCooperativeKernel((void*)xchg, dim3(G), dim3(256), args, smem, 0);
    } else {
      xchg<<<G, 256, smem>>>(ws, iters, out, rows, touch, mode);
    }
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("G=%3d coop=%d smem=%6d rowdata=%d mode=%2d: %lld cyc/step, poll %lld cyc  %s\n", G, coop, smem, rows, mode, h[0], h[1],
           cudaGetErrorString(cudaGetLastError()));
  }
}
