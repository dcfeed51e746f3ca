// Microbenchmark replicating the panel exchange (reducer CTA + broadcast), variants.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE> __device__ __forceinline__ void st4(uint4* p, uint4 v) {
  if (MODE == 0) asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
template <int MODE> __device__ __forceinline__ uint4 ld4(const uint4* p) {
  uint4 v;
  if (MODE == 0) asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  else asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
struct WS { uint4 rec[2][1024][2]; uint4 bc[2][8]; uint4 row[2][1024][64]; };
template <int MODE>
__global__ void panel_like(WS* ws, int iters, long long* out, int rowstores) {
  int c = blockIdx.x, G = gridDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long t0 = clock64();
  for (int j = 0; j < iters; ++j) {
    int par = j & 1; unsigned f = j + 1;
    if (warp == 0) {
      if (rowstores) for (int q = lane; q < 64; q += 32) st4<MODE>(&ws->row[par][c][q], make_uint4(q, f, c, f));
      if (lane == 0) { st4<MODE>(&ws->rec[par][c][0], make_uint4(c, f, 0, f)); st4<MODE>(&ws->rec[par][c][1], make_uint4(c, f, c + 1, f)); }
      int win = 0;
      if (c == 0) {
        int best = -1;
        for (int q = lane; q < G; q += 32) {
          uint4 a, b;
          do { a = ld4<MODE>(&ws->rec[par][q][0]); b = ld4<MODE>(&ws->rec[par][q][1]); } while (a.y != f || a.w != f || b.y != f || b.w != f);
          best = max(best, (int)((a.x * 2654435761u + j) % 1000003u));
        }
        for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(~0u, best, o));
        win = best % G;
        if (lane == 0) { st4<MODE>(&ws->bc[par][0], make_uint4(win, f, 0, f)); }
      } else {
        uint4 h = make_uint4(0,0,0,0);
        if (lane == 0) do { h = ld4<MODE>(&ws->bc[par][0]); } while (h.y != f || h.w != f);
        win = __shfl_sync(~0u, (int)h.x, 0);
      }
      if (rowstores) for (int q = lane; q < 64; q += 32) { uint4 x; do { x = ld4<MODE>(&ws->row[par][win][q]); } while (x.y != f || x.w != f); }
    }
    __syncthreads();
  }
  if (c == 0 && threadIdx.x == 0) out[0] = (clock64() - t0) / iters;
}
int main() {
  WS* ws; long long* out; cudaMalloc(&ws, sizeof(WS)); cudaMalloc(&out, 64);
  for (int G : {16, 148}) for (int threads : {32, 256}) for (int rows : {0, 1}) {
    long long h0, h1;
    cudaMemset(ws, 0, sizeof(WS)); panel_like<0><<<G, threads>>>(ws, 500, out, rows); cudaMemcpy(&h0, out, 8, cudaMemcpyDeviceToHost);
    cudaMemset(ws, 0, sizeof(WS)); panel_like<1><<<G, threads>>>(ws, 500, out, rows); cudaMemcpy(&h1, out, 8, cudaMemcpyDeviceToHost);
    printf("G=%3d threads=%3d rowdata=%d: volatile %lld cyc/step, relaxed.gpu %lld cyc/step %s\n", G, threads, rows, h0, h1, cudaGetErrorString(cudaGetLastError()));
  }
}
