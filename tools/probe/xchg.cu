// All-to-all argmax exchange latency per step across a co-resident grid (the panel's
// per-column critical hop), flat vs thread-block clusters:
//   flat:     every CTA publishes an LL record (value + step flag per 8-byte word) and polls
//             all G records;
//   cluster:  CTAs write their value into the cluster leader's shared memory (st.async +
//             mbarrier complete_tx), the leader reduces and publishes one record, every CTA
//             polls the G/C leader records.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xchg xchg.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ void st_v4(uint4* p, uint4 v) {
  asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint4 ld_v4(const uint4* p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// records: [2][256][8] uint4 (one 128-byte line each).  busy: warps 1-7 run a shared-memory
// rank-1-update loop (the panel's late update) until warp 0 has finished its steps.
__global__ void flat(uint4* rec, int steps, unsigned base, unsigned long long* out, int busy) {
  const int G = gridDim.x, cta = blockIdx.x, lane = threadIdx.x & 31;
  __shared__ double buf[64 * 64];
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) buf[i] = i * 1e-3;
  __syncthreads();
  unsigned best = cta * 2654435761u;
  unsigned long long t0 = clock64();
  if (threadIdx.x >= 32) {
    if (busy) {
      const int w = threadIdx.x / 32 - 1, nw = blockDim.x / 32 - 1;
      double u0 = 0.5, u1 = 0.25;
      while (!done) {
        for (int i = w; i < 64; i += nw) {
          const double l = buf[i * 64 + (lane & 1)];
          buf[i * 64 + ((2 + lane) ^ (i & 31))] -= l * u0;
          buf[i * 64 + ((34 + lane) & 63)] -= l * u1;
        }
      }
    }
  } else {
    for (int j = 0; j < steps; ++j) {
      const unsigned f = base + j + 1, par = j & 1;
      if (lane == 0) st_v4(&rec[(par * 256 + cta) * 8], make_uint4(best ^ j, f, 0, f));
      unsigned m = 0;
      for (int c = lane; c < G; c += 32) {
        uint4 v;
        do { v = ld_v4(&rec[(par * 256 + c) * 8]); } while (v.y != f || v.w != f);
        m = max(m, v.x);
      }
      for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(~0u, m, o));
      best = m * 2654435761u + cta;
    }
    if (lane == 0) done = 1;
  }
  if (threadIdx.x == 0 && cta == 0) out[0] = clock64() - t0;
}

__constant__ int getenv_busy_c;
__constant__ int rowmode_c;  // 0 none, 1 rowdata stores after st.async, 2 before
__device__ uint4 g_rowdata[2][256][64];
#define getenv_busy getenv_busy_c
template <int C>
__global__ void clustered(uint4* rec, int steps, unsigned base, unsigned long long* out) {
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(16) unsigned long long slot[2][16];
  __shared__ double buf[64 * 64];
  __shared__ volatile int done;
  const int busy = getenv_busy;
  if (threadIdx.x == 0) done = 0;
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) buf[i] = i * 1e-3;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  const int L = gridDim.x / C, leader = blockIdx.x / C, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  cl.sync();
  // leader's barrier and slots in the cluster's shared window
  uint32_t rbar, rslot;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(rbar) : "r"(su32(&bar)));
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(rslot) : "r"(su32(&slot[0][0])));
  unsigned best = blockIdx.x * 2654435761u;
  unsigned long long t0 = clock64();
  if (threadIdx.x >= 32) {
    if (busy) {
      const int w = threadIdx.x / 32 - 1, nw = blockDim.x / 32 - 1;
      double u0 = 0.5, u1 = 0.25;
      while (!done) {
        for (int i = w; i < 64; i += nw) {
          const double l = buf[i * 64 + (lane & 1)];
          buf[i * 64 + ((2 + lane) ^ (i & 31))] -= l * u0;
          buf[i * 64 + ((34 + lane) & 63)] -= l * u1;
        }
      }
    }
  } else {
    for (int j = 0; j < steps; ++j) {
      const unsigned f = base + j + 1, par = j & 1;
      if (rowmode_c == 2)
        for (int c = lane; c < 64; c += 32) st_v4(&g_rowdata[par][blockIdx.x][c], make_uint4(best + c, f, c, f));
      if (lane == 0) {
        if (rank == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar)), "r"(C * 8) : "memory");
        const unsigned long long v = (unsigned long long)(best ^ j);
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(
                         rslot + (uint32_t)((par * 16 + rank) * 8)),
                     "l"(v), "r"(rbar)
                     : "memory");
      }
      if (rowmode_c == 1)
        for (int c = lane; c < 64; c += 32) st_v4(&g_rowdata[par][blockIdx.x][c], make_uint4(best + c, f, c, f));
      if (rank == 0) {
        if (lane == 0)
          asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}\n" ::"r"(su32(&bar)), "r"(par) : "memory");
        __syncwarp();
        unsigned m = 0;
        for (int q = 0; q < C; ++q) m = max(m, (unsigned)((volatile unsigned long long*)slot[par])[q]);
        if (lane == 0) st_v4(&rec[(par * 256 + leader) * 8], make_uint4(m, f, 0, f));
      }
      unsigned m = 0;
      for (int c = lane; c < L; c += 32) {
        uint4 v;
        do { v = ld_v4(&rec[(par * 256 + c) * 8]); } while (v.y != f || v.w != f);
        m = max(m, v.x);
      }
      for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(~0u, m, o));
      if (rowmode_c) {  // hop 2: the "winner" CTA's row
        const int wc = (int)(m % gridDim.x);
        for (int c = lane; c < 64; c += 32) {
          uint4 v;
          do { v = ld_v4(&g_rowdata[par][wc][c]); } while (v.y != f || v.w != f);
          m += v.z;
        }
      }
      best = m * 2654435761u + blockIdx.x;
    }
    if (lane == 0) done = 1;
  }
  cl.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int which = argc > 1 ? atoi(argv[1]) : 0;  // 0 flat, 1 flat + busy warps, else the cluster size
  uint4* rec;
  unsigned long long* out;
  cudaMalloc(&rec, 2 * 256 * 8 * sizeof(uint4));
  cudaMemset(rec, 0, 2 * 256 * 8 * sizeof(uint4));
  cudaMalloc(&out, 8);
  const int steps = 2000;
  unsigned base = 0;
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  if (which == 9) {  // many launches at G = 32: per-launch step time (bimodality check)
    for (int rep = 0; rep < 40; ++rep) {
      int G = 32, busy = 0;
      const int st2 = 200;
      void* args[] = {&rec, (void*)&st2, &base, &out, &busy};
      base += 1 << 16;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)flat, G, 256, args, 0, 0);
      cudaEventRecord(e1);
      cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("launch %d: %.3f us/step\n", rep, ms * 1e3 / st2);
    }
  }
  if (which == 0 || which == 1) for (int G : {32, 64, 96, 128, nsm}) {
    int busy = which;
    void* args[] = {&rec, (void*)&steps, &base, &out, &busy};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    base += 1 << 16;
    cudaEventRecord(e0);
    cudaError_t e = cudaLaunchCooperativeKernel((void*)flat, G, 256, args, 0, 0);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc; cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
    printf("flat%s G=%d: %.3f us/step (%llu cycles/step) %s\n", busy ? " +busy warps" : "", G, ms * 1e3 / steps, cyc / steps, cudaGetErrorString(e));
  }
  auto run_cluster = [&](auto kern, int C) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = 256;
    const int dyn = getenv("XCHG_SMEM") ? atoi(getenv("XCHG_SMEM")) : 0;  // e.g. 120000: one CTA per SM
    cfg.dynamicSmemBytes = dyn;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at; cfg.numAttrs = 2;
    int ncl = 0;
    cfg.gridDim = C * 64;
    cudaError_t eo = cudaOccupancyMaxActiveClusters(&ncl, (void*)kern, &cfg);
    for (int G : {C * 8, C * 16, ncl * C}) {
      if (G > ncl * C || G > 148) continue;
      cfg.gridDim = G;
      base += 1 << 16;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cudaError_t e = cudaLaunchKernelEx(&cfg, kern, rec, steps, base, out);
      cudaEventRecord(e1);
      cudaError_t e2 = cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long cyc; cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
      printf("cluster C=%d G=%d (max active clusters %d, %s): %.3f us/step (%llu cycles/step) %s %s\n", C, G, ncl,
             cudaGetErrorString(eo), ms * 1e3 / steps, cyc / steps, cudaGetErrorString(e), cudaGetErrorString(e2));
    }
  };
  { int b = getenv("XCHG_BUSY") ? 1 : 0; cudaMemcpyToSymbol(getenv_busy_c, &b, sizeof(int)); }
  { int b = getenv("XCHG_ROW") ? atoi(getenv("XCHG_ROW")) : 0; cudaMemcpyToSymbol(rowmode_c, &b, sizeof(int));
    cudaMemset((void*)0, 0, 0); }
  if (which == 2) run_cluster(clustered<2>, 2);
  if (which == 4) run_cluster(clustered<4>, 4);
  if (which == 8) run_cluster(clustered<8>, 8);
  if (which == 16) run_cluster(clustered<16>, 16);
  return 0;
}
