// tcgen05.mma issue-rate microbenchmark: one CTA per SM, one thread issues R MMAs
// (SS operands in shared memory) back to back; cycles per MMA by kind and N.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int KIND>
__global__ void rate(int R, uint32_t idesc, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) ((uint4*)sm)[i] = make_uint4(0x01010101u, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    uint64_t da = ((uint64_t)(su32(sm) >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
    uint64_t db = ((uint64_t)((su32(sm) + 32768) >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
    unsigned long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
      uint32_t d = tmem + (uint32_t)((r & 1) * 256);
      if (KIND == 0)
        asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;\n" ::"r"(d), "l"(da), "l"(db), "r"(idesc));
      else if (KIND == 1)
        asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n" ::"r"(d), "l"(da), "l"(db), "r"(idesc));
      else
        asm volatile("tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, 1;\n" ::"r"(d), "l"(da), "l"(db), "r"(idesc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)));
    asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}\n" ::"r"(su32(&bar)));
    unsigned long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int R = 4096;
  for (int kind = 0; kind < 3; ++kind)
    for (int N : {64, 128, 256}) {
      // c_format: i8 -> s32 (2), f16/f8 -> f32 (1); a/b format: i8 signed (1), f16 kind bf16 (1), f8 e4m3 (0)
      uint32_t cf = kind == 0 ? 2 : 1, af = kind == 2 ? 0 : 1;
      uint32_t idesc = (cf << 4) | (af << 7) | (af << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
      void (*k)(int, uint32_t, unsigned long long*) = kind == 0 ? rate<0> : kind == 1 ? rate<1> : rate<2>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 2048);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      k<<<148, 128, 65536 + 2048>>>(R, idesc, d);  // warm
      cudaEventRecord(e0);
      k<<<148, 128, 65536 + 2048>>>(R, idesc, d);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double kk = kind == 1 ? 16 : 32;
      const double ops = 2.0 * 128 * N * kk * R * 148;
      printf("%s N=%d: %.1f cycles/MMA, %.0f TOPS (%s)\n", kind == 0 ? "i8" : kind == 1 ? "bf16" : "e4m3", N,
             (double)h[0] / R, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
    }
  return 0;
}
