// Cycles per k-block of the Ozaki sketch's MMA sequence (ozaki.cu) issued back to back
// without barriers: one CTA per SM, one thread issues R k-blocks.  Orders:
//   0: plane-major, k-steps innermost (the kernel's order)
//   1: k-step-major (each k-step walks all planes)
//   2: same MAC count as N = 256 MMAs only (9 per k-step) -- the rate bound
//   3: order 0 + a tcgen05.commit per A stage (no waits)
//   4: order 3 + the issuing thread waits for the commit of the stage's previous use
//      (a 6-stage ring, as the kernel's producer does)
//   5: the kernel's handshake without data: warp 0 waits for a stage's commit and posts
//      it "full", warp 1 waits for "full", issues the stage's MMAs and commits it
//   6: as 5 with test_wait spinning instead of try_wait
//   7: as 5 with the whole MMA warp waiting in a C++ loop over a single try_wait (converged)
//   8: as 7 without the tcgen05.fence::after_thread_sync per stage
//   9: one thread of the MMA warp waits and issues, no fence, the other lanes leave
//  10: as 9 with the producer backing off 64 ns between polls
//  11: as 9 plus four warps polling a barrier for the whole run (the epilogue's wait)
//  12: as 11 with the pollers sleeping 500 ns between polls
//  13: as 9 with 2-plane (32 KB) stages, 3 of them; 14: 4-plane (64 KB) stages, 2 of them
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_seq tc_seq.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return ((uint64_t)(a >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint32_t idesc(int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ bool try_bar(uint64_t* b, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
               : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t par, bool spin) {
  if (spin)
    asm volatile("{\n\t.reg .pred p;\n\tS_%=:\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra S_%=;\n\t}\n"
                 ::"r"(su32(b)), "r"(par) : "memory");
  else
    asm volatile("{\n\t.reg .pred p;\n\tT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra T_%=;\n\t}\n"
                 ::"r"(su32(b)), "r"(par) : "memory");
}
template <int ORDER_NS>
__global__ void seq(int R, unsigned long long* cyc, int fill) {
  constexpr int ORDER = ORDER_NS % 100, NS = ORDER_NS / 100 ? ORDER_NS / 100 : 6;  // stages in the ring
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint64_t sbar[16];
  __shared__ uint64_t fbar[16];
  __shared__ uint32_t tslot;
  uint32_t x = 12345u + threadIdx.x * 7919u + blockIdx.x;
  for (int i = threadIdx.x; i < (224 << 10) / 4; i += blockDim.x) {
    x = x * 1664525u + 1013904223u;
    uint32_t w = 0;
    for (int b = 0; b < 4; ++b) w |= (uint32_t)(uint8_t)((int)((x >> (8 * b)) & 127) - 63) << (8 * b);
    ((uint32_t*)sm)[i] = fill ? w : 0;
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    for (int i = 0; i < NS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&sbar[i])));
    for (int i = 0; i < NS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&fbar[i])));
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
  if (ORDER >= 5) {
    const uint32_t sa = su32(sm), sb = su32(sm) + NS * 16384;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long t0 = clock64();
    if (warp >= 2 && (ORDER == 11 || ORDER == 12)) {
      // epilogue-like warps: every thread polls a barrier that completes only at the end
      while (!try_bar(&bar, 0)) {
        if (ORDER == 12) __nanosleep(500);
      }
    } else if (warp == 0 && lane == 0) {
      int ai = 0; uint32_t ph = 0;
      constexpr int PPS0 = ORDER == 13 ? 2 : ORDER == 14 ? 4 : 1;
      for (int i = 0; i < R * 8 / PPS0; ++i) {
        if (ORDER >= 7) {
          while (!try_bar(&sbar[ai], ph ^ 1)) {
            if (ORDER == 10) __nanosleep(64);
          }
        } else {
          wait_bar(&sbar[ai], ph ^ 1, ORDER == 6);
        }
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&fbar[ai])) : "memory");
        if (++ai == NS) { ai = 0; ph ^= 1; }
      }
    } else if (warp == 1 && ORDER >= 9) {
      // one thread issues and waits; the other lanes leave.  PPS planes per stage.
      constexpr int PPS = ORDER == 13 ? 2 : ORDER == 14 ? 4 : 1;
      if (lane == 0) {
        int ai = 0; uint32_t ph = 0;
        for (int r = 0; r < R; ++r)
          for (int s = 0; s < 8; ++s) {
            if (s % PPS == 0) {
              while (!try_bar(&fbar[ai], ph)) {
              }
            }
            const uint64_t da = desc(sa + ai * 16384 * PPS + (s % PPS) * 16384);
            for (int t0 = 0; t0 < 8 - s; t0 += 4) {
              const int nt = min(4, 8 - s - t0);
              const uint64_t db = desc(sb + t0 * 8192);
              for (int kk = 0; kk < 4; ++kk)
                mma(tmem + (s + t0) * 64, da + 2 * kk, db + 2 * kk, idesc(64 * nt), (r | s | kk) ? 1 : 0);
            }
            if (s % PPS == PPS - 1) {
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&sbar[ai])) : "memory");
              if (++ai == NS) { ai = 0; ph ^= 1; }
            }
          }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)));
        wait_bar(&bar, 0, false);
        cyc[blockIdx.x] = clock64() - t0;
      }
    } else if (warp == 1) {
      int ai = 0; uint32_t ph = 0;
      for (int r = 0; r < R; ++r)
        for (int s = 0; s < 8; ++s) {
          if (ORDER >= 7) {
            while (!try_bar(&fbar[ai], ph)) {
            }
          } else {
            if (lane == 0) wait_bar(&fbar[ai], ph, ORDER == 6);
            __syncwarp();
          }
          if (ORDER != 8) asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          if (lane == 0) {
            const uint64_t da = desc(sa + ai * 16384);
            for (int t0 = 0; t0 < 8 - s; t0 += 4) {
              const int nt = min(4, 8 - s - t0);
              const uint64_t db = desc(sb + t0 * 8192);
              for (int kk = 0; kk < 4; ++kk)
                mma(tmem + (s + t0) * 64, da + 2 * kk, db + 2 * kk, idesc(64 * nt), (r | s | kk) ? 1 : 0);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&sbar[ai])) : "memory");
          }
          __syncwarp();
          if (++ai == NS) { ai = 0; ph ^= 1; }
        }
      if (lane == 0) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)));
        wait_bar(&bar, 0, false);
        cyc[blockIdx.x] = clock64() - t0;
      }
    }
  } else if (threadIdx.x == 0) {
    const uint32_t sa = su32(sm), sb = su32(sm) + 96 * 1024;
    unsigned long long t0 = clock64();
    int ai = 0;
    int use[6] = {0, 0, 0, 0, 0, 0};
    for (int r = 0; r < R; ++r) {
      if (ORDER == 0 || ORDER == 3 || ORDER == 4) {
        for (int s = 0; s < 8; ++s) {
          if (ORDER == 4 && use[ai] > 0) {
            const uint32_t par = (use[ai] - 1) & 1;
            asm volatile("{\n\t.reg .pred p;\n\tW4_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W4_%=;\n\t}\n"
                         ::"r"(su32(&sbar[ai])), "r"(par) : "memory");
          }
          const uint64_t da = desc(sa + ai * 16384);
          for (int t0 = 0; t0 < 8 - s; t0 += 4) {
            const int nt = min(4, 8 - s - t0);
            const uint64_t db = desc(sb + t0 * 8192);
            for (int kk = 0; kk < 4; ++kk)
              mma(tmem + (s + t0) * 64, da + 2 * kk, db + 2 * kk, idesc(64 * nt), (r | s | kk) ? 1 : 0);
          }
          if (ORDER >= 3) {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&sbar[ai])) : "memory");
            ++use[ai];
          }
          ai = ai == 5 ? 0 : ai + 1;
        }
      } else if (ORDER == 1) {
        for (int kk = 0; kk < 4; ++kk)
          for (int s = 0; s < 8; ++s) {
            const uint64_t da = desc(sa + ((ai + s) % 6) * 16384);
            for (int t0 = 0; t0 < 8 - s; t0 += 4) {
              const int nt = min(4, 8 - s - t0);
              const uint64_t db = desc(sb + t0 * 8192);
              mma(tmem + (s + t0) * 64, da + 2 * kk, db + 2 * kk, idesc(64 * nt), (r | s | kk) ? 1 : 0);
            }
          }
        ai = (ai + 8) % 6;
      } else {
        for (int i = 0; i < 9; ++i) {
          const uint64_t da = desc(sa + (i % 6) * 16384);
          const uint64_t db = desc(sb + (i & 1) * 32768);
          for (int kk = 0; kk < 4; ++kk) mma(tmem + (i & 1) * 256, da + 2 * kk, db + 2 * kk, idesc(256), 1);
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)));
    asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}\n" ::"r"(su32(&bar)));
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int R = 2000;
  const int smem = (224 << 10) + 1024;
  void (*ks[6])(int, unsigned long long*, int) = {seq<0>, seq<4>, seq<9>, seq<313>, seq<214>, seq<11>};
  const int names[6] = {0, 4, 9, 313, 214, 11};
  for (int fill = 1; fill < 2; ++fill)
    for (int o = 0; o < 6; ++o) {
      cudaFuncSetAttribute(ks[o], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      ks[o]<<<148, 192, smem>>>(R, d, fill);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      ks[o]<<<148, 192, smem>>>(R, d, fill);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("order %d (stages %d) %s digits: %.0f cycles per k-block (clock64), %.3f us per k-block wall (%s)\n", names[o] % 100, names[o] / 100 ? names[o] / 100 : 6,
             fill ? "random" : "zero", (double)h[0] / R, ms * 1e3 / R, cudaGetErrorString(err));
    }
  return 0;
}
