// Standalone probe of one tcgen05.mma kind::i8 (M=128, N=64, K=128) from
// SWIZZLE_128B K-major shared-memory tiles; TMEM read back column by column.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const int8_t* ga, const int8_t* gb, int* out, uint32_t idesc, int lbo, int sbo, int layout,
                      int ld_mode) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~uintptr_t(1023));
  uint8_t* sa = sm;            // 16 KB
  uint8_t* sb = sm + 16384;    // 8 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 16384 / 16; i += blockDim.x) ((uint4*)sa)[i] = ((const uint4*)ga)[i];
  for (int i = threadIdx.x; i < 8192 / 16; i += blockDim.x) ((uint4*)sb)[i] = ((const uint4*)gb)[i];
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
    for (int kk = 0; kk < 4; ++kk) {
      uint64_t da = ((uint64_t)((su32(sa) + kk * 32) >> 4) & 0x3FFF) | ((uint64_t)lbo << 16) | ((uint64_t)sbo << 32) |
                    (1ull << 46) | ((uint64_t)layout << 61);
      uint64_t db = ((uint64_t)((su32(sb) + kk * 32) >> 4) & 0x3FFF) | ((uint64_t)lbo << 16) | ((uint64_t)sbo << 32) |
                    (1ull << 46) | ((uint64_t)layout << 61);
      uint32_t acc = kk > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                   "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)));
  }
  asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}\n" ::"r"(
      su32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = (warp & 3) * 32 + lane;
  for (int c = 0; c < 64; ++c) {
    uint32_t v;
    uint32_t ta = tmem + (((uint32_t)(warp & 3) * 32) << 16) + c;
    if (ld_mode == 0) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(ta));
    } else {
      uint32_t r[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(tmem + (((uint32_t)(warp & 3) * 32) << 16) + (c & ~15)));
      v = r[c & 15];
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (warp < 4) out[row * 64 + c] = (int)v;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

static int swz(int r, int c) { return (r / 8) * 1024 + (r % 8) * 128 + (((c / 16) ^ (r % 8)) * 16) + c % 16; }

int main(int argc, char** argv) {
  int lbo = argc > 1 ? atoi(argv[1]) : 1, sbo = argc > 2 ? atoi(argv[2]) : 64, layout = argc > 3 ? atoi(argv[3]) : 2;
  int swizzle_host = argc > 4 ? atoi(argv[4]) : 1;
  unsigned idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  if (argc > 5) idesc = (unsigned)strtoul(argv[5], nullptr, 0);
  int ld_mode = argc > 6 ? atoi(argv[6]) : 0;
  std::vector<int8_t> A(128 * 128), B(64 * 128), ha(16384), hb(8192);
  srand(1);
  for (auto& x : A) x = (int8_t)(rand() % 255 - 127);
  for (auto& x : B) x = (int8_t)(rand() % 255 - 127);
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < 128; ++c) ha[swizzle_host ? swz(r, c) : r * 128 + c] = A[r * 128 + c];
  for (int r = 0; r < 64; ++r)
    for (int c = 0; c < 128; ++c) hb[swizzle_host ? swz(r, c) : r * 128 + c] = B[r * 128 + c];
  int8_t *da, *db;
  int* dout;
  cudaMalloc(&da, 16384); cudaMalloc(&db, 8192); cudaMalloc(&dout, 128 * 64 * 4);
  cudaMemcpy(da, ha.data(), 16384, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), 8192, cudaMemcpyHostToDevice);
  cudaMemset(dout, 0, 128 * 64 * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  probe<<<1, 128, 32768>>>(da, db, dout, idesc, lbo, sbo, layout, ld_mode);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<int> out(128 * 64);
  cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0, first = -1;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 64; ++j) {
      long ref = 0;
      for (int k = 0; k < 128; ++k) ref += (long)A[i * 128 + k] * B[j * 128 + k];
      if (ref != out[i * 64 + j]) { ++bad; if (first < 0) first = i * 64 + j; }
    }
  printf("lbo=%d sbo=%d layout=%d swz=%d idesc=0x%08x ld=%d: err=%s wrong=%d/8192", lbo, sbo, layout, swizzle_host,
         idesc, ld_mode, cudaGetErrorString(e), bad);
  if (first >= 0) {
    int i = first / 64, j = first % 64;
    long ref = 0;
    for (int k = 0; k < 128; ++k) ref += (long)A[i * 128 + k] * B[j * 128 + k];
    printf(" first (%d,%d) got %d ref %ld; row0:", i, j, out[first], ref);
    for (int c = 0; c < 6; ++c) printf(" %d", out[c]);
  }
  printf("\n");
  return 0;
}
