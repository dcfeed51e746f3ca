// Shared device helpers for the randomized-skeleton (sketched LUPP) kernels.
// Target: sm_100a only (B200).  fp64 math runs on the DMMA pipe through
// mma.sync m16n8k4 (tcgen05 has no f64 kind); operands are staged through
// shared memory with cp.async (LDGSTS).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rskel.h"  // status codes

#define RS_DEV __device__ __forceinline__

namespace rs {

// ---- cp.async -------------------------------------------------------------
// 16-byte copy with zero fill: src_bytes in {0, 8, 16}.
RS_DEV void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
// 8-byte copy with zero fill: src_bytes in {0, 8}.
RS_DEV void cp_async8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
RS_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
RS_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- DMMA -----------------------------------------------------------------
// D(16x8) += A(16x4, row) * B(4x8, col), fp64.  Fragment ownership (lane =
// 4*g + t): a0 = A[g][t], a1 = A[g+8][t]; b0 = B[t][g];
// c0 = C[g][2t], c1 = C[g][2t+1], c2 = C[g+8][2t], c3 = C[g+8][2t+1].
RS_DEV void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// ---- memory ordering helpers for the in-kernel grid barrier ----------------
RS_DEV unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
RS_DEV void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
RS_DEV void red_release_gpu_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// Grid-wide barrier for a cooperatively launched kernel.  `bar` is zeroed
// before launch; the k-th barrier (1-based) waits until bar >= k * nblocks.
RS_DEV void grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    red_release_gpu_add(bar, 1u);
    while (ld_acquire_gpu(bar) < target) {
    }
  }
  __syncthreads();
}

// Pivot key ordering of the reference panel (`dense.py:194`): larger |v| wins,
// ties go to the smaller *current* position.  |v| is finite and >= 0, so its
// IEEE bit pattern orders like the value.
RS_DEV bool key_better(double va, int pa, double vb, int pb) {
  return (va > vb) || (va == vb && pa < pb);
}

}  // namespace rs

