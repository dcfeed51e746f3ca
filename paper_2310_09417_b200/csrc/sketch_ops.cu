// Dense device form of the structured embeddings of the reference
// (`sketching.py:134-235`), so every sketch kind runs through the same DMMA
// sketch GEMM:
//
//   SRTT (`make_srtt`): y = scale * (DCT-II_ortho(x[perm]) * signs)[cols], i.e.
//     Omega[perm[p], j] = scale * signs[q] * d(q, p),  q = cols[j],
//     d(q, p) = sqrt((q ? 2 : 1) / n) * cos(pi q (2p + 1) / (2n))
//   with the angle reduced exactly in integers (q (2p+1) mod 4n) and cospi.
//   Sparse sign (`make_sparse_sign`): Omega[r, idx[r, z]] = signs[r, z] * scale.
#include "common.cuh"
#include "rskel_internal.h"

#ifndef RS_SS_RPL  // rows of A per lane in the sparse-sign SpMM (2 or 4)
#define RS_SS_RPL 2
#endif
#ifndef RS_SS_STAGES  // cp.async pipeline depth of the sparse-sign SpMM
#define RS_SS_STAGES 2
#endif
#ifndef RS_SS_CPW  // y columns per warp (a CTA covers 8 x CPW columns)
#define RS_SS_CPW 8
#endif
#ifndef RS_SS_DBG
#define RS_SS_DBG 0
#endif
#ifndef RS_SS_KQ   // 32-column bitmap chunks of A per pipeline stage
#define RS_SS_KQ 1
#endif

namespace rs {

__global__ void srtt_dense_kernel(int n, int ell, const int64_t* __restrict__ perm, const double* __restrict__ signs,
                                  const int64_t* __restrict__ cols, double scale, double* __restrict__ out,
                                  long long ldo) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)n * ell) return;
  const int p = (int)(e / ell), j = (int)(e % ell);
  const long long q = cols[j];
  const long long fourn = 4LL * n;
  const long long r = (q * (2LL * p + 1)) % fourn;  // angle pi * r / (2n), r in [0, 4n)
  const double c = cospi((double)r / (2.0 * n));
  const double norm = q == 0 ? sqrt(1.0 / n) : sqrt(2.0 / n);
  out[perm[p] * ldo + j] = scale * signs[q] * norm * c;
}

int launch_srtt_dense(int n, int ell, const int64_t* perm, const double* signs, const int64_t* cols, double scale,
                      double* out, long long ldo, cudaStream_t st) {
  if (n < 1 || ell < 1 || ell > n || ldo < ell) return RS_ERR_ARG;
  const long long total = (long long)n * ell;
  srtt_dense_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(n, ell, perm, signs, cols, scale, out, ldo);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

__global__ void sparse_sign_dense_kernel(int n, int ell, int zeta, const int64_t* __restrict__ idx,
                                         const double* __restrict__ signs, double scale, double* __restrict__ out,
                                         long long ldo) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)n * zeta) return;
  const long long r = e / zeta;
  out[r * ldo + idx[e]] = signs[e] * scale;
}

int launch_sparse_sign_dense(int n, int ell, int zeta, const int64_t* idx, const double* signs, double scale,
                             double* out, long long ldo, cudaStream_t st) {
  if (n < 1 || ell < 1 || zeta < 1 || zeta > ell || ldo < ell) return RS_ERR_ARG;
  if (cudaMemset2DAsync(out, (size_t)ldo * 8, 0, (size_t)ell * 8, (size_t)n, st) != cudaSuccess) return RS_ERR_CUDA;
  const long long total = (long long)n * zeta;
  sparse_sign_dense_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(n, ell, zeta, idx, signs, scale, out,
                                                                            ldo);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}


// ---- sparse-sign embedding applied as an SpMM (no dense Omega) ---------------
// The reference applies the operator as `(csr.T @ a.T).T` (`sketching.py:176-185`):
// scipy's csc_matvecs walks the operator rows j in ascending order and does
// y[:, c] += v * a[:, j] with v = signs * scale, a separate multiply and add
// (no FMA).  Each output is therefore a sequential sum over the rows j that hold
// column c, in ascending j, starting from 0.  This kernel keeps exactly that
// order and rounding, so its y is bitwise the reference's.
//
// Plan: the operator as two bitmaps per (column c, 32-row chunk q) -- which rows
// of the chunk hold c, and which of them carry a negative sign.  Built with
// atomicOr (order-free, hence deterministic); requires signs of +-1 and no
// repeated index within a row (what `make_sparse_sign` draws; the host checks).
//
// Apply: a CTA owns SS_RB rows of A (lane l: rows l + 32 k) and up to 8 * CPW
// columns of y (warp w: columns w + 8 t).  A's 32-column chunks are staged in
// shared memory with cp.async (3 stages); per chunk each warp walks the set bits
// of its columns' bitmaps, lowest first.  Algorithmic HBM bytes: A once,
// 8 m n; the staged tile is read zeta times per element from shared memory.
namespace {
constexpr int SS_JC = 32;  // operator rows per bitmap word
constexpr int SS_WARPS = 8;
constexpr int SS_STAGES = RS_SS_STAGES;
}  // namespace

// plan: nzm[q * ell + c], then sgm likewise (chunk-major: one stage's words are contiguous)
long long sparse_sign_plan_words(int n, int ell) { return 2LL * ell * ((n + SS_JC - 1) / SS_JC); }

__global__ void sparse_sign_plan_kernel(int n, int zeta, int ell, const int64_t* __restrict__ idx,
                                        const double* __restrict__ signs, unsigned* __restrict__ nzm,
                                        unsigned* __restrict__ sgm, int* __restrict__ bad) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)n * zeta) return;
  const int j = (int)(e / zeta);
  const long long c = idx[e];
  const double sg = signs[e];
  if (c < 0 || c >= ell || !(sg == 1.0 || sg == -1.0)) {
    atomicOr(bad, 1);
    return;
  }
  const unsigned bit = 1u << (j & 31);
  const long long w = (long long)(j >> 5) * ell + c;
  const unsigned old = atomicOr(&nzm[w], bit);
  if (old & bit) atomicOr(bad, 2);  // repeated index in row j
  if (sg < 0) atomicOr(&sgm[w], bit);
}

// One pipeline stage: KQ bitmap chunks (32 KQ columns of A) for RB rows, plus
// the stage's bitmap words of this CTA's columns.
template <int RPL, int CPW, int KQ, bool CM>
__global__ void __launch_bounds__(SS_WARPS * 32) sparse_sign_apply_kernel(
    long long m, int n, int ell, const double* __restrict__ a, long long lda, int nq,
    const unsigned* __restrict__ nzm, const unsigned* __restrict__ sgm, double scale, double* __restrict__ y,
    long long ldy) {
  constexpr int RB = 32 * RPL;
  constexpr int SC = SS_JC * KQ;                               // A columns per stage
  constexpr int CG = SS_WARPS * CPW;                           // y columns per CTA
  constexpr int TILE = CM ? SC * RB : RB * (SC + 1);           // CM: [j][r]; row-major: [r][j], odd pitch
  constexpr int STAGE = TILE + (2 * KQ * CG + 1) / 2;          // + bitmaps, in doubles
  extern __shared__ double ss_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long r0 = (long long)blockIdx.x * RB;
  const int c0 = blockIdx.y * CG;
  const int ns = (nq + KQ - 1) / KQ;
  const int cg = min(CG, ell - c0);
  const unsigned scale_hi = (unsigned)__double2hiint(scale), scale_lo = (unsigned)__double2loint(scale);

  auto stage = [&](int s, int buf) {
    double* t = ss_smem + buf * STAGE;
    unsigned* mw = reinterpret_cast<unsigned*>(t + TILE);
    const int j0 = s * SC;
    if (CM) {
      for (int i = warp; i < SC; i += SS_WARPS) {
        if (j0 + i >= n) break;
#pragma unroll
        for (int k = 0; k < RPL; ++k) {
          const long long r = r0 + lane + 32 * k;
          if (r < m) cp_async8(t + i * RB + lane + 32 * k, a + (long long)(j0 + i) * lda + r, 8);
        }
      }
    } else {
#pragma unroll
      for (int h = 0; h < KQ; ++h) {
        const int j = j0 + 32 * h + lane;
        if (j < n)
          for (int r = warp; r < RB; r += SS_WARPS)
            if (r0 + r < m) cp_async8(t + r * (SC + 1) + 32 * h + lane, a + (r0 + r) * lda + j, 8);
      }
    }
    for (int i = threadIdx.x; i < 2 * KQ * CG; i += SS_WARPS * 32) {
      const int which = i / (KQ * CG), rem = i % (KQ * CG), h = rem / CG, cl = rem % CG;
      const int q = s * KQ + h;
      if (q < nq && cl < cg) {
        const unsigned* src = (which ? sgm : nzm) + (long long)q * ell + c0 + cl;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(
                         (unsigned)__cvta_generic_to_shared(mw + i)),
                     "l"(src));
      }
    }
  };

  double acc[CPW][RPL];
#pragma unroll
  for (int u = 0; u < CPW; ++u)
#pragma unroll
    for (int k = 0; k < RPL; ++k) acc[u][k] = 0.0;

#pragma unroll
  for (int s = 0; s < SS_STAGES - 1; ++s) {
    if (s < ns) stage(s, s);
    cp_async_commit();
  }
  for (int s = 0; s < ns; ++s) {
    cp_async_wait<SS_STAGES - 2>();
    __syncthreads();
    if (s + SS_STAGES - 1 < ns) stage(s + SS_STAGES - 1, (s + SS_STAGES - 1) % SS_STAGES);
    cp_async_commit();
    const double* t = ss_smem + (s % SS_STAGES) * STAGE;
    const unsigned* mw = reinterpret_cast<const unsigned*>(t + TILE);
#pragma unroll
    for (int h = 0; h < KQ; ++h) {
      if (s * KQ + h >= nq) break;
#pragma unroll
      for (int u = 0; u < CPW; ++u) {
        const int cl = warp + SS_WARPS * u;
        if (cl >= cg) break;
        // bit-reversed words: clz walks the operator rows in ascending order and
        // the row's sign bit shifts straight into the sign of `scale`
        // p = 31 - b is the highest set bit of the reversed word: b ascends
        unsigned rm = __brev(mw[h * CG + cl]);
        const unsigned sg = mw[KQ * CG + h * CG + cl];
        const double* end = CM ? t + (32 * h + 31) * RB + lane : t + lane * (SC + 1) + 32 * h + 31;
        if (RS_SS_DBG) rm = 0;  // experiment: staging only
        while (rm) {
          unsigned p;
          asm("bfind.u32 %0, %1;" : "=r"(p) : "r"(rm));
          rm ^= 1u << p;
          const double v = __hiloint2double(scale_hi ^ ((sg << p) & 0x80000000u), scale_lo);
#pragma unroll
          for (int k = 0; k < RPL; ++k) {
            const double x = CM ? end[32 * k - p * RB] : end[32 * k * (SC + 1) - p];
            acc[u][k] = __dadd_rn(acc[u][k], __dmul_rn(v, x));
          }
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < CPW; ++u) {
    const int c = c0 + warp + SS_WARPS * u;
    if (c >= ell) break;
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const long long r = r0 + lane + 32 * k;
      if (r < m) y[r * ldy + c] = acc[u][k];
    }
  }
}

template <int RPL, int CPW, int KQ>
static int ss_launch(long long m, int n, int ell, const double* a, long long lda, bool cm, int nq,
                     const unsigned* nzm, const unsigned* sgm, double scale, double* y, long long ldy,
                     cudaStream_t st) {
  constexpr int RB = 32 * RPL, SC = SS_JC * KQ, CG = SS_WARPS * CPW;
  const size_t stage = (size_t)(cm ? SC * RB : RB * (SC + 1)) + (2 * KQ * CG + 1) / 2;
  const size_t smem = SS_STAGES * stage * sizeof(double);
  auto k = cm ? sparse_sign_apply_kernel<RPL, CPW, KQ, true> : sparse_sign_apply_kernel<RPL, CPW, KQ, false>;
  // set on every launch (cheap), so every device of the process has it
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return RS_ERR_CUDA;
  const dim3 grid((unsigned)((m + RB - 1) / RB), (unsigned)((ell + CG - 1) / CG));
  k<<<grid, SS_WARPS * 32, smem, st>>>(m, n, ell, a, lda, nq, nzm, sgm, scale, y, ldy);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

int launch_sparse_sign_apply(long long m, int n, int ell, int zeta, const double* a, long long lda, int colmajor,
                             const int64_t* idx, const double* signs, double scale, double* y, long long ldy,
                             unsigned* plan, int* bad, cudaStream_t st) {
  if (m < 0 || n < 1 || ell < 1 || zeta < 1 || zeta > ell || ldy < ell || !plan || !bad) return RS_ERR_ARG;
  if (lda < (colmajor ? m : n)) return RS_ERR_ARG;
  const int nq = (n + SS_JC - 1) / SS_JC;
  const long long words = (long long)ell * nq;
  if (cudaMemsetAsync(plan, 0, (size_t)(2 * words) * sizeof(unsigned), st) != cudaSuccess) return RS_ERR_CUDA;
  const long long nnz = (long long)n * zeta;
  sparse_sign_plan_kernel<<<(unsigned)((nnz + 255) / 256), 256, 0, st>>>(n, zeta, ell, idx, signs, plan,
                                                                          plan + words, bad);
  count_launch(1);
  if (cudaGetLastError() != cudaSuccess) return RS_ERR_CUDA;
  if (m == 0) return RS_OK;
  const unsigned* nzm = plan;
  const unsigned* sgm = plan + words;
#define RS_SS_GO(RPL, CPW) ss_launch<RPL, CPW, RS_SS_KQ>(m, n, ell, a, lda, colmajor, nq, nzm, sgm, scale, y, ldy, st)
  constexpr int cpw = RS_SS_CPW;
  constexpr int cpw_small = cpw < 4 ? cpw : 4;
#if RS_SS_RPL == 1
  if (ell <= 32) return RS_SS_GO(1, cpw_small);
  return RS_SS_GO(1, cpw);
#else
  if (ell <= 32) return RS_SS_RPL == 4 ? RS_SS_GO(4, cpw_small) : RS_SS_GO(2, cpw_small);
  return RS_SS_RPL == 4 ? RS_SS_GO(4, cpw) : RS_SS_GO(2, cpw);
#endif
#undef RS_SS_GO
}

}  // namespace rs
