// One-sided (Hestenes) Jacobi SVD of a tall-skinny matrix and the small
// helpers of the CUR linking solve `pinv_apply` (reference `dense.py:166-182`,
// LAPACK gelsd with rcond 1e-12) and of the two-sided ID condition flag
// (`skeleton.py:592-603`).
//
// X (p x q) is held transposed, Xt (q x p row-major: row i = column i of X), so
// every column operation is a contiguous, coalesced stream.  One launch runs
// one round of a round-robin (circle) schedule: CTA r rotates column pair
// (i, j) -- three dot products by a fixed-order block reduction, then the
// rotation of the two columns of X and of V.  Deterministic; converged when
// every |x_i . x_j| <= tol sqrt(|x_i|^2 |x_j|^2).
#include "common.cuh"
#include "rskel_internal.h"

namespace rs {

constexpr int JT = 256;

__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < JT / 32; ++w) s += red[w];
    red[JT / 32] = s;
  }
  __syncthreads();
  s = red[JT / 32];
  __syncthreads();
  return s;
}

__global__ void __launch_bounds__(JT) jacobi_round_kernel(double* __restrict__ Xt, long long ldx, int p,
                                                          double* __restrict__ Vt, long long ldv, int q,
                                                          const int* __restrict__ pairs, double tol,
                                                          unsigned long long* __restrict__ max_off) {
  __shared__ double red[JT / 32 + 1];
  const int i = pairs[2 * blockIdx.x], j = pairs[2 * blockIdx.x + 1];
  if (i < 0 || j < 0) return;  // bye (odd q)
  double* xi = Xt + (long long)i * ldx;
  double* xj = Xt + (long long)j * ldx;
  double a = 0.0, b = 0.0, g = 0.0;
  for (int r = threadIdx.x; r < p; r += JT) {
    const double u = xi[r], w = xj[r];
    a = fma(u, u, a);
    b = fma(w, w, b);
    g = fma(u, w, g);
  }
  a = block_sum(a, red);
  b = block_sum(b, red);
  g = block_sum(g, red);
  const double scale = sqrt(a) * sqrt(b);
  if (!(scale > 0.0)) return;
  const double off = fabs(g) / scale;
  if (threadIdx.x == 0) atomicMax(max_off, (unsigned long long)__double_as_longlong(off));
  if (!(off > tol)) return;
  // rotation annihilating g (Rutishauser's formulas)
  const double zeta = (b - a) / (2.0 * g);
  const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
  for (int r = threadIdx.x; r < p; r += JT) {
    const double u = xi[r], w = xj[r];
    xi[r] = c * u - s * w;
    xj[r] = s * u + c * w;
  }
  double* vi = Vt + (long long)i * ldv;
  double* vj = Vt + (long long)j * ldv;
  for (int r = threadIdx.x; r < q; r += JT) {
    const double u = vi[r], w = vj[r];
    vi[r] = c * u - s * w;
    vj[r] = s * u + c * w;
  }
}

int launch_jacobi_round(double* Xt, long long ldx, int p, double* Vt, long long ldv, int q, const int* pairs,
                        int npairs, double tol, unsigned long long* max_off, cudaStream_t st) {
  if (npairs <= 0) return RS_OK;
  jacobi_round_kernel<<<npairs, JT, 0, st>>>(Xt, ldx, p, Vt, ldv, q, pairs, tol, max_off);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

// A whole sweep in one cooperative launch: CTA c rotates pair c of every
// round, a grid barrier between rounds (the per-round launches of a small
// q x q problem were host-launch bound).  Same arithmetic as the round kernel.
__global__ void __launch_bounds__(JT) jacobi_sweep_kernel(double* __restrict__ Xt, long long ldx, int p,
                                                          double* __restrict__ Vt, long long ldv, int q,
                                                          const int* __restrict__ sched, int nrounds, double tol,
                                                          unsigned long long* __restrict__ max_off,
                                                          unsigned* __restrict__ bar) {
  __shared__ double red[JT / 32 + 1];
  const int G = gridDim.x;
  for (int rd = 0; rd < nrounds; ++rd) {
    const int* pairs = sched + (size_t)rd * 2 * G;
    const int i = pairs[2 * blockIdx.x], j = pairs[2 * blockIdx.x + 1];
    if (i >= 0 && j >= 0) {
      double* xi = Xt + (long long)i * ldx;
      double* xj = Xt + (long long)j * ldx;
      double a = 0.0, b = 0.0, g = 0.0;
      for (int r = threadIdx.x; r < p; r += JT) {
        const double u = xi[r], w = xj[r];
        a = fma(u, u, a);
        b = fma(w, w, b);
        g = fma(u, w, g);
      }
      a = block_sum(a, red);
      b = block_sum(b, red);
      g = block_sum(g, red);
      const double scale = sqrt(a) * sqrt(b);
      const double off = scale > 0.0 ? fabs(g) / scale : 0.0;
      if (threadIdx.x == 0 && scale > 0.0) atomicMax(max_off, (unsigned long long)__double_as_longlong(off));
      if (scale > 0.0 && off > tol) {
        const double zeta = (b - a) / (2.0 * g);
        const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
        for (int r = threadIdx.x; r < p; r += JT) {
          const double u = xi[r], w = xj[r];
          xi[r] = c * u - s * w;
          xj[r] = s * u + c * w;
        }
        double* vi = Vt + (long long)i * ldv;
        double* vj = Vt + (long long)j * ldv;
        for (int r = threadIdx.x; r < q; r += JT) {
          const double u = vi[r], w = vj[r];
          vi[r] = c * u - s * w;
          vj[r] = s * u + c * w;
        }
      }
    }
    __threadfence();
    grid_barrier(bar, (unsigned)((rd + 1) * G));
  }
}

int launch_jacobi_sweep(double* Xt, long long ldx, int p, double* Vt, long long ldv, int q, const int* sched,
                        int nrounds, int npairs, double tol, unsigned long long* max_off, unsigned* bar,
                        cudaStream_t st) {
  if (npairs <= 0 || nrounds <= 0) return RS_OK;
  int dev = 0, nsm = 148, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, jacobi_sweep_kernel, JT, 0);
  if (npairs > occ * nsm) return RS_ERR_CAPACITY;
  if (cudaMemsetAsync(bar, 0, sizeof(unsigned), st) != cudaSuccess) return RS_ERR_CUDA;
  void* args[] = {&Xt, &ldx, &p, &Vt, &ldv, &q, &sched, &nrounds, &tol, &max_off, &bar};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)jacobi_sweep_kernel, dim3(npairs), dim3(JT), args, 0, st);
  count_launch(1);
  return e == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

// sigma_i = |Xt[i, :]|, d_i = 1 / sigma_i^2 if sigma_i > rcond * max sigma else 0;
// scales column i of V (row i of Vt) by d_i.  One CTA.
__global__ void __launch_bounds__(JT) pinv_scale_kernel(const double* __restrict__ Xt, long long ldx, int p,
                                                        double* __restrict__ Vt, long long ldv, int q,
                                                        double rcond, double* __restrict__ sigma) {
  __shared__ double red[JT / 32 + 1];
  __shared__ double smax;
  for (int i = 0; i < q; ++i) {
    double a = 0.0;
    for (int r = threadIdx.x; r < p; r += JT) a = fma(Xt[(long long)i * ldx + r], Xt[(long long)i * ldx + r], a);
    a = block_sum(a, red);
    if (threadIdx.x == 0) sigma[i] = sqrt(a);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < q; ++i) m = fmax(m, sigma[i]);
    smax = m;
  }
  __syncthreads();
  for (int i = 0; i < q; ++i) {
    const double si = sigma[i];
    const double d = (si > rcond * smax && si > 0.0) ? 1.0 / (si * si) : 0.0;
    for (int r = threadIdx.x; r < q; r += JT) Vt[(long long)i * ldv + r] *= d;
  }
}

int launch_pinv_scale(const double* Xt, long long ldx, int p, double* Vt, long long ldv, int q, double rcond,
                      double* sigma, cudaStream_t st) {
  if (q <= 0) return RS_OK;
  pinv_scale_kernel<<<1, JT, 0, st>>>(Xt, ldx, p, Vt, ldv, q, rcond, sigma);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

// out = max_j sum_i |A[i, j]| (1-norm), A row-major rows x cols.  One CTA.
__global__ void __launch_bounds__(JT) norm1_kernel(const double* __restrict__ A, long long lda, int rows, int cols,
                                                   double* __restrict__ out) {
  __shared__ double red[JT / 32 + 1];
  double best = 0.0;
  for (int c0 = 0; c0 < cols; c0 += JT) {
    const int c = c0 + threadIdx.x;
    double s = 0.0;
    if (c < cols)
      for (int r = 0; r < rows; ++r) s += fabs(A[(long long)r * lda + c]);
    best = fmax(best, s);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) best = fmax(best, __shfl_down_sync(0xffffffffu, best, off));
  if (lane == 0) red[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < JT / 32; ++w) m = fmax(m, red[w]);
    *out = m;
  }
}

int launch_norm1(const double* A, long long lda, int rows, int cols, double* out, cudaStream_t st) {
  if (rows < 0 || cols < 0) return RS_ERR_ARG;
  norm1_kernel<<<1, JT, 0, st>>>(A, lda, rows, cols, out);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

// Cholesky G = R^T R of a small SPD matrix (n <= 1024), in place: the upper
// triangle of G becomes R, the strict lower triangle is zeroed.  One CTA,
// right-looking by columns (the Gram matrix of a well-conditioned
// interpolation matrix in the pinv path, cur.py).  *status = 0, or j + 1 if
// pivot j is not positive.
// Right-looking Cholesky of a symmetric n x n (n <= 1024) matrix in place (upper factor R,
// G = R^T R), one CTA.  Per column: the scaled row j is staged in shared memory, then the
// 32 x 32 thread grid updates the trailing upper triangle row by row (no index division;
// the matrix, <= 8 MB, stays in L2).
__global__ void __launch_bounds__(1024) cholesky_kernel(double* __restrict__ G, long long ldg, int n,
                                                        int* __restrict__ status) {
  __shared__ double srow[1024];
  __shared__ int s_bad;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    double* gj = G + (long long)j * ldg;
    const double djj = gj[j];
    if (!(djj > 0.0)) {
      if (threadIdx.x == 0) s_bad = j + 1;
      break;  // uniform: every thread read the same diagonal
    }
    const double d = sqrt(djj);
    for (int c = j + threadIdx.x; c < n; c += blockDim.x) {
      const double v = c == j ? d : gj[c] / d;
      srow[c] = v;
      gj[c] = v;
    }
    __syncthreads();
    // G[r][c] -= R[j][r] R[j][c] for j < r <= c
    for (int r = j + 1 + ty; r < n; r += 32) {
      const double rr = srow[r];
      double* gr = G + (long long)r * ldg;
      for (int c = r + tx; c < n; c += 32) gr[c] -= rr * srow[c];
    }
    __syncthreads();
  }
  __syncthreads();
  for (int r = ty; r < n; r += 32)
    for (int c = tx; c < r; c += 32) G[(long long)r * ldg + c] = 0.0;
  if (threadIdx.x == 0) *status = s_bad;
}

// x <- T^-1 x for a small triangular T (n <= 1024) given by columns (column j at
// cols[j * ldc .. + n)), one CTA, one element of x per thread.  Column-oriented substitution
// in LAPACK dtrsv's order: x_j /= T_jj, then x_i -= T_ij x_j for the rows still to solve.
// One barrier per step (the pivot value alternates between two shared slots) and the next
// column's entry is loaded before the barrier, so a step costs one barrier plus one
// division on the diagonal thread.
__global__ void __launch_bounds__(1024) trsv_cols_kernel(const double* __restrict__ cols, long long ldc, int n,
                                                         int lower, int unit, double* __restrict__ x) {
  __shared__ double s_xj[2];
  const int i = threadIdx.x;
  double xi = i < n ? x[i] : 0.0;
  int j = lower ? 0 : n - 1;
  double c = i < n ? cols[(long long)j * ldc + i] : 0.0;
  for (int s = 0; s < n; ++s) {
    const int jn = lower ? j + 1 : j - 1;
    const double cn = (s + 1 < n && i < n) ? cols[(long long)jn * ldc + i] : 0.0;  // next column, early
    if (i == j) {
      if (!unit) xi = xi / c;
      s_xj[s & 1] = xi;
    }
    __syncthreads();
    const double xj = s_xj[s & 1];
    if (i < n && (lower ? i > j : i < j)) xi = xi - c * xj;
    j = jn;
    c = cn;
  }
  if (i < n) x[i] = xi;
}

int launch_trsv_cols(const double* cols, long long ldc, int n, int lower, int unit, double* x, cudaStream_t st) {
  if (n < 0 || n > 1024 || (n > 0 && ldc < n)) return RS_ERR_ARG;
  if (n == 0) return RS_OK;
  trsv_cols_kernel<<<1, ((n + 31) / 32) * 32, 0, st>>>(cols, ldc, n, lower, unit, x);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

int launch_cholesky(double* G, long long ldg, int n, int* status, cudaStream_t st) {
  if (n < 0 || n > 1024 || ldg < n) return RS_ERR_ARG;
  if (n == 0) return cudaMemsetAsync(status, 0, sizeof(int), st) == cudaSuccess ? RS_OK : RS_ERR_CUDA;
  cholesky_kernel<<<1, 1024, 0, st>>>(G, ldg, n, status);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

}  // namespace rs
