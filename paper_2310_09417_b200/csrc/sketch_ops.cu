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

}  // namespace rs
