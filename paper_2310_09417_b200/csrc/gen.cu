// Device input generators: the synthetic matrices of
// the benchmark configs built in HBM instead of on the host.  Input
// generation, not the skeleton path -- but cfg5 (65536^2 fp64, 34 GB) cannot
// be built by the host in reasonable time, and every generator here is
// restated in numpy by the oracle (oracle/randskel_oracle.py) with the same
// rounding, so the device matrix is bit-identical to the host one.
//
//  * rs_uniform: numpy Generator(Philox(key=[seed, stream])).random(n),
//    C order -- word i of the Philox4x64-10 stream -> (w >> 11) * 2^-53.
//  * rs_hadamard_init / rs_fwht_rows: x <- rowscale (c H x), H the n x n
//    Walsh-Hadamard matrix acting on the row index (every column
//    independently), c = 1/sqrt(n).  The butterflies (a + b, a - b) run in
//    numpy's level order h = 1, 2, ..., n/2, so each element sees the same
//    roundings as the vectorised host loop.  Two passes over HBM: levels
//    h < n1 inside tiles of n1 consecutive rows, levels h >= n1 inside
//    tiles of the n2 = n / n1 rows {i0 + n1 t}; each tile is a 32-column
//    strip staged in shared memory.
//  * rs_kahan / rs_chan: `gen_kahan` / `gen_chan` (zoo.py:78-104).
//  * rs_axpy_cast: out = x + beta * y, fp64 or rounded to fp32 (the
//    low-rank-plus-noise recipe of cfg3).
#include "common.cuh"
#include "rskel_internal.h"

namespace rs {

namespace {

RS_DEV void philox4x64_10g(uint64_t c0, uint64_t k0, uint64_t k1, uint64_t out[4]) {
  uint64_t c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0);
    const uint64_t lo1 = 0xCA5A826395121157ull * c2, hi1 = __umul64hi(0xCA5A826395121157ull, c2);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

__global__ void uniform_kernel(uint64_t k0, uint64_t k1, long long n, double* __restrict__ out) {
  const long long blk = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // 4 words per Philox block
  const long long p0 = blk * 4;
  if (p0 >= n) return;
  uint64_t o[4];
  philox4x64_10g((uint64_t)blk + 1, k0, k1, o);  // numpy pre-increments the counter
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (p0 + q < n) out[p0 + q] = (double)(o[q] >> 11) * (1.0 / 9007199254740992.0);
}

// x[i, j] = (c * (-1)^popc(i & j)) * rowscale[i]  ==  rowscale (c H I), bit for bit
__global__ void hadamard_init_kernel(double* __restrict__ x, long long ld, int n, double c,
                                     const double* __restrict__ rowscale) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  for (int i = blockIdx.y; i < n; i += gridDim.y) {
    double v = (__popc((unsigned)(i & j)) & 1) ? -c : c;
    if (rowscale) v = v * rowscale[i];
    x[(long long)i * ld + j] = v;
  }
}

constexpr int FW_T = 256;
constexpr int FW_CB = 32;  // columns per tile (256-byte row segments)

// In-place levels h = h0, 2 h0, ..., < h1 over the `rows` staged rows of a
// tile (row r of the tile at smem[r * FW_CB + col]); the tile rows are the
// group's rows in index order, so level h pairs tile rows r and r + h / step.
__device__ void fwht_levels(double* t, int rows) {
  for (int h = 1; h < rows; h <<= 1) {
    for (int q = threadIdx.x; q < rows / 2 * FW_CB; q += FW_T) {
      const int col = q % FW_CB, pr = q / FW_CB;
      const int r = (pr / h) * 2 * h + (pr % h);
      const double a = t[r * FW_CB + col], b = t[(r + h) * FW_CB + col];
      t[r * FW_CB + col] = a + b;
      t[(r + h) * FW_CB + col] = a - b;
    }
    __syncthreads();
  }
}

// Tile = rows {base + stride * r : r < rows} x columns [j0, j0 + 32).
// finish: scale by c, then by rowscale (after the last level of the transform).
__global__ void __launch_bounds__(FW_T) fwht_pass_kernel(double* __restrict__ x, long long ld, int n, int rows,
                                                         int stride, int finish, double c,
                                                         const double* __restrict__ rowscale) {
  extern __shared__ double tile[];
  const int j0 = blockIdx.x * FW_CB;
  const int g = blockIdx.y;  // group: low pass base = g * rows, high pass base = g (stride n1)
  const long long base = stride == 1 ? (long long)g * rows : g;
  for (int q = threadIdx.x; q < rows * FW_CB; q += FW_T) {
    const int r = q / FW_CB, col = q % FW_CB;
    const int j = j0 + col;
    tile[q] = j < n ? x[(base + (long long)stride * r) * ld + j] : 0.0;
  }
  __syncthreads();
  fwht_levels(tile, rows);
  for (int q = threadIdx.x; q < rows * FW_CB; q += FW_T) {
    const int r = q / FW_CB, col = q % FW_CB;
    const int j = j0 + col;
    if (j >= n) continue;
    const long long i = base + (long long)stride * r;
    double v = tile[q];
    if (finish) {
      v = v * c;
      if (rowscale) v = v * rowscale[i];
    }
    x[i * ld + j] = v;
  }
}

__global__ void kahan_kernel(double* __restrict__ a, long long ld, int n, const double* __restrict__ rowpow,
                             double negphi) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  for (int i = blockIdx.y; i < n; i += gridDim.y) {
    const double k = j < i ? 0.0 : (j == i ? 1.0 : negphi);
    a[(long long)i * ld + j] = rowpow[i] * k;
  }
}

__global__ void chan_kernel(double* __restrict__ a, long long ld, int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  for (int i = blockIdx.y; i < n; i += gridDim.y)
    a[(long long)i * ld + j] = j == n - 1 ? 1.0 : (j == i ? 1.0 : (j < i ? -1.0 : 0.0));
}

__global__ void axpy_cast_kernel(const double* __restrict__ x, const double* __restrict__ y, double beta,
                                 long long n, double* __restrict__ out64, float* __restrict__ out32) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double v = x[i] + beta * y[i];  // numpy: low + (eta * noise), two roundings
    if (out32) out32[i] = (float)v;
    else out64[i] = v;
  }
}

int ok_or_cuda() { return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA; }

}  // namespace

int launch_uniform(uint64_t k0, uint64_t k1, long long n, double* out, cudaStream_t st) {
  if (n < 0) return RS_ERR_ARG;
  if (n == 0) return RS_OK;
  const long long blocks = (n + 3) / 4;
  uniform_kernel<<<(unsigned)((blocks + 255) / 256), 256, 0, st>>>(k0, k1, n, out);
  count_launch(1);
  return ok_or_cuda();
}

int launch_hadamard_init(double* x, long long ld, int n, double c, const double* rowscale, cudaStream_t st) {
  if (n <= 0 || (n & (n - 1)) || ld < n) return RS_ERR_ARG;
  hadamard_init_kernel<<<dim3((n + 255) / 256, n < 8192 ? n : 8192), 256, 0, st>>>(x, ld, n, c, rowscale);
  count_launch(1);
  return ok_or_cuda();
}

int launch_fwht_rows(double* x, long long ld, int n, double c, const double* rowscale, cudaStream_t st) {
  if (n <= 0 || (n & (n - 1)) || ld < n || n > (1 << 17)) return RS_ERR_ARG;
  const int n1 = n < 256 ? n : 256, n2 = n / n1;
  const dim3 cols((n + FW_CB - 1) / FW_CB);
  const size_t s1 = sizeof(double) * n1 * FW_CB, s2 = sizeof(double) * n2 * FW_CB;
  cudaFuncSetAttribute(fwht_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(s1 > s2 ? s1 : s2));
  // low levels: n2 groups of n1 consecutive rows
  fwht_pass_kernel<<<dim3(cols.x, n2), FW_T, s1, st>>>(x, ld, n, n1, 1, n2 == 1, c, rowscale);
  count_launch(1);
  if (n2 > 1) {  // high levels: n1 groups of the rows {i0 + n1 t}
    fwht_pass_kernel<<<dim3(cols.x, n1), FW_T, s2, st>>>(x, ld, n, n2, n1, 1, c, rowscale);
    count_launch(1);
  }
  return ok_or_cuda();
}

int launch_kahan(double* a, long long ld, int n, const double* rowpow, double negphi, cudaStream_t st) {
  if (n <= 0 || ld < n) return RS_ERR_ARG;
  kahan_kernel<<<dim3((n + 255) / 256, n < 8192 ? n : 8192), 256, 0, st>>>(a, ld, n, rowpow, negphi);
  count_launch(1);
  return ok_or_cuda();
}

int launch_chan(double* a, long long ld, int n, cudaStream_t st) {
  if (n <= 0 || ld < n) return RS_ERR_ARG;
  chan_kernel<<<dim3((n + 255) / 256, n < 8192 ? n : 8192), 256, 0, st>>>(a, ld, n);
  count_launch(1);
  return ok_or_cuda();
}

int launch_axpy_cast(const double* x, const double* y, double beta, long long n, double* out64, float* out32,
                     cudaStream_t st) {
  if (n < 0 || (out64 == nullptr) == (out32 == nullptr)) return RS_ERR_ARG;
  if (n == 0) return RS_OK;
  axpy_cast_kernel<<<148 * 8, 256, 0, st>>>(x, y, beta, n, out64, out32);
  count_launch(1);
  return ok_or_cuda();
}

}  // namespace rs
