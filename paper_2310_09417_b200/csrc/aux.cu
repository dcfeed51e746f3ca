// Bandwidth-bound helper kernels of the skeleton path: row gathers, the
// deterministic Frobenius reduction, the small triangular inverse used for
// W_hat = L_r L_1^{-1}, the permutation update and the interpolation-matrix
// scatter (`skeleton.py:176-182`).
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "rskel_internal.h"


namespace rs {

// ---- row gathers ----------------------------------------------------------
// dst[i, c] = src[idx[i], c] (idx == nullptr: identity; idx[i] < 0: a zero row -- the
// owner-masked gathers of the sharded loop), row-major.  Rows are copied with 16-byte vector
// loads and stores whenever every source and destination row starts on a 16-byte boundary
// (base pointers aligned and both leading dimensions even): a warp moves 512 contiguous
// bytes per instruction, and a row wider than one CTA's span is split over CTAs (grid.x),
// so long skeleton rows (`a[row_idx]`, 16384 doubles) use the whole GPU.  Streaming loads
// bypass L1 (ld.global.nc.L1::no_allocate): every byte is read once.
constexpr int GR_THREADS = 256;

RS_DEV double2 ldg_stream2(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// one CTA per (column span, row); VEC = 2 doubles per access when aligned
template <int VEC>
__global__ void __launch_bounds__(GR_THREADS) gather_rows_vec_kernel(
    const double* __restrict__ src, long long lds, const int64_t* __restrict__ idx, int nrows, int ncols,
    double* __restrict__ dst, long long ldd, int span) {
  const int c0 = blockIdx.x * span, c1 = min(ncols, c0 + span);
  for (int i = blockIdx.y; i < nrows; i += gridDim.y) {
    const long long r = idx ? idx[i] : i;
    double* d = dst + (long long)i * ldd;
    if (r < 0) {
      for (int c = c0 + threadIdx.x; c < c1; c += GR_THREADS) d[c] = 0.0;
      continue;
    }
    const double* s = src + r * lds;
    if (VEC == 2) {
      // 4 independent 16-byte loads in flight per thread
      int c = c0 + threadIdx.x * 2;
      for (; c + 3 * GR_THREADS * 2 + 1 < c1; c += 4 * GR_THREADS * 2) {
        double2 v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = ldg_stream2(reinterpret_cast<const double2*>(s + c + q * GR_THREADS * 2));
#pragma unroll
        for (int q = 0; q < 4; ++q) *reinterpret_cast<double2*>(d + c + q * GR_THREADS * 2) = v[q];
      }
      for (; c < c1; c += GR_THREADS * 2) {
        if (c + 1 < c1) *reinterpret_cast<double2*>(d + c) = ldg_stream2(reinterpret_cast<const double2*>(s + c));
        else d[c] = s[c];
      }
    } else {
      for (int c = c0 + threadIdx.x; c < c1; c += GR_THREADS) d[c] = s[c];
    }
  }
}

// Narrow rows (the 64-column sketch blocks Y[perm]): one warp per row, 16 bytes per lane.
__global__ void __launch_bounds__(GR_THREADS) gather_rows_narrow_kernel(
    const double* __restrict__ src, long long lds, const int64_t* __restrict__ idx, int nrows, int ncols,
    double* __restrict__ dst, long long ldd) {
  const int lane = threadIdx.x & 31;
  const int wid = blockIdx.x * (GR_THREADS / 32) + (threadIdx.x >> 5);
  const int nw = gridDim.x * (GR_THREADS / 32);
  for (int i = wid; i < nrows; i += nw) {
    const long long r = idx ? idx[i] : i;
    double* d = dst + (long long)i * ldd;
    const double* s = r >= 0 ? src + r * lds : nullptr;
    for (int c = 2 * lane; c < ncols; c += 64) {
      double2 v = make_double2(0.0, 0.0);
      if (s) {
        if (c + 1 < ncols) v = ldg_stream2(reinterpret_cast<const double2*>(s + c));
        else v.x = s[c];
      }
      if (c + 1 < ncols) *reinterpret_cast<double2*>(d + c) = v;
      else d[c] = v.x;
    }
  }
}

int launch_gather_rows(const double* src, long long lds, const int64_t* idx, int nrows, int ncols,
                       double* dst, long long ldd, cudaStream_t st) {
  if (nrows < 0 || ncols < 0) return RS_ERR_ARG;
  if (nrows == 0 || ncols == 0) return RS_OK;
  const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0 &&
                   (lds % 2) == 0 && (ldd % 2) == 0;
  if (vec && ncols <= 256) {
    const int warps = GR_THREADS / 32;
    const int grid = std::min((nrows + warps - 1) / warps, 148 * 16);
    gather_rows_narrow_kernel<<<grid, GR_THREADS, 0, st>>>(src, lds, idx, nrows, ncols, dst, ldd);
  } else {
    // column spans of 8 accesses per thread; rows over grid.y, enough CTAs to fill the GPU
    const int span = GR_THREADS * (vec ? 2 : 1) * 8;
    const int gx = (ncols + span - 1) / span;
    const int gy = std::min(nrows, std::min(65535, std::max(1, 148 * 16 / gx)));
    if (vec)
      gather_rows_vec_kernel<2><<<dim3(gx, gy), GR_THREADS, 0, st>>>(src, lds, idx, nrows, ncols, dst, ldd, span);
    else
      gather_rows_vec_kernel<1><<<dim3(gx, gy), GR_THREADS, 0, st>>>(src, lds, idx, nrows, ncols, dst, ldd, span);
  }
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

// ---- deterministic sum of squares ---------------------------------------
// Stage 1: CTA b reduces rows [b*rows_per, ...) in a fixed order; stage 2 adds
// the partials in CTA order.  The result is independent of scheduling.
constexpr int SS_THREADS = 256;
constexpr int SS_MAX_CTAS = 1024;

__global__ void sumsq_stage1(const double* __restrict__ X, long long ldx, int R, int w, int rows_per,
                             double* __restrict__ partial) {
  __shared__ double red[SS_THREADS];
  int r0 = blockIdx.x * rows_per, r1 = min(R, r0 + rows_per);
  double acc = 0.0;
  long long n = (long long)(r1 > r0 ? r1 - r0 : 0) * w;
  // thread t takes elements t, t + 256, ... of the CTA's rows (row-major order), in that order
  if (ldx == w) {  // contiguous rows: the element index is the offset
    const double* base = X + (long long)r0 * ldx;
    for (long long e = threadIdx.x; e < n; e += SS_THREADS) {
      const double v = base[e];
      acc = fma(v, v, acc);
    }
  } else {  // (row, column) advanced by 256 elements per step without a division
    const int q = SS_THREADS / w, rq = SS_THREADS % w;
    int i = threadIdx.x / w, c = threadIdx.x % w;
    for (long long e = threadIdx.x; e < n; e += SS_THREADS) {
      const double v = X[(long long)(r0 + i) * ldx + c];
      acc = fma(v, v, acc);
      i += q;
      c += rq;
      if (c >= w) {
        c -= w;
        ++i;
      }
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = SS_THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void sumsq_stage2(const double* __restrict__ partial, int n, double* __restrict__ out) {
  __shared__ double red[SS_THREADS];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += SS_THREADS) acc += partial[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = SS_THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

size_t sumsq_workspace_bytes() { return SS_MAX_CTAS * sizeof(double); }

int launch_sumsq(const double* X, long long ldx, int R, int w, double* partial_ws, double* out,
                 cudaStream_t st) {
  if (R < 0 || w < 0) return RS_ERR_ARG;
  if (R == 0 || w == 0) {
    cudaMemsetAsync(out, 0, sizeof(double), st);
    return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
  }
  int ctas = (R + 63) / 64;
  if (ctas > 296) ctas = 296;
  int rows_per = (R + ctas - 1) / ctas;
  ctas = (R + rows_per - 1) / rows_per;
  sumsq_stage1<<<ctas, SS_THREADS, 0, st>>>(X, ldx, R, w, rows_per, partial_ws);
  count_launch(1);
  sumsq_stage2<<<1, SS_THREADS, 0, st>>>(partial_ws, ctas, out);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

// ---- small triangular inverse (n <= 64) ---------------------------------
// Element (i, j) of the input triangle is T[ridx(i) * rs + j * cs].  Thread c
// computes column c of the inverse by substitution; out is n x n row-major.
constexpr int TI_MAX = 64;
// Fully unrolled substitution: thread c keeps column c of the inverse in
// registers (x[0..63]); L[i][q] are shared-memory broadcasts.  The problem is
// padded to 64 (identity outside n x n), 4 partial sums shorten the FMA chain.
template <bool LOWER>
__global__ void __launch_bounds__(TI_MAX) trinv_kernel(const double* __restrict__ T, long long rs_,
                                                       long long cs_, const int64_t* __restrict__ ridx,
                                                       int n, int unit, double* __restrict__ out,
                                                       long long ldo) {
  __shared__ double L[TI_MAX][TI_MAX];
  for (int e = threadIdx.x; e < TI_MAX * TI_MAX; e += blockDim.x) {
    const int i = e / TI_MAX, j = e - i * TI_MAX;
    double v;
    if (i < n && j < n) {
      const long long r = ridx ? ridx[i] : i;
      v = T[r * rs_ + (long long)j * cs_];
    } else {
      v = (i == j) ? 1.0 : 0.0;
    }
    L[i][j] = v;
  }
  __syncthreads();
  const int c = threadIdx.x;
  double x[TI_MAX];
  if (LOWER) {
#pragma unroll
    for (int i = 0; i < TI_MAX; ++i) {
      double s0 = (i == c) ? 1.0 : 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int q = 0; q < i; ++q) {
        const double lq = L[i][q];
        if ((q & 3) == 0) s0 -= lq * x[q];
        else if ((q & 3) == 1) s1 -= lq * x[q];
        else if ((q & 3) == 2) s2 -= lq * x[q];
        else s3 -= lq * x[q];
      }
      const double s = (s0 + s1) + (s2 + s3);
      x[i] = unit ? s : s / L[i][i];
    }
  } else {
#pragma unroll
    for (int i = TI_MAX - 1; i >= 0; --i) {
      double s0 = (i == c) ? 1.0 : 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int q = i + 1; q < TI_MAX; ++q) {
        const double lq = L[i][q];
        if ((q & 3) == 0) s0 -= lq * x[q];
        else if ((q & 3) == 1) s1 -= lq * x[q];
        else if ((q & 3) == 2) s2 -= lq * x[q];
        else s3 -= lq * x[q];
      }
      const double s = (s0 + s1) + (s2 + s3);
      x[i] = unit ? s : s / L[i][i];
    }
  }
  if (c < n) {
#pragma unroll
    for (int i = 0; i < TI_MAX; ++i)
      if (i < n) out[(long long)i * ldo + c] = x[i];
  }
}

int launch_trinv(const double* T, long long rs_, long long cs_, const int64_t* ridx, int n, int lower,
                 int unit, double* out, long long ldo, cudaStream_t st) {
  if (n < 0 || n > TI_MAX) return RS_ERR_ARG;
  if (n == 0) return RS_OK;
  if (lower) trinv_kernel<true><<<1, TI_MAX, 0, st>>>(T, rs_, cs_, ridx, n, unit, out, ldo);
  else trinv_kernel<false><<<1, TI_MAX, 0, st>>>(T, rs_, cs_, ridx, n, unit, out, ldo);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

// ---- W_hat = L_r L_1^{-1} by row-parallel substitution ----------------------
// out[i, :nc] solves y L1 = x with x = S[ridx[i], :nc] and L1 the unit lower
// triangle of the pivot rows S[sub[a], b] (b < a < nc): one row per thread,
// right-looking (y_a final once every later column has been folded in, then
// x_j -= y_a L1[a][j] for all j < a -- 63 independent FMAs per step), L1 as
// shared-memory broadcasts.  Replaces the trinv + GEMM pair of the absorb.
constexpr int WH_T = 128;
constexpr int WH_G = 4;  // lanes per row: lane g of a group owns x[j], j = g mod 4

// Four lanes per row (four times the warps of one row per thread, which left ~4 warps per
// SM at R = 20000): step a takes y_a = x[a] from its owner lane by shuffle, then every lane
// folds it into its own x[j], j < a.  Each x[j] sees the same fma sequence in the same order
// as a one-row-per-thread substitution, so the bits are unchanged.
__global__ void __launch_bounds__(WH_T) what_kernel(const double* __restrict__ S, long long lds,
                                                    const int64_t* __restrict__ sub, int nc,
                                                    const int64_t* __restrict__ ridx, int R,
                                                    double* __restrict__ out, long long ldo) {
  __shared__ double L1[TI_MAX][TI_MAX + 1];
  for (int e = threadIdx.x; e < TI_MAX * TI_MAX; e += blockDim.x) {
    const int a = e / TI_MAX, b = e - a * TI_MAX;
    L1[a][b] = (a < nc && b < a) ? S[sub[a] * lds + b] : 0.0;
  }
  __syncthreads();
  constexpr int NJ = TI_MAX / WH_G;
  const int lane = threadIdx.x & 31, g = lane & (WH_G - 1);
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) / WH_G;
  const bool live = i < R;  // every lane takes part in the shuffles
  const double* src = S + (live ? ridx[i] : 0) * lds;
  double x[NJ];
#pragma unroll
  for (int jj = 0; jj < NJ; ++jj) {
    const int j = jj * WH_G + g;
    x[jj] = (live && j < nc) ? src[j] : 0.0;
  }
#pragma unroll
  for (int a = TI_MAX - 1; a > 0; --a) {
    const double ya = __shfl_sync(0xffffffffu, x[a / WH_G], (lane & ~(WH_G - 1)) | (a % WH_G), 32);
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) {
      const int j = jj * WH_G + g;
      if (jj * WH_G < a && j < a) x[jj] = fma(-ya, L1[a][j], x[jj]);
    }
  }
  if (!live) return;
  double* dst = out + (long long)i * ldo;
#pragma unroll
  for (int jj = 0; jj < NJ; ++jj) {
    const int j = jj * WH_G + g;
    if (j < nc) dst[j] = x[jj];
  }
}

int launch_what(const double* S, long long lds, const int64_t* sub, int nc, const int64_t* ridx, int R, double* out,
                long long ldo, cudaStream_t st) {
  if (nc < 0 || nc > TI_MAX || R < 0 || ldo < nc) return RS_ERR_ARG;
  if (nc == 0 || R == 0) return RS_OK;
  what_kernel<<<(unsigned)(((long long)R * WH_G + WH_T - 1) / WH_T), WH_T, 0, st>>>(S, lds, sub, nc, ridx, R, out,
                                                                                  ldo);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

// ---- permutation update: perm'[:k] = perm[:k]; perm'[k+i] = perm[k + sub[i]] ----
__global__ void perm_update_kernel(const int64_t* __restrict__ perm, int64_t* __restrict__ perm_new,
                                   int m, int k, const int64_t* __restrict__ sub) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  perm_new[i] = (i < k) ? perm[i] : perm[k + sub[i - k]];
}

int launch_perm_update(const int64_t* perm, int64_t* perm_new, int m, int k, const int64_t* sub,
                       cudaStream_t st) {
  if (m < 0 || k < 0 || k > m) return RS_ERR_ARG;
  if (m == 0) return RS_OK;
  perm_update_kernel<<<(m + 255) / 256, 256, 0, st>>>(perm, perm_new, m, k, sub);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

__global__ void iota_kernel(int64_t* p, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = i;
}

int launch_iota(int64_t* p, int n, cudaStream_t st) {
  if (n <= 0) return n == 0 ? RS_OK : RS_ERR_ARG;
  iota_kernel<<<(n + 255) / 256, 256, 0, st>>>(p, n);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

// ---- W[perm[p]] = e_p (p < k), W[perm[p]] = T[p - k] (p >= k) ---------------
// One CTA row-sweep per position; writes every W element exactly once.
__global__ void scatter_interp_kernel(const double* __restrict__ T, long long ldt,
                                      const int64_t* __restrict__ perm, int m, int k,
                                      double* __restrict__ W, long long ldw) {
  for (int p = blockIdx.x; p < m; p += gridDim.x) {
    double* wr = W + perm[p] * ldw;
    if (p < k) {
      for (int c = threadIdx.x; c < k; c += blockDim.x) wr[c] = (c == p) ? 1.0 : 0.0;
    } else {
      const double* tr = T + (long long)(p - k) * ldt;
      for (int c = threadIdx.x; c < k; c += blockDim.x) wr[c] = tr[c];
    }
  }
}

int launch_scatter_interp(const double* T, long long ldt, const int64_t* perm, int m, int k, double* W,
                          long long ldw, cudaStream_t st) {
  if (m < 0 || k < 0 || k > m) return RS_ERR_ARG;
  if (m == 0 || k == 0) return RS_OK;
  int threads = k >= 256 ? 256 : ((k + 31) / 32) * 32;
  int grid = m < 148 * 32 ? m : 148 * 32;
  scatter_interp_kernel<<<grid, threads, 0, st>>>(T, ldt, perm, m, k, W, ldw);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

}  // namespace rs

namespace rs {

// ---- dst (cols x rows) = src (rows x cols)^T, 32x32 smem tiles ------------
__global__ void transpose_kernel(const double* __restrict__ src, long long lds, int rows, int cols,
                                 double* __restrict__ dst, long long ldd) {
  __shared__ double tile[32][33];
  int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += 8) {
    int i = by + y, j = bx + threadIdx.x;
    if (i < rows && j < cols) tile[y][threadIdx.x] = src[(long long)i * lds + j];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) {
    int j = bx + y, i = by + threadIdx.x;
    if (i < rows && j < cols) dst[(long long)j * ldd + i] = tile[threadIdx.x][y];
  }
}

int launch_transpose(const double* src, long long lds, int rows, int cols, double* dst, long long ldd,
                     cudaStream_t st) {
  if (rows < 0 || cols < 0) return RS_ERR_ARG;
  if (rows == 0 || cols == 0) return RS_OK;
  dim3 grid((cols + 31) / 32, (rows + 31) / 32);
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(src, lds, rows, cols, dst, ldd);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

}  // namespace rs

namespace rs {

// dst[i, j] = src(r(i), c(j)) with src element (r, c) at src[r * rs + c * cs];
// r(i) = ridx ? ridx[i] : i, c(j) = cidx ? cidx[j] : j.  Skeleton gathers
// a[I], a[:, J], a[ix_(I, J)] for either input layout (skeleton.py:619,639-645).
__global__ void gather2d_kernel(const double* __restrict__ src, long long rs_, long long cs_,
                                const int64_t* __restrict__ ridx, int nr, const int64_t* __restrict__ cidx,
                                int nc, double* __restrict__ dst, long long ldd) {
  for (int i = blockIdx.x; i < nr; i += gridDim.x) {
    const long long r = ridx ? ridx[i] : i;
    const double* s = src + r * rs_;
    double* d = dst + (long long)i * ldd;
    for (int j = threadIdx.x; j < nc; j += blockDim.x) {
      const long long c = cidx ? cidx[j] : j;
      d[j] = s[c * cs_];
    }
  }
}

// Column-contiguous source (rs == 1, a column-major a): the gather is a transpose.  32 x 32
// tiles through shared memory: reads run down the source columns (coalesced along i when
// ridx is absent or local), writes run along the destination rows.
__global__ void __launch_bounds__(256) gather2d_colmajor_kernel(
    const double* __restrict__ src, long long cs_, const int64_t* __restrict__ ridx, int nr,
    const int64_t* __restrict__ cidx, int nc, double* __restrict__ dst, long long ldd) {
  __shared__ double tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  const long long r = i0 + tx < nr ? (ridx ? ridx[i0 + tx] : i0 + tx) : -1;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int j = j0 + ty + 8 * q;
    double v = 0.0;
    if (r >= 0 && j < nc) {
      const long long c = cidx ? cidx[j] : j;
      v = src[r + c * cs_];
    }
    tile[ty + 8 * q][tx] = v;  // tile[j][i]
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = i0 + ty + 8 * q, j = j0 + tx;
    if (i < nr && j < nc) dst[(long long)i * ldd + j] = tile[tx][ty + 8 * q];
  }
}

// dst = a[ridx][:, cidx] in three shapes: whole rows of row-contiguous data (the vectorised
// row gather), a column-contiguous source (the tiled transpose), and scattered columns of
// row-contiguous data (`a[:, col_idx]` of a row-major a: one 8-byte element per index,
// inherent to the layout).
int launch_gather2d(const double* src, long long rs_, long long cs_, const int64_t* ridx, int nr,
                    const int64_t* cidx, int nc, double* dst, long long ldd, cudaStream_t st) {
  if (nr < 0 || nc < 0) return RS_ERR_ARG;
  if (nr == 0 || nc == 0) return RS_OK;
  if (cs_ == 1 && cidx == nullptr) return launch_gather_rows(src, rs_, ridx, nr, nc, dst, ldd, st);
  if (rs_ == 1 && nr > 1 && (nc + 31) / 32 <= 65535) {
    gather2d_colmajor_kernel<<<dim3((nr + 31) / 32, (nc + 31) / 32), 256, 0, st>>>(src, cs_, ridx, nr, cidx, nc,
                                                                                 dst, ldd);
  } else {
    int threads = nc >= 256 ? 256 : ((nc + 31) / 32) * 32;
    int grid = nr < 148 * 16 ? nr : 148 * 16;
    gather2d_kernel<<<grid, threads, 0, st>>>(src, rs_, cs_, ridx, nr, cidx, nc, dst, ldd);
  }
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

}  // namespace rs
