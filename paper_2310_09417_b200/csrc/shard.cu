// Index bookkeeping of the column-sharded adaptive loop.
//
// Rank g owns the contiguous candidate rows [lo, hi) of the matrix whose rows
// are the candidates (A.T for the column ID: A is column-sharded).  The
// position order `perm` is replicated -- every rank runs the same panel LUPP
// on the same all-gathered Schur block -- while the interpolation rows T_g
// of the rank's own remaining candidates stay local, compact, in position
// order.  One single-CTA scan per block turns (perm, k) into the maps the
// block's gathers, GEMMs and scatters need.
#include "common.cuh"
#include "rskel_internal.h"

namespace rs {

constexpr int MAP_T = 1024;

RS_DEV bool owned(int64_t c, long long lo, long long hi) { return c >= lo && c < hi; }

// Block-wide exclusive scan of one int per thread (MAP_T threads).
RS_DEV int block_exclusive_scan(int v, int* total) {
  __shared__ int warp_sum[MAP_T / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = warp_sum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    warp_sum[lane] = w;  // inclusive
  }
  __syncthreads();
  const int before = (wid > 0 ? warp_sum[wid - 1] : 0) + x - v;
  *total = warp_sum[MAP_T / 32 - 1];
  __syncthreads();
  return before;
}

__global__ void __launch_bounds__(MAP_T) shard_maps_kernel(
    const int64_t* __restrict__ perm, int m, int k, long long lo, long long hi,
    const int64_t* __restrict__ lrow_old, const int64_t* __restrict__ sub, int k_old, int nc,
    int64_t* __restrict__ lrow, int64_t* __restrict__ loc, int64_t* __restrict__ spos,
    int64_t* __restrict__ src_row, int64_t* __restrict__ wsrc, int64_t* __restrict__ tp_src,
    int64_t* __restrict__ ytop_src, int* __restrict__ count, int pad_to) {
  const int t = threadIdx.x;
  for (int p = t; p < k; p += MAP_T) {
    const int64_t c = perm[p];
    ytop_src[p] = owned(c, lo, hi) ? c - lo : -1;
    lrow[p] = -1;
  }
  if (sub != nullptr) {
    for (int j = t; j < nc; j += MAP_T) tp_src[j] = lrow_old[k_old + sub[j]];
  }
  const int R = m - k;
  const int per = (R + MAP_T - 1) / MAP_T;
  const int a = k + t * per, b = min(m, a + per);
  int mine = 0;
  for (int p = a; p < b; ++p) mine += owned(perm[p], lo, hi) ? 1 : 0;
  int total;
  int r = block_exclusive_scan(mine, &total);
  for (int p = a; p < b; ++p) {
    const int64_t c = perm[p];
    if (!owned(c, lo, hi)) {
      lrow[p] = -1;
      continue;
    }
    lrow[p] = r;
    loc[r] = c - lo;
    spos[r] = p - k;
    if (sub != nullptr) {
      const int64_t j = sub[p - k_old];
      src_row[r] = lrow_old[k_old + j];
      wsrc[r] = j;
    }
    ++r;
  }
  // rows [total, pad_to): harmless entries for launches sized by an upper
  // bound of the row count (valid gather indices, no scatter)
  for (int r2 = total + t; r2 < pad_to; r2 += MAP_T) {
    loc[r2] = 0;
    spos[r2] = -1;
    if (sub != nullptr) {
      src_row[r2] = 0;
      wsrc[r2] = 0;
    }
  }
  if (t == 0) *count = total;
}

int launch_shard_maps(const int64_t* perm, int m, int k, long long lo, long long hi, const int64_t* lrow_old,
                      const int64_t* sub, int k_old, int nc, int64_t* lrow, int64_t* loc, int64_t* spos,
                      int64_t* src_row, int64_t* wsrc, int64_t* tp_src, int64_t* ytop_src, int* count,
                      int pad_to, cudaStream_t st) {
  if (m < 0 || k < 0 || k > m || lo > hi) return RS_ERR_ARG;
  if (sub != nullptr && (lrow_old == nullptr || src_row == nullptr || wsrc == nullptr || tp_src == nullptr ||
                         k_old < 0 || nc < 0 || k_old + nc != k))
    return RS_ERR_ARG;
  shard_maps_kernel<<<1, MAP_T, 0, st>>>(perm, m, k, lo, hi, lrow_old, sub, k_old, nc, lrow, loc, spos, src_row,
                                         wsrc, tp_src, ytop_src, count, pad_to);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

// *out_max = max over ranks g of #{p >= k : bounds[g] <= perm[p] < bounds[g+1]}:
// every rank's remaining-candidate count from the replicated perm, so all ranks
// agree on the padding of the next all-gather without a collective.
__global__ void __launch_bounds__(MAP_T) shard_max_count_kernel(const int64_t* __restrict__ perm, int m, int k,
                                                                const int64_t* __restrict__ bounds, int world,
                                                                int* __restrict__ out_max) {
  __shared__ int hist[64];
  __shared__ long long bnd[65];
  for (int g = threadIdx.x; g < world; g += MAP_T) hist[g] = 0;
  for (int g = threadIdx.x; g <= world; g += MAP_T) bnd[g] = bounds[g];
  __syncthreads();
  for (int p = k + threadIdx.x; p < m; p += MAP_T) {
    const long long c = perm[p];
    int lo = 0, hi = world;  // largest g with bnd[g] <= c
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (bnd[mid] <= c) lo = mid;
      else hi = mid;
    }
    atomicAdd(hist + lo, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int mx = 0;
    for (int g = 0; g < world; ++g) mx = max(mx, hist[g]);
    *out_max = mx;
  }
}

int launch_shard_max_count(const int64_t* perm, int m, int k, const int64_t* bounds, int world, int* out_max,
                           cudaStream_t st) {
  if (m < 0 || k < 0 || k > m || world < 1 || world > 64) return RS_ERR_ARG;
  shard_max_count_kernel<<<1, MAP_T, 0, st>>>(perm, m, k, bounds, world, out_max);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

// dst[idx[i], :] = src[i, :] for idx[i] >= 0.
__global__ void scatter_rows_kernel(const double* __restrict__ src, long long lds, const int64_t* __restrict__ idx,
                                    int nrows, int ncols, double* __restrict__ dst, long long ldd) {
  for (int i = blockIdx.x; i < nrows; i += gridDim.x) {
    const long long r = idx[i];
    if (r < 0) continue;
    const double* s = src + (long long)i * lds;
    double* d = dst + r * ldd;
    for (int c = threadIdx.x; c < ncols; c += blockDim.x) d[c] = s[c];
  }
}

int launch_scatter_rows(const double* src, long long lds, const int64_t* idx, int nrows, int ncols, double* dst,
                        long long ldd, cudaStream_t st) {
  if (nrows < 0 || ncols < 0 || idx == nullptr) return RS_ERR_ARG;
  if (nrows == 0 || ncols == 0) return RS_OK;
  const int threads = ncols >= 256 ? 256 : ((ncols + 31) / 32) * 32;
  const int grid = nrows < 148 * 16 ? nrows : 148 * 16;
  scatter_rows_kernel<<<grid, threads, 0, st>>>(src, lds, idx, nrows, ncols, dst, ldd);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

// Identity rows of the local W block: W_g[perm[p] - lo, p] = 1 for owned skeletons p < k.
__global__ void shard_identity_kernel(const int64_t* __restrict__ perm, int k, long long lo, long long hi,
                                      double* __restrict__ W, long long ldw) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= k) return;
  const int64_t c = perm[p];
  if (owned(c, lo, hi)) W[(c - lo) * ldw + p] = 1.0;
}

int launch_scatter_interp_local(const double* T, long long ldt, const int64_t* perm, int k, const int64_t* loc,
                                int r, long long lo, long long hi, double* W, long long ldw, cudaStream_t st) {
  if (k < 0 || r < 0 || lo > hi || ldw < k) return RS_ERR_ARG;
  const long long mg = hi - lo;
  if (mg == 0 || k == 0) return RS_OK;
  if (cudaMemset2DAsync(W, (size_t)ldw * 8, 0, (size_t)k * 8, (size_t)mg, st) != cudaSuccess) return RS_ERR_CUDA;
  shard_identity_kernel<<<(k + 255) / 256, 256, 0, st>>>(perm, k, lo, hi, W, ldw);
  count_launch(1);
  if (cudaGetLastError() != cudaSuccess) return RS_ERR_CUDA;
  return launch_scatter_rows(T, ldt, loc, r, k, W, ldw, st);
}

}  // namespace rs
