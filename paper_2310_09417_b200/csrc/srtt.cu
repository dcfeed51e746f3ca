// SRTT embedding applied as a fast transform, the reference's `SrttSketch.apply`
// (`sketching.py:147-155`):
//
//   c = DCT-II_ortho(a[:, perm]) along each row (length n),  c *= signs,  y = scale * c[:, cols]
//
// Makhoul's reordering turns a length-n DCT-II into one length-n real FFT:
//   v[q] = x[2q] (q < ceil(n/2)),  v[n-1-q] = x[2q+1],   V = FFT(v),
//   DCT2[k] = 2 Re(exp(-i pi k / (2n)) V[k]),  ortho scale sqrt(1/(4n)) at k = 0, sqrt(1/(2n)) else,
// and V[k] = conj(V[n-k]) above n/2 (real input).  Per batch of rows:
//   1. srtt_gather_*: v = the reordered, permuted row (one CTA per row, the row staged in shared
//      memory when it fits, so A is read once and coalesced);
//   2. cuFFT D2Z, batched (a plain library FFT, as cuBLAS would be for a GEMM; plans cached);
//   3. srtt_select_kernel: only the ell sampled outputs are formed.
// O(m n log n) work and ~4 passes of m n doubles over HBM, against O(m n ell) for the dense
// embedding: the dense tensor-core product is faster for small ell, this for large ell.
#include <cufft.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "rskel_internal.h"

namespace rs {

namespace {
constexpr int SRTT_STAGE_MAX = 24576;  // doubles of a row staged in shared memory (192 KB)

RS_DEV int makhoul_src(int q, int n) { return q < (n + 1) / 2 ? 2 * q : 2 * (n - 1 - q) + 1; }

struct PlanKey {
  int dev, n, batch;
};
struct PlanSlot {
  PlanKey key;
  cufftHandle plan;
  bool used;
};
PlanSlot g_plans[16];
int g_next = 0;
std::mutex g_mu;

int get_plan(int n, int batch, cufftHandle* out) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& s : g_plans)
    if (s.used && s.key.dev == dev && s.key.n == n && s.key.batch == batch) {
      *out = s.plan;
      return RS_OK;
    }
  PlanSlot& s = g_plans[g_next];
  g_next = (g_next + 1) % 16;
  if (s.used) cufftDestroy(s.plan);
  s.used = false;
  int nn = n, inembed = n, onembed = n / 2 + 1;
  const cufftResult r = cufftPlanMany(&s.plan, 1, &nn, &inembed, 1, n, &onembed, 1, n / 2 + 1, CUFFT_D2Z, batch);
  if (r != CUFFT_SUCCESS) {
    if (getenv("RS_SRTT_DEBUG")) fprintf(stderr, "srtt: cufftPlanMany(n=%d, batch=%d) = %d\n", n, batch, (int)r);
    return RS_ERR_CUDA;
  }
  s.key = {dev, n, batch};
  s.used = true;
  *out = s.plan;
  return RS_OK;
}
}  // namespace

// src[q] = perm[makhoul_src(q)]: the column of A that lands at FFT input position q
__global__ void srtt_index_kernel(int n, const int64_t* __restrict__ perm, int* __restrict__ src) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) src[q] = (int)perm[makhoul_src(q, n)];
}

// one 1024-thread CTA per row: the row staged in shared memory with 16-byte loads (all
// in flight at once), then written out in FFT-input order (coalesced)
template <bool VEC>
__global__ void __launch_bounds__(1024) srtt_gather_staged_kernel(int n, const double* __restrict__ a, long long lda,
                                                                  const int* __restrict__ src,
                                                                  double* __restrict__ v) {
  extern __shared__ double srow[];
  const long long i = blockIdx.x;
  const double* ar = a + i * lda;
  if (VEC) {
    const double2* ar2 = reinterpret_cast<const double2*>(ar);
    double2* s2 = reinterpret_cast<double2*>(srow);
    for (int p = threadIdx.x; p < n / 2; p += blockDim.x) s2[p] = __ldcs(ar2 + p);
    if ((n & 1) && threadIdx.x == 0) srow[n - 1] = ar[n - 1];
  } else {
    for (int p = threadIdx.x; p < n; p += blockDim.x) srow[p] = ar[p];
  }
  __syncthreads();
  double* vr = v + i * (long long)n;
  for (int q = threadIdx.x; q < n; q += blockDim.x) vr[q] = srow[src[q]];
}

// any layout / length: element-wise gather (A's rows stay in L2 across the CTAs of a row)
__global__ void srtt_gather_kernel(long long rows, int n, const double* __restrict__ a, long long lda, int colmajor,
                                   const int* __restrict__ src, double* __restrict__ v) {
  const long long total = rows * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / n;
    const int q = (int)(e - i * n);
    const long long col = src[q];
    v[e] = colmajor ? a[col * lda + i] : a[i * lda + col];
  }
}

__global__ void srtt_select_kernel(long long rows, int n, int ell, const double2* __restrict__ V,
                                   const int64_t* __restrict__ cols, const double* __restrict__ signs, double scale,
                                   double* __restrict__ y, long long ldy) {
  const long long total = rows * ell;
  const int nh = n / 2 + 1;
  const double f0 = sqrt(1.0 / (4.0 * n)), fk = sqrt(1.0 / (2.0 * n));
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / ell;
    const int j = (int)(e - i * ell);
    const int k = (int)cols[j];
    double2 z;
    if (k < nh) {
      z = V[i * nh + k];
    } else {
      z = V[i * nh + (n - k)];
      z.y = -z.y;
    }
    double s, c;
    sincospi((double)k / (2.0 * n), &s, &c);  // exp(-i pi k / (2n)) = c - i s
    const double dct = 2.0 * (z.x * c + z.y * s) * (k == 0 ? f0 : fk);
    y[i * ldy + j] = scale * (dct * signs[k]);
  }
}

long long srtt_workspace_bytes(long long m, int n) {
  // per row: v (n doubles) + V (n/2 + 1 complex doubles); + 16 B to align V for cuFFT,
  // + the composed column index (n ints)
  return m * (8LL * n + 16LL * (n / 2 + 1)) + 16 + 4LL * n + 16;
}

int launch_srtt_apply(long long m, int n, int ell, const double* a, long long lda, int colmajor,
                      const int64_t* perm, const double* signs, const int64_t* cols, double scale, double* y,
                      long long ldy, void* ws, long long ws_bytes, cudaStream_t st) {
  if (m < 0 || n < 1 || ell < 1 || ell > n || ldy < ell || !ws) return RS_ERR_ARG;
  if (lda < (colmajor ? m : n)) return RS_ERR_ARG;
  if (m == 0) return RS_OK;
  const long long fixed = 4LL * n + 32;
  const long long per_row = srtt_workspace_bytes(1, n) - fixed;
  long long batch = (ws_bytes - fixed) / per_row;
  if (batch < 1) return RS_ERR_ARG;
  if (batch > m) batch = m;
  if (batch > (1 << 30) / n) batch = std::max(1LL, (long long)((1 << 30) / n));  // cuFFT int batch sizes
  double* v = static_cast<double*>(ws);
  double2* V = reinterpret_cast<double2*>(v + ((batch * (long long)n + 1) & ~1LL));  // 16-byte aligned
  int* src = reinterpret_cast<int*>(V + batch * (long long)(n / 2 + 1));
  srtt_index_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, perm, src);
  count_launch(1);
  const bool staged = !colmajor && n <= SRTT_STAGE_MAX;
  const bool vec = staged && (lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(a) & 15) == 0);
  auto gk = vec ? srtt_gather_staged_kernel<true> : srtt_gather_staged_kernel<false>;
  if (staged && cudaFuncSetAttribute(gk, cudaFuncAttributeMaxDynamicSharedMemorySize, n * 8) != cudaSuccess)
    return RS_ERR_CUDA;
  for (long long r0 = 0; r0 < m; r0 += batch) {
    const long long rows = std::min(batch, m - r0);
    cufftHandle plan;
    if (get_plan(n, (int)rows, &plan) != RS_OK) return RS_ERR_CUDA;
    const double* ab = colmajor ? a + r0 : a + r0 * lda;
    if (staged) {
      gk<<<(unsigned)rows, 1024, (size_t)n * 8, st>>>(n, ab, lda, src, v);
    } else {
      const long long tot = rows * n;
      srtt_gather_kernel<<<(unsigned)std::min<long long>((tot + 255) / 256, 148LL * 16), 256, 0, st>>>(
          rows, n, ab, lda, colmajor, src, v);
    }
    if (cufftSetStream(plan, st) != CUFFT_SUCCESS) return RS_ERR_CUDA;
    const cufftResult r = cufftExecD2Z(plan, v, reinterpret_cast<cufftDoubleComplex*>(V));
    if (r != CUFFT_SUCCESS) {
      if (getenv("RS_SRTT_DEBUG")) fprintf(stderr, "srtt: cufftExecD2Z = %d\n", (int)r);
      return RS_ERR_CUDA;
    }
    const long long tot = rows * ell;
    srtt_select_kernel<<<(unsigned)std::min<long long>((tot + 255) / 256, 148LL * 16), 256, 0, st>>>(
        rows, n, ell, V, cols, signs, scale, y + r0 * ldy, ldy);
    count_launch(2);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && getenv("RS_SRTT_DEBUG")) fprintf(stderr, "srtt: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

}  // namespace rs
