// fp64 GEMM on the B200 DMMA pipe with optional row gathers.
//
//   C[i, :] = alpha * (op(A) B)[i, :] + beta * Cin[cidx(i), :]
//
// A is M x K, either row-major with an optional row index (row i of A lives
// at aidx[i]) or column-major (the transposed view of a C-ordered matrix, as
// in `a.T @ Gamma`, `sketching.py:266-273`).  B is K x N row-major with an
// optional row index (row k of B lives at bidx[k]), which is how the Schur
// step reads the skeleton rows Y[perm[:k]] without materialising them
// (`skeleton.py:317-323`).  C is row-major.  Every output element is reduced
// in one fixed order by one thread (no split-K, no atomics), so results are
// bitwise reproducible run to run.
//
// Tiling: CTA 128 x 64 x 16, 8 warps as 4 (M) x 2 (N), warp tile 32 x 32 =
// 2 x 4 DMMA m16n8k4 tiles, 3-stage cp.async pipeline, 2 CTAs per SM.
#include "common.cuh"
#include "rskel_internal.h"

namespace rs {

constexpr int GBM = 128, GBN = 64, GBK = 16, GSTAGES = 3;
constexpr int GWARPS_M = 4, GWARPS_N = 2, GTHREADS = GWARPS_M * GWARPS_N * 32;
constexpr int GWTM = GBM / GWARPS_M, GWTN = GBN / GWARPS_N;  // 32 x 32
constexpr int GMT = GWTM / 16, GNT = GWTN / 8;                  // 2 x 4
constexpr int A_COL_LD = GBM + 8;  // As[k][m]
constexpr int A_ROW_LD = GBK + 4;  // As[m][k]
constexpr int B_LD = GBN + 8;      // Bs[k][n]

template <bool A_COL>
__host__ __device__ constexpr int a_stage_elems() { return A_COL ? GBK * A_COL_LD : GBM * A_ROW_LD; }
__host__ __device__ constexpr int b_stage_elems() { return GBK * B_LD; }

template <bool A_COL>
constexpr size_t gemm_smem_bytes() {
  return sizeof(double) * GSTAGES * (a_stage_elems<A_COL>() + b_stage_elems());
}

template <bool A_COL, bool VEC2>
__global__ void __launch_bounds__(GTHREADS, 2) dgemm_kernel(DGemmParams p) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + GSTAGES * a_stage_elems<A_COL>();

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp % GWARPS_M) * GWTM, wn = (warp / GWARPS_M) * GWTN;
  const int n0 = blockIdx.x * GBN, m0 = blockIdx.y * GBM;
  const int M = p.M, N = p.N, K = p.K;
  const int KT = (K + GBK - 1) / GBK;

  // Row pointers of the A tile rows this thread copies (row-major A only).
  constexpr int A_CHUNKS = (GBM * GBK) / (VEC2 ? 2 : 1) / GTHREADS;  // per thread
  const double* arow[A_COL ? 1 : A_CHUNKS];
  if constexpr (!A_COL) {
#pragma unroll
    for (int i = 0; i < A_CHUNKS; ++i) {
      int c = tid + i * GTHREADS;
      int mr = VEC2 ? c / (GBK / 2) : c / GBK;
      int gm = m0 + mr;
      long long r = gm < M ? (p.aidx ? p.aidx[gm] : gm) : 0;
      arow[i] = gm < M ? p.A + r * p.lda : nullptr;
    }
  }

  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * GBK;
    double* as = As + stage * a_stage_elems<A_COL>();
    double* bs = Bs + stage * b_stage_elems();
    // ---- A tile ----
#pragma unroll
    for (int i = 0; i < A_CHUNKS; ++i) {
      int c = tid + i * GTHREADS;
      if constexpr (A_COL) {
        // As[kr][mc..] <- A[(k0+kr)*lda + m0+mc..]
        constexpr int PER_ROW = GBM / (VEC2 ? 2 : 1);
        int kr = c / PER_ROW, mc = (c % PER_ROW) * (VEC2 ? 2 : 1);
        int gk = k0 + kr, gm = m0 + mc;
        const double* src = p.A;
        int bytes = 0;
        if (gk < K && gm < M) {
          src = p.A + (long long)gk * p.lda + gm;
          bytes = (VEC2 && gm + 1 < M) ? 16 : 8;
        }
        if constexpr (VEC2) cp_async16(as + kr * A_COL_LD + mc, src, bytes);
        else cp_async8(as + kr * A_COL_LD + mc, src, bytes);
      } else {
        constexpr int PER_ROW = GBK / (VEC2 ? 2 : 1);
        int mr = c / PER_ROW, kc = (c % PER_ROW) * (VEC2 ? 2 : 1);
        int gk = k0 + kc;
        const double* src = p.A;
        int bytes = 0;
        if (arow[i] != nullptr && gk < K) {
          src = arow[i] + gk;
          bytes = (VEC2 && gk + 1 < K) ? 16 : 8;
        }
        if constexpr (VEC2) cp_async16(as + mr * A_ROW_LD + kc, src, bytes);
        else cp_async8(as + mr * A_ROW_LD + kc, src, bytes);
      }
    }
    // ---- B tile ----
    constexpr int B_CHUNKS = (GBK * GBN) / (VEC2 ? 2 : 1) / GTHREADS;
#pragma unroll
    for (int i = 0; i < B_CHUNKS; ++i) {
      int c = tid + i * GTHREADS;
      constexpr int PER_ROW = GBN / (VEC2 ? 2 : 1);
      int kr = c / PER_ROW, nc = (c % PER_ROW) * (VEC2 ? 2 : 1);
      int gk = k0 + kr, gn = n0 + nc;
      const double* src = p.B;
      int bytes = 0;
      if (gk < K && gn < N) {
        long long r = p.bidx ? p.bidx[gk] : gk;
        src = p.B + r * p.ldb + gn;
        bytes = (VEC2 && gn + 1 < N) ? 16 : 8;
      }
      if constexpr (VEC2) cp_async16(bs + kr * B_LD + nc, src, bytes);
      else cp_async8(bs + kr * B_LD + nc, src, bytes);
    }
  };

  double acc[GMT][GNT][4];
#pragma unroll
  for (int i = 0; i < GMT; ++i)
#pragma unroll
    for (int j = 0; j < GNT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

#pragma unroll
  for (int s = 0; s < GSTAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    {
      int nk = kt + GSTAGES - 1;
      if (nk < KT) load_stage(nk % GSTAGES, nk);
      cp_async_commit();
    }
    const int stage = kt % GSTAGES;
    const double* as = As + stage * a_stage_elems<A_COL>();
    const double* bs = Bs + stage * b_stage_elems();
#pragma unroll
    for (int kk = 0; kk < GBK; kk += 4) {
      double a[GMT][2], b[GNT];
#pragma unroll
      for (int i = 0; i < GMT; ++i) {
        int mr = wm + 16 * i + g;
        if constexpr (A_COL) {
          a[i][0] = as[(kk + t) * A_COL_LD + mr];
          a[i][1] = as[(kk + t) * A_COL_LD + mr + 8];
        } else {
          a[i][0] = as[mr * A_ROW_LD + kk + t];
          a[i][1] = as[(mr + 8) * A_ROW_LD + kk + t];
        }
      }
#pragma unroll
      for (int j = 0; j < GNT; ++j) b[j] = bs[(kk + t) * B_LD + wn + 8 * j + g];
#pragma unroll
      for (int i = 0; i < GMT; ++i)
#pragma unroll
        for (int j = 0; j < GNT; ++j) dmma_16x8x4(acc[i][j], a[i][0], a[i][1], b[j]);
    }
  }
  cp_async_wait<0>();

  // ---- epilogue ----
  const double alpha = p.alpha, beta = p.beta;
#pragma unroll
  for (int i = 0; i < GMT; ++i) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int row = m0 + wm + 16 * i + g + 8 * h;
      if (row >= M) continue;
      double* crow = p.C + (long long)row * p.ldc;
      const double* cin = nullptr;
      if (beta != 0.0) {
        long long r = p.cidx ? p.cidx[row] : row;
        cin = p.Cin + r * p.ldcin;
      }
#pragma unroll
      for (int j = 0; j < GNT; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int col = n0 + wn + 8 * j + 2 * t + e;
          if (col < N) {
            double v = acc[i][j][2 * h + e];
            crow[col] = cin ? fma(alpha, v, beta * cin[col]) : alpha * v;
          }
        }
      }
    }
  }
}

template <bool A_COL, bool VEC2>
static int launch_dgemm_t(const DGemmParams& p, cudaStream_t st) {
  constexpr size_t smem = gemm_smem_bytes<A_COL>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(dgemm_kernel<A_COL, VEC2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  dim3 grid((p.N + GBN - 1) / GBN, (p.M + GBM - 1) / GBM);
  dgemm_kernel<A_COL, VEC2><<<grid, GTHREADS, smem, st>>>(p);
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

static bool al16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; }

int launch_dgemm(const DGemmParams& p, bool a_col, cudaStream_t st) {
  if (p.M < 0 || p.N < 0 || p.K < 0) return RS_ERR_ARG;
  if (p.M == 0 || p.N == 0) return RS_OK;
  bool vec2 = al16(p.A) && al16(p.B) && (p.lda % 2 == 0) && (p.ldb % 2 == 0);
  if (a_col) return vec2 ? launch_dgemm_t<true, true>(p, st) : launch_dgemm_t<true, false>(p, st);
  return vec2 ? launch_dgemm_t<false, true>(p, st) : launch_dgemm_t<false, false>(p, st);
}

}  // namespace rs
