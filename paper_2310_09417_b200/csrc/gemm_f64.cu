// fp64 GEMM on the B200 DMMA pipe with optional row gathers.
//
//   C[i, :] = alpha * (op(A) B)[i, :] + beta * Cin[cidx(i), :]
//
// A is M x K, either row-major with an optional row index (row i of A lives
// at aidx[i]) or column-major (the transposed view of a C-ordered matrix, as
// in `a.T @ Gamma`, `sketching.py:266-273`).  B is K x N row-major with an
// optional row index (row k of B lives at bidx[k]), which is how the Schur
// step reads the skeleton rows Y[perm[:k]] without materialising them
// (`skeleton.py:317-323`).  C is row-major.
//
// Tiling: CTA 128 x 64 x 16, 8 warps as 4 (M) x 2 (N), warp tile 32 x 32 =
// 2 x 4 DMMA m16n8k4 tiles, 3-stage cp.async pipeline, 2 CTAs per SM.
//
// Work distribution: the skeleton GEMMs are tall and skinny (N = 64, M up to
// 65536, K up to 65536), so a plain tile grid leaves most of the 148 SMs idle
// or runs 1.06 waves.  When the tile count is below a few waves the kernel
// runs stream-K: exactly G = 2 x #SM persistent CTAs, CTA c owning the
// contiguous range [c U / G, (c+1) U / G) of the U = tiles x k-tiles work
// units.  Tiles split between CTAs write fragment-ordered partials; a fixup
// kernel adds them in k order (CTA order) and applies the epilogue.  The
// split depends only on (M, N, K, G), so results are bitwise reproducible.
#include "common.cuh"
#include "rskel_internal.h"

namespace rs {

constexpr int GBM = 128, GBN = 64, GBK = 16, GSTAGES = 3;
constexpr int GWARPS_M = 4, GWARPS_N = 2, GTHREADS = GWARPS_M * GWARPS_N * 32;
constexpr int GWTM = GBM / GWARPS_M, GWTN = GBN / GWARPS_N;  // 32 x 32
constexpr int GMT = GWTM / 16, GNT = GWTN / 8;                  // 2 x 4
constexpr int GACC = GMT * GNT * 4;                             // accumulators per thread
// Leading dimensions are = 4 (mod 16) doubles: 64-bit shared loads are served per
// half-warp, and the fragment pattern (t * LD + g, g, t in 0..3) then hits 16
// distinct bank pairs -- conflict-free.
constexpr int A_COL_LD = GBM + 4;  // As[k][m]
constexpr int A_ROW_LD = GBK + 4;  // As[m][k]
constexpr int B_LD = GBN + 4;      // Bs[k][n]
constexpr int SK_CTAS_PER_SM = 2;

template <bool A_COL>
__host__ __device__ constexpr int a_stage_elems() { return A_COL ? GBK * A_COL_LD : GBM * A_ROW_LD; }
__host__ __device__ constexpr int b_stage_elems() { return GBK * B_LD; }

template <bool A_COL>
constexpr size_t gemm_smem_bytes() {
  return sizeof(double) * GSTAGES * (a_stage_elems<A_COL>() + b_stage_elems());
}

size_t gemm_partials_bytes(int nsm) {
  return sizeof(double) * 2 * (size_t)nsm * SK_CTAS_PER_SM * GBM * GBN;
}

struct SkPlan {
  int tiles_n, tiles, KT, G;
  long long U;
};

// First unit of CTA c.
__host__ __device__ inline long long sk_u0(const SkPlan& s, int c) { return (long long)c * s.U / s.G; }

// Epilogue for one accumulator set of tile (m0, n0).
__device__ __forceinline__ void epilogue_store(const DGemmParams& p, int m0, int n0, int wm, int wn,
                                               int g, int t, const double (&acc)[GACC]) {
  const double alpha = p.alpha, beta = p.beta;
#pragma unroll
  for (int i = 0; i < GMT; ++i) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int row = m0 + wm + 16 * i + g + 8 * h;
      if (row >= p.M) continue;
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
          if (col < p.N) {
            double v = acc[(i * GNT + j) * 4 + 2 * h + e];
            crow[col] = cin ? fma(alpha, v, beta * cin[col]) : alpha * v;
          }
        }
      }
    }
  }
}

template <bool A_COL, bool VEC2>
__device__ __forceinline__ void mainloop(const DGemmParams& p, double* As, double* Bs, int m0, int n0,
                                         int kt0, int kt1, double (&acc)[GACC]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp % GWARPS_M) * GWTM, wn = (warp / GWARPS_M) * GWTN;
  const int M = p.M, N = p.N, K = p.K;

  constexpr int A_CHUNKS = (GBM * GBK) / (VEC2 ? 2 : 1) / GTHREADS;
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
#pragma unroll
    for (int i = 0; i < A_CHUNKS; ++i) {
      int c = tid + i * GTHREADS;
      if constexpr (A_COL) {
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

#pragma unroll
  for (int e = 0; e < GACC; ++e) acc[e] = 0.0;

  const int nkt = kt1 - kt0;
#pragma unroll
  for (int s = 0; s < GSTAGES - 1; ++s) {
    if (s < nkt) load_stage(s, kt0 + s);
    cp_async_commit();
  }
  for (int it = 0; it < nkt; ++it) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    {
      int nk = it + GSTAGES - 1;
      if (nk < nkt) load_stage(nk % GSTAGES, kt0 + nk);
      cp_async_commit();
    }
    const int stage = it % GSTAGES;
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
        for (int j = 0; j < GNT; ++j) {
          double(&c4)[4] = *reinterpret_cast<double(*)[4]>(&acc[(i * GNT + j) * 4]);
          dmma_16x8x4(c4, a[i][0], a[i][1], b[j]);
        }
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // stage buffers are reused by the next tile of this CTA
}

template <bool A_COL, bool VEC2>
__global__ void __launch_bounds__(GTHREADS, SK_CTAS_PER_SM) dgemm_kernel(DGemmParams p, SkPlan sk) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + GSTAGES * a_stage_elems<A_COL>();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp % GWARPS_M) * GWTM, wn = (warp / GWARPS_M) * GWTN;
  double acc[GACC];

  if (sk.G == 0) {  // classic tile grid
    const int n0 = blockIdx.x * GBN, m0 = blockIdx.y * GBM;
    mainloop<A_COL, VEC2>(p, As, Bs, m0, n0, 0, sk.KT, acc);
    epilogue_store(p, m0, n0, wm, wn, g, t, acc);
    return;
  }
  // stream-K
  const int c = blockIdx.x;
  long long u = sk_u0(sk, c), u1 = sk_u0(sk, c + 1);
  while (u < u1) {
    const int tile = (int)(u / sk.KT);
    const int i0 = (int)(u - (long long)tile * sk.KT);
    const int i1 = (int)min((long long)sk.KT, i0 + (u1 - u));
    const int m0 = (tile / sk.tiles_n) * GBM, n0 = (tile % sk.tiles_n) * GBN;
    mainloop<A_COL, VEC2>(p, As, Bs, m0, n0, i0, i1, acc);
    if (i0 == 0 && i1 == sk.KT) {
      epilogue_store(p, m0, n0, wm, wn, g, t, acc);
    } else {
      const int slot = (i0 > 0) ? 2 * c : 2 * c + 1;
      double* dst = p.partials + ((size_t)slot * GTHREADS + tid) * GACC;
#pragma unroll
      for (int e = 0; e < GACC; e += 2)
        *reinterpret_cast<double2*>(dst + e) = make_double2(acc[e], acc[e + 1]);
    }
    u += i1 - i0;
  }
}

// Sum the partials of every split tile in k order and apply the epilogue.
__global__ void __launch_bounds__(GTHREADS) dgemm_fixup_kernel(DGemmParams p, SkPlan sk) {
  const int tile = blockIdx.x;
  const long long ub = (long long)tile * sk.KT, ue = ub + sk.KT;
  // owner(u): largest c with u0(c) <= u
  auto owner = [&](long long u) {
    int c = (int)((u * sk.G) / sk.U);
    while (c + 1 < sk.G && sk_u0(sk, c + 1) <= u) ++c;
    while (c > 0 && sk_u0(sk, c) > u) --c;
    return c;
  };
  const int clo = owner(ub), chi = owner(ue - 1);
  if (clo == chi) return;  // complete tile, stored by its CTA
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp % GWARPS_M) * GWTM, wn = (warp / GWARPS_M) * GWTN;
  double acc[GACC];
  {
    const double* src = p.partials + ((size_t)(2 * clo + 1) * GTHREADS + tid) * GACC;
#pragma unroll
    for (int e = 0; e < GACC; ++e) acc[e] = src[e];
  }
  for (int c = clo + 1; c <= chi; ++c) {
    const double* src = p.partials + ((size_t)(2 * c) * GTHREADS + tid) * GACC;
#pragma unroll
    for (int e = 0; e < GACC; ++e) acc[e] += src[e];
  }
  const int m0 = (tile / sk.tiles_n) * GBM, n0 = (tile % sk.tiles_n) * GBN;
  epilogue_store(p, m0, n0, wm, wn, g, t, acc);
}

template <bool A_COL, bool VEC2>
static int launch_dgemm_t(const DGemmParams& p, cudaStream_t st) {
  constexpr size_t smem = gemm_smem_bytes<A_COL>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(dgemm_kernel<A_COL, VEC2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  SkPlan sk;
  sk.tiles_n = (p.N + GBN - 1) / GBN;
  const int tiles_m = (p.M + GBM - 1) / GBM;
  sk.tiles = sk.tiles_n * tiles_m;
  sk.KT = (p.K + GBK - 1) / GBK;
  sk.G = 0;
  sk.U = (long long)sk.tiles * sk.KT;
  const int slots = nsm * SK_CTAS_PER_SM;
  // Stream-K when a plain grid would run fewer than ~4 waves and each CTA
  // still gets a few k-tiles of work.
  if (p.partials != nullptr && sk.tiles < 4 * slots && sk.U >= 4LL * slots && sk.KT >= 8) {
    sk.G = slots;
    dgemm_kernel<A_COL, VEC2><<<sk.G, GTHREADS, smem, st>>>(p, sk);
    dgemm_fixup_kernel<<<sk.tiles, GTHREADS, 0, st>>>(p, sk);
    count_launch(2);
  } else {
    dim3 grid(sk.tiles_n, tiles_m);
    dgemm_kernel<A_COL, VEC2><<<grid, GTHREADS, smem, st>>>(p, sk);
    count_launch(1);
  }
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
