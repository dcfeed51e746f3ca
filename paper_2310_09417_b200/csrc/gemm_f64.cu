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
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "rskel_internal.h"

namespace rs {

// ---------------------------------------------------------------------------
// Tile configuration (compile-time).  Leading dimensions are = 4 (mod 16)
// doubles: 64-bit shared loads are served per half-warp and the fragment
// pattern (t * LD + g, g, t in 0..3) then hits 16 distinct bank pairs.
template <int BM_, int BN_, int BK_, int WARPS_M_, int WARPS_N_, int STAGES_, int MINB_>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_;
  static constexpr int STAGES = STAGES_, MINB = MINB_;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  static constexpr int MT = WTM / 16, NT = WTN / 8;
  static constexpr int ACC = MT * NT * 4;
  static constexpr int A_COL_LD = BM + 4;  // As[k][m]
  static constexpr int A_ROW_LD = BK + 4;  // As[m][k]
  static constexpr int B_LD = BN + 4;      // Bs[k][n]
  template <bool A_COL>
  static constexpr int a_stage() { return A_COL ? BK * A_COL_LD : BM * A_ROW_LD; }
  static constexpr int b_stage() { return BK * B_LD; }
  template <bool A_COL>
  static constexpr size_t smem() { return sizeof(double) * STAGES * (a_stage<A_COL>() + b_stage()); }
};

// Production configuration and the alternatives the tuner compares
// (RSKEL_GEMM_CFG=i selects one at run time, for tools/bench_kernels.py).
using Cfg0 = GemmCfg<128, 64, 16, 4, 2, 3, 2>;   // row-major A (Schur, W_hat, small products): 8 warps of 32x32
using Cfg8 = GemmCfg<128, 64, 32, 2, 2, 2, 2>;   // column-major A (sketch): 4 warps of 64x32, BK 32
using Cfg12 = GemmCfg<128, 64, 32, 4, 2, 2, 2>;  // 8 warps of 32x32, BK 32
// Measured alternatives (tools/tune_gemm.sh, B200, sketch 20000^2 x 64 / Schur k=7000):
// 128x64x16 4 stages 28.x / 24; 64x64x16 4 CTA/SM 26 / 17; 64x32x16 (cuBLAS-like tile) 26.8 / 13.7;
// 256x64 one CTA/SM 29.0 / 21.7; 8 warps BK 32 (Cfg12) 29.1 / 23.3; Cfg8 31.4 / 19.8; Cfg0 28.2 / 25.5.
// Stream-K partial slots: 2 per CTA, THREADS * ACC doubles each; every config
// has MINB * THREADS * ACC <= 16384 doubles per SM.
constexpr int SK_SLOT_DOUBLES_PER_SM = 16384;

size_t gemm_partials_bytes(int nsm) {
  return sizeof(double) * 2 * (size_t)nsm * SK_SLOT_DOUBLES_PER_SM;
}

struct SkPlan {
  int tiles_n, tiles, KT, G;
  long long U;
};

// First unit of CTA c.
__host__ __device__ inline long long sk_u0(const SkPlan& s, int c) { return (long long)c * s.U / s.G; }

// Epilogue for one accumulator set of tile (m0, n0).
template <class C>
__device__ __forceinline__ void epilogue_store(const DGemmParams& p, int m0, int n0, int wm, int wn,
                                               int g, int t, const double (&acc)[C::ACC]) {
  const double alpha = p.alpha, beta = p.beta;
#pragma unroll
  for (int i = 0; i < C::MT; ++i) {
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
      for (int j = 0; j < C::NT; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int col = n0 + wn + 8 * j + 2 * t + e;
          if (col < p.N) {
            double v = acc[(i * C::NT + j) * 4 + 2 * h + e];
            crow[col] = cin ? fma(alpha, v, beta * cin[col]) : alpha * v;
          }
        }
      }
    }
  }
}

template <class C, bool A_COL, bool VEC2>
__device__ __forceinline__ void mainloop(const DGemmParams& p, double* As, double* Bs, int m0, int n0,
                                         int kt0, int kt1, double (&acc)[C::ACC]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp % C::WARPS_M) * C::WTM, wn = (warp / C::WARPS_M) * C::WTN;
  const int M = p.M, N = p.N, K = p.K;
  constexpr int V = VEC2 ? 2 : 1;
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, T = C::THREADS;

  constexpr int A_CHUNKS = (BM * BK) / V / T;
  static_assert(A_CHUNKS * V * T == BM * BK, "A tile must split evenly");
  const double* arow[A_COL ? 1 : A_CHUNKS];
  if constexpr (!A_COL) {
#pragma unroll
    for (int i = 0; i < A_CHUNKS; ++i) {
      int c = tid + i * T;
      int mr = c / (BK / V);
      int gm = m0 + mr;
      long long r = gm < M ? (p.aidx ? p.aidx[gm] : gm) : 0;
      arow[i] = gm < M ? p.A + r * p.lda : nullptr;
    }
  }

  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * BK;
    double* as = As + stage * C::template a_stage<A_COL>();
    double* bs = Bs + stage * C::b_stage();
#pragma unroll
    for (int i = 0; i < A_CHUNKS; ++i) {
      int c = tid + i * T;
      if constexpr (A_COL) {
        constexpr int PER_ROW = BM / V;
        int kr = c / PER_ROW, mc = (c % PER_ROW) * V;
        int gk = k0 + kr, gm = m0 + mc;
        const double* src = p.A;
        int bytes = 0;
        if (gk < K && gm < M) {
          src = p.A + (long long)gk * p.lda + gm;
          bytes = (VEC2 && gm + 1 < M) ? 16 : 8;
        }
        if constexpr (VEC2) cp_async16(as + kr * C::A_COL_LD + mc, src, bytes);
        else cp_async8(as + kr * C::A_COL_LD + mc, src, bytes);
      } else {
        constexpr int PER_ROW = BK / V;
        int mr = c / PER_ROW, kc = (c % PER_ROW) * V;
        int gk = k0 + kc;
        const double* src = p.A;
        int bytes = 0;
        if (arow[i] != nullptr && gk < K) {
          src = arow[i] + gk;
          bytes = (VEC2 && gk + 1 < K) ? 16 : 8;
        }
        if constexpr (VEC2) cp_async16(as + mr * C::A_ROW_LD + kc, src, bytes);
        else cp_async8(as + mr * C::A_ROW_LD + kc, src, bytes);
      }
    }
    constexpr int B_CHUNKS = (BK * BN) / V / T;
    static_assert(B_CHUNKS * V * T == BK * BN, "B tile must split evenly");
#pragma unroll
    for (int i = 0; i < B_CHUNKS; ++i) {
      int c = tid + i * T;
      constexpr int PER_ROW = BN / V;
      int kr = c / PER_ROW, nc = (c % PER_ROW) * V;
      int gk = k0 + kr, gn = n0 + nc;
      const double* src = p.B;
      int bytes = 0;
      if (gk < K && gn < N) {
        long long r = p.bidx ? p.bidx[gk] : gk;
        src = p.B + r * p.ldb + gn;
        bytes = (VEC2 && gn + 1 < N) ? 16 : 8;
      }
      if constexpr (VEC2) cp_async16(bs + kr * C::B_LD + nc, src, bytes);
      else cp_async8(bs + kr * C::B_LD + nc, src, bytes);
    }
  };

#pragma unroll
  for (int e = 0; e < C::ACC; ++e) acc[e] = 0.0;

  const int nkt = kt1 - kt0;
#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    if (s < nkt) load_stage(s, kt0 + s);
    cp_async_commit();
  }
  for (int it = 0; it < nkt; ++it) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    {
      int nk = it + C::STAGES - 1;
      if (nk < nkt) load_stage(nk % C::STAGES, kt0 + nk);
      cp_async_commit();
    }
    const int stage = it % C::STAGES;
    const double* as = As + stage * C::template a_stage<A_COL>();
    const double* bs = Bs + stage * C::b_stage();
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[C::MT][2], b[C::NT];
#pragma unroll
      for (int i = 0; i < C::MT; ++i) {
        int mr = wm + 16 * i + g;
        if constexpr (A_COL) {
          a[i][0] = as[(kk + t) * C::A_COL_LD + mr];
          a[i][1] = as[(kk + t) * C::A_COL_LD + mr + 8];
        } else {
          a[i][0] = as[mr * C::A_ROW_LD + kk + t];
          a[i][1] = as[(mr + 8) * C::A_ROW_LD + kk + t];
        }
      }
#pragma unroll
      for (int j = 0; j < C::NT; ++j) b[j] = bs[(kk + t) * C::B_LD + wn + 8 * j + g];
#pragma unroll
      for (int i = 0; i < C::MT; ++i)
#pragma unroll
        for (int j = 0; j < C::NT; ++j) {
          double(&c4)[4] = *reinterpret_cast<double(*)[4]>(&acc[(i * C::NT + j) * 4]);
          dmma_16x8x4(c4, a[i][0], a[i][1], b[j]);
        }
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // stage buffers are reused by the next tile of this CTA
}

template <class C, bool A_COL, bool VEC2>
__global__ void __launch_bounds__(C::THREADS, C::MINB) dgemm_kernel(DGemmParams p, SkPlan sk) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + C::STAGES * C::template a_stage<A_COL>();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp % C::WARPS_M) * C::WTM, wn = (warp / C::WARPS_M) * C::WTN;
  double acc[C::ACC];

  if (sk.G == 0) {  // classic tile grid
    const int n0 = blockIdx.x * C::BN, m0 = blockIdx.y * C::BM;
    mainloop<C, A_COL, VEC2>(p, As, Bs, m0, n0, 0, sk.KT, acc);
    epilogue_store<C>(p, m0, n0, wm, wn, g, t, acc);
    return;
  }
  // stream-K
  const int c = blockIdx.x;
  long long u = sk_u0(sk, c), u1 = sk_u0(sk, c + 1);
  while (u < u1) {
    const int tile = (int)(u / sk.KT);
    const int i0 = (int)(u - (long long)tile * sk.KT);
    const int i1 = (int)min((long long)sk.KT, i0 + (u1 - u));
    const int m0 = (tile / sk.tiles_n) * C::BM, n0 = (tile % sk.tiles_n) * C::BN;
    mainloop<C, A_COL, VEC2>(p, As, Bs, m0, n0, i0, i1, acc);
    if (i0 == 0 && i1 == sk.KT) {
      epilogue_store<C>(p, m0, n0, wm, wn, g, t, acc);
    } else {
      // element-major slot layout: coalesced writes here and reads in the fixup
      const int slot = (i0 > 0) ? 2 * c : 2 * c + 1;
      double* dst = p.partials + (size_t)slot * C::THREADS * C::ACC + tid;
#pragma unroll
      for (int e = 0; e < C::ACC; ++e) dst[(size_t)e * C::THREADS] = acc[e];
    }
    u += i1 - i0;
  }
}

// Sum the partials of every split tile in k order and apply the epilogue.
template <class C>
__global__ void __launch_bounds__(C::THREADS) dgemm_fixup_kernel(DGemmParams p, SkPlan sk) {
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
  const int wm = (warp % C::WARPS_M) * C::WTM, wn = (warp / C::WARPS_M) * C::WTN;
  double acc[C::ACC];
  {
    const double* src = p.partials + (size_t)(2 * clo + 1) * C::THREADS * C::ACC + tid;
#pragma unroll
    for (int e = 0; e < C::ACC; ++e) acc[e] = src[(size_t)e * C::THREADS];
  }
  for (int c = clo + 1; c <= chi; ++c) {
    const double* src = p.partials + (size_t)(2 * c) * C::THREADS * C::ACC + tid;
#pragma unroll
    for (int e = 0; e < C::ACC; ++e) acc[e] += src[(size_t)e * C::THREADS];
  }
  const int m0 = (tile / sk.tiles_n) * C::BM, n0 = (tile % sk.tiles_n) * C::BN;
  epilogue_store<C>(p, m0, n0, wm, wn, g, t, acc);
}

// Fixup for skinny splits (many CTAs per tile): CTA (tile, e) sums element e
// of every thread's partial over the contributors (in CTA order) and stores it.
template <class C>
__global__ void __launch_bounds__(C::THREADS) dgemm_fixup_elem_kernel(DGemmParams p, SkPlan sk) {
  const int tile = blockIdx.x, e = blockIdx.y;
  const long long ub = (long long)tile * sk.KT, ue = ub + sk.KT;
  auto owner = [&](long long u) {
    int c = (int)((u * sk.G) / sk.U);
    while (c + 1 < sk.G && sk_u0(sk, c + 1) <= u) ++c;
    while (c > 0 && sk_u0(sk, c) > u) --c;
    return c;
  };
  const int clo = owner(ub), chi = owner(ue - 1);
  if (clo == chi) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp % C::WARPS_M) * C::WTM, wn = (warp / C::WARPS_M) * C::WTN;
  double acc = p.partials[(size_t)(2 * clo + 1) * C::THREADS * C::ACC + (size_t)e * C::THREADS + tid];
  for (int c = clo + 1; c <= chi; ++c)
    acc += p.partials[(size_t)(2 * c) * C::THREADS * C::ACC + (size_t)e * C::THREADS + tid];
  // e = ((i * NT + j) * 4 + 2h + ee): fragment row/column of this element
  const int ee = e & 1, h = (e >> 1) & 1, ij = e >> 2, i = ij / C::NT, j = ij % C::NT;
  const int m0 = (tile / sk.tiles_n) * C::BM, n0 = (tile % sk.tiles_n) * C::BN;
  const int row = m0 + wm + 16 * i + g + 8 * h, col = n0 + wn + 8 * j + 2 * t + ee;
  if (row >= p.M || col >= p.N) return;
  double v = p.alpha * acc;
  if (p.beta != 0.0) {
    const long long r = p.cidx ? p.cidx[row] : row;
    v = fma(p.alpha, acc, p.beta * p.Cin[r * p.ldcin + col]);
  }
  p.C[(long long)row * p.ldc + col] = v;
}

template <class C, bool A_COL, bool VEC2>
static int launch_dgemm_t(const DGemmParams& p, cudaStream_t st) {
  static_assert(C::MINB * C::THREADS * C::ACC <= SK_SLOT_DOUBLES_PER_SM, "partials workspace");
  constexpr size_t smem = C::template smem<A_COL>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(dgemm_kernel<C, A_COL, VEC2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  SkPlan sk;
  sk.tiles_n = (p.N + C::BN - 1) / C::BN;
  const int tiles_m = (p.M + C::BM - 1) / C::BM;
  sk.tiles = sk.tiles_n * tiles_m;
  sk.KT = (p.K + C::BK - 1) / C::BK;
  sk.G = 0;
  sk.U = (long long)sk.tiles * sk.KT;
  const int slots = nsm * C::MINB;
  // Stream-K when a plain grid would run fewer than ~4 waves and each CTA
  // still gets a few k-tiles of work.
  // Skinny products (fewer tiles than CTA slots, long K) split K over up to
  // `slots` CTAs with at least 4 k-tiles each.
  int G = 0;
  if (p.partials != nullptr && sk.tiles < 4 * slots && sk.KT >= 8) {
    if (sk.U >= 4LL * slots) G = slots;
    else if (sk.tiles < slots && sk.KT >= 64) G = (int)std::max<long long>(sk.tiles, std::min<long long>(slots, sk.U / 4));
  }
  if (G > 0) {
    sk.G = G;
    dgemm_kernel<C, A_COL, VEC2><<<sk.G, C::THREADS, smem, st>>>(p, sk);
    if (sk.G > 8 * sk.tiles)  // many contributors per tile: element-parallel sum
      dgemm_fixup_elem_kernel<C><<<dim3(sk.tiles, C::ACC), C::THREADS, 0, st>>>(p, sk);
    else
      dgemm_fixup_kernel<C><<<sk.tiles, C::THREADS, 0, st>>>(p, sk);
    count_launch(2);
  } else {
    dim3 grid(sk.tiles_n, tiles_m);
    dgemm_kernel<C, A_COL, VEC2><<<grid, C::THREADS, smem, st>>>(p, sk);
    count_launch(1);
  }
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

static bool al16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; }

template <class C>
static int launch_cfg(const DGemmParams& p, bool a_col, bool vec2, cudaStream_t st) {
  if (a_col) return vec2 ? launch_dgemm_t<C, true, true>(p, st) : launch_dgemm_t<C, true, false>(p, st);
  return vec2 ? launch_dgemm_t<C, false, true>(p, st) : launch_dgemm_t<C, false, false>(p, st);
}

static int selected_cfg() {
  static int cfg = -2;
  if (cfg == -2) {
    const char* e = getenv("RSKEL_GEMM_CFG");
    cfg = e ? atoi(e) : -1;
  }
  return cfg;
}

int launch_dgemm(const DGemmParams& p, bool a_col, cudaStream_t st) {
  if (p.M < 0 || p.N < 0 || p.K < 0) return RS_ERR_ARG;
  if (p.M == 0 || p.N == 0) return RS_OK;
  bool vec2 = al16(p.A) && al16(p.B) && (p.lda % 2 == 0) && (p.ldb % 2 == 0);
  switch (selected_cfg()) {
    case 8: return launch_cfg<Cfg8>(p, a_col, vec2, st);
    case 12: return launch_cfg<Cfg12>(p, a_col, vec2, st);
    default:
      // Measured on B200 (tools/tune_gemm.sh): the column-major sketch operand
      // prefers 64x32 warp tiles (31.4 TF/s vs 28.2), the gathered row-major
      // Schur/interpolation operands the 32x32 tiles of Cfg0.
      return a_col ? launch_cfg<Cfg8>(p, a_col, vec2, st) : launch_cfg<Cfg0>(p, a_col, vec2, st);
  }
}

}  // namespace rs
