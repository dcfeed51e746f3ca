// fp64 GEMM on the B200 DMMA pipe with optional row gathers.
//
//   C[i, :] = alpha * (op(A) B)[i, :] + beta * Cin[cidx(i), :]      (RS_GEMM_PLAIN)
//   C[i, :] = Cin[cidx(i), :] + (op(A) B)[i, :]                      (RS_GEMM_FOLD / _CHAIN)
//
// A is M x K, either row-major with an optional row index (row i of A lives
// at aidx[i]) or column-major (the transposed view of a C-ordered matrix, as
// in `a.T @ Gamma`, `sketching.py:266-273`).  B is K x N row-major with an
// optional row index (row k of B lives at bidx[k]), which is how the Schur
// step reads the skeleton rows Y[perm[:k]] without materialising them
// (`skeleton.py:317-323`).  C is row-major.
//
// Tiling: CTA 128 x 64, DMMA m16n8k4, cp.async multi-stage pipeline, 2 CTAs
// per SM; the summation order is fixed by K alone (see below).
#include <algorithm>
#include <atomic>
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

// Production configurations (measured on B200, tools/tune_gemm.sh: the
// column-major sketch operand prefers 64x32 warp tiles, the gathered
// row-major Schur / interpolation operands the 32x32 tiles).
#if !defined(RS_ROW_VARIANT) || RS_ROW_VARIANT == 0  // (other variants: tools/build_row_cfg.sh experiments)
using CfgRow = GemmCfg<128, 64, 16, 4, 2, 3, 2>;  // row-major A: 8 warps of 32x32, BK 16
#elif RS_ROW_VARIANT == 1
using CfgRow = GemmCfg<128, 64, 32, 4, 2, 2, 2>;
#elif RS_ROW_VARIANT == 2
using CfgRow = GemmCfg<128, 64, 16, 2, 2, 4, 2>;
#elif RS_ROW_VARIANT == 4
using CfgRow = GemmCfg<128, 64, 16, 2, 2, 3, 2>;  // 4 warps of 64x32, 3 stages: two CTAs fit an SM
#elif RS_ROW_VARIANT == 5
using CfgRow = GemmCfg<128, 64, 16, 4, 2, 4, 2>;  // the library config with 4 stages
#elif RS_ROW_VARIANT == 6
using CfgRow = GemmCfg<128, 64, 8, 4, 2, 6, 2>;   // BK 8, 6 stages
#else
using CfgRow = GemmCfg<128, 64, 32, 2, 2, 2, 2>;
#endif
using CfgCol = GemmCfg<128, 64, 32, 2, 2, 2, 2>;  // column-major A: 4 warps of 64x32, BK 32
constexpr int SLOT_DOUBLES = 128 * 64;            // one BM x BN partial tile
static_assert(CfgRow::THREADS * CfgRow::ACC == SLOT_DOUBLES && CfgCol::THREADS * CfgCol::ACC == SLOT_DOUBLES,
              "partial slots hold one tile");

// ---------------------------------------------------------------------------
// Summation order (the determinism contract).
//
// K is cut into chunks of kc = gemm_chunk(K) columns, fixed in global k and
// independent of M, of the tile grid, of the CTA count and of the layout of
// A.  Chunk c of every output element is a DMMA chain from zero over
// k in [c kc, (c+1) kc) in steps of 4; the chunk sums are folded in chunk
// order, v = ((p0 + p1) + p2) + ...  So an element's value depends only on
// its row of A, B and K: a row gives the same bits whether it is one of
// 20000 candidates on one GPU or one of 2500 on rank 3 of 8, whether A is
// column- or row-major, and whether the K range arrives in one call or in
// kc-aligned pieces (mode RS_GEMM_FOLD below).
//
// Scheduling (chained stream-K): the tiles x k-tiles work is cut into G equal
// contiguous ranges, one per persistent CTA, at k-tile granularity -- no wave
// quantisation whatever M is.  A range cuts chunks at its two ends; the head
// of a cut chunk belongs to CTA g-1, its tail to CTA g, and the tail must
// continue the head's DMMA chain.  Each CTA therefore walks its range
// BACKWARDS: its last piece (a chunk head it hands to g+1) is computed first
// and published to a boundary slot with a release flag, its first piece (the
// tail of g-1's head) is computed last, by which time g-1's boundary value is
// long published.  A completed chunk goes to its (tile, chunk) slot; the last
// chunk of a tile to arrive (ticket counter) folds the slots in chunk order
// and applies the epilogue.
size_t gemm_workspace_bytes() {
  return sizeof(double) * (size_t)(GEMM_SLOTS + GEMM_MAX_CTAS) * SLOT_DOUBLES +
         sizeof(int) * (size_t)(GEMM_SLOTS + GEMM_MAX_CTAS);
}

int gemm_chunk(long long K) {
  long long kc = (K + GEMM_MAX_CHUNKS - 1) / GEMM_MAX_CHUNKS;
  kc = (kc + 31) / 32 * 32;
  return (int)std::max<long long>(GEMM_MIN_CHUNK, kc);
}

struct ChunkPlan {
  int tiles_n;     // tiles along N of the full grid
  int tile0;       // first tile of this launch (tile groups when slots run out)
  int KT;          // k-tiles of K
  int kct;         // k-tiles per chunk
  int nch;         // chunks
  long long U;     // (tiles of this launch) x KT k-tile units, split over gridDim.x CTAs
  unsigned epoch;  // boundary-flag value of this launch (flags are never reset)
};

// Fragment coordinates (within the tile) of accumulator element e of this thread.
template <class C>
__device__ __forceinline__ void frag_rc(int e, int wm, int wn, int g, int t, int& r, int& c) {
  const int ee = e & 1, h = (e >> 1) & 1, ij = e >> 2, i = ij / C::NT, j = ij % C::NT;
  r = wm + 16 * i + g + 8 * h;
  c = wn + 8 * j + 2 * t + ee;
}

// acc[e] = the Cin element of fragment e (0 outside the matrix).
template <class C>
__device__ __forceinline__ void load_cin(const DGemmParams& p, int m0, int n0, int wm, int wn, int g, int t,
                                         double (&acc)[C::ACC]) {
#pragma unroll
  for (int e = 0; e < C::ACC; ++e) {
    int r, c;
    frag_rc<C>(e, wm, wn, g, t, r, c);
    r += m0;
    c += n0;
    double v = 0.0;
    if (r < p.M && c < p.N) {
      const long long rr = p.cidx ? p.cidx[r] : r;
      v = p.Cin[rr * p.ldcin + c];
    }
    acc[e] = v;
  }
}

// Epilogue for one accumulator set of tile (m0, n0).
template <class C>
__device__ __forceinline__ void epilogue_store(const DGemmParams& p, int m0, int n0, int wm, int wn,
                                               int g, int t, const double (&acc)[C::ACC]) {
  const double alpha = p.alpha, beta = p.beta;
  const bool plain = p.mode == RS_GEMM_PLAIN;
#pragma unroll
  for (int i = 0; i < C::MT; ++i) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int row = m0 + wm + 16 * i + g + 8 * h;
      if (row >= p.M) continue;
      double* crow = p.C + (long long)row * p.ldc;
      const double* cin = nullptr;
      if (plain && beta != 0.0) {
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
            crow[col] = !plain ? v : cin ? fma(alpha, v, beta * cin[col]) : alpha * v;
          }
        }
      }
    }
  }
}

// DMMA chain over k-tiles [kt0, kt1) of the tile at (m0, n0), continuing
// from the values already in acc.
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
  __syncthreads();  // stage buffers are reused by the next unit of this CTA
}

// One persistent CTA per range of the tiles x k-tiles work (see "Scheduling"
// above); pieces are walked backwards.
template <class C, bool A_COL, bool VEC2>
__global__ void __launch_bounds__(C::THREADS, C::MINB) dgemm_kernel(DGemmParams p, ChunkPlan pl) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_last;
  double* As = smem;
  double* Bs = smem + C::STAGES * C::template a_stage<A_COL>();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp % C::WARPS_M) * C::WTM, wn = (warp / C::WARPS_M) * C::WTN;
  const int G = gridDim.x, cta = blockIdx.x;
  const long long u0 = pl.U * cta / G, u1 = pl.U * (cta + 1) / G;
  double acc[C::ACC];

  long long u = u1;
  while (u > u0) {
    const int lt = (int)((u - 1) / pl.KT);
    const int ke = (int)(u - (long long)lt * pl.KT);              // piece end (k-tiles, exclusive)
    const int ch = (ke - 1) / pl.kct;
    const int cs = ch * pl.kct, ce = min(pl.KT, cs + pl.kct);
    const int kb = (int)max((long long)cs, u0 - (long long)lt * pl.KT);  // piece begin
    u = (long long)lt * pl.KT + kb;
    const int tile = pl.tile0 + lt;
    const int m0 = (tile / pl.tiles_n) * C::BM, n0 = (tile % pl.tiles_n) * C::BN;

    if (kb > cs) {
      // tail of a chunk whose head CTA cta - 1 computed first: continue its chain
      if (tid == 0) {
        while (ld_acquire_gpu(p.bflags + cta - 1) != pl.epoch) {
        }
      }
      __syncthreads();
      const double* src = p.bslots + (size_t)(cta - 1) * SLOT_DOUBLES + tid;
#pragma unroll
      for (int e = 0; e < C::ACC; ++e) acc[e] = __ldcg(src + (size_t)e * C::THREADS);
    } else if (p.mode == RS_GEMM_CHAIN) {
      load_cin<C>(p, m0, n0, wm, wn, g, t, acc);
    } else {
#pragma unroll
      for (int e = 0; e < C::ACC; ++e) acc[e] = 0.0;
    }
    mainloop<C, A_COL, VEC2>(p, As, Bs, m0, n0, kb, ke, acc);

    if (ke < ce) {
      // head of a chunk continued by CTA cta + 1: publish the chain value
      double* dst = p.bslots + (size_t)cta * SLOT_DOUBLES + tid;
#pragma unroll
      for (int e = 0; e < C::ACC; ++e) __stcg(dst + (size_t)e * C::THREADS, acc[e]);
      __threadfence();
      __syncthreads();
      if (tid == 0) st_release_gpu(p.bflags + cta, pl.epoch);
      continue;
    }
    // the chunk is complete
    if (pl.nch == 1) {
      if (p.mode == RS_GEMM_FOLD) {
        double v[C::ACC];
        load_cin<C>(p, m0, n0, wm, wn, g, t, v);
#pragma unroll
        for (int e = 0; e < C::ACC; ++e) v[e] += acc[e];
        epilogue_store<C>(p, m0, n0, wm, wn, g, t, v);
      } else {
        epilogue_store<C>(p, m0, n0, wm, wn, g, t, acc);
      }
      continue;
    }
    // element-major slot layout: coalesced stores here and loads in the fold
    double* slot = p.slots + ((size_t)lt * pl.nch + ch) * SLOT_DOUBLES + tid;
#pragma unroll
    for (int e = 0; e < C::ACC; ++e) __stcg(slot + (size_t)e * C::THREADS, acc[e]);
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(p.tickets + lt, 1) == pl.nch - 1;
    __syncthreads();
    if (!s_last) continue;
    __threadfence();
    // last chunk of the tile to arrive: fold the chunk partials in chunk order
    const double* base = p.slots + (size_t)lt * pl.nch * SLOT_DOUBLES + tid;
    if (p.mode == RS_GEMM_FOLD) {
      load_cin<C>(p, m0, n0, wm, wn, g, t, acc);
#pragma unroll
      for (int e = 0; e < C::ACC; ++e) acc[e] += __ldcg(base + (size_t)e * C::THREADS);
    } else {
#pragma unroll
      for (int e = 0; e < C::ACC; ++e) acc[e] = __ldcg(base + (size_t)e * C::THREADS);
    }
    for (int c = 1; c < pl.nch; ++c) {
      const double* src = base + (size_t)c * SLOT_DOUBLES;
#pragma unroll
      for (int e = 0; e < C::ACC; ++e) acc[e] += __ldcg(src + (size_t)e * C::THREADS);
    }
    epilogue_store<C>(p, m0, n0, wm, wn, g, t, acc);
    if (tid == 0) p.tickets[lt] = 0;  // ready for the next launch on this workspace
  }
}

// Boundary-flag values: one process-wide counter shared by every kernel
// instantiation (they share the flag words), never 0 (the zeroed workspace).
static std::atomic<unsigned> g_epoch{1};
static unsigned next_epoch() {
  unsigned e = g_epoch.fetch_add(1);
  return e != 0 ? e : g_epoch.fetch_add(1);
}

template <class C, bool A_COL, bool VEC2>
static int launch_dgemm_t(const DGemmParams& p, int kc, cudaStream_t st) {
  constexpr size_t smem = C::template smem<A_COL>();
  // set on every launch: the attribute is per device and one process may drive several
  cudaFuncSetAttribute(dgemm_kernel<C, A_COL, VEC2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  ChunkPlan pl;
  pl.tiles_n = (p.N + C::BN - 1) / C::BN;
  const int tiles_m = (p.M + C::BM - 1) / C::BM;
  const long long tiles = (long long)pl.tiles_n * tiles_m;
  pl.KT = std::max(1, (p.K + C::BK - 1) / C::BK);  // K = 0: one empty k-tile, so the epilogue runs
  pl.kct = kc / C::BK;
  pl.nch = std::max(1, (pl.KT + pl.kct - 1) / pl.kct);
  const int slots = std::min(nsm * C::MINB, GEMM_MAX_CTAS);
  // tile groups: as many tiles per launch as the partial slots hold, balanced
  const long long per = pl.nch == 1 ? tiles : std::max<long long>(1, p.nslots / pl.nch);
  const long long ngroups = (tiles + per - 1) / per;
  for (long long gi = 0; gi < ngroups; ++gi) {
    const long long t0 = tiles * gi / ngroups, t1 = tiles * (gi + 1) / ngroups;
    pl.tile0 = (int)t0;
    pl.U = (t1 - t0) * pl.KT;
    pl.epoch = next_epoch();
    const int G = (int)std::min<long long>(std::max<long long>(pl.U, 1), slots);
    dgemm_kernel<C, A_COL, VEC2><<<G, C::THREADS, smem, st>>>(p, pl);
    count_launch(1);
  }
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

static bool al16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; }

int launch_dgemm(const DGemmParams& p, bool a_col, int kc, cudaStream_t st) {
  if (p.M < 0 || p.N < 0 || p.K < 0) return RS_ERR_ARG;
  if (p.mode != RS_GEMM_PLAIN && p.mode != RS_GEMM_FOLD && p.mode != RS_GEMM_CHAIN) return RS_ERR_ARG;
  if (p.mode != RS_GEMM_PLAIN && p.Cin == nullptr) return RS_ERR_ARG;
  if (kc <= 0) kc = gemm_chunk(p.K);
  if (kc >= p.K) kc = std::max(32, (p.K + 31) / 32 * 32);  // one chunk: any kc >= K means the same
  if (kc % 32 != 0) return RS_ERR_ARG;
  if (p.mode == RS_GEMM_CHAIN && kc < p.K) return RS_ERR_ARG;  // a chain continues inside one chunk
  if (p.M == 0 || p.N == 0) return RS_OK;
  if (p.slots == nullptr || p.tickets == nullptr || p.nslots < 1) return RS_ERR_ARG;
  const bool vec2 = al16(p.A) && al16(p.B) && (p.lda % 2 == 0) && (p.ldb % 2 == 0);
  if (a_col)
    return vec2 ? launch_dgemm_t<CfgCol, true, true>(p, kc, st) : launch_dgemm_t<CfgCol, true, false>(p, kc, st);
  return vec2 ? launch_dgemm_t<CfgRow, false, true>(p, kc, st) : launch_dgemm_t<CfgRow, false, false>(p, kc, st);
}

}  // namespace rs
