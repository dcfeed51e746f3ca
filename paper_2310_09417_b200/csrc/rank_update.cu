// Rank-<=64 update with row gathers, the T-form absorb step
// (`_extend_state`, skeleton.py:326-351, on T = L2 L1^{-1}):
//
//   C[i, :] = Cin[cidx[i], :] - A[i, :K] * B[bidx[0..K), :]      (K <= 64)
//
// with C = T_new[:, :k] (M = m-k-nc rows, N = k columns), A = W_hat, B = the
// pivot rows T[P_hat] and Cin = T[Q_hat].  Short K, huge M x N: the kernel is
// a streaming pipeline, not a k-loop.  Every element is one DMMA chain over
// k = 0..K-1 in steps of 4 followed by Cin - acc, whichever kernel runs, so
// the result of a row does not depend on M or on the tile it lands in.
//
//  * rank_update_stream_kernel (default): one CTA per SM walks contiguous
//    128 x 64 tiles; the W_hat strip stays in registers as DMMA fragments,
//    the gathered B and Cin rows stream through a cp.async ring.
//  * rank_update_kernel: the generic cp.async kernel for shapes the
//    streaming kernel cannot take (odd K, N or leading dimensions,
//    misaligned pointers).
#include <cstdlib>

#include "common.cuh"
#include "rskel_internal.h"

namespace rs {

struct RankUpdateParams {
  int M, N, K;
  const double* A;
  long long lda;
  const double* B;
  long long ldb;
  const int64_t* bidx;
  const double* Cin;
  long long ldcin;
  const int64_t* cidx;
  double* C;
  long long ldc;
  int tiles_n, tiles;
};

// -------------------------------------------------- generic cp.async kernel --
constexpr int UBM = 64, UBN = 64, UK = 64;
constexpr int UTHREADS = 256;                       // 8 warps: 2 (M) x 4 (N), warp tile 32 x 16
constexpr int UWM = 2, UWN = 4, UWTM = UBM / UWM, UWTN = UBN / UWN;
constexpr int UMT = UWTM / 16, UNT = UWTN / 8;      // 2 x 2 m16n8 tiles per warp
constexpr int UA_LD = UK + 4, UB_LD = UBN + 4;      // = 4 (mod 16): conflict-free fragment loads
constexpr size_t U_SMEM = sizeof(double) * (UBM * UA_LD + 2 * UK * UB_LD) + sizeof(long long) * UK;

template <bool VEC2>
__device__ __forceinline__ void ru_copy(double* dst, const double* src, int valid) {
  if (valid == 0) {
    dst[0] = 0.0;
    if constexpr (VEC2) dst[1] = 0.0;
    return;
  }
  if constexpr (VEC2) cp_async16(dst, src, valid * 8);
  else cp_async8(dst, src, valid * 8);
}

// Read-only loads as volatile asm: ptxas keeps them ahead of the (volatile)
// DMMA asm, so the Cin stream is in flight during the MMAs.
RS_DEV double2 ldnc2(const double* q) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(q));
  return v;
}
RS_DEV double ldnc1(const double* q) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];\n" : "=d"(v) : "l"(q));
  return v;
}

template <bool VEC2>
__global__ void __launch_bounds__(UTHREADS, 2) rank_update_kernel(RankUpdateParams p) {
  extern __shared__ __align__(16) double usm[];
  double* As = usm;                  // [UBM][UA_LD]
  double* Bs = usm + UBM * UA_LD;    // [2][UK][UB_LD]
  // B row offsets (bidx is fixed for the launch): one global load per row per
  // CTA instead of one dependent load per copied element.
  long long* brow = reinterpret_cast<long long*>(Bs + 2 * UK * UB_LD);  // [UK]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp % UWM) * UWTM, wn = (warp / UWM) * UWTN;
  const int G = gridDim.x, c = blockIdx.x;
  const int t0 = (int)((long long)c * p.tiles / G), t1 = (int)((long long)(c + 1) * p.tiles / G);
  if (t0 >= t1) return;
  constexpr int V = VEC2 ? 2 : 1;
  for (int r = tid; r < UK; r += UTHREADS) brow[r] = r < p.K ? p.bidx[r] * p.ldb : 0;
  __syncthreads();

  auto load_A = [&](int m0) {
    for (int e = tid; e < UBM * (UK / V); e += UTHREADS) {
      const int r = e / (UK / V), kc = (e % (UK / V)) * V;
      const int gm = m0 + r;
      const int valid = (gm < p.M && kc < p.K) ? min(V, p.K - kc) : 0;
      ru_copy<VEC2>(As + r * UA_LD + kc, p.A + (long long)gm * p.lda + kc, valid);
    }
  };
  auto load_B = [&](int n0, int buf) {
    double* bs = Bs + buf * UK * UB_LD;
    for (int e = tid; e < UK * (UBN / V); e += UTHREADS) {
      const int r = e / (UBN / V), nc = (e % (UBN / V)) * V;
      const int gn = n0 + nc;
      const int valid = (r < p.K && gn < p.N) ? min(V, p.N - gn) : 0;
      ru_copy<VEC2>(bs + r * UB_LD + nc, valid ? p.B + brow[r] + gn : p.B, valid);
    }
  };
  // Cin row pointers of this thread's 2 x UMT accumulator rows: they change
  // only with the strip, so the gathered-index loads leave the tile loop.
  const double* crow[UMT][2];
  auto set_rows = [&](int m0) {
#pragma unroll
    for (int i = 0; i < UMT; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gm = m0 + wm + 16 * i + g + 8 * h;
        crow[i][h] = gm < p.M ? p.Cin + p.cidx[gm] * p.ldcin : nullptr;
      }
  };

  int strip = t0 / p.tiles_n;
  set_rows(strip * UBM);
  load_A(strip * UBM);
  load_B((t0 % p.tiles_n) * UBN, 0);
  cp_async_commit();
  for (int tile = t0; tile < t1; ++tile) {
    const int buf = (tile - t0) & 1;
    const int tstrip = tile / p.tiles_n;
    const int m0 = tstrip * UBM, n0 = (tile % p.tiles_n) * UBN;
    if (tstrip != strip) {
      __syncthreads();
      strip = tstrip;
      set_rows(m0);
      load_A(m0);
      cp_async_commit();
    }
    double cin[UMT][2][UNT][2];
#pragma unroll
    for (int i = 0; i < UMT; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double* cr = crow[i][h];
#pragma unroll
        for (int j = 0; j < UNT; ++j) {
          const int gn = n0 + wn + 8 * j + 2 * t;
          if (VEC2 && cr != nullptr && gn + 1 < p.N) {
            const double2 v = ldnc2(cr + gn);
            cin[i][h][j][0] = v.x;
            cin[i][h][j][1] = v.y;
          } else {
            cin[i][h][j][0] = (cr != nullptr && gn < p.N) ? ldnc1(cr + gn) : 0.0;
            cin[i][h][j][1] = (cr != nullptr && gn + 1 < p.N) ? ldnc1(cr + gn + 1) : 0.0;
          }
        }
      }
    if (tile + 1 < t1) load_B(((tile + 1) % p.tiles_n) * UBN, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* bs = Bs + buf * UK * UB_LD;
    double acc[UMT][UNT][4];
#pragma unroll
    for (int i = 0; i < UMT; ++i)
#pragma unroll
      for (int j = 0; j < UNT; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;
#pragma unroll
    for (int kk = 0; kk < UK; kk += 4) {
      double a[UMT][2], b[UNT];
#pragma unroll
      for (int i = 0; i < UMT; ++i) {
        const int mr = wm + 16 * i + g;
        a[i][0] = As[mr * UA_LD + kk + t];
        a[i][1] = As[(mr + 8) * UA_LD + kk + t];
      }
#pragma unroll
      for (int j = 0; j < UNT; ++j) b[j] = bs[(kk + t) * UB_LD + wn + 8 * j + g];
#pragma unroll
      for (int i = 0; i < UMT; ++i)
#pragma unroll
        for (int j = 0; j < UNT; ++j) dmma_16x8x4(acc[i][j], a[i][0], a[i][1], b[j]);
    }
#pragma unroll
    for (int i = 0; i < UMT; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gm = m0 + wm + 16 * i + g + 8 * h;
        if (gm >= p.M) continue;
        double* cw = p.C + (long long)gm * p.ldc;
#pragma unroll
        for (int j = 0; j < UNT; ++j) {
          const int gn = n0 + wn + 8 * j + 2 * t;
          const double v0 = cin[i][h][j][0] - acc[i][j][2 * h];
          const double v1 = cin[i][h][j][1] - acc[i][j][2 * h + 1];
          if (VEC2 && gn + 1 < p.N) {
            *reinterpret_cast<double2*>(cw + gn) = make_double2(v0, v1);
          } else {
            if (gn < p.N) cw[gn] = v0;
            if (gn + 1 < p.N) cw[gn + 1] = v1;
          }
        }
      }
    __syncthreads();
  }
  cp_async_wait<0>();
}

// ------------------------------------------------- streaming kernel (v3) --
// One CTA per SM walks its contiguous range of 64 x 64 output tiles
// (strip-major).  The A strip (64 x K, W_hat) lives in registers as DMMA
// fragments for the whole strip; the B chunk (K x 64, gathered rows of
// T[P_hat]) and the Cin chunk (64 x 64, gathered rows of T[Q_hat]) stream
// through a 3-stage cp.async ring, so the HBM reads of tile i+2 are in flight
// while tile i is multiplied; C = Cin - A B leaves from registers with 16-byte
// stores.  8 warps: 4 (M, 16 rows) x 2 (N, 32 cols); 4 independent
// accumulators per warp.  B rows at ld 68 (= 4 mod 16: conflict-free 64-bit
// fragment loads), Cin rows at ld 72 (= 8 mod 16: conflict-free 128-bit
// epilogue loads).
template <int BM, int WARPS_N, int STAGES>
struct R3Cfg {
  static constexpr int BN = 64, K = 64, THREADS = 256;
  static constexpr int WARPS_M = 8 / WARPS_N;
  static_assert(WARPS_M * 16 == BM, "8 warps: BM = 16 * warps along M");
  static constexpr int NT = BN / 8 / WARPS_N;  // n8 accumulators per warp
  static constexpr int BLD = BN + 4, CLD = BN + 8;
  static constexpr int STAGE = K * BLD + BM * CLD;  // doubles
  static constexpr size_t SMEM = sizeof(double) * STAGES * STAGE;
  static constexpr int BCH = K * BN / 2 / THREADS;   // 16-byte B chunks per thread (8)
  static constexpr int CCH = BM * BN / 2 / THREADS;  // 16-byte Cin chunks per thread
};

template <int BM, int WARPS_N, int STAGES>
__global__ void __launch_bounds__(256, 1) rank_update_stream_kernel(RankUpdateParams p) {
  using C = R3Cfg<BM, WARPS_N, STAGES>;
  extern __shared__ __align__(16) double r3sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp % C::WARPS_M) * 16, wn = (warp / C::WARPS_M) * (C::BN / WARPS_N);
  const int G = gridDim.x, c = blockIdx.x;
  const int t0 = (int)((long long)c * p.tiles / G), t1 = (int)((long long)(c + 1) * p.tiles / G);
  if (t0 >= t1) return;
  const int ntile = t1 - t0;

  // copy geometry: chunk q = tid + 256 i -> row q / 32 (32 chunks = 64 doubles
  // per row), 16-byte column (q % 32) * 2
  const int crow0 = tid >> 5, ccol = (tid & 31) * 2;
  long long boff[C::BCH];  // B row offsets: bidx is fixed for the launch
#pragma unroll
  for (int i = 0; i < C::BCH; ++i) {
    const int r = crow0 + 8 * i;
    boff[i] = r < p.K ? p.bidx[r] * p.ldb : -1;
  }
  long long coff[C::CCH];  // Cin row offsets of the prefetch strip
  int pf_strip = -1;

  auto issue = [&](int li) {  // loads of local tile li into stage li % STAGES
    const int tile = t0 + li;
    const int strip = tile / p.tiles_n;
    const int m0 = strip * BM, n0 = (tile - strip * p.tiles_n) * C::BN;
    if (strip != pf_strip) {
      pf_strip = strip;
#pragma unroll
      for (int i = 0; i < C::CCH; ++i) {
        const int gm = m0 + crow0 + 8 * i;
        coff[i] = gm < p.M ? p.cidx[gm] * p.ldcin : -1;
      }
    }
    double* st = r3sm + (li % STAGES) * C::STAGE;
    double* bs = st;
    double* cs = st + C::K * C::BLD;
    const int gn = n0 + ccol;
    const int nv = gn < p.N ? min(2, p.N - gn) : 0;
#pragma unroll
    for (int i = 0; i < C::BCH; ++i) {
      const bool bv = boff[i] >= 0 && nv > 0;
      cp_async16(bs + (crow0 + 8 * i) * C::BLD + ccol, bv ? p.B + boff[i] + gn : p.B, bv ? nv * 8 : 0);
    }
#pragma unroll
    for (int i = 0; i < C::CCH; ++i) {
      const bool cv = coff[i] >= 0 && nv > 0;
      cp_async16(cs + (crow0 + 8 * i) * C::CLD + ccol, cv ? p.Cin + coff[i] + gn : p.Cin, cv ? nv * 8 : 0);
    }
  };

  double af[16][2];  // A fragments of this warp's 16 rows, all K/4 k-steps
  int a_strip = -1;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ntile) issue(s);
    cp_async_commit();
  }
  for (int li = 0; li < ntile; ++li) {
    const int tile = t0 + li;
    const int strip = tile / p.tiles_n;
    const int m0 = strip * BM, n0 = (tile - strip * p.tiles_n) * C::BN;
    if (strip != a_strip) {  // new strip: A fragments straight from global
      a_strip = strip;
      const int r0 = m0 + wm + g, r1 = r0 + 8;
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) {
        const int kc = 4 * ks + t;
        af[ks][0] = (r0 < p.M && kc < p.K) ? p.A[(long long)r0 * p.lda + kc] : 0.0;
        af[ks][1] = (r1 < p.M && kc < p.K) ? p.A[(long long)r1 * p.lda + kc] : 0.0;
      }
    }
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (li + STAGES - 1 < ntile) issue(li + STAGES - 1);
    cp_async_commit();
    const double* st = r3sm + (li % STAGES) * C::STAGE;
    const double* bs = st;
    const double* cs = st + C::K * C::BLD;
    double acc[C::NT][4];
#pragma unroll
    for (int j = 0; j < C::NT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[j][e] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 16; ++ks) {
#pragma unroll
      for (int j = 0; j < C::NT; ++j) {
        const double b = bs[(4 * ks + t) * C::BLD + wn + 8 * j + g];
        dmma_16x8x4(acc[j], af[ks][0], af[ks][1], b);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int lr = wm + g + 8 * h;
      const int gm = m0 + lr;
      if (gm >= p.M) continue;
      double* cw = p.C + (long long)gm * p.ldc;
#pragma unroll
      for (int j = 0; j < C::NT; ++j) {
        const int ln = wn + 8 * j + 2 * t;
        const int gn = n0 + ln;
        const double2 ci = *reinterpret_cast<const double2*>(cs + lr * C::CLD + ln);
        const double v0 = ci.x - acc[j][2 * h], v1 = ci.y - acc[j][2 * h + 1];
        if (gn + 1 < p.N) {
          *reinterpret_cast<double2*>(cw + gn) = make_double2(v0, v1);
        } else if (gn < p.N) {
          cw[gn] = v0;
        }
      }
    }
  }
  cp_async_wait<0>();
}

template <int BM, int WARPS_N, int STAGES>
static void launch_stream(RankUpdateParams p, int nsm, cudaStream_t st) {
  using C = R3Cfg<BM, WARPS_N, STAGES>;
  p.tiles_n = (p.N + C::BN - 1) / C::BN;
  p.tiles = p.tiles_n * ((p.M + BM - 1) / BM);
  const int G = p.tiles < nsm ? p.tiles : nsm;
  // set on every launch: the attribute is per device
  cudaFuncSetAttribute(rank_update_stream_kernel<BM, WARPS_N, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)C::SMEM);
  rank_update_stream_kernel<BM, WARPS_N, STAGES><<<G, 256, C::SMEM, st>>>(p);
}

int launch_rank_update(int M, int N, int K, const double* A, long long lda, const double* B,
                       long long ldb, const int64_t* bidx, const double* Cin, long long ldcin,
                       const int64_t* cidx, double* C, long long ldc, cudaStream_t st) {
  if (M < 0 || N < 0 || K < 0 || K > UK) return RS_ERR_ARG;
  if (M == 0 || N == 0) return RS_OK;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  const bool vec2 = al16(A) && al16(B) && al16(Cin) && al16(C) && lda % 2 == 0 && ldb % 2 == 0 &&
                    ldcin % 2 == 0 && ldc % 2 == 0;
  RankUpdateParams p{M, N, K, A, lda, B, ldb, bidx, Cin, ldcin, cidx, C, ldc, 0, 0};
  if (vec2 && K > 0 && K % 2 == 0 && N % 2 == 0) {
#if !defined(RS_RU_VARIANT) || RS_RU_VARIANT == 0  // (experiment builds: tools/build_ru_cfg.sh)
    launch_stream<128, 1, 2>(p, nsm, st);
#elif RS_RU_VARIANT == 1
    launch_stream<64, 2, 3>(p, nsm, st);
#else
    launch_stream<64, 2, 2>(p, nsm, st);
#endif
  } else {
    p.tiles_n = (N + UBN - 1) / UBN;
    p.tiles = p.tiles_n * ((M + UBM - 1) / UBM);
    const int G = p.tiles < 2 * nsm ? p.tiles : 2 * nsm;
    if (vec2) {
      cudaFuncSetAttribute(rank_update_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)U_SMEM);
      rank_update_kernel<true><<<G, UTHREADS, U_SMEM, st>>>(p);
    } else {
      cudaFuncSetAttribute(rank_update_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)U_SMEM);
      rank_update_kernel<false><<<G, UTHREADS, U_SMEM, st>>>(p);
    }
  }
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

}  // namespace rs
