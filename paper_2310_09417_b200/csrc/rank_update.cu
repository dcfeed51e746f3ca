// Rank-<=64 update with row gathers, the T-form absorb step
// (`_extend_state`, skeleton.py:326-351, on T = L2 L1^{-1}):
//
//   C[i, :] = Cin[cidx[i], :] - A[i, :K] * B[bidx[0..K), :]      (K <= 64)
//
// with C = T_new[:, :k] (M = m-k-nc rows, N = k columns), A = W_hat, B = the
// pivot rows T[P_hat] and Cin = T[Q_hat].  The shape is short-K / huge-MN, so
// the kernel is organised around the output stream rather than a k-pipeline:
//  * persistent CTAs (2 per SM) walk contiguous chunks of 64 x 64 tiles, so
//    the 64 x 64 A strip stays resident in shared memory across a row strip;
//  * the B tile of the next tile is prefetched with cp.async (double buffer);
//  * the Cin tile is prefetched straight into registers at the top of the
//    tile (read-only path), so its HBM latency hides behind the 16 DMMA
//    k-steps, and C is written with 16-byte stores.
// Per tile: 64x64x64 FMAs, 32 KB of Cin read and 32 KB of C written.
#include "common.cuh"
#include "rskel_internal.h"

namespace rs {

constexpr int UBM = 64, UBN = 64, UK = 64;
constexpr int UTHREADS = 256;                       // 8 warps: 2 (M) x 4 (N), warp tile 32 x 16
constexpr int UWM = 2, UWN = 4, UWTM = UBM / UWM, UWTN = UBN / UWN;
constexpr int UMT = UWTM / 16, UNT = UWTN / 8;      // 2 x 2 m16n8 tiles per warp
constexpr int UA_LD = UK + 4, UB_LD = UBN + 4;  // = 4 (mod 16): conflict-free 64-bit fragment loads
constexpr size_t U_SMEM = sizeof(double) * (UBM * UA_LD + 2 * UK * UB_LD);

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

template <bool VEC2>
__device__ __forceinline__ void ru_copy(double* dst, const double* src, int valid) {
  // valid: number of valid doubles in this chunk (0..2 for VEC2, 0..1 otherwise)
  if (valid == 0) {
    dst[0] = 0.0;
    if constexpr (VEC2) dst[1] = 0.0;
    return;
  }
  if constexpr (VEC2) cp_async16(dst, src, valid * 8);
  else cp_async8(dst, src, valid * 8);
}

template <bool VEC2>
__global__ void __launch_bounds__(UTHREADS, 2) rank_update_kernel(RankUpdateParams p) {
  extern __shared__ __align__(16) double usm[];
  double* As = usm;                  // [UBM][UA_LD]
  double* Bs = usm + UBM * UA_LD;    // [2][UK][UB_LD]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp % UWM) * UWTM, wn = (warp / UWM) * UWTN;
  const int G = gridDim.x, c = blockIdx.x;
  const int t0 = (int)((long long)c * p.tiles / G), t1 = (int)((long long)(c + 1) * p.tiles / G);
  if (t0 >= t1) return;
  constexpr int V = VEC2 ? 2 : 1;

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
      ru_copy<VEC2>(bs + r * UB_LD + nc, valid ? p.B + p.bidx[r] * p.ldb + gn : p.B, valid);
    }
  };

  int strip = t0 / p.tiles_n;
  load_A(strip * UBM);
  load_B((t0 % p.tiles_n) * UBN, 0);
  cp_async_commit();

  for (int tile = t0; tile < t1; ++tile) {
    const int buf = (tile - t0) & 1;
    const int tstrip = tile / p.tiles_n;
    const int m0 = tstrip * UBM, n0 = (tile % p.tiles_n) * UBN;
    if (tstrip != strip) {  // new row strip (rare: chunks are contiguous): reload A
      __syncthreads();       // everyone is done with the old A
      strip = tstrip;
      load_A(m0);
      cp_async_commit();
    }
    // Cin of this tile -> registers (consumed by the epilogue, after the MMAs).
    double cin[UMT][2][UNT][2];
#pragma unroll
    for (int i = 0; i < UMT; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gm = m0 + wm + 16 * i + g + 8 * h;
        const double* crow = gm < p.M ? p.Cin + p.cidx[gm] * p.ldcin : nullptr;
#pragma unroll
        for (int j = 0; j < UNT; ++j) {
          const int gn = n0 + wn + 8 * j + 2 * t;
          if (crow != nullptr && VEC2 && gn + 1 < p.N) {
            const double2 v = __ldg(reinterpret_cast<const double2*>(crow + gn));
            cin[i][h][j][0] = v.x;
            cin[i][h][j][1] = v.y;
          } else {
            cin[i][h][j][0] = (crow != nullptr && gn < p.N) ? __ldg(crow + gn) : 0.0;
            cin[i][h][j][1] = (crow != nullptr && gn + 1 < p.N) ? __ldg(crow + gn + 1) : 0.0;
          }
        }
      }
    // prefetch the next tile's B (its A, if a new strip, is loaded next iteration)
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
    for (int kk = 0; kk < UK; kk += 4) {  // K zero-padded to 64 in shared memory
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
    // epilogue: C = Cin - acc (one rounding, as cin - (a @ b)), 16-byte stores
#pragma unroll
    for (int i = 0; i < UMT; ++i) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gm = m0 + wm + 16 * i + g + 8 * h;
        if (gm >= p.M) continue;
        double* crow = p.C + (long long)gm * p.ldc;
#pragma unroll
        for (int j = 0; j < UNT; ++j) {
          const int gn = n0 + wn + 8 * j + 2 * t;
          const double v0 = cin[i][h][j][0] - acc[i][j][2 * h];
          const double v1 = cin[i][h][j][1] - acc[i][j][2 * h + 1];
          if (VEC2 && gn + 1 < p.N) {
            *reinterpret_cast<double2*>(crow + gn) = make_double2(v0, v1);
          } else {
            if (gn < p.N) crow[gn] = v0;
            if (gn + 1 < p.N) crow[gn + 1] = v1;
          }
        }
      }
    }
    __syncthreads();  // B[buf] is refilled by the next iteration's prefetch
  }
  cp_async_wait<0>();
}

int launch_rank_update(int M, int N, int K, const double* A, long long lda, const double* B,
                       long long ldb, const int64_t* bidx, const double* Cin, long long ldcin,
                       const int64_t* cidx, double* C, long long ldc, cudaStream_t st) {
  if (M < 0 || N < 0 || K < 0 || K > UK) return RS_ERR_ARG;
  if (M == 0 || N == 0) return RS_OK;
  RankUpdateParams p{M, N, K, A, lda, B, ldb, bidx, Cin, ldcin, cidx, C, ldc, 0, 0};
  p.tiles_n = (N + UBN - 1) / UBN;
  p.tiles = p.tiles_n * ((M + UBM - 1) / UBM);
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  const bool vec2 = al16(A) && al16(B) && al16(Cin) && al16(C) && lda % 2 == 0 && ldb % 2 == 0 &&
                    ldcin % 2 == 0 && ldc % 2 == 0;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int slots = 2 * nsm;
  const int G = p.tiles < slots ? p.tiles : slots;
  static bool configured[2] = {false, false};
  if (vec2) {
    if (!configured[1]) {
      cudaFuncSetAttribute(rank_update_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)U_SMEM);
      configured[1] = true;
    }
    rank_update_kernel<true><<<G, UTHREADS, U_SMEM, st>>>(p);
  } else {
    if (!configured[0]) {
      cudaFuncSetAttribute(rank_update_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)U_SMEM);
      configured[0] = true;
    }
    rank_update_kernel<false><<<G, UTHREADS, U_SMEM, st>>>(p);
  }
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

}  // namespace rs
