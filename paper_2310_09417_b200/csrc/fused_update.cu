// Fused absorb(t) + Schur(t+1): one pass over the interpolation block T per
// adaptive step (`skeleton.py:439-454`: `_extend_state` of block t followed by
// `_schur_of_block` of block t+1, on the T form T = L2 L1^{-1}).
//
//   T'[i, :k]      = T[sub[nc+i], :k] - W_hat[i, :] * T[sub[0..nc), :k]   (update)
//   T'[i, k:k+nc]  = W_hat[i, :]                                          (written before)
//   S'[i, :]       = Y'[perm'[k'+i], :] - sum_c T'[i, c] * Y'[perm'[c], :]  (next Schur block)
//
// The unfused path streams T twice per block (rank update, then the Schur
// GEMM re-reads T').  Here every 64 x 32 tile of T' is produced in registers,
// stored once, staged in shared memory and immediately multiplied into the
// 64 x 64 Schur accumulator of its row strip: both DMMA products run on one
// read of T and one write of T', so the pass is DMMA-bound (per tile 2 x 64 x
// 32 x 64 FMAs against 32 KB of HBM traffic).
//
// Work units are (row strip, 32-column tile) pairs in strip-major order,
// split evenly over 2 x #SM persistent CTAs (stream-K over column tiles).  A
// CTA that owns a whole strip finishes S' directly; split strips leave
// partial accumulators that a fixup kernel adds in CTA (= column) order, so
// the result is deterministic.  Preconditions (else the caller uses the
// unfused kernels): nc == 64, k % 32 == 0, 16-byte aligned rows.
#include "common.cuh"
#include "rskel_internal.h"

namespace rs {

constexpr int FBM = 64, FBN = 32, FNB = 64, FK = 64;  // strip rows, tile cols, Schur width, W_hat width
constexpr int FTHREADS = 256;
constexpr int FA_LD = FK + 4;    // W_hat strip [64][68]
constexpr int FB_LD = FBN + 4;   // T_p tile   [64][36]
constexpr int FC_LD = FBN + 4;   // Cin / T' tile [64][36]
constexpr int FY_LD = FNB + 4;   // Y' rows    [32][68]
constexpr int FA_ELEMS = FBM * FA_LD;
constexpr int FSTAGE = FK * FB_LD + FBM * FC_LD + FBN * FY_LD;
constexpr size_t F_SMEM = sizeof(double) * (2 * FA_ELEMS + 2 * FSTAGE);
constexpr int F_CTAS_PER_SM = 1;

struct FusedParams {
  int Rn;                 // rows of T' (= R - nc)
  int k, nc, kn;          // old rank, block width (64), new rank
  const double* T;        // old T, ld = k
  const int64_t* sub;     // panel positions -> rows of old T / S
  double* Tn;             // new T, ld = kn; columns [k, kn) hold W_hat already
  const double* Y;        // next sketch block, m x 64, ld = 64
  const int64_t* perm;    // new perm (skeletons perm[:kn], then T' row order)
  double* S;              // out: next Schur block, Rn x 64
  double* partials;       // stream-K partial accumulators
  int ctiles, strips, G;
  long long U;
};

RS_DEV long long f_u0(const FusedParams& p, int c) { return (long long)c * p.U / p.G; }

__global__ void __launch_bounds__(FTHREADS, F_CTAS_PER_SM) fused_absorb_schur_kernel(FusedParams p) {
  extern __shared__ __align__(16) double fsm[];
  double* Abuf = fsm;                    // [2][FBM][FA_LD]
  double* Sbuf = fsm + 2 * FA_ELEMS;     // [2][stage]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int c = blockIdx.x;
  const long long u_begin = f_u0(p, c), u_end = f_u0(p, c + 1);
  if (u_begin >= u_end) return;
  const int ktiles = p.k / FBN;  // update tiles per strip; the rest are W_hat tiles

  auto load = [&](long long u, int buf, bool with_a) {
    const int s = (int)(u / p.ctiles), j = (int)(u % p.ctiles);
    const int n0 = j * FBN, r0 = s * FBM;
    double* bs = Sbuf + buf * FSTAGE;
    double* cs = bs + FK * FB_LD;
    double* ys = cs + FBM * FC_LD;
    if (with_a) {
      double* as = Abuf + (s & 1) * FA_ELEMS;
      for (int e = tid; e < FBM * (FK / 2); e += FTHREADS) {
        const int r = e / (FK / 2), cc = (e % (FK / 2)) * 2;
        const bool ok = r0 + r < p.Rn;
        cp_async16(as + r * FA_LD + cc, ok ? p.Tn + (long long)(r0 + r) * p.kn + p.k + cc : p.Tn, ok ? 16 : 0);
      }
    }
    const bool upd = j < ktiles;
    if (upd) {  // T_p tile: rows sub[0..nc) of old T
      for (int e = tid; e < FK * (FBN / 2); e += FTHREADS) {
        const int r = e / (FBN / 2), cc = (e % (FBN / 2)) * 2;
        const bool ok = r < p.nc;
        cp_async16(bs + r * FB_LD + cc, ok ? p.T + p.sub[r] * (long long)p.k + n0 + cc : p.T, ok ? 16 : 0);
      }
    }
    for (int e = tid; e < FBM * (FBN / 2); e += FTHREADS) {  // Cin (update) or W_hat columns of T'
      const int r = e / (FBN / 2), cc = (e % (FBN / 2)) * 2;
      const bool ok = r0 + r < p.Rn;
      const double* src = p.T;
      if (ok) src = upd ? p.T + p.sub[p.nc + r0 + r] * (long long)p.k + n0 + cc
                        : p.Tn + (long long)(r0 + r) * p.kn + n0 + cc;
      cp_async16(cs + r * FC_LD + cc, src, ok ? 16 : 0);
    }
    for (int e = tid; e < FBN * (FNB / 2); e += FTHREADS) {  // Y' rows of the tile's skeletons
      const int q = e / (FNB / 2), cc = (e % (FNB / 2)) * 2;
      cp_async16(ys + q * FY_LD + cc, p.Y + p.perm[n0 + q] * (long long)FNB + cc, 16);
    }
  };

  // Schur accumulator: warp tile 16 x 32 of the 64 x 64 strip block.
  const int wm = (warp & 3) * 16;
  const int wn_s = (warp >> 2) * 32;
  const int wn_u = (warp >> 2) * 16;  // update warp tile 16 x 16 of the 64 x 32 tile
  double acc_s[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc_s[j][e] = 0.0;

  auto finish_strip = [&](int s, bool whole, int slot) {
    if (whole) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = s * FBM + wm + g + 8 * h;
        if (r >= p.Rn) continue;
        const double* yrow = p.Y + p.perm[p.kn + r] * (long long)FNB;
        double* srow = p.S + (long long)r * FNB;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int col = wn_s + 8 * j + 2 * t;
          const double2 yv = *reinterpret_cast<const double2*>(yrow + col);
          *reinterpret_cast<double2*>(srow + col) =
              make_double2(yv.x - acc_s[j][2 * h], yv.y - acc_s[j][2 * h + 1]);
        }
      }
    } else {
      double* dst = p.partials + (size_t)slot * (FTHREADS * 16) + tid;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) dst[(j * 4 + e) * FTHREADS] = acc_s[j][e];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc_s[j][e] = 0.0;
  };

  load(u_begin, 0, true);
  cp_async_commit();
  int strip_start_unit_is_mine = (int)(u_begin % p.ctiles == 0);
  for (long long u = u_begin; u < u_end; ++u) {
    const int buf = (int)((u - u_begin) & 1);
    const int s = (int)(u / p.ctiles), j = (int)(u % p.ctiles);
    if (u + 1 < u_end) load(u + 1, buf ^ 1, (u + 1) % p.ctiles == 0);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* as = Abuf + (s & 1) * FA_ELEMS;
    const double* bs = Sbuf + buf * FSTAGE;
    double* cs = const_cast<double*>(bs) + FK * FB_LD;
    const double* ys = cs + FBM * FC_LD;
    const int n0 = j * FBN;
    if (j < ktiles) {
      // ---- update: T' tile = Cin - W_hat T_p (warp tile 16 x 16) ----
      double acc_u[2][4];
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc_u[q][e] = 0.0;
#pragma unroll
      for (int kk = 0; kk < FK; kk += 4) {
        const double a0 = as[(wm + g) * FA_LD + kk + t];
        const double a1 = as[(wm + g + 8) * FA_LD + kk + t];
#pragma unroll
        for (int q = 0; q < 2; ++q) dmma_16x8x4(acc_u[q], a0, a1, bs[(kk + t) * FB_LD + wn_u + 8 * q + g]);
      }
      const int rbase = s * FBM;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = wm + g + 8 * h;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int col = wn_u + 8 * q + 2 * t;
          double2* cp = reinterpret_cast<double2*>(cs + r * FC_LD + col);
          const double2 cin = *cp;
          const double2 v = make_double2(cin.x - acc_u[q][2 * h], cin.y - acc_u[q][2 * h + 1]);
          *cp = v;
          if (rbase + r < p.Rn)
            *reinterpret_cast<double2*>(p.Tn + (long long)(rbase + r) * p.kn + n0 + col) = v;
        }
      }
      __syncthreads();  // T' tile complete in shared memory
    }
    // ---- Schur: S_acc += T' tile (64 x 32) * Y'[perm'[n0..n0+32)] (32 x 64) ----
#pragma unroll
    for (int kk = 0; kk < FBN; kk += 4) {
      const double a0 = cs[(wm + g) * FC_LD + kk + t];
      const double a1 = cs[(wm + g + 8) * FC_LD + kk + t];
#pragma unroll
      for (int q = 0; q < 4; ++q) dmma_16x8x4(acc_s[q], a0, a1, ys[(kk + t) * FY_LD + wn_s + 8 * q + g]);
    }
    const bool strip_end = (j == p.ctiles - 1) || (u + 1 == u_end);
    if (strip_end) {
      const bool whole = strip_start_unit_is_mine && j == p.ctiles - 1;
      // partial slots: 2c = strip tail of this CTA's first strip (started
      // before us), 2c+1 = head of the strip we stop inside
      const int slot = strip_start_unit_is_mine ? 2 * c + 1 : 2 * c;
      finish_strip(s, whole, slot);
      strip_start_unit_is_mine = 1;
    }
    __syncthreads();  // stage `buf` is refilled by the next iteration's prefetch
  }
  cp_async_wait<0>();
}

// Add the partial accumulators of every split strip in CTA order, finish S'.
__global__ void __launch_bounds__(FTHREADS) fused_fixup_kernel(FusedParams p) {
  const int s = blockIdx.x;
  const long long ub = (long long)s * p.ctiles, ue = ub + p.ctiles;
  auto owner = [&](long long u) {
    int c = (int)((u * p.G) / p.U);
    while (c + 1 < p.G && f_u0(p, c + 1) <= u) ++c;
    while (c > 0 && f_u0(p, c) > u) --c;
    return c;
  };
  const int clo = owner(ub), chi = owner(ue - 1);
  if (clo == chi) return;  // whole strip finished by its CTA
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp & 3) * 16, wn_s = (warp >> 2) * 32;
  double acc[16];
  {
    // the first CTA started the strip: its slot is 2c+1 (head)
    const double* src = p.partials + (size_t)(2 * clo + 1) * (FTHREADS * 16) + tid;
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = src[e * FTHREADS];
  }
  for (int c = clo + 1; c <= chi; ++c) {
    // later CTAs entered mid-strip: slot 2c (their first strip)
    const double* src = p.partials + (size_t)(2 * c) * (FTHREADS * 16) + tid;
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] += src[e * FTHREADS];
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = s * FBM + wm + g + 8 * h;
    if (r >= p.Rn) continue;
    const double* yrow = p.Y + p.perm[p.kn + r] * (long long)FNB;
    double* srow = p.S + (long long)r * FNB;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = wn_s + 8 * j + 2 * t;
      srow[col] = yrow[col] - acc[j * 4 + 2 * h];
      srow[col + 1] = yrow[col + 1] - acc[j * 4 + 2 * h + 1];
    }
  }
}

size_t fused_partials_bytes(int nsm) {
  return sizeof(double) * 2 * (size_t)nsm * F_CTAS_PER_SM * FTHREADS * 16;
}

int launch_fused_absorb_schur(int Rn, int k, int nc, const double* T, const int64_t* sub, double* Tn,
                              const double* Y, const int64_t* perm, double* S, double* partials,
                              cudaStream_t st) {
  if (nc != FK || k % FBN != 0 || Rn < 0 || k < 0) return RS_ERR_ARG;
  if (Rn == 0) return RS_OK;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  FusedParams p{};
  p.Rn = Rn; p.k = k; p.nc = nc; p.kn = k + nc;
  p.T = T; p.sub = sub; p.Tn = Tn; p.Y = Y; p.perm = perm; p.S = S; p.partials = partials;
  p.ctiles = p.kn / FBN;
  p.strips = (Rn + FBM - 1) / FBM;
  p.U = (long long)p.ctiles * p.strips;
  const long long slots = (long long)nsm * F_CTAS_PER_SM;
  p.G = (int)(p.U < slots ? p.U : slots);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(fused_absorb_schur_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F_SMEM);
    configured = true;
  }
  fused_absorb_schur_kernel<<<p.G, FTHREADS, F_SMEM, st>>>(p);
  fused_fixup_kernel<<<p.strips, FTHREADS, 0, st>>>(p);
  count_launch(2);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

}  // namespace rs
