// Rank-<=64 update with row gathers, the T-form absorb step
// (`_extend_state`, skeleton.py:326-351, on T = L2 L1^{-1}):
//
//   C[i, :] = Cin[cidx[i], :] - A[i, :K] * B[bidx[0..K), :]      (K <= 64)
//
// with C = T_new[:, :k] (M = m-k-nc rows, N = k columns), A = W_hat, B = the
// pivot rows T[P_hat] and Cin = T[Q_hat].  Short K, huge M x N: the kernel is
// a streaming pipeline, not a k-loop.
//
// Warp-specialised persistent design (one CTA per SM):
//  * 1 producer warp issues 1-D bulk async copies (cp.async.bulk, the TMA
//    engine's non-tensor form) of whole gathered rows -- the K B rows and the
//    64 Cin rows of a 64 x 32 output tile, and the 64 x K A strip -- into a
//    4-stage shared-memory ring, completion tracked by mbarrier transaction
//    counts (no per-thread address math or cp.async groups);
//  * 8 consumer warps (warp tile 16 x 16, DMMA m16n8k4) wait on the stage's
//    full barrier, run the 16 k-steps, write C = Cin - A B with 16-byte
//    stores straight from registers, and release the stage.
// Rows are placed at padded strides (68 / 36 doubles, = 4 mod 16) so the
// 64-bit fragment loads are bank-conflict free.  A generic cp.async kernel
// (rank_update_kernel) remains for shapes the bulk path cannot take
// (odd K, N or leading dimensions, misaligned pointers).
#include <cstdlib>

#include "common.cuh"
#include "rskel_internal.h"

namespace rs {

// ------------------------------------------------------------ mbarrier/bulk --
RS_DEV unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
RS_DEV void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
RS_DEV void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
RS_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
RS_DEV void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
RS_DEV void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ------------------------------------------------------------- bulk kernel --
#ifndef RS_RU_WBN
#define RS_RU_WBN 64
#endif
#ifndef RS_RU_STAGES
#define RS_RU_STAGES 2
#endif
constexpr int WBM = 64, WBN = RS_RU_WBN, WK = 64, WSTAGES = RS_RU_STAGES;
constexpr int W_CONSUMERS = 8;                         // warps 0..7: 4 (M) x 2 (N), warp tile 16 x WBN/2
constexpr int WNT = WBN / 16;                          // n8 tiles per warp
constexpr int W_THREADS = (W_CONSUMERS + 1) * 32;      // + producer warp 8
constexpr int WA_LD = WK + 4, WB_LD = WBN + 4, WC_LD = WBN + 4;  // = 4 (mod 16)
constexpr int WA_ELEMS = WBM * WA_LD;
constexpr int WB_ELEMS = WK * WB_LD, WC_ELEMS = WBM * WC_LD;
constexpr int WSTAGE_ELEMS = WB_ELEMS + WC_ELEMS;
constexpr size_t W_SMEM = sizeof(double) * (2 * WA_ELEMS + WSTAGES * WSTAGE_ELEMS) + 1024;

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

__global__ void __launch_bounds__(W_THREADS, 1) rank_update_bulk_kernel(RankUpdateParams p) {
  extern __shared__ __align__(128) double wsm[];
  double* Abuf = wsm;                              // [2][WBM][WA_LD]
  double* Sbuf = wsm + 2 * WA_ELEMS;               // [WSTAGES][B | C]
  uint64_t* bars = reinterpret_cast<uint64_t*>(Sbuf + WSTAGES * WSTAGE_ELEMS);
  uint64_t* full = bars;                           // [WSTAGES]
  uint64_t* empty = bars + WSTAGES;                // [WSTAGES]
  uint64_t* a_full = bars + 2 * WSTAGES;           // [2]
  uint64_t* a_empty = bars + 2 * WSTAGES + 2;      // [2]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, c = blockIdx.x;
  const int t0 = (int)((long long)c * p.tiles / G), t1 = (int)((long long)(c + 1) * p.tiles / G);

  // Zero the K padding of A and B once (the producer only writes columns /
  // rows < K), then initialise the barriers.
  for (int e = tid; e < 2 * WBM * (WA_LD - p.K); e += W_THREADS) {
    const int r = e / (WA_LD - p.K), cc = p.K + e % (WA_LD - p.K);
    Abuf[(r / WBM) * WA_ELEMS + (r % WBM) * WA_LD + cc] = 0.0;
  }
  for (int e = tid; e < WSTAGES * (WK - p.K) * WB_LD; e += W_THREADS) {
    const int s = e / ((WK - p.K) * WB_LD), rem = e % ((WK - p.K) * WB_LD);
    Sbuf[s * WSTAGE_ELEMS + (p.K + rem / WB_LD) * WB_LD + rem % WB_LD] = 0.0;
  }
  if (tid == 0) {
    for (int s = 0; s < WSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], W_CONSUMERS);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&a_full[s], 1);
      mbar_init(&a_empty[s], W_CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (t0 >= t1) return;

  if (warp == W_CONSUMERS) {
    // ================= producer =================
    int stage = 0, phase = 0, a_slot = -1, strip = -1;
    unsigned a_phase[2] = {0u, 0u};
    const unsigned a_bytes = (unsigned)(p.K * 8);
    for (int tile = t0; tile < t1; ++tile) {
      const int tstrip = tile / p.tiles_n;
      const int m0 = tstrip * WBM, n0 = (tile % p.tiles_n) * WBN;
      const int rows = min(WBM, p.M - m0);
      if (tstrip != strip) {
        strip = tstrip;
        a_slot = (a_slot + 1) & 1;
        mbar_wait(&a_empty[a_slot], a_phase[a_slot] ^ 1u);
        if (lane == 0) mbar_expect_tx(&a_full[a_slot], a_bytes * rows);
        __syncwarp();
        double* dst = Abuf + a_slot * WA_ELEMS;
        for (int r = lane; r < rows; r += 32)
          bulk_g2s(dst + r * WA_LD, p.A + (long long)(m0 + r) * p.lda, a_bytes, &a_full[a_slot]);
        a_phase[a_slot] ^= 1u;
      }
      const int cols = min(WBN, p.N - n0);
      const unsigned row_bytes = (unsigned)(cols * 8);
      mbar_wait(&empty[stage], (unsigned)phase ^ 1u);
      if (lane == 0) mbar_expect_tx(&full[stage], row_bytes * (p.K + rows));
      __syncwarp();
      double* bs = Sbuf + stage * WSTAGE_ELEMS;
      double* cs = bs + WB_ELEMS;
      for (int r = lane; r < p.K; r += 32)
        bulk_g2s(bs + r * WB_LD, p.B + p.bidx[r] * p.ldb + n0, row_bytes, &full[stage]);
      for (int r = lane; r < rows; r += 32)
        bulk_g2s(cs + r * WC_LD, p.Cin + p.cidx[m0 + r] * p.ldcin + n0, row_bytes, &full[stage]);
      if (++stage == WSTAGES) { stage = 0; phase ^= 1; }
    }
    return;
  }

  // ================= consumers =================
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp & 3) * 16, wn = (warp >> 2) * (WBN / 2);
  int stage = 0, phase = 0, a_slot = -1, strip = -1;
  unsigned a_phase[2] = {0u, 0u};
  for (int tile = t0; tile < t1; ++tile) {
    const int tstrip = tile / p.tiles_n;
    const int m0 = tstrip * WBM, n0 = (tile % p.tiles_n) * WBN;
    if (tstrip != strip) {
      if (a_slot >= 0) {  // release the previous strip's A
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_empty[a_slot]);
      }
      strip = tstrip;
      a_slot = (a_slot + 1) & 1;
      mbar_wait(&a_full[a_slot], a_phase[a_slot]);
      a_phase[a_slot] ^= 1u;
    }
    mbar_wait(&full[stage], (unsigned)phase);
    const double* as = Abuf + a_slot * WA_ELEMS;
    const double* bs = Sbuf + stage * WSTAGE_ELEMS;
    const double* cs = bs + WB_ELEMS;
    double acc[WNT][4];
#pragma unroll
    for (int j = 0; j < WNT; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[j][e] = 0.0;
#pragma unroll
    for (int kk = 0; kk < WK; kk += 4) {
      const double a0 = as[(wm + g) * WA_LD + kk + t];
      const double a1 = as[(wm + g + 8) * WA_LD + kk + t];
#pragma unroll
      for (int j = 0; j < WNT; ++j) dmma_16x8x4(acc[j], a0, a1, bs[(kk + t) * WB_LD + wn + 8 * j + g]);
    }
    // epilogue: C = Cin - acc (one rounding, as cin - (a @ b)), 16-byte stores
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = wm + g + 8 * h;
      const int gm = m0 + r;
      if (gm < p.M) {
        double* crow = p.C + (long long)gm * p.ldc;
#pragma unroll
        for (int j = 0; j < WNT; ++j) {
          const int col = wn + 8 * j + 2 * t;
          const int gn = n0 + col;
          const double2 cin = *reinterpret_cast<const double2*>(cs + r * WC_LD + col);
          const double v0 = cin.x - acc[j][2 * h];
          const double v1 = cin.y - acc[j][2 * h + 1];
          if (gn + 1 < p.N) {
            *reinterpret_cast<double2*>(crow + gn) = make_double2(v0, v1);
          } else if (gn < p.N) {
            crow[gn] = v0;
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == WSTAGES) { stage = 0; phase ^= 1; }
  }
}

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
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(rank_update_stream_kernel<BM, WARPS_N, STAGES>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    configured = true;
  }
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
  const bool bulk_ok = K > 0 && K % 2 == 0 && N % 2 == 0 && al16(A) && al16(B) && al16(Cin) && al16(C) &&
                       lda % 2 == 0 && ldb % 2 == 0 && ldcin % 2 == 0 && ldc % 2 == 0;
  RankUpdateParams p{M, N, K, A, lda, B, ldb, bidx, Cin, ldcin, cidx, C, ldc, 0, 0};
  // Default: the 2-CTA/SM cp.async kernel (17-18 TF/s on B200); the bulk-copy
  // pipeline (15 TF/s, per-row copy rate bound) is opt-in via RSKEL_RU_BULK=1.
  static const bool prefer_bulk = [] {
    const char* e = getenv("RSKEL_RU_BULK");
    return e != nullptr && e[0] == '1';
  }();
  static const int ru_kernel = [] {
    // 0: 2-CTA cp.async, 1: bulk, 3: streaming 128 x 64 tiles (default), 4: streaming 64 x 64
    const char* e = getenv("RSKEL_RU_KERNEL");
    return e != nullptr ? atoi(e) : 3;
  }();
  const bool stream_ok = bulk_ok && K <= 64;
  if (stream_ok && (ru_kernel == 3 || ru_kernel == 4) && !prefer_bulk) {
    if (ru_kernel == 4)
      launch_stream<64, 2, 3>(p, nsm, st);
    else
      launch_stream<128, 1, 2>(p, nsm, st);
  } else if (bulk_ok && (prefer_bulk || ru_kernel == 1)) {
    p.tiles_n = (N + WBN - 1) / WBN;
    p.tiles = p.tiles_n * ((M + WBM - 1) / WBM);
    const int G = p.tiles < nsm ? p.tiles : nsm;
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(rank_update_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)W_SMEM);
      configured = true;
    }
    rank_update_bulk_kernel<<<G, W_THREADS, W_SMEM, st>>>(p);
  } else {
    p.tiles_n = (N + UBN - 1) / UBN;
    p.tiles = p.tiles_n * ((M + UBM - 1) / UBM);
    const int G = p.tiles < 2 * nsm ? p.tiles : 2 * nsm;
    const bool vec2 = al16(A) && al16(B) && al16(Cin) && al16(C) && lda % 2 == 0 && ldb % 2 == 0 &&
                      ldcin % 2 == 0 && ldc % 2 == 0;
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
  }
  count_launch(1);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

}  // namespace rs
