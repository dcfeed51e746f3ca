// fp64 / fp32 sketch GEMM on the 5th-generation tensor cores: the Ozaki
// scheme on tcgen05.mma kind::i8 with TMEM int32 accumulators.
//
//   Y = A Omega,  A: M x K (fp64 or fp32, either layout),  Omega: K x N fp64.
//
// Every row i of A and every column j of Omega is cut, per K-chunk c, into
// signed 7-bit digits relative to a power of two above its largest entry in
// the chunk:
//     A[i, k] = 2^{e_ic} sum_{s<SA} a_s[i, k] 2^{-7(s+1)} + (|rem| < 2^{e_ic - 7 SA})
// (exact: scaling by 2^-e and the digit extraction y <- 128 y - trunc(128 y)
// are exact in fp64).  The products of digit planes are exact integers,
// accumulated exactly in int32 by the tensor cores, one TMEM accumulator per
// digit sum g = s + t (pairs with g >= G = max(SA, SB) are dropped: their
// weight is below 2^{-7(G+2)} of the row x column scale):
//     Y_chunk[i, j] = 2^{e_ic + f_jc} sum_{g<G} 2^{-7(g+2)} C_g[i, j],
//     C_g = sum_{s+t=g} a_s b_t^T   (int32, |C_g| <= kc 127^2 min(SA, SB) < 2^31).
// The G terms are converted and added in fp64 in a fixed order (smallest
// first), then the chunk sums are folded in chunk order exactly as the DMMA
// GEMM does (gemm_f64.cu).  Every quantity depends on row i, on Omega and on
// K alone, so the determinism contract of rs_dgemm holds here too: a row's
// bits do not depend on M, on the tile it lands in or on the device count.
//
// A is sliced ONCE per skeleton call (rs_oz_slice; it is multiplied by a
// fresh Omega every block) into digit planes laid out in HBM as the exact
// shared-memory image the MMA reads: 128-row x 128-byte tiles, K-major,
// 128-byte swizzled (16-byte chunk c of row r at r*128 + ((c ^ r%8) * 16)),
// tile order [row tile][k-block][digit plane].  So each pipeline stage is one
// contiguous 16 KB bulk copy (cp.async.bulk, the TMA engine's linear mode)
// and no tensor map is needed.  At SA = 8 the planes take 8 bytes per entry,
// the same HBM traffic as the fp64 matrix, while the int8 tensor pipe does
// the 36 plane products (4.5 POP/s dense) -- the sketch is no longer bound by
// the 37 TF/s DMMA pipe (measured bound: the MMA issue through the stage
// handshake).
//
// Kernel (one CTA per SM, persistent over (tile, chunk) units; the units after
// the last full wave are halved over two CTAs, see oz_item):
//   warp 0  producer: bulk copies of the Omega planes of a k-block (one copy
//           of SB x 8 KB) and of the A planes (one 16 KB stage each);
//   warp 1  TMEM owner + MMA issuer (one thread): for every A plane s and
//           Omega plane t with s + t < G, tcgen05.mma m128 n64..256 k32 into
//           accumulator g = s + t; tcgen05.commit releases the stages;
//   warps 2-9 epilogue, two warps per TMEM lane quadrant splitting the
//           columns: tcgen05.ld of the G int32 accumulators (one TMEM lane =
//           one output row per thread), exact int64 combination, fp64
//           conversion, chunk slot or direct store; the last-arriving unit of
//           a tile folds the chunk slots.
#include <algorithm>
#include <cstdio>
#include <cstdint>

#include "common.cuh"
#include "rskel_internal.h"

#ifndef OZ_DBG  // experiment switch for tools/oz_prof.py builds only (0 in the library):
// 1 no MMAs, 2 no epilogue TMEM reads, 3 no loads (barriers arrive without data),
// 5 = 3 without the epilogue, 6 = 3 with an empty epilogue, 7 = time the MMA issuer's waits
#define OZ_DBG 0
#endif

namespace rs {

namespace {

constexpr int OZ_BM = 128, OZ_BN = 64, OZ_BK = 128;  // rows of A tile, rows of Omega^T tile, k bytes
constexpr int OZ_ATILE = OZ_BM * OZ_BK;               // 16 KB
constexpr int OZ_BTILE = OZ_BN * OZ_BK;               // 8 KB
constexpr int OZ_MAXS = 8;
#ifndef OZ_PPS  // A digit planes per pipeline stage (one bulk copy, one handshake); 2 measured equal
#define OZ_PPS 1
#endif
#ifndef OZ_NA_STAGES
#define OZ_NA_STAGES (6 / OZ_PPS)
#endif
constexpr int OZ_PPS_ = OZ_PPS;
constexpr int OZ_NA = OZ_NA_STAGES;                   // A stages of OZ_PPS planes
constexpr int OZ_NB = 2;                              // Omega k-block stages (SB planes each)
#ifndef OZ_EPI_WARPS  // epilogue warps: 4 (one per TMEM lane quadrant) or 8 (two, splitting the columns)
#define OZ_EPI_WARPS 8
#endif
constexpr int OZ_EPI = OZ_EPI_WARPS * 32;             // epilogue threads
constexpr int OZ_CBS = OZ_EPI_WARPS / 4;              // column groups: each warp takes OZ_BN / OZ_CBS columns
constexpr int OZ_THREADS = 64 + OZ_EPI;
constexpr size_t OZ_SMEM = 1024 + (size_t)OZ_NA * OZ_PPS_ * OZ_ATILE + (size_t)OZ_NB * OZ_MAXS * OZ_BTILE + 512;

// ------------------------------------------------------------------ PTX ----
RS_DEV uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
RS_DEV void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(n));
}
RS_DEV void mb_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
RS_DEV void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
RS_DEV void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
RS_DEV void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
RS_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
RS_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
RS_DEV void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(b))
               : "memory");
}
RS_DEV void tc_mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
RS_DEV void tc_ld16_async(uint32_t taddr, int* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
RS_DEV void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
// 2^e exactly (normal range; the digit exponents of finite fp64 data stay far inside it)
RS_DEV double pow2(int e) {
  return e >= -1022 && e <= 1023 ? __longlong_as_double((long long)(e + 1023) << 52) : ldexp(1.0, e);
}
RS_DEV void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

// K-major, 128-byte swizzled operand tile: rows of 128 bytes, 8-row groups
// 1024 bytes apart (SBO), version 1 (sm_100), layout SWIZZLE_128B.
RS_DEV uint64_t smem_desc(const void* p) {
  const uint64_t addr = su32(p);
  return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// kind::i8, signed x signed -> s32, both K-major, M = 128, N = n (multiple of 16, <= 256)
RS_DEV uint32_t oz_idesc(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(OZ_BM >> 4) << 24);
}

// ---------------------------------------------------------------- slicing ----
template <typename T>
RS_DEV double ld_elem(const T* X, long long ld, bool colmajor, long long i, long long k) {
  return (double)(colmajor ? X[k * ld + i] : X[i * ld + k]);
}

// Row-chunk maxima -> exponents: expo[i * nch + c] = e with
// max_{k in chunk c} |X[i, k]| < 2^e (frexp).  Pass 1 (oz_max_kernel): block
// (32 x 8) covers 32 rows x 256 k of one chunk -- lanes along the contiguous
// dimension, the 8 warps split the k range -- reduces in shared memory and
// folds into mx[i * nch + c] with an atomicMax on the double's bits (|x| >= 0
// orders like its bit pattern).  Pass 2 (oz_expo_kernel) converts.  NaN/inf
// set *nonfinite (fmax would drop a NaN).
template <typename T, bool COLMAJOR>
__global__ void __launch_bounds__(256) oz_max_kernel(const T* __restrict__ X, long long ld, int rows, int K, int kc,
                                                     int c0, int nch, unsigned long long* __restrict__ mx,
                                                     int* __restrict__ nonfinite) {
  const int c = c0 + blockIdx.y;
  const int kb = c * kc + blockIdx.z * 256;
  const int kend = min(K, min(c * kc + kc, kb + 256));
  __shared__ double red[8][33];
  double m = 0.0;
  bool bad = false;
  if constexpr (COLMAJOR) {  // lanes along rows (contiguous), warps along k
    const long long i = (long long)blockIdx.x * 32 + threadIdx.x;
    if (i < rows)
      for (int k = kb + threadIdx.y; k < kend; k += 8) {
        const double x = fabs((double)X[(long long)k * ld + i]);
        m = fmax(m, x);
        bad = bad || !isfinite(x);
      }
    red[threadIdx.y][threadIdx.x] = m;
    __syncthreads();
    if (threadIdx.y == 0 && i < rows) {
      for (int w = 1; w < 8; ++w) m = fmax(m, red[w][threadIdx.x]);
      atomicMax(mx + i * nch + c, (unsigned long long)__double_as_longlong(m));
    }
  } else {  // warp y handles row blockIdx.x * 8 + y, lanes along k (contiguous)
    const long long i = (long long)blockIdx.x * 8 + threadIdx.y;
    if (i < rows)
      for (int k = kb + threadIdx.x; k < kend; k += 32) {
        const double x = fabs((double)X[i * ld + k]);
        m = fmax(m, x);
        bad = bad || !isfinite(x);
      }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    if (threadIdx.x == 0 && i < rows) atomicMax(mx + i * nch + c, (unsigned long long)__double_as_longlong(m));
  }
  if (bad && nonfinite) atomicOr(nonfinite, 1);
}

__global__ void oz_expo_kernel(const unsigned long long* __restrict__ mx, int rows, int c0, int c1, int nch,
                               int* __restrict__ expo) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int nc = c1 - c0;
  if (t >= (long long)rows * nc) return;
  const long long i = t / nc;
  const int c = c0 + (int)(t % nc);
  const double m = __longlong_as_double((long long)mx[i * nch + c]);
  int e = 0;
  if (m > 0.0 && isfinite(m)) frexp(m, &e);
  expo[i * nch + c] = e;
}

// Digit planes of rows [0, rows_pad) x k in [k0, k1_pad) (k0 a multiple of
// 128, k1_pad = k1 rounded up to 128): thread (row, 16-k group); rows >= rows
// and k >= K give zero digits (the tile padding).
template <typename T, bool COLMAJOR>
__global__ void oz_slice_kernel(const T* __restrict__ X, long long ld, int rows, int rows_pad, int K, int k0,
                                int k1_pad, int kc, int nch, int S, int tile_rows, int KB,
                                const int* __restrict__ expo, int8_t* __restrict__ dig) {
  int i, q;
  if constexpr (COLMAJOR) {  // lanes along rows: each k reads 32 consecutive rows
    i = blockIdx.x * 32 + threadIdx.x;
    q = blockIdx.y * blockDim.y + threadIdx.y;
  } else {  // lanes along k groups: each row segment is read contiguously
    i = blockIdx.x * blockDim.y + threadIdx.y;
    q = blockIdx.y * 32 + threadIdx.x;
  }
  const int k = k0 + q * 16;
  if (i >= rows_pad || k >= k1_pad) return;
  // The S digits d_s = trunc(128 y_s), y_{s+1} = 128 y_s - d_s of y = x 2^-e (|y| < 1) are the
  // base-128 digits of trunc(|y| 2^56) with y's sign: one exact conversion per entry instead
  // of S truncations and conversions.
  long long t[16];
  const int e = (i < rows && k < K) ? expo[(long long)i * nch + k / kc] : 0;
  const bool pw = e >= -1023;  // 2^-e representable: x * 2^-e rounds exactly as ldexp(x, -e)
  const double p2 = pw ? ldexp(1.0, -e) : 0.0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int kk = k + j;
    const double x = (i < rows && kk < K) ? ld_elem(X, ld, COLMAJOR, i, kk) : 0.0;
    const double y = pw ? x * p2 : ldexp(x, -e);
    t[j] = __double2ll_rz(y * 72057594037927936.0);  // y 2^56: exact, |.| < 2^56
  }
  const int tile = i / tile_rows, r = i % tile_rows, kb = k / OZ_BK, c16 = (k % OZ_BK) / 16;
  const size_t tile_bytes = (size_t)tile_rows * OZ_BK;
  int8_t* base = dig + ((size_t)tile * KB + kb) * S * tile_bytes + (size_t)(r >> 3) * 1024 + (r & 7) * 128 +
                 ((c16 ^ (r & 7)) * 16);
  for (int s = 0; s < S; ++s) {
    const int sh = 7 * (7 - s);
    uint32_t w[4];
#pragma unroll
    for (int j4 = 0; j4 < 4; ++j4) {
      uint32_t packed = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const long long tj = t[j4 * 4 + b];
        const int mag = (int)(((unsigned long long)(tj < 0 ? -tj : tj) >> sh) & 127u);
        packed |= (uint32_t)(uint8_t)(int8_t)(tj < 0 ? -mag : mag) << (8 * b);
      }
      w[j4] = packed;
    }
    *reinterpret_cast<uint4*>(base + (size_t)s * tile_bytes) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// ------------------------------------------------------------------- GEMM ----
struct OzParams {
  int M, N, K;
  const int8_t* adig;
  const int* aexp;
  int SA;
  const int8_t* bdig;
  const int* bexp;
  int SB;
  int G;             // accumulators (digit sums 0..G-1)
  int KB, kbc, nch;  // k-blocks of K, k-blocks per chunk, chunks
  int tiles_n, tile0, units;
  int mode;
  double alpha, beta;
  const double* Cin;
  long long ldcin;
  double* C;
  long long ldc;
  double* slots;
  int* tickets;
  long long* hl;      // tail split: exact int64 (H, L) partials, 4 tiles of 128 x 64 per tail unit
  int* tail_tickets;  // tail split: arrival counters per tail unit (zero between launches)
  int split;          // 1: the last partial wave's units are halved over two CTAs each
};

// Work item i of this CTA.  Whole units u = blockIdx.x + i * gridDim.x; with the tail split,
// the units after the last full wave are cut in two k-block halves, half (b & 1) of tail
// unit (b >> 1) going to CTA b, so the last wave keeps every SM busy instead of half of
// them.  The halves' int32 accumulators are summed exactly (as int64 Horner words), so a
// split unit has the same bits as an unsplit one.
RS_DEV bool oz_item(const OzParams& p, int i, int& u, int& kb0, int& kb1, int& half) {
  const int G = gridDim.x, b = blockIdx.x;
  const int rounds = p.units / G;
  if (!p.split) {
    u = b + i * G;
    if (u >= p.units) return false;
    half = -1;
  } else if (i < rounds) {
    u = b + i * G;
    half = -1;
  } else if (i == rounds && b < 2 * (p.units - rounds * G)) {
    u = rounds * G + (b >> 1);
    half = b & 1;
  } else {
    return false;
  }
  const int ch = u % p.nch;
  const int k0 = ch * p.kbc, k1 = min(p.KB, k0 + p.kbc);
  if (half < 0) {
    kb0 = k0;
    kb1 = k1;
  } else {
    const int mid = k0 + (k1 - k0 + 1) / 2;
    kb0 = half ? mid : k0;
    kb1 = half ? k1 : mid;
  }
  return true;
}

__global__ void __launch_bounds__(OZ_THREADS, 1) oz_gemm_kernel(OzParams p) {
  extern __shared__ __align__(1024) uint8_t oz_smem[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(oz_smem) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = sm;                                      // OZ_NA x OZ_PPS x 16 KB
  uint8_t* sb = sm + OZ_NA * OZ_PPS_ * OZ_ATILE;         // OZ_NB x SB x 8 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(sb + OZ_NB * OZ_MAXS * OZ_BTILE);
  uint64_t* full_a = bars;
  uint64_t* empty_a = bars + OZ_NA;
  uint64_t* full_b = bars + 2 * OZ_NA;
  uint64_t* empty_b = full_b + OZ_NB;
  uint64_t* tm_full = empty_b + OZ_NB;
  uint64_t* tm_empty = tm_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tm_empty + 1);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);
  int* s_eb = s_last + 1;  // OZ_BN column exponents of the current unit

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < OZ_NA; ++i) { mb_init(full_a + i, 1); mb_init(empty_a + i, 1); }
    for (int i = 0; i < OZ_NB; ++i) { mb_init(full_b + i, 1); mb_init(empty_b + i, 1); }
    mb_init(tm_full, 1);
    mb_init(tm_empty, OZ_EPI);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer --
    if (lane == 0) {
      int ai = 0, bi = 0;
      uint32_t aph = 0, bph = 0;
      int u, kb0, kb1, hf;
      for (int item = 0; oz_item(p, item, u, kb0, kb1, hf); ++item) {
        const int lt = u / p.nch, tile = p.tile0 + lt;
        const int tm = tile / p.tiles_n, tn = tile - tm * p.tiles_n;
        for (int kb = kb0; kb < kb1; ++kb) {
          mb_wait(empty_b + bi, bph ^ 1);
          if (OZ_DBG == 3 || OZ_DBG == 5 || OZ_DBG == 6) {  // no-load experiment modes
            mb_arrive(full_b + bi);
          } else {
            mb_expect_tx(full_b + bi, (uint32_t)(p.SB * OZ_BTILE));
            bulk_load(sb + (size_t)bi * OZ_MAXS * OZ_BTILE,
                      p.bdig + ((size_t)tn * p.KB + kb) * p.SB * OZ_BTILE, p.SB * OZ_BTILE, full_b + bi);
          }
          if (++bi == OZ_NB) { bi = 0; bph ^= 1; }
          const int8_t* asrc = p.adig + ((size_t)tm * p.KB + kb) * p.SA * OZ_ATILE;
          for (int s0 = 0; s0 < p.SA; s0 += OZ_PPS_) {
            // planes s0.. of this k-block are consecutive 16 KB tiles in HBM: one copy
            const uint32_t bytes = (uint32_t)(min(OZ_PPS_, p.SA - s0) * OZ_ATILE);
            mb_wait(empty_a + ai, aph ^ 1);
            if (OZ_DBG == 3 || OZ_DBG == 5 || OZ_DBG == 6) {  // no-load experiment modes
              mb_arrive(full_a + ai);
            } else {
              mb_expect_tx(full_a + ai, bytes);
              bulk_load(sa + (size_t)ai * OZ_PPS_ * OZ_ATILE, asrc + (size_t)s0 * OZ_ATILE, bytes, full_a + ai);
            }
            if (++ai == OZ_NA) { ai = 0; aph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer --
    int ai = 0, bi = 0;
    uint32_t aph = 0, bph = 0, tph = 0;
#if OZ_DBG == 7 || OZ_DBG == 8  // where the MMA issuer waits (7: printf per 37th CTA; 8: no printf)
    unsigned long long w_tm = 0, w_b = 0, w_a = 0, t_mark = 0;
    const unsigned long long t_start = clock64();
#define OZ_T0() (t_mark = clock64())
#define OZ_T1(acc) (acc += clock64() - t_mark)
#else
#define OZ_T0() ((void)0)
#define OZ_T1(acc) ((void)0)
#endif
    // One thread issues and waits; the other lanes of the warp idle until the end (a
    // warp-wide wait + __syncwarp per stage made the k-block ~6 % slower in
    // tools/probe/tc_seq.cu, orders 7 vs 9).
    if (lane == 0) {
      int u, kb0, kb1, hf;
      for (int item = 0; oz_item(p, item, u, kb0, kb1, hf); ++item) {
        OZ_T0();
        if (OZ_DBG != 5) mb_wait(tm_empty, tph ^ 1);  // the epilogue has drained the previous unit
        OZ_T1(w_tm);
        tph ^= 1;
        tc_fence_after();
        for (int kb = kb0; kb < kb1; ++kb) {
          OZ_T0();
          mb_wait(full_b + bi, bph);
          OZ_T1(w_b);
          const uint8_t* bst = sb + (size_t)bi * OZ_MAXS * OZ_BTILE;
          for (int s = 0; s < p.SA; ++s) {
            if (s % OZ_PPS_ == 0) {
              OZ_T0();
              mb_wait(full_a + ai, aph);
              OZ_T1(w_a);
              tc_fence_after();
            }
            // A plane s times Omega planes t = 0..G-1-s in MMAs of up to 4 planes
            // (N <= 256): the planes are consecutive 64-row tiles in shared memory
            // and their accumulators g = s + t consecutive 64-column TMEM blocks, so
            // one MMA covers up to four (s, t) pairs and reads the A plane once.
            const uint64_t da = smem_desc(sa + ((size_t)ai * OZ_PPS_ + s % OZ_PPS_) * OZ_ATILE);
            const int nt = p.G - s;
            for (int t0 = 0; t0 < nt; t0 += 4) {
              const int ntile = min(4, nt - t0);
              const uint64_t db = smem_desc(bst + (size_t)t0 * OZ_BTILE);
              const uint32_t d = tmem + (uint32_t)((s + t0) * OZ_BN);
              const uint32_t idesc = oz_idesc(OZ_BN * ntile);
#pragma unroll
              for (int kk = 0; kk < OZ_BK / 32; ++kk) {
                // s = 0 of the unit's first k-block covers every accumulator: it
                // starts them from zero, everything after accumulates
                const uint32_t acc = (kb > kb0 || s > 0 || kk > 0) ? 1u : 0u;
                if (OZ_DBG != 1) tc_mma_i8(d, da + 2 * kk, db + 2 * kk, idesc, acc);
              }
            }
            if (s % OZ_PPS_ == OZ_PPS_ - 1 || s == p.SA - 1) {
              tc_commit(empty_a + ai);  // the A stage is free once these MMAs have read it
              if (++ai == OZ_NA) { ai = 0; aph ^= 1; }
            }
          }
          tc_commit(empty_b + bi);
          if (++bi == OZ_NB) { bi = 0; bph ^= 1; }
        }
        if (OZ_DBG != 5) tc_commit(tm_full);
      }
    }
    __syncwarp();
#if OZ_DBG == 7
    if (lane == 0 && blockIdx.x % 37 == 0)
      printf("cta %d: total %llu cycles, wait tm_empty %llu, full_b %llu, full_a %llu\n", blockIdx.x,
             clock64() - t_start, w_tm, w_b, w_a);
#endif
  } else if (OZ_DBG != 5) {
    // ------------------------------------------------------------ epilogue --
    const int q = warp & 3;              // TMEM lane quadrant this warp may read
    const int r = q * 32 + lane;         // output row within the tile
    const int et = threadIdx.x - 64;     // 0..OZ_EPI-1
    const int cgrp = (warp - 2) >> 2;    // column group of this warp
    const int cb_lo = cgrp * (OZ_BN / 16 / OZ_CBS), cb_hi = cb_lo + OZ_BN / 16 / OZ_CBS;
    uint32_t tph = 0;
    int u, kb0, kb1, hf;
    for (int item = 0; oz_item(p, item, u, kb0, kb1, hf); ++item) {
      const int lt = u / p.nch, ch = u - lt * p.nch, tile = p.tile0 + lt;
      const int tm = tile / p.tiles_n, tn = tile - tm * p.tiles_n;
      const int row = tm * OZ_BM + r;
      const int ea = row < p.M ? p.aexp[(long long)row * p.nch + ch] : 0;
      mb_wait(tm_full, tph);
      tph ^= 1;
      tc_fence_after();
      if (OZ_DBG == 6) {
        mb_arrive(tm_empty);
        continue;
      }
      double* slot = p.slots + (size_t)u * (OZ_BM * OZ_BN);
      // this unit's column exponents, staged once in shared memory
      named_sync(1, OZ_EPI);
      if (et < OZ_BN) {
        const int col = tn * OZ_BN + et;
        s_eb[et] = col < p.N ? p.bexp[(long long)col * p.nch + ch] : 0;
      }
      named_sync(1, OZ_EPI);
      // tail halves: this half's (H, L) words and the other half's, 128 x 64 int64 each
      const int tt = hf >= 0 ? u - (p.units / gridDim.x) * gridDim.x : 0;
      long long* hl_mine = p.hl + ((size_t)4 * tt + 2 * (hf > 0)) * (OZ_BM * OZ_BN) + r;
      long long* hl_other = p.hl + ((size_t)4 * tt + 2 * (hf == 0)) * (OZ_BM * OZ_BN) + r;
      for (int pass = 0; pass < (hf >= 0 ? 2 : 1); ++pass) {
        if (pass == 1) {
          // both halves of a split unit are in: the second to arrive finishes the unit
          __threadfence();
          named_sync(1, OZ_EPI);
          if (et == 0) *s_last = atomicAdd(p.tail_tickets + tt, 1) == 1;
          named_sync(1, OZ_EPI);
          if (!*s_last) break;
          __threadfence();
          if (et == 0) p.tail_tickets[tt] = 0;
        }
      for (int cb = cb_lo; cb < cb_hi; ++cb) {
        // The G <= 8 exact int32 digit-sum accumulators of 16 columns, combined
        // exactly in two int64 words (H: g = 0..3, L: g = 4..7; 7-bit shifts,
        // |H|, |L| < 2^55), then two conversions and one fma:
        //   v = 2^(ea+eb) (H 2^-35 + L 2^-63).
        long long H[16], L[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) { H[j] = 0; L[j] = 0; }
        if (pass == 1) {
          // the exact sum of the two halves' words
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const size_t o = (size_t)(cb * 16 + j) * OZ_BM;
            H[j] = __ldcg(hl_mine + o) + __ldcg(hl_other + o);
            L[j] = __ldcg(hl_mine + (OZ_BM * OZ_BN) + o) + __ldcg(hl_other + (OZ_BM * OZ_BN) + o);
          }
        } else if (OZ_DBG != 2 && kb1 > kb0) {
          const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(cb * 16);
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            const int g0 = 4 * half;
            if (g0 >= p.G) break;
            int c[4][16];  // four accumulators in flight, one wait
#pragma unroll
            for (int gg = 0; gg < 4; ++gg)
              if (g0 + gg < p.G) tc_ld16_async(tb + (uint32_t)((g0 + gg) * OZ_BN), c[gg]);
            tc_wait_ld();
#pragma unroll
            for (int gg = 0; gg < 4; ++gg) {
              if (g0 + gg >= p.G) break;
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                if (half == 0) H[j] = H[j] * 128 + c[gg][j];
                else L[j] = L[j] * 128 + c[gg][j];
              }
            }
          }
        }
        if (hf >= 0 && pass == 0) {
          // a tail half: publish this half's words; the unit is finished in pass 1
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const size_t o = (size_t)(cb * 16 + j) * OZ_BM;
            __stcg(hl_mine + o, H[j]);
            __stcg(hl_mine + (OZ_BM * OZ_BN) + o, L[j]);
          }
          continue;
        }
        // missing high accumulators (G < 8) still take their 7-bit shifts
        const int gl = p.G > 4 ? p.G - 4 : 0, gh = p.G < 4 ? p.G : 4;
        double v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const double h = (double)H[j] * pow2(-7 * (gh + 1));
          const double l = (double)L[j] * pow2(-7 * (gl + 5));
          v[j] = (h + l) * pow2(ea + s_eb[cb * 16 + j]);
        }
        if (p.nch == 1) {
          if (row < p.M) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int col = tn * OZ_BN + cb * 16 + j;
              if (col >= p.N) continue;
              double out = v[j];
              if (p.mode == RS_GEMM_FOLD) out = p.Cin[(long long)row * p.ldcin + col] + v[j];
              else if (p.beta != 0.0) out = fma(p.alpha, v[j], p.beta * p.Cin[(long long)row * p.ldcin + col]);
              else out = p.alpha * v[j];
              p.C[(long long)row * p.ldc + col] = out;
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) __stcg(slot + (size_t)(cb * 16 + j) * OZ_BM + r, v[j]);
        }
      }
        if (pass == 0) {
          tc_fence_before();
          mb_arrive(tm_empty);  // TMEM may be overwritten by the next unit
        }
      }
      if (hf >= 0 && !*s_last) continue;  // the first half to arrive: the other finishes
      if (p.nch == 1) continue;
      __threadfence();
      named_sync(1, OZ_EPI);
      if (et == 0) *s_last = atomicAdd(p.tickets + lt, 1) == p.nch - 1;
      named_sync(1, OZ_EPI);
      if (!*s_last) continue;
      __threadfence();
      // last chunk of the tile to arrive: fold the chunk partials in chunk order
      const double* base = p.slots + (size_t)lt * p.nch * (OZ_BM * OZ_BN) + r;
      for (int cb = cb_lo; cb < cb_hi; ++cb) {
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = __ldcg(base + (size_t)(cb * 16 + j) * OZ_BM);
        if (p.mode == RS_GEMM_FOLD && row < p.M) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int col = tn * OZ_BN + cb * 16 + j;
            if (col < p.N) acc[j] = p.Cin[(long long)row * p.ldcin + col] + acc[j];
          }
        }
        for (int c = 1; c < p.nch; ++c) {
          const double* src = base + (size_t)c * (OZ_BM * OZ_BN);
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] += __ldcg(src + (size_t)(cb * 16 + j) * OZ_BM);
        }
        if (row < p.M) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int col = tn * OZ_BN + cb * 16 + j;
            if (col >= p.N) continue;
            double out = acc[j];
            if (p.mode == RS_GEMM_PLAIN)
              out = p.beta != 0.0 ? fma(p.alpha, acc[j], p.beta * p.Cin[(long long)row * p.ldcin + col])
                                  : p.alpha * acc[j];
            p.C[(long long)row * p.ldc + col] = out;
          }
        }
      }
      named_sync(1, OZ_EPI);
      if (et == 0) p.tickets[lt] = 0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

int ok_or_cuda() { return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA; }

}  // namespace

int oz_chunk(long long K) {
  long long kc = (K + 7) / 8;
  kc = (kc + OZ_BK - 1) / OZ_BK * OZ_BK;
  return (int)std::min<long long>(16384, std::max<long long>(1024, kc));
}

size_t oz_digits_bytes(int rows, long long K, int S, int tile_rows) {
  const long long tiles = (rows + tile_rows - 1) / tile_rows;
  const long long KB = (K + OZ_BK - 1) / OZ_BK;
  return (size_t)tiles * KB * S * tile_rows * OZ_BK;
}

int launch_oz_slice(const void* X, int fp32, long long ld, int colmajor, int rows, int K, int k0, int k1, int kc,
                    int S, int tile_rows, int8_t* dig, int* expo, int* nonfinite, unsigned long long* mx,
                    size_t mx_bytes, cudaStream_t st) {
  if (rows < 0 || K < 0 || k0 < 0 || k1 > K || k0 > k1 || kc <= 0 || kc % OZ_BK || k0 % kc || S < 1 ||
      S > OZ_MAXS || (tile_rows != OZ_BM && tile_rows != OZ_BN))
    return RS_ERR_ARG;
  if (rows == 0 || k0 == k1) return RS_OK;
  const int nch = (K + kc - 1) / kc;
  if ((size_t)rows * nch * sizeof(unsigned long long) > mx_bytes) return RS_ERR_CAPACITY;
  const int c0 = k0 / kc, c1 = (k1 + kc - 1) / kc;
  const int KB = (K + OZ_BK - 1) / OZ_BK;
  const int rows_pad = (rows + tile_rows - 1) / tile_rows * tile_rows;
  const int k1_pad = k1 == K ? (K + OZ_BK - 1) / OZ_BK * OZ_BK : k1;
  const int groups = (k1_pad - k0) / 16;
  // mx: rows x nch words of scratch (the caller's workspace), zeroed for the atomics
  cudaMemsetAsync(mx, 0, sizeof(unsigned long long) * (size_t)rows * nch, st);
  const dim3 gm_col((rows + 31) / 32, c1 - c0, (kc + 255) / 256), gm_row((rows + 7) / 8, c1 - c0, (kc + 255) / 256);
  const dim3 gs_col((rows_pad + 31) / 32, (groups + 7) / 8), gs_row((rows_pad + 7) / 8, (groups + 31) / 32);
  const long long ne = (long long)rows * (c1 - c0);
  if (colmajor) {
    if (fp32) oz_max_kernel<float, true><<<gm_col, dim3(32, 8), 0, st>>>((const float*)X, ld, rows, K, kc, c0, nch, mx, nonfinite);
    else oz_max_kernel<double, true><<<gm_col, dim3(32, 8), 0, st>>>((const double*)X, ld, rows, K, kc, c0, nch, mx, nonfinite);
  } else {
    if (fp32) oz_max_kernel<float, false><<<gm_row, dim3(32, 8), 0, st>>>((const float*)X, ld, rows, K, kc, c0, nch, mx, nonfinite);
    else oz_max_kernel<double, false><<<gm_row, dim3(32, 8), 0, st>>>((const double*)X, ld, rows, K, kc, c0, nch, mx, nonfinite);
  }
  oz_expo_kernel<<<(unsigned)((ne + 255) / 256), 256, 0, st>>>(mx, rows, c0, c1, nch, expo);
  if (colmajor) {
    if (fp32)
      oz_slice_kernel<float, true><<<gs_col, dim3(32, 8), 0, st>>>((const float*)X, ld, rows, rows_pad, K, k0, k1_pad,
                                                                   kc, nch, S, tile_rows, KB, expo, dig);
    else
      oz_slice_kernel<double, true><<<gs_col, dim3(32, 8), 0, st>>>((const double*)X, ld, rows, rows_pad, K, k0,
                                                                    k1_pad, kc, nch, S, tile_rows, KB, expo, dig);
  } else {
    if (fp32)
      oz_slice_kernel<float, false><<<gs_row, dim3(32, 8), 0, st>>>((const float*)X, ld, rows, rows_pad, K, k0,
                                                                    k1_pad, kc, nch, S, tile_rows, KB, expo, dig);
    else
      oz_slice_kernel<double, false><<<gs_row, dim3(32, 8), 0, st>>>((const double*)X, ld, rows, rows_pad, K, k0,
                                                                     k1_pad, kc, nch, S, tile_rows, KB, expo, dig);
  }
  count_launch(3);
  return ok_or_cuda();
}

int launch_oz_gemm(int M, int N, int K, int kc, int mode, double alpha, const int8_t* adig, const int* aexp, int SA,
                   const int8_t* bdig, const int* bexp, int SB, double beta, const double* Cin, long long ldcin,
                   double* C, long long ldc, double* slots, int* tickets, int nslots, long long* hl, int hl_units,
                   int* tail_tickets, cudaStream_t st) {
  // G = SB accumulators and SA <= SB, so the s = 0 products touch every accumulator
  if (M < 0 || N < 0 || K < 0 || SA < 1 || SB < SA || SB > OZ_MAXS || kc % OZ_BK || kc <= 0 || kc > 16384)
    return RS_ERR_ARG;
  if (mode != RS_GEMM_PLAIN && mode != RS_GEMM_FOLD) return RS_ERR_ARG;
  if ((mode == RS_GEMM_FOLD || beta != 0.0) && Cin == nullptr) return RS_ERR_ARG;
  if (M == 0 || N == 0) return RS_OK;
  if (slots == nullptr || tickets == nullptr) return RS_ERR_ARG;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  OzParams p{};
  p.M = M; p.N = N; p.K = K;
  p.adig = adig; p.aexp = aexp; p.SA = SA;
  p.bdig = bdig; p.bexp = bexp; p.SB = SB;
  p.G = SB;
  p.KB = (K + OZ_BK - 1) / OZ_BK;
  p.kbc = kc / OZ_BK;
  p.nch = std::max(1, (K + kc - 1) / kc);
  p.tiles_n = (N + OZ_BN - 1) / OZ_BN;
  p.mode = mode; p.alpha = alpha; p.beta = beta;
  p.Cin = Cin; p.ldcin = ldcin; p.C = C; p.ldc = ldc;
  p.slots = slots; p.tickets = tickets;
  const long long tiles = (long long)p.tiles_n * ((M + OZ_BM - 1) / OZ_BM);
  cudaFuncSetAttribute(oz_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)OZ_SMEM);
  const long long per = p.nch == 1 ? tiles : std::max<long long>(1, nslots / p.nch);
  const long long ngroups = (tiles + per - 1) / per;
  for (long long gi = 0; gi < ngroups; ++gi) {
    const long long t0 = tiles * gi / ngroups, t1 = tiles * (gi + 1) / ngroups;
    p.tile0 = (int)t0;
    p.units = (int)((t1 - t0) * p.nch);
#ifndef OZ_MAX_CTAS  // experiment builds: leave SMs free for a concurrent kernel
#define OZ_MAX_CTAS 100000
#endif
    const int grid = std::min(std::min(p.units, nsm), OZ_MAX_CTAS);
    const int tail = p.units - (p.units / grid) * grid;
    p.hl = hl;
    p.tail_tickets = tail_tickets;
    p.split = (hl != nullptr && tail > 0 && 2 * tail <= grid && tail <= hl_units) ? 1 : 0;
    oz_gemm_kernel<<<grid, OZ_THREADS, OZ_SMEM, st>>>(p);
    count_launch(1);
  }
  return ok_or_cuda();
}

}  // namespace rs
