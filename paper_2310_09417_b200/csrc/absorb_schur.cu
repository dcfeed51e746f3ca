// Absorb(t) + Schur(t+1) with one read of the interpolation block T
// (`skeleton.py:439-454`: `_extend_state` of block t, then `_schur_of_block`
// of block t+1, on the T form T = L2 L1^{-1}).
//
// With P = sub[:nc] (pivots of block t), Q = sub[nc:] (the rest, new order),
// W = L_r L_1^{-1} (already in T'[:, k:k+nc]) and Y = the next sketch block,
//
//   T'[i, :k] = T[Q_i] - W_i T[P]                                 (rank-nc update)
//   S'[i]     = Y[perm'[k'+i]] - T'[i] Y[perm'[:k']]              (next Schur block)
//             = Z[Q_i] - W_i Z[P],   Z = Y[perm[k:]] - T Y[perm[:k]]
//
// i.e. the next Schur block is the Schur block of Y against the OLD
// factorisation, corrected by the block's own rank-nc update.  So one pass
// streams T[Q] once: every 64 x 64 tile of it feeds both DMMA products,
//   T' tile = Cin - W_strip T[P]_chunk      (A = W fragments in registers)
//   X_strip += Cin Y[perm[n0 : n0+64]]       (A = the Cin tile in smem)
// and a small kernel finishes S'[i] = Y[perm'[k'+i]] - (X[i] + W_i Z[P]) with
// Z[P] = Y[perm'[k:k+nc]] - T[P] Y[perm[:k]] (one skinny GEMM, done before).
//
// Work: tiles (64-row strip, 64-column chunk) in strip-major order, split
// evenly over one persistent CTA per SM; B (T[P]) / Cin (T[Q]) / Y chunks
// stream through a 2-stage cp.async ring.  A strip split between CTAs leaves
// per-CTA partial X sums in workspace slots; the finishing kernel adds them in
// CTA order, so S' is deterministic.
#include "common.cuh"
#include "rskel_internal.h"

namespace rs {

constexpr int AS_BM = 64, AS_BN = 64, AS_K = 64, AS_NB = 64, AS_STAGES = 2, AS_THREADS = 256;
constexpr int AS_LD = 68;  // = 4 (mod 16): conflict-free 64-bit fragment loads
constexpr int AS_STAGE = 3 * 64 * AS_LD;  // B chunk, Cin chunk, Y chunk (doubles)
constexpr size_t AS_SMEM = sizeof(double) * AS_STAGES * AS_STAGE;
constexpr int AS_SLOT = AS_BM * AS_NB;  // doubles per partial X slot

struct AbsorbSchurParams {
  int M;                 // rows of T' (R - nc)
  int N;                 // k: columns of T to update
  int K;                 // nc (<= 64)
  const double* W;       // W_hat rows (new order), ld ldw  (= T' + k)
  long long ldw;
  const double* T;       // old T (R x k), ld ldt
  long long ldt;
  const int64_t* pidx;   // sub[:nc]
  const int64_t* qidx;   // sub[nc:]
  double* Tn;            // T' (first k columns), ld ldn
  long long ldn;
  const double* Y;       // next sketch block (m x 64), ld ldy
  long long ldy;
  const int64_t* ytop;   // perm[:k] (rows of Y multiplying T's columns)
  double* X;             // X strips (M x 64, ld 64) for whole strips
  double* slots;         // partial X of split strips: 2 per CTA
  int tiles_n, tiles;
};

__host__ __device__ inline int as_t0(const AbsorbSchurParams& p, int G, int c) {
  return (int)((long long)c * p.tiles / G);
}

__global__ void __launch_bounds__(AS_THREADS, 1) absorb_schur_kernel(AbsorbSchurParams p) {
  extern __shared__ __align__(16) double assm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp & 3) * 16, wn = (warp >> 2) * 32;
  const int G = gridDim.x, c = blockIdx.x;
  const int t0 = as_t0(p, G, c), t1 = as_t0(p, G, c + 1);
  if (t0 >= t1) return;
  const int ntile = t1 - t0;

  const int crow0 = tid >> 5, ccol = (tid & 31) * 2;  // copy geometry: 8 rows apart, 16-byte column
  long long boff[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = crow0 + 8 * i;
    boff[i] = r < p.K ? p.pidx[r] * p.ldt : -1;
  }
  long long coff[8];
  int pf_strip = -1;

  auto issue = [&](int li) {
    const int tile = t0 + li;
    const int strip = tile / p.tiles_n;
    const int m0 = strip * AS_BM, n0 = (tile - strip * p.tiles_n) * AS_BN;
    if (strip != pf_strip) {
      pf_strip = strip;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int gm = m0 + crow0 + 8 * i;
        coff[i] = gm < p.M ? p.qidx[gm] * p.ldt : -1;
      }
    }
    double* st = assm + (li % AS_STAGES) * AS_STAGE;
    double* bs = st;
    double* cs = st + 64 * AS_LD;
    double* ys = st + 2 * 64 * AS_LD;
    const int gn = n0 + ccol;
    const int nv = gn < p.N ? min(2, p.N - gn) : 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = crow0 + 8 * i;
      const bool bv = boff[i] >= 0 && nv > 0;
      cp_async16(bs + r * AS_LD + ccol, bv ? p.T + boff[i] + gn : p.T, bv ? nv * 8 : 0);
      const bool cv = coff[i] >= 0 && nv > 0;
      cp_async16(cs + r * AS_LD + ccol, cv ? p.T + coff[i] + gn : p.T, cv ? nv * 8 : 0);
      const int yr = n0 + r;  // Y row for T column n0 + r
      const bool yv = yr < p.N;
      cp_async16(ys + r * AS_LD + ccol, yv ? p.Y + p.ytop[yr] * p.ldy + ccol : p.Y, yv ? 16 : 0);
    }
  };

  double af[16][2];
  int a_strip = -1;
  double xacc[4][4];  // X of this warp's 16 rows x 32 Schur columns, over the strip segment
  int seg_first = t0;

#pragma unroll
  for (int s = 0; s < AS_STAGES - 1; ++s) {
    if (s < ntile) issue(s);
    cp_async_commit();
  }
  for (int li = 0; li < ntile; ++li) {
    const int tile = t0 + li;
    const int strip = tile / p.tiles_n;
    const int m0 = strip * AS_BM, n0 = (tile - strip * p.tiles_n) * AS_BN;
    if (strip != a_strip) {
      a_strip = strip;
      seg_first = tile;
      const int r0 = m0 + wm + g, r1 = r0 + 8;
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) {
        const int kc = 4 * ks + t;
        af[ks][0] = (r0 < p.M && kc < p.K) ? p.W[(long long)r0 * p.ldw + kc] : 0.0;
        af[ks][1] = (r1 < p.M && kc < p.K) ? p.W[(long long)r1 * p.ldw + kc] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) xacc[j][e] = 0.0;
    }
    cp_async_wait<AS_STAGES - 2>();
    __syncthreads();
    if (li + AS_STAGES - 1 < ntile) issue(li + AS_STAGES - 1);
    cp_async_commit();
    const double* st = assm + (li % AS_STAGES) * AS_STAGE;
    const double* bs = st;
    const double* cs = st + 64 * AS_LD;
    const double* ys = st + 2 * 64 * AS_LD;

    // T' tile = Cin - W T[P]  and  X += Cin Y_chunk (K = the chunk's 64
    // columns of T, zero-filled past k): the two products interleaved per
    // k-step, 8 independent accumulator chains per warp.
    double acc[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[j][e] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 16; ++ks) {
      const double a0 = cs[(wm + g) * AS_LD + 4 * ks + t];
      const double a1 = cs[(wm + g + 8) * AS_LD + 4 * ks + t];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double b = bs[(4 * ks + t) * AS_LD + wn + 8 * j + g];
        dmma_16x8x4(acc[j], af[ks][0], af[ks][1], b);
        const double y = ys[(4 * ks + t) * AS_LD + wn + 8 * j + g];
        dmma_16x8x4(xacc[j], a0, a1, y);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int lr = wm + g + 8 * h;
      const int gm = m0 + lr;
      if (gm >= p.M) continue;
      double* cw = p.Tn + (long long)gm * p.ldn;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ln = wn + 8 * j + 2 * t;
        const int gn = n0 + ln;
        const double c0 = cs[lr * AS_LD + ln], c1 = cs[lr * AS_LD + ln + 1];
        const double v0 = c0 - acc[j][2 * h], v1 = c1 - acc[j][2 * h + 1];
        if (gn + 1 < p.N) {
          *reinterpret_cast<double2*>(cw + gn) = make_double2(v0, v1);
        } else if (gn < p.N) {
          cw[gn] = v0;
        }
      }
    }
    // end of this CTA's segment of the strip: hand X over
    const bool strip_end = (tile + 1) % p.tiles_n == 0;
    if (strip_end || tile + 1 == t1) {
      const bool whole = strip_end && seg_first == strip * p.tiles_n;
      double* dst;
      long long ldd;
      int row0;
      if (whole) {
        dst = p.X;
        ldd = AS_NB;
        row0 = m0;
      } else {
        // slot rule (as in the finishing kernel): the segment is this CTA's
        // last one iff the CTA's range started before the strip
        dst = p.slots + (size_t)(t0 < strip * p.tiles_n ? 2 * c + 1 : 2 * c) * AS_SLOT;
        ldd = AS_NB;
        row0 = 0;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int lr = wm + g + 8 * h;
        if (whole && m0 + lr >= p.M) continue;
        double* xw = dst + (long long)(row0 + lr) * ldd;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int ln = wn + 8 * j + 2 * t;
          *reinterpret_cast<double2*>(xw + ln) = make_double2(xacc[j][2 * h], xacc[j][2 * h + 1]);
        }
      }
    }
  }
  cp_async_wait<0>();
}

// S'[i] = Y[yrest[i]] - (X[i] + W_i Z[P]) for one 64-row strip per CTA; the X
// of a split strip is the sum of its CTAs' slots in CTA order.
__global__ void __launch_bounds__(256) absorb_schur_finish_kernel(AbsorbSchurParams p, int G,
                                                                  const double* __restrict__ ZP,
                                                                  const int64_t* __restrict__ yrest,
                                                                  double* __restrict__ S) {
  __shared__ double zs[64][65];
  __shared__ double ws[16][65];  // W rows of the 16 strip rows being finished
  const int strip = blockIdx.x, tid = threadIdx.x;
  const int m0 = strip * AS_BM;
  for (int e = tid; e < 64 * 64; e += 256) {
    const int r = e >> 6, cc = e & 63;
    zs[r][cc] = r < p.K ? ZP[r * 64 + cc] : 0.0;
  }
  const int s0 = strip * p.tiles_n, s1 = s0 + p.tiles_n;
  // owners of the first and last tile of the strip
  auto owner = [&](int tile) {
    int c = (int)(((long long)tile * G) / p.tiles);
    while (c + 1 < G && as_t0(p, G, c + 1) <= tile) ++c;
    while (c > 0 && as_t0(p, G, c) > tile) --c;
    return c;
  };
  const int clo = owner(s0), chi = owner(s1 - 1);
  const bool whole = clo == chi && as_t0(p, G, clo) <= s0;
  const int col = tid & 63;
  for (int rb = 0; rb < 64; rb += 16) {  // 16 rows per pass: W rows staged in smem
    __syncthreads();
    for (int e = tid; e < 16 * 64; e += 256) {
      const int r = e >> 6, cc = e & 63, gm = m0 + rb + r;
      ws[r][cc] = (gm < p.M && cc < p.K) ? p.W[(long long)gm * p.ldw + cc] : 0.0;
    }
    __syncthreads();
  for (int r = rb + (tid >> 6); r < rb + 16; r += 4) {
    const int gm = m0 + r;
    if (gm >= p.M) break;
    double x;
    if (whole) {
      x = p.X[(long long)gm * AS_NB + col];
    } else {
      x = 0.0;
      for (int cc = clo; cc <= chi; ++cc) {
        const int slot = as_t0(p, G, cc) < s0 ? 2 * cc + 1 : 2 * cc;
        const double v = p.slots[(size_t)slot * AS_SLOT + r * AS_NB + col];
        x = cc == clo ? v : x + v;
      }
    }
    double acc = x;
    for (int j = 0; j < p.K; ++j) acc = fma(ws[r - rb][j], zs[j][col], acc);
    S[(long long)gm * AS_NB + col] = p.Y[yrest[gm] * p.ldy + col] - acc;
  }
  }
}

size_t absorb_schur_slots_bytes(int nsm) { return sizeof(double) * 2 * (size_t)nsm * AS_SLOT; }

// Tn = T' (ld k + nc, W_hat already in columns k..k+nc), ZP = Z[P] (nc x 64),
// yrest = perm'[k + nc:] (rows of Y for S'), ytop = perm'[:k].
int launch_absorb_schur(int Rn, int k, int nc, const double* T, const int64_t* sub, double* Tn,
                        const double* Y, long long ldy, const int64_t* perm_new, const double* ZP, double* X,
                        double* S, double* slots, cudaStream_t st) {
  if (Rn < 0 || k < 1 || nc < 1 || nc > AS_K) return RS_ERR_ARG;
  if (Rn == 0) return RS_OK;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  AbsorbSchurParams p;
  p.M = Rn;
  p.N = k;
  p.K = nc;
  p.ldn = k + nc;
  p.W = Tn + k;
  p.ldw = k + nc;
  p.T = T;
  p.ldt = k;
  p.pidx = sub;
  p.qidx = sub + nc;
  p.Tn = Tn;
  p.Y = Y;
  p.ldy = ldy;
  p.ytop = perm_new;
  p.X = X;
  p.slots = slots;
  p.tiles_n = (k + AS_BN - 1) / AS_BN;
  p.tiles = p.tiles_n * ((Rn + AS_BM - 1) / AS_BM);
  const int G = p.tiles < nsm ? p.tiles : nsm;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(absorb_schur_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)AS_SMEM);
    configured = true;
  }
  absorb_schur_kernel<<<G, AS_THREADS, AS_SMEM, st>>>(p);
  const int strips = (Rn + AS_BM - 1) / AS_BM;
  absorb_schur_finish_kernel<<<strips, 256, 0, st>>>(p, G, ZP, perm_new + k + nc, S);
  count_launch(2);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

}  // namespace rs
