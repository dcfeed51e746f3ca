// Panel LU with partial pivoting on a tall R x w block (w <= 64), the kernel
// behind `_lupp_panel` (`dense.py:185-207`) for the sketch blocks and Schur
// blocks of the adaptive loop (`skeleton.py:317-351`).
//
// Design (B200): one cooperative grid of G CTAs, CTA g keeps its contiguous
// slice of rows resident in shared memory for the whole panel (a 65472 x 64
// fp64 Schur block is 33.5 MB = 148 CTAs x 226 KB).  Rows never move: the
// reference's full-row swaps are replaced by a position map pos[row] (the
// "current permuted position" that breaks argmax ties, `dense.py:194`).
//
// Per column j the critical path is: every CTA publishes its best candidate
// (|v|, pos, row, the row's values) with a release-store of a per-step
// sequence number; warp 0 of every CTA polls the G sequence numbers (this is
// the grid barrier and the data exchange in one round trip), reduces the G
// candidates identically (deterministic), loads the pivot row, and all
// threads scale column j and update column j+1 of their rows ("early"
// update, one row per thread) to find the next candidate.  The rest of the
// rank-1 update (columns j+2..w-1, "late" update) runs while warp 0 publishes
// and waits for the next column, so it is off the critical path.
//
// Arithmetic follows numpy's rounding exactly: l = s / pivot (IEEE division),
// s' = s - (l * u) with the product rounded before the subtraction (np.outer
// then -=), i.e. no FMA contraction.
//
// Shared memory holds the rows with a 64-double stride and an XOR swizzle
// (column c of local row i at i*64 + (c ^ (i & 31))), conflict-free for both
// the row-per-thread (early) and row-per-warp (late) access patterns.
//
// Large panels (more rows than 148 x 227 KB of shared memory holds, about
// 65,000 x 64): the same kernel with the rows left in place in global memory
// (ROWS_GLOBAL; R x 64 fp64 is 51 MB at R = 100,000 and stays in the 126 MB
// L2), the position map in shared memory.  Same arithmetic, same pivots.
#include <atomic>
#include <cstdio>
#include <cstdlib>

#ifndef PANEL_DBG  // experiment switch: 1 = per-phase clock64 totals of CTA 0 (printf)
#define PANEL_DBG 0
#endif

#include "common.cuh"
#include "rskel_internal.h"

namespace rs {

constexpr int PTHREADS = 256;
#if PANEL_DBG
__device__ unsigned long long tp_late_out[256];
#endif
constexpr int PWARPS = PTHREADS / 32;
constexpr int PMAXW = 64;
constexpr int PMAXG = 256;  // >= CTAs of the cooperative grid (one per SM)

// LL-style exchange: every 8-byte word carries the step flag next to 4 bytes
// of payload, so a reader that sees the flag in a word also sees its payload
// (8-byte single-copy atomicity) -- no fences, no separate barrier.
struct PanelScratch {
  // One 128-byte line per CTA for its record and for its copy of the winner
  // broadcast: no line is shared by two writers or polled by many readers
  // (a hot line serialises in its L2 slice and made each hop ~1.3 us).
  uint4 rec[2][PMAXG][8];           // [0] = {val.lo, f, val.hi, f}, [1] = {pos, f, row + 1, f}
  uint4 rowdata[2][PMAXG][PMAXW];   // candidate row: {x.lo, f, x.hi, f} per column
};

RS_DEV void st_v4(uint4* p, unsigned a, unsigned b, unsigned c, unsigned d) {
  // gpu-scope relaxed: .volatile (= relaxed.sys) stores were serialised (~150 ns each)
  asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
RS_DEV uint4 ld_v4(const uint4* p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
RS_DEV double join(unsigned lo, unsigned hi) {
  return __longlong_as_double((long long)(((unsigned long long)hi << 32) | lo));
}

size_t panel_workspace_bytes() { return sizeof(PanelScratch); }

RS_DEV int swz(int i, int c) { return i * PMAXW + (c ^ (i & 31)); }


// Block-wide argmax of (val desc, pos asc); returns the winner's local row
// (-1 if no thread had a candidate) in every thread.  Uses red_* scratch.
RS_DEV void block_best(double& v, int& p, int& r, double* red_v, int* red_p, int* red_r) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, off);
    int op = __shfl_xor_sync(0xffffffffu, p, off);
    int orr = __shfl_xor_sync(0xffffffffu, r, off);
    if (orr >= 0 && (r < 0 || key_better(ov, op, v, p))) { v = ov; p = op; r = orr; }
  }
  if (lane == 0) { red_v[warp] = v; red_p[warp] = p; red_r[warp] = r; }
  __syncthreads();
  v = red_v[0]; p = red_p[0]; r = red_r[0];
#pragma unroll
  for (int q = 1; q < PWARPS; ++q) {
    if (red_r[q] >= 0 && (r < 0 || key_better(red_v[q], red_p[q], v, p))) {
      v = red_v[q]; p = red_p[q]; r = red_r[q];
    }
  }
  __syncthreads();
}

template <int QMAX, bool ROWS_GLOBAL>
__global__ void __launch_bounds__(PTHREADS, 1)
    panel_kernel(double* __restrict__ S, long long lds, int R, int w, int rows_per,
                 int64_t* __restrict__ perm_out, int* __restrict__ ncols_out, PanelScratch* ws,
                 unsigned flag_base) {
  extern __shared__ __align__(16) double psm[];
  const int G = gridDim.x, cta = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r0 = cta * rows_per;
  int nloc = R - r0;
  nloc = nloc < 0 ? 0 : (nloc > rows_per ? rows_per : nloc);

  // local row i, column c: swizzled shared memory, or the row in place in S
  double* Ss = psm;
  double* const Sg = S + (long long)r0 * lds;
  auto at = [&](int i, int c) -> double& {
    if constexpr (ROWS_GLOBAL) return Sg[(long long)i * lds + c];
    else return Ss[swz(i, c)];
  };
  int* pos = reinterpret_cast<int*>(psm + (ROWS_GLOBAL ? 0 : (size_t)rows_per * PMAXW));  // rows_per
  __shared__ double Urow2[2][PMAXW];  // U row of step j in Urow2[j & 1] (late update reads j-1)
  __shared__ double red_v[PWARPS];
  __shared__ int red_p[PWARPS], red_r[PWARPS];
  __shared__ double s_val;
  __shared__ int s_pos, s_row;

  if constexpr (!ROWS_GLOBAL) {
    for (int idx = tid; idx < nloc * w; idx += PTHREADS) {
      int i = idx / w, c = idx - i * w;
      Ss[swz(i, c)] = S[(long long)(r0 + i) * lds + c];
    }
  }
  for (int i = tid; i < nloc; i += PTHREADS) pos[i] = r0 + i;
  __syncthreads();

  // Candidate for column 0.
  double bv = -1.0;
  int bp = 0x7fffffff, br = -1;
  for (int i = tid; i < nloc; i += PTHREADS) {
    double v = fabs(at(i, 0));
    if (key_better(v, pos[i], bv, bp) || br < 0) { bv = v; bp = pos[i]; br = i; }
  }
  block_best(bv, bp, br, red_v, red_p, red_r);

  unsigned long long tp[6] = {0, 0, 0, 0, 0, 0}, tm0 = clock64(), tm1, tlate = 0;
#define PMARK(k) if (PANEL_DBG && tid == 0) { tm1 = clock64(); tp[k] += tm1 - tm0; tm0 = tm1; }
  int ncols = w;
  int late_j = -1;   // step whose columns late_j+2.. still need the rank-1 update
  int late_skip = -1;
  for (int j = 0; j < w; ++j) {
    const int par = j & 1;
    if (warp == 0) {
      const unsigned f = flag_base + (unsigned)j + 1u;
      // ---- publish this CTA's candidate for column j (no fence needed).
      // The record goes first: it is what every CTA polls; the row values are
      // read only by the winner's readers, one exchange hop later. ----
      if (lane == 0) {
        const double v = br >= 0 ? bv : -1.0;
        const unsigned long long x = (unsigned long long)__double_as_longlong(v);
        st_v4(&ws->rec[par][cta][0], (unsigned)x, f, (unsigned)(x >> 32), f);
        st_v4(&ws->rec[par][cta][1], (unsigned)bp, f, br >= 0 ? (unsigned)(r0 + br + 1) : 0u, f);
      }
      if (br >= 0) {
        for (int c = lane; c < w; c += 32) {
          const unsigned long long x = (unsigned long long)__double_as_longlong(at(br, c));
          st_v4(&ws->rowdata[par][cta][c], (unsigned)x, f, (unsigned)(x >> 32), f);
        }
      }
      PMARK(0);  // publish
#if PANEL_DBG
      unsigned long long gt_pub = 0, gt_poll = 0;
      if (lane == 0 && j == 10) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_pub));
#endif
      // ---- reduce the G candidates: every CTA polls all records itself
      // (all-to-all, one hop; identical reduction order on every CTA) ----
      double v = -1.0;
      int pp = 0x7fffffff, rr = -1, cc = -1;
      {
        // Poll all of this lane's records in one pass (loads issued back to
        // back, then checked), repeat only for the ones not yet published.
        const int nq = (G - lane + 31) / 32;
        unsigned pending = nq >= 32 ? 0xffffffffu : ((1u << nq) - 1u);
        while (pending) {
          uint4 a[QMAX], b[QMAX];
#pragma unroll
          for (int i = 0; i < QMAX; ++i) {
            if ((pending >> i) & 1u) {
              a[i] = ld_v4(&ws->rec[par][lane + 32 * i][0]);
              b[i] = ld_v4(&ws->rec[par][lane + 32 * i][1]);
            }
          }
#pragma unroll
          for (int i = 0; i < QMAX; ++i) {
            if (!((pending >> i) & 1u)) continue;
            if (a[i].y != f || a[i].w != f || b[i].y != f || b[i].w != f) continue;
            pending &= ~(1u << i);
            const int row = (int)b[i].z - 1;
            const double qv = join(a[i].x, a[i].z);
            const int qp = (int)b[i].x;
            if (row >= 0 && (rr < 0 || key_better(qv, qp, v, pp))) {
              v = qv; pp = qp; rr = row; cc = lane + 32 * i;
            }
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          double ov = __shfl_xor_sync(0xffffffffu, v, off);
          int op = __shfl_xor_sync(0xffffffffu, pp, off);
          int orr = __shfl_xor_sync(0xffffffffu, rr, off);
          int oc = __shfl_xor_sync(0xffffffffu, cc, off);
          if (orr >= 0 && (rr < 0 || key_better(ov, op, v, pp))) { v = ov; pp = op; rr = orr; cc = oc; }
        }
      }
      if (lane == 0) { s_val = rr >= 0 ? v : 0.0; s_pos = pp; s_row = rr; }
      PMARK(1);  // poll + reduce (hop 1)
#if PANEL_DBG
      if (lane == 0 && j == 10) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_poll));
        printf("step10 cta %d pub %llu poll_end %llu\n", cta, gt_pub, gt_poll);
      }
#endif
      // ---- pivot row (U row j) straight from the winner's published copy ----
      if (rr >= 0 && v > 0.0) {
        const int c0 = j + lane, c1 = j + lane + 32;
        bool need0 = c0 < w, need1 = c1 < w;
        while (need0 || need1) {  // both words in flight at once
          uint4 x0 = make_uint4(0, 0, 0, 0), x1 = make_uint4(0, 0, 0, 0);
          if (need0) x0 = ld_v4(&ws->rowdata[par][cc][c0]);
          if (need1) x1 = ld_v4(&ws->rowdata[par][cc][c1]);
          if (need0 && x0.y == f && x0.w == f) { Urow2[par][c0] = join(x0.x, x0.z); need0 = false; }
          if (need1 && x1.y == f && x1.w == f) { Urow2[par][c1] = join(x1.x, x1.z); need1 = false; }
        }
      }
    } else if (late_j >= 0) {
      // ---- late update of the previous step (off the critical path) ----
      // Rank-1 update of columns jl+2.. of every live row; each lane owns at
      // most two columns (u0, u1 in registers) and walks 4 rows per trip so
      // the smem load -> dmul -> dsub -> store chains overlap.
      const int jl = late_j;
      const unsigned long long tl0 = PANEL_DBG ? clock64() : 0;
      const int c0 = jl + 2 + lane, c1 = c0 + 32;
      if (c0 < w) {
        const bool h1 = c1 < w;
        const double u0 = Urow2[jl & 1][c0], u1 = h1 ? Urow2[jl & 1][c1] : 0.0;
        constexpr int WS = PWARPS - 1;
        int i = warp - 1;
        for (; i + 3 * WS < nloc; i += 4 * WS) {
          int rr4[4];
          bool ok[4];
          double l[4], a[4], b[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            rr4[q] = i + q * WS;
            ok[q] = pos[rr4[q]] > jl && rr4[q] != late_skip;
            l[q] = at(rr4[q], jl);
            a[q] = at(rr4[q], c0);
            b[q] = h1 ? at(rr4[q], c1) : 0.0;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (!ok[q]) continue;
            at(rr4[q], c0) = __dsub_rn(a[q], __dmul_rn(l[q], u0));
            if (h1) at(rr4[q], c1) = __dsub_rn(b[q], __dmul_rn(l[q], u1));
          }
        }
        for (; i < nloc; i += WS) {
          if (pos[i] <= jl || i == late_skip) continue;
          const double l = at(i, jl);
          at(i, c0) = __dsub_rn(at(i, c0), __dmul_rn(l, u0));
          if (h1) at(i, c1) = __dsub_rn(at(i, c1), __dmul_rn(l, u1));
        }
      }
      if (PANEL_DBG && tid == 32) tlate += clock64() - tl0;
    }
    PMARK(2);  // pivot row (hop 2)
    __syncthreads();
    PMARK(3);  // wait for the late update
    if (!(s_val > 0.0)) { ncols = j; break; }  // exactly-zero pivot column
    const int ppos = s_pos, prow = s_row;

    // ---- swap bookkeeping, scale column j, update column j+1, next candidate ----
    const double upiv = Urow2[par][j];
    const double unext = (j + 1 < w) ? Urow2[par][j + 1] : 0.0;
    bv = -1.0; bp = 0x7fffffff; br = -1;
    for (int i = tid; i < nloc; i += PTHREADS) {
      int pi = pos[i];
      if (pi < j) continue;
      if (r0 + i == prow) { pos[i] = j; continue; }
      if (pi == j) { pi = ppos; pos[i] = pi; }
      const double l = __ddiv_rn(at(i, j), upiv);
      at(i, j) = l;
      if (j + 1 < w) {
        double& a = at(i, j + 1);
        const double v = __dsub_rn(a, __dmul_rn(l, unext));
        a = v;
        const double av = fabs(v);
        if (br < 0 || key_better(av, pi, bv, bp)) { bv = av; bp = pi; br = i; }
      }
    }
    block_best(bv, bp, br, red_v, red_p, red_r);
    PMARK(4);  // early update + block argmax
    // The new local best row is published next step: bring it fully up to date.
    if (warp == 0 && br >= 0) {
      const double l = at(br, j);
      for (int c = j + 2 + lane; c < w; c += 32) {
        double& a = at(br, c);
        a = __dsub_rn(a, __dmul_rn(l, Urow2[par][c]));
      }
      __syncwarp();
    }
    late_j = j;
    late_skip = br;
    PMARK(5);  // best row update
  }
#if PANEL_DBG
  if (PANEL_DBG && tid == 32 && (cta == 0 || cta == G / 2)) tp_late_out[cta] = tlate;
  __syncthreads();
  if (PANEL_DBG && tid == 0 && (cta == 0 || cta == G / 2))
    printf("panel cta %d/%d rows %d: publish %llu poll %llu row %llu sync %llu early %llu best %llu late(warp 1) %llu (cycles, %d cols)\n",
           cta, G, nloc, tp[0], tp[1], tp[2], tp[3], tp[4], tp[5], tp_late_out[cta], w);
#endif
  __syncthreads();

  // ---- write back factors (physical row order) and the position map ----
  if constexpr (!ROWS_GLOBAL) {
    for (int idx = tid; idx < nloc * w; idx += PTHREADS) {
      int i = idx / w, c = idx - i * w;
      S[(long long)(r0 + i) * lds + c] = Ss[swz(i, c)];
    }
  }
  for (int i = tid; i < nloc; i += PTHREADS) perm_out[pos[i]] = r0 + i;
  if (cta == 0 && tid == 0) *ncols_out = ncols;
}

int launch_panel(double* S, long long lds, int R, int w, int64_t* perm_out, int* ncols_dev,
                 void* workspace, cudaStream_t st) {
  if (R < 0 || w < 0 || w > PMAXW || (R > 0 && lds < w)) return RS_ERR_ARG;
  if (R == 0 || w == 0) {
    cudaMemsetAsync(ncols_dev, 0, sizeof(int), st);
    return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  int nsm = 0, max_smem = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // Small panels: fewer CTAs (cheaper exchange).  Large: one CTA per SM.
#ifndef RS_PANEL_ROWS  // rows per CTA before the grid grows (tools/ experiment builds vary it)
#define RS_PANEL_ROWS 64
#endif
  int G = (R + RS_PANEL_ROWS - 1) / RS_PANEL_ROWS;
  if (G > nsm) G = nsm;
  if (G > PMAXG) G = PMAXG;
  if (G < 1) G = 1;
  const int rows_per = (R + G - 1) / G;
  const size_t static_smem = 2048;
  auto round16 = [](size_t x) { return (x + 15) & ~size_t(15); };
  size_t smem = round16((size_t)rows_per * PMAXW * sizeof(double) + (size_t)rows_per * sizeof(int));
  // rows in shared memory when they fit, else in place in global memory (L2)
  const bool rows_global = smem + static_smem > (size_t)max_smem;
  if (rows_global) smem = round16((size_t)rows_per * sizeof(int));
  if (smem + static_smem > (size_t)max_smem) return RS_ERR_CAPACITY;
  // Polled record slots per lane: G <= 32 * QMAX (a small QMAX keeps the
  // exchange loop short).
#ifndef RS_PANEL_QMIN  // smallest polling width used (experiment builds vary it)
#define RS_PANEL_QMIN 0
#endif
  int q = G <= 32 ? 0 : G <= 64 ? 1 : G <= 128 ? 2 : 3;
  if (q < RS_PANEL_QMIN) q = RS_PANEL_QMIN;
  static const void* const kernels[2][4] = {
      {(const void*)panel_kernel<1, false>, (const void*)panel_kernel<2, false>, (const void*)panel_kernel<4, false>,
       (const void*)panel_kernel<8, false>},
      {(const void*)panel_kernel<1, true>, (const void*)panel_kernel<2, true>, (const void*)panel_kernel<4, true>,
       (const void*)panel_kernel<8, true>}};
  const void* kern = kernels[rows_global ? 1 : 0][q];
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, PTHREADS, smem);
  if (occ * nsm < G) return RS_ERR_CAPACITY;
  PanelScratch* ws = static_cast<PanelScratch*>(workspace);
  // Flags of launch e are e*128 + j + 1: stale words of earlier launches never match.
  static std::atomic<unsigned> epoch{1};
  unsigned flag_base = (epoch.fetch_add(1) & 0x1ffffffu) << 7;
  void* args[] = {&S, &lds, &R, &w, (void*)&rows_per, &perm_out, &ncols_dev, &ws, &flag_base};
  cudaError_t e = cudaLaunchCooperativeKernel(kern, dim3(G), dim3(PTHREADS), args, smem, st);
  count_launch(1);
  return e == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

}  // namespace rs
