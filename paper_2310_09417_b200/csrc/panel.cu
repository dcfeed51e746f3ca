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
// candidates identically (deterministic), loads the pivot row, and column j
// is scaled and column j+1 updated for every local row ("early" update) to
// find the next candidate -- by warp 0 alone with a warp argmax when a CTA
// holds at most 192 rows, else by all threads with a block argmax.  The rest
// of the rank-1 update (columns j+2..w-1, "late" update, warps 1-7) runs
// while warp 0 publishes and waits for the next column, so it is off the
// critical path.
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
#include <algorithm>
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
#ifndef RS_PANEL_EU_MAX  // rows per lane up to which warp 0 does the early update alone (0: never)
#define RS_PANEL_EU_MAX 6
#endif
constexpr int EU_MAX = RS_PANEL_EU_MAX;
constexpr int PMAXG = 256;  // >= CTAs of the cooperative grid (one per SM)

// LL-style exchange: every 8-byte word carries the step flag next to 4 bytes
// of payload, so a reader that sees the flag in a word also sees its payload
// (8-byte single-copy atomicity) -- no fences, no separate barrier.
// Each CTA writes its record to NREP replicas in different lines; CTA c polls replica c % NREP,
// so a hot record line has G / NREP pollers instead of G.
#ifndef RS_PANEL_NREP
#define RS_PANEL_NREP 8
#endif
constexpr int NREP = RS_PANEL_NREP;
#ifndef RS_PANEL_RD_NREP  // replicas of the published candidate rows (pivot-row hop)
#define RS_PANEL_RD_NREP 1
#endif
constexpr int RD_NREP = RS_PANEL_RD_NREP;

struct PanelScratch {
  // One 128-byte line per CTA for its record and for its copy of the winner
  // broadcast: no line is shared by two writers or polled by many readers
  // (a hot line serialises in its L2 slice and made each hop ~1.3 us).
  uint4 rec[2][NREP][PMAXG][8];     // [0] = {val.lo, f, val.hi, f}, [1] = {pos, f, row + 1, f}
  uint4 rowdata[2][RD_NREP][PMAXG][PMAXW];  // candidate row: {x.lo, f, x.hi, f} per column
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
RS_DEV uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }


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

RS_DEV void mb_expect_tx_cta(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// 16 bytes into (possibly another CTA's) shared memory, counted on that CTA's mbarrier
RS_DEV void st_async_v4(uint32_t addr, unsigned a, unsigned b, unsigned c, unsigned d, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];\n" ::"r"(
                   addr),
               "r"(a), "r"(b), "r"(c), "r"(d), "r"(bar)
               : "memory");
}
// Wait for a phase of a local mbarrier that remote st.async writes complete.  CTA-scope acquire
// (the default): the transaction count already orders the bytes before the phase flip (a
// cluster-scope acquire adds an L1 invalidation).  Called by the whole warp, with the loop in
// C++: a spin loop inside inline asm run by one lane leaves the warp unconverged for the
// compiler, and every later shuffle then took the slow divergent path (~3.7 us per step).
RS_DEV bool mb_try_wait(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
RS_DEV void mb_wait_cluster(uint64_t* bar, unsigned parity) {
  while (!mb_try_wait(bar, parity)) {
  }
}
RS_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// CL = 1 (the library build): flat exchange, every CTA publishes a record and polls all G of
// them.  CL > 1 (experiment builds, -DRS_PANEL_CLUSTER=8): thread-block clusters; every CTA
// sends its candidate record and row into the cluster leader's shared memory (st.async,
// completion counted on the leader's mbarrier), the leaders exchange one record each through
// global memory, and each leader broadcasts the winner record and U row back into its CTAs'
// shared memory.  The flat hop grows from ~1 us at 64 records to ~3 us at 148
// (tools/probe/xchg.cu), but the cluster version measured slower inside the panel: 334-354 us
// against 272-299 us at R = 6000-20000.
template <int QMAX, bool ROWS_GLOBAL, int CL>
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
  __shared__ int s_pos, s_row, s_skip;
  // Cluster exchange (CL > 1), by step parity: the leader gathers the CL candidates (record +
  // row) in crec/crow (cbar counts their bytes); every CTA receives the step's winner record in
  // brec and its U row straight into Urow2 (bbar counts those bytes).
  constexpr int NCL = CL > 1 ? CL : 1;
  __shared__ __align__(8) uint64_t cbar[2], bbar[2];
  __shared__ __align__(16) uint4 crec[2][NCL];
  __shared__ __align__(16) double crow[2][NCL][CL > 1 ? PMAXW : 1];
  __shared__ __align__(16) uint4 brec[2];
  unsigned crank = 0;
  const int nrec = CL > 1 ? G / CL : G;  // records polled per step
  const int rec_id = CL > 1 ? cta / CL : cta;
  if constexpr (CL > 1) {
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(crank));
    if (tid == 0) {
      for (int q = 0; q < 2; ++q) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&cbar[q])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bbar[q])));
      }
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    cluster_sync_all();
  }

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

  unsigned long long tp[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tm0 = clock64(), tm1, tlate = 0;
  unsigned long long gt0 = 0, ck0 = clock64();
  if (PANEL_DBG) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
#define PMARK(k) if (PANEL_DBG && tid == 0) { tm1 = clock64(); tp[k] += tm1 - tm0; tm0 = tm1; }
  int ncols = w;
  // few rows per CTA: warp 0 does the early update and argmax alone (every CTA of the grid
  // decides for itself; the decision only changes which threads do the same arithmetic)
  const bool warp_early = nloc <= 32 * EU_MAX;
  int late_j = -1;   // step whose columns late_j+2.. still need the rank-1 update
  int late_skip = -1;
#if PANEL_DBG
  unsigned long long tstep[PMAXW + 1];
#endif
  for (int j = 0; j < w; ++j) {
#if PANEL_DBG
    tstep[j] = clock64();
#endif
    const int par = j & 1;
    if (warp == 0) {
     if constexpr (CL > 1) {
      // ---------------- two-level exchange over the thread-block cluster ----------------
      const unsigned f = flag_base + (unsigned)j + 1u;
      const unsigned ph = (unsigned)(j >> 1) & 1u;  // mbarrier phase of this parity's use
      uint32_t lead_cbar, lead_crec, lead_crow;
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(lead_cbar) : "r"(smem_u32(&cbar[par])));
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(lead_crec) : "r"(smem_u32(&crec[par][crank])));
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(lead_crow) : "r"(smem_u32(&crow[par][crank][0])));
      // (1) this CTA's candidate, record and row, into the leader's shared memory
      if (lane == 0) {
        if (crank == 0) mb_expect_tx_cta(&cbar[par], CL * (16 + 8 * PMAXW));
        mb_expect_tx_cta(&bbar[par], 16 + 8 * PMAXW);  // this step's broadcast, received below
        const unsigned long long x = (unsigned long long)__double_as_longlong(br >= 0 ? bv : -1.0);
        st_async_v4(lead_crec, (unsigned)x, (unsigned)(x >> 32), (unsigned)bp,
                    br >= 0 ? (unsigned)(r0 + br + 1) : 0u, lead_cbar);
      }
      {
        const int c = 2 * lane;
        const double x0 = (br >= 0 && c < w) ? at(br, c) : 0.0, x1 = (br >= 0 && c + 1 < w) ? at(br, c + 1) : 0.0;
        const unsigned long long u0 = (unsigned long long)__double_as_longlong(x0);
        const unsigned long long u1 = (unsigned long long)__double_as_longlong(x1);
        st_async_v4(lead_crow + 8u * c, (unsigned)u0, (unsigned)(u0 >> 32), (unsigned)u1, (unsigned)(u1 >> 32),
                    lead_cbar);
      }
      PMARK(0);  // publish
      if (crank == 0) {
        // (2) leader: cluster winner -> global record + row (LL words); poll the G / CL
        // records; fetch the global winner's row; broadcast record + row to the cluster
        mb_wait_cluster(&cbar[par], ph);
        PMARK(6);  // gather wait
        double cv = -1.0;
        int cp = 0x7fffffff, cr = -1, cm = -1;
        if (lane < CL) {
          const uint4 q = crec[par][lane];
          cv = join(q.x, q.y);
          cp = (int)q.z;
          cr = (int)q.w - 1;
          cm = lane;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, cv, off);
          const int op = __shfl_xor_sync(0xffffffffu, cp, off);
          const int orr = __shfl_xor_sync(0xffffffffu, cr, off);
          const int om = __shfl_xor_sync(0xffffffffu, cm, off);
          if (orr >= 0 && (cr < 0 || key_better(ov, op, cv, cp))) { cv = ov; cp = op; cr = orr; cm = om; }
        }
        if (cr >= 0) {
          for (int c = lane; c < w; c += 32) {
            const unsigned long long x = (unsigned long long)__double_as_longlong(crow[par][cm][c]);
            st_v4(&ws->rowdata[par][0][rec_id][c], (unsigned)x, f, (unsigned)(x >> 32), f);
          }
        }
        if (lane == 0) {
          const unsigned long long x = (unsigned long long)__double_as_longlong(cr >= 0 ? cv : -1.0);
          st_v4(&ws->rec[par][0][rec_id][0], (unsigned)x, f, (unsigned)(x >> 32), f);
          st_v4(&ws->rec[par][0][rec_id][1], (unsigned)cp, f, (unsigned)(cr + 1), f);
        }
        PMARK(7);  // cluster reduce + global publish
        double v = -1.0;
        int pp = 0x7fffffff, rr = -1, cc = -1;
        if (lane < nrec) {
          for (;;) {
            const uint4 qa = ld_v4(&ws->rec[par][0][lane][0]);
            const uint4 qb = ld_v4(&ws->rec[par][0][lane][1]);
            if (qa.y != f || qa.w != f || qb.y != f || qb.w != f) continue;
            if ((int)qb.z - 1 >= 0) { v = join(qa.x, qa.z); pp = (int)qb.x; rr = (int)qb.z - 1; cc = lane; }
            break;
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, v, off);
          const int op = __shfl_xor_sync(0xffffffffu, pp, off);
          const int orr = __shfl_xor_sync(0xffffffffu, rr, off);
          const int oc = __shfl_xor_sync(0xffffffffu, cc, off);
          if (orr >= 0 && (rr < 0 || key_better(ov, op, v, pp))) { v = ov; pp = op; rr = orr; cc = oc; }
        }
        PMARK(1);  // gather + global poll
        double u0 = 0.0, u1 = 0.0;  // U row columns 2 lane, 2 lane + 1
        if (rr >= 0 && v > 0.0) {
          const int c0 = 2 * lane, c1 = c0 + 1;
          bool need0 = c0 < w, need1 = c1 < w;
          while (need0 || need1) {
            uint4 x0 = make_uint4(0, 0, 0, 0), x1 = make_uint4(0, 0, 0, 0);
            if (need0) x0 = ld_v4(&ws->rowdata[par][0][cc][c0]);
            if (need1) x1 = ld_v4(&ws->rowdata[par][0][cc][c1]);
            if (need0 && x0.y == f && x0.w == f) { u0 = join(x0.x, x0.z); need0 = false; }
            if (need1 && x1.y == f && x1.w == f) { u1 = join(x1.x, x1.z); need1 = false; }
          }
        }
        const unsigned long long vx = (unsigned long long)__double_as_longlong(rr >= 0 ? v : 0.0);
        const unsigned long long ux0 = (unsigned long long)__double_as_longlong(u0);
        const unsigned long long ux1 = (unsigned long long)__double_as_longlong(u1);
        for (int r = 0; r < CL; ++r) {
          uint32_t m_bar, m_rec, m_row;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(m_bar) : "r"(smem_u32(&bbar[par])), "r"(r));
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(m_rec) : "r"(smem_u32(&brec[par])), "r"(r));
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(m_row) : "r"(smem_u32(&Urow2[par][0])), "r"(r));
          if (lane == 0)
            st_async_v4(m_rec, (unsigned)vx, (unsigned)(vx >> 32), (unsigned)pp, (unsigned)(rr + 1), m_bar);
          st_async_v4(m_row + 16u * lane, (unsigned)ux0, (unsigned)(ux0 >> 32), (unsigned)ux1, (unsigned)(ux1 >> 32),
                      m_bar);
        }
      }
      // (3) every CTA: the step's winner and U row arrive in its own shared memory
      mb_wait_cluster(&bbar[par], ph);
      if (lane == 0) {
        const uint4 q = brec[par];
        s_val = join(q.x, q.y);
        s_pos = (int)q.z;
        s_row = (int)q.w - 1;
      }
      __syncwarp();
      PMARK(2);  // broadcast
     } else {
      const unsigned f = flag_base + (unsigned)j + 1u;
      // ---- publish this CTA's candidate for column j (no fence needed).
      // The record goes first: it is what every CTA polls; the row values are
      // read only by the winner's readers, one exchange hop later. ----
      if (lane < NREP) {  // (bv, bp, br are uniform across the warp)
        const double v = br >= 0 ? bv : -1.0;
        const unsigned long long x = (unsigned long long)__double_as_longlong(v);
        const unsigned growp1 = br >= 0 ? (unsigned)(r0 + br + 1) : 0u;
        st_v4(&ws->rec[par][lane][cta][0], (unsigned)x, f, (unsigned)(x >> 32), f);
        st_v4(&ws->rec[par][lane][cta][1], (unsigned)bp, f, growp1, f);
      }
      if (br >= 0) {
        for (int c = lane; c < w; c += 32) {
          const unsigned long long x = (unsigned long long)__double_as_longlong(at(br, c));
#pragma unroll
          for (int rp = 0; rp < RD_NREP; ++rp)
            st_v4(&ws->rowdata[par][rp][cta][c], (unsigned)x, f, (unsigned)(x >> 32), f);
        }
      }
      PMARK(0);  // publish
      // ---- reduce the published candidates: every CTA polls all records itself
      // (all-to-all, one hop; identical reduction order on every CTA) ----
      double v = -1.0;
      int pp = 0x7fffffff, rr = -1, cc = -1;
      {
        // Poll all of this lane's records in one pass (loads issued back to
        // back, then checked), repeat only for the ones not yet published.
        const int nq = (nrec - lane + 31) / 32;
        unsigned pending = nq >= 32 ? 0xffffffffu : ((1u << nq) - 1u);
        while (pending) {
          uint4 a[QMAX], b[QMAX];
#pragma unroll
          for (int i = 0; i < QMAX; ++i) {
            if ((pending >> i) & 1u) {
              a[i] = ld_v4(&ws->rec[par][cta % NREP][lane + 32 * i][0]);
              b[i] = ld_v4(&ws->rec[par][cta % NREP][lane + 32 * i][1]);
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
              v = qv; pp = qp; rr = row; cc = row / rows_per;  // the winner's CTA
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
      // ---- pivot row (U row j) straight from the winner's published copy ----
      if (rr >= 0 && v > 0.0) {
        const int c0 = j + lane, c1 = j + lane + 32;
        bool need0 = c0 < w, need1 = c1 < w;
        while (need0 || need1) {  // both words in flight at once
          uint4 x0 = make_uint4(0, 0, 0, 0), x1 = make_uint4(0, 0, 0, 0);
          if (need0) x0 = ld_v4(&ws->rowdata[par][cta % RD_NREP][cc][c0]);
          if (need1) x1 = ld_v4(&ws->rowdata[par][cta % RD_NREP][cc][c1]);
          if (need0 && x0.y == f && x0.w == f) { Urow2[par][c0] = join(x0.x, x0.z); need0 = false; }
          if (need1 && x1.y == f && x1.w == f) { Urow2[par][c1] = join(x1.x, x1.z); need1 = false; }
        }
      }
     }
    } else if (late_j >= 0) {
      // ---- late update of the previous step (off the critical path) ----
      // Rank-1 update of columns jl+2.. of every live row; each lane owns at
      // most two columns (u0, u1 in registers) and walks 4 rows per trip so
      // the smem load -> dmul -> dsub -> store chains overlap.
      if (warp_early) {
        // warp 0 did step late_j's early update alone: wait for its scaled column
        asm volatile("bar.sync 2, %0;\n" ::"r"(PTHREADS) : "memory");
        late_skip = s_skip;
      }
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
    if (warp_early) {
      // Few rows per CTA: warp 0 alone scales column j and updates column j + 1 of up to
      // EU_MAX rows per lane (independent rows, so the divisions overlap), then a warp
      // argmax -- no block-wide barrier on the critical path.  Warps 1-7 wait for it on a
      // named barrier before the late update of this column.
      if (warp == 0) {
#pragma unroll
        for (int q = 0; q < EU_MAX; ++q) {
          const int i = lane + 32 * q;
          if (i < nloc) {
            int pi = pos[i];
            if (pi >= j) {
              if (r0 + i == prow) {
                pos[i] = j;
              } else {
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
            }
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
          const int op = __shfl_xor_sync(0xffffffffu, bp, off);
          const int orr = __shfl_xor_sync(0xffffffffu, br, off);
          if (orr >= 0 && (br < 0 || key_better(ov, op, bv, bp))) { bv = ov; bp = op; br = orr; }
        }
        PMARK(4);  // early update + warp argmax
        if (br >= 0) {
          const double l = at(br, j);
          for (int c = j + 2 + lane; c < w; c += 32) {
            double& a = at(br, c);
            a = __dsub_rn(a, __dmul_rn(l, Urow2[par][c]));
          }
        }
        if (lane == 0) s_skip = br;
        __syncwarp();
        // the last column has no late update: no arrival, so the barrier stays balanced
        if (j + 1 < w) asm volatile("bar.arrive 2, %0;\n" ::"r"(PTHREADS) : "memory");
      }
      late_j = j;
      late_skip = br;  // (warps 1-7 read s_skip after the named barrier)
      PMARK(5);  // best row update
      continue;
    }
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
  tstep[ncols < w ? ncols : w] = clock64();
  if (tid == 0) {
    unsigned sm_all;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_all));
    printf("CTASM %d %u %d\n", cta, sm_all, G);
  }
  if (tid == 0 && (cta == 0 || cta == G / 2)) {
    // per-column durations: the five slowest and the median
    unsigned long long d[PMAXW];
    const int nn = ncols < w ? ncols : w;
    for (int q = 0; q < nn; ++q) d[q] = tstep[q + 1] - tstep[q];
    unsigned long long srt[PMAXW];
    for (int q = 0; q < nn; ++q) srt[q] = d[q];
    for (int a = 1; a < nn; ++a) {
      unsigned long long v = srt[a];
      int b2 = a - 1;
      while (b2 >= 0 && srt[b2] > v) { srt[b2 + 1] = srt[b2]; --b2; }
      srt[b2 + 1] = v;
    }
    int top[5] = {-1, -1, -1, -1, -1};
    for (int t = 0; t < 5 && t < nn; ++t) {
      unsigned long long best = 0; int bj = -1;
      for (int q = 0; q < nn; ++q) {
        bool used = false;
        for (int u = 0; u < t; ++u) used |= top[u] == q;
        if (!used && d[q] >= best) { best = d[q]; bj = q; }
      }
      top[t] = bj;
    }
    unsigned smid_;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));
    printf("smid %u ", smid_);
    printf("cta %d steps: median %llu min %llu max %llu cycles; slowest j=%d:%llu j=%d:%llu j=%d:%llu j=%d:%llu j=%d:%llu\n",
           cta, srt[nn / 2], srt[0], srt[nn - 1], top[0], d[top[0]], top[1], d[top[1]], top[2], d[top[2]], top[3],
           d[top[3]], top[4], d[top[4]]);
  }
  if (PANEL_DBG && tid == 32 && (cta == 0 || cta == G / 2 || cta == 1)) tp_late_out[cta] = tlate;
  __syncthreads();
  unsigned long long gt1 = 0;
  if (PANEL_DBG) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
  if (PANEL_DBG && tid == 0 && (cta == 0 || cta == G / 2 || cta == 1))
    printf("panel cta %d/%d rows %d: publish %llu poll %llu row %llu sync %llu early %llu best %llu late(warp 1) %llu"
           " [cluster: gather %llu reduce+publish %llu] (cycles, %d cols); loop %llu cycles in %llu ns\n",
           cta, G, nloc, tp[0], tp[1], tp[2], tp[3], tp[4], tp[5], tp_late_out[cta], tp[6], tp[7], w,
           clock64() - ck0, gt1 - gt0);
#endif
  __syncthreads();
  if constexpr (CL > 1) cluster_sync_all();  // no CTA leaves while its leader may be written

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
#ifndef RS_PANEL_CLUSTER  // cluster size of the two-level exchange; 1 = flat (the default, faster)
#define RS_PANEL_CLUSTER 1
#endif
  constexpr int CL = RS_PANEL_CLUSTER;
  constexpr int FLAT_MAX = 64;  // the flat exchange's hop is ~1 us up to 64 records, ~3 us at 148
#ifndef RS_PANEL_MAXG  // experiment cap on the grid (fewer, fuller CTAs: a cheaper exchange)
#define RS_PANEL_MAXG 1024
#endif
  int G = (R + RS_PANEL_ROWS - 1) / RS_PANEL_ROWS;
  if (G > nsm) G = nsm;
  if (G > RS_PANEL_MAXG) G = RS_PANEL_MAXG;
  if (G > PMAXG) G = PMAXG;
  if (G < 1) G = 1;
  size_t static_smem = 2048;  // >= the kernel's static shared memory (12 KB with the cluster slots)
  auto round16 = [](size_t x) { return (x + 15) & ~size_t(15); };
  auto smem_for = [&](int g, bool& rows_global) {
    const int rp = (R + g - 1) / g;
    size_t sm = round16((size_t)rp * PMAXW * sizeof(double) + (size_t)rp * sizeof(int));
    // rows in shared memory when they fit, else in place in global memory (L2)
    rows_global = sm + static_smem > (size_t)max_smem;
    if (rows_global) sm = round16((size_t)rp * sizeof(int));
    return sm;
  };
  static const void* const flat_kernels[2][4] = {
      {(const void*)panel_kernel<1, false, 1>, (const void*)panel_kernel<2, false, 1>,
       (const void*)panel_kernel<4, false, 1>, (const void*)panel_kernel<8, false, 1>},
      {(const void*)panel_kernel<1, true, 1>, (const void*)panel_kernel<2, true, 1>,
       (const void*)panel_kernel<4, true, 1>, (const void*)panel_kernel<8, true, 1>}};
  static const void* const cluster_kernels[2] = {(const void*)panel_kernel<1, false, CL>,
                                                 (const void*)panel_kernel<1, true, CL>};
  bool rows_global = false;
  size_t smem = 0;
  const void* kern = nullptr;
  bool clustered = false;
  if (CL > 1 && G > FLAT_MAX) {
    // Two-level exchange: G a multiple of CL, no more clusters than fit at once (a cluster
    // lives in one GPC, so with one CTA per SM a few SMs per GPC may stay idle).
    int g = std::min((G + CL - 1) / CL * CL, nsm / CL * CL);
    static_smem = 12288;
    smem = smem_for(g, rows_global);
    // one CTA per SM: a second CTA on an SM would slow every step of the exchange
    const size_t one_per_sm = (size_t)max_smem / 2 + 8192 - static_smem;  // 2 x (this + static + 1 KB) > an SM
    smem = std::max(smem, one_per_sm);
    kern = cluster_kernels[rows_global ? 1 : 0];
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(g);
    cfg.blockDim = dim3(PTHREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // With one CTA per SM forced, the cluster capacity does not depend on the shared-memory
    // size: query it once per device (the query costs more than the panel launch).
    static int maxcl_cache[64];
    static bool maxcl_known[64];
    int maxcl = 0;
    bool ok = true;
    if (dev < 64 && maxcl_known[dev]) {
      maxcl = maxcl_cache[dev];
    } else {
      ok = cudaOccupancyMaxActiveClusters(&maxcl, kern, &cfg) == cudaSuccess;
      if (ok && dev < 64) { maxcl_cache[dev] = maxcl; maxcl_known[dev] = true; }
    }
    if (ok && maxcl * CL >= FLAT_MAX) {
      if (g > maxcl * CL) {
        g = maxcl * CL;
        smem = std::max(smem_for(g, rows_global), one_per_sm);
        kern = cluster_kernels[rows_global ? 1 : 0];
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      }
      G = g;
      clustered = true;
    } else {
      cudaGetLastError();  // no cluster placement: fall back to the flat exchange
      static_smem = 2048;
    }
  }
  if (!clustered) {
    smem = smem_for(G, rows_global);
    const int q = G <= 32 ? 0 : G <= 64 ? 1 : G <= 128 ? 2 : 3;  // polled records per lane <= 32 * QMAX
    kern = flat_kernels[rows_global ? 1 : 0][q];
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  if (smem + static_smem > (size_t)max_smem) return RS_ERR_CAPACITY;
  const int rows_per = (R + G - 1) / G;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, PTHREADS, smem);
  if (occ * nsm < G) return RS_ERR_CAPACITY;
  PanelScratch* ws = static_cast<PanelScratch*>(workspace);
  // Flags of launch e are e*128 + j + 1: stale words of earlier launches never match.
  static std::atomic<unsigned> epoch{1};
  unsigned flag_base = (epoch.fetch_add(1) & 0x1ffffffu) << 7;
  void* args[] = {&S, &lds, &R, &w, (void*)&rows_per, &perm_out, &ncols_dev, &ws, &flag_base};
  cudaError_t e;
  if (clustered) {
    // all CTAs co-resident (the exchange spins on every CTA): cooperative + cluster launch
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(PTHREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    e = cudaLaunchKernelExC(&cfg, kern, args);
  } else {
    e = cudaLaunchCooperativeKernel(kern, dim3(G), dim3(PTHREADS), args, smem, st);
  }
  count_launch(1);
  return e == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

}  // namespace rs
