// Panel LU with partial pivoting on a tall R x w block (w <= 64), the kernel
// behind `_lupp_panel` (`dense.py:185-207`) for the sketch blocks and Schur
// blocks of the adaptive loop (`skeleton.py:317-351`).
//
// Design (B200): one cooperative grid of G CTAs, CTA g keeps its contiguous
// slice of rows resident in shared memory for the whole panel (a 65472 x 64
// fp64 Schur block is 33.5 MB = 148 CTAs x 226 KB).  Rows never move: the
// reference's full-row swaps are replaced by a position map pos[row] (the
// "current permuted position" that breaks argmax ties, `dense.py:194`).  Per
// column j each CTA publishes its best (|v|, pos, row, row values) candidate,
// one grid barrier, then every CTA reduces the G candidates identically
// (deterministic), takes the pivot row from the candidate buffer and applies
// scale + rank-1 update to its own rows while computing its next candidate.
// That is one grid barrier per eliminated column.
//
// Arithmetic follows numpy's rounding exactly: l = s / pivot (IEEE division),
// s' = s - (l * u) with the product rounded before the subtraction (np.outer
// then -=), i.e. no FMA contraction.
#include "common.cuh"
#include "rskel_internal.h"

namespace rs {

constexpr int PTHREADS = 256;
constexpr int PWARPS = PTHREADS / 32;
constexpr int PMAXW = 64;
constexpr int PMAXG = 1024;

struct PanelScratch {
  unsigned bar;
  unsigned pad[31];
  double cval[2][PMAXG];
  int cpos[2][PMAXG];
  int crow[2][PMAXG];
  double crowdata[2][PMAXG][PMAXW];
};

size_t panel_workspace_bytes() { return sizeof(PanelScratch); }

__global__ void __launch_bounds__(PTHREADS, 1)
    panel_kernel(double* __restrict__ S, long long lds, int R, int w, int rows_per,
                 int64_t* __restrict__ perm_out, int* __restrict__ ncols_out, PanelScratch* ws) {
  extern __shared__ __align__(16) double psm[];
  const int G = gridDim.x, cta = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r0 = cta * rows_per;
  int nloc = R - r0;
  nloc = nloc < 0 ? 0 : (nloc > rows_per ? rows_per : nloc);

  double* Ss = psm;                                  // nloc x w
  int* pos = reinterpret_cast<int*>(psm + (size_t)rows_per * w);  // nloc
  __shared__ double Urow[PMAXW];
  __shared__ double wv[PWARPS];
  __shared__ int wp[PWARPS], wr[PWARPS];
  __shared__ double s_val;
  __shared__ int s_pos, s_row, s_cta, s_best_local;

  for (int idx = tid; idx < nloc * w; idx += PTHREADS) {
    int i = idx / w, c = idx - i * w;
    Ss[idx] = S[(long long)(r0 + i) * lds + c];
  }
  for (int i = tid; i < nloc; i += PTHREADS) pos[i] = r0 + i;
  __syncthreads();

  // Warp-uniform running best for the current column.
  double bv = -1.0;
  int bp = 0x7fffffff, br = -1;
  for (int i = warp; i < nloc; i += PWARPS) {
    double v = fabs(Ss[i * w]);
    if (key_better(v, pos[i], bv, bp)) { bv = v; bp = pos[i]; br = i; }
  }

  int ncols = w;
  for (int j = 0; j < w; ++j) {
    const int par = j & 1;
    // ---- CTA candidate ----
    if (lane == 0) { wv[warp] = bv; wp[warp] = bp; wr[warp] = br; }
    __syncthreads();
    if (tid == 0) {
      double v = -1.0; int pp = 0x7fffffff, rr = -1;
      for (int q = 0; q < PWARPS; ++q)
        if (wr[q] >= 0 && key_better(wv[q], wp[q], v, pp)) { v = wv[q]; pp = wp[q]; rr = wr[q]; }
      s_best_local = rr;
      ws->cval[par][cta] = rr >= 0 ? v : -1.0;
      ws->cpos[par][cta] = pp;
      ws->crow[par][cta] = rr >= 0 ? r0 + rr : -1;
    }
    __syncthreads();
    if (tid < w) ws->crowdata[par][cta][tid] = s_best_local >= 0 ? Ss[s_best_local * w + tid] : 0.0;
    __threadfence();
    grid_barrier(&ws->bar, (unsigned)(j + 1) * (unsigned)G);

    // ---- global pivot (every CTA reduces the same candidates in the same way) ----
    if (warp == 0) {
      double v = -1.0; int pp = 0x7fffffff, rr = -1, cc = -1;
      for (int q = lane; q < G; q += 32) {
        int row = __ldcg(&ws->crow[par][q]);
        if (row < 0) continue;
        double qv = __ldcg(&ws->cval[par][q]);
        int qp = __ldcg(&ws->cpos[par][q]);
        if (key_better(qv, qp, v, pp)) { v = qv; pp = qp; rr = row; cc = q; }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, v, off);
        int op = __shfl_xor_sync(0xffffffffu, pp, off);
        int orr = __shfl_xor_sync(0xffffffffu, rr, off);
        int oc = __shfl_xor_sync(0xffffffffu, cc, off);
        if (orr >= 0 && (rr < 0 || key_better(ov, op, v, pp))) { v = ov; pp = op; rr = orr; cc = oc; }
      }
      if (lane == 0) { s_val = rr >= 0 ? v : 0.0; s_pos = pp; s_row = rr; s_cta = cc; }
    }
    __syncthreads();
    if (!(s_val > 0.0)) { ncols = j; break; }  // exactly-zero pivot column (or no rows left)
    const int ppos = s_pos, prow = s_row;
    if (tid >= j && tid < w) Urow[tid] = __ldcg(&ws->crowdata[par][s_cta][tid]);
    __syncthreads();

    // ---- swap bookkeeping, scale, rank-1 update, next candidate ----
    const double upiv = Urow[j];
    bv = -1.0; bp = 0x7fffffff; br = -1;
    for (int i = warp; i < nloc; i += PWARPS) {
      int pi = pos[i];
      if (pi < j) continue;             // pivoted in an earlier column
      if (r0 + i == prow) {             // the pivot row moves to position j
        __syncwarp();
        if (lane == 0) pos[i] = j;
        continue;
      }
      if (pi == j) pi = ppos;           // the row at position j takes the pivot's old slot
      double l = __ddiv_rn(Ss[i * w + j], upiv);
      __syncwarp();
      if (lane == 0) pos[i] = pi;
      double v0 = 0.0, v1 = 0.0;
      {
        int c = lane;
        if (c < w) {
          if (c == j) Ss[i * w + c] = l;
          else if (c > j) { v0 = __dsub_rn(Ss[i * w + c], __dmul_rn(l, Urow[c])); Ss[i * w + c] = v0; }
        }
        c = lane + 32;
        if (c < w) {
          if (c == j) Ss[i * w + c] = l;
          else if (c > j) { v1 = __dsub_rn(Ss[i * w + c], __dmul_rn(l, Urow[c])); Ss[i * w + c] = v1; }
        }
      }
      if (j + 1 < w) {
        int jn = j + 1;
        double nv = __shfl_sync(0xffffffffu, jn >= 32 ? v1 : v0, jn & 31);
        nv = fabs(nv);
        if (key_better(nv, pi, bv, bp)) { bv = nv; bp = pi; br = i; }
      }
    }
    __syncthreads();
  }

  // ---- write back factors (physical row order) and the position map ----
  for (int idx = tid; idx < nloc * w; idx += PTHREADS) {
    int i = idx / w, c = idx - i * w;
    S[(long long)(r0 + i) * lds + c] = Ss[idx];
  }
  for (int i = tid; i < nloc; i += PTHREADS) perm_out[pos[i]] = r0 + i;
  if (cta == 0 && tid == 0) *ncols_out = ncols;
}

int launch_panel(double* S, long long lds, int R, int w, int64_t* perm_out, int* ncols_dev,
                 void* workspace, cudaStream_t st) {
  if (R < 0 || w < 0 || w > PMAXW || (R > 0 && lds < w)) return RS_ERR_ARG;
  if (R == 0 || w == 0) {
    int zero_cols = (R == 0) ? 0 : w;
    (void)zero_cols;
    cudaMemsetAsync(ncols_dev, 0, sizeof(int), st);
    return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  int nsm = 0, max_smem = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // Small panels: fewer CTAs, cheaper barrier.  Large: one CTA per SM.
  int G = (R + 127) / 128;
  if (G > nsm) G = nsm;
  if (G < 1) G = 1;
  int rows_per = (R + G - 1) / G;
  const size_t static_smem = 4096;  // Urow + reduction scratch (upper bound)
  size_t smem = (size_t)rows_per * w * sizeof(double) + (size_t)rows_per * sizeof(int);
  smem = (smem + 15) & ~size_t(15);
  if (smem + static_smem > (size_t)max_smem) return RS_ERR_CAPACITY;
  cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, panel_kernel, PTHREADS, smem);
  if (occ * nsm < G || G > PMAXG) return RS_ERR_CAPACITY;
  PanelScratch* ws = static_cast<PanelScratch*>(workspace);
  cudaMemsetAsync(&ws->bar, 0, sizeof(unsigned), st);
  void* args[] = {&S, &lds, &R, &w, &rows_per, &perm_out, &ncols_dev, &ws};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)panel_kernel, dim3(G), dim3(PTHREADS), args, smem, st);
  count_launch(1);
  return e == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

}  // namespace rs
