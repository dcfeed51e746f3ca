// extern "C" boundary of librskel.so (declared in include/rskel.h).
// Composite calls (Schur block, absorb block) are sequences of the kernels in
// gemm_f64.cu / panel.cu / aux.cu enqueued on the caller's stream.
#include <atomic>
#include <cstdlib>

#include "common.cuh"
#include "rskel_internal.h"

namespace rs {
static std::atomic<unsigned long long> g_launch_count{0};
void count_launch(int n) { g_launch_count.fetch_add((unsigned long long)n, std::memory_order_relaxed); }
}  // namespace rs

namespace {

constexpr int kMaxB = 64;
#ifndef RS_SCHUR_STAGE_B  // experiment builds: 0 = the GEMM gathers Y[perm[:k]] per stage
#define RS_SCHUR_STAGE_B 1
#endif

struct WorkspaceLayout {
  size_t panel_off, sumsq_off, gemm_off, ytop_off, total;
};

// Y[perm[:k]] staged contiguously for the Schur GEMM's B operand (k <= kYtopRows)
constexpr long long kYtopRows = 65536;

// Fixed layout (device independent); the GEMM ticket counters at the end of
// the GEMM region must be zero when the workspace is first used.
WorkspaceLayout layout() {
  WorkspaceLayout L;
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  L.panel_off = 0;
  L.sumsq_off = up(rs::panel_workspace_bytes());
  L.gemm_off = L.sumsq_off + up(rs::sumsq_workspace_bytes());
  L.ytop_off = L.gemm_off + up(rs::gemm_workspace_bytes());
  L.total = L.ytop_off + up(sizeof(double) * (size_t)kYtopRows * kMaxB);
  return L;
}

inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
inline char* W(void* ws, size_t off) { return static_cast<char*>(ws) + off; }

rs::DGemmParams gemm_params(int M, int N, int K, double alpha, const double* A, long long lda, const int64_t* aidx,
                            const double* B, long long ldb, const int64_t* bidx, double beta, const double* Cin,
                            long long ldcin, const int64_t* cidx, double* C, long long ldc, int mode, void* ws) {
  rs::DGemmParams p{M, N, K, A, lda, aidx, B, ldb, bidx, Cin, ldcin, cidx, C, ldc, alpha, beta, mode,
                    nullptr, nullptr, 0, nullptr, nullptr};
  if (ws) {
    // [slots | boundary slots | tickets | boundary flags]
    p.slots = reinterpret_cast<double*>(W(ws, layout().gemm_off));
    p.bslots = p.slots + (size_t)rs::GEMM_SLOTS * 128 * 64;
    p.tickets = reinterpret_cast<int*>(p.bslots + (size_t)rs::GEMM_MAX_CTAS * 128 * 64);
    p.bflags = reinterpret_cast<unsigned*>(p.tickets + rs::GEMM_SLOTS);
    p.nslots = rs::GEMM_SLOTS;
  }
  return p;
}

}  // namespace

extern "C" {

int rs_abi_version(void) { return RS_ABI_VERSION; }

const char* rs_status_string(int status) {
  switch (status) {
    case RS_OK: return "ok";
    case RS_ERR_ARG: return "invalid argument";
    case RS_ERR_CUDA: return "CUDA launch error";
    case RS_ERR_CAPACITY: return "problem exceeds on-chip capacity of the panel kernel";
    default: return "unknown status";
  }
}

size_t rs_workspace_bytes(void) { return layout().total; }

unsigned long long rs_launch_count(void) { return rs::g_launch_count.load(); }

int rs_gemm_chunk(long long K) { return rs::gemm_chunk(K); }

int rs_dgemm_ex(int M, int N, int K, int kc, int mode, double alpha, const double* A, long long lda, int a_colmajor,
                const int64_t* aidx, const double* B, long long ldb, const int64_t* bidx, double beta,
                const double* Cin, long long ldcin, const int64_t* cidx, double* C, long long ldc,
                void* workspace, void* stream) {
  if (a_colmajor && aidx) return RS_ERR_ARG;
  if (mode == RS_GEMM_PLAIN && beta != 0.0 && Cin == nullptr) return RS_ERR_ARG;
  rs::DGemmParams p = gemm_params(M, N, K, alpha, A, lda, aidx, B, ldb, bidx, beta, Cin, ldcin, cidx, C, ldc,
                                  mode, workspace);
  return rs::launch_dgemm(p, a_colmajor != 0, kc, S(stream));
}

int rs_dgemm(int M, int N, int K, double alpha, const double* A, long long lda, int a_colmajor,
             const int64_t* aidx, const double* B, long long ldb, const int64_t* bidx, double beta,
             const double* Cin, long long ldcin, const int64_t* cidx, double* C, long long ldc,
             void* workspace, void* stream) {
  return rs_dgemm_ex(M, N, K, 0, RS_GEMM_PLAIN, alpha, A, lda, a_colmajor, aidx, B, ldb, bidx, beta, Cin, ldcin,
                     cidx, C, ldc, workspace, stream);
}

int rs_sketch_gemm(int m, int n, int ell, const double* A, long long lda, int a_colmajor,
                   const double* Omega, long long ldo, double* Y, long long ldy, void* workspace,
                   void* stream) {
  return rs_dgemm(m, ell, n, 1.0, A, lda, a_colmajor, nullptr, Omega, ldo, nullptr, 0.0, nullptr, 0,
                  nullptr, Y, ldy, workspace, stream);
}

int rs_panel_lupp(double* S_, long long lds, int R, int w, int64_t* perm_out, int* ncols_dev,
                  void* workspace, void* stream) {
  return rs::launch_panel(S_, lds, R, w, perm_out, ncols_dev, W(workspace, layout().panel_off),
                          S(stream));
}

int rs_sumsq(const double* X, long long ldx, int R, int w, double* out, void* workspace, void* stream) {
  return rs::launch_sumsq(X, ldx, R, w, reinterpret_cast<double*>(W(workspace, layout().sumsq_off)),
                          out, S(stream));
}

int rs_schur_block(int m, int k, int b, const double* Y, long long ldy, const int64_t* perm,
                   const double* T, long long ldt, double* S_, long long lds, double* e2_dev,
                   void* workspace, void* stream) {
  if (m < 0 || k < 0 || k > m || b < 0 || b > kMaxB) return RS_ERR_ARG;
  const int R = m - k;
  int rc;
  if (k == 0) {
    rc = rs::launch_gather_rows(Y, ldy, perm, R, b, S_, lds, S(stream));
  } else if (k <= kYtopRows && RS_SCHUR_STAGE_B) {
    // B = Y[perm[:k]] gathered once into a contiguous k x b block (16-byte loads), so the
    // GEMM's B tiles need no per-stage row-index loads
    double* ytop = reinterpret_cast<double*>(W(workspace, layout().ytop_off));
    rc = rs::launch_gather_rows(Y, ldy, perm, k, b, ytop, b, S(stream));
    if (rc != RS_OK) return rc;
    rs::DGemmParams p = gemm_params(R, b, k, -1.0, T, ldt, nullptr, ytop, b, nullptr, 1.0, Y, ldy, perm + k, S_, lds,
                                    RS_GEMM_PLAIN, workspace);
    rc = rs::launch_dgemm(p, false, 0, S(stream));
  } else {
    rs::DGemmParams p = gemm_params(R, b, k, -1.0, T, ldt, nullptr, Y, ldy, perm, 1.0, Y, ldy, perm + k, S_, lds,
                                    RS_GEMM_PLAIN, workspace);
    rc = rs::launch_dgemm(p, false, 0, S(stream));
  }
  if (rc != RS_OK) return rc;
  if (e2_dev) rc = rs_sumsq(S_, lds, R, b, e2_dev, workspace, stream);
  return rc;
}

int rs_absorb_block(int m, int k, int nc, const double* S_, long long lds, const int64_t* sub_perm,
                    const double* T, long long ldt, double* T_new, const int64_t* perm,
                    int64_t* perm_new, void* workspace, void* stream) {
  if (m < 0 || k < 0 || nc < 0 || nc > kMaxB || k + nc > m) return RS_ERR_ARG;
  const int R = m - k;
  const long long ldn = k + nc;
  int rc = RS_OK;
  if (nc > 0) {
    // W_hat = L_r L_1^{-1} -> T_new[:, k:k+nc] (row-parallel substitution
    // against the unit lower triangle of the pivot rows)
    rc = rs::launch_what(S_, lds, sub_perm, nc, sub_perm + nc, R - nc, T_new + k, ldn, S(stream));
    if (rc != RS_OK) return rc;
    if (k > 0) {
      // T_new[:, :k] = T[Q_hat] - W_hat T[P_hat]  (persistent rank-nc update kernel)
      rc = rs::launch_rank_update(R - nc, k, nc, T_new + k, ldn, T, ldt, sub_perm, T, ldt,
                                  sub_perm + nc, T_new, ldn, S(stream));
      if (rc != RS_OK) return rc;
    }
  }
  return rs::launch_perm_update(perm, perm_new, m, k, sub_perm, S(stream));
}

int rs_absorb_schur(int m, int k, int nc, const double* S_, long long lds, const int64_t* sub_perm,
                    const double* T, long long ldt, double* T_new, const int64_t* perm, int64_t* perm_new,
                    const double* Y_next, long long ldy, double* S_next, double* e2_dev, void* workspace,
                    void* stream) {
  int rc = rs_absorb_block(m, k, nc, S_, lds, sub_perm, T, ldt, T_new, perm, perm_new, workspace, stream);
  if (rc != RS_OK) return rc;
  // the next block is 64 columns wide at row stride ldy; S_next is m x 64
  return rs_schur_block(m, k + nc, nc > 0 ? kMaxB : 0, Y_next, ldy, perm_new, T_new, k + nc, S_next, kMaxB,
                        e2_dev, workspace, stream);
}

int rs_rank_update(int M, int N, int K, const double* A, long long lda, const double* B, long long ldb,
                   const int64_t* bidx, const double* Cin, long long ldcin, const int64_t* cidx,
                   double* C, long long ldc, void* stream) {
  if (bidx == nullptr || cidx == nullptr) return RS_ERR_ARG;
  return rs::launch_rank_update(M, N, K, A, lda, B, ldb, bidx, Cin, ldcin, cidx, C, ldc, S(stream));
}

int rs_scatter_interp(const double* T, long long ldt, const int64_t* perm, int m, int k, double* Wm,
                      long long ldw, void* stream) {
  return rs::launch_scatter_interp(T, ldt, perm, m, k, Wm, ldw, S(stream));
}

int rs_gather_rows(const double* src, long long lds, const int64_t* idx, int nrows, int ncols,
                   double* dst, long long ldd, void* stream) {
  return rs::launch_gather_rows(src, lds, idx, nrows, ncols, dst, ldd, S(stream));
}

int rs_trinv(const double* T, long long rs_, long long cs_, const int64_t* ridx, int n, int lower,
             int unit, double* out, long long ldo, void* stream) {
  return rs::launch_trinv(T, rs_, cs_, ridx, n, lower, unit, out, ldo, S(stream));
}

int rs_perm_update(const int64_t* perm, int64_t* perm_new, int m, int k, const int64_t* sub,
                   void* stream) {
  return rs::launch_perm_update(perm, perm_new, m, k, sub, S(stream));
}

int rs_transpose(const double* src, long long lds, int rows, int cols, double* dst, long long ldd,
                 void* stream) {
  return rs::launch_transpose(src, lds, rows, cols, dst, ldd, S(stream));
}

int rs_jacobi_round(double* Xt, long long ldx, int p, double* Vt, long long ldv, int q, const int* pairs,
                    int npairs, double tol, unsigned long long* max_off, void* stream) {
  return rs::launch_jacobi_round(Xt, ldx, p, Vt, ldv, q, pairs, npairs, tol, max_off, S(stream));
}

int rs_pinv_scale(const double* Xt, long long ldx, int p, double* Vt, long long ldv, int q, double rcond,
                  double* sigma, void* stream) {
  return rs::launch_pinv_scale(Xt, ldx, p, Vt, ldv, q, rcond, sigma, S(stream));
}

int rs_jacobi_sweep(double* Xt, long long ldx, int p, double* Vt, long long ldv, int q, const int* sched,
                    int nrounds, int npairs, double tol, unsigned long long* max_off, unsigned* barrier,
                    void* stream) {
  return rs::launch_jacobi_sweep(Xt, ldx, p, Vt, ldv, q, sched, nrounds, npairs, tol, max_off, barrier, S(stream));
}

int rs_what(const double* S_, long long lds, const int64_t* sub, int nc, const int64_t* ridx, int R, double* out,
            long long ldo, void* stream) {
  return rs::launch_what(S_, lds, sub, nc, ridx, R, out, ldo, S(stream));
}

int rs_srtt_dense(int n, int ell, const int64_t* perm, const double* signs, const int64_t* cols, double scale,
                  double* out, long long ldo, void* stream) {
  return rs::launch_srtt_dense(n, ell, perm, signs, cols, scale, out, ldo, S(stream));
}

int rs_sparse_sign_dense(int n, int ell, int zeta, const int64_t* idx, const double* signs, double scale,
                         double* out, long long ldo, void* stream) {
  return rs::launch_sparse_sign_dense(n, ell, zeta, idx, signs, scale, out, ldo, S(stream));
}

long long rs_srtt_workspace_bytes(long long m, int n) {
  if (m < 0 || n < 1) return 0;
  return rs::srtt_workspace_bytes(m, n);
}

int rs_srtt_apply(long long m, int n, int ell, const double* a, long long lda, int a_colmajor, const int64_t* perm,
                  const double* signs, const int64_t* cols, double scale, double* y, long long ldy, void* ws,
                  long long ws_bytes, void* stream) {
  return rs::launch_srtt_apply(m, n, ell, a, lda, a_colmajor, perm, signs, cols, scale, y, ldy, ws, ws_bytes,
                               S(stream));
}

long long rs_sparse_sign_plan_bytes(int n, int ell) {
  if (n < 1 || ell < 1) return 0;
  return rs::sparse_sign_plan_words(n, ell) * (long long)sizeof(unsigned);
}

int rs_sparse_sign_apply(long long m, int n, int ell, int zeta, const double* a, long long lda, int a_colmajor,
                         const int64_t* idx, const double* signs, double scale, double* y, long long ldy, void* plan,
                         int* bad, void* stream) {
  return rs::launch_sparse_sign_apply(m, n, ell, zeta, a, lda, a_colmajor, idx, signs, scale, y, ldy,
                                      static_cast<unsigned*>(plan), bad, S(stream));
}

int rs_cholesky(double* G, long long ldg, int n, int* status_dev, void* stream) {
  return rs::launch_cholesky(G, ldg, n, status_dev, S(stream));
}

int rs_trsv_cols(const double* cols, long long ldc, int n, int lower, int unit, double* x, void* stream) {
  return rs::launch_trsv_cols(cols, ldc, n, lower, unit, x, S(stream));
}

int rs_norm1(const double* A, long long lda, int rows, int cols, double* out, void* stream) {
  return rs::launch_norm1(A, lda, rows, cols, out, S(stream));
}

int rs_gather2d(const double* src, long long rs_, long long cs_, const int64_t* ridx, int nr,
                const int64_t* cidx, int nc, double* dst, long long ldd, void* stream) {
  return rs::launch_gather2d(src, rs_, cs_, ridx, nr, cidx, nc, dst, ldd, S(stream));
}

size_t rs_gaussian_workspace_bytes(long long n) { return rs::gaussian_workspace_bytes(n); }

int rs_gaussian(unsigned long long seed, unsigned long long stream_id, long long n, double scale, double* out,
                void* rng_workspace, size_t ws_bytes, int* status_dev, void* stream) {
  return rs::launch_gaussian(seed, stream_id, n, scale, out, rng_workspace, ws_bytes, status_dev, S(stream));
}

int rs_iota(int64_t* p, int n, void* stream) { return rs::launch_iota(p, n, S(stream)); }

int rs_shard_maps(const int64_t* perm, int m, int k, long long lo, long long hi, const int64_t* lrow_old,
                  const int64_t* sub, int k_old, int nc, int64_t* lrow, int64_t* loc, int64_t* spos,
                  int64_t* src_row, int64_t* wsrc, int64_t* tp_src, int64_t* ytop_src, int* count, int pad_to,
                  void* stream) {
  return rs::launch_shard_maps(perm, m, k, lo, hi, lrow_old, sub, k_old, nc, lrow, loc, spos, src_row, wsrc,
                               tp_src, ytop_src, count, pad_to, S(stream));
}

int rs_shard_max_count(const int64_t* perm, int m, int k, const int64_t* bounds, int world, int* out_max,
                       void* stream) {
  return rs::launch_shard_max_count(perm, m, k, bounds, world, out_max, S(stream));
}

int rs_scatter_rows(const double* src, long long lds, const int64_t* idx, int nrows, int ncols, double* dst,
                    long long ldd, void* stream) {
  return rs::launch_scatter_rows(src, lds, idx, nrows, ncols, dst, ldd, S(stream));
}

int rs_scatter_interp_local(const double* T, long long ldt, const int64_t* perm, int k, const int64_t* loc, int r,
                            long long lo, long long hi, double* W, long long ldw, void* stream) {
  return rs::launch_scatter_interp_local(T, ldt, perm, k, loc, r, lo, hi, W, ldw, S(stream));
}

int rs_oz_chunk(long long K) { return rs::oz_chunk(K); }

size_t rs_oz_digits_bytes(int rows, long long K, int S, int tile_rows) {
  return rs::oz_digits_bytes(rows, K, S, tile_rows);
}

int rs_oz_slice(const void* X, int fp32, long long ld, int colmajor, int rows, int K, int k0, int k1, int kc,
                int planes, int tile_rows, int8_t* digits, int* expo, int* nonfinite, void* workspace,
                void* stream) {
  if (workspace == nullptr) return RS_ERR_ARG;
  // the row-chunk maxima use the GEMM partial-slot region of the workspace as scratch
  unsigned long long* mx = reinterpret_cast<unsigned long long*>(W(workspace, layout().gemm_off));
  return rs::launch_oz_slice(X, fp32, ld, colmajor, rows, K, k0, k1, kc, planes, tile_rows, digits, expo, nonfinite,
                             mx, sizeof(double) * (size_t)rs::GEMM_SLOTS * 128 * 64, S(stream));
}

int rs_oz_gemm(int M, int N, int K, int kc, int mode, double alpha, const int8_t* a_digits, const int* a_expo,
               int SA, const int8_t* b_digits, const int* b_expo, int SB, double beta, const double* Cin,
               long long ldcin, double* C, long long ldc, void* workspace, void* stream) {
  rs::DGemmParams g = gemm_params(0, 0, 0, 0.0, nullptr, 0, nullptr, nullptr, 0, nullptr, 0.0, nullptr, 0, nullptr,
                                  nullptr, 0, RS_GEMM_PLAIN, workspace);
  // tail split of the last wave: exact (H, L) partials in the chain-slot region (4 slots per
  // tail unit), arrival counters in the last 128 ticket words (tile tickets use < 2048)
  return rs::launch_oz_gemm(M, N, K, kc, mode, alpha, a_digits, a_expo, SA, b_digits, b_expo, SB, beta, Cin, ldcin,
                            C, ldc, g.slots, g.tickets, g.nslots, reinterpret_cast<long long*>(g.bslots),
                            rs::GEMM_MAX_CTAS / 4, g.tickets + (rs::GEMM_SLOTS - rs::GEMM_MAX_CTAS / 4), S(stream));
}

int rs_uniform(unsigned long long seed, unsigned long long stream_id, long long n, double* out, void* stream) {
  return rs::launch_uniform(seed, stream_id, n, out, S(stream));
}

int rs_hadamard_init(double* x, long long ld, int n, double c, const double* rowscale, void* stream) {
  return rs::launch_hadamard_init(x, ld, n, c, rowscale, S(stream));
}

int rs_fwht_rows(double* x, long long ld, int n, double c, const double* rowscale, void* stream) {
  return rs::launch_fwht_rows(x, ld, n, c, rowscale, S(stream));
}

int rs_kahan(double* a, long long ld, int n, const double* rowpow, double negphi, void* stream) {
  return rs::launch_kahan(a, ld, n, rowpow, negphi, S(stream));
}

int rs_chan(double* a, long long ld, int n, void* stream) { return rs::launch_chan(a, ld, n, S(stream)); }

int rs_axpy_cast(const double* x, const double* y, double beta, long long n, double* out64, float* out32,
                 void* stream) {
  return rs::launch_axpy_cast(x, y, beta, n, out64, out32, S(stream));
}

}  // extern "C"
