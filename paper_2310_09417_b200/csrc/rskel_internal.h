// Internal launch interfaces shared by the kernel translation units and the
// C-ABI layer (capi.cu).  Nothing here crosses the library boundary.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rs {

// Every kernel launch of the library bumps this counter (rs_launch_count()).
void count_launch(int n);

struct DGemmParams {
  int M, N, K;
  const double* A;
  long long lda;
  const int64_t* aidx;  // row-major A only: row i of A is A[aidx[i]]
  const double* B;
  long long ldb;
  const int64_t* bidx;  // row k of B is B[bidx[k]]
  const double* Cin;
  long long ldcin;
  const int64_t* cidx;  // row i of Cin is Cin[cidx[i]]
  double* C;
  long long ldc;
  double alpha, beta;
  int mode;          // RS_GEMM_PLAIN / RS_GEMM_FOLD / RS_GEMM_CHAIN (rskel.h)
  double* slots;     // partial-tile slots (GEMM_SLOTS x 128 x 64 doubles)
  int* tickets;      // per-tile arrival counters (GEMM_SLOTS ints, zero between launches)
  int nslots;
  double* bslots;    // chain values handed from CTA g to g + 1 (GEMM_MAX_CTAS slots)
  unsigned* bflags;  // their release flags (launch epochs)
};

// Deterministic chunking of K (gemm_f64.cu): at most GEMM_MAX_CHUNKS chunks of
// kc >= GEMM_MIN_CHUNK columns, kc a multiple of 32, a function of K alone.
constexpr int GEMM_SLOTS = 4096;
constexpr int GEMM_MAX_CTAS = 512;  // >= persistent CTAs of one GEMM launch
constexpr int GEMM_MAX_CHUNKS = 32;
constexpr int GEMM_MIN_CHUNK = 1024;
size_t gemm_workspace_bytes();
int gemm_chunk(long long K);
// kc <= 0: gemm_chunk(K)
int launch_dgemm(const DGemmParams& p, bool a_col, int kc, cudaStream_t st);
// C[i, :] = Cin[cidx[i], :] - A[i, :K] B[bidx[0..K), :], K <= 64 (rank_update.cu)
int launch_rank_update(int M, int N, int K, const double* A, long long lda, const double* B,
                       long long ldb, const int64_t* bidx, const double* Cin, long long ldcin,
                       const int64_t* cidx, double* C, long long ldc, cudaStream_t st);

// Panel LUPP (cooperative grid).  Factors the R x w row-major block S in
// place with partial pivoting (first maximum in the current position wins,
// `dense.py:185-207`); rows stay in physical order, the position map is
// returned as perm_out (position -> physical row), *ncols_dev receives the
// number of eliminated columns.  Workspace: see panel_workspace_bytes().
size_t panel_workspace_bytes();
int launch_panel(double* S, long long lds, int R, int w, int64_t* perm_out, int* ncols_dev,
                 void* workspace, cudaStream_t st);

int launch_gather_rows(const double* src, long long lds, const int64_t* idx, int nrows, int ncols,
                       double* dst, long long ldd, cudaStream_t st);
size_t sumsq_workspace_bytes();
int launch_sumsq(const double* X, long long ldx, int R, int w, double* partial_ws, double* out,
                 cudaStream_t st);
int launch_trinv(const double* T, long long rs_, long long cs_, const int64_t* ridx, int n, int lower,
                 int unit, double* out, long long ldo, cudaStream_t st);
int launch_what(const double* S, long long lds, const int64_t* sub, int nc, const int64_t* ridx, int R, double* out,
                long long ldo, cudaStream_t st);
int launch_perm_update(const int64_t* perm, int64_t* perm_new, int m, int k, const int64_t* sub,
                       cudaStream_t st);
int launch_iota(int64_t* p, int n, cudaStream_t st);
int launch_shard_maps(const int64_t* perm, int m, int k, long long lo, long long hi, const int64_t* lrow_old,
                      const int64_t* sub, int k_old, int nc, int64_t* lrow, int64_t* loc, int64_t* spos,
                      int64_t* src_row, int64_t* wsrc, int64_t* tp_src, int64_t* ytop_src, int* count,
                      int pad_to, cudaStream_t st);
int launch_shard_max_count(const int64_t* perm, int m, int k, const int64_t* bounds, int world, int* out_max,
                           cudaStream_t st);
int launch_scatter_rows(const double* src, long long lds, const int64_t* idx, int nrows, int ncols, double* dst,
                        long long ldd, cudaStream_t st);
int launch_scatter_interp_local(const double* T, long long ldt, const int64_t* perm, int k, const int64_t* loc,
                                int r, long long lo, long long hi, double* W, long long ldw, cudaStream_t st);
int launch_scatter_interp(const double* T, long long ldt, const int64_t* perm, int m, int k, double* W,
                          long long ldw, cudaStream_t st);
// One-sided Jacobi SVD / pinv helpers (svd.cu)
int launch_jacobi_round(double* Xt, long long ldx, int p, double* Vt, long long ldv, int q, const int* pairs,
                        int npairs, double tol, unsigned long long* max_off, cudaStream_t st);
int launch_pinv_scale(const double* Xt, long long ldx, int p, double* Vt, long long ldv, int q, double rcond,
                      double* sigma, cudaStream_t st);
int launch_jacobi_sweep(double* Xt, long long ldx, int p, double* Vt, long long ldv, int q, const int* sched,
                        int nrounds, int npairs, double tol, unsigned long long* max_off, unsigned* bar,
                        cudaStream_t st);
int launch_srtt_dense(int n, int ell, const int64_t* perm, const double* signs, const int64_t* cols, double scale,
                      double* out, long long ldo, cudaStream_t st);
int launch_sparse_sign_dense(int n, int ell, int zeta, const int64_t* idx, const double* signs, double scale,
                             double* out, long long ldo, cudaStream_t st);
long long srtt_workspace_bytes(long long m, int n);
int launch_srtt_apply(long long m, int n, int ell, const double* a, long long lda, int colmajor,
                      const int64_t* perm, const double* signs, const int64_t* cols, double scale, double* y,
                      long long ldy, void* ws, long long ws_bytes, cudaStream_t st);
long long sparse_sign_plan_words(int n, int ell);
int launch_sparse_sign_apply(long long m, int n, int ell, int zeta, const double* a, long long lda, int colmajor,
                             const int64_t* idx, const double* signs, double scale, double* y, long long ldy,
                             unsigned* plan, int* bad, cudaStream_t st);
int launch_cholesky(double* G, long long ldg, int n, int* status, cudaStream_t st);
int launch_trsv_cols(const double* cols, long long ldc, int n, int lower, int unit, double* x, cudaStream_t st);
int launch_norm1(const double* A, long long lda, int rows, int cols, double* out, cudaStream_t st);
int launch_gather2d(const double* src, long long rs_, long long cs_, const int64_t* ridx, int nr,
                    const int64_t* cidx, int nc, double* dst, long long ldd, cudaStream_t st);
// numpy Generator(Philox).standard_normal on the device (gaussian_rng.cu)
size_t gaussian_workspace_bytes(long long N);
int launch_gaussian(uint64_t seed, uint64_t stream, long long N, double scale, double* out, void* ws,
                    size_t ws_bytes, int* status_dev, cudaStream_t st);
// Ozaki-scheme sketch GEMM on tcgen05 kind::i8 (ozaki.cu)
int oz_chunk(long long K);
size_t oz_digits_bytes(int rows, long long K, int S, int tile_rows);
int launch_oz_slice(const void* X, int fp32, long long ld, int colmajor, int rows, int K, int k0, int k1, int kc,
                    int S, int tile_rows, int8_t* dig, int* expo, int* nonfinite, unsigned long long* mx,
                    size_t mx_bytes, cudaStream_t st);
int launch_oz_gemm(int M, int N, int K, int kc, int mode, double alpha, const int8_t* adig, const int* aexp, int SA,
                   const int8_t* bdig, const int* bexp, int SB, double beta, const double* Cin, long long ldcin,
                   double* C, long long ldc, double* slots, int* tickets, int nslots, long long* hl, int hl_units, int* tail_tickets, cudaStream_t st);
// Input generators (gen.cu)
int launch_uniform(uint64_t k0, uint64_t k1, long long n, double* out, cudaStream_t st);
int launch_hadamard_init(double* x, long long ld, int n, double c, const double* rowscale, cudaStream_t st);
int launch_fwht_rows(double* x, long long ld, int n, double c, const double* rowscale, cudaStream_t st);
int launch_kahan(double* a, long long ld, int n, const double* rowpow, double negphi, cudaStream_t st);
int launch_chan(double* a, long long ld, int n, cudaStream_t st);
int launch_axpy_cast(const double* x, const double* y, double beta, long long n, double* out64, float* out32,
                     cudaStream_t st);
int launch_transpose(const double* src, long long lds, int rows, int cols, double* dst, long long ldd,
                     cudaStream_t st);

}  // namespace rs
