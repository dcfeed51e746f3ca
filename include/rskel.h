/*
 * rskel.h — C ABI of the B200 randomized-skeleton (sketched LUPP ID/CUR) library
 * `librskel.so` (package paper_2310_09417_b200).
 *
 * The reference (`randskel`, /root/reference/pkg/src/randskel) is a pure
 * Python package with no FFI; its "operator API" is the Python namespace.  The
 * entry points below are the native operations that namespace's hot path
 * reaches through numpy/OpenBLAS/LAPACK, one C function per reference call
 * site (cited per function).  The Python host layer
 * (paper_2310_09417_b200/_lib.py) binds them with ctypes; see INTEGRATION.md.
 *
 * Conventions
 *  - All matrices are fp64, device-resident, row-major with an explicit
 *    leading dimension (elements), unless a `*_colmajor` flag says otherwise.
 *  - Index vectors are int64 (numpy np.intp) device arrays.
 *  - `stream` is a cudaStream_t passed as void*; every call is asynchronous on
 *    it and takes no global lock.  No call allocates or frees device memory:
 *    scratch comes from a caller-owned `workspace` of rs_workspace_bytes().
 *  - Return value: 0 = ok, <0 = error (RS_ERR_*), see rs_status_string().
 *    Numerical outcomes (zero pivots) are reported through device outputs
 *    (`ncols_dev`), mirroring `_lupp_partial`'s ncols (`dense.py:284-298`).
 */
#ifndef RSKEL_H
#define RSKEL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_ABI_VERSION 2
#define RS_OK 0
#define RS_ERR_ARG -1
#define RS_ERR_CUDA -2
#define RS_ERR_CAPACITY -3

/* GEMM accumulation modes (rs_dgemm_ex). */
#define RS_GEMM_PLAIN 0 /* C = alpha * op(A) B + beta * Cin                          */
#define RS_GEMM_FOLD 1  /* C = Cin + op(A) B, the K chunks folded onto Cin in order     */
#define RS_GEMM_CHAIN 2 /* C = Cin + op(A) B, the DMMA chain continued from Cin (K <= kc) */

int rs_abi_version(void);
const char* rs_status_string(int status);

/* Bytes of scratch the composite calls need (panel candidates, reduction
 * partials, GEMM partial tiles and their arrival counters).  One workspace
 * per stream; it must be zero-filled once before its first use (the GEMM
 * counters return to zero after every call). */
size_t rs_workspace_bytes(void);

/* Number of kernels this library has launched in the process (instrumentation). */
unsigned long long rs_launch_count(void);

/* C = alpha * op(A) * B + beta * Cin (row gathers optional, NULL = identity).
 * A: M x K, row-major (A[aidx[i]*lda + k]) or, with a_colmajor, column-major
 * (A[k*lda + i]; aidx must be NULL).  B: K x N row-major, row k at bidx[k].
 * Cin row i at cidx[i].  Replaces the OpenBLAS dgemm calls of `gemm`
 * (dense.py:118-141), `GaussianSketch.apply` (sketching.py:122-128) and the
 * Schur/trailing updates (dense.py:232, skeleton.py:322).
 * Summation order: K is cut into chunks of rs_gemm_chunk(K) columns; each
 * chunk is a DMMA chain from zero and the chunk sums are added in chunk
 * order.  An output element therefore depends only on its row of op(A), on
 * B and on K -- not on M, the layout of A, the grid or the device -- which
 * makes row-sharded and single-GPU sketches / Schur blocks bitwise equal.
 * `workspace` (rs_workspace_bytes, zero-filled once) is required. */
int rs_dgemm(int M, int N, int K, double alpha, const double* A, long long lda, int a_colmajor,
             const int64_t* aidx, const double* B, long long ldb, const int64_t* bidx, double beta,
             const double* Cin, long long ldcin, const int64_t* cidx, double* C, long long ldc,
             void* workspace, void* stream);

/* Chunk length (columns of K, a multiple of 32) of the summation order above. */
int rs_gemm_chunk(long long K);

/* rs_dgemm with an explicit chunk length kc (<= 0: rs_gemm_chunk(K)) and mode:
 * RS_GEMM_FOLD adds the chunk sums to Cin in order, so a K range fed in
 * kc-aligned pieces (C = Cin + piece, piece by piece, kc of the full K)
 * gives the bits of the one-shot product; RS_GEMM_CHAIN continues the DMMA
 * chain from Cin (K <= kc), the same for the single-chunk case.  Used by the
 * host-input pre-sketch, which multiplies row chunks of A as they land. */
int rs_dgemm_ex(int M, int N, int K, int kc, int mode, double alpha, const double* A, long long lda, int a_colmajor,
                const int64_t* aidx, const double* B, long long ldb, const int64_t* bidx, double beta,
                const double* Cin, long long ldcin, const int64_t* cidx, double* C, long long ldc,
                void* workspace, void* stream);

/* Y (m x ell) = A (m x n) * Omega (n x ell): the sketch `a @ omega`
 * (sketching.py:128, 272).  a_colmajor selects the `a.T` view of a C-ordered
 * matrix (column ID / `rand_lupp_adaptive(A.T, ...)`). */
int rs_sketch_gemm(int m, int n, int ell, const double* A, long long lda, int a_colmajor,
                   const double* Omega, long long ldo, double* Y, long long ldy, void* workspace,
                   void* stream);

/* Panel LU with partial pivoting of the R x w (w <= 64) block S, in place,
 * rows kept in physical order: `_lupp_panel` (dense.py:185-207) over one
 * block.  perm_out[p] = physical row at position p afterwards (`sub.perm`);
 * *ncols_dev = eliminated columns (< w iff an exactly-zero pivot column was
 * met, dense.py:195-198).  Physical row r of S then holds, for its position
 * p < ncols, L[p, :p] and U[p, p:], and for p >= ncols the multipliers. */
int rs_panel_lupp(double* S, long long lds, int R, int w, int64_t* perm_out, int* ncols_dev,
                  void* workspace, void* stream);

/* Schur block of a fresh sketch block against the T-form state
 * (`_schur_of_block`, skeleton.py:317-323):
 *   S = Y[perm[k:]] - T * Y[perm[:k]],   *e2_dev = ||S||_F^2
 * with T = L2 L1^{-1} ((m-k) x k, ld ldt) the interpolation block of the
 * current rank-k state.  k = 0 gathers Y[perm].  The norm reduction is
 * deterministic (fixed order), `frobenius_norm` (dense.py:144-146). */
int rs_schur_block(int m, int k, int b, const double* Y, long long ldy, const int64_t* perm,
                   const double* T, long long ldt, double* S, long long lds, double* e2_dev,
                   void* workspace, void* stream);

/* Absorb a factored Schur block (the first nc of its columns) into the
 * T-form state (`_extend_state`, skeleton.py:326-351, expressed on
 * T = L2 L1^{-1}):
 *   W_hat = L_r L_1^{-1},  T_new = [T[Q_hat] - W_hat T[P_hat], W_hat]
 *   perm_new[:k] = perm[:k],  perm_new[k:] = perm[k:][sub_perm]
 * T_new is (m-k-nc) x (k+nc) with ld k+nc and must not alias T. */
int rs_absorb_block(int m, int k, int nc, const double* S, long long lds, const int64_t* sub_perm,
                    const double* T, long long ldt, double* T_new, const int64_t* perm,
                    int64_t* perm_new, void* workspace, void* stream);

/* C[i, :] = Cin[cidx[i], :] - A[i, :K] * B[bidx[0..K), :] with K <= 64: the
 * rank-b interpolation update inside rs_absorb_block (the trailing-update
 * role of dense.py:232 in T form).  Persistent DMMA kernel. */
int rs_rank_update(int M, int N, int K, const double* A, long long lda, const double* B, long long ldb,
                   const int64_t* bidx, const double* Cin, long long ldcin, const int64_t* cidx,
                   double* C, long long ldc, void* stream);

/* rs_absorb_block followed by the Schur block of the NEXT sketch block
 * (the two enqueued back to back, so the host reads one scalar per block):
 *   T_new, perm_new as rs_absorb_block;
 *   S_next = Y_next[perm_new[k+nc:]] - T_new * Y_next[perm_new[:k+nc]],
 *   *e2_dev = ||S_next||_F^2                       (skeleton.py:326-351, 317-323)
 * Y_next is m x 64 (ldy = 64); S_next is (m-k-nc) x 64 and may alias S. */
int rs_absorb_schur(int m, int k, int nc, const double* S, long long lds, const int64_t* sub_perm,
                    const double* T, long long ldt, double* T_new, const int64_t* perm, int64_t* perm_new,
                    const double* Y_next, long long ldy, double* S_next, double* e2_dev, void* workspace,
                    void* stream);

/* W (m x k, row-major) with W[perm[:k]] = I and W[perm[k:]] = T
 * (`_w_from_parts`, skeleton.py:176-182). */
int rs_scatter_interp(const double* T, long long ldt, const int64_t* perm, int m, int k, double* W,
                      long long ldw, void* stream);

/* dst[i, :] = src[idx[i], :]  (skeleton gathers `a[row_idx]`, skeleton.py:569,640);
 * idx[i] < 0 gives a zero row (owner-masked gathers of the sharded loop). */
int rs_gather_rows(const double* src, long long lds, const int64_t* idx, int nrows, int ncols,
                   double* dst, long long ldd, void* stream);

/* *out = ||X||_F^2, deterministic two-stage reduction. */
int rs_sumsq(const double* X, long long ldx, int R, int w, double* out, void* workspace,
             void* stream);

/* Inverse of an n x n (n <= 64) triangular matrix whose (i, j) element is
 * T[ridx(i)*rs + j*cs]; out n x n row-major.  Used for L_1^{-1}. */
int rs_trinv(const double* T, long long rs, long long cs, const int64_t* ridx, int n, int lower,
             int unit, double* out, long long ldo, void* stream);

/* perm_new[:k] = perm[:k], perm_new[k+i] = perm[k + sub[i]] (skeleton.py:345). */
int rs_perm_update(const int64_t* perm, int64_t* perm_new, int m, int k, const int64_t* sub,
                   void* stream);

/* dst (cols x rows, row-major) = src (rows x cols, row-major)^T. */
int rs_transpose(const double* src, long long lds, int rows, int cols, double* dst, long long ldd,
                 void* stream);

/* One round of one-sided Jacobi on Xt (q x p row-major = X^T): for every
 * pair (pairs[2r], pairs[2r+1]) rotate columns i, j of X (and rows of Vt) to
 * make them orthogonal; *max_off = max |x_i.x_j| / (|x_i||x_j|) seen (as
 * double bits, atomicMax).  Drives `pinv_apply` (dense.py:166-182). */
int rs_jacobi_round(double* Xt, long long ldx, int p, double* Vt, long long ldv, int q, const int* pairs,
                    int npairs, double tol, unsigned long long* max_off, void* stream);

/* After Jacobi convergence: sigma_i = |Xt[i,:]|, scale row i of Vt by
 * 1/sigma_i^2 (0 when sigma_i <= rcond * max sigma, gelsd's truncation). */
int rs_pinv_scale(const double* Xt, long long ldx, int p, double* Vt, long long ldv, int q, double rcond,
                  double* sigma, void* stream);

/* *out = max_j sum_i |A[i,j]| (matrix 1-norm, for the cond_1 flag, skeleton.py:592-603). */
int rs_norm1(const double* A, long long lda, int rows, int cols, double* out, void* stream);

/* All nrounds rounds of a Jacobi sweep (sched: nrounds x npairs pairs) in one
 * cooperative launch of npairs CTAs with a grid barrier between rounds;
 * barrier: one caller-owned device unsigned (reset by the call). */
int rs_jacobi_sweep(double* Xt, long long ldx, int p, double* Vt, long long ldv, int q, const int* sched,
                    int nrounds, int npairs, double tol, unsigned long long* max_off, unsigned* barrier,
                    void* stream);

/* W_hat rows of a factored panel: out[i, :nc] = S[ridx[i], :nc] L1^{-1}, L1 the
 * unit lower triangle of the pivot rows S[sub[a], b] (b < a < nc <= 64); one
 * row per thread (`_extend_state`, skeleton.py:326-351, on the T form). */
int rs_what(const double* S, long long lds, const int64_t* sub, int nc, const int64_t* ridx, int R, double* out,
            long long ldo, void* stream);

/* Dense n x ell form of the SRTT embedding (`sketching.py:134-157,207-216`):
 * Omega[perm[p], j] = scale * signs[q] * DCT-II_ortho(q, p), q = cols[j]. */
int rs_srtt_dense(int n, int ell, const int64_t* perm, const double* signs, const int64_t* cols, double scale,
                  double* out, long long ldo, void* stream);

/* Dense n x ell form of the sparse-sign embedding (`sketching.py:160-187,219-235`):
 * zero, then Omega[r, idx[r, z]] = signs[r, z] * scale (zeta entries per row). */
int rs_sparse_sign_dense(int n, int ell, int zeta, const int64_t* idx, const double* signs, double scale,
                         double* out, long long ldo, void* stream);

/* Device scratch for rs_srtt_apply to transform m rows of length n in one batch
 * (fewer bytes are accepted: the rows then go in batches). */
long long rs_srtt_workspace_bytes(long long m, int n);

/* y = a @ Omega for the SRTT embedding as a fast transform, the reference's
 * `SrttSketch.apply` (sketching.py:147-155): per row, the DCT-II (ortho) of
 * a[i, perm] through one length-n real FFT (Makhoul's reordering; cuFFT D2Z),
 * times signs[k], at the sampled frequencies k = cols[j], times scale.
 * O(m n log n); agrees with the reference to floating-point rounding (pocketfft's
 * order cannot be reproduced).  a: m x n row- or column-major; y: m x ell row-major;
 * ws: >= rs_srtt_workspace_bytes(1, n) bytes. */
int rs_srtt_apply(long long m, int n, int ell, const double* a, long long lda, int a_colmajor, const int64_t* perm,
                  const double* signs, const int64_t* cols, double scale, double* y, long long ldy, void* ws,
                  long long ws_bytes, void* stream);

/* Scratch bytes of rs_sparse_sign_apply's plan: two bitmaps (rows holding the
 * column, negative signs) per operator column per 32 operator rows. */
long long rs_sparse_sign_plan_bytes(int n, int ell);

/* y = a @ Omega for the sparse-sign embedding without forming Omega: the
 * reference's `(csr.T @ a.T).T` (`SparseSignSketch.apply`, sketching.py:176-185).
 * a: m x n, row-major (a[i*lda + j]) or column-major (a[j*lda + i]); y: m x ell
 * row-major.  Each y[i, c] is summed over the operator rows j holding c in
 * ascending j with a separate multiply and add, scipy's csc_matvecs order, so
 * the result is bitwise the reference's.  idx/signs: n x zeta (int64, +-1.0);
 * plan: rs_sparse_sign_plan_bytes of device scratch; bad: a caller-zeroed device
 * int, set to 1 (index outside [0, ell) or a sign other than +-1) or 2 (an index
 * repeated within a row) -- y is then not meaningful. */
int rs_sparse_sign_apply(long long m, int n, int ell, int zeta, const double* a, long long lda, int a_colmajor,
                         const int64_t* idx, const double* signs, double scale, double* y, long long ldy, void* plan,
                         int* bad, void* stream);

/* Cholesky G = R^T R of a small SPD matrix (n <= 1024) in place (upper R,
 * strict lower part zeroed); *status_dev = 0 or j + 1 for a non-positive
 * pivot j.  The Gram step of pinv_apply (dense.py:166-182). */
int rs_cholesky(double* G, long long ldg, int n, int* status_dev, void* stream);

/* x <- T^-1 x in place for a small triangular T (n <= 1024) stored by columns: T[i, j] at
 * cols[j * ldc + i] (a row-major T^T).  lower = forward substitution, else backward; unit =
 * implicit unit diagonal.  The solves of dgecon's dlacn2 iteration inside the 1-norm
 * condition estimate (`_condition_estimate_1norm`, skeleton.py:592-603), one launch each. */
int rs_trsv_cols(const double* cols, long long ldc, int n, int lower, int unit, double* x, void* stream);

/* dst[i, j] = src[r(i)*rs + c(j)*cs], r/c via optional index vectors: the
 * skeleton gathers a[I], a[:, J], a[ix_(I, J)] (skeleton.py:619,639-645). */
int rs_gather2d(const double* src, long long rs, long long cs, const int64_t* ridx, int nr,
                const int64_t* cidx, int nc, double* dst, long long ldd, void* stream);

/* n standard normals of numpy's Generator(Philox(key=[seed, stream_id]))
 * in generation order, each divided by `scale` (1.0 = none; sqrt(ell) for the
 * 'inv_sqrt_ell' spec): `make_gaussian` (sketching.py:191-204) on the device.
 * Workspace: rs_gaussian_workspace_bytes(n).  *status_dev = 1 (never seen)
 * if the parallel word->normal resolution hit an unsupported chain; the
 * caller then draws on the host. */
size_t rs_gaussian_workspace_bytes(long long n);
int rs_gaussian(unsigned long long seed, unsigned long long stream_id, long long n, double scale, double* out,
                void* rng_workspace, size_t ws_bytes, int* status_dev, void* stream);

/* p[i] = i. */
int rs_iota(int64_t* p, int n, void* stream);

/* ---- column-sharded adaptive loop (no reference counterpart:
 * the reference is single-process, this shards `rand_lupp_adaptive`,
 * skeleton.py:391-460, over ranks that own candidate rows [lo, hi)). ------ */

/* Per-block maps from the replicated position order perm (rank k):
 *   ytop_src[p] (p < k)   local row of skeleton p, or -1 if another rank owns it
 *   lrow[p]               local T row of position p >= k (or -1), for the next block
 *   loc[r], spos[r]       local candidate and Schur position of local row r
 *   *count                number of local remaining rows
 * With sub != NULL (just after an absorb of nc columns at rank k_old = k - nc,
 * lrow_old the previous lrow): src_row[r] / wsrc[r] = previous local T row /
 * Schur row of local row r, tp_src[j] = previous local T row of pivot j or -1.
 * Rows [*count, pad_to) get harmless entries (loc 0, spos -1, src_row 0,
 * wsrc 0) for launches sized by an upper bound of the row count. */
int rs_shard_maps(const int64_t* perm, int m, int k, long long lo, long long hi, const int64_t* lrow_old,
                  const int64_t* sub, int k_old, int nc, int64_t* lrow, int64_t* loc, int64_t* spos,
                  int64_t* src_row, int64_t* wsrc, int64_t* tp_src, int64_t* ytop_src, int* count, int pad_to,
                  void* stream);

/* *out_max = the largest remaining-candidate count over the ranks: ranks own
 * the contiguous candidate ranges [bounds[g], bounds[g+1]), g < world <= 64;
 * the remaining candidates are perm[k:].  Sizes the per-block all-gather of
 * the Schur rows identically on every rank (no collective). */
int rs_shard_max_count(const int64_t* perm, int m, int k, const int64_t* bounds, int world, int* out_max,
                       void* stream);

/* dst[idx[i], :] = src[i, :] for idx[i] >= 0. */
int rs_scatter_rows(const double* src, long long lds, const int64_t* idx, int nrows, int ncols, double* dst,
                    long long ldd, void* stream);

/* Local rows [lo, hi) of W (m x k): zero, W[perm[p]-lo, p] = 1 for owned
 * skeletons, W[loc[r]] = T[r] for the r local remaining rows. */
int rs_scatter_interp_local(const double* T, long long ldt, const int64_t* perm, int k, const int64_t* loc, int r,
                            long long lo, long long hi, double* W, long long ldw, void* stream);

/* ---- Ozaki-scheme sketch GEMM on the int8 tensor cores (tcgen05 kind::i8,
 * TMEM accumulators; ozaki.cu).  Y = A Omega with A and Omega cut into
 * signed 7-bit digit planes per (row, K-chunk) / (column, K-chunk); the plane
 * products are exact int32 sums, combined in fp64 in a fixed order and the
 * chunk sums folded in chunk order: the same determinism contract as
 * rs_dgemm.  Replaces the OpenBLAS dgemm of `GaussianSketch.apply`
 * (sketching.py:122-128) on the adaptive loop's sketch (skeleton.py:293-295). */

/* K-chunk length (multiple of 128, <= 16384) of the Ozaki sketch for K. */
int rs_oz_chunk(long long K);

/* Bytes of the digit planes of a rows x K operand with S planes, in tiles of
 * tile_rows (128 for A, 64 for Omega^T). */
size_t rs_oz_digits_bytes(int rows, long long K, int S, int tile_rows);

/* Digit planes and exponents of X (rows x K; fp32 if fp32 else fp64; X[i, k]
 * at X[i*ld + k] or, colmajor, X[k*ld + i]) for k in [k0, k1), k0 and k1
 * multiples of kc or k1 = K.  expo: rows x ceil(K / kc) int32.  For Omega
 * (K x N row-major) pass colmajor = 1, rows = N, ld = its row stride.
 * *nonfinite (may be NULL) is or-ed with 1 if X holds a NaN or inf.
 * workspace: rs_workspace_bytes (scratch for the row-chunk maxima). */
int rs_oz_slice(const void* X, int fp32, long long ld, int colmajor, int rows, int K, int k0, int k1, int kc, int S,
                int tile_rows, int8_t* digits, int* expo, int* nonfinite, void* workspace, void* stream);

/* C (M x N row-major) = alpha * A Omega + beta * Cin (mode RS_GEMM_PLAIN) or
 * Cin + A Omega with the chunk sums folded onto Cin (RS_GEMM_FOLD), from the
 * sliced operands (SA, SB <= 8 planes).  workspace: rs_workspace_bytes. */
int rs_oz_gemm(int M, int N, int K, int kc, int mode, double alpha, const int8_t* a_digits, const int* a_expo,
               int SA, const int8_t* b_digits, const int* b_expo, int SB, double beta, const double* Cin,
               long long ldcin, double* C, long long ldc, void* workspace, void* stream);

/* ---- input generators (input generation, not the
 * skeleton path).  Each is restated in numpy by the oracle with the same
 * rounding, so the device matrix equals the host one bit for bit. ------- */

/* out[i] = numpy Generator(Philox(key=[seed, stream_id])).random(n)[i]. */
int rs_uniform(unsigned long long seed, unsigned long long stream_id, long long n, double* out, void* stream);

/* x (n x n, row-major, n a power of two) = rowscale * (c H), H the
 * Walsh-Hadamard matrix: the first factor of the randomized-Hadamard
 * fast-decay generator (cfg5).  rowscale may be NULL. */
int rs_hadamard_init(double* x, long long ld, int n, double c, const double* rowscale, void* stream);

/* x <- rowscale * (c * H x): Walsh-Hadamard transform of every column of the
 * n x n row-major x (n a power of two, <= 2^17), butterflies in numpy's
 * level order, then the scale c and the optional row scale. */
int rs_fwht_rows(double* x, long long ld, int n, double c, const double* rowscale, void* stream);

/* Kahan's matrix `gen_kahan` (zoo.py:78-88): a[i, j] = rowpow[i] * k[i, j],
 * k = 1 on the diagonal, negphi above it, 0 below; rowpow[i] = zeta^i. */
int rs_kahan(double* a, long long ld, int n, const double* rowpow, double negphi, void* stream);

/* `gen_chan` (zoo.py:91-104): 1 on the diagonal, -1 below, last column 1. */
int rs_chan(double* a, long long ld, int n, void* stream);

/* out = x + beta * y elementwise (n values), to out64 or rounded to out32
 * (exactly one non-NULL): the low-rank-plus-noise recipe of cfg3. */
int rs_axpy_cast(const double* x, const double* y, double beta, long long n, double* out64, float* out32,
                 void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RSKEL_H */
