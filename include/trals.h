/* C-ABI of the B200-native TR-ALS hot path (libtrals.so).
 *
 * Conventions (all entry points):
 *   - plain extern "C"; no torch or C++ types cross this boundary;
 *   - every pointer argument named d_* is a caller-owned DEVICE buffer,
 *     h_* is host memory;
 *   - every call takes the CUDA stream (cudaStream_t passed as void*) and is
 *     asynchronous: nothing synchronises the device or allocates memory
 *     inside a call (workspace is caller-provided, sized by the matching
 *     *_ws_elems query);
 *   - every call returns an int status (TRALS_OK or an error code, see
 *     trals_strerror); numerical failures detected on the device are reported
 *     through a caller-provided device int array (d_info), never by a sync;
 *   - results are deterministic (fixed reduction orders), so replicas on
 *     several GPUs stay bitwise identical.
 *
 * Cores are ring cores G_n of shape (R_n, I_n, R_{n+1}) (reference ring.py:1-24).
 * Three device layouts are used (TRALS_LAYOUT_*):
 *   C     : [r_n][i][r_{n+1}]   the reference's C-order array
 *   SLICE : [i][r_n][r_{n+1}]   lateral slices G_n(i) contiguous
 *   ZT    : [i][r_{n+1}][r_n]   = classical 2-unfolding Z[i, r_n + R_n r_{n+1}]
 *                               (tensor_ops.py:100-108), the solve's output
 *   TT    : [r_{n+1}][r_n][i]   (transposed slices; operand of the fused reconstruct)
 *
 * Each entry point cites the reference code it replaces.
 */
#ifndef TRALS_H
#define TRALS_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TRALS_OK = 0,
  TRALS_ERR_ARG = 1,         /* bad shape / stride / pointer */
  TRALS_ERR_CUDA = 2,        /* kernel launch failed */
  TRALS_ERR_WORKSPACE = 3,   /* caller workspace too small */
  TRALS_ERR_UNSUPPORTED = 4  /* size outside the kernels' envelope */
};

enum { TRALS_LAYOUT_C = 0, TRALS_LAYOUT_SLICE = 1, TRALS_LAYOUT_ZT = 2, TRALS_LAYOUT_TT = 3 };

/* d_info slots written by the solve kernels (int32 each, 0 = no event) */
enum {
  TRALS_INFO_CHOL = 0,       /* 1-based index of first non-positive pivot */
  TRALS_INFO_ASYM = 1,       /* 1 if |S - S^T| > 1e-8 max|S| (linalg.py:70-72) */
  TRALS_INFO_DEGEN = 2,      /* 1-based index of diag <= 1e-13 max|R| (linalg.py:96-99) */
  TRALS_INFO_FALLBACKS = 3,  /* number of fallback solves taken (AlsReport.fallback_count) */
  TRALS_INFO_ILLCOND = 4,    /* QR variants: merged R0's smallest diagonal <= sqrt(m eps) max|R0| */
  TRALS_INFO_REFINE = 5,     /* m <= 112 factor with max|U| > 1e4 min diag(U): refine the solve */
  TRALS_INFO_SLOTS = 6
};

const char* trals_strerror(int code);
int trals_version(void);
/* Number of kernels this library has launched in the process (instrumentation). */
long long trals_launch_count(void);

/* Generic strided fp64 contraction on the DMMA pipe (the engine behind every
 * entry point below):  C[p][m][n] (+)= sum_k A(p,m,k) * B[k*ldb + n],
 * A(p,m,k) = d_A[p*sAp + m*sAm + k*sAk] with sAk == 1 or sAm == 1,
 * C address = p*cmap[0] + (m/cmap[1])*cmap[2] + (m%cmap[1])*cmap[3]
 *                       + (n/cmap[4])*cmap[5] + (n%cmap[4])*cmap[6].
 * Replaces the numpy matmul / tensordot / einsum calls on the path
 * (solvers.py:379, ring.py:129,188, tensor_ops.py:161,225). */
int64_t trals_gemm_ws_elems(int64_t P, int64_t M, int64_t K, int64_t N);
int trals_gemm_f64(const double* d_A, int64_t sAp, int64_t sAm, int64_t sAk,
                   int64_t P, int64_t M, int64_t K, int64_t N,
                   const double* d_B, int64_t ldb, double* d_C, const int64_t* h_cmap, int beta,
                   double* d_ws, int64_t ws_elems, void* stream);

/* Core layout moves (tensor_ops.py:52-119 classical fold/unfold of a core). */
int trals_core_relayout_f64(const double* d_src, int src_layout, int Ra, int64_t I, int Rb,
                            double* d_dst, int dst_layout, void* stream);

/* Half chain H[i_u..i_v][r_u][r_{v+1}] = G_u(i_u) ... G_v(i_v) of a contiguous
 * block of cores (ring.py:110-152 subchain_merge/skip restricted to a block).
 * d_cores_c[j] = core u+j in layout C, d_first_slice = core u in layout SLICE.
 * d_tmp must hold the largest intermediate chain (trals_half_chain_tmp_elems).
 * transposed != 0 writes [r_{v+1}][r_u][i_u..i_v] instead (the K x post operand
 * of trals_residual_f64). */
int64_t trals_half_chain_tmp_elems(int nblk, const int64_t* dims, const int32_t* ranks);
int trals_half_chain_f64(int nblk, const int64_t* dims, const int32_t* ranks,
                         const double* d_first_slice, const double* const* h_cores_c,
                         double* d_out, double* d_tmp, double* d_ws, int64_t ws_elems, int transposed,
                         void* stream);

/* Environment of the prefix/suffix segment complementary to a half chain
 * (the X_[n] * G^{!=n}_[2] product of solvers.py:379 restricted to the
 * modes of the half chain).  X is C-contiguous and viewed as [pre][post].
 *  side = 0: half chain covers the suffix (post);  Env[r_0][pre][r_y]
 *  side = 1: half chain covers the prefix (pre);   Env[r_x][post][r_0]
 * r_lo/r_hi are the chain's outer bonds (left, right).  leaf != 0: the
 * segment is a single mode and the result is written as M_n directly. */
int trals_env_f64(const double* d_X, int64_t pre, int64_t post, int side,
                  const double* d_H, int r_lo, int r_hi, double* d_env, int leaf,
                  double* d_ws, int64_t ws_elems, void* stream);

/* ---- fp32 variant (AlsConfig.dtype = "float32"; BASELINE config 4) ----
 * X is stored in fp32 and only the X-streaming environment product changes;
 * cores, Grams, solves and errors stay fp64. */
/* fp32 variant, product path: digit-sliced GEMM on the int8 tensor cores
 * (tcgen05 kind::i8, exact int32 accumulation; tc_int8_gemm.cuh).  Each
 * K-major row r of X is held as ex[r] and four int8 digit planes with
 *   x = 2^ex[r] * sum_{s<4} d_s 2^(-7(s+1)),  |x| < 2^ex[r],
 * stored as the MMA's shared-memory image: [128-row tile][64-k block][plane]
 * [128 x 64 B], each plane in the UMMA K-major SWIZZLE_64B pattern, zero
 * padded (trals_oz_digits_bytes bytes for rows x K).  trals_oz_split_f32
 * slices x [rows][cols] row-major, or its transpose when transpose = 1
 * (out rows = cols, K = rows); ws holds out_rows doubles.
 * trals_env_oz: trals_env_f64 with X given sliced, K-major for `side` (side 0:
 * rows = pre, K = post; side 1: rows = post, K = pre); the half chain is
 * sliced per call. */
int64_t trals_oz_digits_bytes(int64_t rows, int64_t k);
int64_t trals_oz_split_ws_elems(int64_t rows, int64_t cols, int transpose);
int trals_oz_split_f32(const float* d_x, int64_t rows, int64_t cols, int transpose, int8_t* d_digits,
                       int32_t* d_exps, double* d_ws, int64_t ws_elems, void* stream);
int64_t trals_env_oz_ws_elems(int64_t pre, int64_t post, int side, int r_lo, int r_hi);
int trals_env_oz(const int8_t* d_xdigits, const int32_t* d_xexps, int64_t pre, int64_t post, int side,
                 const double* d_H, int r_lo, int r_hi, double* d_env, int leaf, double* d_ws, int64_t ws_elems,
                 void* stream);

/* fp64 environment product on the int8 tensor cores (AlsConfig.fp64_gemm =
 * "ozaki", the default at c3-c5 under the guard of trals_oz_range_f64): trals_env_f64 with X given as
 * seven balanced digit planes per K-major row,
 *   x = 2^ex[r] (d_0 + (d_1 + (d_2 + ...) / 254) / 254) / 127,  |d_s| <= 127  (7 digits),
 * (remainder <= 2^-55.9 2^ex[r], |x| < 2^ex[r]; same tiled layout as above with 7 planes,
 * trals_oz64_digits_bytes bytes), the half chain sliced the same way per call,
 * and the 28 digit-pair products of levels s + t <= 6 accumulated exactly in
 * int32 and combined in fp64.  Accuracy against an extended-precision product
 * is that of the fp64 DMMA product (tests/test_gpu_ops.py).  Replaces the same
 * reference call as trals_env_f64 (solvers.py:379). */
int64_t trals_oz64_digits_bytes(int64_t rows, int64_t k);
int trals_oz64_split_f64(const double* d_x, int64_t rows, int64_t cols, int transpose, int8_t* d_digits,
                         int32_t* d_exps, double* d_ws, int64_t ws_elems, void* stream);
int64_t trals_env_oz64_ws_elems(int64_t pre, int64_t post, int side, int r_lo, int r_hi);
int trals_env_oz64(const int8_t* d_xdigits, const int32_t* d_xexps, int64_t pre, int64_t post, int side,
                   const double* d_H, int r_lo, int r_hi, double* d_env, int leaf, double* d_ws, int64_t ws_elems,
                   void* stream);
/* fp64 environment product on the int8 tensor cores by the Chinese remainder theorem
 * (AlsConfig.fp64_gemm = "crt"; the default for long contractions, K >= 4096 and R^2 <= 512,
 * i.e. BASELINE c5): trals_env_f64 with X given as residue planes.  Every K-major row r of X is
 * scaled by 2^sx[r] (from its 2-norm) and rounded to integers x' = rint(2^sx x) with
 * ||x'||_2 <= 2^trals_crt_row_bits(0) (58; 62 with 16 moduli); plane i holds the residues
 * x' mod p_i in [0, p_i) (unsigned bytes) for the trals_crt_moduli() (15; TRALS_CRT_MODULI=12..16)
 * largest pairwise coprime moduli p_i <= 256, each plane tiled
 * [128-row tile][64-k block][128 x 64 B] in the UMMA K-major SWIZZLE_64B pattern
 * (trals_crt_planes_bytes bytes in total).  The half chain is sliced the same way per call;
 * one exact int8 GEMM per modulus, reduced mod p_i in its epilogue, and an exact 128-bit CRT
 * reconstruction: the result is the correctly rounded exact product of the rounded operands.
 * Accuracy contract: as trals_env_oz64 (below), with each row rounded at 2^-58 of its 2-norm
 * instead of 2^-56.9 of its maximum (measured at K = 25600 on Gaussian operands: 3.8e-16 relative
 * against an extended-precision product, fp64 DMMA 9.2e-16).  Replaces the same reference call as trals_env_f64
 * (solvers.py:379).  trals_crt_supported: 1 when the shape (rows x k) . (k x n) is covered. */
int trals_crt_supported(int64_t rows, int64_t k, int64_t n);
int trals_crt_moduli(void);
int trals_crt_row_bits(int operand); /* log2 of the 2-norm bound of the scaled rows of X (0) / the half chain (1) */
int64_t trals_crt_planes_bytes(int64_t rows, int64_t k);
int64_t trals_crt_split_ws_elems(int64_t rows, int64_t cols, int transpose);
int trals_crt_split_f64(const double* d_x, int64_t rows, int64_t cols, int transpose, int8_t* d_planes,
                        int32_t* d_exps, double* d_ws, int64_t ws_elems, void* stream);
int64_t trals_env_crt_ws_elems(int64_t pre, int64_t post, int side, int r_lo, int r_hi);
int trals_env_crt(const int8_t* d_xplanes, const int32_t* d_xexps, int64_t pre, int64_t post, int side,
                  const double* d_H, int r_lo, int r_hi, double* d_env, int leaf, double* d_ws, int64_t ws_elems,
                  void* stream);
/* The same product stage by stage on the same workspace (stages: bit mask, run in this order):
 * 1 = scales + residue planes of the half chain, 2 = the modular int8 GEMMs, 4 = CRT reconstruction
 * into d_env.  trals_env_crt == stages 7.  Lets the caller time or schedule the stages apart. */
int trals_env_crt_stage(const int8_t* d_xplanes, const int32_t* d_xexps, int64_t pre, int64_t post, int side,
                        const double* d_H, int r_lo, int r_hi, double* d_env, int leaf, double* d_ws,
                        int64_t ws_elems, int stages, void* stream);
/* Absorb the rightmost / leftmost core of an environment segment.
 * Env layout [r_a][i_a .. i_b][r_{b+1}].
 *   right: Out[r_a][pre][r_b]       = sum E[r_a][pre][i_b][r_{b+1}] G_b[r_b,i_b,r_{b+1}]
 *          (d_core in layout ZT)
 *   left : Out[r_{a+1}][rest][r_{b+1}] = sum E[r_a][i_a][rest][r_{b+1}] G_a[r_a,i_a,r_{a+1}]
 *          (d_core in layout C)
 * leaf != 0 writes the single-mode result directly as M_n (I_n x R_n R_{n+1},
 * column r_n + R_n r_{n+1}), the layout of solvers.py:379's product. */
int trals_absorb_right_f64(const double* d_env, int Ra, int64_t pre, int64_t Ib, int Rb, int Rb1,
                           const double* d_core_zt, double* d_out, int leaf,
                           double* d_ws, int64_t ws_elems, void* stream);
int trals_absorb_left_f64(const double* d_env, int Ra, int64_t Ia, int64_t rest, int Ra1, int Rb1,
                          const double* d_core_c, double* d_out, int leaf,
                          double* d_ws, int64_t ws_elems, void* stream);

/* Bond Gram of one core as a transfer matrix
 * E[(a,c)][(b,d)] = sum_i G[a,i,b] G[c,i,d]  (ring.py:173-188, Alg. 2 line 2). */
int trals_core_gram_f64(const double* d_core_slice, int Ra, int64_t I, int Rb, double* d_E,
                        double* d_ws, int64_t ws_elems, void* stream);

/* Householder QR of a core's classical 2-unfolding (mode2_qr, ring.py:236-249;
 * qr_economy sign convention, linalg.py:36-52): d_Gzt = the core in layout ZT
 * viewed as an I x RR row-major matrix; writes R (k x RR, k = min(I, RR),
 * nonnegative diagonal) -- the R-tensor of the QR / QRNE variants.  One CTA
 * when the matrix fits shared memory, TSQR for tall, left-block + parallel Q^T
 * application for wide matrices.  Returns TRALS_ERR_UNSUPPORTED when
 * trals_core_qr_ws_elems is negative. */
int64_t trals_core_qr_ws_elems(int I, int RR);
int trals_core_qr_f64(const double* d_Gzt, int I, int RR, double* d_R, double* d_ws, int64_t ws_elems, void* stream);

/* Coefficient Gram S_n = (G^{!=n}_[2])^T G^{!=n}_[2] from the chain of transfer
 * matrices (ring.py:191-214 gram_chain(_order), Prop. 3).  h_E[j] = transfer
 * matrix of core j; d_tmp holds two R^2 x R^2 buffers. */
int trals_gram_chain_f64(int N, int n, const int32_t* ranks, const double* const* h_E,
                         double* d_S, double* d_tmp, double* d_ws, int64_t ws_elems, void* stream);
/* The same chain in two parts (R = the largest rank in d_tmp's size): part 1 forms every product but
 * the last and leaves the prefix in d_tmp, part 2 multiplies it by the last factor -- the transfer
 * matrix of core n-1, the core solved just before block n -- into d_S; part 0 = both. */
int trals_gram_chain_part_f64(int N, int n, const int32_t* ranks, const double* const* h_E,
                              double* d_S, double* d_tmp, double* d_ws, int64_t ws_elems, int part, void* stream);

/* spd_solve (linalg.py:55-81), factor step: symmetry check (1e-8 relative,
 * -> d_info[TRALS_INFO_ASYM]), symmetrise, upper Cholesky S = U^T U
 * (-> d_U, row-major).  Failing pivot (1-based) -> d_info[TRALS_INFO_CHOL];
 * with check_degen the 1e-13 floor of tri_solve_right (linalg.py:96-99) is
 * evaluated on diag(U) -> d_info[TRALS_INFO_DEGEN].
 *   m <= 112: one CTA, [S | I] resident in shared memory, Gauss-Jordan
 *             elimination yields U and V = U^{-T} together; d_F = U^{-1},
 *             d_aux = V;
 *   m  > 112: blocked (64-row panels: diagonal block + its inverse in one
 *             CTA, panel and trailing updates as DMMA GEMMs); d_F = U^T,
 *             d_aux = diagonal-block inverses + GEMM workspace.
 * d_aux holds trals_cholesky_aux_elems(m) doubles. */
int64_t trals_cholesky_aux_elems(int m);
int trals_cholesky_f64(const double* d_S, int m, double* d_U, double* d_F, double* d_aux, int check_degen,
                       int* d_info, void* stream);

/* spd_solve, solve step (scipy cho_solve, linalg.py:76): Z with Z S = M for the
 * factor written by trals_cholesky_f64.  m <= 112: Z = (M U^{-1}) U^{-T}, two
 * DMMA GEMMs; m > 112: blocked forward/backward substitution (Y U = M,
 * Z U^T = Y) with the diagonal-block inverses.  d_ws holds
 * trals_chol_solve_ws_elems(rows, m) doubles. */
int64_t trals_chol_solve_ws_elems(int64_t rows, int m);
int trals_chol_solve_f64(const double* d_U, const double* d_F, const double* d_aux, int m, const double* d_M,
                         int64_t rows, double* d_Z, double* d_ws, int64_t ws_elems, void* stream);

/* One step of iterative refinement after trals_chol_solve_f64 on the m <= 112 path (explicit-inverse
 * operands F = U^{-1}, aux = U^{-T}): R = M - Z S, Z += (R F) aux.  The explicit inverses are accurate
 * only to ~eps cond(S) where S is ill-conditioned (BASELINE c4: cond(S_n) ~ 5e11); one step brings Z to
 * the accuracy of scipy's cho_solve (linalg.py:76).  Gated on d_info[TRALS_INFO_REFINE], which the
 * factorisation (trals_cholesky_f64 / trals_tri_prepare_f64, m <= 112) sets when max|U| > 1e4 min
 * diag(U); otherwise the kernel returns at once (it stays in the sweep graph). */
int trals_solve_refine_f64(const double* d_F, const double* d_aux, const double* d_S, int m, const double* d_M,
                           int64_t rows, double* d_Z, int* d_info, void* stream);

/* Numerical fallback of spd_solve / solve_triangular_block, run right after
 * trals_chol_solve_f64 on the same stream; it returns immediately unless its
 * trigger flag is set.  mode 0 (NE/QRNE, linalg.py:77-81): on a Cholesky
 * failure, Z = least-squares solution of Z sym = M with the rank cut at
 * rcond * sigma_max (scipy lstsq gelsy with cond = eps: pass rcond = 2.22e-16).
 * mode 1 (QR, solvers.py:262-273 + linalg.py:104-112): on a failed or
 * degenerate R0 = chol(S), the min-norm solve with singular values of R0 cut at
 * rcond * sigma_max(R0) (AlsConfig.svd_rcond).  mode 2: the reference's
 * non-square R0 (prod_{j!=n} k_j < R^2, solvers.py:264-266): always that min-norm
 * solve, not counted as a fallback.  Cuts never go below the Jacobi noise floor
 * m * eps * sigma_max(S).  All via a one-CTA one-sided
 * Jacobi SVD of S.  When it fires it overwrites Z, clears the trigger flag and
 * increments d_info[TRALS_INFO_FALLBACKS]. */
int64_t trals_spd_fallback_ws_elems(int64_t rows, int m);
int trals_spd_fallback_f64(const double* d_S, int m, const double* d_M, int64_t rows, double* d_Z, int* d_info,
                           int mode, double rcond, double* d_ws, int64_t ws_elems, void* stream);

/* Accuracy contract of the digit-sliced fp64 products (trals_env_oz64, trals_residual_oz64):
 * every K-major row a of the sliced operand is held to 2^-56.9 of its own maximum (7 balanced
 * radix-254 digits), so an output's error is <= 2^-56.9 (max|a| sum|h| + max|h| sum|a|) plus
 * the dropped pair level (the same order) -- relative to each row's maximum, where a dgemm's
 * bound is eps sum|a||h|.  The two agree within a small factor when no row has a wide dynamic
 * range; trals_oz_range_f64 measures it for X: d_out[0] = max over the K-major rows (rows of X
 * for transpose = 0, columns for transpose = 1) of rho = max|x| K / sum|x|.  The solvers'
 * fp64_gemm = "auto" takes the int8 engine only when rho <= 2^12 for every X-streaming phase
 * (Gaussian data: rho ~ 5), i.e. when the product's error stays within 2^-44.9 mean|a| sum|h|;
 * otherwise they use the DMMA pipe (trals_env_f64). */
int64_t trals_oz_range_ws_elems(int64_t rows, int64_t cols, int transpose);
int trals_oz_range_f64(const double* d_x, int64_t rows, int64_t cols, int transpose, double* d_out, double* d_ws,
                       int64_t ws_elems, void* stream);

/* R0 of the QR-stabilised variants (tr_als_qr, solvers.py:422-424 `q0, r0 =
 * qr_economy(cyclic_unfold(V, 1))`; Alg. 1 tr_als, solvers.py:337-339, the same with the cores):
 * the nonnegative-diagonal factor with R0^T R0 = V_[2]^T V_[2] = S_n, computed without V and without
 * squaring cond(V) in fp64: the transfer matrices of the R-tensors (of the cores for Alg. 1), their
 * Gram chain (ring.py:191-214) and the Cholesky factorisation all run in double-double arithmetic
 * (~2^-104 relative per operation), so R0 is as accurate as the reference's Householder R0 for
 * cond(V) up to ~2^51 before it is rounded to fp64.  A pivot <= 0 (semidefinite S, rank-deficient V)
 * leaves a zero row, which the 1e-13 floor of trals_tri_prepare_f64 reports as the reference's
 * Householder R0 of such a V does (linalg.py:96-99).
 * trals_dd_transfer_f64: E = sum_i R(i) (x) R(i) of one tensor (layout C, (Ra, k, Rb)) as hi / lo
 * planes, in the layout of trals_core_gram_f64.
 * trals_dd_r0_f64: h_Ehi / h_Elo[j] = those of tensor j; writes R0 (m x m row-major, m = R_n
 * R_{n+1}, columns r_n + R_n r_{n+1}) and, if d_S is not null, the fp64 rounding of S_n. */
int trals_dd_transfer_f64(const double* d_R, int Ra, int k, int Rb, double* d_Ehi, double* d_Elo, void* stream);
int64_t trals_dd_r0_ws_elems(int N, const int32_t* ranks);
int trals_dd_r0_f64(int N, int n, const int32_t* ranks, const double* const* h_Ehi, const double* const* h_Elo,
                    double* d_S, double* d_R0, double* d_ws, int64_t ws_elems, void* stream);

/* solve_triangular_block's factor step (solvers.py:262-273 with linalg.py:84-101) for a given
 * square R0 (d_U, m x m row-major, upper): the operands of trals_chol_solve_f64 (which then
 * computes Z = M R0^{-1} R0^{-T}, i.e. W = M R0^{-1}, Z R0^T = W): m <= 112: d_F = R0^{-1},
 * d_aux = R0^{-T}; m > 112: d_F = R0^T, d_aux = the inverses of the 64 x 64 diagonal blocks
 * (trals_cholesky_aux_elems(m) doubles); the strict lower triangle of d_U is zeroed.  With
 * check_degen the 1e-13 degeneracy floor of linalg.py:96-99 -> d_info[TRALS_INFO_DEGEN]. */
int trals_tri_prepare_f64(double* d_U, int m, double* d_F, double* d_aux, int check_degen, int* d_info,
                          void* stream);

/* The min-norm fallback of the QR variants taken on R0 itself (linalg.py:104-112 pinv with
 * rcond = AlsConfig.svd_rcond, solvers.py:262-273): one-sided Jacobi SVD of the Lr x m factor
 * (R0 V = U Sigma), Z = M V Sigma^{-2} V^T over the singular values above rcond sigma_max
 * (= W pinv(R0)^T for W = M R0^{-1}).  Because the right-hand side is M = W R0 rather than W, the
 * cut is max(rcond, sqrt(m eps)) sigma_max: a component with a smaller singular value is divided by
 * sigma^2 and would only amplify M's rounding.  mode 1: fires on d_info[TRALS_INFO_DEGEN] (counted as
 * a fallback, flag cleared -- the reference's event) or on d_info[TRALS_INFO_ILLCOND] alone (an
 * R0 with min|r_ii| <= sqrt(m eps) max|R0| but above the 1e-13 floor, where the two triangular
 * solves of M would square its condition number: the same min-norm solve, not counted); mode 3
 * (rank_deficient_fallback off): only the ILLCOND case, so a degenerate R0 still raises;
 * mode 2: non-square R0 (Lr < m, solvers.py:264-266), always, uncounted.
 * Workspace: trals_spd_fallback_ws_elems(rows, m). */
int trals_tri_fallback_f64(const double* d_R0, int Lr, int m, const double* d_M, int64_t rows, double* d_Z,
                           int* d_info, int mode, double rcond, double* d_ws, int64_t ws_elems, void* stream);

/* Axis reversal (io.py:10-11, read_tensor's reshape(order="F").copy()): src is
 * first-index-fastest over dims[0..N-1], dst the same tensor last-index-fastest
 * (C order).  N <= 16; src and dst must not alias.  Used to land a .dten payload
 * uploaded verbatim into the engine's C-order X on the device. */
int trals_reverse_axes_f64(const double* d_src, int N, const int64_t* h_dims, double* d_dst, void* stream);

/* Sum of squares of n doubles into d_out[0] (tensor_ops.py:237-239 norm) and the
 * number of non-finite entries into d_out[1] (validation.py:53-54). */
int64_t trals_sumsq_ws_elems(void);
int trals_sumsq_f64(const double* d_x, int64_t n, double* d_out, double* d_ws, void* stream);
/* Same for fp32 input (the fp32 variant's X), accumulated in fp64. */
int trals_sumsq_f32(const float* d_x, int64_t n, double* d_out, double* d_ws, void* stream);

/* Relative error from sweep intermediates (solvers.py:177-212):
 * d_out[0] = sqrt(max(0, |X|^2 - 2<M,Z> + <S, Z^T Z>)) / |X|,
 * d_out[1] = <M,Z>, d_out[2] = <S, Z^T Z>.  d_xnorm2 = |X|^2 on the device. */
int64_t trals_error_ws_elems(int64_t rows, int m);
int trals_error_terms_f64(const double* d_M, const double* d_Z, const double* d_S, int64_t rows, int m,
                          const double* d_xnorm2, double* d_out, double* d_ws, int64_t ws_elems,
                          void* stream);

/* Stateless convenience: M_n = X_[n] G^{!=n}_[2] for one mode, the exact
 * drop-in for solvers.py:375+379 (`cyclic_unfold(x, n) @ a`).  Cores in
 * layout C (h_cores_c) and SLICE (h_cores_s); never materialises the
 * (prod_{j!=n} I_j) x R_n R_{n+1} subchain. */
int64_t trals_mttsp_ws_elems(int N, const int64_t* dims, const int32_t* ranks, int n);
int trals_mttsp_f64(const double* d_X, int N, const int64_t* dims, const int32_t* ranks, int n,
                    const double* const* h_cores_c, const double* const* h_cores_s,
                    const double* const* h_cores_zt, double* d_M, double* d_ws, int64_t ws_elems,
                    void* stream);

/* Exact relative error (solvers.py:164-174, exact_relative_error):
 * ||X - TR(G)||_F / ||X||_F with the dense reconstruction (ring.py:155-170)
 * fused into a DMMA GEMM X_hat = HL * HRt whose epilogue accumulates
 * (X - X_hat)^2 tile by tile -- X_hat is never stored.  X viewed as [pre][post];
 * HL = half chain of the prefix cores [pre][r_0][r_h]; HRt = half chain of the
 * suffix cores written transposed, [r_0][r_h][post]; K = R_0 R_h.
 * d_out[1] = sum of squared residuals, d_out[0] = sqrt(d_out[1] / d_xnorm2[0]). */
int64_t trals_residual_ws_elems(int64_t pre, int64_t post);
int trals_residual_f64(const double* d_X, int64_t pre, int64_t post, const double* d_HL, const double* d_HRt,
                       int64_t K, const double* d_xnorm2, double* d_out, double* d_ws, int64_t ws_elems,
                       void* stream);

/* The same exact error with the product on the int8 tensor cores: HL (rows) and HRt
 * (columns) sliced into 7 balanced digits each, the 28 digit-pair products of levels
 * <= 6 accumulated exactly and combined in fp64 (the scheme of trals_env_oz64), the
 * residual (X - HL HRt)^2 summed in the GEMM epilogue in a fixed order (one partial per
 * CTA, then one fixed-order sum): X_hat is never stored.  K <= 18944. */
int64_t trals_residual_oz64_ws_elems(int64_t pre, int64_t post, int64_t K);
int trals_residual_oz64(const double* d_X, int64_t pre, int64_t post, const double* d_HL, const double* d_HRt,
                        int64_t K, const double* d_xnorm2, double* d_out, double* d_ws, int64_t ws_elems,
                        void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TRALS_H */
