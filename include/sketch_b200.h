/*
 * sketch_b200.h -- C ABI of the B200-native CountSketch (sparse embedding)
 * hot path.  Plain pointers and sizes only; every device pointer is caller-
 * owned (e.g. a torch CUDA tensor's data_ptr), every call is stream-ordered on
 * the cudaStream_t passed as `stream` (NULL = legacy default stream), and no
 * call allocates device memory behind the caller's back (workspace queries
 * give the scratch sizes).  Errors are returned as skt_status; a human-readable
 * message for the calling thread is available from skt_last_error().
 *
 * The reference (/root/reference/pkg/src/sketchnla, pure Python on numpy/scipy)
 * has no FFI of its own; its drop-in boundary is the duck-typed SketchOperator
 * protocol (sketch.py:97-119).  Each entry point below replaces one piece of
 * SparseEmbedding (sketch.py:138-173) or of a caller of it, cited per function.
 * The Python binding is paper_1207_6365_b200/_lib.py (ctypes); see
 * INTEGRATION.md for the binding a maintainer adds to sketchnla.
 */
#ifndef SKETCH_B200_H
#define SKETCH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SKT_ABI_VERSION 1

typedef enum skt_status {
  SKT_OK = 0,
  SKT_EINVAL = 1,    /* bad argument (Python: ValueError, the reference convention) */
  SKT_ECUDA = 2,     /* CUDA runtime / launch failure (Python: RuntimeError) */
  SKT_ENOTSUP = 3,   /* valid but unsupported shape/dtype combination */
  SKT_EWORKSPACE = 4 /* workspace too small */
} skt_status;

typedef enum skt_dtype { SKT_F32 = 0, SKT_F64 = 1 } skt_dtype;
typedef enum skt_itype { SKT_I32 = 0, SKT_I64 = 1 } skt_itype;

/* flags for skt_apply_csr */
#define SKT_CSR_CANONICAL 1u /* no duplicate column inside a row (as_csr output) */
#define SKT_CSR_FAST 2u      /* allow unordered global atomics: not deterministic, SA to rounding */

/* 128-bit PCG64 state (numpy's PCG64: state and odd increment), hi/lo words. */
typedef struct skt_pcg64 {
  uint64_t state_hi, state_lo, inc_hi, inc_lo;
} skt_pcg64;

/* ---- host-side utilities ------------------------------------------------ */
const char *skt_version(void);
/* Message of the last non-OK status returned on this thread. */
const char *skt_last_error(void);
/* Number of CUDA kernels this library has launched in this process. */
uint64_t skt_launch_count(void);

/* numpy.random.SeedSequence(entropy, spawn_key).generate_state(n_out, uint32).
 * entropy = little-endian 32-bit words of the (non-negative) integer seed.
 * Replaces the seeding inside sketch.py:51-53 and the derived-seed idiom
 * SeedSequence(seed, spawn_key=(k,)).generate_state(1)[0] (regress.py:77-78,
 * leverage.py:72-73, lowrank.py:147-150). */
skt_status skt_seedseq_generate(const uint32_t *entropy, int32_t n_entropy,
                                const uint32_t *spawn_key, int32_t n_spawn,
                                uint32_t *out, int32_t n_out);

/* PCG64(SeedSequence(entropy, spawn_key)) initial state: sketch.py:51-53. */
skt_status skt_pcg64_seed(const uint32_t *entropy, int32_t n_entropy,
                          const uint32_t *spawn_key, int32_t n_spawn, skt_pcg64 *out);

/* numpy PCG64.advance(delta): jump ahead delta 64-bit outputs. */
skt_status skt_pcg64_advance(skt_pcg64 *st, uint64_t delta);

/* ---- K1: bucket hash h and sign s --------------------------------------- */
/* Replaces sketch.py:147 (bucket = integers(0, t, n)) and sketch.py:148
 * (sign = choice([-1, 1], n)), bit-exact, for the row range [row_begin,
 * row_end) of an operator with n >= row_end rows.  h[k] / s[k] receive the
 * values of row row_begin + k.  1 <= t <= 2^32.  s may be NULL.
 * When t is not a power of two (Lemire rejection possible), the call
 * synchronises `stream` once to confirm enough draws were generated. */
skt_status skt_hash_signs_workspace(int64_t row_end, uint64_t t, size_t *bytes);
skt_status skt_hash_signs(const skt_pcg64 *bucket_stream, const skt_pcg64 *sign_stream,
                          int64_t row_begin, int64_t row_end, uint64_t t, uint32_t *h,
                          int8_t *s, void *ws, size_t ws_bytes, void *stream);

/* ---- K2: the plan (S as a t x n CSR) ------------------------------------ */
/* Replaces sketch.py:149-151 (csr_array((sign, (bucket, arange(n))))).
 * shift = 0: indptr[t+1] (int64) = bucket offsets, rows[n] = row ids stably
 * sorted by bucket (ascending inside a bucket) -- exactly _mat.indptr /
 * _mat.indices -- with the row's sign in bit 31 (1 = -1.0).
 * shift = k in 1..8: the same rows stably sorted by bucket GROUP h >> k
 * (groups of 2^k consecutive buckets, ascending row order inside a group);
 * indptr has ngroups+1 = ((t-1) >> k) + 2 entries and blo[n] (uint8) gets each
 * row's bucket inside its group.  This is the order the grouped S.A kernels
 * sweep.  n < 2^31.  Deterministic (no atomics on positions). */
skt_status skt_plan_workspace(int64_t n, uint64_t t, int32_t shift, size_t *bytes);
skt_status skt_plan_build(const uint32_t *h, const int8_t *s, int64_t n, uint64_t t,
                          int32_t shift, int64_t *indptr, uint32_t *rows, uint8_t *blo,
                          void *ws, size_t ws_bytes, void *stream);

/* ---- K3: S.A for dense A ------------------------------------------------ */
/* Replaces sketch.py:165 (self._mat @ as_dense(a)) and the finiteness scan of
 * _validation.py:25-26.  A is n x d row-major (leading dim lda, f32 or f64),
 * SA is t x d row-major (ldsa).  Each SA[b, j] is the fp64 sum over the rows
 * of bucket b in ascending order starting from +0.0 -- bit-identical to the
 * reference; sa_dtype = SKT_F32 rounds that fp64 sum once.  If nonfinite_flag
 * (device int32) is non-NULL it is zeroed and then set to 1 if any entry of A
 * is Inf/NaN (the caller raises ValueError). */
skt_status skt_apply_dense(const int64_t *indptr, const uint32_t *rows, uint64_t t,
                           int64_t n, const void *a, skt_dtype a_dtype, int64_t d,
                           int64_t lda, void *sa, skt_dtype sa_dtype, int64_t ldsa,
                           int32_t *nonfinite_flag, void *stream);

/* ---- K4: S.A for CSR A -------------------------------------------------- */
/* Replaces sketch.py:155-164 (repeat + np.bincount): SA[h(i), j] += s(i) v
 * for every stored (i, j, v), fp64, per output in ascending row order and
 * stored order inside a row -- bit-identical to the bincount.  (indptr, rows,
 * blo, shift) is a plan from skt_plan_build; canonical input (flag
 * SKT_CSR_CANONICAL: no duplicate column inside a row) with narrow d runs the
 * grouped sweep kernel for any shift, otherwise a shift-0 plan is required.
 * CSR arrays of A may use int32 or int64 indptr / indices; values f32 or f64;
 * nnz = number of stored entries (a_indptr[n]).
 * Bucket ranges (K3 and K4, e.g. bucket-ownership sharding across GPUs): SA
 * rows [b0, b1) alone are computed by passing indptr + b0 (shift-0 plan; a
 * grouped plan: indptr + (b0 >> shift) with b0 a multiple of 2^shift),
 * t = b1 - b0 and sa + b0 * ldsa; the rows / blo arrays are shared. */
skt_status skt_apply_csr(const int64_t *indptr, const uint32_t *rows, const uint8_t *blo,
                         int32_t shift, uint64_t t, int64_t n, const void *a_indptr,
                         skt_itype indptr_type, const void *a_indices, skt_itype index_type,
                         const void *a_vals, skt_dtype val_dtype, int64_t nnz, int64_t d,
                         void *sa, skt_dtype sa_dtype, int64_t ldsa, uint32_t flags,
                         void *stream);

/* skt_apply_csr_wide: K4 for CSR A whose SA rows are too wide for on-chip
 * accumulators (BASELINE config 5: d = 262,144, t = 400) -- same contract and
 * bit-identical result as skt_apply_csr (ascending row order per output from
 * +0.0), for CANONICAL input (sorted, distinct column indices per row: as_csr
 * output), shift-0 plan (indptr, rows).  The entries are ordered by
 * 1024-column block (stable: row order kept) per 32-row piece of a bucket, then
 * one warp per (bucket, column block) adds them in row order into fp64
 * accumulators in shared memory (csrc/csr_fine.cuh); no atomics.  d > 524,288
 * or SKT_CSR_WIDE=partition|colblock: the 16384-column partition path / the
 * single-kernel column-block path.  Workspace (device, caller-owned):
 * skt_apply_csr_wide_workspace(n, t, d, nnz, val_dtype) bytes -- the piece
 * tables and the ordered entries (~nnz x (2 + value size) bytes). */
skt_status skt_apply_csr_wide_workspace(int64_t n, uint64_t t, int64_t d, int64_t nnz, skt_dtype val_dtype,
                                        size_t *bytes);
skt_status skt_apply_csr_wide(const int64_t *indptr, const uint32_t *rows, uint64_t t, int64_t n,
                              const void *a_indptr, skt_itype indptr_type, const void *a_indices,
                              skt_itype index_type, const void *a_vals, skt_dtype val_dtype, int64_t nnz,
                              int64_t d, void *sa, skt_dtype sa_dtype, int64_t ldsa, void *ws,
                              size_t ws_bytes, void *stream);

/* Row-window kernel for canonical CSR (csrc/csr_window.cuh; replaces
 * sketch.py:155-164 like skt_apply_csr): the same contract and bit-identical
 * result as skt_apply_csr, for fp32 values / int32 column
 * indices with rows of about 16 stored entries and an m x d fp64 SA that fits
 * the chip's shared memory (BASELINE config 4).  A is streamed ONCE in row
 * order: rows are cut into windows of W consecutive rows, every row of a
 * window is written as one 128-byte slot at its rank in the window's stable
 * sort by bucket (an L2-resident ring of windows), and the warp owning a
 * bucket range adds its contiguous slot range in ascending row order into
 * shared-memory fp64 accumulators.  No global data atomics.
 *   skt_csr_window_config: W (rows per window, 0 = shape not supported on this
 *     device) and the window count for an n-row input.
 *   skt_plan_window_build: from the shift-0 plan (indptr, rows) of
 *     skt_plan_build: pos[n] (slot of each row inside its window | sign << 31)
 *     and wpi[n_windows][t + 1] (first slot of every bucket per window).
 *   skt_apply_csr_window: SA (t x d, ldsa) in sa_dtype; SKT_ENOTSUP when the
 *     shape / alignment is outside the kernel's range (call skt_apply_csr). */
skt_status skt_csr_window_config(int64_t n, uint64_t t, int64_t d, int32_t *rows_per_window,
                                 int32_t *n_windows);
skt_status skt_plan_window_build(const int64_t *indptr, const uint32_t *rows, uint64_t t, int64_t n,
                                 int32_t rows_per_window, uint32_t *pos, int32_t *wpi, void *stream);
skt_status skt_apply_csr_window_workspace(int64_t n, int32_t rows_per_window, size_t *bytes);
skt_status skt_apply_csr_window(const uint32_t *pos, const int32_t *wpi, int32_t rows_per_window,
                                uint64_t t, int64_t n, const void *a_indptr, skt_itype indptr_type,
                                const int32_t *a_indices, const float *a_vals, int64_t nnz, int64_t d,
                                void *sa, skt_dtype sa_dtype, int64_t ldsa, void *ws, size_t ws_bytes,
                                void *stream);

/* Window gather kernel for canonical CSR (csrc/csr_cta.cuh; replaces
 * sketch.py:155-164 like skt_apply_csr): same contract and bit-identical
 * result as skt_apply_csr, fp32 values / int32 column indices,
 * m x d fp64 accumulators within the chip's shared memory.  Every SM owns a
 * contiguous bucket range; all SMs walk A window by window (rows of a window
 * stably sorted by bucket: wrows = the inverse of skt_plan_window_build's pos,
 * with the same wpi), loader warps gather the SM's rows of the window into
 * shared-memory slots with cp.async, accumulating half warps add them in
 * ascending row order.  No global workspace, no atomics.
 *   skt_csr_cta_config: rows per window (0 = shape not supported) and windows.
 *   skt_plan_window_rows: wrows[n] from pos[n] (same rows_per_window). */
skt_status skt_csr_cta_config(int64_t n, uint64_t t, int64_t d, int32_t *rows_per_window, int32_t *n_windows);
skt_status skt_plan_window_rows(const uint32_t *pos, int64_t n, int32_t rows_per_window, uint32_t *wrows,
                                void *stream);
skt_status skt_apply_csr_cta(const uint32_t *wrows, const int32_t *wpi, int32_t rows_per_window, uint64_t t,
                             int64_t n, const void *a_indptr, skt_itype indptr_type, const int32_t *a_indices,
                             const float *a_vals, int64_t nnz, int64_t d, void *sa, skt_dtype sa_dtype,
                             int64_t ldsa, void *stream);

/* skt_memcpy_staged: copy between PAGEABLE host memory and the device through
 * a ring of page-locked chunk buffers (host memcpy of chunk i + 1 overlaps the
 * DMA of chunk i; the CUDA driver copies pageable memory at ~11 GB/s here,
 * page-locked at ~55 GB/s).  kind 0 = host -> device: returns once src may be
 * reused, the device data is ordered on `stream`; kind 1 = device -> host:
 * returns when dst holds the data.  Serialised per device (one ring). */
skt_status skt_memcpy_staged(void *dst, const void *src, size_t bytes, int32_t kind, void *stream);

/* ---- column sketch A.S^T ------------------------------------------------ */
/* Replaces apply_right (sketch.py:445-448) = (S.apply(A.T)).T without the
 * transpose: Y[i, h(j)] += s(j) A[i, j], per output ascending j.  A has
 * n_rows rows and ncols = the operator's n columns; h/s are the operator's
 * per-column hash and sign (K1 output).  Y is n_rows x t row-major (ldy). */
skt_status skt_apply_right_dense(const uint32_t *h, const int8_t *s, uint64_t t,
                                 int64_t n_rows, int64_t ncols, const void *a,
                                 skt_dtype a_dtype, int64_t lda, void *y, skt_dtype y_dtype,
                                 int64_t ldy, int32_t *nonfinite_flag, void *stream);
skt_status skt_apply_right_csr(const uint32_t *h, const int8_t *s, uint64_t t,
                               int64_t n_rows, int64_t ncols, const void *a_indptr,
                               skt_itype indptr_type, const void *a_indices,
                               skt_itype index_type, const void *a_vals, skt_dtype val_dtype,
                               void *y, skt_dtype y_dtype, int64_t ldy, void *stream);

/* ---- K5: leverage-score contraction ------------------------------------- */
/* Replaces leverage.py:90-91 (rows = a @ probe; einsum('ij,ij->i', rows, rows))
 * fused: scores[i] = sum_c (sum_j A[i,j] probe[j,c])^2 with the n x k product
 * kept on chip.  probe is d x k row-major fp64 (probe = N G^T, leverage.py:89).
 * fp64 accumulation; scores written as score_dtype. */
skt_status skt_lev_rownorms_csr(int64_t n, int64_t d, const void *a_indptr,
                                skt_itype indptr_type, const void *a_indices,
                                skt_itype index_type, const void *a_vals, skt_dtype val_dtype,
                                const double *probe, int64_t k, void *scores,
                                skt_dtype score_dtype, void *stream);
skt_status skt_lev_rownorms_dense(int64_t n, int64_t d, const void *a, skt_dtype a_dtype,
                                  int64_t lda, const double *probe, int64_t k, void *scores,
                                  skt_dtype score_dtype, int32_t *nonfinite_flag, void *stream);

/* ---- residual pass on the original data --------------------------------- */
/* Replaces regress.py:81-82 (_residual_fro: ||a @ x - b||_F, the step after
 * every sketch-and-solve): *out_sq (device fp64) = sum_ij ((A X)_ij - B_ij)^2,
 * fused with the GEMV / SpMV so A is read once.  X is d x k fp64 row-major,
 * B is n x k (ldb) f32 or f64; A dense (lda) or CSR.  The workspace holds one
 * fp64 partial per block (skt_residual_workspace); the fixed-order block
 * reduction makes the result deterministic. */
skt_status skt_residual_workspace(size_t *bytes);
skt_status skt_residual_dense(int64_t n, int64_t d, const void *a, skt_dtype a_dtype, int64_t lda,
                              const double *x, int64_t k, const void *b, skt_dtype b_dtype,
                              int64_t ldb, double *out_sq, void *ws, size_t ws_bytes, void *stream);
skt_status skt_residual_csr(int64_t n, int64_t d, const void *a_indptr, skt_itype indptr_type,
                            const void *a_indices, skt_itype index_type, const void *a_vals,
                            skt_dtype val_dtype, const double *x, int64_t k, const void *b,
                            skt_dtype b_dtype, int64_t ldb, double *out_sq, void *ws,
                            size_t ws_bytes, void *stream);

/* ---- fused exchange for row-sharded multi-GPU S.A ------------------------ */
/* skt_apply_dense_push: K3 (TMA gather4 kernel; rows of 512 B .. 2 KB) that
 * stores each partial bucket row straight into its owner rank's receive
 * buffer instead of a local SA: owner g holds buckets [bounds[g],
 * bounds[g+1]) (nranks + 1 host int64), peers[g] (host array of nranks
 * pointers) is g's receive buffer -- a peer pointer over NVLink (symmetric
 * memory) or local -- laid out [src rank][cap bucket rows][ldr], and this
 * rank (me) writes slot me.  b0 = global id of local bucket 0 (bucket-range
 * launches).  skt_slot_sum: out[r][c] = sum over src = 0 .. nslots-1, in that
 * order, of recv[src * slot_stride + r * ldr + c] (fp64 accumulation) -- the
 * owner's deterministic reduction after a cross-rank barrier. */
skt_status skt_apply_dense_push(const int64_t *indptr, const uint32_t *rows, uint64_t t, int64_t n,
                                const void *a, skt_dtype a_dtype, int64_t d, int64_t lda,
                                skt_dtype out_dtype, void *const *peers, const int64_t *bounds,
                                int32_t nranks, int32_t me, int64_t cap, int64_t ldr, int64_t b0,
                                int32_t *nonfinite_flag, void *stream);
skt_status skt_slot_sum(const void *recv, skt_dtype dtype, int32_t nslots, int64_t rows, int64_t d,
                        int64_t slot_stride, int64_t ldr, void *out, int64_t ldo, void *stream);

/* ---- passes of the preconditioned iterations and the rank-k residual ----- */
/* SURVEY §8f rank 2, the passes over original data after the sketch.  M is
 * the n x r row-major fp64 product A R (regress.py:200, r <= 256); y, p are
 * r-vectors, b, q, rvec n-vectors (one right-hand-side column per call), all
 * fp64 on the device.  Reductions go through per-block partials in the
 * workspace (skt_lsq_workspace) and one fixed-order pass: deterministic.
 *  skt_lsq_residual_grad: *res2 = ||b - M y||^2, g = M^T (b - M y) (g may be
 *    NULL) -- Richardson's step y + M^T (b - M y) (regress.py:237-241) and the
 *    residual _iterate records (regress.py:209), one read of M.
 *  skt_lsq_matvec_norm: q = M p, *qq = ||q||^2 -- CGNR's mp and denom
 *    (regress.py:274-275).
 *  skt_lsq_update_grad: rvec <- rvec - q * alpha (product rounded, as numpy),
 *    z = M^T rvec, *res2 = ||M y - b||^2 -- CGNR's r, z (regress.py:278-279)
 *    and the residual of the new iterate, one read of M.
 *  skt_spmm_csr: Y = A X (n x k, ldy), A CSR, X d x k fp64 -- M = A R for a
 *    sparse A (regress.py:200).
 *  skt_gram_cross_csr / _dense: out2[0] = sum_i <A_i Mw, L_i>, out2[1] =
 *    ||A||_F^2 for Mw = W diag(d) (ncols x k, k <= 64) and L (n x k): the
 *    Gram-identity residual ||A - L D W^T||^2 = out2[1] - 2 out2[0] + sum d^2
 *    (lowrank.py:100-108), one read of A.  Workspace: skt_lsq_workspace(0). */
skt_status skt_lsq_workspace(int64_t r, size_t *bytes);
skt_status skt_lsq_residual_grad(int64_t n, int64_t r, const double *m, int64_t ldm, const double *y,
                                 const double *b, int64_t ldb, double *g, double *res2, void *ws,
                                 size_t ws_bytes, void *stream);
skt_status skt_lsq_matvec_norm(int64_t n, int64_t r, const double *m, int64_t ldm, const double *p,
                               double *q, int64_t ldq, double *qq, void *ws, size_t ws_bytes,
                               void *stream);
skt_status skt_lsq_update_grad(int64_t n, int64_t r, const double *m, int64_t ldm, const double *q,
                               int64_t ldq, double alpha, double *rvec, int64_t ldr, const double *y,
                               const double *b, int64_t ldb, double *z, double *res2, void *ws,
                               size_t ws_bytes, void *stream);
/* skt_gemm_dense: Y = A X (n x k, ldy), A dense n x d (lda, f32 / f64), X
 * d x k fp64 row-major, k <= 4096 -- M = A R for a dense A (regress.py:200),
 * fp64 dot products in ascending column order (equal to numpy's BLAS product
 * to rounding). */
skt_status skt_gemm_dense(int64_t n, int64_t d, const void *a, skt_dtype a_dtype, int64_t lda, const double *x,
                          int64_t k, double *y, int64_t ldy, void *stream);
skt_status skt_spmm_csr(int64_t n, int64_t d, const void *a_indptr, skt_itype indptr_type,
                        const void *a_indices, skt_itype index_type, const void *a_vals,
                        skt_dtype val_dtype, int64_t nnz, const double *x, int64_t k, double *y,
                        int64_t ldy, void *stream);
skt_status skt_gram_cross_csr(int64_t n, int64_t ncols, const void *a_indptr, skt_itype indptr_type,
                              const void *a_indices, skt_itype index_type, const void *a_vals,
                              skt_dtype val_dtype, const double *mw, int64_t ldm, int64_t k,
                              const double *l, int64_t ldl, double *out2, void *ws, size_t ws_bytes,
                              void *stream);
skt_status skt_gram_cross_dense(int64_t n, int64_t ncols, const void *a, skt_dtype a_dtype,
                                int64_t lda, const double *mw, int64_t ldm, int64_t k,
                                const double *l, int64_t ldl, double *out2, void *ws,
                                size_t ws_bytes, void *stream);

/* ---- SRHT of a tall fp64 matrix ---------------------------------------- */
/* Replaces SrhtOperator.apply (sketch.py:284-291) on device data: rows of A
 * (n x d, lda) zero-padded to n_pad = 2^ceil(log2 n), multiplied by sign[i]
 * (n_pad entries, +-1.0), unnormalised Walsh-Hadamard transform along the
 * rows (_fwht, sketch.py:241-252 -- the same butterflies in the same stage
 * order, so bit-identical), then out[r, :] = scale * H[rows[r], :] for the t
 * sampled rows.  The workspace holds the n_pad x d transform
 * (skt_srht_workspace). */
skt_status skt_srht_workspace(int64_t n, int64_t d, size_t *bytes);
skt_status skt_srht_apply(const double *a, int64_t n, int64_t d, int64_t lda, const int8_t *sign,
                          const uint32_t *rows, int64_t t, double scale, double *out, int64_t ldo,
                          void *ws, size_t ws_bytes, void *stream);

/* ---- generalized sparse embedding ---------------------------------------- */
/* GeneralizedSparseEmbedding (sketch.py:176-238): k_blocks entries per input
 * row j at h_b(j) = outer(j) k v + b v + inner_b(j), weight sign_b(j)/sqrt(k).
 * The plan is the CountSketch plan over k n virtual rows vid = b n + j (the
 * reference's (k, n) draw order): skt_hash_signs draws outer (stream (1, 0),
 * t = q) and inner buckets / signs (streams (1, 1) / (1, 2), t = v, k n rows),
 * skt_gse_buckets combines them into h[vid] (t = q k v < 2^32), skt_plan_build
 * sorts the virtual rows, skt_gse_fold_rows rewrites plan words to j.
 * skt_gse_apply_dense / _csr compute SA = self._mat @ a (sketch.py:222-227)
 * with scipy's per-element order and rounding (fp64, products rounded, no FMA:
 * bit-identical); SA is fp64 t x d (ldsa).  Dense A has n rows (rows of
 * 128 B .. 1 KB use K3's TMA gather4 kernel with weighted terms, |weight| <= 1). */
skt_status skt_gse_buckets(const uint32_t *outer, const uint32_t *inner, int64_t n, int32_t k, uint32_t v,
                           uint64_t q, uint32_t *h, void *stream);
skt_status skt_gse_fold_rows(uint32_t *rows, int64_t count, int64_t n, void *stream);
skt_status skt_gse_apply_dense(const int64_t *indptr, const uint32_t *rows, uint64_t t, int64_t n,
                               const void *a, skt_dtype a_dtype, int64_t d, int64_t lda, double weight,
                               double *sa, int64_t ldsa, int32_t *nonfinite_flag, void *stream);
skt_status skt_gse_apply_csr(const int64_t *indptr, const uint32_t *rows, uint64_t t, const void *a_indptr,
                             skt_itype indptr_type, const void *a_indices, skt_itype index_type,
                             const void *a_vals, skt_dtype val_dtype, int64_t d, double weight, double *sa,
                             int64_t ldsa, void *stream);

/* ---- Matrix Market ingest ------------------------------------------------- */
/* Replaces load_matrix_market (io.py:37-104).  skt_mm_probe reads the header
 * and size line; skt_mm_read_coo parses the coordinate entries on n_threads
 * host threads (0 = all cores) into caller host arrays (0-based, capacity >=
 * n_entries, x2 for symmetric storage, which is expanded as the reference
 * does), with the reference's "path:line: reason" errors (SKT_EINVAL).
 * skt_coo_to_csr canonicalises on the device (io.py:101-102 -> as_csr,
 * _validation.py:30-41): (row, col)-sorted, duplicates summed in file order,
 * zero sums dropped; indptr (n_rows + 1, int64), indices (int32), values
 * (fp64, capacity count), *nnz (device int64); *nonfinite (device int32,
 * may be NULL) is set to 1 when a kept (summed) entry is NaN or +-inf -- the
 * caller raises as_csr's "contains non-finite entries" (_validation.py:39-40). */
typedef struct skt_mm_info {
  int64_t n_rows, n_cols, n_entries;
  int32_t field;     /* 0 real, 1 integer, 2 pattern */
  int32_t symmetric; /* 0 general, 1 symmetric */
} skt_mm_info;
skt_status skt_mm_probe(const char *path, skt_mm_info *info);
skt_status skt_mm_read_coo(const char *path, int64_t capacity, int64_t *rows, int64_t *cols, double *vals,
                           int64_t *count, int32_t n_threads);
skt_status skt_coo_to_csr_workspace(int64_t count, int64_t n_rows, int64_t n_cols, size_t *bytes);
/* skt_csr_check_sorted: *flag (device int32) = 1 if some row's column indices
 * are not strictly increasing (duplicates / unsorted -- not as_csr's canonical
 * form, _validation.py:30-41), else 0.  The device replacement for scipy's
 * O(nnz) host scan (has_canonical_format) ahead of skt_apply_csr's
 * SKT_CSR_CANONICAL flag. */
skt_status skt_csr_check_sorted(int64_t n, const void *a_indptr, skt_itype indptr_type, const void *a_indices,
                                skt_itype index_type, int32_t *flag, void *stream);
skt_status skt_coo_to_csr(const int64_t *rows, const int64_t *cols, const double *vals, int64_t count,
                          int64_t n_rows, int64_t n_cols, int64_t *indptr, int32_t *indices, double *out_vals,
                          int64_t *nnz, int32_t *nonfinite, void *ws, size_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SKETCH_B200_H */
