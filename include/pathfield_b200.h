/*
 * pathfield_b200.h — C ABI of the B200-native divergence-distance hot path.
 *
 * Drop-in boundary for the reference package `pathfield` (pure Python,
 * /root/reference/pkg/src/pathfield).  The reference has no native code, so
 * each entry point below replaces one numpy/scipy computation inside a
 * reference function; the citation on each declaration names it.  The
 * Python mirror (paper_1708_02845_b200/) keeps the reference signatures and
 * calls these through ctypes; a maintainer of the reference would bind them
 * the same way.
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer (buffers owned by the caller, e.g.
 *     torch tensors) unless the parameter name ends in `_host`.
 *   - Every call takes the CUDA stream to launch on (`pf_stream_t`, a
 *     cudaStream_t passed as void*) and is asynchronous on that stream.
 *   - Every call returns 0 on success, otherwise a PF_E_* code or a
 *     cudaError_t value (> 0); pf_last_error() returns the message of the
 *     most recent failure on the calling thread.  Nothing throws.
 *   - No hidden allocation: scratch is passed in by the caller.
 *   - Matrices are row-major with an explicit leading dimension `ld`
 *     (elements).  Dense P rows must be 16-byte aligned: `ld` even and the
 *     base pointer 16-byte aligned.
 *   - Row slabs: a call may cover rows [row0, row0+rows) of the global
 *     matrix (multi-GPU row sharding); `P`, `H`, `is_interior` and `out`
 *     point at the slab, while `target` is a GLOBAL row index.
 */
#ifndef PATHFIELD_B200_H
#define PATHFIELD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *pf_stream_t;

enum {
  PF_OK = 0,
  PF_E_ARG = -1,     /* invalid argument (null pointer, bad size)           */
  PF_E_ALIGN = -2,   /* misaligned pointer or odd leading dimension         */
  PF_E_DOMAIN = -3,  /* value outside the supported domain                  */
  PF_E_LAUNCH = -4,  /* kernel launch failed (message in pf_last_error)     */
  PF_E_CAPACITY = -5 /* output buffer too small (count returned separately) */
};

/* Divergence generators (divergence.py:70-104).  The dense kernels are
 * templated over these; kl and tv are the north-star pair. */
enum {
  PF_DIV_KL = 0,        /* f(x) = -log x,          clamp 1e-300 (:82-83)   */
  PF_DIV_TV = 1,        /* f(x) = |1-x|,           clamp 1e-150 (:79-81)   */
  PF_DIV_CHI2 = 2,      /* f(x) = x^2 - 1,         clamp 1e-150 (:84-86)   */
  PF_DIV_HELLINGER = 3, /* f(x) = (sqrt x - 1)^2,  clamp 1e-150 (:87-89)   */
  PF_DIV_ALPHA = 4,     /* 4/(1-a^2)(1-x^((1+a)/2)), clamp 1e-300 (:90-97) */
  PF_DIV_POWER = 5      /* |1-x|^p,                clamp 1e-150 (:98-103)  */
};

/* Flag words written by the field kernels (uint32 array `flags`, >= 4). */
enum {
  PF_FLAG_CLAMPED = 0,   /* != 0: clamping fired one-sidedly on an interior
                            row — divergence.py:172-175 ("clamped")        */
  PF_FLAG_GUARDED = 1,   /* number of rows recomputed in per-element form  */
  PF_FLAG_NONPOS = 2,    /* reserved                                       */
  PF_FLAG_SPARE = 3
};

int pf_version(void);
const char *pf_last_error(void);
/* Number of SMs of the current device (grid sizing helper). */
int pf_sm_count(void);

/* ---- K0: per-target staging ------------------------------------------
 * From the raw target row Pt (k doubles, device) write
 *   tgt[b]      = max(Pt[b], clamp)            (b < k; pad to k_pad = 1.0)
 *   logt[b]     = log(max(Pt[b], clamp))       (b < k; pad 0.0)
 *   tmask[b]    = Pt[b] < clamp                (b < k; pad 0)
 * and zero flags[0..3].  Replaces the `ps_t = np.maximum(dense[p], clamp)`
 * line of dv_field (divergence.py:170) and the target half of the
 * one-sided compare (:172).  `clamp <= 0` means "no clamp" (identity).
 * Buffers tgt/logt must hold k_pad = round_up(k, 2) doubles and tmask
 * round_up(k, 16) bytes. */
int pf_target_prep_f64(const double *Pt, int64_t k, double clamp, double *tgt,
                       double *logt, uint8_t *tmask, uint32_t *flags,
                       pf_stream_t stream);

/* ---- K1: per-row negentropy -------------------------------------------
 * H[r] = sum_{b<k} c(P[r,b]) * log c(P[r,b]),  c(x) = max(x, clamp).
 * Target-independent; computed once per (P, clamp).  It is the Q log Q half
 * of the reference KL sum (divergence.py:180 with f = -log, :82-83).
 * Also writes min_out[0] = min over the slab of P (for the clamp <= 0
 * domain check, divergence.py:162-165) if min_out != NULL (caller seeds
 * min_out[0] with +inf). */
int pf_row_negentropy_f64(const double *P, int64_t ld, int64_t rows, int64_t k,
                          double clamp, double *H, double *min_out,
                          pf_stream_t stream);

/* ---- K2: dense KL field -------------------------------------------------
 * out[r] = sum_b c(Q_rb) * (-log(c(Pt_b)/c(Q_rb)))  for global row
 * row0 + r, evaluated as H[r] - sum_b c(Q_rb) * logt[b] with a cancellation
 * guard: rows with |out| < tau*(|H|+|cross|) are re-evaluated in the
 * reference's per-element form by the same launch — in 512-element chunks
 * shared by the warps of the CTA that found them, summed in an order fixed by
 * k alone (counted in flags[PF_FLAG_GUARDED]).  Then the settle rule (-1e-10,0) -> 0 and
 * out[target-row0] = 0.  Replaces dv_field's kl evaluation
 * (divergence.py:170-182).  flags[PF_FLAG_CLAMPED] |= one-sided clamp on a
 * row with is_interior[r] != 0 (is_interior may be NULL = all interior). */
int pf_dense_kl_f64(const double *P, int64_t ld, int64_t rows, int64_t k,
                    const double *H, const double *tgt, const double *logt,
                    const uint8_t *tmask, double clamp, double tau,
                    int64_t row0, int64_t target, const uint8_t *is_interior,
                    double *out, uint32_t *flags, pf_stream_t stream);

/* ---- K3: dense TV field ---------------------------------------------------
 * out[r] = sum_b |c(Q_rb) - c(Pt_b)|  (== sum c(Q)|1 - c(Pt)/c(Q)|, the
 * reference tv evaluation divergence.py:79-81,180, within rounding), then
 * settle and out[target-row0] = 0; clamp flag as for K2. */
int pf_dense_tv_f64(const double *P, int64_t ld, int64_t rows, int64_t k,
                    const double *tgt, const uint8_t *tmask, double clamp,
                    int64_t row0, int64_t target, const uint8_t *is_interior,
                    double *out, uint32_t *flags, pf_stream_t stream);

/* ---- K2/K3 generalised: any builtin generator (divergence.py:70-104) ----
 * out[r] = sum_b c(Q) f(c(Pt)/c(Q)) per-element (no split form), settle,
 * target zero, clamp flag.  `kind` is PF_DIV_*, `param` the alpha or the
 * power exponent.  swap_order != 0 evaluates sum_b c(Pt) f(c(Q)/c(Pt))
 * (divergence.py:177-178). */
int pf_dense_generic_f64(const double *P, int64_t ld, int64_t rows, int64_t k,
                         const double *tgt, const uint8_t *tmask, double clamp,
                         int kind, double param, int swap_order, int64_t row0,
                         int64_t target, const uint8_t *is_interior,
                         double *out, uint32_t *flags, pf_stream_t stream);

/* ---- dv_at: the same arithmetic on a gathered subset of query rows ------
 * out[i] = KL/TV/... for query row queries[i] (global index into P, whose
 * slab starts at row0), using the per-element reference form
 * (divergence.py:137-151); out[i] = 0 where queries[i] == target. */
int pf_dense_at_f64(const double *P, int64_t ld, int64_t rows, int64_t k,
                    const double *tgt, double clamp, int kind, double param,
                    int swap_order, int64_t row0, int64_t target,
                    const int64_t *queries, int64_t nq, double *out,
                    pf_stream_t stream);

/* ---- FP32 storage mode (north-star tolerance 1e-5 relative) -------------
 * pf_convert_f32: out (rows x ld32, ld32 % 4 == 0) = (float)P, pad 0.
 * pf_row_negentropy_f32: H[r] = sum c(Q32) log c(Q32) in FP64 over FP32 rows.
 * pf_dense_kl_f32 / pf_dense_tv_f32: the K2 / K3 fields with the query rows
 * read from the FP32 copy (half the bytes); target row, logs, H and all
 * accumulation FP64, H the FP64 negentropy of the FP64 rows
 * (pf_row_negentropy_f64 of P64; the FP32 rounding then only perturbs the
 * cross term, by at most 2^-24 |cross|).  Rows whose value cannot be
 * certified to 1e-5 against that bound (|KL| < tau*|cross|, |TV| < tau; tau = 1e-2)
 * are re-evaluated from the FP64 rows P64 (count in flags[PF_FLAG_GUARDED]):
 * TV exactly; KL in the FP64 split form H64[r] - sum c(Q64) logt when H64
 * (pf_row_negentropy_f64 of P64) is given, falling back to the reference form
 * only where that cancels too (|KL| < tau64*(|H64|+|cross64|), the K2 guard),
 * or directly in the reference form when H64 is NULL.  Staging buffers as for K2/K3 (pf_target_prep_f64);
 * tmask / is_interior are accepted for symmetry but unused: FP32 rounding
 * flushes sub-float-range entries to 0, so the `clamped` flag must come from
 * the FP64 rows — pf_mask_compare_f64 below plus pf_mask_uniform_f64.
 * pf_mask_compare_f64: flag[0] |= 1 if (a[i] < clamp) != (b[i] < clamp) for
 * some i < k. */
int pf_convert_f32(const double *P, int64_t ld, int64_t rows, int64_t k, float *out,
                   int64_t ld32, pf_stream_t stream);
int pf_row_negentropy_f32(const float *P, int64_t ld, int64_t rows, int64_t k, double clamp,
                          double *H, pf_stream_t stream);
int pf_dense_kl_f32(const float *P, int64_t ld, int64_t rows, int64_t k, const double *H,
                    const double *tgt, const double *logt, const uint8_t *tmask, double clamp,
                    double tau, int64_t row0, int64_t target, const uint8_t *is_interior,
                    const double *P64, int64_t ld64, const double *H64, double tau64,
                    double *out, uint32_t *flags, pf_stream_t stream);
int pf_dense_tv_f32(const float *P, int64_t ld, int64_t rows, int64_t k, const double *tgt,
                    const uint8_t *tmask, double clamp, double tau, int64_t row0, int64_t target,
                    const uint8_t *is_interior, const double *P64, int64_t ld64, double *out,
                    uint32_t *flags, pf_stream_t stream);
int pf_mask_compare_f64(const double *a, const double *b, int64_t k, double clamp,
                        uint32_t *flag, pf_stream_t stream);

/* ---- K4: sparsify (divergence.py:194-240) ---------------------------------
 * keep = P >= cut (strict_positive == 0; cut = threshold / k computed by the
 * caller exactly as divergence.py:219) or P > 0 (threshold 0, :220).
 * pf_csr_count_f64 writes the per-row kept count c_r; the caller scans the
 * ROW-ALIGNED lengths c_r + (c_r & 1) into indptr (rows+1, int64, indptr[0]
 * = 0) and sets bit 0 of indptr[r+1] when c_r is odd: every row starts at an
 * even offset (indptr[r] & ~1), and a row with an odd count ends with one zero
 * pad entry (data 0, log 0) that every kernel excludes — so a row's element
 * order never depends on the row's position (a multi-GPU slab reduces each
 * row exactly like the whole CSR).  pf_csr_fill_f64 then
 * writes, in scipy's order (row-major, ascending column):
 *   indices (int32), data = kept P values, log_data = log(data) (:224-225),
 *   hs[r] = sum data*log_data (the split-form KL row term), and
 *   dropped[r] = max(0, 1 - rowsum) with rowsum in numpy reduceat order
 *   (:227-228; bitwise the reference's). */
int pf_csr_count_f64(const double *P, int64_t ld, int64_t rows, int64_t k, double cut,
                     int strict_positive, int64_t *rownnz, pf_stream_t stream);
int pf_csr_fill_f64(const double *P, int64_t ld, int64_t rows, int64_t k, double cut,
                    int strict_positive, const int64_t *indptr, int32_t *indices,
                    double *data, double *log_data, double *hs, double *dropped,
                    pf_stream_t stream);

/* ---- K5/K6 per-target staging ---------------------------------------------
 * From CSR row p_local of the slab: vp[0..round_up(k,2)) = the sparsified
 * target row scattered dense (0 off-support), tscal[0] = S_p = sum of its
 * kept values, tscal[1] = dropped[p], tscal[2] = nnz_p (tscal holds 4 doubles).
 * Replaces _row_support/_aligned for the target side (divergence.py:243-252). */
int pf_csr_target_prep_f64(const int64_t *indptr, const int32_t *indices,
                           const double *data, const double *dropped, int64_t p_local,
                           int64_t k, double *vp, double *tscal, pf_stream_t stream);

/* ---- K5: CSR KL field -------------------------------------------------------
 * out[i] = sum_{j in supp(q)} v_qj (log v_qj - logt[j]),  q = queries[i] (global;
 * slab rows start at row0) or q = row0 + i when queries == NULL; logt[j] =
 * log(max(P[p,j], 1e-300)) is the target's dense log row (log_dense[p],
 * divergence.py:226,277).  Split form hs[q] - sum v logt with a cancellation
 * guard re-evaluated in the reference form; then _settle (:286).
 * ops[i] = |supp(q)| (:276) if ops != NULL; flags[PF_FLAG_GUARDED] counts
 * re-evaluated rows.  With `inline_guard` != 0 (flags and log_data required;
 * flags[PF_FLAG_GUARDED] zero on entry, as pf_target_prep_f64 leaves it) the
 * field kernel re-evaluates a guarded row in place, with the target logs
 * already in shared memory (one launch); with inline_guard == 0 a second pass
 * scans the output for the guard sentinel.  Both re-evaluate in the same
 * order, so the results are identical. */
int pf_csr_kl_f64(const int64_t *indptr, const int32_t *indices, const double *data,
                  const double *log_data, const double *hs, int64_t rows, int64_t k,
                  const double *logt, double tau, int64_t row0, const int64_t *queries,
                  int64_t nq, double *out, int64_t *ops, uint32_t *flags, int inline_guard,
                  pf_stream_t stream);

/* ---- K6: CSR TV field -------------------------------------------------------
 * out[i] = sum_{union} |vp - vq| + dropped[p] + dropped[q] (divergence.py:288-295,
 * no settle), evaluated in one pass over supp(q) with vp/tscal from
 * pf_csr_target_prep_f64; ops[i] = |supp(p) U supp(q)| (:289). */
int pf_csr_tv_f64(const int64_t *indptr, const int32_t *indices, const double *data,
                  const double *dropped, int64_t rows, int64_t k, const double *vp,
                  const double *tscal, int64_t row0, const int64_t *queries, int64_t nq,
                  double *out, int64_t *ops, pf_stream_t stream);

/* ---- K5/K6 over 16-bit column indices (k <= 65,536) -------------------------
 * The same fields with the device CSR's columns narrowed to uint16
 * (pf_csr_narrow_u16, once per CSR): 10 instead of 12 streamed bytes per
 * entry (the algorithmic figure stays scipy's int32 layout). */
/* The row-aligned device CSR in scipy's layout (what sparsify returns,
 * divergence.py:221-226): entries of row r move to sp_indptr[r] (the exclusive
 * prefix of the real row counts), pads dropped; o_data / o_log may be NULL. */
int pf_csr_unpad(const int64_t *indptr, const int64_t *sp_indptr, int64_t rows,
                 const int32_t *indices, const double *data, const double *log_data,
                 int32_t *o_indices, double *o_data, double *o_log, pf_stream_t stream);
int pf_csr_narrow_u16(const int32_t *indices, int64_t n, uint16_t *indices16,
                      pf_stream_t stream);
int pf_csr_kl_u16_f64(const int64_t *indptr, const uint16_t *indices16, const double *data,
                      const double *log_data, const double *hs, int64_t rows, int64_t k,
                      const double *logt, double tau, int64_t row0, const int64_t *queries,
                      int64_t nq, double *out, int64_t *ops, uint32_t *flags, int inline_guard,
                      pf_stream_t stream);
int pf_csr_tv_u16_f64(const int64_t *indptr, const uint16_t *indices16, const double *data,
                      const double *dropped, int64_t rows, int64_t k, const double *vp,
                      const double *tscal, int64_t row0, const int64_t *queries, int64_t nq,
                      double *out, int64_t *ops, pf_stream_t stream);

/* ---- K5/K6 for the other generators (divergence.py:275-299) ---------------
 * kind PF_DIV_ALPHA: sum_{supp q} v (1 - exp(expo (logt - log v))) * scale,
 *   settle; ops = |supp q|.  Needs logt (the target's dense log row).
 * kind PF_DIV_CHI2 / PF_DIV_HELLINGER / PF_DIV_POWER: the union form with
 *   weights clamped at `cut`; prow = the target's DENSE row, p_local its row in
 *   this slab's CSR; ops = |union|.  Both settle the result. */
int pf_csr_generic_f64(const int64_t *indptr, const int32_t *indices, const double *data,
                       const double *log_data, int64_t rows, int64_t k, int kind, double param,
                       double cut, const double *prow, int64_t p_local, const double *logt,
                       int64_t row0, const int64_t *queries, int64_t nq, double *out,
                       int64_t *ops, pf_stream_t stream);

/* Elementwise log view: out[r*k + c] = log(max(P[r*ld + c], clamp)), the
 * reference's log_dense (divergence.py:226), materialised on request. */
int pf_log_clamped_f64(const double *P, int64_t ld, int64_t rows, int64_t k, double clamp,
                       double *out, pf_stream_t stream);

/* ---- K7: KL to a batch of T targets (T x dv_field, divergence.py:154-187) ---
 * pf_batch_prep_f64: from the T raw target rows Pt (T x ldp) write
 *   L[t,b] = log(max(Pt[t,b], clamp)) and Tc[t,b] = max(Pt[t,b], clamp)
 *   (T x ldl, ldl = round_up(k,16), zero / one padded) and
 *   tflag[t] = 1 if the below-clamp mask of Pt[t] differs from that of `ref`
 *   (the mask shared by the interior rows, see pf_mask_uniform_f64).
 * pf_mask_uniform_f64: nonuniform[0] |= 1 if any interior row's mask
 *   (P < clamp) differs from ref's; with it the per-target `clamped` flag of
 *   divergence.py:172-175 is exact: flag_t = nonuniform || tflag[t].
 * pf_batched_kl_f64: out[q*ldo + t] = KL(q, targets[t]) for the slab rows:
 *   H[q] - (Qc L^T)[q,t] as an FP64 GEMM with a fused epilogue (guard,
 *   settle, zero at the target), then the guarded pairs re-evaluated in the
 *   reference's per-element form (count added to *guarded if non-NULL). */
int pf_batch_prep_f64(const double *Pt, int64_t ldp, int64_t T, int64_t k, int64_t ldl,
                      double clamp, const double *ref, double *L, double *Tc, uint32_t *tflag,
                      pf_stream_t stream);
int pf_mask_uniform_f64(const double *P, int64_t ld, int64_t rows, int64_t k, double clamp,
                        const uint8_t *is_interior, const double *ref, uint32_t *nonuniform,
                        pf_stream_t stream);
int pf_batched_kl_f64(const double *P, int64_t ld, int64_t rows, int64_t k, const double *H,
                      const double *L, const double *Tc, int64_t ldl, int64_t T,
                      const int64_t *targets, double clamp, double tau, int64_t row0,
                      double *out, int64_t ldo, uint32_t *guarded, pf_stream_t stream);

/* pf_batched_kl_fixup_f64: the guarded-pair pass of pf_batched_kl_f64 on its
 * own: every out entry holding the guard sentinel is re-evaluated in the
 * reference's per-element form sum c(Q) (-log(c(Pt)/c(Q))) (divergence.py:180)
 * and settled; the count is added to *guarded if non-NULL. */
int pf_batched_kl_fixup_f64(const double *P, int64_t ld, int64_t rows, int64_t k,
                            const double *Tc, int64_t ldl, int64_t T, double clamp, double *out,
                            int64_t ldo, uint32_t *guarded, pf_stream_t stream);
/* The same over the guarded-pair list pf_batched_kl_i8_listed recorded
 * (guard_list[0] = count, then q * T + t): no scan of the output; a list
 * that overflowed guard_cap falls back to the scan.  Same values. */
int pf_batched_kl_fixup_list_f64(const double *P, int64_t ld, int64_t rows, int64_t k,
                                 const double *Tc, int64_t ldl, int64_t T, double clamp,
                                 double *out, int64_t ldo, uint32_t *guarded,
                                 const int64_t *guard_list, int64_t guard_cap, pf_stream_t stream);

/* ---- K7 on the int8 tensor pipe (batched_i8.cu) ----------------------------
 * The same contraction as pf_batched_kl_f64, S = c(P) . (-L)^T, evaluated as
 * an exact-integer emulation of the FP64 GEMM: both operands are non-negative
 * 56-bit fixed-point numbers against a power-of-two scale per row / target,
 * cut into 7 byte planes; the 34 byte-pair GEMMs of levels 2..9 run on
 * tcgen05.mma kind::i8 (u8 x u8 -> s32 in TMEM) and are combined in FP64.
 * pf_slice_rows_u8: slices [7][rows][ldk] and exps[rows] of max(P, clamp)
 *   (target independent, cached per P like H); ldk % 64 == 0, pad zero.
 * pf_slice_targets_u8: slices [7][T][ldk] and exps[T] of -L (L from
 *   pf_batch_prep_f64); bad[0] |= 1 if some -L < 0 (then use the FP64 path).
 * pf_batched_kl_i8: out[q*ldo + t] = H[q] + S[q,t] with the K7 epilogue
 *   (guard sentinel, settle, zero at the target); k <= 4717.  grade 64 keeps
 *   levels 2..9 of all 7 planes (34 pairs, FP64-grade: within 1e-10 of the
 *   reference), grade 32 levels 2..6 of the top 5 planes (15 pairs, the
 *   north-star FP32 tolerance 1e-5).  cta_pair != 0 runs the persistent
 *   CTA-pair kernel (tcgen05 cta_group::2, M256 tiles over two SMs, the
 *   epilogue overlapped with the next tile's MMAs), bitwise the same outputs
 *   as cta_pair == 0 (one CTA per 128 x 128 tile).
 *   Follow with pf_batched_kl_fixup_f64 for
 *   the guarded pairs. */
int pf_slice_rows_u8(const double *P, int64_t ld, int64_t rows, int64_t k, double clamp,
                     int64_t ldk, uint8_t *slices, int32_t *exps, pf_stream_t stream);
int pf_slice_targets_u8(const double *L, int64_t ldl, int64_t T, int64_t k, int64_t ldk,
                        uint8_t *slices, int32_t *exps, uint32_t *bad, pf_stream_t stream);
int pf_batched_kl_i8(const uint8_t *A, const int32_t *ea, int64_t rows, const uint8_t *B,
                     const int32_t *eb, int64_t T, int64_t k, int64_t ldk, const double *H,
                     const int64_t *targets, double tau, int64_t row0, double *out, int64_t ldo,
                     int grade, int cta_pair, pf_stream_t stream);
/* pf_batched_kl_i8 that also appends every guarded pair to guard_list
 * (int64[1 + guard_cap]; guard_list[0] is the count and must be zero before
 * the call): then follow with pf_batched_kl_fixup_list_f64. */
int pf_batched_kl_i8_listed(const uint8_t *A, const int32_t *ea, int64_t rows, const uint8_t *B,
                            const int32_t *eb, int64_t T, int64_t k, int64_t ldk, const double *H,
                            const int64_t *targets, double tau, int64_t row0, double *out,
                            int64_t ldo, int grade, int cta_pair, int64_t *guard_list,
                            int64_t guard_cap, pf_stream_t stream);
/* The tiled operand layout the CTA-pair kernel streams best: byte plane s,
 * tile u, 32-byte K block kb is one contiguous run of R x 32 bytes (R = 128
 * rows for A, 64 targets for B) holding the SWIZZLE_32B shared-memory image,
 * so a TMA box is 256-byte rows (1.6x the L2 ingest rate of the row-major
 * box, 4x from HBM).  Each operand takes pf_i8_tiled_bytes(n, k) bytes (rows
 * / targets padded to 128 with zeros, K to 32), 16-byte aligned.
 * pf_batched_kl_i8_tiled: pf_batched_kl_i8_listed with cta_pair = 1 on the
 * tiled operands (guard_list may be NULL); bitwise the same outputs. */
int64_t pf_i8_tiled_bytes(int64_t n, int64_t k);
int pf_slice_rows_u8_tiled(const double *P, int64_t ld, int64_t rows, int64_t k, double clamp,
                           uint8_t *tiles, int32_t *exps, pf_stream_t stream);
int pf_slice_targets_u8_tiled(const double *L, int64_t ldl, int64_t T, int64_t k, uint8_t *tiles,
                              int32_t *exps, uint32_t *bad, pf_stream_t stream);
int pf_batched_kl_i8_tiled(const uint8_t *A, const int32_t *ea, int64_t rows, const uint8_t *B,
                           const int32_t *eb, int64_t T, int64_t k, const double *H,
                           const int64_t *targets, double tau, int64_t row0, double *out,
                           int64_t ldo, int grade, int64_t *guard_list, int64_t guard_cap,
                           pf_stream_t stream);

/* Diagnostic: back-to-back M128 N256 K32 u8 tcgen05.mma on shared-memory
 * operands, one CTA per SM (*ops_host = integer ops issued): the int8 tensor
 * pipe ceiling pf_batched_kl_i8 is measured against.  random_operands != 0
 * fills the operands with hashed random bytes (K7's slice planes are random
 * bytes, and the tensor pipe's power draw -- hence the clock it holds under
 * the board's power cap -- depends on the operand bits; MEASURED_PEAKS'
 * bf16 figure is likewise taken on random matrices), 0 with a 0..3 pattern. */
int pf_probe_umma_i8(int64_t iters, int random_operands, int64_t *ops_host, uint32_t *sink,
                     pf_stream_t stream);

/* Diagnostic: a pure-DFMA kernel (8 independent FMA chains per thread, all
 * SMs); *flops_host receives its FLOP count so the caller can time it and
 * obtain the sustained FP64 rate K7 is measured against. */
int pf_probe_dfma_f64(int64_t iters, int64_t *flops_host, double *out, pf_stream_t stream);

/* Diagnostic: stream n doubles of buf (16-byte aligned) with the field
 * kernels' loads and nothing else: the pure-read HBM ceiling the dense
 * streams are reported against beside the copy peak. */
int pf_probe_hbm_read(const double *buf, int64_t n, double *sink, pf_stream_t stream);

/* ---- K8: batched triangle-descent tracer (paths.py:101-307) ---------------
 * Device-resident mesh topology (all arrays device pointers):
 *   vertices  (n,2) FP64;  triangles (nt,3) int32 CCW exactly as stored by
 *   TriMesh (mesh.py:57-68);  areas (nt) = TriMesh.triangle_areas;
 *   tri_nbr (nt,3) int32: the triangle across the edge opposite each slot, -1
 *   on the boundary (edge_adjacency, mesh.py:113-126);  vt_ptr/vt_idx: the
 *   ascending incident triangles of each vertex (vertex_triangles);
 *   nb_ptr/nb_idx: ascending neighbours (neighbors);
 *   eps_prog = 1e-14 * bbox_diagonal (paths.py:143). */
typedef struct {
  const double *vertices;
  const int32_t *triangles;
  const double *areas;
  const int32_t *tri_nbr;
  const int64_t *vt_ptr;
  const int32_t *vt_idx;
  const int64_t *nb_ptr;
  const int32_t *nb_idx;
  int64_t n;
  int64_t nt;
  double eps_prog;
  /* optional (nt,6) table of barycentric gradients, rows (G00,G01,G10,G11,
   * G20,G21) = paths.py:105-110 bit for bit; built by pf_mesh_geometry_f64.
   * NULL: recomputed per visit. */
  const double *G;
  /* optional (nt,16) packed records, one 128-byte line per triangle (vertex
   * coordinates, the G row, area, vertex ids, tri_nbr; pf_mesh_pack_f64): a
   * tracer step is then one round trip for the geometry.  NULL: the arrays
   * above. */
  const double *pack;
} pf_mesh_t;

/* Path output: location l of path p is at index p*cap + l:
 *   kind 0 = ("vertex", i), 1 = ("edge", i, j, t); (x, y) the polyline point.
 * count[p] = number of locations (may exceed cap: then only the first cap
 * are written and the caller re-runs p with a larger buffer); status[p]:
 * 0 reached, 1 stuck, 2 max-steps-exceeded (paths.py:27-29); stuck[p] the
 * stuck vertex or -1. */
typedef struct {
  int8_t *kind;
  int32_t *i;
  int32_t *j;
  double *t;
  double *x;
  double *y;
  int64_t cap;
  int64_t *count;
  int32_t *status;
  int64_t *stuck;
  double *qx; /* scratch (npaths): nearest-vertex query point of stuck paths */
  double *qy;
} pf_paths_t;

/* Trace npaths paths: path p descends field field_of[p] (fields is
 * nfields x n FP64, row f = field f; field_of NULL = field 0) from
 * sources[p] toward targets[field_of[p]], at most step_cap state transitions
 * (settings.step_cap_factor * n).  Replaces triangle_descent (paths.py:292-307)
 * for a batch of sources; FP64 rounding follows the reference bit for bit. */
int pf_trace_batch_f64(const pf_mesh_t *mesh, const double *fields, const int64_t *targets,
                       const int64_t *sources, const int32_t *field_of, int64_t npaths,
                       int64_t step_cap, const pf_paths_t *out, pf_stream_t stream);
/* The same over fields in any 2-D layout: field f's value at vertex v is
 * fields[f * field_ld + v * vertex_ld].  pf_trace_batch_f64 is field_ld = n,
 * vertex_ld = 1; the (n, T) row-major output of the batched KL
 * (pf_batched_kl_*) is traced in place with field_ld = 1, vertex_ld = ldo, so
 * a rank tracing the paths of its own target columns copies
 * nothing. */
int pf_trace_fields_f64(const pf_mesh_t *mesh, const double *fields, int64_t field_ld,
                        int64_t vertex_ld, const int64_t *targets, const int64_t *sources,
                        const int32_t *field_of, int64_t npaths, int64_t step_cap,
                        const pf_paths_t *out, pf_stream_t stream);

/* ---- Path metric (paths.py:326-368) ----------------------------------------
 * A polyline instance p is one side of one compared pair: points
 * pts[2*(src_off[p] + i) + {0,1}], i < len[p].
 * pf_polyline_arc_f64: arc[src_off[p] + i] = sequential cumsum of np.hypot
 *   segment lengths (arc[.. + 0] = 0) and segmin[p] = the shortest positive
 *   segment (+inf if none; the default step is min over a pair / 4).
 * pf_polyline_resample_f64: resample_polyline (np.linspace + np.interp) into
 *   out[2*(out_off[p] + i) + {0,1}], i < cnt[p] = out_off[p+1] - out_off[p]
 *   points; the caller computes cnt[p] = max(2, ceil(total/step) + 1) like the
 *   reference, 0 to copy an instance with fewer than 2 points, -1 for a
 *   zero-length one (its first point).  total_out = out_off[ninst].
 * pf_hausdorff_pairs_f64: best_bits[q] = bits of the larger directed squared
 *   term between instances inst_a[q] and inst_b[q], each max_x min_y
 *   (dx*dx) + (dy*dy) over their resampled points (scipy cKDTree's 2-D
 *   arithmetic); the reference's path_hausdorff is its sqrt.  The search over y
 *   visits the source segments of y's instance (pts/arc/src_off/len/cnt as
 *   above) and measures only points next to x's projection on the segments
 *   that can hold the minimum: the exhaustive minimum, bit for bit.
 *   max_points >= every instance's resampled count. */
int pf_polyline_arc_f64(const double *pts, const int64_t *src_off, const int64_t *len,
                        int64_t ninst, double *arc, double *segmin, pf_stream_t stream);
int pf_polyline_resample_f64(const double *pts, const int64_t *src_off, const int64_t *len,
                             const double *arc, const int64_t *cnt, const int64_t *out_off,
                             int64_t ninst, int64_t total_out, double *out, pf_stream_t stream);
int pf_hausdorff_pairs_f64(const double *pts, const double *arc, const int64_t *src_off,
                           const int64_t *len, const int64_t *cnt, const double *rp,
                           const int64_t *out_off, const int64_t *inst_a, const int64_t *inst_b,
                           int64_t npairs, int64_t max_points, uint64_t *best_bits,
                           pf_stream_t stream);

/* ---- Wire formats (fileio.py:37-79, service/app.py:95-114; wire.cu) --------
 * pf_format_lines: line i of `kind` into slots[64*i ..] (lens[i] bytes):
 *   0 field CSV  f"{index0 + i},{v:.17g}\n"          (fileio.py:37-40)
 *   1 path CSV   f"{x:.17g},{y:.17g}\n", vals (n,2)   (fileio.py:72-75)
 *   2 JSON       json.dumps float (repr, NaN/Infinity) + ",\n    " but the last
 *   3 compact    repr + "," but the last; nonfinite[0] |= 1 on NaN/inf
 *   4 repr       float.__repr__        5 .17g   format(v, ".17g")
 * Digits are exact (big-integer dtoa modes 2 / 0, CPython's tie rules) and the
 * layout is CPython's format_float_short: byte-identical to the reference.
 * pf_pack_lines: out[offs[i] ..] = the lens[i] bytes of slot i (offs = the
 * exclusive scan of lens). */
int pf_format_lines(const double *vals, int64_t n, int kind, int64_t index0, char *slots,
                    int32_t *lens, uint32_t *nonfinite, pf_stream_t stream);
int pf_pack_lines(const char *slots, const int32_t *lens, const int64_t *offs, int64_t n,
                  char *out, pf_stream_t stream);

/* Fill the (nt,16) packed triangle records of pf_mesh_t.pack (128-byte aligned). */
int pf_mesh_pack_f64(const pf_mesh_t *mesh, double *pack, pf_stream_t stream);

/* Fill the (nt,6) barycentric-gradient table of pf_mesh_t.G (mesh->G ignored). */
int pf_mesh_geometry_f64(const pf_mesh_t *mesh, double *G, pf_stream_t stream);

/* triangle_gradient (paths.py:113-121) for a batch of triangle ids: out (ntri,2). */
int pf_triangle_gradient_f64(const pf_mesh_t *mesh, const double *vals, const int64_t *tris,
                             int64_t ntri, double *out, pf_stream_t stream);

/* np.hypot as the tracer evaluates it (glibc non-FMA kernel), elementwise. */
int pf_np_hypot_f64(const double *x, const double *y, int64_t n, double *out,
                    pf_stream_t stream);

/* ---- K11: the Poisson kernel P itself ---------------------
 * Replaces the preprocessing that produces the hot path's input:
 *   assemble_cotan      laplacian.py:91-134  -> pf_cotan_laplacian_f64
 *   factor_interior     laplacian.py:29-45, 137-141 (SuperLU of -Lc_II)
 *                       -> pf_nd_plan_build (host) + pf_mf_factor_level
 *   poisson_kernel      solvers.py:278-303 (k back-substitutions)
 *                       -> pf_mf_forward_level + pf_mf_backward_level
 *                          + pf_poisson_residual + pf_poisson_finalize
 *
 * Host symbolic plan (host pointers; opaque handle; the only allocating
 * entry points of the ABI).  Nested dissection of the interior vertices
 * (geometric bisection of the planar mesh), post-order fronts, scatter maps.
 * `nb_ptr/nb_idx` is the sorted vertex-neighbour CSR (mesh.py:151),
 * `is_boundary` the boundary mask (mesh.boundary_vertices), `leaf` the leaf
 * sub-domain size, `tile` the column tile of the solves.
 * pf_nd_plan_array copies the named array into `dst_host` (if not NULL) and
 * returns its length (-1: unknown name); names/dtypes: laplacian.py _I32/_I64. */
int pf_nd_plan_build(int64_t n, const double *xy_host, const int64_t *nb_ptr_host,
                     const int64_t *nb_idx_host, const uint8_t *is_boundary_host, int leaf,
                     int tile, void **plan_out);
void pf_nd_plan_free(void *plan);
int64_t pf_nd_plan_array(void *plan, const char *name, void *dst_host);
/* Host: the sorted vertex-neighbour CSR of a triangle mesh (mesh.py:151
 * `neighbors`), tri_host (nt,3) int64; nb_idx_host capacity 6*nt; *nnz_out
 * receives the entry count. */
int pf_vertex_neighbors(int64_t n, int64_t nt, const int64_t *tri_host, int64_t *nb_ptr_host,
                        int64_t *nb_idx_host, int64_t *nnz_out);
/* out_host[16]: n m k nodes levels f_total v_total nnz_l flops_factor
 * flops_solve max_f max_c max_r ntiles tile leaf */
int pf_nd_plan_stats(void *plan, double *out_host);

/* Device copy of the plan arrays (all device pointers). */
typedef struct {
  const int32_t *c0, *cn, *rn, *fn;  /* per node: first position, |C|, |R|, |C|+|R| */
  const int64_t *foff;               /* per node: offset of its f x f front in F     */
  const int32_t *ch_ptr, *ch_idx;    /* children CSR                                 */
  const int64_t *r_ptr;              /* R lists (original vertex ids)                */
  const int32_t *r_orig;
  const int64_t *relmap_off;         /* per node: its R rows inside the parent front */
  const int32_t *relmap;
  const int64_t *a_ptr, *a_dst, *a_src; /* A entries: F[a_dst] = -(src >= 0 ? off[src]
                                            : diag[-1-src])                          */
  const int64_t *b_ptr;              /* B entries: front row, column, off[] index    */
  const int32_t *b_row, *b_col;
  const int64_t *b_src;
  const int32_t *act_tile;           /* active (node, tile) items of the forward     */
  const int64_t *act_voff;           /* offset of each item's f x tile block [Y_C; V] */
  const int64_t *tile_item;          /* node * ntiles + tile -> item or -1           */
  const int32_t *perm_orig;          /* position -> original vertex id               */
  const int64_t *mt_off;             /* per node: Mt (f x round_up(c,16)) offset     */
  const int64_t *m_off;              /* per node: M = Mt^T (c x round_up(f,16))      */
  const int64_t *rowoff;             /* NULL: vertex v's output row at v * ldp; else
                                        the row-slab build's per-vertex offsets   */
  int64_t nodes, ntiles, k;
  int32_t tile;                      /* must be 64 */
  int32_t pad_;
} pf_mf_plan_t;

/* Cotangent Laplacian, bitwise laplacian.py:91-134: off[e] for every entry e
 * of the neighbour CSR (sum of the <= 2 corner halves 0.5*cot), diag[v] =
 * -(scipy row sum of off: first entry + numpy pairwise sum of the rest).
 * V (n,2) FP64, T (nt,3) int32 as stored.  *bad = min triangle index with a
 * zero cross product (0/pi angle, DegenerateGeometryError) or INT64_MAX;
 * nnz = nb_ptr[n]; callee initialises off and *bad (no host synchronisation). */
int pf_cotan_laplacian_f64(const double *V, const int32_t *T, int64_t nt, const int64_t *nb_ptr,
                           const int32_t *nb_idx, int64_t n, int64_t nnz, double *off,
                           double *diag, int64_t *bad, pf_stream_t stream);

/* Multifrontal Cholesky of A = -Lc_II, the nodes of one tree level: assemble
 * each front (A entries + children's update matrices, in child order), then
 * factor its |C| pivot columns in place (F[:, :c] = [L_CC; L_RC], F[c:, c:] =
 * the update matrix).  err[0] |= 1 on a non-positive pivot.  split = 0: one
 * CTA per front; split = 1 (few large fronts): assembly, pivot block, panel
 * TRSM and trailing update are each spread over CTAs (max_f / max_c bound the
 * level's fronts). */
int pf_mf_factor_level(const pf_mf_plan_t *plan, const double *off, const double *diag,
                       const int32_t *nodes, int64_t count, int32_t max_f, int32_t max_c,
                       int split, double *F, int32_t *err, pf_stream_t stream);

/* Explicit front inverses after the factorisation: Mt = [L_CC^{-1};
 * -L_RC L_CC^{-1}] (f x c, row stride round_up(c,16)) for items (node, 32
 * identity columns), then, if M != NULL, M = Mt^T (c x round_up(f,16)) for
 * `nodes` (the solves read Mt only).  Buffers must be zero-initialised (their
 * row pads stay 0).  Non-negative on
 * M-matrices: the solves below are sums of non-negative products. */
int pf_mf_inverse(const pf_mf_plan_t *plan, const double *F, const int32_t *item_node,
                  const int32_t *item_ct, int64_t count, const int32_t *nodes, int64_t nnodes,
                  double *Mt, double *M, pf_stream_t stream);

/* Forward solve of one level over its active (node, 64-column tile) items:
 * assemble W = [B_C; 0] + children's V (child order) into Wb at asm_woff,
 * then the item block O = Mt W_C + [0; W_R] = [Y_C; V] (items x 32-row
 * blocks g_rb).  O blocks live at plan->act_voff. */
int pf_mf_forward_level(const pf_mf_plan_t *plan, const double *Mt, const double *off,
                        const int32_t *asm_node, const int64_t *asm_item, const int64_t *asm_woff,
                        int64_t n_asm, const int32_t *g_node, const int64_t *g_item,
                        const int64_t *g_woff, const int32_t *g_rb, int64_t n_gemm, double *Wb,
                        double *O, pf_stream_t stream);

/* Backward solve of one level (levels top-down): X_C = Mt^T [Y_C; X_R] for items
 * (node, nb_rows-row block of C, 128-column blocks [cb0, cb1)), Y_C from O
 * (zero for tiles the forward never reached), X_R from P's rows, X_C into P
 * (rows by original vertex id; ldp a multiple of 64).  nb_rows in {8, 16, 32,
 * 64}; max_f / max_ncb bound the items' front sizes and column-block counts
 * (shared-memory sizing). */
int pf_mf_backward_level(const pf_mf_plan_t *plan, const double *Mt, const double *O,
                         const int32_t *item_node, const int32_t *item_rb,
                         const int32_t *item_cb0, const int32_t *item_cb1, int64_t count,
                         int32_t max_f, int32_t max_ncb, int32_t nb_rows, double *P,
                         int64_t ldp, pf_stream_t stream);

/* Gather table of the residual: nrow[e] = nb_idx[e] * ldp for an interior
 * neighbour entry, -1 - bcol[u] for a boundary one (built once per mesh). */
int pf_poisson_residual_table(const int32_t *nb_idx, int64_t nnz, const uint8_t *is_boundary,
                              const int32_t *bcol, int64_t ldp, const int64_t *rowoff,
                              int64_t *nrow, pf_stream_t stream);

/* residual = max |(Lc P)[v, j]| over the interior rows v = order[0..count)
 * and columns j < k with P's boundary rows taken as indicators (= |Lc_II P_IB
 * + Lc_IB|, solvers.py:292), before the clip; out_max[0] holds the max as
 * ordered FP64 bits.  `order` is best the plan's perm_orig (spatially compact
 * row groups share their neighbours' rows in cache).  Every row offset (rowoff,
 * nrow) is a multiple of ldp and names one of fewer than 2^31 rows. */
int pf_poisson_residual(const double *P, int64_t ldp, int64_t k, const int32_t *order,
                        int64_t count, const int64_t *rowoff, const int64_t *nb_ptr,
                        const int64_t *nrow, const double *off, const double *diag,
                        unsigned long long *out_max, pf_stream_t stream);

/* Boundary rows -> indicators of their column, pad columns -> 0, interior
 * entries in (-1e-12, 0) -> 0 (solvers.py:293-296); out_max[0] = max
 * |row sum - 1| (row_sum_error, :297) as ordered FP64 bits.  Fused K1: if H
 * != NULL, H[r] = sum_b c(P) log c(P) with c = max(., clamp), bitwise what
 * pf_row_negentropy_f64 returns, and min_out[0] (seeded +inf by the caller) =
 * min over P[:, :k]. */
int pf_poisson_finalize(double *P, int64_t ldp, int64_t row0, int64_t n, int64_t k,
                        const uint8_t *is_boundary, const int32_t *bcol, double clamp, double *H,
                        double *min_out, unsigned long long *out_max, pf_stream_t stream);

/* Finalize without a second pass over P (bare builds, no fused K1): the
 * residual pass also writes, per interior row r (P row index, rowoff / ldp)
 * and 512-column chunk c, row_part[r * ceil(k / PF_RESIDUAL_COLS) + c] = the
 * chunk's sum of the row's entries, and sets out_max[2] = 1 if any such entry
 * is negative (out_max: 3 words; [0] the residual as above).  Then
 * pf_poisson_finalize_rows writes the boundary indicator rows, zero pads and
 * out_max[0] = max |row sum - 1| over interior rows (sums over the chunks in
 * order).  When out_max[2] is set the clip of solvers.py:293-296 may apply:
 * run pf_poisson_finalize instead (it clips and re-sums). */
#define PF_RESIDUAL_COLS 512
int pf_poisson_residual_rows(const double *P, int64_t ldp, int64_t k, const int32_t *order,
                             int64_t count, const int64_t *rowoff, const int64_t *nb_ptr,
                             const int64_t *nrow, const double *off, const double *diag,
                             double *row_part, unsigned long long *out_max, pf_stream_t stream);
int pf_poisson_finalize_rows(double *P, int64_t ldp, int64_t row0, int64_t n, int64_t k,
                             const uint8_t *is_boundary, const int32_t *bcol,
                             const double *row_part, unsigned long long *out_max,
                             pf_stream_t stream);

/* ---- User-defined generators (divergence.py:42-56: FDivergence(name, f)) --
 * The reference evaluates any numpy generator f as q * f(p / q) per element
 * in dv_field / dv_at / dv_pair (:137-187).  The Python side traces f into a
 * scalar CUDA expression of `x` (arithmetic, comparisons, ternaries and CUDA
 * math functions only; _userf.py); pf_user_compile compiles it with NVRTC
 * (loaded at run time: `nvrtc_path_host` or libnvrtc.so.12) for sm_100a into
 * the two kernels below and, if `load`, loads them on the current device.
 * pf_dense_user_f64 is pf_dense_generic_f64 with f = the expression (same
 * settle, target zero, clamp flag, swap_order); pf_dense_user_at_f64 is
 * pf_dense_at_f64 likewise; pf_csr_user_f64 below pf_csr_generic_f64 likewise.
 * pf_user_cubin_size reports the cubin size (a
 * compile-only check needs no device). */
int pf_user_compile(const char *expr_host, const char *nvrtc_path_host, int load,
                    void **handle_host);
int pf_user_cubin_size(void *handle, int64_t *bytes_host);
int pf_user_free(void *handle);
int pf_dense_user_f64(void *handle, const double *P, int64_t ld, int64_t rows, int64_t k,
                      const double *tgt, const uint8_t *tmask, double clamp, int swap_order,
                      int64_t row0, int64_t target, const uint8_t *is_interior, double *out,
                      uint32_t *flags, pf_stream_t stream);
int pf_dense_user_at_f64(void *handle, const double *P, int64_t ld, int64_t rows, int64_t k,
                         const double *tgt, double clamp, int swap_order, int64_t row0,
                         int64_t target, const int64_t *queries, int64_t nq, double *out,
                         pf_stream_t stream);
/* pf_csr_generic_f64's union form (divergence.py:296-299) with f = the user
 * expression: prow is the target's raw dense row, cut the row cut. */
int pf_csr_user_f64(void *handle, const int64_t *indptr, const int32_t *indices,
                    const double *data, int64_t rows, const double *prow, int64_t p_local,
                    double cut, int64_t row0, const int64_t *queries, int64_t nq, double *out,
                    int64_t *ops, pf_stream_t stream);

/* ---- NCCL plumbing of the row-sharded path (SURVEY §8b pf_nccl_*, §8e) ---
 * The reference is single-process (dv_field, divergence.py:154-187, reads
 * the whole of `pk.dense`); with P partitioned into row slabs over the GPUs
 * of one box the path gains exactly these exchanges: the target row
 * P[t, :] broadcast from its owner (replaces the `dense[p]` read of
 * divergence.py:170 on the other ranks), the all-gather of finished field
 * slabs when the tracer needs the whole field (paths.py:292-307 reads
 * `field.values` at every vertex), and small max/min reductions of the
 * `clamped` flag word and the clamp <= 0 domain check (divergence.py:162-175),
 * so every rank returns the flags / raises exactly as the single process does.
 * NCCL is bound at run time: pf_nccl_load reuses the libnccl.so.2 already in
 * the process (torch's) or dlopens `path_host`.  The 128-byte unique id from
 * pf_nccl_unique_id is exchanged by the caller (rank 0 -> all) before
 * pf_nccl_comm_init.  Collectives are asynchronous on `stream`. */
#define PF_NCCL_ID_BYTES 128
enum { PF_T_U8 = 0, PF_T_I32 = 1, PF_T_I64 = 2, PF_T_F64 = 3 };
enum { PF_OP_SUM = 0, PF_OP_MAX = 1, PF_OP_MIN = 2 };
int pf_nccl_load(const char *path_host);
int pf_nccl_version(int *version_host);
int pf_nccl_unique_id(void *id_host);
int pf_nccl_comm_init(int nranks, const void *id_host, int rank, int device, void **comm_host);
int pf_nccl_comm_destroy(void *comm);
/* in place: buf (count elements) on every rank = root's */
int pf_nccl_broadcast(void *comm, void *buf, int64_t count, int dtype, int root,
                      pf_stream_t stream);
/* recv (nranks * count) = concatenation of every rank's send (count) */
int pf_nccl_all_gather(void *comm, const void *send, void *recv, int64_t count, int dtype,
                       pf_stream_t stream);
/* recv (count) = op over ranks of send (count); send == recv is in place */
int pf_nccl_all_reduce(void *comm, const void *send, void *recv, int64_t count, int dtype,
                       int op, pf_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* PATHFIELD_B200_H */
