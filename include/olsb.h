/* olsb.h — C ABI of the B200-native overlap-and-save (OLS) engine.
 *
 * This is the drop-in boundary for the reference's kernel plugin seam: the
 * reference picks a kernel module `K` at import (olsconv/backend.py:18-36) and
 * calls `K.dif_fwd_batch`, `K.dit_inv_batch` and `K.fused_c2c` with plain
 * arrays (olsconv/_kernels_nb.py:54-63, 265-285).  Each entry point below
 * replaces one of those calls; the Python host layer (paper_1910_01972_b200)
 * keeps the reference's validation and exceptions above it.
 *
 * Conventions (mirroring the reference's ownership model):
 *   - all pointers are DEVICE pointers; the caller allocates everything;
 *   - calls are stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *     default stream), never allocate, never synchronise the host;
 *   - complex data is interleaved (re, im): float2 when precision = 0
 *     (complex64), double2 when precision = 1 (complex128);
 *   - return 0 on success, a positive cudaError_t from the launch, or a
 *     negative OLSB_E_* code for a rejected argument (see olsb_error_string).
 *     Like the reference kernels they never raise: the host layer validates
 *     first and maps non-zero codes to exceptions.
 */
#ifndef OLSB_H_
#define OLSB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OLSB_OK 0
#define OLSB_E_BAD_LENGTH (-1)    /* n not a power of two in [4, 4096] */
#define OLSB_E_BAD_ARG (-2)       /* negative count, null pointer, ... */
#define OLSB_E_BAD_PRECISION (-3) /* precision not 0 (single) or 1 (double) */
#define OLSB_E_UNSUPPORTED (-4)   /* pp_kind not implemented by this build */
#define OLSB_E_GEOMETRY (-5)      /* l_eff / t0 / windows inconsistent */

#define OLSB_PP_NONE 0  /* postproc.py:15  KINDS[0] "none"  */
#define OLSB_PP_SCALE 1 /* postproc.py:15  KINDS[1] "scale" */
#define OLSB_PP_MAG2 2  /* postproc.py:15  KINDS[2] "magnitude_squared" */
#define OLSB_PP_DERIV 3 /* postproc.py:15  KINDS[3] "derivative": central
                           difference, needs the halo geometry (ols.py:137) */

/* Library version (major * 10000 + minor * 100 + patch). */
int olsb_version(void);

/* Human-readable text for a return code. */
const char* olsb_error_string(int code);

/* Number of complex elements of the engine ("device") spectrum layout per
 * filter for FFT length n (== n; the layout is a permutation of the
 * reference's bit-reversed order chosen for coalesced 16-byte loads). */
int olsb_spectra_dev_len(int n);

/* Forward transform of `rows` rows of n natural-order samples into the
 * reference's bit-reversed ("permuted") order, unscaled.
 * Replaces K.dif_fwd_batch(mat, tw) (_kernels_nb.py:54-57, used by
 * fft.fft_forward_permuted fft.py:112-117).  in == out is allowed. */
int olsb_dif_fwd_batch(const void* in, void* out, int rows, int n,
                       int precision, void* stream);

/* Inverse of olsb_dif_fwd_batch including the 1/n scale: bit-reversed in,
 * natural out.  Replaces K.dit_inv_batch(mat, twc) (_kernels_nb.py:60-63,
 * fft.fft_inverse_permuted fft.py:120-125).  in == out is allowed. */
int olsb_dit_inv_batch(const void* in, void* out, int rows, int n,
                       int precision, void* stream);

/* Filter-bank spectra: zero-pad each of the n_fil rows of `taps` (n_fil x m,
 * row-major, complex) to n and forward-transform it with the same in-register
 * FFT the fused kernel uses.  Writes the reference's permuted layout
 * (n_fil x n, may be NULL) and/or the engine layout (n_fil x
 * olsb_spectra_dev_len(n), may be NULL).
 * Replaces the pad + K.dif_fwd_batch of transform_filters (ols.py:195-199). */
int olsb_filter_spectra_c2c(const void* taps, int n_fil, int m, int n,
                            void* spectra_perm, void* spectra_dev,
                            int precision, void* stream);

/* Convert spectra already in the reference's permuted layout (e.g. a
 * FilterSet whose cache was filled elsewhere) into the engine layout. */
int olsb_spectra_perm_to_dev(const void* spectra_perm, int n_fil, int n,
                             void* spectra_dev, int precision, void* stream);

/* The fused OLS engine (the paper's Algorithm 2): for every segment s in
 * [seg_lo, seg_hi): gather the zero-extended window x[s*l_eff + win_off, +n),
 * forward FFT, then for every filter f: multiply by spectra_dev[f], inverse
 * FFT, post-process, and write out[f, s*l_eff + j] = y[t0 + j] for
 * j < min(l_eff, n_s - s*l_eff).
 * Replaces K.fused_c2c(x, spectra, tw, twc, m, origin, l_eff, t0, win_off,
 * seg_lo, seg_hi, pp_kind, pp_c, h0, out, buf, spec_buf)
 * (_kernels_nb.py:265-285); scratch lives in shared memory, twiddles are
 * generated on device.  Extra arguments for sharded signals:
 *   x        points at global sample x_base (x[i] is sample x_base + i); the
 *            caller guarantees every in-range sample a segment reads is
 *            present (its shard plus the (m-1)-sample halo);
 *   n_s      GLOBAL signal length (zero extension outside [0, n_s));
 *   out      row f, global sample g lives at out[f*out_ld + g - out_base].
 * Global segment indices keep results bit-identical for any split. */
int olsb_fused_c2c(const void* x, int64_t x_base, int64_t n_s,
                   const void* spectra_dev, int n_fil, int n, int m,
                   int origin, int64_t l_eff, int t0, int64_t win_off,
                   int64_t seg_lo, int64_t seg_hi, int pp_kind, double pp_c,
                   void* out, int64_t out_ld, int64_t out_base,
                   int precision, void* stream);

/* Output-range form of olsb_fused_c2c for sharded and streamed signals
 * (no reference counterpart): writes outputs [g_lo, g_hi) of every filter
 * for the plain (no post-processing halo) geometry of taps of length m with
 * output origin `origin`.  The engine covers the range with its own segment
 * grid, anchored at global sample 0, so results are bit-identical for any
 * partition of [0, n_s) into ranges.  `x`, `x_base`, `n_s`, `out`, `out_ld`,
 * `out_base` as in olsb_fused_c2c; the input samples a call reads are
 * [x_lo, x_hi) of olsb_input_extent (clipped to [0, n_s)).  pp_kind
 * OLSB_PP_MAG2 selects the |y|^2 epilogue of olsb_fused_c2c_abs2: `out` is
 * then REAL.  OLSB_PP_DERIV uses the halo geometry (olsb_input_extent_pp). */
int olsb_fused_c2c_range(const void* x, int64_t x_base, int64_t n_s,
                         const void* spectra_dev, int n_fil, int n, int m,
                         int origin, int64_t g_lo, int64_t g_hi, int pp_kind,
                         double pp_c, void* out, int64_t out_ld,
                         int64_t out_base, int precision, void* stream);

/* The fused engine's |y|^2 epilogue (postproc "magnitude_squared" on the
 * complex path): same arguments as olsb_fused_c2c, `out` is REAL
 * (float/double, n_fil x out_ld).  Replaces K.fused_c2c_abs2(x, spectra, tw,
 * twc, m, origin, l_eff, t0, win_off, seg_lo, seg_hi, h0, out, buf,
 * spec_buf) (_kernels_nb.py:288-309). */
int olsb_fused_c2c_abs2(const void* x, int64_t x_base, int64_t n_s,
                        const void* spectra_dev, int n_fil, int n, int m,
                        int origin, int64_t l_eff, int t0, int64_t win_off,
                        int64_t seg_lo, int64_t seg_hi, void* out,
                        int64_t out_ld, int64_t out_base, int precision,
                        void* stream);

/* The fused real path: real signal `x`, real taps (their complex spectra in
 * the engine layout, from olsb_filter_spectra_c2c of the taps with zero
 * imaginary parts), REAL output rows.  Two consecutive segments of the
 * engine grid are transformed together as one complex segment (re: segment
 * 2k, im: segment 2k+1): with real taps the complex convolution separates
 * exactly into the two real ones, so no packed-real split/merge is needed.
 * pp_kind: none, scale or magnitude_squared (v*v, fused_r2r pp_kind 2).
 * Arguments as olsb_fused_c2c.  Replaces K.fused_r2r(x, spectra, tw_half,
 * tw_half_conj, pack_tw, pack_tw_conj, m, origin, l_eff, t0, win_off,
 * seg_lo, seg_hi, pp_kind, pp_c, h0, out, rbuf, z_scr, bins, prod)
 * (_kernels_nb.py:312-337). */
int olsb_fused_r2r(const void* x, int64_t x_base, int64_t n_s,
                   const void* spectra_dev, int n_fil, int n, int m,
                   int origin, int64_t l_eff, int t0, int64_t win_off,
                   int64_t seg_lo, int64_t seg_hi, int pp_kind, double pp_c,
                   void* out, int64_t out_ld, int64_t out_base,
                   int precision, void* stream);

/* Output-range form of olsb_fused_r2r (sharded / streamed real signals);
 * reads the input extent of olsb_input_extent_r2r. */
int olsb_fused_r2r_range(const void* x, int64_t x_base, int64_t n_s,
                         const void* spectra_dev, int n_fil, int n, int m,
                         int origin, int64_t g_lo, int64_t g_hi, int pp_kind,
                         double pp_c, void* out, int64_t out_ld,
                         int64_t out_base, int precision, void* stream);

/* Exact mode: the reference's arithmetic, bit for bit.  Same arguments as
 * olsb_fused_c2c plus `tw`, the reference's twiddle table (n/2 complex
 * values e^{-2 pi i j / n} rounded to the precision, fft.py:70-78; device
 * memory), i.e. the `tw` argument of K.fused_c2c (_kernels_nb.py:266).  The
 * engine then keeps the reference's segment grid (no 32-alignment), computes
 * every butterfly as the reference's explicit complex product by the table
 * entry (dif_fwd / dit_inv, _kernels_nb.py:11-51, twc = conj(tw)) with
 * non-contracting IEEE operations, and applies 1/n and pp_c where dit_inv
 * and _store do.  With spectra from olsb_filter_spectra_c2c_ref, outputs are
 * bit-identical to the reference's fp32 (fp64) fused_c2c.  pp_kind: none or
 * scale. */
int olsb_fused_c2c_ref(const void* x, int64_t x_base, int64_t n_s,
                       const void* spectra_dev, int n_fil, int n, int m,
                       int origin, int64_t l_eff, int t0, int64_t win_off,
                       int64_t seg_lo, int64_t seg_hi, int pp_kind,
                       double pp_c, const void* tw, void* out, int64_t out_ld,
                       int64_t out_base, int precision, void* stream);

/* Exact-mode |y|^2 epilogue: replaces K.fused_c2c_abs2(x, spectra, tw, twc,
 * ...) (_kernels_nb.py:288-309) bit for bit. */
int olsb_fused_c2c_abs2_ref(const void* x, int64_t x_base, int64_t n_s,
                            const void* spectra_dev, int n_fil, int n, int m,
                            int origin, int64_t l_eff, int t0, int64_t win_off,
                            int64_t seg_lo, int64_t seg_hi, const void* tw,
                            void* out, int64_t out_ld, int64_t out_base,
                            int precision, void* stream);

/* Exact-mode filter spectra: the pad + K.dif_fwd_batch(mat, tw) of
 * transform_filters (ols.py:195-199, _kernels_nb.py:54-57) with the
 * reference's arithmetic; same outputs as olsb_filter_spectra_c2c. */
int olsb_filter_spectra_c2c_ref(const void* taps, int n_fil, int m, int n,
                                const void* tw, void* spectra_perm,
                                void* spectra_dev, int precision,
                                void* stream);

/* Input samples [*x_lo, *x_hi) that olsb_fused_c2c_range(g_lo, g_hi) reads
 * (before clipping to [0, n_s)): the shard plus its halos. */
int olsb_input_extent(int n, int m, int origin, int64_t g_lo, int64_t g_hi,
                      int64_t* x_lo, int64_t* x_hi);

/* Input extent of a range call with post-processing pp_kind (mode 0: the
 * c2c range entry, 1: the r2r one).  OLSB_PP_DERIV ranges use the halo
 * geometry (t0 = m, L = n - m - 1: each output's neighbours lie in its own
 * segment), which reads one more sample on each side. */
int olsb_input_extent_pp(int mode, int n, int m, int origin, int pp_kind,
                         int64_t g_lo, int64_t g_hi, int64_t* x_lo,
                         int64_t* x_hi);

/* Input samples [*x_lo, *x_hi) that olsb_fused_r2r_range(g_lo, g_hi) reads:
 * the windows of whole segment pairs (both halves of a pair are always
 * transformed together, which keeps results independent of the split). */
int olsb_input_extent_r2r(int n, int m, int origin, int64_t g_lo,
                          int64_t g_hi, int64_t* x_lo, int64_t* x_hi);

/* Tuning knob (not in the reference): number of filters processed per work
 * item (0 = all).  Smaller chunks cut the tail of the last wave at the cost
 * of recomputing the segment's forward FFT per chunk. */
int olsb_set_filter_chunk(int filters_per_item);

/* Stream-ordered strided copy (cudaMemcpy2DAsync, direction inferred from
 * the pointers; `kind` is reserved and must be 0).  Used by the streaming
 * host-memory path of convolve() to move per-chunk (n_fil x chunk) output
 * tiles into the caller's (n_fil x n_s) pinned host array. */
int olsb_copy2d_async(void* dst, int64_t dst_pitch_bytes, const void* src,
                      int64_t src_pitch_bytes, int64_t width_bytes,
                      int64_t height, int kind, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* OLSB_H_ */
