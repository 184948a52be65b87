/*
 * srpb.h -- C ABI of the B200-native SRP-map hot path (libsrpb.so).
 *
 * The reference (srpfast, arXiv 2012.09499) is pure Python/numpy; it has no
 * FFI of its own.  Its drop-in boundary is the Python function API of
 * srpfast.spectral / srpfast.srp (re-exported at pkg/src/srpfast/__init__.py
 * :43-66).  These entry points are what that API binds, one per numpy
 * "kernel" of the reference.  The Python mirror of the
 * reference API (paper_2012_09499_b200/spectral.py, srp.py) calls them via
 * ctypes; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - every pointer argument is a DEVICE pointer unless stated otherwise;
 *    complex data is interleaved (re, im) float pairs ("complex64");
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default);
 *  - calls are asynchronous and stream ordered; nothing is allocated or
 *    freed, no global mutable state is kept (re-entrant);
 *  - return 0 on success, <0 invalid argument (nothing launched),
 *    >0 a cudaError_t from the launch; srpb_last_error() gives a
 *    thread-local message for the last failing call on this thread.
 *
 * Shapes: F frames, M channels, Kb one-sided bins (DC kept, Nyquist dropped,
 * spectral.py:70-73), P pairs in canonical order (geometry.py:141-176),
 * J candidates, T_pad = padded total lattice samples (multiple of 32).
 */
#ifndef SRPB_H
#define SRPB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SRPB_WEIGHT_PHAT 0
#define SRPB_WEIGHT_IDENTITY 1

/* Version of this ABI (bumped on any signature change). */
int srpb_abi_version(void);

/* Message of the last failing call on the calling thread ("" if none). */
const char* srpb_last_error(void);

/* Kernels launched by the calling thread's last srpb_gcc_phat /
 * srpb_gcc_phat_split16 (1 for the frame-resident speculative pass with the
 * relative PHAT floor, else 2).  Bookkeeping for launch counts (ABI v13). */
int srpb_last_gcc_kernels(void);

/*
 * Plan build on the device: candidate TDOAs (geometry.build_tdoa_table,
 * geometry.py:365-398; near field |q - p_m| - |q - p_m'| over c, far field
 * (p_m - p_m') . r / c) and their splits, fp64 in the reference's operation
 * order: conventional x = (omega1 tau) period / 2pi -> conv_ti = rint(x) mod
 * period, conv_tf = x - rint(x); sinc x = tau / sample_period -> sx_i, sx_f
 * (srp.py:310).  Layout [P, J] (candidates fastest); tau [J, P] optional.
 *   mic_pos [M, 3], points [J, 3] float64 (unit directions for far field)
 *   bounds [P] float64 (pair distance / c); *violation set to 1 when some
 *   |tau| > bound + slack (the reference raises AssertionError)
 * Any of the (conv_ti, conv_tf), (sx_i, sx_f), tau outputs may be NULL.
 */
int srpb_tdoa_split(const double* mic_pos, int M, const double* points, int J,
                    const int32_t* pair_m, const int32_t* pair_mp, int P, int far_field,
                    double speed_of_sound, double omega1, int period, double sample_period,
                    const double* bounds, double slack, int32_t* conv_ti, float* conv_tf,
                    int32_t* sx_i, float* sx_f, double* tau, int* violation, void* stream);

/*
 * K0 STFT on the device.  Replaces spectral.stft_analyze (spectral.py:185-215)
 * with FrameSpec's framing and window (:35-99): frame f covers samples
 * [f hop, f hop + N), periodic sqrt-Hann (window 0) or rectangular (1),
 * one-sided bins 0..N/2-1 (DC kept, Nyquist dropped).
 *   x [M, L] float32 audio; N = frame_length even: powers of two <= 8192
 *   take a shared-memory FFT, other N <= 4096 a direct DFT;
 *   F = (L - N) / hop + 1 (trailing samples dropped)
 *   Y [F, M, N/2] complex64 out (the layout srpb_gcc_phat / srpb_gcc_floor /
 *   srpb_lattice_from_spectra read)
 */
int srpb_stft(const float* x, int M, int L, int frame_length, int hop, int window, int F,
              float* Y, void* stream);

/*
 * K1 GCC-PHAT cross-spectra for F frames.
 * Replaces spectral.cross_spectrum (pkg/src/srpfast/spectral.py:218-285),
 * batched over frames.
 *   Y        [F, M, Kb] complex64 STFT frames
 *   pair_m, pair_mp [P] int32 channel indices (index_m, index_m_prime);
 *            M <= 64, P <= 2016
 *   weighting SRPB_WEIGHT_PHAT or SRPB_WEIGHT_IDENTITY
 *   floor_rel adaptive floor factor (DEFAULT_PHAT_FLOOR_REL = 1e-12,
 *             spectral.py:31-32) used when abs_floor <= 0
 *   abs_floor explicit floor (> 0) or <= 0 for the adaptive floor
 *   Psi      [F, P, Kb] complex64 out: psi = raw / max(|raw|, floor), 0 where
 *            raw == 0 (phat) or psi = raw (identity)
 *   floor_out [F] float64 out (may be NULL): the floor applied per frame
 *            (0 under identity weighting)
 */
int srpb_gcc_phat(const float* Y, int F, int M, int Kb, const int32_t* pair_m,
                  const int32_t* pair_mp, int P, int weighting, double floor_rel,
                  double abs_floor, float* Psi, double* floor_out, void* stream);

/*
 * Same cross-spectra (PHAT only) written as the fp16 operand split of the
 * tensor-core K2 -- hi = fp16(s psi), lo = fp16(s psi - hi), s = split_scale
 * (a power of two) -- into Psi_hi / Psi_lo [F, 2 P Kb] (K index p 2Kb + 2k +
 * {re, im}, the layout srpb_f16_split gives the float view of Psi); Psi
 * [F, P, Kb] complex64 is written too when non-NULL.  Kb even; Y and Psi
 * 16-byte, Psi_hi / Psi_lo 8-byte aligned.
 */
int srpb_gcc_phat_split16(const float* Y, int F, int M, int Kb, const int32_t* pair_m,
                          const int32_t* pair_mp, int P, int weighting, double floor_rel,
                          double abs_floor, float* Psi, void* Psi_hi, void* Psi_lo,
                          float split_scale, double* floor_out, void* stream);

/*
 * K1a: the per-frame PHAT floor alone, floor_rel * sqrt(mean_{p,k} |raw|^2)
 * accumulated in fp64 (spectral.py:268-275), and per-frame range flags;
 * feeds srpb_lattice_from_spectra.
 *   floor_out [F] float64 out or NULL
 *   clean_out [F] int32 out or NULL: 1 when every |y_m[k]|^2 (fp32) of the
 *             frame is 0 or inside (1e-30, 1e30) -- the fused lattice then
 *             skips its per-bin range test (results are identical)
 */
int srpb_gcc_floor(const float* Y, int F, int M, int Kb, const int32_t* pair_m,
                   const int32_t* pair_mp, int P, double floor_rel, double* floor_out,
                   int32_t* clean_out, void* stream);

/*
 * K2 conventional SRP maps (harmonic bins w_k = k w_1).
 * Replaces srp.srp_conventional_frames (srp.py:391-429) incl. the steering
 * phases of srp._phase_matrix (srp.py:350-373), generated on the fly:
 *   SRP[f, j] = sum_p 2 Re sum_k psi[f,p,k] e^{j k w_1 tau[j,p]}
 * with w_1 tau[j,p] / 2pi = (tau_i[p,j] + tau_f[p,j]) / period.
 *   Psi      [F, P, Kb] complex64
 *   tau_i    [P, J] int32, tau_f [P, J] float32 (|tau_f| <= 1/2): host split
 *            of x = w_1 tau period / 2pi (fp64) into rint + fraction
 *   period   integer period of the phase (the frame length N = 2 Kb)
 *   maps     [F, J] float32 out, or NULL (argmax only)
 *   keys     [F] uint64 in/out, or NULL: running packed argmax keys
 *            (srpb_argmax_keys_reset first); see srpb_keys_to_index
 */
int srpb_conventional(const float* Psi, int F, int P, int Kb, int period,
                      const int32_t* tau_i, const float* tau_f, int J, float* maps,
                      unsigned long long* keys, void* stream);

/*
 * K2g conventional SRP maps for arbitrary (non-harmonic) bins: the dense
 * exp branch of srp._phase_matrix (srp.py:366-367), phases in fp64.
 *   omega [Kb] float64 rad/s, tau [J, P] float64 seconds
 */
int srpb_conventional_general(const float* Psi, int F, int P, int Kb,
                              const double* omega, const double* tau, int J,
                              float* maps, unsigned long long* keys, void* stream);

/*
 * Lattice twiddles e^{j w_k n T} for the half-lags n in [0, L] (lag -n is the
 * conjugate), fp64 phases rounded to fp32.  Signal-independent table of
 * srp.build_gcc_lattice (srp.py:235-236).
 *   omega [Kb] float64, tw [Kb, Hs] complex64 out (bin-major), Hs = L+1
 *   rounded up to a multiple of 16, columns n > L zero
 */
int srpb_lattice_twiddles(const double* omega, int Kb, double sample_period, int L,
                          float* tw, void* stream);

/*
 * K3 lattice GCC samples for F frames.
 * Replaces srp.build_gcc_lattice (srp.py:201-247):
 *   Xi[f, off[p] + n + reach[p]] = 2 Re sum_k psi[f,p,k] e^{j w_k n T}
 *   with tw [Kb, Hs] from srpb_lattice_twiddles (lag -n via conjugation)
 *   for n in [-reach[p], reach[p]], reach[p] = N_p + n_aux.
 *   off [P+1] int32 prefix sums of 2 reach + 1; pad columns [off[P], T_pad)
 *   are written as 0.
 *   Xi [F, T_pad] float32 out
 */
int srpb_lattice(const float* Psi, int F, int P, int Kb, const float* tw, int L,
                 const int32_t* off, const int32_t* reach, int T_pad, float* Xi,
                 void* stream);

/*
 * K1b+K3 fused: lattice GCC samples straight from the channel spectra.
 * Same output as srpb_gcc_phat followed by srpb_lattice, but the GCC-PHAT
 * cross-spectra are formed in the lattice kernel's staging pass and never
 * stored (spectral.cross_spectrum spectral.py:218-285 feeding
 * srp.build_gcc_lattice srp.py:201-247).
 *   PHAT floor: floors [F] float64 (srpb_gcc_floor), or NULL with
 *   abs_floor > 0 (explicit floor), or NULL with abs_floor <= 0: the
 *   relative floor floor_rel * sqrt(mean |raw|^2) is applied speculatively --
 *   the lattice runs unfloored while accumulating per-(frame, pair) |raw|^2
 *   statistics, and a fix-up pass recomputes exactly every frame in which a
 *   bin could fall below the floor or a power leaves the fast path's range
 *   (identical results, no floor pass).  Ignored for identity weighting.
 *   clean [F] int32 (srpb_gcc_floor) or NULL (every bin range-tested).
 *   spec_scratch: 12 F P bytes for the speculative floor's statistics, or
 *   NULL (then allocated stream-ordered per call).
 *   tw 16-byte aligned.
 *   Xi [F, T_pad] float32 out and/or Xi_hi, Xi_lo [F, T_pad]: its operand
 *   split for the tensor-core K4 -- split_scale == 0: tf32 floats
 *   (hi = rna(Xi), lo = rna(Xi - hi), srpb_interp_tc); split_scale a power
 *   of two: fp16 of split_scale * Xi (srpb_interp_tc16).
 */
int srpb_lattice_from_spectra(const float* Y, int F, int M, int Kb, const int32_t* pair_m,
                              const int32_t* pair_mp, int P, int weighting, const double* floors,
                              double abs_floor, const int32_t* clean, const float* tw, int L,
                              const int32_t* off, const int32_t* reach, int T_pad, float* Xi,
                              void* Xi_hi, void* Xi_lo, float split_scale, double floor_rel,
                              void* spec_scratch, void* stream);

/*
 * Tensor-core form of the same step (replaces spectral.cross_spectrum ->
 * srp.build_gcc_lattice, spectral.py:218-285 + srp.py:201-247, like the
 * entry above): the lattice twiddles do not depend on the pair, so all
 * (frame, pair) rows form one GEMM  C[f P + p, c] = sum_k Re(psi e^{j w_k n T})
 * over lag slots c = n + L, psi generated by PHAT on the fly (3xFP16,
 * tcgen05).  Used for PHAT with the relative floor (speculative + fix-up) and
 * the fp16 split output when Kb % 32 == 0, Kb >= 64 and
 * srpb_lattice_tc_cols(L) <= 1024 (beyond 64 slots the lag slots run in passes
 * of up to 128, each regenerating its rows' psi; frame_counters is then
 * ignored and the fix-up kernel runs after the passes); any other call
 * behaves exactly like srpb_lattice_from_spectra.  Arguments as there, plus
 *   tc_b_hi, tc_b_lo  [srpb_lattice_tc_cols(L), 2 Kb] fp16 from
 *                     srpb_lattice_tc_twiddles (both NULL: SIMT path).
 *   frame_counters    [F] int32, zero on entry and left zero (or NULL): the
 *                     tensor-core kernel then runs the speculative-floor
 *                     fix-up itself -- the CTA completing a frame tests it and
 *                     redoes it exactly if flagged -- instead of a second
 *                     kernel.  Calls sharing the counters must be stream-ordered.
 */
int srpb_lattice_from_spectra_tc(const float* Y, int F, int M, int Kb, const int32_t* pair_m,
                                 const int32_t* pair_mp, int P, int weighting,
                                 const double* floors, double abs_floor, const int32_t* clean,
                                 const float* tw, int L, const int32_t* off, const int32_t* reach,
                                 int T_pad, float* Xi, void* Xi_hi, void* Xi_lo, float split_scale,
                                 double floor_rel, void* spec_scratch, const void* tc_b_hi,
                                 const void* tc_b_lo, int* frame_counters, void* stream);

/* Lag slots of the tensor-core lattice: 2L + 1 rounded up to 16. */
int srpb_lattice_tc_cols(int L);

/* 1 when srpb_lattice_from_spectra_tc takes the tensor-core path for this
 * shape (PHAT, relative floor, fp16 split output assumed), else 0. */
int srpb_lattice_tc_supported(int M, int P, int Kb, int L, int T_pad);

/*
 * Its B operand: row c (lag n = c - L, zero rows past 2L), K = 2 Kb
 * interleaved (cos, -sin)(omega[k] n T) x 2^14, fp16 hi/lo split (fp64
 * phases as srpb_lattice_twiddles).  b_hi, b_lo [srpb_lattice_tc_cols(L), 2 Kb].
 */
int srpb_lattice_tc_twiddles(const double* omega, int Kb, double sample_period, int L, void* b_hi,
                             void* b_lo, void* stream);

/*
 * Sinc interpolation table W[j, off[p] + n + reach[p]] = sinc(x[j,p] - n),
 * exact 1/0 at integer arguments (srp._sinc_kernel srp.py:250-261,
 * srp.precompute_sinc_table srp.py:287-317), x = tau / T split on the host in
 * fp64 into sx_i [P, J] int32 = rint(x) and sx_f [P, J] float32 = x - rint(x).
 *   W [J, T_pad] float32 out (pad columns 0)
 */
int srpb_sinc_table(const int32_t* sx_i, const float* sx_f, int J, int P,
                    const int32_t* off, const int32_t* reach, int T_pad, float* W,
                    void* stream);

/*
 * K4 approximate SRP maps from lattice samples: maps = Xi W^T.
 * Replaces srp.srp_approx (srp.py:320-347), batched over frames.
 *   W [J, T_pad] float32 (srpb_sinc_table), Xi [F, T_pad] float32
 *   maps [F, J] float32 out or NULL; keys [F] as in srpb_conventional
 */
int srpb_interp(const float* W, const float* Xi, int F, int J, int T_pad, float* maps,
                unsigned long long* keys, void* stream);

/*
 * K4f approximate maps with the sinc weights generated on the fly from the
 * split TDOAs (no stored W; the only option when J x T_pad does not fit,
 * e.g. C4's 361 GB table).  Same arithmetic as srpb_sinc_table + srpb_interp.
 */
int srpb_interp_onthefly(const int32_t* sx_i, const float* sx_f, int P,
                         const int32_t* off, const int32_t* reach, const float* Xi,
                         int F, int J, int T_pad, float* maps, unsigned long long* keys,
                         void* stream);

/*
 * Operand split for the 3xTF32 tensor-core kernels: hi = tf32(x),
 * lo = tf32(x - hi) (round to nearest), elementwise over n floats
 * (n % 4 == 0, 16-byte aligned pointers).
 */
int srpb_tf32_split(const float* x, size_t n, float* hi, float* lo, void* stream);

/*
 * K2tc conventional maps on the tcgen05 tensor cores (kind::tf32, 3xTF32):
 * same result as srpb_conventional (srp.py:391-429).  The steering phases
 * are generated on the fly into shared memory; Psi enters pre-split
 * (srpb_tf32_split of the float view of Psi [F, P, Kb]).  Requires
 * Kb % 16 == 0.  kb_per_group = 32-element K blocks accumulated per TMEM
 * buffer before folding into the fp32 totals (the tensor core's accumulation
 * is not round-to-nearest; short groups bound its drift, default 4).
 */
int srpb_conventional_tc(const float* psi_hi, const float* psi_lo, int F, int P, int Kb,
                         int period, const int32_t* tau_i, const float* tau_f, int J,
                         float* maps, unsigned long long* keys, int kb_per_group,
                         void* stream);

/*
 * K4tc approximate maps on the tensor cores (srp.py:320-347): TMA-fed
 * W_hi/W_lo [J, T_pad] and Xi_hi/Xi_lo [F, T_pad] (srpb_tf32_split),
 * kb_per_group = 32-column K blocks per TMEM buffer.
 */
int srpb_interp_tc(const float* w_hi, const float* w_lo, const float* xi_hi, const float* xi_lo,
                   int F, int J, int T_pad, float* maps, unsigned long long* keys,
                   int kb_per_group, void* stream);

/*
 * Dynamic scheduling and in-kernel argmax finish (srpb_conventional_tc16,
 * srpb_interp_tc16, srpb_interp_tc16_onthefly): done_counter points to two
 * zero-initialised unsigned ints -- [0] CTAs finished, [1] the work-item
 * cursor from which CTAs (pairs) take their next tile once their first is
 * done.  The kernel's last CTA resets both to 0; with argmax_out [F] int32
 * also non-NULL it first decodes keys into argmax_out (as
 * srpb_keys_to_index) and resets keys to 0, so a caller that keeps keys and
 * the counters zero-initialised between calls needs neither
 * srpb_argmax_keys_reset nor srpb_keys_to_index.  done_counter NULL: static
 * round-robin tiles.  Calls sharing keys / counter buffers must be
 * stream-ordered.
 */

/*
 * 3xFP16 operand split: hi = fp16(scale x), lo = fp16(scale x - hi), scale a
 * power of two keeping |scale x| < 65504 (fp16 has tf32's 11-bit
 * significand: the split is as exact as the tf32 one).
 *   x [n] float32; hi, lo [n] fp16 out
 */
int srpb_f16_split(const float* x, size_t n, float scale, void* hi, void* lo, void* stream);

/*
 * K2 on the tensor cores in 3xFP16 (kind::f16, twice the kind::tf32 rate);
 * same maps as srpb_conventional_tc.  psi_hi/psi_lo [F, 2 P Kb] fp16 split of
 * Psi prescaled by psi_scale (power of two, |psi_scale psi| < 65504: 2^14 for
 * PHAT cross-spectra); the steering phases are generated prescaled by 2^14.
 * Kb % 32 == 0.
 */
int srpb_conventional_tc16(const void* psi_hi, const void* psi_lo, float psi_scale, int F, int P,
                           int Kb, int period, const int32_t* tau_i, const float* tau_f, int J,
                           float* maps, unsigned long long* keys, int kb_per_group,
                           int32_t* argmax_out, unsigned int* done_counter, void* stream);

/*
 * K4 on the tensor cores in 3xFP16; same maps as srpb_interp_tc.
 *   w_hi/w_lo [J, T_pad] fp16 split of W prescaled by w_scale;
 *   xi_hi/xi_lo [F, T_pad] fp16 split of Xi prescaled by xi_scale
 *   (powers of two); T_pad % 8 == 0.
 */
int srpb_interp_tc16(const void* w_hi, const void* w_lo, float w_scale, const void* xi_hi,
                     const void* xi_lo, float xi_scale, int F, int J, int T_pad, float* maps,
                     unsigned long long* keys, int kb_per_group, int32_t* argmax_out,
                     unsigned int* done_counter, void* stream);

/*
 * K4 on the tensor cores in 3xFP16 without a stored W: the sinc weights are
 * generated in tensor memory by the epilogue warps from the sinc split (the
 * same arithmetic as srpb_sinc_table + srpb_f16_split with w_scale 2^14, so
 * the maps equal srpb_interp_tc16's bit for bit), removing W's HBM footprint
 * (J * T_pad * 8 bytes) and traffic.
 *   sx_i, sx_f [P, J], off [P+1], reach [P] as for srpb_sinc_table;
 *   xi_hi/xi_lo [F, T_pad] fp16 split of xi_scale * Xi; T_pad % 8 == 0.
 */
int srpb_interp_tc16_onthefly(const int32_t* sx_i, const float* sx_f, int P, const int32_t* off,
                              const int32_t* reach, const void* xi_hi, const void* xi_lo,
                              float xi_scale, int F, int J, int T_pad, float* maps,
                              unsigned long long* keys, int kb_per_group, int32_t* argmax_out,
                              unsigned int* done_counter, void* stream);

/*
 * K5 per-frame argmax, lowest index on ties (srp.argmax_candidate,
 * srp.py:107-109) over stored maps [F, J]: folds into keys [F].
 */
int srpb_argmax(const float* maps, int F, int J, unsigned long long* keys, void* stream);

/*
 * K5d argmax over float64 maps [F, J] (maps built on the host, e.g. an
 * SrpMap whose values came from numpy): idx[f] int32 = first maximum,
 * exactly numpy.argmax (srp.py:109).
 */
int srpb_argmax_f64(const double* maps, int F, int J, int32_t* idx, void* stream);

/* keys[f] = 0 for f < F (the identity of the packed-key max). */
int srpb_argmax_keys_reset(unsigned long long* keys, int F, void* stream);

/* idx[f] = candidate index held by keys[f] (int32). */
int srpb_keys_to_index(const unsigned long long* keys, int F, int32_t* idx, void* stream);

/*
 * Strided host -> device copy of `rows` rows of `row_bytes` (one DMA
 * request, cudaMemcpy2DAsync): a frame range of multichannel audio [M, L]
 * is a column block of the host array.  Pinned src for an async copy.
 */
int srpb_copy_rows_h2d(void* dst, size_t dst_pitch, const void* src, size_t src_pitch,
                       size_t row_bytes, int rows, void* stream);

/* ---- device-side cross-checks ---------------------- */

/*
 * Quadratic-form SRP map in fp64 -- replaces srp.srp_oracle
 * (pkg/src/srpfast/srp.py:468-515) for pair cross-spectra:
 *   maps[f, j] = sum_k sum_p 2 Re(Psi[f,p,k] conj(h_m) h_m'),
 *   h_m = exp(-i omega[k] tau_rel[j, m]),  (m, m') = (pair_m[p], pair_mp[p])
 * which equals sum_k [h^H Psi h - tr Psi] for the cross matrix assembled from
 * the pairs (srp.py:432-442).  Every exponential is an fp64 sincos (no
 * recurrence, no tensor cores): an independent check of K2.
 *   Psi [F, P, Kb] complex64; omega [Kb] fp64; tau_rel [J, M] fp64 delays
 *   relative to mic 0 (column 0 = 0, columns 1.. = the first M-1 canonical
 *   TDOA columns, srp.py:495-498); maps [F, J] fp64 out.
 */
int srpb_srp_quadform(const float* Psi, int F, int P, int Kb, const double* omega,
                      const double* tau_rel, int J, int M, const int32_t* pair_m,
                      const int32_t* pair_mp, double* maps, void* stream);

/*
 * Per-frame map error energy for metrics.approximation_error_db
 * (pkg/src/srpfast/metrics.py:22-41): num[f] = sum_j (ref - app)^2,
 * den[f] = sum_j ref^2, fp64 accumulation in a fixed order.
 *   ref, app [F, J], fp32 or fp64 each (ref_f64 / app_f64 = 1 for fp64);
 *   scratch: SRPB_MAP_ERROR_SCRATCH * F doubles; num, den [F] fp64 out.
 */
#define SRPB_MAP_ERROR_SCRATCH 128
int srpb_map_error(const void* ref, int ref_f64, const void* app, int app_f64, int F, int J,
                   double* scratch, double* num, double* den, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SRPB_H */
