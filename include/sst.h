/*
 * sst.h -- C ABI of the B200-native fast downsampled SST
 *          (He & Cao, "Fast implementation of synchrosqueezing transform based on
 *           downsampling for large-scale vibration signal analysis", arXiv 2003.07065).
 *
 * Citations: P:Lnnn = PAPER.md line nnn (section / equation); Rnn = reading in DESIGN.md §3.
 *
 * The problem, as the paper states it: given a real signal x
 * sampled at fs, a window g and its derivative g', a time hop H_t and a DFT
 * length N_f (Eq. 7-9), a band [f1, f2] with subdivision z (Eq. 27-29) and a threshold gamma
 * (Eq. 13), return the synchrosqueezed plane T on the band grid, and invert T back to x
 * (Eq. 25-26).
 *
 * Conventions (every entry point):
 *  - Return an sst_status.  Nothing aborts, exits or prints.  sst_last_error() gives a
 *    message for the last failing call on a plan (or, with plan == NULL, on this thread).
 *  - Ownership: the caller owns every buffer passed in.  "device" pointers are CUDA device
 *    memory on the plan's device; "host" pointers are ordinary host memory.  The plan owns
 *    its copies of the window taps, twiddle tables and scratch.
 *  - Complex arrays are complex64: interleaved float pairs (re, im), row-major.
 *  - Asynchrony: compute calls enqueue work on `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream) and return without synchronising.  Launch errors are
 *    returned synchronously as SST_E_CUDA; asynchronous faults surface on the caller's
 *    next synchronisation.
 *  - Threading: a plan is bound to one device and is not thread-safe.
 *  - Frames: F = floor((N-1)/H_t) + 1; frame m is centred on sample m*H_t and covers samples
 *    [m*H_t - c, m*H_t - c + L) (Eq. 8, R4); samples outside [0, N) read as zero.
 */
#ifndef SST_H
#define SST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SST_ABI_VERSION 4

typedef enum {
    SST_OK = 0,
    SST_E_INVALID_ARGUMENT = 1, /* bad parameter, pointer, size or range                       */
    SST_E_COVERAGE = 2,         /* some n in [0,N) has frame diagonal d[n] = 0 (R20)   */
    SST_E_UNSUPPORTED = 3,      /* valid per the paper, outside this library (N_f, B limits)   */
    SST_E_CUDA = 4,             /* a CUDA runtime call or launch failed                        */
    SST_E_OUT_OF_MEMORY = 5,    /* device allocation failed                                    */
    SST_E_INTERNAL = 6
} sst_status;

/* sst_params.flags */
enum {
    SST_GAMMA_RELATIVE = 1u,    /* gamma is relative: gamma_abs = gamma * max|S| (Eq. 13, R6).
                                   sst_forward computes max|S| over its own frames first (one
                                   extra FFT pass) unless sst_plan_set_absmax() gave a device
                                   scalar (e.g. a global max all-reduced over ranks).           */
    SST_SOURCE_TRUNCATE = 2u,   /* only source bins k in [k1, k2) are reassigned (R12)  */
    SST_DETERMINISTIC = 4u,     /* accepted, no effect: every result is bitwise reproducible run to
                                   run (exact fixed-point squeeze sums, fixed-order OLA)            */
    SST_DISCRETE_CONSTANT = 8u, /* inverse divides by C_d = g[c] sum g / sum g^2 instead of
                                   sqrt 2 (Eq. 24, R15)                                         */
    SST_FILTER_BANK = 16u       /* with SST_SOURCE_TRUNCATE: compute the band's S, S' with the
                                   frequency-domain filter bank (§6) instead of per-frame
                                   FFTs (same results to fp32 rounding).  Without the flag the plan
                                   uses it only where its cost model predicts a gain (measured on B200:
                                   none of C2-C4)                                  */
};

typedef struct {
    int64_t n;            /* N: samples of the whole record (also when sharded), >= 1          */
    double fs;            /* sample rate, Hz, > 0                                              */
    int32_t win_len;      /* L >= 1 taps                                                       */
    int32_t win_center;   /* c in [0, L); -1 -> floor(L/2) (P:L85 for odd L, R3 for even L)     */
    const double* g;      /* HOST [L]: analysis window g (copied into the plan)                */
    const double* gd;     /* HOST [L]: g' = dg/dn per sample (R1) (copied)             */
    double sigma;         /* Gaussian sigma in samples for the packing scale alpha = sigma*sqrt 2
                             (R18); <= 0 -> alpha = sqrt(sum g^2 / sum g'^2)                  */
    int32_t hop;          /* H_t >= 1                                                  */
    int32_t nfft;         /* N_f: power of two, L <= N_f <= N; 128..65536 here:
                             <= 8192 fused single-kernel path, 16384..65536 the multi-pass path
                             (same ABI and results contract; the paper's §5.2 uses 2^15) */
    double f1, f2;        /* band [f1, f2) in Hz, 0 <= f1 < f2 <= fs/2, on the grid fs/N_f (R9)*/
    int32_t zoom;         /* subdivision z >= 1 (Eq. 28-29)                                    */
    double gamma;         /* threshold on |S^g| (Eq. 13, R6), >= 0; absolute unless RELATIVE  */
    uint32_t flags;       /* SST_* flags                                                       */
} sst_params;

typedef struct {
    int64_t n;            /* N                                                                 */
    int64_t frames;       /* F = floor((N-1)/H_t) + 1                                          */
    int32_t bins;         /* B = z * N_r output bins per frame (Eq. 28-29, half-open R10)     */
    int32_t k1, k2;       /* snapped band edges in coarse bins (R9), N_r = k2 - k1             */
    int32_t nfft, zoom, hop, center, win_len;
    int32_t src_bins;     /* N_f/2 + 1 source bins per frame (R7)                              */
    double fs;
    double f0_hz;         /* frequency of output bin 0 = k1 * df                               */
    double df_hz;         /* coarse spacing fs / N_f (Eq. 12)                                  */
    double dfz_hz;        /* output spacing df / z (Eq. 28)                                    */
    double gamma_abs;     /* absolute gamma in use (0 until known when RELATIVE)              */
    double alpha;         /* g' packing scale (R18)                                            */
    double hf;            /* H_f = N / N_f                                             */
    double hf_bound;      /* Eq. 38 bound 3N/(4 pi sigma fs) (sigma in s), 0 if sigma unknown  */
    double sigma_f_hz;    /* frequency diffusion sigma_f = 1/(2 pi sigma) (Eq. 35), 0 if
                             sigma unknown                                                     */
    double df_eq37_hz;    /* Eq. 37 limit 1.5 sigma_f on df; same condition as Eq. 38  */
    double df_eq46_hz;    /* Eq. 46 limit sqrt(2) sigma_f on df                        */
    double hf_bound46;    /* Eq. 46 as an H_f bound: N sqrt(2) sigma_f / fs            */
    uint32_t warnings;    /* SST_WARN_* bits: which of the bounds df exceeds (non-fatal)       */
    int32_t forward_path; /* how sst_forward computes the STFT: SST_PATH_FUSED (one kernel per tile
                             of frames, N_f <= 8192), SST_PATH_MULTIPASS (N_f > 8192) or
                             SST_PATH_FILTERBANK (SST_SOURCE_TRUNCATE with a narrow band: the
                             frequency-domain filter bank of P:L485, §6); set by sst_plan_create  */
    int32_t inverse_path; /* how sst_inverse computes Eq. 25-26 (same results contract):
                             SST_IPATH_RESIDUE (z N_f-point IDFT split into z residue sub-IFFTs
                             per frame pair), SST_IPATH_NARROWBAND (full window, band within 8 of
                             64 rows, hop % 8 == 0: residue sum inside the transform, C2/C3) or
                             SST_IPATH_MULTIPASS (N_f > 8192); SST_INV_NB=0 in the environment at
                             plan creation disables the narrow-band path                        */
} sst_layout;

enum { SST_PATH_FUSED = 0, SST_PATH_MULTIPASS = 1, SST_PATH_FILTERBANK = 2 };
enum { SST_IPATH_RESIDUE = 0, SST_IPATH_NARROWBAND = 1, SST_IPATH_MULTIPASS = 2 };

/* sst_layout.warnings (also reported as text by sst_last_error after sst_plan_create) */
enum {
    SST_WARN_EQ37 = 1u,   /* df >= 1.5 sigma_f (Eq. 37 / Eq. 38): reassignment stops concentrating */
    SST_WARN_EQ46 = 2u    /* df >= sqrt(2) sigma_f (Eq. 46): outside the effective-SST interval    */
};

typedef struct sst_plan sst_plan;

/* ---------------------------------------------------------------- host-only helpers -------- */

/* Unit-energy Gaussian window and its analytic derivative, sigma in samples (R1):
 *   g[j]  = (pi sigma^2)^(-1/4) exp(-(j-c)^2 / (2 sigma^2)),  g'[j] = -((j-c)/sigma^2) g[j].
 * center < 0 -> c = floor(L/2).  g, gd: HOST arrays of L doubles, written.  No GPU needed.
 * Errors: SST_E_INVALID_ARGUMENT for L < 1, sigma <= 0 / non-finite, c outside [0,L), NULL. */
sst_status sst_gaussian_window(int32_t L, double sigma_samples, int32_t center, double* g, double* gd);

/* Validate parameters without a GPU (the checks of sst_plan_create, R9, R20).
 * Returns SST_OK, SST_E_INVALID_ARGUMENT, SST_E_COVERAGE or SST_E_UNSUPPORTED (also when a
 * window / hop needs more than 227 KB of shared memory for the forward, the inverse, or the
 * z = 1 inverse that sst_istft runs).                                                       */
sst_status sst_params_validate(const sst_params* p);

/* Layout a valid parameter set would have (host only, no plan).                            */
sst_status sst_params_layout(const sst_params* p, sst_layout* out);

const char* sst_status_str(sst_status s);
/* Message for the last failing call on `plan`; plan == NULL -> this thread's last failure.
 * Also carries non-fatal warnings after plan creation: df at or above the Eq. 37 limit
 * 1.5 sigma_f (H_f above the Eq. 38 bound) and / or the Eq. 46 limit
 * sqrt(2) sigma_f -- see sst_layout.warnings.                                     */
const char* sst_last_error(const sst_plan* plan);
int32_t sst_abi_version(void);

/* ---------------------------------------------------------------- plan --------------------- */

/* Create a plan on CUDA device `device`: validates p, snaps the band (R9), uploads window taps
 * (g, alpha*g'), twiddle tables and inverse normalisation tables (1/(C d[n]), R2/R15), sizes
 * the launch.  *out receives the plan (NULL on failure).  Synchronous, host-blocking.
 * N_f > 8192 (multi-pass path): the plan also owns two FFT scratch buffers of
 * min(F, 2^27 / (8 N_f)) frames (at least z N_f complex per frame pair) -- at most ~2 x 128 MiB
 * -- and 2 L floats per buffered frame pair; calls on such a plan are ordered on the stream they
 * are given, and, like every plan, it is not thread-safe (one stream at a time).             */
sst_status sst_plan_create(const sst_params* p, int device, sst_plan** out);
sst_status sst_plan_layout(const sst_plan* plan, sst_layout* out);
/* Set the absolute threshold gamma (>= 0) used by later sst_forward / sst_targets calls.     */
sst_status sst_plan_set_gamma(sst_plan* plan, double gamma_abs);
/* RELATIVE mode: take max|S| from this device float (e.g. all-reduced over ranks) instead of
 * computing it per call; NULL restores per-call computation.  Not owned by the plan.        */
sst_status sst_plan_set_absmax(sst_plan* plan, const float* absmax_device);
/* R23 counters since plan creation (sst_forward / sst_targets): out[0] = source bins whose fp32
 * decision was re-taken in fp64 (direct Eq. 8 sum), out[1] = of those, bins whose target changed.
 * HOST uint64_t[2].  Synchronous (waits for the device).                                    */
sst_status sst_plan_counters(sst_plan* plan, uint64_t* out);
void sst_plan_destroy(sst_plan* plan);

/* ---------------------------------------------------------------- forward ------------------ */

/* Fused downsampled SST of frames [frame_begin, frame_end) (Eq. 9, 13, 27-29; P:L110-124,
 * P:L192-210): STFT with g and g', omega_hat with threshold, selective reassignment with
 * subdivision; writes only the band.
 *   x:  device float [x_len] holding global samples [x_off, x_off + x_len); must cover
 *       [frame_begin*H_t - c, (frame_end-1)*H_t - c + L) intersected with [0, N).
 *   T:  device complex64, row i = frame frame_begin + i, T[i*ldT + l] for l in [0, B);
 *       ldT >= B (complex elements).  Entries [B, ldT) of a row are not touched.
 * Errors: SST_E_INVALID_ARGUMENT (NULL, empty or out-of-range frames, x not covering,
 *         ldT < B), SST_E_CUDA.                                                              */
sst_status sst_forward(sst_plan* plan, const float* x, int64_t x_off, int64_t x_len,
                       int64_t frame_begin, int64_t frame_end, float* T, int64_t ldT, void* stream);

/* ---------------------------------------------------------------- inverse ------------------ */

/* Whole-record approximate inverse (Eq. 25-26): T holds all F rows (row stride ldT),
 * y: device float [N], overwritten with x_hat.                                              */
sst_status sst_inverse(sst_plan* plan, const float* T, int64_t ldT, float* y, void* stream);

/* Sharded inverse, step 1: y[n - y_off] += sum over frames m in [frame_begin, frame_end) of
 * g[n - m H_t + c] r~[m, n - m H_t] (Eq. 26 before normalisation).  T row i = frame
 * frame_begin + i.  y: device float [y_len] for global samples [y_off, y_off + y_len), must
 * cover the frames' reach intersected with [0, N).                                          */
sst_status sst_inverse_accumulate(sst_plan* plan, const float* T, int64_t ldT,
                                  int64_t frame_begin, int64_t frame_end,
                                  float* y, int64_t y_off, int64_t y_len, void* stream);
/* Step 2: y[n - y_off] /= C d[n] for global n in [y_off, y_off + y_len) (C = sqrt 2 or C_d). */
sst_status sst_inverse_finalize(sst_plan* plan, float* y, int64_t y_off, int64_t y_len, void* stream);
/* Step 2 on a rank of a time-sharded inverse: the received seam -- the previous
 * rank's partial Eq. 26 sums over global samples [seam_off, seam_off + seam_len), device float --
 * is added and the result normalised in one pass:
 *   y[n - y_off] = (y[n - y_off] + seam[n - seam_off]) / (C d[n])   (seam term only inside its span).
 * The seam span must lie inside the y span (SST_E_INVALID_ARGUMENT otherwise); seam_len = 0 is
 * sst_inverse_finalize.  The transport (NCCL / gloo) only moves the bytes; this is the arithmetic. */
sst_status sst_inverse_finalize_seam(sst_plan* plan, float* y, int64_t y_off, int64_t y_len, const float* seam,
                                     int64_t seam_off, int64_t seam_len, void* stream);

/* ---------------------------------------------------------------- plain STFT synthesis ----- */

/* Downsampled STFT synthesis, Eq. (10)-(11): per frame the N_f-point inverse DFT of
 * the one-sided spectrum S[m, k], k = 0..N_f/2 (as written by sst_stft; conjugate mirror, DC and
 * Nyquist real, window-centred phase of Eq. 9), times g, overlap-added and divided by the frame
 * diagonal d[n] = sum_m g[n - m H_t + c]^2 (R2).  No sqrt 2: this is the plain STFT inverse the
 * paper compares the SST against (Figs 4, 7), exact up to rounding (pin P4).
 *   S: device complex64, row m = frame m (all F rows), S[m*ldS + k], ldS >= N_f/2 + 1.
 *   y: device float [N], overwritten.
 * Errors: SST_E_INVALID_ARGUMENT (NULL, ldS too small), SST_E_CUDA.                        */
sst_status sst_istft(sst_plan* plan, const float* S, int64_t ldS, float* y, void* stream);

/* ---------------------------------------------------------------- analysis ----------------- */

/* Renyi entropy of order alpha of the TF plane P = |T|^2 (Eq. 32):
 *   H_alpha = log2( sum P^alpha / (sum P)^alpha ) / (1 - alpha).
 * T: device complex64 [rows][ldT], columns [0, B).  out: device double [3] receives
 * { sum P, sum P^alpha, H_alpha } (fp64 accumulation in a fixed order: reproducible).
 * alpha > 0, alpha != 1.  Errors: SST_E_INVALID_ARGUMENT, SST_E_CUDA.                    */
sst_status sst_renyi(sst_plan* plan, const float* T, int64_t rows, int64_t ldT, double alpha, double* out,
                     void* stream);

/* ---------------------------------------------------------------- mode retrieval ---------- */
/* Ridge, zone and retrieval of one component (§2.2, §2.3).  The paper names
 * ridge extraction without an algorithm; this is reading R22: maximise
 *   sum_m E[m, l_m] - lambda sum_m (l_{m+1} - l_m)^2,  E = log(|T| + eps), eps = 1e-12 max|T|,
 * ties to the lowest bin, `count` ridges one after another with the zone +-suppress bins of each
 * found ridge set to log(eps) first.
 *
 * sst_ridge_emission: E device double [rows][B] and *floor_out (device double) = log(eps), from
 *   T device complex64 [rows][ldT].
 * sst_ridge: paths device int32 [count][rows] from E (modified: suppressed zones).  One CTA runs
 *   the DP sequentially over frames (exact, O(B log B) per frame); plan-owned scratch holds
 *   rows*B int32 backpointers.  B <= 8000 (SST_E_UNSUPPORTED beyond).
 * sst_zone_mask: in place, T[m, l] = 0 where |l - path[m]| > half (keep_inside = 1) or
 *   <= half (keep_inside = 0); sst_inverse of the masked T retrieves the mode (§2.3).
 * sst_mode_full: Eq. 15 for H_t = 1 (else SST_E_INVALID_ARGUMENT, "invalid for downsampled SST",
 *   P:L130): x[m] = (2 / (N_f g[c])) Re sum_{|l - path[m]| <= half} w_l T[m, l], w = 1/2 at DC;
 *   x device float [rows].                                                                  */
sst_status sst_ridge_emission(sst_plan* plan, const float* T, int64_t ldT, int64_t rows, double* E,
                              double* floor_out, void* stream);
sst_status sst_ridge(sst_plan* plan, double* E, int64_t rows, double lambda, int32_t count, int32_t suppress,
                     const double* floor_in, int32_t* paths, void* stream);
sst_status sst_zone_mask(sst_plan* plan, float* T, int64_t ldT, int64_t rows, const int32_t* path, int32_t half,
                         int32_t keep_inside, void* stream);
sst_status sst_mode_full(sst_plan* plan, const float* T, int64_t ldT, int64_t rows, const int32_t* path,
                         int32_t half, float* x, void* stream);
/* Mode retrieval by the downsampled inverse (§2.3, Eq. 25-26) with the zone applied inside
 * the inverse kernel's loads of T (no masked copy of T, no extra pass): entries with
 * |l - path[m]| <= half are used (keep_inside = 1) or only the others (keep_inside = 0).
 * T as sst_inverse (all F rows); path device int32 [F]; y device float [N], overwritten.        */
sst_status sst_inverse_zone(sst_plan* plan, const float* T, int64_t ldT, const int32_t* path, int32_t half,
                            int32_t keep_inside, float* y, void* stream);

/* ---------------------------------------------------------------- debug / parity ----------- */

/* S^g and S^{g'} (Eq. 9) of frames [fb, fe) for k = 0..N_f/2: S, Sd device complex64
 * [(fe-fb) * (N_f/2+1)].                                                                    */
sst_status sst_stft(sst_plan* plan, const float* x, int64_t x_off, int64_t x_len,
                    int64_t fb, int64_t fe, float* S, float* Sd, void* stream);
/* S^g and S^{g'} of frames [fb, fe) for the band's source bins k in [k1, k2) only, computed by the
 * plan's frequency-domain filter bank (SST_PATH_FILTERBANK plans; SST_E_UNSUPPORTED otherwise):
 * S, Sd device complex64 [(fe-fb) * (k2-k1)], row i = frame fb + i.  Debug / parity.          */
sst_status sst_stft_band(sst_plan* plan, const float* x, int64_t x_off, int64_t x_len,
                         int64_t fb, int64_t fe, float* S, float* Sd, void* stream);
/* Target bin of every source coefficient (Eq. 13, 28): l device int32 [(fe-fb)*(N_f/2+1)];
 * -1 = masked (|S| <= gamma or truncated), -2 = out of band / non-finite (R10, R17).       */
sst_status sst_targets(sst_plan* plan, const float* x, int64_t x_off, int64_t x_len,
                       int64_t fb, int64_t fe, int32_t* l, void* stream);
/* max over frames [fb, fe), k in [0, N_f/2] of |S^g[m,k]| into device float *out (overwritten;
 * the gamma pre-pass for a relative threshold, Eq. 13, R6).                                */
sst_status sst_absmax(sst_plan* plan, const float* x, int64_t x_off, int64_t x_len,
                      int64_t fb, int64_t fe, float* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SST_H */
