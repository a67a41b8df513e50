// Host side of the C ABI declared in include/sst.h: validation, plan creation (window taps,
// twiddle and normalisation tables), argument checks and kernel launches.  No compute runs
// on the host: every step of the transform is a kernel in sst_kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "../../include/sst.h"
#include "sst_internal.h"

namespace {

thread_local std::string g_thread_err;
constexpr int64_t kR23Chunk = 1 << 20;   // frames per deferred R23 launch sequence

constexpr double kPi = 3.14159265358979323846264338327950288;

}  // namespace

struct sst_plan {
    sst_params p{};
    sst_layout lay{};
    int device = 0;
    std::vector<double> g, gd;
    double cst = 0;                 // C (sqrt 2 or C_d)
    // device tables
    float2* d_taps = nullptr;       // [L]  (g, alpha g')
    float* d_gwin = nullptr;        // [L]  g / N_f (narrow-band inverse window table)
    float2* d_tw = nullptr;         // [N_f]
    double2* d_taps64 = nullptr;    // [L]  (g, g') fp64 (R23 re-decision)
    double2* d_tw64 = nullptr;      // [N_f] exp(-2 pi i e/N_f) fp64
    int32_t* d_mpl = nullptr;       // multi-pass: [mp_fwd_frames][N_f/2 + 1] targets
    unsigned long long* d_r23 = nullptr;   // [2] R23 counters (sst_plan_counters)
    int4* d_gq = nullptr;           // R23 deferral queue [gq_cap], one region per CTA
    unsigned int* d_gctr = nullptr; // [1 + fwd_grid]: dirty frames, then each CTA's queued entries
    unsigned int* d_dirty_bits = nullptr;   // [(F + 31) / 32]
    int* d_dirty_list = nullptr;    // [gq_cap]
    unsigned int gq_cap = 0;
    // filter-bank forward (f3b): chosen at plan creation for SST_SOURCE_TRUNCATE with a narrow band
    bool fb = false;
    sst::FbArgs fbt{};              // geometry and device tables (x, frames, planes set per launch)
    float2 *d_fb_gam = nullptr, *d_fb_gamd = nullptr, *d_fb_ph = nullptr, *d_fb_twns = nullptr, *d_fb_twp = nullptr;
    float2 *d_fb_S = nullptr, *d_fb_Sd = nullptr;
    float* d_fb_eta = nullptr;
    int64_t fb_chunk = 0;
    int fb_sq_grid = 0;
    float2* d_phz = nullptr;        // [z][64 + 2 N_f/64]
    double* d_renyi = nullptr;      // [kRenyiBlocks][2] partial sums
    unsigned long long* d_amax2 = nullptr;   // ridge emission: max |T| (double bits)
    int32_t* d_back = nullptr;      // ridge DP backpointers
    size_t back_elems = 0;
    float* d_inv_head = nullptr;    // [n_head]
    float* d_inv_tail = nullptr;    // [n_tail]
    float* d_inv_per = nullptr;     // [hop]
    float* d_absmax = nullptr;      // scratch scalar
    float* d_seam = nullptr;        // [inv_max_grid][2][seam_len]
    // multi-pass large-N_f path (N_f > kMaxFusedNfft)
    bool mp = false;
    float2* d_twN = nullptr;        // [N_f] W_N^k
    float2* d_mp0 = nullptr;        // FFT scratch, mp_elems float2 each
    float2* d_mp1 = nullptr;
    float* d_wf = nullptr;          // [2 mp_inv_pairs][L] windowed frames
    int64_t mp_fwd_frames = 0, mp_inv_pairs = 0;
    int32_t n_head = 0, n_tail = 0;
    int fwd_grid = 0, inv_grid = 0;
    int inv_grid_nb = 0;            // narrow-band inverse (inv_nb_kernel.cuh): resident CTAs, 0 = not used
    bool redecide = true;           // R23 (SST_NO_REDECIDE=1 turns it off: timing experiments only)
    double r23_m = 6.0;             // R23 margin factor over the R21 error model (SST_R23_M: experiments)
    const float* ext_absmax = nullptr;
    double gamma_abs = 0;
    std::string err;
    ~sst_plan() {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        for (void* q : {(void*)d_taps, (void*)d_gwin, (void*)d_tw, (void*)d_taps64, (void*)d_tw64, (void*)d_mpl, (void*)d_r23, (void*)d_gq, (void*)d_gctr,
                        (void*)d_dirty_bits, (void*)d_dirty_list, (void*)d_fb_gam, (void*)d_fb_gamd,
                        (void*)d_fb_ph, (void*)d_fb_twns, (void*)d_fb_twp, (void*)d_fb_S, (void*)d_fb_Sd,
                        (void*)d_fb_eta, (void*)d_phz, (void*)d_renyi, (void*)d_amax2, (void*)d_back, (void*)d_inv_head, (void*)d_inv_tail,
                        (void*)d_inv_per, (void*)d_absmax, (void*)d_seam, (void*)d_twN, (void*)d_mp0, (void*)d_mp1, (void*)d_wf})
            if (q) cudaFree(q);
        cudaSetDevice(prev);
    }
};

namespace {

sst_status fail(sst_plan* plan, sst_status s, const std::string& msg) {
    if (plan) plan->err = msg;
    g_thread_err = msg;
    return s;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        cudaSetDevice(dev);
    }
    ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

int64_t frames_of(int64_t n, int32_t hop) { return (n - 1) / hop + 1; }

// frame diagonal d[n] = sum_m g[n - m H + c]^2 over frames 0..F-1 (Eq. 11 / Eq. 26 normaliser, R2)
double diag_at(const std::vector<double>& g, int64_t n, int64_t N, int32_t hop, int32_t c) {
    const int64_t L = (int64_t)g.size();
    const int64_t F = frames_of(N, hop);
    int64_t m_lo = n + c - L + 1;
    m_lo = m_lo <= 0 ? 0 : (m_lo + hop - 1) / hop;
    int64_t m_hi = (n + c) / hop;
    if (m_hi > F - 1) m_hi = F - 1;
    double d = 0;
    for (int64_t m = m_lo; m <= m_hi; ++m) {
        const int64_t j = n - m * hop + c;
        if (j >= 0 && j < L) d += g[j] * g[j];
    }
    return d;
}

// Validation shared by sst_params_validate / sst_params_layout / sst_plan_create.
sst_status validate(const sst_params* p, sst_layout* lay, std::string& msg) {
    if (!p) { msg = "params is NULL"; return SST_E_INVALID_ARGUMENT; }
    if (!p->g || !p->gd) { msg = "window arrays g/gd are NULL"; return SST_E_INVALID_ARGUMENT; }
    if (p->n < 1) { msg = "N must be >= 1"; return SST_E_INVALID_ARGUMENT; }
    if (!std::isfinite(p->fs) || p->fs <= 0) { msg = "fs must be finite and > 0"; return SST_E_INVALID_ARGUMENT; }
    if (p->win_len < 1) { msg = "window length L must be >= 1"; return SST_E_INVALID_ARGUMENT; }
    const int32_t L = p->win_len;
    const int32_t c = p->win_center < 0 ? L / 2 : p->win_center;
    if (c >= L) { msg = "window centre outside [0, L)"; return SST_E_INVALID_ARGUMENT; }
    if (p->hop < 1) { msg = "hop H_t must be >= 1"; return SST_E_INVALID_ARGUMENT; }
    if (p->nfft < 1) { msg = "N_f must be >= 1"; return SST_E_INVALID_ARGUMENT; }
    if (p->zoom < 1) { msg = "subdivision z must be >= 1"; return SST_E_INVALID_ARGUMENT; }
    if (!std::isfinite(p->gamma) || p->gamma < 0) { msg = "gamma must be finite and >= 0"; return SST_E_INVALID_ARGUMENT; }
    if (!std::isfinite(p->sigma)) { msg = "sigma must be finite"; return SST_E_INVALID_ARGUMENT; }
    if (p->flags & ~(uint32_t)(SST_GAMMA_RELATIVE | SST_SOURCE_TRUNCATE | SST_DETERMINISTIC | SST_DISCRETE_CONSTANT |
                               SST_FILTER_BANK)) {
        msg = "unknown flag bits"; return SST_E_INVALID_ARGUMENT;
    }
    if ((int64_t)L > (int64_t)p->nfft || (int64_t)p->nfft > p->n) {
        msg = "need L <= N_f <= N (P:L89)"; return SST_E_INVALID_ARGUMENT;
    }
    double sg2 = 0, sgd2 = 0;
    for (int32_t j = 0; j < L; ++j) {
        if (!std::isfinite(p->g[j]) || !std::isfinite(p->gd[j])) { msg = "non-finite window tap"; return SST_E_INVALID_ARGUMENT; }
        sg2 += p->g[j] * p->g[j];
        sgd2 += p->gd[j] * p->gd[j];
    }
    if (!(sg2 > 0)) { msg = "window g is identically zero"; return SST_E_INVALID_ARGUMENT; }
    // band snapping (R9)
    const double df = p->fs / p->nfft;
    if (!std::isfinite(p->f1) || !std::isfinite(p->f2) || p->f1 < 0 || p->f2 <= p->f1 || p->f2 > p->fs / 2 * (1 + 1e-15)) {
        msg = "need 0 <= f1 < f2 <= fs/2"; return SST_E_INVALID_ARGUMENT;
    }
    const double k1f = p->f1 / df, k2f = p->f2 / df;
    const double k1r = std::nearbyint(k1f), k2r = std::nearbyint(k2f);
    if (std::fabs(k1f - k1r) > 1e-9 || std::fabs(k2f - k2r) > 1e-9) {
        msg = "band edges must lie on the coarse grid fs/N_f (R9)"; return SST_E_INVALID_ARGUMENT;
    }
    const int64_t k1 = (int64_t)k1r, k2 = (int64_t)k2r;
    if (!(k1 >= 0 && k1 < k2 && k2 <= p->nfft / 2)) { msg = "band outside [0, N_f/2]"; return SST_E_INVALID_ARGUMENT; }
    // library limits
    if (!is_pow2(p->nfft)) { msg = "N_f must be a power of two (P:L93)"; return SST_E_UNSUPPORTED; }
    if (p->nfft < 128 || p->nfft > sst::kMaxNfft) { msg = "this build supports 128 <= N_f <= 65536"; return SST_E_UNSUPPORTED; }
    if (p->zoom > 64 || (int64_t)p->zoom * p->nfft > (1 << 20)) { msg = "z <= 64 and z N_f <= 2^20 supported"; return SST_E_UNSUPPORTED; }
    {
        // shared-memory footprint of the forward / inverse CTAs (227 KB per CTA on sm_100)
        constexpr int kMaxSmem = 227 * 1024;
        const int n2 = p->nfft / 64;
        if (p->hop <= L && p->nfft <= sst::kMaxFusedNfft && (sst::fwd_layout(n2, L, p->hop).total > kMaxSmem - sst::kFwdStaticSmem ||
                            sst::inv_layout(n2, L, p->hop, p->zoom).total > kMaxSmem ||
                            sst::inv_layout(n2, L, p->hop, 1).total > kMaxSmem)) {   // z = 1: sst_istft
            msg = "window / hop too large for this build's shared-memory tiles (227 KB per CTA)";
            return SST_E_UNSUPPORTED;
        }
    }
    // coverage (R20): every n in [0, N) needs d[n] > 0
    const int64_t N = p->n;
    const int64_t F = frames_of(N, p->hop);
    if (p->hop > L || (F - 1) * (int64_t)p->hop - c + L < N) {
        msg = "frames do not cover [0, N): need H_t <= L and (F-1) H_t - c + L >= N (R20)"; return SST_E_COVERAGE;
    }
    {
        std::vector<double> g(p->g, p->g + L);
        // periodic interior part
        for (int32_t i = 0; i < p->hop; ++i) {
            double s = 0;
            for (int32_t j = i; j < L; j += p->hop) s += g[j] * g[j];
            if (!(s > 0)) { msg = "frame diagonal vanishes (window zeros) (R20)"; return SST_E_COVERAGE; }
        }
        const int64_t nh = std::min<int64_t>(N, L), nt = std::min<int64_t>(N, (int64_t)L + p->hop);
        for (int64_t n = 0; n < nh; ++n)
            if (!(diag_at(g, n, N, p->hop, c) > 0)) { msg = "frame diagonal vanishes at the head (R20)"; return SST_E_COVERAGE; }
        for (int64_t n = N - nt; n < N; ++n)
            if (!(diag_at(g, n, N, p->hop, c) > 0)) { msg = "frame diagonal vanishes at the tail (R20)"; return SST_E_COVERAGE; }
    }
    if (lay) {
        std::memset(lay, 0, sizeof(*lay));
        lay->n = N;
        lay->frames = F;
        lay->k1 = (int32_t)k1;
        lay->k2 = (int32_t)k2;
        lay->bins = (int32_t)(p->zoom * (k2 - k1));
        lay->nfft = p->nfft;
        lay->zoom = p->zoom;
        lay->hop = p->hop;
        lay->center = c;
        lay->win_len = L;
        lay->src_bins = p->nfft / 2 + 1;
        lay->fs = p->fs;
        lay->df_hz = df;
        lay->f0_hz = k1 * df;
        lay->dfz_hz = df / p->zoom;
        lay->gamma_abs = (p->flags & SST_GAMMA_RELATIVE) ? 0.0 : p->gamma;
        lay->alpha = p->sigma > 0 ? p->sigma * std::sqrt(2.0) : (sgd2 > 0 ? std::sqrt(sg2 / sgd2) : 1.0);
        lay->hf = (double)N / p->nfft;
        lay->hf_bound = p->sigma > 0 ? 3.0 * (double)N / (4.0 * kPi * p->sigma) : 0.0;   // Eq. 38, sigma_s = sigma/fs
        // Eq. 35: sigma_f = 1/(2 pi sigma_s) Hz with sigma_s = sigma / fs; Eq. 37 / Eq. 46 limits on df
        lay->sigma_f_hz = p->sigma > 0 ? p->fs / (2.0 * kPi * p->sigma) : 0.0;
        lay->df_eq37_hz = 1.5 * lay->sigma_f_hz;
        lay->df_eq46_hz = std::sqrt(2.0) * lay->sigma_f_hz;
        lay->hf_bound46 = lay->df_eq46_hz * (double)N / p->fs;
        lay->warnings = 0;
        if (p->sigma > 0 && df >= lay->df_eq37_hz) lay->warnings |= SST_WARN_EQ37;
        if (p->sigma > 0 && df >= lay->df_eq46_hz) lay->warnings |= SST_WARN_EQ46;
    }
    msg.clear();
    return SST_OK;
}

std::vector<cudaError_t (*)(const float2*)>& w64_uploaders() {
    static std::vector<cudaError_t (*)(const float2*)> v;   // filled at load time (fft.cuh registrars)
    return v;
}

std::mutex g_w64_mu;
uint64_t g_w64_uploaded = 0;   // bitmask of devices with c_w64 set

sst_status ensure_w64(int device, std::string& msg) {
    std::lock_guard<std::mutex> lk(g_w64_mu);
    if (device < 64 && (g_w64_uploaded >> device) & 1ull) return SST_OK;
    float2 w[64];
    for (int e = 0; e < 64; ++e) {
        const double a = -2.0 * kPi * e / 64.0;
        w[e] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
    for (auto fn : w64_uploaders()) {
        cudaError_t ce = fn(w);
        if (ce != cudaSuccess) { msg = std::string("upload twiddles: ") + cudaGetErrorString(ce); return SST_E_CUDA; }
    }
    if (device < 64) g_w64_uploaded |= 1ull << device;
    return SST_OK;
}

template <class T>
sst_status upload(sst_plan* pl, T** dst, const std::vector<T>& src) {
    if (src.empty()) return SST_OK;
    cudaError_t ce = cudaMalloc((void**)dst, sizeof(T) * src.size());
    if (ce == cudaErrorMemoryAllocation) return fail(pl, SST_E_OUT_OF_MEMORY, "cudaMalloc failed (out of memory)");
    if (ce != cudaSuccess) return fail(pl, SST_E_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(ce));
    ce = cudaMemcpy(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) return fail(pl, SST_E_CUDA, std::string("cudaMemcpy: ") + cudaGetErrorString(ce));
    return SST_OK;
}

sst_status cuda_status(sst_plan* pl, cudaError_t ce, const char* what) {
    if (ce == cudaSuccess) return SST_OK;
    cudaGetLastError();
    return fail(pl, SST_E_CUDA, std::string(what) + ": " + cudaGetErrorString(ce));
}

// x slice must cover [fb H - c, (fe-1) H - c + L) intersected with [0, N)
bool covers_input(const sst_plan* pl, int64_t x_off, int64_t x_len, int64_t fb, int64_t fe) {
    const int64_t lo = std::max<int64_t>(0, fb * pl->lay.hop - pl->lay.center);
    const int64_t hi = std::min<int64_t>(pl->lay.n, (fe - 1) * pl->lay.hop - pl->lay.center + pl->lay.win_len);
    if (hi <= lo) return true;
    return x_off <= lo && x_off + x_len >= hi;
}

sst_status check_frames(sst_plan* pl, int64_t fb, int64_t fe) {
    if (!(fb >= 0 && fb < fe && fe <= pl->lay.frames))
        return fail(pl, SST_E_INVALID_ARGUMENT, "frame range must satisfy 0 <= begin < end <= F");
    return SST_OK;
}

sst::FwdArgs fwd_args(const sst_plan* pl, const float* x, int64_t x_off, int64_t x_len, int64_t fb, int64_t fe) {
    sst::FwdArgs a{};
    a.x = x;
    a.x_off = x_off;
    a.x_len = x_len;
    a.n = pl->lay.n;
    a.frame_begin = fb;
    a.frame_end = fe;
    a.hop = pl->lay.hop;
    a.L = pl->lay.win_len;
    a.c = pl->lay.center;
    a.nfft = pl->lay.nfft;
    a.taps = pl->d_taps;
    a.tw = pl->d_tw;
    a.k1 = pl->lay.k1;
    a.k2 = pl->lay.k2;
    a.bins = pl->lay.bins;
    a.zoom = pl->lay.zoom;
    const bool trunc = pl->p.flags & SST_SOURCE_TRUNCATE;
    a.src_lo = trunc ? pl->lay.k1 : 0;
    a.src_hi = trunc ? pl->lay.k2 : pl->lay.nfft / 2 + 1;
    const double gam = pl->gamma_abs;
    a.gamma2x4 = (float)(4.0 * gam * gam);
    a.absmax_dev = nullptr;
    a.gamma_rel = (float)pl->p.gamma;
    a.r_scale = (float)(pl->lay.nfft / (2.0 * kPi * pl->lay.alpha));
    a.zr_scale = (float)(pl->lay.zoom * pl->lay.nfft / (2.0 * kPi * pl->lay.alpha));
    a.r_scale_d = pl->lay.nfft / (2.0 * kPi * pl->lay.alpha);
    a.inv_alpha2 = (float)(1.0 / (2.0 * pl->lay.alpha));
    // R23: margins of the fp32 decision, 8 x the R21 error model eta = 4 u sqrt(log2 N_f) ||z_m||
    const double u = std::ldexp(1.0, -24), sl = std::sqrt(std::log2((double)pl->lay.nfft));
    a.redecide = pl->redecide ? 1 : 0;
    a.cflag = (float)(pl->r23_m * (pl->lay.zoom * pl->lay.nfft / (2.0 * kPi * pl->lay.alpha)) * 4.0 * u * sl);
    a.kflag = (float)(pl->r23_m * 2.0 * u * sl);
    a.gamma_d = pl->gamma_abs;
    a.gamma_rel_d = pl->p.gamma;
    a.taps64 = pl->d_taps64;
    a.tw64 = pl->d_tw64;
    a.lscratch = pl->d_mpl;
    a.r23_count = pl->d_r23;
    a.lay = sst::fwd_layout(pl->lay.nfft / 64, pl->lay.win_len, pl->lay.hop);
    return a;
}

int fwd_grid_for(const sst_plan* pl, int64_t nfr) {
    const int G = sst::groups_of(pl->lay.nfft / 64, true);
    const int64_t tiles = (nfr + G - 1) / G;
    return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, pl->fwd_grid));
}

// forward-family launch on either path; the multi-pass path runs in chunks of mp_fwd_frames
cudaError_t launch_fwd_any(const sst_plan* pl, const sst::FwdArgs& a, int mode, cudaStream_t st) {
    if (!pl->mp) return sst::launch_forward(a, mode, fwd_grid_for(pl, a.frame_end - a.frame_begin), st);
    const int64_t K = pl->lay.nfft / 2 + 1;
    for (int64_t c0 = a.frame_begin; c0 < a.frame_end; c0 += pl->mp_fwd_frames) {
        sst::FwdArgs b = a;
        const int64_t off = c0 - a.frame_begin;
        b.frame_begin = c0;
        b.frame_end = std::min<int64_t>(a.frame_end, c0 + pl->mp_fwd_frames);
        if (b.T) b.T += off * a.ldT;
        if (b.S) b.S += off * K;
        if (b.Sd) b.Sd += off * K;
        if (b.lout) b.lout += off * K;
        cudaError_t e = sst::launch_mp_forward(b, mode, pl->d_twN, pl->d_mp0, pl->d_mp1, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// y (+)= the inverse of frames [fb, fe) on the multi-pass path (chunks of 2 mp_inv_pairs frames)
cudaError_t mp_inverse_accumulate(const sst_plan* pl, const float2* T, int64_t ldT, int64_t fb, int64_t fe,
                                  int32_t k1, int32_t bins, int32_t zoom, float* y, int64_t y_off, int64_t y_len,
                                  cudaStream_t st, const int32_t* zone_path = nullptr, int32_t zone_half = 0,
                                  int32_t zone_keep = 1) {
    sst::MpInvArgs a{};
    a.ldT = ldT;
    a.n = pl->lay.n;
    a.hop = pl->lay.hop;
    a.L = pl->lay.win_len;
    a.c = pl->lay.center;
    a.nfft = pl->lay.nfft;
    a.zoom = zoom;
    a.k1 = k1;
    a.bins = bins;
    a.taps = pl->d_taps;
    a.twN = pl->d_twN;
    a.inv_n = (float)(1.0 / pl->lay.nfft);
    a.buf0 = pl->d_mp0;
    a.buf1 = pl->d_mp1;
    a.wf = pl->d_wf;
    a.y = y;
    a.y_off = y_off;
    a.y_len = y_len;
    // direct band sum when its cost B L (complex FMAs per frame) is below the FFT path's, measured
    // on B200 at ~4.3 z N_f log2 N_f in the same units; SST_MP_INVERSE=fft|direct overrides (tests)
    const double lg = std::log2((double)pl->lay.nfft);
    a.direct = ((double)bins * pl->lay.win_len < 4.3 * zoom * (double)pl->lay.nfft * lg && bins <= 6144) ? 1 : 0;
    if (const char* ov = std::getenv("SST_MP_INVERSE")) {
        if (!std::strcmp(ov, "fft")) a.direct = 0;
        else if (!std::strcmp(ov, "direct") && bins <= 6144) a.direct = 1;
    }
    const int64_t step = 2 * pl->mp_inv_pairs;        // buffers hold mp_inv_pairs x plan z >= zoom transforms
    for (int64_t c0 = fb; c0 < fe; c0 += step) {
        a.frame_begin = c0;
        a.frame_end = std::min<int64_t>(fe, c0 + step);
        a.T = T + (c0 - fb) * ldT;
        a.zone_path = zone_path ? zone_path + (c0 - fb) : nullptr;
        a.zone_half = zone_half;
        a.zone_keep = zone_keep;
        cudaError_t e = sst::launch_mp_inverse_accumulate(a, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace

namespace {

// f3b: filter-bank geometry and tables (see filterbank.cu).  Returns false (plan keeps the fused
// forward) when the band is not narrow, H does not divide the segment, or the tiles do not fit.
// in-place iterative radix-2 DFT, fp64: a[k] <- sum_n a[n] e^{sign 2 pi i n k / n_pts}
void fft64(std::vector<std::pair<double, double>>& a, int sign) {
    const size_t n = a.size();
    for (size_t i = 1, j = 0; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i], a[j]);
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        for (size_t i = 0; i < n; i += len)
            for (size_t k = 0; k < len / 2; ++k) {
                const double ang = sign * 2.0 * kPi * (double)k / (double)len;
                const double wr = std::cos(ang), wi = std::sin(ang);
                auto& u = a[i + k];
                auto& v = a[i + k + len / 2];
                const double tr = v.first * wr - v.second * wi, ti = v.first * wi + v.second * wr;
                v = {u.first - tr, u.second - ti};
                u = {u.first + tr, u.second + ti};
            }
    }
}

bool setup_filterbank(sst_plan* pl) {
    const sst_layout& ly = pl->lay;
    // SST_FILTER_BANK requests it; SST_FILTERBANK=0 / =1 (environment, tests only) forbid / force it
    const char* env = std::getenv("SST_FILTERBANK");
    int force = (pl->p.flags & SST_FILTER_BANK) ? 1 : 0;
    if (env) force = env[0] == '1' ? 1 : (env[0] == '0' ? -1 : force);
    if (force < 0 || pl->mp || !(pl->p.flags & SST_SOURCE_TRUNCATE)) return false;
    const int32_t Nf = ly.nfft, L = ly.win_len, H = ly.hop, kb = ly.k2 - ly.k1;
    if (ly.bins > 1024 || kb > 1024) return false;
    int64_t ns = 1;
    while (ns < 4 * (int64_t)L) ns <<= 1;
    if (ns < Nf) ns = Nf;
    if (ns > 16384 || ns % H != 0) return false;
    const int32_t P = (int32_t)(ns / H);
    if ((P & (P - 1)) != 0 || P < 32) return false;
    const int32_t fbn = (int32_t)((ns - L) / H + 1);
    int lgP = 0;
    while ((1 << lgP) < P) ++lgP;
    // cost model (complex multiply-adds per frame): folds + P-point inverse FFTs of 2 K_b bins per
    // block and the block FFT, against the fused path's packed N_f-point FFT
    // measured on B200 (tools/time_fb.py): the filter bank ran 1.8x / 2.0x / 3.1x the fused forward on
    // C2 / C3 / C4 at modelled cost ratios 0.53 / 0.79 / 2.0 (its folds and P-point transforms are
    // shared-memory-latency bound), so it is picked only below a modelled ratio of 0.25
    const double fb_cost = (2.0 * kb * ((double)ns + 0.5 * P * lgP) + 0.5 * ns * std::log2((double)ns)) / fbn;
    const double fused_cost = 0.5 * Nf * std::log2((double)Nf);
    if (!force && fb_cost > 0.25 * fused_cost) return false;
    // Gamma[d] = sum_j g[j] e^{2 pi i d j / Ns} for every d (an fp64 inverse-sign DFT of the zero-padded
    // taps), and the same for g'
    std::vector<std::pair<double, double>> G(ns, {0.0, 0.0}), Gd(ns, {0.0, 0.0});
    for (int32_t j = 0; j < L; ++j) { G[j] = {pl->g[j], 0.0}; Gd[j] = {pl->gd[j], 0.0}; }
    fft64(G, +1);
    fft64(Gd, +1);
    // staging chunk: the largest power of two <= 32 bins that fits the transform CTA's shared memory
    // together with one window's Gamma (Ns float2, staged per pass); without it if even 4 bins do not fit
    auto smem_of = [&](int kcv, bool gsm) { return (ns + 8 * P + (int64_t)fbn * kcv * 2 + (gsm ? ns : 0)) * 8; };
    int kc = 32;
    while (kc > 4 && smem_of(kc, true) > 227 * 1024 - 1024) kc >>= 1;
    if (smem_of(kc, true) > 227 * 1024 - 1024) {
        kc = 32;
        while (kc > 1 && smem_of(kc, false) > 227 * 1024 - 1024) kc >>= 1;
        if (smem_of(kc, false) > 227 * 1024 - 1024) return false;
    }
    std::vector<float2> gam(ns), gamd(ns), ph(kb), twns(ns / 2), twp(P / 2);
    for (int64_t d = 0; d < ns; ++d) {
        gam[d] = make_float2((float)G[d].first, (float)G[d].second);
        gamd[d] = make_float2((float)Gd[d].first, (float)Gd[d].second);
    }
    for (int32_t kk = 0; kk < kb; ++kk) {
        const int64_t k = ly.k1 + kk;
        const double a = 2.0 * kPi * (double)((k * ly.center) % Nf) / (double)Nf;
        ph[kk] = make_float2((float)(std::cos(a) / ns), (float)(std::sin(a) / ns));
    }
    for (int64_t e = 0; e < ns / 2; ++e) {
        const double a = -2.0 * kPi * (double)e / (double)ns;
        twns[e] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
    for (int32_t e = 0; e < P / 2; ++e) {
        const double a = 2.0 * kPi * (double)e / (double)P;
        twp[e] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
    if (upload(pl, &pl->d_fb_gam, gam) != SST_OK || upload(pl, &pl->d_fb_gamd, gamd) != SST_OK ||
        upload(pl, &pl->d_fb_ph, ph) != SST_OK || upload(pl, &pl->d_fb_twns, twns) != SST_OK ||
        upload(pl, &pl->d_fb_twp, twp) != SST_OK)
        return false;
    pl->fb_chunk = std::min<int64_t>(ly.frames, 1 << 18);
    if (cudaMalloc((void**)&pl->d_fb_S, sizeof(float2) * (size_t)pl->fb_chunk * kb) != cudaSuccess ||
        cudaMalloc((void**)&pl->d_fb_Sd, sizeof(float2) * (size_t)pl->fb_chunk * kb) != cudaSuccess ||
        cudaMalloc((void**)&pl->d_fb_eta, sizeof(float) * (size_t)pl->fb_chunk) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    sst::FbArgs& f = pl->fbt;
    f.hop = H;
    f.c = ly.center;
    f.ns = (int32_t)ns;
    f.lg_ns = 0;
    while ((1ll << f.lg_ns) < ns) ++f.lg_ns;
    f.P = P;
    f.lg_P = 0;
    while ((1 << f.lg_P) < P) ++f.lg_P;
    f.fb = fbn;
    f.kc = kc;
    f.ratio = (int32_t)(ns / Nf);
    f.kb0 = ly.k1;
    f.kb = kb;
    f.gam = pl->d_fb_gam;
    f.gamd = pl->d_fb_gamd;
    f.ph = pl->d_fb_ph;
    f.twns = pl->d_fb_twns;
    f.twp = pl->d_fb_twp;
    f.S = pl->d_fb_S;
    f.Sd = pl->d_fb_Sd;
    f.eta = pl->d_fb_eta;
    f.alpha = (float)ly.alpha;
    // R23 error model of the filter-bank S (calibrated on the GPU like the fused one,
    // tools/diag_fb_margin.py: r errors <= 3.3 x the model with the constant 4, so 8 is used): one S
    // value off by eta_S = 8 u sqrt(log2(Ns P)) ||x_b|| ||g|| / sqrt(Ns) (S' likewise with ||g'||,
    // taken through alpha); margins M times that, in the fused kernel's units (its eta is twice an S error)
    double g2 = 0, gd2 = 0;
    for (int32_t j = 0; j < L; ++j) { g2 += pl->g[j] * pl->g[j]; gd2 += pl->gd[j] * pl->gd[j]; }
    const double gnorm = std::sqrt(g2) * std::max(1.0, ly.alpha * std::sqrt(gd2 / g2));
    const double u = std::ldexp(1.0, -24);
    const double etaS = 8.0 * u * std::sqrt(std::log2((double)ns * P)) * gnorm / std::sqrt((double)ns);
    const double zr_scale = ly.zoom * Nf / (2.0 * kPi * ly.alpha);
    f.cflag = (float)(pl->r23_m * zr_scale * 2.0 * etaS);
    f.kflag = (float)(pl->r23_m * etaS);
    pl->fb_sq_grid = sst::fb_squeeze_grid(pl->device);
    pl->fb = true;
    pl->lay.forward_path = SST_PATH_FILTERBANK;
    return true;
}

}  // namespace

namespace sst {
void register_w64_uploader(cudaError_t (*fn)(const float2*)) { w64_uploaders().push_back(fn); }
}  // namespace sst

extern "C" {

const char* sst_status_str(sst_status s) {
    switch (s) {
        case SST_OK: return "SST_OK";
        case SST_E_INVALID_ARGUMENT: return "SST_E_INVALID_ARGUMENT";
        case SST_E_COVERAGE: return "SST_E_COVERAGE";
        case SST_E_UNSUPPORTED: return "SST_E_UNSUPPORTED";
        case SST_E_CUDA: return "SST_E_CUDA";
        case SST_E_OUT_OF_MEMORY: return "SST_E_OUT_OF_MEMORY";
        case SST_E_INTERNAL: return "SST_E_INTERNAL";
    }
    return "SST_E_UNKNOWN";
}

const char* sst_last_error(const sst_plan* plan) {
    return plan ? plan->err.c_str() : g_thread_err.c_str();
}

int32_t sst_abi_version(void) { return SST_ABI_VERSION; }

sst_status sst_gaussian_window(int32_t L, double sigma, int32_t center, double* g, double* gd) {
    if (L < 1 || !std::isfinite(sigma) || sigma <= 0 || !g || !gd)
        return fail(nullptr, SST_E_INVALID_ARGUMENT, "sst_gaussian_window: need L >= 1, sigma > 0, non-NULL outputs");
    const int32_t c = center < 0 ? L / 2 : center;
    if (c >= L) return fail(nullptr, SST_E_INVALID_ARGUMENT, "sst_gaussian_window: centre outside [0, L)");
    const double amp = std::pow(kPi * sigma * sigma, -0.25);           // (pi sigma^2)^(-1/4)
    for (int32_t j = 0; j < L; ++j) {
        const double t = (double)(j - c);
        const double e = amp * std::exp(-(t * t) / (2.0 * sigma * sigma));
        g[j] = e;
        gd[j] = -(t / (sigma * sigma)) * e;                              // analytic g'
    }
    return SST_OK;
}

sst_status sst_params_validate(const sst_params* p) {
    std::string msg;
    sst_status s = validate(p, nullptr, msg);
    if (s != SST_OK) g_thread_err = msg;
    return s;
}

sst_status sst_params_layout(const sst_params* p, sst_layout* out) {
    if (!out) return fail(nullptr, SST_E_INVALID_ARGUMENT, "layout output is NULL");
    std::string msg;
    sst_status s = validate(p, out, msg);
    if (s != SST_OK) g_thread_err = msg;
    return s;
}

sst_status sst_plan_create(const sst_params* p, int device, sst_plan** out) {
    if (!out) return fail(nullptr, SST_E_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    sst_plan* pl = new (std::nothrow) sst_plan();
    if (!pl) return fail(nullptr, SST_E_INTERNAL, "host allocation failed");
    std::string msg;
    sst_status s = validate(p, &pl->lay, msg);
    if (s != SST_OK) { delete pl; return fail(nullptr, s, msg); }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        delete pl;
        return fail(nullptr, ndev == 0 ? SST_E_CUDA : SST_E_INVALID_ARGUMENT, "no such CUDA device");
    }
    pl->p = *p;
    pl->device = device;
    const int32_t L = pl->lay.win_len, c = pl->lay.center, H = pl->lay.hop, Nf = pl->lay.nfft, z = pl->lay.zoom;
    const int64_t N = pl->lay.n;
    pl->g.assign(p->g, p->g + L);
    pl->gd.assign(p->gd, p->gd + L);
    pl->p.g = nullptr;
    pl->p.gd = nullptr;
    pl->gamma_abs = pl->lay.gamma_abs;
    {
        double sg = 0, sg2 = 0;
        for (double v : pl->g) { sg += v; sg2 += v * v; }
        pl->cst = (p->flags & SST_DISCRETE_CONSTANT) ? pl->g[c] * sg / sg2 : std::sqrt(2.0);   // Eq. 24 / R15
    }
    DeviceGuard guard(device);
    if ((s = ensure_w64(device, msg)) != SST_OK) { delete pl; return fail(nullptr, s, msg); }

    const double alpha = pl->lay.alpha;
    // tw[k1 * N2 + t] = W_N^{t k1} (four-step twiddle, laid out so a warp's lanes t read
    // consecutive entries).  Inverse phase exp(+2 pi i b tau/(z N)) of residue b at output
    // p = col + 64 k2 (tau = p, or p - N where the window wraps): phz[b][col] * phz[b][64 + w N2 + k2]
    // with phz[b][col] = e(b col), phz[b][64 + k2] = e(64 b k2), phz[b][64 + N2 + k2] = e(b (64 k2 - N)),
    // e(x) = exp(2 pi i x/(z N)); all rounded once from fp64.
    const int32_t N2 = Nf / 64;
    const int32_t PH = 64 + 2 * N2;
    std::vector<float2> taps(L), tw(Nf), phz((size_t)z * PH);
    for (int32_t j = 0; j < L; ++j) taps[j] = make_float2((float)pl->g[j], (float)(alpha * pl->gd[j]));
    for (int32_t k1 = 0; k1 < 64; ++k1)
        for (int32_t t = 0; t < N2; ++t) {
            const double a = -2.0 * kPi * (double)((int64_t)t * k1 % Nf) / Nf;
            tw[(size_t)k1 * N2 + t] = make_float2((float)std::cos(a), (float)std::sin(a));
        }
    const int64_t zN = (int64_t)z * Nf;
    auto ez = [&](int64_t x) {
        const int64_t e = ((x % zN) + zN) % zN;
        const double a = 2.0 * kPi * (double)e / (double)zN;
        return make_float2((float)std::cos(a), (float)std::sin(a));
    };
    for (int32_t b = 0; b < z; ++b) {
        for (int32_t col = 0; col < 64; ++col) phz[(size_t)b * PH + col] = ez((int64_t)b * col);
        for (int32_t k2 = 0; k2 < N2; ++k2) {
            phz[(size_t)b * PH + 64 + k2] = ez((int64_t)b * 64 * k2);
            phz[(size_t)b * PH + 64 + N2 + k2] = ez((int64_t)b * (64 * k2 - Nf));
        }
    }
    // 1/(C d[n]): head [0, n_head), tail [N - n_tail, N), interior periodic in (n + c) mod H
    pl->n_head = (int32_t)std::min<int64_t>(N, L);
    pl->n_tail = (int32_t)std::min<int64_t>(N, (int64_t)L + H);
    std::vector<float> head(pl->n_head), tail(pl->n_tail), per(H);
    for (int32_t n = 0; n < pl->n_head; ++n) head[n] = (float)(1.0 / (pl->cst * diag_at(pl->g, n, N, H, c)));
    for (int32_t i = 0; i < pl->n_tail; ++i)
        tail[i] = (float)(1.0 / (pl->cst * diag_at(pl->g, N - pl->n_tail + i, N, H, c)));
    for (int32_t i = 0; i < H; ++i) {
        double d = 0;
        for (int32_t j = i; j < L; j += H) d += pl->g[j] * pl->g[j];
        per[i] = (float)(1.0 / (pl->cst * d));
    }
    std::vector<double2> taps64(L), tw64(Nf);
    for (int32_t j = 0; j < L; ++j) taps64[j] = make_double2(pl->g[j], pl->gd[j]);
    for (int32_t e = 0; e < Nf; ++e) {
        const double a = -2.0 * kPi * (double)e / Nf;
        tw64[e] = make_double2(std::cos(a), std::sin(a));
    }
    if (const char* nr = std::getenv("SST_NO_REDECIDE")) pl->redecide = !(nr[0] == '1');
    if (const char* mm = std::getenv("SST_R23_M")) { const double v = std::atof(mm); if (v > 0) pl->r23_m = v; }
    std::vector<float> gwin(L);
    for (int32_t j = 0; j < L; ++j) gwin[j] = (float)(pl->g[j] / Nf);
    if ((s = upload(pl, &pl->d_taps, taps)) != SST_OK || (s = upload(pl, &pl->d_tw, tw)) != SST_OK ||
        (s = upload(pl, &pl->d_gwin, gwin)) != SST_OK ||
        (s = upload(pl, &pl->d_taps64, taps64)) != SST_OK || (s = upload(pl, &pl->d_tw64, tw64)) != SST_OK ||
        (s = upload(pl, &pl->d_phz, phz)) != SST_OK || (s = upload(pl, &pl->d_inv_head, head)) != SST_OK ||
        (s = upload(pl, &pl->d_inv_tail, tail)) != SST_OK || (s = upload(pl, &pl->d_inv_per, per)) != SST_OK) {
        msg = pl->err;
        delete pl;
        return fail(nullptr, s, msg);
    }
    cudaError_t ce = cudaMalloc((void**)&pl->d_absmax, sizeof(float));
    if (ce != cudaSuccess) { delete pl; cudaGetLastError(); return fail(nullptr, SST_E_OUT_OF_MEMORY, "cudaMalloc absmax"); }
    ce = cudaMalloc((void**)&pl->d_r23, 2 * sizeof(unsigned long long));
    if (ce == cudaSuccess) ce = cudaMemset(pl->d_r23, 0, 2 * sizeof(unsigned long long));
    if (ce != cudaSuccess) { delete pl; cudaGetLastError(); return fail(nullptr, SST_E_OUT_OF_MEMORY, "cudaMalloc counters"); }
    if (Nf > sst::kMaxFusedNfft) {
        // multi-pass path: W_N table and scratch for a bounded chunk of frames (kMpScratch per buffer)
        pl->mp = true;
        pl->lay.forward_path = SST_PATH_MULTIPASS;
        pl->lay.inverse_path = SST_IPATH_MULTIPASS;
        std::vector<float2> twN(Nf);
        for (int32_t k = 0; k < Nf; ++k) {
            const double a = -2.0 * kPi * k / Nf;
            twN[k] = make_float2((float)std::cos(a), (float)std::sin(a));
        }
        if ((s = upload(pl, &pl->d_twN, twN)) != SST_OK) { msg = pl->err; delete pl; return fail(nullptr, s, msg); }
        constexpr int64_t kMpScratch = 128ll << 20;
        const int64_t F = pl->lay.frames, per = (int64_t)Nf * 8;
        pl->mp_fwd_frames = std::max<int64_t>(1, std::min<int64_t>(F, kMpScratch / per));
        pl->mp_inv_pairs = std::max<int64_t>(1, std::min<int64_t>((F + 1) / 2, kMpScratch / (per * z)));
        const size_t elems = (size_t)std::max<int64_t>(pl->mp_fwd_frames, pl->mp_inv_pairs * z) * Nf;
        if (cudaMalloc((void**)&pl->d_mp0, elems * sizeof(float2)) != cudaSuccess ||
            cudaMalloc((void**)&pl->d_mp1, elems * sizeof(float2)) != cudaSuccess ||
            cudaMalloc((void**)&pl->d_wf, sizeof(float) * (size_t)(2 * pl->mp_inv_pairs) * L) != cudaSuccess ||
            cudaMalloc((void**)&pl->d_mpl, sizeof(int32_t) * (size_t)pl->mp_fwd_frames * (Nf / 2 + 1)) != cudaSuccess) {
            cudaGetLastError();
            delete pl;
            return fail(nullptr, SST_E_OUT_OF_MEMORY, "cudaMalloc multi-pass scratch");
        }
    } else {
        pl->fwd_grid = sst::forward_max_grid(Nf, L, H, device);
        // R23 deferral: a queue of up to 2^22 flagged bins per chunk of 2^20 frames (measured rates:
        // 0.01-1.3 per frame on C2-C5, ~20 on C1), split into one region per CTA; a CTA whose region is
        // full re-decides inline
        pl->gq_cap = 1u << 22;
        const size_t words = (size_t)((std::min<int64_t>(pl->lay.frames, kR23Chunk) + 31) / 32);
        if (cudaMalloc((void**)&pl->d_gq, sizeof(int4) * pl->gq_cap) != cudaSuccess ||
            cudaMalloc((void**)&pl->d_gctr, (1 + (size_t)std::max(1, pl->fwd_grid)) * sizeof(unsigned int)) != cudaSuccess ||
            cudaMalloc((void**)&pl->d_dirty_bits, sizeof(unsigned int) * words) != cudaSuccess ||
            cudaMalloc((void**)&pl->d_dirty_list, sizeof(int) * pl->gq_cap) != cudaSuccess) {
            cudaGetLastError();
            delete pl;
            return fail(nullptr, SST_E_OUT_OF_MEMORY, "cudaMalloc R23 queue");
        }
        pl->inv_grid = sst::inverse_max_grid(Nf, H, L, z, device);
        // narrow-band inverse where it applies (SST_INV_NB=0: the residue-split kernel, A/B and tests)
        const char* nbe = std::getenv("SST_INV_NB");
        if (!(nbe && nbe[0] == '0') &&
            sst::inv_nb_applicable(Nf, L, pl->lay.center, H, z, pl->lay.k1, pl->lay.bins))
            pl->inv_grid_nb = sst::inverse_nb_max_grid(Nf, H, L, z, pl->lay.k1, pl->lay.bins, device);
        pl->lay.inverse_path = pl->inv_grid_nb > 0 ? SST_IPATH_NARROWBAND : SST_IPATH_RESIDUE;
        const int32_t seam_len = std::max(0, L - H);
        if (seam_len > 0) {
            ce = cudaMalloc((void**)&pl->d_seam,
                            sizeof(float) * (size_t)std::max(pl->inv_grid, pl->inv_grid_nb) * 2 * seam_len);
            if (ce != cudaSuccess) { delete pl; cudaGetLastError(); return fail(nullptr, SST_E_OUT_OF_MEMORY, "cudaMalloc seams"); }
        }
        if (pl->fwd_grid <= 0 || pl->inv_grid <= 0) { delete pl; return fail(nullptr, SST_E_CUDA, "occupancy query failed"); }
    }
    if (!pl->mp) setup_filterbank(pl);
    pl->err.clear();
    if (pl->lay.warnings) {
        char buf[512];
        std::string w = "warning:";
        if (pl->lay.warnings & SST_WARN_EQ37) {
            std::snprintf(buf, sizeof buf,
                          " df = %.4g Hz >= 1.5 sigma_f = %.4g Hz (Eq. 37, P:L353), i.e. H_f = %.4g >= %.4g (Eq. 38, P:L357):"
                          " reassignment no longer concentrates, SST degenerates to the STFT;",
                          pl->lay.df_hz, pl->lay.df_eq37_hz, pl->lay.hf, pl->lay.hf_bound);
            w += buf;
        }
        if (pl->lay.warnings & SST_WARN_EQ46) {
            std::snprintf(buf, sizeof buf, " df = %.4g Hz >= sqrt(2) sigma_f = %.4g Hz, H_f = %.4g >= %.4g (Eq. 46, P:L413)",
                          pl->lay.df_hz, pl->lay.df_eq46_hz, pl->lay.hf, pl->lay.hf_bound46);
            w += buf;
        }
        pl->err = w;
    }
    *out = pl;
    return SST_OK;
}

sst_status sst_plan_layout(const sst_plan* plan, sst_layout* out) {
    if (!plan || !out) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan or output");
    *out = plan->lay;
    out->gamma_abs = plan->gamma_abs;
    return SST_OK;
}

sst_status sst_plan_set_gamma(sst_plan* plan, double gamma_abs) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    if (!std::isfinite(gamma_abs) || gamma_abs < 0) return fail(plan, SST_E_INVALID_ARGUMENT, "gamma must be finite and >= 0");
    plan->gamma_abs = gamma_abs;
    plan->p.flags &= ~(uint32_t)SST_GAMMA_RELATIVE;
    return SST_OK;
}

sst_status sst_plan_set_absmax(sst_plan* plan, const float* absmax_device) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    plan->ext_absmax = absmax_device;
    return SST_OK;
}

sst_status sst_plan_counters(sst_plan* plan, uint64_t* out) {
    if (!plan || !out) return fail(plan, SST_E_INVALID_ARGUMENT, "NULL plan or out");
    DeviceGuard guard(plan->device);
    unsigned long long h[2] = {0, 0};
    sst_status s = cuda_status(plan, cudaMemcpy(h, plan->d_r23, sizeof h, cudaMemcpyDeviceToHost), "counters");
    out[0] = h[0];
    out[1] = h[1];
    return s;
}

void sst_plan_destroy(sst_plan* plan) { delete plan; }

// f3b forward: per chunk of frames, the filter-bank transform (S, S' planes of the band's source
// bins), the decision + exact squeeze per frame (flagged bins queued, R23), the fp64 re-decisions and
// a list-mode re-squeeze of the frames whose target changed
static sst_status run_forward_fb(sst_plan* plan, const sst::FwdArgs& a, cudaStream_t st) {
    for (int64_t c0 = a.frame_begin; c0 < a.frame_end; c0 += plan->fb_chunk) {
        sst::FwdArgs b = a;
        b.frame_begin = c0;
        b.frame_end = std::min<int64_t>(a.frame_end, c0 + plan->fb_chunk);
        b.T = a.T + (c0 - a.frame_begin) * a.ldT;
        const int64_t n = b.frame_end - b.frame_begin;
        sst::FbArgs f = plan->fbt;
        f.x = b.x;
        f.x_off = b.x_off;
        f.x_len = b.x_len;
        f.n = b.n;
        f.frame_begin = b.frame_begin;
        f.frame_end = b.frame_end;
        sst_status s = cuda_status(plan, sst::launch_fb_transform(f, st), "filter-bank transform");
        if (s != SST_OK) return s;
        const int grid = (int)std::min<int64_t>(plan->fb_sq_grid, (n + 7) / 8);
        const bool defer = b.redecide && plan->d_gq;
        if (defer) {
            s = cuda_status(plan, cudaMemsetAsync(plan->d_gctr, 0, sizeof(unsigned int), st), "memset");
            if (s == SST_OK)
                s = cuda_status(plan, cudaMemsetAsync(plan->d_dirty_bits, 0, sizeof(unsigned int) * (size_t)((n + 31) / 32), st),
                                "memset");
            if (s != SST_OK) return s;
            b.gq = plan->d_gq;
            b.gq_n = plan->d_gctr;
            b.gq_counts = plan->d_gctr + 1;
            b.gq_cap = plan->gq_cap;
            b.gq_ctas = grid;
        }
        s = cuda_status(plan, sst::launch_fb_squeeze(f, b, grid, st), "filter-bank squeeze");
        if (s != SST_OK || !defer) {
            if (s != SST_OK) return s;
            continue;
        }
        s = cuda_status(plan, sst::launch_redecide(b, sst::kModeForward, plan->d_dirty_bits, plan->d_dirty_list, st),
                        "redecide launch");
        if (s != SST_OK) return s;
        sst::FwdArgs r = b;
        r.gq = nullptr;
        r.flist = plan->d_dirty_list;
        r.flist_n = plan->d_gctr;
        s = cuda_status(plan, sst::launch_fb_squeeze(f, r, plan->fb_sq_grid, st), "filter-bank repair");
        if (s != SST_OK) return s;
    }
    return SST_OK;
}

static sst_status run_forward_mode(sst_plan* plan, int mode, const float* x, int64_t x_off, int64_t x_len, int64_t fb,
                                   int64_t fe, sst::FwdArgs& a, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (mode != sst::kModeAbsmax && (plan->p.flags & SST_GAMMA_RELATIVE)) {
        if (plan->ext_absmax) {
            a.absmax_dev = plan->ext_absmax;
        } else {
            sst::FwdArgs m = a;
            m.absmax_out = plan->d_absmax;
            m.redecide = 0;
            sst_status s = cuda_status(plan, cudaMemsetAsync(plan->d_absmax, 0, sizeof(float), st), "memset");
            if (s != SST_OK) return s;
            s = cuda_status(plan, launch_fwd_any(plan, m, sst::kModeAbsmax, st), "absmax launch");
            if (s != SST_OK) return s;
            a.absmax_dev = plan->d_absmax;
        }
    }
    (void)x; (void)x_off; (void)x_len;
    if (plan->fb && mode == sst::kModeForward) return run_forward_fb(plan, a, st);
    const int64_t nfr = a.frame_end - a.frame_begin;
    const bool defer = !plan->mp && a.redecide && plan->d_gq &&
                       (mode == sst::kModeForward || mode == sst::kModeTargets);
    if (!defer) return cuda_status(plan, launch_fwd_any(plan, a, mode, st), "forward launch");
    // R23 deferred, per chunk of frames: forward (fp32 decisions, flagged bins queued) -> fp64
    // re-decisions -> repair of the rows whose decision changed (forward) / fp64 targets (targets)
    const int64_t K = plan->lay.nfft / 2 + 1;
    for (int64_t c0 = a.frame_begin; c0 < a.frame_end; c0 += kR23Chunk) {
        sst::FwdArgs b = a;
        b.frame_begin = c0;
        b.frame_end = std::min<int64_t>(a.frame_end, c0 + kR23Chunk);
        const int64_t off = c0 - a.frame_begin, n = b.frame_end - b.frame_begin;
        if (b.T) b.T += off * a.ldT;
        if (b.lout) b.lout += off * K;
        const int grid = fwd_grid_for(plan, n);
        sst_status s = cuda_status(plan, cudaMemsetAsync(plan->d_gctr, 0, sizeof(unsigned int), st), "memset");
        if (s == SST_OK && mode == sst::kModeForward)
            s = cuda_status(plan, cudaMemsetAsync(plan->d_dirty_bits, 0, sizeof(unsigned int) * (size_t)((n + 31) / 32), st),
                            "memset");
        if (s != SST_OK) return s;
        b.gq = plan->d_gq;
        b.gq_n = plan->d_gctr;
        b.gq_counts = plan->d_gctr + 1;
        b.gq_cap = plan->gq_cap;
        b.gq_ctas = grid;
        s = cuda_status(plan, sst::launch_forward(b, mode, grid, st), "forward launch");
        if (s != SST_OK) return s;
        s = cuda_status(plan, sst::launch_redecide(b, mode, plan->d_dirty_bits, plan->d_dirty_list, st), "redecide launch");
        if (s != SST_OK) return s;
        if (mode != sst::kModeForward) continue;
        sst::FwdArgs r = b;
        r.gq = nullptr;
        r.flist = plan->d_dirty_list;
        r.flist_n = plan->d_gctr;
        s = cuda_status(plan, sst::launch_forward(r, mode, plan->fwd_grid, st), "repair launch");
        if (s != SST_OK) return s;
    }
    return SST_OK;
}

sst_status sst_forward(sst_plan* plan, const float* x, int64_t x_off, int64_t x_len, int64_t frame_begin,
                       int64_t frame_end, float* T, int64_t ldT, void* stream) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    if (!x || !T) return fail(plan, SST_E_INVALID_ARGUMENT, "NULL x or T");
    sst_status s = check_frames(plan, frame_begin, frame_end);
    if (s != SST_OK) return s;
    if (ldT < plan->lay.bins) return fail(plan, SST_E_INVALID_ARGUMENT, "ldT < B");
    if (x_len < 0 || !covers_input(plan, x_off, x_len, frame_begin, frame_end))
        return fail(plan, SST_E_INVALID_ARGUMENT, "x slice does not cover the frames' samples");
    DeviceGuard guard(plan->device);
    sst::FwdArgs a = fwd_args(plan, x, x_off, x_len, frame_begin, frame_end);
    a.T = reinterpret_cast<float2*>(T);
    a.ldT = ldT;
    return run_forward_mode(plan, sst::kModeForward, x, x_off, x_len, frame_begin, frame_end, a, stream);
}

sst_status sst_stft(sst_plan* plan, const float* x, int64_t x_off, int64_t x_len, int64_t fb, int64_t fe, float* S,
                    float* Sd, void* stream) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    if (!x || !S || !Sd) return fail(plan, SST_E_INVALID_ARGUMENT, "NULL pointer");
    sst_status s = check_frames(plan, fb, fe);
    if (s != SST_OK) return s;
    if (x_len < 0 || !covers_input(plan, x_off, x_len, fb, fe))
        return fail(plan, SST_E_INVALID_ARGUMENT, "x slice does not cover the frames' samples");
    DeviceGuard guard(plan->device);
    sst::FwdArgs a = fwd_args(plan, x, x_off, x_len, fb, fe);
    a.S = reinterpret_cast<float2*>(S);
    a.Sd = reinterpret_cast<float2*>(Sd);
    a.gamma2x4 = -1.0f;   // report every bin
    a.redecide = 0;
    a.src_lo = 0;
    a.src_hi = plan->lay.nfft / 2 + 1;
    return cuda_status(plan, launch_fwd_any(plan, a, sst::kModeStft, (cudaStream_t)stream),
                       "stft launch");
}

sst_status sst_stft_band(sst_plan* plan, const float* x, int64_t x_off, int64_t x_len, int64_t fb, int64_t fe, float* S,
                         float* Sd, void* stream) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    if (!plan->fb) return fail(plan, SST_E_UNSUPPORTED, "the plan does not use the filter-bank forward");
    if (!x || !S || !Sd) return fail(plan, SST_E_INVALID_ARGUMENT, "NULL pointer");
    sst_status s = check_frames(plan, fb, fe);
    if (s != SST_OK) return s;
    if (x_len < 0 || !covers_input(plan, x_off, x_len, fb, fe))
        return fail(plan, SST_E_INVALID_ARGUMENT, "x slice does not cover the frames' samples");
    DeviceGuard guard(plan->device);
    sst::FbArgs f = plan->fbt;
    f.x = x;
    f.x_off = x_off;
    f.x_len = x_len;
    f.n = plan->lay.n;
    f.frame_begin = fb;
    f.frame_end = fe;
    f.S = reinterpret_cast<float2*>(S);
    f.Sd = reinterpret_cast<float2*>(Sd);
    f.eta = nullptr;
    return cuda_status(plan, sst::launch_fb_transform(f, (cudaStream_t)stream), "filter-bank transform");
}

sst_status sst_targets(sst_plan* plan, const float* x, int64_t x_off, int64_t x_len, int64_t fb, int64_t fe, int32_t* l,
                       void* stream) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    if (!x || !l) return fail(plan, SST_E_INVALID_ARGUMENT, "NULL pointer");
    sst_status s = check_frames(plan, fb, fe);
    if (s != SST_OK) return s;
    if (x_len < 0 || !covers_input(plan, x_off, x_len, fb, fe))
        return fail(plan, SST_E_INVALID_ARGUMENT, "x slice does not cover the frames' samples");
    DeviceGuard guard(plan->device);
    sst::FwdArgs a = fwd_args(plan, x, x_off, x_len, fb, fe);
    a.lout = l;
    return run_forward_mode(plan, sst::kModeTargets, x, x_off, x_len, fb, fe, a, stream);
}

sst_status sst_absmax(sst_plan* plan, const float* x, int64_t x_off, int64_t x_len, int64_t fb, int64_t fe, float* out,
                      void* stream) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    if (!x || !out) return fail(plan, SST_E_INVALID_ARGUMENT, "NULL pointer");
    sst_status s = check_frames(plan, fb, fe);
    if (s != SST_OK) return s;
    if (x_len < 0 || !covers_input(plan, x_off, x_len, fb, fe))
        return fail(plan, SST_E_INVALID_ARGUMENT, "x slice does not cover the frames' samples");
    DeviceGuard guard(plan->device);
    cudaStream_t st = (cudaStream_t)stream;
    s = cuda_status(plan, cudaMemsetAsync(out, 0, sizeof(float), st), "memset");
    if (s != SST_OK) return s;
    sst::FwdArgs a = fwd_args(plan, x, x_off, x_len, fb, fe);
    a.absmax_out = out;
    a.gamma2x4 = -1.0f;
    a.redecide = 0;
    return cuda_status(plan, launch_fwd_any(plan, a, sst::kModeAbsmax, st), "absmax launch");
}

static sst::InvArgs inv_args(const sst_plan* pl, const float* T, int64_t ldT, int64_t fb, int64_t fe, float* y,
                             int64_t y_off, int64_t y_len, int normalize, int* grid, bool allow_nb = true) {
    sst::InvArgs a{};
    a.T = reinterpret_cast<const float2*>(T);
    a.ldT = ldT;
    a.n = pl->lay.n;
    a.frame_begin = fb;
    a.frame_end = fe;
    a.hop = pl->lay.hop;
    a.L = pl->lay.win_len;
    a.c = pl->lay.center;
    a.nfft = pl->lay.nfft;
    a.zoom = pl->lay.zoom;
    a.k1 = pl->lay.k1;
    a.bins = pl->lay.bins;
    a.taps = pl->d_taps;
    a.gwin = pl->d_gwin;
    a.tw = pl->d_tw;
    a.phz = pl->d_phz;
    a.inv_n = (float)(1.0 / pl->lay.nfft);
    a.y = y;
    a.y_off = y_off;
    a.y_len = y_len;
    a.normalize = normalize;
    a.out_scale = 1.0f;
    a.inv_head = pl->d_inv_head;
    a.n_head = pl->n_head;
    a.inv_tail = pl->d_inv_tail;
    a.n_tail = pl->n_tail;
    a.inv_per = pl->d_inv_per;
    a.seam = pl->d_seam;
    a.seam_len = std::max(0, pl->lay.win_len - pl->lay.hop);
    a.lay = sst::inv_layout(pl->lay.nfft / 64, pl->lay.win_len, pl->lay.hop, pl->lay.zoom);
    a.nb = (allow_nb && pl->inv_grid_nb > 0) ? 1 : 0;
    if (a.nb) a.lay = sst::inv_nb_layout(pl->lay.nfft / 64, pl->lay.win_len, pl->lay.hop, pl->lay.zoom, pl->lay.bins);
    const int ctas = a.nb ? pl->inv_grid_nb : pl->inv_grid;
    const int64_t F = fe - fb;
    const int64_t min_fpc = (pl->lay.win_len + pl->lay.hop - 1) / pl->lay.hop;
    int64_t fpc = (F + ctas - 1) / ctas;
    if (fpc < min_fpc) fpc = min_fpc;
    a.frames_per_cta = fpc;
    *grid = (int)((F + fpc - 1) / fpc);
    return a;
}

// plain STFT synthesis (Eq. 10-11): the inverse kernel on the full one-sided band, z = 1,
// with the normalisation 1/(C d) rescaled by C (tables hold 1/(C d[n]))
static sst::InvArgs istft_args(const sst_plan* pl, const float* S, int64_t ldS, float* y, int* grid) {
    sst::InvArgs a = inv_args(pl, S, ldS, 0, pl->lay.frames, y, 0, pl->lay.n, 1, grid, false);
    a.zoom = 1;
    a.k1 = 0;
    a.bins = pl->lay.nfft / 2 + 1;
    a.out_scale = (float)pl->cst;
    a.lay = sst::inv_layout(pl->lay.nfft / 64, pl->lay.win_len, pl->lay.hop, 1);
    return a;
}

static sst_status run_inverse(sst_plan* plan, const float* T, int64_t ldT, int64_t fb, int64_t fe, float* y, int64_t y_off,
                              int64_t y_len, int normalize, void* stream, const int32_t* zone_path = nullptr,
                              int32_t zone_half = 0, int32_t zone_keep = 1) {
    if (plan->mp) {
        cudaStream_t st = (cudaStream_t)stream;
        sst_status s = SST_OK;
        if (normalize) s = cuda_status(plan, cudaMemsetAsync(y, 0, sizeof(float) * (size_t)y_len, st), "memset");
        if (s != SST_OK) return s;
        s = cuda_status(plan, mp_inverse_accumulate(plan, reinterpret_cast<const float2*>(T), ldT, fb, fe, plan->lay.k1,
                                                    plan->lay.bins, plan->lay.zoom, y, y_off, y_len, st, zone_path,
                                                    zone_half, zone_keep), "inverse launch");
        if (s != SST_OK || !normalize) return s;
        return sst_inverse_finalize(plan, y, y_off, y_len, stream);
    }
    int grid = 0;
    sst::InvArgs a = inv_args(plan, T, ldT, fb, fe, y, y_off, y_len, normalize, &grid, zone_path == nullptr);
    a.zone_path = zone_path;
    a.zone_half = zone_half;
    a.zone_keep = zone_keep;
    cudaStream_t st = (cudaStream_t)stream;
    sst_status s = cuda_status(plan, sst::launch_inverse(a, grid, st), "inverse launch");
    if (s != SST_OK) return s;
    return cuda_status(plan, sst::launch_inverse_seams(a, grid, st), "seam launch");
}

sst_status sst_inverse(sst_plan* plan, const float* T, int64_t ldT, float* y, void* stream) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    if (!T || !y) return fail(plan, SST_E_INVALID_ARGUMENT, "NULL T or y");
    if (ldT < plan->lay.bins) return fail(plan, SST_E_INVALID_ARGUMENT, "ldT < B");
    DeviceGuard guard(plan->device);
    return run_inverse(plan, T, ldT, 0, plan->lay.frames, y, 0, plan->lay.n, 1, stream);
}

sst_status sst_inverse_zone(sst_plan* plan, const float* T, int64_t ldT, const int32_t* path, int32_t half,
                            int32_t keep_inside, float* y, void* stream) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    if (!T || !y || !path) return fail(plan, SST_E_INVALID_ARGUMENT, "NULL T, path or y");
    if (ldT < plan->lay.bins || half < 0) return fail(plan, SST_E_INVALID_ARGUMENT, "ldT < B or half < 0");
    DeviceGuard guard(plan->device);
    return run_inverse(plan, T, ldT, 0, plan->lay.frames, y, 0, plan->lay.n, 1, stream, path, half, keep_inside ? 1 : 0);
}

sst_status sst_inverse_accumulate(sst_plan* plan, const float* T, int64_t ldT, int64_t frame_begin, int64_t frame_end,
                                  float* y, int64_t y_off, int64_t y_len, void* stream) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    if (!T || !y) return fail(plan, SST_E_INVALID_ARGUMENT, "NULL T or y");
    sst_status s = check_frames(plan, frame_begin, frame_end);
    if (s != SST_OK) return s;
    if (ldT < plan->lay.bins) return fail(plan, SST_E_INVALID_ARGUMENT, "ldT < B");
    if (y_len < 0 || !covers_input(plan, y_off, y_len, frame_begin, frame_end))
        return fail(plan, SST_E_INVALID_ARGUMENT, "y span does not cover the frames' reach");
    DeviceGuard guard(plan->device);
    return run_inverse(plan, T, ldT, frame_begin, frame_end, y, y_off, y_len, 0, stream);
}

sst_status sst_istft(sst_plan* plan, const float* S, int64_t ldS, float* y, void* stream) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    if (!S || !y) return fail(plan, SST_E_INVALID_ARGUMENT, "NULL S or y");
    if (ldS < plan->lay.nfft / 2 + 1) return fail(plan, SST_E_INVALID_ARGUMENT, "ldS < N_f/2 + 1");
    DeviceGuard guard(plan->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (plan->mp) {
        const int64_t N = plan->lay.n;
        sst_status s = cuda_status(plan, cudaMemsetAsync(y, 0, sizeof(float) * (size_t)N, st), "memset");
        if (s != SST_OK) return s;
        s = cuda_status(plan, mp_inverse_accumulate(plan, reinterpret_cast<const float2*>(S), ldS, 0, plan->lay.frames, 0,
                                                    plan->lay.nfft / 2 + 1, 1, y, 0, N, st), "istft launch");
        if (s != SST_OK) return s;
        return cuda_status(plan, sst::launch_finalize(y, 0, N, N, plan->lay.hop, plan->lay.center, plan->d_inv_head,
                                                      plan->n_head, plan->d_inv_tail, plan->n_tail, plan->d_inv_per,
                                                      (float)plan->cst, st), "istft finalize");
    }
    int grid = 0;
    sst::InvArgs a = istft_args(plan, S, ldS, y, &grid);
    sst_status s = cuda_status(plan, sst::launch_inverse(a, grid, st), "istft launch");
    if (s != SST_OK) return s;
    return cuda_status(plan, sst::launch_inverse_seams(a, grid, st), "istft seam launch");
}

sst_status sst_renyi(sst_plan* plan, const float* T, int64_t rows, int64_t ldT, double alpha, double* out,
                     void* stream) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    if (!T || !out) return fail(plan, SST_E_INVALID_ARGUMENT, "NULL T or out");
    if (rows < 1 || ldT < plan->lay.bins) return fail(plan, SST_E_INVALID_ARGUMENT, "rows < 1 or ldT < B");
    if (!(alpha > 0.0) || alpha == 1.0 || !std::isfinite(alpha))
        return fail(plan, SST_E_INVALID_ARGUMENT, "alpha must be > 0, finite and != 1 (Eq. 32)");
    DeviceGuard guard(plan->device);
    if (!plan->d_renyi) {
        cudaError_t ce = cudaMalloc((void**)&plan->d_renyi, sizeof(double) * 2 * sst::kRenyiBlocks);
        if (ce != cudaSuccess) { cudaGetLastError(); return fail(plan, SST_E_OUT_OF_MEMORY, "cudaMalloc renyi"); }
    }
    return cuda_status(plan, sst::launch_renyi(reinterpret_cast<const float2*>(T), rows, plan->lay.bins, ldT, alpha,
                                               plan->d_renyi, out, (cudaStream_t)stream), "renyi launch");
}

sst_status sst_ridge_emission(sst_plan* plan, const float* T, int64_t ldT, int64_t rows, double* E,
                              double* floor_out, void* stream) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    if (!T || !E || !floor_out) return fail(plan, SST_E_INVALID_ARGUMENT, "NULL T, E or floor");
    if (rows < 1 || ldT < plan->lay.bins) return fail(plan, SST_E_INVALID_ARGUMENT, "rows < 1 or ldT < B");
    DeviceGuard guard(plan->device);
    if (!plan->d_amax2) {
        cudaError_t ce = cudaMalloc((void**)&plan->d_amax2, sizeof(unsigned long long));
        if (ce != cudaSuccess) { cudaGetLastError(); return fail(plan, SST_E_OUT_OF_MEMORY, "cudaMalloc amax"); }
    }
    return cuda_status(plan, sst::launch_ridge_emission(reinterpret_cast<const float2*>(T), rows, plan->lay.bins, ldT,
                                                        plan->d_amax2, E, floor_out, (cudaStream_t)stream),
                       "emission launch");
}

sst_status sst_ridge(sst_plan* plan, double* E, int64_t rows, double lambda, int32_t count, int32_t suppress,
                     const double* floor_in, int32_t* paths, void* stream) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    if (!E || !floor_in || !paths) return fail(plan, SST_E_INVALID_ARGUMENT, "NULL E, floor or paths");
    if (rows < 1 || count < 1 || suppress < 0 || !(lambda >= 0.0) || !std::isfinite(lambda))
        return fail(plan, SST_E_INVALID_ARGUMENT, "rows >= 1, count >= 1, suppress >= 0, finite lambda >= 0");
    const int cols = plan->lay.bins;
    if (cols > sst::kRidgeMaxCols) return fail(plan, SST_E_UNSUPPORTED, "ridge DP supports B <= 8000");
    DeviceGuard guard(plan->device);
    const size_t need = (size_t)rows * (size_t)cols;
    if (plan->back_elems < need) {
        if (plan->d_back) cudaFree(plan->d_back);
        plan->d_back = nullptr;
        plan->back_elems = 0;
        cudaError_t ce = cudaMalloc((void**)&plan->d_back, sizeof(int32_t) * need);
        if (ce != cudaSuccess) { cudaGetLastError(); return fail(plan, SST_E_OUT_OF_MEMORY, "cudaMalloc backpointers"); }
        plan->back_elems = need;
    }
    return cuda_status(plan, sst::launch_ridge_dp(E, rows, cols, lambda, count, suppress, floor_in, plan->d_back, paths,
                                                  (cudaStream_t)stream), "ridge launch");
}

sst_status sst_zone_mask(sst_plan* plan, float* T, int64_t ldT, int64_t rows, const int32_t* path, int32_t half,
                         int32_t keep_inside, void* stream) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    if (!T || !path) return fail(plan, SST_E_INVALID_ARGUMENT, "NULL T or path");
    if (rows < 1 || ldT < plan->lay.bins || half < 0) return fail(plan, SST_E_INVALID_ARGUMENT, "rows, ldT or half");
    DeviceGuard guard(plan->device);
    return cuda_status(plan, sst::launch_zone_mask(reinterpret_cast<float2*>(T), rows, plan->lay.bins, ldT, path, half,
                                                   keep_inside ? 1 : 0, (cudaStream_t)stream), "zone launch");
}

sst_status sst_mode_full(sst_plan* plan, const float* T, int64_t ldT, int64_t rows, const int32_t* path,
                         int32_t half, float* x, void* stream) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    if (plan->lay.hop != 1) return fail(plan, SST_E_INVALID_ARGUMENT, "Eq. 15 needs H_t = 1 (invalid for downsampled SST, P:L130)");
    if (!T || !path || !x) return fail(plan, SST_E_INVALID_ARGUMENT, "NULL T, path or x");
    if (rows < 1 || ldT < plan->lay.bins || half < 0) return fail(plan, SST_E_INVALID_ARGUMENT, "rows, ldT or half");
    DeviceGuard guard(plan->device);
    const int dc_bin = (plan->lay.k1 == 0) ? 0 : -1;                  // z k1 + l = 0
    const double scale = 2.0 / ((double)plan->lay.nfft * plan->g[plan->lay.center]);
    return cuda_status(plan, sst::launch_mode_full(reinterpret_cast<const float2*>(T), rows, plan->lay.bins, ldT, path,
                                                   half, dc_bin, scale, x, (cudaStream_t)stream), "mode launch");
}

sst_status sst_inverse_finalize(sst_plan* plan, float* y, int64_t y_off, int64_t y_len, void* stream) {
    return sst_inverse_finalize_seam(plan, y, y_off, y_len, nullptr, 0, 0, stream);
}

sst_status sst_inverse_finalize_seam(sst_plan* plan, float* y, int64_t y_off, int64_t y_len, const float* seam,
                                     int64_t seam_off, int64_t seam_len, void* stream) {
    if (!plan) return fail(nullptr, SST_E_INVALID_ARGUMENT, "NULL plan");
    if (!y || y_len < 0) return fail(plan, SST_E_INVALID_ARGUMENT, "NULL y or negative length");
    if (y_off < 0 || y_off + y_len > plan->lay.n) return fail(plan, SST_E_INVALID_ARGUMENT, "y span outside [0, N)");
    if (seam_len < 0 || (seam_len > 0 && (!seam || seam_off < y_off || seam_off + seam_len > y_off + y_len)))
        return fail(plan, SST_E_INVALID_ARGUMENT, "seam span must lie inside the y span");
    DeviceGuard guard(plan->device);
    return cuda_status(plan,
                       sst::launch_finalize(y, y_off, y_len, plan->lay.n, plan->lay.hop, plan->lay.center, plan->d_inv_head,
                                            plan->n_head, plan->d_inv_tail, plan->n_tail, plan->d_inv_per, 1.0f,
                                            (cudaStream_t)stream, seam_len > 0 ? seam : nullptr, seam_off, seam_len),
                       "finalize launch");
}

}  // extern "C"
