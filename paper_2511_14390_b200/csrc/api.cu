// api.cu -- the C ABI of libiirgrad.so (see include/iirgrad.h): host-side
// validation, workspace / tape layout, kernel dispatch and instrumentation.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/iirgrad.h"
#include "lti.cuh"
#include "host.h"
#include "lti_host.cuh"
#include "lti2.cuh"

using namespace iirg;

// ---------------------------------------------------------------- errors ----
static thread_local std::string g_err;
namespace iirg {
iir_status_t fail(iir_status_t st, const std::string& msg) {
    g_err = msg;
    return st;
}
SideStream& side_stream() {
    thread_local SideStream per_dev[64];
    int dev = 0;
    cudaGetDevice(&dev);
    SideStream& s = per_dev[dev & 63];
    if (s.st == nullptr) {
        cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&s.join, cudaEventDisableTiming);
    }
    return s;
}
}  // namespace iirg

// ------------------------------------------------------- instrumentation ----
static const char* kKindNames[K_NUM] = {"lti_prep", "lti_fwd", "lti_bwd", "tv_phi", "tv_chain", "tv_fwd",
                                        "tv_bwd_agg", "tv_bwd", "rec_fwd", "rec_bwd", "state_carry", "tv_fir",
                                        "diag_prep", "diag_agg", "diag_scan", "diag_fwd", "diag_bwd", "diag_red",
                                        "tv_skew", "tv_wagg"};
static std::atomic<int64_t> g_launches{0};
struct ProfRec { int kind; cudaEvent_t e0, e1; };
static std::mutex g_pmu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_pending;
static std::vector<cudaEvent_t> g_pool;
static double g_ms[K_NUM];
static int64_t g_cnt[K_NUM];

static cudaEvent_t ev_get() {
    if (!g_pool.empty()) { cudaEvent_t e = g_pool.back(); g_pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

namespace iirg {
// Under stream capture a plain cudaEventRecord is only a dependency edge: the
// profiling events must be external record nodes to be timestamped at replay.
static unsigned rec_flags(cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    return cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
}
LaunchGuard::LaunchGuard(int k, cudaStream_t s) : kind(k), st(s) {
    std::lock_guard<std::mutex> lk(g_pmu);
    if (g_prof_on) { e0 = ev_get(); e1 = ev_get(); }
    if (e0) cudaEventRecordWithFlags(e0, st, rec_flags(st));
}
iir_status_t LaunchGuard::done() {
    cudaError_t err = cudaGetLastError();
    if (e0) {
        cudaEventRecordWithFlags(e1, st, rec_flags(st));
        std::lock_guard<std::mutex> lk(g_pmu);
        g_pending.push_back({kind, e0, e1});
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (err != cudaSuccess)
        return fail(IIR_ECUDA, std::string(kKindNames[kind]) + " launch failed: " + cudaGetErrorString(err));
    return IIR_OK;
}
}  // namespace iirg

// ------------------------------------------------------------- layout -------
static size_t dsize(int dtype) { return dtype == IIR_F64 ? 8 : 4; }
static int tile_samples(int dtype, int M) {
    const int L = dtype == IIR_F64 ? (M >= IIRG_LONG_CHUNK_M ? Chunk<double, 8>::L : Chunk<double, 1>::L)
                                   : (M >= IIRG_LONG_CHUNK_M ? Chunk<float, 8>::L : Chunk<float, 1>::L);
    return NT * L;
}

static int tab_size(int M) {
    switch (M) {
        case 1: return Tab<1>::SIZE; case 2: return Tab<2>::SIZE; case 3: return Tab<3>::SIZE;
        case 4: return Tab<4>::SIZE; case 5: return Tab<5>::SIZE; case 6: return Tab<6>::SIZE;
        case 7: return Tab<7>::SIZE; case 8: return Tab<8>::SIZE;
    }
    return 0;
}

namespace iirg {
int rec_tile_samples(int dtype, int M);
iir_status_t rec_run(bool fwd, int dtype, int M, const Layout& L, const LtiFwdArgs& fa, const LtiBwdArgs& ba,
                     cudaStream_t st);
}  // namespace iirg

// Engine choice for fp32 TDF-II with fixed coefficients.  The round-2 engine (lti2.cuh:
// persistent warp tiles, TMEM parking, fp32 carries, fused backward) is the default from
// order 4 up; below it the round-1 engine (lti.cuh: one CTA per tile) is faster on the
// measured shapes (B200, graph-timed us/step: C5 M=8 162 vs 216,
// C4 M=4 168 vs 174, C2 M=2 42 vs 33).  IIR_FLAG_ENGINE_V2 / IIR_FLAG_LEGACY_LTI force either one.
static bool v2_capable(const iir_desc_t* d) {
    return d->form == IIR_TDF2 && d->dtype == IIR_F32 &&
           (d->coef_mode == IIR_COEF_SHARED || d->coef_mode == IIR_COEF_PER_SEQ) && d->order >= 1 && d->order <= 8 &&
           !(d->flags & IIR_FLAG_LEGACY_LTI);
}
// Chunk<T, M>::L of the round-1 engine (samples per thread chunk): the DF tape's state grid
static int64_t df_chunk_len(const iir_desc_t* d) {
    return (d->dtype == IIR_F64 ? 16 : 32) * (d->order >= IIRG_LONG_CHUNK_M ? 2 : 1);
}
static_assert(Chunk<float, 1>::L == 32 && Chunk<double, 1>::L == 16, "df_chunk_len");
static_assert(Chunk<float, IIRG_LONG_CHUNK_M>::L == 64 && Chunk<double, IIRG_LONG_CHUNK_M>::L == 32, "df_chunk_len");

static bool use_v2(const iir_desc_t* d) {
    if (!v2_capable(d)) return false;
    if (d->flags & IIR_FLAG_ENGINE_V2) return true;
    return d->order >= 4;
}

static int scan_tile_samples(const iir_desc_t* d) {
    if (use_v2(d)) return v2::tile_samples(d->order);
    return d->form == IIR_SS ? rec_tile_samples(d->dtype, d->order) : tile_samples(d->dtype, d->order);
}

static iir_status_t check_desc(const iir_desc_t* d) {
    if (d == nullptr) return fail(IIR_EINVAL, "desc is NULL");
    if (d->batch < 1) return fail(IIR_EINVAL, "batch must be >= 1");
    if (d->length < 1) return fail(IIR_EINVAL, "length must be >= 1");
    if (d->dtype != IIR_F32 && d->dtype != IIR_F64) return fail(IIR_EINVAL, "dtype must be IIR_F32 or IIR_F64");
    if (d->form != IIR_DF2 && d->form != IIR_TDF2 && d->form != IIR_SS)
        return fail(IIR_EINVAL, "form must be IIR_DF2, IIR_TDF2 or IIR_SS");
    if (d->form == IIR_SS) {
        if (d->coef_mode != IIR_COEF_SHARED && d->coef_mode != IIR_COEF_PER_SEQ)
            return fail(IIR_EUNSUPPORTED, "bare recurrence: A is SHARED or PER_SEQ");
        if (d->order < 1 || d->order > 4) return fail(IIR_EUNSUPPORTED, "bare recurrence: order must be 1..4");
        if ((d->flags & IIR_FLAG_DIAG) && d->order > 4)
            return fail(IIR_EUNSUPPORTED, "Diag-EXT (IIR_FLAG_DIAG): order must be 1..4");
    }
    if (d->flags & IIR_FLAG_THREE_PHASE_REMOVED)
        return fail(IIR_EUNSUPPORTED, "the three-phase LTI schedule was removed (it lost on every measured shape)");
    if ((d->flags & IIR_FLAG_DIAG) && d->form != IIR_SS)
        return fail(IIR_EINVAL, "IIR_FLAG_DIAG applies to the bare recurrence (form IIR_SS)");
    if ((d->flags & IIR_FLAG_PER_SAMPLE_B) && d->coef_mode != IIR_COEF_PER_SAMPLE)
        return fail(IIR_EINVAL, "IIR_FLAG_PER_SAMPLE_B needs IIR_COEF_PER_SAMPLE");
    if (d->coef_mode == IIR_COEF_PER_SAMPLE) {
        if (d->form != IIR_DF2 && d->form != IIR_TDF2)
            return fail(IIR_EUNSUPPORTED, "per-sample coefficients: DF or TDF form");
        if (d->form == IIR_TDF2 && !(d->flags & IIR_FLAG_PER_SAMPLE_B))
            return fail(IIR_EUNSUPPORTED, "per-sample TDF: the general filter only (IIR_FLAG_PER_SAMPLE_B)");
        if (d->order < 1 || d->order > TV_MAX_M) return fail(IIR_EUNSUPPORTED, "per-sample order must be 1..32");
        if (!tv_supported(d->order)) return fail(IIR_EUNSUPPORTED, "per-sample order not compiled in");
        return IIR_OK;
    }
    if (d->coef_mode != IIR_COEF_SHARED && d->coef_mode != IIR_COEF_PER_SEQ)
        return fail(IIR_EINVAL, "coef_mode must be SHARED, PER_SEQ or PER_SAMPLE");
    if (d->order < 1 || d->order > 8) return fail(IIR_EUNSUPPORTED, "order must be 1..8 for LTI filters");
    const int64_t TS = scan_tile_samples(d);
    if ((d->length + TS - 1) / TS > (int64_t(1) << (5 * MAX_LEVELS)))
        return fail(IIR_EUNSUPPORTED, "length exceeds 32^4 tiles per sequence");
    if (d->batch * ((d->length + TS - 1) / TS) >= (int64_t(1) << 31))
        return fail(IIR_EUNSUPPORTED, "batch x tiles exceeds 2^31 CTAs");
    return IIR_OK;
}

static Layout diag_layout(const iir_desc_t* d) {
    Layout L;
    const int M = d->order;
    L.ncoef = d->coef_mode == IIR_COEF_SHARED ? 1 : d->batch;
    L.ntiles = (d->length + diag_chunk() - 1) / diag_chunk();        // chunks per sequence
    L.ntot = L.ntiles * d->batch;
    size_t o = 256;                                                  // (counters block unused; error word)
    L.ws_err = 64;
    L.ws_clear = 256;
    L.ws_part = o; o += al256((size_t)L.ntot * 2 * M * 8);         // chunk aggregates (complex)
    L.ws_part2 = o; o += al256((size_t)L.ntot * 2 * M * 8);        // carries entering each chunk
    L.ws_psi = o; o += al256((size_t)L.ntot * M * M * 8);          // grad_A partial sums per chunk
    L.ws_bytes = o;
    L.tp_tab = 0;
    L.tp_bytes = al256((size_t)L.ncoef * diag_tab_doubles(M) * 8);
    return L;
}

static Layout layout(const iir_desc_t* d) {
    if (d->form == IIR_SS && (d->flags & IIR_FLAG_DIAG)) return diag_layout(d);
    if (d->coef_mode == IIR_COEF_PER_SAMPLE) return tv_layout(d);
    Layout L;
    const int M = d->order;
    const int64_t TS = scan_tile_samples(d);
    const int NGP = d->form == IIR_SS ? M * M : 2 * M + 1;   // coefficient partial sums per tile
    L.ntiles = (d->length + TS - 1) / TS;
    L.ntot = L.ntiles * d->batch;
    L.ncoef = d->coef_mode == IIR_COEF_SHARED ? 1 : d->batch;
    L.nlev = 1;
    while (L.nlev < MAX_LEVELS && (int64_t(1) << (5 * L.nlev)) < L.ntiles) ++L.nlev;
    for (int l = 0; l < MAX_LEVELS; ++l)
        L.nblk[l] = l < L.nlev ? (L.ntiles + (int64_t(1) << (5 * l)) - 1) >> (5 * l) : 0;
    // partial-sum rows per coefficient set: one per tile (the round-2 SHARED path: one per
    // warp of the grid, at most ntot + 63)
    const int64_t per_set = (d->coef_mode == IIR_COEF_SHARED ? L.ntot : L.ntiles) + (d->coef_mode == IIR_COEF_SHARED ? 64 : 0);
    const int64_t ng_set = (per_set + 31) / 32;
    L.ngroups = ng_set * L.ncoef;
    size_t o = 0;
    L.ws_ticket = o; L.ws_done = o + 4; L.ws_epoch = o + 8; L.ws_err = o + 64; o += 256;
    L.ws_gcnt = o; o += al256(L.ngroups * 4);
    L.ws_scnt = o; o += al256(L.ncoef * 4);
    L.ws_clear = o;
    L.ws_sent = o;
    for (int l = 0; l < L.nlev; ++l) { L.ws_agg[l] = o; o += al256(d->batch * L.nblk[l] * M * 8); }
    L.ws_bank = o - L.ws_sent;                           // two banks of look-back slots (epoch parity),
    o += 3 * L.ws_bank;                                  // for the forward and for the backward
    L.ws_sent_bytes = o - L.ws_sent;
    L.ws_part = o; o += al256((L.ntot + 64) * NGP * 8);
    L.ws_part2 = o; o += al256(L.ngroups * NGP * 8);
    L.v2 = use_v2(d);
    L.ws_bytes = o;
    o = 0;
    if (L.v2) {
        L.tp_t64 = o; o += al256((size_t)L.ncoef * v2::tab64_doubles(M) * 8);
        L.tp_t32 = o; o += al256((size_t)L.ncoef * v2::tab32_floats(M) * 4);
        L.tp_tab = L.tp_t64;
        L.tp_u = o;
        L.tp_bytes = o;
        return L;
    }
    L.tp_tab = o; o += al256((size_t)L.ncoef * tab_size(M) * 8);
    L.tp_u = o;                                            // DF: the state entering every chunk
    if (d->form == IIR_DF2) {                              // (B, ceil(T / L), M): M values per L samples
        const int64_t Lc = df_chunk_len(d);
        o += al256((size_t)d->batch * ((d->length + Lc - 1) / Lc) * d->order * dsize(d->dtype));
    }
    L.tp_bytes = o;
    return L;
}

// -------------------------------------------------------------- kernels -----
// Instantiated in lti_<dtype>_<form>.cu (split for parallel compilation).
namespace iirg {
template <typename T, int FORM> iir_status_t run_lti_m(int M, LtiCall& c);
extern template iir_status_t run_lti_m<float, 0>(int, LtiCall&);
extern template iir_status_t run_lti_m<float, 1>(int, LtiCall&);
extern template iir_status_t run_lti_m<double, 0>(int, LtiCall&);
extern template iir_status_t run_lti_m<double, 1>(int, LtiCall&);
}  // namespace iirg

static iir_status_t run_lti_any(LtiCall& c) {
    const iir_desc_t* d = c.d;
    if (d->dtype == IIR_F32)
        return d->form == IIR_DF2 ? run_lti_m<float, 0>(d->order, c) : run_lti_m<float, 1>(d->order, c);
    return d->form == IIR_DF2 ? run_lti_m<double, 0>(d->order, c) : run_lti_m<double, 1>(d->order, c);
}

static unsigned long long* g_trace = nullptr;
// The forward and the backward have separate counters and slot banks, so a
// backward launched with PDL may run its dy-only phases while the forward ends.
static CarryWs carry_ws(const Layout& L, char* w, bool bwd) {
    CarryWs c{};
    const size_t co = bwd ? 16 : 0, bo = bwd ? 2 * L.ws_bank : 0;
    c.ticket = reinterpret_cast<unsigned*>(w + L.ws_ticket + co);
    c.done = reinterpret_cast<unsigned*>(w + L.ws_done + co);
    c.epoch = reinterpret_cast<unsigned*>(w + L.ws_epoch + co);
    c.bank = (int64_t)(L.ws_bank / 8);
    for (int l = 0; l < MAX_LEVELS; ++l) {
        c.agg[l] = l < L.nlev ? reinterpret_cast<double*>(w + L.ws_agg[l] + bo) : nullptr;
        c.nblk[l] = L.nblk[l];
    }
    c.nlev = L.nlev;
    c.err = reinterpret_cast<unsigned*>(w + L.ws_err);
    return c;
}

static iir_status_t ws_reset(const Layout& L, void* ws, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(ws, 0, L.ws_clear, st);
    if (e == cudaSuccess && L.ws_sent_bytes)
        e = cudaMemsetAsync(static_cast<char*>(ws) + L.ws_sent, 0xFF, L.ws_sent_bytes, st);
    if (e != cudaSuccess) return fail(IIR_ECUDA, std::string("workspace memset: ") + cudaGetErrorString(e));
    return IIR_OK;
}

static bool aligned16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ------------------------------------------------------------- C ABI --------
extern "C" {

int iir_abi_version(void) { return IIRGRAD_ABI_VERSION; }
const char* iir_last_error(void) { return g_err.c_str(); }

size_t iir_tape_bytes(const iir_desc_t* d) {
    if (check_desc(d) != IIR_OK) return 0;
    return layout(d).tp_bytes;
}
size_t iir_workspace_bytes(const iir_desc_t* d) {
    if (check_desc(d) != IIR_OK) return 0;
    return layout(d).ws_bytes;
}

iir_status_t iir_workspace_init(const iir_desc_t* d, void* ws, size_t ws_bytes, iir_stream_t stream) {
    iir_status_t s = check_desc(d);
    if (s != IIR_OK) return s;
    const Layout L = layout(d);
    if (ws == nullptr || ws_bytes < L.ws_bytes) return fail(IIR_EWORKSPACE, "workspace missing or too small");
    return ws_reset(L, ws, static_cast<cudaStream_t>(stream));
}

iir_status_t iir_forward(const iir_desc_t* d, const void* b, const void* a, const void* x, const void* zi, void* y,
                         void* zf, void* tape, size_t tape_bytes, void* ws, size_t ws_bytes, iir_stream_t stream) {
    iir_status_t s = check_desc(d);
    if (s != IIR_OK) return s;
    const Layout L = layout(d);
    if (x == nullptr || y == nullptr) return fail(IIR_EINVAL, "x and y must be non-NULL");
    if (a == nullptr) return fail(IIR_EINVAL, "a must be non-NULL");
    if (d->coef_mode == IIR_COEF_PER_SAMPLE && (d->flags & IIR_FLAG_PER_SAMPLE_B)) {
        if (b == nullptr) return fail(IIR_EINVAL, "IIR_FLAG_PER_SAMPLE_B: b (B, T, M+1) must be non-NULL");
    } else if (d->coef_mode == IIR_COEF_PER_SAMPLE || d->form == IIR_SS) {
        if (b != nullptr) return fail(IIR_EINVAL, "per-sample all-pole / bare recurrence: b must be NULL");
    } else if (b == nullptr) {
        return fail(IIR_EINVAL, "b must be non-NULL");
    }
    if (tape == nullptr || tape_bytes < L.tp_bytes) return fail(IIR_EWORKSPACE, "tape missing or too small");
    if (ws == nullptr || ws_bytes < L.ws_bytes) return fail(IIR_EWORKSPACE, "workspace missing or too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    char* w = static_cast<char*>(ws);
    char* t = static_cast<char*>(tape);
    if (!(d->flags & IIR_FLAG_WS_READY)) {
        iir_status_t rs = ws_reset(L, w, st);
        if (rs != IIR_OK) return rs;
    }
    const int W = d->dtype == IIR_F64 ? 2 : 4;
    const int64_t rowlen = d->length * (d->form == IIR_SS ? d->order : 1);
    const bool vec = (rowlen % W == 0) && aligned16(x) && aligned16(y);
    if (d->coef_mode == IIR_COEF_PER_SAMPLE) return tv_forward(d, L, b, a, x, zi, y, zf, t, w, vec, st);
    if (L.v2) {
        v2::Call c{};
        c.st = st;
        c.b = static_cast<const float*>(b);
        c.a = static_cast<const float*>(a);
        c.cstride = d->coef_mode == IIR_COEF_SHARED ? 0 : d->order + 1;
        c.ncoef = L.ncoef;
        c.nlev = L.nlev;
        v2::FwdArgs& f = c.f;
        f.x = static_cast<const float*>(x); f.y = static_cast<float*>(y);
        f.zi = static_cast<const float*>(zi); f.zf = static_cast<float*>(zf);
        f.t32 = reinterpret_cast<const float*>(t + L.tp_t32);
        f.t32_stride = d->coef_mode == IIR_COEF_SHARED ? 0 : (int64_t)v2::tab32_floats(d->order);
        f.t64 = reinterpret_cast<const double*>(t + L.tp_t64);
        f.t64_stride = d->coef_mode == IIR_COEF_SHARED ? 0 : (int64_t)v2::tab64_doubles(d->order);
        f.cw = carry_ws(L, w, false);
        f.B = d->batch; f.T = d->length; f.ntiles = (int)L.ntiles; f.ntot = L.ntot;
        f.vec = (d->length % 4 == 0) && aligned16(x) && aligned16(y);
        f.trace = g_trace;
        return v2::run(true, d->order, c);
    }

    LtiCall c{};
    c.d = d; c.L = &L; c.st = st; c.is_fwd = true; c.b = b; c.a = a;
    LtiFwdArgs& fa = c.fa;
    fa.b = b; fa.a = a; fa.coef_stride = d->coef_mode == IIR_COEF_SHARED ? 0 : d->order + 1;
    fa.x = x; fa.zi = zi; fa.y = y; fa.zf = zf;
    fa.u = d->form == IIR_DF2 ? t + L.tp_u : nullptr;
    fa.tab = reinterpret_cast<const double*>(t + L.tp_tab);
    fa.tab_stride = d->coef_mode == IIR_COEF_SHARED ? 0 : tab_size(d->order);
    fa.cw = carry_ws(L, w, false);
    fa.B = d->batch; fa.Tlen = d->length; fa.ntiles = (int)L.ntiles; fa.vec = vec;
    fa.trace = g_trace;
    fa.span = g_trace == nullptr ? nullptr : g_trace + L.ntot * 16 + 2;   // [prep][fwd][bwd]
    if (d->form == IIR_SS && (d->flags & IIR_FLAG_DIAG))
        return diag_run(true, d, a, x, zi, y, nullptr, nullptr, nullptr, nullptr, nullptr,
                        reinterpret_cast<double*>(t + L.tp_tab), reinterpret_cast<double*>(w + L.ws_part),
                        reinterpret_cast<double*>(w + L.ws_part2), reinterpret_cast<double*>(w + L.ws_psi), st);
    if (d->form == IIR_SS) {
        fa.coef_stride = d->coef_mode == IIR_COEF_SHARED ? 0 : (int64_t)d->order * d->order;
        return rec_run(true, d->dtype, d->order, L, fa, LtiBwdArgs{}, st);
    }
    return run_lti_any(c);
}

iir_status_t iir_backward(const iir_desc_t* d, const void* grad_y, const void* grad_zf, const void* b, const void* a,
                          const void* x, const void* y, const void* zi, const void* tape, size_t tape_bytes,
                          void* grad_x, void* grad_b, void* grad_a, void* grad_zi, void* ws, size_t ws_bytes,
                          iir_stream_t stream) {
    iir_status_t s = check_desc(d);
    if (s != IIR_OK) return s;
    const Layout L = layout(d);
    if (tape == nullptr || tape_bytes < L.tp_bytes) return fail(IIR_EWORKSPACE, "tape missing or too small");
    if (ws == nullptr || ws_bytes < L.ws_bytes) return fail(IIR_EWORKSPACE, "workspace missing or too small");
    if (d->coef_mode != IIR_COEF_PER_SAMPLE && d->form == IIR_TDF2 && (x == nullptr || y == nullptr))
        return fail(IIR_EINVAL, "TDF backward needs the forward's x and y");
    if (d->coef_mode != IIR_COEF_PER_SAMPLE && d->form == IIR_DF2 && x == nullptr)
        return fail(IIR_EINVAL, "DF backward needs the forward's x (u is re-run from the tape's chunk states)");
    if (d->form == IIR_SS && (a == nullptr || y == nullptr))
        return fail(IIR_EINVAL, "bare-recurrence backward needs A and the forward's v");
    if (d->form == IIR_SS && grad_b != nullptr) return fail(IIR_EINVAL, "bare recurrence: grad_b must be NULL");
    if (d->coef_mode == IIR_COEF_PER_SAMPLE && (d->flags & IIR_FLAG_PER_SAMPLE_B) && b == nullptr)
        return fail(IIR_EINVAL, "IIR_FLAG_PER_SAMPLE_B backward needs the forward's b");
    if (d->coef_mode == IIR_COEF_PER_SAMPLE && !(d->flags & IIR_FLAG_PER_SAMPLE_B) && grad_b != nullptr)
        return fail(IIR_EINVAL, "per-sample all-pole: grad_b must be NULL");
    if (d->coef_mode == IIR_COEF_PER_SAMPLE && (a == nullptr || y == nullptr))
        return fail(IIR_EINVAL, "per-sample backward needs the forward's a and y");
    if (d->coef_mode == IIR_COEF_PER_SAMPLE && d->form == IIR_TDF2 && x == nullptr)
        return fail(IIR_EINVAL, "per-sample TDF backward needs the forward's x");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    char* w = static_cast<char*>(ws);
    const char* t = static_cast<const char*>(tape);
    if (!(d->flags & IIR_FLAG_WS_READY)) {
        iir_status_t rs = ws_reset(L, w, st);
        if (rs != IIR_OK) return rs;
    }
    const int W = d->dtype == IIR_F64 ? 2 : 4;
    const int64_t rowlen = d->length * (d->form == IIR_SS ? d->order : 1);
    const bool vec = (rowlen % W == 0) && aligned16(grad_y) && aligned16(x) && aligned16(y) &&
                     aligned16(grad_x);
    if (d->coef_mode == IIR_COEF_PER_SAMPLE)
        return tv_backward(d, L, grad_y, grad_zf, b, a, y, zi, t, grad_x, grad_b, grad_a, grad_zi, w, vec, st, x);
    if (L.v2) {
        v2::Call c{};
        c.st = st;
        c.ncoef = L.ncoef;
        c.nlev = L.nlev;
        v2::BwdArgs& g = c.g;
        g.gy = static_cast<const float*>(grad_y); g.gzf = static_cast<const float*>(grad_zf);
        g.x = static_cast<const float*>(x); g.y = static_cast<const float*>(y);
        g.gx = static_cast<float*>(grad_x); g.gzi = static_cast<float*>(grad_zi);
        g.gb = static_cast<float*>(grad_b); g.ga = static_cast<float*>(grad_a);
        g.want_coef = (grad_b != nullptr || grad_a != nullptr);
        g.t32 = reinterpret_cast<const float*>(t + L.tp_t32);
        g.t32_stride = d->coef_mode == IIR_COEF_SHARED ? 0 : (int64_t)v2::tab32_floats(d->order);
        g.t64 = reinterpret_cast<const double*>(t + L.tp_t64);
        g.t64_stride = d->coef_mode == IIR_COEF_SHARED ? 0 : (int64_t)v2::tab64_doubles(d->order);
        g.cw = carry_ws(L, w, true);
        g.partial = reinterpret_cast<double*>(w + L.ws_part);
        g.partial2 = reinterpret_cast<double*>(w + L.ws_part2);
        g.gcnt = reinterpret_cast<unsigned*>(w + L.ws_gcnt);
        g.scnt = reinterpret_cast<unsigned*>(w + L.ws_scnt);
        g.ncoef = L.ncoef;
        g.B = d->batch; g.T = d->length; g.ntiles = (int)L.ntiles; g.ntot = L.ntot;
        g.vec = (d->length % 4 == 0) && aligned16(grad_y) && aligned16(x) && aligned16(y) && aligned16(grad_x);
        g.trace = g_trace;
        g.gy_early = (d->flags & IIR_FLAG_GRAD_Y_EARLY) != 0;
        return v2::run(false, d->order, c);
    }

    LtiCall c{};
    c.d = d; c.L = &L; c.st = st; c.is_fwd = false;
    LtiBwdArgs& ba = c.ba;
    ba.gy = grad_y; ba.gzf = grad_zf; ba.x = x; ba.y = y;
    ba.u = d->form == IIR_DF2 ? t + L.tp_u : nullptr;
    ba.zi = zi; ba.gx = grad_x; ba.gzi = grad_zi;
    ba.gb = grad_b; ba.ga = grad_a;
    ba.partial = reinterpret_cast<double*>(w + L.ws_part);
    ba.partial2 = reinterpret_cast<double*>(w + L.ws_part2);
    ba.gcnt = reinterpret_cast<unsigned*>(w + L.ws_gcnt);
    ba.scnt = reinterpret_cast<unsigned*>(w + L.ws_scnt);
    ba.ncoef = L.ncoef;
    ba.want_coef = (grad_b != nullptr || grad_a != nullptr);
    ba.gy_early = (d->flags & IIR_FLAG_GRAD_Y_EARLY) != 0;
    ba.tab = reinterpret_cast<const double*>(t + L.tp_tab);
    ba.tab_stride = d->coef_mode == IIR_COEF_SHARED ? 0 : tab_size(d->order);
    ba.cw = carry_ws(L, w, true);
    ba.B = d->batch; ba.Tlen = d->length; ba.ntiles = (int)L.ntiles; ba.vec = vec;
    ba.trace = g_trace;
    ba.span = g_trace == nullptr ? nullptr : g_trace + L.ntot * 16 + 4;
    (void)b;
    if (d->form == IIR_SS && (d->flags & IIR_FLAG_DIAG))
        return diag_run(false, d, a, nullptr, zi, nullptr, grad_y, y, grad_x, grad_a, grad_zi,
                        reinterpret_cast<double*>(const_cast<char*>(t) + L.tp_tab),
                        reinterpret_cast<double*>(w + L.ws_part), reinterpret_cast<double*>(w + L.ws_part2),
                        reinterpret_cast<double*>(w + L.ws_psi), st);
    if (d->form == IIR_SS) {
        ba.a = a;
        ba.coef_stride = d->coef_mode == IIR_COEF_SHARED ? 0 : (int64_t)d->order * d->order;
        return rec_run(false, d->dtype, d->order, L, LtiFwdArgs{}, ba, st);
    }
    return run_lti_any(c);
}

iir_status_t iir_check_workspace(const iir_desc_t* d, void* ws, size_t ws_bytes, iir_stream_t stream) {
    iir_status_t s = check_desc(d);
    if (s != IIR_OK) return s;
    const Layout L = layout(d);
    if (ws == nullptr || ws_bytes < L.ws_bytes) return fail(IIR_EWORKSPACE, "workspace missing or too small");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    unsigned flag = 0;
    unsigned* p = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + L.ws_err);
    cudaError_t e = cudaMemcpyAsync(&flag, p, sizeof(flag), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(IIR_ECUDA, std::string("iir_check_workspace: ") + cudaGetErrorString(e));
    if (flag != 0) {
        cudaMemsetAsync(p, 0, sizeof(unsigned), st);
        cudaStreamSynchronize(st);
        return fail(IIR_ECUDA, "a look-back wait timed out (outputs of the affected call are NaN)");
    }
    return IIR_OK;
}

int64_t iir_launch_count(void) { return g_launches.load(); }
void iir_debug_trace(void* buf) { g_trace = static_cast<unsigned long long*>(buf); }
int iir_num_kernels(void) { return K_NUM; }
const char* iir_kernel_name(int kind) { return (kind >= 0 && kind < K_NUM) ? kKindNames[kind] : ""; }

void iir_profile_enable(int on) {
    std::lock_guard<std::mutex> lk(g_pmu);
    g_prof_on = on != 0;
}
void iir_profile_reset(void) {
    std::lock_guard<std::mutex> lk(g_pmu);
    for (auto& r : g_pending) { g_pool.push_back(r.e0); g_pool.push_back(r.e1); }
    g_pending.clear();
    for (int k = 0; k < K_NUM; ++k) { g_ms[k] = 0; g_cnt[k] = 0; }
}
int iir_profile_query(int kind, double* total_ms, int64_t* launches) {
    if (kind < 0 || kind >= K_NUM) return 1;
    std::lock_guard<std::mutex> lk(g_pmu);
    for (auto& r : g_pending) {
        float ms = 0.f;
        cudaEventSynchronize(r.e1);
        if (cudaEventElapsedTime(&ms, r.e0, r.e1) != cudaSuccess) { ms = 0.f; (void)cudaGetLastError(); }
        g_ms[r.kind] += ms;
        g_cnt[r.kind] += 1;
        g_pool.push_back(r.e0);
        g_pool.push_back(r.e1);
    }
    g_pending.clear();
    if (total_ms) *total_ms = g_ms[kind];
    if (launches) *launches = g_cnt[kind];
    return 0;
}

}  // extern "C"
