// tv.cu -- host side of the per-sample (time-varying) all-pole DF path
// (IIR_COEF_PER_SAMPLE): layout and dispatch; the per-order kernels are
// instantiated in tv_o1.cu .. tv_o4.cu (every order 1..32).
#include <mutex>

#include "host.h"
#include "tv_impl.cuh"
#include "tvtdf.cuh"

namespace iirg {

#define IIRG_TV_ORDERS(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30) X(31) X(32)
#define IIRG_EXTERN(m)                                                                                         \
    extern template iir_status_t tv_order<float, m>(int, const iir_desc_t*, const Layout&, TvArgs&,            \
                                                    const void*, const void*, const void*, const void*, void*, \
                                                    void*, void*, void*, cudaStream_t);                        \
    extern template iir_status_t tv_order<double, m>(int, const iir_desc_t*, const Layout&, TvArgs&,           \
                                                     const void*, const void*, const void*, const void*,      \
                                                     void*, void*, void*, void*, cudaStream_t);
IIRG_TV_ORDERS(IIRG_EXTERN)
#undef IIRG_EXTERN



bool tv_supported(int M) {
    switch (M) {
#define IIRG_CASE(m) case m: return true;
        IIRG_TV_ORDERS(IIRG_CASE)
#undef IIRG_CASE
    }
    return false;
}

Layout tv_layout(const iir_desc_t* d) {
    Layout L;
    const int M = d->order;
    const size_t ts = d->dtype == IIR_F64 ? 8 : 4;
    L.ntiles = (d->length + TV_SEG - 1) / TV_SEG;          // segments per sequence
    L.ntot = L.ntiles * d->batch;
    L.ncoef = d->batch;
    size_t o = 0;
    L.ws_clear = 0;                                        // no counters: nothing to initialise
    L.ws_part = o; o += al256((size_t)L.ntot * M * 8);     // w: segment aggregates
    L.ws_part2 = o; o += al256((size_t)L.ntot * M * 8);    // carry: entering states
    const int64_t ngrp = (L.ntiles + TV_GS - 1) / TV_GS;
    L.ngroups = ngrp;
    L.ws_psi = o; o += al256((size_t)d->batch * ngrp * M * M * 8);
    L.ws_omega = o; o += al256((size_t)d->batch * ngrp * M * 8);
    L.ws_sgrp = o; o += al256((size_t)d->batch * ngrp * M * 8);
    L.ws_bytes = o;
    L.tp_tab = 0;
    L.tp_bytes = al256((size_t)L.ntot * M * M * ts);       // Phi_k per segment (reused by the backward)
    L.tp_u = L.tp_bytes;
    if (d->flags & IIR_FLAG_PER_SAMPLE_B) {
        const size_t bt = (size_t)d->batch * d->length;
        if (d->form == IIR_DF2) L.tp_bytes += al256(bt * ts);   // general DF: the all-pole output u (B, T)
        L.ws_du = o; o += al256(bt * ts);                  // DF: FIR-stage adjoint of u(0..T-1); TDF: g = dL/df
        L.ws_duneg = o; o += al256((size_t)d->batch * M * ts);   //   ... and of u(-1..-M)
        if (d->form == IIR_TDF2) {                         // general TDF (tvtdf.cuh)
            L.ws_f = o; o += al256(bt * ts);               // f (forward) / grad_y + zf tail (backward)
            L.ws_gas = o; o += al256(bt * M * ts);         // gradient of the skewed rows a~
            L.ws_as = L.tp_bytes; L.tp_bytes += al256(bt * M * ts);        // the skewed rows a~ on the tape
                                                                           // (offset into the tape)
        }
        L.ws_bytes = o;
    }
    return L;
}

template <typename T>
static iir_status_t tv_op(int op, const iir_desc_t* d, const Layout& L, TvArgs& a, const void* b, const void* u,
                          const void* zi, const void* gy, void* y, void* du, void* duneg, void* gb, cudaStream_t st) {
    switch (d->order) {
#define IIRG_CASE(m) case m: return tv_order<T, m>(op, d, L, a, b, u, zi, gy, y, du, duneg, gb, st);
        IIRG_TV_ORDERS(IIRG_CASE)
#undef IIRG_CASE
    }
    return fail(IIR_EUNSUPPORTED, "per-sample order must be 1..32");
}
template <typename T>
static iir_status_t fir_dispatch(bool fwd, const iir_desc_t* d, const void* b, const void* u, const void* zi,
                                 const void* gy, void* y, void* du, void* duneg, void* gb, cudaStream_t st,
                                 bool skew = false) {
    static Layout none;
    TvArgs dummy{};
    return tv_op<T>(skew ? (fwd ? 4 : 5) : (fwd ? 2 : 3), d, none, dummy, b, u, zi, gy, y, du, duneg, gb, st);
}
template <typename T>
static iir_status_t tv_dispatch(bool fwd, int, const Layout& L, TvArgs& a, cudaStream_t st, const iir_desc_t* d) {
    return tv_op<T>(fwd ? 0 : 1, d, L, a, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, st);
}

// 16 B staging copies of coefficient rows need aligned rows and pieces that
// never straddle two samples.
static int tv_vec(const iir_desc_t* d, const void* a) {
    const size_t ts = d->dtype == IIR_F64 ? 8 : 4;
    return (((size_t)d->order * ts) % 16 == 0) && ((reinterpret_cast<uintptr_t>(a) & 15u) == 0);
}

// ---- general time-varying TDF (tvtdf.cuh, reading R20) -------------------------------
// (row tiles, sequences) grid of the skew kernels, their shared memory (> 48 KB opt-in per device)
template <typename T>
static dim3 skew_grid(int64_t B, int64_t N) { return dim3((unsigned)((N + tdf::SR - 1) / tdf::SR), (unsigned)B); }
template <typename T>
static void skew_attrs(int M) {
    static PerDevice attrs;
    attrs.once([] {
        cudaFuncSetAttribute(tdf::skew_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tdf::skew_smem<T>(TV_MAX_M));
        cudaFuncSetAttribute(tdf::unskew_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tdf::skew_smem<T>(TV_MAX_M));
    });
    (void)M;
}
static TvArgs tv_args(const iir_desc_t* d, const Layout& L, char* tape, char* ws) {
    TvArgs ta{};
    ta.phi = tape;
    ta.w = reinterpret_cast<double*>(ws + L.ws_part);
    ta.carry = reinterpret_cast<double*>(ws + L.ws_part2);
    ta.B = d->batch; ta.T = d->length; ta.nseg = (int)L.ntiles;
    ta.psi = reinterpret_cast<double*>(ws + L.ws_psi);
    ta.omega = reinterpret_cast<double*>(ws + L.ws_omega);
    ta.sgrp = reinterpret_cast<double*>(ws + L.ws_sgrp);
    ta.ngrp = (int)L.ngroups;
    return ta;
}
template <typename T>
static iir_status_t tdf_forward(const iir_desc_t* d, const Layout& L, const void* b, const void* a, const void* x,
                                const void* zi, void* y, void* zf, char* tape, char* ws, cudaStream_t st) {
    const int64_t B = d->batch, N = d->length;
    const int M = d->order;
    T* as = reinterpret_cast<T*>(tape + L.ws_as);                    // skewed rows: tape (reused backward)
    T* f = reinterpret_cast<T*>(ws + L.ws_f);
    skew_attrs<T>(M);
    iir_status_t s = launch(K_TV_SKEW, st, [&] {
        tdf::skew_kernel<T><<<skew_grid<T>(B, N), tdf::NT, tdf::skew_smem<T>(M), st>>>(static_cast<const T*>(a),
            as, N, M);
    });
    if (s != IIR_OK) return s;
    // f(n) = sum_k b~_k(n) x(n-k) (b read at skewed rows; zero history), + zi(n) for n < M
    s = fir_dispatch<T>(true, d, b, x, nullptr, nullptr, f, nullptr, nullptr, nullptr, st, true);
    if (s != IIR_OK) return s;
    if (zi != nullptr) {
        s = launch(K_TV_SKEW, st, [&] {
            tdf::zi_add_kernel<T><<<(unsigned)((B * M + 127) / 128), 128, 0, st>>>(f, static_cast<const T*>(zi), B, N, M);
        });
        if (s != IIR_OK) return s;
    }
    // y(n) = f(n) - sum_i a~_i(n) y(n-i), zero history
    TvArgs ta = tv_args(d, L, tape, ws);
    ta.a = as; ta.x = f; ta.zi = nullptr; ta.y = y; ta.zf = nullptr;
    ta.vec = (((size_t)M * sizeof(T)) % 16 == 0) && ((reinterpret_cast<uintptr_t>(as) & 15u) == 0);
    s = tv_dispatch<T>(true, M, L, ta, st, d);
    if (s != IIR_OK || zf == nullptr) return s;
    return launch(K_TV_SKEW, st, [&] {
        tdf::zf_kernel<T><<<(unsigned)((B * M + 127) / 128), 128, 0, st>>>(static_cast<const T*>(a),
            static_cast<const T*>(b), static_cast<const T*>(x), static_cast<const T*>(y), static_cast<const T*>(zi),
            static_cast<T*>(zf), B, N, M);
    });
}
template <typename T>
static iir_status_t tdf_backward(const iir_desc_t* d, const Layout& L, const void* gy, const void* gzf, const void* b,
                                 const void* a, const void* x, const void* y, const char* tape, void* gx, void* gb,
                                 void* ga, void* gzi, char* ws, cudaStream_t st) {
    const int64_t B = d->batch, N = d->length;
    const int M = d->order;
    const T* as = reinterpret_cast<const T*>(tape + L.ws_as);        // the forward's skewed rows (tape)
    T* gas = reinterpret_cast<T*>(ws + L.ws_gas);
    T* gye = reinterpret_cast<T*>(ws + L.ws_f);
    T* g = reinterpret_cast<T*>(ws + L.ws_du);
    T* duneg = reinterpret_cast<T*>(ws + L.ws_duneg);
    skew_attrs<T>(M);
    iir_status_t s = launch(K_TV_SKEW, st, [&] {
        tdf::gy_eff_kernel<T><<<dim3((unsigned)((N + tdf::NT - 1) / tdf::NT), (unsigned)B), tdf::NT, 0, st>>>(
            static_cast<const T*>(gy), static_cast<const T*>(gzf), static_cast<const T*>(a), gye, N, M);
    });
    if (s != IIR_OK) return s;
    // all-pole adjoint on the skewed rows: g = dL/df, grad_a~
    TvArgs ta = tv_args(d, L, const_cast<char*>(tape), ws);
    ta.a = as; ta.zi = nullptr; ta.gy = gye; ta.gzf = nullptr; ta.yin = y;
    ta.gx = g; ta.ga = gas; ta.gzi = nullptr;
    ta.vec = (((size_t)M * sizeof(T)) % 16 == 0) && ((reinterpret_cast<uintptr_t>(as) & 15u) == 0) &&
             ((reinterpret_cast<uintptr_t>(gas) & 15u) == 0);
    s = tv_dispatch<T>(false, M, L, ta, st, d);
    if (s != IIR_OK) return s;
    // FIR adjoint on the skewed rows (b read in place): grad_x, grad_b (unskewed)
    s = fir_dispatch<T>(false, d, b, x, nullptr, g, nullptr, gx != nullptr ? gx : static_cast<void*>(gye), duneg,
                        gb, st, true);
    if (s != IIR_OK) return s;
    if (ga != nullptr) {
        s = launch(K_TV_SKEW, st, [&] {
            tdf::unskew_kernel<T><<<skew_grid<T>(B, N), tdf::NT, tdf::skew_smem<T>(M), st>>>(gas,
                static_cast<T*>(ga), N, M);
        });
        if (s != IIR_OK) return s;
    }
    return launch(K_TV_SKEW, st, [&] {
        tdf::tail_kernel<T><<<(unsigned)((B * M + 127) / 128), 128, 0, st>>>(static_cast<const T*>(gzf),
            static_cast<const T*>(a), static_cast<const T*>(b), static_cast<const T*>(x), static_cast<const T*>(y), g,
            static_cast<T*>(gx), static_cast<T*>(ga), static_cast<T*>(gb), static_cast<T*>(gzi), B, N, M);
    });
}

iir_status_t tv_forward(const iir_desc_t* d, const Layout& L, const void* b, const void* a, const void* x,
                        const void* zi, void* y, void* zf, char* tape, char* ws, bool, cudaStream_t st) {
    const bool fir = (d->flags & IIR_FLAG_PER_SAMPLE_B) != 0;
    if (d->form == IIR_TDF2)
        return d->dtype == IIR_F64 ? tdf_forward<double>(d, L, b, a, x, zi, y, zf, tape, ws, st)
                                   : tdf_forward<float>(d, L, b, a, x, zi, y, zf, tape, ws, st);
    void* u = fir ? static_cast<void*>(tape + L.tp_u) : y;   // general DF: the recursion's output is u
    TvArgs ta{};
    ta.a = a; ta.x = x; ta.zi = zi; ta.y = u; ta.zf = zf;
    ta.phi = tape;
    ta.w = reinterpret_cast<double*>(ws + L.ws_part);
    ta.carry = reinterpret_cast<double*>(ws + L.ws_part2);
    ta.B = d->batch; ta.T = d->length; ta.nseg = (int)L.ntiles;
    ta.vec = tv_vec(d, a);
    ta.psi = reinterpret_cast<double*>(ws + L.ws_psi);
    ta.omega = reinterpret_cast<double*>(ws + L.ws_omega);
    ta.sgrp = reinterpret_cast<double*>(ws + L.ws_sgrp);
    ta.ngrp = (int)L.ngroups;
    iir_status_t s = d->dtype == IIR_F64 ? tv_dispatch<double>(true, d->order, L, ta, st, d)
                                         : tv_dispatch<float>(true, d->order, L, ta, st, d);
    if (s != IIR_OK || !fir) return s;
    return d->dtype == IIR_F64 ? fir_dispatch<double>(true, d, b, u, zi, nullptr, y, nullptr, nullptr, nullptr, st)
                               : fir_dispatch<float>(true, d, b, u, zi, nullptr, y, nullptr, nullptr, nullptr, st);
}

iir_status_t tv_backward(const iir_desc_t* d, const Layout& L, const void* gy, const void* gzf, const void* b,
                         const void* a, const void* y, const void* zi, const char* tape, void* gx, void* gb,
                         void* ga, void* gzi, char* ws, bool, cudaStream_t st, const void* x) {
    if (d->form == IIR_TDF2)
        return d->dtype == IIR_F64 ? tdf_backward<double>(d, L, gy, gzf, b, a, x, y, tape, gx, gb, ga, gzi, ws, st)
                                   : tdf_backward<float>(d, L, gy, gzf, b, a, x, y, tape, gx, gb, ga, gzi, ws, st);
    const bool fir = (d->flags & IIR_FLAG_PER_SAMPLE_B) != 0;
    const void* u = fir ? static_cast<const void*>(tape + L.tp_u) : y;
    void* du = fir ? static_cast<void*>(ws + L.ws_du) : nullptr;
    void* duneg = fir ? static_cast<void*>(ws + L.ws_duneg) : nullptr;
    if (fir) {                                             // FIR stage adjoint first: du, grad_b
        iir_status_t s = d->dtype == IIR_F64
            ? fir_dispatch<double>(false, d, b, u, zi, gy, nullptr, du, duneg, gb, st)
            : fir_dispatch<float>(false, d, b, u, zi, gy, nullptr, du, duneg, gb, st);
        if (s != IIR_OK) return s;
    }
    TvArgs ta{};
    ta.a = a; ta.zi = zi; ta.gy = fir ? du : gy; ta.gzf = gzf; ta.yin = u;
    ta.gx = gx; ta.ga = ga; ta.gzi = gzi;
    ta.phi = const_cast<char*>(tape);
    ta.w = reinterpret_cast<double*>(ws + L.ws_part);
    ta.carry = reinterpret_cast<double*>(ws + L.ws_part2);
    ta.B = d->batch; ta.T = d->length; ta.nseg = (int)L.ntiles;
    ta.vec = tv_vec(d, a) && (reinterpret_cast<uintptr_t>(ga) & 15u) == 0;
    ta.psi = reinterpret_cast<double*>(ws + L.ws_psi);
    ta.omega = reinterpret_cast<double*>(ws + L.ws_omega);
    ta.sgrp = reinterpret_cast<double*>(ws + L.ws_sgrp);
    ta.ngrp = (int)L.ngroups;
    iir_status_t s = d->dtype == IIR_F64 ? tv_dispatch<double>(false, d->order, L, ta, st, d)
                                         : tv_dispatch<float>(false, d->order, L, ta, st, d);
    if (s != IIR_OK || !fir || gzi == nullptr) return s;
    const int64_t n = d->batch * d->order;                 // grad_zi += the FIR stage's direct terms
    return launch(K_TV_FIR, st, [&] {
        if (d->dtype == IIR_F64)
            tv_add_kernel<double><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(static_cast<double*>(gzi),
                static_cast<const double*>(duneg), n);
        else
            tv_add_kernel<float><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(static_cast<float*>(gzi),
                static_cast<const float*>(duneg), n);
    });
}

}  // namespace iirg
