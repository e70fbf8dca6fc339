#include <type_traits>
// tv.cu -- host side of the per-sample (time-varying) all-pole DF path
// (IIR_COEF_PER_SAMPLE): layout, dispatch, instantiations.
#include "host.h"
#include "tv.cuh"

#include <mutex>

namespace iirg {

#define IIRG_TV_ORDERS(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(10) X(12) X(16) X(20) X(24) X(28) X(31)

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
    return L;
}

template <typename T, int M, int MODE>
static void tv_seq_launch(unsigned nseg_tot, const TvArgs& a, cudaStream_t st) {
    const size_t smem = TvStage<T, M, MODE>::bytes(MODE);
    static std::once_flag once;
    std::call_once(once, [&] {
        cudaFuncSetAttribute(tv_seq_kernel<T, M, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    const unsigned per = 32 * TV_SEQ_WARPS;
    tv_seq_kernel<T, M, MODE><<<(nseg_tot + per - 1) / per, per, smem, st>>>(a);
}

// phase 2 (both directions): group maps, chain over the groups, expansion
template <typename T, int M, bool BWD>
static iir_status_t tv_chain2(const TvArgs& a, const void* x0, cudaStream_t st) {
    const unsigned ng = (unsigned)(a.B * a.ngrp);
    const unsigned blocks = (ng + TV_GRP_WARPS - 1) / TV_GRP_WARPS;
    iir_status_t s = launch(K_TV_CHAIN, st, [&] {
        tv_group_kernel<T, M, BWD><<<blocks, 32 * TV_GRP_WARPS, 0, st>>>(a);
    });
    if (s != IIR_OK) return s;
    s = launch(K_TV_CHAIN, st, [&] {
        tv_groupchain_kernel<M, BWD><<<(unsigned)a.B, 32, 0, st>>>(a, x0, (int)sizeof(T));
    });
    if (s != IIR_OK) return s;
    return launch(K_TV_CHAIN, st, [&] { tv_expand_kernel<T, M, BWD><<<blocks, 32 * TV_GRP_WARPS, 0, st>>>(a); });
}

template <typename T, int M>
static iir_status_t tv_fwd_m(const Layout& L, TvArgs& a, cudaStream_t st) {
    const unsigned nseg_tot = (unsigned)L.ntot;
    iir_status_t s = launch(K_TV_PHI, st, [&] {
        if constexpr (std::is_same<T, float>::value) {
            const unsigned per = 2 * TV_PHI2_WARPS;          // segments per CTA
            tv_phi2_kernel<M><<<(nseg_tot + per - 1) / per, 32 * TV_PHI2_WARPS, 0, st>>>(a);
        } else {
            tv_phi_kernel<T, M><<<(nseg_tot + TV_PHI_WARPS - 1) / TV_PHI_WARPS, 32 * TV_PHI_WARPS, 0, st>>>(a);
        }
    });
    if (s != IIR_OK) return s;
    s = tv_chain2<T, M, false>(a, a.zi, st);
    if (s != IIR_OK) return s;
    return launch(K_TV_FWD, st, [&] { tv_seq_launch<T, M, TV_FWD_EMIT>(nseg_tot, a, st); });
}

template <typename T, int M>
static iir_status_t tv_bwd_m(const Layout& L, TvArgs& a, cudaStream_t st) {
    const unsigned nseg_tot = (unsigned)L.ntot;
    iir_status_t s = launch(K_TV_BWD_AGG, st, [&] { tv_seq_launch<T, M, TV_BWD_AGG>(nseg_tot, a, st); });
    if (s != IIR_OK) return s;
    s = tv_chain2<T, M, true>(a, a.gzf, st);
    if (s != IIR_OK) return s;
    return launch(K_TV_BWD, st, [&] { tv_seq_launch<T, M, TV_BWD_EMIT>(nseg_tot, a, st); });
}

template <typename T>
static iir_status_t tv_dispatch(bool fwd, int M, const Layout& L, TvArgs& a, cudaStream_t st) {
    switch (M) {
#define IIRG_CASE(m) case m: return fwd ? tv_fwd_m<T, m>(L, a, st) : tv_bwd_m<T, m>(L, a, st);
        IIRG_TV_ORDERS(IIRG_CASE)
#undef IIRG_CASE
    }
    return fail(IIR_EUNSUPPORTED, "per-sample order not compiled in");
}

// 16 B staging copies of coefficient rows need aligned rows and pieces that
// never straddle two samples.
static int tv_vec(const iir_desc_t* d, const void* a) {
    const size_t ts = d->dtype == IIR_F64 ? 8 : 4;
    return (((size_t)d->order * ts) % 16 == 0) && ((reinterpret_cast<uintptr_t>(a) & 15u) == 0);
}

iir_status_t tv_forward(const iir_desc_t* d, const Layout& L, const void* a, const void* x, const void* zi, void* y,
                        void* zf, char* tape, char* ws, bool, cudaStream_t st) {
    TvArgs ta{};
    ta.a = a; ta.x = x; ta.zi = zi; ta.y = y; ta.zf = zf;
    ta.phi = tape;
    ta.w = reinterpret_cast<double*>(ws + L.ws_part);
    ta.carry = reinterpret_cast<double*>(ws + L.ws_part2);
    ta.B = d->batch; ta.T = d->length; ta.nseg = (int)L.ntiles;
    ta.vec = tv_vec(d, a);
    ta.psi = reinterpret_cast<double*>(ws + L.ws_psi);
    ta.omega = reinterpret_cast<double*>(ws + L.ws_omega);
    ta.sgrp = reinterpret_cast<double*>(ws + L.ws_sgrp);
    ta.ngrp = (int)L.ngroups;
    return d->dtype == IIR_F64 ? tv_dispatch<double>(true, d->order, L, ta, st)
                               : tv_dispatch<float>(true, d->order, L, ta, st);
}

iir_status_t tv_backward(const iir_desc_t* d, const Layout& L, const void* gy, const void* gzf, const void* a,
                         const void* y, const void* zi, const char* tape, void* gx, void* ga, void* gzi, char* ws,
                         bool, cudaStream_t st) {
    TvArgs ta{};
    ta.a = a; ta.zi = zi; ta.gy = gy; ta.gzf = gzf; ta.yin = y;
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
    return d->dtype == IIR_F64 ? tv_dispatch<double>(false, d->order, L, ta, st)
                               : tv_dispatch<float>(false, d->order, L, ta, st);
}

}  // namespace iirg
