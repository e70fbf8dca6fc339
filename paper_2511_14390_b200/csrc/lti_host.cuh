// lti_host.cuh -- host-side launchers of the LTI kernels (included by the
// per-(dtype, form) instantiation units and by api.cu for the declarations).
#pragma once
#include "host.h"
#include "lti.cuh"

namespace iirg {

template <typename K>
inline void set_smem(K kernel, size_t bytes) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// Launch with programmatic stream serialization (PDL): the kernel may start
// while its predecessor finishes; it synchronises with griddepcontrol.wait.
template <typename K, typename A>
inline void launch_pdl(K kernel, unsigned grid, unsigned block, size_t smem, cudaStream_t st, const A& args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, args);
}

template <typename T, int M, int FORM>
struct LtiOps {
    using SM = Smem<T, M>;
    static void attrs() {
        static std::once_flag once;
        std::call_once(once, [] {
            set_smem(lti_prep_kernel<T, M, FORM>, PrepSlots<M>::bytes());
            set_smem(lti_fwd_kernel<T, M, FORM>, SM::fwd(FORM));
            set_smem(lti_fwd_kernel<T, M, FORM, true>, SM::fwd(FORM));
            set_smem(lti_red_kernel<T, M, FORM, false>, RedSmem<T, M>::bytes());
            set_smem(lti_red_kernel<T, M, FORM, true>, RedSmem<T, M>::bytes());
            set_smem(lti_bwd_kernel<T, M, FORM>, SM::bwd(FORM));
            set_smem(lti_bwd_kernel<T, M, FORM, true>, SM::bwd(FORM));
            if constexpr (FORM == 1) {
                set_smem(lti_bwd_tdf_kernel<T, M>, SM::bwd_tdf());
                set_smem(lti_bwd_tdf_kernel<T, M, true>, SM::bwd_tdf());
            }
        });
    }
    // Persistent grid of the reduce kernel: every resident slot, at most one CTA per tile.
    static unsigned red_grid(int64_t ntot) {
        static int64_t cap = 0;
        static std::once_flag once;
        std::call_once(once, [] {
            int dev = 0, sms = 0, per = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, lti_red_kernel<T, M, FORM, false>, NT,
                                                          RedSmem<T, M>::bytes());
            cap = (int64_t)sms * (per > 0 ? per : 1);
        });
        return (unsigned)(ntot < cap ? ntot : cap);
    }
    // Schedule (iir_flags_t).  Default: single pass.  Measured on B200 (DESIGN.md
    // §6), three-phase lost at every BASELINE shape: its extra pass over the data
    // costs more issue slots than the look-back waits it removes (C2 44.6 vs 35.5,
    // C4 181.6 vs 186.2, C5 252 vs 231 us/step), so it is opt-in only.
    static bool three_phase(const iir_desc_t* d, const Layout&) {
        if (d->flags & IIR_FLAG_SINGLE_PASS) return false;
        return (d->flags & IIR_FLAG_THREE_PHASE) != 0;
    }
    // a1 prologue, then the scan (PDL throughout: each kernel's loads and local
    // pass overlap its predecessor; it waits before reading the predecessor's output)
    static iir_status_t forward(const iir_desc_t* d, const Layout& L, const void* b, const void* a,
                                const LtiFwdArgs& fa, cudaStream_t st) {
        attrs();
        const int64_t cstride = d->coef_mode == IIR_COEF_SHARED ? 0 : (M + 1);
        iir_status_t s = launch(K_LTI_PREP, st, [&] {
            lti_prep_kernel<T, M, FORM><<<(unsigned)L.ncoef, PREP_THREADS, PrepSlots<M>::bytes(), st>>>(
                static_cast<const T*>(b), static_cast<const T*>(a), cstride, const_cast<double*>(fa.tab),
                Tab<M>::SIZE, L.nlev, fa.span == nullptr ? nullptr : fa.span - 2);
        });
        if (s != IIR_OK) return s;
        if (!three_phase(d, L))
            return launch(K_LTI_FWD, st, [&] {
                launch_pdl(lti_fwd_kernel<T, M, FORM>, (unsigned)L.ntot, NT, SM::fwd(FORM), st, fa);
            });
        unsigned long long* dbg = fa.span == nullptr ? nullptr : fa.span - 2;   // [prep][fwd][bwd] spans, then ours
        const LtiRedArgs ra{fa.x, b, a, cstride, fa.tab, fa.tab_stride, fa.car, fa.B, fa.Tlen, fa.ntiles, fa.vec,
                            dbg == nullptr ? nullptr : dbg + 8};
        s = launch(K_LTI_RED_F, st, [&] {
            launch_pdl(lti_red_kernel<T, M, FORM, false>, red_grid(L.ntot), NT, RedSmem<T, M>::bytes(), st, ra);
        });
        if (s != IIR_OK) return s;
        const LtiScanArgs sa{fa.car, fa.zi, fa.tab, fa.tab_stride, fa.B, fa.ntiles,
                             dbg == nullptr ? nullptr : dbg + 10, dbg == nullptr ? nullptr : dbg + 16};
        s = launch(K_LTI_CSCAN, st, [&] { launch_pdl(lti_cscan_kernel<T, M, false>, (unsigned)fa.B, cs_nt<M>(), 0, st, sa); });
        if (s != IIR_OK) return s;
        return launch(K_LTI_FWD, st, [&] {
            launch_pdl(lti_fwd_kernel<T, M, FORM, true>, (unsigned)L.ntot, NT, SM::fwd(FORM), st, fa);
        });
    }
    static iir_status_t backward(const iir_desc_t* d, const Layout& L, const LtiBwdArgs& ba, cudaStream_t st) {
        attrs();
        if (!three_phase(d, L))
            return launch(K_LTI_BWD, st, [&] {
                if constexpr (FORM == 1) launch_pdl(lti_bwd_tdf_kernel<T, M>, (unsigned)L.ntot, NT, SM::bwd_tdf(), st, ba);
                else lti_bwd_kernel<T, M, FORM><<<(unsigned)L.ntot, NT, SM::bwd(FORM), st>>>(ba);
            });
        unsigned long long* dbg = ba.span == nullptr ? nullptr : ba.span - 4;
        const LtiRedArgs ra{ba.gy, nullptr, nullptr, 0, ba.tab, ba.tab_stride, ba.car, ba.B, ba.Tlen, ba.ntiles, ba.vec,
                            dbg == nullptr ? nullptr : dbg + 12};
        iir_status_t s = launch(K_LTI_RED_B, st, [&] {
            launch_pdl(lti_red_kernel<T, M, FORM, true>, red_grid(L.ntot), NT, RedSmem<T, M>::bytes(), st, ra);
        });
        if (s != IIR_OK) return s;
        const LtiScanArgs sa{ba.car, ba.gzf, ba.tab, ba.tab_stride, ba.B, ba.ntiles,
                             dbg == nullptr ? nullptr : dbg + 14, dbg == nullptr ? nullptr : dbg + 32};
        s = launch(K_LTI_CSCAN, st, [&] { launch_pdl(lti_cscan_kernel<T, M, true>, (unsigned)ba.B, cs_nt<M>(), 0, st, sa); });
        if (s != IIR_OK) return s;
        return launch(K_LTI_BWD, st, [&] {
            if constexpr (FORM == 1)
                launch_pdl(lti_bwd_tdf_kernel<T, M, true>, (unsigned)L.ntot, NT, SM::bwd_tdf(), st, ba);
            else launch_pdl(lti_bwd_kernel<T, M, FORM, true>, (unsigned)L.ntot, NT, SM::bwd(FORM), st, ba);
        });
    }
};

struct LtiCall {
    const iir_desc_t* d; const Layout* L; cudaStream_t st;
    const void *b, *a;
    LtiFwdArgs fa;
    LtiBwdArgs ba;
    bool is_fwd;
};

template <typename T, int M, int FORM>
inline iir_status_t run_lti(LtiCall& c) {
    using Ops = LtiOps<T, M, FORM>;
    if (c.is_fwd) return Ops::forward(c.d, *c.L, c.b, c.a, c.fa, c.st);
    return Ops::backward(c.d, *c.L, c.ba, c.st);
}

template <typename T, int FORM>
iir_status_t run_lti_m(int M, LtiCall& c) {
    switch (M) {
        case 1: return run_lti<T, 1, FORM>(c);
        case 2: return run_lti<T, 2, FORM>(c);
        case 3: return run_lti<T, 3, FORM>(c);
        case 4: return run_lti<T, 4, FORM>(c);
        case 5: return run_lti<T, 5, FORM>(c);
        case 6: return run_lti<T, 6, FORM>(c);
        case 7: return run_lti<T, 7, FORM>(c);
        case 8: return run_lti<T, 8, FORM>(c);
    }
    return fail(IIR_EUNSUPPORTED, "order");
}

}  // namespace iirg
