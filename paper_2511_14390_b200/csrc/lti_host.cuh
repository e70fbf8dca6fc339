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
    // the max-dynamic-smem attribute is per device: set once for every device that calls in
    static void attrs() {
        static std::mutex mu;
        static bool done[64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lk(mu);
        if (done[dev & 63]) return;
        set_smem(lti_prep_kernel<T, M, FORM>, PrepSlots<M>::bytes());
        set_smem(lti_fwd_kernel<T, M, FORM>, SM::fwd(FORM));
        set_smem(lti_bwd_kernel<T, M, FORM>, SM::bwd(FORM));
        if constexpr (FORM == 1) set_smem(lti_bwd_tdf_kernel<T, M>, SM::bwd_tdf());
        done[dev & 63] = true;
    }
    // a1 prologue, then the single-pass scan (PDL: each kernel's tile loads overlap its
    // predecessor's tail; it waits before reading the predecessor's output)
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
        return launch(K_LTI_FWD, st, [&] {
            launch_pdl(lti_fwd_kernel<T, M, FORM>, (unsigned)L.ntot, NT, SM::fwd(FORM), st, fa);
        });
    }
    static iir_status_t backward(const iir_desc_t*, const Layout& L, const LtiBwdArgs& ba, cudaStream_t st) {
        attrs();
        return launch(K_LTI_BWD, st, [&] {
            if constexpr (FORM == 1) launch_pdl(lti_bwd_tdf_kernel<T, M>, (unsigned)L.ntot, NT, SM::bwd_tdf(), st, ba);
            else lti_bwd_kernel<T, M, FORM><<<(unsigned)L.ntot, NT, SM::bwd(FORM), st>>>(ba);
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
