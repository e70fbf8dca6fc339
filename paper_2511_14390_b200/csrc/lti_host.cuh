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

// Persistent grid: as many CTAs as are co-resident (cached per device).
template <typename K>
inline unsigned resident_grid(K kernel, size_t smem, int64_t work, int* cache) {
    int dev = 0;
    cudaGetDevice(&dev);
    int g = (dev >= 0 && dev < 64) ? cache[dev] : 0;
    if (g == 0) {
        int nsm = 0, per = 0;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, NT, smem);
        g = nsm * (per > 0 ? per : 1);
        if (dev >= 0 && dev < 64) cache[dev] = g;
    }
    return (unsigned)(work < (int64_t)g ? work : (int64_t)g);
}

template <typename T, int M, int FORM>
struct LtiOps {
    using SM = Smem<T, M>;
    static void attrs() {
        static std::once_flag once;
        std::call_once(once, [] {
            set_smem(lti_carry_kernel<M, false>, carry_smem<M>());
            set_smem(lti_carry_kernel<M, true>, carry_smem<M>());
            set_smem(lti_prep_kernel<T, M, FORM>, PrepSlots<M>::bytes());
            set_smem(lti_fwd_kernel<T, M, FORM, 1>, SM::fwd(FORM, 1));
            set_smem(lti_fwd_kernel<T, M, FORM, 3>, SM::fwd(FORM, 3));
            set_smem(lti_bwd_kernel<T, M, FORM, 1>, SM::bwd(FORM, 1));
            set_smem(lti_bwd_kernel<T, M, FORM, 3>, SM::bwd(FORM, 3));
        });
    }
    // a1 prologue -> phase 1 (tile aggregates) -> phase 2 (carries) -> phase 3 (emit)
    static iir_status_t forward(const iir_desc_t* d, const Layout& L, const void* b, const void* a,
                                const LtiFwdArgs& fa, const CarryArgs& ca, cudaStream_t st) {
        attrs();
        const int64_t cstride = d->coef_mode == IIR_COEF_SHARED ? 0 : (M + 1);
        iir_status_t s = launch(K_LTI_PREP, st, [&] {
            lti_prep_kernel<T, M, FORM><<<(unsigned)L.ncoef, PREP_THREADS, PrepSlots<M>::bytes(), st>>>(
                static_cast<const T*>(b), static_cast<const T*>(a), cstride, const_cast<double*>(fa.tab),
                Tab<M>::SIZE, L.nlev);
        });
        if (s != IIR_OK) return s;
        static int c1[64], c3[64];
        const unsigned g1 = resident_grid(lti_fwd_kernel<T, M, FORM, 1>, SM::fwd(FORM, 1), L.ntot, c1);
        const unsigned g3 = resident_grid(lti_fwd_kernel<T, M, FORM, 3>, SM::fwd(FORM, 3), L.ntot, c3);
        s = launch(K_LTI_FWD1, st, [&] {
            launch_pdl(lti_fwd_kernel<T, M, FORM, 1>, g1, NT, SM::fwd(FORM, 1), st, fa);
        });
        if (s != IIR_OK) return s;
        s = launch(K_LTI_CARRY, st, [&] {
            launch_pdl(lti_carry_kernel<M, false>, (unsigned)d->batch, CARRY_THREADS, carry_smem<M>(), st, ca);
        });
        if (s != IIR_OK) return s;
        return launch(K_LTI_FWD3, st, [&] {
            launch_pdl(lti_fwd_kernel<T, M, FORM, 3>, g3, NT, SM::fwd(FORM, 3), st, fa);
        });
    }
    static iir_status_t backward(const iir_desc_t* d, const Layout& L, const LtiBwdArgs& ba, const CarryArgs& ca,
                                 cudaStream_t st) {
        attrs();
        static int c1[64], c3[64];
        const unsigned g1 = resident_grid(lti_bwd_kernel<T, M, FORM, 1>, SM::bwd(FORM, 1), L.ntot, c1);
        const unsigned g3 = resident_grid(lti_bwd_kernel<T, M, FORM, 3>, SM::bwd(FORM, 3), L.ntot, c3);
        iir_status_t s = launch(K_LTI_BWD1, st, [&] {
            lti_bwd_kernel<T, M, FORM, 1><<<g1, NT, SM::bwd(FORM, 1), st>>>(ba);
        });
        if (s != IIR_OK) return s;
        s = launch(K_LTI_CARRY, st, [&] {
            launch_pdl(lti_carry_kernel<M, true>, (unsigned)d->batch, CARRY_THREADS, carry_smem<M>(), st, ca);
        });
        if (s != IIR_OK) return s;
        return launch(K_LTI_BWD3, st, [&] {
            launch_pdl(lti_bwd_kernel<T, M, FORM, 3>, g3, NT, SM::bwd(FORM, 3), st, ba);
        });
    }
};

struct LtiCall {
    const iir_desc_t* d; const Layout* L; cudaStream_t st;
    const void *b, *a;
    LtiFwdArgs fa;
    LtiBwdArgs ba;
    CarryArgs ca;
    bool is_fwd;
};

template <typename T, int M, int FORM>
inline iir_status_t run_lti(LtiCall& c) {
    using Ops = LtiOps<T, M, FORM>;
    if (c.is_fwd) return Ops::forward(c.d, *c.L, c.b, c.a, c.fa, c.ca, c.st);
    return Ops::backward(c.d, *c.L, c.ba, c.ca, c.st);
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
