// lti_host.cuh -- host-side launchers of the LTI kernels (included by the
// per-(dtype, form) instantiation units and by api.cu for the declarations).
#pragma once
#include "host.h"
#include "lti.cuh"

namespace iirg {

template <typename K>
inline void set_smem(K kernel, size_t bytes) {
    if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <typename T, int M, int FORM>
struct LtiOps {
    static constexpr int TS = NT * Chunk<T>::L;
    static size_t fwd_smem() { return Smem<T, M>::fwd(FORM); }
    static size_t bwd_smem() { return Smem<T, M>::bwd(FORM); }
    // persistent grid: as many CTAs as fit on the device at once (<= tiles)
    template <typename K>
    static unsigned grid_for(K kernel, size_t smem, int64_t ntot) {
        static int cache[64] = {0};                 // resident CTAs per device
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
        return (unsigned)(ntot < (int64_t)g ? ntot : (int64_t)g);
    }
    static iir_status_t prep(const iir_desc_t* d, const Layout& L, const void* b, const void* a, double* tab,
                             cudaStream_t st) {
        static std::once_flag once;
        std::call_once(once, [] { set_smem(lti_prep_kernel<T, M, FORM>, PrepSlots<M>::bytes()); });
        const int64_t cstride = d->coef_mode == IIR_COEF_SHARED ? 0 : (M + 1);
        return launch(K_LTI_PREP, st, [&] {
            lti_prep_kernel<T, M, FORM><<<(unsigned)L.ncoef, PREP_THREADS, PrepSlots<M>::bytes(), st>>>(
                static_cast<const T*>(b), static_cast<const T*>(a), cstride, tab, Tab<M>::SIZE, L.nlev);
        });
    }
    // The scan kernel is launched as a programmatic dependent of the prologue: its
    // tile loads and local pass overlap the prologue; it waits (griddepcontrol.wait)
    // before touching the power tables.
    static iir_status_t fwd(const iir_desc_t* d, const Layout& L, const LtiFwdArgs& args, cudaStream_t st) {
        static std::once_flag once;
        std::call_once(once, [] { set_smem(lti_fwd_kernel<T, M, FORM>, fwd_smem()); });
        const unsigned grid = grid_for(lti_fwd_kernel<T, M, FORM>, fwd_smem(), L.ntot);
        return launch(K_LTI_FWD, st, [&] {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(NT);
            cfg.dynamicSmemBytes = fwd_smem();
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, lti_fwd_kernel<T, M, FORM>, args);
        });
    }
    static iir_status_t bwd(const iir_desc_t* d, const Layout& L, const LtiBwdArgs& args, cudaStream_t st) {
        static std::once_flag once;
        std::call_once(once, [] { set_smem(lti_bwd_kernel<T, M, FORM>, bwd_smem()); });
        const unsigned grid = grid_for(lti_bwd_kernel<T, M, FORM>, bwd_smem(), L.ntot);
        return launch(K_LTI_BWD, st, [&] {
            lti_bwd_kernel<T, M, FORM><<<grid, NT, bwd_smem(), st>>>(args);
        });
    }
};

struct LtiCall {
    const iir_desc_t* d; const Layout* L; cudaStream_t st;
    // forward
    const void *b, *a; LtiFwdArgs fa;
    // backward
    LtiBwdArgs ba;
    bool is_fwd;
};

template <typename T, int M, int FORM>
inline iir_status_t run_lti(LtiCall& c) {
    using Ops = LtiOps<T, M, FORM>;
    if (c.is_fwd) {
        iir_status_t s = Ops::prep(c.d, *c.L, c.b, c.a, const_cast<double*>(c.fa.tab), c.st);
        if (s != IIR_OK) return s;
        return Ops::fwd(c.d, *c.L, c.fa, c.st);
    }
    return Ops::bwd(c.d, *c.L, c.ba, c.st);
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
