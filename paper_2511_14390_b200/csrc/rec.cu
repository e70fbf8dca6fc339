// rec.cu -- host side of the bare recurrence (form IIR_SS, rec.cuh): launchers
// and instantiations (fp32 / fp64, M = 1..4).
#include "host.h"
#include "lti_host.cuh"
#include "rec.cuh"

namespace iirg {

template <typename T, int M>
struct RecOps {
    using RS = RecSmem<T, M>;
    static void attrs() {
        static std::once_flag once;
        std::call_once(once, [] {
            set_smem(lti_prep_kernel<T, M, 2, RS::L>, PrepSlots<M>::bytes());
            set_smem(rec_fwd_kernel<T, M>, RS::fwd());
            set_smem(rec_bwd_kernel<T, M>, RS::bwd());
        });
    }
    static iir_status_t forward(const Layout& L, const LtiFwdArgs& fa, cudaStream_t st) {
        attrs();
        iir_status_t s = launch(K_LTI_PREP, st, [&] {
            lti_prep_kernel<T, M, 2, RS::L><<<(unsigned)L.ncoef, PREP_THREADS, PrepSlots<M>::bytes(), st>>>(
                nullptr, static_cast<const T*>(fa.a), fa.coef_stride, const_cast<double*>(fa.tab), Tab<M>::SIZE,
                L.nlev, fa.span == nullptr ? nullptr : fa.span - 2);
        });
        if (s != IIR_OK) return s;
        return launch(K_REC_FWD, st, [&] { launch_pdl(rec_fwd_kernel<T, M>, (unsigned)L.ntot, NT, RS::fwd(), st, fa); });
    }
    static iir_status_t backward(const Layout& L, const LtiBwdArgs& ba, cudaStream_t st) {
        attrs();
        return launch(K_REC_BWD, st, [&] {
            rec_bwd_kernel<T, M><<<(unsigned)L.ntot, NT, RS::bwd(), st>>>(ba);
        });
    }
};

int rec_tile_samples(int dtype, int M) {
    if (dtype == IIR_F64) return M > 2 ? RecSmem<double, 3>::TS : RecSmem<double, 1>::TS;
    return M > 2 ? RecSmem<float, 3>::TS : RecSmem<float, 1>::TS;
}

template <typename T>
static iir_status_t rec_m(bool fwd, int M, const Layout& L, const LtiFwdArgs& fa, const LtiBwdArgs& ba,
                          cudaStream_t st) {
    switch (M) {
#define IIRG_CASE(m) \
    case m: return fwd ? RecOps<T, m>::forward(L, fa, st) : RecOps<T, m>::backward(L, ba, st);
        IIRG_CASE(1) IIRG_CASE(2) IIRG_CASE(3) IIRG_CASE(4)
#undef IIRG_CASE
    }
    return fail(IIR_EUNSUPPORTED, "recurrence order must be 1..4");
}

iir_status_t rec_run(bool fwd, int dtype, int M, const Layout& L, const LtiFwdArgs& fa, const LtiBwdArgs& ba,
                     cudaStream_t st) {
    return dtype == IIR_F64 ? rec_m<double>(fwd, M, L, fa, ba, st) : rec_m<float>(fwd, M, L, fa, ba, st);
}

}  // namespace iirg
