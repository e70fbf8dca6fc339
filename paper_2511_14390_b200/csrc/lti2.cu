// lti2.cu -- host launchers of the round-2 LTI engine (lti2.cuh): fp32 TDF-II,
// SHARED or PER_SEQ coefficients, orders 1..8.  Three launches per call pair:
// prologue (plain launch), then the persistent forward / backward scans, each
// launched with programmatic stream serialization (their griddepcontrol.wait comes
// before any read of a predecessor's output, so PDL only hides launch latency).
#include <mutex>

#include "host.h"
#include "lti2.cuh"
#include "lti_host.cuh"

namespace iirg {
namespace v2 {

constexpr int NWF = IIRG_V2_NWF;   // warps per CTA, forward
constexpr int NWB = IIRG_V2_NWB;   // warps per CTA, backward

template <int M>
constexpr size_t smem_bytes(bool gt, int nwp, int nbuf) {
    return (gt ? 0 : (size_t)Cfg<M>::STAGE * 4) + (size_t)nwp * nbuf * Cfg<M>::BUF * 4;
}
// shared buffers per warp: forward x in / y out; backward dy in, x -> dx, y
template <int M, bool GT>
constexpr auto fwd_kernel() { return lti2_fwd_kernel<M, NWF, GT>; }
template <int M>
constexpr size_t fwd_smem(bool gt) { return smem_bytes<M>(gt, NWF, 2); }

// Per-device launch setup: the max-dynamic-smem attribute is per device, so it is
// set (and the resident-CTA counts queried) once for every device that calls in.
struct DevInfo {
    bool ready = false;
    int sms = 0;
    int occ[4] = {0, 0, 0, 0};   // fwd shared, fwd global, bwd shared, bwd global
};

template <int M>
struct Ops {
    static const DevInfo& dev_info() {
        static std::mutex mu;
        static DevInfo info[64];
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lk(mu);
        DevInfo& d = info[dev & 63];
        if (!d.ready) {
            cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
            set_smem(lti2_prep_kernel<M>, Prep2Slots<M>::bytes());
            set_smem(fwd_kernel<M, false>(), fwd_smem<M>(false));
            set_smem(fwd_kernel<M, true>(), fwd_smem<M>(true));
            set_smem(lti2_bwd_kernel<M, NWB, false>, smem_bytes<M>(false, NWB, 3));
            set_smem(lti2_bwd_kernel<M, NWB, true>, smem_bytes<M>(true, NWB, 3));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.occ[0], fwd_kernel<M, false>(), NWF * 32,
                                                          fwd_smem<M>(false));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.occ[1], fwd_kernel<M, true>(), NWF * 32,
                                                          fwd_smem<M>(true));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.occ[2], lti2_bwd_kernel<M, NWB, false>, NWB * 32,
                                                          smem_bytes<M>(false, NWB, 3));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.occ[3], lti2_bwd_kernel<M, NWB, true>, NWB * 32,
                                                          smem_bytes<M>(true, NWB, 3));
            (void)cudaGetLastError();
            d.ready = true;
        }
        return d;
    }
    // one resident wave, at most one warp per tile
    static unsigned grid(const DevInfo& d, int k, int64_t ntot, int nwp) {
        const int64_t cap = (int64_t)d.sms * (d.occ[k] > 0 ? d.occ[k] : 1);
        const int64_t need = (ntot + nwp - 1) / nwp;
        return (unsigned)(need < cap ? need : cap);
    }
    static iir_status_t forward(const Call& c) {
        const DevInfo& d = dev_info();
        iir_status_t s = launch(K_LTI_PREP, c.st, [&] {
            lti2_prep_kernel<M><<<dim3((unsigned)c.ncoef, 2 + c.nlev), PREP_NT, Prep2Slots<M>::bytes(), c.st>>>(
                c.b, c.a, c.cstride, const_cast<float*>(c.f.t32), c.f.t32_stride, const_cast<double*>(c.f.t64),
                c.f.t64_stride, c.nlev);
        });
        if (s != IIR_OK) return s;
        const bool gt = c.ncoef > 1;
        return launch(K_LTI_FWD, c.st, [&] {
            if (gt) launch_pdl(fwd_kernel<M, true>(), grid(d, 1, c.f.ntot, NWF), NWF * 32, fwd_smem<M>(true), c.st, c.f);
            else launch_pdl(fwd_kernel<M, false>(), grid(d, 0, c.f.ntot, NWF), NWF * 32, fwd_smem<M>(false), c.st, c.f);
        });
    }
    static iir_status_t backward(const Call& c) {
        const DevInfo& d = dev_info();
        const bool gt = c.ncoef > 1;
        return launch(K_LTI_BWD, c.st, [&] {
            if (gt)
                launch_pdl(lti2_bwd_kernel<M, NWB, true>, grid(d, 3, c.g.ntot, NWB), NWB * 32, smem_bytes<M>(true, NWB, 3),
                           c.st, c.g);
            else
                launch_pdl(lti2_bwd_kernel<M, NWB, false>, grid(d, 2, c.g.ntot, NWB), NWB * 32,
                           smem_bytes<M>(false, NWB, 3), c.st, c.g);
        });
    }
};

iir_status_t run(bool fwd, int M, const Call& c) {
    switch (M) {
#define IIRG_V2_CASE(m) \
        case m: return fwd ? Ops<m>::forward(c) : Ops<m>::backward(c);
#ifdef IIRG_V2_ONLY                      // kernel experiments: one order only (tools/sass_loop.sh)
        IIRG_V2_CASE(IIRG_V2_ONLY)
#else
        IIRG_V2_CASE(1) IIRG_V2_CASE(2) IIRG_V2_CASE(3) IIRG_V2_CASE(4)
        IIRG_V2_CASE(5) IIRG_V2_CASE(6) IIRG_V2_CASE(7) IIRG_V2_CASE(8)
#endif
#undef IIRG_V2_CASE
    }
    return fail(IIR_EUNSUPPORTED, "order");
}

int tile_samples(int M) {
    (void)M;
    return Cfg<8>::TS;
}
size_t tab32_floats(int M) {
    switch (M) {
        case 1: return Cfg<1>::SIZE32; case 2: return Cfg<2>::SIZE32; case 3: return Cfg<3>::SIZE32;
        case 4: return Cfg<4>::SIZE32; case 5: return Cfg<5>::SIZE32; case 6: return Cfg<6>::SIZE32;
        case 7: return Cfg<7>::SIZE32; case 8: return Cfg<8>::SIZE32;
    }
    return 0;
}
size_t tab64_doubles(int M) {
    switch (M) {
        case 1: return Cfg<1>::SIZE64; case 2: return Cfg<2>::SIZE64; case 3: return Cfg<3>::SIZE64;
        case 4: return Cfg<4>::SIZE64; case 5: return Cfg<5>::SIZE64; case 6: return Cfg<6>::SIZE64;
        case 7: return Cfg<7>::SIZE64; case 8: return Cfg<8>::SIZE64;
    }
    return 0;
}

}  // namespace v2
}  // namespace iirg
