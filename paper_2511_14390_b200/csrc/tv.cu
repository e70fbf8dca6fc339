// tv.cu -- per-sample (time-varying) all-pole DF path.  Stub
// until the kernels land: reports IIR_EUNSUPPORTED.
#include "host.h"

namespace iirg {
bool tv_supported(int) { return false; }
Layout tv_layout(const iir_desc_t*) { return Layout{}; }
iir_status_t tv_forward(const iir_desc_t*, const Layout&, const void*, const void*, const void*, void*, void*, char*,
                        char*, bool, cudaStream_t) {
    return fail(IIR_EUNSUPPORTED, "per-sample path not built");
}
iir_status_t tv_backward(const iir_desc_t*, const Layout&, const void*, const void*, const void*, const void*,
                         const void*, const char*, void*, void*, void*, char*, bool, cudaStream_t) {
    return fail(IIR_EUNSUPPORTED, "per-sample path not built");
}
}  // namespace iirg
