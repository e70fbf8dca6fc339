// Instantiation unit: LTI kernels for T = double, form = TDF-II, M = 1..8.
#include "lti_host.cuh"
namespace iirg {
template iir_status_t run_lti_m<double, 1>(int, LtiCall&);
}  // namespace iirg
