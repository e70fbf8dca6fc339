// Instantiation unit: LTI kernels for T = double, form = DF-II, M = 1..8.
#include "lti_host.cuh"
namespace iirg {
template iir_status_t run_lti_m<double, 0>(int, LtiCall&);
}  // namespace iirg
