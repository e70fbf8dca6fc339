// tv_o3.cu -- per-sample path instantiations, orders 17..24 (tv_impl.cuh).
#include "tv_impl.cuh"

namespace iirg {
IIRG_TV_INST(17)
IIRG_TV_INST(18)
IIRG_TV_INST(19)
IIRG_TV_INST(20)
IIRG_TV_INST(21)
IIRG_TV_INST(22)
IIRG_TV_INST(23)
IIRG_TV_INST(24)
}  // namespace iirg
