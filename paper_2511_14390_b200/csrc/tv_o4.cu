// tv_o4.cu -- per-sample path instantiations, orders 25..32 (tv_impl.cuh).
#include "tv_impl.cuh"

namespace iirg {
IIRG_TV_INST(25)
IIRG_TV_INST(26)
IIRG_TV_INST(27)
IIRG_TV_INST(28)
IIRG_TV_INST(29)
IIRG_TV_INST(30)
IIRG_TV_INST(31)
IIRG_TV_INST(32)
}  // namespace iirg
