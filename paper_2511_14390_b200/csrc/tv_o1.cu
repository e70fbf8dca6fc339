// tv_o1.cu -- per-sample path instantiations, orders 1..8 (tv_impl.cuh).
#include "tv_impl.cuh"

namespace iirg {
IIRG_TV_INST(1)
IIRG_TV_INST(2)
IIRG_TV_INST(3)
IIRG_TV_INST(4)
IIRG_TV_INST(5)
IIRG_TV_INST(6)
IIRG_TV_INST(7)
IIRG_TV_INST(8)
}  // namespace iirg
