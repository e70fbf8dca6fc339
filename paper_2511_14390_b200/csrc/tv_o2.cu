// tv_o2.cu -- per-sample path instantiations, orders 9..16 (tv_impl.cuh).
#include "tv_impl.cuh"

namespace iirg {
IIRG_TV_INST(9)
IIRG_TV_INST(10)
IIRG_TV_INST(11)
IIRG_TV_INST(12)
IIRG_TV_INST(13)
IIRG_TV_INST(14)
IIRG_TV_INST(15)
IIRG_TV_INST(16)
}  // namespace iirg
