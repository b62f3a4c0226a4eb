// camelot_inst_c4_p1.cu -- instantiations of the search launchers (camelot_inst.cuh): CM=4, NS in {4,6,8}, policy in {1}.
#define CAMELOT_INST_TU
#include "camelot_inst.cuh"

namespace cam {
#ifndef CAMELOT_SHARED_POLICY
CAMELOT_INSTANTIATE(4, 4, 1)
CAMELOT_INSTANTIATE(4, 6, 1)
CAMELOT_INSTANTIATE(4, 8, 1)
#endif
}  // namespace cam
