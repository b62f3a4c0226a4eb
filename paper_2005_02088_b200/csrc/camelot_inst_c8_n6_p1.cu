// camelot_inst_c8_n6_p1.cu -- instantiations of the search launchers (camelot_inst.cuh): CM=8, NS in {6}, policy in {1}.
#define CAMELOT_INST_TU
#include "camelot_inst.cuh"

namespace cam {
#ifndef CAMELOT_SHARED_POLICY
CAMELOT_INSTANTIATE(8, 6, 1)
#endif
}  // namespace cam
