// camelot_inst_c8_n4.cu -- instantiations of the search launchers (camelot_inst.cuh): CM=8, NS in {4}, policy in {0,1}.
#define CAMELOT_INST_TU
#include "camelot_inst.cuh"

namespace cam {
#ifdef CAMELOT_SHARED_POLICY   // one instantiation serves both policies (policy = runtime argument)
CAMELOT_INSTANTIATE(8, 4, 2)
#else
CAMELOT_INSTANTIATE(8, 4, 0)
CAMELOT_INSTANTIATE(8, 4, 1)
#endif
}  // namespace cam
