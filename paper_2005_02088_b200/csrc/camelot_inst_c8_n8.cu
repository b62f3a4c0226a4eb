// camelot_inst_c8_n8.cu -- instantiations of the search launchers (camelot_inst.cuh): CM=8, NS in {8}, policy in {0,1}.
#define CAMELOT_INST_TU
#include "camelot_inst.cuh"

namespace cam {
#ifdef CAMELOT_SHARED_POLICY   // one instantiation serves both policies (policy = runtime argument)
CAMELOT_INSTANTIATE(8, 8, 2)
#else
CAMELOT_INSTANTIATE(8, 8, 0)
CAMELOT_INSTANTIATE(8, 8, 1)
#endif
}  // namespace cam
