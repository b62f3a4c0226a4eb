// camelot_inst_c8_n6_p0.cu -- instantiations of the search launchers (camelot_inst.cuh): CM=8, NS in {6}, policy in {0}.
#define CAMELOT_INST_TU
#include "camelot_inst.cuh"

namespace cam {
#ifdef CAMELOT_SHARED_POLICY   // one instantiation serves both policies (policy = runtime argument)
CAMELOT_INSTANTIATE(8, 6, 2)
#else
CAMELOT_INSTANTIATE(8, 6, 0)
#endif
}  // namespace cam
