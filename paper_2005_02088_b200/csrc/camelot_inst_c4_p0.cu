// camelot_inst_c4_p0.cu -- instantiations of the search launchers (camelot_inst.cuh): CM=4, NS in {4,6,8}, policy in {0}.
#define CAMELOT_INST_TU
#include "camelot_inst.cuh"

namespace cam {
#ifdef CAMELOT_SHARED_POLICY   // one instantiation serves both policies (policy = runtime argument)
CAMELOT_INSTANTIATE(4, 4, 2)
CAMELOT_INSTANTIATE(4, 6, 2)
CAMELOT_INSTANTIATE(4, 8, 2)
#else
CAMELOT_INSTANTIATE(4, 4, 0)
CAMELOT_INSTANTIATE(4, 6, 0)
CAMELOT_INSTANTIATE(4, 8, 0)
#endif
}  // namespace cam
