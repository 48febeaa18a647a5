// sqv_eval_tc_cm_b.cu — instantiations of the tcgen05 evaluator for C <= 16
#include "sqv_eval_tc_impl.cuh"

namespace sqv {
template int launch_tc<16>(const EvalArgs&, int, int, cudaStream_t);
}  // namespace sqv
