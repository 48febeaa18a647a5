// sqv_eval_tc_cm_c.cu — instantiations of the tcgen05 evaluator for C <= 18
#include "sqv_eval_tc_impl.cuh"

namespace sqv {
template int launch_tc<18>(const EvalArgs&, int, int, cudaStream_t);
}  // namespace sqv
