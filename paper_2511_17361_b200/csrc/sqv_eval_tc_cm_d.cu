// sqv_eval_tc_cm_d.cu — instantiations of the tcgen05 evaluator for C <= 24
#include "sqv_eval_tc_impl.cuh"

namespace sqv {
template int launch_tc<24>(const EvalArgs&, int, int, cudaStream_t);
}  // namespace sqv
