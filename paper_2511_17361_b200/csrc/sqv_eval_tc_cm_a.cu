// sqv_eval_tc_cm_a.cu — instantiations of the tcgen05 evaluator for C <= 2/4/8/12
#include "sqv_eval_tc_impl.cuh"

namespace sqv {
template int launch_tc<2>(const EvalArgs&, int, int, cudaStream_t);
template int launch_tc<4>(const EvalArgs&, int, int, cudaStream_t);
template int launch_tc<8>(const EvalArgs&, int, int, cudaStream_t);
template int launch_tc<12>(const EvalArgs&, int, int, cudaStream_t);
}  // namespace sqv
