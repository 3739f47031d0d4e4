// diag_dG_safe.cu -- instantiation of the generalized diagonal-block kernel (Alg. 7/8) for scalar
// double, safe variant.
#include "diag_launch.cuh"

namespace mstrsm {
namespace rt {
template int launch_diag_gen<double, true>(const DiagArgs<double> &, int);
}  // namespace rt
}  // namespace mstrsm
