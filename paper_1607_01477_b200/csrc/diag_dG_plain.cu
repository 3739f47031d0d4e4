// diag_dG_plain.cu -- instantiation of the generalized diagonal-block kernel (Alg. 7/8) for scalar
// double, plain variant.
#include "diag_launch.cuh"

namespace mstrsm {
namespace rt {
template int launch_diag_gen<double, false>(const DiagArgs<double> &, int);
}  // namespace rt
}  // namespace mstrsm
