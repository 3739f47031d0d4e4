// diag_zG_safe.cu -- instantiation of the generalized diagonal-block kernel (Alg. 7/8) for scalar
// cplx, safe variant.
#include "diag_launch.cuh"

namespace mstrsm {
namespace rt {
template int launch_diag_gen<cplx, true>(const DiagArgs<cplx> &, int);
}  // namespace rt
}  // namespace mstrsm
