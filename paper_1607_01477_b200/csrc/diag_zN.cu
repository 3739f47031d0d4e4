// diag_zN.cu -- instantiation of the diagonal-block kernel for scalar cplx, op N.
#include "diag_launch.cuh"

namespace mstrsm {
namespace rt {
template int launch_diag<cplx, false, 0>(const DiagArgs<cplx> &, int);
template int launch_diag<cplx, true, 0>(const DiagArgs<cplx> &, int);
}  // namespace rt
}  // namespace mstrsm
