// diag_zC.cu -- instantiation of the diagonal-block kernel for scalar cplx, op C.
#include "diag_launch.cuh"

namespace mstrsm {
namespace rt {
template int launch_diag<cplx, false, 1>(const DiagArgs<cplx> &, int);
template int launch_diag<cplx, true, 1>(const DiagArgs<cplx> &, int);
}  // namespace rt
}  // namespace mstrsm
