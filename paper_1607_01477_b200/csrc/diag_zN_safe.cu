// diag_zN_safe.cu -- instantiation of the diagonal-block kernel for scalar cplx, op N, safe variant
// (one translation unit per instantiation set so the build compiles them in parallel).
#include "diag_launch.cuh"

namespace mstrsm {
namespace rt {
template int launch_diag<cplx, true, 0>(const DiagArgs<cplx> &, int);
}  // namespace rt
}  // namespace mstrsm
