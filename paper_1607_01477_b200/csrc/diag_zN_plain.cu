// diag_zN_plain.cu -- instantiation of the diagonal-block kernel for scalar cplx, op N, plain variant
// (one translation unit per instantiation set so the build compiles them in parallel).
#include "diag_launch.cuh"

namespace mstrsm {
namespace rt {
template int launch_diag<cplx, false, 0>(const DiagArgs<cplx> &, int);
}  // namespace rt
}  // namespace mstrsm
