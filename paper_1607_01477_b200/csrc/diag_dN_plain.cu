// diag_dN_plain.cu -- instantiation of the diagonal-block kernel for scalar double, op N, plain variant
// (one translation unit per instantiation set so the build compiles them in parallel).
#include "diag_launch.cuh"

namespace mstrsm {
namespace rt {
template int launch_diag<double, false, 0>(const DiagArgs<double> &, int);
}  // namespace rt
}  // namespace mstrsm
