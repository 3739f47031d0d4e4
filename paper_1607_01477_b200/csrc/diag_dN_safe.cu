// diag_dN_safe.cu -- instantiation of the diagonal-block kernel for scalar double, op N, safe variant
// (one translation unit per instantiation set so the build compiles them in parallel).
#include "diag_launch.cuh"

namespace mstrsm {
namespace rt {
template int launch_diag<double, true, 0>(const DiagArgs<double> &, int);
}  // namespace rt
}  // namespace mstrsm
