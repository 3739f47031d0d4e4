// diag_dC.cu -- instantiation of the diagonal-block kernel for scalar double, op C.
#include "diag_launch.cuh"

namespace mstrsm {
namespace rt {
template int launch_diag<double, false, 1>(const DiagArgs<double> &, int);
template int launch_diag<double, true, 1>(const DiagArgs<double> &, int);
}  // namespace rt
}  // namespace mstrsm
