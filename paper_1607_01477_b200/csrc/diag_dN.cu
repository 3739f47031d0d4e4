// diag_dN.cu -- instantiation of the diagonal-block kernel for scalar double, op N.
#include "diag_launch.cuh"

namespace mstrsm {
namespace rt {
template int launch_diag<double, false, 0>(const DiagArgs<double> &, int);
template int launch_diag<double, true, 0>(const DiagArgs<double> &, int);
}  // namespace rt
}  // namespace mstrsm
