// Explicit instantiation of the n = 7 kernels (compiled in parallel by build.py).
#include "oaa_launch.cuh"
namespace oaa_host {
OAA_INSTANTIATE_N(7)
}  // namespace oaa_host
