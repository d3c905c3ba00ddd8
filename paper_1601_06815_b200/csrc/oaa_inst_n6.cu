// Explicit instantiation of the n = 6 kernels (compiled in parallel by build.py).
#include "oaa_launch.cuh"
namespace oaa_host {
OAA_INSTANTIATE_N(6)
}  // namespace oaa_host
