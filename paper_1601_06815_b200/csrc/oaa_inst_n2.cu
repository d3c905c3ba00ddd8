// Explicit instantiation of the n = 2 kernels (compiled in parallel by build.py).
#include "oaa_launch.cuh"
namespace oaa_host {
OAA_INSTANTIATE_N(2)
}  // namespace oaa_host
