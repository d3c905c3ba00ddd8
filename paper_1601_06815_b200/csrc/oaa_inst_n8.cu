// Explicit instantiation of the n = 8 kernels (compiled in parallel by build.py).
#include "oaa_launch.cuh"
namespace oaa_host {
OAA_INSTANTIATE_N(8)
}  // namespace oaa_host
