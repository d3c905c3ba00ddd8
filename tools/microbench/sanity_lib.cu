// Minimal shared library with one kernel, loaded through ctypes after torch has created the
// CUDA context -- the same loading pattern as liboaa.so.  Used to check whether
// compute-sanitizer's "CUDA_ERROR_INVALID_HANDLE on cuKernelGetFunction" at the first
// launch comes from the runtime's lazy kernel lookup rather than from liboaa.
#include <cuda_runtime.h>
__global__ void sanity_kernel(float* p) { p[threadIdx.x] = 1.f; }
extern "C" int sanity_launch(float* p, void* stream) {
  sanity_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(p);
  return (int)cudaGetLastError();
}
