// Second translation unit for the two-object variant of sanity_lib.cu (see tools/sanity_lib.py).
#include <cuda_runtime.h>
template <int N> __global__ void sanity_kernel2(float* p) { p[threadIdx.x] += (float)N; }
template __global__ void sanity_kernel2<1>(float*);
extern "C" int sanity_launch2(float* p, void* stream) {
  sanity_kernel2<1><<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(p);
  return (int)cudaGetLastError();
}
