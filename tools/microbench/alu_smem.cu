// Microbenchmark: FP32 issue rates (3-reg FFMA, imm FFMA, FADD) and LDS bandwidth on sm_100a.
// Used only to derive roofline denominators for DESIGN.md (not product code).
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void ffma_reg(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  float c = a, d = b;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = fmaf(x0, c, d); x1 = fmaf(x1, c, d); x2 = fmaf(x2, c, d); x3 = fmaf(x3, c, d);
      x4 = fmaf(x4, c, d); x5 = fmaf(x5, c, d); x6 = fmaf(x6, c, d); x7 = fmaf(x7, c, d);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void ffma_imm(float* out) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = fmaf(x0, 0.99f, 0.5f); x1 = fmaf(x1, 0.98f, 0.25f); x2 = fmaf(x2, 0.97f, 0.125f); x3 = fmaf(x3, 0.96f, 0.3f);
      x4 = fmaf(x4, 0.95f, 0.7f); x5 = fmaf(x5, 0.94f, 0.6f); x6 = fmaf(x6, 0.93f, 0.1f); x7 = fmaf(x7, 0.92f, 0.2f);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void fadd_reg(float* out, float a) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  float y0 = a, y1 = a * 2, y2 = a * 3, y3 = a * 4;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = x0 + y0; x1 = x1 - y1; x2 = x2 + y2; x3 = x3 - y3;
      x4 = x4 + y1; x5 = x5 - y2; x6 = x6 + y3; x7 = x7 - y0;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void lds_bw(float* out, int stride) {
  extern __shared__ float sm[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
  __syncthreads();
  float acc = 0;
  int base = threadIdx.x;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += sm[(base + j * 32 * stride) & 8191];
    base += 37;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void lds128_bw(float* out) {
  extern __shared__ float4 sm4[];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm4[i] = make_float4(i, i, i, i);
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  int base = threadIdx.x;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { float4 v = sm4[(base + j * 32) & 2047]; acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
    base += 37;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  printf("device %s sms %d clock(kHz) %d\n", p.name, sms, p.clockRate);
  float* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int threads = 512, blocks = sms * 4;
  double ops = (double)blocks * threads * ITERS * 32;  // lane-ops
  auto run = [&](const char* name, auto launch, double lane_ops) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    printf("%-10s %8.3f ms  %8.2f Tlane-op/s  %6.1f lane-op/clk/SM@1.9GHz\n", name, ms, lane_ops / ms / 1e9,
           lane_ops / (ms * 1e-3) / sms / 1.9e9);
  };
  run("ffma_reg", [&] { ffma_reg<<<blocks, threads>>>(out, 0.999f, 0.001f); }, ops);
  run("ffma_imm", [&] { ffma_imm<<<blocks, threads>>>(out); }, ops);
  run("fadd_reg", [&] { fadd_reg<<<blocks, threads>>>(out, 0.001f); }, ops);
  double lds_ops = (double)blocks * threads * ITERS * 8;
  run("lds32", [&] { lds_bw<<<blocks, threads, 8192 * 4>>>(out, 1); }, lds_ops);
  run("lds128", [&] { lds128_bw<<<blocks, threads, 8192 * 4>>>(out); }, lds_ops);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
