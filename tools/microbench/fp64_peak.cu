// DFMA/FFMA-chain microbenchmark: measures the B200 FP64 and FP32 CUDA-core
// peaks that the roofline in DESIGN.md divides by (MEASURED_PEAKS.json has
// neither).  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int CHAINS, class T = double>
__global__ void dfma_kernel(T* out, int iters, T a, T b) {
  T x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == T(12345.678)) out[threadIdx.x] = s;
}
__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, ", p.name, p.multiProcessorCount);
  double* out; cudaMalloc(&out, 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000; int blocks = p.multiProcessorCount * 8; int threads = 256;
  dfma_kernel<8><<<blocks, threads>>>(out, 100, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * 8 * (double)iters * blocks * threads;
  printf("\"fp64_tflops\": %.3f, ", flops / (best * 1e-3) / 1e12);
  // sustained: back to back for ~3 s
  cudaEventRecord(e0);
  int reps = 0; float tot = 0;
  while (tot < 3000.f) {
    for (int k = 0; k < 10; ++k) dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    reps += 10; cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&tot, e0, e1);
  }
  printf("\"fp64_tflops_sustained\": %.3f, ", flops * reps / (tot * 1e-3) / 1e12);
  {  // FP32: 16 independent FFMA chains per thread
    float* outf; cudaMalloc(&outf, 1024 * 4);
    dfma_kernel<16, float><<<blocks, threads>>>(outf, 100, 0.999999f, 1e-7f);
    cudaDeviceSynchronize();
    best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      dfma_kernel<16, float><<<blocks, threads>>>(outf, iters, 0.999999f, 1e-7f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("\"fp32_tflops\": %.3f, ", 2.0 * 16 * (double)iters * blocks * threads / (best * 1e-3) / 1e12);
  }
  size_t n = (size_t)1 << 28;  // 2^28 double2 = 4 GiB each
  double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16);
  copy_kernel<<<p.multiProcessorCount * 16, 512>>>(a, b, n); cudaDeviceSynchronize();
  best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0); copy_kernel<<<p.multiProcessorCount * 16, 512>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf("\"copy_gbs\": %.1f}\n", 2.0 * n * 16 / (best * 1e-3) / 1e9);
  return 0;
}
