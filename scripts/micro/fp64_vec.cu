// FP64 vector-pipe throughput and latency, LDS broadcast throughput (microbenchmark).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_tp(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void dfma_lat(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x;
  for (int i = 0; i < iters; ++i) x0 = fma(x0, a, b);
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0;
}
__global__ void dsqrt_lat(double* out, int iters) {
  double x0 = threadIdx.x + 2.0;
  for (int i = 0; i < iters; ++i) x0 = 1.0 / sqrt(x0) + 1.5;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0;
}
__global__ void lds_bcast(double* out, int iters) {
  __shared__ __align__(16) double s[256];
  s[threadIdx.x & 255] = threadIdx.x;
  __syncthreads();
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  for (int i = 0; i < iters; ++i) {
    const double* p = s + ((i * 8) & 255);
    acc0 += p[0]; acc1 += p[1]; acc2 += p[2]; acc3 += p[3];
    acc0 += p[4]; acc1 += p[5]; acc2 += p[6]; acc3 += p[7];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}
int main() {
  double* d; cudaMalloc(&d, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int iters = 1 << 14;
  for (int bs : {128, 256, 512}) {
    int grid = 148 * (2048 / bs);
    dfma_tp<<<grid, bs>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e0); dfma_tp<<<grid, bs>>>(d, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)grid * bs;
    printf("dfma throughput bs=%d: %.2f TFLOP/s (%.1f DFMA/clk/SM at 1.965 GHz)\n", bs, fl / ms / 1e9,
           fl / 2 / (ms * 1e-3) / 148 / 1.965e9);
  }
  dfma_lat<<<1, 32>>>(d, iters, 1.0000001, 1e-9);
  cudaEventRecord(e0); dfma_lat<<<1, 32>>>(d, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("dfma latency: %.1f clk\n", ms * 1e-3 * 1.965e9 / iters);
  dsqrt_lat<<<1, 32>>>(d, 1024);
  cudaEventRecord(e0); dsqrt_lat<<<1, 32>>>(d, 1024); cudaEventRecord(e1);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("1/sqrt + add latency: %.1f clk\n", ms * 1e-3 * 1.965e9 / 1024);
  for (int bs : {64, 256}) {
    int grid = 148 * (1024 / bs);
    lds_bcast<<<grid, bs>>>(d, iters);
    cudaEventRecord(e0); lds_bcast<<<grid, bs>>>(d, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double nld = 8.0 * iters * grid * (bs / 32);
    printf("broadcast LDS.64 bs=%d: %.2f warp-loads/clk/SM\n", bs, nld / (ms * 1e-3) / 148 / 1.965e9);
  }
  return 0;
}
