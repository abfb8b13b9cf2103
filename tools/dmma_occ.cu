// DMMA throughput vs warps per SM and independent accumulator chains (development tool)
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[CH][2];
  for (int t = 0; t < CH; ++t) c[t][0] = c[t][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < CH; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < CH; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
void run(int sms, int blocks_per_sm, int threads, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  k<CH><<<sms * blocks_per_sm, threads>>>(out, 10);
  cudaEventRecord(e0);
  k<CH><<<sms * blocks_per_sm, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 256 * CH * iters * (double)(threads / 32) * sms * blocks_per_sm;
  printf("chains=%2d warps/SM=%2d : %.1f TFLOP/s\n", CH, blocks_per_sm * threads / 32, flops / ms / 1e9);
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 4 * 1024);
  for (int w : {4, 8, 12, 16}) {
    run<4>(sms, 1, w * 32, out);
    run<8>(sms, 1, w * 32, out);
    run<16>(sms, 1, w * 32, out);
  }
  return 0;
}
