// DMMA (mma.sync m8n8k4 f64) throughput vs resident warps and independent
// accumulators per warp.  Development tool: what fraction of the FP64 tensor
// peak is reachable at the occupancy the on-the-fly GEMMs run at.
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[NACC][2];
#pragma unroll
  for (int t = 0; t < NACC; ++t) c[t][0] = c[t][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < NACC; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < NACC; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
void run(int sms, double* out, int warps_per_sm) {
  const int threads = 256;
  const int ctas = sms * warps_per_sm / 8;
  const int iters = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dmma<NACC><<<ctas, threads>>>(out, 10);
  cudaEventRecord(e0);
  k_dmma<NACC><<<ctas, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 512.0 * NACC * iters * (threads / 32) * (double)ctas;
  printf("warps/SM=%2d acc/warp=%2d : %6.2f TFLOP/s\n", warps_per_sm, NACC, flops / ms / 1e9);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 64 * 32);
  for (int w : {8, 16, 24, 32}) {
    run<4>(sms, out, w);
    run<8>(sms, out, w);
    run<16>(sms, out, w);
    run<26>(sms, out, w);
  }
  return 0;
}
