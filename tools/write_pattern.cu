// Store-pattern microbenchmark for the O-row writer (development tool): CTAs
// (row block b, column tile c) write rows [lo_b, hi_b) x units [c*W, (c+1)*W) of
// an N x ld_u (16-byte units) matrix, PPT units per thread per row, streaming
// stores.  Compares tile counts at the cfg2 and cfg5 shapes.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_write(double2* O, long n_rows, long ld_u, int ppt, int nb, int C) {
  const int rank = blockIdx.x % C, blk = blockIdx.x / C;
  const long lo = n_rows * blk / nb, hi = n_rows * (blk + 1) / nb;
  const long c0 = ld_u * rank / C, c1 = ld_u * (rank + 1) / C;
  const int nt = blockDim.x;
  for (long r = lo; r < hi; ++r) {
    double2* row = O + r * ld_u;
    for (int k = 0; k < ppt; ++k) {
      const long u = c0 + threadIdx.x + (long)k * nt;
      if (u < c1) {
        double2 v = make_double2((double)r, (double)u);
        asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(row + u), "d"(v.x), "d"(v.y) : "memory");
      }
    }
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double2* O;
  const long maxb = 65536L * 104512 * 16;
  if (cudaMalloc(&O, maxb) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct G { long N, ld; int C, nt, ppt, per_sm; } gs[] = {
      {65536, 3312, 1, 416, 8, 1},      {65536, 104512, 26, 512, 8, 2},  {65536, 104512, 26, 512, 8, 1},
      {65536, 104512, 52, 512, 4, 2},   {65536, 104512, 13, 1024, 8, 1}, {65536, 104512, 1, 1024, 103, 1},
      {65536, 104512, 2, 1024, 52, 1}};
  for (auto g : gs) {
    const int nb = (sms * g.per_sm + g.C - 1) / g.C;
    k_write<<<nb * g.C, g.nt>>>(O, g.N, g.ld, g.ppt, nb, g.C);
    cudaEventRecord(e0);
    for (int i = 0; i < 2; ++i) k_write<<<nb * g.C, g.nt>>>(O, g.N, g.ld, g.ppt, nb, g.C);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("N %ld ld_u %ld C %3d nt %4d ppt %3d nb %3d : %.3f ms  %.0f GB/s  (%s)\n", g.N, g.ld, g.C, g.nt, g.ppt, nb,
           ms / 2, g.N * g.ld * 16.0 / (ms / 2 * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
