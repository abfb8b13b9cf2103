// Development probe: does every SM stream its column slice of every row at
// the same rate?  One CTA per SM, CTA c reads columns [c W, (c+1) W) of every
// row of an N x ld f64 matrix through a TMA bulk-copy ring (the wide
// product's access pattern, no exchange).  Prints per-CTA finish times.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ssp tools/slice_stream_probe.cu
//   /tmp/ssp <rows> <ld_units> <rows_per_stage> <stages> [align_units] [test_wait 0/1]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <bool TEST>
__global__ void __launch_bounds__(64, 1) k_probe(const double2* O, long long n, long long ld_u, int W, int RS,
                                                 int NS, unsigned long long* fin, int align) {
  extern __shared__ __align__(16) unsigned char sm[];
  double2* ring = (double2*)sm;
  unsigned long long* full = (unsigned long long*)(sm + (size_t)NS * RS * W * 16);
  const int c = blockIdx.x, G = gridDim.x;
  long long col0 = (ld_u * c) / G;
  col0 = (col0 / align) * align;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const long long NB = (n + RS - 1) / RS;
  if (tid == 0) {
    for (long long b = 0; b < NB; ++b) {
      const int s = b % NS;
      if (b >= NS) {  // wait for the previous use of this stage to land (consumer = us)
        const unsigned ph = ((b / NS) - 1) & 1;
        unsigned ok = 0;
        while (!ok) {
          if (TEST)
            asm volatile("{.reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(smem_addr(&full[s])), "r"(ph) : "memory");
          else
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(smem_addr(&full[s])), "r"(ph) : "memory");
        }
      }
      const long long r0 = b * RS;
      const int rows = (int)min((long long)RS, n - r0);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&full[s])),
                   "r"(rows * W * 16) : "memory");
      for (int i = 0; i < rows; ++i)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_addr(ring + ((size_t)s * RS + i) * W)),
                     "l"(O + (r0 + i) * ld_u + col0), "r"(W * 16), "r"(smem_addr(&full[s]))
                     : "memory");
    }
    for (long long b = max(0LL, NB - NS); b < NB; ++b) {
      const int s = b % NS;
      const unsigned ph = (b / NS) & 1;
      unsigned ok = 0;
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"(smem_addr(&full[s])), "r"(ph) : "memory");
    }
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    fin[c * 2] = t1 - t0;
    fin[c * 2 + 1] = smid;
  }
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : 131072;
  const long long ld_u = argc > 2 ? atoll(argv[2]) : 29344;
  const int RS = argc > 3 ? atoi(argv[3]) : 4;
  const int NS = argc > 4 ? atoi(argv[4]) : 16;
  const int align = argc > 5 ? atoi(argv[5]) : 1;
  const int test = argc > 6 ? atoi(argv[6]) : 0;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int W = (int)((ld_u + sms - 1) / sms) + align;
  double2* O;
  if (cudaMalloc(&O, (size_t)n * ld_u * 16 + 4096) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(O, 0, (size_t)n * ld_u * 16);
  unsigned long long* fin;
  cudaMalloc(&fin, sms * 16);
  const size_t smem = (size_t)NS * RS * W * 16 + NS * 8;
  auto kern = test ? k_probe<true> : k_probe<false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<sms, 64, smem>>>(O, n, ld_u, W, RS, NS, fin, align);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h(sms * 2);
    cudaMemcpy(h.data(), fin, sms * 16, cudaMemcpyDeviceToHost);
    std::vector<std::pair<double, int>> t;
    for (int c = 0; c < sms; ++c) t.push_back({h[c * 2] / 1e6, (int)h[c * 2 + 1]});
    std::sort(t.begin(), t.end());
    const double bytes = (double)n * sms * W * 16;
    printf("rep %d: %.3f ms (%.0f GB/s of slices; %s)  per-CTA ms: min %.3f (sm %d) median %.3f max %.3f (sm %d) | 5 slowest:",
           rep, ms, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()), t[0].first, t[0].second,
           t[sms / 2].first, t.back().first, t.back().second);
    for (int i = sms - 5; i < sms; ++i) printf(" %.3f(sm%d)", t[i].first, t[i].second);
    printf("\n");
  }
  return 0;
}
