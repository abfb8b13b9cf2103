#include "../paper_2601_01437_b200/csrc/otf.cuh"
#include <cstdio>
using namespace irl;
int main() {
  size_t smem = 1024 + (size_t)OTF_ACC_STAGES * (OTF_TILE * 8 + OTF_BM * OTF_XW * 8 + OTF_BM * 16 + 16);
  auto fn = k_otf_acc_c<8>;
  int optin; cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  for (int carve : {-1, 100}) {
    if (carve >= 0) cudaFuncSetAttribute((const void*)fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, 288, smem);
    cudaFuncAttributes at; cudaFuncGetAttributes(&at, (const void*)fn);
    printf("carve %d smem %zu optin %d occ %d regs %d static %zu maxdyn %d\n", carve, smem, optin, occ, at.numRegs, at.sharedSizeBytes, at.maxDynamicSharedSizeBytes);
  }
  int per_sm; cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, 0);
  int rsv; cudaDeviceGetAttribute(&rsv, cudaDevAttrReservedSharedMemoryPerBlock, 0);
  printf("smem/SM %d reserved/block %d\n", per_sm, rsv);
}
