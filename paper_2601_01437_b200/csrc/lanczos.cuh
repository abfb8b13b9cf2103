// Lanczos step for short vectors (kry:96-116) fused into ONE single-CTA kernel.
//
// On entry W = A v_j.  The kernel performs, on device scalars only:
//   alpha_j = v_j . W ;  W -= alpha_j v_j + beta_{j-1} v_{j-1}
//   twice:   h = V_{0..j} W ;  W -= V^T h          (full reorthogonalisation)
//   beta_j = ||W|| ;  V[j+1] = W / max(beta_j, tiny)
// and stores (alpha_j, beta_j) into ab[0][j], ab[1][j].  It replaces ~14
// separate BLAS-1/2 launches per Lanczos step when L is small enough that one
// SM streams V faster than the launch latency of the multi-kernel version.
// All reductions are fixed-order (warp butterflies, warps in index order).
#pragma once
#include "common.cuh"

namespace irl {

__device__ __forceinline__ double block_sum_f64(double x, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  x = warp_sum<false>(x);
  __syncthreads();  // sh reuse
  if (lane == 0) sh[warp] = x;
  __syncthreads();
  double t = (lane < nw) ? sh[lane] : 0.0;
  return warp_sum<false>(t);
}

__global__ void __launch_bounds__(1024) k_lanczos_small(double* __restrict__ V, int64_t ldv, double* __restrict__ W,
                                                         int64_t L, int j, int m, double* __restrict__ ab) {
  __shared__ double sh[32];
  __shared__ double hs[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const double* vj = V + (int64_t)j * ldv;
  // alpha
  double p = 0.0;
  for (int64_t e = tid; e < L; e += blockDim.x) p = fma(vj[e], W[e], p);
  const double alpha = block_sum_f64(p, sh);
  const double bprev = j > 0 ? ab[m + j - 1] : 0.0;
  const double* vp = j > 0 ? V + (int64_t)(j - 1) * ldv : nullptr;
  for (int64_t e = tid; e < L; e += blockDim.x) {
    double w = W[e] - alpha * vj[e];
    if (vp) w -= bprev * vp[e];
    W[e] = w;
  }
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    // h_i = V_i . W, one warp per basis row
    for (int i = warp; i <= j; i += nw) {
      const double* vi = V + (int64_t)i * ldv;
      double q = 0.0;
      for (int64_t e = lane; e < L; e += 32) q = fma(vi[e], W[e], q);
      q = warp_sum<false>(q);
      if (lane == 0) hs[i] = q;
    }
    __syncthreads();
    for (int64_t e = tid; e < L; e += blockDim.x) {
      double acc = 0.0;
      for (int i = 0; i <= j; ++i) acc = fma(hs[i], V[(int64_t)i * ldv + e], acc);
      W[e] -= acc;
    }
    __syncthreads();
  }
  double nrm = 0.0;
  for (int64_t e = tid; e < L; e += blockDim.x) nrm = fma(W[e], W[e], nrm);
  const double beta = sqrt(block_sum_f64(nrm, sh));
  const double inv = 1.0 / fmax(beta, 1e-300);
  double* vn = V + (int64_t)(j + 1) * ldv;
  for (int64_t e = tid; e < L; e += blockDim.x) vn[e] = W[e] * inv;
  if (tid == 0) {
    ab[j] = alpha;
    ab[m + j] = beta;
  }
}

}  // namespace irl

namespace irl {

// ---------------------------------------------------------------------------
// The same Lanczos step (kry:96-116) for medium L on ONE thread-block cluster:
// CTA r of the cluster owns the element slice [L r / CS, L (r+1) / CS) of V and
// W.  Each dot product (alpha, the two reorthogonalisation coefficient vectors,
// beta) is a per-CTA partial followed by a fixed-order sum over the cluster's
// shared memories (DSMEM), so every CTA holds bit-identical scalars and the
// result does not depend on timing.  Four exchanges, one cluster barrier each;
// every exchange has its own buffer, so no buffer is rewritten while a peer
// may still read it.
// ---------------------------------------------------------------------------
constexpr int LZ_MAXJ = 64;

// fixed-order cluster sum of part[0..cnt) (this CTA's partials) -> out[0..cnt)
__device__ __forceinline__ void lz_cluster_sum(const double* part, double* out, int cnt, int cs) {
  cluster_sync();  // release this CTA's partials / acquire the peers'
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const uint32_t a = smem_addr(part + i);
    double s = 0.0;
    for (int r = 0; r < cs; ++r) s += ld_cluster(map_to_rank(a, (uint32_t)r), (double*)nullptr);
    out[i] = s;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(512) k_lanczos_cluster(double* __restrict__ V, int64_t ldv, double* __restrict__ W,
                                                          int64_t L, int j, int m, double* __restrict__ ab) {
  __shared__ double sh[32];
  __shared__ double p_alpha[1], p_beta[1], p_h0[LZ_MAXJ], p_h1[LZ_MAXJ];
  __shared__ double s_alpha[1], s_beta[1], s_h[LZ_MAXJ];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int cs = (int)(gridDim.x * gridDim.y * gridDim.z);  // one cluster spans the grid
  const int rank = (int)cluster_rank();
  const int64_t lo = L * rank / cs, hi = L * (rank + 1) / cs;
  const double* vj = V + (int64_t)j * ldv;

  double p = 0.0;
  for (int64_t e = lo + tid; e < hi; e += blockDim.x) p = fma(vj[e], W[e], p);
  p = block_sum_f64(p, sh);
  if (tid == 0) p_alpha[0] = p;
  lz_cluster_sum(p_alpha, s_alpha, 1, cs);
  const double alpha = s_alpha[0];
  const double bprev = j > 0 ? ab[m + j - 1] : 0.0;
  const double* vp = j > 0 ? V + (int64_t)(j - 1) * ldv : nullptr;
  for (int64_t e = lo + tid; e < hi; e += blockDim.x) {
    double w = W[e] - alpha * vj[e];
    if (vp) w -= bprev * vp[e];
    W[e] = w;
  }
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    double* ph = pass == 0 ? p_h0 : p_h1;
    for (int i = warp; i <= j; i += nw) {  // one warp per basis row over this slice
      const double* vi = V + (int64_t)i * ldv;
      double q = 0.0;
      for (int64_t e = lo + lane; e < hi; e += 32) q = fma(vi[e], W[e], q);
      q = warp_sum<false>(q);
      if (lane == 0) ph[i] = q;
    }
    lz_cluster_sum(ph, s_h, j + 1, cs);
    for (int64_t e = lo + tid; e < hi; e += blockDim.x) {
      double acc = 0.0;
      for (int i = 0; i <= j; ++i) acc = fma(s_h[i], V[(int64_t)i * ldv + e], acc);
      W[e] -= acc;
    }
    __syncthreads();  // s_h is rewritten by the next pass
  }
  double nrm = 0.0;
  for (int64_t e = lo + tid; e < hi; e += blockDim.x) nrm = fma(W[e], W[e], nrm);
  nrm = block_sum_f64(nrm, sh);
  if (tid == 0) p_beta[0] = nrm;
  lz_cluster_sum(p_beta, s_beta, 1, cs);
  const double beta = sqrt(s_beta[0]);
  const double inv = 1.0 / fmax(beta, 1e-300);
  double* vn = V + (int64_t)(j + 1) * ldv;
  for (int64_t e = lo + tid; e < hi; e += blockDim.x) vn[e] = W[e] * inv;
  if (rank == 0 && tid == 0) {
    ab[j] = alpha;
    ab[m + j] = beta;
  }
  cluster_sync();  // no CTA leaves while a peer may still read its partials
}

}  // namespace irl

namespace irl {

// The one-cluster step with the CTA's slice of V (rows 0..j) and W staged in
// shared memory by TMA bulk copies at kernel start: the four passes over the
// basis then read shared memory instead of L2, which removes three L2 round
// trips from the step's critical path.  Slices are whole 16-byte units (L is
// even for every bordered layout; the host checks).  Same arithmetic order as
// k_lanczos_cluster.
__global__ void __launch_bounds__(512) k_lanczos_cluster_smem(double* __restrict__ V, int64_t ldv,
                                                               double* __restrict__ W, int64_t L, int j, int m,
                                                               double* __restrict__ ab) {
  extern __shared__ __align__(16) double lz_sm[];
  __shared__ double sh[32];
  __shared__ double p_alpha[1], p_beta[1], p_h0[LZ_MAXJ], p_h1[LZ_MAXJ];
  __shared__ double s_alpha[1], s_beta[1], s_h[LZ_MAXJ];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int cs = (int)(gridDim.x * gridDim.y * gridDim.z);
  const int rank = (int)cluster_rank();
  const int64_t units = L >> 1;
  const int64_t lo = 2 * (units * rank / cs), hi = 2 * (units * (rank + 1) / cs);
  const int S = (int)(hi - lo);
  double* vs = lz_sm;                           // [j+1][S]
  double* ws = lz_sm + (int64_t)(j + 1) * S;    // [S]
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar, (uint32_t)((j + 2) * S * 8));
    for (int i = 0; i <= j; ++i) bulk_g2s(vs + (int64_t)i * S, V + (int64_t)i * ldv + lo, (uint32_t)S * 8u, &bar);
    bulk_g2s(ws, W + lo, (uint32_t)S * 8u, &bar);
  }
  mbar_wait(&bar, 0);
  const double* vj = vs + (int64_t)j * S;

  double p = 0.0;
  for (int e = tid; e < S; e += blockDim.x) p = fma(vj[e], ws[e], p);
  p = block_sum_f64(p, sh);
  if (tid == 0) p_alpha[0] = p;
  lz_cluster_sum(p_alpha, s_alpha, 1, cs);
  const double alpha = s_alpha[0];
  const double bprev = j > 0 ? ab[m + j - 1] : 0.0;
  const double* vp = j > 0 ? vs + (int64_t)(j - 1) * S : nullptr;
  for (int e = tid; e < S; e += blockDim.x) {
    double w = ws[e] - alpha * vj[e];
    if (vp) w -= bprev * vp[e];
    ws[e] = w;
  }
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    double* ph = pass == 0 ? p_h0 : p_h1;
    for (int i = warp; i <= j; i += nw) {
      const double* vi = vs + (int64_t)i * S;
      double q = 0.0;
      for (int e = lane; e < S; e += 32) q = fma(vi[e], ws[e], q);
      q = warp_sum<false>(q);
      if (lane == 0) ph[i] = q;
    }
    lz_cluster_sum(ph, s_h, j + 1, cs);
    for (int e = tid; e < S; e += blockDim.x) {
      double acc = 0.0;
      for (int i = 0; i <= j; ++i) acc = fma(s_h[i], vs[(int64_t)i * S + e], acc);
      ws[e] -= acc;
    }
    __syncthreads();
  }
  double nrm = 0.0;
  for (int e = tid; e < S; e += blockDim.x) nrm = fma(ws[e], ws[e], nrm);
  nrm = block_sum_f64(nrm, sh);
  if (tid == 0) p_beta[0] = nrm;
  lz_cluster_sum(p_beta, s_beta, 1, cs);
  const double beta = sqrt(s_beta[0]);
  const double inv = 1.0 / fmax(beta, 1e-300);
  double* vn = V + (int64_t)(j + 1) * ldv + lo;
  for (int e = tid; e < S; e += blockDim.x) {
    const double w = ws[e];
    W[lo + e] = w;
    vn[e] = w * inv;
  }
  if (rank == 0 && tid == 0) {
    ab[j] = alpha;
    ab[m + j] = beta;
  }
  cluster_sync();
}

}  // namespace irl
