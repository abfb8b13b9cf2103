// Two-configuration completion of H_eff and batched log psi.
//
// heff_offdiag_matvec (estimators.py:254-294) adds to the single-configuration
// product the couplings <x|H|y> psi(y)/psi(x) between every sampled
// configuration x_n and its connected partners y:
//
//   corr_n = sum_{e in seg(k_n)} coeff_e (q_part[row_e] - q_n),   k_n = dist_index[n]
//   out    = Re( (w corr) @ conj(O_c) ),        q = (O - Obar) v,  q_part = (O_part - Obar) v
//
// Split per row into a coefficient on the row's own q_n and a term that does
// not depend on it:
//
//   w_n corr_n = -(w_n S_k) q_n + w_n R_k,   S_k = sum coeff_e,  R_k = sum coeff_e q_part[row_e]
//
// so the whole connected product (diagonal + completion, optimizer.py:144-147)
// is ONE ordinary streaming product over the batch O with per-row coefficient
// a_n = c_n - w_n S_k and additive term d_n = w_n R_k (StreamArgs::yadd).
// q_part comes from a MODE_DOT pass over the partner rows; k_connected_rows
// forms a_n, d_n with one warp per row (fixed-order lane strides + butterfly:
// deterministic).
//
// k_logamp_part / k_logamp_finish: log psi for the shallow NQS (the role of
// ansatz.log_amplitude, ansatz.py:200-247, for the RBM / MLP of BASELINE.json),
// needed for the partner amplitude ratios psi(y)/psi(x):
//   RBM  log psi = a.x + sum_j log cosh(b_j + W_j.x)       (complex for complex theta)
//   MLP  log psi = u.tanh(b + W x) + c
#pragma once
#include "common.cuh"
#include "obuild.cuh"  // MODEL_RBM / MODEL_MLP

namespace irl {

// ------------------------------------------------------------ completion ---
template <bool CPLX>
__global__ void __launch_bounds__(256) k_connected_rows(
    const int64_t* __restrict__ dist_index, const int64_t* __restrict__ indptr, const int64_t* __restrict__ prow,
    const typename Traits<CPLX>::S* __restrict__ pcoeff, const typename Traits<CPLX>::S* __restrict__ tpart_p,
    int C, int64_t m, const typename Traits<CPLX>::S* __restrict__ spart, const double* __restrict__ w,
    const typename Traits<CPLX>::S* __restrict__ cdiag, int64_t n, typename Traits<CPLX>::S* __restrict__ a_out,
    typename Traits<CPLX>::S* __restrict__ d_out) {
  using T = Traits<CPLX>;
  using S = typename T::S;
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // s = Obar . v, summed over the DOT pass's column slices in order (as MODE_ACC does)
  S s = T::zero();  // spart == nullptr: tpart_p already holds centred dots
  if (m > 0 && spart)
    for (int c = 0; c < C; ++c) s = T::add(s, spart[c]);
  for (int64_t r = warp0; r < n; r += nwarps) {
    const int64_t k = dist_index[r];
    const int64_t e0 = indptr[k], e1 = indptr[k + 1];
    S R = T::zero(), Ssum = T::zero();
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const S ce = pcoeff[e];
      const int64_t pr = prow[e];
      S q = T::zero();
      for (int c = 0; c < C; ++c) q = T::add(q, tpart_p[(int64_t)c * m + pr]);
      q = T::sub(q, s);
      R = T::add(R, T::mul(ce, q));
      Ssum = T::add(Ssum, ce);
    }
    R = warp_sum<CPLX>(R);
    Ssum = warp_sum<CPLX>(Ssum);
    if (lane == 0) {
      const double wr = w[r];
      S wS, wR;
      if constexpr (CPLX) {
        wS = make_double2(wr * Ssum.x, wr * Ssum.y);
        wR = make_double2(wr * R.x, wr * R.y);
      } else {
        wS = wr * Ssum;
        wR = wr * R;
      }
      a_out[r] = T::sub(cdiag ? cdiag[r] : T::zero(), wS);
      d_out[r] = wR;
    }
  }
}

// ---------------------------------------------------------------- log psi ---
__device__ __forceinline__ double2 clogcosh(double2 z) {
  // principal log of cosh(z) = cosh x cos y + i sinh x sin y  (numpy: log(cosh(z)))
  double sy, cy;
  sincos(z.y, &sy, &cy);
  const double re = cosh(z.x) * cy, im = sinh(z.x) * sy;
  return make_double2(log(hypot(re, im)), atan2(im, re));
}

// Partial sums over 32 hidden units per (row, j-tile): part[jt * n + row].
// Grid (row blocks, j tiles); W tile staged transposed in shared memory as in
// k_hidden (obuild.cuh); theta_j = b_j + sum over the row's set bits.
template <bool CPLX, int MODEL>
__global__ void __launch_bounds__(256) k_logamp_part(const uint8_t* __restrict__ x, int64_t n_rows, int n_vis,
                                                     int hidden, const typename Traits<CPLX>::S* __restrict__ Wm,
                                                     const typename Traits<CPLX>::S* __restrict__ bvec,
                                                     const double* __restrict__ uvec,
                                                     typename Traits<CPLX>::S* __restrict__ part) {
  using S = typename Traits<CPLX>::S;
  extern __shared__ __align__(16) unsigned char smem_l[];
  S* Wt = reinterpret_cast<S*>(smem_l);  // [n_vis][32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j0 = blockIdx.y * 32;
  const int j = j0 + lane;
  const bool jok = j < hidden;
  for (int e = threadIdx.x; e < n_vis * 32; e += blockDim.x) {
    const int i = e / 32, jj = e % 32;
    S val = Traits<CPLX>::zero();
    if (j0 + jj < hidden) val = Wm[(int64_t)(j0 + jj) * n_vis + i];
    Wt[i * 32 + jj] = val;
  }
  __syncthreads();
  const S bj = jok ? bvec[j] : Traits<CPLX>::zero();
  const double uj = (MODEL == MODEL_MLP && jok) ? uvec[j] : 0.0;
  const int64_t rows_per_blk = (n_rows + gridDim.x - 1) / gridDim.x;
  const int64_t r_lo = blockIdx.x * rows_per_blk;
  const int64_t r_hi = min(n_rows, r_lo + rows_per_blk);
  for (int64_t r = r_lo + warp; r < r_hi; r += 8) {
    S acc = bj;
    const uint8_t* xr = x + r * n_vis;
    for (int i0 = 0; i0 < n_vis; i0 += 32) {
      const bool on = (i0 + lane < n_vis) && xr[i0 + lane] != 0;
      uint32_t bits = __ballot_sync(0xffffffffu, on);
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        acc = Traits<CPLX>::add(acc, Wt[(i0 + b) * 32 + lane]);
      }
    }
    S f = Traits<CPLX>::zero();
    if (jok) {
      if constexpr (CPLX) {
        f = clogcosh(acc);
      } else if constexpr (MODEL == MODEL_RBM) {
        f = log(cosh(acc));
      } else {
        f = uj * tanh(acc);
      }
    }
    f = warp_sum<CPLX>(f);
    if (lane == 0) part[(int64_t)blockIdx.y * n_rows + r] = f;
  }
}

// log psi_n = sum_jt part[jt][n] (+ a . x_n for the RBM, + c for the MLP)
template <bool CPLX, int MODEL>
__global__ void __launch_bounds__(256) k_logamp_finish(const uint8_t* __restrict__ x, int64_t n_rows, int n_vis,
                                                       int jt_count, const typename Traits<CPLX>::S* __restrict__ avec,
                                                       const double* __restrict__ cval,
                                                       const typename Traits<CPLX>::S* __restrict__ part,
                                                       typename Traits<CPLX>::S* __restrict__ out) {
  using T = Traits<CPLX>;
  using S = typename T::S;
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  S lin = T::zero();
  if constexpr (MODEL == MODEL_RBM) {
    const uint8_t* xr = x + r * n_vis;
    for (int i = 0; i < n_vis; ++i)
      if (xr[i]) lin = T::add(lin, avec[i]);
  } else {
    if constexpr (CPLX) lin = make_double2(*cval, 0.0); else lin = *cval;
  }
  S h = T::zero();
  for (int jt = 0; jt < jt_count; ++jt) h = T::add(h, part[(int64_t)jt * n_rows + r]);
  out[r] = T::add(lin, h);
}

// Row lookup of partner configurations among the batch's sorted distinct
// configurations (binary search): out[q] = index of queries[q] in keys, or -1.
// In exact mode every partner lies in the batch, so the partner rows are the
// batch's own O rows and no partner O is built or stored.
__global__ void k_sorted_lookup(const uint64_t* __restrict__ keys, int64_t nk, const uint64_t* __restrict__ q,
                                int64_t nq, int64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t v = q[i];
    int64_t lo = 0, hi = nk;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < v) lo = mid + 1; else hi = mid;
    }
    out[i] = (lo < nk && keys[lo] == v) ? lo : -1;
  }
}

}  // namespace irl
