// O-row producers (K1 RBM f64/c128, K2 MLP f64) and the energy statistics.
//
// Replaces the per-sample `ans.log_derivative` loop inside `build_batch`
// (est:112-126 -> ans:249-290) with two launches over all N_s rows:
//   k_hidden : pre-activation  b + W x_n  for every row (x is 0/1, so this is
//              a gather-sum over the occupied inputs, summed in ascending
//              input order), then tanh (and g = u (1 - t^2) for the MLP).
//   k_orows  : writes the rows  O_n  (row-major, padded ld) with streaming
//              16-B stores and, in the same pass, accumulates the column
//              statistics  sum w conj(O)  and  sum c conj(O)  that give
//              Obar (est:167) and the gradient F (est:156-163).
//
// Parameter layout:
//   RBM : [a (n), b (h), W (h x n) row-major, index j*n + i]
//   MLP : [W (h x n_in) row-major, b (h), u (h), c (1)]   (mirrors _Weights, ans:67-83)
#pragma once
#include "common.cuh"

namespace irl {

enum { MODEL_RBM = 0, MODEL_MLP = 1 };

// complex tanh: (sinh 2a + i sin 2b) / (cosh 2a + cos 2b)
__device__ __forceinline__ double2 ctanh(double2 z) {
  const double d = cosh(2.0 * z.x) + cos(2.0 * z.y);
  return make_double2(sinh(2.0 * z.x) / d, sin(2.0 * z.y) / d);
}

// pre[n][j] = b_j + sum_{i : x[n][i] = 1} W[j][i]  ->  T = tanh(pre), G = u (1 - T^2)
template <bool CPLX, int MODEL>
__global__ void __launch_bounds__(256) k_hidden(const uint8_t* __restrict__ x, int64_t n_rows, int n_vis, int hidden,
                                                const typename Traits<CPLX>::S* __restrict__ Wm,
                                                const typename Traits<CPLX>::S* __restrict__ bvec,
                                                const double* __restrict__ uvec, typename Traits<CPLX>::S* Tout,
                                                double* Gout) {
  using S = typename Traits<CPLX>::S;
  extern __shared__ __align__(16) unsigned char smem_h[];
  S* Wt = reinterpret_cast<S*>(smem_h);  // [n_vis][32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j0 = blockIdx.y * 32;
  const int j = j0 + lane;
  const bool jok = j < hidden;
  for (int e = threadIdx.x; e < n_vis * 32; e += blockDim.x) {
    const int i = e / 32, jj = e % 32;
    S val;
    if constexpr (CPLX) val = make_double2(0.0, 0.0); else val = 0.0;
    if (j0 + jj < hidden) val = Wm[(int64_t)(j0 + jj) * n_vis + i];
    Wt[i * 32 + jj] = val;
  }
  __syncthreads();
  S bj;
  if constexpr (CPLX) bj = make_double2(0.0, 0.0); else bj = 0.0;
  double uj = 0.0;
  if (jok) {
    bj = bvec[j];
    if (MODEL == MODEL_MLP) uj = uvec[j];
  }
  const int64_t rows_per_blk = (n_rows + gridDim.x - 1) / gridDim.x;
  const int64_t r_lo = blockIdx.x * rows_per_blk;
  const int64_t r_hi = min(n_rows, r_lo + rows_per_blk);
  for (int64_t n = r_lo + warp; n < r_hi; n += 8) {
    S acc = bj;
    const uint8_t* xr = x + n * n_vis;
    for (int i0 = 0; i0 < n_vis; i0 += 32) {
      const bool on = (i0 + lane < n_vis) && xr[i0 + lane] != 0;
      uint32_t bits = __ballot_sync(0xffffffffu, on);
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        const S wv = Wt[(i0 + b) * 32 + lane];
        if constexpr (CPLX) {
          acc.x += wv.x;
          acc.y += wv.y;
        } else {
          acc += wv;
        }
      }
    }
    if (jok) {
      if constexpr (CPLX) {
        Tout[n * hidden + j] = ctanh(acc);
      } else {
        const double t = tanh(acc);
        Tout[n * hidden + j] = t;
        if (MODEL == MODEL_MLP) Gout[n * hidden + j] = uj * (1.0 - t * t);
      }
    }
  }
}

struct ORowArgs {
  const uint8_t* x;
  int64_t n_rows;
  int n_vis;
  int hidden;
  int64_t p;  // true parameter count
  const void* T;   // S[N][hidden]
  const double* G; // MLP only
  double2* O;
  int64_t ld_u;
  const double* w;
  const void* coeff;  // S[N] : w (e - E)
  double2* part0;     // [nb][ld_u]  sum w conj(O)
  double2* part1;     // [nb][ld_u]  sum c conj(O)
  int W, C, nb;
};

// Per-row factor table (S-typed, in shared memory):
//   [0] = 0, [1] = 1, [2, 2+h) = t_n, [2+h, 2+2h) = g_n (MLP), then x_n (0/1).
// Every element of O_n is tab[ia] * tab[ib] with (ia, ib) fixed per column:
//   RBM  x_i -> (x_i, 1)   t_j -> (t_j, 1)   t_j x_i -> (t_j, x_i)
//   MLP  g_j x_k -> (g_j, x_k)   g_j -> (g_j, 1)   t_j -> (t_j, 1)   1 -> (1, 1)
//   padding -> (0, 1)
// so the row writer is one multiply per element, no per-element branching.
template <int MODEL>
__host__ __device__ __forceinline__ int orow_tab_len(int n, int h) {
  return 2 + h * (MODEL == MODEL_MLP ? 2 : 1) + n;
}

template <int MODEL>
__device__ __forceinline__ uint32_t elem_pair(int64_t p, int n, int h, int64_t P) {
  const int OT = 2, OG = 2 + h, OX = 2 + h * (MODEL == MODEL_MLP ? 2 : 1);
  uint32_t ia = 0, ib = 1;
  if (p < P) {
    if constexpr (MODEL == MODEL_RBM) {
      if (p < n) {
        ia = OX + (uint32_t)p;
      } else if (p < n + h) {
        ia = OT + (uint32_t)(p - n);
      } else {
        const int64_t q = p - n - h;
        ia = OT + (uint32_t)(q / n);
        ib = OX + (uint32_t)(q % n);
      }
    } else {
      const int64_t hn = (int64_t)h * n;
      if (p < hn) {
        ia = OG + (uint32_t)(p / n);
        ib = OX + (uint32_t)(p % n);
      } else if (p < hn + h) {
        ia = OG + (uint32_t)(p - hn);
      } else if (p < hn + 2 * h) {
        ia = OT + (uint32_t)(p - hn - h);
      } else {
        ia = 1;
      }
    }
  }
  return (ia << 16) | ib;
}

// stage the factor table of row n into tab (cp.async for t/g, direct for x)
template <bool CPLX, int MODEL>
__device__ __forceinline__ void orow_stage(const ORowArgs& a, int64_t n, typename Traits<CPLX>::S* tab, int tid,
                                           int nthreads) {
  using S = typename Traits<CPLX>::S;
  const int h = a.hidden, nv = a.n_vis;
  const int OX = 2 + h * (MODEL == MODEL_MLP ? 2 : 1);
  const S* trow = reinterpret_cast<const S*>(a.T) + (size_t)n * h;
  if (CPLX || (h & 1) == 0) {  // rows 16-B aligned: async copy
    const int tchunks = (int)((size_t)h * sizeof(S) / 16);
    for (int c = tid; c < tchunks; c += nthreads) {
      const uint32_t d = smem_addr(reinterpret_cast<char*>(tab + 2) + 16 * c);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(reinterpret_cast<const char*>(trow) + 16 * c)
                   : "memory");
    }
    if constexpr (MODEL == MODEL_MLP) {
      const char* grow = reinterpret_cast<const char*>(a.G + (size_t)n * h);
      for (int c = tid; c < h / 2; c += nthreads) {
        const uint32_t d = smem_addr(reinterpret_cast<char*>(tab + 2 + h) + 16 * c);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(grow + 16 * c) : "memory");
      }
    }
  } else {  // odd hidden width (real): plain loads
    for (int j = tid; j < h; j += nthreads) tab[2 + j] = trow[j];
    if constexpr (MODEL == MODEL_MLP)
      for (int j = tid; j < h; j += nthreads) tab[2 + h + j] = a.G[(size_t)n * h + j];
  }
  for (int i = tid; i < nv; i += nthreads) {
    const double xv = a.x[n * nv + i] ? 1.0 : 0.0;
    if constexpr (CPLX) tab[OX + i] = make_double2(xv, 0.0); else tab[OX + i] = xv;
  }
}

// STATS: accumulate the column statistics in the writer (complex RBM); real
// models get them from the DMMA GEMMs of otf.cuh instead (lighter writer).
template <bool CPLX, int MODEL, int PPT, bool STATS>
__global__ void __launch_bounds__(512) k_orows(const ORowArgs a, int R) {
  using T = Traits<CPLX>;
  using S = typename T::S;
  extern __shared__ __align__(16) unsigned char smem_r[];
  const int NT = blockDim.x;
  const int tid = threadIdx.x;
  const int rank = blockIdx.x % a.C, blk = blockIdx.x / a.C;
  const int64_t lo = (a.n_rows * blk) / a.nb, hi = (a.n_rows * (blk + 1)) / a.nb;
  const int64_t col0 = (a.ld_u * rank) / a.C;  // uneven split: any tile count
  const int W = (int)((a.ld_u * (rank + 1)) / a.C - col0);
  constexpr int E = Traits<CPLX>::kElemsPerUnit;
  const int TL = (orow_tab_len<MODEL>(a.n_vis, a.hidden) + 1) & ~1;
  S* tabs = reinterpret_cast<S*>(smem_r);  // [2][R][TL] factor tables, R rows per group

  // smem byte offsets of the two factors of each element (relative to the row table)
  uint32_t pr[PPT][E];
  double2 acc0[PPT], acc1[PPT];
  const int kval = (W > tid) ? min(PPT, (W - tid + NT - 1) / NT) : 0;
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int idx = tid + k * NT;
    const int64_t u = col0 + idx;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t q = (idx < W) ? elem_pair<MODEL>(u * E + e, a.n_vis, a.hidden, a.p) : 1u;
      pr[k][e] = (((q >> 16) * (uint32_t)sizeof(S)) << 16) | ((q & 0xffffu) * (uint32_t)sizeof(S));
    }
    acc0[k] = make_double2(0.0, 0.0);
    acc1[k] = make_double2(0.0, 0.0);
  }
  for (int e = tid; e < 2 * R; e += NT) {
    if constexpr (CPLX) {
      tabs[e * TL] = make_double2(0.0, 0.0);
      tabs[e * TL + 1] = make_double2(1.0, 0.0);
    } else {
      tabs[e * TL] = 0.0;
      tabs[e * TL + 1] = 1.0;
    }
  }
  const S* cf = reinterpret_cast<const S*>(a.coeff);
  const int G = (int)((hi - lo + R - 1) / R);
  auto stage_group = [&](int g) {
    const int64_t n0 = lo + (int64_t)g * R;
    const int rows = (int)min((int64_t)R, hi - n0);
    S* base = tabs + (size_t)(g & 1) * R * TL;
    for (int r = 0; r < rows; ++r) orow_stage<CPLX, MODEL>(a, n0 + r, base + (size_t)r * TL, tid, NT);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (G > 0) stage_group(0);
  for (int g = 0; g < G; ++g) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // group g staged; every thread is done with group g-1's buffer
    if (g + 1 < G) stage_group(g + 1);
    const int64_t n0 = lo + (int64_t)g * R;
    const int rows = (int)min((int64_t)R, hi - n0);
    const S* base = tabs + (size_t)(g & 1) * R * TL;
    double2* orow = a.O + n0 * a.ld_u + col0 + tid;
    const char* tbase = reinterpret_cast<const char*>(base);
    for (int r = 0; r < rows; ++r, orow += a.ld_u, tbase += (size_t)TL * sizeof(S)) {
      const int64_t n = n0 + r;
      double wn = 0.0;
      S cn = T::zero();
      if constexpr (STATS) {
        wn = __ldg(a.w + n);
        cn = cf[n];
      }
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        if (k < kval) {
          double2 u;
          if constexpr (CPLX) {
            const S fa = *reinterpret_cast<const S*>(tbase + (pr[k][0] >> 16));
            const S fb = *reinterpret_cast<const S*>(tbase + (pr[k][0] & 0xffffu));
            u = T::mul(fa, fb);
            if constexpr (STATS) {
              acc0[k].x = fma(wn, u.x, acc0[k].x);
              acc0[k].y = fma(-wn, u.y, acc0[k].y);
              T::axpy(acc1[k], u, cn);
            }
          } else {
            u.x = *reinterpret_cast<const double*>(tbase + (pr[k][0] >> 16)) *
                  *reinterpret_cast<const double*>(tbase + (pr[k][0] & 0xffffu));
            u.y = *reinterpret_cast<const double*>(tbase + (pr[k][1] >> 16)) *
                  *reinterpret_cast<const double*>(tbase + (pr[k][1] & 0xffffu));
            if constexpr (STATS) {
              acc0[k].x = fma(wn, u.x, acc0[k].x);
              acc0[k].y = fma(wn, u.y, acc0[k].y);
              acc1[k].x = fma(cn, u.x, acc1[k].x);
              acc1[k].y = fma(cn, u.y, acc1[k].y);
            }
          }
          st_stream(orow + k * NT, u);
        }
      }
    }
  }
  if constexpr (STATS) {
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int idx = tid + k * NT;
      if (idx < W) {
        a.part0[(int64_t)blk * a.ld_u + col0 + idx] = acc0[k];
        a.part1[(int64_t)blk * a.ld_u + col0 + idx] = acc1[k];
      }
    }
  }
}

// Energy statistics (est:146-153) and the H_eff coefficient c_n = w_n (e_n - E)
// (est:166-168, est:186).  One CTA, fixed-order tree: deterministic.
//   stats[0] = E = Re sum w e ; stats[1] = Im sum w e ; stats[2] = sum w |e - E|^2
// hermitian (complex only): c_n = w_n Re(e_n - E)
template <bool CPLX>
__global__ void __launch_bounds__(1024) k_energy(const double* __restrict__ w, const void* e_, int64_t n,
                                                 int hermitian, double* stats, void* coeff_) {
  using T = Traits<CPLX>;
  using S = typename T::S;
  const S* e = reinterpret_cast<const S*>(e_);
  S* coeff = reinterpret_cast<S*>(coeff_);
  __shared__ S sh[32];
  __shared__ double shd[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  S acc = T::zero();
  for (int64_t i = tid; i < n; i += blockDim.x) {
    const S ei = e[i];
    if constexpr (CPLX) {
      acc.x = fma(w[i], ei.x, acc.x);
      acc.y = fma(w[i], ei.y, acc.y);
    } else {
      acc = fma(w[i], ei, acc);
    }
  }
  acc = warp_sum<CPLX>(acc);
  if (lane == 0) sh[warp] = acc;
  __syncthreads();
  S tot = T::zero();
  for (int k = 0; k < nw; ++k) tot = T::add(tot, sh[k]);
  double E, Ei;
  if constexpr (CPLX) {
    E = tot.x;
    Ei = tot.y;
  } else {
    E = tot;
    Ei = 0.0;
  }
  double v = 0.0;
  for (int64_t i = tid; i < n; i += blockDim.x) {
    const S ei = e[i];
    if constexpr (CPLX) {
      const double dr = ei.x - E, di = ei.y;
      v = fma(w[i], dr * dr + di * di, v);
      coeff[i] = hermitian ? make_double2(w[i] * dr, 0.0) : make_double2(w[i] * dr, w[i] * di);
    } else {
      const double d = ei - E;
      v = fma(w[i], d * d, v);
      coeff[i] = w[i] * d;
    }
  }
  v = warp_sum<false>(v);
  if (lane == 0) shd[warp] = v;
  __syncthreads();
  if (tid == 0) {
    double var = 0.0;
    for (int k = 0; k < nw; ++k) var += shd[k];
    stats[0] = E;
    stats[1] = Ei;
    stats[2] = var;
  }
}

}  // namespace irl
