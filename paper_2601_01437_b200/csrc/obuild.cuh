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

enum { MODEL_RBM = 0, MODEL_MLP = 1, MODEL_NONE = 2 };  // NONE: Hamiltonian only (ratio 1)

constexpr int ORW_NBUF = 3;   // staging buffers of the O-row writer
constexpr int ORW_RMAX = 32;  // rows per staging group at most

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
  const void* xd;     // S[N][xrow]: the inputs as table entries (0/1), or null
  int xrow;
};

// x (N x n uint8) -> S[N][xrow] 0/1 table entries (zero padded), for the
// asynchronous row staging of the O-row writer
template <bool CPLX>
__global__ void k_x_expand(const uint8_t* __restrict__ x, int64_t n_rows, int n_vis, int xrow,
                           typename Traits<CPLX>::S* __restrict__ xd) {
  const int64_t total = n_rows * xrow;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / xrow;
    const int i = (int)(e % xrow);
    const double v = (i < n_vis && x[r * n_vis + i]) ? 1.0 : 0.0;
    if constexpr (CPLX) xd[e] = make_double2(v, 0.0); else xd[e] = v;
  }
}

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

// Compact per-tile factor table.  A column tile only touches a contiguous
// range of hidden units, so each CTA stages just that range:
//   [0] = 0, [1] = 1, [2, 2+tl) = t[t_lo ..], [2+tl, 2+tl+gl) = g[g_lo ..], then x.
struct TabRange {
  int t_lo, tl, tn;  // first unit, table slots (even), units to stage (<= tl, inside [0, h))
  int g_lo, gl, gn;
  int len;           // table entries, even
};

template <int MODEL>
__device__ __forceinline__ TabRange tab_range(int64_t e0, int64_t e1, int n, int h, int64_t P, bool even_align) {
  // element range [e0, e1) of this tile (clipped to P) -> hidden-unit hulls
  e1 = min(e1, P);
  int tlo = h, thi = -1, glo = h, ghi = -1;
  auto addt = [&](int64_t a, int64_t b) { if (a <= b) { tlo = min(tlo, (int)a); thi = max(thi, (int)b); } };
  auto addg = [&](int64_t a, int64_t b) { if (a <= b) { glo = min(glo, (int)a); ghi = max(ghi, (int)b); } };
  if (e0 < e1) {
    if constexpr (MODEL == MODEL_RBM) {
      const int64_t bb = n, wb = (int64_t)n + h;
      addt(max(e0, bb) - bb, min(e1, wb) - 1 - bb);                               // b block: t_j
      if (e1 > wb) addt((max(e0, wb) - wb) / n, (e1 - 1 - wb) / n);              // W block: t_j x_i
    } else {
      const int64_t hn = (int64_t)h * n;
      if (e0 < hn) addg(e0 / n, (min(e1, hn) - 1) / n);                          // W block: g_j x_k
      addg(max(e0, hn) - hn, min(e1, hn + h) - 1 - hn);                          // b block: g_j
      addt(max(e0, hn + h) - hn - h, min(e1, hn + 2 * h) - 1 - hn - h);          // u block: t_j
    }
  }
  TabRange r;
  if (thi < tlo) { tlo = 0; thi = -1; }
  if (ghi < glo) { glo = 0; ghi = -1; }
  if (even_align) {  // 16-byte cp.async chunks of a real (8-byte) row
    tlo &= ~1;
    thi = (thi < 0) ? -1 : min(h - 1, thi | 1);
    glo &= ~1;
    ghi = (ghi < 0) ? -1 : min(h - 1, ghi | 1);
  }
  r.t_lo = tlo;
  r.tn = thi - tlo + 1;
  r.tl = (r.tn + 1) & ~1;  // even slot counts keep the x block 16-byte aligned
  r.g_lo = glo;
  r.gn = ghi - glo + 1;
  r.gl = (r.gn + 1) & ~1;
  r.len = (2 + r.tl + r.gl + n + 1) & ~1;
  return r;
}

// full-layout factor index (elem_pair) -> compact index
__device__ __forceinline__ uint32_t tab_remap(uint32_t ia, const TabRange& r, int h, int mlp) {
  const uint32_t OT = 2, OG = 2 + h, OX = 2 + h * (mlp ? 2 : 1);
  if (ia < OT) return ia;
  if (ia < OT + h) return 2 + (ia - OT - r.t_lo);
  if (mlp && ia < OG + h) return 2 + r.tl + (ia - OG - r.g_lo);
  return 2 + r.tl + r.gl + (ia - OX);
}

// stage the compact factor table of row n into tab (cp.async for t/g, direct for x)
template <bool CPLX, int MODEL>
__device__ __forceinline__ void orow_stage(const ORowArgs& a, int64_t n, const TabRange& rg,
                                           typename Traits<CPLX>::S* tab, int tid, int nthreads) {
  using S = typename Traits<CPLX>::S;
  const int h = a.hidden, nv = a.n_vis;
  const int OX = 2 + rg.tl + rg.gl;
  const S* trow = reinterpret_cast<const S*>(a.T) + (size_t)n * h;
  if (CPLX || (h & 1) == 0) {  // rows 16-B aligned: async copy
    const int tchunks = (int)((size_t)rg.tn * sizeof(S) / 16);
    const char* tsrc = reinterpret_cast<const char*>(trow + rg.t_lo);
    for (int c = tid; c < tchunks; c += nthreads) {
      const uint32_t d = smem_addr(reinterpret_cast<char*>(tab + 2) + 16 * c);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(tsrc + 16 * c) : "memory");
    }
    if constexpr (MODEL == MODEL_MLP) {
      const char* gsrc = reinterpret_cast<const char*>(a.G + (size_t)n * h + rg.g_lo);
      for (int c = tid; c < rg.gn / 2; c += nthreads) {
        const uint32_t d = smem_addr(reinterpret_cast<char*>(tab + 2 + rg.tl) + 16 * c);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc + 16 * c) : "memory");
      }
    }
  } else {  // odd hidden width (real): plain loads
    for (int j = tid; j < rg.tn; j += nthreads) tab[2 + j] = trow[rg.t_lo + j];
    if constexpr (MODEL == MODEL_MLP)
      for (int j = tid; j < rg.gn; j += nthreads) tab[2 + rg.tl + j] = a.G[(size_t)n * h + rg.g_lo + j];
  }
  if (a.xd) {  // expanded inputs: 16-byte asynchronous chunks
    const int xchunks = (int)((size_t)a.xrow * sizeof(S) / 16);
    const char* xsrc = reinterpret_cast<const char*>(reinterpret_cast<const S*>(a.xd) + (size_t)n * a.xrow);
    for (int c = tid; c < xchunks; c += nthreads) {
      const uint32_t d = smem_addr(reinterpret_cast<char*>(tab + OX) + 16 * c);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(xsrc + 16 * c) : "memory");
    }
    return;
  }
  for (int i = tid; i < nv; i += nthreads) {
    const double xv = a.x[n * nv + i] ? 1.0 : 0.0;
    if constexpr (CPLX) tab[OX + i] = make_double2(xv, 0.0); else tab[OX + i] = xv;
  }
}

// STATS: accumulate the column statistics in the writer (complex RBM); real
// models get them from the DMMA GEMMs of otf.cuh instead (lighter writer).
template <bool CPLX, int MODEL, int PPT, bool STATS>
__global__ void __launch_bounds__(512) k_orows(const ORowArgs a, int buf_bytes) {
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
  const TabRange rg = tab_range<MODEL>(col0 * E, (col0 + W) * E, a.n_vis, a.hidden, a.p, !CPLX);
  const int TL = rg.len;
  // rows per staging group: as many compact tables as one buffer holds (<= ORW_RMAX)
  const int R = max(1, min(ORW_RMAX, buf_bytes / (TL * (int)sizeof(S))));
  // 3 staging buffers of R rows: factor tables, then the rows' w_n and c_n
  constexpr int NBUF = ORW_NBUF;
  S* tabs = reinterpret_cast<S*>(smem_r);                                   // [NBUF][R][TL]
  double* wsm = reinterpret_cast<double*>(smem_r + (size_t)NBUF * buf_bytes); // [NBUF][RMAX]
  S* csm = reinterpret_cast<S*>(wsm + NBUF * ORW_RMAX);                       // [NBUF][RMAX]

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
      const uint32_t ia = tab_remap(q >> 16, rg, a.hidden, MODEL == MODEL_MLP);
      const uint32_t ib = tab_remap(q & 0xffffu, rg, a.hidden, MODEL == MODEL_MLP);
      pr[k][e] = ((ia * (uint32_t)sizeof(S)) << 16) | (ib * (uint32_t)sizeof(S));
    }
    acc0[k] = make_double2(0.0, 0.0);
    acc1[k] = make_double2(0.0, 0.0);
  }
  for (int e = tid; e < NBUF * R; e += NT) {
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
    const int b = g % NBUF;
    S* base = tabs + (size_t)b * R * TL;
    for (int r = 0; r < rows; ++r) orow_stage<CPLX, MODEL>(a, n0 + r, rg, base + (size_t)r * TL, tid, NT);
    if constexpr (STATS) {
      for (int r = tid; r < rows; r += NT) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(wsm + b * ORW_RMAX + r)),
                     "l"(a.w + n0 + r)
                     : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_addr(csm + b * ORW_RMAX + r)),
                     "l"(cf + n0 + r), "n"(sizeof(S))
                     : "memory");
      }
    }
  };
  // two groups in flight: group g is waited for at iteration g, with g + 1 still pending
  for (int g = 0; g < NBUF - 1; ++g) {
    if (g < G) stage_group(g);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int g = 0; g < G; ++g) {
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();  // group g staged; every thread is done with group g-1's buffer
    if (g + NBUF - 1 < G) stage_group(g + NBUF - 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const int64_t n0 = lo + (int64_t)g * R;
    const int rows = (int)min((int64_t)R, hi - n0);
    const int b = g % NBUF;
    const S* base = tabs + (size_t)b * R * TL;
    double2* orow = a.O + n0 * a.ld_u + col0 + tid;
    const char* tbase = reinterpret_cast<const char*>(base);
    for (int r = 0; r < rows; ++r, orow += a.ld_u, tbase += (size_t)TL * sizeof(S)) {
      double wn = 0.0;
      S cn = T::zero();
      if constexpr (STATS) {
        wn = wsm[b * ORW_RMAX + r];
        cn = csm[b * ORW_RMAX + r];
      }
      // every unit computed (invalid ones read the table's constant slots): only
      // the store is predicated, so the table loads of all PPT units issue together
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
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
        if (k < kval) st_stream(orow + k * NT, u);
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

namespace irl {

// Row-sweeping O writer (stats come from the DMMA GEMMs, so no column
// ownership is needed): CTA c writes whole rows c, c + grid, ... front to
// back with streaming 16-B stores -- the store pattern that sustains the
// HBM write rate on very wide rows (1.67 MB at cfg5), where column tiles of
// many CTAs interleaving inside one row do not.  The outer-product block
// (t_j x_i for the RBM, g_j x_k for the MLP) is written j-segment by
// j-segment: a lane owns fixed input positions (units) of the segment, so its
// x values are loaded once per row and every store is factor_j * x.
//   real RBM  [x (n), t (h), W (h x n)]     needs n, h even (unit-aligned blocks)
//   c128 RBM  same, one complex element per unit
//   MLP       [W (h x n), g (h), t (h), 1]  needs n even
constexpr int SWEEP_NT = 512;
constexpr int SWEEP_UQ = 4;  // units per lane per segment: n <= 128 (complex) / 256 (real)

template <bool CPLX, int MODEL>
__global__ void __launch_bounds__(SWEEP_NT, 2) k_orows_sweep(const uint8_t* __restrict__ x, int64_t n_rows, int n,
                                                            int h, const void* __restrict__ Tv,
                                                            const double* __restrict__ G, double2* __restrict__ O,
                                                            int64_t ld_u, int dbuf) {
  using S = typename Traits<CPLX>::S;
  extern __shared__ __align__(16) unsigned char smem_sw[];
  S* fs = reinterpret_cast<S*>(smem_sw);  // [2][h] factor rows (t or g), double-buffered
  const S* T = reinterpret_cast<const S*>(Tv);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = SWEEP_NT / 32;
  const int upj = CPLX ? n : n / 2;  // units per j segment
  const int JW = upj >= 32 ? 1 : 32 / upj;
  const int jo = upj >= 32 ? 0 : lane / upj;
  const int u0 = upj >= 32 ? lane : lane % upj;
  const bool active = jo < JW;
  const int64_t hn = (int64_t)h * n;
  const int64_t P = MODEL == MODEL_RBM ? (int64_t)n + h + hn : hn + 2 * (int64_t)h + 1;
  const int64_t wb = MODEL == MODEL_MLP ? 0 : (CPLX ? (int64_t)n + h : ((int64_t)n + h) / 2);  // W block, units
  const int64_t we = wb + (int64_t)h * upj;
  // the factor row (t or g) of the next row is copied into the other half of a
  // double buffer with cp.async while this row is written (h * sizeof(S) is a
  // multiple of 16 bytes: h even for real rows)
  const S* F = MODEL == MODEL_MLP ? reinterpret_cast<const S*>(G) : T;
  const int fchunks = (int)((size_t)h * sizeof(S) / 16);
  auto prefetch = [&](int64_t row, S* dst) {
    if (row < n_rows) {
      const char* src = reinterpret_cast<const char*>(F + row * h);
      for (int q = tid; q < fchunks; q += SWEEP_NT)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(reinterpret_cast<char*>(dst) + 16 * q)),
                     "l"(src + 16 * q)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // dbuf = 0 (long rows, whose writes dwarf the factor load): one buffer, loaded
  // in place at the top of every row
  int cur = 0;
  if (dbuf) prefetch(blockIdx.x, fs);
  for (int64_t r = blockIdx.x; r < n_rows; r += gridDim.x, cur ^= dbuf) {
    const uint8_t* xr = x + r * n;
    if (!dbuf) {
      __syncthreads();  // previous row's factors consumed
      prefetch(r, fs);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // this row's factors landed; the other buffer's previous row is consumed
    if (dbuf) prefetch(r + gridDim.x, fs + (cur ^ 1) * h);
    const S* fr = fs + cur * h;
    // this lane's x values (its units of every segment)
    double xa[SWEEP_UQ], xb[SWEEP_UQ];
#pragma unroll
    for (int q = 0; q < SWEEP_UQ; ++q) {
      const int u = u0 + 32 * q;
      xa[q] = xb[q] = 0.0;
      if (u < upj) {
        if constexpr (CPLX) {
          xa[q] = xr[u] ? 1.0 : 0.0;
        } else {
          xa[q] = xr[2 * u] ? 1.0 : 0.0;
          xb[q] = xr[2 * u + 1] ? 1.0 : 0.0;
        }
      }
    }
    double2* orow = O + r * ld_u;
    if (active) {
      for (int j = warp * JW + jo; j < h; j += NW * JW) {
        const S f = fr[j];
        double2* seg = orow + wb + (int64_t)j * upj;
#pragma unroll
        for (int q = 0; q < SWEEP_UQ; ++q) {
          const int u = u0 + 32 * q;
          if (u < upj) {
            if constexpr (CPLX) st_stream(seg + u, make_double2(f.x * xa[q], f.y * xa[q]));
            else st_stream(seg + u, make_double2(f * xa[q], f * xb[q]));
          }
        }
      }
    }
    // the short blocks and the padding, element by element
    auto elem = [&](int64_t e) -> S {
      S v = Traits<CPLX>::zero();
      if (e >= P) return v;
      if constexpr (MODEL == MODEL_RBM) {
        if (e < n) {
          if constexpr (CPLX) v.x = xr[e] ? 1.0 : 0.0; else v = xr[e] ? 1.0 : 0.0;
        } else if (e < (int64_t)n + h) {
          v = fr[e - n];
        }
      } else {
        if (e >= hn && e < hn + h) {
          v = G[r * h + (e - hn)];
        } else if (e >= hn + h && e < hn + 2 * h) {
          if constexpr (!CPLX) v = reinterpret_cast<const double*>(Tv)[r * h + (e - hn - h)];
        } else if (e == hn + 2 * h) {
          if constexpr (!CPLX) v = 1.0;
        }
      }
      return v;
    };
    for (int64_t u = tid; u < ld_u - (we - wb); u += SWEEP_NT) {
      const int64_t uu = u < wb ? u : u + (we - wb);  // skip the W block
      if constexpr (CPLX) {
        st_stream(orow + uu, elem(uu));
      } else {
        const double lo = elem(2 * uu), hi = elem(2 * uu + 1);
        st_stream(orow + uu, make_double2(lo, hi));
      }
    }
  }
}

}  // namespace irl
