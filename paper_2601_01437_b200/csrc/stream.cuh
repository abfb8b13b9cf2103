// Streaming kernel family over the stored log-derivative matrix O.
//
// One templated kernel, four modes, all streaming O row-slices through a
// shared-memory ring filled by the TMA bulk-copy engine (cp.async.bulk ->
// mbarrier complete_tx) from a dedicated producer warp:
//
//   MODE_FUSED  single-pass centred product (K5 in SURVEY §2):
//                 t_n = O_n . v ;  y_n = c_n (t_n - s) , s = Obar . v
//                 acc += conj(O_n) y_n           (same smem tile, read once)
//               Columns are split over a thread-block CLUSTER of C CTAs; the
//               per-row partial dots are exchanged CTA-to-CTA through DSMEM
//               with st.async + mbarrier complete_tx.  Replaces est:184-186
//               (`_centered` copy + two GEMVs) with one HBM pass.
//   MODE_DOT    two-pass pass 1 (K3): partial t per column tile -> global.
//   MODE_ACC    two-pass pass 2 (K4): y from the tile partials, acc.
//   MODE_STATS  column statistics (A4/A5): acc0 = sum w conj(O),
//               acc1 = sum c conj(O)   -> Obar (est:167), F/2 (est:162).
//
// Every reduction has a fixed order (warp butterfly, warps in index order,
// cluster ranks in order, row blocks in order): results are bit-identical
// run to run, no float atomics anywhere.
#pragma once
#include "common.cuh"

namespace irl {

enum StreamMode { MODE_FUSED = 0, MODE_DOT = 1, MODE_ACC = 2, MODE_STATS = 3 };

struct StreamArgs {
  const double2* O;  // units; row stride ld_u
  int64_t n_rows;
  int64_t ld_u;
  int W;       // units per column slice
  int C;       // column slices (cluster size in MODE_FUSED)
  int nb;      // row blocks (clusters in MODE_FUSED)
  int stages;  // ring depth
  // input vectors (unit-indexed).  real: v_re is the f64 array viewed as units;
  // complex: planar re/im (im may be null = 0).
  const double* v_re;
  const double* v_im;
  const double* hf_re;  // bordered half gradient (null = not bordered)
  const double* hf_im;
  const double2* obar;  // centring vector (units); null = uncentred
  const void* coeff0;   // FUSED/ACC: S[N] ; STATS: double[N] (weights)
  const void* coeff1;   // STATS: S[N]
  // outputs / workspace
  double2* part0;  // [nb][ld_u]
  double2* part1;  // [nb][ld_u]   (STATS)
  void* ysum;      // S[nb]
  void* tpart;     // S[C][n_rows]  (DOT -> ACC)
  void* spart;     // S[C]          (DOT -> ACC; FUSED writes [0])
  double* gpart;   // double[C]     (DOT; FUSED writes [0])
};

template <bool CPLX>
__device__ __forceinline__ double2 load_vec_unit(const double* re, const double* im, int64_t u) {
  if constexpr (!CPLX) {
    return reinterpret_cast<const double2*>(re)[u];
  } else {
    return make_double2(re[u], im ? im[u] : 0.0);
  }
}

__host__ __device__ constexpr int stream_max_nt(int ppt) {
  return ppt <= 2 ? 992 : ppt <= 4 ? 768 : ppt <= 8 ? 480 : 320;
}

template <bool CPLX, int PPT, int R, int MODE>
__global__ void __launch_bounds__(stream_max_nt(PPT) + 32, 1) k_stream(const StreamArgs a) {
  using T = Traits<CPLX>;
  using S = typename T::S;
  extern __shared__ __align__(128) unsigned char smem[];

  const int NT = blockDim.x - 32;  // consumer threads; last warp = producer
  const int NW = NT >> 5;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int W = a.W, C = a.C, NS = a.stages;
  const int RP = NW + 1;
  const int64_t N = a.n_rows;

  double2* ring = reinterpret_cast<double2*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NS * R * W * 16);
  uint64_t* empty = full + NS;
  uint64_t* xbar = empty + NS;                  // [2]
  S* red = reinterpret_cast<S*>(xbar + 2);      // [2][R][RP]
  S* xch = red + 2 * R * RP;                    // [2][C][R]
  S* scr_s = xch + 2 * C * R;                   // [32] block-reduce scratch
  S* pro_s = scr_s + 32;                        // [1] cluster-visible prologue slot
  double* scr_g = reinterpret_cast<double*>(pro_s + 1);  // [32]
  double* pro_g = scr_g + 32;                            // [1]

  const bool clustered = (MODE == MODE_FUSED) && (C > 1);
  int rank, blk;
  if (MODE == MODE_FUSED) {
    rank = clustered ? (int)cluster_rank() : 0;
    blk = blockIdx.x / C;
  } else {
    rank = blockIdx.x % C;
    blk = blockIdx.x / C;
  }
  const int64_t lo = (N * blk) / a.nb, hi = (N * (blk + 1)) / a.nb;
  const int G = (int)((hi - lo + R - 1) / R);
  const int64_t col0 = (int64_t)rank * W;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (clustered) cluster_sync();  // peers' barriers initialised before any st.async

  // ------------------------------------------------------------ producer --
  if (warp == NW) {
    if (clustered) cluster_arrive();  // prologue exchange barrier (no data needed here)
    if (lane == 0) {
      const uint32_t slice_bytes = (uint32_t)W * 16u;
      for (int g = 0; g < G; ++g) {
        const int s = g % NS;
        if (g >= NS) mbar_wait(&empty[s], ((g / NS) - 1) & 1);
        const int64_t r0 = lo + (int64_t)g * R;
        const int rows = (int)min((int64_t)R, hi - r0);
        mbar_arrive_expect_tx(&full[s], slice_bytes * rows);
        double2* dst = ring + (size_t)s * R * W;
        const double2* src = a.O + r0 * a.ld_u + col0;
        for (int r = 0; r < rows; ++r) bulk_g2s(dst + (size_t)r * W, src + r * a.ld_u, slice_bytes, &full[s]);
      }
    }
    __syncwarp();
    if (clustered) {
      cluster_wait();
      cluster_sync();  // final: keep smem alive until every peer is done with it
    }
    return;
  }

  // ----------------------------------------------------------- consumers --
  double2 vreg[PPT];
  double2 acc0[PPT];
  double2 acc1[PPT];
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    vreg[k] = make_double2(0.0, 0.0);
    acc0[k] = make_double2(0.0, 0.0);
    acc1[k] = make_double2(0.0, 0.0);
  }

  S s_val = T::zero();
  if constexpr (MODE == MODE_FUSED || MODE == MODE_DOT) {
    S sp = T::zero();
    double gp = 0.0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int idx = tid + k * NT;
      if (idx < W) {
        const int64_t u = col0 + idx;
        vreg[k] = load_vec_unit<CPLX>(a.v_re, a.v_im, u);
        if (a.obar) T::dot_acc(sp, a.obar[u], vreg[k]);
        if (a.hf_re) {
          const double2 h = load_vec_unit<CPLX>(a.hf_re, a.hf_im, u);
          gp = fma(h.x, vreg[k].x, gp);
          gp = fma(h.y, vreg[k].y, gp);
        }
      }
    }
    sp = warp_sum<CPLX>(sp);
    gp = warp_sum<false>(gp);
    if (lane == 0) {
      scr_s[warp] = sp;
      scr_g[warp] = gp;
    }
    named_bar_sync(1, NT);
    S sc = T::zero();
    double gc = 0.0;
    for (int w = 0; w < NW; ++w) {
      sc = T::add(sc, scr_s[w]);
      gc += scr_g[w];
    }
    if (MODE == MODE_DOT) {
      if (blk == 0 && tid == 0) {
        reinterpret_cast<S*>(a.spart)[rank] = sc;
        a.gpart[rank] = gc;
      }
    } else if (clustered) {
      if (tid == 0) {
        *pro_s = sc;
        *pro_g = gc;
      }
      cluster_arrive();
      cluster_wait();
      const uint32_t as = smem_addr(pro_s), ag = smem_addr(pro_g);
      sc = T::zero();
      gc = 0.0;
      for (int q = 0; q < C; ++q) {
        sc = T::add(sc, ld_cluster(map_to_rank(as, q), (S*)nullptr));
        gc += ld_cluster(map_to_rank(ag, q), (double*)nullptr);
      }
    }
    s_val = sc;
    if (MODE == MODE_FUSED && blockIdx.x == 0 && tid == 0) {
      reinterpret_cast<S*>(a.spart)[0] = sc;
      a.gpart[0] = gc;
    }
  } else if constexpr (MODE == MODE_ACC) {
    for (int c = 0; c < C; ++c) s_val = T::add(s_val, reinterpret_cast<const S*>(a.spart)[c]);
  }

  S ys = T::zero();
  for (int g = 0; g < G; ++g) {
    const int s = g % NS;
    const int64_t r0 = lo + (int64_t)g * R;
    const int rows = (int)min((int64_t)R, hi - r0);

    // per-row scalars, lane r owns row r of the group (prefetched before the wait)
    S cf0 = T::zero();
    S cf1 = T::zero();
    S tin = T::zero();
    if (lane < rows) {
      if constexpr (MODE == MODE_STATS) {
        const double w = reinterpret_cast<const double*>(a.coeff0)[r0 + lane];
        if constexpr (CPLX) cf0 = make_double2(w, 0.0); else cf0 = w;
        cf1 = reinterpret_cast<const S*>(a.coeff1)[r0 + lane];
      } else if constexpr (MODE != MODE_DOT) {
        cf0 = reinterpret_cast<const S*>(a.coeff0)[r0 + lane];
      }
      if constexpr (MODE == MODE_ACC) {
        for (int c = 0; c < C; ++c) tin = T::add(tin, reinterpret_cast<const S*>(a.tpart)[(int64_t)c * N + r0 + lane]);
      }
    }

    mbar_wait(&full[s], (g / NS) & 1);
    const double2* st = ring + (size_t)s * R * W;

    S yv = T::zero();
    if constexpr (MODE == MODE_FUSED || MODE == MODE_DOT) {
      S dp[R];
#pragma unroll
      for (int r = 0; r < R; ++r) dp[r] = T::zero();
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        const int idx = tid + k * NT;
        if (idx < W) {
#pragma unroll
          for (int r = 0; r < R; ++r)
            if (r < rows) T::dot_acc(dp[r], st[(size_t)r * W + idx], vreg[k]);
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) dp[r] = warp_sum<CPLX>(dp[r]);
      S* rb = red + (g & 1) * R * RP;
      if (lane == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) rb[r * RP + warp] = dp[r];
      }
      named_bar_sync(1, NT);
      S t = T::zero();
      if (lane < rows)
        for (int w = 0; w < NW; ++w) t = T::add(t, rb[lane * RP + w]);
      if constexpr (MODE == MODE_DOT) {
        if (warp == 0 && lane < rows) reinterpret_cast<S*>(a.tpart)[(int64_t)rank * N + r0 + lane] = t;
      } else {
        if (clustered) {
          const int b = g & 1;
          if (warp == 0) {
            if (lane == 0) mbar_arrive_expect_tx(&xbar[b], (uint32_t)(C * rows * sizeof(S)));
            if (lane < rows) {
              const uint32_t la = smem_addr(&xch[(b * C + rank) * R + lane]);
              const uint32_t lb = smem_addr(&xbar[b]);
              for (int q = 0; q < C; ++q) st_async(map_to_rank(la, q), t, map_to_rank(lb, q));
            }
          }
          mbar_wait(&xbar[b], (g >> 1) & 1);
          t = T::zero();
          if (lane < rows)
            for (int q = 0; q < C; ++q) t = T::add(t, xch[(b * C + q) * R + lane]);
        }
        if (lane < rows) yv = T::mul(cf0, T::sub(t, s_val));
      }
    } else if constexpr (MODE == MODE_ACC) {
      if (lane < rows) yv = T::mul(cf0, T::sub(tin, s_val));
    } else {
      yv = cf0;
    }

    if constexpr (MODE != MODE_DOT) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r < rows) {
          const S y = T::shfl(yv, r);
          S y1 = T::zero();
          if constexpr (MODE == MODE_STATS) y1 = T::shfl(cf1, r);
          if (MODE != MODE_STATS && tid == 0) ys = T::add(ys, y);
#pragma unroll
          for (int k = 0; k < PPT; ++k) {
            const int idx = tid + k * NT;
            if (idx < W) {
              const double2 u = st[(size_t)r * W + idx];
              T::axpy(acc0[k], u, y);
              if constexpr (MODE == MODE_STATS) T::axpy(acc1[k], u, y1);
            }
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  if constexpr (MODE != MODE_DOT) {
    double2* p0 = a.part0 + (int64_t)blk * a.ld_u + col0;
    double2* p1 = (MODE == MODE_STATS) ? a.part1 + (int64_t)blk * a.ld_u + col0 : nullptr;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int idx = tid + k * NT;
      if (idx < W) {
        p0[idx] = acc0[k];
        if constexpr (MODE == MODE_STATS) p1[idx] = acc1[k];
      }
    }
    if (MODE != MODE_STATS && rank == 0 && tid == 0) reinterpret_cast<S*>(a.ysum)[blk] = ys;
  }
  if (clustered) cluster_sync();
}

// out = sum_b part[b] - conj(obar) * sum_b ysum[b]  (+ u0 * hf)    ; out0 = sum gpart
template <bool CPLX>
__global__ void k_finish_mvp(const double2* __restrict__ part, int nb, int64_t ld_u, const void* ysum,
                             const double2* __restrict__ obar, const double* hf_re, const double* hf_im,
                             const double* u0, double* out_re, double* out_im, const double* gpart, int n_gpart,
                             double* out0) {
  using T = Traits<CPLX>;
  using S = typename T::S;
  S Y = T::zero();
  const S* ys = reinterpret_cast<const S*>(ysum);
  for (int b = 0; b < nb; ++b) Y = T::add(Y, ys[b]);
  const double uu = (hf_re && u0) ? *u0 : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ld_u; i += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int b = 0; b < nb; ++b) {
      const double2 p = part[(int64_t)b * ld_u + i];
      acc.x += p.x;
      acc.y += p.y;
    }
    if (obar) {
      S negY;
      if constexpr (CPLX) negY = make_double2(-Y.x, -Y.y); else negY = -Y;
      T::axpy(acc, obar[i], negY);
    }
    if (hf_re && u0) {
      const double2 h = load_vec_unit<CPLX>(hf_re, hf_im, i);
      acc.x = fma(uu, h.x, acc.x);
      acc.y = fma(uu, h.y, acc.y);
    }
    if constexpr (!CPLX) {
      reinterpret_cast<double2*>(out_re)[i] = acc;
    } else {
      out_re[i] = acc.x;
      if (out_im) out_im[i] = acc.y;
    }
  }
  if (out0 && blockIdx.x == 0 && threadIdx.x == 0) {
    double g = 0.0;
    if (hf_re)
      for (int c = 0; c < n_gpart; ++c) g += gpart[c];
    *out0 = g;
  }
}

// obar = sum_b part0[b] (conjugated back for complex) ; g = sum_b part1[b]
template <bool CPLX>
__global__ void k_finish_stats(const double2* __restrict__ part0, const double2* __restrict__ part1, int nb,
                               int64_t ld_u, double2* obar, double2* g) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ld_u; i += (int64_t)gridDim.x * blockDim.x) {
    double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
    for (int b = 0; b < nb; ++b) {
      const double2 p = part0[(int64_t)b * ld_u + i];
      const double2 q = part1[(int64_t)b * ld_u + i];
      a0.x += p.x;
      a0.y += p.y;
      a1.x += q.x;
      a1.y += q.y;
    }
    if (CPLX) a0.y = -a0.y;
    obar[i] = a0;
    g[i] = a1;
  }
}

}  // namespace irl
