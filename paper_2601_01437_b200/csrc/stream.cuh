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
// The consumer loop is software-pipelined one row group deep: the dot
// product, block reduction and DSMEM send of group g+1 are issued before
// group g's exchange is awaited and accumulated, so the exchange latency
// hides behind the next tile instead of stalling the HBM stream.
//
// Every reduction has a fixed order (warp butterfly, warps in index order,
// cluster ranks in order, row blocks in order): results are bit-identical
// run to run, no float atomics anywhere.
#pragma once
#include "common.cuh"

namespace irl {

enum StreamMode { MODE_FUSED = 0, MODE_DOT = 1, MODE_ACC = 2, MODE_STATS = 3 };

constexpr int kXchSlots = 4;  // DSMEM exchange ring depth (lookahead 1 needs 4, see below)

struct StreamArgs {
  const double2* O;  // units; row stride ld_u
  int64_t n_rows;
  int64_t ld_u;
  int Wmax;    // max units per column slice (ring slot width)
  int C;       // column slices (cluster size in MODE_FUSED)
  int nb;      // row blocks (clusters in MODE_FUSED)
  int stages;  // ring depth
  int dbg;     // reserved (0)
  // input vectors (unit-indexed).  real: v_re is the f64 array viewed as units;
  // complex: planar re/im (im may be null = 0).
  const double* v_re;
  const double* v_im;
  const double* hf_re;  // bordered half gradient (null = not bordered)
  const double* hf_im;
  const double2* obar;  // centring vector (units); null = uncentred
  const void* coeff0;   // FUSED/ACC: S[N] ; STATS: double[N] (weights)
  const void* coeff1;   // STATS: S[N]
  const void* yadd;     // FUSED/ACC: S[N] additive row term, y_n += yadd_n (connected completion); null = none
  // outputs / workspace
  double2* part0;  // [nb][ld_u]
  double2* part1;  // [nb][ld_u]   (STATS)
  void* ysum;      // S[nb]
  void* ysum1;     // S[nb]         (FUSED DUAL: the second product's sum of y)
  size_t vs_off;   // FUSED DUAL: shared-memory offset of the v slice (the second accumulator takes v's registers)
  void* tpart;     // S[C][n_rows]  (DOT -> ACC)
  void* spart;     // S[C]          (DOT -> ACC; FUSED writes [0])
  double* gpart;   // double[C]     (DOT; FUSED writes [0])
};

// Column split: slice r covers units [slice_lo(r), slice_lo(r+1)).  Uneven
// splits let any cluster size tile the row (every unit is 16-B aligned).
__host__ __device__ __forceinline__ int64_t slice_lo(int64_t ld_u, int C, int r) { return (ld_u * r) / C; }

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

// ADD (MODE_FUSED only): the additive row term yadd is compiled in only for the
// connected product, so the plain fused product keeps its exact schedule
// (a runtime test cost the clustered cfg3 product 2.15 -> 2.72 ms).  MODE_ACC
// tests yadd at run time (no measurable cost there).
//
// DUAL (MODE_FUSED only): two products over the same read of O for the same
// v -- y0 = coeff0 (t - s), y1 = coeff1 (t - s), acc0 / acc1 -> part0 / part1
// (the GEVP form needs H_eff v and S v together, PAPER Eq. 11).
template <bool CPLX, int PPT, int R, int MODE, bool ADD = false, bool DUAL = false>
__global__ void __launch_bounds__(stream_max_nt(PPT) + 32, 1) k_stream(const StreamArgs a) {
  static_assert(!DUAL || (MODE == MODE_FUSED && !ADD), "DUAL is a plain fused product with two coefficient vectors");
  constexpr bool kAdd = (MODE == MODE_FUSED && ADD) || MODE == MODE_ACC;
  using T = Traits<CPLX>;
  using S = typename T::S;
  extern __shared__ __align__(128) unsigned char smem[];

  const int NT = blockDim.x - 32;  // consumer threads; last warp = producer
  const int NW = NT >> 5;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int C = a.C, NS = a.stages, WM = a.Wmax;
  const int64_t N = a.n_rows;

  double2* ring = reinterpret_cast<double2*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NS * R * WM * 16);
  uint64_t* empty = full + NS;
  uint64_t* xbar = empty + NS;                       // [kXchSlots]
  S* red = reinterpret_cast<S*>(xbar + kXchSlots);   // [2][R][32]
  S* xch = red + 2 * R * 32;                         // [kXchSlots][C][R]
  S* tslot = xch + kXchSlots * C * R;                // [kXchSlots][R] CTA-level t (C == 1)
  S* pro_s = tslot + kXchSlots * R;                  // [1] cluster-visible prologue slot
  double* pro_g = reinterpret_cast<double*>(pro_s + 1);  // [1]

  const bool clustered = (MODE == MODE_FUSED) && (C > 1);
  const bool xchg = clustered;
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
  const int64_t col0 = slice_lo(a.ld_u, C, rank);
  const int W = (int)(slice_lo(a.ld_u, C, rank + 1) - col0);

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    for (int s = 0; s < kXchSlots; ++s) mbar_init(&xbar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (clustered) cluster_sync();  // peers' barriers initialised before any st.async
  // let the (PDL-launched) finisher get scheduled; it waits for our completion
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // ------------------------------------------------------------ producer --
  if (warp == NW) {
    if (clustered) cluster_arrive();  // prologue exchange barrier (no data needed here)
    if (lane == 0) {
      const uint32_t slice_bytes = (uint32_t)W * 16u;
      for (int g = 0, s = 0, ph = 0; g < G; ++g) {
        if (g >= NS) mbar_wait(&empty[s], ph ^ 1);
        const int64_t r0 = lo + (int64_t)g * R;
        const int rows = (int)min((int64_t)R, hi - r0);
        mbar_arrive_expect_tx(&full[s], slice_bytes * rows);
        double2* dst = ring + (size_t)s * R * WM;
        const double2* src = a.O + r0 * a.ld_u + col0;
        for (int r = 0; r < rows; ++r) bulk_g2s(dst + (size_t)r * WM, src + r * a.ld_u, slice_bytes, &full[s]);
        if (++s == NS) {
          s = 0;
          ph ^= 1;
        }
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
  // number of this thread's units inside the slice (units tid + k*NT)
  const int kval = (W > tid) ? min(PPT, (W - tid + NT - 1) / NT) : 0;
  double2 vreg[PPT];
  double2 acc0[PPT];
  double2 acc1[PPT];
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    vreg[k] = make_double2(0.0, 0.0);
    acc0[k] = make_double2(0.0, 0.0);
    acc1[k] = make_double2(0.0, 0.0);
  }

  // warp-parallel block reduction of per-warp values v[w] stored at buf[w]:
  // every lane of every warp returns the same fixed-order butterfly sum.
  auto block_sum = [&](const S* buf) -> S {
    S x = (lane < NW) ? buf[lane] : T::zero();
    return warp_sum<CPLX>(x);
  };

  S s_val = T::zero();
  if constexpr (MODE == MODE_FUSED || MODE == MODE_DOT) {
    S sp = T::zero();
    double gp = 0.0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      if (k < kval) {
        const int64_t u = col0 + tid + k * NT;
        vreg[k] = load_vec_unit<CPLX>(a.v_re, a.v_im, u);
        if (a.obar) T::dot_acc(sp, a.obar[u], vreg[k]);
        if (a.hf_re) {
          const double2 h = load_vec_unit<CPLX>(a.hf_re, a.hf_im, u);
          gp = fma(h.x, vreg[k].x, gp);
          gp = fma(h.y, vreg[k].y, gp);
        }
      }
    }
    if constexpr (DUAL) {  // each thread reads back only what it wrote: no barrier needed
      double2* vsm = reinterpret_cast<double2*>(smem + a.vs_off);
#pragma unroll
      for (int k = 0; k < PPT; ++k)
        if (k < kval) vsm[tid + k * NT] = vreg[k];
    }
    sp = warp_sum<CPLX>(sp);
    gp = warp_sum<false>(gp);
    S* scr = red;  // red[0][0][*] is free before the main loop
    double* scrg = reinterpret_cast<double*>(red + 32);
    if (lane == 0) {
      scr[warp] = sp;
      scrg[warp] = gp;
    }
    named_bar_sync(1, NT);
    S sc = block_sum(scr);
    double gc = warp_sum<false>((lane < NW) ? scrg[lane] : 0.0);
    named_bar_sync(1, NT);  // scratch reused by the main loop
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

  auto rows_of = [&](int g) -> int { return (int)min((int64_t)R, hi - (lo + (int64_t)g * R)); };
  // ring position of a group: (stage s, phase parity ph), advanced incrementally
  struct Pos {
    int s, ph;
  };
  auto advance = [&](Pos& p) {
    if (++p.s == NS) {
      p.s = 0;
      p.ph ^= 1;
    }
  };

  // dot + block reduction (+ DSMEM send) of group g.  Only warp 0 reduces the
  // per-warp partials; the result reaches the other warps through smem
  // (tslot, C == 1), the DSMEM exchange (xch, C > 1) or global (tpart, DOT).
  auto dot_group = [&](int g, Pos p) {
    const int rows = rows_of(g);
    mbar_wait(&full[p.s], p.ph);
    const double2* st = ring + (size_t)p.s * R * WM;
    S dp[R];
#pragma unroll
    for (int r = 0; r < R; ++r) dp[r] = T::zero();
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      if (k < kval) {
        const int idx = tid + k * NT;
        double2 vk;
        if constexpr (DUAL) vk = reinterpret_cast<const double2*>(smem + a.vs_off)[idx]; else vk = vreg[k];
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (r < rows) T::dot_acc(dp[r], st[(size_t)r * WM + idx], vk);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) dp[r] = warp_sum<CPLX>(dp[r]);
    S* rb = red + (g & 1) * R * 32;
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r) rb[r * 32 + warp] = dp[r];
    }
    named_bar_sync(1, NT);
    if (warp == 0) {
      S t = T::zero();
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const S tr = block_sum(rb + r * 32);
        if (lane == r) t = tr;
      }
      const int b = g % kXchSlots;
      if constexpr (MODE == MODE_DOT) {
        if (lane < rows) reinterpret_cast<S*>(a.tpart)[(int64_t)rank * N + lo + (int64_t)g * R + lane] = t;
      } else if (xchg) {
        if (lane == 0) mbar_arrive_expect_tx(&xbar[b], (uint32_t)(C * rows * sizeof(S)));
        if (lane < rows) {
          const uint32_t la = smem_addr(&xch[(b * C + rank) * R + lane]);
          const uint32_t lb = smem_addr(&xbar[b]);
          for (int q = 0; q < C; ++q) st_async(map_to_rank(la, q), t, map_to_rank(lb, q));
        }
      } else {
        if (lane < rows) tslot[b * R + lane] = t;
      }
    }
  };

  // finish group g: cluster-summed t -> y -> accumulate -> release the stage
  S ys = T::zero();
  S ys1 = T::zero();
  auto acc_group = [&](int g, Pos p, S tin, S cf0, S cf1) {
    const int rows = rows_of(g);
    const double2* st = ring + (size_t)p.s * R * WM;
    S yv = T::zero();
    S yv1 = T::zero();  // DUAL: the second product's y
    if constexpr (MODE == MODE_FUSED || MODE == MODE_ACC) {
      S t = tin;
      if constexpr (MODE == MODE_FUSED) {
        const int b = g % kXchSlots;
        if (xchg) {
          mbar_wait(&xbar[b], (g / kXchSlots) & 1);
          t = T::zero();
          if (lane < rows)
            for (int q = 0; q < C; ++q) t = T::add(t, xch[(b * C + q) * R + lane]);
        } else {
          t = (lane < rows) ? tslot[b * R + lane] : T::zero();
        }
      }
      if (lane < rows) {
        yv = T::mul(cf0, T::sub(t, s_val));
        if constexpr (kAdd) yv = T::add(yv, cf1);  // cf1 = yadd_n (0 without)
        if constexpr (DUAL) yv1 = T::mul(cf1, T::sub(t, s_val));
      }
    } else {
      yv = cf0;
    }
    if constexpr (MODE == MODE_ACC || MODE == MODE_STATS) mbar_wait(&full[p.s], p.ph);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r < rows) {
        const S y = T::shfl(yv, r);
        S y1 = T::zero();
        if constexpr (MODE == MODE_STATS) y1 = T::shfl(cf1, r);
        if constexpr (DUAL) y1 = T::shfl(yv1, r);
        if (MODE != MODE_STATS && tid == 0) ys = T::add(ys, y);
        if (DUAL && tid == 0) ys1 = T::add(ys1, y1);
        if constexpr (DUAL) {
          // all the row's units in flight before the two axpys (the per-unit
          // branches of the loop below serialise the shared-memory loads here);
          // units past the slice add 0 to accumulators that are never stored
          double2 u[PPT];
#pragma unroll
          for (int k = 0; k < PPT; ++k)
            u[k] = (k < kval) ? st[(size_t)r * WM + tid + k * NT] : make_double2(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < PPT; ++k) {
            T::axpy(acc0[k], u[k], y);
            T::axpy(acc1[k], u[k], y1);
          }
        } else {
#pragma unroll
          for (int k = 0; k < PPT; ++k) {
            if (k < kval) {
              const double2 u = st[(size_t)r * WM + tid + k * NT];
              T::axpy(acc0[k], u, y);
              if constexpr (MODE == MODE_STATS) T::axpy(acc1[k], u, y1);
            }
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[p.s]);
  };

  // per-row coefficients for group g (lane r owns row r)
  auto load_coeffs = [&](int g, S& cf0, S& cf1, S& tin) {
    const int64_t r0 = lo + (int64_t)g * R;
    const int rows = rows_of(g);
    cf0 = T::zero();
    cf1 = T::zero();
    tin = T::zero();
    if (lane < rows) {
      if constexpr (MODE == MODE_STATS) {
        const double w = reinterpret_cast<const double*>(a.coeff0)[r0 + lane];
        if constexpr (CPLX) cf0 = make_double2(w, 0.0); else cf0 = w;
        cf1 = reinterpret_cast<const S*>(a.coeff1)[r0 + lane];
      } else if constexpr (MODE != MODE_DOT) {
        cf0 = reinterpret_cast<const S*>(a.coeff0)[r0 + lane];
        if constexpr (kAdd) {
          if (a.yadd) cf1 = reinterpret_cast<const S*>(a.yadd)[r0 + lane];
        }
        if constexpr (DUAL) cf1 = reinterpret_cast<const S*>(a.coeff1)[r0 + lane];
      }
      if constexpr (MODE == MODE_ACC) {
        for (int c = 0; c < C; ++c)
          tin = T::add(tin, reinterpret_cast<const S*>(a.tpart)[(int64_t)c * N + r0 + lane]);
      }
    }
  };

  if constexpr (MODE == MODE_DOT) {
    Pos p{0, 0};
    for (int g = 0; g < G; ++g, advance(p)) {
      dot_group(g, p);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[p.s]);
    }
  } else if constexpr (MODE == MODE_FUSED) {
    if (G > 0) {
      S cf0, cf1, tin;
      load_coeffs(0, cf0, cf1, tin);
      Pos pa{0, 0}, pd{0, 0};
      dot_group(0, pd);
      advance(pd);
      for (int g = 0; g < G; ++g) {
        S cn0 = T::zero(), cn1 = T::zero(), tn = T::zero();
        if (g + 1 < G) {
          load_coeffs(g + 1, cn0, cn1, tn);
          dot_group(g + 1, pd);  // lookahead: its barrier also publishes tslot[g] (C == 1)
          advance(pd);
        } else if (!xchg) {
          named_bar_sync(1, NT);  // publish the last group's tslot
        }
        acc_group(g, pa, T::zero(), cf0, cf1);
        advance(pa);
        cf0 = cn0;
        if constexpr (kAdd || DUAL) cf1 = cn1;
      }
    }
  } else {
    Pos p{0, 0};
    for (int g = 0; g < G; ++g, advance(p)) {
      S cf0, cf1, tin;
      load_coeffs(g, cf0, cf1, tin);
      acc_group(g, p, tin, cf0, cf1);
    }
  }

  if constexpr (MODE != MODE_DOT) {
    double2* p0 = a.part0 + (int64_t)blk * a.ld_u + col0;
    double2* p1 = (MODE == MODE_STATS || DUAL) ? a.part1 + (int64_t)blk * a.ld_u + col0 : nullptr;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      if (k < kval) {
        p0[tid + k * NT] = acc0[k];
        if constexpr (MODE == MODE_STATS || DUAL) p1[tid + k * NT] = acc1[k];
      }
    }
    if (MODE != MODE_STATS && rank == 0 && tid == 0) reinterpret_cast<S*>(a.ysum)[blk] = ys;
    if (DUAL && rank == 0 && tid == 0) reinterpret_cast<S*>(a.ysum1)[blk] = ys1;
  }
  if (clustered) cluster_sync();
}

// Deterministic fixed-order sum of nb per-block partials, 32 units x 8 row
// groups per CTA.  Launched with programmatic dependent launch: the CTA is
// resident before the producer kernel ends and waits in griddepcontrol.wait.
//
// out = sum_b part[b] - conj(obar) * sum_b ysum[b]  (+ u0 * hf)    ; out0 = sum gpart
template <bool CPLX>
__global__ void __launch_bounds__(256) k_finish_mvp(const double2* __restrict__ part, int nb, int64_t ld_u, int upb,
                                                    const void* ysum, const double2* __restrict__ obar,
                                                    const double* hf_re, const double* hf_im, const double* u0,
                                                    double* out_re, double* out_im, const double* gpart,
                                                    int n_gpart, double* out0) {
  using T = Traits<CPLX>;
  using S = typename T::S;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ double2 sh[256];
  __shared__ S shy[1];
  // upb units x (256 / upb) row groups per block
  const int groups = 256 / upb;
  const int tx = threadIdx.x % upb, ty = threadIdx.x / upb;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // Y = sum_b ysum[b]: warp 0, fixed-order strided partial + butterfly
  if (warp == 0) {
    const S* ysv = reinterpret_cast<const S*>(ysum);
    S yp = T::zero();
    for (int b = lane; b < nb; b += 32) yp = T::add(yp, ysv[b]);
    yp = warp_sum<CPLX>(yp);
    if (lane == 0) shy[0] = yp;
  }
  const int64_t i = blockIdx.x * (int64_t)upb + tx;
  double2 acc = make_double2(0.0, 0.0);
  if (i < ld_u) {
    for (int b = ty; b < nb; b += groups) {
      const double2 p = part[(int64_t)b * ld_u + i];
      acc.x += p.x;
      acc.y += p.y;
    }
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  if (ty == 0) {
    const S Y = shy[0];
    acc = sh[tx];
    for (int k = 1; k < groups; ++k) {
      acc.x += sh[k * upb + tx].x;
      acc.y += sh[k * upb + tx].y;
    }
    if (i < ld_u) {
      if (obar) {
        S negY;
        if constexpr (CPLX) negY = make_double2(-Y.x, -Y.y); else negY = -Y;
        T::axpy(acc, obar[i], negY);
      }
      if (hf_re && u0) {
        const double uu = *u0;
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
    if (out0 && blockIdx.x == 0 && tx == 0) {
      double g = 0.0;
      if (hf_re)
        for (int c = 0; c < n_gpart; ++c) g += gpart[c];
      *out0 = g;
    }
  }
}

// obar = sum_b part0[b] (conjugated back for complex) ; g = sum_b part1[b]
template <bool CPLX>
__global__ void __launch_bounds__(256) k_finish_stats(const double2* __restrict__ part0,
                                                      const double2* __restrict__ part1, int nb, int64_t ld_u,
                                                      double2* obar, double2* g) {
  __shared__ double2 sh0[8][33], sh1[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t i = blockIdx.x * 32 + tx;
  double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
  if (i < ld_u) {
    for (int b = ty; b < nb; b += 8) {
      const double2 p = part0[(int64_t)b * ld_u + i];
      const double2 q = part1[(int64_t)b * ld_u + i];
      a0.x += p.x;
      a0.y += p.y;
      a1.x += q.x;
      a1.y += q.y;
    }
  }
  sh0[ty][tx] = a0;
  sh1[ty][tx] = a1;
  __syncthreads();
  if (ty == 0 && i < ld_u) {
    a0 = sh0[0][tx];
    a1 = sh1[0][tx];
    for (int k = 1; k < 8; ++k) {
      a0.x += sh0[k][tx].x;
      a0.y += sh0[k][tx].y;
      a1.x += sh1[k][tx].x;
      a1.y += sh1[k][tx].y;
    }
    if (CPLX) a0.y = -a0.y;
    obar[i] = a0;
    g[i] = a1;
  }
}

}  // namespace irl
