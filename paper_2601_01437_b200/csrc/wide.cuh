// Single-HBM-read product for very wide rows (cfg4: 470 KB rows, cfg5: 1.67 MB).
//
// The fused cluster kernel needs a whole row slice per CTA in shared memory
// while the row's dot is exchanged, which limits rows in flight when rows are
// this wide; the two-pass path reads O twice from HBM.  Here the GPU runs one
// persistent, cooperatively launched grid with one CTA per SM:
//
//   * CTA c owns the column slice c of EVERY row (G = #SMs slices), so its
//     slice of the output needs no cross-CTA reduction at all;
//   * rows go in blocks of R (~30 MB per block).  Phase D(b): stream the slice
//     of block b through a TMA ring, per-row partial dots (minus the slice's
//     share of Obar.v) -> tpart[b % 4][r][c]; arrive on block b's counter.
//   * Phase A(b), one block later: wait until all G CTAs have arrived for b,
//     every CTA forms y_r = c_r sum_c tpart[..][r][c] in the same fixed order,
//     then streams its slice of block b again -- now from L2, the block was
//     read one block earlier -- and accumulates conj(O_r) y_r in registers.
//
// The producer warp streams D(0), D(1), A(0), D(2), A(1), ..., so the barrier
// of block b is hidden behind D(b+1) and the ring keeps prefetching A(b) while
// consumers wait.  HBM reads O once; L2 serves the second pass.  Each block
// has its own arrival counter (a shared running total could be satisfied by a
// fast CTA's later arrivals while a slow CTA had not yet published block b).
// tpart has four buffers: a CTA writes block b+1's partials (into b-3's
// buffer) only after its A(b-1), i.e. after every CTA arrived for b-1 and so
// finished A(b-3); with three buffers a slow CTA could still be reading A(b-2)
// (seen as a rare 1e-7 error on cfg5).  All sums are fixed-order.
#pragma once
#include "stream.cuh"

namespace irl {

constexpr int WIDE_NT = 256;  // consumer threads
constexpr int WIDE_NW = WIDE_NT / 32;

struct WideArgs {
  const double2* O;
  int64_t n_rows, ld_u;
  const double* v_re;
  const double* v_im;
  const double* hf_re;
  const double* hf_im;
  const double2* obar;
  const void* coeff;  // S[N]
  const void* yadd;   // S[N] additive row term (connected completion); null = none
  const double* u0;
  double* out_re;
  double* out_im;
  double* out0;
  void* tpart;              // S[4][R][G]
  double* gpart;            // [G]
  unsigned int* counter;    // [NB] per-block arrival counters, zero at launch
  int* error;               // set on a barrier timeout (never expected)
  int R;                    // rows per block
  int NS;                   // ring stages
  int RB;                   // row slices per stage (<= WIDE_RB)
  int WM;                   // row slice width in the ring (units)
};

constexpr int WIDE_RB = 8;

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned int* p, unsigned int v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// mbarrier wait that gives up (and flags the error) after ~30 s instead of
// hanging the GPU if the ring ever desynchronised
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t parity, int* error) {
  const uint32_t addr = smem_addr(bar);
  if (mbar_try_wait(addr, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(addr, parity)) {
    if (clock64() - t0 > (1LL << 36)) {
      atomicExch(error, 2);
      return;
    }
  }
}

// Consumers work warp-per-row: a ring stage holds WIDE_NW row slices and warp w
// takes slice w, so a row's partial dot over the CTA's slice is one warp
// butterfly (no cross-warp reduction per row) and each lane owns the units
// lane + 32 k (k < UPL) of the slice; v sits in shared memory.  The warps'
// accumulators meet in shared memory once, at the end, in warp order.
template <bool CPLX, int UPL>
__global__ void __launch_bounds__(WIDE_NT + 32, 1) k_wide(const WideArgs a) {
  using T = Traits<CPLX>;
  using S = typename T::S;
  extern __shared__ __align__(16) unsigned char smem_w[];
  const int NS = a.NS, WM = a.WM, R = a.R;
  const int RB = a.RB;  // WIDE_NW * rpw row slices per stage
  const int rpw = RB / WIDE_NW;
  double2* ring = reinterpret_cast<double2*>(smem_w);                          // [NS][RB][WM]
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)NS * RB * WM);  // [NS]
  uint64_t* empty = full + NS;                                                 // [NS]
  S* ys = reinterpret_cast<S*>(empty + NS);                                    // [R]
  double2* vs = reinterpret_cast<double2*>(ys + R);                            // [WM] v slice
  __shared__ S shs[WIDE_NW];
  __shared__ double shg[WIDE_NW];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, c = blockIdx.x;
  const int64_t N = a.n_rows;
  const int64_t col0 = slice_lo(a.ld_u, G, c);
  const int W = (int)(slice_lo(a.ld_u, G, c + 1) - col0);
  const int NB = (int)((N + R - 1) / R);
  S* tpart = reinterpret_cast<S*>(a.tpart);

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], WIDE_NW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // ------------------------------------------------------------ producer --
  // item sequence: D(0), then for each b: D(b+1) (if any), A(b)
  if (warp == WIDE_NW) {
    if (lane == 0) {
      const uint32_t slice_bytes = (uint32_t)W * 16u;
      int s = 0, ph = 0;
      int64_t issued = 0;
      auto stream_block = [&](int b) {
        const int64_t r0 = (int64_t)b * R;
        const int rows = (int)min((int64_t)R, N - r0);
        for (int r = 0; r < rows; r += RB) {  // one stage = up to RB row slices
          const int rs = min(RB, rows - r);
          if (issued >= NS) mbar_wait_bounded(&empty[s], ph ^ 1, a.error);
          mbar_arrive_expect_tx(&full[s], slice_bytes * (uint32_t)rs);
          for (int i = 0; i < rs; ++i)
            bulk_g2s(ring + ((size_t)s * RB + i) * WM, a.O + (r0 + r + i) * a.ld_u + col0, slice_bytes, &full[s]);
          ++issued;
          if (++s == NS) {
            s = 0;
            ph ^= 1;
          }
        }
      };
      stream_block(0);
      for (int b = 0; b < NB; ++b) {
        if (b + 1 < NB) stream_block(b + 1);
        stream_block(b);
      }
    }
    return;
  }

  // ----------------------------------------------------------- consumers --
  // v slice -> smem; this slice's shares of Obar . v and (F/2) . v
  S sp = T::zero();
  double gp = 0.0;
  for (int u = tid; u < W; u += WIDE_NT) {
    const double2 v = load_vec_unit<CPLX>(a.v_re, a.v_im, col0 + u);
    vs[u] = v;
    if (a.obar) T::dot_acc(sp, a.obar[col0 + u], v);
    if (a.hf_re) {
      const double2 h = load_vec_unit<CPLX>(a.hf_re, a.hf_im, col0 + u);
      gp = fma(h.x, v.x, gp);
      gp = fma(h.y, v.y, gp);
    }
  }
  sp = warp_sum<CPLX>(sp);
  gp = warp_sum<false>(gp);
  if (lane == 0) {
    shs[warp] = sp;
    shg[warp] = gp;
  }
  named_bar_sync(1, WIDE_NT);
  S s_c = T::zero();
  double g_c = 0.0;
  for (int w = 0; w < WIDE_NW; ++w) {
    s_c = T::add(s_c, shs[w]);
    g_c += shg[w];
  }
  if (tid == 0) a.gpart[c] = g_c;  // published with the first arrive

  double2 acc[UPL];
#pragma unroll
  for (int k = 0; k < UPL; ++k) acc[k] = make_double2(0.0, 0.0);
  int s = 0, ph = 0;
  auto advance = [&]() {
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
  };
  const S* coeff = reinterpret_cast<const S*>(a.coeff);
  S ysum = T::zero();  // lane 0 of each warp: sum of the y it formed

  auto phase_d = [&](int b) {
    const int64_t r0 = (int64_t)b * R;
    const int rows = (int)min((int64_t)R, N - r0);
    S* tp = tpart + ((size_t)(b & 3) * R) * G;
    for (int r = 0; r < rows; r += RB) {
      mbar_wait_bounded(&full[s], ph, a.error);
      // this warp's rows of the stage: warp, warp + NW (rpw <= 2); two partial
      // accumulators per row keep the FMA chains short
      S t[2][2];
#pragma unroll
      for (int i = 0; i < 2; ++i) t[i][0] = t[i][1] = T::zero();
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int rr = warp + i * WIDE_NW;
        if (i < rpw && r + rr < rows) {
          const double2* row = ring + ((size_t)s * RB + rr) * WM;
#pragma unroll
          for (int k = 0; k < UPL; ++k) {
            const int u = lane + 32 * k;
            if (u < W) T::dot_acc(t[i][k & 1], row[u], vs[u]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int rr = warp + i * WIDE_NW;
        if (i < rpw && r + rr < rows) {
          const S tt = warp_sum<CPLX>(T::add(t[i][0], t[i][1]));
          if (lane == 0) tp[(size_t)(r + rr) * G + c] = T::sub(tt, s_c);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      advance();
    }
    named_bar_sync(1, WIDE_NT);  // every warp's partials written
    if (tid == 0) red_release_add(a.counter + b, 1u);
  };

  auto phase_a = [&](int b) {
    const int64_t r0 = (int64_t)b * R;
    const int rows = (int)min((int64_t)R, N - r0);
    if (tid == 0) {  // wait until every CTA has published block b
      // one counter per block: a single running total could reach G (b + 1)
      // with a fast CTA's later arrivals standing in for a slow CTA's missing
      // one, and block b's partials would be read before they were all written
      const unsigned int target = (unsigned int)G;
      const long long t0 = clock64();
      while (ld_acquire_u32(a.counter + b) < target) {
        if (clock64() - t0 > (1LL << 36)) {  // ~30 s: never expected; no hang
          atomicExch(a.error, 1);
          break;
        }
      }
    }
    named_bar_sync(1, WIDE_NT);
    const S* tp = tpart + ((size_t)(b & 3) * R) * G;
    // 4 rows per warp at a time: their partial loads are independent (in flight together)
    for (int r = warp * 4; r < rows; r += WIDE_NW * 4) {
      S t[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) t[i] = T::zero();
      for (int q = lane; q < G; q += 32) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (r + i < rows) t[i] = T::add(t[i], __ldcg(tp + (size_t)(r + i) * G + q));
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (r + i >= rows) break;
        const S tt = warp_sum<CPLX>(t[i]);
        S y = T::mul(coeff[r0 + r + i], tt);
        if (a.yadd) y = T::add(y, reinterpret_cast<const S*>(a.yadd)[r0 + r + i]);
        if (lane == 0) {
          ys[r + i] = y;
          ysum = T::add(ysum, y);
        }
      }
    }
    named_bar_sync(1, WIDE_NT);
    for (int r = 0; r < rows; r += RB) {
      mbar_wait_bounded(&full[s], ph, a.error);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int rr = warp + i * WIDE_NW;
        if (i < rpw && r + rr < rows) {
          const double2* row = ring + ((size_t)s * RB + rr) * WM;
          const S y = ys[r + rr];
#pragma unroll
          for (int k = 0; k < UPL; ++k) {
            const int u = lane + 32 * k;
            if (u < W) T::axpy(acc[k], row[u], y);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      advance();
    }
    named_bar_sync(1, WIDE_NT);  // ys reused by the next block
  };

  phase_d(0);
  for (int b = 0; b < NB; ++b) {
    if (b + 1 < NB) phase_d(b + 1);
    phase_a(b);
  }

  // the warps' accumulators meet in shared memory (ring is free: every stage consumed)
  double2* red = ring;  // [NW][WM]
#pragma unroll
  for (int k = 0; k < UPL; ++k) {
    const int u = lane + 32 * k;
    if (u < W) red[(size_t)warp * WM + u] = acc[k];
  }
  if (lane == 0) shs[warp] = ysum;
  named_bar_sync(1, WIDE_NT);
  S Y = T::zero();  // sum over all rows of y, the same fixed order in every CTA
  for (int w = 0; w < WIDE_NW; ++w) Y = T::add(Y, shs[w]);
  const double uu = (a.hf_re && a.u0) ? *a.u0 : 0.0;
  for (int u = tid; u < W; u += WIDE_NT) {
    double2 o = red[u];
    for (int w = 1; w < WIDE_NW; ++w) {
      o.x += red[(size_t)w * WM + u].x;
      o.y += red[(size_t)w * WM + u].y;
    }
    const int64_t gu = col0 + u;
    if (a.obar) {
      S negY;
      if constexpr (CPLX) negY = make_double2(-Y.x, -Y.y); else negY = -Y;
      T::axpy(o, a.obar[gu], negY);
    }
    if (a.hf_re && a.u0) {
      const double2 h = load_vec_unit<CPLX>(a.hf_re, a.hf_im, gu);
      o.x = fma(uu, h.x, o.x);
      o.y = fma(uu, h.y, o.y);
    }
    if constexpr (!CPLX) {
      reinterpret_cast<double2*>(a.out_re)[gu] = o;
    } else {
      a.out_re[gu] = o.x;
      if (a.out_im) a.out_im[gu] = o.y;
    }
  }
  if (a.out0 && c == 0 && tid == 0) {  // every CTA arrived for the last block: gpart complete
    double g = 0.0;
    if (a.hf_re)
      for (int q = 0; q < G; ++q) g += __ldcg(a.gpart + q);
    *a.out0 = g;
  }
}

}  // namespace irl
