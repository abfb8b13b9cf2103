// Warp-per-row fused product for narrow rows (ld <= 32 * UPL units), e.g. cfg1
// (8192 x 860: 432 units of 16 B per row).
//
// The TMA-ring kernel (k_stream) pays a block-wide reduction per row group;
// at 28 rows per CTA that latency chain, not bandwidth, sets its time.  Here
// one warp owns a whole row: each lane loads its UPL units (coalesced 512-B
// warp loads), the row dot t_n = O_n . v is a warp butterfly, y_n = c_n (t_n -
// Obar.v) is known to every lane at once, and conj(O_n) y_n is accumulated
// from the same registers -- O is read once and nothing crosses warps until the
// CTA epilogue, which sums the warp partials in fixed order into part[blk].
// k_finish_mvp (PDL) then reduces the CTA partials exactly as for k_stream.
#pragma once
#include "stream.cuh"

namespace irl {

// Every warp keeps two rows in flight: the loads of row r + stride are issued
// before row r is reduced and accumulated, and the first row's loads are
// issued before the prologue (v staging, Obar.v), so HBM latency overlaps the
// butterflies instead of adding to them row after row.
// UPL <= 4: 8 warps per CTA, 2 CTAs per SM; larger UPL (two row buffers +
// accumulators, up to ~210 registers at UPL = 16): 8 warps, one CTA per SM.
template <int UPL>
struct RowsGeom {
  static constexpr int NW = 8;
  static constexpr int MINB = UPL <= 4 ? 2 : 1;
};

template <bool CPLX, int UPL>
__global__ void __launch_bounds__(RowsGeom<UPL>::NW * 32, RowsGeom<UPL>::MINB) k_rows_mvp(const StreamArgs a) {
  constexpr int NW = RowsGeom<UPL>::NW;
  using T = Traits<CPLX>;
  using S = typename T::S;
  extern __shared__ __align__(16) unsigned char smem_rw[];
  const int64_t ld_u = a.ld_u;
  double2* vs = reinterpret_cast<double2*>(smem_rw);  // [32 UPL] v units, zero past ld_u
  double2* red = vs + 32 * UPL;                       // [NW][ld_u] warp partials
  __shared__ S shs[NW], shy[NW];
  __shared__ double shg[NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t nw = (int64_t)gridDim.x * NW;

  const S* coeff = reinterpret_cast<const S*>(a.coeff0);
  const S* yadd = reinterpret_cast<const S*>(a.yadd);
  // row r's O units and its coefficient / additive term, all issued at once
  auto load_row = [&](int64_t r, double2 (&o)[UPL], S& c, S& d) {
    c = T::zero();
    d = T::zero();
    if (r < a.n_rows) {
      c = coeff[r];
      if (yadd) d = yadd[r];
    }
    const double2* orow = a.O + r * ld_u + lane;
    // units read per lane: up to 32 UPL (units past ld_u read into the
    // following rows -- finite O entries -- and meet v = 0 in the dot; their
    // accumulators are never stored), but never past the end of the last row:
    // O may sit at the very end of the caller's allocation
    const int64_t left = (r < a.n_rows) ? (a.n_rows - r) * ld_u : 0;
    const int lim = (int)min((int64_t)(32 * UPL), left);
#pragma unroll
    for (int k = 0; k < UPL; ++k) o[k] = (lane + 32 * k < lim) ? __ldg(orow + 32 * k) : make_double2(0.0, 0.0);
  };
  // first row in flight before the prologue
  double2 o0[UPL], o1[UPL];
  S c0, c1, d0, d1;
  int64_t r = (int64_t)blockIdx.x * NW + warp;
  load_row(r, o0, c0, d0);

  // prologue: v -> shared memory; s = Obar . v and g = (F/2) . v in a fixed order
  S sp = T::zero();
  double gp = 0.0;
  for (int64_t u = ld_u + tid; u < 32 * UPL; u += blockDim.x) vs[u] = make_double2(0.0, 0.0);
  for (int64_t u = tid; u < ld_u; u += blockDim.x) {
    const double2 v = load_vec_unit<CPLX>(a.v_re, a.v_im, u);
    vs[u] = v;
    if (a.obar) T::dot_acc(sp, a.obar[u], v);
    if (a.hf_re) {
      const double2 h = load_vec_unit<CPLX>(a.hf_re, a.hf_im, u);
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
  __syncthreads();
  S s_val = T::zero();
  double g_val = 0.0;
  for (int w = 0; w < NW; ++w) {
    s_val = T::add(s_val, shs[w]);
    g_val += shg[w];
  }
  if (blockIdx.x == 0 && tid == 0) {
    reinterpret_cast<S*>(a.spart)[0] = s_val;
    a.gpart[0] = g_val;
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  double2 acc[UPL];
#pragma unroll
  for (int k = 0; k < UPL; ++k) acc[k] = make_double2(0.0, 0.0);
  S ys = T::zero();
  auto row_step = [&](const double2 (&o)[UPL], S c, S d) {
    S t = T::zero();
#pragma unroll
    for (int k = 0; k < UPL; ++k)
      if (lane + 32 * k < ld_u) T::dot_acc(t, o[k], vs[lane + 32 * k]);
    t = warp_sum<CPLX>(t);  // butterfly: every lane holds t_n
    const S y = T::add(T::mul(c, T::sub(t, s_val)), d);  // d: connected completion term (0 without)
#pragma unroll
    for (int k = 0; k < UPL; ++k) T::axpy(acc[k], o[k], y);
    ys = T::add(ys, y);
  };
  // two row buffers, alternating: the next row's loads are in flight while
  // the current row is reduced and accumulated
  while (r < a.n_rows) {
    load_row(r + nw, o1, c1, d1);
    row_step(o0, c0, d0);
    r += nw;
    if (r >= a.n_rows) break;
    load_row(r + nw, o0, c0, d0);
    row_step(o1, c1, d1);
    r += nw;
  }
  // epilogue: the warp partials, summed in warp order
#pragma unroll
  for (int k = 0; k < UPL; ++k) {
    const int64_t u = lane + 32 * k;
    if (u < ld_u) red[warp * ld_u + u] = acc[k];
  }
  if (lane == 0) shy[warp] = ys;
  __syncthreads();
  double2* p0 = a.part0 + (int64_t)blockIdx.x * ld_u;
  for (int64_t u = tid; u < ld_u; u += blockDim.x) {
    double2 t2 = red[u];
    for (int w = 1; w < NW; ++w) {
      t2.x += red[w * ld_u + u].x;
      t2.y += red[w * ld_u + u].y;
    }
    p0[u] = t2;
  }
  if (tid == 0) {
    S yt = shy[0];
    for (int w = 1; w < NW; ++w) yt = T::add(yt, shy[w]);
    reinterpret_cast<S*>(a.ysum)[blockIdx.x] = yt;
  }
}

}  // namespace irl
