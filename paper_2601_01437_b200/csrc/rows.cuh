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

// UPL <= 8: 8 warps per CTA, 2 CTAs per SM; UPL = 16 (up to 512 units, ~160
// registers): 12 warps per CTA, one CTA per SM.
template <int UPL>
struct RowsGeom {
  static constexpr int NW = UPL <= 8 ? 8 : 12;
  static constexpr int MINB = UPL <= 8 ? 2 : 1;
};

template <bool CPLX, int UPL>
__global__ void __launch_bounds__(RowsGeom<UPL>::NW * 32, RowsGeom<UPL>::MINB) k_rows_mvp(const StreamArgs a) {
  constexpr int NW = RowsGeom<UPL>::NW;
  using T = Traits<CPLX>;
  using S = typename T::S;
  extern __shared__ __align__(16) unsigned char smem_rw[];
  const int64_t ld_u = a.ld_u;
  double2* vs = reinterpret_cast<double2*>(smem_rw);  // [ld_u] v units
  double2* red = vs + ld_u;                           // [NW][ld_u] warp partials
  __shared__ S shs[NW], shy[NW];
  __shared__ double shg[NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // prologue: v -> shared memory; s = Obar . v and g = (F/2) . v in a fixed order
  S sp = T::zero();
  double gp = 0.0;
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

  const S* coeff = reinterpret_cast<const S*>(a.coeff0);
  const S* yadd = reinterpret_cast<const S*>(a.yadd);
  double2 acc[UPL];
#pragma unroll
  for (int k = 0; k < UPL; ++k) acc[k] = make_double2(0.0, 0.0);
  S ys = T::zero();
  const int64_t nw = (int64_t)gridDim.x * NW;
  for (int64_t r = (int64_t)blockIdx.x * NW + warp; r < a.n_rows; r += nw) {
    const double2* orow = a.O + r * ld_u;
    double2 o[UPL];
#pragma unroll
    for (int k = 0; k < UPL; ++k) {
      const int64_t u = lane + 32 * k;
      o[k] = (u < ld_u) ? __ldg(orow + u) : make_double2(0.0, 0.0);
    }
    S t = T::zero();
#pragma unroll
    for (int k = 0; k < UPL; ++k) {
      const int64_t u = lane + 32 * k;
      if (u < ld_u) T::dot_acc(t, o[k], vs[u]);
    }
    t = warp_sum<CPLX>(t);  // butterfly: every lane holds t_n
    S y = T::mul(coeff[r], T::sub(t, s_val));
    if (yadd) y = T::add(y, yadd[r]);  // connected completion term
#pragma unroll
    for (int k = 0; k < UPL; ++k) T::axpy(acc[k], o[k], y);
    ys = T::add(ys, y);
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
