// The reference's own NQS on the device: the autoregressive
// ansatz of ansatz.py (ans:1-290) -- batched log psi, log-derivative rows and
// exact ancestral sampling.
//
// One warp per configuration, lanes over hidden units (h <= 32 HPL).  The
// conditional network's pre-activation for position i,
//   z_i = b1 + W1 u_i,   u_i = [+-1 prefix (j < i), 0 ..., onehot(M + i)]  (ans:156-162)
// is carried incrementally: r_i = b1 + sum_{j<i} s_j W1[:, j], z_i = r_i + W1[:, M+i].
// Logits l = b2 + W2 tanh(z_i) are warp sums; the particle-number mask of
// _channel_state (ans:130-153) forces a channel's outcome once it is filled or
// must be filled; ln p sums the masked log-softmax (ans:165-183, 239-247).
// The phase head phi = w_lin.s + up.tanh(Wp s + bp) + c (ans:243-247).
//
// Rows (ans:249-290): the amplitude-head gradient (real part) accumulates over
// the unforced positions g = (onehot - p)/2, dW2 += g a^T, db2 += g,
// dz = (W2^T g)(1 - a^2), dW1 += dz u^T, db1 += dz; the W1 prefix columns are
// s_j times the suffix sums of dz (kept per warp in shared memory); the phase
// gradient (imaginary part) is [dt s^T, dt, t, s, 1] with dt = up (1 - t^2).
//
// Sampling (ans:215-236): the reference draws one uniform per position from a
// per-sample numpy PCG64 stream (SeedSequence(seed).spawn(count)); the host
// hands over each stream's 128-bit state and increment and lane 0 replays the
// generator bit for bit (XSL-RR output, next_double = (x >> 11) 2^-53).
#pragma once
#include "common.cuh"

namespace irl {

enum ArMode { AR_LOGAMP = 0, AR_ROWS = 1, AR_SAMPLE = 2 };
constexpr int AR_WARPS = 4;  // warps (configurations) per CTA

struct ArArgs {
  const uint64_t* xbits;  // LOGAMP / ROWS: [n] configurations
  int64_t n;
  int M, h, n_up, n_down;
  const double* theta;  // [W1 (h x 2M), b1, W2 (2 x h), b2, Wp (h x M), bp, up, w_lin, c]
  double2* logpsi;      // LOGAMP: [n] (ln p / 2, phase)
  double2* O;           // ROWS: [n][ld] complex rows
  int64_t ld;
  const uint64_t* rng;  // SAMPLE: [n][4] = state hi, state lo, inc hi, inc lo
  uint64_t* out_bits;   // SAMPLE: [n]
  int* error;           // set when a configuration is outside the sector (ROWS) or a prefix is infeasible
};

__device__ __forceinline__ double ar_logaddexp(double a, double b) {
  const double m = fmax(a, b);
  return m + log1p(exp(-fabs(a - b)));
}

// 128-bit PCG64 step + XSL-RR output (numpy's PCG64)
struct Pcg64 {
  uint64_t shi, slo, ihi, ilo;
  __device__ __forceinline__ double next_double() {
    const uint64_t MH = 0x2360ED051FC65DA4ull, ML = 0x4385DF649FCCF645ull;
    // state = state * MULT + inc  (mod 2^128)
    const uint64_t lo = slo * ML;
    const uint64_t hi = __umul64hi(slo, ML) + slo * MH + shi * ML;
    const uint64_t nlo = lo + ilo;
    const uint64_t nhi = hi + ihi + (nlo < lo ? 1ull : 0ull);
    shi = nhi;
    slo = nlo;
    const uint64_t x = nhi ^ nlo;
    const unsigned rot = (unsigned)(nhi >> 58);
    const uint64_t out = (x >> rot) | (x << ((64u - rot) & 63u));
    return (double)(out >> 11) * (1.0 / 9007199254740992.0);
  }
};

template <int HPL, int MODE>
__global__ void __launch_bounds__(AR_WARPS * 32) k_autoreg(const ArArgs a) {
  extern __shared__ __align__(16) double dz_s[];  // ROWS: [AR_WARPS][M][32 HPL]
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int M = a.M, h = a.h, half = M / 2;
  const double* th = a.theta;
  const double* W1 = th;
  const double* b1 = W1 + (size_t)h * 2 * M;
  const double* W2 = b1 + h;
  const double* b2 = W2 + 2 * h;
  const double* Wp = b2 + 2;
  const double* bp = Wp + (size_t)h * M;
  const double* up = bp + h;
  const double* wl = up + h;
  const double* cc = wl + M;
  double* dzw = dz_s + (size_t)wib * M * 32 * HPL;

  for (int64_t r = (int64_t)blockIdx.x * AR_WARPS + wib; r < a.n; r += (int64_t)gridDim.x * AR_WARPS) {
    uint64_t x = (MODE == AR_SAMPLE) ? 0ull : a.xbits[r];
    const uint64_t upmask = (half >= 64) ? ~0ull : ((1ull << half) - 1ull);
    if (MODE != AR_SAMPLE) {
      const int cu = __popcll(x & upmask), cd = __popcll(x >> half);
      if (cu != a.n_up || cd != a.n_down || (M < 64 && (x >> M) != 0)) {
        // outside the sector: ln psi = -inf (ans:237-238); rows are an error (ans:256-257)
        if (MODE == AR_LOGAMP) {
          if (lane == 0) a.logpsi[r] = make_double2(-INFINITY, 0.0);
        } else {
          if (lane == 0) atomicExch(a.error, 1);
          for (int64_t u = lane; u < a.ld; u += 32) a.O[r * a.ld + u] = make_double2(0.0, 0.0);
        }
        continue;
      }
    }
    Pcg64 rng{};
    if (MODE == AR_SAMPLE && lane == 0) {
      rng.shi = a.rng[4 * r];
      rng.slo = a.rng[4 * r + 1];
      rng.ihi = a.rng[4 * r + 2];
      rng.ilo = a.rng[4 * r + 3];
    }
    double rk[HPL], gb1[HPL], gw2a[HPL], gw2b[HPL];
#pragma unroll
    for (int q = 0; q < HPL; ++q) {
      const int k = lane + 32 * q;
      rk[q] = k < h ? b1[k] : 0.0;
      gb1[q] = gw2a[q] = gw2b[q] = 0.0;
    }
    double logp_sum = 0.0, gb2a = 0.0, gb2b = 0.0;
    int cnt_up = 0, cnt_dn = 0;
    for (int i = 0; i < M; ++i) {
      // _channel_state (ans:130-153)
      int needed, remaining;
      if (i < half) {
        needed = a.n_up - cnt_up;
        remaining = half - i;
      } else {
        needed = a.n_down - cnt_dn;
        remaining = M - i;
      }
      if (needed < 0 || needed > remaining) {
        if (lane == 0) atomicExch(a.error, 2);
      }
      const bool f_empty = needed == 0, f_occ = needed == remaining;
      double av[HPL];
      double l0 = 0.0, l1 = 0.0;
#pragma unroll
      for (int q = 0; q < HPL; ++q) {
        const int k = lane + 32 * q;
        av[q] = 0.0;
        if (k < h) {
          av[q] = tanh(rk[q] + W1[(size_t)k * 2 * M + M + i]);
          l0 = fma(W2[k], av[q], l0);
          l1 = fma(W2[h + k], av[q], l1);
        }
      }
      l0 = warp_sum<false>(l0) + b2[0];
      l1 = warp_sum<false>(l1) + b2[1];
      double lp0, lp1;
      if (f_empty) {
        lp0 = 0.0;
        lp1 = -INFINITY;
      } else if (f_occ) {
        lp0 = -INFINITY;
        lp1 = 0.0;
      } else {
        const double lz = ar_logaddexp(l0, l1);
        lp0 = l0 - lz;
        lp1 = l1 - lz;
      }
      bool occ;
      if constexpr (MODE == AR_SAMPLE) {
        int take = 0;
        if (lane == 0) take = rng.next_double() < exp(lp1) ? 1 : 0;
        occ = __shfl_sync(0xffffffffu, take, 0) != 0;
        if (occ) x |= 1ull << i;
      } else {
        occ = (x >> i) & 1ull;
      }
      logp_sum += occ ? lp1 : lp0;
      if constexpr (MODE == AR_ROWS) {
        const bool forced = f_empty || f_occ;
        double g0 = 0.0, g1 = 0.0;
        if (!forced) {
          g0 = 0.5 * ((occ ? 0.0 : 1.0) - exp(lp0));
          g1 = 0.5 * ((occ ? 1.0 : 0.0) - exp(lp1));
          gb2a += g0;
          gb2b += g1;
        }
#pragma unroll
        for (int q = 0; q < HPL; ++q) {
          const int k = lane + 32 * q;
          double dz = 0.0;
          if (!forced && k < h) {
            gw2a[q] = fma(g0, av[q], gw2a[q]);
            gw2b[q] = fma(g1, av[q], gw2b[q]);
            dz = (W2[k] * g0 + W2[h + k] * g1) * (1.0 - av[q] * av[q]);
            gb1[q] += dz;
          }
          dzw[(size_t)i * 32 * HPL + k] = dz;
        }
      }
      // advance the prefix: r += s_i W1[:, i]
      const double si = occ ? 1.0 : -1.0;
#pragma unroll
      for (int q = 0; q < HPL; ++q) {
        const int k = lane + 32 * q;
        if (k < h) rk[q] = fma(si, W1[(size_t)k * 2 * M + i], rk[q]);
      }
      if (occ) {
        if (i < half) ++cnt_up; else ++cnt_dn;
      }
    }
    if constexpr (MODE == AR_SAMPLE) {
      if (lane == 0) a.out_bits[r] = x;
      continue;
    }
    // phase head (ans:243-247)
    double tk[HPL], ph = 0.0;
#pragma unroll
    for (int q = 0; q < HPL; ++q) {
      const int k = lane + 32 * q;
      tk[q] = 0.0;
      if (k < h) {
        double z = bp[k];
        for (int j = 0; j < M; ++j) z = fma(Wp[(size_t)k * M + j], ((x >> j) & 1ull) ? 1.0 : -1.0, z);
        tk[q] = tanh(z);
        ph = fma(up[k], tk[q], ph);
      }
    }
    for (int j = lane; j < M; j += 32) ph = fma(wl[j], ((x >> j) & 1ull) ? 1.0 : -1.0, ph);
    ph = warp_sum<false>(ph) + cc[0];
    if constexpr (MODE == AR_LOGAMP) {
      if (lane == 0) a.logpsi[r] = make_double2(0.5 * logp_sum, ph);
      continue;
    }
    // ---- rows: [W1 (h x 2M), b1, W2 (2 x h), b2 | Wp (h x M), bp, up, w_lin, c]
    __syncwarp();
    double2* row = a.O + r * a.ld;
    const size_t o_b1 = (size_t)h * 2 * M, o_w2 = o_b1 + h, o_b2 = o_w2 + 2 * h, o_wp = o_b2 + 2;
    const size_t o_bp = o_wp + (size_t)h * M, o_up = o_bp + h, o_wl = o_up + h, o_c = o_wl + M;
#pragma unroll
    for (int q = 0; q < HPL; ++q) {
      const int k = lane + 32 * q;
      if (k >= h) continue;
      double2* w1r = row + (size_t)k * 2 * M;
      double suf = 0.0;  // sum_{i > j} dz_i[k]
      for (int j = M - 1; j >= 0; --j) {
        const double dzj = dzw[(size_t)j * 32 * HPL + k];
        w1r[M + j] = make_double2(dzj, 0.0);
        w1r[j] = make_double2(((x >> j) & 1ull) ? suf : -suf, 0.0);
        suf += dzj;
      }
      row[o_b1 + k] = make_double2(gb1[q], 0.0);
      row[o_w2 + k] = make_double2(gw2a[q], 0.0);
      row[o_w2 + h + k] = make_double2(gw2b[q], 0.0);
      const double dt = up[k] * (1.0 - tk[q] * tk[q]);
      double2* wpr = row + o_wp + (size_t)k * M;
      for (int j = 0; j < M; ++j) wpr[j] = make_double2(0.0, ((x >> j) & 1ull) ? dt : -dt);
      row[o_bp + k] = make_double2(0.0, dt);
      row[o_up + k] = make_double2(0.0, tk[q]);
    }
    for (int j = lane; j < M; j += 32) row[o_wl + j] = make_double2(0.0, ((x >> j) & 1ull) ? 1.0 : -1.0);
    if (lane == 0) {
      row[o_b2] = make_double2(gb2a, 0.0);
      row[o_b2 + 1] = make_double2(gb2b, 0.0);
      row[o_c] = make_double2(0.0, 1.0);
    }
    for (int64_t u = (int64_t)o_c + 1 + lane; u < a.ld; u += 32) row[u] = make_double2(0.0, 0.0);
    __syncwarp();
  }
}

// E_loc = diag + sum_e element_e exp(ln psi(y_e) - ln psi(x)) per sample, fixed order (ham:290-302)
__global__ void k_eloc_combine(const int64_t* __restrict__ indptr, const double* __restrict__ elem,
                               const double2* __restrict__ lp_part, const double2* __restrict__ lp_x,
                               const double* __restrict__ diag, int64_t n, double2* __restrict__ eloc) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < n; r += nw) {
    const double2 lx = lp_x[r];
    double re = 0.0, im = 0.0;
    for (int64_t e = indptr[r] + lane; e < indptr[r + 1]; e += 32) {
      const double2 ly = lp_part[e];
      if (ly.x == -INFINITY) continue;  // est:246 / ham:297
      double s, c;
      sincos(ly.y - lx.y, &s, &c);
      const double m = elem[e] * exp(ly.x - lx.x);
      re = fma(m, c, re);
      im = fma(m, s, im);
    }
    re = warp_sum<false>(re);
    im = warp_sum<false>(im);
    if (lane == 0) eloc[r] = make_double2(diag[r] + re, im);
  }
}

}  // namespace irl
