// Local energies and connected configurations of a molecular Hamiltonian
// (hamiltonian.py:238-302, the step before the hot path).
//
// One CTA per sample x (a bitmask over M <= 64 spin-orbitals, blocked
// layout: 0..ns-1 spin up, ns..2ns-1 spin down, hilbert.py:1-5).  The CTA
//   1. lists the occupied / empty orbitals of each spin and the hole / particle
//      pair tables in shared memory,
//   2. forms theta_j(x) = b_j + sum_{i occ} W_ji and the per-unit factors of
//      the amplitude ratio (threads over hidden units),
//   3. enumerates every spin-conserving single and double excitation
//      (ham:255-274) -- thread t owns the contiguous index range
//      [t T / B, (t+1) T / B) of the T candidates -- computes its
//      Slater-Condon element (ham:180-235) with the fermionic sign of
//      classify_excitation (hilbert.py:137-158), drops |element| <= drop
//      (ham:282-285), and the amplitude ratio psi(y)/psi(x) from the updated
//      hidden pre-activations theta_j(y) = theta_j(x) + W_jp + W_jq - W_jm - W_jn:
//        RBM  exp(a.(y - x)) prod_j (P_j e^{D_j} + Q_j e^{-D_j}),
//             P_j = (1 + tanh theta_j)/2, Q_j = (1 - tanh theta_j)/2
//             (= prod_j cosh(theta_j + D_j)/cosh(theta_j); complex theta too)
//        MLP  exp(sum_j u_j (tanh(theta_j + D_j) - tanh theta_j)),
//   4. MODE_ELOC: E_loc(x) = <x|H|x> + sum element * ratio (local_energy,
//      ham:290-302), block-reduced in a fixed order;
//      MODE_COUNT: number of kept partners;  MODE_FILL: the kept partners'
//      bitmasks, elements and coefficients element * ratio written in
//      enumeration order at offsets[r] (build_connected_cache, est:221-251).
#pragma once
#include "common.cuh"
#include "obuild.cuh"  // MODEL_RBM / MODEL_MLP, ctanh

namespace irl {

enum HamMode { HAM_ELOC = 0, HAM_COUNT = 1, HAM_FILL = 2 };
constexpr int HAM_NT = 128;
constexpr int HAM_MAXPAIR = 496;  // C(32, 2)

struct HamArgs {
  const uint64_t* xbits;
  int64_t n;
  int ns;      // spatial orbitals (M = 2 ns <= 64)
  int hidden;
  double e_core;
  const double* h1;  // ns x ns
  const double* g2;  // ns^4, chemists' (ij|kl)
  double drop;
  const void* avec;  // RBM a (M), S
  const void* bvec;  // b (h), S
  const void* WT;    // (M x h) transposed W, S
  const void* EX;    // (M x h x 2) {exp(W^T), exp(-W^T)}, S (RBM)
  const double* uvec;  // MLP u (h)
  void* out;         // ELOC: S[n]
  int64_t* counts;   // COUNT: [n]
  double* diag;      // COUNT (optional): [n] diagonal elements <x|H|x>
  const int64_t* offsets;  // FILL: [n] start of each sample's partners
  uint64_t* pbits;   // FILL
  double* pelem;     // FILL
  void* pcoeff;      // FILL: S
};

__device__ __forceinline__ int ham_spatial(int i, int ns) { return i < ns ? i : i - ns; }
__device__ __forceinline__ bool ham_same(int i, int j, int ns) { return (i < ns) == (j < ns); }

// parity of moving one electron hole -> particle on `bits` (hilbert.py:126-134)
__device__ __forceinline__ double ham_move_sign(uint64_t bits, int hole, int part) {
  const int lo = min(hole, part), hi = max(hole, part);
  const uint64_t below_hi = (hi >= 64) ? ~0ull : ((1ull << hi) - 1ull);
  const uint64_t upto_lo = (lo + 1 >= 64) ? ~0ull : ((1ull << (lo + 1)) - 1ull);
  return (__popcll(bits & (below_hi ^ upto_lo)) & 1) ? -1.0 : 1.0;
}

template <bool CPLX>
__device__ __forceinline__ typename Traits<CPLX>::S ham_exp(typename Traits<CPLX>::S z);
template <>
__device__ __forceinline__ double ham_exp<false>(double z) { return exp(z); }
template <>
__device__ __forceinline__ double2 ham_exp<true>(double2 z) {
  double s, c;
  sincos(z.y, &s, &c);
  const double m = exp(z.x);
  return make_double2(m * c, m * s);
}

// SMT: the RBM exp table lives in shared memory (rows padded by one entry so
// lanes on different orbitals hit different banks); one CTA of NT threads per SM.
template <bool CPLX, int MODEL, int MODE, int NT = HAM_NT, bool SMT = false>
__global__ void __launch_bounds__(NT) k_local_energy(const HamArgs a) {
  using T = Traits<CPLX>;
  using S = typename T::S;
  extern __shared__ __align__(16) unsigned char smem_hm[];
  const int h = a.hidden, ns = a.ns, M = 2 * ns;
  S* th = reinterpret_cast<S*>(smem_hm);  // [h] theta_j(x)
  S* fp = th + h;                         // [h] RBM P_j / MLP tanh theta_j
  S* fq = fp + h;                         // [h] RBM Q_j
  // SMT: [M][h + 1][2] exp table, 16-B aligned for the paired loads
  S* ex_s = reinterpret_cast<S*>(smem_hm + ((3 * (size_t)h * sizeof(S) + 15) & ~(size_t)15));
  __shared__ int occ_l[4][32];            // occ up, vir up, occ down, vir down
  __shared__ int cnt_l[4];
  __shared__ int occ_all[64];
  __shared__ int n_occ_all;
  __shared__ unsigned short pairs[4][HAM_MAXPAIR];
  __shared__ S red[NT / 32];
  __shared__ int64_t scan[NT];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ex_ld = SMT ? h + 1 : h;  // table row stride (entries)
  if constexpr (SMT) {
    const S* src = reinterpret_cast<const S*>(a.EX);
    for (int64_t e = tid; e < (int64_t)M * h; e += NT) {
      const int row = (int)(e / h), j = (int)(e % h);
      ex_s[2 * ((int64_t)row * ex_ld + j)] = src[2 * e];
      ex_s[2 * ((int64_t)row * ex_ld + j) + 1] = src[2 * e + 1];
    }
  }

  for (int64_t r = blockIdx.x; r < a.n; r += gridDim.x) {
    const uint64_t x = a.xbits[r];
    __syncthreads();  // smem reuse across samples
    if (tid < 4) {
      // tid 0: occ up, 1: vir up, 2: occ down, 3: vir down
      const int base = (tid < 2) ? 0 : ns;
      const bool want = (tid & 1) == 0;
      int c = 0;
      for (int i = 0; i < ns; ++i)
        if ((((x >> (base + i)) & 1ull) != 0) == want) occ_l[tid][c++] = base + i;
      cnt_l[tid] = c;
      int k = 0;
      for (int p = 0; p < c; ++p)
        for (int q = p + 1; q < c; ++q) pairs[tid][k++] = (unsigned short)(p | (q << 8));
    } else if (tid == 4) {
      int c = 0;
      for (int i = 0; i < M; ++i)
        if ((x >> i) & 1ull) occ_all[c++] = i;
      n_occ_all = c;
    }
    // theta_j(x) and the ratio factors
    const S* WT = reinterpret_cast<const S*>(a.WT);
    for (int j = tid; j < (MODEL == MODEL_NONE ? 0 : h); j += NT) {
      S acc = reinterpret_cast<const S*>(a.bvec)[j];
      uint64_t bits = x;
      while (bits) {
        const int i = __ffsll((long long)bits) - 1;
        bits &= bits - 1;
        acc = T::add(acc, WT[(int64_t)i * h + j]);
      }
      th[j] = acc;
      if constexpr (CPLX) {
        const double2 t = ctanh(acc);
        fp[j] = make_double2(0.5 * (1.0 + t.x), 0.5 * t.y);
        fq[j] = make_double2(0.5 * (1.0 - t.x), -0.5 * t.y);
      } else if constexpr (MODEL == MODEL_RBM) {
        const double t = tanh(acc);
        fp[j] = 0.5 * (1.0 + t);
        fq[j] = 0.5 * (1.0 - t);
      } else {
        fp[j] = tanh(acc);
      }
    }
    __syncthreads();
    const int nou = cnt_l[0], nvu = cnt_l[1], nod = cnt_l[2], nvd = cnt_l[3];
    const int64_t S_u = (int64_t)nou * nvu, S_d = (int64_t)nod * nvd;
    const int64_t D_u = (int64_t)(nou * (nou - 1) / 2) * (nvu * (nvu - 1) / 2);
    const int64_t D_d = (int64_t)(nod * (nod - 1) / 2) * (nvd * (nvd - 1) / 2);
    const int64_t D_o = (int64_t)nou * nod * nvu * nvd;
    const int64_t Tot = S_u + S_d + D_u + D_d + D_o;
    const int64_t lo = Tot * tid / NT, hi = Tot * (tid + 1) / NT;
    const double* g = a.g2;
    auto G = [&](int p, int q, int s, int t) { return __ldg(g + (((int64_t)p * ns + q) * ns + s) * ns + t); };

    // candidate idx -> (holes m < n, particles p < q; n = q = -1 for singles)
    auto decode = [&](int64_t idx, int& m, int& n, int& p, int& q) {
      n = q = -1;
      if (idx < S_u) {
        m = occ_l[0][idx / nvu];
        p = occ_l[1][idx % nvu];
        return;
      }
      idx -= S_u;
      if (idx < S_d) {
        m = occ_l[2][idx / nvd];
        p = occ_l[3][idx % nvd];
        return;
      }
      idx -= S_d;
      for (int sp = 0; sp < 2; ++sp) {
        const int64_t D = sp == 0 ? D_u : D_d;
        if (idx < D) {
          const int nv = cnt_l[2 * sp + 1];
          const int64_t npv = nv * (nv - 1) / 2;
          const unsigned short ph = pairs[2 * sp][idx / npv], pp = pairs[2 * sp + 1][idx % npv];
          m = occ_l[2 * sp][ph & 0xff];
          n = occ_l[2 * sp][ph >> 8];
          p = occ_l[2 * sp + 1][pp & 0xff];
          q = occ_l[2 * sp + 1][pp >> 8];
          return;
        }
        idx -= D;
      }
      // opposite-spin double: (hu, hd) -> (pu, pd); idx = ((hu * nod + hd) * nvu + pu) * nvd + pd
      const int pd = (int)(idx % nvd);
      idx /= nvd;
      const int pu = (int)(idx % nvu);
      idx /= nvu;
      const int hd = (int)(idx % nod);
      const int hu = (int)(idx / nod);
      m = occ_l[0][hu];
      n = occ_l[2][hd];
      p = occ_l[1][pu];
      q = occ_l[3][pd];
    };
    // Slater-Condon element <y|H|x> (ham:203-235) with the fermionic sign
    auto element = [&](int m, int n, int p, int q) -> double {
      const int sm = ham_spatial(m, ns), sp = ham_spatial(p, ns);
      if (n < 0) {
        double val = __ldg(a.h1 + sm * ns + sp);
        const int no = n_occ_all;
        for (int k = 0; k < no; ++k) {
          const int j = occ_all[k];
          if (j == m) continue;
          const int sj = ham_spatial(j, ns);
          val += G(sm, sp, sj, sj);
          if (ham_same(m, j, ns)) val -= G(sm, sj, sj, sp);
        }
        return ham_move_sign(x, m, p) * val;
      }
      const int sn = ham_spatial(n, ns), sq = ham_spatial(q, ns);
      const double direct = (ham_same(m, p, ns) && ham_same(n, q, ns)) ? G(sm, sp, sn, sq) : 0.0;
      const double cross = (ham_same(m, q, ns) && ham_same(n, p, ns)) ? G(sm, sq, sn, sp) : 0.0;
      const uint64_t x1 = (x & ~(1ull << m)) | (1ull << p);
      return ham_move_sign(x, m, p) * ham_move_sign(x1, n, q) * (direct - cross);
    };
    // psi(y) / psi(x) for the excitation (m, n) -> (p, q)
    auto ratio = [&](int m, int n, int p, int q) -> S {
      if constexpr (MODEL == MODEL_NONE) {
        S one;
        if constexpr (CPLX) one = make_double2(1.0, 0.0); else one = 1.0;
        return one;
      }
      const S* wm = WT + (int64_t)m * h;
      const S* wp = WT + (int64_t)p * h;
      const S* wn = n >= 0 ? WT + (int64_t)n * h : nullptr;
      const S* wq = n >= 0 ? WT + (int64_t)q * h : nullptr;
      if constexpr (MODEL == MODEL_RBM) {
        // e^{D_j} = e^{W_jp} e^{W_jq} e^{-W_jm} e^{-W_jn} from the exp table: no exp, no
        // division; {e^{W}, e^{-W}} of one (orbital, unit) share a 16-B (32-B complex) entry
        const S* EX = SMT ? ex_s : reinterpret_cast<const S*>(a.EX);  // [M][ex_ld][2]
        const S* av = reinterpret_cast<const S*>(a.avec);
        S lin = T::sub(av[p], av[m]);
        if (n >= 0) lin = T::add(lin, T::sub(av[q], av[n]));
        S prod;
        if constexpr (CPLX) prod = make_double2(1.0, 0.0); else prod = 1.0;
        const S* tp = EX + (int64_t)p * ex_ld * 2;
        const S* tm = EX + (int64_t)m * ex_ld * 2;
        auto ld2 = [](const S* t, int j, S& plus, S& minus) {
          if constexpr (CPLX) {
            plus = SMT ? t[2 * j] : __ldg(t + 2 * j);
            minus = SMT ? t[2 * j + 1] : __ldg(t + 2 * j + 1);
          } else {
            const double2 v = SMT ? reinterpret_cast<const double2*>(t)[j] : __ldg(reinterpret_cast<const double2*>(t) + j);
            plus = v.x;
            minus = v.y;
          }
        };
        if (n < 0) {
          for (int j = 0; j < h; ++j) {
            S pp, ip, pm, im;
            ld2(tp, j, pp, ip);
            ld2(tm, j, im, pm);
            const S e = T::mul(pp, pm), ei = T::mul(ip, im);
            prod = T::mul(prod, T::add(T::mul(fp[j], e), T::mul(fq[j], ei)));
          }
        } else {
          const S* tq = EX + (int64_t)q * ex_ld * 2;
          const S* tn = EX + (int64_t)n * ex_ld * 2;
          for (int j = 0; j < h; ++j) {
            S pp, ip, pm, im, pq, iq, pn, in_;
            ld2(tp, j, pp, ip);
            ld2(tm, j, im, pm);
            ld2(tq, j, pq, iq);
            ld2(tn, j, in_, pn);
            const S e = T::mul(T::mul(pp, pm), T::mul(pq, pn));
            const S ei = T::mul(T::mul(ip, im), T::mul(iq, in_));
            prod = T::mul(prod, T::add(T::mul(fp[j], e), T::mul(fq[j], ei)));
          }
        }
        return T::mul(ham_exp<CPLX>(lin), prod);
      } else {
        double sum = 0.0;
        for (int j = 0; j < h; ++j) {
          double d = __ldg(wp + j) - __ldg(wm + j);
          if (n >= 0) d += __ldg(wq + j) - __ldg(wn + j);
          sum = fma(a.uvec[j], tanh(th[j] + d) - fp[j], sum);
        }
        return exp(sum);
      }
    };

    // diagonal element <x|H|x> (ham:190-201)
    auto diag_element = [&]() -> double {
      double val = a.e_core;
      const int no = n_occ_all;
      for (int k = 0; k < no; ++k) {
        const int i = occ_all[k], si = ham_spatial(i, ns);
        val += __ldg(a.h1 + si * ns + si);
      }
      for (int k = 0; k < no; ++k) {
        const int i = occ_all[k], si = ham_spatial(i, ns);
        for (int l = k + 1; l < no; ++l) {
          const int j = occ_all[l], sj = ham_spatial(j, ns);
          val += G(si, si, sj, sj);
          if (ham_same(i, j, ns)) val -= G(si, sj, sj, si);
        }
      }
      return val;
    };

    if constexpr (MODE == HAM_ELOC) {
      // strided: neighbouring lanes share holes and walk the particles, so
      // their table rows coincide or sit close in L1
      S acc = T::zero();
      for (int64_t idx = tid; idx < Tot; idx += NT) {
        int m, n, p, q;
        decode(idx, m, n, p, q);
        const double el = element(m, n, p, q);
        if (fabs(el) <= a.drop) continue;
        const S rt = ratio(m, n, p, q);
        if constexpr (CPLX) acc = make_double2(fma(el, rt.x, acc.x), fma(el, rt.y, acc.y)); else acc = fma(el, rt, acc);
      }
      if (tid == 0) {
        const double val = diag_element();  // ratio 1
        if constexpr (CPLX) acc.x += val; else acc += val;
      }
      acc = warp_sum<CPLX>(acc);
      if (lane == 0) red[warp] = acc;
      __syncthreads();
      if (tid == 0) {
        S e = red[0];
        for (int w = 1; w < NT / 32; ++w) e = T::add(e, red[w]);
        reinterpret_cast<S*>(a.out)[r] = e;
      }
    } else {
      int64_t kept = 0;
      for (int64_t idx = lo; idx < hi; ++idx) {
        int m, n, p, q;
        decode(idx, m, n, p, q);
        if (fabs(element(m, n, p, q)) > a.drop) ++kept;
      }
      if constexpr (MODE == HAM_COUNT) {
        scan[tid] = kept;
        __syncthreads();
        if (tid == 0) {
          int64_t s = 0;
          for (int t = 0; t < NT; ++t) s += scan[t];
          a.counts[r] = s;
          if (a.diag) a.diag[r] = diag_element();
        }
      } else {
        scan[tid] = kept;
        __syncthreads();
        if (tid == 0) {
          int64_t s = 0;
          for (int t = 0; t < NT; ++t) {
            const int64_t c = scan[t];
            scan[t] = s;
            s += c;
          }
        }
        __syncthreads();
        int64_t pos = a.offsets[r] + scan[tid];
        for (int64_t idx = lo; idx < hi; ++idx) {
          int m, n, p, q;
          decode(idx, m, n, p, q);
          const double el = element(m, n, p, q);
          if (fabs(el) <= a.drop) continue;
          const S rt = ratio(m, n, p, q);
          uint64_t y = (x & ~(1ull << m)) | (1ull << p);
          if (n >= 0) y = (y & ~(1ull << n)) | (1ull << q);
          a.pbits[pos] = y;
          a.pelem[pos] = el;
          S c;
          if constexpr (CPLX) c = make_double2(el * rt.x, el * rt.y); else c = el * rt;
          reinterpret_cast<S*>(a.pcoeff)[pos] = c;
          ++pos;
        }
      }
    }
  }
}

// W (h x M, row-major) -> WT (M x h) and, for the RBM ratio, EX = {exp(W^T), exp(-W^T)}
template <bool CPLX>
__global__ void k_transpose_w(const typename Traits<CPLX>::S* __restrict__ W, int h, int M,
                              typename Traits<CPLX>::S* __restrict__ WT, typename Traits<CPLX>::S* __restrict__ EX) {
  using S = typename Traits<CPLX>::S;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)h * M) return;
  const int j = (int)(e / M), i = (int)(e % M);
  const S w = W[e];
  const int64_t o = (int64_t)i * h + j;
  WT[o] = w;
  if (EX) {
    EX[2 * o] = ham_exp<CPLX>(w);
    if constexpr (CPLX) EX[2 * o + 1] = ham_exp<CPLX>(make_double2(-w.x, -w.y)); else EX[2 * o + 1] = ham_exp<CPLX>(-w);
  }
}

}  // namespace irl
