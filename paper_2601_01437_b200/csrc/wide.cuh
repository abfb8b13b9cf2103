// Single-HBM-read product for very wide rows (cfg4: 470 KB rows, cfg5: 1.67 MB).
//
// The fused cluster kernel (stream.cuh) splits a row over at most a few CTAs
// of one cluster, and its per-row DSMEM exchange stops paying beyond C = 2; the
// two-pass path reads O twice from HBM.  Here the whole GPU works on every
// row at once: one persistent, cooperatively launched grid with one CTA per SM.
//
//   * CTA c owns the column slice c of EVERY row (G = #SMs slices), so its
//     slice of the output lives in registers for the whole product and needs
//     no cross-CTA reduction at all.
//   * Rows go in blocks of RS rows; a block is one stage of a shared-memory
//     ring (TMA bulk copies, one per row slice).  O is read from HBM exactly
//     once and never re-read (not even from L2): between its dot and its
//     accumulate a block waits for the grid-wide exchange of its row dots, and
//     during that wait it is parked in TENSOR MEMORY -- each consumer warp
//     moves its part of the block from shared memory to registers for the dot
//     and from there to its TMEM columns (tcgen05.st), and frees the stage at
//     once.  Shared memory then only has to cover the HBM latency and the
//     256 KB of TMEM cover the exchange latency: a 1-CTA-per-SM stream needs
//     about (HBM latency + exchange latency) x 45 GB/s in flight, more than
//     the 227 KB of shared memory alone.
//   * Only the per-row dots cross CTAs.  Every exchanged value travels as a
//     self-validating "LL" record: each 32-bit half of a double shares a 64-bit
//     word with a 32-bit tag (block + 1), and aligned 64-bit accesses are
//     single-copy atomic, so a reader that sees the tag sees the data -- no
//     fences, no counters, no atomics on the hot path.  The records are zeroed
//     before every launch, so a stale tag can never match.
//
// Exchange of block b (RS rows):
//   publish    every CTA writes its RS partial dots (minus its share of
//              Obar.v) to part[b % NBUF][row][c];
//   aggregate  CTA r % G polls the G partials of row r, sums them in a
//              fixed order (the same order whichever CTA aggregates) and
//              writes t_r to fin[copy][b % NBUF][row], WIDE_FIN_COPIES replicas
//              (every CTA polls the totals: one copy is an L2 hot spot);
//   reduce     every CTA polls its replica (c % copies), forms
//              y_row = c_row t_row (+ yadd) -- bit-identical in every CTA --
//              and accumulates with it.
//
// Warp roles (one CTA, WIDE_THREADS threads):
//   dot warps (WIDE_CW)        warp w owns rows (w / Q) RPW ... + RPW - 1 of a
//       stage, part w % Q of the slice (RS = RPW WIDE_CW / Q rows per block;
//       several rows per warp-step hide the step's latencies).  D(b): wait for
//       slot b % K to be free and for the stage; part -> registers -> partial
//       dots -> smem, arrive dotdone (published at once); part -> TMEM slot,
//       arrive empty (the stage refills); wait::st, arrive parked.
//   accumulate warps (WIDE_CW) warp w + WIDE_CW shares warp w's place and TMEM
//       columns (same warp % 4 = TMEM lane quarter).  A(b): wait parked,
//       part back from TMEM into registers, arrive slotfree (the slot is free
//       before y arrives: the window is K blocks in TMEM plus this one), wait
//       ydone, acc += conj(O) y.
//       A single warp doing D(b) and A(b - K) in turn was the bound of the CTA
//       (their dependent latencies add up per block); split, every wait is a
//       blocking mbarrier wait on the one thing the warp needs next.
//   producer (1 warp)          lane 0 streams block after block into the ring.
//   publisher (1 warp)         sums the Q part dots of each row, writes part.
//   aggregators (WIDE_AW warps) the rows this CTA aggregates.
//   reducers (WIDE_RW warps)   block b (b = k mod RW): fin -> y -> smem,
//       arrive ydone; several warps keep several blocks' polls in flight.
//
// Slot reuse: a slot holds one pending block, so CTA X publishes block b only
// after its accumulate warps fetched b - K, i.e. after fin of b - K existed,
// i.e. after every CTA published b - K; a CTA publishes b - K only after it
// fetched b - 2 K, i.e. after its reducers finished every block <= b - 2 K.
// With NBUF >= 2 K + 2 no record is overwritten while some CTA may still read
// it; tags are unique within a launch.
//
// Replaces est:184-186 (centring copy + the two GEMVs) for stored O.
#pragma once
#include "stream.cuh"

namespace irl {

constexpr int WIDE_CW = 8;  // dot warps, and as many accumulate warps (warp w + WIDE_CW takes what warp w parked)
constexpr int WIDE_AW = 3;  // aggregator warps
constexpr int WIDE_RW = 3;  // reducer warps
constexpr int WIDE_THREADS = (2 * WIDE_CW + 2 + WIDE_AW + WIDE_RW) * 32;
// Registers: the CTA launches at WIDE_REGS_LAUNCH per thread; then the dot and
// accumulate warpgroups grow and the other roles shrink (setmaxnreg, issued
// inside each role's branch so that ptxas allocates per role).  The pool is
// the launch allocation: asking for more than the others gave back never returns.
constexpr int WIDE_REGS_LAUNCH = (65536 / WIDE_THREADS) / 8 * 8;
constexpr int WIDE_REGS_DOT = 88;
constexpr int WIDE_REGS_ACC = 104;
constexpr int WIDE_REGS_AUX = 48;
static_assert(WIDE_CW % 4 == 0 && (WIDE_THREADS / 32) % 4 == 0, "setmaxnreg works on whole warpgroups");
static_assert(WIDE_CW * 32 * (WIDE_REGS_DOT + WIDE_REGS_ACC) + (WIDE_THREADS - 2 * WIDE_CW * 32) * WIDE_REGS_AUX <=
                  WIDE_THREADS * WIDE_REGS_LAUNCH,
              "setmaxnreg.inc can only take what the CTA's own warps gave back");
#define WIDE_SET_REGS(op, n) asm volatile("setmaxnreg." op ".sync.aligned.u32 %0;" ::"n"(n))
constexpr int WIDE_MAX_NS = 24;  // shared-memory stages
constexpr int WIDE_MAX_K = 24;   // blocks parked in TMEM per consumer warp (pending exchange)
constexpr int WIDE_NBUF = 64;    // exchange record ring (>= 2 K + 2)
static_assert(WIDE_NBUF >= 2 * (WIDE_MAX_K + 1) + 2, "exchange ring too short for the deepest pending window");
constexpr int WIDE_QPL = 2;  // partials per aggregator lane: 2 * 32 * WIDE_AW >= G
static_assert(WIDE_QPL * 32 * WIDE_AW >= 160, "aggregator lanes must cover every SM");
constexpr int WIDE_MAX_RS = 32;  // rows per block: one reducer lane each
constexpr int WIDE_FIN_COPIES = 16;  // replicas of the row totals (every CTA polls them: one copy is an L2 hot spot)
constexpr int WIDE_TMEM_COLS = 512;  // whole TMEM: one CTA per SM
// TMEM words (32-bit columns) one consumer lane parks per block: UPL 16-byte units
__host__ __device__ constexpr int wide_tm_words(int upl) { return 4 * upl; }
// consumer warps w and w + 4 share a 32-lane quarter of TMEM, so each owns half the columns
constexpr int WIDE_TM_COLS_PER_WARP = WIDE_TMEM_COLS / (WIDE_CW / 4);

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
  ulonglong2* part;  // LL records [NBUF][RS][G][S doubles]   (zeroed per launch)
  ulonglong2* fin;   // LL records [copies][NBUF][RS][S doubles]   (zeroed per launch)
  int fin_copies;    // replicas of fin written by the aggregator; CTA c polls copy c % fin_copies
  size_t fin_stride;  // records between replicas
  ulonglong2* gpart;  // LL records [G]: each slice's (F/2) . v share   (zeroed per launch)
  int RS;            // rows per block (= per stage), WIDE_CW / Q
  int Q;             // parts per row slice
  int PU;            // units per part (ceil(WM / Q))
  int NS;            // ring stages
  int K;             // TMEM slots per dot / accumulate warp pair (blocks in flight between dot and accumulate)
  int UT;            // a lane's first UT units of a row part go to TMEM ...
  int PR;            // ... and the PR units of the partly filled last lane-row (units 32 UT ..) to a side buffer in
  size_t side_off;   // shared memory [K][RS][Q][PR]: TMEM columns are not spent on empty lanes (cfg4: 100 units a
                     // part = 3 full lane-rows + 4 units; K = 5 instead of 4)
  int WM;            // max slice width (units): ring row pitch
  size_t ring_bytes;  // ring + epilogue scratch (>= both)
  size_t vsl_off;     // shared-memory offset of the v slice
  unsigned long long* trace;  // debug (IRL_WIDE_TRACE): [G][WIDE_TRACE_B][8] globaltimer stamps; null = off
  int trace_stride;           // every trace_stride-th block is stamped
  int poll_ns;                // reducer / aggregator poll back-off (ns)
  int rot;                    // debug: CTA c takes column slice (c + rot) % G
  int red_delay_ns;           // reducers: pause between this CTA's own publish and the first poll of the totals
  int agg_delay_ns;           // aggregators: the same before the first poll of a row's partials
};

constexpr int WIDE_TRACE_B = 512;  // traced blocks per CTA
constexpr uint32_t WIDE_GPART_TAG = 0xffffffffu;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define WIDE_STAMP(b, k)                                                                      \
  do {                                                                                        \
    if (a.trace && ((b) % a.trace_stride) == 0 && (b) / a.trace_stride < WIDE_TRACE_B)        \
      a.trace[((size_t)c * WIDE_TRACE_B + (b) / a.trace_stride) * 8 + (k)] = gtimer();        \
  } while (0)

// ------------------------------------------------------------- LL records --
__device__ __forceinline__ void st_ll(ulonglong2* p, double d, uint32_t tag) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(d);
  const unsigned long long t = (unsigned long long)tag << 32;
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(t | (u & 0xffffffffull)),
               "l"(t | (u >> 32))
               : "memory");
}
// returns true (and the value) when both halves carry `tag`
__device__ __forceinline__ bool ld_ll(const ulonglong2* p, uint32_t tag, double& d) {
  unsigned long long lo, hi;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(p) : "memory");
  d = __longlong_as_double((long long)((hi << 32) | (lo & 0xffffffffull)));
  return (uint32_t)(lo >> 32) == tag && (uint32_t)(hi >> 32) == tag;
}
template <bool CPLX>
__device__ __forceinline__ void st_ll_s(ulonglong2* p, typename Traits<CPLX>::S v, uint32_t tag) {
  if constexpr (CPLX) {
    st_ll(p, v.x, tag);
    st_ll(p + 1, v.y, tag);
  } else {
    st_ll(p, v, tag);
  }
}
template <bool CPLX>
__device__ __forceinline__ bool ld_ll_s(const ulonglong2* p, uint32_t tag, typename Traits<CPLX>::S& v) {
  if constexpr (CPLX) {
    const bool a = ld_ll(p, tag, v.x);
    const bool b = ld_ll(p + 1, tag, v.y);
    return a && b;
  } else {
    return ld_ll(p, tag, v);
  }
}

// ------------------------------------------------------------------ TMEM --
// 32x32b shapes: thread t of the warp moves 32-bit words to / from TMEM lane
// (lane quarter base + t), consecutive columns.
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// One 16-byte unit per TMEM access: the four words are the registers an
// LDS.128 delivered (wider accesses cost register shuffles and measured slower).
__device__ __forceinline__ void tm_st4(uint32_t ta, int4 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ta), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void tm_ld4(uint32_t ta, int4& v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(ta)
               : "memory");
}
__device__ __forceinline__ double2 unit_of(int4 w) {
  return make_double2(__hiloint2double(w.y, w.x), __hiloint2double(w.w, w.z));
}
// park UPL units (4 UPL words) of one lane
template <int UPL>
__device__ __forceinline__ void tm_park(uint32_t ta, const int4 (&x)[UPL]) {
#pragma unroll
  for (int k = 0; k < UPL; ++k) tm_st4(ta + 4 * k, x[k]);
}

// Sum NV values per lane over the warp with the fewest shuffles: while more
// than one value is left, the lanes of a butterfly pair split them (one keeps
// the lower half, its partner the upper half, each adds what the other sent),
// then plain butterflies.  Lane l ends with the warp total of value
// l / (32 / NV) in v[0]; the order of the additions is fixed.
template <int NV>
__device__ __forceinline__ void warp_sum_split(double (&v)[NV], int lane) {
  static_assert(NV == 1 || NV == 2 || NV == 4 || NV == 8 || NV == 16, "power of two");
  int n = NV;
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    if (n > 1) {
      n >>= 1;
      const bool up = (lane & m) != 0;
#pragma unroll
      for (int i = 0; i < NV / 2; ++i) {
        if (i < n) {
          const double send = up ? v[i] : v[i + n];
          const double keep = up ? v[i + n] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
        }
      }
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], m);
    }
  }
}

// SIDE: the last lane-row of a part (k = UPL - 1) is only partly filled and
// waits in the shared-memory side buffer; TMEM takes the UT = UPL - 1 full ones.
template <bool CPLX, int UPL, int RPW, bool SIDE = false>
__global__ void __launch_bounds__(WIDE_THREADS, 1) k_wide(const WideArgs a) {
  using T = Traits<CPLX>;
  using S = typename T::S;
  constexpr int SW = CPLX ? 2 : 1;  // LL records per scalar
  constexpr int UT = SIDE ? UPL - 1 : UPL;
  const int PR = a.PR;
  constexpr int TMW = RPW * 4 * UT;  // TMEM words a lane parks per block
  constexpr int SC = CPLX ? 2 : 1;               // doubles per scalar
  constexpr int NV = RPW * SC;                   // doubles a lane reduces per warp-step
  constexpr int RB = UPL >= 8 ? 1 : (RPW * UPL <= 16 ? RPW : (RPW >= 2 && (RPW / 2) * UPL <= 16 ? RPW / 2 : 1));  // rows per TMEM fetch
  extern __shared__ __align__(16) unsigned char smem_w[];
  const int NS = a.NS, K = a.K, WM = a.WM, RS = a.RS, Q = a.Q, PU = a.PU;
  double2* ring = reinterpret_cast<double2*>(smem_w);                    // [NS][RS][WM]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_w + a.ring_bytes);  // [NS]
  uint64_t* empty = full + NS;                                           // [NS]
  uint64_t* dotdone = empty + NS;                                        // [K]
  // y of the rows has one slot more than the pending ring: an accumulate warp fetches block b into registers as
  // soon as it is parked and frees its slot, so block b + K may get its y while block b still waits for its own
  const int KY = K + 1;
  uint64_t* ydone = dotdone + K;                                         // [KY]
  uint64_t* parked = ydone + KY + 1;                                     // [K] (+ 1: pd stays 16-byte aligned) block b is in TMEM
  uint64_t* slotfree = parked + K;                                       // [K] block b left TMEM (accumulate warps -> dot warps)
  S* pd = reinterpret_cast<S*>(slotfree + K);                            // [K][RS][Q] part dots
  S* ys = pd + (size_t)K * RS * Q;                                       // [KY][RS] y of the rows
  double2* vsl = reinterpret_cast<double2*>(a.vsl_off + smem_w);         // [WM + 1] v slice (+ a zero unit)
  double2* side = reinterpret_cast<double2*>(a.side_off + smem_w);       // [K][RS][Q][PR] last lane-rows of pending blocks
  __shared__ S shs[WIDE_CW];
  __shared__ double shg[WIDE_CW];
  __shared__ S shy[WIDE_RW];
  __shared__ S shagg[WIDE_AW];
  __shared__ S s_c_sh;
  __shared__ volatile int published;  // blocks this CTA has published (paces its aggregator)
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, c = blockIdx.x;
  const int64_t N = a.n_rows;
  const int sl = (c + a.rot) % G;  // column slice of this CTA
  const int64_t col0 = slice_lo(a.ld_u, G, sl);
  const int W = (int)(slice_lo(a.ld_u, G, sl + 1) - col0);
  const int NB = (int)((N + RS - 1) / RS);
  const S* coeff = reinterpret_cast<const S*>(a.coeff);
  const S* yadd = reinterpret_cast<const S*>(a.yadd);
  constexpr int W_ACC = WIDE_CW, W_PROD = 2 * WIDE_CW, W_PUB = W_PROD + 1, W_AGG = W_PROD + 2, W_RED = W_AGG + WIDE_AW;
  constexpr int NTC = WIDE_CW * 32;

  if (tid == 0) {
    if (a.trace) {
      unsigned int smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      a.trace[(size_t)c * WIDE_TRACE_B * 8 + 7] = smid;
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], WIDE_CW);
    }
    for (int j = 0; j < K; ++j) {
      mbar_init(&dotdone[j], WIDE_CW);
      mbar_init(&parked[j], WIDE_CW);
      mbar_init(&slotfree[j], WIDE_CW);
    }
    for (int j = 0; j <= K; ++j) mbar_init(&ydone[j], 1);
    published = 0;
    fence_mbar_init();
  }
  if (warp == 0) {  // the whole TMEM (one CTA per SM); warp 0 also frees it
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_base_sh)),
                 "n"(WIDE_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }

  // prologue (consumer warps): the v slice, this slice's shares of Obar . v and (F/2) . v
  if (warp < WIDE_CW) {
    for (int u = W + tid; u <= WM; u += NTC) vsl[u] = make_double2(0.0, 0.0);  // past the slice: 0
    S sp = T::zero();
    double gp = 0.0;
    for (int u = tid; u < W; u += NTC) {
      const double2 v = load_vec_unit<CPLX>(a.v_re, a.v_im, col0 + u);
      vsl[u] = v;
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
    named_bar_sync(1, NTC);
    if (tid == 0) {
      S s_c = T::zero();
      double g_c = 0.0;
      for (int w = 0; w < WIDE_CW; ++w) {
        s_c = T::add(s_c, shs[w]);
        g_c += shg[w];
      }
      s_c_sh = s_c;
      st_ll(a.gpart + c, g_c, WIDE_GPART_TAG);  // read by CTA 0 at the end
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // ------------------------------------------------------------ producer --
  if (warp == W_PROD) {
    WIDE_SET_REGS("dec", WIDE_REGS_AUX);
    if (lane == 0) {
      const uint32_t slice_bytes = (uint32_t)W * 16u;
      for (int b = 0; b < NB; ++b) {
        const int s = b % NS;
        if (b >= NS) mbar_wait(&empty[s], ((b / NS) & 1) ^ 1);
        const int64_t r0 = (int64_t)b * RS;
        const int rows = (int)min((int64_t)RS, N - r0);
        WIDE_STAMP(b, 0);
        mbar_arrive_expect_tx(&full[s], slice_bytes * (uint32_t)rows);
        for (int i = 0; i < rows; ++i)
          bulk_g2s(ring + ((size_t)s * RS + i) * WM, a.O + (r0 + i) * a.ld_u + col0, slice_bytes, &full[s]);
      }
    }
    return;
  }

  // ----------------------------------------------------------- publisher --
  if (warp == W_PUB) {
    WIDE_SET_REGS("dec", WIDE_REGS_AUX);
    const S s_c = s_c_sh;
    for (int b = 0; b < NB; ++b) {
      const int j = b % K;
      mbar_wait(&dotdone[j], (b / K) & 1);
      if (lane < RS) {
        S t = T::zero();
        for (int q = 0; q < Q; ++q) t = T::add(t, pd[(j * RS + lane) * Q + q]);
        st_ll_s<CPLX>(a.part + (((size_t)(b % WIDE_NBUF) * RS + lane) * G + c) * SW, T::sub(t, s_c), (uint32_t)b + 1);
      }
      __syncwarp();
      if (lane == 0) {
        published = b + 1;
        WIDE_STAMP(b, 2);
      }
    }
    return;
  }

  // --------------------------------------------------------- aggregators --
  // row r of the matrix is aggregated by CTA r % G: one row's G partials per
  // visit, two per aggregator lane
  if (warp >= W_AGG && warp < W_RED) {
    WIDE_SET_REGS("dec", WIDE_REGS_AUX);
    constexpr int AL = WIDE_AW * 32;            // aggregator lanes
    const int al = (warp - W_AGG) * 32 + lane;  // partials al, al + AL
    for (int64_t r = c; r < N; r += G) {
      const int b = (int)(r / RS), i = (int)(r - (int64_t)b * RS);
      // pace: start once this CTA has published block b itself (the others are
      // close); a row comes up every ~G / RS blocks, so sleep long
      while (published <= b) __nanosleep(256);
      if (a.agg_delay_ns) __nanosleep(a.agg_delay_ns);
      const uint32_t tag = (uint32_t)b + 1;
      const ulonglong2* src = a.part + ((size_t)(b % WIDE_NBUF) * RS + i) * G * SW;
      S x[WIDE_QPL];
      uint32_t pending = 0;  // bit j: record al + AL j not seen yet
#pragma unroll
      for (int j = 0; j < WIDE_QPL; ++j) {
        x[j] = T::zero();
        if (al + AL * j < G) pending |= 1u << j;
      }
      while (true) {
#pragma unroll
        for (int j = 0; j < WIDE_QPL; ++j)
          if (pending & (1u << j))
            if (ld_ll_s<CPLX>(src + (size_t)(al + AL * j) * SW, tag, x[j])) pending &= ~(1u << j);
        if (__all_sync(0xffffffffu, pending == 0)) break;
        __nanosleep(a.poll_ns);
      }
      // fixed order: per lane j = 0, 1, ..., butterfly, then the aggregator warps in order
      S t = x[0];
#pragma unroll
      for (int j = 1; j < WIDE_QPL; ++j) t = T::add(t, x[j]);
      t = warp_sum<CPLX>(t);
      if (lane == 0) shagg[warp - W_AGG] = t;
      named_bar_sync(3, WIDE_AW * 32);
      if (warp == W_AGG && lane < a.fin_copies) {  // one replica per lane, the same total in each
        S tt = T::zero();
        for (int w = 0; w < WIDE_AW; ++w) tt = T::add(tt, shagg[w]);
        st_ll_s<CPLX>(a.fin + (size_t)lane * a.fin_stride + ((size_t)(b % WIDE_NBUF) * RS + i) * SW, tt, tag);
      }
      named_bar_sync(3, WIDE_AW * 32);  // shagg reused by the next row
    }
    return;
  }

  // ------------------------------------------------------------ reducers --
  if (warp >= W_RED) {
    WIDE_SET_REGS("dec", WIDE_REGS_AUX);
    const int k = warp - W_RED;
    S ysum = T::zero();
    for (int b = k; b < NB; b += WIDE_RW) {
      const int j = b % KY;  // slot of the y ring
      const int64_t r0 = (int64_t)b * RS;
      const int rows = (int)min((int64_t)RS, N - r0);
      const uint32_t tag = (uint32_t)b + 1;
      // the row's coefficient loads while the exchange completes
      const S cf = (lane < rows) ? coeff[r0 + lane] : T::zero();
      const S ya = (yadd && lane < rows) ? yadd[r0 + lane] : T::zero();
      const ulonglong2* src = a.fin + (size_t)(c % a.fin_copies) * a.fin_stride + ((size_t)(b % WIDE_NBUF) * RS + lane) * SW;
      S t = T::zero();
      bool ok = lane >= rows;
      while (published <= b) __nanosleep(64);  // no total before this CTA's own share
      if (a.red_delay_ns) __nanosleep(a.red_delay_ns);
      const long long t0 = clock64();
      while (true) {
        if (!ok) ok = ld_ll_s<CPLX>(src, tag, t);
        if (__all_sync(0xffffffffu, ok)) break;
        if (clock64() - t0 > (1LL << 36)) __trap();  // ~30 s: a lost CTA; fail loudly, never hang
        __nanosleep(a.poll_ns);
      }
      if (lane == 0) WIDE_STAMP(b, 3);
      S y = T::mul(cf, t);
      if (yadd) y = T::add(y, ya);
      if (lane < rows) ys[j * RS + lane] = y;
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&ydone[j]);
        WIDE_STAMP(b, 4);
      }
      for (int i = 0; i < rows; ++i) ysum = T::add(ysum, T::shfl(y, i));  // row order (off the critical path)
    }
    if (lane == 0) shy[k] = ysum;
    named_bar_sync(2, (WIDE_CW + WIDE_RW) * 32);  // epilogue (accumulate warps): shy complete
    return;
  }

  // ------------------------------------------------- dot / accumulate warps --
  // Dot warp w and accumulate warp w + WIDE_CW own the same place: part
  // pq = w % Q of rows rg RPW .. rg RPW + RPW - 1 (rg = w / Q) of every block,
  // and the same TMEM columns (warp % 4 is the TMEM lane quarter of both).
  // A warp that did both steps of a block one after the other was the bound of
  // the CTA (~0.65 + 0.45 us of dependent latencies per block whatever the
  // rows per step); split, the block rate is that of the slower step.
  const int wi = warp % WIDE_CW;
  const int rg = wi / Q;
  const int pq = wi % Q;
  const int u0p = pq * PU;
  const int u1p = min(W, u0p + PU);
  static_assert(WIDE_CW % 4 == 0, "a warp's TMEM lane quarter is warp % 4");
  // this place's TMEM: lane quarter wi % 4, column half wi / 4, K slots of TMW words
  const uint32_t tm = tmem_base_sh + ((uint32_t)(32 * (wi & 3)) << 16) + (uint32_t)((wi >> 2) * WIDE_TM_COLS_PER_WARP);
  bool inpart[UPL];
#pragma unroll
  for (int k = 0; k < UPL; ++k) inpart[k] = u0p + lane + 32 * k < u1p;

  if (warp < W_ACC) {
    // ---- dot warps: stage -> registers -> partial dots (published at once) -> TMEM
    WIDE_SET_REGS("inc", WIDE_REGS_DOT);
    int sd = 0, pdp = 0, jd = 0, pk = 0;  // stage / parity, slot, parity of nd / K
    for (int nd = 0; nd < NB; ++nd) {
      const int s = sd, j = jd;
      if (nd >= K) mbar_wait(&slotfree[j], pk ^ 1);  // block nd - K left this slot (window of K pending blocks)
      if (wi == 0 && lane == 0) WIDE_STAMP(nd, 6);
      mbar_wait(&full[s], pdp);
      const int64_t r0 = (int64_t)nd * RS + rg * RPW;
      const int nlive = (int)min((int64_t)RPW, N - r0);
      double t[NV];
      // row by row: shared memory -> registers -> dot -> TMEM (the TMEM
      // stores are asynchronous, so the next row's loads overlap them)
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const int4* row = reinterpret_cast<const int4*>(ring + ((size_t)s * RS + rg * RPW + r) * WM + u0p + lane);
        const bool live = r < nlive;
        int4 x[UPL];  // the unit's four words as loaded: parked as they are
#pragma unroll
        for (int k = 0; k < UPL; ++k) x[k] = (live && inpart[k]) ? row[32 * k] : make_int4(0, 0, 0, 0);
        S t0 = T::zero(), t1 = T::zero();
#pragma unroll
        for (int k = 0; k < UPL; ++k)  // x = 0 past the part, so any finite v will do there
          T::dot_acc((k & 1) ? t1 : t0, unit_of(x[k]), vsl[min(u0p + lane + 32 * k, WM)]);
        const S tr = T::add(t0, t1);
        if constexpr (CPLX) {
          t[2 * r] = tr.x;
          t[2 * r + 1] = tr.y;
        } else {
          t[r] = tr;
        }
        if (live) {
          const uint32_t tr0 = tm + (uint32_t)(j * TMW + r * 4 * UT);
#pragma unroll
          for (int k = 0; k < UPL; ++k) {
            if (k < UT) {
              tm_st4(tr0 + 4 * k, x[k]);
            } else if (SIDE && k == UT && lane < PR) {
              reinterpret_cast<int4*>(side)[((size_t)(j * RS + rg * RPW + r) * Q + pq) * PR + lane] = x[k];
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // the stage is in registers / TMEM: refill it
      warp_sum_split<NV>(t, lane);            // lane l: the total of value l / (32 / NV)
      if ((lane & (32 / NV - 1)) == 0)
        reinterpret_cast<double*>(pd)[((j * RS + rg * RPW) * Q) * SC + ((lane / (32 / NV)) / SC * Q + pq) * SC +
                                      (lane / (32 / NV)) % SC] = t[0];
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&dotdone[j]);
        if (wi == 0) WIDE_STAMP(nd, 1);
      }
      // the park has landed: hand the slot to the accumulate warps
      tm_wait_st();
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&parked[j]);
      if (++sd == NS) {
        sd = 0;
        pdp ^= 1;
      }
      if (++jd == K) {
        jd = 0;
        pk ^= 1;
      }
    }
    // TMEM is no longer needed once the accumulate warps are done: warp 0 frees it
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    named_bar_sync(4, 2 * NTC);
    if (warp == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base_sh), "n"(WIDE_TMEM_COLS)
                   : "memory");
    }
    return;
  }

  // ---- accumulate warps: y and the parked block -> registers -> acc += conj(O) y
  WIDE_SET_REGS("inc", WIDE_REGS_ACC);
  double2 acc[UPL];
#pragma unroll
  for (int k = 0; k < UPL; ++k) acc[k] = make_double2(0.0, 0.0);
  {
    // EARLY (all the rows of a step fit one TMEM round trip): the block is fetched into registers as soon as it
    // is parked and its slot freed before its y arrives, so the window is K blocks in TMEM plus this one
    constexpr bool EARLY = RB == RPW;
    int ja = 0, pap = 0, jy = 0, py = 0;
    for (int na = 0; na < NB; ++na) {
      const int j = ja;
      if (!EARLY) mbar_wait(&ydone[jy], py);
      mbar_wait(&parked[j], pap);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t r0 = (int64_t)na * RS + rg * RPW;
      const int nlive = (int)min((int64_t)RPW, N - r0);  // rows of this warp that exist (<= 0: none)
      // RB rows per TMEM round trip: all their loads in flight, one wait
#pragma unroll
      for (int rb = 0; rb < RPW; rb += RB) {
        int4 w[RB][UPL];
        if (rb < nlive) {
#pragma unroll
          for (int r = 0; r < RB; ++r)
#pragma unroll
            for (int k = 0; k < UPL; ++k) {
              if (k < UT) {
                tm_ld4(tm + (uint32_t)(j * TMW + (rb + r) * 4 * UT + 4 * k), w[r][k]);
              } else {
                w[r][k] = (SIDE && k == UT && lane < PR)
                              ? reinterpret_cast<const int4*>(
                                    side)[((size_t)(j * RS + rg * RPW + rb + r) * Q + pq) * PR + lane]
                              : make_int4(0, 0, 0, 0);
              }
            }
          tm_wait_ld();
        }
        if (rb + RB >= RPW) {  // the slot's last rows are in registers: the dot warps may park block na + K
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&slotfree[j]);
          if (EARLY) mbar_wait(&ydone[jy], py);
        }
        if (rb < nlive) {
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            if (rb + r < nlive) {
              const S y = ys[jy * RS + rg * RPW + rb + r];
#pragma unroll
              for (int k = 0; k < UPL; ++k) T::axpy(acc[k], unit_of(w[r][k]), y);  // x = 0 past the part
            }
          }
        }
      }
      if (lane == 0 && wi == 0) WIDE_STAMP(na, 5);
      if (++ja == K) {
        ja = 0;
        pap ^= 1;
      }
      if (++jy == KY) {
        jy = 0;
        py ^= 1;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  named_bar_sync(4, 2 * NTC);  // with the dot warps: TMEM may go

  // the part accumulators of the RS warps sharing a part meet in shared memory
  // (the ring is free: every stage consumed), in row order
  named_bar_sync(2, (WIDE_CW + WIDE_RW) * 32);
  double2* red = ring;  // [CW][32 * UPL] (ring_bytes covers it)
  const int pitch = 32 * UPL;
  const int ta = tid - W_ACC * 32;  // thread index among the accumulate warps
#pragma unroll
  for (int k = 0; k < UPL; ++k) red[(size_t)wi * pitch + lane + 32 * k] = acc[k];
  S Y = T::zero();  // sum over all rows of y, the same fixed order in every CTA
  for (int k = 0; k < WIDE_RW; ++k) Y = T::add(Y, shy[k]);
  named_bar_sync(5, NTC);
  const double uu = (a.hf_re && a.u0) ? *a.u0 : 0.0;
  for (int u = ta; u < W; u += NTC) {
    const int q = u / PU, j = u - q * PU;
    double2 o = red[(size_t)q * pitch + j];
    for (int i = 1; i < WIDE_CW / Q; ++i) {  // the row groups sharing part q, in order
      const double2 x = red[(size_t)(i * Q + q) * pitch + j];
      o.x += x.x;
      o.y += x.y;
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
  if (a.out0 && c == 0 && wi == 0) {  // (F/2) . u over the slices, fixed order
    double g = 0.0;
    if (a.hf_re) {
      for (int q0 = 0; q0 < G; q0 += 32) {
        double x = 0.0;
        if (q0 + lane < G)
          while (!ld_ll(a.gpart + q0 + lane, WIDE_GPART_TAG, x)) __nanosleep(32);
        g += warp_sum<false>(x);
      }
    }
    if (lane == 0) *a.out0 = g;
  }
}

}  // namespace irl
