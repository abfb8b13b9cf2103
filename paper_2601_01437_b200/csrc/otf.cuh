// On-the-fly O regeneration for the shallow MLP (K6).
//
// O_n = [g_n (x) x_n (h x n_in, j-major), g_n (h), t_n (h), 1] is never stored.
// The centred product out = O_c^T (c (O_c v)) is regenerated from the 0/1
// inputs X (bit-packed), T = tanh(W x + b) and G = u (1 - T^2) as two FP64
// tensor-core GEMMs (mma.sync m8n8k4 f64, SASS DMMA) with fused epilogues:
//
//   k_otf_dot : A = X V_W^T (+ v_b)  ->  t_n = sum_j G_nj A_nj + T_nj v_u,j
//               (the N x h product is reduced with G/T in registers, never stored;
//                per-j-chunk row partials go to tpart)
//   k_otf_y   : y_n = c_n (sum_chunks tpart + v_c - Obar.v), fixed order
//   k_otf_acc : out_W = (G (.) y)^T X, out_b = (G (.) y)^T 1, out_u = (T (.) y)^T 1
//               (split over row blocks; partials reduced in k_otf_finish)
//
// With y = w or y = w (e - E) the same k_otf_acc yields Obar and the gradient
// (est:167, est:156-163) without ever materialising O.
#pragma once
#include "common.cuh"
#include "obuild.cuh"

namespace irl {

constexpr int OTF_BJ = 64;   // hidden units per CTA chunk
constexpr int OTF_BM = 64;   // rows per tile
constexpr int OTF_KC = 104;  // k columns of the acc GEMM: n_in (<=100) + ones column, padded to 13 n-tiles
constexpr int OTF_MAX_NIN = 100;
constexpr int OTF_XW = 2;    // 64-bit words per packed input row (n_in <= 128)
constexpr int OTF_ACC_STAGES = 3;  // TMA ring stages of the acc GEMMs
constexpr int OTF_DOT_STAGES = 2;  // TMA ring stages of the dot GEMMs (v_W also lives in shared memory)

struct OtfArgs {
  const uint64_t* xbits;  // [N][OTF_XW]
  const double* T;        // [N][h]
  const double* G;        // [N][h]
  int64_t n_rows;
  int n_in, hidden;
  int nb;                 // row blocks
  // parameter layout offsets (elements of v): W block, b, u (-1: none, RBM)
  int64_t offW, offb, offu;
  // dot
  const double* v;        // padded parameter vector
  double* tpart;          // [JC][N]
  // acc
  const double* y;        // [N]
  const double* y2;       // [N] second weight vector (NY = 2)
  double* part;           // [NY][nb][h][KC]
  double* partu;          // [NY][nb][h]
  // MLP only: output weights u (length h).  Non-null: G = u (1 - T^2) is formed
  // from the T tile in registers and G is never read (half the activation
  // traffic; the on-the-fly MLP product at small n_in is HBM-bound on T and G)
  const double* u;
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Programmatic dependent launch: the product chain (vdot -> dot -> y -> acc ->
// xsum -> finish) is launched with programmatic stream serialisation, so a
// kernel's CTAs are set up while its predecessor drains.  Every kernel of the
// chain waits for its predecessor's completion (and memory) before touching
// global memory and lets its own successor launch right away; without the
// launch attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// 0/1 -> 0.0/1.0 without a conversion instruction (1.0 = 0x3FF00000:00000000)
__device__ __forceinline__ double bit_to_double(uint32_t bit) {
  return __hiloint2double((int)((0u - bit) & 0x3FF00000u), 0);
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, bool pred) {
  const uint32_t d = smem_addr(smem_dst);
  const int sz = pred ? 16 : 0;  // zero-fill when out of range
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gsrc), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Fixed-order block sum of src[0..count) (every thread gets the total).
__device__ __forceinline__ double block_sum_fixed(const double* __restrict__ src, int count, double* sh) {
  const int tid = threadIdx.y * blockDim.x + threadIdx.x, nt = blockDim.x * blockDim.y;
  double v = 0.0;
  for (int q = tid; q < count; q += nt) v += src[q];
  v = warp_sum<false>(v);
  if ((tid & 31) == 0) sh[tid >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (nt >> 5); ++w) t += sh[w];
  __syncthreads();
  return t;
}

// Column reduction of the row-block partials: blockDim (32, 8); lane x owns one
// output, the 8 y-phases split the partial blocks (b = y, y + 8, ...), then a
// fixed-order sum over y (valid on threadIdx.y == 0).
__device__ __forceinline__ double ysum8(double v, double (*sm)[33]) {
  sm[threadIdx.y][threadIdx.x] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.y == 0)
#pragma unroll
    for (int q = 0; q < 8; ++q) t += sm[q][threadIdx.x];
  __syncthreads();
  return t;
}

// x (N x n_in uint8) -> bit-packed rows
__global__ void k_pack_bits(const uint8_t* __restrict__ x, int64_t n, int n_in, uint64_t* __restrict__ xbits) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    uint64_t w[OTF_XW] = {0, 0};
    for (int k = 0; k < n_in; ++k)
      if (x[r * n_in + k]) w[k >> 6] |= 1ull << (k & 63);
    for (int q = 0; q < OTF_XW; ++q) xbits[r * OTF_XW + q] = w[q];
  }
}

// Tile loader: G (and T unless ts is null) rows [r0, r0+BM) x columns [j0, j0+BJ), packed bits.
__device__ __forceinline__ void otf_load_tile(const OtfArgs& a, int64_t r0, int64_t hi, int j0, double* gs, double* ts,
                                              uint64_t* xs, int tid, int nthreads) {
  // 64 rows x 64 doubles = 512 B per row = 32 x 16 B per row, for G and T
  for (int e = tid; e < OTF_BM * (OTF_BJ / 2); e += nthreads) {
    const int r = e / (OTF_BJ / 2), c = (e % (OTF_BJ / 2)) * 2;
    const int64_t row = r0 + r;
    const bool ok = row < hi && (j0 + c) < a.hidden;
    const int64_t off = ok ? row * a.hidden + j0 + c : 0;
    cp_async16(gs + r * OTF_BJ + c, a.G + off, ok);
    if (ts) cp_async16(ts + r * OTF_BJ + c, a.T + off, ok);  // ts == nullptr: G-only tiles (RBM)
  }
  for (int e = tid; e < OTF_BM; e += nthreads) {
    const int64_t row = r0 + e;
    const bool ok = row < hi;
    cp_async16(xs + e * OTF_XW, a.xbits + (ok ? row * OTF_XW : 0), ok);
  }
}

// Tiles of the OTF GEMMs are 64 rows x 64 columns of doubles loaded by four
// 2-D TMA boxes of 64 rows x 16 columns (128 bytes) with the 128-byte swizzle:
// box b holds columns [16 b, 16 b + 16); row r's 16-byte chunk q sits at chunk
// q ^ (r & 7).  Offset (in doubles) of element (r, c) of such a tile:
__device__ __forceinline__ int swz64(int r, int c) {
  return ((c >> 4) << 10) + (r << 4) + ((((c & 15) >> 1) ^ (r & 7)) << 1) + (c & 1);
}
constexpr int OTF_TILE = OTF_BM * OTF_BJ;  // doubles per swizzled tile (32 KB, 1024-byte aligned)

// Dynamic shared memory, rounded up to the 1024-byte alignment the swizzle needs.
__device__ __forceinline__ unsigned char* smem_1k(unsigned char* p) {
  const uint32_t a = smem_addr(p);
  return p + (((a + 1023u) & ~1023u) - a);
}

// Row stride (doubles) of the v_W chunk in shared memory: >= n_in, a multiple
// of 4 and == 4 (mod 16), so the B-fragment loads (8 rows x 4 k per half warp
// pair) hit 16 distinct 8-byte bank pairs.
__host__ __device__ __forceinline__ int otf_vstride(int nin) {
  int vs = (nin + 3) & ~3;
  while ((vs & 15) != 4) vs += 4;
  return vs;
}

// Persistent tile range of CTA c: linear tiles t = jc * ntiles + row_tile,
// split evenly over the grid (a range spans at most two hidden chunks while
// JC < gridDim.x).
__device__ __forceinline__ void otf_cta_range(int64_t total, int64_t& t0, int64_t& t1) {
  t0 = (total * blockIdx.x) / gridDim.x;
  t1 = (total * (blockIdx.x + 1)) / gridDim.x;
}

// grid (persistent, 1-D), 288 threads = 8 consumer warps + 1 producer warp:
// t partials (tpart[jc][row]) for every (hidden chunk, 64-row tile) of this
// CTA's range.  Consumers: 2 (32 rows) x 4 (16 hidden units).  HAS_T: MLP
// (G tile for X V_W^T, T tile for v_u); RBM: G == T, G-only tiles, no u block.
// The producer streams the G/T tiles (2-D swizzled TMA boxes) and the packed
// bits through a 2-stage mbarrier ring; the per-row cross-warp sums use a
// double-buffered exchange and one named barrier of the consumers per tile.
// LOWREG (short input rows, n_in <= 40): 80 registers, so two 288-thread CTAs
// share an SM (a short K loop leaves the tile epilogue latency-bound; twice
// the warps hide it); long rows keep the register budget for the K loop.
template <bool HAS_T, bool LOWREG = false>
__global__ void __maxnreg__(LOWREG ? 80 : (HAS_T ? 168 : 96))
    k_otf_dot(const OtfArgs a, const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmT) {
  extern __shared__ __align__(16) unsigned char smem_o[];
  constexpr int ST = OTF_DOT_STAGES;
  // tiles per stage: G (+ T for the MLP); with G formed from T (a.u) only T,
  // which then sits in the first slot -- half the shared memory, 2 CTAs per SM
  const bool gu = HAS_T && a.u != nullptr;
  const int NM = (HAS_T && !gu) ? 2 : 1;
  const int nin = a.n_in, vs = otf_vstride(nin);
  double* tiles = reinterpret_cast<double*>(smem_1k(smem_o));              // [ST][NM][TILE]
  uint64_t* xs = reinterpret_cast<uint64_t*>(tiles + ST * NM * OTF_TILE);  // [ST][BM][XW]
  double* red = reinterpret_cast<double*>(xs + ST * OTF_BM * OTF_XW);      // [2][4][BM]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 2 * 4 * OTF_BM);      // [ST]
  uint64_t* empty = full + ST;                                             // [ST]
  double* vb = reinterpret_cast<double*>(empty + ST);                      // [BJ]
  double* vu = vb + OTF_BJ;                                                // [BJ]
  double* vw = vu + OTF_BJ;                                                // [BJ][vs]
  double* uw = vw + OTF_BJ * vs;                                           // [BJ] u chunk (gu)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t N = a.n_rows;
  const int64_t ntiles = (N + OTF_BM - 1) / OTF_BM;
  const int h = a.hidden;
  const int jcount = (h + OTF_BJ - 1) / OTF_BJ;
  int64_t t0, t1;
  otf_cta_range(ntiles * jcount, t0, t1);
  if (t0 >= t1) return;
  for (int e = tid; e < ST * NM * OTF_TILE; e += blockDim.x) tiles[e] = 0.0;
  for (int e = tid; e < ST * OTF_BM * OTF_XW; e += blockDim.x) xs[e] = 0ull;
  if (tid == 0) {
    for (int q = 0; q < ST; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 8);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_enter();

  if (warp == 8) {  // ---------------------------------------------- producer
    if (lane == 0) {
      for (int64_t t = t0; t < t1; ++t) {
        const int k = (int)(t - t0), st = k % ST;
        if (k >= ST) mbar_wait(&empty[st], ((uint32_t)(k / ST) & 1u) ^ 1u);
        const int jc = (int)(t / ntiles);
        const int64_t r0 = (t % ntiles) * OTF_BM;
        const int nrows = (int)min((int64_t)OTF_BM, N - r0);
        const int j0 = jc * OTF_BJ;
        const int nbox = min(4, (h - j0 + 15) >> 4);
        mbar_arrive_expect_tx(&full[st], (uint32_t)(nbox * NM * OTF_BM * 128) + (uint32_t)nrows * OTF_XW * 8u);
        double* tg = tiles + st * NM * OTF_TILE;
        for (int b = 0; b < nbox; ++b) {
          if (!gu) tma_load_2d(tg + b * 1024, &tmG, j0 + 16 * b, (int)r0, &full[st]);
          if (HAS_T) tma_load_2d(tg + (NM - 1) * OTF_TILE + b * 1024, &tmT, j0 + 16 * b, (int)r0, &full[st]);
        }
        bulk_g2s(xs + st * OTF_BM * OTF_XW, a.xbits + r0 * OTF_XW, (uint32_t)nrows * OTF_XW * 8u, &full[st]);
      }
    }
    return;
  }
  // ------------------------------------------------------------ consumers
  const int wr = warp >> 2, wj = warp & 3;  // rows [wr*32, +32), j [wj*16, +16)
  auto load_v = [&](int jc) {  // v_W chunk, v_b, v_u (zero beyond h / n_in)
    const int j0 = jc * OTF_BJ;
    for (int e = tid; e < OTF_BJ * vs; e += 256) {
      const int jj = e / vs, k = e % vs;
      vw[e] = (j0 + jj < h && k < nin) ? a.v[a.offW + (int64_t)(j0 + jj) * nin + k] : 0.0;
    }
    for (int e = tid; e < OTF_BJ; e += 256) {
      vb[e] = (j0 + e < h) ? a.v[a.offb + j0 + e] : 0.0;
      if (HAS_T) vu[e] = (j0 + e < h) ? a.v[a.offu + j0 + e] : 0.0;
      if (gu) uw[e] = (j0 + e < h) ? a.u[j0 + e] : 0.0;
    }
  };
  const int ksteps = (nin + 3) / 4;
  int cur_jc = -1;
  for (int64_t t = t0; t < t1; ++t) {
    const int k = (int)(t - t0), st = k % ST;
    const int jc = (int)(t / ntiles);
    const int64_t r0 = (t % ntiles) * OTF_BM;
    if (jc != cur_jc) {  // (re)load the B operand for this hidden chunk
      named_bar_sync(1, 256);
      load_v(jc);
      named_bar_sync(1, 256);
      cur_jc = jc;
    }
    mbar_wait(&full[st], (uint32_t)(k / ST) & 1u);
    const double* G = tiles + st * NM * OTF_TILE;
    const double* Tt = G + (NM - 1) * OTF_TILE;
    const uint64_t* X = xs + st * OTF_BM * OTF_XW;

    // C = v_b (broadcast per column) + X V_W^T
    double c[4][2][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int jl = wj * 16 + nt * 8 + (lane & 3) * 2;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        c[mt][nt][0] = vb[jl];
        c[mt][nt][1] = vb[jl + 1];
      }
    }
    // m-tile mt holds tile rows wr*32 + mt + 4 i (i = lane >> 2): the 8 lanes of a
    // quarter-warp then read rows of both parities, so the 128-byte TMA swizzle
    // (chunk ^ row % 8) spreads their epilogue LDS.128 over all 8 chunks (the
    // consecutive-row mapping hit 4 chunks twice: 2-way bank conflicts)
    uint64_t xr[4][OTF_XW];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int q = 0; q < OTF_XW; ++q) xr[mt][q] = X[(wr * 32 + mt + 4 * (lane >> 2)) * OTF_XW + q];
    const double* vrow0 = vw + (wj * 16 + (lane >> 2)) * vs + (lane & 3);
    // a warp whose 16 hidden units all lie past h (tail chunk, e.g. h = 160)
    // skips its GEMM: c stays v_b = 0 there and meets zero v_u
    const int kend = (jc * OTF_BJ + wj * 16 < h) ? ksteps : 0;
    for (int kk = 0; kk < kend; ++kk) {
      const int kq = kk * 4 + (lane & 3);
      const double b0 = vrow0[kk * 4];
      const double b1 = vrow0[kk * 4 + 8 * vs];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const uint64_t word = (kq < 64) ? xr[mt][0] : xr[mt][1];
        const double av = bit_to_double((uint32_t)(word >> (kq & 63)) & 1u);
        dmma(c[mt][0][0], c[mt][0][1], av, b0);
        dmma(c[mt][1][0], c[mt][1][1], av, b1);
      }
    }
    // epilogue: row sums of G (.) C (+ T (.) v_u)
    double rs[4];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int rl = wr * 32 + mt + 4 * (lane >> 2);
      double sacc = 0.0;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int jl = wj * 16 + nt * 8 + (lane & 3) * 2;
        const int o = swz64(rl, jl);
        double2 g2;
        if (HAS_T && gu) {
          const double2 t2 = *reinterpret_cast<const double2*>(Tt + o);
          g2 = make_double2(uw[jl] * (1.0 - t2.x * t2.x), uw[jl + 1] * (1.0 - t2.y * t2.y));
        } else {
          g2 = *reinterpret_cast<const double2*>(G + o);
        }
        sacc = fma(g2.x, c[mt][nt][0], sacc);
        sacc = fma(g2.y, c[mt][nt][1], sacc);
        if (HAS_T) {
          const double2 t2 = *reinterpret_cast<const double2*>(Tt + o);
          sacc = fma(t2.x, vu[jl], sacc);
          sacc = fma(t2.y, vu[jl + 1], sacc);
        }
      }
      sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
      sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
      rs[mt] = sacc;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with the stage
    double* rd = red + (k & 1) * 4 * OTF_BM;
    if ((lane & 3) == 0) {
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) rd[wj * OTF_BM + wr * 32 + mt + 4 * (lane >> 2)] = rs[mt];
    }
    named_bar_sync(1, 256);
    if (tid < OTF_BM) {
      const int64_t row = r0 + tid;
      if (row < N) {
        const double tv = ((rd[tid] + rd[OTF_BM + tid]) + rd[2 * OTF_BM + tid]) + rd[3 * OTF_BM + tid];
        a.tpart[(int64_t)jc * N + row] = tv;
      }
    }
  }
}

// y_n = c_n (sum_jc tpart + v_c - s) ; s, g0 from per-CTA partial dots (fixed order)
// Y partials per CTA.
// p_last >= 0: MLP constant parameter v_c; offa >= 0: RBM visible block, adds x_n . v_a
__global__ void __launch_bounds__(256) k_otf_y(const double* __restrict__ tpart, int jc_count, int64_t n,
                                               const double* __restrict__ coeff, const double* v, int64_t p_last,
                                               const double* __restrict__ dpart, int n_dpart, double* y,
                                               double* ypart, const uint64_t* __restrict__ xbits, int64_t offa,
                                               int n_in, const double* __restrict__ yadd = nullptr) {
  pdl_enter();
  // coeff == nullptr: y = q (the centred row dot itself; connected completion)
  __shared__ double sh[8];
  __shared__ double va[OTF_MAX_NIN];
  if (offa >= 0)
    for (int i = threadIdx.x; i < n_in; i += blockDim.x) va[i] = v[offa + i];
  __syncthreads();
  const double s = block_sum_fixed(dpart, n_dpart, sh);  // same fixed order in every CTA
  const double vc = p_last >= 0 ? v[p_last] : 0.0;
  double acc = 0.0;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = min(n, lo + per);
  for (int64_t r = lo + threadIdx.x; r < hi; r += blockDim.x) {
    double t = 0.0;
#pragma unroll 4
    for (int q = 0; q < jc_count; ++q) t += tpart[(int64_t)q * n + r];
    if (offa >= 0) {
      double xa = 0.0;
      for (int w = 0; w < OTF_XW; ++w) {
        uint64_t bits = xbits[r * OTF_XW + w];
        while (bits) {
          const int b = __ffsll((long long)bits) - 1;
          bits &= bits - 1;
          xa += va[w * 64 + b];
        }
      }
      t += xa;
    }
    double yy = (coeff ? coeff[r] : 1.0) * ((t + vc) - s);
    if (yadd) yy += yadd[r];
    y[r] = yy;
    acc += yy;
  }
  acc = warp_sum<false>(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += sh[w];
    ypart[blockIdx.x] = tot;
  }
}

// grid (JC, nb), 288 threads = 8 consumer warps + 1 producer warp.
// part[y][blk][j][kc] = sum_rows y g_j x_kc (kc = n_in is the ones column),
// partu[y][blk][j] = sum y t_j (HAS_T).  NKT n-tiles of 8 k columns cover
// n_in + 1; NY weight vectors share one read of the G/T tiles and the B
// fragments.
//
// Pipeline: the producer warp fills an ST-stage ring (2-D TMA boxes of G/T,
// a bulk copy of the packed bits and of y), completing on the stage's `full`
// mbarrier; consumers release a stage through its `empty` mbarrier, so there
// is no CTA-wide barrier in the main loop.
//
// Consumer warp w: hidden units j0 + 16 (w & 3) + {0..7, 8..15} (two A
// fragments per B fragment: every 0/1 input fragment built from the bits
// feeds two DMMAs) over the row quads kk = w >> 2, +2, ...; the two row halves
// are summed through shared memory at the end.
template <int NKT, int NY, bool HAS_T>
__global__ void __maxnreg__((NKT <= 8 && NY == 1 && !HAS_T) ? 96 : 168)
    k_otf_acc(const OtfArgs a, const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmT) {
  extern __shared__ __align__(16) unsigned char smem_o[];
  constexpr int ST = OTF_ACC_STAGES;
  constexpr int KC = 8 * NKT;
  // G formed from T (a.u, product only): T alone per stage, in the first slot
  const bool gu = HAS_T && NY == 1 && a.u != nullptr;
  const int NM = (HAS_T && !gu) ? 2 : 1;
  double* tiles = reinterpret_cast<double*>(smem_1k(smem_o));                          // [ST][NM][TILE]
  uint64_t* xs = reinterpret_cast<uint64_t*>(tiles + ST * NM * OTF_TILE);              // [ST][BM][XW]
  double* ys = reinterpret_cast<double*>(xs + ST * OTF_BM * OTF_XW);                  // [ST][NY][BM]
  uint64_t* full = reinterpret_cast<uint64_t*>(ys + ST * NY * OTF_BM);                // [ST]
  uint64_t* empty = full + ST;                                                         // [ST]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int jc = blockIdx.x, j0 = jc * OTF_BJ;
  const int64_t N = a.n_rows;
  // row blocks start on even rows, so every tile's y slice is a 16-byte aligned bulk copy
  const int64_t lo = ((N * blockIdx.y) / a.nb) & ~1LL;
  const int64_t hi = blockIdx.y + 1 == (unsigned)a.nb ? N : ((N * (blockIdx.y + 1)) / a.nb) & ~1LL;
  const int nin = a.n_in, h = a.hidden;
  const int nbox = min(4, (h - j0 + 15) >> 4);  // boxes of this chunk inside [0, h)
  const int ntiles = (int)((hi - lo + OTF_BM - 1) / OTF_BM);

  // zero every stage once: boxes past h are never loaded and rows past the
  // block keep finite data (their y is zero)
  for (int e = tid; e < ST * NM * OTF_TILE; e += blockDim.x) tiles[e] = 0.0;
  for (int e = tid; e < ST * OTF_BM * OTF_XW; e += blockDim.x) xs[e] = 0ull;
  if (tid == 0) {
    for (int q = 0; q < ST; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 8);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_enter();

  double c[NY][2][NKT][2];
  double cu[NY][2][2];
#pragma unroll
  for (int q = 0; q < NY; ++q)
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      cu[q][f][0] = cu[q][f][1] = 0.0;
#pragma unroll
      for (int nt = 0; nt < NKT; ++nt) c[q][f][nt][0] = c[q][f][nt][1] = 0.0;
    }
  const int wj = warp & 3, wk = (warp >> 2) & 1;
  // A rows of this lane: hidden units jl (m-tile 0) and jl + 1 (m-tile 1), jl even, so one
  // 16-byte load gives both.  A quarter-warp (8 lanes) reads 4 tile rows (lane & 3) x 2
  // chunks; row r's chunk q sits at bank group q ^ (r & 7), so the two chunks must differ
  // in bit 2 for the 8 accesses to hit 8 distinct groups (chunks q, q + 1 collided
  // pairwise: ncu counted 2 wavefronts per ideal one on this load).  MMA row g = lane >> 2
  // therefore takes unit pair ((g & 1) << 2) | (g >> 1); the accumulator rows follow the
  // same lane, so the epilogue's jl is all that changes.
  const int jl = wj * 16 + 2 * ((((lane >> 2) & 1) << 2) | (lane >> 3));
  const double u_lo = (gu && j0 + jl < h) ? a.u[j0 + jl] : 0.0;
  const double u_hi = (gu && j0 + jl + 1 < h) ? a.u[j0 + jl + 1] : 0.0;

  if (warp == 8) {  // ---------------------------------------------- producer
    const double* yv_src[2] = {a.y, a.y2};
    for (int it = 0; it < ntiles; ++it) {
      const int st = it % ST;
      const uint32_t ph = (uint32_t)(it / ST) & 1u;
      if (it >= ST) mbar_wait(&empty[st], ph ^ 1u);
      const int64_t r0 = lo + (int64_t)it * OTF_BM;
      const int nrows = (int)min((int64_t)OTF_BM, hi - r0);
      // y: bulk copy of the even part; an odd last row (N odd) and the tail by plain stores
      const int nev = nrows & ~1;
      if (nrows < OTF_BM) {
        for (int e = lane; e < NY * OTF_BM; e += 32) {
          const int q = e / OTF_BM, r = e % OTF_BM;
          if (r >= nev) ys[(st * NY + q) * OTF_BM + r] = r < nrows ? yv_src[q][r0 + r] : 0.0;
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_expect_tx(&full[st], (uint32_t)(nbox * NM * OTF_BM * 128) +
                                             (uint32_t)nrows * OTF_XW * 8u + (uint32_t)(NY * nev * 8));
        double* tg = tiles + (st * NM) * OTF_TILE;
        for (int b = 0; b < nbox; ++b) {
          if (!gu) tma_load_2d(tg + b * 1024, &tmG, j0 + 16 * b, (int)r0, &full[st]);
          if (HAS_T) tma_load_2d(tg + (NM - 1) * OTF_TILE + b * 1024, &tmT, j0 + 16 * b, (int)r0, &full[st]);
        }
        bulk_g2s(xs + st * OTF_BM * OTF_XW, a.xbits + r0 * OTF_XW, (uint32_t)nrows * OTF_XW * 8u, &full[st]);
      }
      if (lane < NY && nev > 0) bulk_g2s(ys + (st * NY + lane) * OTF_BM, yv_src[lane] + r0, (uint32_t)nev * 8u, &full[st]);
    }
  } else {  // ---------------------------------------------------- consumers
    const int sh_base = lane >> 2;  // B column offset within an n-tile
    // the ones column (k = n_in) is bit n_in of every packed row
    const uint64_t one0 = nin < 64 ? (1ull << nin) : 0ull, one1 = nin >= 64 ? (1ull << (nin - 64)) : 0ull;
    for (int it = 0; it < ntiles; ++it) {
      const int st = it % ST;
      mbar_wait(&full[st], (uint32_t)(it / ST) & 1u);
      const double* G = tiles + (st * NM) * OTF_TILE;
      const double* Tt = G + (NM - 1) * OTF_TILE;
      const uint64_t* X = xs + st * OTF_BM * OTF_XW;
      const double* Y = ys + st * NY * OTF_BM;
      // warps whose 16 hidden units all lie past h never store: skip the GEMM
      const int kk_end = (j0 + wj * 16 < h) ? OTF_BM / 4 : 0;
#pragma unroll 2
      for (int kk = wk; kk < kk_end; kk += 2) {
        const int rl = kk * 4 + (lane & 3);
        const int o0 = swz64(rl, jl);  // jl even: (jl, jl + 1) is one 16-byte chunk
        double g0, g1, t0 = 0.0, t1 = 0.0;
        if (HAS_T) {
          const double2 tt = *reinterpret_cast<const double2*>(Tt + o0);
          t0 = tt.x;
          t1 = tt.y;
        }
        if (HAS_T && gu) {
          g0 = u_lo * (1.0 - t0 * t0);
          g1 = u_hi * (1.0 - t1 * t1);
        } else {
          const double2 gg = *reinterpret_cast<const double2*>(G + o0);
          g0 = gg.x;
          g1 = gg.y;
        }
        const uint64_t w0 = (X[rl * OTF_XW] | one0) >> sh_base, w1 = (X[rl * OTF_XW + 1] | one1) >> sh_base;
        // the row weight rides on the B operand: B = x ? y : 0 (integer selects, no FP64
        // multiply competing with the DMMA pipe)
#pragma unroll
        for (int q = 0; q < NY; ++q) {
          const double yq = Y[q * OTF_BM + rl];
#pragma unroll
          for (int nt = 0; nt < NKT; ++nt) {
            const uint32_t bit = nt < 8 ? (uint32_t)(w0 >> (nt * 8)) & 1u : (uint32_t)(w1 >> ((nt - 8) * 8)) & 1u;
            const double bv = bit ? yq : 0.0;
            dmma(c[q][0][nt][0], c[q][0][nt][1], g0, bv);
            dmma(c[q][1][nt][0], c[q][1][nt][1], g1, bv);
          }
          if (HAS_T) {  // u block sum_n T_nj y_n: two FMAs per lane (a DMMA here would be 7/8 zeros)
            cu[q][0][0] = fma(t0, yq, cu[q][0][0]);
            cu[q][1][0] = fma(t1, yq, cu[q][1][0]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
  if (HAS_T) {  // the u-block partials: lanes of a quad hold rows kk*4 + (lane & 3): sum the quad
#pragma unroll
    for (int q = 0; q < NY; ++q)
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        double v = cu[q][f][0];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        cu[q][f][0] = v;
        cu[q][f][1] = 0.0;
      }
  }
  __syncthreads();  // every stage consumed and every copy landed: the tiles are free
  // row halves: warps 4..7 hand their fragments to warps 0..3
  constexpr int NV = NY * 2 * (NKT + (HAS_T ? 1 : 0)) * 2;
  // (the G-from-T layout, one tile per stage, only occurs with NY == 1)
  static_assert(NV * 128 <= ST * (HAS_T && NY != 1 ? 2 : 1) * OTF_TILE, "exchange must fit the tile buffers");
  double* xch = tiles;  // [NV][128]
  const int xl = wj * 32 + lane;
  if (warp >= 4 && warp < 8) {
    int v = 0;
#pragma unroll
    for (int q = 0; q < NY; ++q)
#pragma unroll
      for (int f = 0; f < 2; ++f) {
#pragma unroll
        for (int nt = 0; nt < NKT; ++nt) {
          xch[(v++) * 128 + xl] = c[q][f][nt][0];
          xch[(v++) * 128 + xl] = c[q][f][nt][1];
        }
        if (HAS_T) {
          xch[(v++) * 128 + xl] = cu[q][f][0];
          xch[(v++) * 128 + xl] = cu[q][f][1];
        }
      }
  }
  __syncthreads();
  if (warp >= 4) return;
  {
    int v = 0;
#pragma unroll
    for (int q = 0; q < NY; ++q)
#pragma unroll
      for (int f = 0; f < 2; ++f) {
#pragma unroll
        for (int nt = 0; nt < NKT; ++nt) {
          c[q][f][nt][0] += xch[(v++) * 128 + xl];
          c[q][f][nt][1] += xch[(v++) * 128 + xl];
        }
        if (HAS_T) {
          cu[q][f][0] += xch[(v++) * 128 + xl];
          cu[q][f][1] += xch[(v++) * 128 + xl];
        }
      }
  }
  // partials: C[j][kc] fragment -> part[q][blk][j][kc]
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    const int jrow = j0 + jl + f;
    if (jrow >= h) continue;
#pragma unroll
    for (int q = 0; q < NY; ++q) {
      double* pb = a.part + (((int64_t)q * a.nb + blockIdx.y) * h + jrow) * KC;
#pragma unroll
      for (int nt = 0; nt < NKT; ++nt) {
        const int kc = nt * 8 + (lane & 3) * 2;
        pb[kc] = c[q][f][nt][0];
        pb[kc + 1] = c[q][f][nt][1];
      }
      if (HAS_T && (lane & 3) == 0) a.partu[((int64_t)q * a.nb + blockIdx.y) * h + jrow] = cu[q][f][0];
    }
  }
}

// Assemble the MLP-layout parameter vector from the acc partials:
//   mode 0 (product): out = sum part - obar * Y (+ u0 hf), out0 = g0
//   mode 1 (stats)  : out = sum part          (Y, obar unused)
// MLP assembly in the layout [W (h x n_in), b, u, c]; blockDim (32, 8)
__global__ void __launch_bounds__(256) k_otf_finish(const double* __restrict__ part, const double* __restrict__ partu,
                                                    int nb, int hidden, int n_in, int kc, int64_t ld,
                                                    const double* __restrict__ ypart, int n_ypart,
                                                    const double* __restrict__ obar, const double* hf,
                                                    const double* u0, const double* dgpart, int n_dgpart,
                                                    double* out, double* out0) {
  pdl_enter();
  __shared__ double sh[8];
  __shared__ double sm[8][33];
  const double Y = block_sum_fixed(ypart, n_ypart, sh);
  const int64_t hn = (int64_t)hidden * n_in;
  const int64_t P = hn + 2 * hidden + 1;
  const double uu = (hf && u0) ? *u0 : 0.0;
  const int ty = threadIdx.y;
  for (int64_t p0 = blockIdx.x * 32LL; p0 < ld; p0 += gridDim.x * 32LL) {
    const int64_t p = p0 + threadIdx.x;
    double acc = 0.0;
    if (p < hn) {
      const int64_t j = p / n_in, k = p % n_in;
      for (int b = ty; b < nb; b += 8) acc += part[((int64_t)b * hidden + j) * kc + k];
    } else if (p < hn + hidden) {
      const int64_t j = p - hn;
      for (int b = ty; b < nb; b += 8) acc += part[((int64_t)b * hidden + j) * kc + n_in];
    } else if (p < hn + 2 * hidden) {
      const int64_t j = p - hn - hidden;
      for (int b = ty; b < nb; b += 8) acc += partu[(int64_t)b * hidden + j];
    }
    acc = ysum8(acc, sm);
    if (ty == 0 && p < ld) {
      if (p == P - 1) acc = Y;
      if (p < P) {
        if (obar) acc = fma(-obar[p], Y, acc);
        if (hf && u0) acc = fma(uu, hf[p], acc);
      } else {
        acc = 0.0;
      }
      out[p] = acc;
    }
  }
  if (out0 && blockIdx.x == 0) {
    const double g = hf ? block_sum_fixed(dgpart, n_dgpart, sh) : 0.0;
    if (threadIdx.x == 0 && threadIdx.y == 0) *out0 = g;
  }
}

// per-CTA partial dots s = obar . v and g0 = hf . v over the padded vector
__global__ void __launch_bounds__(256) k_vdot2(const double* __restrict__ a1, const double* __restrict__ a2,
                                               const double* __restrict__ v, int64_t len, double* p1, double* p2) {
  pdl_enter();
  __shared__ double s1[8], s2[8];
  double x1 = 0.0, x2 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    const double vi = v[i];
    if (a1) x1 = fma(a1[i], vi, x1);
    if (a2) x2 = fma(a2[i], vi, x2);
  }
  x1 = warp_sum<false>(x1);
  x2 = warp_sum<false>(x2);
  if ((threadIdx.x & 31) == 0) {
    s1[threadIdx.x >> 5] = x1;
    s2[threadIdx.x >> 5] = x2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t1 = 0.0, t2 = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      t1 += s1[w];
      t2 += s2[w];
    }
    p1[blockIdx.x] = t1;
    p2[blockIdx.x] = t2;
  }
}

}  // namespace irl

namespace irl {
// per-CTA partial sums of y (fixed order)
__global__ void __launch_bounds__(256) k_vsum(const double* __restrict__ y, int64_t n, double* part) {
  __shared__ double s[8];
  double x = 0.0;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = min(n, lo + per);
  for (int64_t r = lo + threadIdx.x; r < hi; r += blockDim.x) x += y[r];
  x = warp_sum<false>(x);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    part[blockIdx.x] = t;
  }
}
}  // namespace irl

namespace irl {
// Hidden layer on FP64 tensor cores (the MLP "forward contraction" of the north
// star; also the RBM's theta = b + W x): PRE = X W^T + b for a 64-column chunk
// of the (real) weight matrix, then the activation epilogue.
//   real    : columns = hidden units;            T = tanh(PRE), MLP: G = u (1 - T^2)
//   complex : columns (2j, 2j+1) = (Re, Im) of W row j, so each C fragment pair
//             holds one complex theta_j;       T = tanh(theta) (complex)
// grid (ceil(ncols/64), nb), 256 threads; X as packed bits (n_in <= 100).
template <bool CPLX, int MODEL>
__global__ void __launch_bounds__(256) k_hidden_mma(const uint64_t* __restrict__ xbits, int64_t n_rows, int n_in,
                                                    int hidden, const double* __restrict__ Wm,
                                                    const double* __restrict__ bvec, const double* __restrict__ uvec,
                                                    double* __restrict__ Tout, double* __restrict__ Gout, int nb) {
  extern __shared__ __align__(16) unsigned char smem_h2[];
  double* ws = reinterpret_cast<double*>(smem_h2);  // [64][OTF_MAX_NIN] weight chunk (real columns)
  double* bs = ws + 64 * OTF_MAX_NIN;              // [64]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp >> 2, wj = warp & 3;
  const int ncols = CPLX ? 2 * hidden : hidden;
  const int c0 = blockIdx.x * 64;
  const int64_t lo = (n_rows * blockIdx.y) / nb, hi = (n_rows * (blockIdx.y + 1)) / nb;
  // real column c <-> weight element: real: W[c][k]; complex: (Re|Im) W[c/2][k]
  for (int e = tid; e < 64 * OTF_MAX_NIN; e += blockDim.x) {
    const int cc = e / OTF_MAX_NIN, k = e % OTF_MAX_NIN;
    const int col = c0 + cc;
    double val = 0.0;
    if (col < ncols && k < n_in) {
      if constexpr (CPLX) val = Wm[((int64_t)(col >> 1) * n_in + k) * 2 + (col & 1)];
      else val = Wm[(int64_t)col * n_in + k];
    }
    ws[e] = val;
  }
  for (int e = tid; e < 64; e += blockDim.x) {
    const int col = c0 + e;
    double bv = 0.0;
    if (col < ncols) {
      if constexpr (CPLX) bv = bvec[(col >> 1) * 2 + (col & 1)];
      else bv = bvec[col];
    }
    bs[e] = bv;
  }
  __syncthreads();
  const int ksteps = (n_in + 3) / 4;
  const double* wrow0 = ws + (wj * 16 + (lane >> 2)) * OTF_MAX_NIN + (lane & 3);
  for (int64_t r0 = lo; r0 < hi; r0 += 64) {
    double c[4][2][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int cl = wj * 16 + nt * 8 + (lane & 3) * 2;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        c[mt][nt][0] = bs[cl];
        c[mt][nt][1] = bs[cl + 1];
      }
    }
    uint64_t xr[4][OTF_XW];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int64_t row = r0 + wr * 32 + mt * 8 + (lane >> 2);
#pragma unroll
      for (int q = 0; q < OTF_XW; ++q) xr[mt][q] = row < hi ? __ldg(xbits + row * OTF_XW + q) : 0ull;
    }
    for (int kk = 0; kk < ksteps; ++kk) {
      const int k = kk * 4 + (lane & 3);
      const double b0 = wrow0[kk * 4];
      const double b1 = wrow0[kk * 4 + 8 * OTF_MAX_NIN];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const uint64_t word = (k < 64) ? xr[mt][0] : xr[mt][1];
        const double av = bit_to_double((uint32_t)(word >> (k & 63)) & 1u);
        dmma(c[mt][0][0], c[mt][0][1], av, b0);
        dmma(c[mt][1][0], c[mt][1][1], av, b1);
      }
    }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int64_t row = r0 + wr * 32 + mt * 8 + (lane >> 2);
      if (row >= hi) continue;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int col = c0 + wj * 16 + nt * 8 + (lane & 3) * 2;
        if (col >= ncols) continue;
        if constexpr (CPLX) {
          const double2 t = ctanh(make_double2(c[mt][nt][0], c[mt][nt][1]));
          reinterpret_cast<double2*>(Tout)[row * hidden + (col >> 1)] = t;
        } else {
          const double t0 = tanh(c[mt][nt][0]), t1 = tanh(c[mt][nt][1]);
          *reinterpret_cast<double2*>(Tout + row * hidden + col) = make_double2(t0, t1);
          if (MODEL == MODEL_MLP) {
            const double u0 = uvec[col], u1 = uvec[col + 1];
            *reinterpret_cast<double2*>(Gout + row * hidden + col) =
                make_double2(u0 * (1.0 - t0 * t0), u1 * (1.0 - t1 * t1));
          }
        }
      }
    }
  }
}
}  // namespace irl

namespace irl {
// xpart[blk][i] = sum_{rows of blk} y_r x_ri (thread i < n_in owns feature i; the
// packed row words are broadcast), plus ypart[blk] = sum y_r.  Fixed order.
__global__ void __launch_bounds__(128) k_xsum(const uint64_t* __restrict__ xbits, const double* __restrict__ y,
                                              int64_t n, int n_in, double* xpart, double* ypart) {
  pdl_enter();
  __shared__ uint64_t xb[128][OTF_XW];
  __shared__ double yb[128];
  __shared__ double sh[4];
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = min(n, lo + per);
  const int i = threadIdx.x;
  const int wsel = i >> 6, sft = i & 63;
  double acc = 0.0, ys = 0.0;
  for (int64_t r0 = lo; r0 < hi; r0 += 128) {  // stage 128 rows (coalesced), then scan them from smem
    const int64_t r = r0 + i;
    if (r < hi) {
      xb[i][0] = xbits[r * OTF_XW];
      xb[i][1] = xbits[r * OTF_XW + 1];
      yb[i] = y[r];
      ys += yb[i];
    }
    __syncthreads();
    const int cnt = (int)min((int64_t)128, hi - r0);
    if (i < n_in)
      for (int q = 0; q < cnt; ++q)
        if ((xb[q][wsel] >> sft) & 1ull) acc += yb[q];
    __syncthreads();
  }
  if (i < n_in) xpart[(int64_t)blockIdx.x * n_in + i] = acc;
  ys = warp_sum<false>(ys);
  if ((i & 31) == 0) sh[i >> 5] = ys;
  __syncthreads();
  if (i == 0) ypart[blockIdx.x] = ((sh[0] + sh[1]) + sh[2]) + sh[3];
}

// RBM real column statistics in the parameter layout [a (n), b (h), W (h x n)]:
//   a_i = sum y x_i ; b_j = sum y t_j (ones column) ; W_ji = sum y t_j x_i
__global__ void __launch_bounds__(256) k_rbm_stats_finish(const double* __restrict__ part, int nb, int hidden,
                                                          int n_in, int kc, const double* __restrict__ xpart, int nbx,
                                                          int64_t ld, double* out) {
  __shared__ double sm[8][33];
  const int64_t P = (int64_t)n_in + hidden + (int64_t)hidden * n_in;
  const int ty = threadIdx.y;
  for (int64_t p0 = blockIdx.x * 32LL; p0 < ld; p0 += gridDim.x * 32LL) {
    const int64_t p = p0 + threadIdx.x;
    double acc = 0.0;
    if (p < n_in) {
      for (int b = ty; b < nbx; b += 8) acc += xpart[(int64_t)b * n_in + p];
    } else if (p < n_in + hidden) {
      const int64_t j = p - n_in;
      for (int b = ty; b < nb; b += 8) acc += part[((int64_t)b * hidden + j) * kc + n_in];
    } else if (p < P) {
      const int64_t q = p - n_in - hidden, j = q / n_in, i = q % n_in;
      for (int b = ty; b < nb; b += 8) acc += part[((int64_t)b * hidden + j) * kc + i];
    }
    acc = ysum8(acc, sm);
    if (ty == 0 && p < ld) out[p] = acc;
  }
}
}  // namespace irl

namespace irl {
// RBM on-the-fly product assembled in the layout [a (n), b (h), W (h x n)]:
//   out = sum_blocks (x / ones-column / W partials) - obar * Y (+ u0 hf) ; out0 = g0
__global__ void __launch_bounds__(256) k_rbm_otf_finish(const double* __restrict__ part, int nb, int hidden,
                                                        int n_in, int kc, const double* __restrict__ xpart, int nbx,
                                                        const double* __restrict__ ypart, int n_ypart, int64_t ld,
                                                        const double* __restrict__ obar, const double* hf,
                                                        const double* u0, const double* dgpart, int n_dgpart,
                                                        double* out, double* out0) {
  pdl_enter();
  __shared__ double sh[8];
  __shared__ double sm[8][33];
  const double Y = block_sum_fixed(ypart, n_ypart, sh);
  const int64_t P = (int64_t)n_in + hidden + (int64_t)hidden * n_in;
  const double uu = (hf && u0) ? *u0 : 0.0;
  const int ty = threadIdx.y;
  for (int64_t p0 = blockIdx.x * 32LL; p0 < ld; p0 += gridDim.x * 32LL) {
    const int64_t p = p0 + threadIdx.x;
    double acc = 0.0;
    if (p < n_in) {
      for (int b = ty; b < nbx; b += 8) acc += xpart[(int64_t)b * n_in + p];
    } else if (p < n_in + hidden) {
      const int64_t j = p - n_in;
      for (int b = ty; b < nb; b += 8) acc += part[((int64_t)b * hidden + j) * kc + n_in];
    } else if (p < P) {
      const int64_t q = p - n_in - hidden, j = q / n_in, i = q % n_in;
      for (int b = ty; b < nb; b += 8) acc += part[((int64_t)b * hidden + j) * kc + i];
    }
    acc = ysum8(acc, sm);
    if (ty == 0 && p < ld) {
      if (p < P) {
        if (obar) acc = fma(-obar[p], Y, acc);
        if (hf && u0) acc = fma(uu, hf[p], acc);
      } else {
        acc = 0.0;
      }
      out[p] = acc;
    }
  }
  if (out0 && blockIdx.x == 0) {
    const double g = hf ? block_sum_fixed(dgpart, n_dgpart, sh) : 0.0;
    if (threadIdx.x == 0 && threadIdx.y == 0) *out0 = g;
  }
}
}  // namespace irl

// ============================================================================
// Complex-parameter (Hermitian, cfg4) RBM on the fly.  T (N x h complex) is
// viewed as a real N x 2h matrix (Re/Im column pairs), so the same DMMA tiles
// apply: the pair (2j, 2j+1) of every C fragment is one complex value.
//   dot : A = X V_W^T + v_b (complex) ; t_n = x.v_a + sum_j T_nj A_nj
//   acc : out[2j+p][kc] = sum_n (conj(T_nj) y_n)_p x_n,kc   (ones column kc = n_in)
// ============================================================================
namespace irl {

struct OtfCArgs {
  const uint64_t* xbits;
  const double* T;   // [N][2h] real view of the complex activations
  int64_t n_rows;
  int n_in, hidden;  // hidden = complex units h
  int nb;
  int64_t offW, offb;  // complex parameter offsets (RBM layout [a, b, W])
  const double* v_re;
  const double* v_im;
  double2* tpart;      // [JC][N]
  const double2* y;    // [N] complex row weights, or
  const double* yr;    // [N] real row weights (y == nullptr)
  double* part;        // [nb][2h][KC]
};

__device__ __forceinline__ void otf_load_ctile(const OtfCArgs& a, int64_t r0, int64_t hi, int c0, double* gs,
                                               uint64_t* xs, int tid, int nthreads) {
  const int ncols = 2 * a.hidden;
  for (int e = tid; e < OTF_BM * (OTF_BJ / 2); e += nthreads) {
    const int r = e / (OTF_BJ / 2), c = (e % (OTF_BJ / 2)) * 2;
    const int64_t row = r0 + r;
    const bool ok = row < hi && (c0 + c) < ncols;
    cp_async16(gs + r * OTF_BJ + c, a.T + (ok ? row * ncols + c0 + c : 0), ok);
  }
  for (int e = tid; e < OTF_BM; e += nthreads) {
    const int64_t row = r0 + e;
    const bool ok = row < hi;
    cp_async16(xs + e * OTF_XW, a.xbits + (ok ? row * OTF_XW : 0), ok);
  }
}

// grid (persistent, 1-D), 288 threads: complex t partials over this CTA's
// range of (real column chunk, 64-row tile) pairs; same pipeline as k_otf_dot.
__global__ void __maxnreg__(96) k_otf_dot_c(const OtfCArgs a,
                                                                  const __grid_constant__ CUtensorMap tmT) {
  extern __shared__ __align__(16) unsigned char smem_c[];
  constexpr int ST = OTF_DOT_STAGES;
  const int nin = a.n_in, vs = otf_vstride(nin);
  double* tiles = reinterpret_cast<double*>(smem_1k(smem_c));          // [ST][TILE]
  uint64_t* xs = reinterpret_cast<uint64_t*>(tiles + ST * OTF_TILE);   // [ST][BM][XW]
  double2* red = reinterpret_cast<double2*>(xs + ST * OTF_BM * OTF_XW);  // [2][4][BM]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 2 * 4 * OTF_BM);  // [ST]
  uint64_t* empty = full + ST;
  double* vb = reinterpret_cast<double*>(empty + ST);  // [64]
  double* vw = vb + OTF_BJ;                            // [64][vs]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ncols = 2 * a.hidden;
  const int64_t N = a.n_rows;
  const int64_t ntiles = (N + OTF_BM - 1) / OTF_BM;
  const int jcount = (ncols + OTF_BJ - 1) / OTF_BJ;
  int64_t t0, t1;
  otf_cta_range(ntiles * jcount, t0, t1);
  if (t0 >= t1) return;
  for (int e = tid; e < ST * OTF_TILE; e += blockDim.x) tiles[e] = 0.0;
  for (int e = tid; e < ST * OTF_BM * OTF_XW; e += blockDim.x) xs[e] = 0ull;
  if (tid == 0) {
    for (int q = 0; q < ST; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 8);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 8) {  // producer
    if (lane == 0) {
      for (int64_t t = t0; t < t1; ++t) {
        const int k = (int)(t - t0), st = k % ST;
        if (k >= ST) mbar_wait(&empty[st], ((uint32_t)(k / ST) & 1u) ^ 1u);
        const int jc = (int)(t / ntiles);
        const int64_t r0 = (t % ntiles) * OTF_BM;
        const int nrows = (int)min((int64_t)OTF_BM, N - r0);
        const int c0 = jc * OTF_BJ;
        const int nbox = min(4, (ncols - c0 + 15) >> 4);
        mbar_arrive_expect_tx(&full[st], (uint32_t)(nbox * OTF_BM * 128) + (uint32_t)nrows * OTF_XW * 8u);
        for (int b = 0; b < nbox; ++b)
          tma_load_2d(tiles + st * OTF_TILE + b * 1024, &tmT, c0 + 16 * b, (int)r0, &full[st]);
        bulk_g2s(xs + st * OTF_BM * OTF_XW, a.xbits + r0 * OTF_XW, (uint32_t)nrows * OTF_XW * 8u, &full[st]);
      }
    }
    return;
  }
  const int wr = warp >> 2, wj = warp & 3;
  auto load_v = [&](int jc) {
    const int c0 = jc * OTF_BJ;
    for (int e = tid; e < OTF_BJ * vs; e += 256) {
      const int cc = e / vs, k = e % vs;
      const int col = c0 + cc;
      double val = 0.0;
      if (col < ncols && k < nin) {
        const int64_t idx = a.offW + (int64_t)(col >> 1) * nin + k;
        val = (col & 1) ? a.v_im[idx] : a.v_re[idx];
      }
      vw[e] = val;
    }
    for (int e = tid; e < OTF_BJ; e += 256) {
      const int col = c0 + e;
      vb[e] = col < ncols ? ((col & 1) ? a.v_im[a.offb + (col >> 1)] : a.v_re[a.offb + (col >> 1)]) : 0.0;
    }
  };
  const int ksteps = (nin + 3) / 4;
  int cur_jc = -1;
  for (int64_t t = t0; t < t1; ++t) {
    const int k = (int)(t - t0), st = k % ST;
    const int jc = (int)(t / ntiles);
    const int64_t r0 = (t % ntiles) * OTF_BM;
    if (jc != cur_jc) {
      named_bar_sync(1, 256);
      load_v(jc);
      named_bar_sync(1, 256);
      cur_jc = jc;
    }
    mbar_wait(&full[st], (uint32_t)(k / ST) & 1u);
    const double* G = tiles + st * OTF_TILE;
    const uint64_t* X = xs + st * OTF_BM * OTF_XW;
    double c[4][2][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int cl = wj * 16 + nt * 8 + (lane & 3) * 2;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        c[mt][nt][0] = vb[cl];
        c[mt][nt][1] = vb[cl + 1];
      }
    }
    uint64_t xr[4][OTF_XW];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int q = 0; q < OTF_XW; ++q) xr[mt][q] = X[(wr * 32 + mt + 4 * (lane >> 2)) * OTF_XW + q];
    const double* vrow0 = vw + (wj * 16 + (lane >> 2)) * vs + (lane & 3);
    for (int kk = 0; kk < ksteps; ++kk) {
      const int kq = kk * 4 + (lane & 3);
      const double b0 = vrow0[kk * 4];
      const double b1 = vrow0[kk * 4 + 8 * vs];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const uint64_t word = (kq < 64) ? xr[mt][0] : xr[mt][1];
        const double av = bit_to_double((uint32_t)(word >> (kq & 63)) & 1u);
        dmma(c[mt][0][0], c[mt][0][1], av, b0);
        dmma(c[mt][1][0], c[mt][1][1], av, b1);
      }
    }
    // epilogue: complex row sums of T_nj A_nj over this chunk's units
    double2 rs[4];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int rl = wr * 32 + mt + 4 * (lane >> 2);
      double sre = 0.0, sim = 0.0;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int cl = wj * 16 + nt * 8 + (lane & 3) * 2;
        const double2 t2 = *reinterpret_cast<const double2*>(G + swz64(rl, cl));
        sre = fma(t2.x, c[mt][nt][0], sre);
        sre = fma(-t2.y, c[mt][nt][1], sre);
        sim = fma(t2.x, c[mt][nt][1], sim);
        sim = fma(t2.y, c[mt][nt][0], sim);
      }
      sre += __shfl_xor_sync(0xffffffffu, sre, 1);
      sim += __shfl_xor_sync(0xffffffffu, sim, 1);
      sre += __shfl_xor_sync(0xffffffffu, sre, 2);
      sim += __shfl_xor_sync(0xffffffffu, sim, 2);
      rs[mt] = make_double2(sre, sim);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    double2* rd = red + (k & 1) * 4 * OTF_BM;
    if ((lane & 3) == 0) {
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) rd[wj * OTF_BM + wr * 32 + mt + 4 * (lane >> 2)] = rs[mt];
    }
    named_bar_sync(1, 256);
    if (tid < OTF_BM) {
      const int64_t row = r0 + tid;
      if (row < N) {
        double2 tv = rd[tid];
        for (int w = 1; w < 4; ++w) {
          tv.x += rd[w * OTF_BM + tid].x;
          tv.y += rd[w * OTF_BM + tid].y;
        }
        a.tpart[(int64_t)jc * N + row] = tv;
      }
    }
  }
}

// s = sum obar_p v_p (complex, obar interleaved, v planar), g0 = sum hf_re v_re + hf_im v_im
__global__ void __launch_bounds__(256) k_vdot_c(const double2* __restrict__ obar, const double* __restrict__ v_re,
                                                const double* __restrict__ v_im, const double* __restrict__ h_re,
                                                const double* __restrict__ h_im, int64_t len, double2* sp,
                                                double* gp) {
  __shared__ double sh[3][8];
  double xr = 0.0, xi = 0.0, g = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    const double vr = v_re[i], vi = v_im ? v_im[i] : 0.0;
    if (obar) {
      const double2 o = obar[i];
      xr = fma(o.x, vr, fma(-o.y, vi, xr));
      xi = fma(o.x, vi, fma(o.y, vr, xi));
    }
    if (h_re) g = fma(h_re[i], vr, fma(h_im ? h_im[i] : 0.0, vi, g));
  }
  xr = warp_sum<false>(xr);
  xi = warp_sum<false>(xi);
  g = warp_sum<false>(g);
  if ((threadIdx.x & 31) == 0) {
    sh[0][threadIdx.x >> 5] = xr;
    sh[1][threadIdx.x >> 5] = xi;
    sh[2][threadIdx.x >> 5] = g;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0, c = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += sh[0][w];
      b += sh[1][w];
      c += sh[2][w];
    }
    sp[blockIdx.x] = make_double2(a, b);
    gp[blockIdx.x] = c;
  }
}

// y_n = c_n (sum_jc tpart + x_n . v_a - s), complex; Y partials per CTA
__global__ void __launch_bounds__(256) k_otf_y_c(const double2* __restrict__ tpart, int jc_count, int64_t n,
                                                 const double2* __restrict__ coeff, const double* v_re,
                                                 const double* v_im, int64_t offa, int n_in,
                                                 const uint64_t* __restrict__ xbits, const double2* __restrict__ sp,
                                                 int n_sp, double2* y, double2* ypart,
                                                 const double2* __restrict__ yadd = nullptr) {
  __shared__ double2 va[OTF_MAX_NIN];
  __shared__ double2 sh[8];
  for (int i = threadIdx.x; i < n_in; i += blockDim.x)
    va[i] = make_double2(v_re[offa + i], v_im ? v_im[offa + i] : 0.0);
  __syncthreads();
  double sr = 0.0, si = 0.0;
  {  // fixed-order block sum of the complex partials (same order in every CTA)
    __shared__ double2 shs[8];
    double2 v = make_double2(0.0, 0.0);
    for (int q = threadIdx.x; q < n_sp; q += blockDim.x) {
      v.x += sp[q].x;
      v.y += sp[q].y;
    }
    v.x = warp_sum<false>(v.x);
    v.y = warp_sum<false>(v.y);
    if ((threadIdx.x & 31) == 0) shs[threadIdx.x >> 5] = v;
    __syncthreads();
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      sr += shs[w].x;
      si += shs[w].y;
    }
  }
  double ar = 0.0, ai = 0.0;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = min(n, lo + per);
  for (int64_t r = lo + threadIdx.x; r < hi; r += blockDim.x) {
    double tr = 0.0, ti = 0.0;
    for (int q = 0; q < jc_count; ++q) {
      const double2 p = tpart[(int64_t)q * n + r];
      tr += p.x;
      ti += p.y;
    }
    for (int w = 0; w < OTF_XW; ++w) {
      uint64_t bits = xbits[r * OTF_XW + w];
      while (bits) {
        const int b = __ffsll((long long)bits) - 1;
        bits &= bits - 1;
        tr += va[w * 64 + b].x;
        ti += va[w * 64 + b].y;
      }
    }
    tr -= sr;
    ti -= si;
    const double2 c = coeff ? coeff[r] : make_double2(1.0, 0.0);
    double2 yy = make_double2(c.x * tr - c.y * ti, c.x * ti + c.y * tr);
    if (yadd) {
      yy.x += yadd[r].x;
      yy.y += yadd[r].y;
    }
    y[r] = yy;
    ar += yy.x;
    ai += yy.y;
  }
  ar = warp_sum<false>(ar);
  ai = warp_sum<false>(ai);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = make_double2(ar, ai);
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 t = make_double2(0.0, 0.0);
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      t.x += sh[w].x;
      t.y += sh[w].y;
    }
    ypart[blockIdx.x] = t;
  }
}

// part[blk][2j+p][kc] = sum_rows (conj(T_nj) y_n)_p x_n,kc  (kc = n_in: ones column).
// Same structure as k_otf_acc (producer warp, 2-D swizzled TMA tiles of the
// real N x 2h view of T, two A fragments per B fragment, row quads split over
// two warp halves).
// Register caps of the 9-warp (288-thread) GEMM kernels: one SM sub-partition
// holds a 16K-register slice and receives up to 3 warps of one CTA (168
// registers per thread at most) or 5 warps of two CTAs (96).
template <int NKT>
__global__ void __maxnreg__(NKT <= 8 ? 96 : 168)
    k_otf_acc_c(const OtfCArgs a, const __grid_constant__ CUtensorMap tmT) {
  extern __shared__ __align__(16) unsigned char smem_c[];
  constexpr int ST = OTF_ACC_STAGES;
  constexpr int KC = 8 * NKT;
  double* tiles = reinterpret_cast<double*>(smem_1k(smem_c));              // [ST][TILE]
  uint64_t* xs = reinterpret_cast<uint64_t*>(tiles + ST * OTF_TILE);       // [ST][BM][XW]
  double2* ys = reinterpret_cast<double2*>(xs + ST * OTF_BM * OTF_XW);     // [ST][BM]
  uint64_t* full = reinterpret_cast<uint64_t*>(ys + ST * OTF_BM);          // [ST]
  uint64_t* empty = full + ST;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c0 = blockIdx.x * OTF_BJ;
  const int64_t N = a.n_rows;
  const int64_t lo = (N * blockIdx.y) / a.nb, hi = (N * (blockIdx.y + 1)) / a.nb;
  const int nin = a.n_in, ncols = 2 * a.hidden;
  const int nbox = min(4, (ncols - c0 + 15) >> 4);
  const int ntiles = (int)((hi - lo + OTF_BM - 1) / OTF_BM);
  for (int e = tid; e < ST * OTF_TILE; e += blockDim.x) tiles[e] = 0.0;
  for (int e = tid; e < ST * OTF_BM * OTF_XW; e += blockDim.x) xs[e] = 0ull;
  if (tid == 0) {
    for (int q = 0; q < ST; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 8);
    }
    fence_mbar_init();
  }
  __syncthreads();
  double c[2][NKT][2];
#pragma unroll
  for (int f = 0; f < 2; ++f)
#pragma unroll
    for (int nt = 0; nt < NKT; ++nt) c[f][nt][0] = c[f][nt][1] = 0.0;
  const int wj = warp & 3, wk = (warp >> 2) & 1;
  const int jl = wj * 16 + (lane >> 2);  // real rows (2j + p) jl and jl + 8 within the chunk

  if (warp == 8) {  // producer
    for (int it = 0; it < ntiles; ++it) {
      const int st = it % ST;
      const uint32_t ph = (uint32_t)(it / ST) & 1u;
      if (it >= ST) mbar_wait(&empty[st], ph ^ 1u);
      const int64_t r0 = lo + (int64_t)it * OTF_BM;
      const int nrows = (int)min((int64_t)OTF_BM, hi - r0);
      if (!a.y || nrows < OTF_BM)
        for (int r = lane; r < OTF_BM; r += 32)
          ys[st * OTF_BM + r] = r >= nrows ? make_double2(0.0, 0.0)
                                : a.y ? a.y[r0 + r] : make_double2(a.yr[r0 + r], 0.0);
      __syncwarp();
      if (lane == 0) {
        const bool ybulk = a.y && nrows == OTF_BM;
        mbar_arrive_expect_tx(&full[st], (uint32_t)(nbox * OTF_BM * 128) + (uint32_t)nrows * OTF_XW * 8u +
                                             (ybulk ? OTF_BM * 16u : 0u));
        for (int b = 0; b < nbox; ++b)
          tma_load_2d(tiles + st * OTF_TILE + b * 1024, &tmT, c0 + 16 * b, (int)r0, &full[st]);
        bulk_g2s(xs + st * OTF_BM * OTF_XW, a.xbits + r0 * OTF_XW, (uint32_t)nrows * OTF_XW * 8u, &full[st]);
        if (ybulk) bulk_g2s(ys + st * OTF_BM, a.y + r0, OTF_BM * 16u, &full[st]);
      }
    }
  } else {  // consumers
    const int pj = jl & 1, jb = jl & ~1;
    const int sh_base = lane >> 2;
    const uint64_t one0 = nin < 64 ? (1ull << nin) : 0ull, one1 = nin >= 64 ? (1ull << (nin - 64)) : 0ull;
    for (int it = 0; it < ntiles; ++it) {
      const int st = it % ST;
      mbar_wait(&full[st], (uint32_t)(it / ST) & 1u);
      const double* G = tiles + st * OTF_TILE;
      const uint64_t* X = xs + st * OTF_BM * OTF_XW;
      const double2* Y = ys + st * OTF_BM;
#pragma unroll 2
      for (int kk = wk; kk < OTF_BM / 4; kk += 2) {
        const int rl = kk * 4 + (lane & 3);
        const double2 ta = *reinterpret_cast<const double2*>(G + swz64(rl, jb));
        const double2 tb = *reinterpret_cast<const double2*>(G + swz64(rl, jb + 8));
        const double2 yv = Y[rl];
        // conj(t) y = (t.x y.x + t.y y.y) + i (t.x y.y - t.y y.x): the lane's part p
        // is t.x u + t.y w with (u, w) selected once per row (no divergent FP64 paths)
        const double u = pj ? yv.y : yv.x, w = pj ? -yv.x : yv.y;
        const double a0 = fma(ta.x, u, ta.y * w);
        const double a1 = fma(tb.x, u, tb.y * w);
        const uint64_t w0 = (X[rl * OTF_XW] | one0) >> sh_base, w1 = (X[rl * OTF_XW + 1] | one1) >> sh_base;
#pragma unroll
        for (int nt = 0; nt < NKT; ++nt) {
          const uint32_t bit = nt < 8 ? (uint32_t)(w0 >> (nt * 8)) & 1u : (uint32_t)(w1 >> ((nt - 8) * 8)) & 1u;
          const double bv = bit_to_double(bit);
          dmma(c[0][nt][0], c[0][nt][1], a0, bv);
          dmma(c[1][nt][0], c[1][nt][1], a1, bv);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
  __syncthreads();
  constexpr int NV = 2 * NKT * 2;
  static_assert(NV * 128 <= ST * OTF_TILE, "exchange must fit the tile buffers");
  double* xch = tiles;  // [NV][128]
  const int xl = wj * 32 + lane;
  if (warp >= 4 && warp < 8) {
#pragma unroll
    for (int f = 0; f < 2; ++f)
#pragma unroll
      for (int nt = 0; nt < NKT; ++nt) {
        xch[((f * NKT + nt) * 2) * 128 + xl] = c[f][nt][0];
        xch[((f * NKT + nt) * 2 + 1) * 128 + xl] = c[f][nt][1];
      }
  }
  __syncthreads();
  if (warp >= 4) return;
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    const int col = c0 + jl + 8 * f;
#pragma unroll
    for (int nt = 0; nt < NKT; ++nt) {
      c[f][nt][0] += xch[((f * NKT + nt) * 2) * 128 + xl];
      c[f][nt][1] += xch[((f * NKT + nt) * 2 + 1) * 128 + xl];
    }
    if (col >= ncols) continue;
    double* pb = a.part + ((int64_t)blockIdx.y * ncols + col) * KC;
#pragma unroll
    for (int nt = 0; nt < NKT; ++nt) {
      const int kc = nt * 8 + (lane & 3) * 2;
      pb[kc] = c[f][nt][0];
      pb[kc + 1] = c[f][nt][1];
    }
  }
}

// xpart[blk][i] = sum y_r x_ri (complex y, or real yr); rows staged in smem
__global__ void __launch_bounds__(128) k_xsum_c(const uint64_t* __restrict__ xbits, const double2* __restrict__ y,
                                                const double* __restrict__ yr, int64_t n, int n_in, double2* xpart) {
  __shared__ uint64_t xb[128][OTF_XW];
  __shared__ double2 yb[128];
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = min(n, lo + per);
  const int i = threadIdx.x;
  const int wsel = i >> 6, sft = i & 63;
  double ar = 0.0, ai = 0.0;
  for (int64_t r0 = lo; r0 < hi; r0 += 128) {
    const int64_t r = r0 + i;
    if (r < hi) {
      xb[i][0] = xbits[r * OTF_XW];
      xb[i][1] = xbits[r * OTF_XW + 1];
      yb[i] = y ? y[r] : make_double2(yr[r], 0.0);
    }
    __syncthreads();
    const int cnt = (int)min((int64_t)128, hi - r0);
    if (i < n_in)
      for (int q = 0; q < cnt; ++q)
        if ((xb[q][wsel] >> sft) & 1ull) {
          ar += yb[q].x;
          ai += yb[q].y;
        }
    __syncthreads();
  }
  if (i < n_in) xpart[(int64_t)blockIdx.x * n_in + i] = make_double2(ar, ai);
}

// Assemble the complex RBM vector [a, b, W] from the partials.
//   product mode (out_re/out_im planar): out = R - conj(obar) Y (+ u0 hf) ; out0 = g0
//   stats mode (out_c interleaved): out = R, or conj(R) when conj_out (obar from y = w)
__global__ void __launch_bounds__(256) k_rbm_otf_finish_c(const double* __restrict__ part, int nb, int hidden,
                                                          int n_in, int kc, const double2* __restrict__ xpart, int nbx,
                                                          const double2* __restrict__ ypart, int n_ypart, int64_t ld,
                                                          const double2* __restrict__ obar, const double* hf_re,
                                                          const double* hf_im, const double* u0,
                                                          const double* gpart, int n_gpart, double* out_re,
                                                          double* out_im, double* out0, double2* out_c, int conj_out) {
  __shared__ double sh[8];
  __shared__ double sm[8][33];
  // ypart as 2 n_ypart doubles (re, im interleaved): sum the two lanes separately
  double Yr = 0.0, Yi = 0.0;
  if (ypart) {
    const int tid = threadIdx.y * 32 + threadIdx.x;
    for (int q = tid; q < n_ypart; q += 256) {
      Yr += ypart[q].x;
      Yi += ypart[q].y;
    }
    Yr = warp_sum<false>(Yr);
    Yi = warp_sum<false>(Yi);
    __shared__ double2 shy[8];
    if ((tid & 31) == 0) shy[tid >> 5] = make_double2(Yr, Yi);
    __syncthreads();
    Yr = Yi = 0.0;
    for (int w = 0; w < 8; ++w) {
      Yr += shy[w].x;
      Yi += shy[w].y;
    }
  }
  const int ncols = 2 * hidden;
  const int64_t P = (int64_t)n_in + hidden + (int64_t)hidden * n_in;
  const double uu = (hf_re && u0) ? *u0 : 0.0;
  const int ty = threadIdx.y;
  for (int64_t p0 = blockIdx.x * 32LL; p0 < ld; p0 += gridDim.x * 32LL) {
    const int64_t p = p0 + threadIdx.x;
    double ar = 0.0, ai = 0.0;
    if (p < n_in) {
      for (int b = ty; b < nbx; b += 8) {
        const double2 q = xpart[(int64_t)b * n_in + p];
        ar += q.x;
        ai += q.y;
      }
    } else if (p < n_in + hidden) {
      const int64_t j = p - n_in;
      for (int b = ty; b < nb; b += 8) {
        ar += part[((int64_t)b * ncols + 2 * j) * kc + n_in];
        ai += part[((int64_t)b * ncols + 2 * j + 1) * kc + n_in];
      }
    } else if (p < P) {
      const int64_t q = p - n_in - hidden, j = q / n_in, i = q % n_in;
      for (int b = ty; b < nb; b += 8) {
        ar += part[((int64_t)b * ncols + 2 * j) * kc + i];
        ai += part[((int64_t)b * ncols + 2 * j + 1) * kc + i];
      }
    }
    ar = ysum8(ar, sm);
    ai = ysum8(ai, sm);
    if (ty != 0 || p >= ld) continue;
    if (p >= P) ar = ai = 0.0;
    if (out_c) {
      out_c[p] = make_double2(ar, conj_out ? -ai : ai);
      continue;
    }
    if (p < P) {
      if (obar) {  // - conj(obar) Y
        const double2 o = obar[p];
        ar -= o.x * Yr + o.y * Yi;
        ai -= o.x * Yi - o.y * Yr;
      }
      if (hf_re && u0) {
        ar = fma(uu, hf_re[p], ar);
        if (hf_im) ai = fma(uu, hf_im[p], ai);
      }
    }
    out_re[p] = ar;
    if (out_im) out_im[p] = ai;
  }
  if (out0 && blockIdx.x == 0) {
    const double g = hf_re ? block_sum_fixed(gpart, n_gpart, sh) : 0.0;
    if (threadIdx.x == 0 && threadIdx.y == 0) *out0 = g;
  }
}

}  // namespace irl
