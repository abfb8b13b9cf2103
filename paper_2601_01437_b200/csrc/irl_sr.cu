// Host side of the C-ABI (include/irl_sr.h): argument checks, launch plans,
// workspace carving, kernel dispatch.  No allocation, no synchronisation.
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>
#include <set>
#include <string>
#include <unordered_map>
#include <unordered_set>

#include <cudaTypedefs.h>

#include "../../include/irl_sr.h"
#include "obuild.cuh"
#include "otf.cuh"
#include "lanczos.cuh"
#include "stream.cuh"
#include "rows.cuh"
#include <utility>
#include "wide.cuh"
#include "connected.cuh"
#include "hamiltonian.cuh"
#include "autoreg.cuh"

using namespace irl;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return IRL_OK;
  cudaGetLastError();
  return fail(IRL_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define IRL_TRY(expr)            \
  do {                           \
    int _rc = (expr);            \
    if (_rc != IRL_OK) return _rc; \
  } while (0)

struct DevInfo {
  int sms = 0;
  int smem_optin = 0;
  int major = 0;
};

int dev_info(DevInfo& d) {
  static DevInfo cache[64];
  static std::mutex mu;
  int dev = 0;
  IRL_TRY(cuda_check(cudaGetDevice(&dev), "cudaGetDevice"));
  if (dev < 0 || dev >= 64) return fail(IRL_ERR_DEVICE, "device index %d", dev);
  std::lock_guard<std::mutex> lk(mu);
  if (cache[dev].sms == 0) {
    DevInfo t;
    IRL_TRY(cuda_check(cudaDeviceGetAttribute(&t.sms, cudaDevAttrMultiProcessorCount, dev), "attr"));
    IRL_TRY(cuda_check(cudaDeviceGetAttribute(&t.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "attr"));
    IRL_TRY(cuda_check(cudaDeviceGetAttribute(&t.major, cudaDevAttrComputeCapabilityMajor, dev), "attr"));
    cache[dev] = t;
  }
  d = cache[dev];
  if (d.major != 10) return fail(IRL_ERR_DEVICE, "compute capability %d.x: this library is built for sm_100a", d.major);
  return IRL_OK;
}

// Function attributes are per device: the cache is keyed by (device, function)
// so a process that launches on a second GPU sets them there too.
int ensure_fn_attrs(const void* fn, int smem_optin) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  IRL_TRY(cuda_check(cudaGetDevice(&dev), "cudaGetDevice"));
  const std::pair<int, const void*> key(dev, fn);
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(key)) return IRL_OK;
  cudaFuncAttributes fa;
  IRL_TRY(cuda_check(cudaFuncGetAttributes(&fa, fn), "cudaFuncGetAttributes"));
  // dynamic + static shared memory must fit the opt-in limit
  IRL_TRY(cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          smem_optin - (int)fa.sharedSizeBytes),
                     "cudaFuncSetAttribute(smem)"));
  // cluster size 16 is non-portable; harmless for non-cluster launches
  cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaGetLastError();
  done.insert(key);
  return IRL_OK;
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t rup(int64_t a, int64_t b) { return cdiv(a, b) * b; }
inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

bool aligned16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ----------------------------------------------------------- kernels ----
using StreamFn = void (*)(StreamArgs);

template <bool CPLX, int MODE, bool ADD = false, bool DUAL = false>
StreamFn pick_stream(int ppt, int R) {
#define IRL_CASE(P, RR) \
  if (ppt == P && R == RR) return k_stream<CPLX, P, RR, MODE, ADD, DUAL>;
  IRL_CASE(2, 1) IRL_CASE(2, 2) IRL_CASE(2, 4) IRL_CASE(4, 1) IRL_CASE(4, 2) IRL_CASE(4, 4)
  IRL_CASE(8, 1) IRL_CASE(8, 2) IRL_CASE(8, 4) IRL_CASE(16, 1) IRL_CASE(16, 2) IRL_CASE(16, 4)
#undef IRL_CASE
  return nullptr;
}

StreamFn pick_stream_any(bool cplx, int mode, int ppt, int R) {
  switch (mode) {
    case MODE_FUSED: return cplx ? pick_stream<true, MODE_FUSED>(ppt, R) : pick_stream<false, MODE_FUSED>(ppt, R);
    case MODE_DOT: return cplx ? pick_stream<true, MODE_DOT>(ppt, R) : pick_stream<false, MODE_DOT>(ppt, R);
    case MODE_ACC: return cplx ? pick_stream<true, MODE_ACC>(ppt, R) : pick_stream<false, MODE_ACC>(ppt, R);
    default: return cplx ? pick_stream<true, MODE_STATS>(ppt, R) : pick_stream<false, MODE_STATS>(ppt, R);
  }
}

struct Plan {
  int mode = 0;
  int C = 0, W = 0, PPT = 0, R = 0, NT = 0, NS = 0, nb = 0;
  size_t smem = 0;
  StreamFn fn = nullptr;
  StreamFn fn_add = nullptr;  // MODE_FUSED with the additive row term (connected product)
  StreamFn fn_dual = nullptr;  // MODE_FUSED with two coefficient vectors (H_eff v and S v over one read)
};

size_t stream_extra_smem(bool cplx, int R, int C, int NS) {
  const size_t sS = cplx ? 16 : 8;
  return (size_t)(2 * NS + kXchSlots) * 8 + (size_t)2 * R * 32 * sS + (size_t)kXchSlots * C * R * sS +
         (size_t)kXchSlots * R * sS + sS + 8;
}

// Geometry for C column slices (uneven split, slot width Wmax = ceil(ld_u / C)).
bool choose_geom(int64_t ld_u, int C, bool cplx, int mode, int budget, Plan& p, int ns_cap = 8) {
  if (C < 1 || C > ld_u) return false;
  const int64_t W = cdiv(ld_u, C);
  if (W > INT_MAX / 16) return false;
  int best_ppt = 0, best_nt = 0;
  int64_t best_waste = INT64_MAX;
  for (int ppt : {16, 8, 4, 2}) {
    int64_t nt = rup(cdiv(W, ppt), 32);
    if (nt < 64) nt = 64;
    if (nt > stream_max_nt(ppt)) continue;
    const int64_t waste = nt * ppt - W;
    if (waste < best_waste) {
      best_waste = waste;
      best_ppt = ppt;
      best_nt = (int)nt;
    }
  }
  if (!best_ppt) return false;
  const size_t slice = (size_t)W * 16;
  // rows per stage: amortise the per-group reduction over up to 4 rows while
  // keeping >= 3 stages in flight
  const int R = (4 * slice <= 64 * 1024) ? 4 : (2 * slice <= 64 * 1024) ? 2 : 1;
  const size_t extra = stream_extra_smem(cplx, R, C, 8);
  if ((size_t)budget <= extra) return false;
  int NS = (int)std::min<size_t>((size_t)ns_cap, ((size_t)budget - extra) / (R * slice));
  if (NS < 2) return false;
  p.mode = mode;
  p.C = C;
  p.W = (int)W;
  p.PPT = best_ppt;
  p.R = R;
  p.NT = best_nt;
  p.NS = NS;
  p.smem = (size_t)NS * R * slice + stream_extra_smem(cplx, R, C, NS);
  p.fn = pick_stream_any(cplx, mode, best_ppt, R);
  if (mode == MODE_FUSED) {
    p.fn_add = cplx ? pick_stream<true, MODE_FUSED, true>(best_ppt, R) : pick_stream<false, MODE_FUSED, true>(best_ppt, R);
    p.fn_dual = cplx ? pick_stream<true, MODE_FUSED, false, true>(best_ppt, R)
                     : pick_stream<false, MODE_FUSED, false, true>(best_ppt, R);
  }
  return p.fn != nullptr;
}

int occupancy_blocks(const Plan& p, int& occ) {
  IRL_TRY(cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)p.fn, p.NT + 32, p.smem),
                     "occupancy"));
  if (occ < 1) return fail(IRL_ERR_DEVICE, "kernel does not fit on an SM (smem %zu)", p.smem);
  return IRL_OK;
}

int active_clusters(const Plan& p, int sms) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(p.C * std::max(1, sms / p.C));
  cfg.blockDim = dim3(p.NT + 32);
  cfg.dynamicSmemBytes = p.smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, (const void*)p.fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return ncl;
}

struct PlanKey {
  int64_t n, ld_u;
  int cplx, mode, dev;
  bool operator==(const PlanKey& o) const {
    return n == o.n && ld_u == o.ld_u && cplx == o.cplx && mode == o.mode && dev == o.dev;
  }
};
struct PlanKeyHash {
  size_t operator()(const PlanKey& k) const {
    return std::hash<int64_t>()(k.ld_u * 131 + k.n * 1000003 + k.cplx * 17 + k.mode * 3 + k.dev * 7919);
  }
};

constexpr int kMaxFusedCluster = 2;

int make_plan_uncached(int64_t n, int64_t ld_u, bool cplx, int mode, Plan& out) {
  DevInfo d;
  IRL_TRY(dev_info(d));
  const int budget = d.smem_optin;
  if (mode == MODE_FUSED) {
    // pick the cluster size that keeps the most SMs streaming (GPC packing
    // limits how many clusters of a given size are co-resident)
    Plan best;
    int best_active = 0;
    const char* force = getenv("IRL_FUSED_CLUSTER");  // tuning override
    const int c_force = force ? atoi(force) : 0;
    // clusters of at most kMaxFusedCluster CTAs: beyond two, the per-row DSMEM
    // exchange and GPC packing cost more than a second HBM pass (cfg4 C = 6:
    // 26.6 ms against 17.4 two-pass), and rows that wide take the single-read
    // wide product instead
    for (int C = 1; C <= kMaxFusedCluster; ++C) {
      if (c_force > 0 && C != c_force) continue;
      Plan p;
      if (!choose_geom(ld_u, C, cplx, mode, budget, p)) continue;
      IRL_TRY(ensure_fn_attrs((const void*)p.fn, budget));
      if (p.fn_add) IRL_TRY(ensure_fn_attrs((const void*)p.fn_add, budget));
      if (p.fn_dual) IRL_TRY(ensure_fn_attrs((const void*)p.fn_dual, budget));
      int active = 0;
      if (C == 1) {
        int occ = 0;
        IRL_TRY(occupancy_blocks(p, occ));
        p.nb = d.sms * occ;
        active = p.nb;
        // short problems: each CTA would see only a few row groups, so trade
        // ring depth for a second CTA per SM (twice the warps, half the chain)
        if (occ == 1 && n < (int64_t)d.sms * 8 * p.R * p.NS) {
          Plan q;
          const size_t extra = stream_extra_smem(cplx, p.R, 1, 3);
          const size_t stage = (size_t)p.R * p.W * 16;
          const int ns2 = (int)(((size_t)budget / 2 - 1024 - extra) / stage);
          if (ns2 >= 3 && choose_geom(ld_u, 1, cplx, mode, budget, q, ns2)) {
            int occ2 = 0;
            IRL_TRY(occupancy_blocks(q, occ2));
            if (occ2 >= 2) {
              q.nb = d.sms * occ2;
              p = q;
            }
          }
        }
      } else {
        p.nb = active_clusters(p, d.sms);
        active = p.nb * C;
      }
      active = std::min(active, d.sms);  // SMs kept streaming; extra co-resident CTAs buy nothing
      if (active > best_active * 1.04) {  // a bigger cluster must buy > 4% more SMs
        best = p;
        best_active = active;
      }
    }
    if (best_active == 0) return fail(IRL_ERR_DEVICE, "no fused single-pass geometry for ld=%lld units", (long long)ld_u);
    out = best;
    return IRL_OK;
  }
  for (int C = 1; C <= 256; ++C) {
    Plan p;
    if (!choose_geom(ld_u, C, cplx, mode, budget, p)) continue;
    IRL_TRY(ensure_fn_attrs((const void*)p.fn, budget));
    if (p.fn_add) IRL_TRY(ensure_fn_attrs((const void*)p.fn_add, budget));
    int occ = 0;
    IRL_TRY(occupancy_blocks(p, occ));
    // ~2 waves of CTAs over the SMs
    p.nb = std::max(1, (int)((2LL * d.sms * occ + C / 2) / C));
    out = p;
    return IRL_OK;
  }
  return fail(IRL_ERR_DEVICE, "no streaming geometry for ld=%lld units", (long long)ld_u);
}

int make_plan(int64_t n, int64_t ld_u, bool cplx, int mode, Plan& p) {
  static std::mutex mu;
  struct Entry {
    int rc;
    Plan plan;
    std::string err;
  };
  static std::unordered_map<PlanKey, Entry, PlanKeyHash> cache;
  int dev = 0;
  IRL_TRY(cuda_check(cudaGetDevice(&dev), "cudaGetDevice"));
  PlanKey key{n, ld_u, cplx ? 1 : 0, mode, dev};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      p = it->second.plan;
      if (it->second.rc != IRL_OK) g_err = it->second.err;
      return it->second.rc;
    }
  }
  Plan q;
  const int rc = make_plan_uncached(n, ld_u, cplx, mode, q);
  const std::string err = rc != IRL_OK ? g_err : std::string();
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = Entry{rc, q, err};
  p = q;
  return rc;
}

int launch_stream(const Plan& p, const StreamArgs& a, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.gridDim = dim3((unsigned)(p.nb * p.C));
  cfg.blockDim = dim3(p.NT + 32);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cfg.numAttrs = 0;
  if (p.mode == MODE_FUSED && p.C > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  StreamArgs args = a;
  args.Wmax = p.W;
  args.C = p.C;
  args.nb = p.nb;
  args.stages = p.NS;
  args.dbg = 0;
  void* kargs[] = {&args};
  const StreamFn fn = (p.mode == MODE_FUSED && args.coeff1) ? p.fn_dual
                      : (args.yadd && p.mode == MODE_FUSED) ? p.fn_add
                                                             : p.fn;
  if (!fn) return fail(IRL_ERR_DEVICE, "no stream kernel instance");
  return cuda_check(cudaLaunchKernelExC(&cfg, (const void*)fn, kargs), "stream kernel launch");
}

// finisher launched with programmatic dependent launch (overlaps its launch
// with the streaming kernel's tail; it waits in griddepcontrol.wait)
template <bool CPLX>
int launch_finish_mvp(const double2* part, int nb, int64_t ld_u, const void* ysum, const double2* obar,
                      const double* hf_re, const double* hf_im, const double* u0, double* out_re, double* out_im,
                      const double* gpart, int n_gpart, double* out0, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  // units per block: 32 normally; narrow vectors spread the nb-way sums over
  // more row groups per block so the grid still covers the SMs
  const int upb = ld_u >= 32 * 148 ? 32 : (ld_u >= 16 * 148 ? 16 : 8);
  cfg.gridDim = dim3((unsigned)cdiv(ld_u, upb));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cuda_check(cudaLaunchKernelEx(&cfg, k_finish_mvp<CPLX>, part, nb, ld_u, upb, ysum, obar, hf_re, hf_im, u0,
                                       out_re, out_im, gpart, n_gpart, out0),
                    "finish kernel launch");
}


// MVP workspace layout for one plan
struct MvpWs {
  double2* part;
  void* ysum;
  void* tpart;
  void* spart;
  double* gpart;
  size_t bytes;
};

MvpWs mvp_ws_layout(const Plan& p, int64_t n, int64_t ld_u, bool cplx, void* base) {
  const size_t sS = cplx ? 16 : 8;
  size_t off = 0;
  MvpWs w{};
  auto carve = [&](size_t b) {
    void* r = base ? static_cast<char*>(base) + off : nullptr;
    off += align256(b);
    return r;
  };
  w.part = (double2*)carve((size_t)p.nb * ld_u * 16);
  w.ysum = carve((size_t)p.nb * sS);
  w.tpart = carve(p.mode == MODE_FUSED ? 0 : (size_t)p.C * n * sS);
  w.spart = carve((size_t)std::max(p.C, 1) * sS);
  w.gpart = (double*)carve((size_t)std::max(p.C, 1) * 8);
  w.bytes = off;
  return w;
}

// warp-per-row path (rows.cuh): narrow rows only
constexpr int64_t kRowsMaxUnits = 512;

using RowsFn = void (*)(StreamArgs);
RowsFn pick_rows(bool cplx, int64_t ld_u) {
  const int upl = (int)cdiv(ld_u, 32);
  if (upl <= 4) return cplx ? k_rows_mvp<true, 4> : k_rows_mvp<false, 4>;
  if (upl <= 8) return cplx ? k_rows_mvp<true, 8> : k_rows_mvp<false, 8>;
  if (upl <= 12) return cplx ? k_rows_mvp<true, 12> : k_rows_mvp<false, 12>;
  if (upl <= 14) return cplx ? k_rows_mvp<true, 14> : k_rows_mvp<false, 14>;
  if (upl <= 16) return cplx ? k_rows_mvp<true, 16> : k_rows_mvp<false, 16>;
  return nullptr;
}

// rows plan: 2 CTAs per SM (or fewer for short problems); a Plan carrying the
// partial count for the workspace layout
int make_rows_plan(int64_t n, int64_t ld_u, Plan& p) {
  if (ld_u > kRowsMaxUnits) return fail(IRL_ERR_DEVICE, "rows path needs ld <= %lld units", (long long)kRowsMaxUnits);
  DevInfo d;
  IRL_TRY(dev_info(d));
  p = Plan{};
  p.mode = MODE_FUSED;  // no tpart in the workspace
  p.C = 1;
  const int upl = (int)cdiv(ld_u, 32);
  const int nw = 8, per_sm = upl <= 4 ? 2 : 1;  // RowsGeom<UPL>
  p.nb = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * d.sms, cdiv(n, 2 * nw)));
  p.NT = nw * 32;
  const int upl_t = upl <= 4 ? 4 : upl <= 8 ? 8 : upl <= 12 ? 12 : upl <= 14 ? 14 : 16;  // pick_rows' instance
  p.smem = ((size_t)nw * ld_u + 32 * upl_t) * 16;
  return IRL_OK;
}

int launch_rows(const Plan& p, bool cplx, const StreamArgs& a, cudaStream_t st) {
  RowsFn fn = pick_rows(cplx, a.ld_u);
  if (!fn) return fail(IRL_ERR_DEVICE, "no rows instance for ld=%lld units", (long long)a.ld_u);
  DevInfo d;
  IRL_TRY(dev_info(d));
  IRL_TRY(ensure_fn_attrs((const void*)fn, d.smem_optin));
  fn<<<p.nb, p.NT, p.smem, st>>>(a);
  return cuda_check(cudaGetLastError(), "rows kernel launch");
}

// ----------------------------------------------------------------- wide ---
// Rows of at least kWideMinUnits 16-byte units (cfg4, cfg5) take the
// single-read wide kernel (wide.cuh): every SM owns a column slice of every
// row, so O is read from HBM once with no cluster exchange.
constexpr int64_t kWideMinUnits = 16384;

struct WidePlan {
  int G, WM, RS, Q, PU, NS, K, upl, rpw, ut, pr;
  size_t smem, ws, part_bytes, fin_bytes, fin_copy_bytes, ring_bytes, vsl_off, side_off;
};

using WideFn = void (*)(WideArgs);
// instances: units per lane x rows per warp-step <= 16 (register budget)
constexpr bool wide_inst(int upl, int rpw) { return upl * rpw <= 16; }
template <bool CPLX>
WideFn pick_wide_c(int upl, int rpw, bool side) {
#define WIDE_CASE(U, R) if (upl == U && rpw == R && !side) return k_wide<CPLX, U, R>;
  WIDE_CASE(2, 1) WIDE_CASE(2, 2) WIDE_CASE(2, 4) WIDE_CASE(4, 1) WIDE_CASE(4, 2) WIDE_CASE(4, 4)
  WIDE_CASE(6, 1) WIDE_CASE(6, 2) WIDE_CASE(8, 1) WIDE_CASE(8, 2)
#undef WIDE_CASE
#define WIDE_CASE(U, R) if (upl == U && rpw == R && side) return k_wide<CPLX, U, R, true>;
  WIDE_CASE(4, 1) WIDE_CASE(4, 2) WIDE_CASE(4, 4) WIDE_CASE(6, 1) WIDE_CASE(6, 2)
#undef WIDE_CASE
  return nullptr;
}
// side-buffer instances exist for 4 and 6 units per lane
constexpr bool wide_side_inst(int upl) { return upl == 4 || upl == 6; }
WideFn pick_wide(bool cplx, int upl, int rpw, bool side) {
  return cplx ? pick_wide_c<true>(upl, rpw, side) : pick_wide_c<false>(upl, rpw, side);
}

int wide_upl(int need) { return need <= 2 ? 2 : need <= 4 ? 4 : need <= 6 ? 6 : need <= 8 ? 8 : 0; }

int make_wide_plan(int64_t n, int64_t ld_u, bool cplx, WidePlan& p) {
  DevInfo d;
  IRL_TRY(dev_info(d));
  p.G = d.sms;
  if (getenv("IRL_WIDE_G")) p.G = std::max(2, std::min(d.sms, atoi(getenv("IRL_WIDE_G"))));  // tuning: fewer, wider slices
  if (p.G > WIDE_QPL * 32 * WIDE_AW) return fail(IRL_ERR_DEVICE, "wide path: %d SMs exceed the aggregator lanes", p.G);
  p.WM = (int)cdiv(ld_u, p.G);
  // fewest parts per row slice (most rows per block, the biggest TMA stages)
  // whose per-lane share fits a kernel instance
  // (at most 6 units per lane: the 8-unit instances spill with two rows per step)
  p.Q = 0;
  for (int q = 1; q <= WIDE_CW; q *= 2) {
    const int upl = wide_upl((int)cdiv(cdiv(p.WM, q), 32));
    if (upl && upl <= 6) {
      p.Q = q;
      p.upl = upl;
      break;
    }
  }
  if (!p.Q) return fail(IRL_ERR_DEVICE, "wide path needs <= %d units per SM slice", 8 * 32 * WIDE_CW);
  if (getenv("IRL_WIDE_Q")) {  // tuning: more parts per row = fewer rows per stage
    const int q = atoi(getenv("IRL_WIDE_Q"));
    if (q >= p.Q && q <= WIDE_CW && (WIDE_CW % q) == 0) {
      p.Q = q;
      p.upl = wide_upl((int)cdiv(cdiv(p.WM, q), 32));
    }
  }
  // rows per warp-step: each consumer step has fixed latencies (barrier probes,
  // butterfly, TMEM round trip), so a step should move ~5 KB or more
  const int part_bytes_row = (int)cdiv(p.WM, p.Q) * 16;
  p.PU = (int)cdiv(p.WM, p.Q);
  // TMEM takes a lane's full lane-rows of a part (units lane + 32 k, k < ut);
  // a partly filled last lane-row (pr units) waits in a shared-memory side
  // buffer instead, so no TMEM columns are spent on empty lanes: the TMEM slots
  // set the number of pending blocks, which bounds the product (cfg4: 100 units
  // a part = 3 lane-rows + 4 units, 5 slots instead of 4; cfg5: 5 + 17 units, 6
  // instead of 5)
  p.ut = p.upl;
  p.pr = 0;
  {
    const int ut = p.PU / 32, pr = p.PU - 32 * ut;
    if (!getenv("IRL_WIDE_NOSIDE") && ut == p.upl - 1 && wide_side_inst(p.upl) && pr > 0 && pr <= 24) {
      p.ut = ut;
      p.pr = pr;
    }
  }
  p.rpw = 1;
  while (p.rpw < 4 && part_bytes_row * p.rpw < 4096 && wide_inst(p.upl, 2 * p.rpw) &&
         2 * p.rpw * WIDE_CW / p.Q <= WIDE_MAX_RS && 2 * p.rpw * 4 * p.ut * 2 <= WIDE_TM_COLS_PER_WARP)
    p.rpw *= 2;
  if (getenv("IRL_WIDE_RPW")) {
    const int r = atoi(getenv("IRL_WIDE_RPW"));
    if ((r == 1 || r == 2 || r == 4) && wide_inst(p.upl, r) && r * WIDE_CW / p.Q <= WIDE_MAX_RS &&
        r * 4 * p.ut * 2 <= WIDE_TM_COLS_PER_WARP)
      p.rpw = r;
  }
  p.RS = p.rpw * WIDE_CW / p.Q;
  const size_t sS = cplx ? 16 : 8;
  // TMEM slots per dot / accumulate warp pair: its half of the 512 columns over 4 ut words a row
  p.K = std::min(WIDE_MAX_K, WIDE_TM_COLS_PER_WARP / (p.rpw * 4 * p.ut));
  if (getenv("IRL_WIDE_K")) p.K = std::min(p.K, std::max(2, atoi(getenv("IRL_WIDE_K"))));
  const size_t stage = (size_t)p.RS * p.WM * 16;
  const size_t per_slot = 4 * 8 + (size_t)p.RS * p.Q * sS + (size_t)p.RS * sS;  // dotdone, ydone, parked, slotfree, pd, ys
  const size_t budget = (size_t)d.smem_optin - 2048;  // static smem of the kernel
  const size_t side_bytes = (size_t)p.K * p.RS * p.Q * p.pr * 16;
  const size_t fixed = (size_t)p.K * per_slot + 16 + (size_t)p.RS * sS;  // + the y ring's extra slot (ydone + pad, ys)
  const size_t vbytes = (size_t)(p.WM + 1) * 16 + 32 + side_bytes;
  p.NS = (int)std::min<size_t>(WIDE_MAX_NS, (budget - fixed - vbytes) / (stage + 16));
  if (getenv("IRL_WIDE_NS")) p.NS = std::min(p.NS, std::max(2, atoi(getenv("IRL_WIDE_NS"))));
  if (p.NS < 2) return fail(IRL_ERR_DEVICE, "wide path: row slices too wide for the ring");
  p.ring_bytes = std::max((size_t)p.NS * stage, (size_t)WIDE_CW * 32 * p.upl * 16);  // ring / epilogue scratch
  p.vsl_off = p.ring_bytes + (size_t)p.NS * 16 + fixed;
  p.vsl_off = (p.vsl_off + 15) / 16 * 16;
  p.side_off = (p.vsl_off + (size_t)(p.WM + 1) * 16 + 15) / 16 * 16;
  p.smem = p.side_off + side_bytes;
  if (p.smem > budget) return fail(IRL_ERR_DEVICE, "wide path: shared memory");
  const size_t rec = cplx ? 32 : 16;  // LL record bytes per scalar
  p.part_bytes = align256((size_t)WIDE_NBUF * p.RS * p.G * rec);
  p.fin_copy_bytes = align256((size_t)WIDE_NBUF * p.RS * rec) + 256;  // + 256: replicas start on different L2 slices
  p.fin_bytes = (size_t)WIDE_FIN_COPIES * p.fin_copy_bytes;
  p.ws = p.part_bytes + p.fin_bytes + align256((size_t)p.G * 16);
  (void)n;
  return IRL_OK;
}

// development tracing (IRL_WIDE_TRACE=1): per-block globaltimer stamps of
// every CTA into one process-wide device buffer, read by irl_debug_wide_trace
unsigned long long* g_wide_trace = nullptr;
size_t g_wide_trace_bytes = 0;
unsigned long long* wide_trace_buffer(int G) {
  static const bool on = getenv("IRL_WIDE_TRACE") != nullptr;
  if (!on) return nullptr;
  const size_t bytes = (size_t)G * WIDE_TRACE_B * 8 * 8;
  if (!g_wide_trace) {
    if (cudaMalloc(&g_wide_trace, bytes) != cudaSuccess) return nullptr;
    cudaMemset(g_wide_trace, 0, bytes);
    g_wide_trace_bytes = bytes;
  }
  return g_wide_trace;
}

int launch_wide(const WidePlan& p, bool cplx, WideArgs a, void* ws, cudaStream_t st) {
  WideFn fn = pick_wide(cplx, p.upl, p.rpw, p.pr > 0);
  if (!fn) return fail(IRL_ERR_DEVICE, "no wide instance for %d units per lane, %d rows per warp", p.upl, p.rpw);
  DevInfo d;
  IRL_TRY(dev_info(d));
  IRL_TRY(ensure_fn_attrs((const void*)fn, d.smem_optin));
  char* base = static_cast<char*>(ws);
  a.part = reinterpret_cast<ulonglong2*>(base);
  a.fin = reinterpret_cast<ulonglong2*>(base + p.part_bytes);
  a.gpart = reinterpret_cast<ulonglong2*>(base + p.part_bytes + p.fin_bytes);
  a.fin_copies = WIDE_FIN_COPIES;
  if (getenv("IRL_WIDE_FINC")) a.fin_copies = std::min(WIDE_FIN_COPIES, std::max(1, atoi(getenv("IRL_WIDE_FINC"))));
  a.fin_stride = p.fin_copy_bytes / sizeof(ulonglong2);
  a.RS = p.RS;
  a.Q = p.Q;
  a.PU = p.PU;
  a.NS = p.NS;
  a.K = p.K;
  a.WM = p.WM;
  a.ring_bytes = p.ring_bytes;
  a.vsl_off = p.vsl_off;
  a.UT = p.ut;
  a.PR = p.pr;
  a.side_off = p.side_off;
  a.trace = wide_trace_buffer(p.G);
  a.trace_stride = getenv("IRL_WIDE_TRACE") ? std::max(1, atoi(getenv("IRL_WIDE_TRACE"))) : 1;
  a.poll_ns = getenv("IRL_WIDE_POLL_NS") ? atoi(getenv("IRL_WIDE_POLL_NS")) : 160;
  // aggregators start polling a row's partials 0.5 us after this CTA's own publish: the other CTAs' shares land
  // within about that time, and the earlier polls only added L2 traffic (cfg4 12.6 -> 12.25 ms, cfg5 18.6 -> 18.2)
  a.agg_delay_ns = getenv("IRL_WIDE_ADELAY") ? atoi(getenv("IRL_WIDE_ADELAY")) : 500;
  a.rot = getenv("IRL_WIDE_ROT") ? atoi(getenv("IRL_WIDE_ROT")) % p.G : 0;
  a.red_delay_ns = getenv("IRL_WIDE_RDELAY") ? atoi(getenv("IRL_WIDE_RDELAY")) : 0;
  // tags are block numbers: zeroed records can never match a stale one
  IRL_TRY(cuda_check(cudaMemsetAsync(base, 0, p.ws, st), "wide record reset"));
  int occ = 0;
  IRL_TRY(cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, WIDE_THREADS, p.smem), "occ"));
  if (occ < 1) return fail(IRL_ERR_DEVICE, "wide kernel does not fit on an SM");
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all G CTAs co-resident: the exchange cannot deadlock
  attr[0].val.cooperative = 1;
  cfg.gridDim = dim3(p.G);
  cfg.blockDim = dim3(WIDE_THREADS);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cuda_check(cudaLaunchKernelEx(&cfg, fn, a), "wide kernel launch");
}

int mvp_impl(bool cplx, const double* O, int64_t n, int64_t p, int64_t ld, const double* obar, const double* coeff,
             const void* yadd, const double* v_re, const double* v_im, double* out_re, double* out_im, const double* hf_re,
             const double* hf_im, const double* u0, double* out0, int mode, void* ws, size_t ws_bytes,
             cudaStream_t st) {
  if (!O || !coeff || !v_re || !out_re) return fail(IRL_ERR_ARG, "null required pointer");
  if (n < 1 || p < 1 || ld < p) return fail(IRL_ERR_ARG, "bad shape n=%lld p=%lld ld=%lld", (long long)n,
                                            (long long)p, (long long)ld);
  if (ld != irl_padded_ld(p, cplx)) return fail(IRL_ERR_ALIGN, "ld must equal irl_padded_ld(p)");
  if (!aligned16(O) || !aligned16(obar) || !aligned16(ws) || (!cplx && (!aligned16(v_re) || !aligned16(out_re) ||
                                                                       !aligned16(hf_re))))
    return fail(IRL_ERR_ALIGN, "pointers must be 16-byte aligned");
  const int64_t ld_u = cplx ? ld : ld / 2;
  int path = mode;
  Plan pl;
  WidePlan wp{};
  if ((mode == IRL_MVP_AUTO && ld_u <= kRowsMaxUnits) || mode == IRL_MVP_ROWS) {
    IRL_TRY(make_rows_plan(n, ld_u, pl));
    path = IRL_MVP_ROWS;
  } else if ((mode == IRL_MVP_AUTO && ld_u >= kWideMinUnits && make_wide_plan(n, ld_u, cplx, wp) == IRL_OK) ||
             mode == IRL_MVP_WIDE) {
    IRL_TRY(make_wide_plan(n, ld_u, cplx, wp));
    if (ws_bytes < wp.ws) return fail(IRL_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, wp.ws);
    WideArgs wa{};
    wa.O = reinterpret_cast<const double2*>(O);
    wa.n_rows = n;
    wa.ld_u = ld_u;
    wa.v_re = v_re;
    wa.v_im = v_im;
    wa.hf_re = hf_re;
    wa.hf_im = hf_im;
    wa.obar = reinterpret_cast<const double2*>(obar);
    wa.coeff = coeff;
    wa.yadd = yadd;
    wa.u0 = u0;
    wa.out_re = out_re;
    wa.out_im = out_im;
    wa.out0 = out0;
    return launch_wide(wp, cplx, wa, ws, st);
  } else if (mode == IRL_MVP_AUTO || mode == IRL_MVP_FUSED) {
    int rc = make_plan(n, ld_u, cplx, MODE_FUSED, pl);
    if (rc == IRL_OK) {
      path = IRL_MVP_FUSED;
    } else if (mode == IRL_MVP_FUSED) {
      return rc;
    } else {
      path = IRL_MVP_TWO_PASS;
    }
  } else if (mode != IRL_MVP_TWO_PASS) {
    return fail(IRL_ERR_ARG, "bad mvp mode %d", mode);
  }
  StreamArgs a{};
  a.O = reinterpret_cast<const double2*>(O);
  a.n_rows = n;
  a.ld_u = ld_u;
  a.v_re = v_re;
  a.v_im = v_im;
  a.hf_re = hf_re;
  a.hf_im = hf_im;
  a.obar = reinterpret_cast<const double2*>(obar);
  a.coeff0 = coeff;
  a.yadd = yadd;
  if (path == IRL_MVP_FUSED || path == IRL_MVP_ROWS) {
    MvpWs w = mvp_ws_layout(pl, n, ld_u, cplx, ws);
    if (ws_bytes < w.bytes) return fail(IRL_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, w.bytes);
    a.part0 = w.part;
    a.ysum = w.ysum;
    a.spart = w.spart;
    a.gpart = w.gpart;
    if (path == IRL_MVP_ROWS) {
      a.n_rows = n;
      IRL_TRY(launch_rows(pl, cplx, a, st));
    } else {
      IRL_TRY(launch_stream(pl, a, st));
    }
    if (cplx)
      return launch_finish_mvp<true>(w.part, pl.nb, ld_u, w.ysum, a.obar, hf_re, hf_im, u0, out_re, out_im, w.gpart, 1,
                                     out0, st);
    return launch_finish_mvp<false>(w.part, pl.nb, ld_u, w.ysum, a.obar, hf_re, hf_im, u0, out_re, out_im, w.gpart, 1,
                                    out0, st);
  }
  Plan p1, p2;
  IRL_TRY(make_plan(n, ld_u, cplx, MODE_DOT, p1));
  IRL_TRY(make_plan(n, ld_u, cplx, MODE_ACC, p2));
  // both passes must agree on the column split (ACC sums the DOT tile partials)
  if (p1.C != p2.C) return fail(IRL_ERR_DEVICE, "two-pass plans disagree on column split");
  Plan pw = p1;
  pw.nb = std::max(p1.nb, p2.nb);
  MvpWs w = mvp_ws_layout(pw, n, ld_u, cplx, ws);
  if (ws_bytes < w.bytes) return fail(IRL_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, w.bytes);
  a.part0 = w.part;
  a.ysum = w.ysum;
  a.tpart = w.tpart;
  a.spart = w.spart;
  a.gpart = w.gpart;
  IRL_TRY(launch_stream(p1, a, st));
  IRL_TRY(launch_stream(p2, a, st));
  if (cplx)
    return launch_finish_mvp<true>(w.part, p2.nb, ld_u, w.ysum, a.obar, hf_re, hf_im, u0, out_re, out_im, w.gpart,
                                   p1.C, out0, st);
  return launch_finish_mvp<false>(w.part, p2.nb, ld_u, w.ysum, a.obar, hf_re, hf_im, u0, out_re, out_im, w.gpart,
                                  p1.C, out0, st);
}

size_t mvp_ws_bytes(int64_t n, int64_t ld, bool cplx) {
  const int64_t ld_u = cplx ? ld : ld / 2;
  size_t best = 0;
  Plan p;
  if (make_plan(n, ld_u, cplx, MODE_FUSED, p) == IRL_OK) best = std::max(best, mvp_ws_layout(p, n, ld_u, cplx, nullptr).bytes);
  if (make_rows_plan(n, ld_u, p) == IRL_OK) best = std::max(best, mvp_ws_layout(p, n, ld_u, cplx, nullptr).bytes);
  WidePlan wp;
  if (make_wide_plan(n, ld_u, cplx, wp) == IRL_OK) best = std::max(best, wp.ws);
  Plan p1, p2;
  if (make_plan(n, ld_u, cplx, MODE_DOT, p1) == IRL_OK && make_plan(n, ld_u, cplx, MODE_ACC, p2) == IRL_OK) {
    p1.nb = std::max(p1.nb, p2.nb);
    best = std::max(best, mvp_ws_layout(p1, n, ld_u, cplx, nullptr).bytes);
  }
  g_err.clear();
  return best;
}

// ------------------------------------------------------ dual product ---
// H_eff v and S v for the same v (the GEVP form applies both to every
// iterate): rows on the fused single-pass path read O once for both
// (k_stream DUAL); other shapes (rows, wide) run two products.
bool mvp2_fused(int64_t n, int64_t ld_u, bool cplx, Plan& pl) {
  if (ld_u <= kRowsMaxUnits) return false;
  WidePlan wp{};
  if (ld_u >= kWideMinUnits && make_wide_plan(n, ld_u, cplx, wp) == IRL_OK) return false;
  // single-CTA rows only: the 2-CTA cluster plans (cfg3) run their 4-unit instances at 80 registers, where the
  // second accumulator spills and the pair measured slower than two products (4.38 against 4.23 ms)
  // (one ring stage is given to the v slice, so the plan needs four)
  const bool ok = make_plan(n, ld_u, cplx, MODE_FUSED, pl) == IRL_OK && pl.C == 1 && pl.fn_dual && pl.NS >= 4;
  g_err.clear();
  return ok;
}

size_t mvp2_ws_bytes(int64_t n, int64_t ld, bool cplx) {
  const int64_t ld_u = cplx ? ld : ld / 2;
  size_t best = mvp_ws_bytes(n, ld, cplx);
  Plan pl;
  if (mvp2_fused(n, ld_u, cplx, pl))
    best = std::max(best, mvp_ws_layout(pl, n, ld_u, cplx, nullptr).bytes + align256((size_t)pl.nb * ld_u * 16) +
                              align256((size_t)pl.nb * (cplx ? 16 : 8)));
  return best;
}

int mvp2_impl(bool cplx, const double* O, int64_t n, int64_t p, int64_t ld, const double* obar, const double* coeff_a,
              const double* coeff_b, const double* v_re, const double* v_im, double* outa_re, double* outa_im,
              double* outb_re, double* outb_im, const double* hf_re, const double* hf_im, const double* u0,
              double* out0, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!O || !coeff_a || !coeff_b || !v_re || !outa_re || !outb_re) return fail(IRL_ERR_ARG, "null required pointer");
  if (n < 1 || p < 1 || ld < p) return fail(IRL_ERR_ARG, "bad shape n=%lld p=%lld ld=%lld", (long long)n,
                                            (long long)p, (long long)ld);
  if (ld != irl_padded_ld(p, cplx)) return fail(IRL_ERR_ALIGN, "ld must equal irl_padded_ld(p)");
  if (!aligned16(O) || !aligned16(obar) || !aligned16(ws) ||
      (!cplx && (!aligned16(v_re) || !aligned16(outa_re) || !aligned16(outb_re) || !aligned16(hf_re))))
    return fail(IRL_ERR_ALIGN, "pointers must be 16-byte aligned");
  const int64_t ld_u = cplx ? ld : ld / 2;
  Plan pl;
  if (!mvp2_fused(n, ld_u, cplx, pl)) {  // two products (each picks its own path)
    IRL_TRY(mvp_impl(cplx, O, n, p, ld, obar, coeff_a, nullptr, v_re, v_im, outa_re, outa_im, hf_re, hf_im, u0, out0,
                     IRL_MVP_AUTO, ws, ws_bytes, st));
    return mvp_impl(cplx, O, n, p, ld, obar, coeff_b, nullptr, v_re, v_im, outb_re, outb_im, nullptr, nullptr, nullptr,
                    nullptr, IRL_MVP_AUTO, ws, ws_bytes, st);
  }
  const size_t sS = cplx ? 16 : 8;
  MvpWs w = mvp_ws_layout(pl, n, ld_u, cplx, ws);
  const size_t part_b = align256((size_t)pl.nb * ld_u * 16), ysum_b = align256((size_t)pl.nb * sS);
  if (ws_bytes < w.bytes + part_b + ysum_b) return fail(IRL_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes,
                                                        w.bytes + part_b + ysum_b);
  char* extra = static_cast<char*>(ws) + w.bytes;
  StreamArgs a{};
  a.O = reinterpret_cast<const double2*>(O);
  a.n_rows = n;
  a.ld_u = ld_u;
  a.v_re = v_re;
  a.v_im = v_im;
  a.hf_re = hf_re;
  a.hf_im = hf_im;
  a.obar = reinterpret_cast<const double2*>(obar);
  a.coeff0 = coeff_a;
  a.coeff1 = coeff_b;
  a.part0 = w.part;
  a.part1 = reinterpret_cast<double2*>(extra);
  a.ysum = w.ysum;
  a.ysum1 = extra + part_b;
  a.spart = w.spart;
  a.gpart = w.gpart;
  // the second accumulator takes the registers of the v slice: v goes to the
  // shared memory of the last ring stage, the ring runs on one stage less
  Plan pd = pl;
  pd.NS = pl.NS - 1;
  a.vs_off = (pl.smem - (size_t)pl.R * pl.W * 16) & ~size_t(15);
  IRL_TRY(launch_stream(pd, a, st));
  if (cplx) {
    IRL_TRY(launch_finish_mvp<true>(a.part0, pl.nb, ld_u, a.ysum, a.obar, hf_re, hf_im, u0, outa_re, outa_im, w.gpart, 1,
                                    out0, st));
    return launch_finish_mvp<true>(a.part1, pl.nb, ld_u, a.ysum1, a.obar, nullptr, nullptr, nullptr, outb_re, outb_im,
                                   w.gpart, 1, nullptr, st);
  }
  IRL_TRY(launch_finish_mvp<false>(a.part0, pl.nb, ld_u, a.ysum, a.obar, hf_re, hf_im, u0, outa_re, outa_im, w.gpart, 1,
                                   out0, st));
  return launch_finish_mvp<false>(a.part1, pl.nb, ld_u, a.ysum1, a.obar, nullptr, nullptr, nullptr, outb_re, outb_im,
                                  w.gpart, 1, nullptr, st);
}

// --------------------------------------------------------- colstats ----
size_t colstats_bytes(const Plan& p, int64_t ld_u) { return 2 * align256((size_t)p.nb * ld_u * 16); }

int colstats_impl(bool cplx, const double* O, int64_t n, int64_t ld, const double* w, const double* coeff,
                  double* obar, double* g, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!O || !w || !coeff || !obar || !g) return fail(IRL_ERR_ARG, "null pointer");
  if (n < 1 || ld < 1 || (!cplx && (ld & 1))) return fail(IRL_ERR_ARG, "bad shape");
  if (!aligned16(O) || !aligned16(obar) || !aligned16(g) || !aligned16(ws)) return fail(IRL_ERR_ALIGN, "alignment");
  const int64_t ld_u = cplx ? ld : ld / 2;
  Plan p;
  IRL_TRY(make_plan(n, ld_u, cplx, MODE_STATS, p));
  const size_t need = colstats_bytes(p, ld_u);
  if (ws_bytes < need) return fail(IRL_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  StreamArgs a{};
  a.O = reinterpret_cast<const double2*>(O);
  a.n_rows = n;
  a.ld_u = ld_u;
  a.coeff0 = w;
  a.coeff1 = coeff;
  a.part0 = static_cast<double2*>(ws);
  a.part1 = reinterpret_cast<double2*>(static_cast<char*>(ws) + align256((size_t)p.nb * ld_u * 16));
  IRL_TRY(launch_stream(p, a, st));
  const unsigned blocks = (unsigned)cdiv(ld_u, 32);
  if (cplx)
    k_finish_stats<true><<<blocks, 256, 0, st>>>(a.part0, a.part1, p.nb, ld_u, (double2*)obar, (double2*)g);
  else
    k_finish_stats<false><<<blocks, 256, 0, st>>>(a.part0, a.part1, p.nb, ld_u, (double2*)obar, (double2*)g);
  return cuda_check(cudaGetLastError(), "colstats finish launch");
}

// --------------------------------------------------------------- otf ----
// partial-reduction kernels: 32 outputs per CTA (blockDim (32, 8))
unsigned fin_grid(int64_t ld) { return (unsigned)std::min<int64_t>(cdiv(ld, 32), 1 << 20); }

struct OtfPlan {
  int jc, nb, ny;  // nb: the largest row-block count of any acc variant (workspace bound)
  int nkt, kc;     // n-tiles of the acc GEMM (k columns = n_in + ones column, padded to 8)
  int nb_v[2][3];  // row blocks per acc variant [ny - 1][0: RBM, 1: MLP (G and T), 2: MLP (G from T)]
};

// Row blocks for a (jc x nb) grid of equal CTAs: the wave count k in 1..3
// whose floor(k * slots / jc) * jc fills the resident slots best.
int best_row_blocks(int slots, int jc, int64_t n) {
  const int64_t tiles = std::max<int64_t>(1, cdiv(n, OTF_BM));
  int best = 1;
  double best_eff = -1.0;
  for (int k = 1; k <= 3; ++k) {
    const int nb = (int)std::min<int64_t>(tiles, std::max(1, k * slots / jc));
    const int64_t ctas = (int64_t)nb * jc;
    const double eff = (double)ctas / (double)(cdiv(ctas, slots) * slots);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = nb;
    }
  }
  return best;
}

using AccFn = void (*)(OtfArgs, CUtensorMap, CUtensorMap);

// 2-D TMA descriptor of a row-major rows x cols f64 matrix, boxes of 64 rows x
// 16 columns with the 128-byte swizzle (the acc GEMM tiles).  Cached per
// (pointer, shape): encoding is host work on every product otherwise.
int tile_map(CUtensorMap& m, const double* base, int64_t cols, int64_t rows) {
  static std::once_flag once;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    cudaGetLastError();
  });
  if (!encode) return fail(IRL_ERR_DEVICE, "cuTensorMapEncodeTiled is unavailable");
  struct Key {
    const double* p;
    int64_t c, r;
  };
  thread_local Key keys[16];
  thread_local CUtensorMap maps[16];
  thread_local int used = 0, next = 0;
  for (int i = 0; i < used; ++i)
    if (keys[i].p == base && keys[i].c == cols && keys[i].r == rows) {
      m = maps[i];
      return IRL_OK;
    }
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((cols * 8) & 15))
    return fail(IRL_ERR_ALIGN, "tile map needs 16-byte aligned rows");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 8};
  cuuint32_t box[2] = {16, (cuuint32_t)OTF_BM};
  cuuint32_t es[2] = {1, 1};
  const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(IRL_ERR_ARG, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  const int slot = used < 16 ? used++ : (next++ & 15);
  keys[slot] = Key{base, cols, rows};
  maps[slot] = m;
  return IRL_OK;
}

AccFn pick_acc(int nkt, int nyv, bool has_t) {
#define IRL_ACC(NK, NYV, HT) \
  if (nkt == NK && nyv == NYV && has_t == HT) return k_otf_acc<NK, NYV, HT>;
  IRL_ACC(3, 1, true) IRL_ACC(3, 2, true) IRL_ACC(3, 1, false) IRL_ACC(3, 2, false)
  IRL_ACC(6, 1, true) IRL_ACC(6, 2, true) IRL_ACC(6, 1, false) IRL_ACC(6, 2, false)
  IRL_ACC(13, 1, true) IRL_ACC(13, 1, false)
#undef IRL_ACC
  return nullptr;
}

// gu: G formed from T inside the kernel (OtfArgs::u), one tile per stage
size_t acc_smem(int nyv, bool has_t, bool gu = false) {
  const size_t st = OTF_ACC_STAGES;
  return 1024 + (st * OTF_TILE * (has_t && !gu ? 2 : 1) + st * OTF_BM * OTF_XW + (size_t)nyv * st * OTF_BM) * 8 +
         2 * st * 8;
}

int make_otf_plan_uncached(int64_t n, int n_in, int hidden, OtfPlan& p) {
  DevInfo d;
  IRL_TRY(dev_info(d));
  if (n_in < 1 || n_in > OTF_MAX_NIN) return fail(IRL_ERR_ARG, "on-the-fly mode supports n_in <= %d", OTF_MAX_NIN);
  p.jc = (int)cdiv(hidden, OTF_BJ);
  p.ny = 4 * d.sms;  // row-parallel helper kernels (y, dots): 4 CTAs per SM
  p.nkt = (n_in + 1 + 7) / 8 <= 3 ? 3 : (n_in + 1 + 7) / 8 <= 6 ? 6 : 13;
  p.kc = 8 * p.nkt;
  p.nb = 1;
  IRL_TRY(ensure_fn_attrs((const void*)k_otf_dot<true>, d.smem_optin));
  IRL_TRY(ensure_fn_attrs((const void*)k_otf_dot<true, true>, d.smem_optin));
  IRL_TRY(ensure_fn_attrs((const void*)k_otf_dot<false>, d.smem_optin));
  IRL_TRY(ensure_fn_attrs((const void*)k_otf_dot<false, true>, d.smem_optin));
  for (int nyv = 1; nyv <= 2; ++nyv)
    for (int ht = 0; ht < 3; ++ht) {
      p.nb_v[nyv - 1][ht] = 0;
      if (ht == 2 && nyv != 1) continue;  // G from T: product only
      AccFn f = pick_acc(p.nkt, nyv, ht != 0);
      if (!f) continue;
      IRL_TRY(ensure_fn_attrs((const void*)f, d.smem_optin));
      int occ = 0;
      IRL_TRY(cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)f, 288,
                                                                       acc_smem(nyv, ht != 0, ht == 2)),
                         "occ"));
      p.nb_v[nyv - 1][ht] = best_row_blocks(d.sms * std::max(occ, 1), p.jc, n);
      p.nb = std::max(p.nb, p.nb_v[nyv - 1][ht]);
    }
  return IRL_OK;
}

int make_otf_plan(int64_t n, int n_in, int hidden, OtfPlan& p) {
  struct Entry {
    int rc;
    OtfPlan plan;
    std::string err;
  };
  static std::mutex mu;
  static std::unordered_map<std::string, Entry> cache;
  int dev = 0;
  IRL_TRY(cuda_check(cudaGetDevice(&dev), "cudaGetDevice"));
  char key[96];
  snprintf(key, sizeof(key), "%lld/%d/%d/%d", (long long)n, n_in, hidden, dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      p = it->second.plan;
      if (it->second.rc != IRL_OK) g_err = it->second.err;
      return it->second.rc;
    }
  }
  Entry e{};
  e.rc = make_otf_plan_uncached(n, n_in, hidden, e.plan);
  if (e.rc == IRL_ERR_CUDA) return e.rc;  // transient: do not cache
  if (e.rc != IRL_OK) e.err = g_err;
  p = e.plan;
  std::lock_guard<std::mutex> lk(mu);
  cache.emplace(key, e);
  return e.rc;
}

struct OtfWs {
  double *tpart, *y, *ypart, *dpart, *gpart, *part, *partu, *xpart, *ypart2;
  size_t bytes;
};

OtfWs otf_ws_layout(const OtfPlan& p, int64_t n, int hidden, void* base) {
  OtfWs w{};
  size_t off = 0;
  auto carve = [&](size_t b) {
    double* r = base ? reinterpret_cast<double*>(static_cast<char*>(base) + off) : nullptr;
    off += align256(b);
    return r;
  };
  w.tpart = carve((size_t)p.jc * n * 8);
  w.y = carve((size_t)n * 8);
  w.ypart = carve((size_t)p.ny * 8);
  w.dpart = carve((size_t)p.ny * 8);
  w.gpart = carve((size_t)p.ny * 8);
  w.part = carve((size_t)2 * p.nb * hidden * p.kc * 8);
  w.partu = carve((size_t)2 * p.nb * hidden * 8);
  w.xpart = carve((size_t)4 * 148 * (OTF_MAX_NIN + 1) * 8);
  w.ypart2 = carve((size_t)4 * 148 * 8);
  w.bytes = off;
  return w;
}

int otf_check(const uint64_t* xbits, const double* t, const double* g, int64_t n, int n_in, int hidden, int64_t ld) {
  if (!xbits || !t || !g) return fail(IRL_ERR_ARG, "null pointer");
  if (n < 1 || hidden < 1 || n_in < 1) return fail(IRL_ERR_ARG, "bad shape");
  const int64_t P = (int64_t)hidden * n_in + 2 * (int64_t)hidden + 1;
  if (ld != irl_padded_ld(P, 0)) return fail(IRL_ERR_ALIGN, "ld must equal irl_padded_ld(P=%lld)", (long long)P);
  if (!aligned16(xbits) || !aligned16(t) || !aligned16(g) || (hidden & 1))
    return fail(IRL_ERR_ALIGN, "on-the-fly operands must be 16-byte aligned with an even hidden width");
  return IRL_OK;
}

size_t otf_dot_smem(int n_in, bool has_t, bool cplx, bool gu = false) {
  const int vs = otf_vstride(n_in);
  const size_t st = OTF_DOT_STAGES;
  const size_t tiles = st * OTF_TILE * (has_t && !gu ? 2 : 1);
  const size_t red = (size_t)2 * 4 * OTF_BM * (cplx ? 2 : 1);
  return 1024 + (tiles + st * OTF_BM * OTF_XW + red + 2 * st + OTF_BJ * 3 + (size_t)OTF_BJ * vs) * 8;
}

// persistent grid of the dot kernels: every resident CTA slot, occupancy cached per (kernel, n_in)
int otf_dot_grid(const void* fn, size_t smem, int key, int& grid) {
  static std::mutex mu;
  static std::unordered_map<int, int> cache;
  DevInfo d;
  IRL_TRY(dev_info(d));
  int dev = 0;
  cudaGetDevice(&dev);
  const int k = (key << 8) ^ dev;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(k);
    if (it != cache.end()) {
      grid = it->second;
      return IRL_OK;
    }
  }
  IRL_TRY(ensure_fn_attrs(fn, d.smem_optin));
  int occ = 0;
  IRL_TRY(cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 288, smem), "occ"));
  grid = d.sms * std::max(occ, 1);
  std::lock_guard<std::mutex> lk(mu);
  cache[k] = grid;
  return IRL_OK;
}

// Launch with programmatic stream serialisation (the kernel must begin its
// global-memory work with griddepcontrol.wait: pdl_enter() in otf.cuh).
template <typename... KArgs, typename... Args>
int launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, const char* what,
               Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cuda_check(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...), what);
}

constexpr int kOtfLowRegMaxNin = 40;

int otf_dot_launch(OtfArgs& a, bool has_t, cudaStream_t st) {
  const bool low = a.n_in <= kOtfLowRegMaxNin && !getenv("IRL_OTF_NO_LOWREG");
  const void* fn = has_t ? (low ? (const void*)k_otf_dot<true, true> : (const void*)k_otf_dot<true>)
                         : (low ? (const void*)k_otf_dot<false, true> : (const void*)k_otf_dot<false>);
  const bool gu = has_t && a.u != nullptr;
  const size_t smem = otf_dot_smem(a.n_in, has_t, false, gu);
  int grid = 0;
  IRL_TRY(otf_dot_grid(fn, smem, (a.n_in << 4) | (low ? 8 : 0) | (gu ? 4 : 0) | (has_t ? 1 : 0), grid));
  CUtensorMap mg, mt;
  IRL_TRY(tile_map(mg, a.G, a.hidden, a.n_rows));
  if (has_t)
    IRL_TRY(tile_map(mt, a.T, a.hidden, a.n_rows));
  else
    mt = mg;
  if (has_t && low) return launch_pdl(k_otf_dot<true, true>, dim3(grid), dim3(288), smem, st, "otf dot launch", a, mg, mt);
  if (has_t) return launch_pdl(k_otf_dot<true>, dim3(grid), dim3(288), smem, st, "otf dot launch", a, mg, mt);
  if (low) return launch_pdl(k_otf_dot<false, true>, dim3(grid), dim3(288), smem, st, "otf dot launch", a, mg, mt);
  return launch_pdl(k_otf_dot<false>, dim3(grid), dim3(288), smem, st, "otf dot launch", a, mg, mt);
}

// launches the acc GEMM variant; a.nb = its row-block count (the partial stride)
int otf_acc_launch(const OtfPlan& pl, OtfArgs& a, cudaStream_t st, int nyv, bool has_t) {
  AccFn f = pick_acc(pl.nkt, nyv, has_t);
  if (!f) return fail(IRL_ERR_DEVICE, "no acc GEMM instance for nkt=%d ny=%d", pl.nkt, nyv);
  const bool gu = has_t && nyv == 1 && a.u != nullptr;
  a.nb = pl.nb_v[nyv - 1][has_t ? (gu ? 2 : 1) : 0];
  dim3 grid((unsigned)pl.jc, (unsigned)a.nb);
  CUtensorMap mg, mt;
  IRL_TRY(tile_map(mg, a.G, a.hidden, a.n_rows));
  if (has_t)
    IRL_TRY(tile_map(mt, a.T, a.hidden, a.n_rows));
  else
    mt = mg;
  return launch_pdl(f, grid, dim3(288), acc_smem(nyv, has_t, gu), st, "otf acc launch", a, mg, mt);
}

// column statistics (obar = sum w O, grad = sum c O) of a real model from the
// hidden activations: one GEMM pass for both weight vectors when they fit
int otf_stats(const OtfPlan& pl, OtfArgs a, const OtfWs& wl, int model, int64_t n, int n_in, int hidden,
              int64_t ld, const double* w, const double* coeff, double* obar, double* grad, double* xpart, int nbx,
              cudaStream_t st) {
  const bool has_t = model == MODEL_MLP;  // the RBM has no u block: G-only tiles
  const double* ys[2] = {w, coeff};
  double* outs[2] = {obar, grad};
  a.part = wl.part;
  a.partu = wl.partu;
  const int nyv = pl.nkt <= 6 ? 2 : 1;
  for (int q0 = 0; q0 < 2; q0 += nyv) {
    a.y = ys[q0];
    a.y2 = nyv == 2 ? ys[q0 + 1] : nullptr;
    IRL_TRY(otf_acc_launch(pl, a, st, nyv, has_t));
    for (int q = q0; q < q0 + nyv; ++q) {
      const double* part = wl.part + (size_t)(q - q0) * a.nb * hidden * pl.kc;
      const double* partu = wl.partu + (size_t)(q - q0) * a.nb * hidden;
      if (model == MODEL_MLP) {
        k_vsum<<<pl.ny, 256, 0, st>>>(ys[q], n, wl.ypart);
        k_otf_finish<<<fin_grid(ld), dim3(32, 8), 0, st>>>(part, partu, a.nb, hidden, n_in, pl.kc, ld, wl.ypart,
                                                             pl.ny, nullptr, nullptr, nullptr, nullptr, 0, outs[q],
                                                             nullptr);
      } else {
        double* xp = xpart ? xpart : wl.xpart;
        k_xsum<<<nbx, 128, 0, st>>>(a.xbits, ys[q], n, n_in, xp, wl.ypart2);
        k_rbm_stats_finish<<<fin_grid(ld), dim3(32, 8), 0, st>>>(part, a.nb, hidden, n_in, pl.kc, xp, nbx, ld,
                                                                    outs[q]);
      }
      IRL_TRY(cuda_check(cudaGetLastError(), "stats finish launch"));
    }
  }
  return IRL_OK;
}


// complex-parameter RBM on the fly (hermitian kind): T viewed as N x 2h real
struct OtfCPlan {
  int jc, nb_dot, nb_acc, ny, nbx;
  int nkt, kc;
  size_t smem_dot, smem_acc;
};

using AccCFn = void (*)(OtfCArgs, CUtensorMap);

AccCFn pick_acc_c(int nkt) {
  switch (nkt) {
    case 3: return k_otf_acc_c<3>;
    case 6: return k_otf_acc_c<6>;
    case 8: return k_otf_acc_c<8>;
    case 13: return k_otf_acc_c<13>;
    default: return nullptr;
  }
}

int make_otfc_plan_uncached(int64_t n, int n_in, int hidden, OtfCPlan& p) {
  DevInfo d;
  IRL_TRY(dev_info(d));
  if (n_in < 1 || n_in > OTF_MAX_NIN) return fail(IRL_ERR_ARG, "on-the-fly mode supports n_in <= %d", OTF_MAX_NIN);
  p.jc = (int)cdiv(2LL * hidden, OTF_BJ);
  const int k8 = (n_in + 1 + 7) / 8;
  p.nkt = k8 <= 3 ? 3 : k8 <= 6 ? 6 : k8 <= 8 ? 8 : 13;
  p.kc = 8 * p.nkt;
  p.smem_dot = otf_dot_smem(n_in, false, true);
  p.smem_acc = 1024 + (size_t)OTF_ACC_STAGES * (OTF_TILE * 8 + OTF_BM * OTF_XW * 8 + OTF_BM * 16 + 16);
  AccCFn acc = pick_acc_c(p.nkt);
  IRL_TRY(ensure_fn_attrs((const void*)k_otf_dot_c, d.smem_optin));
  IRL_TRY(ensure_fn_attrs((const void*)acc, d.smem_optin));
  int occ_d = 1, occ_a = 1;
  IRL_TRY(cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_d, (const void*)k_otf_dot_c, 288, p.smem_dot),
                     "occ"));
  IRL_TRY(cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_a, (const void*)acc, 288, p.smem_acc), "occ"));
  p.nb_dot = d.sms * std::max(occ_d, 1);  // persistent grid
  p.nb_acc = best_row_blocks(d.sms * std::max(occ_a, 1), p.jc, n);
  p.ny = 4 * d.sms;  // row-parallel helper kernels (y, dots): 4 CTAs per SM
  p.nbx = std::min<int>(4 * d.sms, (int)std::max<int64_t>(1, n / 64));
  return IRL_OK;
}

int make_otfc_plan(int64_t n, int n_in, int hidden, OtfCPlan& p) {
  struct Entry {
    int rc;
    OtfCPlan plan;
    std::string err;
  };
  static std::mutex mu;
  static std::unordered_map<std::string, Entry> cache;
  int dev = 0;
  IRL_TRY(cuda_check(cudaGetDevice(&dev), "cudaGetDevice"));
  char key[96];
  snprintf(key, sizeof(key), "%lld/%d/%d/%d", (long long)n, n_in, hidden, dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      p = it->second.plan;
      if (it->second.rc != IRL_OK) g_err = it->second.err;
      return it->second.rc;
    }
  }
  Entry e{};
  e.rc = make_otfc_plan_uncached(n, n_in, hidden, e.plan);
  if (e.rc == IRL_ERR_CUDA) return e.rc;
  if (e.rc != IRL_OK) e.err = g_err;
  p = e.plan;
  std::lock_guard<std::mutex> lk(mu);
  cache.emplace(key, e);
  return e.rc;
}

struct OtfCWs {
  double2 *tpart, *y, *ypart, *dpart, *xpart;
  double *gpart, *part;
  size_t bytes;
};

OtfCWs otfc_ws_layout(const OtfCPlan& p, int64_t n, int n_in, int hidden, void* base) {
  OtfCWs w{};
  size_t off = 0;
  auto carve = [&](size_t b) {
    char* r = base ? static_cast<char*>(base) + off : nullptr;
    off += align256(b);
    return r;
  };
  w.tpart = reinterpret_cast<double2*>(carve((size_t)p.jc * n * 16));
  w.y = reinterpret_cast<double2*>(carve((size_t)n * 16));
  w.ypart = reinterpret_cast<double2*>(carve((size_t)p.ny * 16));
  w.dpart = reinterpret_cast<double2*>(carve((size_t)p.ny * 16));
  w.xpart = reinterpret_cast<double2*>(carve((size_t)p.nbx * n_in * 16));
  w.gpart = reinterpret_cast<double*>(carve((size_t)p.ny * 8));
  w.part = reinterpret_cast<double*>(carve((size_t)p.nb_acc * 2 * hidden * p.kc * 8));
  w.bytes = off;
  return w;
}

int otfc_check(const uint64_t* xbits, const double* t, int64_t n, int n_vis, int hidden, int64_t ld) {
  if (!xbits || !t) return fail(IRL_ERR_ARG, "null pointer");
  if (n < 1 || hidden < 1 || n_vis < 1) return fail(IRL_ERR_ARG, "bad shape");
  if (n_vis > OTF_MAX_NIN) return fail(IRL_ERR_ARG, "on-the-fly mode supports n_vis <= %d", OTF_MAX_NIN);
  const int64_t P = (int64_t)n_vis + hidden + (int64_t)hidden * n_vis;
  if (ld != irl_padded_ld(P, 1)) return fail(IRL_ERR_ALIGN, "ld must equal irl_padded_ld(P=%lld, complex)", (long long)P);
  if (!aligned16(xbits) || !aligned16(t)) return fail(IRL_ERR_ALIGN, "on-the-fly operands must be 16-byte aligned");
  return IRL_OK;
}

// Sum_n conj(O_n) y_n for the complex RBM -> out_c (interleaved), conj'd when conj_out
int otfc_colsum(const OtfCPlan& pl, OtfCArgs a, const OtfCWs& wl, int64_t ld, const double2* y, const double* yr,
                double2* out_c, int conj_out, cudaStream_t st) {
  a.y = y;
  a.yr = yr;
  a.part = wl.part;
  a.nb = pl.nb_acc;
  {
    CUtensorMap mt;
    IRL_TRY(tile_map(mt, a.T, 2LL * a.hidden, a.n_rows));
    pick_acc_c(pl.nkt)<<<dim3((unsigned)pl.jc, (unsigned)pl.nb_acc), 288, pl.smem_acc, st>>>(a, mt);
  }
  IRL_TRY(cuda_check(cudaGetLastError(), "otf acc (complex) launch"));
  k_xsum_c<<<pl.nbx, 128, 0, st>>>(a.xbits, y, yr, a.n_rows, a.n_in, wl.xpart);
  k_rbm_otf_finish_c<<<fin_grid(ld), dim3(32, 8), 0, st>>>(wl.part, pl.nb_acc, a.hidden, a.n_in, pl.kc, wl.xpart,
                                                             pl.nbx, nullptr, 0, ld, nullptr, nullptr, nullptr,
                                                             nullptr, nullptr, 0, nullptr, nullptr, nullptr, out_c,
                                                             conj_out);
  return cuda_check(cudaGetLastError(), "otf finish (complex) launch");
}

// ------------------------------------------------------------ obuild ----
struct OPlan {
  int C, W, PPT, NT, nb;
  size_t smem;
  void (*fn)(ORowArgs, int);
};

template <bool CPLX, int MODEL, bool STATS>
void (*pick_orows(int ppt))(ORowArgs, int) {
  switch (ppt) {
    case 1: return k_orows<CPLX, MODEL, 1, STATS>;
    case 2: return k_orows<CPLX, MODEL, 2, STATS>;
    case 4: return k_orows<CPLX, MODEL, 4, STATS>;
    default: return k_orows<CPLX, MODEL, 8, STATS>;
  }
}

// real models with n_in <= 100 and an even hidden width take their column
// statistics from the DMMA GEMM (k_otf_acc) instead of the row writer
// (measured: for the narrow RBM hidden layers the fused writer statistics win)
// Row-sweeping writer (k_orows_sweep): real models with unit-aligned blocks
// (even n; the RBM also needs an even h), its statistics from the DMMA GEMMs.
// Measured (B200): MLP cfg5 37.7 -> 23.3 ms, cfg3 equal; the RBM's column-tile
// writer with fused statistics stays faster (cfg2 0.78 vs 1.00 ms), so the RBM
// sweeps only with IRL_OBUILD_SWEEP=2; IRL_OBUILD_SWEEP=0 disables it.
bool sweep_ok(bool cplx, int model, int n_vis, int hidden) {
  static const int mode = getenv("IRL_OBUILD_SWEEP") ? atoi(getenv("IRL_OBUILD_SWEEP")) : 1;
  if (mode == 0) return false;
  if (cplx)  // complex-theta RBM (cfg4: 470 KB rows): statistics from the complex DMMA colsums
    return model == MODEL_RBM && n_vis <= OTF_MAX_NIN && n_vis <= 32 * SWEEP_UQ;
  if ((n_vis & 1) || (hidden & 1) || n_vis > 2 * 32 * SWEEP_UQ) return false;  // 16-byte factor rows
  return model == MODEL_MLP || mode == 2;
}

bool gemm_stats(bool cplx, int model, int n_vis, int hidden) {
  if (cplx) return sweep_ok(cplx, model, n_vis, hidden);
  if (n_vis > OTF_MAX_NIN || (hidden & 1)) return false;
  return model == MODEL_MLP || sweep_ok(cplx, model, n_vis, hidden);
}

int make_oplan(int64_t ld_u, bool cplx, int model, OPlan& p, bool stats_in_writer) {
  DevInfo d;
  IRL_TRY(dev_info(d));
  // write-bound: prefer few units per thread (low registers, several CTAs per
  // SM with independent row barriers); column tiles may be uneven
  const char* fc = getenv("IRL_OBUILD_C");     // tuning overrides
  const char* fp = getenv("IRL_OBUILD_PPT");
  const int c_force = fc ? atoi(fc) : 0, p_force = fp ? atoi(fp) : 0;
  for (int64_t C = std::max(1, c_force); C <= 4096; ++C) {
    for (int ppt : {1, 2, 4, 8}) {
      if (p_force && ppt != p_force) continue;
      const int64_t W = cdiv(ld_u, C);
      int64_t nt = rup(cdiv(W, ppt), 32);
      if (nt > 512) continue;
      if (nt < 64) nt = 64;
      p.C = (int)C;
      p.W = (int)W;
      p.PPT = ppt;
      p.NT = (int)nt;
      if (cplx)
        p.fn = pick_orows<true, MODEL_RBM, true>(ppt);
      else if (stats_in_writer)
        p.fn = model == MODEL_RBM ? pick_orows<false, MODEL_RBM, true>(ppt) : pick_orows<false, MODEL_MLP, true>(ppt);
      else
        p.fn = model == MODEL_RBM ? pick_orows<false, MODEL_RBM, false>(ppt) : pick_orows<false, MODEL_MLP, false>(ppt);
      p.smem = 0;
      int occ = 0;
      IRL_TRY(cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)p.fn, p.NT, 0), "occ"));
      occ = std::max(occ, 1);
      p.nb = std::max(1, (int)((d.sms * occ + C - 1) / C));
      return IRL_OK;
    }
  }
  return fail(IRL_ERR_DEVICE, "no O-build geometry");
}

size_t obuild_bytes(const OPlan& p, int model, int64_t n, int n_vis, int hidden, int64_t ld_u, bool cplx) {
  const size_t sS = cplx ? 16 : 8;
  size_t b = align256((size_t)n * hidden * sS);                    // t
  if (model == MODEL_MLP) b += align256((size_t)n * hidden * 8);    // g
  b += align256((size_t)n * OTF_XW * 8);                           // packed inputs
  b += align256((size_t)n * (cplx ? n_vis : (n_vis + 1) & ~1) * sS);  // inputs as table entries
  if (gemm_stats(cplx, model, n_vis, hidden)) {                           // DMMA stats scratch
    if (cplx) {
      OtfCPlan op;
      if (make_otfc_plan(n, n_vis, hidden, op) == IRL_OK) b += otfc_ws_layout(op, n, n_vis, hidden, nullptr).bytes;
    } else {
      OtfPlan op;
      if (make_otf_plan(n, n_vis, hidden, op) == IRL_OK) b += otf_ws_layout(op, n, hidden, nullptr).bytes;
    }
    b += align256((size_t)148 * 4 * (n_vis + 1) * 8);             // x sums
  }
  b += 2 * align256((size_t)p.nb * ld_u * 16);                     // partials
  return b;
}

template <bool CPLX, int MODEL>
int launch_hidden(const uint8_t* x, const uint64_t* xbits, int64_t n, int n_vis, int hidden, const void* Wm,
                  const void* bvec, const double* uvec, void* T, double* G, cudaStream_t st) {
  using S = typename Traits<CPLX>::S;
  DevInfo d;
  IRL_TRY(dev_info(d));
  if (xbits && n_vis <= OTF_MAX_NIN && (CPLX || (hidden & 1) == 0)) {
    // FP64 tensor-core path (DMMA): PRE = X W^T + b, activation in the epilogue
    auto fn = k_hidden_mma<CPLX, MODEL>;
    const size_t smem = (size_t)(64 * OTF_MAX_NIN + 64) * 8;
    IRL_TRY(ensure_fn_attrs((const void*)fn, d.smem_optin));
    const int ncols = CPLX ? 2 * hidden : hidden;
    const int jc = (int)cdiv(ncols, 64);
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 64), cdiv((int64_t)d.sms * 4, jc)));
    fn<<<dim3((unsigned)jc, (unsigned)nb), 256, smem, st>>>(xbits, n, n_vis, hidden, (const double*)Wm,
                                                           (const double*)bvec, uvec, (double*)T, G, nb);
    return cuda_check(cudaGetLastError(), "hidden (mma) kernel launch");
  }
  const size_t smem = (size_t)n_vis * 32 * sizeof(S);
  if (smem > (size_t)d.smem_optin) return fail(IRL_ERR_ARG, "n_vis too large");
  auto fn = k_hidden<CPLX, MODEL>;
  IRL_TRY(ensure_fn_attrs((const void*)fn, d.smem_optin));
  const int jt = (int)cdiv(hidden, 32);
  int64_t rb = std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 8), cdiv((int64_t)d.sms * 8, jt)));
  dim3 grid((unsigned)rb, (unsigned)jt);
  fn<<<grid, 256, smem, st>>>(x, n, n_vis, hidden, (const S*)Wm, (const S*)bvec, uvec, (S*)T, G);
  return cuda_check(cudaGetLastError(), "hidden kernel launch");
}

int pack_bits(const uint8_t* x, int64_t n, int n_vis, uint64_t* xbits, cudaStream_t st) {
  DevInfo d;
  IRL_TRY(dev_info(d));
  k_pack_bits<<<(unsigned)std::min<int64_t>(cdiv(n, 256), 4 * d.sms), 256, 0, st>>>(x, n, n_vis, xbits);
  return cuda_check(cudaGetLastError(), "pack bits launch");
}

// A second stream per device for work that overlaps the caller's stream (the
// O-build's hidden layer and FP64-tensor statistics beside its HBM-write-bound
// row writer).  Fork / join by events recorded per call, so the caller's
// stream order (and graph capture of it) is kept.
int side_stream(cudaStream_t& out) {
  static std::mutex mu;
  static cudaStream_t streams[64] = {};
  int dev = 0;
  IRL_TRY(cuda_check(cudaGetDevice(&dev), "cudaGetDevice"));
  if (dev < 0 || dev >= 64) return fail(IRL_ERR_DEVICE, "device index %d", dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!streams[dev]) IRL_TRY(cuda_check(cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking), "side stream"));
  out = streams[dev];
  return IRL_OK;
}

struct Fork {
  cudaStream_t main = nullptr, side = nullptr;
  cudaEvent_t ev = nullptr;
  int begin(cudaStream_t st) {  // side waits for everything issued on st so far
    main = st;
    IRL_TRY(side_stream(side));
    IRL_TRY(cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "fork event"));
    IRL_TRY(cuda_check(cudaEventRecord(ev, st), "fork record"));
    return cuda_check(cudaStreamWaitEvent(side, ev, 0), "fork wait");
  }
  int join() {  // st waits for everything issued on side since begin()
    IRL_TRY(cuda_check(cudaEventRecord(ev, side), "join record"));
    IRL_TRY(cuda_check(cudaStreamWaitEvent(main, ev, 0), "join wait"));
    return cuda_check(cudaEventDestroy(ev), "join event");
  }
};

// column statistics Obar = sum w conj(O), F/2 = sum c conj(O) from the hidden
// activations and the packed inputs (no O read): the DMMA GEMMs of the
// on-the-fly product with y = w and y = c
int obuild_stats(bool cplx, int model, const uint64_t* xbits, const void* T, const double* G, int64_t n, int n_vis,
                 int hidden, int64_t ld, const double* w, const double* coeff, double* obar, double* g, char* scratch,
                 cudaStream_t st) {
  if (cplx) {
    // complex theta: obar = conj(sum w conj(O)), grad = sum c conj(O) from the
    // real N x 2h view of T (as irl_otf_colstats_rbm_c128)
    OtfCPlan op;
    IRL_TRY(make_otfc_plan(n, n_vis, hidden, op));
    OtfCWs wl = otfc_ws_layout(op, n, n_vis, hidden, scratch);
    OtfCArgs oa{};
    oa.xbits = xbits;
    oa.T = reinterpret_cast<const double*>(T);
    oa.n_rows = n;
    oa.n_in = n_vis;
    oa.hidden = hidden;
    IRL_TRY(otfc_colsum(op, oa, wl, ld, nullptr, w, reinterpret_cast<double2*>(obar), 1, st));
    return otfc_colsum(op, oa, wl, ld, reinterpret_cast<const double2*>(coeff), nullptr,
                       reinterpret_cast<double2*>(g), 0, st);
  }
  OtfPlan op;
  IRL_TRY(make_otf_plan(n, n_vis, hidden, op));
  OtfWs wl = otf_ws_layout(op, n, hidden, scratch);
  double* xpart = reinterpret_cast<double*>(scratch + align256(wl.bytes));
  OtfArgs oa{};
  oa.xbits = xbits;
  oa.T = reinterpret_cast<const double*>(T);
  oa.G = model == MODEL_MLP ? G : reinterpret_cast<const double*>(T);
  oa.n_rows = n;
  oa.n_in = n_vis;
  oa.hidden = hidden;
  DevInfo d;
  IRL_TRY(dev_info(d));
  const int nbx = std::min<int>(4 * d.sms, (int)std::max<int64_t>(1, n / 64));
  return otf_stats(op, oa, wl, model, n, n_vis, hidden, ld, w, coeff, obar, g, xpart, nbx, st);
}

int obuild_impl(bool cplx, int model, const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta,
                double* O, int64_t ld, const double* w, const double* coeff, double* obar, double* g, void* ws,
                size_t ws_bytes, cudaStream_t st) {
  if (!x || !theta || !O || !w || !coeff || !obar || !g) return fail(IRL_ERR_ARG, "null pointer");
  if (n < 1 || n_vis < 1 || hidden < 1 || n_vis > 4095 || hidden > 65535) return fail(IRL_ERR_ARG, "bad shape");
  const int64_t P = model == MODEL_RBM ? (int64_t)n_vis + hidden + (int64_t)hidden * n_vis
                                       : (int64_t)hidden * n_vis + 2 * (int64_t)hidden + 1;
  if (ld != irl_padded_ld(P, cplx)) return fail(IRL_ERR_ALIGN, "ld must equal irl_padded_ld(P=%lld)", (long long)P);
  if (!aligned16(O) || !aligned16(obar) || !aligned16(g) || !aligned16(ws)) return fail(IRL_ERR_ALIGN, "alignment");
  const int64_t ld_u = cplx ? ld : ld / 2;
  const bool gstats = gemm_stats(cplx, model, n_vis, hidden);
  OPlan p;
  IRL_TRY(make_oplan(ld_u, cplx, model, p, !gstats));
  const size_t need = obuild_bytes(p, model, n, n_vis, hidden, ld_u, cplx);
  if (ws_bytes < need) return fail(IRL_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  const size_t sS = cplx ? 16 : 8;
  char* base = static_cast<char*>(ws);
  void* T = base;
  size_t off = align256((size_t)n * hidden * sS);
  double* G = nullptr;
  if (model == MODEL_MLP) {
    G = reinterpret_cast<double*>(base + off);
    off += align256((size_t)n * hidden * 8);
  }
  double2* part0 = reinterpret_cast<double2*>(base + off);
  off += align256((size_t)p.nb * ld_u * 16);
  double2* part1 = reinterpret_cast<double2*>(base + off);
  off += align256((size_t)p.nb * ld_u * 16);
  uint64_t* xbits = nullptr;
  if (n_vis <= OTF_MAX_NIN) {
    xbits = reinterpret_cast<uint64_t*>(base + off);
    IRL_TRY(pack_bits(x, n, n_vis, xbits, st));
  }
  off += align256((size_t)n * OTF_XW * 8);
  const int xrow = cplx ? n_vis : (n_vis + 1) & ~1;
  void* xd = base + off;
  off += align256((size_t)n * xrow * sS);
  const bool sweep = gstats && sweep_ok(cplx, model, n_vis, hidden);
  if (!sweep) {  // table entries of the inputs: the column-tile writer only
    const int64_t total = n * xrow;
    const unsigned grid = (unsigned)std::min<int64_t>(cdiv(total, 256), 4 * 148 * 8);
    if (cplx)
      k_x_expand<true><<<grid, 256, 0, st>>>(x, n, n_vis, xrow, reinterpret_cast<double2*>(xd));
    else
      k_x_expand<false><<<grid, 256, 0, st>>>(x, n, n_vis, xrow, reinterpret_cast<double*>(xd));
    IRL_TRY(cuda_check(cudaGetLastError(), "x expand launch"));
  }
  // hidden layer of rows [r0, r0 + rows) (row offsets into x, xbits, T, G)
  auto hidden_rows = [&](int64_t r0, int64_t rows, cudaStream_t hs) -> int {
    const uint8_t* xr = x + r0 * n_vis;
    const uint64_t* xb = xbits ? xbits + r0 * OTF_XW : nullptr;
    if (model == MODEL_RBM) {
      const double* bvec = theta + (size_t)n_vis * (cplx ? 2 : 1);
      const double* Wm = theta + (size_t)(n_vis + hidden) * (cplx ? 2 : 1);
      void* Tr = static_cast<char*>(T) + (size_t)r0 * hidden * sS;
      if (cplx) return launch_hidden<true, MODEL_RBM>(xr, xb, rows, n_vis, hidden, Wm, bvec, nullptr, Tr, nullptr, hs);
      return launch_hidden<false, MODEL_RBM>(xr, xb, rows, n_vis, hidden, Wm, bvec, nullptr, Tr, nullptr, hs);
    }
    const double* Wm = theta;
    const double* bvec = theta + (size_t)hidden * n_vis;
    const double* uvec = bvec + hidden;
    return launch_hidden<false, MODEL_MLP>(xr, xb, rows, n_vis, hidden, Wm, bvec, uvec,
                                           static_cast<char*>(T) + (size_t)r0 * hidden * sS, G + (size_t)r0 * hidden, hs);
  };
  if (sweep) {
    // row-chunk pipeline: the side stream computes the hidden layer chunk by
    // chunk (FP64 tensor cores) and then the column statistics, while the
    // caller's stream writes O (HBM-write bound) for each chunk once its
    // activations exist; only the first chunk's hidden layer is exposed
    DevInfo d;
    IRL_TRY(dev_info(d));
    auto fn = cplx ? k_orows_sweep<true, MODEL_RBM>
                   : (model == MODEL_MLP ? k_orows_sweep<false, MODEL_MLP> : k_orows_sweep<false, MODEL_RBM>);
    // short rows (cfg3: 90 KB) double-buffer the factor row, long rows load it in place
    const int dbuf = ld_u * 16 < (256 << 10) ? 1 : 0;
    const size_t sm = (size_t)(1 + dbuf) * hidden * (cplx ? 16 : 8);
    IRL_TRY(ensure_fn_attrs((const void*)fn, d.smem_optin));
    const int64_t want = getenv("IRL_OBUILD_CHUNKS") ? atoi(getenv("IRL_OBUILD_CHUNKS")) : 4;
    const int nc = (int)std::max<int64_t>(1, std::min<int64_t>(want, n / 4096));
    Fork fork;
    IRL_TRY(fork.begin(st));
    std::vector<cudaEvent_t> evs((size_t)nc, nullptr);
    for (int c = 0; c < nc; ++c) {
      const int64_t r0 = n * c / nc, r1 = n * (c + 1) / nc;
      IRL_TRY(hidden_rows(r0, r1 - r0, fork.side));
      IRL_TRY(cuda_check(cudaEventCreateWithFlags(&evs[c], cudaEventDisableTiming), "chunk event"));
      IRL_TRY(cuda_check(cudaEventRecord(evs[c], fork.side), "chunk record"));
    }
    for (int c = 0; c < nc; ++c) {
      const int64_t r0 = n * c / nc, r1 = n * (c + 1) / nc;
      IRL_TRY(cuda_check(cudaStreamWaitEvent(st, evs[c], 0), "chunk wait"));
      IRL_TRY(cuda_check(cudaEventDestroy(evs[c]), "chunk event"));
      const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(r1 - r0, 2 * (int64_t)d.sms));
      fn<<<grid, SWEEP_NT, sm, st>>>(x + r0 * n_vis, r1 - r0, n_vis, hidden,
                                     static_cast<char*>(T) + (size_t)r0 * hidden * sS,
                                     G ? G + (size_t)r0 * hidden : nullptr, reinterpret_cast<double2*>(O) + r0 * ld_u,
                                     ld_u, dbuf);
      IRL_TRY(cuda_check(cudaGetLastError(), "orows sweep launch"));
    }
    IRL_TRY(obuild_stats(cplx, model, xbits, T, G, n, n_vis, hidden, ld, w, coeff, obar, g, base + off, fork.side));
    return fork.join();
  }
  IRL_TRY(hidden_rows(0, n, st));
  ORowArgs a{};
  a.x = x;
  a.xd = xd;
  a.xrow = xrow;
  a.n_rows = n;
  a.n_vis = n_vis;
  a.hidden = hidden;
  a.p = P;
  a.T = T;
  a.G = G;
  a.O = reinterpret_cast<double2*>(O);
  a.ld_u = ld_u;
  a.w = w;
  a.coeff = coeff;
  a.part0 = part0;
  a.part1 = part1;
  a.W = p.W;
  a.C = p.C;
  a.nb = p.nb;
  const int tab_len = model == MODEL_MLP ? orow_tab_len<MODEL_MLP>(n_vis, hidden) : orow_tab_len<MODEL_RBM>(n_vis, hidden);
  const size_t tab_bytes = (size_t)((tab_len + 1) & ~1) * sS;
  // per staging buffer: at least one full-width table (tiles spanning the short
  // blocks), else 16 KB of compact per-tile tables (k_orows sizes its groups)
  const size_t buf_bytes = rup(std::max<size_t>(tab_bytes, 16 * 1024), 16);
  const size_t smem = ORW_NBUF * (buf_bytes + (size_t)ORW_RMAX * (8 + sS));
  {
    DevInfo d;
    IRL_TRY(dev_info(d));
    if (smem > (size_t)d.smem_optin) return fail(IRL_ERR_ARG, "hidden layer too wide for the row table");
    IRL_TRY(ensure_fn_attrs((const void*)p.fn, d.smem_optin));
  }
  p.fn<<<(unsigned)(p.nb * p.C), p.NT, smem, st>>>(a, (int)buf_bytes);
  IRL_TRY(cuda_check(cudaGetLastError(), "orows launch"));
  if (gstats) {  // statistics on FP64 tensor cores beside the writer (they read T, G, not O)
    Fork fork;
    IRL_TRY(fork.begin(st));
    IRL_TRY(obuild_stats(cplx, model, xbits, T, G, n, n_vis, hidden, ld, w, coeff, obar, g, base + off, fork.side));
    return fork.join();
  }
  const unsigned blocks = (unsigned)cdiv(ld_u, 32);
  if (cplx)
    k_finish_stats<true><<<blocks, 256, 0, st>>>(part0, part1, p.nb, ld_u, (double2*)obar, (double2*)g);
  else
    k_finish_stats<false><<<blocks, 256, 0, st>>>(part0, part1, p.nb, ld_u, (double2*)obar, (double2*)g);
  return cuda_check(cudaGetLastError(), "obuild finish launch");
}

// ------------------------------------------------------------ connected ---
// Full connected product (est:171-186 + est:254-294, summed as opt:144-147):
// partner DOT pass -> per-row (a_n, d_n) -> one ordinary product over the batch
// O with coefficient a and additive row term d (connected.cuh).
struct ConnWs {
  size_t mvp, tpart, spart, gpart, a, d, bytes;
};

ConnWs conn_ws_layout(int64_t n, int64_t m, int64_t ld, bool cplx, const Plan* pp) {
  const size_t sS = cplx ? 16 : 8;
  ConnWs w{};
  size_t off = 0;
  auto carve = [&](size_t b) {
    const size_t r = off;
    off += align256(std::max<size_t>(b, 1));
    return r;
  };
  w.mvp = carve(mvp_ws_bytes(n, ld, cplx));
  const int C = pp ? std::max(pp->C, 1) : 1;
  w.tpart = carve((size_t)C * std::max<int64_t>(m, 1) * sS);
  w.spart = carve((size_t)C * sS);
  w.gpart = carve((size_t)C * 8);
  w.a = carve((size_t)n * sS);
  w.d = carve((size_t)n * sS);
  w.bytes = off;
  return w;
}

size_t connected_ws_bytes(int64_t n, int64_t m, int64_t ld, bool cplx) {
  const int64_t ld_u = cplx ? ld : ld / 2;
  Plan pp;
  const bool ok = m > 0 && make_plan(m, ld_u, cplx, MODE_DOT, pp) == IRL_OK;
  g_err.clear();
  return conn_ws_layout(n, m, ld, cplx, ok ? &pp : nullptr).bytes;
}

// Partners that are the batch's own rows (partner_O == O, exact mode): the
// product's first pass already gives q at every row, so the completion costs no
// extra read of O -- DOT pass over O, the per-row CSR kernel on those partial
// dots, then the ACC pass with coefficient a and additive term d (two passes
// instead of a partner pass plus the fused pass).
int connected_self_impl(bool cplx, const double* O, int64_t n, int64_t ld, const double* obar, const double* w,
                        const double* coeff, const int64_t* dist_index, const int64_t* indptr, const int64_t* prow,
                        const double* pcoeff, const double* v_re, const double* v_im, double* out_re, double* out_im,
                        const double* hf_re, const double* hf_im, const double* u0, double* out0, void* ws,
                        size_t ws_bytes, cudaStream_t st) {
  const int64_t ld_u = cplx ? ld : ld / 2;
  Plan p1, p2;
  IRL_TRY(make_plan(n, ld_u, cplx, MODE_DOT, p1));
  IRL_TRY(make_plan(n, ld_u, cplx, MODE_ACC, p2));
  if (p1.C != p2.C) return fail(IRL_ERR_DEVICE, "two-pass plans disagree on column split");
  const ConnWs wl = conn_ws_layout(n, 0, ld, cplx, nullptr);
  if (ws_bytes < wl.bytes) return fail(IRL_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, wl.bytes);
  char* base = static_cast<char*>(ws);
  Plan pw = p1;
  pw.nb = std::max(p1.nb, p2.nb);
  MvpWs mw = mvp_ws_layout(pw, n, ld_u, cplx, base + wl.mvp);
  if ((size_t)(wl.a - wl.mvp) < mw.bytes) return fail(IRL_ERR_WORKSPACE, "connected workspace layout");
  StreamArgs a{};
  a.O = reinterpret_cast<const double2*>(O);
  a.n_rows = n;
  a.ld_u = ld_u;
  a.v_re = v_re;
  a.v_im = v_im;
  a.hf_re = hf_re;
  a.hf_im = hf_im;
  a.obar = reinterpret_cast<const double2*>(obar);
  a.part0 = mw.part;
  a.ysum = mw.ysum;
  a.tpart = mw.tpart;
  a.spart = mw.spart;
  a.gpart = mw.gpart;
  IRL_TRY(launch_stream(p1, a, st));
  DevInfo d;
  IRL_TRY(dev_info(d));
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 8), (int64_t)d.sms * 8));
  void* av = base + wl.a;
  void* dv = base + wl.d;
  if (cplx)
    k_connected_rows<true><<<blocks, 256, 0, st>>>(dist_index, indptr, prow, reinterpret_cast<const double2*>(pcoeff),
                                                   reinterpret_cast<const double2*>(mw.tpart), p1.C, n,
                                                   reinterpret_cast<const double2*>(mw.spart), w,
                                                   reinterpret_cast<const double2*>(coeff), n,
                                                   reinterpret_cast<double2*>(av), reinterpret_cast<double2*>(dv));
  else
    k_connected_rows<false><<<blocks, 256, 0, st>>>(dist_index, indptr, prow, pcoeff,
                                                    reinterpret_cast<const double*>(mw.tpart), p1.C, n,
                                                    reinterpret_cast<const double*>(mw.spart), w, coeff, n,
                                                    reinterpret_cast<double*>(av), reinterpret_cast<double*>(dv));
  IRL_TRY(cuda_check(cudaGetLastError(), "connected rows launch"));
  a.coeff0 = av;
  a.yadd = dv;
  IRL_TRY(launch_stream(p2, a, st));
  if (cplx)
    return launch_finish_mvp<true>(mw.part, p2.nb, ld_u, mw.ysum, a.obar, hf_re, hf_im, u0, out_re, out_im, mw.gpart,
                                   p1.C, out0, st);
  return launch_finish_mvp<false>(mw.part, p2.nb, ld_u, mw.ysum, a.obar, hf_re, hf_im, u0, out_re, out_im, mw.gpart,
                                  p1.C, out0, st);
}

int connected_impl(bool cplx, const double* O, int64_t n, int64_t p, int64_t ld, const double* obar, const double* w,
                   const double* coeff, const int64_t* dist_index, const int64_t* indptr, const int64_t* prow,
                   const double* pcoeff, const double* Op, int64_t m, const double* v_re, const double* v_im,
                   double* out_re, double* out_im, const double* hf_re, const double* hf_im, const double* u0,
                   double* out0, int mode, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!O || !w || !dist_index || !indptr || !v_re || !out_re) return fail(IRL_ERR_ARG, "null required pointer");
  if (m < 0 || (m > 0 && (!Op || !prow || !pcoeff))) return fail(IRL_ERR_ARG, "bad partner arguments");
  if (n < 1 || p < 1 || ld < p) return fail(IRL_ERR_ARG, "bad shape n=%lld p=%lld ld=%lld", (long long)n,
                                            (long long)p, (long long)ld);
  if (ld != irl_padded_ld(p, cplx)) return fail(IRL_ERR_ALIGN, "ld must equal irl_padded_ld(p)");
  if (!aligned16(O) || !aligned16(Op) || !aligned16(obar) || !aligned16(ws))
    return fail(IRL_ERR_ALIGN, "pointers must be 16-byte aligned");
  const int64_t ld_u = cplx ? ld : ld / 2;
  if (Op == O && m == n) return connected_self_impl(cplx, O, n, ld, obar, w, coeff, dist_index, indptr, prow, pcoeff,
                                                    v_re, v_im, out_re, out_im, hf_re, hf_im, u0, out0, ws,
                                                    ws_bytes, st);
  Plan pp{};
  if (m > 0) IRL_TRY(make_plan(m, ld_u, cplx, MODE_DOT, pp));
  const ConnWs wl = conn_ws_layout(n, m, ld, cplx, m > 0 ? &pp : nullptr);
  if (ws_bytes < wl.bytes) return fail(IRL_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, wl.bytes);
  char* base = static_cast<char*>(ws);
  if (m > 0) {
    StreamArgs a{};
    a.O = reinterpret_cast<const double2*>(Op);
    a.n_rows = m;
    a.ld_u = ld_u;
    a.v_re = v_re;
    a.v_im = v_im;
    a.obar = reinterpret_cast<const double2*>(obar);
    a.tpart = base + wl.tpart;
    a.spart = base + wl.spart;
    a.gpart = reinterpret_cast<double*>(base + wl.gpart);
    IRL_TRY(launch_stream(pp, a, st));
  }
  DevInfo d;
  IRL_TRY(dev_info(d));
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 8), (int64_t)d.sms * 8));
  if (cplx) {
    k_connected_rows<true><<<blocks, 256, 0, st>>>(
        dist_index, indptr, prow, reinterpret_cast<const double2*>(pcoeff),
        reinterpret_cast<const double2*>(base + wl.tpart), std::max(pp.C, 1), m,
        reinterpret_cast<const double2*>(base + wl.spart), w, reinterpret_cast<const double2*>(coeff), n,
        reinterpret_cast<double2*>(base + wl.a), reinterpret_cast<double2*>(base + wl.d));
  } else {
    k_connected_rows<false><<<blocks, 256, 0, st>>>(
        dist_index, indptr, prow, pcoeff, reinterpret_cast<const double*>(base + wl.tpart), std::max(pp.C, 1), m,
        reinterpret_cast<const double*>(base + wl.spart), w, coeff, n, reinterpret_cast<double*>(base + wl.a),
        reinterpret_cast<double*>(base + wl.d));
  }
  IRL_TRY(cuda_check(cudaGetLastError(), "connected rows launch"));
  return mvp_impl(cplx, O, n, p, ld, obar, reinterpret_cast<const double*>(base + wl.a), base + wl.d, v_re, v_im,
                  out_re, out_im, hf_re, hf_im, u0, out0, mode, base + wl.mvp, wl.a - wl.mvp, st);
}

// ------------------------------------------------------------- log psi ---
size_t logamp_ws_bytes(int64_t n, int hidden, bool cplx) {
  return align256((size_t)cdiv(hidden, 32) * std::max<int64_t>(n, 1) * (cplx ? 16 : 8));
}

template <bool CPLX, int MODEL>
int logamp_impl(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta, double* out, void* ws,
                size_t ws_bytes, cudaStream_t st) {
  using S = typename Traits<CPLX>::S;
  if (!x || !theta || !out || n < 1 || n_vis < 1 || hidden < 1) return fail(IRL_ERR_ARG, "bad log-amplitude arguments");
  if (ws_bytes < logamp_ws_bytes(n, hidden, CPLX)) return fail(IRL_ERR_WORKSPACE, "workspace too small");
  const size_t smem = (size_t)n_vis * 32 * sizeof(S);
  DevInfo d;
  IRL_TRY(dev_info(d));
  if (smem > (size_t)d.smem_optin) return fail(IRL_ERR_ARG, "n_vis too large");
  const S* th = reinterpret_cast<const S*>(theta);
  const S *avec, *bvec, *Wm;
  const double *uvec = nullptr, *cval = nullptr;
  if (MODEL == MODEL_RBM) {
    avec = th;
    bvec = th + n_vis;
    Wm = th + n_vis + hidden;
  } else {
    Wm = th;
    bvec = th + (size_t)hidden * n_vis;
    uvec = theta + (size_t)hidden * n_vis + hidden;
    cval = uvec + hidden;
    avec = nullptr;
  }
  auto fn = k_logamp_part<CPLX, MODEL>;
  IRL_TRY(ensure_fn_attrs((const void*)fn, d.smem_optin));
  const int jt = (int)cdiv(hidden, 32);
  const int64_t rb = std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 8), cdiv((int64_t)d.sms * 8, jt)));
  S* part = static_cast<S*>(ws);
  fn<<<dim3((unsigned)rb, (unsigned)jt), 256, smem, st>>>(x, n, n_vis, hidden, Wm, bvec, uvec, part);
  IRL_TRY(cuda_check(cudaGetLastError(), "log-amplitude kernel launch"));
  k_logamp_finish<CPLX, MODEL><<<(unsigned)cdiv(n, 256), 256, 0, st>>>(x, n, n_vis, jt, avec, cval, part,
                                                                       reinterpret_cast<S*>(out));
  return cuda_check(cudaGetLastError(), "log-amplitude finish launch");
}

// ---------------------------------------------------------- hamiltonian ---
size_t ham_ws_bytes(int n_vis, int hidden, bool cplx) {
  return 3 * align256((size_t)n_vis * std::max(hidden, 1) * (cplx ? 16 : 8));  // W^T, exp(W^T), exp(-W^T)
}

template <bool CPLX, int MODEL, int MODE>
int ham_launch(const HamArgs& a, size_t smem, cudaStream_t st) {
  DevInfo d;
  IRL_TRY(dev_info(d));
  if (smem > (size_t)d.smem_optin - 8192) return fail(IRL_ERR_ARG, "hidden width too large for the local-energy kernel");
  // E_loc and the partner coefficients of the RBM: the exp table in shared
  // memory when it fits (one 512-thread CTA per SM)
  if constexpr ((MODE == HAM_ELOC || MODE == HAM_FILL) && MODEL == MODEL_RBM) {
    const size_t tab = (size_t)2 * a.ns * (a.hidden + 1) * 2 * (CPLX ? 16 : 8);
    if (!getenv("IRL_HAM_NO_SMT") && rup(smem, 16) + tab <= (size_t)d.smem_optin - 16384) {
      auto fn = k_local_energy<CPLX, MODEL, MODE, 512, true>;
      IRL_TRY(ensure_fn_attrs((const void*)fn, d.smem_optin));
      const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(a.n, (int64_t)d.sms));
      fn<<<grid, 512, rup(smem, 16) + tab, st>>>(a);
      return cuda_check(cudaGetLastError(), "local-energy kernel launch");
    }
  }
  auto fn = k_local_energy<CPLX, MODEL, MODE>;
  IRL_TRY(ensure_fn_attrs((const void*)fn, d.smem_optin));
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(a.n, (int64_t)d.sms * 16));
  fn<<<grid, HAM_NT, smem, st>>>(a);
  return cuda_check(cudaGetLastError(), "local-energy kernel launch");
}

int ham_impl(int model, bool cplx, int mode, const uint64_t* xbits, int64_t n, int ns, double e_core, const double* h1,
             const double* g2, double drop, int hidden, const double* theta, void* out, int64_t* counts,
             const int64_t* offsets, uint64_t* pbits, double* pelem, double* pcoeff, void* ws, size_t ws_bytes,
             cudaStream_t st, double* diag = nullptr) {
  const bool none = model == MODEL_NONE;
  if (!xbits || !h1 || !g2 || (!none && !theta) || n < 0 || ns < 1 || ns > 32 || (!none && hidden < 1))
    return fail(IRL_ERR_ARG, "bad local-energy arguments");
  if (model != MODEL_RBM && model != MODEL_MLP && !none) return fail(IRL_ERR_ARG, "unknown model %d", model);
  if (none) {
    if (mode == HAM_ELOC) return fail(IRL_ERR_ARG, "local energies need an ansatz");
    cplx = false;
    hidden = 0;
  }
  if (cplx && model != MODEL_RBM) return fail(IRL_ERR_ARG, "complex parameters are an RBM feature");
  if (mode == HAM_ELOC && !out) return fail(IRL_ERR_ARG, "null output");
  if (mode == HAM_COUNT && !counts) return fail(IRL_ERR_ARG, "null counts");
  if (mode == HAM_FILL && (!offsets || !pbits || !pelem || !pcoeff)) return fail(IRL_ERR_ARG, "null fill outputs");
  const int M = 2 * ns;
  if (!none && ws_bytes < ham_ws_bytes(M, hidden, cplx)) return fail(IRL_ERR_WORKSPACE, "workspace too small");
  if (n == 0) return IRL_OK;
  const size_t sS = cplx ? 16 : 8;
  HamArgs a{};
  a.xbits = xbits;
  a.n = n;
  a.ns = ns;
  a.hidden = hidden;
  a.e_core = e_core;
  a.h1 = h1;
  a.g2 = g2;
  a.drop = drop;
  a.diag = diag;
  a.out = out;
  a.counts = counts;
  a.offsets = offsets;
  a.pbits = pbits;
  a.pelem = pelem;
  a.pcoeff = pcoeff;
  if (none) {
    if (mode == HAM_COUNT) return ham_launch<false, MODEL_NONE, HAM_COUNT>(a, 0, st);
    return ham_launch<false, MODEL_NONE, HAM_FILL>(a, 0, st);
  }
  const char* th = reinterpret_cast<const char*>(theta);
  const char* Wm;
  if (model == MODEL_RBM) {
    a.avec = th;
    a.bvec = th + (size_t)M * sS;
    Wm = th + (size_t)(M + hidden) * sS;
  } else {
    Wm = th;
    a.bvec = th + (size_t)hidden * M * sS;
    a.uvec = theta + (size_t)hidden * M + hidden;
  }
  const size_t tab = align256((size_t)M * hidden * sS);
  a.WT = ws;
  void* EX = model == MODEL_RBM ? static_cast<char*>(ws) + tab : nullptr;
  a.EX = EX;
  a.out = out;
  a.counts = counts;
  a.offsets = offsets;
  a.pbits = pbits;
  a.pelem = pelem;
  a.pcoeff = pcoeff;
  const int64_t ne = (int64_t)hidden * M;
  if (cplx)
    k_transpose_w<true><<<(unsigned)cdiv(ne, 256), 256, 0, st>>>((const double2*)Wm, hidden, M, (double2*)ws,
                                                                 (double2*)EX);
  else
    k_transpose_w<false><<<(unsigned)cdiv(ne, 256), 256, 0, st>>>((const double*)Wm, hidden, M, (double*)ws,
                                                                  (double*)EX);
  IRL_TRY(cuda_check(cudaGetLastError(), "transpose launch"));
  const size_t smem = (size_t)3 * hidden * sS;
#define IRL_HAM(C, MD, MO) \
  if (cplx == C && model == MD && mode == MO) return ham_launch<C, MD, MO>(a, smem, st);
  IRL_HAM(false, MODEL_RBM, HAM_ELOC)
  IRL_HAM(false, MODEL_RBM, HAM_COUNT)
  IRL_HAM(false, MODEL_RBM, HAM_FILL)
  IRL_HAM(true, MODEL_RBM, HAM_ELOC)
  IRL_HAM(true, MODEL_RBM, HAM_COUNT)
  IRL_HAM(true, MODEL_RBM, HAM_FILL)
  IRL_HAM(false, MODEL_MLP, HAM_ELOC)
  IRL_HAM(false, MODEL_MLP, HAM_COUNT)
  IRL_HAM(false, MODEL_MLP, HAM_FILL)
#undef IRL_HAM
  return fail(IRL_ERR_ARG, "unsupported local-energy variant");
}

// ------------------------------------------------------- autoregressive ---
int ar_check(int64_t n, int M, int h, int n_up, int n_down, const double* theta) {
  if (n < 0 || M < 2 || M > 64 || (M & 1) || h < 1 || h > 64 || !theta) return fail(IRL_ERR_ARG, "bad autoregressive shape");
  if (n_up < 0 || n_down < 0 || n_up > M / 2 || n_down > M / 2) return fail(IRL_ERR_ARG, "bad sector");
  return IRL_OK;
}

template <int MODE>
int ar_launch(ArArgs& a, cudaStream_t st) {
  if (a.n == 0) return IRL_OK;
  DevInfo d;
  IRL_TRY(dev_info(d));
  const int hpl = a.h <= 32 ? 1 : 2;
  const size_t smem = MODE == AR_ROWS ? (size_t)AR_WARPS * a.M * 32 * hpl * 8 : 0;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(a.n, AR_WARPS), (int64_t)d.sms * 16));
  auto fn = hpl == 1 ? k_autoreg<1, MODE> : k_autoreg<2, MODE>;
  IRL_TRY(ensure_fn_attrs((const void*)fn, d.smem_optin));
  fn<<<grid, AR_WARPS * 32, smem, st>>>(a);
  return cuda_check(cudaGetLastError(), "autoregressive kernel launch");
}

// ------------------------------------------------ connected, on the fly ---
// The completion on an on-the-fly batch (O never stored): partner dots from
// stored partner rows (a k_stream DOT pass) or, when the partners are batch
// rows (partner_O == NULL, exact mode), from the batch's own centred dots (a
// first k_otf_y pass with unit coefficient); then k_connected_rows, and the
// product's y pass takes coefficient a and additive term d.
struct OtfConn {
  const int64_t* dist_index;
  const int64_t* indptr;
  const int64_t* prow;
  const void* pcoeff;
  const double* w;
  const void* cdiag;
  const double* partner_O;  // null: partners are batch rows (or regenerated, below)
  const uint64_t* pxbits;   // partners regenerated on the fly: packed inputs, t (and MLP g)
  const double* pt;
  const double* pg;
  int64_t m;
  Plan pp;
  OtfPlan ppl;
  OtfWs pwl;
  void* tpart_p;
  void* spart_p;
  double* gpart_p;
  void* q;
  void* qpart;
  void* a;
  void* d;
};

size_t otf_conn_carve(OtfConn& cx, int64_t n, int64_t m, bool cplx, bool stored, void* base, bool regen = false,
                      int hidden = 0) {
  const size_t sS = cplx ? 16 : 8;
  size_t off = 0;
  auto carve = [&](size_t b) {
    void* r = base ? static_cast<char*>(base) + off : nullptr;
    off += align256(std::max<size_t>(b, 1));
    return r;
  };
  const int C = stored ? std::max(cx.pp.C, 1) : 1;
  cx.tpart_p = carve(stored ? (size_t)C * std::max<int64_t>(m, 1) * sS : 0);
  cx.spart_p = carve((size_t)C * sS);
  cx.gpart_p = reinterpret_cast<double*>(carve((size_t)C * 8));
  cx.q = carve(stored ? 0 : (size_t)(regen ? m : n) * sS);
  if (regen) {
    const size_t pb = otf_ws_layout(cx.ppl, m, hidden, nullptr).bytes;
    void* pbase = carve(pb);
    cx.pwl = otf_ws_layout(cx.ppl, m, hidden, pbase);
  }
  cx.qpart = carve((size_t)4 * 148 * sS);
  cx.a = carve((size_t)n * sS);
  cx.d = carve((size_t)n * sS);
  return off;
}

int otf_conn_partner_dot(OtfConn& cx, bool cplx, int64_t ld, const double* v_re, const double* v_im,
                         const double* obar, cudaStream_t st) {
  if (!cx.partner_O || cx.m == 0) return IRL_OK;
  StreamArgs a{};
  a.O = reinterpret_cast<const double2*>(cx.partner_O);
  a.n_rows = cx.m;
  a.ld_u = cplx ? ld : ld / 2;
  a.v_re = v_re;
  a.v_im = v_im;
  a.obar = reinterpret_cast<const double2*>(obar);
  a.tpart = cx.tpart_p;
  a.spart = cx.spart_p;
  a.gpart = cx.gpart_p;
  return launch_stream(cx.pp, a, st);
}

int otf_conn_rows(OtfConn& cx, bool cplx, int64_t n, cudaStream_t st) {
  DevInfo d;
  IRL_TRY(dev_info(d));
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 8), (int64_t)d.sms * 8));
  const bool stored = cx.partner_O != nullptr;
  const void* tp = stored ? cx.tpart_p : cx.q;
  const int C = stored ? std::max(cx.pp.C, 1) : 1;
  const int64_t m = (stored || cx.pxbits) ? cx.m : n;
  const void* sp = stored ? cx.spart_p : nullptr;
  if (cplx)
    k_connected_rows<true><<<blocks, 256, 0, st>>>(cx.dist_index, cx.indptr, cx.prow, (const double2*)cx.pcoeff,
                                                   (const double2*)tp, C, m, (const double2*)sp, cx.w,
                                                   (const double2*)cx.cdiag, n, (double2*)cx.a, (double2*)cx.d);
  else
    k_connected_rows<false><<<blocks, 256, 0, st>>>(cx.dist_index, cx.indptr, cx.prow, (const double*)cx.pcoeff,
                                                    (const double*)tp, C, m, (const double*)sp, cx.w,
                                                    (const double*)cx.cdiag, n, (double*)cx.a, (double*)cx.d);
  return cuda_check(cudaGetLastError(), "connected rows launch");
}

// Partner dots regenerated from the partners' packed inputs and hidden
// activations with the batch's own DMMA dot GEMM: q_p = O_p v - Obar.v.
int otf_conn_regen_dots(OtfConn& cx, const OtfArgs& batch_args, bool has_t, int64_t p_last, int64_t offa,
                        const double* dpart, int n_dpart, cudaStream_t st) {
  if (!cx.pxbits || cx.m == 0) return IRL_OK;
  OtfArgs ap = batch_args;
  ap.xbits = cx.pxbits;
  ap.T = cx.pt;
  ap.G = has_t ? cx.pg : cx.pt;
  ap.n_rows = cx.m;
  ap.nb = cx.ppl.nb;
  ap.tpart = cx.pwl.tpart;
  IRL_TRY(otf_dot_launch(ap, has_t, st));
  k_otf_y<<<cx.ppl.ny, 256, 0, st>>>(cx.pwl.tpart, cx.ppl.jc, cx.m, nullptr, batch_args.v, p_last, dpart, n_dpart,
                                     (double*)cx.q, cx.pwl.ypart, offa >= 0 ? cx.pxbits : nullptr, offa,
                                     batch_args.n_in);
  return cuda_check(cudaGetLastError(), "partner dot launch");
}

}  // namespace

// =================================================================== ABI ==
extern "C" {

int irl_version(void) { return 100; }

const char* irl_last_error(void) { return g_err.c_str(); }

size_t irl_debug_wide_trace(void* host, size_t bytes) {
  if (!g_wide_trace || !host) return 0;
  const size_t n = bytes < g_wide_trace_bytes ? bytes : g_wide_trace_bytes;
  if (cudaMemcpy(host, g_wide_trace, n, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  return n;
}

int64_t irl_padded_ld(int64_t p, int is_complex) {
  if (p < 1) return 0;
  const int64_t E = is_complex ? 1 : 2;
  const int64_t units = cdiv(p, E);
  const int64_t A = units < 32768 ? 16 : 64;
  return rup(units, A) * E;
}

int irl_energy_f64(const double* w, const double* e, int64_t n, double* stats3, double* coeff, void* stream) {
  if (!w || !e || !stats3 || !coeff || n < 1) return fail(IRL_ERR_ARG, "bad energy arguments");
  DevInfo d;
  IRL_TRY(dev_info(d));
  k_energy<false><<<1, 1024, 0, (cudaStream_t)stream>>>(w, e, n, 0, stats3, coeff);
  return cuda_check(cudaGetLastError(), "energy launch");
}

int irl_energy_c128(const double* w, const double* e, int64_t n, int hermitian, double* stats3, double* coeff,
                    void* stream) {
  if (!w || !e || !stats3 || !coeff || n < 1) return fail(IRL_ERR_ARG, "bad energy arguments");
  DevInfo d;
  IRL_TRY(dev_info(d));
  k_energy<true><<<1, 1024, 0, (cudaStream_t)stream>>>(w, e, n, hermitian, stats3, coeff);
  return cuda_check(cudaGetLastError(), "energy launch");
}

size_t irl_colstats_workspace_bytes(int64_t n, int64_t ld, int is_complex) {
  const int64_t ld_u = is_complex ? ld : ld / 2;
  Plan p;
  if (make_plan(n, ld_u, is_complex != 0, MODE_STATS, p) != IRL_OK) return 0;
  return colstats_bytes(p, ld_u);
}

int irl_colstats_f64(const double* O, int64_t n, int64_t ld, const double* w, const double* coeff, double* obar,
                     double* g, void* ws, size_t ws_bytes, void* stream) {
  return colstats_impl(false, O, n, ld, w, coeff, obar, g, ws, ws_bytes, (cudaStream_t)stream);
}

int irl_colstats_c128(const double* O, int64_t n, int64_t ld, const double* w, const double* coeff, double* obar,
                      double* g, void* ws, size_t ws_bytes, void* stream) {
  return colstats_impl(true, O, n, ld, w, coeff, obar, g, ws, ws_bytes, (cudaStream_t)stream);
}

size_t irl_obuild_workspace_bytes(int model, int64_t n, int n_vis, int hidden, int64_t ld, int is_complex) {
  const int64_t ld_u = is_complex ? ld : ld / 2;
  OPlan p;
  if (make_oplan(ld_u, is_complex != 0, model, p, !gemm_stats(is_complex != 0, model, n_vis, hidden)) != IRL_OK) return 0;
  return obuild_bytes(p, model, n, n_vis, hidden, ld_u, is_complex != 0);
}

int irl_obuild_rbm_f64(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta, double* O,
                       int64_t ld, const double* w, const double* coeff, double* obar, double* g, void* ws,
                       size_t ws_bytes, void* stream) {
  return obuild_impl(false, MODEL_RBM, x, n, n_vis, hidden, theta, O, ld, w, coeff, obar, g, ws, ws_bytes,
                     (cudaStream_t)stream);
}

int irl_obuild_rbm_c128(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta, double* O,
                        int64_t ld, const double* w, const double* coeff, double* obar, double* g, void* ws,
                        size_t ws_bytes, void* stream) {
  return obuild_impl(true, MODEL_RBM, x, n, n_vis, hidden, theta, O, ld, w, coeff, obar, g, ws, ws_bytes,
                     (cudaStream_t)stream);
}

int irl_obuild_mlp_f64(const uint8_t* x, int64_t n, int n_in, int hidden, const double* theta, double* O,
                       int64_t ld, const double* w, const double* coeff, double* obar, double* g, void* ws,
                       size_t ws_bytes, void* stream) {
  return obuild_impl(false, MODEL_MLP, x, n, n_in, hidden, theta, O, ld, w, coeff, obar, g, ws, ws_bytes,
                     (cudaStream_t)stream);
}

int irl_hidden_rbm_f64(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta, double* t,
                       void* stream) {
  if (!x || !theta || !t || n < 1 || n_vis < 1 || hidden < 1) return fail(IRL_ERR_ARG, "bad hidden arguments");
  return launch_hidden<false, MODEL_RBM>(x, nullptr, n, n_vis, hidden, theta + n_vis + hidden, theta + n_vis, nullptr,
                                         t, nullptr, (cudaStream_t)stream);
}

int irl_hidden_rbm_c128(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta, double* t,
                        void* stream) {
  if (!x || !theta || !t || n < 1 || n_vis < 1 || hidden < 1) return fail(IRL_ERR_ARG, "bad hidden arguments");
  return launch_hidden<true, MODEL_RBM>(x, nullptr, n, n_vis, hidden, theta + 2 * (n_vis + hidden), theta + 2 * n_vis,
                                        nullptr, t, nullptr, (cudaStream_t)stream);
}

int irl_hidden_mlp_f64(const uint8_t* x, int64_t n, int n_in, int hidden, const double* theta, double* t,
                       double* g, void* stream) {
  if (!x || !theta || !t || !g || n < 1 || n_in < 1 || hidden < 1) return fail(IRL_ERR_ARG, "bad hidden arguments");
  const double* bvec = theta + (size_t)hidden * n_in;
  return launch_hidden<false, MODEL_MLP>(x, nullptr, n, n_in, hidden, theta, bvec, bvec + hidden, t, g,
                                         (cudaStream_t)stream);
}

size_t irl_mvp_workspace_bytes(int64_t n, int64_t ld, int is_complex) { return mvp_ws_bytes(n, ld, is_complex != 0); }

int irl_mvp_f64(const double* O, int64_t n, int64_t p, int64_t ld, const double* obar, const double* coeff,
                const double* v, double* out, const double* half_f, const double* u0, double* out0, int mode,
                void* ws, size_t ws_bytes, void* stream) {
  return mvp_impl(false, O, n, p, ld, obar, coeff, nullptr, v, nullptr, out, nullptr, half_f, nullptr, u0, out0, mode, ws,
                  ws_bytes, (cudaStream_t)stream);
}

int irl_mvp_c128(const double* O, int64_t n, int64_t p, int64_t ld, const double* obar, const double* coeff,
                 const double* v_re, const double* v_im, double* out_re, double* out_im, const double* hf_re,
                 const double* hf_im, const double* u0, double* out0, int mode, void* ws, size_t ws_bytes,
                 void* stream) {
  return mvp_impl(true, O, n, p, ld, obar, coeff, nullptr, v_re, v_im, out_re, out_im, hf_re, hf_im, u0, out0, mode, ws,
                  ws_bytes, (cudaStream_t)stream);
}

size_t irl_mvp2_workspace_bytes(int64_t n, int64_t ld, int is_complex) { return mvp2_ws_bytes(n, ld, is_complex != 0); }

int irl_mvp2_f64(const double* O, int64_t n, int64_t p, int64_t ld, const double* obar, const double* coeff_a,
                 const double* coeff_b, const double* v, double* out_a, double* out_b, const double* half_f,
                 const double* u0, double* out0, void* ws, size_t ws_bytes, void* stream) {
  return mvp2_impl(false, O, n, p, ld, obar, coeff_a, coeff_b, v, nullptr, out_a, nullptr, out_b, nullptr, half_f,
                   nullptr, u0, out0, ws, ws_bytes, (cudaStream_t)stream);
}

int irl_mvp2_c128(const double* O, int64_t n, int64_t p, int64_t ld, const double* obar, const double* coeff_a,
                  const double* coeff_b, const double* v_re, const double* v_im, double* outa_re, double* outa_im,
                  double* outb_re, double* outb_im, const double* hf_re, const double* hf_im, const double* u0,
                  double* out0, void* ws, size_t ws_bytes, void* stream) {
  return mvp2_impl(true, O, n, p, ld, obar, coeff_a, coeff_b, v_re, v_im, outa_re, outa_im, outb_re, outb_im, hf_re,
                   hf_im, u0, out0, ws, ws_bytes, (cudaStream_t)stream);
}

int irl_mvp_plan(int64_t n, int64_t ld, int is_complex, int mode, int* out_path, int* out_geom7) {
  if (!out_path || !out_geom7) return fail(IRL_ERR_ARG, "null output");
  const int64_t ld_u = is_complex ? ld : ld / 2;
  Plan p;
  int path = IRL_MVP_TWO_PASS;
  WidePlan wp{};
  if ((mode == IRL_MVP_AUTO && ld_u <= kRowsMaxUnits) || mode == IRL_MVP_ROWS) {
    IRL_TRY(make_rows_plan(n, ld_u, p));
    path = IRL_MVP_ROWS;
  } else if ((mode == IRL_MVP_AUTO && ld_u >= kWideMinUnits && make_wide_plan(n, ld_u, is_complex != 0, wp) == IRL_OK) ||
             mode == IRL_MVP_WIDE) {
    IRL_TRY(make_wide_plan(n, ld_u, is_complex != 0, wp));
    *out_path = IRL_MVP_WIDE;
    int g[7] = {wp.G, wp.WM, WIDE_THREADS, wp.RS, wp.NS, wp.K, wp.upl};  // slices, units/slice, threads, rows/stage, stages, TMEM slots, units/lane
    memcpy(out_geom7, g, sizeof(g));
    return IRL_OK;
  } else if (mode == IRL_MVP_AUTO || mode == IRL_MVP_FUSED) {
    if (make_plan(n, ld_u, is_complex != 0, MODE_FUSED, p) == IRL_OK) {
      path = IRL_MVP_FUSED;
    } else if (mode == IRL_MVP_FUSED) {
      return IRL_ERR_DEVICE;
    }
  }
  if (path == IRL_MVP_TWO_PASS) IRL_TRY(make_plan(n, ld_u, is_complex != 0, MODE_DOT, p));
  *out_path = path;
  int g[7] = {p.C, p.W, p.NT, p.R, p.NS, p.nb, p.PPT};
  memcpy(out_geom7, g, sizeof(g));
  return IRL_OK;
}

size_t irl_otf_workspace_bytes(int64_t n, int n_in, int hidden) {
  OtfPlan p;
  if (make_otf_plan(n, n_in, hidden, p) != IRL_OK) return 0;
  return otf_ws_layout(p, n, hidden, nullptr).bytes;
}

int irl_otf_prepare_mlp_f64(const uint8_t* x, int64_t n, int n_in, int hidden, const double* theta, uint64_t* xbits,
                            double* t, double* g, void* stream) {
  if (!x || !theta || !xbits || !t || !g || n < 1 || n_in < 1 || hidden < 1)
    return fail(IRL_ERR_ARG, "bad prepare arguments");
  if (n_in > OTF_MAX_NIN) return fail(IRL_ERR_ARG, "on-the-fly mode supports n_in <= %d", OTF_MAX_NIN);
  cudaStream_t st = (cudaStream_t)stream;
  DevInfo d;
  IRL_TRY(dev_info(d));
  IRL_TRY(pack_bits(x, n, n_in, xbits, st));
  const double* bvec = theta + (size_t)hidden * n_in;
  return launch_hidden<false, MODEL_MLP>(x, xbits, n, n_in, hidden, theta, bvec, bvec + hidden, t, g, st);
}

int irl_otf_colstats_mlp_f64(const uint64_t* xbits, const double* t, const double* g, int64_t n, int n_in, int hidden,
                             int64_t ld, const double* w, const double* coeff, double* obar, double* grad,
                             void* ws, size_t ws_bytes, void* stream) {
  IRL_TRY(otf_check(xbits, t, g, n, n_in, hidden, ld));
  if (!w || !coeff || !obar || !grad) return fail(IRL_ERR_ARG, "null pointer");
  OtfPlan pl;
  IRL_TRY(make_otf_plan(n, n_in, hidden, pl));
  OtfWs wl = otf_ws_layout(pl, n, hidden, ws);
  if (ws_bytes < wl.bytes) return fail(IRL_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, wl.bytes);
  cudaStream_t st = (cudaStream_t)stream;
  OtfArgs a{};
  a.xbits = xbits;
  a.T = t;
  a.G = g;
  a.n_rows = n;
  a.n_in = n_in;
  a.hidden = hidden;
  return otf_stats(pl, a, wl, MODEL_MLP, n, n_in, hidden, ld, w, coeff, obar, grad, nullptr, 0, st);
}

static int otf_mvp_mlp_core(const uint64_t* xbits, const double* t, const double* g, int64_t n, int n_in, int hidden,
                        int64_t ld, const double* obar, const double* coeff, const double* v, double* out,
                        const double* half_f, const double* u0, double* out0, void* ws, size_t ws_bytes,
                        void* stream, const OtfConn* cx, const double* uvec = nullptr) {
  // uvec: G = u (1 - T^2) formed in the GEMM kernels from T (g unused; any valid pointer)
  IRL_TRY(otf_check(xbits, t, g, n, n_in, hidden, ld));
  if ((!coeff && !cx) || !v || !out) return fail(IRL_ERR_ARG, "null pointer");
  OtfPlan pl;
  IRL_TRY(make_otf_plan(n, n_in, hidden, pl));
  OtfWs wl = otf_ws_layout(pl, n, hidden, ws);
  if (ws_bytes < wl.bytes) return fail(IRL_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, wl.bytes);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t P = (int64_t)hidden * n_in + 2 * (int64_t)hidden + 1;
  IRL_TRY(launch_pdl(k_vdot2, dim3(pl.ny), dim3(256), 0, st, "otf vdot launch", obar, half_f, v, (int64_t)ld,
                     wl.dpart, wl.gpart));
  OtfArgs a{};
  a.xbits = xbits;
  a.T = t;
  a.G = g;
  a.n_rows = n;
  a.n_in = n_in;
  a.hidden = hidden;
  a.nb = pl.nb;
  a.offW = 0;
  a.offb = (int64_t)hidden * n_in;
  a.offu = a.offb + hidden;
  a.v = v;
  a.tpart = wl.tpart;
  a.y = wl.y;
  a.part = wl.part;
  a.partu = wl.partu;
  a.u = cx ? nullptr : uvec;
  if (cx) IRL_TRY(otf_conn_partner_dot(*const_cast<OtfConn*>(cx), false, ld, v, nullptr, obar, st));
  IRL_TRY(otf_dot_launch(a, true, st));
  const double* ceff = coeff;
  const double* yadd = nullptr;
  if (cx) {
    if (cx->pxbits)
      IRL_TRY(otf_conn_regen_dots(*const_cast<OtfConn*>(cx), a, true, P - 1, -1, wl.dpart, obar ? pl.ny : 0, st));
    else if (!cx->partner_O)
      k_otf_y<<<pl.ny, 256, 0, st>>>(wl.tpart, pl.jc, n, nullptr, v, P - 1, wl.dpart, obar ? pl.ny : 0,
                                     (double*)cx->q, (double*)cx->qpart, nullptr, -1, n_in);
    IRL_TRY(otf_conn_rows(*const_cast<OtfConn*>(cx), false, n, st));
    ceff = (const double*)cx->a;
    yadd = (const double*)cx->d;
  }
  IRL_TRY(launch_pdl(k_otf_y, dim3(pl.ny), dim3(256), 0, st, "otf y launch", (const double*)wl.tpart, (int)pl.jc,
                     (int64_t)n, ceff, v, (int64_t)(P - 1), (const double*)wl.dpart, obar ? pl.ny : 0, wl.y,
                     wl.ypart, (const uint64_t*)nullptr, (int64_t)-1, n_in, yadd));
  IRL_TRY(otf_acc_launch(pl, a, st, 1, true));
  return launch_pdl(k_otf_finish, fin_grid(ld), dim3(32, 8), 0, st, "otf finish launch", (const double*)wl.part,
                    (const double*)wl.partu, (int)a.nb, hidden, n_in, (int)pl.kc, (int64_t)ld,
                    (const double*)wl.ypart, (int)pl.ny, obar, half_f, u0, (const double*)wl.gpart, (int)pl.ny, out,
                    out0);
}

int irl_otf_mvp_mlp_f64(const uint64_t* xbits, const double* t, const double* g, int64_t n, int n_in, int hidden,
                        int64_t ld, const double* obar, const double* coeff, const double* v, double* out,
                        const double* half_f, const double* u0, double* out0, void* ws, size_t ws_bytes,
                        void* stream) {
  return otf_mvp_mlp_core(xbits, t, g, n, n_in, hidden, ld, obar, coeff, v, out, half_f, u0, out0, ws, ws_bytes, stream, nullptr);
}

int irl_otf_mvp_mlp_u_f64(const uint64_t* xbits, const double* t, const double* u, int64_t n, int n_in, int hidden,
                          int64_t ld, const double* obar, const double* coeff, const double* v, double* out,
                          const double* half_f, const double* u0, double* out0, void* ws, size_t ws_bytes,
                          void* stream) {
  if (!u) return fail(IRL_ERR_ARG, "null pointer");
  return otf_mvp_mlp_core(xbits, t, t, n, n_in, hidden, ld, obar, coeff, v, out, half_f, u0, out0, ws, ws_bytes, stream,
                          nullptr, u);
}

int irl_otf_prepare_rbm_f64(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta, uint64_t* xbits,
                            double* t, void* stream) {
  if (!x || !theta || !xbits || !t || n < 1 || n_vis < 1 || hidden < 1) return fail(IRL_ERR_ARG, "bad prepare arguments");
  if (n_vis > OTF_MAX_NIN || (hidden & 1)) return fail(IRL_ERR_ARG, "on-the-fly RBM needs n_vis <= %d, even hidden", OTF_MAX_NIN);
  cudaStream_t st = (cudaStream_t)stream;
  IRL_TRY(pack_bits(x, n, n_vis, xbits, st));
  return launch_hidden<false, MODEL_RBM>(x, xbits, n, n_vis, hidden, theta + n_vis + hidden, theta + n_vis, nullptr, t,
                                         nullptr, st);
}

int irl_otf_colstats_rbm_f64(const uint64_t* xbits, const double* t, int64_t n, int n_vis, int hidden, int64_t ld,
                             const double* w, const double* coeff, double* obar, double* grad, void* ws,
                             size_t ws_bytes, void* stream) {
  if (!xbits || !t || !w || !coeff || !obar || !grad || n < 1) return fail(IRL_ERR_ARG, "null pointer");
  const int64_t P = (int64_t)n_vis + hidden + (int64_t)hidden * n_vis;
  if (ld != irl_padded_ld(P, 0)) return fail(IRL_ERR_ALIGN, "ld must equal irl_padded_ld(P=%lld)", (long long)P);
  OtfPlan pl;
  IRL_TRY(make_otf_plan(n, n_vis, hidden, pl));
  OtfWs wl = otf_ws_layout(pl, n, hidden, ws);
  if (ws_bytes < wl.bytes) return fail(IRL_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, wl.bytes);
  OtfArgs a{};
  a.xbits = xbits;
  a.T = t;
  a.G = t;
  a.n_rows = n;
  a.n_in = n_vis;
  a.hidden = hidden;
  DevInfo d;
  IRL_TRY(dev_info(d));
  const int nbx = std::min<int>(4 * d.sms, (int)std::max<int64_t>(1, n / 64));
  return otf_stats(pl, a, wl, MODEL_RBM, n, n_vis, hidden, ld, w, coeff, obar, grad, nullptr, nbx,
                   (cudaStream_t)stream);
}

static int otf_mvp_rbm_core(const uint64_t* xbits, const double* t, int64_t n, int n_vis, int hidden, int64_t ld,
                        const double* obar, const double* coeff, const double* v, double* out, const double* half_f,
                        const double* u0, double* out0, void* ws, size_t ws_bytes, void* stream, const OtfConn* cx) {
  if (!xbits || !t || (!coeff && !cx) || !v || !out || n < 1) return fail(IRL_ERR_ARG, "null pointer");
  const int64_t P = (int64_t)n_vis + hidden + (int64_t)hidden * n_vis;
  if (ld != irl_padded_ld(P, 0)) return fail(IRL_ERR_ALIGN, "ld must equal irl_padded_ld(P=%lld)", (long long)P);
  if (n_vis > OTF_MAX_NIN || (hidden & 1) || !aligned16(t)) return fail(IRL_ERR_ARG, "unsupported on-the-fly shape");
  OtfPlan pl;
  IRL_TRY(make_otf_plan(n, n_vis, hidden, pl));
  OtfWs wl = otf_ws_layout(pl, n, hidden, ws);
  if (ws_bytes < wl.bytes) return fail(IRL_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, wl.bytes);
  cudaStream_t st = (cudaStream_t)stream;
  DevInfo d;
  IRL_TRY(dev_info(d));
  IRL_TRY(launch_pdl(k_vdot2, dim3(pl.ny), dim3(256), 0, st, "otf vdot launch", obar, half_f, v, (int64_t)ld,
                     wl.dpart, wl.gpart));
  OtfArgs a{};
  a.xbits = xbits;
  a.T = t;
  a.G = t;
  a.n_rows = n;
  a.n_in = n_vis;
  a.hidden = hidden;
  a.nb = pl.nb;
  a.offW = (int64_t)n_vis + hidden;
  a.offb = n_vis;
  a.offu = -1;
  a.v = v;
  a.tpart = wl.tpart;
  a.y = wl.y;
  a.part = wl.part;
  a.partu = wl.partu;
  if (cx) IRL_TRY(otf_conn_partner_dot(*const_cast<OtfConn*>(cx), false, ld, v, nullptr, obar, st));
  IRL_TRY(otf_dot_launch(a, false, st));
  const double* ceff = coeff;
  const double* yadd = nullptr;
  if (cx) {
    if (cx->pxbits)
      IRL_TRY(otf_conn_regen_dots(*const_cast<OtfConn*>(cx), a, false, -1, 0, wl.dpart, obar ? pl.ny : 0, st));
    else if (!cx->partner_O)
      k_otf_y<<<pl.ny, 256, 0, st>>>(wl.tpart, pl.jc, n, nullptr, v, -1, wl.dpart, obar ? pl.ny : 0,
                                     (double*)cx->q, (double*)cx->qpart, xbits, 0, n_vis);
    IRL_TRY(otf_conn_rows(*const_cast<OtfConn*>(cx), false, n, st));
    ceff = (const double*)cx->a;
    yadd = (const double*)cx->d;
  }
  IRL_TRY(launch_pdl(k_otf_y, dim3(pl.ny), dim3(256), 0, st, "otf y launch", (const double*)wl.tpart, (int)pl.jc,
                     (int64_t)n, ceff, v, (int64_t)-1, (const double*)wl.dpart, obar ? pl.ny : 0, wl.y, wl.ypart,
                     xbits, (int64_t)0, n_vis, yadd));
  IRL_TRY(otf_acc_launch(pl, a, st, 1, false));
  const int nbx = std::min<int>(4 * d.sms, (int)std::max<int64_t>(1, n / 64));
  IRL_TRY(launch_pdl(k_xsum, dim3(nbx), dim3(128), 0, st, "otf xsum launch", xbits, (const double*)wl.y, (int64_t)n,
                     n_vis, wl.xpart, wl.ypart2));
  return launch_pdl(k_rbm_otf_finish, fin_grid(ld), dim3(32, 8), 0, st, "otf rbm finish launch",
                    (const double*)wl.part, (int)a.nb, hidden, n_vis, (int)pl.kc, (const double*)wl.xpart, nbx,
                    (const double*)wl.ypart, (int)pl.ny, (int64_t)ld, obar, half_f, u0, (const double*)wl.gpart,
                    (int)pl.ny, out, out0);
}

int irl_otf_mvp_rbm_f64(const uint64_t* xbits, const double* t, int64_t n, int n_vis, int hidden, int64_t ld,
                        const double* obar, const double* coeff, const double* v, double* out, const double* half_f,
                        const double* u0, double* out0, void* ws, size_t ws_bytes, void* stream) {
  return otf_mvp_rbm_core(xbits, t, n, n_vis, hidden, ld, obar, coeff, v, out, half_f, u0, out0, ws, ws_bytes, stream, nullptr);
}

int irl_otf_prepare_rbm_c128(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta,
                             uint64_t* xbits, double* t, void* stream) {
  if (!x || !theta || !xbits || !t || n < 1 || n_vis < 1 || hidden < 1) return fail(IRL_ERR_ARG, "bad prepare arguments");
  if (n_vis > OTF_MAX_NIN) return fail(IRL_ERR_ARG, "on-the-fly RBM needs n_vis <= %d", OTF_MAX_NIN);
  cudaStream_t st = (cudaStream_t)stream;
  IRL_TRY(pack_bits(x, n, n_vis, xbits, st));
  const double2* th = reinterpret_cast<const double2*>(theta);
  return launch_hidden<true, MODEL_RBM>(x, xbits, n, n_vis, hidden, th + n_vis + hidden, th + n_vis, nullptr, t,
                                        nullptr, st);
}

size_t irl_otf_workspace_bytes_c128(int64_t n, int n_vis, int hidden) {
  OtfCPlan p;
  if (make_otfc_plan(n, n_vis, hidden, p) != IRL_OK) return 0;
  return otfc_ws_layout(p, n, n_vis, hidden, nullptr).bytes;
}

int irl_otf_colstats_rbm_c128(const uint64_t* xbits, const double* t, int64_t n, int n_vis, int hidden, int64_t ld,
                              const double* w, const double* coeff, double* obar, double* grad, void* ws,
                              size_t ws_bytes, void* stream) {
  IRL_TRY(otfc_check(xbits, t, n, n_vis, hidden, ld));
  if (!w || !coeff || !obar || !grad) return fail(IRL_ERR_ARG, "null pointer");
  OtfCPlan pl;
  IRL_TRY(make_otfc_plan(n, n_vis, hidden, pl));
  OtfCWs wl = otfc_ws_layout(pl, n, n_vis, hidden, ws);
  if (ws_bytes < wl.bytes) return fail(IRL_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, wl.bytes);
  cudaStream_t st = (cudaStream_t)stream;
  OtfCArgs a{};
  a.xbits = xbits;
  a.T = t;
  a.n_rows = n;
  a.n_in = n_vis;
  a.hidden = hidden;
  // obar = sum w O = conj(sum w conj(O)) ; grad = sum c conj(O)
  IRL_TRY(otfc_colsum(pl, a, wl, ld, nullptr, w, reinterpret_cast<double2*>(obar), 1, st));
  return otfc_colsum(pl, a, wl, ld, reinterpret_cast<const double2*>(coeff), nullptr,
                     reinterpret_cast<double2*>(grad), 0, st);
}

static int otf_mvp_rbmc_core(const uint64_t* xbits, const double* t, int64_t n, int n_vis, int hidden, int64_t ld,
                         const double* obar, const double* coeff, const double* v_re, const double* v_im,
                         double* out_re, double* out_im, const double* half_f_re, const double* half_f_im,
                         const double* u0, double* out0, void* ws, size_t ws_bytes, void* stream, const OtfConn* cx) {
  IRL_TRY(otfc_check(xbits, t, n, n_vis, hidden, ld));
  if ((!coeff && !cx) || !v_re || !v_im || !out_re || !out_im) return fail(IRL_ERR_ARG, "null pointer");
  if ((half_f_re || u0 || out0) && !(half_f_re && half_f_im && u0 && out0))
    return fail(IRL_ERR_ARG, "bordered product needs half_f_re, half_f_im, u0 and out0");
  OtfCPlan pl;
  IRL_TRY(make_otfc_plan(n, n_vis, hidden, pl));
  OtfCWs wl = otfc_ws_layout(pl, n, n_vis, hidden, ws);
  if (ws_bytes < wl.bytes) return fail(IRL_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, wl.bytes);
  cudaStream_t st = (cudaStream_t)stream;
  const double2* ob = reinterpret_cast<const double2*>(obar);
  k_vdot_c<<<pl.ny, 256, 0, st>>>(ob, v_re, v_im, half_f_re, half_f_im, ld, wl.dpart, wl.gpart);
  if (cx) IRL_TRY(otf_conn_partner_dot(*const_cast<OtfConn*>(cx), true, ld, v_re, v_im, obar, st));
  OtfCArgs a{};
  a.xbits = xbits;
  a.T = t;
  a.n_rows = n;
  a.n_in = n_vis;
  a.hidden = hidden;
  a.nb = pl.nb_dot;
  a.offW = (int64_t)n_vis + hidden;
  a.offb = n_vis;
  a.v_re = v_re;
  a.v_im = v_im;
  a.tpart = wl.tpart;
  {
    CUtensorMap mt;
    IRL_TRY(tile_map(mt, t, 2LL * hidden, n));
    k_otf_dot_c<<<pl.nb_dot, 288, pl.smem_dot, st>>>(a, mt);
  }
  IRL_TRY(cuda_check(cudaGetLastError(), "otf dot (complex) launch"));
  const double2* ceff = reinterpret_cast<const double2*>(coeff);
  const double2* yadd = nullptr;
  if (cx) {
    if (!cx->partner_O)
      k_otf_y_c<<<pl.ny, 256, 0, st>>>(wl.tpart, pl.jc, n, nullptr, v_re, v_im, 0, n_vis, xbits, wl.dpart,
                                       obar ? pl.ny : 0, (double2*)cx->q, (double2*)cx->qpart);
    IRL_TRY(otf_conn_rows(*const_cast<OtfConn*>(cx), true, n, st));
    ceff = (const double2*)cx->a;
    yadd = (const double2*)cx->d;
  }
  k_otf_y_c<<<pl.ny, 256, 0, st>>>(wl.tpart, pl.jc, n, ceff, v_re, v_im, 0, n_vis, xbits, wl.dpart,
                                   obar ? pl.ny : 0, wl.y, wl.ypart, yadd);
  a.y = wl.y;
  a.yr = nullptr;
  a.part = wl.part;
  a.nb = pl.nb_acc;
  {
    CUtensorMap mt;
    IRL_TRY(tile_map(mt, a.T, 2LL * a.hidden, a.n_rows));
    pick_acc_c(pl.nkt)<<<dim3((unsigned)pl.jc, (unsigned)pl.nb_acc), 288, pl.smem_acc, st>>>(a, mt);
  }
  IRL_TRY(cuda_check(cudaGetLastError(), "otf acc (complex) launch"));
  k_xsum_c<<<pl.nbx, 128, 0, st>>>(xbits, wl.y, nullptr, n, n_vis, wl.xpart);
  k_rbm_otf_finish_c<<<fin_grid(ld), dim3(32, 8), 0, st>>>(wl.part, pl.nb_acc, hidden, n_vis, pl.kc, wl.xpart,
                                                             pl.nbx, wl.ypart, pl.ny, ld, ob, half_f_re, half_f_im,
                                                             u0, wl.gpart, pl.ny, out_re, out_im, out0, nullptr, 0);
  return cuda_check(cudaGetLastError(), "otf finish (complex) launch");
}

int irl_otf_mvp_rbm_c128(const uint64_t* xbits, const double* t, int64_t n, int n_vis, int hidden, int64_t ld,
                         const double* obar, const double* coeff, const double* v_re, const double* v_im,
                         double* out_re, double* out_im, const double* half_f_re, const double* half_f_im,
                         const double* u0, double* out0, void* ws, size_t ws_bytes, void* stream) {
  return otf_mvp_rbmc_core(xbits, t, n, n_vis, hidden, ld, obar, coeff, v_re, v_im, out_re, out_im, half_f_re, half_f_im, u0, out0, ws, ws_bytes, stream, nullptr);
}

int irl_lanczos_step_small(double* V, int64_t ldv, double* W, int64_t L, int j, int m, double* ab, void* stream) {
  if (!V || !W || !ab || L < 1 || j < 0 || j >= m || j + 1 > 63 || ldv < L) return fail(IRL_ERR_ARG, "bad lanczos step");
  k_lanczos_small<<<1, 1024, 0, (cudaStream_t)stream>>>(V, ldv, W, L, j, m, ab);
  return cuda_check(cudaGetLastError(), "lanczos step launch");
}

int irl_lanczos_step_cluster(double* V, int64_t ldv, double* W, int64_t L, int j, int m, double* ab, void* stream) {
  if (!V || !W || !ab || L < 1 || j < 0 || j >= m || j + 1 > LZ_MAXJ || ldv < L)
    return fail(IRL_ERR_ARG, "bad lanczos step");
  DevInfo d;
  IRL_TRY(dev_info(d));
  // static shared memory only; allow 16-CTA clusters (per device, via ensure_fn_attrs)
  IRL_TRY(ensure_fn_attrs((const void*)k_lanczos_cluster, d.smem_optin));
  const int cs = (int)std::min<int64_t>(16, std::max<int64_t>(2, cdiv(L, 512)));
  // shared-memory staged variant when this CTA's slice of rows 0..j (+ W) fits
  const int64_t slice = 2 * cdiv(L / 2, cs);
  const size_t stage_bytes = (size_t)(j + 2) * slice * 8;
  IRL_TRY(ensure_fn_attrs((const void*)k_lanczos_cluster_smem, d.smem_optin));
  const bool staged = (L % 2 == 0) && (ldv % 2 == 0) && aligned16(V) && aligned16(W) &&
                      stage_bytes + 4096 <= (size_t)d.smem_optin && getenv("IRL_LANCZOS_NOSTAGE") == nullptr;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = staged ? stage_bytes : 0;
  cfg.stream = (cudaStream_t)stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (staged)
    return cuda_check(cudaLaunchKernelEx(&cfg, k_lanczos_cluster_smem, V, ldv, W, L, j, m, ab),
                      "lanczos cluster launch");
  return cuda_check(cudaLaunchKernelEx(&cfg, k_lanczos_cluster, V, ldv, W, L, j, m, ab), "lanczos cluster launch");
}

int irl_host_qr_sweeps(int m, double* T, double* Q, const double* shifts, int nshift) {
  if (m < 2 || !T || !Q || (nshift > 0 && !shifts)) return fail(IRL_ERR_ARG, "bad qr sweep arguments");
  // kry:165-190 per shift, same operation order (full rows / columns, t <- G^T t G, q <- q G)
  for (int sidx = 0; sidx < nshift; ++sidx) {
    double x = T[0] - shifts[sidx], z = T[m];
    for (int k = 0; k < m - 1; ++k) {
      const double r = hypot(x, z);
      double c = 1.0, s = 0.0;
      if (r != 0.0) {
        c = x / r;
        s = z / r;
      }
      for (int col = 0; col < m; ++col) {
        const double a0 = T[k * m + col], a1 = T[(k + 1) * m + col];
        T[k * m + col] = c * a0 + s * a1;
        T[(k + 1) * m + col] = -s * a0 + c * a1;
      }
      for (int row = 0; row < m; ++row) {
        const double a0 = T[row * m + k], a1 = T[row * m + k + 1];
        T[row * m + k] = c * a0 + s * a1;
        T[row * m + k + 1] = -s * a0 + c * a1;
      }
      for (int row = 0; row < m; ++row) {
        const double a0 = Q[row * m + k], a1 = Q[row * m + k + 1];
        Q[row * m + k] = c * a0 + s * a1;
        Q[row * m + k + 1] = -s * a0 + c * a1;
      }
      if (k < m - 2) {
        x = T[(k + 1) * m + k];
        z = T[(k + 2) * m + k];
      }
    }
  }
  return IRL_OK;
}

size_t irl_connected_workspace_bytes(int64_t n, int64_t n_partner, int64_t ld, int is_complex) {
  return connected_ws_bytes(n, n_partner, ld, is_complex != 0);
}

int irl_connected_mvp_f64(const double* O, int64_t n, int64_t p, int64_t ld, const double* obar, const double* w,
                          const double* coeff, const int64_t* dist_index, const int64_t* indptr,
                          const int64_t* partner_row, const double* pcoeff, const double* partner_O,
                          int64_t n_partner, const double* v, double* out, const double* half_f, const double* u0,
                          double* out0, int mode, void* ws, size_t ws_bytes, void* stream) {
  return connected_impl(false, O, n, p, ld, obar, w, coeff, dist_index, indptr, partner_row, pcoeff, partner_O,
                        n_partner, v, nullptr, out, nullptr, half_f, nullptr, u0, out0, mode, ws, ws_bytes,
                        (cudaStream_t)stream);
}

int irl_connected_mvp_c128(const double* O, int64_t n, int64_t p, int64_t ld, const double* obar, const double* w,
                           const double* coeff, const int64_t* dist_index, const int64_t* indptr,
                           const int64_t* partner_row, const double* pcoeff, const double* partner_O,
                           int64_t n_partner, const double* v_re, const double* v_im, double* out_re,
                           double* out_im, const double* hf_re, const double* hf_im, const double* u0, double* out0,
                           int mode, void* ws, size_t ws_bytes, void* stream) {
  return connected_impl(true, O, n, p, ld, obar, w, coeff, dist_index, indptr, partner_row, pcoeff, partner_O,
                        n_partner, v_re, v_im, out_re, out_im, hf_re, hf_im, u0, out0, mode, ws, ws_bytes,
                        (cudaStream_t)stream);
}

size_t irl_logamp_workspace_bytes(int64_t n, int hidden, int is_complex) {
  return logamp_ws_bytes(n, hidden, is_complex != 0);
}

int irl_logamp_rbm_f64(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta, double* logpsi,
                       void* ws, size_t ws_bytes, void* stream) {
  return logamp_impl<false, MODEL_RBM>(x, n, n_vis, hidden, theta, logpsi, ws, ws_bytes, (cudaStream_t)stream);
}

int irl_logamp_rbm_c128(const uint8_t* x, int64_t n, int n_vis, int hidden, const double* theta, double* logpsi,
                        void* ws, size_t ws_bytes, void* stream) {
  return logamp_impl<true, MODEL_RBM>(x, n, n_vis, hidden, theta, logpsi, ws, ws_bytes, (cudaStream_t)stream);
}

int irl_logamp_mlp_f64(const uint8_t* x, int64_t n, int n_in, int hidden, const double* theta, double* logpsi,
                       void* ws, size_t ws_bytes, void* stream) {
  return logamp_impl<false, MODEL_MLP>(x, n, n_in, hidden, theta, logpsi, ws, ws_bytes, (cudaStream_t)stream);
}

size_t irl_ham_workspace_bytes(int n_spatial, int hidden, int is_complex) {
  return ham_ws_bytes(2 * n_spatial, hidden, is_complex != 0);
}

int irl_ham_local_energy(int model, int is_complex, const uint64_t* xbits, int64_t n, int n_spatial, double e_core,
                         const double* h1, const double* g2, double drop, int hidden, const double* theta,
                         double* eloc, void* ws, size_t ws_bytes, void* stream) {
  return ham_impl(model, is_complex != 0, HAM_ELOC, xbits, n, n_spatial, e_core, h1, g2, drop, hidden, theta, eloc,
                  nullptr, nullptr, nullptr, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

int irl_ham_connected_count(int model, int is_complex, const uint64_t* xbits, int64_t n, int n_spatial, double e_core,
                            const double* h1, const double* g2, double drop, int hidden, const double* theta,
                            int64_t* counts, void* ws, size_t ws_bytes, void* stream) {
  return ham_impl(model, is_complex != 0, HAM_COUNT, xbits, n, n_spatial, e_core, h1, g2, drop, hidden, theta,
                  nullptr, counts, nullptr, nullptr, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

int irl_ham_connected_fill(int model, int is_complex, const uint64_t* xbits, int64_t n, int n_spatial, double e_core,
                           const double* h1, const double* g2, double drop, int hidden, const double* theta,
                           const int64_t* offsets, uint64_t* partner_bits, double* elements, double* coeff, void* ws,
                           size_t ws_bytes, void* stream) {
  return ham_impl(model, is_complex != 0, HAM_FILL, xbits, n, n_spatial, e_core, h1, g2, drop, hidden, theta, nullptr,
                  nullptr, offsets, partner_bits, elements, coeff, ws, ws_bytes, (cudaStream_t)stream);
}

int irl_ham_diagonal_and_count(const uint64_t* xbits, int64_t n, int n_spatial, double e_core, const double* h1,
                               const double* g2, double drop, double* diag, int64_t* counts, void* stream) {
  return ham_impl(MODEL_NONE, false, HAM_COUNT, xbits, n, n_spatial, e_core, h1, g2, drop, 0, nullptr, nullptr, counts,
                  nullptr, nullptr, nullptr, nullptr, nullptr, 256, (cudaStream_t)stream, diag);
}

int irl_ham_partners_fill(const uint64_t* xbits, int64_t n, int n_spatial, double e_core, const double* h1,
                          const double* g2, double drop, const int64_t* offsets, uint64_t* partner_bits,
                          double* elements, void* stream) {
  return ham_impl(MODEL_NONE, false, HAM_FILL, xbits, n, n_spatial, e_core, h1, g2, drop, 0, nullptr, nullptr, nullptr,
                  offsets, partner_bits, elements, elements, nullptr, 256, (cudaStream_t)stream);
}

int irl_ar_logamp(const uint64_t* xbits, int64_t n, int n_orbitals, int hidden, int n_up, int n_down,
                  const double* theta, double* logpsi, int* error, void* stream) {
  IRL_TRY(ar_check(n, n_orbitals, hidden, n_up, n_down, theta));
  if (!xbits || !logpsi || !error) return fail(IRL_ERR_ARG, "null pointer");
  ArArgs a{};
  a.xbits = xbits;
  a.n = n;
  a.M = n_orbitals;
  a.h = hidden;
  a.n_up = n_up;
  a.n_down = n_down;
  a.theta = theta;
  a.logpsi = reinterpret_cast<double2*>(logpsi);
  a.error = error;
  return ar_launch<AR_LOGAMP>(a, (cudaStream_t)stream);
}

int irl_ar_rows(const uint64_t* xbits, int64_t n, int n_orbitals, int hidden, int n_up, int n_down,
                const double* theta, double* O, int64_t ld, int* error, void* stream) {
  IRL_TRY(ar_check(n, n_orbitals, hidden, n_up, n_down, theta));
  if (!xbits || !O || !error) return fail(IRL_ERR_ARG, "null pointer");
  const int64_t p = (int64_t)hidden * 2 * n_orbitals + hidden + 2 * hidden + 2 + (int64_t)hidden * n_orbitals + 2 * hidden +
                    n_orbitals + 1;
  if (ld < p) return fail(IRL_ERR_ARG, "ld %lld < param count %lld", (long long)ld, (long long)p);
  ArArgs a{};
  a.xbits = xbits;
  a.n = n;
  a.M = n_orbitals;
  a.h = hidden;
  a.n_up = n_up;
  a.n_down = n_down;
  a.theta = theta;
  a.O = reinterpret_cast<double2*>(O);
  a.ld = ld;
  a.error = error;
  return ar_launch<AR_ROWS>(a, (cudaStream_t)stream);
}

int irl_ar_sample(const uint64_t* rng_states, int64_t n, int n_orbitals, int hidden, int n_up, int n_down,
                  const double* theta, uint64_t* out_bits, int* error, void* stream) {
  IRL_TRY(ar_check(n, n_orbitals, hidden, n_up, n_down, theta));
  if (!rng_states || !out_bits || !error) return fail(IRL_ERR_ARG, "null pointer");
  ArArgs a{};
  a.n = n;
  a.M = n_orbitals;
  a.h = hidden;
  a.n_up = n_up;
  a.n_down = n_down;
  a.theta = theta;
  a.rng = rng_states;
  a.out_bits = out_bits;
  a.error = error;
  return ar_launch<AR_SAMPLE>(a, (cudaStream_t)stream);
}

int irl_eloc_combine(const int64_t* indptr, const double* elements, const double* logpsi_partner,
                     const double* logpsi_x, const double* diag, int64_t n, double* eloc, void* stream) {
  if (!indptr || !logpsi_x || !diag || !eloc || n < 0) return fail(IRL_ERR_ARG, "bad combine arguments");
  if (n == 0) return IRL_OK;
  k_eloc_combine<<<(unsigned)std::min<int64_t>(cdiv(n, 8), 148 * 16), 256, 0, (cudaStream_t)stream>>>(
      indptr, elements, reinterpret_cast<const double2*>(logpsi_partner), reinterpret_cast<const double2*>(logpsi_x),
      diag, n, reinterpret_cast<double2*>(eloc));
  return cuda_check(cudaGetLastError(), "combine launch");
}

int irl_sorted_lookup(const uint64_t* keys, int64_t n_keys, const uint64_t* queries, int64_t n_queries, int64_t* out,
                      void* stream) {
  if ((!keys && n_keys) || (!queries && n_queries) || (!out && n_queries) || n_keys < 0 || n_queries < 0)
    return fail(IRL_ERR_ARG, "bad lookup arguments");
  if (n_queries == 0) return IRL_OK;
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(n_queries, 256), 148 * 32);
  k_sorted_lookup<<<blocks, 256, 0, (cudaStream_t)stream>>>(keys, n_keys, queries, n_queries, out);
  return cuda_check(cudaGetLastError(), "lookup launch");
}

// ---- connected completion on on-the-fly batches (partner_O: stored partner
// rows, or NULL when partner_row indexes batch rows)
static int otf_conn_setup(OtfConn& cx, bool cplx, int64_t n, int64_t ld, const double* w, const double* coeff,
                          const int64_t* dist_index, const int64_t* indptr, const int64_t* partner_row,
                          const double* pcoeff, const double* partner_O, int64_t n_partner, void* ws,
                          size_t ws_bytes, size_t base_bytes, const uint64_t* pxbits = nullptr,
                          const double* pt = nullptr, const double* pg = nullptr, int n_in = 0, int hidden = 0) {
  if (!w || !dist_index || !indptr) return fail(IRL_ERR_ARG, "null cache pointer");
  if (n_partner < 0 || (n_partner > 0 && (!partner_row || !pcoeff))) return fail(IRL_ERR_ARG, "bad partner arguments");
  if (partner_O && !aligned16(partner_O)) return fail(IRL_ERR_ALIGN, "partner_O must be 16-byte aligned");
  cx = OtfConn{};
  cx.dist_index = dist_index;
  cx.indptr = indptr;
  cx.prow = partner_row;
  cx.pcoeff = pcoeff;
  cx.w = w;
  cx.cdiag = coeff;
  cx.partner_O = partner_O;
  cx.pxbits = pxbits;
  cx.pt = pt;
  cx.pg = pg;
  const bool regen = pxbits != nullptr;
  if (regen && (partner_O || cplx || !pt)) return fail(IRL_ERR_ARG, "bad regenerated-partner arguments");
  cx.m = (partner_O || regen) ? n_partner : n;
  const bool stored = partner_O != nullptr;
  if (stored && n_partner > 0) IRL_TRY(make_plan(n_partner, cplx ? ld : ld / 2, cplx, MODE_DOT, cx.pp));
  if (regen && n_partner > 0) IRL_TRY(make_otf_plan(n_partner, n_in, hidden, cx.ppl));
  const size_t need =
      align256(base_bytes) + otf_conn_carve(cx, n, cx.m, cplx, stored, nullptr, regen && n_partner > 0, hidden);
  if (ws_bytes < need) return fail(IRL_ERR_WORKSPACE, "workspace %zu < %zu", ws_bytes, need);
  otf_conn_carve(cx, n, cx.m, cplx, stored, static_cast<char*>(ws) + align256(base_bytes), regen && n_partner > 0,
                 hidden);
  if (regen && n_partner == 0) cx.pxbits = nullptr;
  return IRL_OK;
}

size_t irl_otf_connected_workspace_bytes(int model, int64_t n, int64_t n_partner, int n_in, int hidden, int64_t ld,
                                         int is_complex) {
  const bool cplx = is_complex != 0;
  const size_t base = cplx ? irl_otf_workspace_bytes_c128(n, n_in, hidden) : irl_otf_workspace_bytes(n, n_in, hidden);
  (void)model;
  OtfConn cx{};
  size_t extra = otf_conn_carve(cx, n, n, cplx, false, nullptr);
  if (n_partner > 0 && make_plan(n_partner, cplx ? ld : ld / 2, cplx, MODE_DOT, cx.pp) == IRL_OK)
    extra = std::max(extra, otf_conn_carve(cx, n, n_partner, cplx, true, nullptr));
  if (n_partner > 0 && !cplx && make_otf_plan(n_partner, n_in, hidden, cx.ppl) == IRL_OK)
    extra = std::max(extra, otf_conn_carve(cx, n, n_partner, cplx, false, nullptr, true, hidden));
  g_err.clear();
  return align256(base) + extra;
}

int irl_otf_connected_mvp_rbm_f64(const uint64_t* xbits, const double* t, int64_t n, int n_vis, int hidden,
                                  int64_t ld, const double* obar, const double* w, const double* coeff,
                                  const int64_t* dist_index, const int64_t* indptr, const int64_t* partner_row,
                                  const double* pcoeff, const double* partner_O, const uint64_t* partner_xbits,
                                  const double* partner_t, const double* partner_g, int64_t n_partner, const double* v,
                                  double* out, const double* half_f, const double* u0, double* out0, void* ws,
                                  size_t ws_bytes, void* stream) {
  const size_t base = irl_otf_workspace_bytes(n, n_vis, hidden);
  OtfConn cx;
  IRL_TRY(otf_conn_setup(cx, false, n, ld, w, coeff, dist_index, indptr, partner_row, pcoeff, partner_O, n_partner,
                         ws, ws_bytes, base, partner_xbits, partner_t, partner_g, n_vis, hidden));
  return otf_mvp_rbm_core(xbits, t, n, n_vis, hidden, ld, obar, coeff, v, out, half_f, u0, out0, ws, base, stream,
                          &cx);
}

int irl_otf_connected_mvp_mlp_f64(const uint64_t* xbits, const double* t, const double* g, int64_t n, int n_in,
                                  int hidden, int64_t ld, const double* obar, const double* w, const double* coeff,
                                  const int64_t* dist_index, const int64_t* indptr, const int64_t* partner_row,
                                  const double* pcoeff, const double* partner_O, const uint64_t* partner_xbits,
                                  const double* partner_t, const double* partner_g, int64_t n_partner, const double* v,
                                  double* out, const double* half_f, const double* u0, double* out0, void* ws,
                                  size_t ws_bytes, void* stream) {
  const size_t base = irl_otf_workspace_bytes(n, n_in, hidden);
  OtfConn cx;
  IRL_TRY(otf_conn_setup(cx, false, n, ld, w, coeff, dist_index, indptr, partner_row, pcoeff, partner_O, n_partner,
                         ws, ws_bytes, base, partner_xbits, partner_t, partner_g, n_in, hidden));
  return otf_mvp_mlp_core(xbits, t, g, n, n_in, hidden, ld, obar, coeff, v, out, half_f, u0, out0, ws, base, stream,
                          &cx);
}

int irl_otf_connected_mvp_rbm_c128(const uint64_t* xbits, const double* t, int64_t n, int n_vis, int hidden,
                                   int64_t ld, const double* obar, const double* w, const double* coeff,
                                   const int64_t* dist_index, const int64_t* indptr, const int64_t* partner_row,
                                   const double* pcoeff, const double* partner_O, int64_t n_partner,
                                   const double* v_re, const double* v_im, double* out_re, double* out_im,
                                   const double* hf_re, const double* hf_im, const double* u0, double* out0, void* ws,
                                   size_t ws_bytes, void* stream) {
  const size_t base = irl_otf_workspace_bytes_c128(n, n_vis, hidden);
  OtfConn cx;
  IRL_TRY(otf_conn_setup(cx, true, n, ld, w, coeff, dist_index, indptr, partner_row, pcoeff, partner_O, n_partner,
                         ws, ws_bytes, base));
  return otf_mvp_rbmc_core(xbits, t, n, n_vis, hidden, ld, obar, coeff, v_re, v_im, out_re, out_im, hf_re, hf_im, u0,
                           out0, ws, base, stream, &cx);
}

}  // extern "C"
