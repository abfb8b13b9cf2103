// Shared device helpers for the IRL-SR hot path (sm_100a only).
//
// Element model: every kernel streams O in 16-byte "units".  A real (f64)
// unit holds two consecutive parameters; a complex (c128) unit holds one
// complex parameter (re, im).  Traits<CPLX> gives the scalar type S of the
// per-row quantities (t_n = O_n . v, y_n, coefficients) and the two inner
// products the MVP needs:
//   dot_acc : d += O_unit . v_unit               (no conjugation, est:185)
//   axpy    : a += conj(O_unit) * y              (est:186 `@ o_c.conj()`)
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#if !defined(__CUDA_ARCH__) || (__CUDA_ARCH__ >= 1000)
#else
#error "this library targets sm_100a only"
#endif

namespace irl {

template <bool CPLX> struct Traits;

template <> struct Traits<false> {
  using S = double;
  static constexpr int kElemsPerUnit = 2;
  __device__ __forceinline__ static S zero() { return 0.0; }
  __device__ __forceinline__ static void dot_acc(S& d, double2 u, double2 v) {
    d = fma(u.x, v.x, d);
    d = fma(u.y, v.y, d);
  }
  __device__ __forceinline__ static void axpy(double2& a, double2 u, S y) {
    a.x = fma(u.x, y, a.x);
    a.y = fma(u.y, y, a.y);
  }
  __device__ __forceinline__ static S add(S a, S b) { return a + b; }
  __device__ __forceinline__ static S sub(S a, S b) { return a - b; }
  __device__ __forceinline__ static S mul(S a, S b) { return a * b; }
  __device__ __forceinline__ static S shfl_xor(S a, int m) { return __shfl_xor_sync(0xffffffffu, a, m); }
  __device__ __forceinline__ static S shfl(S a, int src) { return __shfl_sync(0xffffffffu, a, src); }
};

template <> struct Traits<true> {
  using S = double2;
  static constexpr int kElemsPerUnit = 1;
  __device__ __forceinline__ static S zero() { return make_double2(0.0, 0.0); }
  // d += u * v  (complex, no conjugation)
  __device__ __forceinline__ static void dot_acc(S& d, double2 u, double2 v) {
    d.x = fma(u.x, v.x, d.x);
    d.x = fma(-u.y, v.y, d.x);
    d.y = fma(u.x, v.y, d.y);
    d.y = fma(u.y, v.x, d.y);
  }
  // a += conj(u) * y
  __device__ __forceinline__ static void axpy(double2& a, double2 u, S y) {
    a.x = fma(u.x, y.x, a.x);
    a.x = fma(u.y, y.y, a.x);
    a.y = fma(u.x, y.y, a.y);
    a.y = fma(-u.y, y.x, a.y);
  }
  __device__ __forceinline__ static S add(S a, S b) { return make_double2(a.x + b.x, a.y + b.y); }
  __device__ __forceinline__ static S sub(S a, S b) { return make_double2(a.x - b.x, a.y - b.y); }
  __device__ __forceinline__ static S mul(S a, S b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
  }
  __device__ __forceinline__ static S shfl_xor(S a, int m) {
    return make_double2(__shfl_xor_sync(0xffffffffu, a.x, m), __shfl_xor_sync(0xffffffffu, a.y, m));
  }
  __device__ __forceinline__ static S shfl(S a, int src) {
    return make_double2(__shfl_sync(0xffffffffu, a.x, src), __shfl_sync(0xffffffffu, a.y, src));
  }
};

template <bool CPLX>
__device__ __forceinline__ typename Traits<CPLX>::S warp_sum(typename Traits<CPLX>::S v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v = Traits<CPLX>::add(v, Traits<CPLX>::shfl_xor(v, m));
  return v;
}

// ---------------------------------------------------------------- PTX ----
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

// non-blocking probe (try_wait may suspend the thread for a system-dependent
// time before failing, which stalls a warp that polls two barriers in turn)
__device__ __forceinline__ bool mbar_test_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_addr(bar);
  while (!mbar_try_wait(a, parity)) {
  }
}

// 1-D bulk copy global -> shared (TMA engine, SASS UBLKCP), completes on bar.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// 2-D tensor-map copy global -> shared (TMA engine, SASS UTMALDG), completes on bar.
// c0 = inner (column) coordinate, c1 = row coordinate; out-of-bounds elements are zero.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_sync() {
  cluster_arrive();
  cluster_wait();
}

// shared::cta address -> shared::cluster address of the same offset in CTA `rank`
__device__ __forceinline__ uint32_t map_to_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

// Remote store that completes `bytes` of tx on the destination CTA's mbarrier.
__device__ __forceinline__ void st_async(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async(uint32_t raddr, double2 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(
                   raddr),
               "l"(__double_as_longlong(v.x)), "l"(__double_as_longlong(v.y)), "r"(rbar)
               : "memory");
}

__device__ __forceinline__ double ld_cluster(uint32_t addr, double*) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ double2 ld_cluster(uint32_t addr, double2*) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
  return v;
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Streaming 16-B store (evict-first): O is written once and read by later passes.
__device__ __forceinline__ void st_stream(double2* p, double2 v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

}  // namespace irl
