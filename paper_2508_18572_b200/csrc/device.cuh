// device.cuh — sm_100a device primitives shared by the libstrata kernels (kernels.cu, ring.cu):
// 16-byte vector accesses, mbarriers, cp.async.bulk (TMA, non-tensor) copies, completion fences.
// Inline PTX, sm_100a only.  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace strata {
namespace dev {

constexpr unsigned kFull = 0xffffffffu;

// ---- 16-byte vectors.  Sources are read once: no L1 allocation. ----
__device__ __forceinline__ int4 ld_stream(const void* ptr) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(ptr));
  return r;
}
__device__ __forceinline__ void st_vec(void* ptr, const int4& v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" :: "l"(ptr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ int4 ld_shared_v4(const void* p) {
  int4 r;
  asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void st_shared_v4(void* p, const int4& v) {
  asm volatile("st.shared.v4.s32 [%0], {%1,%2,%3,%4};" :: "r"(smem_u32(p)), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}

// Address of 16-byte vector w of a row on one side: rows whose heads are adjacent are contiguous;
// otherwise head h = w / vph sits at h * stride (device HND / padded heads, head-major host tiers).
// P: any parameter block with vph / vph_shift (XferParams).
template <bool CONTIG, class P>
__device__ __forceinline__ uint64_t row_vec(uint64_t base, int w, const P& p, int64_t stride) {
  if (CONTIG) return base + static_cast<uint64_t>(w) * 16;
  const int h = p.vph_shift >= 0 ? (w >> p.vph_shift) : (w / p.vph);
  return base + h * stride + static_cast<uint64_t>(w - h * p.vph) * 16;
}

// ---- mbarriers ----
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" :: "r"(smem_u32(b)), "r"(parity) : "memory");
}

// ---- cp.async.bulk (TMA engine, non-tensor) ----
// global (device or mapped host) -> shared, completes `bytes` on barrier `bar`
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// the same with an L2 cache-policy operand (A/B: evict-first host reads, STRATA_RING_DEBUG bit 1)
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               :: "r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
// shared -> global (device or mapped host), tracked by this thread's bulk async-groups
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// this thread's bulk groups: all but the newest N have finished reading shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}
// GPU global timer (ns)
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// this thread's bulk groups: all complete (writes performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the async proxy (a following bulk store)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// async-proxy global writes (completed bulk stores) -> ordered before this thread's generic accesses
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ---- cp.async (LSU asynchronous global -> shared, 16 bytes), completion on an mbarrier ----
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
// arrive on `bar` once every cp.async this thread issued so far has landed (counts as one of the
// barrier's expected arrivals: .noinc)
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" :: "r"(smem_u32(bar)) : "memory");
}

// ---- completion publication ----
// Loads land in HBM and are consumed by GPU work: GPU-scope fences.  Offloads land in host memory,
// which the host may read after the event: system scope.
template <int DIR>
__device__ __forceinline__ void layer_fence() {
  if (DIR == 0) __threadfence();
  else __threadfence_system();
}
template <int DIR>
__device__ __forceinline__ void st_release(uint32_t* a, uint32_t v) {
  if (DIR == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(a), "r"(v) : "memory");
  else asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(a), "r"(v) : "memory");
}

// Launch through cudaLaunchKernel: the return value is this launch's own status, never an error
// another component left pending on the thread (<<<>>> + cudaGetLastError would report, and
// clear, that error as ours).
template <class P>
inline cudaError_t launch_k(void (*kernel)(P), int grid, int block, size_t smem, cudaStream_t s, const P& p) {
  void* args[] = {const_cast<P*>(&p)};
  return cudaLaunchKernel(reinterpret_cast<const void*>(kernel), dim3(grid), dim3(block), args, smem, s);
}

}  // namespace dev
}  // namespace strata
