// Box probe for the Strata I/O path.
//
// Measures, on one B200, the ceilings every later number is divided by:
//   * contiguous pinned cudaMemcpyAsync H2D / D2H (the link roofline),
//   * SM-issued zero-copy reads of mapped host memory (LDG.128 from host VA),
//     swept over CTAs x threads x unroll x cache hint (Little's law, §3.1),
//   * SM-issued zero-copy writes to mapped host memory (offload direction),
//   * TMA bulk copies (cp.async.bulk) with a host-VA source / destination,
//   * host-read round-trip latency (pointer chase).
// Output: one JSON object per line on stdout.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o probe probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>
#include <algorithm>
#include <string>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

static float median(std::vector<float> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; }

// ----------------------------------------------------------------------------------------------
// LDG/STG copy: warp w moves segments of 32*U int4 (512*U bytes) contiguous; grid-stride.
template <int U, int HINT>
__device__ __forceinline__ int4 ld_src(const int4* p) {
  int4 r;
  if (HINT == 0) {
    asm volatile("ld.global.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  } else if (HINT == 1) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  }
  return r;
}

template <int U, int HINT>
__global__ void copy_kernel(const int4* __restrict__ src, int4* __restrict__ dst, size_t nvec) {
  const int lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = (gridDim.x * (size_t)blockDim.x) >> 5;
  const size_t seg = 32 * U;
  const size_t nseg = nvec / seg;
  for (size_t s = warp; s < nseg; s += nwarps) {
    const int4* sp = src + s * seg + lane;
    int4* dp = dst + s * seg + lane;
    int4 v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) v[j] = ld_src<U, HINT>(sp + j * 32);
#pragma unroll
    for (int j = 0; j < U; ++j) {
      if (HINT == 0) dp[j * 32] = v[j];
      else asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" :: "l"(dp + j * 32),
                        "r"(v[j].x), "r"(v[j].y), "r"(v[j].z), "r"(v[j].w) : "memory");
    }
  }
}

// ----------------------------------------------------------------------------------------------
// TMA bulk copy: one elected thread per CTA; S stages of B bytes in shared memory.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" :: "r"(smem_u32(b)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__global__ void tma_copy_kernel(const char* __restrict__ src, char* __restrict__ dst, size_t nchunks,
                                uint32_t B, int S) {
  extern __shared__ __align__(128) char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  char* buf = smem + 128;
  if (threadIdx.x != 0) return;
  for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  // chunks of this CTA: blockIdx.x, +gridDim.x, ...
  size_t my = (nchunks > blockIdx.x) ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto chunk = [&](size_t k) { return (size_t)blockIdx.x + k * gridDim.x; };
  for (size_t k = 0; k < (size_t)S && k < my; ++k) {
    mbar_expect_tx(&bars[k], B);
    bulk_g2s(buf + k * B, src + chunk(k) * B, B, &bars[k]);
  }
  for (size_t k = 0; k < my; ++k) {
    int s = k % S;
    mbar_wait(&bars[s], (k / S) & 1);
    bulk_s2g(dst + chunk(k) * B, buf + s * B, B);
    bulk_commit();
    size_t nx = k + S;
    if (nx < my) {
      bulk_wait_read<0>();
      mbar_expect_tx(&bars[s], B);
      bulk_g2s(buf + s * B, src + chunk(nx) * B, B, &bars[s]);
    }
  }
  bulk_wait_all();
}

// ----------------------------------------------------------------------------------------------
__global__ void chase_kernel(const uint64_t* __restrict__ chain, int hops, uint64_t start, long long* out,
                             uint64_t* sink) {
  uint64_t idx = start;
  long long t0 = clock64();
  for (int i = 0; i < hops; ++i) idx = *reinterpret_cast<const volatile uint64_t*>(chain + idx);
  long long t1 = clock64();
  out[0] = t1 - t0;
  sink[0] = idx;
}

// ----------------------------------------------------------------------------------------------
struct Timer {
  cudaEvent_t a, b; cudaStream_t s;
  Timer(cudaStream_t s_) : s(s_) { CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); }
  void start() { CK(cudaEventRecord(a, s)); }
  float stop() { CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b)); float ms; CK(cudaEventElapsedTime(&ms, a, b)); return ms; }
};

template <int U, int HINT>
static void launch_copy(int ctas, int threads, const void* src, void* dst, size_t bytes, cudaStream_t s) {
  copy_kernel<U, HINT><<<ctas, threads, 0, s>>>((const int4*)src, (int4*)dst, bytes / 16);
}
typedef void (*copy_fn)(int, int, const void*, void*, size_t, cudaStream_t);
static copy_fn pick(int U, int hint) {
#define P(u) if (U == u) { if (hint == 0) return launch_copy<u, 0>; if (hint == 1) return launch_copy<u, 1>; return launch_copy<u, 2>; }
  P(1) P(2) P(4) P(8) P(16)
#undef P
  return nullptr;
}

int main(int argc, char** argv) {
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int pageable = 0, canmap = 0, hostreg = 0, pciBus = 0, pciDev = 0;
  cudaDeviceGetAttribute(&pageable, cudaDevAttrPageableMemoryAccess, dev);
  cudaDeviceGetAttribute(&canmap, cudaDevAttrCanMapHostMemory, dev);
  cudaDeviceGetAttribute(&hostreg, cudaDevAttrHostRegisterSupported, dev);
  cudaDeviceGetAttribute(&pciBus, cudaDevAttrPciBusId, dev);
  cudaDeviceGetAttribute(&pciDev, cudaDevAttrPciDeviceId, dev);
  printf("{\"kind\":\"device\",\"name\":\"%s\",\"sms\":%d,\"cc\":\"%d.%d\",\"pageable_access\":%d,\"can_map\":%d,"
         "\"host_register\":%d,\"pci_bus\":%d,\"smem_optin\":%zu,\"param_max\":%d}\n",
         prop.name, prop.multiProcessorCount, prop.major, prop.minor, pageable, canmap, hostreg, pciBus,
         prop.sharedMemPerBlockOptin, 32764);
  fflush(stdout);

  const size_t big = (size_t)1 << 30;      // 1 GiB contiguous
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  char* h = nullptr; CK(cudaHostAlloc(&h, big, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(h, 0x5a, big);
  char* hd = nullptr; CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
  char* d = nullptr; CK(cudaMalloc(&d, big));
  char* d2 = nullptr; CK(cudaMalloc(&d2, big));
  Timer t(s);

  // 1. contiguous memcpy (the roofline)
  for (size_t sz : {(size_t)64 << 20, (size_t)256 << 20, big}) {
    for (int dir = 0; dir < 2; ++dir) {
      std::vector<float> v;
      for (int i = 0; i < 23; ++i) {
        t.start();
        if (dir == 0) CK(cudaMemcpyAsync(d, h, sz, cudaMemcpyHostToDevice, s));
        else CK(cudaMemcpyAsync(h, d, sz, cudaMemcpyDeviceToHost, s));
        float ms = t.stop();
        if (i >= 3) v.push_back(ms);
      }
      float m = median(v);
      printf("{\"kind\":\"memcpy\",\"dir\":\"%s\",\"bytes\":%zu,\"ms\":%.4f,\"gbs\":%.2f,\"min_ms\":%.4f}\n",
             dir == 0 ? "h2d" : "d2h", sz, m, sz / m / 1e6, *std::min_element(v.begin(), v.end()));
      fflush(stdout);
    }
  }
  // bidirectional memcpy
  {
    cudaStream_t s2; CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    char* h2; CK(cudaHostAlloc(&h2, (size_t)256 << 20, cudaHostAllocMapped | cudaHostAllocPortable));
    const size_t sz = (size_t)256 << 20;
    std::vector<float> v;
    cudaEvent_t e0, e1, e2; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
    for (int i = 0; i < 13; ++i) {
      CK(cudaEventRecord(e0, s)); CK(cudaStreamWaitEvent(s2, e0));
      CK(cudaMemcpyAsync(d, h, sz, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(h2, d2, sz, cudaMemcpyDeviceToHost, s2));
      CK(cudaEventRecord(e2, s2)); CK(cudaStreamWaitEvent(s, e2)); CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (i >= 3) v.push_back(ms);
    }
    float m = median(v);
    printf("{\"kind\":\"memcpy_bidir\",\"bytes_each\":%zu,\"ms\":%.4f,\"gbs_total\":%.2f}\n", sz, m, 2 * sz / m / 1e6);
    fflush(stdout);
    cudaFreeHost(h2);
  }

  // 2. zero-copy read sweep (host -> device)  and  3. zero-copy write sweep (device -> host)
  const size_t zsz = (size_t)256 << 20;
  for (int dir = 0; dir < 2; ++dir) {
    for (int hint : {0, 1, 2}) {
      if (dir == 1 && hint == 2) continue;
      for (int U : {1, 2, 4, 8, 16}) {
        for (int threads : {256, 512, 1024}) {
          if (U == 16 && threads == 1024) continue;
          for (int ctas : {1, 2, 4, 8, 16, 32, 64, 148, 296}) {
            if (dir == 1 && hint == 1 && U == 16) continue;
            copy_fn f = pick(U, hint);
            const void* src = dir == 0 ? (const void*)hd : (const void*)d;
            void* dst = dir == 0 ? (void*)d : (void*)hd;
            size_t sz = zsz;
            if (ctas <= 2) sz = (size_t)64 << 20;
            std::vector<float> v;
            for (int i = 0; i < 5; ++i) {
              t.start(); f(ctas, threads, src, dst, sz, s); float ms = t.stop();
              if (i >= 2) v.push_back(ms);
            }
            CK(cudaGetLastError());
            float m = median(v);
            printf("{\"kind\":\"zc\",\"dir\":\"%s\",\"hint\":%d,\"U\":%d,\"threads\":%d,\"ctas\":%d,\"bytes\":%zu,"
                   "\"inflight_kb\":%.1f,\"ms\":%.4f,\"gbs\":%.2f}\n",
                   dir == 0 ? "h2d" : "d2h", hint, U, threads, ctas, sz, ctas * threads * U * 16 / 1024.0, m,
                   sz / m / 1e6);
            fflush(stdout);
          }
        }
      }
    }
  }
  // correctness spot check of the zero-copy read
  {
    for (size_t i = 0; i < (size_t)(1 << 20); ++i) h[i] = (char)(i * 7 + 3);
    copy_kernel<4, 1><<<8, 512, 0, s>>>((const int4*)hd, (int4*)d, (1 << 20) / 16);
    CK(cudaStreamSynchronize(s));
    std::vector<char> back(1 << 20);
    CK(cudaMemcpy(back.data(), d, 1 << 20, cudaMemcpyDeviceToHost));
    printf("{\"kind\":\"zc_check\",\"ok\":%d}\n", memcmp(back.data(), h, 1 << 20) == 0);
    fflush(stdout);
  }

  // 4. TMA bulk copy with host VA as source (h2d) and as destination (d2h)
  CK(cudaFuncSetAttribute(tma_copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (int dir = 0; dir < 2; ++dir) {
    for (uint32_t B : {4096u, 16384u, 32768u}) {
      for (int S : {2, 4, 8}) {
        if ((size_t)B * S > 190 * 1024) continue;
        for (int ctas : {1, 2, 4, 8, 16, 32, 148}) {
          size_t sz = ctas <= 2 ? ((size_t)64 << 20) : zsz;
          size_t nchunks = sz / B;
          const char* src = dir == 0 ? hd : d;
          char* dst = dir == 0 ? d : hd;
          std::vector<float> v;
          cudaError_t err = cudaSuccess;
          for (int i = 0; i < 5; ++i) {
            t.start();
            tma_copy_kernel<<<ctas, 32, 128 + B * S, s>>>(src, dst, nchunks, B, S);
            float ms = t.stop();
            err = cudaGetLastError();
            if (err != cudaSuccess) break;
            if (i >= 2) v.push_back(ms);
          }
          if (err != cudaSuccess) {
            printf("{\"kind\":\"tma\",\"dir\":\"%s\",\"error\":\"%s\"}\n", dir == 0 ? "h2d" : "d2h", cudaGetErrorString(err));
            fflush(stdout);
            return 0;
          }
          float m = median(v);
          printf("{\"kind\":\"tma\",\"dir\":\"%s\",\"B\":%u,\"S\":%d,\"ctas\":%d,\"bytes\":%zu,\"inflight_kb\":%.1f,"
                 "\"ms\":%.4f,\"gbs\":%.2f}\n", dir == 0 ? "h2d" : "d2h", B, S, ctas, sz, ctas * B * S / 1024.0, m,
                 sz / m / 1e6);
          fflush(stdout);
        }
      }
    }
  }
  {
    for (size_t i = 0; i < (size_t)(1 << 20); ++i) h[i] = (char)(i * 13 + 1);
    CK(cudaMemset(d, 0, 1 << 20));
    tma_copy_kernel<<<4, 32, 128 + 16384 * 4, s>>>(hd, d, (1 << 20) / 16384, 16384, 4);
    CK(cudaStreamSynchronize(s));
    std::vector<char> back(1 << 20);
    CK(cudaMemcpy(back.data(), d, 1 << 20, cudaMemcpyDeviceToHost));
    printf("{\"kind\":\"tma_check\",\"ok\":%d}\n", memcmp(back.data(), h, 1 << 20) == 0);
    fflush(stdout);
  }

  // 5. pointer-chase latency over host memory (stride 4 KiB + random permutation)
  {
    const size_t n = (size_t)64 << 20;  // 64 MiB of chain
    uint64_t* chain = reinterpret_cast<uint64_t*>(h);
    const size_t stride = 4096 / 8 + 8;  // elements
    size_t cnt = n / 8 / stride;
    std::vector<size_t> perm(cnt);
    for (size_t i = 0; i < cnt; ++i) perm[i] = i;
    srand(1);
    for (size_t i = cnt - 1; i > 0; --i) std::swap(perm[i], perm[rand() % (i + 1)]);
    for (size_t i = 0; i < cnt; ++i) chain[perm[i] * stride] = perm[(i + 1) % cnt] * stride;
    long long* out; uint64_t* sink; CK(cudaMalloc(&out, 8)); CK(cudaMalloc(&sink, 8));
    for (int rep = 0; rep < 3; ++rep) {
      chase_kernel<<<1, 1, 0, s>>>(reinterpret_cast<const uint64_t*>(hd), 2000, perm[0] * stride, out, sink);
      CK(cudaStreamSynchronize(s));
      long long cyc; CK(cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost));
      int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
      printf("{\"kind\":\"host_latency\",\"cycles_per_hop\":%.1f,\"clock_khz\":%d,\"ns_per_hop_at_max\":%.1f}\n",
             cyc / 2000.0, clk, cyc / 2000.0 / (clk / 1e6));
      fflush(stdout);
    }
  }
  return 0;
}
