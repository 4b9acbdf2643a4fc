// TMA bulk-copy probe at a small SM quota: what limits one TMA warp reading mapped host memory?
// Each CTA (one warp) runs an S-stage ring of B-byte stages (host -> smem -> HBM) and varies:
//   ld_split : the stage's host run arrives as 1 bulk load (1) or as B/2KiB loads (16 at 32 KiB)
//   st_split : the stage leaves as 1 bulk store, B/2KiB bulk stores, or 0 (no store)
//   lag      : refill the stage right after its stores drained (0) or one iteration later (1)
// One JSON object per line.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void g2s(void* s, const void* g, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(su(s)), "l"(g), "r"(n), "r"(su(b)) : "memory");
}
__device__ __forceinline__ void s2g(void* g, const void* s, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(g), "r"(su(s)), "r"(n) : "memory");
}

__global__ void ring(const char* __restrict__ src, char* __restrict__ dst, size_t nchunks, uint32_t B, int S,
                     int ld_split, int st_split, int lag) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  unsigned char* buf = smem + 256;
  const int lane = threadIdx.x;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const size_t my = nchunks > blockIdx.x ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto chunk = [&](size_t k) { return (size_t)blockIdx.x + k * gridDim.x; };
  const uint32_t piece = 2048;
  const int nld = ld_split ? B / piece : 1, nst = st_split == 2 ? B / piece : st_split;
  auto issue = [&](size_t k) {
    const int s = k % S;
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&bar[s])), "r"(B) : "memory");
    __syncwarp();
    if (nld == 1) {
      if (lane == 0) g2s(buf + s * B, src + chunk(k) * B, B, &bar[s]);
    } else if (lane < nld) {
      g2s(buf + s * B + lane * piece, src + chunk(k) * B + lane * piece, piece, &bar[s]);
    }
  };
  for (size_t k = 0; k < (size_t)S && k < my; ++k) issue(k);
  for (size_t k = 0; k < my; ++k) {
    const int s = k % S;
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n"
                 :: "r"(su(&bar[s])), "r"((uint32_t)((k / S) & 1)) : "memory");
    if (nst == 1) {
      if (lane == 0) s2g(dst + chunk(k) * B, buf + s * B, B);
    } else if (nst > 1 && lane < nst) {
      s2g(dst + chunk(k) * B + lane * piece, buf + s * B + lane * piece, piece);
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (!lag) {
      if (k + S < my) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
        issue(k + S);
      }
    } else if (k >= 1 && k - 1 + S < my) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
      issue(k - 1 + S);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Warp-specialised variant: warp 0 issues one B-byte bulk load per stage; NC consumer warps copy the
// stage to HBM with ld.shared.v4 / st.global.v4 (contiguous or 2 KiB-scattered destinations) and
// release it on an `empty` mbarrier.
__global__ void ring_ws(const char* __restrict__ src, char* __restrict__ dst, size_t nchunks, uint32_t B, int S,
                        int scatter, unsigned long long dst_slots) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 16;
  unsigned char* buf = smem + 256;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NC = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su(&empty[s])), "r"(NC));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t my = nchunks > blockIdx.x ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto chunk = [&](size_t k) { return (size_t)blockIdx.x + k * gridDim.x; };
  auto waitp = [&](uint64_t* b, uint32_t par) {
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n"
                 :: "r"(su(b)), "r"(par) : "memory");
  };
  if (warp == 0) {
    for (size_t k = 0; k < my; ++k) {
      const int s = k % S;
      if (k >= (size_t)S) waitp(&empty[s], ((k / S) - 1) & 1);
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(&full[s])), "r"(B) : "memory");
        g2s(buf + s * B, src + chunk(k) * B, B, &full[s]);
      }
      __syncwarp();
    }
  } else {
    const int ct = threadIdx.x - 32, nt = NC * 32;
    const int nvec = B / 16;
    for (size_t k = 0; k < my; ++k) {
      const int s = k % S;
      waitp(&full[s], (k / S) & 1);
      for (int v = ct; v < nvec; v += nt) {
        int4 val;
        asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(val.x), "=r"(val.y), "=r"(val.z), "=r"(val.w)
                     : "r"(su(buf + s * B + v * 16)));
        size_t off = chunk(k) * B + v * 16;
        if (scatter) {   // each 2 KiB row to a pseudo-random 2 KiB slot
          const size_t row = off >> 11;
          off = (((row * 2654435761ull) % dst_slots) << 11) + (off & 2047);
        }
        *reinterpret_cast<int4*>(dst + off) = val;
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su(&empty[s])) : "memory");
    }
  }
}

int main() {
  const size_t bytes = size_t(256) << 20;
  char *h, *hd, *d;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(h, 1, bytes);
  CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
  CK(cudaMalloc(&d, bytes));
  CK(cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const uint32_t B = 32768;
  CK(cudaFuncSetAttribute(ring_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  for (int S : {4, 6}) {
    for (int nc : {1, 2, 4, 8}) {
      for (int scatter : {0, 1}) {
        for (int ctas : {1, 2}) {
          std::vector<float> ms;
          for (int rep = 0; rep < 4; ++rep) {
            CK(cudaEventRecord(a));
            ring_ws<<<ctas, 32 * (1 + nc), 256 + S * B>>>(hd, d, bytes / B, B, S, scatter, bytes / 2048);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float t;
            CK(cudaEventElapsedTime(&t, a, b));
            if (rep) ms.push_back(t);
          }
          std::sort(ms.begin(), ms.end());
          printf("{\"kind\":\"tma_ws\",\"S\":%d,\"consumers\":%d,\"scatter\":%d,\"ctas\":%d,\"gbs\":%.2f}\n", S, nc, scatter,
                 ctas, bytes / ms[1] / 1e6);
          fflush(stdout);
        }
      }
    }
  }
  for (int S : {4, 6}) {
    for (int ld : {0, 1}) {
      for (int st : {1, 2, 0}) {
        for (int lag : {0, 1}) {
          for (int ctas : {1, 2}) {
            std::vector<float> ms;
            for (int rep = 0; rep < 4; ++rep) {
              CK(cudaEventRecord(a));
              ring<<<ctas, 32, 256 + S * B>>>(hd, d, bytes / B, B, S, ld, st, lag);
              CK(cudaEventRecord(b));
              CK(cudaEventSynchronize(b));
              float t;
              CK(cudaEventElapsedTime(&t, a, b));
              if (rep) ms.push_back(t);
            }
            std::sort(ms.begin(), ms.end());
            printf("{\"kind\":\"tma_ring\",\"S\":%d,\"ld_split\":%d,\"st_split\":%d,\"lag\":%d,\"ctas\":%d,\"gbs\":%.2f}\n", S,
                   ld, st, lag, ctas, bytes / ms[1] / 1e6);
            fflush(stdout);
          }
        }
      }
    }
  }
  return 0;
}
