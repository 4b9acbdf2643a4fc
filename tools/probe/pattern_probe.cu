// Access-pattern probe for SM zero-copy reads at a small SM quota (1-2 CTAs).
// Same copy loop as probe.cu (warp moves U*512 B: U LDG.128 from mapped host memory, then U STG.128),
// but the 2 KiB segment -> address maps vary:
//   src: "seq"   contiguous host stream
//        "run<K>" runs of K KiB at random 8 MiB-aligned chunk offsets (the page-first tier: one
//               chunk-layer's K rows are a 128 KiB run inside an 8 MiB chunk)
//   dst: "seq"   contiguous device stream
//        "rand"  each 2 KiB segment to a random 2 KiB slot (page size 1)
// One JSON object per line.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pattern_probe pattern_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ int4 ldnc(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z),
               "=r"(r.w) : "l"(p));
  return r;
}

// segment s (2 KiB) reads src + soff[s], writes dst + doff[s]
template <int U>
__global__ void seg_copy(const char* __restrict__ src, char* __restrict__ dst, const long long* __restrict__ soff,
                         const long long* __restrict__ doff, int nseg) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  constexpr int SEG = 2048, PER = 32 * U * 16;   // bytes per warp iteration
  constexpr int SPI = PER / SEG;                 // segments per iteration
  for (int it = warp; it * SPI < nseg; it += nwarps) {
    int4 v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int b = (j * 32 + lane) * 16;      // byte inside the iteration
      const int s = it * SPI + b / SEG;
      v[j] = ldnc(src + soff[s] + (b % SEG));
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int b = (j * 32 + lane) * 16;
      const int s = it * SPI + b / SEG;
      *reinterpret_cast<int4*>(dst + doff[s] + (b % SEG)) = v[j];
    }
  }
}

int main() {
  const size_t host_bytes = size_t(4) << 30, total = size_t(256) << 20, dev_bytes = size_t(1) << 30;
  const int nseg = int(total / 2048);
  char *h, *hd, *d;
  CK(cudaHostAlloc(&h, host_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(h, 3, host_bytes);
  CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
  CK(cudaMalloc(&d, dev_bytes));
  long long *soff, *doff;
  CK(cudaMalloc(&soff, nseg * 8));
  CK(cudaMalloc(&doff, nseg * 8));
  std::mt19937_64 rng(5);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  struct Src { const char* name; size_t run; };
  const Src srcs[] = {{"seq", 0}, {"run32", 32 << 10}, {"run128", 128 << 10}, {"run512", 512 << 10},
                      {"run2048", 2 << 20}};
  for (const Src& sp : srcs) {
    std::vector<long long> so(nseg);
    if (!sp.run) {
      for (int s = 0; s < nseg; ++s) so[s] = (long long)s * 2048;
    } else {
      const size_t per_run = sp.run / 2048, nchunks = host_bytes / (8 << 20);
      std::vector<size_t> chunk(nchunks);
      std::iota(chunk.begin(), chunk.end(), 0);
      std::shuffle(chunk.begin(), chunk.end(), rng);
      for (int s = 0; s < nseg; ++s) {
        const size_t r = s / per_run, within = s % per_run;
        // run r: chunk[r % nchunks], run slot (r / nchunks) inside the 8 MiB chunk
        const size_t c = chunk[r % nchunks], slot = (r / nchunks) % ((8 << 20) / sp.run);
        so[s] = (long long)(c * (8 << 20) + slot * sp.run + within * 2048);
      }
    }
    CK(cudaMemcpy(soff, so.data(), nseg * 8, cudaMemcpyHostToDevice));
    for (int dr = 0; dr < 2; ++dr) {
      std::vector<long long> dof(nseg);
      std::vector<long long> slots(dev_bytes / 2048);
      std::iota(slots.begin(), slots.end(), 0);
      if (dr) std::shuffle(slots.begin(), slots.end(), rng);
      for (int s = 0; s < nseg; ++s) dof[s] = slots[s] * 2048;
      CK(cudaMemcpy(doff, dof.data(), nseg * 8, cudaMemcpyHostToDevice));
      for (int ctas : {1, 2, 4}) {
        for (int threads : {512, 1024}) {
          std::vector<float> ms;
          for (int rep = 0; rep < 4; ++rep) {
            CK(cudaEventRecord(a));
            seg_copy<4><<<ctas, threads>>>(hd, d, soff, doff, nseg);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float t;
            CK(cudaEventElapsedTime(&t, a, b));
            if (rep) ms.push_back(t);
          }
          std::sort(ms.begin(), ms.end());
          printf("{\"kind\":\"pattern\",\"src\":\"%s\",\"dst\":\"%s\",\"ctas\":%d,\"threads\":%d,\"gbs\":%.2f}\n", sp.name,
                 dr ? "rand" : "seq", ctas, threads, total / ms[ms.size() / 2] / 1e6);
          fflush(stdout);
        }
      }
    }
  }
  return 0;
}
