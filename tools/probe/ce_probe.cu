// Copy-engine probe: how fast can DMA move chunk-sized host runs (SURVEY.md §8f hybrid variant)?
// H2D copies of S bytes each from random positions of a pinned host buffer into a contiguous device
// staging buffer, submitted as a cudaMemcpyAsync loop, over 1..4 streams (round 1 also timed a batched
// submission; that API is closed on the GPU pool after Xid 32 faults).
// One JSON object per line.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ce_probe ce_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

int main() {
  const size_t host_bytes = size_t(4) << 30, total = size_t(1) << 30;
  char* h;
  CK(cudaHostAlloc(&h, host_bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(h, 1, host_bytes);
  char* d;
  CK(cudaMalloc(&d, total));
  std::vector<cudaStream_t> ss(4);
  for (auto& s : ss) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<cudaEvent_t> done(4);
  for (auto& e : done) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  std::mt19937_64 rng(1);
  for (size_t S : {size_t(32) << 10, size_t(128) << 10, size_t(256) << 10, size_t(1) << 20, size_t(4) << 20}) {
    const size_t n = total / S;
    std::vector<size_t> slot(host_bytes / S);
    std::iota(slot.begin(), slot.end(), 0);
    std::shuffle(slot.begin(), slot.end(), rng);
    std::vector<void*> dsts(n), srcs(n);
    std::vector<size_t> sizes(n, S);
    for (size_t i = 0; i < n; ++i) {
      dsts[i] = d + i * S;
      srcs[i] = h + slot[i] * S;
    }
    for (int mode = 0; mode < 1; ++mode) {
      for (int nstreams : {1, 2, 4}) {
        std::vector<float> ms;
        std::vector<double> wall;
        for (int rep = 0; rep < 6; ++rep) {
          CK(cudaDeviceSynchronize());
          auto w0 = std::chrono::steady_clock::now();
          CK(cudaEventRecord(e0, ss[0]));
          for (int k = 1; k < nstreams; ++k) CK(cudaStreamWaitEvent(ss[k], e0));
          const size_t per = (n + nstreams - 1) / nstreams;
          for (int k = 0; k < nstreams; ++k) {
            const size_t lo = k * per, hi = std::min(n, lo + per);
            if (lo >= hi) continue;
            for (size_t i = lo; i < hi; ++i) CK(cudaMemcpyAsync(dsts[i], srcs[i], S, cudaMemcpyHostToDevice, ss[k]));
            if (k) {
              CK(cudaEventRecord(done[k], ss[k]));
              CK(cudaStreamWaitEvent(ss[0], done[k]));
            }
          }
          CK(cudaEventRecord(e1, ss[0]));
          CK(cudaEventSynchronize(e1));
          auto w1 = std::chrono::steady_clock::now();
          float t;
          CK(cudaEventElapsedTime(&t, e0, e1));
          if (rep >= 1) {
            ms.push_back(t);
            wall.push_back(std::chrono::duration<double, std::milli>(w1 - w0).count());
          }
        }
        std::sort(ms.begin(), ms.end());
        std::sort(wall.begin(), wall.end());
        const float m = ms[ms.size() / 2];
        printf("{\"kind\":\"ce\",\"mode\":\"%s\",\"copy_bytes\":%zu,\"copies\":%zu,\"streams\":%d,\"ms\":%.3f,"
               "\"wall_ms\":%.3f,\"gbs\":%.2f}\n", "loop", S, n, nstreams, m, wall[wall.size() / 2],
               total / m / 1e6);
        fflush(stdout);
      }
    }
  }
  return 0;
}
