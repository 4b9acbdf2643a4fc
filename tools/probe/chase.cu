// chase.cu — device-memory latency probe (interference mechanism): one thread
// follows a random cyclic chain of 128-byte-spaced slots over a buffer larger than L2, so every step
// is one dependent HBM access; the mean step time is the loaded latency of device memory.  Run
// beside strata_load on another stream of the same process (tools/interference_latency.py) to see
// whether queued host reads lengthen device-memory latency for everyone.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fPIC -shared -o libchase.so chase.cu
#include <cuda_runtime.h>
#include <cstdint>

__global__ void chase_kernel(const uint32_t* next, uint32_t start, int64_t steps, uint64_t* out) {
  uint32_t i = start;
  const long long t0 = clock64();
  for (int64_t s = 0; s < steps; ++s) i = __ldcg(next + size_t(i) * 32);   // 128-byte slots, L1 bypass
  const long long t1 = clock64();
  out[0] = static_cast<uint64_t>(t1 - t0);
  out[1] = i;
}

// launches one chase on `stream`; out[0] = SM cycles for `steps` dependent loads
// smem_bytes > 0: the chase CTA requests that much dynamic shared memory, so it cannot share an SM
// with a ring CTA (which holds ~115 KiB) — separates a GPU-wide effect from SM co-location
extern "C" int chase_launch(const void* next, unsigned start, long long steps, void* out, void* stream,
                            int smem_bytes) {
  if (smem_bytes > 48 * 1024)
    cudaFuncSetAttribute(chase_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  chase_kernel<<<1, 1, smem_bytes, static_cast<cudaStream_t>(stream)>>>(static_cast<const uint32_t*>(next), start,
                                                                         steps, static_cast<uint64_t*>(out));
  return static_cast<int>(cudaGetLastError());
}
