// G5 exchange kernels (include/rf.h, "G5"): the owner-side sum of the peers' tiles and the device epoch flags that
// order the exchange without the host.
#pragma once
#include <stdint.h>

namespace rfk {

// recv[e] = Σ_{r < world} staging[r][e], in rank order (deterministic), 16-B vectors, for e in [off4, off4 + cnt4);
// staging is [source rank][stride4].  One launch per G5 chunk: launched on the context's reduce stream as soon as
// every source's tiles of the chunk have landed, it runs beside K4 (no shared memory, few registers: it fits next to
// a K4 CTA on the same SM: 1 KB of reserved shared memory and 128 × ≤ 96 registers fit beside the packed K4's 225.5 KB
// and 12 warps × 136 registers) while K4 computes the later chunks — with one CTA per SM it must keep many loads in
// flight, so each thread sums kV vectors per iteration, source by source (kV loads in flight per source step).
constexpr int kReduceV = 8, kReduceThreads = 128;
__global__ void __launch_bounds__(kReduceThreads) k_pack_reduce(const float4* __restrict__ staging, int64_t stride4, int64_t off4,
                                                     int64_t cnt4, int world, float4* __restrict__ recv) {
  const int64_t step = (int64_t)gridDim.x * kReduceThreads;
  const int64_t end = off4 + cnt4;
  for (int64_t e0 = off4 + (int64_t)blockIdx.x * kReduceThreads + threadIdx.x; e0 < end; e0 += step * kReduceV) {
    float4 s[kReduceV];
#pragma unroll
    for (int j = 0; j < kReduceV; ++j) {
      const int64_t e = e0 + j * step;
      s[j] = e < end ? staging[e] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int r = 1; r < world; ++r) {
      float4 v[kReduceV];
#pragma unroll
      for (int j = 0; j < kReduceV; ++j) {
        const int64_t e = e0 + j * step;
        v[j] = e < end ? staging[(int64_t)r * stride4 + e] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < kReduceV; ++j) {
        s[j].x += v[j].x; s[j].y += v[j].y; s[j].z += v[j].z; s[j].w += v[j].w;
      }
    }
#pragma unroll
    for (int j = 0; j < kReduceV; ++j) {
      const int64_t e = e0 + j * step;
      if (e < end) recv[e] = s[j];
    }
  }
}

struct SignalArgs {
  uint32_t* dst[16];
  int count;
  uint32_t value;
};
// One thread: a system-scope fence (everything this stream wrote before — the K4 stores into the peers' staging
// buffers, or the owner-side sum — is ordered before the flags) and one release store per destination flag, which may
// live in another GPU's memory (peer-mapped through CUDA IPC).  The reader waits with a stream-memory wait.
__global__ void k_signal(SignalArgs a) {
  asm volatile("fence.sc.sys;" ::: "memory");
  for (int i = 0; i < a.count; ++i)
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.dst[i]), "r"(a.value) : "memory");
}

}  // namespace rfk
