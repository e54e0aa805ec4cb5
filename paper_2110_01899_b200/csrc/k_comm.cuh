// G5 exchange kernels (include/rf.h, "G5"): the owner-side sum of the peers' tiles and the device epoch flags that
// order the exchange without the host.
#pragma once
#include <stdint.h>

namespace rfk {

// recv[e] = Σ_{r < world} staging[r][e], in rank order (deterministic), 16-B vectors; staging is [source rank][recv4].
__global__ void __launch_bounds__(256) k_pack_reduce(const float4* __restrict__ staging, int64_t recv4, int world,
                                                     float4* __restrict__ recv) {
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < recv4; e += (int64_t)gridDim.x * 256) {
    float4 s = staging[e];
    for (int r = 1; r < world; ++r) {
      const float4 v = staging[(int64_t)r * recv4 + e];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    recv[e] = s;
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
