// Write-path probe for K5's epilogue (experiment, not product code): how fast can 148 persistent CTAs write an
// n × n fp32 matrix tile by tile (256 × 256 tiles, upper triangle in a grouped raster) with
//   mode 0: plain grid-stride st.global.v4 over the whole buffer (reference fill)
//   mode 1: per warp 32 × 32 TMA stores (SWIZZLE_128B), 8 warps × 4 chunks per tile half — K5's pattern
//   mode 2: as 1 but each warp's 4 chunks go out as ONE 3-D TMA store {32 cols, 32 rows, 4 col blocks}
//   mode 3: st.global.v4 from registers, lanes across columns (coalesced 512-B row segments), no smem
//   mode 4: TMA stores of 32 × 32 boxes but the tile rows are written by consecutive warps (row-major within tile)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_probe store_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void fill_kernel(float4* p, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}

struct TileList { int ntiles; const int2* tiles; };

// 256 threads = 8 warps; warp w: rows 32*(w&3) of the tile's row half (w>>2 selects the second 128 rows?)
// We mimic K5: a "CTA" covers a 128 × 256 half tile (rank r of the pair); warp (q, h): rows 32q, cols 128h.
__global__ void __launch_bounds__(256) tma_kernel(const __grid_constant__ CUtensorMap tm2,
                                                  const __grid_constant__ CUtensorMap tm3, TileList tl, int mode,
                                                  float* out, long long ld) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, h = warp >> 2;
  uint8_t* buf = smem + warp * 16384;
  int cur = 0;
  for (int t = blockIdx.x; t < tl.ntiles * 2; t += gridDim.x) {
    const int2 tile = tl.tiles[t >> 1];
    const int half = t & 1;                       // which 128-row half of the 256 × 256 tile
    const long long row0 = (long long)tile.x * 256 + half * 128 + q * 32;
    const long long col0 = (long long)tile.y * 256 + h * 128;
    if (mode == 3) {
      for (int r = 0; r < 32; ++r) {
        float4* dst = reinterpret_cast<float4*>(out + (row0 + r) * ld + col0);
        dst[lane] = make_float4(r, lane, 1.f, 2.f);                   // 32 lanes × 16 B = one 512-B row segment
      }
      continue;
    }
    if (mode == 2) {
      uint8_t* b = buf;                                  // one 16-KB buffer per warp
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
      for (int cc = 0; cc < 4; ++cc)
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<float4*>(b + cc * 4096 + lane * 128 + ((c ^ (lane & 7)) << 4)) = make_float4(1, 2, 3, 4);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(&tm3),
                     "r"(smem_u32(b)), "r"(0), "r"((int)row0), "r"((int)(col0 / 32)) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      cur ^= 1;
      continue;
    }
    for (int cc = 0; cc < 4; ++cc) {
      const int wmode = mode >= 10 ? mode - 5 : mode;   // 10..14: same work as 5..9 but no proxy fence
      if (wmode >= 5) {   // fake EQ1-like work per chunk
        float v[32];
        for (int e = 0; e < 32; ++e) v[e] = (float)(e + lane) * 1e-3f;
        for (int it = 0; it < (wmode - 4) * 2; ++it)
          for (int e = 0; e < 32; ++e) v[e] = fmaf(v[e], 0.999f, 1e-4f);
        float acc = 0.f;
        for (int e = 0; e < 32; ++e) acc += v[e];
        if (acc == 123.456f) out[0] = acc;
      }
      uint8_t* b = buf + cur * 4096;
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<float4*>(b + lane * 128 + ((c ^ (lane & 7)) << 4)) = make_float4(1, 2, 3, 4);
      if (mode < 10) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        int c0 = (int)(col0 + cc * 32), r0 = (int)row0;
        if (mode == 4) { c0 = (int)(tile.y * 256 + (warp * 32 + cc * 256) % 256); r0 = (int)(tile.x * 256 + half * 128 + cc * 32); }
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(&tm2),
                     "r"(smem_u32(b)), "r"(c0), "r"(r0) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      cur ^= 1;
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef CUresult (*PFN_enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : 65536;
  const int gm = argc > 2 ? atoi(argv[2]) : 16;
  float* out;
  CK(cudaMalloc(&out, (size_t)n * n * 4));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
  PFN_enc enc = (PFN_enc)fn;
  CUtensorMap tm2, tm3;
  {
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
    cuuint64_t str[1] = {(cuuint64_t)n * 4};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    if (enc(&tm2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) { printf("enc2\n"); return 1; }
    // 3-D view {32 cols, n rows, n/32 col blocks}: strides row = n·4, col block = 128 B
    cuuint64_t d3[3] = {32, (cuuint64_t)n, (cuuint64_t)n / 32};
    cuuint64_t s3[2] = {(cuuint64_t)n * 4, 128};
    cuuint32_t b3[3] = {32, 32, 4}, e3[3] = {1, 1, 1};
    CUresult r = enc(&tm3, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, out, d3, s3, b3, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("enc3 failed (%d): mode 2 skipped\n", (int)r);
  }
  // upper-triangle tile list in grouped raster (gm row tiles, column-major inside a group)
  const int T = (int)(n / 256);
  std::vector<int2> tiles;
  for (int I0 = 0; I0 < T; I0 += gm)
    for (int J = I0; J < T; ++J)
      for (int I = I0; I < I0 + gm && I < T; ++I)
        if (J >= I) tiles.push_back(make_int2(I, J));
  int2* dtiles;
  CK(cudaMalloc(&dtiles, tiles.size() * sizeof(int2)));
  CK(cudaMemcpy(dtiles, tiles.data(), tiles.size() * sizeof(int2), cudaMemcpyHostToDevice));
  TileList tl{(int)tiles.size(), dtiles};
  const double bytes_tri = (double)tiles.size() * 256 * 256 * 4;
  CK(cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode <= 14; ++mode) {
    if (mode == 6 || mode == 8 || mode == 11 || mode == 13 || mode == 2) continue;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) fill_kernel<<<148 * 8, 256>>>((float4*)out, (size_t)(bytes_tri / 16));
      else tma_kernel<<<148, 256, 8 * 16384>>>(tm2, tm3, tl, mode, out, n);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("n=%lld gm=%d mode %d: %.3f ms  %.0f GB/s\n", n, gm, mode, ms, bytes_tri / ms / 1e6);
    }
    CK(cudaGetLastError());
  }
  return 0;
}
