// Standalone check of the layer-1 raw-box TMA load (3D tensor map over NHWC
// frames, negative start coordinates -> zero fill).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap tmap, float* out, int x, int y, int z, int bx) {
  __shared__ __align__(128) float buf[20 * 128];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(20 * bx * 4) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(smem_u32(buf)), "l"(&tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
  for (int i = threadIdx.x; i < 20 * bx; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  const int bx = argc > 1 ? atoi(argv[1]) : 108;
  const int cx = argc > 2 ? atoi(argv[2]) : -18, cy = argc > 3 ? atoi(argv[3]) : -6;
  const int l2p = argc > 4 ? atoi(argv[4]) : 1;
  const int H = 96, W = 96, C = 3, F = 6;
  std::vector<float> h((size_t)F * H * W * C);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(i % 9973);
  float *d, *o;
  cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 20 * 108 * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)W * C, (cuuint64_t)H, (cuuint64_t)F};
  cuuint64_t str[2] = {(cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4};
  cuuint32_t box[3] = {(cuuint32_t)bx, 20, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)l2p, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("{\"encode\": %d, \"q\": %d}\n", (int)r, (int)q);
  const int cases[1][3] = {{cx, cy, 1}};
  for (auto& c : cases) {
    k<<<1, 128>>>(m, o, c[0], c[1], c[2], bx);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> g(20 * 108);
    cudaMemcpy(g.data(), o, g.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int yy = 0; yy < 20; ++yy)
      for (int xx = 0; xx < 108; ++xx) {
        int gx = c[0] + xx, gy = c[1] + yy;
        if (xx >= bx) continue;
        float want = (gx >= 0 && gx < W * C && gy >= 0 && gy < H) ? h[((size_t)c[2] * H + gy) * W * C + gx] : 0.f;
        bad += g[yy * bx + xx] != want;
      }
    printf("{\"bx\": %d, \"l2p\": %d, \"case\": [%d, %d, %d], \"status\": \"%s\", \"mismatches\": %d}\n", bx, l2p, c[0], c[1], c[2], cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
