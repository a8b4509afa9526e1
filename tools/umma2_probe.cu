// 2-CTA (cta_group::2) tcgen05.mma throughput probe: a cluster of 2 CTAs,
// the even CTA issues M=256 bf16 MMAs (each CTA supplies 128 rows of A and
// N/2 rows of B from its own shared memory), N in {32, 64, 128}; cycles per
// MMA measured on the leader.  Also a correctness check of D against a CPU
// reference for one K-step.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e_), __LINE__); return 1;} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ uint32_t idesc_bf16(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r;
}

// A: [128 rows][16 K] bf16 per CTA in core layout [row/8][kb(2)][row%8][8]
// B: [N/2 rows][16 K] per CTA, same layout.  D (TMEM): 128 lanes x N columns per CTA.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
mma2(int n, int iters, const uint16_t* Ag, const uint16_t* Bg, float* Dout, long long* cyc) {
  __shared__ __align__(1024) uint16_t sa[128 * 16];
  __shared__ __align__(1024) uint16_t sb[128 * 16];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t rank = cluster_rank();
  const int tid = threadIdx.x, warp = tid >> 5;
  const int cta = blockIdx.x;
  for (int i = tid; i < 128 * 16; i += 128) sa[i] = Ag[(cta & 1) * 128 * 16 + i];
  for (int i = tid; i < (n / 2) * 16; i += 128) sb[i] = Bg[(cta & 1) * (n / 2) * 16 + i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  long long t0 = clock64();
  if (rank == 0 && warp == 0) {
    uint32_t e;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
    if (e) {
      const uint64_t da = sdesc(smem_u32(sa), 128, 256), db = sdesc(smem_u32(sb), 128, 256);
      const uint32_t id = idesc_bf16(256, n);
      for (int i = 0; i < iters; ++i)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(da), "l"(db), "r"(id), "r"(i > 0 ? 1 : 0));
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
    }
    __syncwarp();
  }
  // both CTAs wait for the multicast completion
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
  long long t1 = clock64();
  if (rank == 0 && tid == 0 && blockIdx.x == 0) *cyc = t1 - t0;
  asm volatile("tcgen05.fence::after_thread_sync;");
  // D: this CTA's 128 lanes x n columns (first 32 columns checked)
  uint32_t r[32];
  const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                 "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                 "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  if (blockIdx.x < 2)
    for (int c = 0; c < 32; ++c) Dout[((cta & 1) * 128 + tid) * 32 + c] = __uint_as_float(r[c]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

static uint16_t bf(float x) { __nv_bfloat16 b = __float2bfloat16_rn(x); uint16_t u; memcpy(&u, &b, 2); return u; }
static float fb(uint16_t u) { uint32_t v = (uint32_t)u << 16; float f; memcpy(&f, &v, 4); return f; }

int main() {
  // logical A [256 x 16], B [N x 16]; per-CTA core layouts
  for (int n : {32, 64, 128}) {
    std::vector<float> A(256 * 16), Bm(n * 16);
    for (int i = 0; i < 256 * 16; ++i) A[i] = fb(bf(((i * 37) % 17) / 8.0f - 1.0f));
    for (int i = 0; i < n * 16; ++i) Bm[i] = fb(bf(((i * 11) % 13) / 6.0f - 1.0f));
    std::vector<uint16_t> Ah(256 * 16), Bh(n * 16);
    for (int c = 0; c < 2; ++c)
      for (int r = 0; r < 128; ++r)
        for (int k = 0; k < 16; ++k)
          Ah[c * 128 * 16 + ((r / 8) * 2 + k / 8) * 64 + (r % 8) * 8 + k % 8] = bf(A[(c * 128 + r) * 16 + k]);
    for (int c = 0; c < 2; ++c)
      for (int r = 0; r < n / 2; ++r)
        for (int k = 0; k < 16; ++k)
          Bh[c * (n / 2) * 16 + ((r / 8) * 2 + k / 8) * 64 + (r % 8) * 8 + k % 8] = bf(Bm[(c * n / 2 + r) * 16 + k]);
    uint16_t *dA, *dB; float* dD; long long* dc;
    CK(cudaMalloc(&dA, Ah.size() * 2)); CK(cudaMalloc(&dB, Bh.size() * 2));
    CK(cudaMalloc(&dD, 256 * 32 * 4)); CK(cudaMalloc(&dc, 8));
    CK(cudaMemcpy(dA, Ah.data(), Ah.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, Bh.data(), Bh.size() * 2, cudaMemcpyHostToDevice));
    // correctness: 1 MMA
    mma2<<<2, 128>>>(n, 1, dA, dB, dD, dc);
    CK(cudaDeviceSynchronize());
    std::vector<float> D(256 * 32);
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    double err = 0;
    for (int m = 0; m < 256; ++m)
      for (int c = 0; c < 32 && c < n; ++c) {
        double ref = 0;
        for (int k = 0; k < 16; ++k) ref += (double)A[m * 16 + k] * Bm[c * 16 + k];
        err = fmax(err, fabs(ref - D[m * 32 + c]));
      }
    // throughput: 148 CTAs (74 clusters)
    const int iters = 8192;
    mma2<<<148, 128>>>(n, iters, dA, dB, dD, dc);
    CK(cudaDeviceSynchronize());
    long long c; CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
    printf("{\"probe\": \"umma2\", \"N\": %d, \"max_abs_err\": %.3e, \"cyc_per_mma\": %.2f}\n", n, err, (double)c / iters);
    cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
  }
  return 0;
}
