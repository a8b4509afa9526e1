// tcgen05 convention probe: D[128 x N] = A[128 x K] * B[N x K]^T in tf32 with
// fp32 accumulation in TMEM; A and B staged K-major, no swizzle, core
// matrices (8 rows x 16 B) laid out [row/8][k/4][row%8][k%4].  Prints max
// error vs a CPU reference for each (LBO, SBO) role assignment so the
// descriptor convention is established on hardware.
#include <cstdio>
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int M = 128, N = 32, K = 64, KC = 32;   // two K chunks

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;            // version (sm100)
  return d;                          // base offset 0, SWIZZLE_NONE
}
__device__ __forceinline__ uint32_t idesc_tf32(int m, int n) {
  uint32_t d = 0;
  d |= 1u << 4;                      // D = f32
  d |= 2u << 7;                      // A = tf32
  d |= 2u << 10;                     // B = tf32
  d |= (uint32_t)(n >> 3) << 17;
  d |= (uint32_t)(m >> 4) << 24;
  return d;
}

__global__ void probe(const float* A, const float* B, float* D, int swap) {
  __shared__ __align__(1024) float sa[M * KC];
  __shared__ __align__(1024) float sb[N * KC];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&tmem_base)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t core_k_stride = 128;              // bytes between core matrices along K
  const uint32_t core_m_stride = (KC / 4) * 128;   // bytes between core matrices along M/N
  const uint32_t lbo = swap ? core_m_stride : core_k_stride;
  const uint32_t sbo = swap ? core_k_stride : core_m_stride;
  for (int kc = 0; kc < K / KC; ++kc) {
    for (int e = tid; e < M * KC; e += blockDim.x) {
      int m = e / KC, k = e % KC;
      int off = ((m / 8) * (KC / 4) + k / 4) * 32 + (m % 8) * 4 + k % 4;   // floats
      sa[off] = A[m * K + kc * KC + k];
    }
    for (int e = tid; e < N * KC; e += blockDim.x) {
      int n = e / KC, k = e % KC;
      int off = ((n / 8) * (KC / 4) + k / 4) * 32 + (n % 8) * 4 + k % 4;
      sb[off] = B[n * K + kc * KC + k];
    }
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int ks = 0; ks < KC / 8; ++ks) {      // K = 8 per tf32 MMA = 2 core matrices
        uint64_t da = sdesc(sa + ks * 2 * 32, lbo, sbo);
        uint64_t db = sdesc(sb + ks * 2 * 32, lbo, sbo);
        uint32_t acc = (kc | ks) ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     :: "r"(tmem), "l"(da), "l"(db), "r"(idesc_tf32(M, N)), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   :: "r"(smem_u32(&bar)) : "memory");
    }
    // wait for this chunk's MMAs before overwriting smem
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}"
                 :: "r"(smem_u32(&bar)), "r"(kc & 1) : "memory");
    __syncthreads();
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // each warp reads its 32-lane quarter: 32 columns
  uint32_t r[32];
  const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                 "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                 "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  const int m = warp * 32 + lane;
  for (int n = 0; n < N; ++n) D[m * N + n] = __uint_as_float(r[n]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(32));
}

int main() {
  static float hA[M * K], hB[N * K], hD[M * N], ref[M * N];
  for (int i = 0; i < M * K; ++i) hA[i] = ((i * 37) % 101) / 50.0f - 1.0f;
  for (int i = 0; i < N * K; ++i) hB[i] = ((i * 53) % 97) / 48.0f - 1.0f;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)hA[m * K + k] * hB[n * K + k];
      ref[m * N + n] = (float)s;
    }
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  for (int swap = 0; swap < 2; ++swap) {
    cudaMemset(D, 0, sizeof hD);
    probe<<<1, 128>>>(A, B, D, swap);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
    double worst = 0;
    for (int i = 0; i < M * N; ++i) worst = fmax(worst, fabs(hD[i] - ref[i]) / fmax(1.0, fabs(ref[i])));
    printf("{\"swap\": %d, \"status\": \"%s\", \"max_rel_err\": %.3e, \"D00\": %f, \"ref00\": %f}\n",
           swap, cudaGetErrorString(e), worst, hD[0], ref[0]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
