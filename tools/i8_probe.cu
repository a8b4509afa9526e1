// tcgen05 kind::i8 probe (run under gpurun) for a conv layer with int8 limbs:
//  C1  TS MMA, A u8 in TMEM (tcgen05.st, 4 bytes per column, K = 32), B s8 in
//      shared memory (canonical K-major no-swizzle core matrices, 8 rows x 16 B),
//      D s32: exact against the CPU
//  C2  the same with B [N = 64] (two column blocks) in one MMA
//  R   throughput on 148 CTAs of TS i8 MMAs (N = 32, 64; K = 32) against TS bf16
//      (N = 32, 64; K = 16) -- cycles per MMA and MACs per clock per SM
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// D s32 (2 << 4), A u8 (0 << 7), B s8 (1 << 10)
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (128u >> 4 << 24);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (128u >> 4 << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a),
               "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a),
               "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit_wait(uint64_t* bar, uint32_t& phase) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar)) : "memory");
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                   smem_u32(bar)), "r"(phase) : "memory");
  phase ^= 1;
}
__device__ void setup(uint32_t* tmem_slot, uint64_t* bar, int cols) {
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
}
__device__ void teardown(uint32_t tmem, int cols) {
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if ((threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
}
// [rows][32] int8, K-major no-swizzle: core (r/8, k/16) at ((r/8)*2 + k/16)*128 B
__host__ __device__ inline int core_off8(int r, int k) {
  return ((r >> 3) * 2 + (k >> 4)) * 128 + (r & 7) * 16 + (k & 15);
}

template <int N>
__global__ void i8_correct(const uint8_t* A, const int8_t* B, int32_t* D) {
  __shared__ __align__(1024) int8_t sb[N * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < N * 32; e += blockDim.x) sb[core_off8(e / 32, e % 32)] = B[e];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  setup(&tslot, &bar, 128);
  const uint32_t tmem = tslot;
  const uint32_t acol = 64;
  uint32_t w[8];
  for (int j = 0; j < 8; ++j)
    w[j] = (uint32_t)A[tid * 32 + 4 * j] | ((uint32_t)A[tid * 32 + 4 * j + 1] << 8) |
           ((uint32_t)A[tid * 32 + 4 * j + 2] << 16) | ((uint32_t)A[tid * 32 + 4 * j + 3] << 24);
  const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + acol;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta),
               "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    uint32_t phase = 0;
    mma_i8(tmem, tmem + acol, sdesc(smem_u32(sb), 128, 256), idesc_i8(N), 0);
    // accumulate a second time: D = 2 A B
    mma_i8(tmem, tmem + acol, sdesc(smem_u32(sb), 128, 256), idesc_i8(N), 1);
    commit_wait(&bar, phase);
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                   "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                   "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int n = 0; n < 32; ++n) D[tid * N + c0 + n] = (int32_t)r[n];
  }
  teardown(tmem, 128);
}

// WHAT 0: i8 K32, 1: bf16 K16 (A columns: i8 8, bf16 8 per MMA)
template <int N, int WHAT>
__global__ void tput(int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 16 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  setup(&tslot, &bar, 512);
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    uint32_t phase = 0;
    const uint64_t db = sdesc(smem_u32(sm), 128, 256);
    const uint32_t id = WHAT == 0 ? idesc_i8(N) : idesc_bf16(N);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 16) {
      uint32_t e;
      asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
      if (e) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const uint32_t acol = 256 + (u & 7) * 8;
          const uint32_t d = tmem + ((u >> 1) & 1) * 128;
          if (WHAT == 0) mma_i8(d, tmem + acol, db, id, 1);
          else mma_f16(d, tmem + acol, db, id, 1);
        }
        if (((i / 16) & 7) == 7) commit_wait(&bar, phase);
      }
      __syncwarp();
    }
    uint32_t e;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
    if (e) commit_wait(&bar, phase);
    __syncwarp();
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = t1 - t0;
  }
  teardown(tmem, 512);
}

template <int N, int WHAT>
static void run_tput(const char* name) {
  long long* cyc;
  CK(cudaMalloc(&cyc, 8));
  CK(cudaFuncSetAttribute(tput<N, WHAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 1024));
  const int iters = 16384;
  tput<N, WHAT><<<148, 128, 16 * 1024>>>(iters, cyc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  tput<N, WHAT><<<148, 128, 16 * 1024>>>(iters, cyc);
  cudaEventRecord(b);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const int K = WHAT == 0 ? 32 : 16;
  const double ops = 2.0 * 128 * N * K * (double)iters * 148;
  printf("{\"probe\": \"%s\", \"N\": %d, \"K\": %d, \"cyc_per_mma\": %.2f, \"macs_per_clk_sm\": %.0f, \"tops\": %.1f}\n",
         name, N, K, (double)c / iters, 128.0 * N * K / ((double)c / iters), ops / (ms * 1e-3) / 1e12);
  cudaFree(cyc);
}

template <int N>
static void run_correct() {
  std::vector<uint8_t> hA(128 * 32);
  std::vector<int8_t> hB(N * 32);
  std::vector<int32_t> hD(128 * N);
  for (int i = 0; i < 128 * 32; ++i) hA[i] = (uint8_t)((i * 37 + 11) % 256);
  for (int i = 0; i < N * 32; ++i) hB[i] = (int8_t)((i * 53 + 7) % 256 - 128);
  uint8_t* A; int8_t* B; int32_t* D;
  CK(cudaMalloc(&A, hA.size())); CK(cudaMalloc(&B, hB.size())); CK(cudaMalloc(&D, hD.size() * 4));
  CK(cudaMemcpy(A, hA.data(), hA.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(B, hB.data(), hB.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(D, 0, hD.size() * 4));
  i8_correct<N><<<1, 128>>>(A, B, D);
  cudaError_t e = cudaDeviceSynchronize();
  CK(cudaMemcpy(hD.data(), D, hD.size() * 4, cudaMemcpyDeviceToHost));
  long long bad = 0, first = -1;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      long long s = 0;
      for (int k = 0; k < 32; ++k) s += (long long)hA[m * 32 + k] * hB[n * 32 + k];
      if (hD[m * N + n] != 2 * s) { ++bad; if (first < 0) first = m * N + n; }
    }
  printf("{\"probe\": \"i8_ts_correct\", \"N\": %d, \"status\": \"%s\", \"mismatches\": %lld, \"first\": %lld}\n",
         N, cudaGetErrorString(e), bad, first);
}

int main() {
  run_correct<32>();
  run_correct<64>();
  run_tput<32, 0>("ts_i8");
  run_tput<64, 0>("ts_i8");
  run_tput<128, 0>("ts_i8");
  run_tput<32, 1>("ts_bf16");
  run_tput<64, 1>("ts_bf16");
  run_tput<128, 1>("ts_bf16");
  return 0;
}
