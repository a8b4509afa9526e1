// tcgen05 probe for a conv design with the A operand in tensor memory
// ("TS" MMAs, A from TMEM, B from shared memory), run under gpurun:
//  T1  A written to TMEM with tcgen05.st, D = A*B^T by a TS MMA: correctness
//  T2  A copied smem -> TMEM with tcgen05.cp.128x256b (canonical K-major
//      no-swizzle source), D by a TS MMA: correctness (cp -> mma ordering)
//  T3  TS MMA throughput, M=128, N in {32, 64, 128}, bf16, on 148 CTAs
//  T4  SS MMA throughput for the same shapes (the round-1 design)
//  T5  tcgen05.cp.128x256b throughput alone, and cp + TS MMA interleaved
//      (one cp of a fresh A tile per MMA / per 3 MMAs)
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ uint32_t idesc_bf16(int m, int n) {
  uint32_t d = 1u << 4;      // D f32
  d |= 1u << 7;              // A bf16
  d |= 1u << 10;             // B bf16
  d |= (uint32_t)(n >> 3) << 17;
  d |= (uint32_t)(m >> 4) << 24;
  return d;
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a),
               "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a),
               "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void cp128x256(uint32_t taddr, uint64_t sd) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sd));
}
__device__ __forceinline__ void commit_wait(uint64_t* bar, uint32_t& phase) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar)) : "memory");
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                   smem_u32(bar)), "r"(phase) : "memory");
  phase ^= 1;
}
__device__ void setup(uint32_t* tmem_slot, uint64_t* bar, int cols) {
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
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
// canonical K-major no-swizzle core-matrix layout of a [rows][16] bf16 tile:
// core matrix (r/8, k/8) at ((r/8)*2 + k/8)*128 B, row r%8 at 16 B, k%8 at 2 B
// -> LBO (K-adjacent core matrices) = 128 B, SBO (8-row groups) = 256 B
__device__ __forceinline__ int core_off(int r, int k) {   // in bf16 elements
  return ((r >> 3) * 2 + (k >> 3)) * 64 + (r & 7) * 8 + (k & 7);
}

// ------------------------------------------------------------ T1 / T2
// mode 0: A via tcgen05.st; mode 1: A via tcgen05.cp
__global__ void ts_correct(const float* A, const float* B, float* D, int mode) {
  __shared__ __align__(1024) __nv_bfloat16 sa[128 * 16];
  __shared__ __align__(1024) __nv_bfloat16 sb[64 * 16];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 128 * 16; e += blockDim.x)
    sa[core_off(e / 16, e % 16)] = __float2bfloat16_rn(A[e]);
  for (int e = tid; e < 32 * 16; e += blockDim.x)
    sb[core_off(e / 16, e % 16)] = __float2bfloat16_rn(B[e]);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  setup(&tslot, &bar, 64);
  const uint32_t tmem = tslot;
  const uint32_t acol = 32;                      // A at columns 32..39, D at 0..31
  if (mode == 0) {
    // lane m = row m: 8 words, word j = (A[m][2j] lo half, A[m][2j+1] hi half)
    uint32_t w[8];
    for (int j = 0; j < 8; ++j) {
      __nv_bfloat162 p = __floats2bfloat162_rn(A[tid * 16 + 2 * j], A[tid * 16 + 2 * j + 1]);
      w[j] = *reinterpret_cast<uint32_t*>(&p);
    }
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + acol;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta),
                 "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]),
                 "r"(w[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    uint32_t phase = 0;
    if (mode == 1) cp128x256(tmem + acol, sdesc(smem_u32(sa), 128, 256));
    mma_ts(tmem, tmem + acol, sdesc(smem_u32(sb), 128, 256), idesc_bf16(128, 32), 0);
    commit_wait(&bar, phase);
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[32];
  const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                 "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                 "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int n = 0; n < 32; ++n) D[tid * 32 + n] = __uint_as_float(r[n]);
  teardown(tmem, 64);
}

// ------------------------------------------------------------ T3 / T4 / T5
// what: 0 = TS mma, 1 = SS mma, 2 = cp only, 3 = cp + TS mma per step,
//       4 = one cp per 3 TS mmas
// T6: issue cost of the pipeline bookkeeping in one thread: tcgen05.commit
// (nothing pending / after one MMA), mbarrier try_wait on a completed phase,
// tcgen05.fence::after_thread_sync, mbarrier arrive
__global__ void overhead(long long* out) {
  __shared__ __align__(1024) uint8_t sm[8192];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tslot;
  setup(&tslot, &bar[0], 128);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(smem_u32(&bar[2])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const int n = 1000;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[2])) : "memory");
    long long t1 = clock64();
    const uint64_t db = sdesc(smem_u32(sm), 128, 256);
    for (int i = 0; i < n; ++i) {
      mma_ts(tmem, tmem + 64, db, idesc_bf16(128, 32), 1);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[2])) : "memory");
    }
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) mma_ts(tmem, tmem + 64, db, idesc_bf16(128, 32), 1);
    long long t3 = clock64();
    // completed phase: wait for parity 1 of a fresh barrier
    for (int i = 0; i < n; ++i)
      asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 1;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(&bar[1])) : "memory");
    long long t4 = clock64();
    for (int i = 0; i < n; ++i) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    long long t5 = clock64();
    for (int i = 0; i < n; ++i)
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar[2])) : "memory");
    long long t6 = clock64();
    out[0] = (t1 - t0) / n; out[1] = (t2 - t1) / n; out[2] = (t3 - t2) / n;
    out[3] = (t4 - t3) / n; out[4] = (t5 - t4) / n; out[5] = (t6 - t5) / n;
    uint32_t ph = 0;
    commit_wait(&bar[0], ph);
  }
  teardown(tmem, 128);
}

template <int N, int WHAT>
__global__ void tput(int iters, long long* cyc) {
  constexpr int what = WHAT;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  setup(&tslot, &bar, 512);
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    uint32_t phase = 0;
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 65536);
    const uint32_t id = idesc_bf16(128, N);
    const uint64_t db = sdesc(b, 128, 256);
    uint64_t das[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) das[u] = sdesc(a + u * 4096, 128, 256);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 16) {
      uint32_t e;
      asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
      if (e) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const uint32_t acol = 256 + (u & 7) * 8;            // 8 A tiles at columns 256..319
          const uint64_t da = das[u & 7];
          if (what == 0) mma_ts(tmem, tmem + acol, db, id, 1);
          if (what == 1) mma_ss(tmem, da, db, id, 1);
          if (what == 2) cp128x256(tmem + acol, da);
          if (what == 3) { cp128x256(tmem + acol, da); mma_ts(tmem, tmem + acol, db, id, 1); }
          if (what == 4) { if (u % 3 == 0) cp128x256(tmem + acol, da); mma_ts(tmem, tmem + acol, db, id, 1); }
          // conv pattern: pairs (N=64 then N=32) into D slot (u/2) % 5 of 64 columns
          if (what == 5) {
            const uint32_t d = tmem + ((u / 2) % 5) * 64;
            if (u & 1) mma_ts(d, tmem + 384 + 8, db, idesc_bf16(128, 32), 1);
            else mma_ts(d, tmem + 384, db, idesc_bf16(128, 64), 1);
          }
          // same pairs, one D
          if (what == 6) {
            if (u & 1) mma_ts(tmem, tmem + 384 + 8, db, idesc_bf16(128, 32), 1);
            else mma_ts(tmem, tmem + 384, db, idesc_bf16(128, 64), 1);
          }
          // four MMAs per D before switching
          if (what == 7) {
            const uint32_t d = tmem + ((u / 4) % 5) * 64;
            if (u & 1) mma_ts(d, tmem + 384 + 8, db, idesc_bf16(128, 32), 1);
            else mma_ts(d, tmem + 384, db, idesc_bf16(128, 64), 1);
          }
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

template <int N, int what>
static void run_tput(const char* name) {
  long long* cyc;
  CK(cudaMalloc(&cyc, 8));
  CK(cudaFuncSetAttribute(tput<N, what>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
  const int iters = 16384;
  tput<N, what><<<148, 128, 96 * 1024>>>(iters, cyc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  tput<N, what><<<148, 128, 96 * 1024>>>(iters, cyc);
  cudaEventRecord(b);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double mmas = (what == 2) ? 0 : iters;
  const double flops = 2.0 * 128 * N * 16 * mmas * 148;
  printf("{\"probe\": \"%s\", \"N\": %d, \"cyc_per_step\": %.2f, \"mma_tflops\": %.1f}\n", name, N,
         (double)c / iters, flops / (ms * 1e-3) / 1e12);
  cudaFree(cyc);
}

static void run_correct(int mode) {
  std::vector<float> hA(128 * 16), hB(32 * 16), hD(128 * 32);
  for (int i = 0; i < 128 * 16; ++i) hA[i] = ((i * 37) % 101) / 64.0f - 0.75f;
  for (int i = 0; i < 32 * 16; ++i) hB[i] = ((i * 53) % 97) / 64.0f - 0.7f;
  auto bf = [](float x) { return __bfloat162float(__float2bfloat16_rn(x)); };
  float *A, *B, *D;
  CK(cudaMalloc(&A, hA.size() * 4)); CK(cudaMalloc(&B, hB.size() * 4)); CK(cudaMalloc(&D, hD.size() * 4));
  CK(cudaMemcpy(A, hA.data(), hA.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(B, hB.data(), hB.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(D, 0, hD.size() * 4));
  ts_correct<<<1, 128>>>(A, B, D, mode);
  cudaError_t e = cudaDeviceSynchronize();
  CK(cudaMemcpy(hD.data(), D, hD.size() * 4, cudaMemcpyDeviceToHost));
  double worst = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n) {
      double s = 0;
      for (int k = 0; k < 16; ++k) s += (double)bf(hA[m * 16 + k]) * bf(hB[n * 16 + k]);
      worst = fmax(worst, fabs(hD[m * 32 + n] - s));
    }
  printf("{\"probe\": \"%s\", \"status\": \"%s\", \"max_abs_err\": %.3e}\n",
         mode == 0 ? "ts_st_correct" : "ts_cp_correct", cudaGetErrorString(e), worst);
}

static void run_overhead() {
  long long* d;
  CK(cudaMalloc(&d, 64));
  overhead<<<1, 128>>>(d);
  CK(cudaDeviceSynchronize());
  long long h[6];
  CK(cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost));
  printf("{\"probe\": \"overhead_cycles\", \"commit_idle\": %lld, \"mma_plus_commit\": %lld, "
         "\"mma_only\": %lld, \"try_wait_done\": %lld, \"fence_after\": %lld, \"arrive\": %lld}\n",
         h[0], h[1], h[2], h[3], h[4], h[5]);
}

int main() {
  run_overhead();
  run_tput<64, 5>("pairs_5_accumulators");
  run_tput<64, 6>("pairs_1_accumulator");
  run_tput<64, 7>("pairs_switch_every_4");
  run_correct(0);
  run_correct(1);
  run_tput<32, 0>("ts_mma");
  run_tput<64, 0>("ts_mma");
  run_tput<128, 0>("ts_mma");
  run_tput<32, 1>("ss_mma");
  run_tput<64, 1>("ss_mma");
  run_tput<128, 1>("ss_mma");
  run_tput<32, 2>("cp_only");
  run_tput<32, 3>("cp_plus_ts_mma");
  run_tput<32, 4>("cp_per_3_ts_mma");
  run_tput<64, 4>("cp_per_3_ts_mma");
  return 0;
}
