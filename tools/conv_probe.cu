// tcgen05 probes for the conv redesign (run under gpurun):
//  1. SS-mode MMA throughput, M=128, N in {32,64,128,256}, kind::tf32 and
//     kind::f16 (bf16): cycles per instruction on 148 CTAs.
//  2. "Shifted-window" operand layouts: A rows are consecutive pixels of a
//     planar patch P[cb][pix][16 B] (LBO = plane stride, SBO = 128 B) and the
//     Toeplitz layout P[pix][16 B] (LBO = 16 B, SBO = 128 B), checked against
//     a CPU reference.
//  3. Whether kind::tf32 truncates or rounds the fp32 operand.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
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
// kind: 0 = tf32, 1 = bf16
__device__ __forceinline__ uint32_t idesc(int kind, int m, int n) {
  uint32_t d = 1u << 4;
  const uint32_t f = kind == 0 ? 2u : 1u;
  d |= f << 7;
  d |= f << 10;
  d |= (uint32_t)(n >> 3) << 17;
  d |= (uint32_t)(m >> 4) << 24;
  return d;
}
__device__ __forceinline__ void mma(int kind, uint32_t tmem, uint64_t a, uint64_t b, uint32_t id,
                                    uint32_t acc) {
  if (kind == 0)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
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

// ------------------------------------------------------------ 1. throughput
__global__ void tput(int kind, int n, int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  setup(&tslot, &bar, 256);
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    uint32_t phase = 0;
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    const uint32_t id = idesc(kind, 128, n);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t da = sdesc(a + (i & 3) * 32, 128, 1024);
      const uint64_t db = sdesc(b + (i & 3) * 32, 128, 1024);
      mma(kind, tmem, da, db, id, i ? 1u : 0u);
      if ((i & 63) == 63) commit_wait(&bar, phase);
    }
    commit_wait(&bar, phase);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cyc = t1 - t0;
  }
  teardown(tmem, 256);
}


// 1b. unrolled issue: descriptors hoisted, whole warp 0 converged, one elected lane
template <int KIND, int N, int UNROLL>
__global__ void tput2(int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  setup(&tslot, &bar, 256);
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    uint32_t phase = 0;
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    const uint32_t id = idesc(KIND, 128, N);
    uint64_t da[UNROLL], db[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) { da[u] = sdesc(a + (u & 3) * 32, 128, 1024); db[u] = sdesc(b + (u & 3) * 32, 128, 1024); }
    long long t0 = clock64();
    for (int i = 0; i < iters; i += UNROLL) {
      uint32_t e;
      asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
      if (e) {
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
          if (KIND == 0)
            asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(da[u]), "l"(db[u]), "r"(id));
          else
            asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(da[u]), "l"(db[u]), "r"(id));
        }
        if (((i / UNROLL) & 7) == 7) commit_wait(&bar, phase);
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
  teardown(tmem, 256);
}

template <int KIND, int N>
static void run_tput2() {
  long long* cyc;
  CK(cudaMalloc(&cyc, 8));
  CK(cudaFuncSetAttribute(tput2<KIND, N, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  const int iters = 16384;
  tput2<KIND, N, 16><<<148, 128, 64 * 1024>>>(iters, cyc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  tput2<KIND, N, 16><<<148, 128, 64 * 1024>>>(iters, cyc);
  cudaEventRecord(b);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double kk = KIND == 0 ? 8 : 16;
  const double flops = 2.0 * 128 * N * kk * iters * 148;
  printf("{\"probe\": \"tput2\", \"kind\": \"%s\", \"N\": %d, \"cyc_per_mma\": %.2f, \"tflops\": %.1f}\n",
         KIND == 0 ? "tf32" : "bf16", N, (double)c / iters, flops / (ms * 1e-3) / 1e12);
  cudaFree(cyc);
}


// 1c. A-operand layout cost: bf16, M=128, N given; A start offset / LBO / SBO
// varied (the conv patch uses unaligned starts, LBO = plane stride, SBO = row).
template <int N>
__global__ void tput3(int iters, uint32_t aoff, uint32_t lbo, uint32_t sbo, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  setup(&tslot, &bar, 256);
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    uint32_t phase = 0;
    const uint32_t a = smem_u32(sm) + aoff, b = smem_u32(sm + 128 * 1024);
    const uint32_t id = idesc(1, 128, N);
    const uint64_t da = sdesc(a, lbo, sbo), db = sdesc(b, 128, 256);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 16) {
      uint32_t e;
      asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
      if (e) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
          asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(tmem), "l"(da + (u & 3) * 8), "l"(db), "r"(id));
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
  teardown(tmem, 256);
}

template <int N>
static void run_tput3(const char* name, uint32_t aoff, uint32_t lbo, uint32_t sbo) {
  long long* cyc;
  CK(cudaMalloc(&cyc, 8));
  CK(cudaFuncSetAttribute(tput3<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  const int iters = 16384;
  tput3<N><<<148, 128, 160 * 1024>>>(iters, aoff, lbo, sbo, cyc);
  CK(cudaDeviceSynchronize());
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"probe\": \"layout\", \"case\": \"%s\", \"N\": %d, \"aoff\": %u, \"lbo\": %u, \"sbo\": %u, \"cyc_per_mma\": %.2f}\n",
         name, N, aoff, lbo, sbo, (double)c / iters);
  cudaFree(cyc);
}


// 1d. the layer-1 conv MMA stream: per super-tile 4 tiles x 5 K-steps x 3
// N=32 MMAs (xh*wh, xl*wh, xh*wl), A from the planar entry patch
// (LBO = plane stride 10240 B, SBO = 512 B), B 2 KB per step; one commit per
// super-tile, 3 accumulator sets in flight.  mode 1: every A at one address.
__global__ void tput4(int supertiles, int mode, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[3];
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    const uint32_t id = idesc(1, 128, 32);
    const uint32_t wbase = smem_u32(sm), pbase = smem_u32(sm + 16384);
    const uint64_t db0 = sdesc(wbase, 128, 256);
    uint32_t ph[3] = {0, 0, 0};
    long long t0 = clock64();
    for (int it = 0; it < supertiles; ++it) {
      const int b = it % 3;
      if (it >= 3) {   // accumulator set b was committed 3 super-tiles ago
        asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(&bar[b])), "r"(ph[b]) : "memory");
        ph[b] ^= 1;
      }
      const uint64_t da0 = sdesc(pbase + (b % 2) * 40960, 10240, 512);
      uint32_t e;
      asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(e));
      if (e) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const uint32_t d = tmem + (uint32_t)((b * 4 + t) * 32);
#pragma unroll
          for (int s = 0; s < 5; ++s) {
            const uint64_t dah = mode ? da0 : da0 + (uint64_t)((s * 512 + t * 128) >> 4);
            const uint64_t dal = mode ? da0 : dah + (uint64_t)((2 * 10240) >> 4);
            const uint64_t dbs = db0 + (uint64_t)(s * 128);
            asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, %4;" ::"r"(d), "l"(dah), "l"(dbs), "r"(id), "n"(0));
            asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(dal), "l"(dbs), "r"(id));
            asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(dah), "l"(dbs + 64), "r"(id));
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[b])) : "memory");
      }
      __syncwarp();
    }
    for (int b = 0; b < 3 && b < supertiles; ++b) {
      asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(&bar[b])), "r"(ph[b]) : "memory");
    }
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if ((threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ------------------------------------------------- 2. shifted-window layouts
// mode 0 (planar, tf32): P[cb][pix][4 f32], npix pixels, 8 planes (32 ch);
//   D[r][o] = sum_shift sum_ci P[ci][shift + r] * W[shift][o][ci]
//   A desc for (shift, kstep): start = plane 2*kstep, pixel shift; LBO = plane
//   stride, SBO = 128.
// mode 1 (Toeplitz, tf32): P[pix][4 f32]; K index k = 4*j + c reads pixel
//   shift + r + j channel c; LBO = 16, SBO = 128; 3 MMAs (K = 24) per shift.
// mode 2 (planar, bf16): P[cb][pix][8 bf16], 4 planes (32 ch), K=16 per MMA.
constexpr int kPix = 256 + 64;
constexpr int kShifts = 5;
__global__ void window(int mode, const float* P, const float* Wt, float* D) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int N = 32;
  // stage P as given (already in the device layout, fp32 or bf16 bits)
  const int pbytes = (mode == 1) ? kPix * 16 : (mode == 0 ? 8 * kPix * 16 : 4 * kPix * 16);
  for (int i = tid; i < pbytes / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = P[i];
  // W per shift: K-major core layout [n/8][kb][n%8][16 B], kb = K blocks
  const int kb = (mode == 1) ? 6 : (mode == 0 ? 8 : 4);
  const int wbytes = kShifts * N * kb * 16;
  uint8_t* sw = sm + ((pbytes + 1023) & ~1023);
  for (int i = tid; i < wbytes / 4; i += blockDim.x) reinterpret_cast<float*>(sw)[i] = Wt[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  setup(&tslot, &bar, 32);
  const uint32_t tmem = tslot;
  if (tid == 0) {
    uint32_t phase = 0;
    const int kind = mode == 2 ? 1 : 0;
    const uint32_t id = idesc(kind, 128, N);
    int q = 0;
    for (int s = 0; s < kShifts; ++s) {
      const int shift = s * 3;   // arbitrary pixel shifts
      for (int ks = 0; ks < kb / 2; ++ks) {
        uint64_t da;
        if (mode == 1) da = sdesc(smem_u32(sm) + (shift + 2 * ks) * 16, 16, 128);
        else da = sdesc(smem_u32(sm) + (2 * ks) * kPix * 16 + shift * 16, kPix * 16, 128);
        const uint64_t db = sdesc(smem_u32(sw) + s * N * kb * 16 + 2 * ks * 128, 128, kb * 128);
        mma(kind, tmem, da, db, id, q++ ? 1u : 0u);
      }
    }
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
  for (int o = 0; o < 32; ++o) D[tid * 32 + o] = __uint_as_float(r[o]);
  teardown(tmem, 32);
}

static float tf32_trunc(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  memcpy(&x, &u, 4);
  return x;
}
static uint16_t bf16_bits(float x) {
  __nv_bfloat16 b = __float2bfloat16_rn(x);
  uint16_t u;
  memcpy(&u, &b, 2);
  return u;
}
static float bf16_val(float x) {
  uint32_t u = (uint32_t)bf16_bits(x) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static void run_window(int mode) {
  const int N = 32;
  const int C = mode == 1 ? 4 : 32;            // channels per pixel (logical)
  const int kb = mode == 1 ? 6 : (mode == 0 ? 8 : 4);
  std::vector<float> x((size_t)kPix * C), w((size_t)kShifts * N * (mode == 1 ? 24 : 32));
  srand(7);
  for (auto& v : x) v = (float)rand() / RAND_MAX - 0.5f;
  for (auto& v : w) v = (float)rand() / RAND_MAX - 0.5f;
  const int K = mode == 1 ? 24 : 32;
  // device images
  std::vector<uint32_t> P, Wd((size_t)kShifts * N * kb * 4, 0);
  if (mode == 0) {
    P.assign(8 * kPix * 4, 0);
    for (int p = 0; p < kPix; ++p)
      for (int c = 0; c < 32; ++c) memcpy(&P[((c / 4) * kPix + p) * 4 + c % 4], &x[p * 32 + c], 4);
  } else if (mode == 1) {
    P.assign(kPix * 4, 0);
    for (int p = 0; p < kPix; ++p)
      for (int c = 0; c < 4; ++c) memcpy(&P[p * 4 + c], &x[p * 4 + c], 4);
  } else {
    P.assign(4 * kPix * 4, 0);
    uint16_t* ph = reinterpret_cast<uint16_t*>(P.data());
    for (int p = 0; p < kPix; ++p)
      for (int c = 0; c < 32; ++c) ph[((c / 8) * kPix + p) * 8 + c % 8] = bf16_bits(x[p * 32 + c]);
  }
  const int epb = mode == 2 ? 8 : 4;   // elements per 16 B
  for (int s = 0; s < kShifts; ++s)
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) {
        const float v = w[((size_t)s * N + n) * K + k];
        const size_t off = (size_t)s * N * kb * 16 + ((n / 8) * kb + k / epb) * 128 + (n % 8) * 16;
        if (mode == 2) {
          reinterpret_cast<uint16_t*>(Wd.data())[(off + (k % epb) * 2) / 2] = bf16_bits(v);
        } else {
          memcpy(reinterpret_cast<uint8_t*>(Wd.data()) + off + (k % epb) * 4, &v, 4);
        }
      }
  // CPU reference with the operand rounding the hardware applies
  double worst = 0;
  std::vector<float> ref(128 * N);
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < N; ++n) {
      double acc = 0;
      for (int s = 0; s < kShifts; ++s) {
        const int shift = s * 3;
        for (int k = 0; k < K; ++k) {
          float a;
          if (mode == 1) a = x[(shift + r + k / 4) * 4 + k % 4];
          else a = x[(shift + r) * 32 + k];
          float b = w[((size_t)s * N + n) * K + k];
          if (mode == 2) { a = bf16_val(a); b = bf16_val(b); }
          else { a = tf32_trunc(a); b = tf32_trunc(b); }
          acc += (double)a * b;
        }
      }
      ref[r * N + n] = (float)acc;
    }
  float *dP, *dW, *dD;
  CK(cudaMalloc(&dP, P.size() * 4));
  CK(cudaMalloc(&dW, Wd.size() * 4));
  CK(cudaMalloc(&dD, 128 * N * 4));
  CK(cudaMemcpy(dP, P.data(), P.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dW, Wd.data(), Wd.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(window, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  window<<<1, 128, 100 * 1024>>>(mode, dP, dW, dD);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> got(128 * N);
  cudaMemcpy(got.data(), dD, got.size() * 4, cudaMemcpyDeviceToHost);
  for (int i = 0; i < 128 * N; ++i) worst = fmax(worst, fabs(got[i] - ref[i]) / fmax(1.0, fabs(ref[i])));
  printf("{\"probe\": \"window\", \"mode\": %d, \"status\": \"%s\", \"max_rel_err\": %.3e, \"got0\": %f, \"ref0\": %f}\n",
         mode, cudaGetErrorString(e), worst, got[0], ref[0]);
  cudaFree(dP); cudaFree(dW); cudaFree(dD);
}

int main() {
  long long* cyc;
  CK(cudaMalloc(&cyc, 8));
  CK(cudaFuncSetAttribute(tput, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  const int iters = 8192;
  for (int kind = 0; kind < 2; ++kind)
    for (int n = 32; n <= 256; n *= 2) {
      tput<<<148, 128, 64 * 1024>>>(kind, n, iters, cyc);
      CK(cudaDeviceSynchronize());
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      tput<<<148, 128, 64 * 1024>>>(kind, n, iters, cyc);
      cudaEventRecord(b);
      CK(cudaDeviceSynchronize());
      float ms; cudaEventElapsedTime(&ms, a, b);
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double kk = kind == 0 ? 8 : 16;
      const double flops = 2.0 * 128 * n * kk * iters * 148;
      printf("{\"probe\": \"tput\", \"kind\": \"%s\", \"N\": %d, \"cyc_per_mma\": %.2f, \"tflops\": %.1f}\n",
             kind == 0 ? "tf32" : "bf16", n, (double)c / iters, flops / (ms * 1e-3) / 1e12);
    }
  const char* only = getenv("PROBE_ONLY");
  if (!only || (strcmp(only, "layout") && strcmp(only, "conv1"))) {
  run_tput2<0, 32>(); run_tput2<0, 64>(); run_tput2<0, 128>(); run_tput2<0, 256>();
  run_tput2<1, 32>(); run_tput2<1, 64>(); run_tput2<1, 128>(); run_tput2<1, 256>();
  }
  for (int pass = 0; pass < 2; ++pass) {
    // dense core layout (aligned), then misaligned starts, then the conv's planar layout
    if (pass == 0) {
      run_tput3<32>("dense", 0, 128, 1024); run_tput3<64>("dense", 0, 128, 1024);
      run_tput3<32>("dense+16", 16, 128, 1024); run_tput3<64>("dense+16", 16, 128, 1024);
      run_tput3<32>("dense+64", 64, 128, 1024); run_tput3<64>("dense+64", 64, 128, 1024);
    } else {
      run_tput3<32>("planar", 0, 6400, 320); run_tput3<64>("planar", 0, 6400, 320);
      run_tput3<32>("planar+16", 16, 6400, 320); run_tput3<64>("planar+16", 16, 6400, 320);
      run_tput3<32>("planar_sbo256", 0, 6400, 256); run_tput3<64>("planar_sbo256", 0, 6400, 256);
      run_tput3<32>("planar_sbo384", 0, 6400, 384); run_tput3<64>("planar_sbo384", 0, 6400, 384);
      run_tput3<32>("planar+16_sbo256", 16, 6400, 256); run_tput3<64>("planar+16_sbo256", 16, 6400, 256);
      run_tput3<32>("toeplitz", 0, 16, 128); run_tput3<64>("toeplitz", 0, 16, 128);
    }
  }
  if (only && !strcmp(only, "layout")) return 0;
  if (only && !strcmp(only, "conv1")) {
    long long* cyc;
    CK(cudaMalloc(&cyc, 8));
    CK(cudaFuncSetAttribute(tput4, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (int mode = 0; mode < 2; ++mode) {
      tput4<<<148, 128, 200 * 1024>>>(2000, mode, cyc);
      CK(cudaDeviceSynchronize());
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("{\"probe\": \"conv1_stream\", \"mode\": %d, \"cyc_per_mma\": %.2f, \"cyc_per_supertile\": %.1f}\n",
             mode, (double)c / (2000.0 * 60), (double)c / 2000.0);
    }
    return 0;
  }
  for (int mode = 0; mode < 3; ++mode) run_window(mode);
  return 0;
}
