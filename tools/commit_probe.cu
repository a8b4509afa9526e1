// tcgen05.commit cost probe (run under gpurun): one CTA per SM, warp 0's
// elected lane issues K TS MMAs (M=128, N=32, K=16, bf16, A in TMEM) and then
// a tcgen05.commit to an mbarrier, R times; a second warp waits on every
// commit (as the conv kernel's converters / epilogue do).  Reports cycles per
// MMA, the clock cycles the issuing thread spends in the MMA run and in the
// commit instruction, for K in {0, 15, 60, 240}, and with 0 / 1 / 2 extra
// commits per run (the conv kernel issues 1 + ~2 commits per 60 MMAs).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e_), __LINE__); return 1;} } while (0)

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a),
               "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(su(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ bool elect() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(e));
  return e;
}

__global__ void probe(int K, int R, int extra, unsigned long long* out) {
  __shared__ __align__(1024) uint8_t bsm[32 * 16 * 2 * 4];
  __shared__ uint64_t bars[8];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < (int)sizeof(bsm); i += blockDim.x) bsm[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | (4u << 17) | (8u << 24);   // N=32 M=128
  const uint64_t bd = sdesc(su(bsm), 128, 256);
  long long t_mma = 0, t_commit = 0, t0 = clock64();
  if (warp == 0) {
    for (int r = 0; r < R; ++r) {
      if (elect()) {
        long long a = clock64();
        for (int k = 0; k < K; ++k) mma_ts((k & 7) * 32, 256 + (k & 3) * 16, bd, id, 1u);
        long long b = clock64();
        for (int e = 0; e < extra; ++e) commit(&bars[2 + (r & 1) * 2 + e]);
        commit(&bars[r & 1]);
        long long c = clock64();
        t_mma += b - a;
        t_commit += c - b;
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    for (int r = 0; r < R; ++r) {
      wait(&bars[r & 1], (r >> 1) & 1);
      for (int e = 0; e < extra; ++e) wait(&bars[2 + (r & 1) * 2 + e], (r >> 1) & 1);
    }
  }
  long long t1 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 4 + 0] = clock64() - t0;
    out[blockIdx.x * 4 + 1] = t_mma;
    out[blockIdx.x * 4 + 2] = t_commit;
    out[blockIdx.x * 4 + 3] = t1 - t0;
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  unsigned long long* d;
  CK(cudaMalloc(&d, 148 * 4 * 8));
  unsigned long long h[148 * 4];
  int Ks[] = {0, 15, 60, 240};
  for (int extra = 0; extra <= 2; ++extra)
    for (int K : Ks) {
      const int R = K ? 48000 / K : 1000;
      probe<<<148, 64>>>(K, R, extra, d);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
      double tot = 0, tm = 0, tc = 0;
      for (int b = 0; b < 148; ++b) { tot += h[b * 4]; tm += h[b * 4 + 1]; tc += h[b * 4 + 2]; }
      tot /= 148; tm /= 148; tc /= 148;
      printf("{\"K\": %d, \"runs\": %d, \"extra_commits\": %d, \"cycles_per_run\": %.1f, "
             "\"cycles_per_mma\": %.2f, \"issue_cycles_per_run\": %.1f, \"commit_cycles_per_run\": %.1f}\n",
             K, R, extra, tot / R, K ? tot / R / K : 0.0, tm / R, tc / R);
    }
  return 0;
}
