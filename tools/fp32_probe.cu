// FP32 pipe throughput probe on B200: scalar FMUL/FADD vs paired FMUL2/FADD2
// (and FFMA for reference).  Prints lane-ops per second per kind; used to
// bound the bit-exact FIR (no FMA allowed) in DESIGN.md.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b){u64 r; asm("mov.b64 %0,{%1,%2};":"=l"(r):"f"(a),"f"(b)); return r;}
__device__ __forceinline__ u64 mul2(u64 a,u64 b){u64 r; asm volatile("mul.rn.f32x2 %0,%1,%2;":"=l"(r):"l"(a),"l"(b)); return r;}
__device__ __forceinline__ u64 add2(u64 a,u64 b){u64 r; asm volatile("add.rn.f32x2 %0,%1,%2;":"=l"(r):"l"(a),"l"(b)); return r;}
constexpr int CH = 8, IT = 4096;
template<int KIND> __global__ void probe(float* out, float s) {
  float a[CH]; u64 b[CH];
  for (int c = 0; c < CH; ++c) { a[c] = threadIdx.x * 1e-3f + c; b[c] = pk(a[c], a[c] + 1); }
  u64 sc = pk(s, s);
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (KIND == 0) a[c] = __fmul_rn(a[c], s);
      if (KIND == 1) a[c] = __fadd_rn(a[c], s);
      if (KIND == 2) b[c] = mul2(b[c], sc);
      if (KIND == 3) b[c] = add2(b[c], sc);
      if (KIND == 4) a[c] = __fmaf_rn(a[c], s, s);
      if (KIND == 5) { b[c] = mul2(b[c], sc); a[c] = __fadd_rn(a[c], s); }
    }
  }
  float acc = 0; for (int c = 0; c < CH; ++c) { float x,y; asm("mov.b64 {%0,%1},%2;":"=f"(x),"=f"(y):"l"(b[c])); acc += a[c] + x + y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template<int KIND> double run(float* d, int blocks, int threads, double lanes_per_instr) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  probe<KIND><<<blocks, threads>>>(d, 1.0001f);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) probe<KIND><<<blocks, threads>>>(d, 1.0001f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double instr = 5.0 * blocks * threads * (double)IT * CH * (KIND == 5 ? 2 : 1);
  return instr * lanes_per_instr / (ms * 1e-3) / 1e12;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* d; int blocks = sms * 8, threads = 256;
  cudaMalloc(&d, blocks * threads * 4);
  printf("{\"sms\": %d, \"clock_khz\": %d,\n", sms, clk);
  printf(" \"fmul_tops\": %.2f,\n", run<0>(d, blocks, threads, 1));
  printf(" \"fadd_tops\": %.2f,\n", run<1>(d, blocks, threads, 1));
  printf(" \"fmul2_lane_tops\": %.2f,\n", run<2>(d, blocks, threads, 2));
  printf(" \"fadd2_lane_tops\": %.2f,\n", run<3>(d, blocks, threads, 2));
  printf(" \"ffma_tops\": %.2f,\n", run<4>(d, blocks, threads, 1));
  printf(" \"fmul2+fadd_mixed_instr_tops\": %.2f}\n", run<5>(d, blocks, threads, 1));
  return 0;
}
