// Microbenchmark: cycles per (tap, output) of bit-identical FIR inner-loop
// instruction mixes on B200.  All variants compute exactly
//   acc = fl(acc + fl(fl(cr*xr) - fl(ci*xi))), fl(acc_i + fl(fl(cr*xi) + fl(ci*xr)))
// and the probe checks their outputs are bitwise equal.
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b){u64 r; asm("mov.b64 %0,{%1,%2};":"=l"(r):"f"(a),"f"(b)); return r;}
__device__ __forceinline__ void up(u64 v, float&a, float&b){asm("mov.b64 {%0,%1},%2;":"=f"(a),"=f"(b):"l"(v));}
__device__ __forceinline__ u64 mul2(u64 a,u64 b){u64 r; asm("mul.rn.f32x2 %0,%1,%2;":"=l"(r):"l"(a),"l"(b)); return r;}
__device__ __forceinline__ u64 add2(u64 a,u64 b){u64 r; asm("add.rn.f32x2 %0,%1,%2;":"=l"(r):"l"(a),"l"(b)); return r;}
constexpr int V = 8, T = 10, W = V + 12;
template <int VAR>
__device__ __forceinline__ void fir(const float (&wr)[W], const float (&wi)[W], const float4* taps, float (&yr)[V], float (&yi)[V]) {
  if (VAR == 0) {            // current: 2 FMUL2 + 2 FADD + 1 FADD2
    u64 y[V];
#pragma unroll
    for (int v = 0; v < V; ++v) y[v] = pk(0.f, 0.f);
#pragma unroll
    for (int t = 0; t < T; ++t) { float4 c = taps[t]; u64 P = pk(c.x, c.y), Q = pk(c.z, c.w);
#pragma unroll
      for (int v = 0; v < V; ++v) { float xr = wr[12+v-t], xi = wi[12+v-t]; float a,b,cc,d;
        up(mul2(P, pk(xr,xr)), a, b); up(mul2(Q, pk(xi,xi)), cc, d);
        y[v] = add2(y[v], pk(__fsub_rn(a, cc), __fadd_rn(d, b))); } }
#pragma unroll
    for (int v = 0; v < V; ++v) up(y[v], yr[v], yi[v]);
  } else if (VAR == 1) {     // scalar: 4 FMUL + 4 FADD
#pragma unroll
    for (int v = 0; v < V; ++v) { yr[v] = 0.f; yi[v] = 0.f; }
#pragma unroll
    for (int t = 0; t < T; ++t) { float4 c = taps[t];
#pragma unroll
      for (int v = 0; v < V; ++v) { float xr = wr[12+v-t], xi = wi[12+v-t];
        yr[v] = __fadd_rn(yr[v], __fsub_rn(__fmul_rn(c.x, xr), __fmul_rn(c.y, xi)));
        yi[v] = __fadd_rn(yi[v], __fadd_rn(__fmul_rn(c.x, xi), __fmul_rn(c.y, xr))); } }
  } else if (VAR == 2) {     // 4 FMUL + 2 FADD + 1 FADD2
    u64 y[V];
#pragma unroll
    for (int v = 0; v < V; ++v) y[v] = pk(0.f, 0.f);
#pragma unroll
    for (int t = 0; t < T; ++t) { float4 c = taps[t];
#pragma unroll
      for (int v = 0; v < V; ++v) { float xr = wr[12+v-t], xi = wi[12+v-t];
        float u = __fsub_rn(__fmul_rn(c.x, xr), __fmul_rn(c.y, xi));
        float w = __fadd_rn(__fmul_rn(c.x, xi), __fmul_rn(c.y, xr));
        y[v] = add2(y[v], pk(u, w)); } }
#pragma unroll
    for (int v = 0; v < V; ++v) up(y[v], yr[v], yi[v]);
  } else if (VAR == 3) {     // 2 FMUL2 + 4 FADD
#pragma unroll
    for (int v = 0; v < V; ++v) { yr[v] = 0.f; yi[v] = 0.f; }
#pragma unroll
    for (int t = 0; t < T; ++t) { float4 c = taps[t]; u64 P = pk(c.x, c.y), Q = pk(c.z, c.w);
#pragma unroll
      for (int v = 0; v < V; ++v) { float xr = wr[12+v-t], xi = wi[12+v-t]; float a,b,cc,d;
        up(mul2(P, pk(xr,xr)), a, b); up(mul2(Q, pk(xi,xi)), cc, d);
        yr[v] = __fadd_rn(yr[v], __fsub_rn(a, cc)); yi[v] = __fadd_rn(yi[v], __fadd_rn(d, b)); } }
  } else if (VAR == 4) {     // pair over outputs: FMUL2 of {xr[v],xr[v+1]} x cr broadcast...
    // products for two adjacent outputs share a tap: {cr*xr[n], cr*xr[n+1]}
    u64 Yr[V/2], Yi[V/2];
#pragma unroll
    for (int v = 0; v < V/2; ++v) { Yr[v] = pk(0.f,0.f); Yi[v] = pk(0.f,0.f); }
#pragma unroll
    for (int t = 0; t < T; ++t) { float4 c = taps[t];
#pragma unroll
      for (int v = 0; v < V; v += 2) {
        u64 XR = pk(wr[12+v-t], wr[13+v-t]), XI = pk(wi[12+v-t], wi[13+v-t]);
        float a0,a1,b0,b1,c0,c1,d0,d1;
        up(mul2(XR, pk(c.x,c.x)), a0, a1); up(mul2(XI, pk(c.y,c.y)), b0, b1);
        up(mul2(XI, pk(c.x,c.x)), c0, c1); up(mul2(XR, pk(c.y,c.y)), d0, d1);
        Yr[v/2] = add2(Yr[v/2], pk(__fsub_rn(a0,b0), __fsub_rn(a1,b1)));
        Yi[v/2] = add2(Yi[v/2], pk(__fadd_rn(c0,d0), __fadd_rn(c1,d1))); } }
#pragma unroll
    for (int v = 0; v < V; v += 2) { up(Yr[v/2], yr[v], yr[v+1]); up(Yi[v/2], yi[v], yi[v+1]); }
  }
}
template <int VAR>
__global__ void __launch_bounds__(128, 4) probe(const float* x, const float* tp, float* out, int iters) {
  __shared__ float4 taps[T];
  __shared__ float sr[1024 + 12], si[1024 + 12];
  if (threadIdx.x < T) taps[threadIdx.x] = make_float4(tp[threadIdx.x], tp[T+threadIdx.x], tp[T+threadIdx.x], tp[threadIdx.x]);
  for (int i = threadIdx.x; i < 1036; i += blockDim.x) { sr[i] = x[(blockIdx.x * 7 + i) % 4096]; si[i] = x[(blockIdx.x * 13 + i + 77) % 4096]; }
  __syncthreads();
  float accr[V] = {}, acci[V] = {};
  for (int it = 0; it < iters; ++it) {
    float wr[W], wi[W];
    int base = (8 * threadIdx.x + it * 8) % 1016;
#pragma unroll
    for (int k = 0; k < W; ++k) { wr[k] = sr[base + k]; wi[k] = si[base + k]; }
    float yr[V], yi[V];
    fir<VAR>(wr, wi, taps, yr, yi);
#pragma unroll
    for (int v = 0; v < V; ++v) { accr[v] = __fadd_rn(accr[v], yr[v]); acci[v] = __fadd_rn(acci[v], yi[v]); }
  }
  for (int v = 0; v < V; ++v) { out[(blockIdx.x * 128 + threadIdx.x) * 2 * V + v] = accr[v]; out[(blockIdx.x * 128 + threadIdx.x) * 2 * V + V + v] = acci[v]; }
}
template <int VAR> float run(const float* x, const float* tp, float* out, int blocks, int iters) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  probe<VAR><<<blocks, 128>>>(x, tp, out, iters);
  cudaEventRecord(a); probe<VAR><<<blocks, 128>>>(x, tp, out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float hx[4096], htp[2*T];
  for (int i = 0; i < 4096; ++i) hx[i] = ((i * 2654435761u) % 20001) / 10000.0f - 1.0f;
  for (int t = 0; t < T; ++t) { htp[t] = 0.05f * 3 / (t + 1); htp[T+t] = 0.002f * 3 * (t - 4.5f); }
  float *x, *tp, *out; int blocks = sms * 16, iters = 400;
  size_t n = (size_t)blocks * 128 * 2 * V;
  cudaMalloc(&x, sizeof hx); cudaMalloc(&tp, sizeof htp); cudaMalloc(&out, n * 4 * 5);
  cudaMemcpy(x, hx, sizeof hx, cudaMemcpyHostToDevice); cudaMemcpy(tp, htp, sizeof htp, cudaMemcpyHostToDevice);
  float ms[5];
  ms[0] = run<0>(x, tp, out + 0*n, blocks, iters); ms[1] = run<1>(x, tp, out + 1*n, blocks, iters);
  ms[2] = run<2>(x, tp, out + 2*n, blocks, iters); ms[3] = run<3>(x, tp, out + 3*n, blocks, iters);
  ms[4] = run<4>(x, tp, out + 4*n, blocks, iters);
  float* h = new float[n * 5]; cudaMemcpy(h, out, n * 4 * 5, cudaMemcpyDeviceToHost);
  double tapouts = (double)blocks * 128 * iters * V * T;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[5] = {"2FMUL2+2FADD+FADD2", "4FMUL+4FADD", "4FMUL+2FADD+FADD2", "2FMUL2+4FADD", "4FMUL2(out-pairs)+4FADD+2FADD2"};
  printf("{\n");
  for (int k = 0; k < 5; ++k) {
    bool same = memcmp(h, h + k * n, n * 4) == 0;
    double cyc = ms[k] * 1e-3 * clk * 1e3 * sms * 4 / (tapouts / 32);   // SMSP-cycles per warp tap-output
    printf(" \"%s\": {\"ms\": %.3f, \"smsp_cycles_per_warp_tap_output\": %.2f, \"bitwise_equal_to_v0\": %s}%s\n", names[k], ms[k], cyc, same ? "true" : "false", k < 4 ? "," : "");
  }
  printf("}\n");
}
