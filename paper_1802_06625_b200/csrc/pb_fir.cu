// Complex FIR firings of the DPD filter bank (apps/predistortion.py:41-83).
//
// Bit-exactness contract with FirBranch.fire (predistortion.py:51-65):
//   acc_r = +0, acc_i = +0
//   for t in 0..9 (ascending):
//     acc_r = fl(acc_r + fl(fl(cr[t]*xr[n-t]) - fl(ci[t]*xi[n-t])))
//     acc_i = fl(acc_i + fl(fl(cr[t]*xi[n-t]) + fl(ci[t]*xr[n-t])))
// Every product and sum is rounded on its own (numpy evaluates one binary op
// at a time), so no FMA may appear.  Blackwell's paired FP32 pipe is used
// without contraction: FMUL2 forms {cr*x, ci*x} for one sample plane at a
// time with the sample broadcast to both lanes, two scalar FADDs combine the
// cross terms and one FADD2 accumulates {acc_r, acc_i}.  ptxas fuses a
// mul.rn.f32x2 feeding an add.rn.f32x2 into FFMA2 even with -fmad=false, so
// the products never feed a paired add directly (checked in the SASS: no
// FFMA/FFMA2 in these kernels).
#include <algorithm>

#include "pb_common.cuh"

namespace {

typedef unsigned long long u64;

constexpr int kTaps = PB_TAPS;
constexpr int kHist = PB_TAPS - 1;
constexpr int kThreads = 128;
constexpr int kPerThread = 8;                    // consecutive outputs per thread
constexpr int kTile = kThreads * kPerThread;     // outputs per CTA tile
constexpr int kPad = 12;                         // halo slots in front of the tile (>= 9, x4)
constexpr int kWin = kPerThread + kPad;          // per-thread window (20 samples)

__device__ __forceinline__ u64 pack2(float lo, float hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack2(u64 v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ u64 fmul2(u64 a, u64 b) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

struct Taps {
  u64 p[kTaps];  // {cr, ci}
  u64 q[kTaps];  // {ci, cr}
};

__device__ __forceinline__ void load_taps(const float* taps, Taps& tp) {
#pragma unroll
  for (int t = 0; t < kTaps; ++t) {
    float cr = __ldg(taps + t), ci = __ldg(taps + kTaps + t);
    tp.p[t] = pack2(cr, ci);
    tp.q[t] = pack2(ci, cr);
  }
}

// One output sample: returns {acc_r, acc_i} packed.  wr/wi index i holds
// sample (first output of the thread) - kPad + i.
template <int V>
__device__ __forceinline__ u64 fir_point(const float (&wr)[kWin], const float (&wi)[kWin],
                                         const Taps& tp) {
  u64 acc = pack2(0.0f, 0.0f);
#pragma unroll
  for (int t = 0; t < kTaps; ++t) {
    const float xr = wr[kPad + V - t], xi = wi[kPad + V - t];
    u64 P = fmul2(tp.p[t], pack2(xr, xr));  // {cr*xr, ci*xr}
    u64 Q = fmul2(tp.q[t], pack2(xi, xi));  // {ci*xi, cr*xi}
    float prr, pir, qii, qri;
    unpack2(P, prr, pir);
    unpack2(Q, qii, qri);
    const float u = __fsub_rn(prr, qii);  // cr*xr - ci*xi
    const float w = __fadd_rn(qri, pir);  // cr*xi + ci*xr
    acc = fadd2(acc, pack2(u, w));
  }
  return acc;
}

template <int V>
struct Unroll {
  __device__ __forceinline__ static void run(const float (&wr)[kWin], const float (&wi)[kWin],
                                             const Taps& tp, u64 (&y)[kPerThread]) {
    Unroll<V - 1>::run(wr, wi, tp, y);
    y[V - 1] = fir_point<V - 1>(wr, wi, tp);
  }
};
template <>
struct Unroll<0> {
  __device__ __forceinline__ static void run(const float (&)[kWin], const float (&)[kWin],
                                             const Taps&, u64 (&)[kPerThread]) {}
};

// Stage tile [t0, t0+kTile) of both planes (clamped to B) into shared memory
// behind kPad halo slots.  Returns nothing; halo filled separately.
__device__ __forceinline__ void stage_tile(const float* __restrict__ span, int64_t B, int t0,
                                           float* sr, float* si) {
  // 2 planes x kTile floats = 2*kTile/4 float4
  const float4* pr = reinterpret_cast<const float4*>(span + t0);
  const float4* pi = reinterpret_cast<const float4*>(span + B + t0);
  const int64_t rem = B - t0;
  const int n4 = (int)(rem < kTile ? rem : kTile) / 4;
  for (int k = threadIdx.x; k < n4; k += kThreads) {
    float4 a = __ldg(pr + k);
    float4 b = __ldg(pi + k);
    reinterpret_cast<float4*>(sr + kPad)[k] = a;
    reinterpret_cast<float4*>(si + kPad)[k] = b;
  }
}

__device__ __forceinline__ void load_window(const float* sr, const float* si, float (&wr)[kWin],
                                            float (&wi)[kWin]) {
  const float4* a = reinterpret_cast<const float4*>(sr + kPerThread * threadIdx.x);
  const float4* b = reinterpret_cast<const float4*>(si + kPerThread * threadIdx.x);
#pragma unroll
  for (int k = 0; k < kWin / 4; ++k) {
    float4 x = a[k], y = b[k];
    wr[4 * k + 0] = x.x; wr[4 * k + 1] = x.y; wr[4 * k + 2] = x.z; wr[4 * k + 3] = x.w;
    wi[4 * k + 0] = y.x; wi[4 * k + 1] = y.y; wi[4 * k + 2] = y.z; wi[4 * k + 3] = y.w;
  }
}

__device__ __forceinline__ void store_out(float* __restrict__ out, int64_t B, int n0,
                                          const u64 (&y)[kPerThread]) {
  float r[kPerThread], i[kPerThread];
#pragma unroll
  for (int v = 0; v < kPerThread; ++v) unpack2(y[v], r[v], i[v]);
  float4* orr = reinterpret_cast<float4*>(out + n0);
  float4* oi = reinterpret_cast<float4*>(out + B + n0);
#pragma unroll
  for (int k = 0; k < kPerThread / 4; ++k) {
    orr[k] = make_float4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
    oi[k] = make_float4(i[4 * k], i[4 * k + 1], i[4 * k + 2], i[4 * k + 3]);
  }
}

// History source of a fir_branch firing: state (first firing of the epoch) or
// the last kHist samples of the actor's previous input span.
__device__ __forceinline__ void history_ptrs(const pb_fir_actor& a, const pb_resolved& res, int s,
                                             int j, int64_t B, const float*& hr,
                                             const float*& hi) {
  if (j == 0) {
    hr = a.state + (int64_t)s * 2 * kHist;
    hi = hr + kHist;
  } else {
    int np = pb::firing_iter(res, a.cond, s, j - 1);
    const float* prev = reinterpret_cast<const float*>(pb::span_ptr(a.in, res, s, np));
    hr = prev + B - kHist;
    hi = prev + 2 * B - kHist;
  }
}

// ------------------------------------------------- per-actor batched firings

__global__ void __launch_bounds__(kThreads, 4)
fir_kernel(const pb_fir_actor* __restrict__ actors, pb_resolved res, int64_t B, int tiles) {
  const pb_fir_actor& a = actors[blockIdx.z];
  const int s = blockIdx.y;
  const int j = blockIdx.x / tiles;
  const int tile = blockIdx.x % tiles;
  if (j >= pb::cond_count(res, a.cond, s)) return;
  const int n = pb::firing_iter(res, a.cond, s, j);
  const int t0 = tile * kTile;

  __shared__ __align__(16) float sr[kPad + kTile];
  __shared__ __align__(16) float si[kPad + kTile];

  const float* in = reinterpret_cast<const float*>(pb::span_ptr(a.in, res, s, n));
  float* out = reinterpret_cast<float*>(pb::span_ptr(a.out, res, s, n));
  stage_tile(in, B, t0, sr, si);
  if (threadIdx.x < kHist) {
    const int k = threadIdx.x;
    float hr_v, hi_v;
    if (t0 > 0) {
      hr_v = in[t0 - kHist + k];
      hi_v = in[B + t0 - kHist + k];
    } else {
      const float *hr, *hi;
      history_ptrs(a, res, s, j, B, hr, hi);
      hr_v = hr[k];
      hi_v = hi[k];
    }
    sr[kPad - kHist + k] = hr_v;
    si[kPad - kHist + k] = hi_v;
  } else if (threadIdx.x < kPad) {
    sr[threadIdx.x - kHist] = 0.f;
    si[threadIdx.x - kHist] = 0.f;
  }
  Taps tp;
  load_taps(a.taps, tp);
  __syncthreads();

  const int n0 = t0 + kPerThread * threadIdx.x;
  if (n0 >= B) return;
  float wr[kWin], wi[kWin];
  load_window(sr, si, wr, wi);
  u64 y[kPerThread];
  Unroll<kPerThread>::run(wr, wi, tp, y);
  store_out(out, B, n0, y);
}

__global__ void fir_carry_kernel(const pb_fir_actor* __restrict__ actors, pb_resolved res,
                                 int64_t B) {
  const pb_fir_actor& a = actors[blockIdx.y];
  const int s = blockIdx.x;
  const int cnt = pb::cond_count(res, a.cond, s);
  if (cnt == 0 || threadIdx.x >= 2 * kHist) return;
  const int nl = pb::firing_iter(res, a.cond, s, cnt - 1);
  const float* in = reinterpret_cast<const float*>(pb::span_ptr(a.in, res, s, nl));
  const int plane = threadIdx.x / kHist, k = threadIdx.x % kHist;
  a.state[(int64_t)s * 2 * kHist + plane * kHist + k] = in[plane * B + B - kHist + k];
}

// --------------------------------------------------------- fused filter bank

__global__ void __launch_bounds__(kThreads, 4)
filter_bank_kernel(pb_filter_bank bank, pb_resolved res, int64_t B, int tiles) {
  const int s = blockIdx.y;
  const int n = blockIdx.x / tiles;
  const int tile = blockIdx.x % tiles;
  if (n >= res.n_iter) return;
  if (!pb::active(res, bank.actor_cond, s, n)) return;
  const int t0 = tile * kTile;

  __shared__ __align__(16) float sr[kPad + kTile];
  __shared__ __align__(16) float si[kPad + kTile];
  __shared__ float hist[PB_MAX_BRANCHES][2][kHist];

  const float* in = reinterpret_cast<const float*>(pb::span_ptr(bank.in, res, s, n));
  float* out = reinterpret_cast<float*>(pb::span_ptr(bank.out, res, s, n));
  stage_tile(in, B, t0, sr, si);
  if (t0 > 0) {
    if (threadIdx.x < kHist) {
      const int k = threadIdx.x;
      sr[kPad - kHist + k] = in[t0 - kHist + k];
      si[kPad - kHist + k] = in[B + t0 - kHist + k];
    }
  } else {
    // per-branch history: only branches active at this iteration matter
    for (int e = threadIdx.x; e < bank.n_branches * 2 * kHist; e += kThreads) {
      const int b = e / (2 * kHist), plane = (e / kHist) & 1, k = e % kHist;
      const pb_fir_actor& a = bank.branches[b];
      float v = 0.f;
      if (pb::active(res, a.cond, s, n)) {
        const int j = a.cond < 0 ? n
                                 : res.prefix[((int64_t)a.cond * res.n_streams + s) * res.cap + n];
        const float *hr, *hi;
        history_ptrs(a, res, s, j, B, hr, hi);
        v = plane ? hi[k] : hr[k];
      }
      hist[b][plane][k] = v;
    }
  }
  if (threadIdx.x < kPad - kHist) {
    sr[threadIdx.x] = 0.f;
    si[threadIdx.x] = 0.f;
  }
  __syncthreads();

  const int n0 = t0 + kPerThread * threadIdx.x;
  if (n0 >= B) return;
  float wr[kWin], wi[kWin];
  load_window(sr, si, wr, wi);
  // samples of the window that lie before the span start come from the
  // branch's own history (tile 0, threads 0 and 1 only)
  const bool patch = (n0 - kPad) < 0;

  u64 sum[kPerThread];
#pragma unroll
  for (int v = 0; v < kPerThread; ++v) sum[v] = pack2(0.0f, 0.0f);

  for (int b = 0; b < bank.n_branches; ++b) {
    const pb_fir_actor& a = bank.branches[b];
    if (!pb::active(res, a.cond, s, n)) continue;  // uniform across the CTA
    if (patch) {
#pragma unroll
      for (int i = 0; i < kPad; ++i) {
        const int m = n0 - kPad + i;  // sample index relative to span start
        if (m < 0 && m >= -kHist) {
          wr[i] = hist[b][0][m + kHist];
          wi[i] = hist[b][1][m + kHist];
        }
      }
    }
    Taps tp;
    load_taps(a.taps, tp);
    u64 y[kPerThread];
    Unroll<kPerThread>::run(wr, wi, tp, y);
#pragma unroll
    for (int v = 0; v < kPerThread; ++v) sum[v] = fadd2(sum[v], y[v]);
  }
  store_out(out, B, n0, sum);
}

int check_span(int64_t span_bytes, int64_t* B) {
  if (span_bytes % 8 != 0)
    return pb::fail(PB_E_UNSUPPORTED, "fir_branch span must hold complex fp32 planes");
  *B = span_bytes / 8;
  if (*B % kPerThread != 0 || *B < kPad)
    return pb::fail(PB_E_UNSUPPORTED, "fir_branch block length " + std::to_string(*B) +
                                          " must be a multiple of 8 and >= 12");
  return PB_OK;
}

}  // namespace

extern "C" {

int pb_fire_fir(const pb_fir_actor* actors, int n_actors, pb_resolved res, int64_t block,
                void* stream) {
  if (n_actors == 0 || res.n_iter == 0) return PB_OK;
  int64_t B = block;
  int rc = check_span(block * 8, &B);
  if (rc) return rc;
  const int tiles = (int)((B + kTile - 1) / kTile);
  dim3 grid((unsigned)(tiles * res.n_iter), res.n_streams, n_actors);
  fir_kernel<<<grid, kThreads, 0, pb::as_stream(stream)>>>(actors, res, B, tiles);
  PB_LAUNCHED("fir_kernel");
  return PB_OK;
}

int pb_fir_carry(const pb_fir_actor* actors, int n_actors, pb_resolved res, int64_t block,
                 void* stream) {
  if (n_actors == 0 || res.n_iter == 0) return PB_OK;
  dim3 grid(res.n_streams, n_actors);
  fir_carry_kernel<<<grid, 32, 0, pb::as_stream(stream)>>>(actors, res, block);
  PB_LAUNCHED("fir_carry_kernel");
  return PB_OK;
}

int pb_fire_filter_bank(pb_filter_bank bank, pb_resolved res, int64_t block, void* stream) {
  if (res.n_iter == 0) return PB_OK;
  if (bank.n_branches < 1 || bank.n_branches > PB_MAX_BRANCHES)
    return pb::fail(PB_E_UNSUPPORTED, "filter bank needs 1.." + std::to_string(PB_MAX_BRANCHES) +
                                          " branches");
  int64_t B = block;
  int rc = check_span(block * 8, &B);
  if (rc) return rc;
  const int tiles = (int)((B + kTile - 1) / kTile);
  dim3 grid((unsigned)(tiles * res.n_iter), res.n_streams);
  filter_bank_kernel<<<grid, kThreads, 0, pb::as_stream(stream)>>>(bank, res, B, tiles);
  PB_LAUNCHED("filter_bank_kernel");
  return PB_OK;
}

}  // extern "C"
