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
// the products never feed a paired add directly (SASS of this file has no
// FFMA/FFMA2; tests/test_native_host.py::test_no_fma_in_fir_kernels checks).
//
// Kernel structure (persistent, warp-specialised):
//   warp 0   producer: walks the work items (stream, iteration, tile), waits
//            for a free stage, streams the tile of both sample planes into
//            shared memory with cp.async.bulk (TMA bulk copy, completion on
//            the stage's mbarrier) and resolves the firing on the side: the
//            active branches in the combiner's port order and, for the first
//            tile of a span, each branch's 9-sample history.
//   warps 1-4 consumers: wait for a full stage, run the FIR of every active
//            branch over 8 consecutive outputs per thread, sum (bank) or
//            store per branch, release the stage.
// kStages stages keep the next tiles in flight while the FP32 pipe works.
#include <algorithm>
#include <string>

#include "pb_common.cuh"

namespace {

typedef unsigned long long u64;

constexpr int kTaps = PB_TAPS;
constexpr int kHist = PB_TAPS - 1;
constexpr int kConsumerWarps = 4;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kThreads = kConsumers + 32;        // + producer warp
constexpr int kPerThread = 8;                    // consecutive outputs per thread
constexpr int kTile = kConsumers * kPerThread;   // outputs per work item
constexpr int kPad = 12;                         // halo slots in front of the tile (>= 9, x4)
constexpr int kWin = kPerThread + kPad;          // per-thread window (20 samples)
constexpr int kStages = 4;
constexpr int kMaxBr = PB_MAX_BRANCHES;
constexpr int kChunkSpans = 4;               // spans per dynamic work grab

struct __align__(16) StageBuf {
  float re[kPad + kTile];
  float im[kPad + kTile];
};

struct __align__(16) Desc {
  u64 out;        // output span tile base (float*), bank mode and per-actor mode
  int valid;      // 0 terminates the consumers
  int t0;
  int n_act;
  int first;      // tile 0: window entries before the span come from hist
  int8_t br[kMaxBr];
  float hist[kMaxBr][2][kHist];
};

struct __align__(16) Smem {
  StageBuf buf[kStages];
  Desc desc[kStages];
  float4 taps[kMaxBr][kTaps];   // {cr, ci, ci, cr}
  u64 full[kStages];
  u64 empty[kStages];
};

// ----------------------------------------------------------- PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(u64* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(u64* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
      smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(u64* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
// try_wait with a suspend-time hint: the warp sleeps in hardware until the
// phase completes (or the hint elapses) instead of spinning on issue slots
// the FP32 consumers need.
__device__ __forceinline__ void mbar_wait(u64* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

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

// ------------------------------------------------------------- FIR math

// y[v] for the thread's 8 outputs; w*[i] holds sample (first output) - kPad + i.
__device__ __forceinline__ void fir8(const float (&wr)[kWin], const float (&wi)[kWin],
                                     const float4* __restrict__ taps, u64 (&y)[kPerThread]) {
#pragma unroll
  for (int v = 0; v < kPerThread; ++v) y[v] = pack2(0.0f, 0.0f);
#pragma unroll
  for (int t = 0; t < kTaps; ++t) {
    const float4 c = taps[t];
    const u64 P = pack2(c.x, c.y);  // {cr, ci}
    const u64 Q = pack2(c.z, c.w);  // {ci, cr}
#pragma unroll
    for (int v = 0; v < kPerThread; ++v) {
      const float xr = wr[kPad + v - t], xi = wi[kPad + v - t];
      float prr, pir, qii, qri;
      unpack2(fmul2(P, pack2(xr, xr)), prr, pir);  // {cr*xr, ci*xr}
      unpack2(fmul2(Q, pack2(xi, xi)), qii, qri);  // {ci*xi, cr*xi}
      y[v] = fadd2(y[v], pack2(__fsub_rn(prr, qii), __fadd_rn(qri, pir)));
    }
  }
}

// Same roundings with scalar FMUL/FADD only (8 issue slots per tap-output
// instead of 5, same FP32 pipe cycles); selected with kScalarMath.
__device__ __forceinline__ void fir8_scalar(const float (&wr)[kWin], const float (&wi)[kWin],
                                            const float4* __restrict__ taps,
                                            u64 (&y)[kPerThread]) {
  float yr[kPerThread], yi[kPerThread];
#pragma unroll
  for (int v = 0; v < kPerThread; ++v) yr[v] = yi[v] = 0.0f;
#pragma unroll
  for (int t = 0; t < kTaps; ++t) {
    const float4 c = taps[t];
#pragma unroll
    for (int v = 0; v < kPerThread; ++v) {
      const float xr = wr[kPad + v - t], xi = wi[kPad + v - t];
      yr[v] = __fadd_rn(yr[v], __fsub_rn(__fmul_rn(c.x, xr), __fmul_rn(c.y, xi)));
      yi[v] = __fadd_rn(yi[v], __fadd_rn(__fmul_rn(c.x, xi), __fmul_rn(c.y, xr)));
    }
  }
#pragma unroll
  for (int v = 0; v < kPerThread; ++v) y[v] = pack2(yr[v], yi[v]);
}

// Tolerance mode: one fused multiply-add per tap term (4 FFMA per
// tap-output instead of 8 rounded ops); not bit-exact.
__device__ __forceinline__ void fir8_fma(const float (&wr)[kWin], const float (&wi)[kWin],
                                         const float4* __restrict__ taps, u64 (&y)[kPerThread]) {
  float yr[kPerThread], yi[kPerThread];
#pragma unroll
  for (int v = 0; v < kPerThread; ++v) yr[v] = yi[v] = 0.0f;
#pragma unroll
  for (int t = 0; t < kTaps; ++t) {
    const float4 c = taps[t];
#pragma unroll
    for (int v = 0; v < kPerThread; ++v) {
      const float xr = wr[kPad + v - t], xi = wi[kPad + v - t];
      yr[v] = __fmaf_rn(-c.y, xi, __fmaf_rn(c.x, xr, yr[v]));
      yi[v] = __fmaf_rn(c.y, xr, __fmaf_rn(c.x, xi, yi[v]));
    }
  }
#pragma unroll
  for (int v = 0; v < kPerThread; ++v) y[v] = pack2(yr[v], yi[v]);
}

__device__ __forceinline__ void load_window(const StageBuf& sb, int ct, float (&wr)[kWin],
                                            float (&wi)[kWin]) {
  const float4* a = reinterpret_cast<const float4*>(sb.re + kPerThread * ct);
  const float4* b = reinterpret_cast<const float4*>(sb.im + kPerThread * ct);
#pragma unroll
  for (int k = 0; k < kWin / 4; ++k) {
    float4 x = a[k], z = b[k];
    wr[4 * k + 0] = x.x; wr[4 * k + 1] = x.y; wr[4 * k + 2] = x.z; wr[4 * k + 3] = x.w;
    wi[4 * k + 0] = z.x; wi[4 * k + 1] = z.y; wi[4 * k + 2] = z.z; wi[4 * k + 3] = z.w;
  }
}

__device__ __forceinline__ void store8(float* out, int64_t B, int n0, const u64 (&y)[kPerThread]) {
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

// ---------------------------------------------------------------- kernel
//
// kBank = true : items (s, n, tile) of the fused route -> fir* -> branch_sum
//                region; output = sum over active branches (combiner order)
// kBank = false: items (actor, s, j, tile) of per-actor batched firings;
//                output = the actor's own output span
template <bool kBank, int kMath>
__global__ void __launch_bounds__(kThreads, 4)
fir_persistent(const pb_filter_bank bank, const pb_fir_actor* __restrict__ actors, int n_actors,
               pb_resolved res, int64_t B, int tiles) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const pb_fir_actor* br = kBank ? bank.branches : actors;
  const int nb = kBank ? bank.n_branches : n_actors;

  for (int e = threadIdx.x; e < nb * kTaps; e += blockDim.x) {
    const int b = e / kTaps, t = e % kTaps;
    const float cr = br[b].taps[t], ci = br[b].taps[kTaps + t];
    sm.taps[b][t] = make_float4(cr, ci, ci, cr);
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < kStages; ++k) {
      mbar_init(&sm.full[k], 2);
      mbar_init(&sm.empty[k], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t per_unit = (int64_t)res.n_iter * tiles;  // items per (actor, stream)
  const int64_t total = (kBank ? 1 : (int64_t)n_actors) * res.n_streams * per_unit;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // Contiguous tile range per CTA: the tiles of one span are consecutive,
    // so a span's firing (active branches, histories) is resolved once, and
    // consecutive spans of one stream let each lane track when its branch
    // last fired (its history source) without global lookups.
    // Bank launches with a scheduler pointer grab chunks of kChunkSpans spans
    // dynamically (the active-branch count per span varies 1..K, so static
    // ranges leave a tail); otherwise each CTA takes one contiguous range.
    const bool dynamic = kBank && bank.sched != nullptr;
    const int64_t chunk = dynamic ? (int64_t)kChunkSpans * tiles : 0;
    int64_t w0 = total * blockIdx.x / gridDim.x;
    int64_t w1 = total * (blockIdx.x + 1) / gridDim.x;
    int k = 0;
    int64_t cur_unit = -1;
    int cur_it = -1;
    int n = 0;
    bool have = false;
    unsigned mask = 0;
    int prev_n = -2;   // lane b: iteration branch b last fired at (-1: none yet, -2: unknown)
    for (;;) {
    if (dynamic) {
      int64_t c = 0;
      if (lane == 0) c = atomicAdd(bank.sched, 1u);
      c = __shfl_sync(0xffffffffu, c, 0);
      w0 = c * chunk;
      if (w0 >= total) break;
      w1 = min(total, w0 + chunk);
      cur_unit = -1;   // chunks are not contiguous with the previous one
    }
    for (int64_t w = w0; w < w1; ++w) {
      int64_t r = w;
      int a = 0;
      if (!kBank) {
        a = (int)(r / ((int64_t)res.n_streams * per_unit));
        r %= (int64_t)res.n_streams * per_unit;
      }
      const int s = (int)(r / per_unit);
      r %= per_unit;
      const int it = (int)(r / tiles);
      const int tile = (int)(r % tiles);
      const int64_t unit = (int64_t)a * res.n_streams + s;
      if (unit != cur_unit || it != cur_it) {
        // ---- new span: resolve its firing
        if (unit != cur_unit) prev_n = -2;
        cur_unit = unit;
        cur_it = it;
        bool act = false;
        if (kBank) {
          n = it;
          have = pb::active(res, bank.actor_cond, s, n);
          if (have && lane < nb) act = pb::active(res, br[lane].cond, s, n);
        } else {
          have = it < pb::cond_count(res, actors[a].cond, s);
          n = have ? pb::firing_iter(res, actors[a].cond, s, it) : 0;
          act = have && lane == 0;
        }
        mask = __ballot_sync(0xffffffffu, act);
      }
      if (!have) continue;
      const int stage = k % kStages;
      mbar_wait(&sm.empty[stage], ((k / kStages) & 1) ^ 1);
      Desc& d = sm.desc[stage];
      StageBuf& sb = sm.buf[stage];
      const pb_span_ref& in_ref = kBank ? bank.in : actors[a].in;
      const float* in = reinterpret_cast<const float*>(pb::span_ptr(in_ref, res, s, n));
      const int t0 = tile * kTile;
      const int64_t rem = B - t0;
      const int len = (int)(rem < kTile ? rem : kTile);
      if (lane == 0) {
        const int lead = t0 > 0 ? kPad : 0;  // tile > 0: halo from the same span
        const uint32_t bytes = (uint32_t)(len + lead) * 4u;
        mbar_arrive_tx(&sm.full[stage], 2 * bytes);
        bulk_g2s(sb.re + kPad - lead, in + t0 - lead, bytes, &sm.full[stage]);
        bulk_g2s(sb.im + kPad - lead, in + B + t0 - lead, bytes, &sm.full[stage]);
      }
      const bool act = (mask >> lane) & 1u;
      if (act) {
        const int rank = __popc(mask & ((1u << lane) - 1u));
        d.br[rank] = (int8_t)(kBank ? lane : a);
        if (t0 == 0) {
          const pb_fir_actor& fa = br[kBank ? lane : a];
          int src = prev_n;  // iteration of the branch's previous firing
          if (src == -2) {
            const int j = kBank ? (fa.cond < 0 ? n
                                   : res.prefix[((int64_t)fa.cond * res.n_streams + s) * res.cap + n])
                                : it;
            src = j == 0 ? -1 : pb::firing_iter(res, fa.cond, s, j - 1);
          }
          const float *hr, *hi;
          if (src < 0) {
            hr = fa.state + (int64_t)s * 2 * kHist;
            hi = hr + kHist;
          } else {
            const float* prev = reinterpret_cast<const float*>(pb::span_ptr(fa.in, res, s, src));
            hr = prev + B - kHist;
            hi = prev + 2 * B - kHist;
          }
          float h[2 * kHist];
#pragma unroll
          for (int q = 0; q < kHist; ++q) {
            h[q] = hr[q];
            h[kHist + q] = hi[q];
          }
#pragma unroll
          for (int q = 0; q < kHist; ++q) {
            d.hist[rank][0][q] = h[q];
            d.hist[rank][1][q] = h[kHist + q];
          }
        }
      }
      if (lane == 0) {
        const pb_span_ref& out_ref = kBank ? bank.out : actors[a].out;
        float* out = reinterpret_cast<float*>(pb::span_ptr(out_ref, res, s, n));
        d.out = reinterpret_cast<u64>(out);
        d.valid = 1;
        d.t0 = t0;
        d.n_act = __popc(mask);
        d.first = t0 == 0;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.full[stage]);
      // the span's last tile: its active branches have now fired at n
      if (tile == tiles - 1 || w + 1 == w1) {
        if (act) prev_n = n;
      }
      ++k;
    }
    if (!dynamic) break;
    }
    if (dynamic && lane == 0) {
      // the last CTA out resets the scheduler for the next launch
      __threadfence();
      const unsigned done = atomicAdd(bank.sched + 1, 1u);
      if (done == gridDim.x - 1) {
        bank.sched[0] = 0;
        bank.sched[1] = 0;
        __threadfence();
      }
    }
    // terminator: consumers leave after the last produced stage
    {
      const int stage = k % kStages;
      mbar_wait(&sm.empty[stage], ((k / kStages) & 1) ^ 1);
      if (lane == 0) {
        sm.desc[stage].valid = 0;
        mbar_arrive_tx(&sm.full[stage], 0);
        mbar_arrive(&sm.full[stage]);
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int ct = threadIdx.x - 32;
  for (int k = 0;; ++k) {
    const int stage = k % kStages;
    mbar_wait(&sm.full[stage], (k / kStages) & 1);
    const Desc& d = sm.desc[stage];
    if (!d.valid) break;
    const int n0 = d.t0 + kPerThread * ct;
    const int n_act = d.n_act;
    float* out = reinterpret_cast<float*>(d.out);
    if (n0 < B) {
      float wr[kWin], wi[kWin];
      load_window(sm.buf[stage], ct, wr, wi);
      const bool patch = d.first && ct * kPerThread < kPad;
      u64 acc[kPerThread];
#pragma unroll
      for (int v = 0; v < kPerThread; ++v) acc[v] = pack2(0.0f, 0.0f);
      for (int r = 0; r < n_act; ++r) {
        if (patch) {
#pragma unroll
          for (int i = 0; i < kPad; ++i) {
            const int m = kPerThread * ct - kPad + i;  // sample index relative to the span
            if (m < 0 && m >= -kHist) {
              wr[i] = d.hist[r][0][m + kHist];
              wi[i] = d.hist[r][1][m + kHist];
            }
          }
        }
        u64 y[kPerThread];
        if (kMath == PB_FIR_EXACT)
          fir8_scalar(wr, wi, sm.taps[d.br[r]], y);
        else if (kMath == PB_FIR_EXACT_PAIRED)
          fir8(wr, wi, sm.taps[d.br[r]], y);
        else
          fir8_fma(wr, wi, sm.taps[d.br[r]], y);
        if (kBank) {
#pragma unroll
          for (int v = 0; v < kPerThread; ++v) acc[v] = fadd2(acc[v], y[v]);
        } else {
          store8(out, B, n0, y);
        }
      }
      if (kBank) store8(out, B, n0, acc);
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&sm.empty[stage]);
  }
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

int check_block(int64_t B) {
  if (B % kPerThread != 0 || B < kPad)
    return pb::fail(PB_E_UNSUPPORTED, "fir_branch block length " + std::to_string(B) +
                                          " must be a multiple of 8 and >= 12");
  return PB_OK;
}

template <bool kBank, int kMath>
int launch_variant(const pb_filter_bank& bank, const pb_fir_actor* actors, int n_actors,
                   const pb_resolved& res, int64_t B, cudaStream_t st) {
  const int tiles = (int)((B + kTile - 1) / kTile);
  const size_t smem = sizeof(Smem);
  static bool configured = false;
  if (!configured) {
    PB_CUDA(cudaFuncSetAttribute(fir_persistent<kBank, kMath>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  static int sms = 0, per_sm = 0;
  if (sms == 0) {
    int dev = 0;
    PB_CUDA(cudaGetDevice(&dev));
    PB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    PB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fir_persistent<kBank, kMath>,
                                                          kThreads, smem));
    per_sm = std::max(per_sm, 1);
  }
  const int64_t items =
      (kBank ? 1 : (int64_t)n_actors) * res.n_streams * (int64_t)res.n_iter * tiles;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)sms * per_sm));
  fir_persistent<kBank, kMath><<<grid, kThreads, smem, st>>>(bank, actors, n_actors, res, B, tiles);
  PB_LAUNCHED(kBank ? "fir_persistent<bank>" : "fir_persistent<actors>");
  return PB_OK;
}

// Scalar FMUL/FADD is the exact default: on B200 the paired FMUL2/FADD2 ops
// give no FP32 lane throughput (profiles/r1_fp32_probe.json) and the scalar
// mix measured 3% faster in this kernel (profiles/r1_fir_mix.json).
template <bool kBank>
int launch(const pb_filter_bank& bank, const pb_fir_actor* actors, int n_actors,
           const pb_resolved& res, int64_t B, int math, cudaStream_t st) {
  switch (math) {
    case PB_FIR_EXACT:
      return launch_variant<kBank, PB_FIR_EXACT>(bank, actors, n_actors, res, B, st);
    case PB_FIR_EXACT_PAIRED:
      return launch_variant<kBank, PB_FIR_EXACT_PAIRED>(bank, actors, n_actors, res, B, st);
    case PB_FIR_FMA:
      return launch_variant<kBank, PB_FIR_FMA>(bank, actors, n_actors, res, B, st);
    default:
      return pb::fail(PB_E_INVALID, "unknown FIR math mode " + std::to_string(math));
  }
}

}  // namespace

extern "C" {

int pb_fire_fir(const pb_fir_actor* actors, int n_actors, pb_resolved res, int64_t block,
                int math, void* stream) {
  if (n_actors == 0 || res.n_iter == 0) return PB_OK;
  if (n_actors > kMaxBr)
    return pb::fail(PB_E_UNSUPPORTED, "pb_fire_fir: at most " + std::to_string(kMaxBr) +
                                          " actors per launch");
  int rc = check_block(block);
  if (rc) return rc;
  pb_filter_bank none{};
  return launch<false>(none, actors, n_actors, res, block, math, pb::as_stream(stream));
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
  if (bank.n_branches < 1 || bank.n_branches > kMaxBr)
    return pb::fail(PB_E_UNSUPPORTED, "filter bank needs 1.." + std::to_string(kMaxBr) +
                                          " branches");
  int rc = check_block(block);
  if (rc) return rc;
  return launch<true>(bank, nullptr, 0, res, block, bank.math, pb::as_stream(stream));
}

}  // extern "C"
