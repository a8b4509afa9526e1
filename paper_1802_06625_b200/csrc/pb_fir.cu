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
#ifndef PB_FIR_CWARPS
#define PB_FIR_CWARPS 4
#endif
#ifndef PB_FIR_PER_THREAD
#define PB_FIR_PER_THREAD 8
#endif
constexpr int kConsumerWarps = PB_FIR_CWARPS;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kThreads = kConsumers + 32;        // + producer warp
constexpr int kPerThread = PB_FIR_PER_THREAD;    // consecutive outputs per thread
constexpr int kTile = kConsumers * kPerThread;   // outputs per work item
constexpr int kPad = 12;                         // halo slots in front of the tile (>= 9, x4)
constexpr int kWin = kPerThread + kPad;          // per-thread window (20 samples)
#ifndef PB_FIR_STAGES
#define PB_FIR_STAGES 4
#endif
constexpr int kStages = PB_FIR_STAGES;
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
  float pf_hist[2][kMaxBr][2][kHist];   // bank: next span's branch histories (cp.async)
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
// try_wait: kSuspendHint > 0 passes a suspend-time hint (the warp may sleep
// in hardware until the phase completes instead of spinning on issue slots
// the FP32 consumers need); PB_FIR_SUSPEND_NS at build time overrides it.
#ifndef PB_FIR_SUSPEND_NS
#define PB_FIR_SUSPEND_NS 0
#endif
__device__ __forceinline__ void mbar_wait(u64* bar, uint32_t parity) {
  if (PB_FIR_SUSPEND_NS > 0) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"((uint32_t)PB_FIR_SUSPEND_NS)
        : "memory");
  } else {
    pb::mbar_wait_trap(smem_u32(bar), parity);
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, u64* bar,
                                              u64 policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
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

__device__ __forceinline__ void cp_async16_plan(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}

// span_ptr with the stream's ring base already loaded (pb_common.cuh)
__device__ __forceinline__ const uint8_t* span_ptr_b(const pb_span_ref& r, int64_t base,
                                                     const pb_resolved& res, int s, int n) {
  int64_t idx = n;
  if (r.index_cond >= 0)
    idx = res.prefix[((int64_t)r.index_cond * res.n_streams + s) * res.cap + n];
  const int64_t x = base + idx + r.offset;
  const int64_t chunk = (uint64_t)x <= 0xFFFFFFFFull ? (int64_t)((uint32_t)x % (uint32_t)r.slots)
                                                     : x % r.slots;
  return r.data + (int64_t)s * r.stream_stride + chunk * r.span_bytes;
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
  for (int k = 0; k < kPerThread / 4; ++k) {   // streaming stores: output is not re-read here
    __stcs(orr + k, make_float4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]));
    __stcs(oi + k, make_float4(i[4 * k], i[4 * k + 1], i[4 * k + 2], i[4 * k + 3]));
  }
}

// ---------------------------------------------------------------- kernel
//
// kBank = true : items (s, n, tile) of the fused route -> fir* -> branch_sum
//                region; output = sum over active branches (combiner order)
// kBank = false: items (actor, s, j, tile) of per-actor batched firings;
//                output = the actor's own output span
// (The tolerance mode of the bank, PB_FIR_MERGED, runs as bank_plan_par_kernel
// + bank_stream_kernel below; this kernel serves the bit-exact bank and the
// per-actor firings.)
template <bool kBank, int kMath>
__global__ void __launch_bounds__(kThreads, 4)
fir_persistent(const pb_filter_bank bank, const pb_fir_actor* __restrict__ actors, int n_actors,
               pb_resolved res, int64_t B, int tiles) {
  pb::pdl_enter();
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
    // (MERGED work per span is constant: static ranges balance, and keep the
    // per-branch history source in registers across the CTA's spans)
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
    int64_t in_base = 0, out_base = 0;               // ring bases of the current stream
    const float* span_in = nullptr;                  // current span's input / output
    u64 span_out = 0;
    // bank: the next span's activity and each branch's history candidate are
    // loaded one span ahead (registers / cp.async into pf_hist), so resolving
    // a span costs no dependent global-load round trips
    int64_t pf_unit = -1;
    int pf_n = -1;
    bool pf_have = false, pf_act = false, pf_ok = false, cur_pf_ok = false;
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
    // decode w0 once, then step (a, s, it, tile) incrementally
    int a = 0, s = 0, it = 0, tile = 0;
    {
      int64_t r = w0;
      if (!kBank) {
        a = (int)(r / ((int64_t)res.n_streams * per_unit));
        r %= (int64_t)res.n_streams * per_unit;
      }
      s = (int)(r / per_unit);
      r %= per_unit;
      it = (int)(r / tiles);
      tile = (int)(r % tiles);
    }
    for (int64_t w = w0; w < w1; ++w) {
      if (w > w0 && ++tile == tiles) {
        tile = 0;
        if (++it == res.n_iter) {
          it = 0;
          if (++s == res.n_streams) {
            s = 0;
            ++a;
          }
        }
      }
      const int64_t unit = (int64_t)a * res.n_streams + s;
      if (unit != cur_unit || it != cur_it) {
        // ---- new span: resolve its firing
        if (unit != cur_unit) {
          prev_n = -2;
          const pb_span_ref& ir = kBank ? bank.in : actors[a].in;
          const pb_span_ref& orf = kBank ? bank.out : actors[a].out;
          in_base = ir.base ? ir.base[s] : 0;
          out_base = orf.base ? orf.base[s] : 0;
        }
        cur_unit = unit;
        cur_it = it;
        bool act = false;
        if (kBank) {
          n = it;
          const bool use_pf = unit == pf_unit && it == pf_n;
          if (use_pf) {
            have = pf_have;
            act = have && pf_act;
          } else {
            have = pb::active(res, bank.actor_cond, s, n);
            if (have && lane < nb) act = pb::active(res, br[lane].cond, s, n);
          }
          cur_pf_ok = use_pf && pf_ok;
          // prefetch span n + 1 of this stream
          if (it + 1 < res.n_iter) {
            pf_unit = unit;
            pf_n = it + 1;
            pf_have = pb::active(res, bank.actor_cond, s, it + 1);
            pf_act = lane < nb && pb::active(res, br[lane].cond, s, it + 1);
            const int src = act ? n : prev_n;   // branch's latest firing before n + 1
            pf_ok = lane < nb && src != -2;
            if (pf_ok) {
              const float* hr;
              const float* hi;
              if (src < 0) {
                hr = br[lane].state + (int64_t)s * 2 * kHist;
                hi = hr + kHist;
              } else {   // every branch fired on the bank's own input span
                const float* prev = reinterpret_cast<const float*>(
                    span_ptr_b(bank.in, in_base, res, s, src));
                hr = prev + B - kHist;
                hi = prev + 2 * B - kHist;
              }
              float* dst = sm.pf_hist[(it + 1) & 1][lane][0];
#pragma unroll
              for (int q = 0; q < kHist; ++q) {
                cp_async4(dst + q, hr + q);
                cp_async4(dst + kHist + q, hi + q);
              }
            }
          }
          // one group per span, possibly empty: "wait_group 1" at the next
          // span's first tile then covers exactly the groups issued before it
          asm volatile("cp.async.commit_group;" ::: "memory");
        } else {
          have = it < pb::cond_count(res, actors[a].cond, s);
          n = have ? pb::firing_iter(res, actors[a].cond, s, it) : 0;
          act = have && lane == 0;
        }
        mask = __ballot_sync(0xffffffffu, act);
        if (have) {   // the span's input / output, once per span
          span_in = reinterpret_cast<const float*>(
              span_ptr_b(kBank ? bank.in : actors[a].in, in_base, res, s, n));
          span_out = reinterpret_cast<u64>(
              span_ptr_b(kBank ? bank.out : actors[a].out, out_base, res, s, n));
        }
      }
      if (!have) continue;
      const int stage = k % kStages;
      mbar_wait(&sm.empty[stage], ((k / kStages) & 1) ^ 1);
      Desc& d = sm.desc[stage];
      StageBuf& sb = sm.buf[stage];
      const float* in = span_in;
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
        if (kBank && t0 == 0 && cur_pf_ok) {
          // prefetched one span ago (this lane's own cp.async groups)
          asm volatile("cp.async.wait_group 1;" ::: "memory");
          const float* ph = sm.pf_hist[it & 1][lane][0];
#pragma unroll
          for (int q = 0; q < kHist; ++q) {
            d.hist[rank][0][q] = ph[q];
            d.hist[rank][1][q] = ph[kHist + q];
          }
        } else if (t0 == 0) {
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
        d.out = span_out;
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
  pb::pdl_enter();
  const pb_fir_actor& a = actors[blockIdx.y];
  const int s = blockIdx.x;
  const int cnt = pb::cond_count(res, a.cond, s);
  if (cnt == 0 || threadIdx.x >= 2 * kHist) return;
  const int nl = pb::firing_iter(res, a.cond, s, cnt - 1);
  const float* in = reinterpret_cast<const float*>(pb::span_ptr(a.in, res, s, nl));
  const int plane = threadIdx.x / kHist, k = threadIdx.x % kHist;
  a.state[(int64_t)s * 2 * kHist + plane * kHist + k] = in[plane * B + B - kHist + k];
}


// ------------------------------------------------- PB_FIR_MERGED filter bank
// Tolerance mode of the fused bank as two plain data-parallel kernels: the
// bank is then an HBM-bound stencil (8 B read + 8 B written per sample, one
// 10-tap complex FMA FIR), with no producer warp on the critical path.
//   bank_plan_kernel: one warp per span (s, n): the active branches' taps
//     summed per tap, and the correction of outputs 0..8 for the pre-span
//     samples (each branch's own 9-sample history).
//   bank_merged_kernel: 8 consecutive outputs per thread, window straight
//     from global memory (neighbouring threads share it through L1).
struct __align__(16) BankPlan {
  float4 taps[kTaps];   // merged {cr, ci, ci, cr}
  float2 corr[kHist];   // added to outputs 0..8
  int have;             // the bank fires at (s, n)
  int pad_[3];
};

constexpr int kPlanWarps = 8;   // spans per block (one warp each)

__global__ void __launch_bounds__(32 * kPlanWarps)
bank_plan_kernel(pb_filter_bank bank, pb_resolved res, int64_t B, BankPlan* plan) {
  pb::pdl_enter();
  const int n = blockIdx.x * kPlanWarps + threadIdx.y, s = blockIdx.y, lane = threadIdx.x;
  if (n >= res.n_iter) return;
  BankPlan& p = plan[(int64_t)s * res.n_iter + n];
  if (!pb::active(res, bank.actor_cond, s, n)) {
    if (lane == 0) p.have = 0;
    return;
  }
  const pb_fir_actor* br = bank.branches;
  const int nb = bank.n_branches;
  // dynamic shared memory sized for this bank's branch count (more resident
  // warps than a kMaxBr-sized static array): per warp the taps and the
  // histories of its span
  extern __shared__ float4 plan_smem[];
  float4 (*taps)[kTaps] =
      reinterpret_cast<float4 (*)[kTaps]>(plan_smem + threadIdx.y * nb * (kTaps + 5));
  float (*hist)[2][kHist] = reinterpret_cast<float (*)[2][kHist]>(
      plan_smem + threadIdx.y * nb * (kTaps + 5) + nb * kTaps);
  for (int e = lane; e < nb * kTaps; e += 32) {
    const int b = e / kTaps, t = e % kTaps;
    const float cr = br[b].taps[t], ci = br[b].taps[kTaps + t];
    taps[b][t] = make_float4(cr, ci, ci, cr);
  }
  const bool act = lane < nb && pb::active(res, br[lane].cond, s, n);
  const unsigned mask = __ballot_sync(0xffffffffu, act);
  if (act) {
    const pb_fir_actor& fa = br[lane];
    const int j = fa.cond < 0 ? n : res.prefix[((int64_t)fa.cond * res.n_streams + s) * res.cap + n];
    const int src = j == 0 ? -1 : pb::firing_iter(res, fa.cond, s, j - 1);
    const float *hr, *hi;
    if (src < 0) {
      hr = fa.state + (int64_t)s * 2 * kHist;
      hi = hr + kHist;
    } else {
      const float* prev = reinterpret_cast<const float*>(pb::span_ptr(fa.in, res, s, src));
      hr = prev + B - kHist;
      hi = prev + 2 * B - kHist;
    }
#pragma unroll
    for (int q = 0; q < kHist; ++q) {
      hist[lane][0][q] = hr[q];
      hist[lane][1][q] = hi[q];
    }
  }
  __syncwarp();
  if (lane < kTaps) {
    float4 m = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int b = 0; b < nb; ++b)
      if ((mask >> b) & 1u) {
        const float4 c = taps[b][lane];
        m.x += c.x; m.y += c.y; m.z += c.z; m.w += c.w;
      }
    p.taps[lane] = m;
  }
  if (lane < kHist) {   // output `lane` reads pre-span sample lane - t for taps t > lane
    float cr = 0.f, ci = 0.f;
    for (int b = 0; b < nb; ++b) {
      if (!((mask >> b) & 1u)) continue;
      for (int t = lane + 1; t < kTaps; ++t) {
        const int q = lane - t + kHist;
        const float hr = hist[b][0][q], hi = hist[b][1][q];
        const float4 c = taps[b][t];
        cr = __fmaf_rn(-c.y, hi, __fmaf_rn(c.x, hr, cr));
        ci = __fmaf_rn(c.y, hr, __fmaf_rn(c.x, hi, ci));
      }
    }
    p.corr[lane] = make_float2(cr, ci);
  }
  if (lane == 0) p.have = 1;
}

// One block per stream: the whole epoch's plans at once.  Activity masks of
// every span go to shared memory, each branch's "previous firing" index is a
// warp max-scan over the spans, and every thread then plans one span: its
// branch histories are one independent load each (the bank's own input span
// at that firing -- the route copied the same samples to the branch), not a
// prefix -> worklist -> ring-base chain.  Used when the tables fit in 48 KB.
constexpr int kPlanStreamThreads = 256;

__host__ __device__ inline size_t plan_stream_smem(int n_iter, int nb) {
  return (size_t)n_iter * 4 + (size_t)n_iter + 15 + (size_t)nb * n_iter * 4 + (size_t)nb * kTaps * 16 + 16;
}

__global__ void __launch_bounds__(kPlanStreamThreads)
bank_plan_stream_kernel(pb_filter_bank bank, pb_resolved res, int64_t B, BankPlan* plan) {
  pb::pdl_enter();
  const int s = blockIdx.x, E = res.n_iter, tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const pb_fir_actor* br = bank.branches;
  const int nb = bank.n_branches;
  extern __shared__ float4 pss[];
  float4* taps = pss;                                            // [nb][kTaps]
  uint32_t* mask = reinterpret_cast<uint32_t*>(taps + nb * kTaps);   // [E]
  int* prev = reinterpret_cast<int*>(mask + E);                  // [nb][E]
  uint8_t* have = reinterpret_cast<uint8_t*>(prev + nb * E);     // [E]
  for (int e = tid; e < nb * kTaps; e += kPlanStreamThreads) {
    const int b = e / kTaps, t = e % kTaps;
    const float cr = br[b].taps[t], ci = br[b].taps[kTaps + t];
    taps[e] = make_float4(cr, ci, ci, cr);
  }
  for (int n = tid; n < E; n += kPlanStreamThreads) {
    const bool h = pb::active(res, bank.actor_cond, s, n);
    uint32_t m = 0;
    if (h)
      for (int b = 0; b < nb; ++b)
        if (pb::active(res, br[b].cond, s, n)) m |= 1u << b;
    mask[n] = m;
    have[n] = h;
  }
  __syncthreads();
  // previous firing of each branch before span n (exclusive max-scan)
  const int chunk = (E + 31) / 32;
  for (int b = warp; b < nb; b += kPlanStreamThreads / 32) {
    const int lo = lane * chunk, hi = min(E, lo + chunk);
    int last = -1;
    for (int n = lo; n < hi; ++n)
      if ((mask[n] >> b) & 1u) last = n;
    int carry = last;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, carry, d);
      if (lane >= d) carry = max(carry, o);
    }
    int cur = __shfl_up_sync(0xffffffffu, carry, 1);
    if (lane == 0) cur = -1;
    for (int n = lo; n < hi; ++n) {
      prev[b * E + n] = cur;
      if ((mask[n] >> b) & 1u) cur = n;
    }
  }
  __syncthreads();
  for (int n = tid; n < E; n += kPlanStreamThreads) {
    BankPlan& p = plan[(int64_t)s * E + n];
    if (!have[n]) {
      p.have = 0;
      continue;
    }
    const uint32_t m = mask[n];
    float4 mt[kTaps];
#pragma unroll
    for (int t = 0; t < kTaps; ++t) mt[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    float cr[kHist], ci[kHist];
#pragma unroll
    for (int k = 0; k < kHist; ++k) cr[k] = ci[k] = 0.f;
    for (int b = 0; b < nb; ++b) {
      if (!((m >> b) & 1u)) continue;
      const int src = prev[b * E + n];
      const float *hr, *hi;
      if (src < 0) {
        hr = br[b].state + (int64_t)s * 2 * kHist;
        hi = hr + kHist;
      } else {
        const float* pv = reinterpret_cast<const float*>(pb::span_ptr(bank.in, res, s, src));
        hr = pv + B - kHist;
        hi = pv + 2 * B - kHist;
      }
      float h_r[kHist], h_i[kHist];
#pragma unroll
      for (int q = 0; q < kHist; ++q) {
        h_r[q] = hr[q];
        h_i[q] = hi[q];
      }
      const float4* tb = taps + b * kTaps;
#pragma unroll
      for (int t = 0; t < kTaps; ++t) {
        const float4 c = tb[t];
        mt[t].x += c.x; mt[t].y += c.y; mt[t].z += c.z; mt[t].w += c.w;
      }
      // output k reads pre-span sample k - t (history slot k - t + 9) for t > k
#pragma unroll
      for (int k = 0; k < kHist; ++k)
#pragma unroll
        for (int t = k + 1; t < kTaps; ++t) {
          const float4 c = tb[t];
          const float xr = h_r[k - t + kHist], xi = h_i[k - t + kHist];
          cr[k] = __fmaf_rn(-c.y, xi, __fmaf_rn(c.x, xr, cr[k]));
          ci[k] = __fmaf_rn(c.y, xr, __fmaf_rn(c.x, xi, ci[k]));
        }
    }
#pragma unroll
    for (int t = 0; t < kTaps; ++t) p.taps[t] = mt[t];
#pragma unroll
    for (int k = 0; k < kHist; ++k) p.corr[k] = make_float2(cr[k], ci[k]);
    p.have = 1;
  }
}

// Chunk-parallel planner: block (s, c) plans spans [c*kPC, (c+1)*kPC) of
// stream s.  The activity masks of spans 0..hi-1 (one byte load per
// condition, all independent) and each branch's previous-firing max-scan are
// recomputed per block -- cheap -- so the epoch is planned by
// n_streams * E / kPC blocks instead of n_streams, and every dependent load
// of a span's plan is issued at once: the branch histories are gathered into
// shared memory by a flat (span, branch, sample) loop in one round trip, then
// merged taps and corrections are one thread per (span, tap | output).
#ifndef PB_PLAN_PAR
#define PB_PLAN_PAR 1
#endif
#ifndef PB_PLAN_TAILS
#define PB_PLAN_TAILS 1
#endif
#ifndef PB_PLAN_PREFIX   // previous firings from the resolution's prefix / worklist
#define PB_PLAN_PREFIX 1
#endif
#ifndef PB_PLAN_STOP   // profiling: end the planner after phase 1/2/3
#define PB_PLAN_STOP 0
#endif
#ifndef PB_PLAN_PC
#define PB_PLAN_PC 64
#endif
constexpr int kPC = PB_PLAN_PC;         // spans per block
constexpr int kPlanParThreads = 256;

__host__ __device__ inline size_t plan_par_smem(int n_iter, int nb) {
  return (size_t)nb * kTaps * 16                 // taps
         + (size_t)kPC * nb * 8                  // history source pointers
         + (size_t)kPC * nb * 2 * kHist * 4      // hist
         + (size_t)n_iter * 4                    // mask
         + (size_t)nb * kPC * 4                  // prev
         + (size_t)((n_iter + 15) & ~15);        // have
}
// kTails: the 48-byte aligned tail window (last 12 samples) of both planes of
// the spans [lo - kTailWin, hi), and the branch states
constexpr int kTailWin = 32;                      // spans before the chunk with staged tails
constexpr int kTailF = 12;                        // floats per plane window (16-B multiple)
__host__ __device__ inline size_t plan_par_tails_smem(int n_iter, int nb) {
  return plan_par_smem(n_iter, nb) + 16 + (size_t)(kPC + kTailWin) * 2 * kTailF * 4 +
         (size_t)nb * 2 * kHist * 4;
}

// kTails: every span tail of the stream's spans 0..hi-1 (and each branch's
// carried state) is requested at kernel start, before the activity masks and
// the scan are known -- a branch's history is the tail of the bank input at
// its previous firing, the same bytes for every branch -- so the gather's
// round trip overlaps phases 1-2 instead of following them.
#ifndef PB_PLAN_QUAD   // 1: four threads per span in phase 4 (measured 0.2072 vs 0.2064 ms per
#define PB_PLAN_QUAD 0    // C2 step: the one-thread form stays the default)
#endif

// One quarter of the plans of a block's spans (bank_plan_par_kernel phase 4):
// merged taps t and corrections k with t % 4 == k % 4 == PART, every sum in the
// order of the one-thread-per-span form.
template <int PART, bool kTails>
__device__ __forceinline__ void plan_part(const pb_filter_bank& bank, const pb_resolved& res,
                                          int64_t B, BankPlan* plan, int s, int E, int lo, int np,
                                          int i0, int nb, const float4* taps, const float* hist,
                                          const uint32_t* mask, const int* prev,
                                          const uint8_t* have, const float* tails,
                                          const float* stails, int t0, int64_t in_base) {
  constexpr int NT = (kTaps - PART + 3) / 4, NK = (kHist - PART + 3) / 4;
  for (int i = i0; i < np; i += kPlanParThreads / 4) {
    const int n = lo + i;
    BankPlan& p = plan[(int64_t)s * E + n];
    if (!have[n]) {
      if (PART == 0) p.have = 0;
      continue;
    }
    const uint32_t m = mask[n];
    float4 mt[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) mt[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    float cr[NK], ci[NK];
#pragma unroll
    for (int j = 0; j < NK; ++j) cr[j] = ci[j] = 0.f;
    for (int b = 0; b < nb; ++b) {
      if (!((m >> b) & 1u)) continue;
      const int pv = prev[b * kPC + i];
      float h_r[kHist], h_i[kHist];
      if (!kTails) {
        const float* h = hist + (i * nb + b) * 2 * kHist;
#pragma unroll
        for (int q = 0; q < kHist; ++q) {
          h_r[q] = h[q];
          h_i[q] = h[kHist + q];
        }
      } else if (pv < 0) {
        const float* h = stails + b * 2 * kHist;
#pragma unroll
        for (int q = 0; q < kHist; ++q) {
          h_r[q] = h[q];
          h_i[q] = h[kHist + q];
        }
      } else if (pv >= t0) {
        const float* h = tails + (pv - t0) * 2 * kTailF;
#pragma unroll
        for (int q = 0; q < kHist; ++q) {
          h_r[q] = h[kTailF - kHist + q];
          h_i[q] = h[kTailF + kTailF - kHist + q];
        }
      } else {
        const float* pvp = reinterpret_cast<const float*>(span_ptr_b(bank.in, in_base, res, s, pv));
#pragma unroll
        for (int q = 0; q < kHist; ++q) {
          h_r[q] = pvp[B - kHist + q];
          h_i[q] = pvp[2 * B - kHist + q];
        }
      }
      const float4* tb = taps + b * kTaps;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const float4 c = tb[PART + 4 * j];
        mt[j].x += c.x; mt[j].y += c.y; mt[j].z += c.z; mt[j].w += c.w;
      }
#pragma unroll
      for (int j = 0; j < NK; ++j) {
        constexpr int dummy = 0;
        (void)dummy;
        const int k = PART + 4 * j;
#pragma unroll
        for (int t = k + 1; t < kTaps; ++t) {
          const float4 c = tb[t];
          const float xr = h_r[k - t + kHist], xi = h_i[k - t + kHist];
          cr[j] = __fmaf_rn(-c.y, xi, __fmaf_rn(c.x, xr, cr[j]));
          ci[j] = __fmaf_rn(c.y, xr, __fmaf_rn(c.x, xi, ci[j]));
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) p.taps[PART + 4 * j] = mt[j];
#pragma unroll
    for (int j = 0; j < NK; ++j) p.corr[PART + 4 * j] = make_float2(cr[j], ci[j]);
    if (PART == 0) p.have = 1;
  }
}

template <bool kTails>
__global__ void __launch_bounds__(kPlanParThreads)
bank_plan_par_kernel(pb_filter_bank bank, pb_resolved res, int64_t B, BankPlan* plan) {
  pb::pdl_enter();
  const int s = blockIdx.x, E = res.n_iter, tid = threadIdx.x;
  const int lo = blockIdx.y * kPC, hi = min(E, lo + kPC), np = hi - lo;
  const int warp = tid >> 5, lane = tid & 31;
  const pb_fir_actor* br = bank.branches;
  const int nb = bank.n_branches;
  extern __shared__ float4 ppar[];
  float4* taps = ppar;                                                  // [nb][kTaps]
  const float** hsrc = reinterpret_cast<const float**>(taps + nb * kTaps);   // [kPC][nb]
  float* hist = reinterpret_cast<float*>(hsrc + kPC * nb);             // [kPC][nb][2][kHist]
  uint32_t* mask = reinterpret_cast<uint32_t*>(hist + kPC * nb * 2 * kHist);  // [hi]
  int* prev = reinterpret_cast<int*>(mask + E);                         // [nb][kPC]
  uint8_t* have = reinterpret_cast<uint8_t*>(prev + nb * kPC);          // [hi]
  const int64_t in_base = bank.in.base ? bank.in.base[s] : 0;
  // kTails layout: tails[t0 .. hi)[2][kTailF] (16-byte copies of each plane's
  // last 12 samples; the history is samples 3..11), then the states [nb][2][kHist]
  const int t0 = max(0, lo - kTailWin);
  float* tails = reinterpret_cast<float*>(
      (reinterpret_cast<uintptr_t>(have + E) + 15) & ~uintptr_t(15));   // 16-B copies
  float* stails = tails + (size_t)(kPC + kTailWin) * 2 * kTailF;
  if (kTails) {
    const int nt = hi - t0;
    for (int e = tid; e < nt * 6; e += kPlanParThreads) {   // 2 planes x 3 x 16 B per span
      const int t = e / 6, r = e - t * 6, plane = r / 3, part = r - plane * 3;
      const float* src = reinterpret_cast<const float*>(span_ptr_b(bank.in, in_base, res, s, t0 + t)) +
                         plane * B + B - kTailF + 4 * part;
      cp_async16_plan(tails + (t * 2 + plane) * kTailF + 4 * part, src);
    }
    for (int e = tid; e < nb * 2 * kHist; e += kPlanParThreads)
      cp_async4(stails + e, br[e / (2 * kHist)].state + (int64_t)s * 2 * kHist + e % (2 * kHist));
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // 1. taps and activity masks: every load of a thread issued before use
  for (int e = tid; e < nb * kTaps; e += kPlanParThreads) {
    const int b = e / kTaps, t = e % kTaps;
    const float* tp = br[b].taps;
    const float cr = tp[t], ci = tp[kTaps + t];
    taps[e] = make_float4(cr, ci, ci, cr);
  }
  if (PB_PLAN_PREFIX && kTails && bank.actor_cond < 0) {
    // 1-2 from the resolution: per (span of this chunk, branch) the activity
    // and the previous firing (worklist[prefix - 1]), two dependent loads, no
    // mask walk over [0, hi) and no scan
    for (int n = lo + tid; n < hi; n += kPlanParThreads) {
      mask[n] = 0u;
      have[n] = 1;
    }
    __syncthreads();
    for (int e = tid; e < np * nb; e += kPlanParThreads) {
      const int i = e / nb, b = e - i * nb, n = lo + i;
      const int c = br[b].cond;
      bool act = true;
      int pv = n - 1;   // a branch without its own condition fires every iteration
      if (c >= 0) {
        const int64_t row = ((int64_t)c * res.n_streams + s) * res.cap;
        act = res.act[row + n] != 0;
        const int j = res.prefix[row + n];
        pv = j == 0 ? -1 : res.worklist[row + j - 1];
      }
      prev[b * kPC + i] = pv;
      if (act) atomicOr(&mask[n], 1u << b);
    }
    __syncthreads();
  } else {
  for (int n = tid; n < hi; n += kPlanParThreads) {
      const int64_t col = (int64_t)s * res.cap + n;
      const int64_t stride = (int64_t)res.n_streams * res.cap;
      uint8_t a[kMaxBr];
  #pragma unroll
      for (int b = 0; b < kMaxBr; ++b) {
        const int c = b < nb ? br[b].cond : -1;
        a[b] = c < 0 ? 1 : res.act[c * stride + col];
      }
      const bool h = bank.actor_cond < 0 || res.act[bank.actor_cond * stride + col];
      uint32_t m = 0;
  #pragma unroll
      for (int b = 0; b < kMaxBr; ++b)
        if (b < nb && a[b]) m |= 1u << b;
      mask[n] = h ? m : 0u;
      have[n] = h;
    }
    __syncthreads();
  #if PB_PLAN_STOP == 1
    return;
  #endif
    // 2. previous firing of each branch before span n, n in [lo, hi): warp
    //    max-scan over [0, hi)
    const int chunk = (hi + 31) / 32;
    for (int b = warp; b < nb; b += kPlanParThreads / 32) {
      const int a0 = lane * chunk, a1 = min(hi, a0 + chunk);
      int last = -1;
      for (int n = a0; n < a1; ++n)
        if ((mask[n] >> b) & 1u) last = n;
      int carry = last;
  #pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, carry, d);
        if (lane >= d) carry = max(carry, o);
      }
      int cur = __shfl_up_sync(0xffffffffu, carry, 1);
      if (lane == 0) cur = -1;
      for (int n = a0; n < a1; ++n) {
        if (n >= lo) prev[b * kPC + n - lo] = cur;
        if ((mask[n] >> b) & 1u) cur = n;
      }
    }
    __syncthreads();
  }
#if PB_PLAN_STOP == 2
  return;
#endif
  // 3. history sources (one pointer per active (span, branch)), then every
  //    history sample in flight at once (cp.async into shared memory)
  if (kTails) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
  } else {
    for (int e = tid; e < np * nb; e += kPlanParThreads) {
      const int i = e / nb, b = e - i * nb;
      const int src = prev[b * kPC + i];
      const float* p = nullptr;
      if ((mask[lo + i] >> b) & 1u) {
        if (src < 0)   // first firing of the branch: its carried state [2][kHist]
          p = br[b].state + (int64_t)s * 2 * kHist;
        else           // re plane tail; the im plane tail is p + B
          p = reinterpret_cast<const float*>(span_ptr_b(bank.in, in_base, res, s, src)) + B - kHist;
      }
      hsrc[e] = p;
    }
    __syncthreads();
    for (int e = tid; e < np * nb * 2 * kHist; e += kPlanParThreads) {
      const int ib = e / (2 * kHist), q = e - ib * 2 * kHist;
      const float* p = hsrc[ib];
      if (!p) continue;
      const int b = ib % nb, i = ib / nb;
      const bool state = prev[b * kPC + i] < 0;
      const int plane = q / kHist, kk = q - plane * kHist;
      cp_async4(hist + e, p + (state ? q : plane * B + kk));
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
  }
#if PB_PLAN_STOP == 3
  return;
#endif
  // 4. the span plans.  PB_PLAN_QUAD: four threads per span, warp w taking
  //    part w % 4 -- merged taps t and corrections k with t, k = part (mod 4)
  //    (the same sums in the same order as one thread per span, so the same
  //    plan); otherwise one thread per span, everything fully unrolled.
#if PB_PLAN_QUAD
  {
    const int part = warp & 3;
    const int i0 = (warp >> 2) * 32 + lane;
    switch (part) {
      case 0: plan_part<0, kTails>(bank, res, B, plan, s, E, lo, np, i0, nb, taps, hist, mask, prev, have, tails, stails, t0, in_base); break;
      case 1: plan_part<1, kTails>(bank, res, B, plan, s, E, lo, np, i0, nb, taps, hist, mask, prev, have, tails, stails, t0, in_base); break;
      case 2: plan_part<2, kTails>(bank, res, B, plan, s, E, lo, np, i0, nb, taps, hist, mask, prev, have, tails, stails, t0, in_base); break;
      default: plan_part<3, kTails>(bank, res, B, plan, s, E, lo, np, i0, nb, taps, hist, mask, prev, have, tails, stails, t0, in_base); break;
    }
  }
#else
  for (int i = tid; i < np; i += kPlanParThreads) {
    const int n = lo + i;
    BankPlan& p = plan[(int64_t)s * E + n];
    if (!have[n]) {
      p.have = 0;
      continue;
    }
    const uint32_t m = mask[n];
    float4 mt[kTaps];
#pragma unroll
    for (int t = 0; t < kTaps; ++t) mt[t] = make_float4(0.f, 0.f, 0.f, 0.f);
    float cr[kHist], ci[kHist];
#pragma unroll
    for (int k = 0; k < kHist; ++k) cr[k] = ci[k] = 0.f;
    for (int b = 0; b < nb; ++b) {
      if (!((m >> b) & 1u)) continue;
      const int pv = prev[b * kPC + i];
      float h_r[kHist], h_i[kHist];
      if (!kTails) {
        const float* h = hist + (i * nb + b) * 2 * kHist;
#pragma unroll
        for (int q = 0; q < kHist; ++q) {
          h_r[q] = h[q];
          h_i[q] = h[kHist + q];
        }
      } else if (pv < 0) {   // first firing of the branch: its carried state
        const float* h = stails + b * 2 * kHist;
#pragma unroll
        for (int q = 0; q < kHist; ++q) {
          h_r[q] = h[q];
          h_i[q] = h[kHist + q];
        }
      } else if (pv >= t0) {   // a staged tail window: samples 3..11
        const float* h = tails + (pv - t0) * 2 * kTailF;
#pragma unroll
        for (int q = 0; q < kHist; ++q) {
          h_r[q] = h[kTailF - kHist + q];
          h_i[q] = h[kTailF + kTailF - kHist + q];
        }
      } else {   // a firing further back than the window: straight from the ring
        const float* pvp = reinterpret_cast<const float*>(span_ptr_b(bank.in, in_base, res, s, pv));
#pragma unroll
        for (int q = 0; q < kHist; ++q) {
          h_r[q] = pvp[B - kHist + q];
          h_i[q] = pvp[2 * B - kHist + q];
        }
      }
      const float4* tb = taps + b * kTaps;
#pragma unroll
      for (int t = 0; t < kTaps; ++t) {
        const float4 c = tb[t];
        mt[t].x += c.x; mt[t].y += c.y; mt[t].z += c.z; mt[t].w += c.w;
      }
      // output k reads pre-span sample k - t (history slot k - t + 9) for t > k
#pragma unroll
      for (int k = 0; k < kHist; ++k)
#pragma unroll
        for (int t = k + 1; t < kTaps; ++t) {
          const float4 c = tb[t];
          const float xr = h_r[k - t + kHist], xi = h_i[k - t + kHist];
          cr[k] = __fmaf_rn(-c.y, xi, __fmaf_rn(c.x, xr, cr[k]));
          ci[k] = __fmaf_rn(c.y, xr, __fmaf_rn(c.x, xi, ci[k]));
        }
    }
#pragma unroll
    for (int t = 0; t < kTaps; ++t) p.taps[t] = mt[t];
#pragma unroll
    for (int k = 0; k < kHist; ++k) p.corr[k] = make_float2(cr[k], ci[k]);
    p.have = 1;
  }
#endif
}

#ifndef PB_MERGED_PT
#define PB_MERGED_PT 8
#endif
#ifndef PB_MERGED_MINB
#define PB_MERGED_MINB 4
#endif
#ifndef PB_MERGED_STREAMING   // 1: evict-first loads, 2: + streaming stores
#define PB_MERGED_STREAMING 2
#endif

constexpr int kMergedThreads = 256;
constexpr int kMPT = PB_MERGED_PT;             // outputs per thread
constexpr int kMWin = kMPT + kPad;             // window (samples)

__global__ void __launch_bounds__(kMergedThreads, PB_MERGED_MINB)
bank_merged_kernel(pb_filter_bank bank, pb_resolved res, int64_t B, const BankPlan* plan,
                   int blocks_per_span) {
  pb::pdl_enter();
  const int64_t span = blockIdx.x / blocks_per_span;
  const int part = (int)(blockIdx.x % blocks_per_span);
  const int s = (int)(span / res.n_iter), n = (int)(span % res.n_iter);
  __shared__ BankPlan sp;
  // the window loads go out before the plan is known (an inactive span's
  // input is still valid ring memory), so the block's start-up costs one
  // memory round trip, not two
  const float* in = reinterpret_cast<const float*>(pb::span_ptr(bank.in, res, s, n));
  if (threadIdx.x < (int)(sizeof(BankPlan) / 16))
    reinterpret_cast<uint4*>(&sp)[threadIdx.x] =
        __ldg(reinterpret_cast<const uint4*>(plan + span) + threadIdx.x);
  const int64_t n0 = ((int64_t)part * kMergedThreads + threadIdx.x) * kMPT;
  const bool live = n0 < B;
  float wr[kMWin], wi[kMWin];
#pragma unroll
  for (int k = 0; k < kMWin / 4; ++k) {
    const int64_t idx = n0 - kPad + 4 * k;   // multiple of 4: all-or-nothing pre-span
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
    if (live && idx >= 0) {
#if PB_MERGED_STREAMING
      a = __ldcs(reinterpret_cast<const float4*>(in + idx));
      b = __ldcs(reinterpret_cast<const float4*>(in + B + idx));
#else
      a = __ldg(reinterpret_cast<const float4*>(in + idx));
      b = __ldg(reinterpret_cast<const float4*>(in + B + idx));
#endif
    }
    wr[4 * k] = a.x; wr[4 * k + 1] = a.y; wr[4 * k + 2] = a.z; wr[4 * k + 3] = a.w;
    wi[4 * k] = b.x; wi[4 * k + 1] = b.y; wi[4 * k + 2] = b.z; wi[4 * k + 3] = b.w;
  }
  __syncthreads();
  if (!sp.have || !live) return;
  float* out = reinterpret_cast<float*>(pb::span_ptr(bank.out, res, s, n));
  float yr[kMPT], yi[kMPT];
#pragma unroll
  for (int v = 0; v < kMPT; ++v) yr[v] = yi[v] = 0.0f;
#ifdef PB_MERGED_COPYONLY   // profiling variant: memory traffic without the FIR
#pragma unroll
  for (int v = 0; v < kMPT; ++v) { yr[v] = wr[kPad + v]; yi[v] = wi[kPad + v]; }
  if (0)
#endif
#pragma unroll
  for (int t = 0; t < kTaps; ++t) {
    const float4 c = sp.taps[t];
#pragma unroll
    for (int v = 0; v < kMPT; ++v) {
      const float xr = wr[kPad + v - t], xi = wi[kPad + v - t];
      yr[v] = __fmaf_rn(-c.y, xi, __fmaf_rn(c.x, xr, yr[v]));
      yi[v] = __fmaf_rn(c.y, xr, __fmaf_rn(c.x, xi, yi[v]));
    }
  }
  if (n0 < kHist) {
#pragma unroll
    for (int v = 0; v < kMPT; ++v)
      if (n0 + v < kHist) {
        yr[v] += sp.corr[n0 + v].x;
        yi[v] += sp.corr[n0 + v].y;
      }
  }
  float4* orr = reinterpret_cast<float4*>(out + n0);
  float4* oi = reinterpret_cast<float4*>(out + B + n0);
#pragma unroll
  for (int k = 0; k < kMPT / 4; ++k) {
#if PB_MERGED_STREAMING >= 2
    __stcs(orr + k, make_float4(yr[4 * k], yr[4 * k + 1], yr[4 * k + 2], yr[4 * k + 3]));
    __stcs(oi + k, make_float4(yi[4 * k], yi[4 * k + 1], yi[4 * k + 2], yi[4 * k + 3]));
#else
    orr[k] = make_float4(yr[4 * k], yr[4 * k + 1], yr[4 * k + 2], yr[4 * k + 3]);
    oi[k] = make_float4(yi[4 * k], yi[4 * k + 1], yi[4 * k + 2], yi[4 * k + 3]);
#endif
  }
}

// Persistent form of the merged stencil: one CTA per SM slot walks a
// contiguous range of (span, tile) items.  A producer warp streams each
// tile's two sample planes (with the 12-sample halo from the same span) and
// the span's BankPlan into a shared-memory stage with cp.async.bulk, kMSStages
// tiles ahead; the consumer warps read their 20-sample windows from shared
// memory, run the merged FIR and store straight to the output span.  Memory
// requests therefore never wait on the FMA work, and the span addressing
// (ring index arithmetic) runs once per 2048-sample tile in the producer
// instead of once per thread.
#ifndef PB_MS_WARPS
#define PB_MS_WARPS 4
#endif
#ifndef PB_MS_EARLY   // 1: the first stages' input tiles load while the planner runs
#define PB_MS_EARLY 0    // (measured 0.2075 vs 0.2052 ms per C2 step: not adopted)
#endif
#ifndef PB_MS_CARRY   // 1: the stream kernel also carries the branch histories
#define PB_MS_CARRY 1
#endif
#ifndef PB_MS_L2HINT   // input planes are read once: evict-first in L2
#define PB_MS_L2HINT 1
#endif
#ifndef PB_MS_STAGES
#define PB_MS_STAGES 5
#endif
constexpr int kMSWarps = PB_MS_WARPS;
constexpr int kMSThreads = 32 * (kMSWarps + 1);
#ifndef PB_MS_PASSES   // consumer passes per tile (8 outputs per thread each)
#define PB_MS_PASSES 2
#endif
constexpr int kMSPass = 32 * kMSWarps * kPerThread;   // samples per consumer pass
constexpr int kMSTile = kMSPass * PB_MS_PASSES;       // samples per item
constexpr int kMSStages = PB_MS_STAGES;

struct __align__(16) MSStage {
  BankPlan plan;
  float re[kPad + kMSTile];
  float im[kPad + kMSTile];
};
struct __align__(16) MSSmem {
  MSStage st[kMSStages];
  u64 out[kMSStages];   // output span base of the staged tile
  int t0[kMSStages];    // its first sample
  u64 full[kMSStages];
  u64 empty[kMSStages];
};
static_assert(sizeof(BankPlan) % 16 == 0, "BankPlan is bulk-copied");

#ifndef PB_MS_MINB
#define PB_MS_MINB 1
#endif
__global__ void __launch_bounds__(kMSThreads, PB_MS_MINB)
bank_stream_kernel(pb_filter_bank bank, pb_resolved res, int64_t B, const BankPlan* plan,
                   int tiles) {
  // PDL: this grid may start while the planner (its predecessor) still runs.
  // Everything before the planner has completed by then (the planner waited
  // for it before it let this grid launch), so the input spans are final and
  // the output spans free; only the plans and the carried states the planner
  // reads need the planner's completion (griddepcontrol.wait below).
#if PB_MS_EARLY
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#else
  pb::pdl_enter();
#endif
  extern __shared__ __align__(128) uint8_t ms_raw[];
  MSSmem& sm = *reinterpret_cast<MSSmem*>(ms_raw);
  if (threadIdx.x == 0) {
    for (int k = 0; k < kMSStages; ++k) {
      mbar_init(&sm.full[k], 1);
      mbar_init(&sm.empty[k], kMSWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t total = (int64_t)res.n_streams * res.n_iter * tiles;
  // a contiguous item range per CTA (measured faster than interleaving the
  // CTAs over neighbouring tiles: 75% vs 66% of the HBM roofline)
  const int64_t w0 = total * blockIdx.x / gridDim.x;
  const int64_t n_items = total * (blockIdx.x + 1) / gridDim.x - w0;
  const int warp = threadIdx.x >> 5;

  if (warp == kMSWarps) {
    if ((threadIdx.x & 31) != 0) {
#if PB_MS_CARRY
      // lanes 1..18 of the producer warp: the history carry of this CTA's
      // (stream, branch) items -- state <- the last 9 input samples of the
      // branch's last firing this epoch (fir_carry_kernel's work; the planner
      // that reads the old state has completed before this grid started)
      const int q = (threadIdx.x & 31) - 1;
      asm volatile("griddepcontrol.wait;" ::: "memory");   // the planner read the old state
      if (q < 2 * kHist) {
        const int nb = bank.n_branches, plane = q / kHist, k = q - plane * kHist;
        for (int64_t i = blockIdx.x; i < (int64_t)res.n_streams * nb; i += gridDim.x) {
          const int s = (int)(i / nb);
          const pb_fir_actor& fa = bank.branches[i - (int64_t)s * nb];
          const int cnt = pb::cond_count(res, fa.cond, s);
          if (cnt == 0) continue;
          const int nl = pb::firing_iter(res, fa.cond, s, cnt - 1);
          const float* in = reinterpret_cast<const float*>(pb::span_ptr(fa.in, res, s, nl));
          fa.state[(int64_t)s * 2 * kHist + plane * kHist + k] = in[plane * B + B - kHist + k];
        }
      }
#endif
      return;
    }
    // ------------------------------------------------------------ producer
#if PB_MS_L2HINT
    u64 pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
    int64_t span = w0 / tiles;
    int tile = (int)(w0 - span * tiles) - 1;
    const float* in = nullptr;
    u64 out = 0;
    // the first ring's worth of tiles streams in before the planner finished;
    // their plans follow once it has (the stage barriers count both)
    const int64_t pre = !PB_MS_EARLY ? 0 : n_items < kMSStages ? n_items : kMSStages;
    if (pre == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int64_t k = 0; k < n_items; ++k) {
      if (k == 0 || ++tile == tiles) {   // (next) span: its ring addresses
        if (k > 0) {
          tile = 0;
          ++span;
        } else {
          ++tile;
        }
        const int s = (int)(span / res.n_iter), n = (int)(span - (int64_t)s * res.n_iter);
        in = reinterpret_cast<const float*>(pb::span_ptr(bank.in, res, s, n));
        out = reinterpret_cast<u64>(pb::span_ptr(bank.out, res, s, n));
      }
      const int stage = (int)(k % kMSStages);
      mbar_wait(&sm.empty[stage], (uint32_t)(((k / kMSStages) & 1) ^ 1));
      MSStage& sb = sm.st[stage];
      const int64_t t0 = (int64_t)tile * kMSTile;
      const int64_t rem = B - t0;
      const int len = (int)(rem < kMSTile ? rem : kMSTile);
      const int lead = t0 > 0 ? kPad : 0;   // tile > 0: halo from the same span
      const uint32_t bytes = (uint32_t)(len + lead) * 4u;
      sm.out[stage] = out;
      sm.t0[stage] = (int)t0;
      mbar_arrive_tx(&sm.full[stage], 2 * bytes + (uint32_t)sizeof(BankPlan));
      if (k >= pre) bulk_g2s(&sb.plan, plan + span, (uint32_t)sizeof(BankPlan), &sm.full[stage]);
#if PB_MS_L2HINT
      bulk_g2s_hint(sb.re + kPad - lead, in + t0 - lead, bytes, &sm.full[stage], pol);
      bulk_g2s_hint(sb.im + kPad - lead, in + B + t0 - lead, bytes, &sm.full[stage], pol);
#else
      bulk_g2s(sb.re + kPad - lead, in + t0 - lead, bytes, &sm.full[stage]);
      bulk_g2s(sb.im + kPad - lead, in + B + t0 - lead, bytes, &sm.full[stage]);
#endif
      if (k == pre - 1) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        for (int64_t j = 0; j < pre; ++j)
          bulk_g2s(&sm.st[j].plan, plan + (w0 + j) / tiles, (uint32_t)sizeof(BankPlan),
                   &sm.full[j]);
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int ct = threadIdx.x;   // 0 .. 32*kMSWarps-1
  for (int64_t k = 0; k < n_items; ++k) {
    const int stage = (int)(k % kMSStages);
    mbar_wait(&sm.full[stage], (uint32_t)((k / kMSStages) & 1));
    const MSStage& sb = sm.st[stage];
    const int64_t t0 = sm.t0[stage];
#pragma unroll 1
    for (int pass = 0; pass < PB_MS_PASSES; ++pass) {
    const int off = pass * kMSPass + kPerThread * ct;   // first output, relative to t0
    const int64_t n0 = t0 + off;
    if (sb.plan.have && n0 < B) {
      float wr[kWin], wi[kWin];
      {
        const float4* a = reinterpret_cast<const float4*>(sb.re + off);
        const float4* b = reinterpret_cast<const float4*>(sb.im + off);
#pragma unroll
        for (int q = 0; q < kWin / 4; ++q) {
          const float4 x = a[q], z = b[q];
          wr[4 * q + 0] = x.x; wr[4 * q + 1] = x.y; wr[4 * q + 2] = x.z; wr[4 * q + 3] = x.w;
          wi[4 * q + 0] = z.x; wi[4 * q + 1] = z.y; wi[4 * q + 2] = z.z; wi[4 * q + 3] = z.w;
        }
      }
      const bool patch = n0 < kPad;   // pre-span samples: zero here, history in corr
      if (patch) {
#pragma unroll
        for (int i = 0; i < kPad; ++i)
          if (n0 - kPad + i < 0) wr[i] = wi[i] = 0.0f;
      }
      u64 y[kPerThread];
#ifdef PB_MS_COPYONLY   // profiling variant: the memory pipeline without the FIR
#pragma unroll
      for (int v = 0; v < kPerThread; ++v) y[v] = pack2(wr[kPad + v], wi[kPad + v]);
#else
      fir8_fma(wr, wi, sb.plan.taps, y);
#endif
      if (patch) {
#pragma unroll
        for (int v = 0; v < kPerThread; ++v)
          if (n0 + v < kHist) {
            float yr, yi;
            unpack2(y[v], yr, yi);
            y[v] = pack2(yr + sb.plan.corr[n0 + v].x, yi + sb.plan.corr[n0 + v].y);
          }
      }
      store8(reinterpret_cast<float*>(sm.out[stage]), B, (int)n0, y);
    }
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&sm.empty[stage]);
  }
}

#ifndef PB_MERGED_STREAM
#define PB_MERGED_STREAM 1
#endif

int launch_merged_bank(const pb_filter_bank& bank, const pb_resolved& res, int64_t B,
                       cudaStream_t st) {
  const int64_t spans = (int64_t)res.n_streams * res.n_iter;
  BankPlan* plan = nullptr;
  int rc = pb::scratch(pb::kScratchBankPlan, sizeof(BankPlan) * spans,
                       reinterpret_cast<void**>(&plan));
  if (rc) return rc;
  const int dev = pb::device();
  if (dev < 0) return PB_E_CUDA;
  dim3 pgrid((res.n_iter + kPlanWarps - 1) / kPlanWarps, res.n_streams);
  const size_t ssmem = plan_stream_smem(res.n_iter, bank.n_branches);
  const size_t parsmem = plan_par_smem(res.n_iter, bank.n_branches);
  const size_t tailsmem = plan_par_tails_smem(res.n_iter, bank.n_branches);
  if (PB_PLAN_PAR && PB_PLAN_TAILS && tailsmem <= 48 * 1024) {
    dim3 g(res.n_streams, (res.n_iter + kPC - 1) / kPC);
    PB_LAUNCH_PDL(bank_plan_par_kernel<true>, g, kPlanParThreads, tailsmem, st, bank, res, B, plan);
  } else if (PB_PLAN_PAR && parsmem <= 48 * 1024) {
    dim3 g(res.n_streams, (res.n_iter + kPC - 1) / kPC);
    PB_LAUNCH_PDL(bank_plan_par_kernel<false>, g, kPlanParThreads, parsmem, st, bank, res, B, plan);
  } else if (ssmem <= 48 * 1024) {
    PB_LAUNCH_PDL(bank_plan_stream_kernel, res.n_streams, kPlanStreamThreads, ssmem, st, bank, res, B, plan);
  } else {
    // per warp: nb x kTaps float4 taps + nb x 2 x kHist histories (<= 5 float4 per branch)
    const size_t psmem = sizeof(float4) * kPlanWarps * bank.n_branches * (kTaps + 5);
    PB_LAUNCH_PDL(bank_plan_kernel, pgrid, dim3(32, kPlanWarps), psmem, st, bank, res, B, plan);
  }
  PB_LAUNCHED("bank_plan_kernel");
  if (PB_MERGED_STREAM) {
    const int tiles = (int)((B + kMSTile - 1) / kMSTile);
    const size_t smem = sizeof(MSSmem);
    static int sms_d[pb::kMaxDevices] = {}, per_sm_d[pb::kMaxDevices] = {};
    int& sms = sms_d[dev];
    int& per_sm = per_sm_d[dev];
    if (sms == 0) {
      PB_CUDA(cudaFuncSetAttribute(bank_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
      PB_CUDA(cudaFuncSetAttribute(bank_stream_kernel,
                                   cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      PB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      PB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bank_stream_kernel,
                                                            kMSThreads, smem));
      per_sm = std::max(per_sm, 1);
    }
    const int64_t items = spans * tiles;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)sms * per_sm));
    PB_LAUNCH_PDL(bank_stream_kernel, grid, kMSThreads, smem, st, bank, res, B, plan, tiles);
    PB_LAUNCHED("bank_stream_kernel");
    return PB_OK;
  }
  const int bps = (int)((B / kMPT + kMergedThreads - 1) / kMergedThreads);
  const int64_t blocks = spans * bps;
  if (blocks >= ((int64_t)1 << 31)) return pb::fail(PB_E_UNSUPPORTED, "filter bank: too many spans");
  bank_merged_kernel<<<(unsigned)blocks, kMergedThreads, 0, st>>>(bank, res, B, plan, bps);
  PB_LAUNCHED("bank_merged_kernel");
  return PB_OK;
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
  const int dev = pb::device();
  if (dev < 0) return PB_E_CUDA;
  static int sms_d[pb::kMaxDevices] = {}, per_sm_d[pb::kMaxDevices] = {};
  int& sms = sms_d[dev];
  int& per_sm = per_sm_d[dev];
  if (sms == 0) {
    PB_CUDA(cudaFuncSetAttribute(fir_persistent<kBank, kMath>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
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
    case PB_FIR_MERGED:   // per-actor launches have nothing to merge: FMA
      return kBank ? launch_merged_bank(bank, res, B, st)
                   : launch_variant<kBank, PB_FIR_FMA>(bank, actors, n_actors, res, B, st);
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
  PB_LAUNCH_PDL(fir_carry_kernel, grid, 32, 0, pb::as_stream(stream), actors, res, block);
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
  rc = launch<true>(bank, nullptr, 0, res, block, bank.math, pb::as_stream(stream));
  if (rc) return rc;
  // the history carry is part of the bank's firing: done inside the stream
  // kernel on the merged path, a carry launch otherwise
  if (bank.math == PB_FIR_MERGED && PB_MERGED_STREAM == 1 && PB_MS_CARRY) return PB_OK;
  dim3 grid(res.n_streams, bank.n_branches);
  PB_LAUNCH_PDL(fir_carry_kernel, grid, 32, 0, pb::as_stream(stream), bank.branches, res, block);
  PB_LAUNCHED("fir_carry_kernel");
  return PB_OK;
}

}  // extern "C"
