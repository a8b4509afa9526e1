// CNN actors of the vision example: the only
// tensor-core path.  The reference package ships no DNN;
// the graph and its oracle are builder-defined (apps/vision.py,
// oracle/cnn.py) and parity is stated as a tolerance, not bit-exactness.
//
// conv_pool_kernel: 5x5 convolution (NHWC fp32, zero padding) + bias + ReLU
// + 2x2 max-pool as an implicit GEMM on tcgen05 (kind::f16, bf16 operands,
// fp32 accumulation in TMEM), persistent and warp-specialised:
//
//   * GEMM tile: M = 128 conv pixels laid out as 16 image rows x 8 columns,
//     2 (layer 2) or 4 (layer 1) tiles side by side per super-tile,
//     N = 32 output channels, K = 25 * Cin.  A 2x2 pool window is then two
//     neighbouring lanes of two neighbouring 8-lane groups of ONE warp.
//   * Accuracy: split bf16 ("bf16x3"): x = xh + xl, w = wh + wl (each bf16,
//     round-to-nearest), D = xh*wh + xl*wh + xh*wl; the dropped xl*wl and
//     the rounding of xl are ~2^-17 relative per product.  The B operand of
//     the xh MMA is [wh; wl] (N = 64), so three products cost two MMAs;
//     the epilogue adds the two 32-column halves.
//   * No im2col: the converter warps stage each super-tile's input patch in
//     shared memory ONCE, as bf16 hi / lo 16-byte "entry planes" in the UMMA
//     K-major no-swizzle core layout, and every tap's A operand is just a
//     shifted descriptor into that patch: rows of a core matrix are
//     consecutive entries (16 B apart), SBO = one patch row (next image
//     row), LBO = the plane stride (next 8 K elements).
//       mode 1 (Cin % 16 == 0, layer 2): entry = one pixel, plane q holds
//         channels 8q..8q+7; a K-step is one tap x 16 channels.
//       mode 0 (Cin == 3, layer 1): entry (y, x) holds the 5*Cin values
//         x[y][x..x+4][0..Cin) (zero-padded to 16); a K-step is one kernel
//         row ky, so 5 MMA pairs cover the whole 5x5xCin window.
//     Probed on hardware in tools/conv_probe.cu (window modes 0-2).
//   * Roles: warps 0-7 epilogue (TMEM lane quarter = warp % 4), warp 8 MMA issue
//     (one elected lane), warps 9-15 converters (global fp32 -> bf16 hi/lo
//     patch).  Patches and TMEM accumulators are double-buffered and handed
//     over with mbarriers (converters -> MMA: 128 arrivals; MMA -> converter
//     and epilogue: tcgen05.commit; epilogue -> MMA: 128 arrivals).
//   * All weights stay resident in shared memory for the whole launch.
//   * Patches and accumulators: NB buffers (layer 1: 3, layer 2: 2).
#include <algorithm>

#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "pb_common.cuh"

namespace {

constexpr int kTW = 8, kTH = 16;            // conv pixels per MMA tile (M = 128)
constexpr int kPH = kTH + 4;                // patch rows
constexpr int kEpiWarps = 8, kCvtWarps = 6;   // + MMA + scheduler = 16 warps: 4 per SMSP, 128 regs
constexpr int kMmaWarp = kEpiWarps;
constexpr int kCvtWarp0 = kMmaWarp + 1;
constexpr int kSchedWarp = kCvtWarp0 + kCvtWarps;   // walks the work list
constexpr int kSchedRing = 16;
constexpr int kConvThreads = (kEpiWarps + 1 + kCvtWarps + 1) * 32;
constexpr int kCvtThreads = kCvtWarps * 32;
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kTmemCols = 512;              // NB accumulator sets x ST tiles x ACC columns
constexpr int kMaxNB = 4;
constexpr int kStepBytes = 64 * 16 * 2;     // one K-step of [wh; wl]: 64 rows x 16 bf16
constexpr int kCout = 32;
constexpr int kRawBufs = 6;                 // layer-1 raw boxes in flight (prefetch depth 5)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Shared-memory matrix descriptor, K-major, no swizzle (sm100 version 1).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

// kind::f16 instruction descriptor: bf16 A/B, fp32 D, K-major, M = 128 (256: a CTA pair).
__host__ __device__ constexpr uint32_t idesc_bf16(int n, int m = 128) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem, uint64_t a, uint64_t b, uint32_t id,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// ---- CTA-pair (cta_group::2) helpers, layer 2 with PB_CONV_PAIR
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// M = 256 over the pair: A rows 0-127 from the leader's shared memory, 128-255
// from the peer's (same offset); B split by N (first half leader, second
// half peer); D = each CTA's own 128 TMEM lanes.  Issued by the leader.
__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem, uint64_t a, uint64_t b, uint32_t id,
                                              uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
// completion of the leader's MMAs arrives on the barrier at this offset in
// both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)), "h"((uint16_t)3)
      : "memory");
}
// arrive on the leader's (rank 0) barrier at this offset, release at cluster scope
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  pb::mbar_wait_trap_cluster(smem_u32(bar), parity);
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  pb::mbar_wait_trap(smem_u32(bar), parity);
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)), "r"(bytes)
               : "memory");
}

// x = hi + lo, each bf16 round-to-nearest; packs 8 values per 16 bytes.
__device__ __forceinline__ uint32_t pack_hi(float a, float b, float& ra, float& rb) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  ra = a - __low2float(h);
  rb = b - __high2float(h);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t pack_lo(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ void split8(const float* v, uint4& hi, uint4& lo) {
  float r[8];
  hi.x = pack_hi(v[0], v[1], r[0], r[1]);
  hi.y = pack_hi(v[2], v[3], r[2], r[3]);
  hi.z = pack_hi(v[4], v[5], r[4], r[5]);
  hi.w = pack_hi(v[6], v[7], r[6], r[7]);
  lo.x = pack_lo(r[0], r[1]);
  lo.y = pack_lo(r[2], r[3]);
  lo.z = pack_lo(r[4], r[5]);
  lo.w = pack_lo(r[6], r[7]);
}

// Geometry of one conv layer.  MODE/CIN are template parameters (layer 1:
// <0, 3>, layer 2: <1, 32>), so every shared-memory offset and every MMA
// descriptor step is a compile-time constant and the issue loop is a straight
// run of tcgen05.mma with immediate descriptor offsets.
template <int MODE, int CIN>
struct ConvCfg {
#ifndef PB_CONV_ST0
#define PB_CONV_ST0 4
#endif
#ifndef PB_CONV_SPLIT3_0
#define PB_CONV_SPLIT3_0 1
#endif
  static constexpr int CIN_ = CIN;
  static constexpr int ST = MODE ? 2 : PB_CONV_ST0;       // tiles per super-tile
  static constexpr int NP = MODE ? CIN / 8 : 2;           // 16-B planes per precision piece
  static constexpr int PW = ST * kTW + (MODE ? 4 : 0);    // patch width (entries)
  static constexpr int PS = kPH * PW * 16;                // plane stride (bytes)
  static constexpr int STEPS = MODE ? 25 * (CIN / 16) : 5;
  // layer 2 is MMA-bound: B = [wh; wl] (N = 64) gives two products per MMA and
  // the epilogue adds the column halves; layer 1 is epilogue-bound: three
  // N = 32 MMAs accumulate all products into 32 columns
  static constexpr bool SPLIT3 = MODE == 0 && PB_CONV_SPLIT3_0;
  static constexpr int ACC = SPLIT3 ? 32 : 64;            // TMEM columns per tile
  static constexpr int PATCH = 2 * NP * PS;
  static constexpr int WBYTES = STEPS * kStepBytes;
  // layer-1 raw input box staged by one TMA tensor load: kPH rows x
  // (PW + 4) pixels x 3 channels fp32, zero-filled outside the frame; the box
  // starts on a 16-byte boundary (a TMA requirement for the inner
  // coordinate), so it carries up to 3 extra leading floats
  static constexpr int RAW_W = MODE ? 0 : ((PW + 4) * 3 + 3 + 3) / 4 * 4;   // floats per raw row
  static constexpr int RAW_TX = kPH * RAW_W * 4;          // bytes per box
  static constexpr int RAW = MODE ? 0 : ((RAW_TX + 127) / 128) * 128;
#ifndef PB_CONV_L1_EPT   // layer-1 entries per converter thread per batch (loads in flight)
#define PB_CONV_L1_EPT 4
#endif
#ifndef PB_CONV_PAIR_STAGED
#define PB_CONV_PAIR_STAGED 1
#endif
#ifndef PB_CONV_NB0
#define PB_CONV_NB0 3
#endif
  // patch / accumulator buffers in flight (layer 2 is shared-memory-limited)
  static constexpr int NB = MODE ? 2 : PB_CONV_NB0;
  static constexpr int SMEM = WBYTES + NB * PATCH + kRawBufs * RAW;
  static_assert(NB <= kMaxNB && NB * ST * ACC <= kTmemCols, "conv buffers");
  static __host__ __device__ constexpr int a_off(int s) {   // bytes, tile 0, hi piece
    return MODE ? 2 * (s % (CIN / 16)) * PS + (((s / (CIN / 16)) / 5) * PW + (s / (CIN / 16)) % 5) * 16
                : s * PW * 16;
  }
};

// n / d for 0 <= n < 2^24 without an integer divide: float reciprocal, then
// an exact one-step correction.
struct FastDiv {
  int d;
  float inv;
};
__device__ __forceinline__ FastDiv fast_div(int d) { return FastDiv{d, 1.0f / (float)d}; }
__device__ __forceinline__ int fdiv(int n, FastDiv f) {
  int q = __float2int_rz(__int2float_rn(n) * f.inv);
  const int r = n - q * f.d;
  if (r < 0) --q;
  else if (r >= f.d) ++q;
  return q;
}

struct ConvRun {   // runtime geometry
  int H, W, pad, Ho, Wo, Hp, Wp, sx_n, per_frame, per_unit, n_units;
  int64_t in_frame, out_frame;
  FastDiv d_iter, d_frame, d_sx;   // n_iter, per_frame, sx_n
};

template <class Cfg>
__device__ __forceinline__ ConvRun conv_run(const pb_conv_actor& a, const pb_resolved& res) {
  ConvRun g;
  g.H = a.h; g.W = a.w; g.pad = a.pad;
  g.Ho = g.H + 2 * g.pad - 4; g.Wo = g.W + 2 * g.pad - 4;
  g.Hp = g.Ho / 2; g.Wp = g.Wo / 2;
  g.sx_n = (g.Wo + Cfg::ST * kTW - 1) / (Cfg::ST * kTW);
  g.per_frame = ((g.Ho + kTH - 1) / kTH) * g.sx_n;
  g.per_unit = a.frames * g.per_frame;
  g.n_units = res.n_streams * res.n_iter;
  g.in_frame = (int64_t)g.H * g.W * a.cin;
  g.out_frame = (int64_t)g.Hp * g.Wp * kCout;
  g.d_iter = fast_div(res.n_iter);
  g.d_frame = fast_div(g.per_frame);
  g.d_sx = fast_div(g.sx_n);
  return g;
}

constexpr int kMaxStreams = 1024;          // per-stream firing counts cached in smem

// Role timing (profiling builds only: -DPB_CONV_PROF=1, tools/build_variant.sh):
// one thread per role accumulates clock64 deltas per phase into g_conv_prof
// [CTA][slot]; read with pb_conv_debug_counters.
#ifndef PB_CONV_PROF
#define PB_CONV_PROF 0
#endif
constexpr int kProfCtas = 160, kProfSlots = 16;
__device__ unsigned long long g_conv_prof[kProfCtas][kProfSlots];
#define PROF_START() long long prof_t_ = PB_CONV_PROF ? clock64() : 0
#define PROF(on, slot)                                                              \
  do {                                                                              \
    if (PB_CONV_PROF && (on)) {                                                     \
      const long long n_ = clock64();                                               \
      atomicAdd(&g_conv_prof[blockIdx.x % kProfCtas][slot], (unsigned long long)(n_ - prof_t_)); \
      prof_t_ = n_;                                                                 \
    }                                                                               \
  } while (0)

struct SuperTile {
  const float* fin;   // input frame
  float* fout;        // output frame
  int oy0, ox0;       // conv-output origin
  int frame;          // global input frame index (layer-1 TMA coordinate)
  int pad_;
};

// Super-tile descriptors the converters publish with each patch (the MMA warp
// and the epilogue never walk the work list or touch global memory for it).
// A slot is rewritten 8 super-tiles later; the converters run at most NB
// super-tiles ahead of the MMA warp and it at most NB ahead of the epilogue.
constexpr int kDescRing = 8;
static_assert(2 * kMaxNB <= kDescRing, "descriptor ring");

struct ConvBars {
  uint64_t full[kMaxNB], empty[kMaxNB], acc_full[kMaxNB], acc_empty[kMaxNB], raw_full[kRawBufs];
  SuperTile desc[kDescRing];                  // fin unused; fout == nullptr: end of work
  SuperTile sched[kSchedRing];                // the scheduler warp's work list ring
  uint64_t sched_full[kSchedRing], sched_empty[kSchedRing];
  int cnt[kMaxStreams];                       // live firings per stream (cond_count)
  uint32_t tmem_base;
  float bias[kCout];
};

// Walks this CTA's super-tiles (w = blockIdx.x, += gridDim.x) over the live
// firings without 64-bit divisions: unit = (stream, iteration), rem = the
// super-tile within the unit's frames.
struct Cursor {
  int unit, rem, s, j;
  bool live;
};

// cnt: the per-stream live-firing counts, cached in shared memory, so walking
// the cursor never waits on global memory
__device__ __forceinline__ void cursor_fix(Cursor& c, const ConvRun& g, const int* cnt,
                                           const pb_resolved& res) {
  if (c.unit < g.n_units) {
    c.s = fdiv(c.unit, g.d_iter);
    c.j = c.unit - c.s * res.n_iter;
    c.live = c.j < cnt[c.s];
  }
}

__device__ __forceinline__ Cursor cursor_first(const ConvRun& g, const int* cnt,
                                               const pb_resolved& res) {
  Cursor c;
  c.unit = blockIdx.x / g.per_unit;
  c.rem = blockIdx.x - c.unit * g.per_unit;
  c.live = false;
  cursor_fix(c, g, cnt, res);
  return c;
}

__device__ __forceinline__ void cursor_step(Cursor& c, const ConvRun& g, const int* cnt,
                                            const pb_resolved& res) {
  c.rem += gridDim.x;
  if (c.rem >= g.per_unit) {
    while (c.rem >= g.per_unit) {
      c.rem -= g.per_unit;
      ++c.unit;
    }
    cursor_fix(c, g, cnt, res);
  }
}

// next live super-tile (including the current one)
__device__ __forceinline__ bool cursor_live(Cursor& c, const ConvRun& g, const int* cnt,
                                            const pb_resolved& res) {
  while (c.unit < g.n_units && !c.live) cursor_step(c, g, cnt, res);
  return c.unit < g.n_units;
}

// Firing spans of every (stream, iteration) unit, resolved once per launch by
// conv_units_kernel (nullptr: the actor does not fire there): a super-tile's
// pointers are then one independent 16-byte load, not a chain of three.
struct UnitSpans {
  const float* in;
  float* out;
  int frame0;   // global frame index of the input span (layer-1 TMA coordinate)
  int pad_;
};

__global__ void conv_units_kernel(pb_conv_actor a, pb_resolved res, UnitSpans* units) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= res.n_streams * res.n_iter) return;
  const int s = u / res.n_iter, j = u - s * res.n_iter;
  UnitSpans r{nullptr, nullptr, 0, 0};
  if (j < pb::cond_count(res, a.cond, s)) {
    const int n = pb::firing_iter(res, a.cond, s, j);
    r.in = reinterpret_cast<const float*>(pb::span_ptr(a.in, res, s, n));
    r.out = reinterpret_cast<float*>(pb::span_ptr(a.out, res, s, n));
    r.frame0 = (int)((r.in - reinterpret_cast<const float*>(a.in.data)) /
                     ((int64_t)a.h * a.w * a.cin));
  }
  units[u] = r;
}

// A super-tile in two halves: the geometry and the (issued, not yet used)
// load of its unit's spans, then the pointer arithmetic once the load is back
// -- so the load latency overlaps a whole iteration of the caller.
struct PendingTile {
  UnitSpans u;
  int f, oy0, ox0;
};

template <class Cfg>
__device__ __forceinline__ PendingTile pending_tile(const Cursor& c, const ConvRun& g,
                                                    const UnitSpans* units) {
  PendingTile p;
  p.f = fdiv(c.rem, g.d_frame);
  const int st = c.rem - p.f * g.per_frame;
  const int sy = fdiv(st, g.d_sx);
  p.oy0 = sy * kTH;
  p.ox0 = (st - sy * g.sx_n) * (Cfg::ST * kTW);
  p.u = units[c.unit];
  return p;
}

__device__ __forceinline__ SuperTile finish_tile(const PendingTile& p, const ConvRun& g) {
  SuperTile t;
  t.fin = p.u.in + p.f * g.in_frame;
  t.fout = p.u.out + p.f * g.out_frame;
  t.frame = p.u.frame0 + p.f;
  t.oy0 = p.oy0;
  t.ox0 = p.ox0;
  t.pad_ = 0;
  return t;
}

// Layer 1: one TMA tensor load of the raw box a super-tile needs (rows
// oy0-pad .. +kPH, pixels ox0-pad .. +PW+4, all 3 channels); the tensor map
// spans every frame of the input ring, so padding is the TMA zero fill.
template <class Cfg>
__device__ __forceinline__ void raw_issue(uint8_t* raw, uint64_t* bar, const CUtensorMap* tmap,
                                          const ConvRun& g, const pb_conv_actor& a,
                                          const SuperTile& t) {
  const int frame = t.frame;
  mbar_arrive_tx(bar, Cfg::RAW_TX);
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(raw)),
      "l"(tmap), "r"(((t.ox0 - g.pad) * 3) & ~3), "r"(t.oy0 - g.pad), "r"(frame), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}

// Layer-2 converter with a cp.async staging ring (CTA-pair kernel, which has
// the 25 KB the single-CTA weights would occupy free): each thread copies the
// fp32 items it will convert, two batches ahead, straight into shared memory
// (out-of-frame items as a zero-size copy, i.e. zero fill) and splits a batch
// once its own copies have landed -- no registers held across the global-load
// latency and no barrier (a thread converts exactly the items it copied).
template <class Cfg>
__device__ __forceinline__ void fill_patch_staged(uint8_t* patch, uint8_t* stage,
                                                  const ConvRun& g, const SuperTile& t, int ct) {
  constexpr int kS = 2;                                   // items per thread per batch
  constexpr int kBatch = kS * kCvtThreads;
  constexpr int items = kPH * Cfg::PW * Cfg::NP;
  constexpr int nb = (items + kBatch - 1) / kBatch;
  constexpr int kBufBytes = kBatch * 32;
  auto issue = [&](int bt) {
    float4* buf = reinterpret_cast<float4*>(stage + (bt & 1) * kBufBytes);
#pragma unroll
    for (int u = 0; u < kS; ++u) {
      const int i = bt * kBatch + u * kCvtThreads + ct;
      if (i < items) {
        const int e = i / Cfg::NP, q = i % Cfg::NP;
        const int iy = t.oy0 + e / Cfg::PW - g.pad, ix = t.ox0 + e % Cfg::PW - g.pad;
        const bool in = iy >= 0 && iy < g.H && ix >= 0 && ix < g.W;
        const float* src = in ? t.fin + ((int64_t)iy * g.W + ix) * Cfg::CIN_ + 8 * q : t.fin;
        float4* d = buf + 2 * (u * kCvtThreads + ct);
        cp_async16(d, src, in ? 16u : 0u);
        cp_async16(d + 1, in ? src + 4 : src, in ? 16u : 0u);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue(0);
  if (nb > 1) issue(1);
#pragma unroll 1
  for (int bt = 0; bt < nb; ++bt) {
    if (bt + 1 < nb) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    const float4* buf = reinterpret_cast<const float4*>(stage + (bt & 1) * kBufBytes);
#pragma unroll
    for (int u = 0; u < kS; ++u) {
      const int i = bt * kBatch + u * kCvtThreads + ct;
      if (i >= items) break;
      const float4 a = buf[2 * (u * kCvtThreads + ct)], b = buf[2 * (u * kCvtThreads + ct) + 1];
      const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      const int e = i / Cfg::NP, q = i % Cfg::NP;
      uint4 hi, lo;
      split8(v, hi, lo);
      *reinterpret_cast<uint4*>(patch + q * Cfg::PS + e * 16) = hi;
      *reinterpret_cast<uint4*>(patch + (Cfg::NP + q) * Cfg::PS + e * 16) = lo;
    }
    if (bt + 2 < nb) issue(bt + 2);
  }
}

// Converter: build the bf16 hi/lo entry planes of super-tile `t` in `patch`.
template <int MODE, int CIN>
__device__ __forceinline__ void fill_patch(uint8_t* patch, const uint8_t* raw, const ConvRun& g,
                                           const SuperTile& t, int ct) {
  using Cfg = ConvCfg<MODE, CIN>;
  if constexpr (MODE == 1) {
    constexpr int kB = 4;
    constexpr int items = kPH * Cfg::PW * Cfg::NP;
#pragma unroll 1
    for (int i0 = ct; i0 < items; i0 += kB * kCvtThreads) {
      float v[kB][8];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int i = i0 + u * kCvtThreads;
        const int e = i / Cfg::NP, q = i % Cfg::NP;
        const int iy = t.oy0 + e / Cfg::PW - g.pad, ix = t.ox0 + e % Cfg::PW - g.pad;
        if (i < items && iy >= 0 && iy < g.H && ix >= 0 && ix < g.W) {
          const float4* src = reinterpret_cast<const float4*>(
              t.fin + ((int64_t)iy * g.W + ix) * CIN + 8 * q);
          const float4 a = __ldg(src), b = __ldg(src + 1);
          v[u][0] = a.x; v[u][1] = a.y; v[u][2] = a.z; v[u][3] = a.w;
          v[u][4] = b.x; v[u][5] = b.y; v[u][6] = b.z; v[u][7] = b.w;
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) v[u][k] = 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int i = i0 + u * kCvtThreads;
        if (i >= items) break;
        const int e = i / Cfg::NP, q = i % Cfg::NP;
        uint4 hi, lo;
        split8(v[u], hi, lo);
        *reinterpret_cast<uint4*>(patch + q * Cfg::PS + e * 16) = hi;
        *reinterpret_cast<uint4*>(patch + (Cfg::NP + q) * Cfg::PS + e * 16) = lo;
      }
    }
  } else {
    // entries from the raw box in shared memory (out-of-frame pixels are
    // already zero); one entry per thread keeps the 16-byte stores of a warp
    // on consecutive entries (conflict-free)
    constexpr int items = kPH * Cfg::PW;
    const float* rawf = reinterpret_cast<const float*>(raw) + (((t.ox0 - g.pad) * 3) & 3);
    // entries in pairs: both entries' 30 loads are issued before either is
    // split (one shared-memory latency per pair)
#pragma unroll 1
    for (int e0 = ct; e0 < items; e0 += PB_CONV_L1_EPT * kCvtThreads) {
      float v[PB_CONV_L1_EPT][16];
#pragma unroll
      for (int u = 0; u < PB_CONV_L1_EPT; ++u) {
        const int e = min(e0 + u * kCvtThreads, items - 1);
        const int r = e / Cfg::PW, c = e % Cfg::PW;
        const float* src = rawf + r * Cfg::RAW_W + c * 3;
#pragma unroll
        for (int k = 0; k < 15; ++k) v[u][k] = src[k];
        v[u][15] = 0.f;
      }
#pragma unroll
      for (int u = 0; u < PB_CONV_L1_EPT; ++u) {
        const int e = e0 + u * kCvtThreads;
        if (e >= items) break;
        uint4 h0, l0, h1, l1;
        split8(v[u], h0, l0);
        split8(v[u] + 8, h1, l1);
        *reinterpret_cast<uint4*>(patch + 0 * Cfg::PS + e * 16) = h0;
        *reinterpret_cast<uint4*>(patch + 1 * Cfg::PS + e * 16) = h1;
        *reinterpret_cast<uint4*>(patch + 2 * Cfg::PS + e * 16) = l0;
        *reinterpret_cast<uint4*>(patch + 3 * Cfg::PS + e * 16) = l1;
      }
    }
  }
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(p));
  return p != 0;
}

// PAIR (layer 2): clusters of two CTAs; each CTA still builds the patch of
// its own super-tiles, and the even CTA issues cta_group::2 MMAs (M = 256)
// that read both patches, so each SM reads only half of B (the weights) per
// MMA.  Both CTAs walk the pair's two work lists in lockstep (a half without
// a live super-tile gets a dummy one), so every MMA has both halves.
template <int MODE, int CIN, bool PAIR = false>
__global__ void __launch_bounds__(kConvThreads, 1)
conv_pool_kernel(pb_conv_actor a, pb_resolved res, const UnitSpans* __restrict__ units,
                 const __grid_constant__ CUtensorMap tmap) {
  using Cfg = ConvCfg<MODE, CIN>;
  constexpr bool kPair = PAIR && MODE == 1;
  const uint32_t crank = kPair ? cluster_ctarank() : 0u;
  // pair weights per K-step: 32 B rows (the N = 64 MMA's half: wh on the
  // leader, wl on the peer) then 16 B rows (the N = 32 MMA's half of wh)
  constexpr int kPairStep = 1536;
  // the converters' cp.async staging ring lives in the tail of the weights
  // region the pair weights leave free (when it fits: Cin = 32)
  constexpr bool kStaged = kPair && PB_CONV_PAIR_STAGED &&
                           Cfg::STEPS * kPairStep + 2 * 2 * kCvtThreads * 32 <= Cfg::WBYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const ConvRun G = conv_run<Cfg>(a, res);
  uint8_t* wsm = base;                                   // [STEPS][2 KB]
  uint8_t* patch0 = base + Cfg::WBYTES;                  // [2][PATCH]
  uint8_t* raw0 = patch0 + Cfg::NB * Cfg::PATCH;         // [kRawBufs][RAW] (layer 1)
  ConvBars& B = *reinterpret_cast<ConvBars*>(base + Cfg::SMEM);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- prologue: weights, bias, barriers, TMEM
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.weights);
    uint4* dst = reinterpret_cast<uint4*>(wsm);
    if constexpr (kPair) {
      for (int i = tid; i < Cfg::STEPS * (kPairStep / 16); i += kConvThreads) {
        const int st = i / (kPairStep / 16), o = i - st * (kPairStep / 16);   // 16-B units
        const int srco = o < 64 ? (int)crank * 64 + o : (int)crank * 32 + (o - 64);
        dst[i] = __ldg(src + st * (kStepBytes / 16) + srco);
      }
    } else {
      for (int i = tid; i < Cfg::WBYTES / 16; i += kConvThreads) dst[i] = __ldg(src + i);
    }
    if (tid < kCout) B.bias[tid] = __ldg(a.bias + tid);
    for (int st = tid; st < res.n_streams; st += kConvThreads) B.cnt[st] = pb::cond_count(res, a.cond, st);
  }
  if (warp == 0) {
    if constexpr (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&B.tmem_base)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&B.tmem_base)),
                   "r"(kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (tid == 0) {
    for (int b = 0; b < Cfg::NB; ++b) {
      // pair: the leader's full / acc_empty also count the peer's converters
      // and epilogue; acc_full is the multicast MMA completion alone
      mbar_init(&B.full[b], kPair ? 2 * kCvtThreads : kCvtThreads);
      mbar_init(&B.empty[b], 1);
      // acc_full: the MMA completion (tcgen05.commit) and a plain release
      // arrive of the MMA thread, which orders the descriptor it read
      mbar_init(&B.acc_full[b], kPair ? 1 : 2);
      mbar_init(&B.acc_empty[b], kPair ? 2 * kEpiThreads : kEpiThreads);
    }
    for (int b = 0; b < kRawBufs; ++b) mbar_init(&B.raw_full[b], 1);
    for (int k = 0; k < kSchedRing; ++k) {
      mbar_init(&B.sched_full[k], 1);
      mbar_init(&B.sched_empty[k], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if constexpr (kPair) cluster_sync();   // both CTAs' barriers exist before any remote arrive
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = B.tmem_base;

  if (kPair && warp == kSchedWarp) {
    // ================================================ pair scheduler
    // both halves' cursors (super-tiles w0 + k*grid and w0 + 1 + k*grid),
    // stepped together; steps where neither half is live are skipped
    const int w0 = (int)(blockIdx.x & ~1u);
    auto at = [&](int w) {
      Cursor c;
      c.unit = w / G.per_unit;
      c.rem = w - c.unit * G.per_unit;
      c.live = false;
      cursor_fix(c, G, B.cnt, res);
      return c;
    };
    Cursor c0 = at(w0), c1 = at(w0 + 1);
    auto live = [&](const Cursor& c) { return c.unit < G.n_units && c.live; };
    for (int k = 0;; ++k) {
      while (c0.unit < G.n_units && !live(c0) && !live(c1)) {
        cursor_step(c0, G, B.cnt, res);
        cursor_step(c1, G, B.cnt, res);
      }
      const bool more = c0.unit < G.n_units;
      const int slot = k % kSchedRing;
      mbar_wait(&B.sched_empty[slot], ((uint32_t)(k / kSchedRing) & 1) ^ 1);
      SuperTile t{};
      if (more) {
        const Cursor& me = crank ? c1 : c0;
        if (live(me)) {
          t = finish_tile(pending_tile<Cfg>(me, G, units), G);
        } else {   // dummy half: converters skip it, the epilogue stores nothing
          t.fout = reinterpret_cast<float*>(uintptr_t(16));
          t.pad_ = 1;
        }
        cursor_step(c0, G, B.cnt, res);
        cursor_step(c1, G, B.cnt, res);
      }
      if (lane == 0) {
        B.sched[slot] = t;
        mbar_arrive(&B.sched_full[slot]);
      }
      __syncwarp();
      if (!more) break;
    }
  } else if (warp == kSchedWarp) {
    // ================================================ scheduler
    // Walks this CTA's work list (the latency-bound cursor arithmetic and the
    // unit-table loads, one super-tile ahead) and publishes one SuperTile per
    // slot of a ring the converters consume; fout == nullptr ends the list.
    const bool pon = lane == 0;
    PROF_START();
    Cursor c = cursor_first(G, B.cnt, res);
    bool live = cursor_live(c, G, B.cnt, res);
    PendingTile p_next{};
    if (live) p_next = pending_tile<Cfg>(c, G, units);
    for (int k = 0;; ++k) {
      const int slot = k % kSchedRing;
      mbar_wait(&B.sched_empty[slot], ((uint32_t)(k / kSchedRing) & 1) ^ 1);
      SuperTile t{};
      const bool more = live;
      if (more) {
        const PendingTile p = p_next;
        cursor_step(c, G, B.cnt, res);
        live = cursor_live(c, G, B.cnt, res);
        if (live) p_next = pending_tile<Cfg>(c, G, units);
        t = finish_tile(p, G);
      }
      if (lane == 0) {
        B.sched[slot] = t;   // zero-initialised: fout == nullptr when !more
        mbar_arrive(&B.sched_full[slot]);
      }
      __syncwarp();
      PROF(pon, 15);
      if (!more) break;
    }
  } else if (warp >= kCvtWarp0) {
    // ================================================ converters
    const int ct = tid - kCvtWarp0 * 32;
    constexpr int kRawIssuer = kCvtThreads - 32;   // layer 1: issues the raw-box TMA loads
    const bool pon = ct == 0;
    PROF_START();
    bool raw_more = true;                          // (issuer) the list has not ended yet
    auto issue_raw = [&](int k) {                  // raw box of super-tile k
      if (ct != kRawIssuer || !raw_more) return;
      mbar_wait(&B.sched_full[k % kSchedRing], (uint32_t)(k / kSchedRing) & 1);
      const SuperTile tk = B.sched[k % kSchedRing];
      if (tk.fout == nullptr) {
        raw_more = false;
        return;
      }
      if (!(a.debug & 8))
        raw_issue<Cfg>(raw0 + (k % kRawBufs) * Cfg::RAW, &B.raw_full[k % kRawBufs], &tmap, G, a, tk);
    };
    if constexpr (MODE == 0)
      for (int k = 0; k < kRawBufs - 1; ++k) issue_raw(k);
    for (int it = 0;; ++it) {
      const int slot = it % kSchedRing;
      const int b = it % Cfg::NB;
      const uint32_t use = (uint32_t)(it / Cfg::NB);
      mbar_wait(&B.sched_full[slot], (uint32_t)(it / kSchedRing) & 1);
      const SuperTile t = B.sched[slot];
      PROF(pon, 0);
      if (t.fout == nullptr) {   // end of work: an empty descriptor through the normal handoff
        mbar_wait(&B.empty[b], (use & 1) ^ 1);
        if (ct == 0) B.desc[it % kDescRing].fout = nullptr;
        if (kPair && crank) mbar_arrive_leader(&B.full[b]);
        else mbar_arrive(&B.full[b]);
        break;
      }
      const int rb = it % kRawBufs;
      if constexpr (MODE == 0)
        if (!(a.debug & 8)) mbar_wait(&B.raw_full[rb], (uint32_t)(it / kRawBufs) & 1);
      PROF(pon, 1);
      mbar_wait(&B.empty[b], (use & 1) ^ 1);
      PROF(pon, 2);
      if (!(a.debug & 1) && t.pad_ == 0) {
        if constexpr (kStaged)   // the free tail of the weights region
          fill_patch_staged<Cfg>(patch0 + b * Cfg::PATCH, wsm + Cfg::STEPS * kPairStep, G, t, ct);
        else
          fill_patch<MODE, CIN>(patch0 + b * Cfg::PATCH, raw0 + rb * Cfg::RAW, G, t, ct);
      }
      if (ct == 0) B.desc[it % kDescRing] = t;
      PROF(pon, 3);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (kPair && crank) mbar_arrive_leader(&B.full[b]);
      else mbar_arrive(&B.full[b]);
      PROF(pon, 4);
      // all converters are done with sched[slot] (and, layer 1, raw[rb])
      asm volatile("bar.sync 2, %0;" ::"n"(kCvtThreads));
      if (ct == 0) mbar_arrive(&B.sched_empty[slot]);
      PROF(pon, 5);
      if constexpr (MODE == 0) issue_raw(it + kRawBufs - 1);
      PROF(pon, 6);
    }
  } else if (kPair && warp == kMmaWarp) {
    // ================================================ pair MMA issue (the leader only)
    if (crank == 0) {
      constexpr uint32_t id64 = idesc_bf16(64, 256), id32 = idesc_bf16(32, 256);
      const uint64_t db0 = sdesc(smem_u32(wsm), 128, 256);
      for (int it = 0;; ++it) {
        const int b = it % Cfg::NB;
        const uint32_t use = (uint32_t)(it / Cfg::NB);
        mbar_wait_cluster(&B.full[b], use & 1);   // both CTAs' converters
        const SuperTile& t = B.desc[it % kDescRing];
        const bool end = t.fout == nullptr;
        mbar_wait_cluster(&B.acc_empty[b], (use & 1) ^ 1);   // both CTAs' epilogues
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (end) {   // let both epilogues see the end
          if (elect_one()) mma_commit_pair(&B.acc_full[b]);
          __syncwarp();
          break;
        }
        const uint64_t da0 = sdesc(smem_u32(patch0 + b * Cfg::PATCH), Cfg::PS, Cfg::PW * 16);
        if (elect_one()) {
#pragma unroll
          for (int tt = 0; tt < Cfg::ST; ++tt) {
            if (a.debug & 4) break;
            const uint32_t d = tmem + (uint32_t)((b * Cfg::ST + tt) * Cfg::ACC);
#pragma unroll
            for (int st = 0; st < Cfg::STEPS; ++st) {
              const uint64_t dah = da0 + (uint64_t)((Cfg::a_off(st) + tt * kTW * 16) >> 4);
              const uint64_t dal = dah + (uint64_t)((Cfg::NP * Cfg::PS) >> 4);
              const uint64_t db = db0 + (uint64_t)(st * (kPairStep >> 4));
              mma_bf16_pair(d, dah, db, id64, st > 0 ? 1u : 0u);            // [xh*wh | xh*wl]
              mma_bf16_pair(d, dal, db + (1024 >> 4), id32, 1u);            // + xl*wh
            }
          }
          mma_commit_pair(&B.empty[b]);
          mma_commit_pair(&B.acc_full[b]);
        }
        __syncwarp();
      }
    }
  } else if (warp == kMmaWarp) {
    // ================================================ MMA issue (warp-uniform loop, one lane issues)
    constexpr uint32_t id64 = idesc_bf16(64), id32 = idesc_bf16(32);
    const uint64_t db0 = sdesc(smem_u32(wsm), 128, 256);
    const bool pon = lane == 0;
    PROF_START();
    for (int it = 0;; ++it) {
      const int b = it % Cfg::NB;
      const uint32_t use = (uint32_t)(it / Cfg::NB);
      mbar_wait(&B.full[b], use & 1);
      PROF(pon, 8);
      const SuperTile& t = B.desc[it % kDescRing];
      if (t.fout == nullptr) {   // end of work: let the epilogue see it too
        mbar_wait(&B.acc_empty[b], (use & 1) ^ 1);
        if (elect_one()) {
          mma_commit(&B.acc_full[b]);
          mbar_arrive(&B.acc_full[b]);
        }
        __syncwarp();
        break;
      }
      const int ox0 = t.ox0;
      PROF(pon, 7);
      mbar_wait(&B.acc_empty[b], (use & 1) ^ 1);
      PROF(pon, 9);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint64_t da0 = sdesc(smem_u32(patch0 + b * Cfg::PATCH), Cfg::PS, Cfg::PW * 16);
      if (elect_one()) {
#pragma unroll
        for (int t = 0; t < Cfg::ST; ++t) {
          if (ox0 + t * kTW >= G.Wo || (a.debug & 4)) break;
          const uint32_t d = tmem + (uint32_t)((b * Cfg::ST + t) * Cfg::ACC);
#pragma unroll
          for (int s = 0; s < Cfg::STEPS; ++s) {
            const uint64_t dah = da0 + (uint64_t)((Cfg::a_off(s) + t * kTW * 16) >> 4);
            const uint64_t dal = dah + (uint64_t)((Cfg::NP * Cfg::PS) >> 4);
            const uint64_t dbs = db0 + (uint64_t)(s * (kStepBytes >> 4));
            if constexpr (Cfg::SPLIT3) {
              mma_bf16(d, dah, dbs, id32, s > 0 ? 1u : 0u);      // xh * wh
              mma_bf16(d, dal, dbs, id32, 1u);                   // xl * wh
              mma_bf16(d, dah, dbs + (1024 >> 4), id32, 1u);     // xh * wl (B rows 32-63)
            } else {
              mma_bf16(d, dah, dbs, id64, s > 0 ? 1u : 0u);      // [xh*wh | xh*wl]
              mma_bf16(d, dal, dbs, id32, 1u);                   // + xl*wh
            }
          }
        }
        mma_commit(&B.empty[b]);
        mma_commit(&B.acc_full[b]);
        mbar_arrive(&B.acc_full[b]);
      }
      __syncwarp();
      PROF(pon, 10);
    }
  } else {
    // ================================================ epilogue (warps 0-7)
    // warp w reads TMEM lanes 32*(w%4).. of the tiles t = w/4, w/4 + 2, ...
    const int q = warp & 3, h = warp >> 2;
    const int gr = q * 4 + (lane >> 3), x = lane & 7;   // tile row / column of this lane
    const bool pon = tid == 0;
    PROF_START();
    for (int it = 0;; ++it) {
      const int b = it % Cfg::NB;
      const uint32_t use = (uint32_t)(it / Cfg::NB);
      mbar_wait(&B.acc_full[b], use & 1);
      PROF(pon, 12);
      const SuperTile t = B.desc[it % kDescRing];
      if (t.fout == nullptr) break;
      PROF(pon, 11);
      asm volatile("tcgen05.fence::after_thread_sync;");
      // all of this warp's tiles leave TMEM first (one wait), so the
      // accumulator set is released before the pooling math
      constexpr int TPW = Cfg::ST / 2;        // tiles per warp
      float v[TPW][32];
      bool ok[TPW];
#pragma unroll
      for (int u = 0; u < TPW; ++u) {
        const int tt = h + 2 * u;
        ok[u] = t.ox0 + tt * kTW < G.Wo && !(a.debug & 2) && t.pad_ == 0;
        if (ok[u]) {
          const uint32_t taddr =
              tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((b * Cfg::ST + tt) * Cfg::ACC);
          tmem_ld32(taddr, v[u]);
          if constexpr (!Cfg::SPLIT3) {
            float v1[32];
            tmem_ld32(taddr + 32, v1);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int ch = 0; ch < 32; ++ch) v[u][ch] = __fadd_rn(v[u][ch], v1[ch]);
          }
        }
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      if (kPair && crank) mbar_arrive_leader(&B.acc_empty[b]);
      else mbar_arrive(&B.acc_empty[b]);
      PROF(pon, 13);
#pragma unroll
      for (int u = 0; u < TPW; ++u) {
        if (!ok[u]) continue;
        const int tt = h + 2 * u;
        // 2x2 max pool before bias + ReLU (both monotone, bias is per channel),
        // as a halving butterfly: after the x-pair step a lane keeps 16
        // channels, after the row-pair step 8, and all four lanes of a window
        // store their 8 channels
        const bool xodd = lane & 1, yodd = (lane >> 3) & 1;
        float h16[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float send = xodd ? v[u][i] : v[u][16 + i];
          const float keep = xodd ? v[u][16 + i] : v[u][i];
          h16[i] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, 1));
        }
        float h8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float send = yodd ? h16[i] : h16[8 + i];
          const float keep = yodd ? h16[8 + i] : h16[i];
          h8[i] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, 8));
        }
        const int c0 = (xodd ? 16 : 0) + (yodd ? 8 : 0);
#pragma unroll
        for (int i = 0; i < 8; ++i) h8[i] = fmaxf(__fadd_rn(h8[i], B.bias[c0 + i]), 0.0f);
        const int oy = t.oy0 + (gr & ~1), ox = t.ox0 + tt * kTW + (x & ~1);
        if (oy < G.Ho && ox < G.Wo) {
          float4* dst = reinterpret_cast<float4*>(
              t.fout + ((int64_t)(oy >> 1) * G.Wp + (ox >> 1)) * kCout + c0);
          dst[0] = make_float4(h8[0], h8[1], h8[2], h8[3]);
          dst[1] = make_float4(h8[4], h8[5], h8[6], h8[7]);
        }
      }
      PROF(pon, 14);
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if constexpr (kPair) {
    cluster_sync();   // the peer's TMEM is written by this pair's MMAs until both are done
    if (warp == 0)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(kTmemCols));
  } else if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

using EncodeTiled = PFN_cuTensorMapEncodeTiled_v12000;

int tensor_map_encoder(EncodeTiled* fn) {
  static EncodeTiled enc = nullptr;
  if (enc == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    PB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (p == nullptr || q != cudaDriverEntryPointSuccess)
      return pb::fail(PB_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    enc = reinterpret_cast<EncodeTiled>(p);
  }
  *fn = enc;
  return PB_OK;
}

template <int MODE, int CIN>
int launch_conv(const pb_conv_actor& actor, const pb_resolved& res, cudaStream_t st, int sms) {
  using Cfg = ConvCfg<MODE, CIN>;
  const size_t smem = 1024 + Cfg::SMEM + sizeof(ConvBars);
  static_assert(1024 + Cfg::SMEM + sizeof(ConvBars) <= 227 * 1024, "conv smem");
  const int dev = pb::device();
  if (dev < 0) return PB_E_CUDA;
  static bool configured[pb::kMaxDevices] = {};
  if (!configured[dev]) {
    PB_CUDA(cudaFuncSetAttribute(conv_pool_kernel<MODE, CIN>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured[dev] = true;
  }
  const int Ho = actor.h + 2 * actor.pad - 4, Wo = actor.w + 2 * actor.pad - 4;
  const int64_t per_frame = (int64_t)((Ho + kTH - 1) / kTH) * ((Wo + Cfg::ST * kTW - 1) / (Cfg::ST * kTW));
  const int64_t total = per_frame * actor.frames * res.n_streams * res.n_iter;
  if (total >= (int64_t)1 << 31) return pb::fail(PB_E_UNSUPPORTED, "conv: too many tiles per launch");
  if (res.n_streams > kMaxStreams)
    return pb::fail(PB_E_UNSUPPORTED, "conv: more than 1024 streams per launch");
  const int grid = (int)std::min<int64_t>(total, sms);
  if (grid == 0) return PB_OK;
  CUtensorMap tmap{};
  if constexpr (MODE == 0) {
    // the input ring as [frames][H][W*3] fp32; box = one super-tile's raw rows
    const int64_t fbytes = (int64_t)actor.h * actor.w * CIN * 4;
    if (actor.in.stream_stride % fbytes || actor.in.span_bytes % fbytes ||
        (reinterpret_cast<uintptr_t>(actor.in.data) & 15))
      return pb::fail(PB_E_UNSUPPORTED, "conv: input ring is not a whole number of frames");
    EncodeTiled enc;
    if (int rc = tensor_map_encoder(&enc)) return rc;
    const cuuint64_t dims[3] = {(cuuint64_t)actor.w * CIN, (cuuint64_t)actor.h,
                                (cuuint64_t)(actor.in.stream_stride / fbytes * res.n_streams)};
    const cuuint64_t strides[2] = {(cuuint64_t)actor.w * CIN * 4, (cuuint64_t)fbytes};
    const cuuint32_t box[3] = {(cuuint32_t)Cfg::RAW_W, (cuuint32_t)kPH, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, actor.in.data, dims, strides,
                           box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return pb::fail(PB_E_CUDA, "conv: cuTensorMapEncodeTiled failed");
  }
  const int64_t n_units = (int64_t)res.n_streams * res.n_iter;
  UnitSpans* units = nullptr;
  int rc = pb::scratch(pb::kScratchConvUnits, sizeof(UnitSpans) * n_units,
                       reinterpret_cast<void**>(&units));
  if (rc) return rc;
  conv_units_kernel<<<(unsigned)((n_units + 255) / 256), 256, 0, st>>>(actor, res, units);
  PB_LAUNCHED("conv_units_kernel");
  if constexpr (MODE == 1) {
    // CTA pairs (cta_group::2; clusters of 2, an even grid): the default for
    // layer 2; PB_CONV_PAIR=0 selects the single-CTA kernel
    const char* pe = getenv("PB_CONV_PAIR");
    if (!(pe && pe[0] == '0') && grid >= 2) {
      static bool pconf[pb::kMaxDevices] = {};
      if (!pconf[dev]) {
        PB_CUDA(cudaFuncSetAttribute(conv_pool_kernel<MODE, CIN, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        pconf[dev] = true;
      }
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3((unsigned)(grid & ~1));
      cfg.blockDim = dim3(kConvThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      PB_CUDA(cudaLaunchKernelEx(&cfg, conv_pool_kernel<MODE, CIN, true>, actor, res,
                                 (const UnitSpans*)units, tmap));
      PB_LAUNCHED("conv_pool_kernel<pair>");
      return PB_OK;
    }
  }
  conv_pool_kernel<MODE, CIN><<<grid, kConvThreads, smem, st>>>(actor, res, units, tmap);
  PB_LAUNCHED("conv_pool_kernel");
  return PB_OK;
}

// ------------------------------------------------------------- dense (L3)
// out[f] = W x[f] + b, W [nout][nin], as a tcgen05 GEMM with the same bf16x3
// split as the convolutions: M = 128 frames gathered across the launch's
// live firings (rows of a tile may come from different firings and
// streams), N = [wh; wl] padded to 2 x 112 rows so one MMA gives xh*wh and
// xh*wl and a second (N = 112) adds xl*wh into the first half, K = nin in
// 64-wide chunks through a 3-stage ring: the weight chunk arrives by one
// cp.async.bulk (pre-split on the host, cnn_weights.dense_device_layout),
// the frame chunk is split to bf16 hi/lo by the converter warps.  When there
// are fewer M-tiles than SMs the K range is split across CTAs and the last
// CTA of a tile sums the partials in split order (deterministic).
#ifndef PB_DENSE_PF
#define PB_DENSE_PF 0   // 1: L2 prefetch of the frame chunk after next (measured: no gain)
#endif
constexpr int kDN = 112;                    // padded outputs per precision half
constexpr int kDKC = 64;                    // K per pipeline chunk (4 K16 steps)
#ifndef PB_DENSE_CPASYNC   // 1: frame chunks into a 3-deep shared-memory ring by cp.async
#define PB_DENSE_CPASYNC 0   // measured 0.201 vs 0.162 ms (the A / weight ring drops to 2 stages)
#endif
constexpr int kDStages = PB_DENSE_CPASYNC ? 2 : 3;   // A / weight ring
constexpr int kDRaw = 3;                             // raw frame chunks in flight (cp.async)
constexpr int kDStepBytes = 2 * kDN * 16 * 2;       // [wh; wl] 224 rows x 16 bf16
constexpr int kDChunkBytes = 4 * kDStepBytes;       // 28 KB
constexpr int kDAPiece = 128 * kDKC * 2;            // 16 KB (one precision piece)
constexpr int kDTmemCols = 256;
constexpr int kDEpiWarps = 4, kDMmaWarp = 4;       // warps 0-3 epilogue, 4 MMA, 5-12 converters
constexpr int kDEpiThreads = kDEpiWarps * 32;
#ifndef PB_DENSE_CVT
#define PB_DENSE_CVT 512   // 256: 0.168 ms, 512: 0.163 ms per 6144 frames
#endif
constexpr int kDCvtThreads = PB_DENSE_CVT;   // converter threads (frame loads in flight)
constexpr int kDItems = 512 / kDCvtThreads;        // (row, 16-K quarter) items per thread per chunk
constexpr int kDThreads = (kDEpiWarps + 1) * 32 + kDCvtThreads;

struct DenseSmem {
  uint8_t a[kDStages][2][kDAPiece];        // K-major core layout [row/8][kb][row%8][16 B]
  uint8_t b[kDStages][kDChunkBytes];
#if PB_DENSE_CPASYNC
  uint8_t raw[kDRaw][kDCvtThreads * 64];   // each converter thread's 16 floats of a chunk
#endif
  uint64_t full[kDStages], empty[kDStages], acc_full;
  uint32_t tmem_base;
  int last;
  const float* rowp[128];
  float* outp[128];
};

__global__ void __launch_bounds__(kDThreads, 1)
dense_kernel(pb_dense_actor a, pb_resolved res, float* partial, int* counters, int chunks_per_split) {
  extern __shared__ uint8_t smem_raw[];
  DenseSmem& S = *reinterpret_cast<DenseSmem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mt = blockIdx.x, split = blockIdx.y, splits = gridDim.y;
  const int n_chunks = a.nin / kDKC;
  const int c0 = split * chunks_per_split;
  const int c1 = min(n_chunks, c0 + chunks_per_split);

  // ---- rows of this tile: the m-th frame over the live firings, stream-major
  if (tid < 128) {
    const int64_t m = (int64_t)mt * 128 + tid;
    const int64_t unit = m / a.frames;
    const int f = (int)(m % a.frames);
    const float* rp = nullptr;
    float* op = nullptr;
    int64_t acc = 0;
    for (int s = 0; s < res.n_streams; ++s) {
      const int cnt = pb::cond_count(res, a.cond, s);
      if (unit < acc + cnt) {
        const int n = pb::firing_iter(res, a.cond, s, (int)(unit - acc));
        rp = reinterpret_cast<const float*>(pb::span_ptr(a.in, res, s, n)) + (int64_t)f * a.nin;
        op = reinterpret_cast<float*>(pb::span_ptr(a.out, res, s, n)) + (int64_t)f * a.nout;
        break;
      }
      acc += cnt;
    }
    S.rowp[tid] = rp;
    S.outp[tid] = op;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&S.tmem_base)), "r"(kDTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int st = 0; st < kDStages; ++st) {
      mbar_init(&S.full[st], kDCvtThreads);
      mbar_init(&S.empty[st], 1);
    }
    mbar_init(&S.acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = S.tmem_base;
  bool any_row = false;
  for (int r = 0; r < 128 && !any_row; ++r) any_row = S.rowp[r] != nullptr;
  const uint8_t* wg = reinterpret_cast<const uint8_t*>(a.weights);

  if (!any_row) {
    // nothing to do (tile beyond the live frames)
  } else if (warp >= kDMmaWarp + 1) {
    // ================================================ converters + weight copies
    const int ct = tid - (kDMmaWarp + 1) * 32;
    // the next chunk's frame values are loaded while the current one is split
    // (registers double-buffered), so a chunk costs no global-load latency
    float4 nxt[kDItems][4];
    auto load_chunk = [&](int c) {
#pragma unroll
      for (int k = 0; k < kDItems; ++k) {
        const int i = ct + k * kDCvtThreads;
        const int r = i >> 2, q = i & 3;
        const float* rp = S.rowp[r];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          nxt[k][u] = rp != nullptr
                          ? __ldg(reinterpret_cast<const float4*>(rp + (int64_t)c * kDKC + 16 * q) + u)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    // chunk c + 2 is requested into L2 (no registers) while c + 1 is in
    // flight into registers: twice the frame bytes in flight per SM
    auto prefetch_chunk = [&](int c) {
#pragma unroll
      for (int k = 0; k < kDItems; ++k) {
        const int i = ct + k * kDCvtThreads;
        const int r = i >> 2, q = i & 3;
        const float* rp = S.rowp[r];
        if (PB_DENSE_PF && rp != nullptr && (q & 1) == 0)   // one request per 128-B line
          asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + (int64_t)c * kDKC + 16 * q));
      }
    };
#if PB_DENSE_CPASYNC
    static_assert(kDItems == 1, "cp.async ring: one item per converter thread");
    // this thread's 64 bytes of chunk c into raw slot `slot` (zero rows of
    // frames beyond the launch); one commit group per chunk, empty ones too
    auto issue = [&](int c, int slot) {
      if (c < c1) {
        const int r = ct >> 2, q = ct & 3;
        const float* rp = S.rowp[r];
        const float* src = rp != nullptr ? rp + (int64_t)c * kDKC + 16 * q : a.bias;
        const uint32_t dst = smem_u32(S.raw[slot] + ct * 64);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + 16 * u),
                       "l"(src + 4 * u), "r"(rp != nullptr ? 16 : 0)
                       : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue(c0, 0);
    issue(c0 + 1, 1);
#else
    if (c0 < c1) load_chunk(c0);
    if (c0 + 1 < c1) prefetch_chunk(c0 + 1);
#endif
    for (int c = c0, it = 0; c < c1; ++c, ++it) {
      const int st = it % kDStages;
      const uint32_t use = (uint32_t)(it / kDStages);
      float4 cur[kDItems][4];
#if PB_DENSE_CPASYNC
      issue(c + 2, (it + 2) % kDRaw);
      asm volatile("cp.async.wait_group 2;" ::: "memory");   // chunk c has landed
#pragma unroll
      for (int u = 0; u < 4; ++u)
        cur[0][u] = *reinterpret_cast<const float4*>(S.raw[it % kDRaw] + ct * 64 + 16 * u);
#else
#pragma unroll
      for (int k = 0; k < kDItems; ++k)
#pragma unroll
        for (int u = 0; u < 4; ++u) cur[k][u] = nxt[k][u];
      if (c + 2 < c1) prefetch_chunk(c + 2);
      if (c + 1 < c1) load_chunk(c + 1);
#endif
      mbar_wait(&S.empty[st], (use & 1) ^ 1);
      if (ct == 0) {
        mbar_arrive_tx(&S.full[st], kDChunkBytes);
        bulk_g2s(S.b[st], wg + (int64_t)c * kDChunkBytes, kDChunkBytes, &S.full[st]);
      }
      // 128 rows x 4 quarters of 16 K, 4 threads per row
#pragma unroll
      for (int k = 0; k < kDItems; ++k) {
        const int i = ct + k * kDCvtThreads;
        const int r = i >> 2, q = i & 3;
        float v[16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          v[4 * u] = cur[k][u].x; v[4 * u + 1] = cur[k][u].y;
          v[4 * u + 2] = cur[k][u].z; v[4 * u + 3] = cur[k][u].w;
        }
        uint4 h0, l0, h1, l1;
        split8(v, h0, l0);
        split8(v + 8, h1, l1);
        // K-blocks 2q and 2q+1 of row r
        const int o0 = ((r >> 3) * 8 + 2 * q) * 128 + (r & 7) * 16;
        *reinterpret_cast<uint4*>(S.a[st][0] + o0) = h0;
        *reinterpret_cast<uint4*>(S.a[st][0] + o0 + 128) = h1;
        *reinterpret_cast<uint4*>(S.a[st][1] + o0) = l0;
        *reinterpret_cast<uint4*>(S.a[st][1] + o0 + 128) = l1;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (ct != 0) mbar_arrive(&S.full[st]);
    }
  } else if (warp == kDMmaWarp) {
    // ================================================ MMA issue
    if (lane == 0) {
      const uint32_t id224 = idesc_bf16(2 * kDN), id112 = idesc_bf16(kDN);
      for (int c = c0, it = 0; c < c1; ++c, ++it) {
        const int st = it % kDStages;
        const uint32_t use = (uint32_t)(it / kDStages);
        mbar_wait(&S.full[st], use & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint64_t dah = sdesc(smem_u32(S.a[st][0]), 128, 1024);
        const uint64_t dal = sdesc(smem_u32(S.a[st][1]), 128, 1024);
        const uint64_t db = sdesc(smem_u32(S.b[st]), 128, 256);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ak = (uint64_t)(k * 256 >> 4), bk = (uint64_t)(k * kDStepBytes >> 4);
          mma_bf16(tmem, dah + ak, db + bk, id224, (it | k) ? 1u : 0u);
          mma_bf16(tmem, dal + ak, db + bk, id112, 1u);
        }
        mma_commit(&S.empty[st]);
      }
      mma_commit(&S.acc_full);
    }
    __syncwarp();
  } else {
    // ================================================ epilogue (warps 0-3)
    const int r = warp * 32 + lane;
    mbar_wait(&S.acc_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
    const int64_t m = (int64_t)mt * 128 + r;
    float* op = S.outp[r];
    float* mine = splits > 1 ? partial + ((int64_t)split * gridDim.x * 128 + m) * kDN : nullptr;
    // 32 outputs at a time: [xh*wh + xl*wh] + [xh*wl]
#pragma unroll 1
    for (int c = 0; c < kDN; c += 32) {
      float t0[32], t1[32];
      tmem_ld32(tl + c, t0);
      tmem_ld32(tl + kDN + c, t1);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int u = 0; u < 32; ++u) t0[u] = __fadd_rn(t0[u], t1[u]);
      if (splits == 1) {
        if (op != nullptr) {
#pragma unroll
          for (int u = 0; u < 32; ++u)
            if (c + u < a.nout) op[c + u] = __fadd_rn(t0[u], __ldg(a.bias + c + u));
        }
      } else {
#pragma unroll
        for (int u = 0; u < 32; u += 4)
          if (c + u < kDN)
            *reinterpret_cast<float4*>(mine + c + u) = make_float4(t0[u], t0[u + 1], t0[u + 2], t0[u + 3]);
      }
    }
    if (splits > 1) {
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"n"(kDEpiThreads));
      if (r == 0) S.last = (atomicAdd(counters + mt, 1) == splits - 1);
      asm volatile("bar.sync 1, %0;" ::"n"(kDEpiThreads));
      if (S.last) {
        __threadfence();
        // the tile's partials are [split][128 rows][kDN] contiguous: the 128
        // threads sum them as float4s (coalesced, every load independent) in
        // split order, then scatter each row's outputs to its frame
        constexpr int kQ = kDN / 4;                       // float4 per row
        const float4* pp = reinterpret_cast<const float4*>(partial) + (int64_t)mt * 128 * kQ;
        const int64_t split_stride = (int64_t)gridDim.x * 128 * kQ;
#pragma unroll 4
        for (int i = r; i < 128 * kQ; i += kDEpiThreads) {
          const int row = i / kQ, q = i - row * kQ;
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int sp = 0; sp < splits; ++sp) {
            const float4 v = __ldcg(pp + sp * split_stride + i);
            acc.x = __fadd_rn(acc.x, v.x); acc.y = __fadd_rn(acc.y, v.y);
            acc.z = __fadd_rn(acc.z, v.z); acc.w = __fadd_rn(acc.w, v.w);
          }
          float* orow = S.outp[row];
          if (orow != nullptr) {
            const float o4[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (4 * q + u < a.nout) orow[4 * q + u] = __fadd_rn(o4[u], __ldg(a.bias + 4 * q + u));
          }
        }
        if (r == 0) counters[mt] = 0;
      }
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kDTmemCols));
}

// ------------------------------------------------- classify / bypass merge
// Live chain input: logits = W5 relu(W4 relu(x) + b4) + b5; bypass input:
// every logit = marker.  Exactly one live input per firing.
__global__ void classify_kernel(pb_classify_actor a, pb_resolved res) {
  const int s = blockIdx.y;
  const int n = blockIdx.x;
  if (!pb::active(res, a.cond, s, n)) return;
  const bool chain = pb::active(res, a.chain.act_cond, s, n);
  const bool bypass = pb::active(res, a.bypass.act_cond, s, n);
  if (chain == bypass) {
    if (threadIdx.x == 0) atomicExch(a.error_flag, 1);
    return;
  }
  float* out = reinterpret_cast<float*>(pb::span_ptr(a.out, res, s, n));
  if (bypass) {
    for (int e = threadIdx.x; e < a.frames * a.nout; e += blockDim.x) out[e] = a.marker;
    return;
  }
  const float* x = reinterpret_cast<const float*>(pb::span_ptr(a.chain, res, s, n));
  // the firing's inputs (ReLU applied once) and both weight matrices are
  // staged in shared memory with coalesced loads; the dot products then run
  // from shared memory in the same order as before
  extern __shared__ float csm[];
  float* hid = csm;                                   // [frames][nhid]
  float* xs = hid + a.frames * a.nhid;                // [frames][nin], relu(x)
  const int ws = a.nin | 1;                           // odd row stride: conflict-free rows
  float* w4 = xs + a.frames * a.nin;                  // [nhid][ws]
  float* w5 = w4 + a.nhid * ws;                       // [nout][nhid]
  for (int e = threadIdx.x; e < a.frames * a.nin; e += blockDim.x) xs[e] = fmaxf(x[e], 0.f);
  for (int e = threadIdx.x; e < a.nhid * a.nin; e += blockDim.x)
    w4[(e / a.nin) * ws + e % a.nin] = a.w4[e];
  for (int e = threadIdx.x; e < a.nout * a.nhid; e += blockDim.x) w5[e] = a.w5[e];
  __syncthreads();
  for (int e = threadIdx.x; e < a.frames * a.nhid; e += blockDim.x) {
    const int f = e / a.nhid, h = e % a.nhid;
    float acc = a.b4[h];
    const float* wr = w4 + h * ws;
    const float* xr = xs + f * a.nin;
    for (int k = 0; k < a.nin; ++k) acc = fmaf(wr[k], xr[k], acc);
    hid[e] = fmaxf(acc, 0.f);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < a.frames * a.nout; e += blockDim.x) {
    const int f = e / a.nout, o = e % a.nout;
    float acc = a.b5[o];
    for (int k = 0; k < a.nhid; ++k) acc = fmaf(w5[o * a.nhid + k], hid[f * a.nhid + k], acc);
    out[e] = acc;
  }
}

}  // namespace

extern "C" {

int pb_conv_debug_counters(unsigned long long* out, int reset) {
  PB_CUDA(cudaMemcpyFromSymbol(out, g_conv_prof, sizeof(g_conv_prof)));
  if (reset) {
    static unsigned long long zero[kProfCtas][kProfSlots] = {};
    PB_CUDA(cudaMemcpyToSymbol(g_conv_prof, zero, sizeof(zero)));
  }
  return PB_OK;
}

int pb_fire_conv_pool(pb_conv_actor actor, pb_resolved res, void* stream) {
  if (res.n_iter == 0) return PB_OK;
  if (actor.cout != kCout) return pb::fail(PB_E_UNSUPPORTED, "conv: 32 output channels only");
  const int Ho = actor.h + 2 * actor.pad - 4, Wo = actor.w + 2 * actor.pad - 4;
  if (Ho < 2 || Wo < 2 || Ho % 2 || Wo % 2)
    return pb::fail(PB_E_UNSUPPORTED, "conv: output must be even-sized for the 2x2 pool");
  const int dev = pb::device();
  if (dev < 0) return PB_E_CUDA;
  static int sms_d[pb::kMaxDevices] = {};
  int& sms = sms_d[dev];
  if (sms == 0) PB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaStream_t st = pb::as_stream(stream);
  // default: the row-streaming kernel with A in TMEM (pb_conv_rows.cu);
  // PB_CONV_IMPL=tiles selects the round-1 tile kernel below
  const char* impl = getenv("PB_CONV_IMPL");
  if ((actor.cin == 3 || actor.cin == 32) && !(impl && impl[0] == 't')) {
    const int rc = pb::fire_conv_rows(actor, res, st, sms);
    if (rc != 1) return rc;   // 1: shape declined by the row kernel, use the tile kernel
  }
  int rc;
  switch (actor.cin) {
    case 3: rc = launch_conv<0, 3>(actor, res, st, sms); break;
    case 16: rc = launch_conv<1, 16>(actor, res, st, sms); break;
    case 32: rc = launch_conv<1, 32>(actor, res, st, sms); break;
    default: return pb::fail(PB_E_UNSUPPORTED, "conv: Cin must be 3, 16 or 32");
  }
  // the tile kernel does not record its output scale: a separate pass
  if (rc == PB_OK && actor.absmax_out) rc = pb::conv_absmax_out(actor, res, st);
  return rc;
}

int pb_fire_dense(pb_dense_actor actor, pb_resolved res, void* stream) {
  if (res.n_iter == 0) return PB_OK;
  if (actor.nout > kDN || actor.nin % kDKC != 0)
    return pb::fail(PB_E_UNSUPPORTED, "dense: nout <= 112 and nin a multiple of 64");
  const int dev = pb::device();
  if (dev < 0) return PB_E_CUDA;
  static int sms_d[pb::kMaxDevices] = {};
  int& sms = sms_d[dev];
  float* partial = nullptr;
  int* counters = nullptr;
  if (sms == 0) {
    PB_CUDA(cudaFuncSetAttribute(dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(sizeof(DenseSmem) + 1024)));
    PB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int64_t rows = (int64_t)res.n_streams * res.n_iter * actor.frames;
  const int m_tiles = (int)((rows + 127) / 128);
  const int n_chunks = actor.nin / kDKC;
  int splits = std::max(1, std::min({sms / std::max(1, m_tiles), 16, n_chunks}));
  const int cps = (n_chunks + splits - 1) / splits;
  splits = (n_chunks + cps - 1) / cps;
  cudaStream_t st = pb::as_stream(stream);
  if (splits > 1) {
    const size_t need = (size_t)splits * m_tiles * 128 * kDN * sizeof(float);
    int rc = pb::scratch(pb::kScratchDensePartial, need, reinterpret_cast<void**>(&partial));
    if (rc) return rc;
    // arrival counters: zero when allocated, left zero by each launch's last CTA
    rc = pb::scratch(pb::kScratchDenseCounters, sizeof(int) * m_tiles,
                     reinterpret_cast<void**>(&counters), true, st);
    if (rc) return rc;
  }
  dim3 grid(m_tiles, splits);
  dense_kernel<<<grid, kDThreads, sizeof(DenseSmem) + 1024, st>>>(actor, res, partial, counters,
                                                                      cps);
  PB_LAUNCHED("dense_kernel");
  return PB_OK;
}

int pb_fire_classify(pb_classify_actor actor, pb_resolved res, void* stream) {
  if (res.n_iter == 0) return PB_OK;
  dim3 grid(res.n_iter, res.n_streams);
  const size_t smem = sizeof(float) * ((size_t)actor.frames * actor.nhid +
                                       (size_t)actor.frames * actor.nin +
                                       (size_t)actor.nhid * (actor.nin | 1) +
                                       (size_t)actor.nout * actor.nhid);
  if (smem > 200 * 1024) return pb::fail(PB_E_UNSUPPORTED, "classify: layers too large");
  const int dev = pb::device();
  if (dev < 0) return PB_E_CUDA;
  static bool attr[pb::kMaxDevices] = {};
  if (!attr[dev]) {
    PB_CUDA(cudaFuncSetAttribute(classify_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 200 * 1024));
    attr[dev] = true;
  }
  classify_kernel<<<grid, 256, smem, pb::as_stream(stream)>>>(actor, res);
  PB_LAUNCHED("classify_kernel");
  return PB_OK;
}

}  // extern "C"
