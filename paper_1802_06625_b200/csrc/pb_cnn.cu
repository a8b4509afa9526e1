// CNN actors of the vision example: the only
// tensor-core path.  The reference package ships no DNN;
// the graph and its oracle are builder-defined (apps/vision.py,
// oracle/cnn.py) and parity is stated as a tolerance, not bit-exactness.
//
// conv_pool_kernel: 5x5 convolution (NHWC fp32, zero padding) + bias + ReLU
// + 2x2 max-pool as an implicit GEMM on tcgen05:
//   D[128 conv pixels x 32 channels] += A[128 x K] * W[32 x K]^T,
//   K = 25*Cin ordered (ky, kx, ci), chunks of 32.
// Rows are 32 pooled pixels x their 4 conv pixels, so a pool window is 4
// consecutive TMEM lanes of one warp.  Accuracy: split TF32 (3 MMAs,
// hi*hi + hi*lo + lo*hi with x = hi + lo exactly), ~1e-6 relative.
//   * all 4 warps gather the im2col chunk (hi and lo planes) into shared
//     memory in the UMMA K-major no-swizzle core-matrix layout
//     [row/8][k/4][row%8][k%4] (LBO = K-direction core stride 128 B,
//     SBO = row-direction core stride 1024 B; probed in tools/umma_probe.cu);
//   * weights are pre-split on the host into the same layout per chunk;
//   * one thread issues 12 tcgen05.mma (kind::tf32, M=128 N=32 K=8) per
//     chunk and commits them to the stage's mbarrier; two stages overlap the
//     next gather with the running MMAs;
//   * epilogue: tcgen05.ld 32 columns per lane, bias, ReLU, max over the
//     four lanes of a window (warp shuffles), one 128 B NHWC store.
#include <algorithm>

#include "pb_common.cuh"

namespace {

constexpr int kRows = 128;            // conv pixels per tile (GEMM M)
constexpr int kPool = kRows / 4;      // pooled pixels per tile
constexpr int kCout = 32;             // GEMM N
constexpr int kKC = 32;               // K per chunk
constexpr int kThreadsConv = 128;
constexpr int kChunkFloats = kRows * kKC;        // A plane per chunk
constexpr int kWChunkFloats = kCout * kKC;       // W plane per chunk
constexpr int kRawStride = kKC + 4;              // padded raw row (conflict-free LDS.128)
constexpr int kAhead = 4;                        // chunks in flight ahead of the split
constexpr int kRing = kAhead + 2;                // raw/W ring slots
constexpr int kStages = 2;                       // split A planes (MMA operands)

struct __align__(1024) ConvSmem {
  float a_hi[kStages][kChunkFloats];             // UMMA operand, K-major core layout
  float a_lo[kStages][kChunkFloats];
  float w[kRing][2][kWChunkFloats];              // pre-split weights (hi, lo), cp.async ring
  float raw[kRing][kRows * kRawStride];          // gathered im2col rows, cp.async ring
  uint64_t mma_done[kStages];
  uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t sdesc(const void* p) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) & 0x3FFFF) >> 4);
  d |= (uint64_t)(128 >> 4) << 16;                      // LBO: next core matrix along K
  d |= (uint64_t)(((kKC / 4) * 128) >> 4) << 32;        // SBO: next core matrix along rows
  d |= (uint64_t)1 << 46;                                // sm100 descriptor version
  return d;                                              // SWIZZLE_NONE, base offset 0
}

__device__ __forceinline__ uint32_t idesc_tf32() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kCout >> 3) << 17) |
         ((uint32_t)(kRows >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc_tf32()), "r"(acc));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t@!p bra W_%=;\n\t}" ::"r"(
          smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}

// cp.async with zero fill: copies src_bytes (0 or size) and zero-fills the rest
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ int core_off(int row, int k) {  // float offset in a plane
  return ((row >> 3) * (kKC / 4) + (k >> 2)) * 32 + (row & 7) * 4 + (k & 3);
}

__device__ __forceinline__ void split(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = __fsub_rn(x, hi);
}

// Geometry of one conv layer launch.
struct ConvGeom {
  int H, W, Cin, pad, Ho, Wo, Hp, Wp, K, n_chunks;
  int64_t per_frame, per_unit, tiles_per_unit, total, in_frame, out_frame;
};

__device__ __forceinline__ ConvGeom geom(const pb_conv_actor& a, const pb_resolved& res) {
  ConvGeom g;
  g.H = a.h; g.W = a.w; g.Cin = a.cin; g.pad = a.pad;
  g.Ho = g.H + 2 * g.pad - 4; g.Wo = g.W + 2 * g.pad - 4;
  g.Hp = g.Ho / 2; g.Wp = g.Wo / 2;
  g.K = 25 * g.Cin;
  g.n_chunks = (g.K + kKC - 1) / kKC;
  g.per_frame = (int64_t)g.Hp * g.Wp;
  g.per_unit = (int64_t)a.frames * g.per_frame;
  g.tiles_per_unit = (g.per_unit + kPool - 1) / kPool;
  g.total = (int64_t)res.n_streams * res.n_iter * g.tiles_per_unit;
  g.in_frame = (int64_t)g.H * g.W * g.Cin;
  g.out_frame = g.per_frame * kCout;
  return g;
}

// This thread's GEMM row of tile w: its input frame base and conv pixel.
struct RowCtx {
  const float* fin;   // input frame (nullptr: the tile is skipped)
  float* out;         // output span of the firing
  int64_t g;          // pooled pixel index within the firing
  bool ok;
  int oy, ox;
};

__device__ __forceinline__ bool tile_live(const pb_conv_actor& a, const pb_resolved& res,
                                          const ConvGeom& G, int64_t w) {
  const int64_t unit = w / G.tiles_per_unit;
  const int s = (int)(unit / res.n_iter), j = (int)(unit % res.n_iter);
  return j < pb::cond_count(res, a.cond, s);
}

__device__ __forceinline__ RowCtx row_ctx(const pb_conv_actor& a, const pb_resolved& res,
                                          const ConvGeom& G, int64_t w, int tid) {
  RowCtx r;
  const int64_t unit = w / G.tiles_per_unit, tile = w % G.tiles_per_unit;
  const int s = (int)(unit / res.n_iter), j = (int)(unit % res.n_iter);
  const int n = pb::firing_iter(res, a.cond, s, j);
  const float* in = reinterpret_cast<const float*>(pb::span_ptr(a.in, res, s, n));
  r.out = reinterpret_cast<float*>(pb::span_ptr(a.out, res, s, n));
  r.g = tile * kPool + (tid >> 2);
  r.ok = r.g < G.per_unit;
  int frame = 0;
  r.oy = r.ox = 0;
  if (r.ok) {
    frame = (int)(r.g / G.per_frame);
    const int p = (int)(r.g % G.per_frame);
    r.oy = 2 * (p / G.Wp) + ((tid >> 1) & 1);
    r.ox = 2 * (p % G.Wp) + (tid & 1);
  }
  r.fin = in + frame * G.in_frame;
  return r;
}

// Issue the asynchronous gather of chunk c of this thread's row (and its
// share of the chunk's pre-split weights) into ring slot `slot`.
__device__ __forceinline__ void prefetch(ConvSmem& sm, const pb_conv_actor& a, const ConvGeom& G,
                                         const RowCtx& r, int c, int slot, int tid) {
  float* dst = sm.raw[slot] + tid * kRawStride;
  const int k0 = c * kKC;
  if (G.Cin % kKC == 0) {
    const int tap = k0 / G.Cin, ci0 = k0 % G.Cin;
    const int iy = r.oy + tap / 5 - G.pad, ix = r.ox + tap % 5 - G.pad;
    const bool ok = r.ok && iy >= 0 && iy < G.H && ix >= 0 && ix < G.W;
    const float* src = ok ? r.fin + ((int64_t)iy * G.W + ix) * G.Cin + ci0 : r.fin;
#pragma unroll
    for (int q = 0; q < kKC / 4; ++q) cp_async16(dst + 4 * q, src + 4 * q, ok);
  } else {
#pragma unroll 8
    for (int kk = 0; kk < kKC; ++kk) {
      const int k = k0 + kk;
      bool ok = r.ok && k < G.K;
      const float* src = r.fin;
      if (ok) {
        const int tap = k / G.Cin, ci = k % G.Cin;
        const int iy = r.oy + tap / 5 - G.pad, ix = r.ox + tap % 5 - G.pad;
        ok = iy >= 0 && iy < G.H && ix >= 0 && ix < G.W;
        if (ok) src = r.fin + ((int64_t)iy * G.W + ix) * G.Cin + ci;
      }
      cp_async4(dst + kk, src, ok);
    }
  }
  const float4* wsrc = reinterpret_cast<const float4*>(a.weights + (int64_t)c * 2 * kWChunkFloats);
  float4* wdst = reinterpret_cast<float4*>(&sm.w[slot][0][0]);
#pragma unroll
  for (int e = tid; e < 2 * kWChunkFloats / 4; e += kThreadsConv) cp_async16(wdst + e, wsrc + e, true);
}

__global__ void __launch_bounds__(kThreadsConv, 1)
conv_pool_kernel(pb_conv_actor a, pb_resolved res) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  ConvSmem& sm = *reinterpret_cast<ConvSmem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5;
  const ConvGeom G = geom(a, res);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)),
                 "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sm.mma_done[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = sm.tmem_base;

  // The CTA's work is a linear sequence of (tile, chunk) steps over its live
  // tiles; the prefetcher runs kAhead steps ahead of the consumer.
  int64_t pf_tile = blockIdx.x - (int64_t)gridDim.x;   // prefetch cursor
  int pf_chunk = G.n_chunks;
  RowCtx pf_row{};
  auto advance_pf = [&]() -> bool {   // move the prefetch cursor one step
    if (++pf_chunk >= G.n_chunks) {
      pf_chunk = 0;
      do {
        pf_tile += gridDim.x;
      } while (pf_tile < G.total && !tile_live(a, res, G, pf_tile));
      if (pf_tile >= G.total) return false;
      pf_row = row_ctx(a, res, G, pf_tile, tid);
    }
    return true;
  };
  int64_t step_pf = 0;   // steps issued
  bool pf_more = true;
  for (int d = 0; d < kAhead; ++d) {
    pf_more = pf_more && advance_pf();
    if (pf_more) prefetch(sm, a, G, pf_row, pf_chunk, (int)(step_pf % kRing), tid);
    cp_commit();
    ++step_pf;
  }

  int64_t tile = blockIdx.x - (int64_t)gridDim.x;
  int64_t step = 0;
  uint32_t issued[kStages] = {0, 0};
  for (;;) {
    do {
      tile += gridDim.x;
    } while (tile < G.total && !tile_live(a, res, G, tile));
    if (tile >= G.total) break;
    const RowCtx r = row_ctx(a, res, G, tile, tid);
    for (int c = 0; c < G.n_chunks; ++c, ++step) {
      const int stage = (int)(step & 1);
      const int slot = (int)(step % kRing);
      // the MMAs of step-2 used A stage `stage` and ring slot (step-2)%kRing
      if (issued[stage] > 0) mbar_wait(&sm.mma_done[stage], (issued[stage] - 1) & 1);
      // refill the freed ring slot kAhead steps ahead
      pf_more = pf_more && advance_pf();
      if (pf_more) prefetch(sm, a, G, pf_row, pf_chunk, (int)(step_pf % kRing), tid);
      cp_commit();
      ++step_pf;
      cp_wait<kAhead>();    // this step's group has landed (own row + own W share)
      // split the own row into the MMA operand planes
      const float* raw = sm.raw[slot] + tid * kRawStride;
      float* ahi = sm.a_hi[stage];
      float* alo = sm.a_lo[stage];
#pragma unroll
      for (int q = 0; q < kKC / 4; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(raw + 4 * q);
        float4 h, l;
        split(v.x, h.x, l.x);
        split(v.y, h.y, l.y);
        split(v.z, h.z, l.z);
        split(v.w, h.w, l.w);
        const int off = core_off(tid, 4 * q);
        *reinterpret_cast<float4*>(ahi + off) = h;
        *reinterpret_cast<float4*>(alo + off) = l;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();   // all rows split, all W shares landed
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        const float* whi = sm.w[slot][0];
        const float* wlo = sm.w[slot][1];
#pragma unroll
        for (int ks = 0; ks < kKC / 8; ++ks) {
          const uint64_t dah = sdesc(ahi + ks * 64), dal = sdesc(alo + ks * 64);
          const uint64_t dwh = sdesc(whi + ks * 64), dwl = sdesc(wlo + ks * 64);
          mma_tf32(tmem, dah, dwh, (c | ks) ? 1u : 0u);
          mma_tf32(tmem, dah, dwl, 1u);
          mma_tf32(tmem, dal, dwh, 1u);
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&sm.mma_done[stage]))
            : "memory");
      }
      issued[stage] += 1;
    }
    // ---- epilogue: the tile's last commit covers all of its MMAs
    const int last = (int)((step - 1) & 1);
    mbar_wait(&sm.mma_done[last], (issued[last] - 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t v32[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v32[0]), "=r"(v32[1]), "=r"(v32[2]), "=r"(v32[3]), "=r"(v32[4]), "=r"(v32[5]),
          "=r"(v32[6]), "=r"(v32[7]), "=r"(v32[8]), "=r"(v32[9]), "=r"(v32[10]), "=r"(v32[11]),
          "=r"(v32[12]), "=r"(v32[13]), "=r"(v32[14]), "=r"(v32[15]), "=r"(v32[16]),
          "=r"(v32[17]), "=r"(v32[18]), "=r"(v32[19]), "=r"(v32[20]), "=r"(v32[21]),
          "=r"(v32[22]), "=r"(v32[23]), "=r"(v32[24]), "=r"(v32[25]), "=r"(v32[26]),
          "=r"(v32[27]), "=r"(v32[28]), "=r"(v32[29]), "=r"(v32[30]), "=r"(v32[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    float v[32];
#pragma unroll
    for (int ch = 0; ch < 32; ++ch) {
      float x = fmaxf(__fadd_rn(__uint_as_float(v32[ch]), __ldg(a.bias + ch)), 0.0f);
      x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 1));
      x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 2));
      v[ch] = x;
    }
    if ((tid & 3) == 0 && r.ok) {
      const int frame = (int)(r.g / G.per_frame);
      const int p = (int)(r.g % G.per_frame);
      float4* dst = reinterpret_cast<float4*>(r.out + frame * G.out_frame + (int64_t)p * kCout);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    // TMEM reads done before the next tile's first MMA overwrites D
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
  }
  cp_wait<0>();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}

// ------------------------------------------------------------- dense (L3)
// out[f][o] = b[o] + sum_k x[f][k] * w[o][k], k ascending (fp32 FMA, one
// accumulator per output: deterministic).  One CTA per firing: the firing's
// frames and 32-wide K slices of all weight rows are staged in shared memory,
// so each weight element is read once per firing.
constexpr int kDenseThreads = 256;
constexpr int kDenseKC = 32;
constexpr int kDenseMaxF = 32;
constexpr int kDenseMaxOut = 128;

__global__ void __launch_bounds__(kDenseThreads)
dense_kernel(pb_dense_actor a, pb_resolved res) {
  const int s = blockIdx.y;
  const int j = blockIdx.x;
  if (j >= pb::cond_count(res, a.cond, s)) return;
  const int n = pb::firing_iter(res, a.cond, s, j);
  const float* x = reinterpret_cast<const float*>(pb::span_ptr(a.in, res, s, n));
  float* out = reinterpret_cast<float*>(pb::span_ptr(a.out, res, s, n));
  __shared__ float xs[kDenseMaxF][kDenseKC + 1];
  __shared__ float ws[kDenseMaxOut][kDenseKC + 1];
  const int o = threadIdx.x % kDenseMaxOut;
  const int fg = threadIdx.x / kDenseMaxOut;                 // 0 or 1
  float acc[kDenseMaxF / 2];
#pragma unroll
  for (int i = 0; i < kDenseMaxF / 2; ++i) acc[i] = 0.f;
  for (int k0 = 0; k0 < a.nin; k0 += kDenseKC) {
    __syncthreads();
    for (int e = threadIdx.x; e < a.frames * kDenseKC; e += kDenseThreads) {
      const int f = e / kDenseKC, k = e % kDenseKC;
      xs[f][k] = k0 + k < a.nin ? __ldg(x + (int64_t)f * a.nin + k0 + k) : 0.f;
    }
    for (int e = threadIdx.x; e < a.nout * kDenseKC; e += kDenseThreads) {
      const int r = e / kDenseKC, k = e % kDenseKC;
      ws[r][k] = k0 + k < a.nin ? __ldg(a.weights + (int64_t)r * a.nin + k0 + k) : 0.f;
    }
    __syncthreads();
    if (o < a.nout) {
#pragma unroll 4
      for (int k = 0; k < kDenseKC; ++k) {
        const float wv = ws[o][k];
#pragma unroll
        for (int i = 0; i < kDenseMaxF / 2; ++i) {
          const int f = fg + 2 * i;
          if (f < a.frames) acc[i] = fmaf(xs[f][k], wv, acc[i]);
        }
      }
    }
  }
  if (o < a.nout) {
#pragma unroll
    for (int i = 0; i < kDenseMaxF / 2; ++i) {
      const int f = fg + 2 * i;
      if (f < a.frames) out[(int64_t)f * a.nout + o] = __fadd_rn(acc[i], a.bias[o]);
    }
  }
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
  extern __shared__ float hid[];   // [frames][nhid]
  for (int e = threadIdx.x; e < a.frames * a.nhid; e += blockDim.x) {
    const int f = e / a.nhid, h = e % a.nhid;
    float acc = a.b4[h];
    for (int k = 0; k < a.nin; ++k) acc = fmaf(a.w4[h * a.nin + k], fmaxf(x[f * a.nin + k], 0.f), acc);
    hid[e] = fmaxf(acc, 0.f);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < a.frames * a.nout; e += blockDim.x) {
    const int f = e / a.nout, o = e % a.nout;
    float acc = a.b5[o];
    for (int k = 0; k < a.nhid; ++k) acc = fmaf(a.w5[o * a.nhid + k], hid[f * a.nhid + k], acc);
    out[e] = acc;
  }
}

}  // namespace

extern "C" {

int pb_fire_conv_pool(pb_conv_actor actor, pb_resolved res, void* stream) {
  if (res.n_iter == 0) return PB_OK;
  if (actor.cout != kCout) return pb::fail(PB_E_UNSUPPORTED, "conv: 32 output channels only");
  const int Ho = actor.h + 2 * actor.pad - 4, Wo = actor.w + 2 * actor.pad - 4;
  if (Ho < 2 || Wo < 2 || Ho % 2 || Wo % 2)
    return pb::fail(PB_E_UNSUPPORTED, "conv: output must be even-sized for the 2x2 pool");
  if (actor.cin % kKC != 0 && actor.cin > kKC)
    return pb::fail(PB_E_UNSUPPORTED, "conv: Cin must be a multiple of 32 or < 32");
  const size_t smem = sizeof(ConvSmem) + 1024;
  static bool configured = false;
  static int sms = 0;
  if (!configured) {
    PB_CUDA(cudaFuncSetAttribute(conv_pool_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    int dev = 0;
    PB_CUDA(cudaGetDevice(&dev));
    PB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    configured = true;
  }
  conv_pool_kernel<<<sms, kThreadsConv, smem, pb::as_stream(stream)>>>(actor, res);
  PB_LAUNCHED("conv_pool_kernel");
  return PB_OK;
}

int pb_fire_dense(pb_dense_actor actor, pb_resolved res, void* stream) {
  if (res.n_iter == 0) return PB_OK;
  if (actor.frames > kDenseMaxF || actor.nout > kDenseMaxOut)
    return pb::fail(PB_E_UNSUPPORTED, "dense: at most 32 frames and 128 outputs per firing");
  dim3 grid(res.n_iter, res.n_streams);
  dense_kernel<<<grid, kDenseThreads, 0, pb::as_stream(stream)>>>(actor, res);
  PB_LAUNCHED("dense_kernel");
  return PB_OK;
}

int pb_fire_classify(pb_classify_actor actor, pb_resolved res, void* stream) {
  if (res.n_iter == 0) return PB_OK;
  dim3 grid(res.n_iter, res.n_streams);
  const size_t smem = sizeof(float) * actor.frames * actor.nhid;
  classify_kernel<<<grid, 256, smem, pb::as_stream(stream)>>>(actor, res);
  PB_LAUNCHED("classify_kernel");
  return PB_OK;
}

}  // extern "C"
