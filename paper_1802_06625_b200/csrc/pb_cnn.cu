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
constexpr int kStages = 2;
constexpr int kThreadsConv = 128;
constexpr int kChunkFloats = kRows * kKC;        // A plane per chunk
constexpr int kWChunkFloats = kCout * kKC;       // W plane per chunk

struct __align__(1024) ConvSmem {
  float a_hi[kStages][kChunkFloats];
  float a_lo[kStages][kChunkFloats];
  float w_hi[kStages][kWChunkFloats];
  float w_lo[kStages][kWChunkFloats];
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

__device__ __forceinline__ int core_off(int row, int k) {  // float offset in a plane
  return ((row >> 3) * (kKC / 4) + (k >> 2)) * 32 + (row & 7) * 4 + (k & 3);
}

__device__ __forceinline__ void split(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = __fsub_rn(x, hi);
}

__global__ void __launch_bounds__(kThreadsConv, 2)
conv_pool_kernel(pb_conv_actor a, pb_resolved res) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  ConvSmem& sm = *reinterpret_cast<ConvSmem*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int H = a.h, W = a.w, Cin = a.cin, pad = a.pad;
  const int Ho = H + 2 * pad - 4, Wo = W + 2 * pad - 4;
  const int Hp = Ho / 2, Wp = Wo / 2;
  const int K = 25 * Cin;
  const int n_chunks = (K + kKC - 1) / kKC;
  const int64_t per_frame = (int64_t)Hp * Wp;
  const int64_t per_unit = (int64_t)a.frames * per_frame;          // pooled pixels per firing
  const int64_t tiles_per_unit = (per_unit + kPool - 1) / kPool;
  const int64_t total = (int64_t)res.n_streams * res.n_iter * tiles_per_unit;
  const int64_t in_frame_floats = (int64_t)H * W * Cin;
  const int64_t out_frame_floats = per_frame * kCout;

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

  uint32_t issued[kStages] = {0, 0};   // commits issued per stage (phase tracking)
  int stage = 0;

  for (int64_t w = blockIdx.x; w < total; w += gridDim.x) {
    const int64_t unit = w / tiles_per_unit;
    const int64_t tile = w % tiles_per_unit;
    const int s = (int)(unit / res.n_iter);
    const int j = (int)(unit % res.n_iter);
    if (j >= pb::cond_count(res, a.cond, s)) continue;   // uniform across the CTA
    const int n = pb::firing_iter(res, a.cond, s, j);
    const float* in = reinterpret_cast<const float*>(pb::span_ptr(a.in, res, s, n));
    float* out = reinterpret_cast<float*>(pb::span_ptr(a.out, res, s, n));

    // this thread's GEMM row: pooled pixel q = tid/4, window position tid%4
    const int64_t g = tile * kPool + (tid >> 2);
    const bool row_ok = g < per_unit;
    int frame = 0, oy = 0, ox = 0;
    if (row_ok) {
      frame = (int)(g / per_frame);
      const int p = (int)(g % per_frame);
      oy = 2 * (p / Wp) + ((tid >> 1) & 1);
      ox = 2 * (p % Wp) + (tid & 1);
    }
    const float* fin = in + frame * in_frame_floats;

    for (int c = 0; c < n_chunks; ++c) {
      // the stage's previous MMAs must have drained before it is rewritten
      if (issued[stage] > 0) mbar_wait(&sm.mma_done[stage], (issued[stage] - 1) & 1);
      float* ahi = sm.a_hi[stage];
      float* alo = sm.a_lo[stage];
      // ---- im2col gather of 32 K values for this row
      const int k0 = c * kKC;
      if (Cin % kKC == 0) {
        // one (ky, kx) tap per chunk: 32 contiguous channels
        const int tap = k0 / Cin, ci0 = k0 % Cin;
        const int iy = oy + tap / 5 - pad, ix = ox + tap % 5 - pad;
        const bool ok = row_ok && iy >= 0 && iy < H && ix >= 0 && ix < W;
        const float4* src = reinterpret_cast<const float4*>(fin + ((int64_t)iy * W + ix) * Cin + ci0);
#pragma unroll
        for (int q = 0; q < kKC / 4; ++q) {
          float4 v = ok ? __ldg(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
          float4 h, l;
          split(v.x, h.x, l.x);
          split(v.y, h.y, l.y);
          split(v.z, h.z, l.z);
          split(v.w, h.w, l.w);
          const int off = core_off(tid, 4 * q);
          *reinterpret_cast<float4*>(ahi + off) = h;
          *reinterpret_cast<float4*>(alo + off) = l;
        }
      } else {
#pragma unroll 4
        for (int q = 0; q < kKC / 4; ++q) {
          float v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = k0 + 4 * q + e;
            float x = 0.f;
            if (row_ok && k < K) {
              const int tap = k / Cin, ci = k % Cin;
              const int iy = oy + tap / 5 - pad, ix = ox + tap % 5 - pad;
              if (iy >= 0 && iy < H && ix >= 0 && ix < W) x = __ldg(fin + ((int64_t)iy * W + ix) * Cin + ci);
            }
            v[e] = x;
          }
          float4 h, l;
          split(v[0], h.x, l.x);
          split(v[1], h.y, l.y);
          split(v[2], h.z, l.z);
          split(v[3], h.w, l.w);
          const int off = core_off(tid, 4 * q);
          *reinterpret_cast<float4*>(ahi + off) = h;
          *reinterpret_cast<float4*>(alo + off) = l;
        }
      }
      // ---- weights of this chunk (pre-split, pre-laid-out on the host)
      {
        const float4* whi = reinterpret_cast<const float4*>(a.weights + (int64_t)c * 2 * kWChunkFloats);
        const float4* wlo = whi + kWChunkFloats / 4;
        float4* dhi = reinterpret_cast<float4*>(sm.w_hi[stage]);
        float4* dlo = reinterpret_cast<float4*>(sm.w_lo[stage]);
        for (int e = tid; e < kWChunkFloats / 4; e += kThreadsConv) {
          dhi[e] = __ldg(whi + e);
          dlo[e] = __ldg(wlo + e);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int ks = 0; ks < kKC / 8; ++ks) {
          const uint64_t dah = sdesc(ahi + ks * 64), dal = sdesc(alo + ks * 64);
          const uint64_t dwh = sdesc(sm.w_hi[stage] + ks * 64), dwl = sdesc(sm.w_lo[stage] + ks * 64);
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
      stage ^= 1;
    }
    // ---- epilogue: wait for the tile's last commit (it covers all MMAs)
    const int last = stage ^ 1;
    mbar_wait(&sm.mma_done[last], (issued[last] - 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t r[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    float v[32];
#pragma unroll
    for (int ch = 0; ch < 32; ++ch) {
      float x = fmaxf(__fadd_rn(__uint_as_float(r[ch]), __ldg(a.bias + ch)), 0.0f);
      x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 1));
      x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 2));
      v[ch] = x;
    }
    if ((tid & 3) == 0 && row_ok) {
      const int p = (int)(g % per_frame);
      float4* dst = reinterpret_cast<float4*>(out + frame * out_frame_floats + (int64_t)p * kCout);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    // TMEM reads done before the next tile's first MMA overwrites D
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
  }
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
  conv_pool_kernel<<<2 * sms, kThreadsConv, smem, pb::as_stream(stream)>>>(actor, res);
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
