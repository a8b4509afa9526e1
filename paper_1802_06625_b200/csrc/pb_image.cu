// Image actors of the motion-detection app (apps/motion.py:29-71): 8-bit
// frames, integer arithmetic, bit-exact with the reference.  One CTA per
// firing (stream, iteration) of the epoch; the frame is staged in shared
// memory once and every output pixel is computed from it.
//
//   gauss_blur (motion.py:29-47): out = a; out[y][x] = (sum_{dy,dx} k[dy] k[dx]
//     a[y-2+dy][x-2+dx]) >> 8 for 2 <= y, x < side-2 with k = (1 4 6 4 1).  The
//     reference sums rows first, then columns, in int32: the same integer for
//     any order (max 255 * 256 < 2^31), and the shift of a non-negative sum
//     is the floor.
//   frame_diff_threshold (:50-58): 255 where |cur - prev| > threshold, else 0.
//   plus_median (:61-71): the middle of the sorted (centre, up, down, left,
//     right) for interior pixels; the 1-pixel border passes through.
#include "pb_common.cuh"

namespace {

constexpr int kImgThreads = 256;
#ifndef PB_IMG_FAST
#define PB_IMG_FAST 1
#endif
constexpr int kMaxSide = 128;
#ifndef PB_MED_PRMT
#define PB_MED_PRMT 1
#endif

__global__ void __launch_bounds__(kImgThreads)
image_kernel(pb_image_actor a, pb_resolved res) {
  const int s = blockIdx.y, j = blockIdx.x;
  if (j >= pb::cond_count(res, a.cond, s)) return;
  const int n = pb::firing_iter(res, a.cond, s, j);
  const int side = a.side, npx = side * side;
  __shared__ uint8_t fr[kMaxSide * kMaxSide];
  const uint8_t* in0 = pb::span_ptr(a.in[0], res, s, n);
  if (a.op == PB_IMG_DIFF) {
    const uint8_t* in1 = pb::span_ptr(a.in[1], res, s, n);
    const int thr = a.threshold;
    for (int w = threadIdx.x; w < npx / 4; w += kImgThreads) {
      const uint32_t c = reinterpret_cast<const uint32_t*>(in0)[w];
      const uint32_t p = reinterpret_cast<const uint32_t*>(in1)[w];
      uint32_t m = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int d = (int)((c >> (8 * b)) & 0xFF) - (int)((p >> (8 * b)) & 0xFF);
        if ((d < 0 ? -d : d) > thr) m |= 0xFFu << (8 * b);
      }
      for (int k = 0; k < a.n_out; ++k)
        if (pb::active(res, a.out[k].act_cond, s, n))
          reinterpret_cast<uint32_t*>(pb::span_ptr(a.out[k], res, s, n))[w] = m;
    }
    return;
  }
  for (int w = threadIdx.x; w < npx / 4; w += kImgThreads)
    reinterpret_cast<uint32_t*>(fr)[w] = reinterpret_cast<const uint32_t*>(in0)[w];
  __syncthreads();
  uint8_t* outs[PB_MAX_PORTS];
  int n_live = 0;
  for (int k = 0; k < a.n_out; ++k)
    if (pb::active(res, a.out[k].act_cond, s, n)) outs[n_live++] = pb::span_ptr(a.out[k], res, s, n);
  for (int w = threadIdx.x; w < npx / 4; w += kImgThreads) {
    uint32_t word = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int p = 4 * w + b, y = p / side, x = p % side;
      int v = fr[p];
      if (a.op == PB_IMG_BLUR) {
        if (y >= 2 && y < side - 2 && x >= 2 && x < side - 2) {
          const int k5[5] = {1, 4, 6, 4, 1};
          int acc = 0;
#pragma unroll
          for (int dy = 0; dy < 5; ++dy) {
            const uint8_t* row = fr + (y - 2 + dy) * side + (x - 2);
            const int r = row[0] + 4 * row[1] + 6 * row[2] + 4 * row[3] + row[4];
            acc += k5[dy] * r;
          }
          v = acc >> 8;
        }
      } else {   // PB_IMG_MEDIAN
        if (y >= 1 && y < side - 1 && x >= 1 && x < side - 1) {
          int q0 = v, q1 = fr[p - side], q2 = fr[p + side], q3 = fr[p - 1], q4 = fr[p + 1];
          // median of five: sorting network
#define PB_SW(a_, b_) { const int lo_ = min(a_, b_), hi_ = max(a_, b_); a_ = lo_; b_ = hi_; }
          PB_SW(q0, q1); PB_SW(q3, q4); PB_SW(q0, q3); PB_SW(q1, q4); PB_SW(q1, q2);
          PB_SW(q2, q3); PB_SW(q1, q2);
#undef PB_SW
          v = q2;
        }
      }
      word |= (uint32_t)v << (8 * b);
    }
    for (int k = 0; k < n_live; ++k) reinterpret_cast<uint32_t*>(outs[k])[w] = word;
  }
}

// Word-parallel path for power-of-two sides 8..128 (64 in the reference
// app): a thread owns 4-pixel words, 128 threads per firing.
//   blur: horizontal pass with __dp4a over byte windows assembled by
//     __byte_perm (taps 1 4 6 4 | 1), int16 rows in shared memory, then the
//     vertical pass on two packed 16-bit lanes per register (max 255*16*16 =
//     65280 fits a lane) -- the same integers as the reference's row-then-
//     column int32 sums, so the >> 8 is the same floor;
//   diff: __vabsdiffu4 + __vcmpgtu4 on 16 pixels per thread;
//   median: the 7-exchange network of the generic kernel on 4 byte lanes at
//     once (__vminu4 / __vmaxu4), left/right neighbours by __byte_perm.
constexpr int kFastThreads = 128;

// median of five per 16-bit lane (byte values), 10 VIMNMX.U16x2:
// median3(e, max(min(a,b), min(c,d)), min(max(a,b), max(c,d)))
__device__ __forceinline__ uint32_t med5_u16(uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                             uint32_t e) {
  const uint32_t f = __vmaxu2(__vminu2(a, b), __vminu2(c, d));
  const uint32_t g = __vminu2(__vmaxu2(a, b), __vmaxu2(c, d));
  return __vmaxu2(__vminu2(e, f), __vminu2(__vmaxu2(e, f), g));
}
// byte-wise median of five words: even and odd bytes as two u16x2 lane sets
__device__ __forceinline__ uint32_t med5(uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                         uint32_t e) {
#if PB_MED_PRMT
  auto ev = [](uint32_t x) { return __byte_perm(x, 0u, 0x4240); };   // bytes 0, 2
  auto od = [](uint32_t x) { return __byte_perm(x, 0u, 0x4341); };   // bytes 1, 3
  const uint32_t me = med5_u16(ev(a), ev(b), ev(c), ev(d), ev(e));
  const uint32_t mo = med5_u16(od(a), od(b), od(c), od(d), od(e));
  return __byte_perm(me, mo, 0x6240);   // pixels 0 (me.b0), 1 (mo.b0), 2 (me.b2), 3 (mo.b2)
#else
  constexpr uint32_t M = 0x00FF00FFu;
  const uint32_t ev = med5_u16(a & M, b & M, c & M, d & M, e & M);
  const uint32_t od = med5_u16((a >> 8) & M, (b >> 8) & M, (c >> 8) & M, (d >> 8) & M,
                               (e >> 8) & M);
  return ev | (od << 8);
#endif
}

// The median of five values that are each 0x00 or 0xFF is their majority, and
// for such bytes the bitwise majority of the five words is the per-byte one:
// the fused motion region's median runs on the threshold mask, which is only
// ever 0 or 255 per pixel (frame_diff_threshold), so it takes the med5 network
// with min = AND and max = OR (a handful of LOP3s per 4 pixels).
__device__ __forceinline__ uint32_t maj5(uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                         uint32_t e) {
  const uint32_t f = (a & b) | (c & d);   // max(min(a, b), min(c, d))
  const uint32_t g = (a | b) & (c | d);   // min(max(a, b), max(c, d))
  return (e & f) | ((e | f) & g);         // med3(e, f, g) with f <= g
}

// frames per CTA: the span addressing of each frame (ring index arithmetic)
// is done once per frame by one thread and shared, not by every thread
constexpr int kFPC = 4;

struct FramePtrs {
  const uint8_t* in0;
  const uint8_t* in1;
  uint32_t* o0;
  uint32_t* o1;
};

template <int LW>   // words per row = 1 << LW, side = 4 << LW (compile time)
__global__ void __launch_bounds__(kFastThreads)
image_fast_kernel(pb_image_actor a, pb_resolved res) {
  constexpr int lw = LW;
  const int s = blockIdx.y, tid = threadIdx.x;
  constexpr int W = 1 << lw, side = 4 * W, nw = side * W;
  __shared__ FramePtrs fp[kFPC];
  __shared__ int n_frames;
  if (tid < kFPC) {
    const int cnt = pb::cond_count(res, a.cond, s);
    const int j = blockIdx.x * kFPC + tid;
    if (tid == 0) n_frames = max(0, min(kFPC, cnt - (int)blockIdx.x * kFPC));
    if (j < cnt) {
      const int n = pb::firing_iter(res, a.cond, s, j);
      FramePtrs f{pb::span_ptr(a.in[0], res, s, n),
                  a.op == PB_IMG_DIFF ? pb::span_ptr(a.in[1], res, s, n) : nullptr, nullptr,
                  nullptr};
      // live outputs (at most two on this path: blur feeds f_cur and the
      // delayed f_prev)
      for (int k = 0; k < a.n_out; ++k)
        if (pb::active(res, a.out[k].act_cond, s, n)) {
          uint32_t* o = reinterpret_cast<uint32_t*>(pb::span_ptr(a.out[k], res, s, n));
          if (!f.o0) f.o0 = o;
          else f.o1 = o;
        }
      fp[tid] = f;
    }
  }
  __syncthreads();
  const int nf = n_frames;
  extern __shared__ uint4 img_smem[];
  uint32_t* fr = reinterpret_cast<uint32_t*>(img_smem);            // [side][W] words
  uint32_t* hs = fr + nw;                                          // [side][W][2] int16 pairs
  const int xw0 = tid & (W - 1);
  constexpr int rows = kFastThreads >> lw;
  uint4 pre[2];
  for (int f = 0; f < nf; ++f) {
    const FramePtrs P = fp[f];
    uint32_t* const o0 = P.o0;
    uint32_t* const o1 = P.o1;
    auto put = [&](int idx, uint32_t w) {
      if (o0) o0[idx] = w;
      if (o1) o1[idx] = w;
    };
    if (a.op == PB_IMG_DIFF) {
      const uint4* c4 = reinterpret_cast<const uint4*>(P.in0);
      const uint4* p4 = reinterpret_cast<const uint4*>(P.in1);
      const int thr = a.threshold;
      const uint32_t t4 = (uint32_t)min(max(thr, 0), 255) * 0x01010101u;
      auto m4 = [&](uint32_t c, uint32_t p) -> uint32_t {
        if (thr < 0) return 0xFFFFFFFFu;
        if (thr >= 255) return 0u;
        return __vcmpgtu4(__vabsdiffu4(c, p), t4);
      };
      for (int i = tid; i < nw / 4; i += kFastThreads) {
        const uint4 c = c4[i], p = p4[i];
        const uint4 m = make_uint4(m4(c.x, p.x), m4(c.y, p.y), m4(c.z, p.z), m4(c.w, p.w));
        if (o0) reinterpret_cast<uint4*>(o0)[i] = m;
        if (o1) reinterpret_cast<uint4*>(o1)[i] = m;
      }
      continue;
    }
    // this frame into shared memory: its words were loaded into registers
    // while the previous frame was computed (side <= 64: at most 2 uint4 per
    // thread; larger sides load here)
    if (f > 0) __syncthreads();   // the previous frame's readers are done with fr / hs
    if (nw / 4 <= 2 * kFastThreads) {
      if (f == 0) {
#pragma unroll
        for (int q = 0; q < 2; ++q)
          if (tid + q * kFastThreads < nw / 4)
            pre[q] = reinterpret_cast<const uint4*>(P.in0)[tid + q * kFastThreads];
      }
#pragma unroll
      for (int q = 0; q < 2; ++q)
        if (tid + q * kFastThreads < nw / 4) img_smem[tid + q * kFastThreads] = pre[q];
      if (f + 1 < nf) {   // next frame's words in flight during this frame's math
#pragma unroll
        for (int q = 0; q < 2; ++q)
          if (tid + q * kFastThreads < nw / 4)
            pre[q] = reinterpret_cast<const uint4*>(fp[f + 1].in0)[tid + q * kFastThreads];
      }
    } else {
      for (int i = tid; i < nw / 4; i += kFastThreads)
        img_smem[i] = reinterpret_cast<const uint4*>(P.in0)[i];
    }
    __syncthreads();
    if (a.op == PB_IMG_BLUR) {
      constexpr uint32_t K4 = 0x04060401u;   // taps 1 4 6 4 on bytes 0..3 of a window
      for (int y = tid >> lw; y < side; y += rows) {
        const int xw = xw0;
        const uint32_t* row = fr + y * W;
        const uint32_t wa = xw > 0 ? row[xw - 1] : 0u, wb = row[xw];
        const uint32_t wc = xw < W - 1 ? row[xw + 1] : 0u;
        const uint32_t h0 = __dp4a(__byte_perm(wa, wb, 0x5432), K4, (wb >> 16) & 0xFFu);
        const uint32_t h1 = __dp4a(__byte_perm(wa, wb, 0x6543), K4, wb >> 24);
        const uint32_t h2 = __dp4a(wb, K4, wc & 0xFFu);
        const uint32_t h3 = __dp4a(__byte_perm(wb, wc, 0x4321), K4, (wc >> 8) & 0xFFu);
        reinterpret_cast<uint2*>(hs)[y * W + xw] = make_uint2(h0 | (h1 << 16), h2 | (h3 << 16));
      }
      __syncthreads();
      for (int y = tid >> lw; y < side; y += rows) {
        const int xw = xw0;
        const uint32_t orig = fr[y * W + xw];
        uint32_t word = orig;
        if (y >= 2 && y < side - 2) {
          const uint2* h = reinterpret_cast<const uint2*>(hs) + (y - 2) * W + xw;
          const uint2 r0 = h[0], r1 = h[W], r2 = h[2 * W], r3 = h[3 * W], r4 = h[4 * W];
          uint32_t lo = r0.x + 4u * r1.x + 6u * r2.x + 4u * r3.x + r4.x;
          uint32_t hi = r0.y + 4u * r1.y + 6u * r2.y + 4u * r3.y + r4.y;
          lo = (lo >> 8) & 0x00FF00FFu;
          hi = (hi >> 8) & 0x00FF00FFu;
          word = __byte_perm(lo, hi, 0x6420);
          if (xw == 0) word = __byte_perm(word, orig, 0x3254);       // x = 0, 1 pass through
          if (xw == W - 1) word = __byte_perm(word, orig, 0x7610);   // x = side-2, side-1
        }
        put(y * W + xw, word);
      }
      continue;
    }
    // PB_IMG_MEDIAN
    for (int y = tid >> lw; y < side; y += rows) {
      const int xw = xw0;
      const uint32_t c = fr[y * W + xw];
      uint32_t word = c;
      if (y >= 1 && y < side - 1) {
        const uint32_t up = fr[(y - 1) * W + xw], dn = fr[(y + 1) * W + xw];
        const uint32_t pl = xw > 0 ? fr[y * W + xw - 1] : 0u;
        const uint32_t nx = xw < W - 1 ? fr[y * W + xw + 1] : 0u;
        const uint32_t lf = __byte_perm(pl, c, 0x6543), rt = __byte_perm(c, nx, 0x4321);
        word = med5(c, up, dn, lf, rt);
        if (xw == 0) word = __byte_perm(word, c, 0x3214);       // x = 0 passes through
        if (xw == W - 1) word = __byte_perm(word, c, 0x7210);   // x = side-1
      }
      put(y * W + xw, word);
    }
  }
}

// ---------------------------------------------- fused motion region
// blur -> diff(cur, prev) -> median per frame, frames of one stream in order
// (kMRF per CTA): the word-parallel arithmetic of image_fast_kernel, with the
// blurred frame and the mask kept in shared memory.
#ifndef PB_MRF
#define PB_MRF 16
#endif
constexpr int kMRF = PB_MRF;   // frames per CTA (one extra blur per run)
#ifndef PB_MR_MAJ   // the region's median on the 0/255 mask as a bitwise majority
#define PB_MR_MAJ 1
#endif
#ifndef PB_MR_REG
#define PB_MR_REG 1   // sides 32 / 64: the register form below
#endif
#ifndef PB_MR_T64
#define PB_MR_T64 128   // threads per CTA of the register form at side 64 (8 rows each; 256: 0.377 vs 0.335 ms)
#endif

template <int LW>
__device__ __forceinline__ void mr_blur(const uint32_t* fr, uint32_t* hs, uint32_t* out, int tid) {
  constexpr int W = 1 << LW, side = 4 * W, rows = kFastThreads >> LW;
  constexpr uint32_t K4 = 0x04060401u;
  const int xw = tid & (W - 1);
  for (int y = tid >> LW; y < side; y += rows) {
    const uint32_t* row = fr + y * W;
    const uint32_t wa = xw > 0 ? row[xw - 1] : 0u, wb = row[xw];
    const uint32_t wc = xw < W - 1 ? row[xw + 1] : 0u;
    const uint32_t h0 = __dp4a(__byte_perm(wa, wb, 0x5432), K4, (wb >> 16) & 0xFFu);
    const uint32_t h1 = __dp4a(__byte_perm(wa, wb, 0x6543), K4, wb >> 24);
    const uint32_t h2 = __dp4a(wb, K4, wc & 0xFFu);
    const uint32_t h3 = __dp4a(__byte_perm(wb, wc, 0x4321), K4, (wc >> 8) & 0xFFu);
    reinterpret_cast<uint2*>(hs)[y * W + xw] = make_uint2(h0 | (h1 << 16), h2 | (h3 << 16));
  }
  __syncthreads();
  for (int y = tid >> LW; y < side; y += rows) {
    const uint32_t orig = fr[y * W + xw];
    uint32_t word = orig;
    if (y >= 2 && y < side - 2) {
      const uint2* h = reinterpret_cast<const uint2*>(hs) + (y - 2) * W + xw;
      const uint2 r0 = h[0], r1 = h[W], r2 = h[2 * W], r3 = h[3 * W], r4 = h[4 * W];
      uint32_t lo = r0.x + 4u * r1.x + 6u * r2.x + 4u * r3.x + r4.x;
      uint32_t hi = r0.y + 4u * r1.y + 6u * r2.y + 4u * r3.y + r4.y;
      lo = (lo >> 8) & 0x00FF00FFu;
      hi = (hi >> 8) & 0x00FF00FFu;
      word = __byte_perm(lo, hi, 0x6420);
      if (xw == 0) word = __byte_perm(word, orig, 0x3254);
      if (xw == W - 1) word = __byte_perm(word, orig, 0x7610);
    }
    out[y * W + xw] = word;
  }
}

template <int LW>
__global__ void __launch_bounds__(kFastThreads)
motion_region_kernel(pb_motion_region r, pb_resolved res) {
  constexpr int W = 1 << LW, side = 4 * W, nw = side * W, rows = kFastThreads >> LW;
  const int s = blockIdx.y, tid = threadIdx.x;
  const int n0 = blockIdx.x * kMRF, n1 = min(res.n_iter, n0 + kMRF);
  if (n0 >= res.n_iter) return;
  extern __shared__ uint4 mr_smem[];
  uint32_t* fr = reinterpret_cast<uint32_t*>(mr_smem);   // [nw] source frame
  uint32_t* hs = fr + nw;                                 // [2 nw] horizontal sums
  uint32_t* bl[2] = {hs + 2 * nw, hs + 3 * nw};           // blurred frames (cur / prev)
  uint32_t* mk = hs + 4 * nw;                             // [nw] mask
  const int thr = r.threshold;
  const uint32_t t4 = (uint32_t)min(max(thr, 0), 255) * 0x01010101u;
  auto load = [&](const uint8_t* src, uint32_t* dst) {
    for (int i = tid; i < nw / 4; i += kFastThreads)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  };
  // the frame before n0: the delayed channel's token at the epoch's first
  // iteration (its initial token, or the previous epoch's last blurred
  // frame), else this epoch's source frame n0 - 1 blurred again
  int cur = 0;
  if (n0 == 0) {
    load(pb::span_ptr(r.prev_in, res, s, 0), bl[1]);
  } else {
    load(pb::span_ptr(r.in, res, s, n0 - 1), fr);
    __syncthreads();
    mr_blur<LW>(fr, hs, bl[1], tid);
  }
  // the next frame's words are in flight (registers) while this one is computed
  constexpr int kPre = (nw / 4 + kFastThreads - 1) / kFastThreads;
  uint4 pre[kPre];
  auto fetch = [&](int n) {
    const uint4* src = reinterpret_cast<const uint4*>(pb::span_ptr(r.in, res, s, n));
#pragma unroll
    for (int q = 0; q < kPre; ++q)
      if (tid + q * kFastThreads < nw / 4) pre[q] = src[tid + q * kFastThreads];
  };
  fetch(n0);
  for (int n = n0; n < n1; ++n) {
    __syncthreads();   // fr / hs free again
#pragma unroll
    for (int q = 0; q < kPre; ++q)
      if (tid + q * kFastThreads < nw / 4) reinterpret_cast<uint4*>(fr)[tid + q * kFastThreads] = pre[q];
    if (n + 1 < n1) fetch(n + 1);
    __syncthreads();
    uint32_t* const c = bl[cur];
    const uint32_t* const pv = bl[cur ^ 1];
    mr_blur<LW>(fr, hs, c, tid);
    __syncthreads();
    for (int i = tid; i < nw; i += kFastThreads)
      mk[i] = thr < 0 ? 0xFFFFFFFFu : thr >= 255 ? 0u : __vcmpgtu4(__vabsdiffu4(c[i], pv[i]), t4);
    if (n == res.n_iter - 1) {   // the next epoch's first "prev"
      uint32_t* po = reinterpret_cast<uint32_t*>(pb::span_ptr(r.prev_out, res, s, n));
      for (int i = tid; i < nw / 4; i += kFastThreads)
        reinterpret_cast<uint4*>(po)[i] = reinterpret_cast<const uint4*>(c)[i];
    }
    __syncthreads();
    uint32_t* o = reinterpret_cast<uint32_t*>(pb::span_ptr(r.out, res, s, n));
    const int xw = tid & (W - 1);
    for (int y = tid >> LW; y < side; y += rows) {
      const uint32_t cw = mk[y * W + xw];
      uint32_t word = cw;
      if (y >= 1 && y < side - 1) {
        const uint32_t up = mk[(y - 1) * W + xw], dn = mk[(y + 1) * W + xw];
        const uint32_t pl = xw > 0 ? mk[y * W + xw - 1] : 0u;
        const uint32_t nx = xw < W - 1 ? mk[y * W + xw + 1] : 0u;
        const uint32_t lf = __byte_perm(pl, cw, 0x6543), rt = __byte_perm(cw, nx, 0x4321);
        word = PB_MR_MAJ ? maj5(cw, up, dn, lf, rt) : med5(cw, up, dn, lf, rt);
        if (xw == 0) word = __byte_perm(word, cw, 0x3214);
        if (xw == W - 1) word = __byte_perm(word, cw, 0x7210);
      }
      o[y * W + xw] = word;
    }
    cur ^= 1;
  }
}

// Register form for sides 32 and 64: thread (band, xw) owns word column xw
// of R consecutive rows for the whole run, so the blurred frame, the previous
// one and the mask never leave registers; horizontal neighbours come from
// warp shuffles, and only the two rows above and below each band cross
// threads (a double-buffered shared-memory halo, two barriers per frame).
template <int LW, int T>
__global__ void __launch_bounds__(T)
motion_region_reg_kernel(pb_motion_region r, pb_resolved res) {
  constexpr int W = 1 << LW, side = 4 * W, bands = T / W, R = side / bands;
  static_assert(R >= 2 && R * bands == side, "register motion region: sides 32, 64");
  const int s = blockIdx.y, tid = threadIdx.x;
  const int n0 = blockIdx.x * kMRF, n1 = min(res.n_iter, n0 + kMRF);
  if (n0 >= res.n_iter) return;
  const int xw = tid & (W - 1), band = tid >> LW, y0 = band * R;
  __shared__ uint2 hh[2][bands][4][W];      // blur: rows y0, y0+1, y0+R-2, y0+R-1 of each band
  __shared__ uint32_t mh[2][bands][2][W];   // mask: rows y0, y0+R-1
  const int thr = r.threshold;
  const uint32_t t4 = (uint32_t)min(max(thr, 0), 255) * 0x01010101u;
  auto fetch = [&](const uint8_t* src, uint32_t (&x)[R]) {
#pragma unroll
    for (int j = 0; j < R; ++j) x[j] = reinterpret_cast<const uint32_t*>(src)[(y0 + j) * W + xw];
  };
  int hb = 0;   // halo buffer parity
  // the blur of one frame held in x (every thread takes part: two barriers)
  auto blur = [&](const uint32_t (&x)[R], uint32_t (&out)[R]) {
    constexpr uint32_t K4 = 0x04060401u;
    uint2 h[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      uint32_t wa = __shfl_up_sync(0xffffffffu, x[j], 1, W);
      uint32_t wc = __shfl_down_sync(0xffffffffu, x[j], 1, W);
      if (xw == 0) wa = 0u;
      if (xw == W - 1) wc = 0u;
      const uint32_t wb = x[j];
      const uint32_t h0 = __dp4a(__byte_perm(wa, wb, 0x5432), K4, (wb >> 16) & 0xFFu);
      const uint32_t h1 = __dp4a(__byte_perm(wa, wb, 0x6543), K4, wb >> 24);
      const uint32_t h2 = __dp4a(wb, K4, wc & 0xFFu);
      const uint32_t h3 = __dp4a(__byte_perm(wb, wc, 0x4321), K4, (wc >> 8) & 0xFFu);
      h[j] = make_uint2(h0 | (h1 << 16), h2 | (h3 << 16));
    }
    hh[hb][band][0][xw] = h[0];
    hh[hb][band][1][xw] = h[1];
    hh[hb][band][2][xw] = h[R - 2];
    hh[hb][band][3][xw] = h[R - 1];
    __syncthreads();
    const uint2 zero = make_uint2(0u, 0u);
    const uint2 a2 = band > 0 ? hh[hb][band - 1][2][xw] : zero;   // row y0 - 2
    const uint2 a1 = band > 0 ? hh[hb][band - 1][3][xw] : zero;   // row y0 - 1
    const uint2 b1 = band < bands - 1 ? hh[hb][band + 1][0][xw] : zero;   // row y0 + R
    const uint2 b2 = band < bands - 1 ? hh[hb][band + 1][1][xw] : zero;   // row y0 + R + 1
    hb ^= 1;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int y = y0 + j;
      uint32_t word = x[j];
      if (y >= 2 && y < side - 2) {
        const uint2 r0 = j >= 2 ? h[j - 2] : (j == 1 ? a1 : a2);
        const uint2 r1 = j >= 1 ? h[j - 1] : a1;
        const uint2 r3 = j + 1 < R ? h[j + 1] : b1;
        const uint2 r4 = j + 2 < R ? h[j + 2] : (j + 1 < R ? b1 : b2);
        const uint2 r2 = h[j];
        uint32_t lo = r0.x + 4u * r1.x + 6u * r2.x + 4u * r3.x + r4.x;
        uint32_t hi = r0.y + 4u * r1.y + 6u * r2.y + 4u * r3.y + r4.y;
        lo = (lo >> 8) & 0x00FF00FFu;
        hi = (hi >> 8) & 0x00FF00FFu;
        word = __byte_perm(lo, hi, 0x6420);
        if (xw == 0) word = __byte_perm(word, x[j], 0x3254);
        if (xw == W - 1) word = __byte_perm(word, x[j], 0x7610);
      }
      out[j] = word;
    }
  };
  uint32_t x[R], xn[R], cur[R], prev[R];
  if (n0 == 0) {
    fetch(pb::span_ptr(r.prev_in, res, s, 0), prev);
  } else {
    fetch(pb::span_ptr(r.in, res, s, n0 - 1), x);
    blur(x, prev);
  }
  fetch(pb::span_ptr(r.in, res, s, n0), xn);
  for (int n = n0; n < n1; ++n) {
#pragma unroll
    for (int j = 0; j < R; ++j) x[j] = xn[j];
    if (n + 1 < n1) fetch(pb::span_ptr(r.in, res, s, n + 1), xn);
    blur(x, cur);
    uint32_t mk[R];
#pragma unroll
    for (int j = 0; j < R; ++j)
      mk[j] = thr < 0 ? 0xFFFFFFFFu : thr >= 255 ? 0u : __vcmpgtu4(__vabsdiffu4(cur[j], prev[j]), t4);
    if (n == res.n_iter - 1) {   // the next epoch's first "prev"
      uint32_t* po = reinterpret_cast<uint32_t*>(pb::span_ptr(r.prev_out, res, s, n));
#pragma unroll
      for (int j = 0; j < R; ++j) po[(y0 + j) * W + xw] = cur[j];
    }
    mh[hb][band][0][xw] = mk[0];
    mh[hb][band][1][xw] = mk[R - 1];
    __syncthreads();
    const uint32_t above = band > 0 ? mh[hb][band - 1][1][xw] : 0u;
    const uint32_t below = band < bands - 1 ? mh[hb][band + 1][0][xw] : 0u;
    hb ^= 1;
    uint32_t* o = reinterpret_cast<uint32_t*>(pb::span_ptr(r.out, res, s, n));
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int y = y0 + j;
      const uint32_t cw = mk[j];
      uint32_t pl = __shfl_up_sync(0xffffffffu, cw, 1, W);
      uint32_t nx = __shfl_down_sync(0xffffffffu, cw, 1, W);
      uint32_t word = cw;
      if (y >= 1 && y < side - 1) {
        const uint32_t up = j > 0 ? mk[j - 1] : above, dn = j + 1 < R ? mk[j + 1] : below;
        if (xw == 0) pl = 0u;
        if (xw == W - 1) nx = 0u;
        const uint32_t lf = __byte_perm(pl, cw, 0x6543), rt = __byte_perm(cw, nx, 0x4321);
        word = PB_MR_MAJ ? maj5(cw, up, dn, lf, rt) : med5(cw, up, dn, lf, rt);
        if (xw == 0) word = __byte_perm(word, cw, 0x3214);
        if (xw == W - 1) word = __byte_perm(word, cw, 0x7210);
      }
      o[y * W + xw] = word;
    }
#pragma unroll
    for (int j = 0; j < R; ++j) prev[j] = cur[j];
  }
}

}  // namespace

extern "C" {

int pb_fire_motion_region(pb_motion_region r, pb_resolved res, void* stream) {
  if (res.n_iter == 0) return PB_OK;
  const int side = r.side;
  if (side < 8 || side > kMaxSide || (side & (side - 1)))
    return pb::fail(PB_E_UNSUPPORTED, "motion region: power-of-two sides 8..128");
  const size_t smem = (size_t)side * side * 6;   // frame, sums (2x), two blurred, mask
  static bool attr[pb::kMaxDevices] = {};
  const int dev = pb::device();
  if (dev < 0) return PB_E_CUDA;
  if (!attr[dev]) {
    PB_CUDA(cudaFuncSetAttribute(motion_region_kernel<5>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 6 * kMaxSide * kMaxSide));
    attr[dev] = true;
  }
  dim3 grid((res.n_iter + kMRF - 1) / kMRF, res.n_streams);
  cudaStream_t st = pb::as_stream(stream);
  switch (side) {
    case 8: motion_region_kernel<1><<<grid, kFastThreads, smem, st>>>(r, res); break;
    case 16: motion_region_kernel<2><<<grid, kFastThreads, smem, st>>>(r, res); break;
    case 32:
      if (PB_MR_REG) motion_region_reg_kernel<3, 128><<<grid, 128, 0, st>>>(r, res);
      else motion_region_kernel<3><<<grid, kFastThreads, smem, st>>>(r, res);
      break;
    case 64:
      if (PB_MR_REG) motion_region_reg_kernel<4, PB_MR_T64><<<grid, PB_MR_T64, 0, st>>>(r, res);
      else motion_region_kernel<4><<<grid, kFastThreads, smem, st>>>(r, res);
      break;
    default: motion_region_kernel<5><<<grid, kFastThreads, smem, st>>>(r, res); break;
  }
  PB_LAUNCHED("motion_region_kernel");
  return PB_OK;
}

int pb_fire_image(pb_image_actor actor, pb_resolved res, void* stream) {
  if (res.n_iter == 0) return PB_OK;
  if (actor.side < 5 || actor.side > kMaxSide || (actor.side * actor.side) % 4)
    return pb::fail(PB_E_UNSUPPORTED, "image actor: frames of 5..128 pixels a side, "
                                      "a multiple of 4 bytes");
  if (actor.op < PB_IMG_BLUR || actor.op > PB_IMG_MEDIAN || actor.n_out < 0 ||
      actor.n_out > PB_MAX_PORTS)
    return pb::fail(PB_E_INVALID, "image actor: bad op or output count");
  dim3 grid(res.n_iter, res.n_streams);
  const int side = actor.side;
  if (PB_IMG_FAST && side >= 8 && (side & (side - 1)) == 0 && actor.n_out <= 2) {
    const size_t smem = actor.op == PB_IMG_DIFF ? 0 : (size_t)side * side * 3;
    static bool attr[pb::kMaxDevices] = {};   // side 128: 48 KB dynamic + the static part
    const int dev = pb::device();
    if (dev < 0) return PB_E_CUDA;
    if (!attr[dev]) {
      PB_CUDA(cudaFuncSetAttribute(image_fast_kernel<5>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   3 * kMaxSide * kMaxSide));
      attr[dev] = true;
    }
    dim3 fgrid((res.n_iter + kFPC - 1) / kFPC, res.n_streams);
    cudaStream_t st = pb::as_stream(stream);
    switch (side) {
      case 8: image_fast_kernel<1><<<fgrid, kFastThreads, smem, st>>>(actor, res); break;
      case 16: image_fast_kernel<2><<<fgrid, kFastThreads, smem, st>>>(actor, res); break;
      case 32: image_fast_kernel<3><<<fgrid, kFastThreads, smem, st>>>(actor, res); break;
      case 64: image_fast_kernel<4><<<fgrid, kFastThreads, smem, st>>>(actor, res); break;
      default: image_fast_kernel<5><<<fgrid, kFastThreads, smem, st>>>(actor, res); break;
    }
    PB_LAUNCHED("image_fast_kernel");
    return PB_OK;
  }
  image_kernel<<<grid, kImgThreads, 0, pb::as_stream(stream)>>>(actor, res);
  PB_LAUNCHED("image_kernel");
  return PB_OK;
}

}  // extern "C"
