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
constexpr int kMaxSide = 128;

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

}  // namespace

extern "C" {

int pb_fire_image(pb_image_actor actor, pb_resolved res, void* stream) {
  if (res.n_iter == 0) return PB_OK;
  if (actor.side < 5 || actor.side > kMaxSide || (actor.side * actor.side) % 4)
    return pb::fail(PB_E_UNSUPPORTED, "image actor: frames of 5..128 pixels a side, "
                                      "a multiple of 4 bytes");
  if (actor.op < PB_IMG_BLUR || actor.op > PB_IMG_MEDIAN || actor.n_out < 0 ||
      actor.n_out > PB_MAX_PORTS)
    return pb::fail(PB_E_INVALID, "image actor: bad op or output count");
  dim3 grid(res.n_iter, res.n_streams);
  image_kernel<<<grid, kImgThreads, 0, pb::as_stream(stream)>>>(actor, res);
  PB_LAUNCHED("image_kernel");
  return PB_OK;
}

}  // extern "C"
