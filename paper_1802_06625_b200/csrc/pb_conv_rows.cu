// conv2d_relu_pool (apps/vision.py): 5x5 convolution
// (NHWC fp32, zero padding) + bias + ReLU + 2x2 max pool, as a row-streaming
// implicit GEMM whose A operand lives in TENSOR MEMORY ("TS" tcgen05 MMAs).
//
// Why: with A in shared memory an M = 128 MMA reads 4 KB of A per K-step,
// so the N = 32/64 MMAs this layer has (32 output channels) run at the
// shared-memory read rate, not the tensor rate (tools/conv_probe.cu: 43 / 51
// cycles for N = 32 / 64).  With A in TMEM only B is read from shared memory
// and the same MMAs take 20.6 / 34.7 cycles (tools/tmem_a_probe.cu), within
// 30% of the math rate.
//
// Layout: the live frames of a launch (every firing's R frames) are laid side
// by side as one "virtual image" Wo columns per frame; a work tile is 128
// consecutive virtual output columns = the 128 TMEM lanes / MMA rows (lane v
// -> frame v / Wo, column v % Wo), and a tile streams through the input rows
// top to bottom.  For every input row y the converter warps build the row's
// im2col-along-x entries directly in TMEM (lane v, K = (dx, ci):
// x[y][xo + dx - pad][ci], bf16 hi and lo planes), and the MMA warp adds them
// into the accumulators of the five output rows o = y + pad - dy that row
// feeds (B = the weights of kernel row dy, resident in shared memory).  An
// output row is complete once its last input row is in; the epilogue warps
// read it, keep even rows in registers and max-pool each odd row with the
// one before it (vertical) and with the neighbouring lane (horizontal), then
// add the bias and apply ReLU (both monotone, so after the max) and store.
//
//   layer 1 (Cin = 3):  K per kernel row = 5 dx x 3 ci = 15 (+1 zero) -> one
//                       K16 chunk per input row
//   layer 2 (Cin = 32): K per kernel row = 5 dx x 32 ci = 160 -> ten chunks
//
// Accuracy: bf16x3 as the tile kernel (pb_cnn.cu): x = xh + xl, w = wh + wl,
// D = xh*[wh; wl] (N = 64, two products) + xl*wh (N = 32, into the first
// half); the epilogue adds the column halves.
//
// TMEM (512 columns): 4 accumulator slots x 64 columns, one per pair of
// output rows (2p at +0, 2p + 1 at +32; pair p uses slot p % 4) -- the
// max-pool consumes rows in pairs -- and a ring of A steps.  Every product
// is an N = 32 MMA into the row's 32 columns (xh*wh, xh*wl, xl*wh), so the
// epilogue reads one column set per row and adds nothing.
// Work moves in STEPS: layer 1 two input rows (two K16 chunks), layer 2 one
// channel half of one input row (five K16 chunks, dx = 0..4), so the
// per-step bookkeeping (barrier waits, commits) is amortised over 30 / 75
// MMAs.  Roles: warp 0 MMA issue (warp-uniform loop, one elected lane issues)
// and the weight load, warps 1-4 epilogue (TMEM lane quarter = warp % 4),
// warps 5-12 converters in two groups of four warps (one per lane quarter);
// step s of the row stream is built by group s % 2.  Hand-offs: a_full
// (converters -> MMA, 4 warp arrivals), a_empty (tcgen05.commit), acc_full
// (tcgen05.commit), acc_empty (4 epilogue warp arrivals).
#include <algorithm>
#include <cstdlib>

#include <cub/block/block_scan.cuh>
#include <cuda_bf16.h>

#include "pb_common.cuh"

namespace {

constexpr int kMaxPairSlots = 8;
constexpr int kMaxPairsPerTile = 256;
constexpr int kMaxStepsPerTile = 512;
constexpr int kPairCols = 64;                    // accumulator columns of a pair of rows
constexpr int kCoutR = 32;
constexpr int kUnitsThreads = 1024;
constexpr int kDeclined = 1;   // fire_conv_rows: shape not handled here (nothing launched)

// The epilogue's horizontal pool splits the 32 channels of a pooled pixel
// between the lane pair (m, m ^ 1): lane `odd`'s i-th channel.  PB_EPI_SECTOR:
// channels in runs of four alternating between the lanes, so the pair's q-th
// 16-byte stores are adjacent and fill one 32-byte sector; else halves 0-15 /
// 16-31 (two half sectors 64 bytes apart per store).
#ifndef PB_EPI_SECTOR
#define PB_EPI_SECTOR 1
#endif
__host__ __device__ constexpr int epi_channel(int i, bool odd) {
  return PB_EPI_SECTOR ? (i / 4) * 8 + (odd ? 4 : 0) + (i % 4) : (odd ? 16 : 0) + i;
}

__device__ __forceinline__ uint32_t s_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t s_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr & 0x3FFFF) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t i_desc(int n) {   // bf16 x bf16 -> f32, M = 128
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (128u >> 4 << 24);
}
// int8 limbs: s8 x s8 -> s32, M = 128 (tools/i8_probe.cu: exact, and an N = 64,
// K = 32 MMA issues in the 34.7 cycles of an N = 64, K = 16 bf16 one)
__host__ __device__ constexpr uint32_t i_desc_i8(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (128u >> 4 << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint32_t a, uint64_t b, uint32_t id,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   s_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(bar)), "r"(count));
}
__device__ __forceinline__ void bar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(s_u32(bar)) : "memory");
}
// pipeline waits trap after 5 s instead of hanging the device (pb_common.cuh);
// PB_WAIT_TRAP=0 builds the plain spin
#ifndef PB_WAIT_TRAP
#define PB_WAIT_TRAP 1
#endif
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  if (PB_WAIT_TRAP) {
    pb::mbar_wait_trap(s_u32(bar), parity);
    return;
  }
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
          s_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   s_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          s_u32(dst)),
      "l"(src), "r"(bytes), "r"(s_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&w)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                   taddr),
               "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]),
               "r"(w[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld16i(uint32_t taddr, int (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32z(uint32_t taddr) {   // 32 zero columns
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
      "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(0u)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
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
  uint32_t e;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
               : "=r"(e));
  return e != 0;
}

// x = hi + lo, each bf16 round-to-nearest (the tile kernel's converter).
__device__ __forceinline__ void split16(const float (&v)[16], uint32_t (&hi)[8], uint32_t (&lo)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
    const __nv_bfloat162 l =
        __floats2bfloat162_rn(v[2 * j] - __low2float(h), v[2 * j + 1] - __high2float(h));
    hi[j] = *reinterpret_cast<const uint32_t*>(&h);
    lo[j] = *reinterpret_cast<const uint32_t*>(&l);
  }
}

// int8 limbs of 16 values: X = rint(v * q) (q = 32639 / max |v| of the frame,
// so |X| <= 32639) as X = 256 h + l with h = (X + 128) >> 8 and l in
// [-128, 127].  One FFMA per value: v * q + (1.5 * 2^23 + 128) rounds the
// exact product to the nearest integer (ties to even) into the low mantissa
// bits, whose low 16 bits are Y = X + 128: h is byte 1 of Y, l is byte 0 of Y
// with its top bit flipped.  Words 0-3 carry h (K bytes 0-15), words 4-7 l.
__device__ __forceinline__ void quant16(const float (&v)[16], float q, uint32_t (&w)[8]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t y[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) y[b] = __float_as_uint(fmaf(v[4 * j + b], q, 12583040.f));
    const uint32_t p0 = __byte_perm(y[0], y[1], 0x5140);   // y0.b0 y1.b0 y0.b1 y1.b1
    const uint32_t p1 = __byte_perm(y[2], y[3], 0x5140);
    w[j] = __byte_perm(p0, p1, 0x7632);                     // byte 1 of y0..y3: h
    w[4 + j] = __byte_perm(p0, p1, 0x5410) ^ 0x80808080u;   // byte 0 flipped: l
  }
}

// role timing for experiments (pb_conv_actor.debug bit 4): cycles spent
// waiting per barrier kind, printed by CTA 0 at the end
struct WaitClock {
  bool on;
  long long t0, acc;
  __device__ __forceinline__ void start() { if (on) t0 = clock64(); }
  __device__ __forceinline__ void stop() { if (on) acc += clock64() - t0; }
};

// I8 (layer 2 only): int8 limbs instead of bf16x3.  x = (256 xh + xl) / qx
// per frame, w = (256 wh + wl) / qw per output channel; per 16 input channels
// ONE N = 64, K = 32 MMA with A = [xh | xl] and B = [wh 0; wl wh] gives the
// row's "hi" columns (xh wh) and "mid" columns (xh wl + xl wh); the epilogue
// dequantises (256 hi + mid) * 256 / (qx qw).  Each output row then owns 64
// accumulator columns (a pair 128) and a chunk of A 8 columns.
template <int CIN, bool I8 = false>
struct RowCfg {
  static_assert(!I8 || CIN == 32, "int8 limbs: layer 2 only");
  static constexpr int KC = CIN == 3 ? 1 : 5 * CIN / 16;   // K16 chunks per input row
  static constexpr int STEPS = 5 * KC;                     // weight K-steps (kernel row, chunk)
  static constexpr int WBYTES = STEPS * 64 * 16 * 2;       // [wh; wl] (I8: [wh 0; wl wh]) per K-step
  static constexpr int PAIR_COLS = I8 ? 128 : kPairCols;   // accumulator columns of a row pair
  static constexpr int ROW_COLS = PAIR_COLS / 2;
  static constexpr int CHUNK_COLS = I8 ? 8 : 16;           // A columns of one K chunk
  // a step: layer 1 two input rows, layer 2 one channel half of one row
  static constexpr int STEP_ROWS = CIN == 3 ? 4 : 1;
  static constexpr int STEP_CHUNKS = CIN == 3 ? 4 : 5;
  static constexpr int STEP_COLS = STEP_CHUNKS * CHUNK_COLS;
  // TMEM: PAIRS accumulator slots, then a ring of RING A steps.  Layer 1
  // (a step feeds 4 pairs) keeps two pairs of slack for the epilogue.
#ifndef PB_ROWS_PAIRS1
#define PB_ROWS_PAIRS1 6
#endif
  static constexpr int PAIRS = CIN == 3 ? PB_ROWS_PAIRS1 : (I8 ? 3 : 4);
  static constexpr int A0 = PAIRS * PAIR_COLS;             // first A-ring column
  static constexpr int RING = (512 - A0) / STEP_COLS;     // A steps in flight
#ifndef PB_ROWS_GROUPS1   // layer 1 with the row-parity MMA split: 1 converter group
#define PB_ROWS_GROUPS1 1    // + 2 epilogue groups 1.12 ms, 2 + 1 1.20 ms per 6144 frames
#endif
  static constexpr int GROUPS = CIN == 3 ? PB_ROWS_GROUPS1 : 2;   // converter groups of 4 warps
  // layer 2: each converter warp stages its lanes' row-half pixels in shared
  // memory (coalesced loads; 80-byte pixel pitch makes the per-lane 16-byte
  // reads conflict-free): up to 32 + 2 x 4 pixels, double-buffered
  static constexpr int STAGE_PIX = 40, STAGE_PITCH = 80;
  static constexpr int STAGE_BYTES = CIN == 3 ? 0 : 2 * STAGE_PIX * STAGE_PITCH * 4 * GROUPS;
  // layer 1: a loader warp (the last) streams each step's raw input rows into
  // a shared-memory ring by bulk copies; the converters split from there
  static constexpr int LOADER = CIN == 3 ? 1 : 0;
  static constexpr int RAW = 4;                            // raw steps in flight
  // epilogue groups of 4 warps taking alternate pairs: layer 1 has 2.2 pairs
  // per step to drain (its epilogue chain per pair is latency-bound)
#ifndef PB_ROWS_EPI1
#define PB_ROWS_EPI1 2
#endif
  static constexpr int EPI = CIN == 3 ? PB_ROWS_EPI1 : 1;
  static constexpr int CVT0 = 1 + 4 * EPI;                 // first converter warp
  // I8: a second MMA warp (the last) issues the channel-half-1 steps while
  // warp 0 issues the half-0 steps, so one warp's per-step bookkeeping runs
  // while the other's MMAs keep the tensor pipe busy (integer sums: the
  // interleaving cannot change a result)
  // ROWSPLIT (layer 1, fp32 accumulation): the two MMA warps split every
  // step by OUTPUT ROW parity instead -- each accumulator is written by one
  // warp in one order, so the fp32 sums stay deterministic
#ifndef PB_ROWS_SPLIT1
#define PB_ROWS_SPLIT1 1
#endif
  static constexpr bool ROWSPLIT = CIN == 3 && PB_ROWS_SPLIT1;
  static constexpr int MMA2 = (I8 || ROWSPLIT) ? CVT0 + 4 * GROUPS + LOADER : -1;
  static constexpr int THREADS = (CVT0 + 4 * GROUPS + LOADER + (MMA2 >= 0 ? 1 : 0)) * 32;
  static_assert(RING >= 2, "TMEM budget");
};

// Layer-1 raw ring geometry: a step's STEP_ROWS input rows, each as up to
// `segs` frame segments (the frames a 128-column tile touches); a segment is
// one frame row with zero margins (lm pixels left -- the padding rounded up
// so the bulk copy's destination is 16-byte aligned -- and >= pad right), so
// the converters read every entry without bounds checks.
struct RawGeom {
  int lm, seg_px, segs;
  int64_t seg_bytes, slot_bytes;
};
__host__ __device__ inline RawGeom raw_geom(int w, int pad, int wo, int rows) {
  RawGeom r;
  r.lm = (pad + 3) & ~3;
  r.seg_px = (r.lm + w + pad + 3) & ~3;
  r.segs = (127 + wo - 1) / wo + 1;
  r.seg_bytes = (int64_t)r.seg_px * 12;
  r.slot_bytes = r.seg_bytes * r.segs * rows;
  return r;
}

// One live firing of the launch: its input and output spans.
struct LiveSpan {
  const float* in;
  float* out;
};

// The live firings of every stream, compacted in (stream, firing) order with
// a block-wide scan of the per-stream counts; n_live[0] = their number.
__global__ void __launch_bounds__(kUnitsThreads)
conv_rows_units_kernel(pb_conv_actor a, pb_resolved res, LiveSpan* list, int* n_live) {
  using Scan = cub::BlockScan<int, kUnitsThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int base[kUnitsThreads];
  __shared__ int cnt[kUnitsThreads];
  const int s = threadIdx.x;
  const int c = s < res.n_streams ? pb::cond_count(res, a.cond, s) : 0;
  int b, total;
  Scan(tmp).ExclusiveSum(c, b, total);
  base[s] = b;
  cnt[s] = c;
  __syncthreads();
  if (s == 0) *n_live = total;
  // this launch's per-frame max |output| starts at 0 (the epilogue's atomicMax)
  if (a.absmax_out)
    for (int f = s; f < total * a.frames; f += kUnitsThreads) a.absmax_out[f] = 0.f;
  const int n_units = res.n_streams * res.n_iter;
  for (int u = s; u < n_units; u += kUnitsThreads) {
    const int st = u / res.n_iter, j = u - st * res.n_iter;
    if (j >= cnt[st]) continue;
    const int n = pb::firing_iter(res, a.cond, st, j);
    LiveSpan r;
    r.in = reinterpret_cast<const float*>(pb::span_ptr(a.in, res, st, n));
    r.out = reinterpret_cast<float*>(pb::span_ptr(a.out, res, st, n));
    list[base[st] + j] = r;
  }
}

struct RowBars {
  uint64_t a_full[8], a_empty[8], acc_full[kMaxPairSlots], acc_empty[kMaxPairSlots], w_full;
  uint64_t raw_full[8], raw_empty[8];
  // commit batches: every pair completed by the same input step is signalled
  // by ONE tcgen05.commit (the MMA warp feeds the tensor pipe and every
  // instruction it spends elsewhere is a bubble); batch_of[p] = the batch of
  // pair p within a tile, n_batches per tile (same for every tile)
  uint8_t batch_of[kMaxPairsPerTile];
  int n_batches;
  // per input step of a tile: bits 0-14 the last pair to acquire before its
  // MMAs, bit 15 set if a commit batch follows it; pre_sig = pairs committed
  // before the first step (above the first input row)
  uint16_t step_info[kMaxStepsPerTile];
  int pre_sig;
  uint32_t tmem_base;
  float bias[kCoutR];
  float wdq[kCoutR];   // I8: per output channel dequantisation factor max|w| / 32511
};

struct RowGeom {
  int H, W, pad, Ho, Wo, R, frames, tiles;
  int64_t in_frame, out_frame;
};

__device__ __forceinline__ RowGeom row_geom(const pb_conv_actor& a, int n_live, int cin) {
  RowGeom g;
  g.H = a.h; g.W = a.w; g.pad = a.pad; g.R = a.frames;
  g.Ho = g.H + 2 * g.pad - 4; g.Wo = g.W + 2 * g.pad - 4;
  g.frames = n_live * g.R;
  g.tiles = (int)(((int64_t)g.frames * g.Wo + 127) / 128);
  g.in_frame = (int64_t)g.H * g.W * cin;
  g.out_frame = (int64_t)(g.Ho / 2) * (g.Wo / 2) * kCoutR;
  return g;
}

// lane v of tile t: its frame's spans and its output column
struct LaneFrame {
  const float* in;
  float* out;
  int xo, fr;   // column in the frame, live frame index (virtual image order)
  bool valid;
};
__device__ __forceinline__ LaneFrame lane_frame(const RowGeom& g, const LiveSpan* list, int t,
                                                int m) {
  LaneFrame f;
  const int64_t v = (int64_t)t * 128 + m;
  const int fr = (int)(v / g.Wo);
  f.xo = (int)(v - (int64_t)fr * g.Wo);
  f.fr = fr;
  f.valid = fr < g.frames;
  f.in = nullptr;
  f.out = nullptr;
  if (f.valid) {
    const int u = fr / g.R, k = fr - u * g.R;
    const LiveSpan s = list[u];
    f.in = s.in + k * g.in_frame;
    f.out = s.out + k * g.out_frame;
  }
  return f;
}

// Step s of a tile -> its input rows and chunks.  Layer 1: rows 4s .. 4s+3 (one
// chunk each, K = the whole 5x3 entry).  Layer 2: row s/2, channel half s%2,
// chunks dx = 0..4 (weight K-step dy*10 + 2 dx + half).
template <int CIN>
__device__ __forceinline__ int step_row(int s, int i) {
  return CIN == 3 ? 4 * s + i : s >> 1;
}
template <int CIN>
__device__ __forceinline__ int step_wk(int s, int i) {   // weight K-step of chunk i at dy = 0
  return CIN == 3 ? 0 : 2 * i + (s & 1);
}

// absmax: I8, per live input frame max |x| (the quantisation scale)
template <int CIN, bool I8>
__global__ void __launch_bounds__(RowCfg<CIN, I8>::THREADS, 1)
conv_rows_kernel(pb_conv_actor a, const LiveSpan* __restrict__ list,
                 const int* __restrict__ n_live_p, const float* __restrict__ absmax) {
  using Cfg = RowCfg<CIN, I8>;
  constexpr int RING = Cfg::RING;
  constexpr int kPairSlots = Cfg::PAIRS;
  constexpr int kA0 = Cfg::A0;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* wsm = smem;
  RowBars& B = *reinterpret_cast<RowBars*>(smem + Cfg::WBYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const RowGeom g = row_geom(a, *n_live_p, CIN);
  const int n_steps = CIN == 3 ? g.H / 4 : 2 * g.H;   // steps per tile
  const int n_pairs = g.Ho / 2;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        s_u32(&B.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < RING; ++i) {
      bar_init(&B.a_full[i], 4);
      bar_init(&B.a_empty[i], Cfg::ROWSPLIT ? 2 : 1);
    }
    for (int i = 0; i < kPairSlots; ++i) {
      bar_init(&B.acc_full[i], Cfg::MMA2 >= 0 ? 2 : 1);
      bar_init(&B.acc_empty[i], 4);
    }
    bar_init(&B.w_full, 1);
    for (int i = 0; i < Cfg::RAW; ++i) {
      bar_init(&B.raw_full[i], 1);
      bar_init(&B.raw_empty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < kCoutR) {
    B.bias[threadIdx.x] = a.bias[threadIdx.x];
    if (I8)
      B.wdq[threadIdx.x] =
          reinterpret_cast<const float*>(static_cast<const uint8_t*>(a.weights_i8) +
                                         Cfg::WBYTES)[threadIdx.x];
  }
  if (threadIdx.x == 32) {
    // the MMA warp's commit points: before the first row, after every step
    // (layer 2: every row), after the last row
    int sig = 0, nb = 0;
    auto batch = [&](int rp_done) {
      bool any = false;
      for (; sig < n_pairs && min(2 * sig + 5, g.pad + g.H - 1) <= rp_done; ++sig) {
        B.batch_of[sig] = (uint8_t)nb;
        any = true;
      }
      nb += any;
      return any;
    };
    batch(g.pad - 1);
    B.pre_sig = sig;
    for (int st = 0; st < n_steps; ++st) {
      const int rp_hi = step_row<CIN>(st, Cfg::STEP_ROWS - 1) + g.pad;
      const bool cm = (CIN == 3 || (st & 1)) && batch(rp_hi);
      const int acq = max(min(rp_hi, g.Ho - 1) >> 1, sig - 1);
      B.step_info[st] = (uint16_t)(acq | (cm ? 0x8000 : 0));
    }
    batch(1 << 30);
    B.n_batches = nb;
  }
  uint8_t* raw = smem + Cfg::WBYTES + ((sizeof(RowBars) + 127) & ~size_t(127));
  const RawGeom rg = raw_geom(g.W, g.pad, g.Wo, Cfg::STEP_ROWS);
  if constexpr (CIN == 3) {
    // zero margins: the bulk copies only ever write segment interiors
    const int64_t n16 = rg.slot_bytes * Cfg::RAW / 16;
    for (int64_t i = threadIdx.x; i < n16; i += blockDim.x)
      reinterpret_cast<float4*>(raw)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = B.tmem_base;
  if constexpr (I8) {
    // every MMA accumulates (two warps issue into the same rows in either
    // order): the accumulators start at zero and the epilogue re-zeroes a
    // pair's columns when it releases the slot
    if (warp >= 1 && warp < 5) {
      const uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int col = 0; col < Cfg::A0; col += 8)
        tmem_st8(tmem + ((uint32_t)((warp & 3) * 32) << 16) + col, z);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  const bool prof = (a.debug & 16) && blockIdx.x == 0;
  const long long t_begin = clock64();
  WaitClock w1{prof, 0, 0}, w2{prof, 0, 0}, w3{prof, 0, 0}, w4{prof, 0, 0};
  const int y_last = g.pad + g.H - 1;                      // last padded input row with data
  // output row o has data iff some input row feeds it; pair p is complete
  // once the last input row feeding row 2p + 1 is in
  auto has_data = [&](int o) { return max(o, g.pad) <= min(o + 4, y_last); };
  auto pair_done_after = [&](int p) { return min(2 * p + 5, y_last); };

  if (warp == 0 || warp == Cfg::MMA2) {
    // ------------------------------------------------------------ MMA issue
    // A warp-uniform loop (every lane waits on the barriers); one elected lane
    // issues each step's MMAs and the commits: tcgen05 instructions from a
    // diverged single thread issue ~3x slower (tools/tmem_a_probe.cu).
    // I8: warp 0 takes the steps of channel half 0, warp MMA2 half 1; both
    // commit every batch (acc_full counts two arrivals).
    const int mw = warp == 0 ? 0 : 1;
    if (warp == 0 && elect_one()) {
      bar_expect_tx(&B.w_full, Cfg::WBYTES);
      const uint8_t* wsrc = static_cast<const uint8_t*>(I8 ? a.weights_i8 : a.weights);
      for (int off = 0; off < Cfg::WBYTES; off += 16384)
        bulk_load(wsm + off, wsrc + off, min(16384, Cfg::WBYTES - off), &B.w_full);
    }
    __syncwarp();
    bar_wait(&B.w_full, 0);
    const uint64_t bd0 = s_desc(s_u32(wsm), 128, 256);
    constexpr uint32_t id32 = i_desc(32);
    const bool run_mma = !(a.debug & 4);
    uint32_t c = 0;           // step counter (A ring)
    uint32_t pbase = 0;       // pair counter of this tile's pair 0
    uint32_t kbase = 0;       // commit batch counter (acc_full[k % slots])
    // Pair q owns accumulator slot q % 4.  Pairs are ACQUIRED in order (wait
    // until the epilogue drained pair q - 4 of the slot) and COMMITTED in order
    // (acc_full once complete), never committed before acquired: no mbarrier
    // phase of a slot runs more than one ahead of the epilogue.
    const int pre_sig = B.pre_sig;
    for (int t = blockIdx.x; t < g.tiles; t += gridDim.x, pbase += n_pairs) {
      int acq = 0, sig = 0;   // next pair to acquire / to commit
      auto acquire_to = [&](int p_last) {
        for (; acq <= p_last && acq < n_pairs; ++acq) {
          const uint32_t q = pbase + acq;
          w1.start();
          if (q >= kPairSlots) bar_wait(&B.acc_empty[q % kPairSlots], ((q / kPairSlots) - 1) & 1);
          w1.stop();
        }
      };
      // pairs with no input rows above / below the frame: one batch each
      auto commit_rest = [&](int upto) {
        if (upto <= sig) return;
        acquire_to(upto - 1);
        if (elect_one()) commit(&B.acc_full[kbase % kPairSlots]);
        __syncwarp();
        ++kbase;
        sig = upto;
      };
      commit_rest(pre_sig);
      uint32_t info = B.step_info[0];
      for (int st = 0; st < n_steps; ++st, ++c) {
        const int rp_hi = step_row<CIN>(st, Cfg::STEP_ROWS - 1) + g.pad;
        const bool batch_after = info & 0x8000;
        if (I8 && (st & 1) != mw) {
          // the other MMA warp's step: this warp only joins its batch commit
          // (which covers this warp's MMAs of the same input row)
          if (batch_after) {
            if (elect_one()) commit(&B.acc_full[kbase % kPairSlots]);
            __syncwarp();
            ++kbase;
            while (sig < n_pairs && pair_done_after(sig) <= rp_hi) ++sig;
          }
          info = B.step_info[min(st + 1, n_steps - 1)];
          continue;
        }
        const int rp0 = step_row<CIN>(st, 0) + g.pad;
        // interior step: every (chunk, dy) feeds a row inside the output
        // whose first contribution is its dy = 0 MMA -- straight-line issue
        // with the accumulator columns precomputed per step
        const bool interior = rp0 - 4 >= g.pad && rp0 - 4 >= 0 &&
                              step_row<CIN>(st, Cfg::STEP_ROWS - 1) + g.pad < g.Ho && run_mma;
        // I8 (3 pair slots): an interior step issues its dy = 4..1 MMAs
        // (rows in pairs already held) before it waits for the slot of a
        // pair its newest row opens, so the epilogue drains that slot
        // behind them instead of in front
        if (I8 && interior) acquire_to(min((int)(info & 0x7FFF), (rp0 - 1) >> 1));
        else acquire_to((int)(info & 0x7FFF));   // pairs this step writes or completes
        const uint32_t next_info = B.step_info[min(st + 1, n_steps - 1)];
        const uint32_t kb = kbase % kPairSlots;
        const uint32_t slot = c % RING;
        w2.start();
        bar_wait(&B.a_full[slot], (c / RING) & 1);
        w2.stop();
        asm volatile("tcgen05.fence::after_thread_sync;");
        w3.start();
        if (interior) {
          constexpr int NR = Cfg::STEP_ROWS;
          // rows o_min .. o_min + NR + 3 span pairs pmin .. pmin + (NR + 5) / 2:
          // their slot columns from one modulo, then increments with wrap
          const int o_min = rp0 - 4;
          const int odd = o_min & 1;
          constexpr int NB = (NR + 6) / 2;
          uint32_t base[NB];
          uint32_t sl = (pbase + (uint32_t)(o_min >> 1)) % kPairSlots;
#pragma unroll
          for (int k = 0; k < NB; ++k) {
            base[k] = tmem + sl * Cfg::PAIR_COLS;
            sl = sl + 1 == kPairSlots ? 0 : sl + 1;
          }
          uint32_t dcol[NR][5];
#pragma unroll
          for (int r = 0; r < NR; ++r)
#pragma unroll
            for (int dy = 0; dy < 5; ++dy) {
              const int rel = 4 + r - dy;   // o - o_min, compile-time
              dcol[r][dy] = odd ? base[(rel + 1) >> 1] + ((rel + 1) & 1) * Cfg::ROW_COLS
                                : base[rel >> 1] + (rel & 1) * Cfg::ROW_COLS;
            }
          const uint32_t abase = tmem + kA0 + slot * Cfg::STEP_COLS;
          const uint64_t bstep = bd0 + (uint64_t)((step_wk<CIN>(st, 0) * 2048) >> 4);
          const bool lead = CIN == 3 || (st & 1) == 0;
          if constexpr (I8) {
            constexpr uint32_t id64 = i_desc_i8(64);
            if (elect_one()) {
#pragma unroll
              for (int dy = 4; dy >= 1; --dy)
#pragma unroll
                for (int i = 0; i < Cfg::STEP_CHUNKS; ++i)
                  mma_i8(dcol[0][dy], abase + i * Cfg::CHUNK_COLS,
                         bstep + (uint64_t)(((dy * Cfg::KC + 2 * i) * 2048) >> 4), id64, 1u);
            }
            __syncwarp();
            acquire_to((int)(info & 0x7FFF));
            // the epilogue's zeroing of a re-acquired slot before these MMAs
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (elect_one()) {
#pragma unroll
              for (int i = 0; i < Cfg::STEP_CHUNKS; ++i)
                mma_i8(dcol[0][0], abase + i * Cfg::CHUNK_COLS,
                       bstep + (uint64_t)(((2 * i) * 2048) >> 4), id64, 1u);
              commit(&B.a_empty[slot]);
              if (batch_after) commit(&B.acc_full[kb]);
            }
          } else if (elect_one()) {
            const int par = mw ^ odd;   // ROWSPLIT: this warp's rows have rel & 1 == par
#pragma unroll
            for (int i = 0; i < Cfg::STEP_CHUNKS; ++i) {
              const int r = CIN == 3 ? i : 0;
              const uint32_t ahi = abase + i * 16;
#pragma unroll
              for (int dy = 0; dy < 5; ++dy) {
                if (Cfg::ROWSPLIT && ((4 + r - dy) & 1) != par) continue;
                const uint32_t d = dcol[r][dy];
                const uint64_t bd = bstep + (uint64_t)(((dy * Cfg::KC + (CIN == 3 ? 0 : 2 * i)) *
                                                        2048) >> 4);
                const uint32_t en = (dy == 0 && (CIN == 3 || (i == 0 && lead))) ? 0u : 1u;
                mma_ts(d, ahi, bd, id32, en);                    // xh * wh
                mma_ts(d, ahi, bd + (1024 >> 4), id32, 1u);      // xh * wl
                mma_ts(d, ahi + 8, bd, id32, 1u);                // xl * wh
              }
            }
            commit(&B.a_empty[slot]);
            if (batch_after) commit(&B.acc_full[kb]);
          }
        } else if (elect_one()) {
#pragma unroll
          for (int i = 0; i < Cfg::STEP_CHUNKS; ++i) {
            const int rp = step_row<CIN>(st, i) + g.pad;
            const uint32_t ahi = tmem + kA0 + slot * Cfg::STEP_COLS + i * Cfg::CHUNK_COLS;
            const bool lead = CIN == 3 || (i == 0 && (st & 1) == 0);   // first chunk of its row
#pragma unroll
            for (int dy = 0; dy < 5; ++dy) {
              const int o = rp - dy;
              if (o < 0 || o >= g.Ho || !run_mma) continue;
              if (Cfg::ROWSPLIT && (o & 1) != mw) continue;
              const uint32_t d = tmem +
                                 ((pbase + (uint32_t)(o >> 1)) % kPairSlots) * Cfg::PAIR_COLS +
                                 (o & 1) * Cfg::ROW_COLS;
              const uint64_t bd =
                  bd0 + (uint64_t)(((dy * Cfg::KC + step_wk<CIN>(st, i)) * 2048) >> 4);
              const bool first = lead && rp == max(o, g.pad);
              if (I8) {
                mma_i8(d, ahi, bd, i_desc_i8(64), 1u);   // [xh|xl] [wh 0; wl wh], zeroed acc
              } else {
                mma_ts(d, ahi, bd, id32, first ? 0u : 1u);        // xh * wh
                mma_ts(d, ahi, bd + (1024 >> 4), id32, 1u);       // xh * wl
                mma_ts(d, ahi + 8, bd, id32, 1u);                 // xl * wh
              }
            }
          }
          commit(&B.a_empty[slot]);
          if (batch_after) commit(&B.acc_full[kb]);
        }
        __syncwarp();
        w3.stop();
        // the batch of pairs this step completed (its last input row is in)
        if (batch_after) {
          ++kbase;
          while (sig < n_pairs && pair_done_after(sig) <= rp_hi) ++sig;
        }
        info = next_info;
      }
      commit_rest(n_pairs);   // pairs below the last input row
    }
  } else if (warp < Cfg::CVT0) {
    // ------------------------------------------------------------- epilogue
    // group e drains pairs e, e + 2, ... (each pair's 4 warps cover the lanes)
    const int egroup = (warp - 1) >> 2;
    const int quarter = warp & 3;
    const int m = quarter * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(quarter * 32) << 16);
    const bool odd = m & 1;
    float bias[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) bias[i] = B.bias[epi_channel(i, odd)];
    uint32_t pbase = 0, tnum = 0;
    for (int t = blockIdx.x; t < g.tiles; t += gridDim.x, pbase += n_pairs, ++tnum) {
      const LaneFrame f = lane_frame(g, list, t, m);
      // I8: the lane's frame dequantisation 256 * max|x| / 32639
      const float xdq = I8 && f.valid ? absmax[f.fr] * (256.f / 32639.f) : 0.f;
      float fmax_out = 0.f;   // running max |output| of the lane's frame (absmax_out)
      for (int pr = 0; pr < n_pairs; ++pr) {
        const uint32_t q = pbase + pr;
        if ((int)(q % Cfg::EPI) != egroup) continue;
        const uint32_t sl = q % kPairSlots;
        const bool h0 = has_data(2 * pr), h1 = has_data(2 * pr + 1);
        w2.start();
        w1.start();
        {
          const uint32_t k = tnum * (uint32_t)B.n_batches + B.batch_of[pr];
          bar_wait(&B.acc_full[k % kPairSlots], (k / kPairSlots) & 1);
        }
        w1.stop();
        asm volatile("tcgen05.fence::after_thread_sync;");
        float r0[32], r1[32];
        if (!(a.debug & 2)) {
          if constexpr (I8) {
            // row = (256 hi + mid) * 256 / (qx qw): hi and mid are exact s32
            // sums (|hi| < 2^24), the conversion rounds mid only.  Sixteen
            // channels of one row per round trip; r0 ends as the vertical max
            // of both rows (a row without data is 0, as below) and r1 is not
            // used.  Then the pair's columns are re-zeroed (the slot's next
            // pair accumulates from zero) and the slot released.
#pragma unroll
            for (int row = 0; row < 2; ++row) {
              if (!(row ? h1 : h0)) continue;
#pragma unroll
              for (int hf = 0; hf < 2; ++hf) {
                int hi[16], mid[16];
                const uint32_t c0 = tl + sl * Cfg::PAIR_COLS + row * 64 + hf * 16;
                tmem_ld16i(c0, hi);
                tmem_ld16i(c0 + 32, mid);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                  const float v = fmaf((float)hi[i], 256.f, (float)mid[i]) *
                                  (xdq * B.wdq[hf * 16 + i]);
                  r0[hf * 16 + i] = row == 0 ? v : (h0 ? fmaxf(r0[hf * 16 + i], v) : fmaxf(v, 0.f));
                }
              }
            }
            if (h0 && !h1) {
#pragma unroll
              for (int i = 0; i < 32; ++i) r0[i] = fmaxf(r0[i], 0.f);
            }
#pragma unroll
            for (int col = 0; col < Cfg::PAIR_COLS; col += 32) tmem_st32z(tl + sl * Cfg::PAIR_COLS + col);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          } else {
            if (h0) tmem_ld32(tl + sl * kPairCols, r0);
            if (h1) tmem_ld32(tl + sl * kPairCols + 32, r1);
            if (h0 || h1) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          }
        }
        if (I8 ? (!h0 && !h1) || (a.debug & 2) : !h0 || (a.debug & 2)) {
#pragma unroll
          for (int i = 0; i < 32; ++i) r0[i] = 0.f;
        }
        if (!I8 && (!h1 || (a.debug & 2))) {
#pragma unroll
          for (int i = 0; i < 32; ++i) r1[i] = 0.f;
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) bar_arrive(&B.acc_empty[sl]);
        w2.stop();
        w3.start();
        // 2x2 max: rows (2p, 2p+1) in registers, columns (xo, xo+1) on lanes
        // (m, m^1); the even lane keeps channels 0-15, the odd lane 16-31
        float res[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          // channel sets: the even lane pools epi_channel(i, 0), the odd lane
          // epi_channel(i, 1) (compile-time indices into r0 / r1)
          constexpr int dummy = 0;
          (void)dummy;
          const int ca = epi_channel(i, false), cb = epi_channel(i, true);
          const float lo_c = I8 ? r0[ca] : fmaxf(r0[ca], r1[ca]);
          const float hi_c = I8 ? r0[cb] : fmaxf(r0[cb], r1[cb]);
          const float send = odd ? lo_c : hi_c;
          const float keep = odd ? hi_c : lo_c;
          const float other = __shfl_xor_sync(0xffffffffu, send, 1);
          res[i] = fmaxf(fmaxf(keep, other) + bias[i], 0.f);
        }
        if (a.absmax_out) {
#pragma unroll
          for (int i = 0; i < 16; ++i) fmax_out = fmaxf(fmax_out, fabsf(res[i]));
        }
        if (f.valid && !(a.debug & 2)) {
          // PB_EPI_SECTOR: store q writes channels epi_channel(4q .. 4q+3): the
          // lane pair fills one whole 32-byte sector of the pixel per store
          float4* dst = reinterpret_cast<float4*>(
              f.out + ((int64_t)pr * (g.Wo >> 1) + (f.xo >> 1)) * kCoutR);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[epi_channel(4 * i, odd) / 4] =
                make_float4(res[4 * i], res[4 * i + 1], res[4 * i + 2], res[4 * i + 3]);
        }
        w3.stop();
      }
      // non-negative floats order like their bit patterns
      if (a.absmax_out && f.valid)
        atomicMax(reinterpret_cast<int*>(a.absmax_out) + f.fr, __float_as_int(fmax_out));
    }
  } else if (Cfg::LOADER && warp == Cfg::CVT0 + 4 * Cfg::GROUPS) {
    // ------------------------------------------------- layer-1 row loader
    // step c: rows 4s .. 4s+3 of every frame the tile touches, one bulk copy
    // per (row, frame) issued by one lane each, into raw slot c % RAW
    uint32_t c = 0;
    const uint32_t row_bytes = (uint32_t)g.W * 12;
    for (int t = blockIdx.x; t < g.tiles; t += gridDim.x) {
      const int64_t v0 = (int64_t)t * 128;
      const int fr0 = (int)(v0 / g.Wo);
      const int fr1 = min((int)((v0 + 127) / g.Wo), g.frames - 1);
      const int nseg = fr1 - fr0 + 1;
      const float* fin = nullptr;     // lane's frame (segment lane % segs)
      const int j = lane % rg.segs, i = lane / rg.segs;
      if (j < nseg) {
        const int fr = fr0 + j, u = fr / g.R;
        fin = list[u].in + (fr - u * g.R) * g.in_frame;
      }
      const bool mine = j < nseg && i < Cfg::STEP_ROWS && !(a.debug & 1);
      for (int st = 0; st < n_steps; ++st, ++c) {
        const uint32_t rslot = c % Cfg::RAW;
        w1.start();
        bar_wait(&B.raw_empty[rslot], ((c / Cfg::RAW) & 1) ^ 1);
        w1.stop();
        if (lane == 0)
          bar_expect_tx(&B.raw_full[rslot],
                        (a.debug & 1) ? 0u : row_bytes * nseg * Cfg::STEP_ROWS);
        __syncwarp();
        if (mine) {
          const int y = step_row<CIN>(st, i);
          bulk_load(raw + rslot * rg.slot_bytes + (i * rg.segs + j) * rg.seg_bytes + rg.lm * 12,
                    fin + (int64_t)y * g.W * 3, row_bytes, &B.raw_full[rslot]);
        }
        __syncwarp();
      }
    }
  } else {
    // ----------------------------------------------------------- converters
    // This group's steps s = group, group + 2, ... of the row stream; within
    // a step the next chunk's loads are in flight while the current one is
    // split and stored; a step's first chunk prefetches the lane's pixels of
    // the next input row into L2 (later chunks re-read lines the first brought
    // into L1).
    const int quarter = warp & 3;
    const int m = quarter * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(quarter * 32) << 16) + kA0;
    const int group = (warp - Cfg::CVT0) >> 2;
    auto load = [&](const LaneFrame& lf, int yy, int k, float (&v)[16]) {
      const float* row = lf.in + (int64_t)yy * g.W * CIN;
      if constexpr (CIN == 3) {
        // entry x[y][xo-pad .. xo-pad+4][0..2], zero outside the frame
        const int x0 = lf.xo - g.pad;
#pragma unroll
        for (int dx = 0; dx < 5; ++dx) {
          const int x = x0 + dx;
          const bool in = lf.valid && x >= 0 && x < g.W && !(a.debug & 1);
#pragma unroll
          for (int ci = 0; ci < 3; ++ci) v[dx * 3 + ci] = in ? __ldg(row + x * 3 + ci) : 0.f;
        }
        v[15] = 0.f;
      } else {
        // K-step k = 2 dx + half: x[y][xo - pad + dx][16 half .. 16 half + 15]
        const int x = lf.xo - g.pad + (k >> 1);
        if (lf.valid && x >= 0 && x < g.W && !(a.debug & 1)) {
          const float4* p = reinterpret_cast<const float4*>(row + x * CIN + (k & 1) * 16);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 q = __ldg(p + i);
            v[4 * i] = q.x; v[4 * i + 1] = q.y; v[4 * i + 2] = q.z; v[4 * i + 3] = q.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
      }
    };
    if constexpr (CIN == 3) {
      // entry of lane m at chunk (row) i: 15 consecutive floats of its frame's
      // segment, x = xo - pad .. xo - pad + 4 (margins are zero)
      uint32_t c = 0;
      for (int t = blockIdx.x; t < g.tiles; t += gridDim.x) {
        const LaneFrame f = lane_frame(g, list, t, m);
        const int fr0 = (int)((int64_t)t * 128 / g.Wo);
        const int64_t v = (int64_t)t * 128 + m;
        const int seg = (int)(v / g.Wo) - fr0;
        const int64_t lane_off =
            f.valid ? seg * rg.seg_bytes + (int64_t)(rg.lm - g.pad + f.xo) * 12 : 0;
        for (int st = 0; st < n_steps; ++st, ++c) {
          if ((int)(c % Cfg::GROUPS) != group) continue;
          const uint32_t slot = c % RING;
          const uint32_t rslot = c % Cfg::RAW;
          w1.start();
          bar_wait(&B.raw_full[rslot], (c / Cfg::RAW) & 1);
          bar_wait(&B.a_empty[slot], ((c / RING) & 1) ^ 1);
          w1.stop();
          asm volatile("tcgen05.fence::after_thread_sync;");
          const float* src = reinterpret_cast<const float*>(raw + rslot * rg.slot_bytes + lane_off);
          float ev[Cfg::STEP_CHUNKS][16];
#pragma unroll
          for (int i = 0; i < Cfg::STEP_CHUNKS; ++i) {
            const float* r = src + i * rg.segs * rg.seg_bytes / 4;
#pragma unroll
            for (int k = 0; k < 15; ++k) ev[i][k] = (f.valid && !(a.debug & 1)) ? r[k] : 0.f;
            ev[i][15] = 0.f;
          }
#pragma unroll
          for (int i = 0; i < Cfg::STEP_CHUNKS; ++i) {
            uint32_t hi[8], lo[8];
            split16(ev[i], hi, lo);
            if (!(a.debug & 8)) {
              tmem_st8(tl + slot * Cfg::STEP_COLS + i * 16, hi);
              tmem_st8(tl + slot * Cfg::STEP_COLS + i * 16 + 8, lo);
            }
          }
          __syncwarp();
          if (lane == 0) bar_arrive(&B.raw_empty[rslot]);
          w2.start();
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) bar_arrive(&B.a_full[slot]);
          w2.stop();
        }
      }
    } else {
      // Layer 2: group h builds channel half h of every input row (steps
      // 2y + h).  The warp's 32 lanes are at most two frame segments of
      // consecutive output columns; their pixels x = xo - pad .. xo - pad + 4
      // (per segment a contiguous run of <= 36 pixels of one frame row) are
      // fetched with coalesced 16-byte loads (pieces: pixel, quarter of the
      // 64-byte half) into this warp's staging buffer, one row ahead, and
      // every chunk dx reads lane-private 16-byte pieces from there.
      const int h = group;
      uint8_t* stage = smem + Cfg::WBYTES + ((sizeof(RowBars) + 127) & ~size_t(127)) +
                       (size_t)(warp - Cfg::CVT0) * 2 * Cfg::STAGE_PIX * Cfg::STAGE_PITCH;
      struct Seg {   // this warp's lanes in one tile
        const float* in1;
        const float* in2;
        int a, n1, np, my_idx;
        bool v1, v2;
        float q;   // I8: this lane's frame quantisation factor 32639 / max|x|
      };
      auto segs = [&](int t) {
        Seg sg;
        const int64_t v0 = (int64_t)t * 128 + quarter * 32;
        const int f1 = (int)(v0 / g.Wo);
        sg.a = (int)(v0 - (int64_t)f1 * g.Wo);
        sg.n1 = min(32, g.Wo - sg.a);
        const int n2 = 32 - sg.n1;
        sg.np = sg.n1 + 4 + (n2 > 0 ? n2 + 4 : 0);
        sg.v1 = f1 < g.frames;
        sg.v2 = n2 > 0 && f1 + 1 < g.frames;
        sg.in1 = nullptr;
        sg.in2 = nullptr;
        if (sg.v1) {
          const int u = f1 / g.R;
          sg.in1 = list[u].in + (f1 - u * g.R) * g.in_frame;
        }
        if (sg.v2) {
          const int u = (f1 + 1) / g.R;
          sg.in2 = list[u].in + (f1 + 1 - u * g.R) * g.in_frame;
        }
        sg.my_idx = lane < sg.n1 ? lane : sg.n1 + 4 + (lane - sg.n1);
        sg.q = 0.f;
        if (I8) {
          const int myf = lane < sg.n1 ? f1 : f1 + 1;
          const float mx = myf < g.frames ? absmax[myf] : 0.f;
          sg.q = mx > 0.f ? 32639.f / mx : 0.f;
        }
        return sg;
      };
      // piece j of the staged run: pixel p = j / 4, 16-byte quarter j % 4
      auto fetch = [&](const Seg& sg, int y, float4 (&r)[5]) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int j = lane + 32 * k;
          const int p = j >> 2;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (p < sg.np && !(a.debug & 1)) {
            const bool s1 = p < sg.n1 + 4;
            const int x = (s1 ? sg.a + p : p - (sg.n1 + 4)) - g.pad;
            const float* base = s1 ? sg.in1 : sg.in2;
            if ((s1 ? sg.v1 : sg.v2) && x >= 0 && x < g.W)
              v = __ldg(reinterpret_cast<const float4*>(base + ((int64_t)y * g.W + x) * CIN +
                                                        h * 16) + (j & 3));
          }
          r[k] = v;
        }
      };
      auto put = [&](int buf, const float4 (&r)[5]) {
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int j = lane + 32 * k;
          if ((j >> 2) < Cfg::STAGE_PIX)
            *reinterpret_cast<float4*>(stage + (buf * Cfg::STAGE_PIX + (j >> 2)) *
                                                   Cfg::STAGE_PITCH + (j & 3) * 16) = r[k];
        }
      };
      int t = blockIdx.x, y = 0, buf = 0;
      uint32_t c = h;
      if (t < g.tiles) {
        Seg sg = segs(t);
        float4 r[5];
        fetch(sg, 0, r);
        put(0, r);
        __syncwarp();
        while (t < g.tiles) {
          // next row of this group (possibly the next tile's first)
          int t2 = t, y2 = y + 1;
          if (y2 == g.H) {
            y2 = 0;
            t2 += gridDim.x;
          }
          Seg sg2 = sg;
          if (t2 != t && t2 < g.tiles) sg2 = segs(t2);
          if (t2 < g.tiles) fetch(sg2, y2, r);
          const uint32_t slot = c % RING;
          w1.start();
          bar_wait(&B.a_empty[slot], ((c / RING) & 1) ^ 1);
          w1.stop();
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint8_t* src = stage + (buf * Cfg::STAGE_PIX + sg.my_idx) * Cfg::STAGE_PITCH;
#pragma unroll
          for (int dx = 0; dx < 5; ++dx) {
            float v[16];
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              const float4 q = *reinterpret_cast<const float4*>(src + dx * Cfg::STAGE_PITCH + q4 * 16);
              v[4 * q4] = q.x; v[4 * q4 + 1] = q.y; v[4 * q4 + 2] = q.z; v[4 * q4 + 3] = q.w;
            }
            if constexpr (I8) {
              uint32_t w[8];
              quant16(v, sg.q, w);
              if (!(a.debug & 8)) tmem_st8(tl + slot * Cfg::STEP_COLS + dx * Cfg::CHUNK_COLS, w);
            } else {
              uint32_t hi[8], lo[8];
              split16(v, hi, lo);
              if (!(a.debug & 8)) {
                tmem_st8(tl + slot * Cfg::STEP_COLS + dx * 16, hi);
                tmem_st8(tl + slot * Cfg::STEP_COLS + dx * 16 + 8, lo);
              }
            }
          }
          w2.start();
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) bar_arrive(&B.a_full[slot]);
          w2.stop();
          if (t2 < g.tiles) put(buf ^ 1, r);
          __syncwarp();
          buf ^= 1;
          c += 2;
          t = t2;
          y = y2;
          sg = sg2;
        }
      }
    }
  }

  if (prof && lane == 0 && (warp == 0 || warp == 1 || warp == Cfg::CVT0 || warp == Cfg::CVT0 + 4 ||
                            warp == Cfg::MMA2 || (Cfg::LOADER && warp == Cfg::CVT0 + 4 * Cfg::GROUPS)))
    printf("{\"conv_rows_prof\": %d, \"warp\": %d, \"total\": %lld, \"wait1\": %lld, \"wait2\": %lld, \"w3\": %lld, \"w4\": %lld}\n",
           CIN, warp, clock64() - t_begin, w1.acc, w2.acc, w3.acc, w4.acc);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Per live frame max |x| of the launch's input (of_in) or output frames, one
// block per frame: the quantisation scale of an int8 layer whose producer did
// not record it (pb_conv_actor.absmax_in == NULL), or the absmax_out of a
// launch that ran the tile kernel.
constexpr int kAbsmaxThreads = 256;
__global__ void __launch_bounds__(kAbsmaxThreads)
frame_absmax_kernel(const LiveSpan* __restrict__ list, const int* __restrict__ n_live_p, int R,
                    int64_t frame_floats, bool of_in, float* __restrict__ out) {
  const int f = blockIdx.x;
  if (f >= *n_live_p * R) return;
  const int u = f / R, k = f - u * R;
  const float* p = (of_in ? list[u].in : list[u].out) + k * frame_floats;
  float m = 0.f;
  if ((reinterpret_cast<uintptr_t>(p) & 15) == 0 && frame_floats % 4 == 0) {
    const float4* p4 = reinterpret_cast<const float4*>(p);
    for (int64_t i = threadIdx.x; i < frame_floats / 4; i += kAbsmaxThreads) {
      const float4 v = __ldg(p4 + i);
      m = fmaxf(fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y))), fmaxf(fabsf(v.z), fabsf(v.w)));
    }
  } else {
    for (int64_t i = threadIdx.x; i < frame_floats; i += kAbsmaxThreads) m = fmaxf(m, fabsf(p[i]));
  }
#pragma unroll
  for (int d = 16; d; d >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, d));
  __shared__ float wm[kAbsmaxThreads / 32];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kAbsmaxThreads / 32; ++w) m = fmaxf(m, wm[w]);
    out[f] = m;
  }
}

template <int CIN, bool I8 = false>
int launch_rows(const pb_conv_actor& actor, const pb_resolved& res, cudaStream_t st, int sms) {
  using Cfg = RowCfg<CIN, I8>;
  // one CTA per SM: the kernel allocates all 512 TMEM columns
  const int Wo_ = actor.w + 2 * actor.pad - 4, Ho_ = actor.h + 2 * actor.pad - 4;
  const RawGeom rg = raw_geom(actor.w, actor.pad, Wo_, Cfg::STEP_ROWS);
  const size_t raw_bytes = CIN == 3 ? (size_t)rg.slot_bytes * Cfg::RAW : 0;
  const int steps_ = CIN == 3 ? actor.h / 4 : 2 * actor.h;
  if (Ho_ / 2 > kMaxPairsPerTile || steps_ > kMaxStepsPerTile || (CIN == 3 && (actor.w % 4 || rg.segs * Cfg::STEP_ROWS > 32)))
    return kDeclined;   // not for this kernel: the caller uses the tile kernel
  const size_t smem = std::max<size_t>(
      1024 + Cfg::WBYTES + ((sizeof(RowBars) + 127) & ~size_t(127)) + Cfg::STAGE_BYTES + raw_bytes,
      120 * 1024);
  if (smem > 227 * 1024) return kDeclined;
  const int dev = pb::device();
  if (dev < 0) return PB_E_CUDA;
  static size_t configured[pb::kMaxDevices] = {};
  if (configured[dev] < smem) {
    PB_CUDA(cudaFuncSetAttribute(conv_rows_kernel<CIN, I8>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured[dev] = smem;
  }
  if (res.n_streams > kUnitsThreads)
    return pb::fail(PB_E_UNSUPPORTED, "conv: more than 1024 streams per launch");
  if (CIN == 3 && actor.h % 4)
    return pb::fail(PB_E_UNSUPPORTED, "conv: layer-1 frames need a height divisible by 4");
  const int64_t n_units = (int64_t)res.n_streams * res.n_iter;
  const int Wo = actor.w + 2 * actor.pad - 4;
  const int64_t max_tiles = (n_units * actor.frames * Wo + 127) / 128;
  if (max_tiles >= (int64_t)1 << 31) return pb::fail(PB_E_UNSUPPORTED, "conv: launch too large");
  void* scratch = nullptr;
  int rc = pb::scratch(pb::kScratchConvRows, sizeof(LiveSpan) * n_units + 16, &scratch);
  if (rc) return rc;
  LiveSpan* list = reinterpret_cast<LiveSpan*>(static_cast<uint8_t*>(scratch) + 16);
  int* n_live = static_cast<int*>(scratch);
  conv_rows_units_kernel<<<1, kUnitsThreads, 0, st>>>(actor, res, list, n_live);
  PB_LAUNCHED("conv_rows_units_kernel");
  const int grid = (int)std::min<int64_t>(max_tiles, sms);
  if (grid == 0) return PB_OK;
  const float* absmax = actor.absmax_in;
  if (I8 && !absmax) {
    float* buf = nullptr;
    rc = pb::scratch(pb::kScratchConvAbsmax, sizeof(float) * n_units * actor.frames,
                     reinterpret_cast<void**>(&buf));
    if (rc) return rc;
    frame_absmax_kernel<<<(unsigned)(n_units * actor.frames), kAbsmaxThreads, 0, st>>>(
        list, n_live, actor.frames, (int64_t)actor.h * actor.w * CIN, true, buf);
    PB_LAUNCHED("frame_absmax_kernel");
    absmax = buf;
  }
  conv_rows_kernel<CIN, I8><<<grid, Cfg::THREADS, smem, st>>>(actor, list, n_live, absmax);
  PB_LAUNCHED("conv_rows_kernel");
  return PB_OK;
}

}  // namespace

namespace pb {
// pb_fire_conv_pool (pb_cnn.cu) dispatches here for Cin 3 and 32 unless
// PB_CONV_IMPL=tiles selects the round-1 tile kernel.
int fire_conv_rows(const pb_conv_actor& actor, const pb_resolved& res, cudaStream_t st, int sms) {
  switch (actor.cin) {
    case 3: return launch_rows<3>(actor, res, st, sms);
    case 32:
      if (actor.math == PB_CONV_I8 && actor.weights_i8) return launch_rows<32, true>(actor, res, st, sms);
      return launch_rows<32>(actor, res, st, sms);
    default: return PB_E_UNSUPPORTED;
  }
}

// absmax_out of a launch that ran the tile kernel: the output frames' max |y|
// by a separate pass (the row kernel records it in its epilogue)
int conv_absmax_out(const pb_conv_actor& actor, const pb_resolved& res, cudaStream_t st) {
  if (res.n_streams > kUnitsThreads)
    return pb::fail(PB_E_UNSUPPORTED, "conv: more than 1024 streams per launch");
  const int64_t n_units = (int64_t)res.n_streams * res.n_iter;
  if (n_units * actor.frames == 0) return PB_OK;
  void* scratch = nullptr;
  int rc = pb::scratch(pb::kScratchConvRows, sizeof(LiveSpan) * n_units + 16, &scratch);
  if (rc) return rc;
  LiveSpan* list = reinterpret_cast<LiveSpan*>(static_cast<uint8_t*>(scratch) + 16);
  int* n_live = static_cast<int*>(scratch);
  pb_conv_actor a = actor;
  a.absmax_out = nullptr;   // the pass below writes every live frame
  conv_rows_units_kernel<<<1, kUnitsThreads, 0, st>>>(a, res, list, n_live);
  PB_LAUNCHED("conv_rows_units_kernel");
  const int64_t out_floats = (int64_t)((actor.h + 2 * actor.pad - 4) / 2) *
                             ((actor.w + 2 * actor.pad - 4) / 2) * kCoutR;
  frame_absmax_kernel<<<(unsigned)(n_units * actor.frames), kAbsmaxThreads, 0, st>>>(
      list, n_live, actor.frames, out_floats, false, actor.absmax_out);
  PB_LAUNCHED("frame_absmax_kernel");
  return PB_OK;
}
}  // namespace pb
