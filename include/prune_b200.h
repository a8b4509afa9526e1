/*
 * prune_b200.h — C-ABI of the B200 execution path for PRUNE data-parallel actors.
 *
 * Plain pointers and sizes only (no torch / no C++ types).  Every entry point
 * returns an int status: PB_OK (0) or a negative PB_E_* code; pb_last_error()
 * returns the text of the last failure on the calling thread.  Device memory
 * referenced by the descriptor structs below is owned by the caller of the
 * pb_fire_* entry points (normally the Python engine, through pb_malloc);
 * rings own their storage.  Host buffers are always owned by the caller.
 *
 * Reference interfaces each group replaces (paths relative to the reference
 * root, /root/reference):
 *   - FIFO channel engine ........ pkg/src/tokenflow/fifos.py:49-338
 *       (CapacityPlan/layout_plan :49-98, writer_gate/reader_gate/copy_gate
 *        :106-139, FifoChannel :142-338, errors InvalidParams/ProtocolError/
 *        EndOfStream/Poisoned :25-46)
 *   - per-firing rate gating ..... pkg/src/tokenflow/runtime.py:107-116 (Eq. 1),
 *       Eq. 1 recheck :195-220, oracle twin interp.py:126-148,
 *       decode_control behavior.py:34-38
 *   - actor firings .............. FirBranch.fire apps/predistortion.py:41-65,
 *       BranchSum.fire :68-83, Route.fire behavior.py:176-184,
 *       Passthrough :158-165, AddMod :168-173, Merge :187-199,
 *       MatMul.fire apps/bypass.py:36-49, PathMerge.fire :52-66
 *   - host configuration actors .. _PolicyBase/FixedPolicy/AlternatePolicy/
 *       SeededPolicy/SubsetPolicy behavior.py:202-256 (CPython `random`)
 *
 * Error codes map onto the reference exception types (fifos.py:25-46,
 * runtime.py:26-48): PB_E_INVALID -> InvalidParams/ValueError,
 * PB_E_PROTOCOL -> ProtocolError, PB_E_EOS -> EndOfStream,
 * PB_E_POISONED -> Poisoned, PB_E_CUDA / PB_E_ACTOR -> ActorPanic.
 */
#ifndef PRUNE_B200_H
#define PRUNE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PB_ABI_VERSION 1

enum {
  PB_OK = 0,
  PB_E_INVALID = -1,     /* InvalidParams / ValueError */
  PB_E_PROTOCOL = -2,    /* ProtocolError (span protocol misuse, ring overflow) */
  PB_E_EOS = -3,         /* EndOfStream */
  PB_E_POISONED = -4,    /* Poisoned */
  PB_E_CUDA = -5,        /* device runtime failure */
  PB_E_NOMEM = -6,       /* allocation failure */
  PB_E_UNSUPPORTED = -7, /* shape the kernels do not cover */
  PB_E_ACTOR = -8,       /* an actor firing reported a failure (ActorPanic) */
  PB_E_TIMEOUT = -9      /* a blocking ring transfer timed out (Timeout) */
};

#define PB_TAPS 10          /* FIR taps, predistortion.py:24 (TAPS) */
#define PB_MAX_BRANCHES 32  /* branches one fused filter-bank launch covers */
#define PB_MAX_PORTS 16     /* data ports of one actor in the byte kernels */

/* ------------------------------------------------------------------ runtime */
int pb_abi_version(void);
const char* pb_last_error(void);
int pb_device_count(int* n);
int pb_set_device(int device);
int pb_device_sync(void);
int pb_sm_count(int* n);
int pb_malloc(void** dptr, size_t bytes);
int pb_free(void* dptr);
int pb_host_alloc(void** hptr, size_t bytes); /* page-locked host memory */
int pb_host_free(void* hptr);
/* Page-lock caller-owned host memory in place (cudaHostRegister) so ring
 * copies DMA straight from the caller's source buffers (FileSource / sources=
 * data, behavior.py:124-140) without a staging copy.  Returns PB_OK, or 1 when
 * the range was already registered by someone else (do not unregister it). */
int pb_host_register(void* hptr, size_t bytes);
int pb_host_unregister(void* hptr);
int pb_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream);
int pb_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream);
int pb_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream);
int pb_memset(void* dst, int value, size_t bytes, void* stream);
/* pitched copies: height rows of width bytes; kind 1 = H2D, 2 = D2H, 3 = D2D */
int pb_memcpy_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                 size_t height, int kind, void* stream);
int pb_stream_create(void** stream);
int pb_stream_destroy(void* stream);
int pb_stream_sync(void* stream);
int pb_event_create(void** event);
int pb_event_destroy(void* event);
int pb_event_record(void* event, void* stream);
int pb_event_elapsed_ms(void* start, void* end, float* ms);
int pb_event_sync(void* event);
/* make `stream` wait for `event` (cudaStreamWaitEvent) */
int pb_stream_wait(void* stream, void* event);
/* Number of device kernels this library has launched (process lifetime). */
int64_t pb_launch_count(void);

/* --------------------------------------------- capacity plan (fifos.py:49-139) */
typedef struct {
  int32_t rate, token_bytes, delay, factor;
  int32_t aligned; /* 1 when delay % rate == 0 */
  int32_t pad_;
  int64_t slots;   /* token slots */
  int64_t nbytes;  /* slots * token_bytes */
  int64_t copy_src, copy_dst, copy_count; /* wrap copy (unaligned), else -1 */
} pb_plan;

/* layout_plan, fifos.py:87-98 */
int pb_layout_plan(int rate, int delay, int factor, int token_bytes, pb_plan* out);
/* writer_gate fifos.py:106-121, reader_gate :124-127, copy_gate :130-139 */
int64_t pb_writer_gate(int64_t w, int rate, int delay, int factor, int aligned);
int64_t pb_reader_gate(int64_t i, int rate, int delay);
int64_t pb_copy_gate(int64_t n, int rate, int delay, int factor);

/* ------------------------------------- device rings (FifoChannel, fifos.py:142) */
/* One ring per FIFO, replicated over n_streams independent streams.  Storage
 * and the per-stream counters (chunk writes, chunk reads, max occupancy in
 * tokens, wrap copies done) live in HBM; kernels address spans through pb_span_ref. */
typedef struct pb_ring pb_ring;
int pb_ring_create(int rate, int token_bytes, int delay, int factor, int n_streams,
                   const void* delay_payload, pb_ring** out);
int pb_ring_destroy(pb_ring* ring);
int pb_ring_plan(const pb_ring* ring, pb_plan* out);
int pb_ring_storage(const pb_ring* ring, void** data, int64_t* stream_stride,
                    int64_t** counters /* device int64[4][n_streams] */);
/* write n_chunks spans (rate tokens each) from host memory; PB_E_PROTOCOL if
 * the writer gate (fifos.py:106) would block, PB_E_PROTOCOL after close. */
int pb_ring_push_host(pb_ring* ring, int stream, const void* src, int64_t n_chunks,
                      void* cuda_stream);
/* read n_chunks spans into host memory; PB_E_EOS when closed and short,
 * PB_E_PROTOCOL when open and short (the reference would block). */
int pb_ring_pop_host(pb_ring* ring, int stream, void* dst, int64_t n_chunks,
                     void* cuda_stream);
/* Blocking variants (FifoChannel.write_start / read_start wait,
 * fifos.py:223-323): wait until the gate opens, the ring closes (pop:
 * PB_E_EOS when short) or is poisoned (PB_E_POISONED), or timeout_ms elapses
 * (PB_E_TIMEOUT; timeout_ms < 0 waits without limit).  A push and a pop may
 * run concurrently on different threads (single producer, single consumer
 * per stream); every host transfer of a ring is serialised by its lock. */
int pb_ring_push_host_wait(pb_ring* ring, int stream, const void* src, int64_t n_chunks,
                           void* cuda_stream, int64_t timeout_ms);
int pb_ring_pop_host_wait(pb_ring* ring, int stream, void* dst, int64_t n_chunks,
                          void* cuda_stream, int64_t timeout_ms);
int pb_ring_counters(const pb_ring* ring, int stream, int64_t* writes, int64_t* reads,
                     int64_t* max_occupancy);
int pb_ring_close(pb_ring* ring);
int pb_ring_poison(pb_ring* ring, const char* reason);

/* ------------------------------------------ epoch resolution (Eq. 1 on device) */
/* A condition is one (control output port, element) pair of the control
 * table (model.py:137-163).  Its control tokens for the epoch are resident in
 * HBM: token of iteration n of stream s at
 *   tokens + s*stream_stride + ((base + n) % slots) * token_stride. */
typedef struct {
  const uint8_t* tokens;
  int64_t stream_stride;
  int32_t token_stride; /* FIFO token_bytes of the control channel */
  int32_t element;      /* 0-based: T[p] - 1 */
  int32_t slots;        /* ring chunk positions of the control channel */
  int32_t base;         /* chunk index of iteration 0 */
} pb_condition;

/* Device-resident resolution of one epoch: per condition c and stream s,
 * act[c][s][n] (0/1), prefix[c][s][n] (exclusive count of active iterations
 * before n), count[c][s] and worklist[c][s][j] (iteration of the j-th active
 * firing).  Strides: act/prefix/worklist use cap per (c, s) row. */
typedef struct {
  uint8_t* act;
  int32_t* prefix;
  int32_t* count;
  int32_t* worklist;
  int32_t n_cond, n_streams, n_iter, cap;
} pb_resolved;

/* Decode control tokens into per-iteration activity (decode_control,
 * behavior.py:34-38; Eq. 1 runtime.py:107-116) and compact the firings. */
int pb_resolve(const pb_condition* conds /* host array [n_cond] */, pb_resolved res,
               void* stream);

/* Eq. 1 recheck (runtime.py:195-220): for each DRP, the rate implied by the
 * dynamic actor's own control token must equal the span the engine moved.
 * counters: device int64[2] {checks, failures}, accumulated. */
typedef struct {
  int32_t own_cond;   /* condition decoded from the actor's control channel */
  int32_t moved_cond; /* condition that gated the FIFO attached to the DRP */
  int32_t actor_cond; /* condition of the dynamic actor itself (-1: always) */
  int32_t pad_;
} pb_eq1_port;
int pb_eq1_check(const pb_eq1_port* ports /* host array */, int n_ports, pb_resolved res,
                 int64_t* counters, void* stream);

/* Advance ring counters after an epoch (write_end/read_end in bulk).  For
 * ring r: writes += rate_chunks * tokens_in_epoch, reads likewise, and the
 * max occupancy (fifos.py:177-181,256) is updated. */
typedef struct {
  int64_t* counters;  /* ring counters, device int64[4][n_streams] */
  int32_t cond;       /* condition gating the FIFO (-1 always) */
  int32_t rate;       /* tokens per chunk */
  int32_t delay;
  int32_t pad_;
} pb_ring_advance_t;
int pb_rings_advance(const pb_ring_advance_t* rings /* host array */, int n_rings,
                     pb_resolved res, void* stream);

/* pb_eq1_check + pb_rings_advance of one epoch in one launch (independent
 * blocks; at most 256 ports and 256 rings).  The Eq. 1 recheck only reads the
 * resolution, so it can close the epoch after the actor firings. */
int pb_epoch_close(const pb_eq1_port* ports /* host array */, int n_ports, int64_t* counters,
                   const pb_ring_advance_t* rings /* host array */, int n_rings,
                   pb_resolved res, void* stream);

/* --------------------------------------------------------- span addressing */
/* Where the span of a port lives for firing at iteration n of stream s:
 *   idx   = index_cond < 0 ? n : prefix[index_cond][s][n]
 *   chunk = (base[s] + idx + offset) % slots     (base NULL -> 0)
 *   ptr   = data + s*stream_stride + chunk*span_bytes
 * act_cond is the condition gating the port (-1: always active).  offset is
 * the producer side of a FIFO with initial delay tokens: delay / rate chunks
 * (fifos.py:87-98 aligned plan; the consumer side uses 0 and first reads the
 * delay payload). */
typedef struct {
  uint8_t* data;
  int64_t stream_stride;
  int64_t span_bytes;
  const int64_t* base;
  int32_t slots;
  int32_t index_cond;
  int32_t act_cond;
  int32_t offset;
} pb_span_ref;

/* ------------------------------------------------------------- actor kernels */
/* fir_branch (predistortion.py:41-65): planar complex fp32 span
 * [re[B], im[B]], 10-tap complex FIR in ascending tap order, every product
 * and sum rounded separately (no FMA), accumulator from +0.  History = last
 * 9 input samples of the actor's previous firing (state[s] at the first
 * firing of an epoch). */
typedef struct {
  pb_span_ref in;
  pb_span_ref out;
  const float* taps;  /* device [2][PB_TAPS]: re then im */
  float* state;       /* device [n_streams][2][PB_TAPS-1] */
  int32_t cond;       /* actor activity condition (-1 always) */
  int32_t pad_;
} pb_fir_actor;

/* FIR arithmetic modes.  EXACT reproduces FirBranch.fire bit for bit (every
 * product and sum rounded, scalar FMUL/FADD); EXACT_PAIRED is the same
 * roundings with FMUL2/FADD2; FMA contracts each tap into fused multiply-adds
 * (one rounding per tap term, about half the FP32 work) and is accurate to
 * ~1e-7 relative, inside the 1e-5 tolerance the north star states. */
#define PB_FIR_EXACT 0
#define PB_FIR_EXACT_PAIRED 1
#define PB_FIR_FMA 2
#define PB_FIR_MERGED 3   /* bank only: one FMA FIR with the active branches' taps summed */

/* All firings of n_actors fir_branch actors in one launch.  actors is a
 * DEVICE array. */
int pb_fire_fir(const pb_fir_actor* actors, int n_actors, pb_resolved res, int64_t block,
                int math, void* stream);
/* History carry after pb_fire_fir / pb_fire_filter_bank: state[s] <- last 9
 * input samples of the epoch's last firing (if any). */
int pb_fir_carry(const pb_fir_actor* actors, int n_actors, pb_resolved res, int64_t block,
                 void* stream);

/* Fused dynamic region route -> K x fir_branch -> branch_sum
 * (behavior.py:176-184, predistortion.py:41-83): one pass over each input
 * span, branch outputs summed from +0 in the combiner's sorted port order
 * (predistortion.py:75) without materialising the branch channels. */
typedef struct {
  pb_span_ref in;                    /* route input */
  pb_span_ref out;                   /* combiner output */
  const pb_fir_actor* branches;      /* device array, combiner sorted port order */
  int32_t n_branches;
  int32_t actor_cond;                /* condition of route/combiner (-1) */
  uint32_t* sched;                   /* device uint32[2], zeroed once: dynamic work
                                        counter reset by the last CTA; NULL = static */
  int32_t math;                      /* PB_FIR_* arithmetic mode */
  int32_t pad_;
} pb_filter_bank;
/* The call includes the history carry of every branch (pb_fir_carry's work:
 * state[s] <- the last 9 input samples of the branch's last firing this
 * epoch); callers do not carry bank branches themselves. */
int pb_fire_filter_bank(pb_filter_bank bank, pb_resolved res, int64_t block, void* stream);

/* branch_sum (predistortion.py:68-83): ins in sorted port-id order. */
typedef struct {
  pb_span_ref in[PB_MAX_PORTS];
  pb_span_ref out;
  int32_t n_in;
  int32_t cond;
} pb_sum_actor;
int pb_fire_branch_sum(pb_sum_actor actor, pb_resolved res, int64_t block, void* stream);

/* Byte actors: out[k] = (sum of active inputs + offset) mod 256 for every
 * active output — covers route (behavior.py:176-184, used when not
 * aliased), passthrough (:158-165), add_mod (:168-173) and merge (:187-199). */
typedef struct {
  pb_span_ref in[PB_MAX_PORTS];
  pb_span_ref out[PB_MAX_PORTS];
  int32_t n_in, n_out;
  int32_t offset;
  int32_t cond;
} pb_bytes_actor;
int pb_fire_bytes(pb_bytes_actor actor, pb_resolved res, void* stream);

/* matmul (bypass.py:36-49): out = W @ x, N x N fp32, ascending k, separate
 * mul/add roundings.  N = 8 in the reference. */
typedef struct {
  pb_span_ref in;
  pb_span_ref out;
  const float* weights; /* device [N][N] row-major */
  int32_t n;
  int32_t cond;
} pb_matmul_actor;
int pb_fire_matmul(pb_matmul_actor actor, pb_resolved res, void* stream);

/* A chain of matmul actors fired as one launch (the engine fuses consecutive
 * matmul actors under one condition whose link channels are exclusive and
 * undelayed; those channels are then not materialised): out = W_{L-1} ...
 * W_1 W_0 x, every layer in MatMul.fire's order (bypass.py:36-49: ascending k,
 * separate mul/add roundings), so the result is bit-identical to L
 * pb_fire_matmul launches.  N = 8 (16 lanes per firing). */
typedef struct {
  pb_span_ref in;
  pb_span_ref out;
  const float* weights; /* device [layers][N][N] row-major */
  int32_t n;
  int32_t layers;       /* 2 .. 8 */
  int32_t cond;
  int32_t pad_;
} pb_matmul_chain_actor;
int pb_fire_matmul_chain(pb_matmul_chain_actor actor, pb_resolved res, void* stream);

/* The whole adaptive-bypass region (bypass.py:69-132: route -> matmul chain ->
 * path_merge, the route's other output straight into the merge's bypass port)
 * as ONE launch: per merge firing the live path is read once -- the chain's
 * input through its layers (pb_fire_matmul_chain's arithmetic) or the bypass
 * token plus the marker (PathMerge.fire) -- and written to the merge's output;
 * the chain's link channels and its output channel are not materialised.  A
 * firing with != 1 live path sets *error_flag.  N = 8. */
typedef struct {
  pb_span_ref chain_in;   /* the chain's first input channel (consumer side) */
  pb_span_ref bypass_in;  /* the merge's bypass input channel (consumer side) */
  pb_span_ref out;        /* the merge's output channel (producer side) */
  const float* weights;   /* device [layers][8][8] */
  int32_t layers;
  int32_t chain_live;     /* condition of the chain's output channel (its path is live) */
  int32_t cond;           /* the merge's activity condition */
  float marker;
  int32_t* error_flag;
} pb_bypass_region;
int pb_fire_bypass_region(pb_bypass_region region, pb_resolved res, void* stream);

/* path_merge (bypass.py:52-66): exactly one live input is forwarded; the
 * marker is added when it is the bypass port.  A firing with != 1 live input
 * sets *error_flag (device int32) -> ActorPanic. */
typedef struct {
  pb_span_ref in[PB_MAX_PORTS];
  pb_span_ref out;
  int32_t n_in;
  int32_t bypass_index; /* index into in[] of the bypass port, -1 none */
  float marker;
  int32_t cond;
  int32_t* error_flag;
} pb_path_merge_actor;
int pb_fire_path_merge(pb_path_merge_actor actor, pb_resolved res, void* stream);

/* ------------------------------------------- image actors (motion detection) */
/* apps/motion.py:29-71: 8-bit side x side frames, integer arithmetic, bit-exact.
 *   PB_IMG_BLUR   gauss_blur: separable 5x5 binomial (1 4 6 4 1), >> 8, the
 *                 2-pixel border passes through; in[0] -> every out[k]
 *   PB_IMG_DIFF   frame_diff_threshold: |in[0] - in[1]| > threshold ? 255 : 0
 *                 (in[0] = "cur", in[1] = "prev")
 *   PB_IMG_MEDIAN plus_median: median of the pixel and its 4-neighbourhood, the
 *                 1-pixel border passes through */
#define PB_IMG_BLUR 0
#define PB_IMG_DIFF 1
#define PB_IMG_MEDIAN 2
typedef struct {
  pb_span_ref in[2];
  pb_span_ref out[PB_MAX_PORTS];
  int32_t n_out;
  int32_t op;
  int32_t side;
  int32_t threshold;
  int32_t cond;
  int32_t pad_;
} pb_image_actor;
int pb_fire_image(pb_image_actor actor, pb_resolved res, void* stream);

/* The motion region blur -> frame_diff_threshold(cur = blur, prev = blur one
 * frame earlier through a delay-1 channel) -> plus_median as ONE launch
 * (motion.py:74-108; the engine fuses it when all three always fire): a CTA
 * takes a run of consecutive frames of one stream, blurs each once and keeps
 * the previous blurred frame in shared memory, so the f_cur and f_mask
 * channels never reach HBM.  The delayed channel stays a ring: its token is
 * read at the epoch's first iteration and written at the last (the next
 * epoch's first).  Same integers as the three image actors.  Power-of-two
 * sides 8..128. */
typedef struct {
  pb_span_ref in;        /* blur's input */
  pb_span_ref prev_in;   /* frame_diff_threshold.prev (consumer side of the delayed ring) */
  pb_span_ref prev_out;  /* blur -> delayed ring (producer side) */
  pb_span_ref out;       /* plus_median's output */
  int32_t side;
  int32_t threshold;
} pb_motion_region;
int pb_fire_motion_region(pb_motion_region region, pb_resolved res, void* stream);

/* ------------------------------------------------ CNN actors (vision example) */
/* The paper's adaptive DNN is not in the reference
 * package; these actors and their oracle (oracle/cnn.py) are builder-defined.
 * Tokens are NHWC fp32 frames; `frames` = frames per firing (port rate). */

/* conv2d_relu_pool: 5x5 conv (zero pad), bias, ReLU, 2x2 max pool, 32 output
 * channels, as a warp-specialised tcgen05 implicit GEMM (bf16x3 split
 * operands, fp32 accumulation in TMEM).  cin must be 3 or a multiple of 16.
 * weights: the host-prepared device layout of W[32][25*cin] ((ky,kx,ci)
 * order): per 16-wide K-step a 64-row [bf16 hi; bf16 lo] UMMA operand
 * (paper_1802_06625_b200/cnn_weights.py conv_device_layout). */
typedef struct {
  pb_span_ref in;
  pb_span_ref out;
  const void* weights;
  const float* bias;       /* [32] */
  int32_t frames;
  int32_t h, w, cin, cout, pad;
  int32_t cond;
  int32_t debug;           /* 0; profiling only: bit0 skip patch fill, bit1 skip
                              epilogue, bit2 skip MMAs, bit3 skip the layer-1 raw
                              TMA loads (results are garbage) */
  int32_t math;            /* PB_CONV_BF16X3 or PB_CONV_I8 (cin 32 only; other
                              shapes run bf16x3 whatever this says) */
  const void* weights_i8;  /* PB_CONV_I8: cnn_weights.conv_device_layout_i8 (per
                              K-step a 64-row [w0 0; w1 w0] int8 operand, then
                              32 float dequantisation factors); may be NULL
                              when math is PB_CONV_BF16X3 */
  float* absmax_out;       /* NULL, or [live frames] max |output| of every
                              output frame of this launch (in live-firing order;
                              feeds the next conv's int8 quantisation) */
  const float* absmax_in;  /* NULL, or the producer launch's absmax_out for
                              this launch's input frames (same condition, same
                              live firings); NULL: computed by a pre-pass */
} pb_conv_actor;
enum { PB_CONV_BF16X3 = 0, PB_CONV_I8 = 1 };
int pb_fire_conv_pool(pb_conv_actor actor, pb_resolved res, void* stream);
/* Profiling builds (-DPB_CONV_PROF=1) only: per-CTA role timing counters of
 * conv_pool_kernel, uint64 [160][16] clock cycles (slots in csrc/pb_cnn.cu);
 * all zero in normal builds.  reset != 0 zeroes them after the copy. */
int pb_conv_debug_counters(unsigned long long* out, int reset);

/* dense: out[f] = W x[f] + b, W [nout][nin] (nout <= 112, nin % 64 == 0), as a
 * tcgen05 GEMM over 128 frames gathered across firings (bf16x3 split, fp32
 * accumulation; split-K with a deterministic last-CTA reduction when there
 * are fewer frame tiles than SMs).  weights: cnn_weights.dense_device_layout. */
typedef struct {
  pb_span_ref in;
  pb_span_ref out;
  const void* weights;
  const float* bias;
  int32_t frames, nin, nout, cond;
} pb_dense_actor;
int pb_fire_dense(pb_dense_actor actor, pb_resolved res, void* stream);

/* classify_merge: live chain input -> W5 relu(W4 relu(x) + b4) + b5; live
 * bypass input -> every logit = marker; != 1 live input sets *error_flag. */
typedef struct {
  pb_span_ref chain;
  pb_span_ref bypass;
  pb_span_ref out;
  const float* w4;
  const float* b4;
  const float* w5;
  const float* b5;
  int32_t frames, nin, nhid, nout;
  float marker;
  int32_t cond;
  int32_t* error_flag;
} pb_classify_actor;
int pb_fire_classify(pb_classify_actor actor, pb_resolved res, void* stream);

/* ------------------------------------------ host configuration actors (native) */
/* Control tokens of _PolicyBase.fire (behavior.py:212-218) with CPython's
 * Mersenne Twister (random.Random(seed)) reproduced bit for bit:
 * kind 0 fixed_policy(element), 1 alternate_policy, 2 seeded_policy,
 * 3 subset_policy(min_active).  Writes n_firings tokens of token_bytes
 * (values zero-padded) starting at firing `first`; the generator state is
 * kept in *state (opaque, PB_POLICY_STATE_BYTES) so successive epochs continue
 * the same sequence.  pb_policy_init seeds it (seed < 0 -> None -> 0). */
#define PB_POLICY_STATE_BYTES 2560
int pb_policy_init(void* state, int64_t seed);
int pb_policy_tokens(void* state, int kind, int length, int param, int64_t first,
                     int64_t n_firings, uint8_t* out, int token_bytes);
/* Seeding many streams at once: states is n_streams * PB_POLICY_STATE_BYTES,
 * seeds[n_streams]; tokens out[s][n_firings][token_bytes]; threads <= 0 ->
 * hardware concurrency. */
int pb_policy_tokens_streams(void* states, int n_streams, int kind, int length, int param,
                             int64_t first, int64_t n_firings, uint8_t* out, int token_bytes,
                             int threads);
/* zlib.crc32 as used by actor_seed (behavior.py:17-21). */
uint32_t pb_crc32(const uint8_t* data, size_t n);

#ifdef __cplusplus
}
#endif
#endif /* PRUNE_B200_H */
