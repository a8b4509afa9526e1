// Runtime plumbing of libprune_b200: errors, device memory, streams, events,
// the Eq. 2 capacity plan (fifos.py:49-139) and device-resident rings
// (FifoChannel, fifos.py:142-338).
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "pb_common.cuh"

namespace pb {

static thread_local std::string g_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_error = msg; }

int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}

int cuda_fail(cudaError_t err, const char* what) {
  g_error = std::string(what) + ": " + cudaGetErrorName(err) + " (" + cudaGetErrorString(err) + ")";
  return err == cudaErrorMemoryAllocation ? PB_E_NOMEM : PB_E_CUDA;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int device() {
  int dev = 0;
  const cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) {
    cuda_fail(err, "cudaGetDevice");
    return -1;
  }
  if (dev >= kMaxDevices) {
    fail(PB_E_UNSUPPORTED, "device ordinal " + std::to_string(dev) + " >= " +
                               std::to_string(kMaxDevices));
    return -1;
  }
  return dev;
}

int scratch(int slot, size_t bytes, void** out, bool zero_new, cudaStream_t st) {
  static std::mutex mu;
  static void* bufs[kMaxDevices][kScratchSlots] = {};
  static size_t sizes[kMaxDevices][kScratchSlots] = {};
  const int dev = device();
  if (dev < 0) return PB_E_CUDA;
  std::lock_guard<std::mutex> lock(mu);
  if (bytes > sizes[dev][slot]) {
    if (bufs[dev][slot]) PB_CUDA(cudaFree(bufs[dev][slot]));   // synchronising
    bufs[dev][slot] = nullptr;
    sizes[dev][slot] = 0;
    PB_CUDA(cudaMalloc(&bufs[dev][slot], bytes));
    sizes[dev][slot] = bytes;
    if (zero_new) PB_CUDA(cudaMemsetAsync(bufs[dev][slot], 0, bytes, st));
  }
  *out = bufs[dev][slot];
  return PB_OK;
}

}  // namespace pb

using pb::fail;

extern "C" {

int pb_abi_version(void) { return PB_ABI_VERSION; }
const char* pb_last_error(void) { return pb::g_error.c_str(); }
int64_t pb_launch_count(void) { return pb::g_launches.load(); }

int pb_device_count(int* n) {
  if (!n) return fail(PB_E_INVALID, "pb_device_count: null out");
  int c = 0;
  cudaError_t err = cudaGetDeviceCount(&c);
  if (err != cudaSuccess) {
    cudaGetLastError();
    *n = 0;
    return pb::cuda_fail(err, "cudaGetDeviceCount");
  }
  *n = c;
  return PB_OK;
}

int pb_set_device(int device) {
  PB_CUDA(cudaSetDevice(device));
  return PB_OK;
}

int pb_device_sync(void) {
  PB_CUDA(cudaDeviceSynchronize());
  return PB_OK;
}

int pb_sm_count(int* n) {
  int dev = 0;
  PB_CUDA(cudaGetDevice(&dev));
  PB_CUDA(cudaDeviceGetAttribute(n, cudaDevAttrMultiProcessorCount, dev));
  return PB_OK;
}

int pb_malloc(void** dptr, size_t bytes) {
  if (!dptr) return fail(PB_E_INVALID, "pb_malloc: null out");
  *dptr = nullptr;
  if (bytes == 0) bytes = 16;
  PB_CUDA(cudaMalloc(dptr, bytes));
  return PB_OK;
}

int pb_free(void* dptr) {
  if (dptr) PB_CUDA(cudaFree(dptr));
  return PB_OK;
}

int pb_host_alloc(void** hptr, size_t bytes) {
  if (!hptr) return fail(PB_E_INVALID, "pb_host_alloc: null out");
  if (bytes == 0) bytes = 16;
  PB_CUDA(cudaHostAlloc(hptr, bytes, cudaHostAllocPortable));
  return PB_OK;
}

int pb_host_free(void* hptr) {
  if (hptr) PB_CUDA(cudaFreeHost(hptr));
  return PB_OK;
}

int pb_host_register(void* hptr, size_t bytes) {
  if (!hptr || !bytes) return fail(PB_E_INVALID, "pb_host_register: empty range");
  cudaError_t e = cudaHostRegister(hptr, bytes, cudaHostRegisterPortable);
  if (e == cudaErrorHostMemoryAlreadyRegistered) {
    (void)cudaGetLastError();
    return 1;  /* already page-locked by the caller: nothing to undo later */
  }
  PB_CUDA(e);
  return PB_OK;
}

int pb_host_unregister(void* hptr) {
  if (!hptr) return PB_OK;
  cudaError_t e = cudaHostUnregister(hptr);
  if (e == cudaErrorHostMemoryNotRegistered) {
    (void)cudaGetLastError();
    return PB_OK;
  }
  PB_CUDA(e);
  return PB_OK;
}

int pb_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes) PB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, pb::as_stream(stream)));
  return PB_OK;
}

int pb_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes) PB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, pb::as_stream(stream)));
  return PB_OK;
}

int pb_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes) PB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, pb::as_stream(stream)));
  return PB_OK;
}

int pb_memset(void* dst, int value, size_t bytes, void* stream) {
  if (bytes) PB_CUDA(cudaMemsetAsync(dst, value, bytes, pb::as_stream(stream)));
  return PB_OK;
}

int pb_memcpy_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                 size_t height, int kind, void* stream) {
  cudaMemcpyKind k = kind == 1 ? cudaMemcpyHostToDevice
                   : kind == 2 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (kind < 1 || kind > 3) return fail(PB_E_INVALID, "pb_memcpy_2d: bad kind");
  if (width && height)
    PB_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, k, pb::as_stream(stream)));
  return PB_OK;
}

int pb_stream_create(void** stream) {
  cudaStream_t s;
  PB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *stream = s;
  return PB_OK;
}

int pb_stream_destroy(void* stream) {
  if (stream) PB_CUDA(cudaStreamDestroy(pb::as_stream(stream)));
  return PB_OK;
}

int pb_stream_sync(void* stream) {
  PB_CUDA(cudaStreamSynchronize(pb::as_stream(stream)));
  return PB_OK;
}

int pb_event_create(void** event) {
  // blocking sync: a host thread waiting on the event sleeps instead of
  // spinning on a core the pipelined runtime's hashing threads need
  cudaEvent_t e;
  PB_CUDA(cudaEventCreateWithFlags(&e, cudaEventBlockingSync));
  *event = e;
  return PB_OK;
}

int pb_event_destroy(void* event) {
  if (event) PB_CUDA(cudaEventDestroy(reinterpret_cast<cudaEvent_t>(event)));
  return PB_OK;
}

int pb_event_record(void* event, void* stream) {
  PB_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(event), pb::as_stream(stream)));
  return PB_OK;
}

int pb_event_elapsed_ms(void* start, void* end, float* ms) {
  PB_CUDA(cudaEventSynchronize(reinterpret_cast<cudaEvent_t>(end)));
  PB_CUDA(cudaEventElapsedTime(ms, reinterpret_cast<cudaEvent_t>(start),
                               reinterpret_cast<cudaEvent_t>(end)));
  return PB_OK;
}

int pb_event_sync(void* event) {
  PB_CUDA(cudaEventSynchronize(reinterpret_cast<cudaEvent_t>(event)));
  return PB_OK;
}

int pb_stream_wait(void* stream, void* event) {
  PB_CUDA(cudaStreamWaitEvent(pb::as_stream(stream), reinterpret_cast<cudaEvent_t>(event), 0));
  return PB_OK;
}

// ------------------------------------------------------------ capacity plan

int pb_layout_plan(int rate, int delay, int factor, int token_bytes, pb_plan* out) {
  // _validate, fifos.py:76-84
  if (rate < 1) return fail(PB_E_INVALID, "rate must be >= 1, got " + std::to_string(rate));
  if (token_bytes < 1)
    return fail(PB_E_INVALID, "token size must be >= 1 byte, got " + std::to_string(token_bytes));
  if (delay < 0) return fail(PB_E_INVALID, "delay must be >= 0, got " + std::to_string(delay));
  if (factor < 2)
    return fail(PB_E_INVALID, "buffering factor must be >= 2, got " + std::to_string(factor));
  pb_plan p{};
  p.rate = rate;
  p.token_bytes = token_bytes;
  p.delay = delay;
  p.factor = factor;
  p.aligned = (delay % rate) == 0;
  if (p.aligned) {
    p.slots = std::max<int64_t>((int64_t)rate * factor, delay);
    p.copy_src = p.copy_dst = p.copy_count = -1;
  } else {
    p.slots = (int64_t)rate * factor + delay;
    p.copy_src = (int64_t)rate * factor;
    p.copy_dst = 0;
    p.copy_count = delay;
  }
  p.nbytes = p.slots * token_bytes;
  if (out) *out = p;
  return PB_OK;
}

static int64_t floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

int64_t pb_copy_gate(int64_t n, int rate, int delay, int factor) {
  int64_t span = std::min<int64_t>(delay, (int64_t)rate * factor);
  return n * factor + floordiv(span - 1, rate) + 1;
}

int64_t pb_writer_gate(int64_t w, int rate, int delay, int factor, int aligned) {
  if (aligned) {
    int64_t slots = std::max<int64_t>((int64_t)rate * factor, delay);
    int64_t last = delay + (w + 1) * rate - 1 - slots;
    return last < 0 ? 0 : last / rate + 1;
  }
  int64_t n = w / factor, c = w % factor;
  if (n == 0) return 0;
  if (delay > (int64_t)rate * factor) return pb_copy_gate(n - 1, rate, delay, factor);
  return floordiv(delay + (n - 1) * (int64_t)rate * factor + (c + 1) * rate - 1, rate) + 1;
}

int64_t pb_reader_gate(int64_t i, int rate, int delay) {
  int64_t need = (i + 1) * rate - delay;
  if (need <= 0) return 0;
  return (need + rate - 1) / rate;
}

}  // extern "C"

// ------------------------------------------------------------------- rings

struct pb_ring {
  pb_plan plan;
  int n_streams;
  uint8_t* data;        // device [n_streams][nbytes]
  int64_t* counters;    // device int64[4][n_streams]: writes, reads, max_occ, copies
  bool closed;
  std::string poisoned;
  bool is_poisoned;
  // host-side transfers are single-producer / single-consumer across threads
  // (FifoChannel's contract, fifos.py:142-160): one lock serialises the
  // counter read-modify-write of a push and a pop, and the blocking variants
  // wait on `cv` for space / tokens / close / poison
  std::mutex mu;
  std::condition_variable cv;
};

namespace {

enum { C_WRITES = 0, C_READS = 1, C_MAXOCC = 2, C_COPIES = 3, C_N = 4 };

int load_counters(const pb_ring* r, int s, int64_t c[C_N]) {
  for (int k = 0; k < C_N; ++k)
    PB_CUDA(cudaMemcpy(&c[k], r->counters + (int64_t)k * r->n_streams + s, sizeof(int64_t),
                       cudaMemcpyDeviceToHost));
  return PB_OK;
}

int store_counters(const pb_ring* r, int s, const int64_t c[C_N]) {
  for (int k = 0; k < C_N; ++k)
    PB_CUDA(cudaMemcpy(r->counters + (int64_t)k * r->n_streams + s, &c[k], sizeof(int64_t),
                       cudaMemcpyHostToDevice));
  return PB_OK;
}

// _run_copy, fifos.py:206-215 (unaligned layouts only)
int run_copy(pb_ring* r, int s, int64_t c[C_N], cudaStream_t st) {
  const pb_plan& p = r->plan;
  uint8_t* base = r->data + (int64_t)s * p.nbytes;
  int64_t tb = p.token_bytes;
  // source [copy_src, copy_src+count) and destination [0, count) may overlap
  // only when delay > rate*factor; stage through a temporary like the
  // reference's bytes() snapshot.
  size_t n = (size_t)(p.copy_count * tb);
  if (n) {
    void* tmp = nullptr;
    PB_CUDA(cudaMallocAsync(&tmp, n, st));
    PB_CUDA(cudaMemcpyAsync(tmp, base + p.copy_src * tb, n, cudaMemcpyDeviceToDevice, st));
    PB_CUDA(cudaMemcpyAsync(base + p.copy_dst * tb, tmp, n, cudaMemcpyDeviceToDevice, st));
    PB_CUDA(cudaFreeAsync(tmp, st));
  }
  c[C_COPIES] += 1;
  return PB_OK;
}

bool copy_ready(const pb_plan& p, const int64_t c[C_N]) {
  return c[C_READS] >= pb_copy_gate(c[C_COPIES], p.rate, p.delay, p.factor);
}

bool copy_pending(const pb_plan& p, const int64_t c[C_N]) {
  return !p.aligned && c[C_COPIES] < c[C_WRITES] / p.factor;
}

}  // namespace

extern "C" {

int pb_ring_create(int rate, int token_bytes, int delay, int factor, int n_streams,
                   const void* delay_payload, pb_ring** out) {
  if (!out) return fail(PB_E_INVALID, "pb_ring_create: null out");
  *out = nullptr;
  if (n_streams < 1) return fail(PB_E_INVALID, "n_streams must be >= 1");
  pb_plan plan;
  int rc = pb_layout_plan(rate, delay, factor, token_bytes, &plan);
  if (rc) return rc;
  pb_ring* r = new pb_ring();
  r->plan = plan;
  r->n_streams = n_streams;
  r->closed = false;
  r->is_poisoned = false;
  cudaError_t err = cudaMalloc(&r->data, (size_t)plan.nbytes * n_streams);
  if (err != cudaSuccess) {
    delete r;
    return pb::cuda_fail(err, "pb_ring_create: cudaMalloc data");
  }
  err = cudaMalloc(&r->counters, sizeof(int64_t) * C_N * n_streams);
  if (err != cudaSuccess) {
    cudaFree(r->data);
    delete r;
    return pb::cuda_fail(err, "pb_ring_create: cudaMalloc counters");
  }
  std::vector<int64_t> init((size_t)C_N * n_streams, 0);
  for (int s = 0; s < n_streams; ++s) init[(size_t)C_MAXOCC * n_streams + s] = delay;
  cudaMemcpy(r->counters, init.data(), init.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
  cudaMemset(r->data, 0, (size_t)plan.nbytes * n_streams);
  if (delay_payload && delay > 0) {
    for (int s = 0; s < n_streams; ++s)
      cudaMemcpy(r->data + (int64_t)s * plan.nbytes, delay_payload, (size_t)delay * token_bytes,
                 cudaMemcpyHostToDevice);
  }
  err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    cudaFree(r->data);
    cudaFree(r->counters);
    delete r;
    return pb::cuda_fail(err, "pb_ring_create: init");
  }
  *out = r;
  return PB_OK;
}

int pb_ring_destroy(pb_ring* ring) {
  if (!ring) return PB_OK;
  cudaFree(ring->data);
  cudaFree(ring->counters);
  delete ring;
  return PB_OK;
}

int pb_ring_plan(const pb_ring* ring, pb_plan* out) {
  if (!ring || !out) return fail(PB_E_INVALID, "pb_ring_plan: null argument");
  *out = ring->plan;
  return PB_OK;
}

int pb_ring_storage(const pb_ring* ring, void** data, int64_t* stream_stride,
                    int64_t** counters) {
  if (!ring) return fail(PB_E_INVALID, "pb_ring_storage: null ring");
  if (data) *data = ring->data;
  if (stream_stride) *stream_stride = ring->plan.nbytes;
  if (counters) *counters = ring->counters;
  return PB_OK;
}

static int check_stream(const pb_ring* r, int s) {
  if (!r) return fail(PB_E_INVALID, "null ring");
  if (s < 0 || s >= r->n_streams)
    return fail(PB_E_INVALID, "stream " + std::to_string(s) + " outside 0.." +
                                  std::to_string(r->n_streams - 1));
  if (r->is_poisoned) return fail(PB_E_POISONED, "channel poisoned: " + r->poisoned);
  return PB_OK;
}

namespace {
constexpr int kWouldBlock = 1;   // internal: the gate is not open yet
}

// write_start/write_end for n chunks, fifos.py:223-269 (ring->mu held)
static int push_locked(pb_ring* ring, int stream, const void* src, int64_t n_chunks,
                       void* cuda_stream) {
  int rc = check_stream(ring, stream);
  if (rc) return rc;
  if (ring->closed) return fail(PB_E_PROTOCOL, "write after close");
  if (n_chunks < 0) return fail(PB_E_INVALID, "negative chunk count");
  const pb_plan& p = ring->plan;
  cudaStream_t st = pb::as_stream(cuda_stream);
  int64_t c[C_N];
  rc = load_counters(ring, stream, c);
  if (rc) return rc;
  if (n_chunks == 0) return PB_OK;
  // the writer gate is monotone in w: the last chunk's gate bounds them all
  int64_t need = pb_writer_gate(c[C_WRITES] + n_chunks - 1, p.rate, p.delay, p.factor, p.aligned);
  if (c[C_READS] < need) {
    fail(PB_E_PROTOCOL, "write of " + std::to_string(n_chunks) +
                            " chunks would block: ring full (" + std::to_string(c[C_READS]) +
                            " reads done, " + std::to_string(need) + " needed)");
    return kWouldBlock;
  }
  const uint8_t* h = static_cast<const uint8_t*>(src);
  uint8_t* base = ring->data + (int64_t)stream * p.nbytes;
  int64_t span = (int64_t)p.rate * p.token_bytes;
  for (int64_t k = 0; k < n_chunks; ++k) {
    if (copy_pending(p, c)) {
      rc = run_copy(ring, stream, c, st);
      if (rc) return rc;
    }
    int64_t w = c[C_WRITES];
    int64_t slot = p.aligned ? (p.delay + w * p.rate) % p.slots : p.delay + (w % p.factor) * p.rate;
    PB_CUDA(cudaMemcpyAsync(base + slot * p.token_bytes, h + k * span, (size_t)span,
                            cudaMemcpyHostToDevice, st));
    c[C_WRITES] += 1;
    int64_t occ = p.delay + (int64_t)p.rate * (c[C_WRITES] - c[C_READS]);
    c[C_MAXOCC] = std::max(c[C_MAXOCC], occ);
    if (!p.aligned && w % p.factor == p.factor - 1 && copy_ready(p, c)) {
      rc = run_copy(ring, stream, c, st);
      if (rc) return rc;
    }
  }
  PB_CUDA(cudaStreamSynchronize(st));
  return store_counters(ring, stream, c);
}

// read_start/read_end for n chunks, fifos.py:280-323 (ring->mu held)
static int pop_locked(pb_ring* ring, int stream, void* dst, int64_t n_chunks,
                      void* cuda_stream) {
  int rc = check_stream(ring, stream);
  if (rc) return rc;
  if (n_chunks < 0) return fail(PB_E_INVALID, "negative chunk count");
  const pb_plan& p = ring->plan;
  cudaStream_t st = pb::as_stream(cuda_stream);
  int64_t c[C_N];
  rc = load_counters(ring, stream, c);
  if (rc) return rc;
  uint8_t* h = static_cast<uint8_t*>(dst);
  const uint8_t* base = ring->data + (int64_t)stream * p.nbytes;
  int64_t span = (int64_t)p.rate * p.token_bytes;
  // all-or-nothing: check every chunk is available before moving bytes
  int64_t last = c[C_READS] + n_chunks - 1;
  if (n_chunks > 0 && c[C_WRITES] < pb_reader_gate(last, p.rate, p.delay)) {
    if (ring->closed)
      return fail(PB_E_EOS, "channel closed with fewer tokens than requested");
    fail(PB_E_PROTOCOL, "read would block: not enough tokens published");
    return kWouldBlock;
  }
  for (int64_t k = 0; k < n_chunks; ++k) {
    int64_t i = c[C_READS];
    while (!p.aligned && c[C_COPIES] < i / p.factor) {
      if (copy_ready(p, c) && (copy_pending(p, c) || ring->closed)) {
        rc = run_copy(ring, stream, c, st);
        if (rc) return rc;
      } else {
        fail(PB_E_PROTOCOL, "read would block: wrap copy not ready");
        return kWouldBlock;
      }
    }
    int64_t slot = p.aligned ? (i * p.rate) % p.slots : (i % p.factor) * p.rate;
    PB_CUDA(cudaMemcpyAsync(h + k * span, base + slot * p.token_bytes, (size_t)span,
                            cudaMemcpyDeviceToHost, st));
    c[C_READS] += 1;
  }
  PB_CUDA(cudaStreamSynchronize(st));
  return store_counters(ring, stream, c);
}

}  // extern "C"

// one transfer attempt, or (timeout_ms != 0) wait until it can proceed, the
// ring closes / is poisoned, or timeout_ms elapses (< 0: no limit)
template <typename Op>
static int transfer(pb_ring* ring, int64_t timeout_ms, Op op) {
  if (!ring) return fail(PB_E_INVALID, "null ring");
  std::unique_lock<std::mutex> lk(ring->mu);
  const auto until = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms);
  for (;;) {
    const int rc = op();
    if (rc != kWouldBlock) {
      if (rc == PB_OK) ring->cv.notify_all();
      return rc;
    }
    if (timeout_ms == 0) return PB_E_PROTOCOL;
    if (timeout_ms < 0) {
      ring->cv.wait(lk);
    } else if (ring->cv.wait_until(lk, until) == std::cv_status::timeout) {
      const int again = op();   // a last look after the deadline
      if (again != kWouldBlock) {
        if (again == PB_OK) ring->cv.notify_all();
        return again;
      }
      return fail(PB_E_TIMEOUT, "ring transfer timed out after " + std::to_string(timeout_ms) +
                                    " ms");
    }
  }
}

extern "C" {

int pb_ring_push_host(pb_ring* ring, int stream, const void* src, int64_t n_chunks,
                      void* cuda_stream) {
  return transfer(ring, 0, [&] { return push_locked(ring, stream, src, n_chunks, cuda_stream); });
}

int pb_ring_pop_host(pb_ring* ring, int stream, void* dst, int64_t n_chunks, void* cuda_stream) {
  return transfer(ring, 0, [&] { return pop_locked(ring, stream, dst, n_chunks, cuda_stream); });
}

int pb_ring_push_host_wait(pb_ring* ring, int stream, const void* src, int64_t n_chunks,
                           void* cuda_stream, int64_t timeout_ms) {
  return transfer(ring, timeout_ms,
                  [&] { return push_locked(ring, stream, src, n_chunks, cuda_stream); });
}

int pb_ring_pop_host_wait(pb_ring* ring, int stream, void* dst, int64_t n_chunks,
                          void* cuda_stream, int64_t timeout_ms) {
  return transfer(ring, timeout_ms,
                  [&] { return pop_locked(ring, stream, dst, n_chunks, cuda_stream); });
}

int pb_ring_counters(const pb_ring* ring, int stream, int64_t* writes, int64_t* reads,
                     int64_t* max_occupancy) {
  if (!ring) return fail(PB_E_INVALID, "null ring");
  std::lock_guard<std::mutex> lk(const_cast<pb_ring*>(ring)->mu);
  if (stream < 0 || stream >= ring->n_streams) return fail(PB_E_INVALID, "bad stream");
  int64_t c[C_N];
  int rc = load_counters(ring, stream, c);
  if (rc) return rc;
  if (writes) *writes = c[C_WRITES];
  if (reads) *reads = c[C_READS];
  if (max_occupancy) *max_occupancy = c[C_MAXOCC];
  return PB_OK;
}

int pb_ring_close(pb_ring* ring) {
  if (!ring) return fail(PB_E_INVALID, "null ring");
  {
    std::lock_guard<std::mutex> lk(ring->mu);
    if (!ring->is_poisoned) ring->closed = true;
  }
  ring->cv.notify_all();
  return PB_OK;
}

int pb_ring_poison(pb_ring* ring, const char* reason) {
  if (!ring) return fail(PB_E_INVALID, "null ring");
  {
    std::lock_guard<std::mutex> lk(ring->mu);
    ring->is_poisoned = true;
    ring->poisoned = (reason && *reason) ? reason : "failure elsewhere in the graph";
  }
  ring->cv.notify_all();
  return PB_OK;
}

}  // extern "C"
