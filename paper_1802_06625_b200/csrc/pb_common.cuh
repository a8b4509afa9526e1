// Shared internals of libprune_b200: error plumbing, launch accounting and
// the device-side span addressing every actor kernel uses.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/prune_b200.h"

namespace pb {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t err, const char* what);
void count_launch(int n = 1);

// Per-device library state (one process may drive several devices in turn):
// the current device's ordinal, and grow-only scratch buffers owned by the
// library, one per (device, slot).  Launches on one device are stream-ordered
// by the caller (one compute stream per runtime).
constexpr int kMaxDevices = 16;
int device();   // current device ordinal, < kMaxDevices, or -1 on error (pb_last_error set)
enum ScratchSlot { kScratchBankPlan = 0, kScratchConvUnits, kScratchDensePartial,
                   kScratchDenseCounters, kScratchConvRows, kScratchConvAbsmax, kScratchSlots };
// at least `bytes` of device memory for `slot` on the current device; newly
// allocated memory is zeroed on `st` when zero_new
int scratch(int slot, size_t bytes, void** out, bool zero_new = false, cudaStream_t st = 0);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// the row-streaming conv kernel with A in TMEM (pb_conv_rows.cu); Cin 3 / 32;
// returns 1 without launching when it does not handle the shape
int fire_conv_rows(const pb_conv_actor& actor, const pb_resolved& res, cudaStream_t st, int sms);
int conv_absmax_out(const pb_conv_actor& actor, const pb_resolved& res, cudaStream_t st);

}  // namespace pb

// Programmatic dependent launch for the short kernels of an epoch step: the
// next kernel of the stream is scheduled while this one runs and parks in
// griddepcontrol.wait, so the launch latency between the step's kernels
// overlaps work.  Every PDL kernel calls pb::pdl_wait() before its first
// global memory access, so stream order semantics are unchanged.
#ifndef PB_PDL
#define PB_PDL 1
#endif
namespace pb {
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = PB_PDL;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}
}  // namespace pb

#define PB_LAUNCH_PDL(kern, grid, block, smem, st, ...)                            \
  do {                                                                           \
    cudaError_t err__ = pb::launch_pdl(kern, grid, block, smem, st, __VA_ARGS__); \
    if (err__ != cudaSuccess) return pb::cuda_fail(err__, #kern);                \
  } while (0)

#define PB_CUDA(call)                                        \
  do {                                                       \
    cudaError_t err__ = (call);                              \
    if (err__ != cudaSuccess) return pb::cuda_fail(err__, #call); \
  } while (0)

// Check the launch that was just issued.
#define PB_LAUNCHED(name)                                    \
  do {                                                       \
    cudaError_t err__ = cudaGetLastError();                  \
    if (err__ != cudaSuccess) return pb::cuda_fail(err__, name); \
    pb::count_launch();                                      \
  } while (0)

// ----------------------------------------------------------------- device side
namespace pb {

// mbarrier phase wait that cannot hang the device: after 5 s of failed
// try_waits (no pipeline wait in these kernels legitimately lasts longer than a
// launch) it traps, so a protocol fault becomes a launch error instead of a
// hung GPU.  One inline loop; %globaltimer is read every 1024 failed tries.
// SCOPE_CLUSTER: acquire at cluster scope (CTA-pair pipelines).
#define PB_MBAR_WAIT_TRAP(addr, parity, TRYWAIT)                                   \
  asm volatile(                                                                   \
      "{\n\t.reg .pred p, q;\n\t.reg .u64 t0, t1;\n\t.reg .u32 i;\n\t"              \
      "mov.u32 i, 0;\n\t"                                                          \
      "mov.u64 t0, %%globaltimer;\n"                                               \
      "W_%=:\n\t" TRYWAIT " p, [%0], %1;\n\t"                                         \
      "@p bra D_%=;\n\t"                                                            \
      "add.u32 i, i, 1;\n\t"                                                        \
      "and.b32 i, i, 1023;\n\t"                                                     \
      "setp.ne.u32 q, i, 0;\n\t"                                                    \
      "@q bra W_%=;\n\t"                                                            \
      "mov.u64 t1, %%globaltimer;\n\t"                                              \
      "sub.u64 t1, t1, t0;\n\t"                                                     \
      "setp.gt.u64 q, t1, 5000000000;\n\t"                                          \
      "@q trap;\n\t"                                                                \
      "bra W_%=;\n"                                                                  \
      "D_%=:\n\t}" ::"r"(addr),                                                     \
      "r"(parity)                                                                   \
      : "memory")

__device__ __forceinline__ void mbar_wait_trap(uint32_t addr, uint32_t parity) {
  PB_MBAR_WAIT_TRAP(addr, parity, "mbarrier.try_wait.parity.shared::cta.b64");
}
__device__ __forceinline__ void mbar_wait_trap_cluster(uint32_t addr, uint32_t parity) {
  PB_MBAR_WAIT_TRAP(addr, parity, "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64");
}

// wait for the previous kernel of the stream (PDL), then let the next one be
// scheduled
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Index of the span a port uses at iteration n of stream s (pb_span_ref doc).
__device__ __forceinline__ int64_t span_index(const pb_span_ref& r, const pb_resolved& res,
                                              int s, int n) {
  int64_t idx = n;
  if (r.index_cond >= 0)
    idx = res.prefix[((int64_t)r.index_cond * res.n_streams + s) * res.cap + n];
  int64_t b = r.base ? r.base[s] : 0;
  const int64_t x = b + idx + r.offset;
  // 32-bit remainder while the ring counter fits (the 64-bit one is a long
  // software sequence, executed per firing by every actor kernel)
  if ((uint64_t)x <= 0xFFFFFFFFull) return (int64_t)((uint32_t)x % (uint32_t)r.slots);
  return x % r.slots;
}

__device__ __forceinline__ uint8_t* span_ptr(const pb_span_ref& r, const pb_resolved& res,
                                             int s, int n) {
  return r.data + (int64_t)s * r.stream_stride + span_index(r, res, s, n) * r.span_bytes;
}

__device__ __forceinline__ bool active(const pb_resolved& res, int cond, int s, int n) {
  if (cond < 0) return true;
  return res.act[((int64_t)cond * res.n_streams + s) * res.cap + n] != 0;
}

__device__ __forceinline__ int32_t cond_count(const pb_resolved& res, int cond, int s) {
  if (cond < 0) return res.n_iter;
  return res.count[(int64_t)cond * res.n_streams + s];
}

// Iteration of the j-th firing of an actor gated by cond.
__device__ __forceinline__ int32_t firing_iter(const pb_resolved& res, int cond, int s, int j) {
  if (cond < 0) return j;
  return res.worklist[((int64_t)cond * res.n_streams + s) * res.cap + j];
}

}  // namespace pb
