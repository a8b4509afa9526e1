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

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace pb

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

// Index of the span a port uses at iteration n of stream s (pb_span_ref doc).
__device__ __forceinline__ int64_t span_index(const pb_span_ref& r, const pb_resolved& res,
                                              int s, int n) {
  int64_t idx = n;
  if (r.index_cond >= 0)
    idx = res.prefix[((int64_t)r.index_cond * res.n_streams + s) * res.cap + n];
  int64_t b = r.base ? r.base[s] : 0;
  return (b + idx + r.offset) % r.slots;
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
