// Batched firings of the remaining data-parallel actors:
//   branch_sum  apps/predistortion.py:68-83
//   route / passthrough / add_mod / merge   behavior.py:158-199
//   matmul      apps/bypass.py:36-49
//   path_merge  apps/bypass.py:52-66
// One CTA covers one (stream, iteration) firing (or a tile of its span).
#include <algorithm>

#include "pb_common.cuh"

namespace {

constexpr int kSumThreads = 256;

// BranchSum.fire: acc = +0; for pid in sorted(inputs): if span: acc = acc + x.
__global__ void __launch_bounds__(kSumThreads)
branch_sum_kernel(pb_sum_actor a, pb_resolved res, int64_t B, int tiles) {
  const int s = blockIdx.y;
  const int n = blockIdx.x / tiles;
  const int tile = blockIdx.x % tiles;
  if (!pb::active(res, a.cond, s, n)) return;
  const int64_t n4 = (2 * B) / 4;  // both planes, float4 units
  const int64_t k = (int64_t)tile * kSumThreads + threadIdx.x;
  if (k >= n4) return;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int p = 0; p < a.n_in; ++p) {
    const pb_span_ref& r = a.in[p];
    if (!pb::active(res, r.act_cond, s, n)) continue;
    const float4 x = __ldg(reinterpret_cast<const float4*>(pb::span_ptr(r, res, s, n)) + k);
    acc.x = __fadd_rn(acc.x, x.x);
    acc.y = __fadd_rn(acc.y, x.y);
    acc.z = __fadd_rn(acc.z, x.z);
    acc.w = __fadd_rn(acc.w, x.w);
  }
  reinterpret_cast<float4*>(pb::span_ptr(a.out, res, s, n))[k] = acc;
}

// Byte actors: out = (sum of active inputs + offset) mod 256 on every active
// output span.  Route/passthrough (one input, offset 0) reduce to a copy;
// merge with one live input is a copy and otherwise the bytewise sum.  The
// engine admits only actors whose every input span is at least as long as
// every output span (the reference indexes each input over the output span,
// behavior.py:153-199), so no input is read past its span.
__global__ void bytes_kernel(pb_bytes_actor a, pb_resolved res) {
  const int s = blockIdx.y;
  const int n = blockIdx.x;
  if (!pb::active(res, a.cond, s, n)) return;
  const uint8_t* ins[PB_MAX_PORTS];
  int n_live = 0;
  for (int p = 0; p < a.n_in; ++p) {
    if (!pb::active(res, a.in[p].act_cond, s, n)) continue;
    ins[n_live++] = pb::span_ptr(a.in[p], res, s, n);
  }
  for (int o = 0; o < a.n_out; ++o) {
    const pb_span_ref& r = a.out[o];
    if (!pb::active(res, r.act_cond, s, n)) continue;
    uint8_t* dst = pb::span_ptr(r, res, s, n);
    for (int64_t b = threadIdx.x; b < r.span_bytes; b += blockDim.x) {
      unsigned v = (unsigned)a.offset;
      for (int p = 0; p < n_live; ++p) v += ins[p][b];
      dst[b] = (uint8_t)(v & 0xFFu);
    }
  }
}

// MatMul.fire: acc = 0; for k: acc = acc + outer(w[:, k], x[k, :]).
// One thread per output element, one CTA per batch of firings.
__global__ void matmul_kernel(pb_matmul_actor a, pb_resolved res, int per_cta) {
  const int s = blockIdx.y;
  const int N = a.n;
  const int NN = N * N;
  extern __shared__ float smem[];
  float* w = smem;  // [N][N]
  for (int e = threadIdx.x; e < NN; e += blockDim.x) w[e] = a.weights[e];
  __syncthreads();
  const int slot = threadIdx.x / NN;
  const int e = threadIdx.x % NN;
  const int i = e / N, jj = e % N;
  const int cnt = pb::cond_count(res, a.cond, s);
  const int j = blockIdx.x * per_cta + slot;
  if (slot >= per_cta || j >= cnt) return;
  const int n = pb::firing_iter(res, a.cond, s, j);
  const float* x = reinterpret_cast<const float*>(pb::span_ptr(a.in, res, s, n));
  float acc = 0.0f;
  for (int k = 0; k < N; ++k) acc = __fadd_rn(acc, __fmul_rn(w[i * N + k], __ldg(x + k * N + jj)));
  reinterpret_cast<float*>(pb::span_ptr(a.out, res, s, n))[e] = acc;
}

// PathMerge.fire: (pid, span), = live; x + marker if pid is the bypass port.
__global__ void path_merge_kernel(pb_path_merge_actor a, pb_resolved res) {
  const int s = blockIdx.y;
  const int n = blockIdx.x;
  if (!pb::active(res, a.cond, s, n)) return;
  int live = -1, n_live = 0;
  for (int p = 0; p < a.n_in; ++p)
    if (pb::active(res, a.in[p].act_cond, s, n)) {
      live = p;
      ++n_live;
    }
  if (n_live != 1) {
    if (threadIdx.x == 0) atomicExch(a.error_flag, 1);
    return;
  }
  const float* x = reinterpret_cast<const float*>(pb::span_ptr(a.in[live], res, s, n));
  float* out = reinterpret_cast<float*>(pb::span_ptr(a.out, res, s, n));
  const int64_t len = a.out.span_bytes / 4;
  const bool add = live == a.bypass_index;
  for (int64_t k = threadIdx.x; k < len; k += blockDim.x) {
    float v = x[k];
    out[k] = add ? __fadd_rn(v, a.marker) : v;
  }
}

#ifndef PB_MATMUL_MF
#define PB_MATMUL_MF 4
#endif
constexpr int kMF = PB_MATMUL_MF;   // firings per lane group (matmul_packed_kernel)

// MatMul.fire for N*N/4 <= 32 dividing 32 (the reference's 8x8: 16 lanes
// per firing, two firings per warp): the group's first lane resolves the
// firing's spans once; each lane computes 4 consecutive outputs of one row
// (acc = 0, then acc + w[i][k] * x[k][j] in ascending k, every product and
// sum rounded) from float4 rows of x.
__global__ void __launch_bounds__(256)
matmul_packed_kernel(pb_matmul_actor a, pb_resolved res, int L) {
  const int s = blockIdx.y, lane = threadIdx.x & 31, N = a.n;
  __shared__ float w[32 * 4];   // N*N <= 128
  for (int e = threadIdx.x; e < N * N; e += blockDim.x) w[e] = a.weights[e];
  __syncthreads();
  const int fpw = 32 / L;
  const int g = lane / L, sub = lane - g * L;
  // each lane group takes kMF consecutive firings: the leader resolves all of
  // them at once (independent load chains), every lane then has kMF x N
  // row loads in flight
  const int j0 = (((int)blockIdx.x * 8 + (threadIdx.x >> 5)) * fpw + g) * kMF;
  const int leader = g * L;
  const unsigned grp = (L == 32 ? 0xffffffffu : ((1u << L) - 1u) << leader);
  const int cnt = pb::cond_count(res, a.cond, s);
  if (j0 >= cnt) return;   // whole lane groups leave together
  const float* x[kMF];
  float* out[kMF];
#pragma unroll
  for (int f = 0; f < kMF; ++f) {
    x[f] = nullptr;
    out[f] = nullptr;
    if (sub == 0 && j0 + f < cnt) {
      const int n = pb::firing_iter(res, a.cond, s, j0 + f);
      x[f] = reinterpret_cast<const float*>(pb::span_ptr(a.in, res, s, n));
      out[f] = reinterpret_cast<float*>(pb::span_ptr(a.out, res, s, n));
    }
  }
#pragma unroll
  for (int f = 0; f < kMF; ++f) {
    x[f] = reinterpret_cast<const float*>(
        __shfl_sync(grp, reinterpret_cast<unsigned long long>(x[f]), leader));
    out[f] = reinterpret_cast<float*>(
        __shfl_sync(grp, reinterpret_cast<unsigned long long>(out[f]), leader));
  }
  const int e0 = 4 * sub, i = e0 / N, c0 = e0 - i * N;
#pragma unroll
  for (int f = 0; f < kMF; ++f) {
    if (x[f] == nullptr) continue;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int k = 0; k < N; ++k) {
      const float4 xv = __ldg(reinterpret_cast<const float4*>(x[f] + k * N + c0));
      const float wk = w[i * N + k];
      acc[0] = __fadd_rn(acc[0], __fmul_rn(wk, xv.x));
      acc[1] = __fadd_rn(acc[1], __fmul_rn(wk, xv.y));
      acc[2] = __fadd_rn(acc[2], __fmul_rn(wk, xv.z));
      acc[3] = __fadd_rn(acc[3], __fmul_rn(wk, xv.w));
    }
    reinterpret_cast<float4*>(out[f])[sub] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  }
}

// A fused chain of 8x8 matmul layers (pb_matmul_chain_actor), in the column
// form of bypass_region_kernel below: lane j of an 8-lane group carries column
// j of its firing through every layer in registers.  Same products and sums
// in the same order as one matmul_packed_kernel launch per layer.
constexpr int kChainMax = 8;
constexpr int kCMF = 2;   // firings per 8-lane group
__global__ void __launch_bounds__(256)
matmul_chain_kernel(pb_matmul_chain_actor a, pb_resolved res) {
  constexpr int N = 8;
  const int s = blockIdx.y, lane = threadIdx.x & 31;
  __shared__ float w[kChainMax * N * N];
  for (int e = threadIdx.x; e < a.layers * N * N; e += blockDim.x) w[e] = a.weights[e];
  __syncthreads();
  const int g = lane >> 3, j = lane & 7;
  const int j0 = (((int)blockIdx.x * 8 + (threadIdx.x >> 5)) * 4 + g) * kCMF;
  const int leader = g * 8;
  const unsigned grp = 0xFFu << leader;
  const int cnt = pb::cond_count(res, a.cond, s);
  if (j0 >= cnt) return;   // whole lane groups leave together
  const float* x[kCMF];
  float* out[kCMF];
#pragma unroll
  for (int f = 0; f < kCMF; ++f) {
    x[f] = nullptr;
    out[f] = nullptr;
    if (j == 0 && j0 + f < cnt) {
      const int n = pb::firing_iter(res, a.cond, s, j0 + f);
      x[f] = reinterpret_cast<const float*>(pb::span_ptr(a.in, res, s, n));
      out[f] = reinterpret_cast<float*>(pb::span_ptr(a.out, res, s, n));
    }
  }
#pragma unroll
  for (int f = 0; f < kCMF; ++f) {
    x[f] = reinterpret_cast<const float*>(
        __shfl_sync(grp, reinterpret_cast<unsigned long long>(x[f]), leader));
    out[f] = reinterpret_cast<float*>(
        __shfl_sync(grp, reinterpret_cast<unsigned long long>(out[f]), leader));
  }
  float c[kCMF][N];
#pragma unroll
  for (int f = 0; f < kCMF; ++f)
#pragma unroll
    for (int k = 0; k < N; ++k) c[f][k] = x[f] != nullptr ? __ldg(x[f] + k * N + j) : 0.f;
#pragma unroll
  for (int f = 0; f < kCMF; ++f) {
    if (x[f] == nullptr) continue;
    for (int l = 0; l < a.layers; ++l) {
      const float* wl = w + l * N * N;
      float y[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        float acc = 0.0f;
#pragma unroll
        for (int k = 0; k < N; ++k) acc = __fadd_rn(acc, __fmul_rn(wl[i * N + k], c[f][k]));
        y[i] = acc;
      }
#pragma unroll
      for (int i = 0; i < N; ++i) c[f][i] = y[i];
    }
#pragma unroll
    for (int k = 0; k < N; ++k) out[f][k * N + j] = c[f][k];
  }
}

// The fused bypass region (pb_bypass_region).  Column form: output column j
// of W x depends only on input column j, so lane j of an 8-lane group carries
// column j of its firing through every layer in registers (no exchange between
// lanes, ~30 registers: many firings in flight per SM, which is what a
// latency-bound per-firing kernel needs); each row load / store of the group
// is 32 contiguous bytes.  kBMF firings per group, resolved together by the
// group's first lane.  Same products and sums in the same order as MatMul.fire.
#ifndef PB_BYPASS_MF
#define PB_BYPASS_MF 2   // firings per 8-lane group (2: 5.6, 4: 5.2, 8: 4.5 G matrices/s)
#endif
constexpr int kBMF = PB_BYPASS_MF;
__global__ void __launch_bounds__(256)
bypass_region_kernel(pb_bypass_region a, pb_resolved res) {
  constexpr int N = 8;
  const int s = blockIdx.y, lane = threadIdx.x & 31;
  __shared__ float w[kChainMax * N * N];
  for (int e = threadIdx.x; e < a.layers * N * N; e += blockDim.x) w[e] = a.weights[e];
  __syncthreads();
  const int g = lane >> 3, j = lane & 7;   // group of the warp, column
  const int j0 = (((int)blockIdx.x * 8 + (threadIdx.x >> 5)) * 4 + g) * kBMF;
  const int leader = g * 8;
  const unsigned grp = 0xFFu << leader;
  const int cnt = pb::cond_count(res, a.cond, s);
  if (j0 >= cnt) return;   // whole lane groups leave together
  const float* x[kBMF];
  float* out[kBMF];
  int path[kBMF];   // 0 none, 1 chain, 2 bypass
#pragma unroll
  for (int f = 0; f < kBMF; ++f) {
    x[f] = nullptr;
    out[f] = nullptr;
    path[f] = 0;
    if (j == 0 && j0 + f < cnt) {
      const int n = pb::firing_iter(res, a.cond, s, j0 + f);
      const bool ch = pb::active(res, a.chain_live, s, n);
      const bool by = pb::active(res, a.bypass_in.act_cond, s, n);
      if (ch == by) {
        atomicExch(a.error_flag, 1);
      } else {
        path[f] = ch ? 1 : 2;
        x[f] = reinterpret_cast<const float*>(pb::span_ptr(ch ? a.chain_in : a.bypass_in, res, s, n));
        out[f] = reinterpret_cast<float*>(pb::span_ptr(a.out, res, s, n));
      }
    }
  }
#pragma unroll
  for (int f = 0; f < kBMF; ++f) {
    path[f] = __shfl_sync(grp, path[f], leader);
    x[f] = reinterpret_cast<const float*>(
        __shfl_sync(grp, reinterpret_cast<unsigned long long>(x[f]), leader));
    out[f] = reinterpret_cast<float*>(
        __shfl_sync(grp, reinterpret_cast<unsigned long long>(out[f]), leader));
  }
  float c[kBMF][N];   // column j of each firing's token
#pragma unroll
  for (int f = 0; f < kBMF; ++f)
#pragma unroll
    for (int k = 0; k < N; ++k) c[f][k] = path[f] ? __ldg(x[f] + k * N + j) : 0.f;
#pragma unroll
  for (int f = 0; f < kBMF; ++f) {
    if (path[f] == 2) {   // bypass: the token plus the marker (PathMerge.fire)
#pragma unroll
      for (int k = 0; k < N; ++k) out[f][k * N + j] = __fadd_rn(c[f][k], a.marker);
    } else if (path[f] == 1) {
      for (int l = 0; l < a.layers; ++l) {
        const float* wl = w + l * N * N;
        float y[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          float acc = 0.0f;
#pragma unroll
          for (int k = 0; k < N; ++k) acc = __fadd_rn(acc, __fmul_rn(wl[i * N + k], c[f][k]));
          y[i] = acc;
        }
#pragma unroll
        for (int i = 0; i < N; ++i) c[f][i] = y[i];
      }
#pragma unroll
      for (int k = 0; k < N; ++k) out[f][k * N + j] = c[f][k];
    }
  }
}

// Packed form for tokens of 16..512 bytes in 16-byte units (the reference's
// 256-B matrices: 16 lanes per firing, two firings per warp): the first lane
// of each firing's lane group resolves the firing (activity, live input,
// span addresses) once and broadcasts it; every lane moves one float4.
__global__ void __launch_bounds__(256)
path_merge_packed_kernel(pb_path_merge_actor a, pb_resolved res, int L) {
  const int s = blockIdx.y, lane = threadIdx.x & 31;
  const int fpw = 32 / L;                                // lane groups per warp
  const int g = lane / L, sub = lane - g * L;
  // kMF consecutive iterations per lane group, resolved together by its leader
  const int n0 = (((int)blockIdx.x * 8 + (threadIdx.x >> 5)) * fpw + g) * kMF;
  const int leader = g * L;
  const unsigned grp = (L == 32 ? 0xffffffffu : ((1u << L) - 1u) << leader);
  if (n0 >= res.n_iter) return;   // whole lane groups leave together
  int state[kMF];                 // 0: idle, 1: forward, 2: forward + marker, 3: error
  const float4* x[kMF];
  float4* out[kMF];
#pragma unroll
  for (int f = 0; f < kMF; ++f) {
    const int n = n0 + f;
    state[f] = 0;
    x[f] = nullptr;
    out[f] = nullptr;
    if (sub == 0 && n < res.n_iter && pb::active(res, a.cond, s, n)) {
      int live = -1, n_live = 0;
      for (int p = 0; p < a.n_in; ++p)
        if (pb::active(res, a.in[p].act_cond, s, n)) {
          live = p;
          ++n_live;
        }
      if (n_live != 1) {
        state[f] = 3;
      } else {
        x[f] = reinterpret_cast<const float4*>(pb::span_ptr(a.in[live], res, s, n));
        out[f] = reinterpret_cast<float4*>(pb::span_ptr(a.out, res, s, n));
        state[f] = live == a.bypass_index ? 2 : 1;
      }
    }
  }
#pragma unroll
  for (int f = 0; f < kMF; ++f) {
    state[f] = __shfl_sync(grp, state[f], leader);
    x[f] = reinterpret_cast<const float4*>(
        __shfl_sync(grp, reinterpret_cast<unsigned long long>(x[f]), leader));
    out[f] = reinterpret_cast<float4*>(
        __shfl_sync(grp, reinterpret_cast<unsigned long long>(out[f]), leader));
  }
  float4 v[kMF];
#pragma unroll
  for (int f = 0; f < kMF; ++f)
    if (state[f] == 1 || state[f] == 2) v[f] = x[f][sub];
#pragma unroll
  for (int f = 0; f < kMF; ++f) {
    if (state[f] == 3) {
      if (sub == 0) atomicExch(a.error_flag, 1);
    } else if (state[f] != 0) {
      float4 w = v[f];
      if (state[f] == 2) {
        w.x = __fadd_rn(w.x, a.marker); w.y = __fadd_rn(w.y, a.marker);
        w.z = __fadd_rn(w.z, a.marker); w.w = __fadd_rn(w.w, a.marker);
      }
      out[f][sub] = w;
    }
  }
}

}  // namespace

extern "C" {

int pb_fire_branch_sum(pb_sum_actor actor, pb_resolved res, int64_t block, void* stream) {
  if (res.n_iter == 0) return PB_OK;
  if (actor.n_in < 0 || actor.n_in > PB_MAX_PORTS)
    return pb::fail(PB_E_INVALID, "branch_sum: bad input count");
  if ((2 * block) % 4 != 0) return pb::fail(PB_E_UNSUPPORTED, "branch_sum: block must be even");
  const int64_t n4 = 2 * block / 4;
  const int tiles = (int)((n4 + kSumThreads - 1) / kSumThreads);
  dim3 grid((unsigned)(tiles * res.n_iter), res.n_streams);
  branch_sum_kernel<<<grid, kSumThreads, 0, pb::as_stream(stream)>>>(actor, res, block, tiles);
  PB_LAUNCHED("branch_sum_kernel");
  return PB_OK;
}

int pb_fire_bytes(pb_bytes_actor actor, pb_resolved res, void* stream) {
  if (res.n_iter == 0) return PB_OK;
  if (actor.n_in > PB_MAX_PORTS || actor.n_out > PB_MAX_PORTS)
    return pb::fail(PB_E_INVALID, "byte actor: too many ports");
  dim3 grid(res.n_iter, res.n_streams);
  bytes_kernel<<<grid, 128, 0, pb::as_stream(stream)>>>(actor, res);
  PB_LAUNCHED("bytes_kernel");
  return PB_OK;
}

int pb_fire_matmul(pb_matmul_actor actor, pb_resolved res, void* stream) {
  if (res.n_iter == 0) return PB_OK;
  const int NN = actor.n * actor.n;
  if (actor.n < 1 || NN > 1024) return pb::fail(PB_E_UNSUPPORTED, "matmul: N*N must be <= 1024");
  if (actor.n % 4 == 0 && NN <= 128 && 32 % (NN / 4) == 0) {
    const int L = NN / 4, per_cta = 8 * (32 / L) * kMF;
    dim3 grid((unsigned)((res.n_iter + per_cta - 1) / per_cta), res.n_streams);
    matmul_packed_kernel<<<grid, 256, 0, pb::as_stream(stream)>>>(actor, res, L);
    PB_LAUNCHED("matmul_packed_kernel");
    return PB_OK;
  }
  const int per_cta = std::max(1, 256 / NN);
  dim3 grid((unsigned)((res.n_iter + per_cta - 1) / per_cta), res.n_streams);
  matmul_kernel<<<grid, per_cta * NN, NN * sizeof(float), pb::as_stream(stream)>>>(actor, res,
                                                                                   per_cta);
  PB_LAUNCHED("matmul_kernel");
  return PB_OK;
}

int pb_fire_matmul_chain(pb_matmul_chain_actor actor, pb_resolved res, void* stream) {
  if (res.n_iter == 0) return PB_OK;
  if (actor.n != 8 || actor.layers < 1 || actor.layers > kChainMax)
    return pb::fail(PB_E_UNSUPPORTED, "matmul chain: N = 8 and 1..8 layers");
  const int per_cta = 8 * 4 * kCMF;
  dim3 grid((unsigned)((res.n_iter + per_cta - 1) / per_cta), res.n_streams);
  matmul_chain_kernel<<<grid, 256, 0, pb::as_stream(stream)>>>(actor, res);
  PB_LAUNCHED("matmul_chain_kernel");
  return PB_OK;
}

int pb_fire_bypass_region(pb_bypass_region r, pb_resolved res, void* stream) {
  if (res.n_iter == 0) return PB_OK;
  if (r.layers < 1 || r.layers > kChainMax)
    return pb::fail(PB_E_UNSUPPORTED, "bypass region: 1..8 matmul layers");
  const int per_cta = 8 * 4 * kBMF;
  dim3 grid((unsigned)((res.n_iter + per_cta - 1) / per_cta), res.n_streams);
  bypass_region_kernel<<<grid, 256, 0, pb::as_stream(stream)>>>(r, res);
  PB_LAUNCHED("bypass_region_kernel");
  return PB_OK;
}

int pb_fire_path_merge(pb_path_merge_actor actor, pb_resolved res, void* stream) {
  if (res.n_iter == 0) return PB_OK;
  if (actor.n_in > PB_MAX_PORTS) return pb::fail(PB_E_INVALID, "path_merge: too many ports");
  const int64_t sb = actor.out.span_bytes;
  if (sb % 16 == 0 && sb >= 16 && sb <= 512 && 32 % (sb / 16) == 0) {
    const int L = (int)(sb / 16), per_cta = 8 * (32 / L) * kMF;
    dim3 grid((res.n_iter + per_cta - 1) / per_cta, res.n_streams);
    path_merge_packed_kernel<<<grid, 256, 0, pb::as_stream(stream)>>>(actor, res, L);
    PB_LAUNCHED("path_merge_packed_kernel");
    return PB_OK;
  }
  dim3 grid(res.n_iter, res.n_streams);
  path_merge_kernel<<<grid, 128, 0, pb::as_stream(stream)>>>(actor, res);
  PB_LAUNCHED("path_merge_kernel");
  return PB_OK;
}

}  // extern "C"
