// Epoch resolution on the device: control tokens -> per-iteration activity of
// every (control port, element) condition, compacted firing lists, the Eq. 1
// recheck and bulk ring-counter advance.  This replaces the per-firing host
// work of runtime.py:126-163 (control read, decode, _rates) and the Eq. 1
// recheck runtime.py:195-220 with a handful of batched launches per epoch.
#include <algorithm>

#include "pb_common.cuh"

namespace {

constexpr int kMaxConds = 64;
constexpr int kMaxEq1 = 256;
constexpr int kMaxRings = 256;

struct CondTable {
  pb_condition c[kMaxConds];
};
struct Eq1Table {
  pb_eq1_port p[kMaxEq1];
};
struct RingTable {
  pb_ring_advance_t r[kMaxRings];
};

constexpr int kScanThreads = 256;
constexpr int kScanItems = 4;  // iterations per thread per tile

// One CTA per (stream, condition): decode_control (behavior.py:34-38) of the
// condition's element for every iteration, exclusive scan, compaction.
__global__ void __launch_bounds__(kScanThreads) resolve_kernel(CondTable table, int cond0,
                                                               pb_resolved res) {
  pb::pdl_enter();
  const int s = blockIdx.x;
  const int c = cond0 + blockIdx.y;
  const pb_condition& cd = table.c[blockIdx.y];
  const int64_t row = ((int64_t)c * res.n_streams + s) * res.cap;
  const uint8_t* tok = cd.tokens + (int64_t)s * cd.stream_stride;
  __shared__ int warp_sums[kScanThreads / 32];
  __shared__ int carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t0 = 0; t0 < res.n_iter; t0 += kScanThreads * kScanItems) {
    int flags[kScanItems];
    int local = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      int n = t0 + threadIdx.x * kScanItems + k;
      int f = 0;
      if (n < res.n_iter) {
        const int64_t chunk = (uint32_t)(cd.base + n) % (uint32_t)cd.slots;   // base, n >= 0, int32
        f = tok[chunk * cd.token_stride + cd.element] != 0;
      }
      flags[k] = f;
      local += f;
    }
    // block exclusive scan of `local`
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    int warp_off = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w) {
      int v = warp_sums[w];
      if (w < warp) warp_off += v;
      total += v;
    }
    const int carry = carry_s;
    int run = carry + warp_off + incl - local;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      int n = t0 + threadIdx.x * kScanItems + k;
      if (n < res.n_iter) {
        res.act[row + n] = (uint8_t)flags[k];
        res.prefix[row + n] = run;
        if (flags[k]) res.worklist[row + run] = n;
        run += flags[k];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + total;
    __syncthreads();
  }
  if (threadIdx.x == 0) res.count[(int64_t)c * res.n_streams + s] = carry_s;
}

// Eq. 1 recheck: one CTA per (stream, DRP).
__global__ void eq1_kernel(Eq1Table table, int n_ports, pb_resolved res, int64_t* counters) {
  pb::pdl_enter();
  const int s = blockIdx.x;
  const pb_eq1_port& p = table.p[blockIdx.y];
  int checks = 0, failures = 0;
  for (int n = threadIdx.x; n < res.n_iter; n += blockDim.x) {
    if (!pb::active(res, p.actor_cond, s, n)) continue;
    ++checks;
    bool expected = pb::active(res, p.own_cond, s, n);
    bool moved = pb::active(res, p.moved_cond, s, n);
    failures += expected != moved;
  }
  for (int o = 16; o > 0; o >>= 1) {
    checks += __shfl_down_sync(0xffffffffu, checks, o);
    failures += __shfl_down_sync(0xffffffffu, failures, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (checks) atomicAdd((unsigned long long*)&counters[0], (unsigned long long)checks);
    if (failures) atomicAdd((unsigned long long*)&counters[1], (unsigned long long)failures);
  }
}

// write_end/read_end in bulk for every ring of the epoch (fifos.py:247-269,
// 310-323): producer kernels publish all their spans before the consumer
// kernels run, so the epoch's peak occupancy is delay + rate*(w + cnt - r).
__global__ void advance_kernel(RingTable table, int n_rings, pb_resolved res) {
  pb::pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rings * res.n_streams) return;
  const int r = i / res.n_streams, s = i % res.n_streams;
  const pb_ring_advance_t& ra = table.r[r];
  int64_t* w = ra.counters + s;
  int64_t* rd = ra.counters + res.n_streams + s;
  int64_t* mx = ra.counters + 2 * (int64_t)res.n_streams + s;
  int64_t cnt = pb::cond_count(res, ra.cond, s);
  int64_t occ = ra.delay + (int64_t)ra.rate * (*w + cnt - *rd);
  if (occ > *mx) *mx = occ;
  *w += cnt;
  *rd += cnt;
}

// Eq. 1 recheck and ring advance of one epoch in one launch: blocks
// [0, S * n_ports) are eq1_kernel's (stream, port) blocks, the rest
// advance_kernel's.  The two touch disjoint data (Eq. 1 reads the resolution
// and adds to its counters; the advance updates ring counters), so the
// launch is one kernel's latency instead of two.
__global__ void __launch_bounds__(128)
epoch_close_kernel(Eq1Table eq, int n_ports, int64_t* counters, RingTable rings, int n_rings,
                   pb_resolved res) {
  pb::pdl_enter();
  const int n_eq1_blocks = res.n_streams * n_ports;
  if ((int)blockIdx.x < n_eq1_blocks) {
    const int s = blockIdx.x % res.n_streams;
    const pb_eq1_port& p = eq.p[blockIdx.x / res.n_streams];
    int checks = 0, failures = 0;
    for (int n = threadIdx.x; n < res.n_iter; n += blockDim.x) {
      if (!pb::active(res, p.actor_cond, s, n)) continue;
      ++checks;
      failures += pb::active(res, p.own_cond, s, n) != pb::active(res, p.moved_cond, s, n);
    }
    for (int o = 16; o > 0; o >>= 1) {
      checks += __shfl_down_sync(0xffffffffu, checks, o);
      failures += __shfl_down_sync(0xffffffffu, failures, o);
    }
    if ((threadIdx.x & 31) == 0) {
      if (checks) atomicAdd((unsigned long long*)&counters[0], (unsigned long long)checks);
      if (failures) atomicAdd((unsigned long long*)&counters[1], (unsigned long long)failures);
    }
    return;
  }
  const int i = ((int)blockIdx.x - n_eq1_blocks) * blockDim.x + threadIdx.x;
  if (i >= n_rings * res.n_streams) return;
  const int r = i / res.n_streams, s = i % res.n_streams;
  const pb_ring_advance_t& ra = rings.r[r];
  int64_t* w = ra.counters + s;
  int64_t* rd = ra.counters + res.n_streams + s;
  int64_t* mx = ra.counters + 2 * (int64_t)res.n_streams + s;
  const int64_t cnt = pb::cond_count(res, ra.cond, s);
  const int64_t occ = ra.delay + (int64_t)ra.rate * (*w + cnt - *rd);
  if (occ > *mx) *mx = occ;
  *w += cnt;
  *rd += cnt;
}

}  // namespace

extern "C" {

int pb_epoch_close(const pb_eq1_port* ports, int n_ports, int64_t* counters,
                   const pb_ring_advance_t* rings, int n_rings, pb_resolved res, void* stream) {
  if (n_ports < 0 || n_ports > kMaxEq1 || n_rings < 0 || n_rings > kMaxRings)
    return pb::fail(PB_E_UNSUPPORTED, "pb_epoch_close: at most " + std::to_string(kMaxEq1) +
                                          " ports and " + std::to_string(kMaxRings) + " rings");
  if (res.n_iter == 0) n_ports = 0;
  if (n_ports == 0 && n_rings == 0) return PB_OK;
  Eq1Table e{};
  for (int k = 0; k < n_ports; ++k) e.p[k] = ports[k];
  RingTable t{};
  for (int k = 0; k < n_rings; ++k) t.r[k] = rings[k];
  const int blocks = res.n_streams * n_ports + (n_rings * res.n_streams + 127) / 128;
  PB_LAUNCH_PDL(epoch_close_kernel, blocks, 128, 0, pb::as_stream(stream), e, n_ports, counters,
                t, n_rings, res);
  PB_LAUNCHED("epoch_close_kernel");
  return PB_OK;
}


int pb_resolve(const pb_condition* conds, pb_resolved res, void* stream) {
  if (res.n_cond == 0 || res.n_iter == 0) return PB_OK;
  if (!conds) return pb::fail(PB_E_INVALID, "pb_resolve: null conditions");
  if (res.n_iter > res.cap) return pb::fail(PB_E_INVALID, "pb_resolve: n_iter exceeds cap");
  for (int c0 = 0; c0 < res.n_cond; c0 += kMaxConds) {
    int nc = std::min(kMaxConds, res.n_cond - c0);
    CondTable t{};
    for (int k = 0; k < nc; ++k) {
      t.c[k] = conds[c0 + k];
      if (t.c[k].slots <= 0 || t.c[k].element < 0 || t.c[k].element >= t.c[k].token_stride)
        return pb::fail(PB_E_INVALID, "pb_resolve: bad condition " + std::to_string(c0 + k));
    }
    dim3 grid(res.n_streams, nc);
    PB_LAUNCH_PDL(resolve_kernel, grid, kScanThreads, 0, pb::as_stream(stream), t, c0, res);
    PB_LAUNCHED("resolve_kernel");
  }
  return PB_OK;
}

int pb_eq1_check(const pb_eq1_port* ports, int n_ports, pb_resolved res, int64_t* counters,
                 void* stream) {
  if (n_ports == 0 || res.n_iter == 0) return PB_OK;
  for (int p0 = 0; p0 < n_ports; p0 += kMaxEq1) {
    int np = std::min(kMaxEq1, n_ports - p0);
    Eq1Table t{};
    for (int k = 0; k < np; ++k) t.p[k] = ports[p0 + k];
    dim3 grid(res.n_streams, np);
    PB_LAUNCH_PDL(eq1_kernel, grid, 128, 0, pb::as_stream(stream), t, np, res, counters);
    PB_LAUNCHED("eq1_kernel");
  }
  return PB_OK;
}

int pb_rings_advance(const pb_ring_advance_t* rings, int n_rings, pb_resolved res,
                     void* stream) {
  if (n_rings == 0) return PB_OK;
  for (int r0 = 0; r0 < n_rings; r0 += kMaxRings) {
    int nr = std::min(kMaxRings, n_rings - r0);
    RingTable t{};
    for (int k = 0; k < nr; ++k) t.r[k] = rings[r0 + k];
    int total = nr * res.n_streams;
    PB_LAUNCH_PDL(advance_kernel, (total + 127) / 128, 128, 0, pb::as_stream(stream), t, nr, res);
    PB_LAUNCHED("advance_kernel");
  }
  return PB_OK;
}

}  // extern "C"
