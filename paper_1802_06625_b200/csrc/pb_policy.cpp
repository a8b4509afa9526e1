// Native host configuration actors.  The reference's policies draw from
// CPython's `random.Random` (behavior.py:202-256); this file reproduces the
// exact generator and call sequence so control tokens match bit for bit:
//   - MT19937 with init_by_array seeding from the 32-bit words of abs(seed)
//     (CPython Modules/_randommodule.c: random_seed / init_by_array)
//   - getrandbits(k) = genrand_uint32() >> (32 - k)   (k <= 32)
//   - _randbelow_with_getrandbits(n): k = n.bit_length(); rejection sampling
//   - randrange(a, b) = a + _randbelow(b - a); randint(a, b) = randrange(a, b + 1)
//   - sample(population, k): pool method when n <= setsize (21, plus
//     4**ceil(log(3k, 4)) when k > 5), set-rejection method otherwise
// Pinned by tests/test_policy_native.py against CPython itself and against
// the reference's frozen sequences (pkg/tests/test_behavior.py:320-360).
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "../../include/prune_b200.h"

namespace pb {
int fail(int code, const std::string& msg);
}

namespace {

constexpr int kN = 624;
constexpr int kM = 397;

struct PolicyState {
  uint32_t mt[kN];
  int32_t mti;
  int32_t pad_;
  int64_t firing;  // _PolicyBase.firing
};
static_assert(sizeof(PolicyState) <= PB_POLICY_STATE_BYTES, "policy state too large");

void init_genrand(PolicyState* st, uint32_t s) {
  st->mt[0] = s;
  for (int i = 1; i < kN; ++i)
    st->mt[i] = 1812433253u * (st->mt[i - 1] ^ (st->mt[i - 1] >> 30)) + (uint32_t)i;
  st->mti = kN;
}

void init_by_array(PolicyState* st, const uint32_t* key, int len) {
  init_genrand(st, 19650218u);
  int i = 1, j = 0;
  for (int k = std::max(kN, len); k; --k) {
    st->mt[i] = (st->mt[i] ^ ((st->mt[i - 1] ^ (st->mt[i - 1] >> 30)) * 1664525u)) + key[j] +
                (uint32_t)j;
    ++i;
    ++j;
    if (i >= kN) {
      st->mt[0] = st->mt[kN - 1];
      i = 1;
    }
    if (j >= len) j = 0;
  }
  for (int k = kN - 1; k; --k) {
    st->mt[i] = (st->mt[i] ^ ((st->mt[i - 1] ^ (st->mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
    ++i;
    if (i >= kN) {
      st->mt[0] = st->mt[kN - 1];
      i = 1;
    }
  }
  st->mt[0] = 0x80000000u;
}

uint32_t genrand_uint32(PolicyState* st) {
  static const uint32_t mag01[2] = {0u, 0x9908b0dfu};
  uint32_t y;
  if (st->mti >= kN) {
    int kk;
    for (kk = 0; kk < kN - kM; ++kk) {
      y = (st->mt[kk] & 0x80000000u) | (st->mt[kk + 1] & 0x7fffffffu);
      st->mt[kk] = st->mt[kk + kM] ^ (y >> 1) ^ mag01[y & 1u];
    }
    for (; kk < kN - 1; ++kk) {
      y = (st->mt[kk] & 0x80000000u) | (st->mt[kk + 1] & 0x7fffffffu);
      st->mt[kk] = st->mt[kk + (kM - kN)] ^ (y >> 1) ^ mag01[y & 1u];
    }
    y = (st->mt[kN - 1] & 0x80000000u) | (st->mt[0] & 0x7fffffffu);
    st->mt[kN - 1] = st->mt[kM - 1] ^ (y >> 1) ^ mag01[y & 1u];
    st->mti = 0;
  }
  y = st->mt[st->mti++];
  y ^= (y >> 11);
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= (y >> 18);
  return y;
}

int bit_length(uint64_t n) {
  int k = 0;
  while (n) {
    ++k;
    n >>= 1;
  }
  return k;
}

uint32_t getrandbits(PolicyState* st, int k) {
  if (k == 0) return 0;
  return genrand_uint32(st) >> (32 - k);
}

// _randbelow_with_getrandbits, n > 0
uint32_t randbelow(PolicyState* st, uint32_t n) {
  const int k = bit_length(n);
  uint32_t r = getrandbits(st, k);
  while (r >= n) r = getrandbits(st, k);
  return r;
}

// random.sample(range(1, n + 1), k) -> marks chosen elements (1-based) in v
void sample_into(PolicyState* st, int n, int k, uint8_t* v) {
  int setsize = 21;
  if (k > 5) setsize += (int)pow(4.0, ceil(log((double)k * 3) / log(4.0)));
  if (n <= setsize) {
    std::vector<int> pool(n);
    for (int i = 0; i < n; ++i) pool[i] = i + 1;
    for (int i = 0; i < k; ++i) {
      int j = (int)randbelow(st, (uint32_t)(n - i));
      v[pool[j] - 1] = 1;
      pool[j] = pool[n - i - 1];
    }
  } else {
    std::vector<uint8_t> selected(n, 0);
    for (int i = 0; i < k; ++i) {
      int j = (int)randbelow(st, (uint32_t)n);
      while (selected[j]) j = (int)randbelow(st, (uint32_t)n);
      selected[j] = 1;
      v[j] = 1;
    }
  }
}

int tokens(PolicyState* st, int kind, int length, int param, int64_t first, int64_t n_firings,
           uint8_t* out, int token_bytes) {
  if (length < 1) return pb::fail(PB_E_INVALID, "policy length must be >= 1");
  if (length > token_bytes)
    return pb::fail(PB_E_INVALID, std::to_string(length) + " control elements exceed " +
                                      std::to_string(token_bytes) + " bytes");
  for (int64_t f = 0; f < n_firings; ++f) {
    uint8_t* v = out + f * token_bytes;
    memset(v, 0, (size_t)token_bytes);
    const int64_t firing = first + f;
    switch (kind) {
      case 0: {  // FixedPolicy, behavior.py:221-227
        if (param >= 1 && param <= length) v[param - 1] = 1;
        break;
      }
      case 1: {  // AlternatePolicy, behavior.py:230-236
        v[firing % length] = 1;
        break;
      }
      case 2: {  // SeededPolicy, behavior.py:239-245: randrange(1, length + 1)
        v[randbelow(st, (uint32_t)length)] = 1;
        break;
      }
      case 3: {  // SubsetPolicy, behavior.py:248-256
        const int lo = std::min(param, length);
        if (lo > length || length - lo + 1 <= 0)
          return pb::fail(PB_E_INVALID, "subset_policy: empty randint range");
        const int size = lo + (int)randbelow(st, (uint32_t)(length - lo + 1));
        if (size < 0) return pb::fail(PB_E_INVALID, "Sample larger than population or is negative");
        sample_into(st, length, size, v);
        break;
      }
      default:
        return pb::fail(PB_E_INVALID, "unknown policy kind " + std::to_string(kind));
    }
  }
  st->firing = first + n_firings;
  return PB_OK;
}

}  // namespace

extern "C" {

int pb_policy_init(void* state, int64_t seed) {
  if (!state) return pb::fail(PB_E_INVALID, "pb_policy_init: null state");
  PolicyState* st = static_cast<PolicyState*>(state);
  memset(st, 0, sizeof(PolicyState));
  uint64_t n = seed < 0 ? 0 : (uint64_t)seed;  // seed None -> Random(0), behavior.py:207
  uint32_t key[2] = {(uint32_t)(n & 0xffffffffu), (uint32_t)(n >> 32)};
  int used = (n >> 32) ? 2 : 1;
  init_by_array(st, key, used);
  st->firing = 0;
  return PB_OK;
}

int pb_policy_tokens(void* state, int kind, int length, int param, int64_t first,
                     int64_t n_firings, uint8_t* out, int token_bytes) {
  if (!state || (!out && n_firings > 0)) return pb::fail(PB_E_INVALID, "pb_policy_tokens: null argument");
  return tokens(static_cast<PolicyState*>(state), kind, length, param, first, n_firings, out,
                token_bytes);
}

int pb_policy_tokens_streams(void* states, int n_streams, int kind, int length, int param,
                             int64_t first, int64_t n_firings, uint8_t* out, int token_bytes,
                             int threads) {
  if (!states || (!out && n_firings > 0)) return pb::fail(PB_E_INVALID, "pb_policy_tokens_streams: null argument");
  if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  threads = std::min(threads, n_streams);
  // thread start-up costs ~10-20 us each: small batches run inline (the
  // pipelined runtime calls this per sub-epoch while its hashers hold the cores)
  if ((int64_t)n_streams * n_firings < 65536) threads = 1;
  std::vector<int> rcs(n_streams, PB_OK);
  auto work = [&](int t) {
    for (int s = t; s < n_streams; s += threads) {
      PolicyState* st = reinterpret_cast<PolicyState*>(static_cast<uint8_t*>(states) +
                                                       (int64_t)s * PB_POLICY_STATE_BYTES);
      rcs[s] = tokens(st, kind, length, param, first, n_firings,
                      out + (int64_t)s * n_firings * token_bytes, token_bytes);
    }
  };
  if (threads <= 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  for (int s = 0; s < n_streams; ++s)
    if (rcs[s] != PB_OK) return rcs[s];
  return PB_OK;
}

uint32_t pb_crc32(const uint8_t* data, size_t n) {
  static uint32_t table[256];
  static bool ready = false;
  if (!ready) {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      table[i] = c;
    }
    ready = true;
  }
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < n; ++i) c = table[(c ^ data[i]) & 0xFFu] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

}  // extern "C"
