// Host-side helpers of the filter runtime (no device code).
//
// ssm_seedseq_state: numpy's SeedSequence hashing (bit_generator.pyx:
// hashmix / mix / generate_state, the reference RngStream's key derivation,
// rng.py:16-34) for many streams at once.  The theta-level loops of PMMH and
// SMC^2 derive a few hundred fresh child streams per step (device Philox keys,
// the first uniforms of each stream); in C this is a few microseconds instead
// of ~0.5 ms of small numpy operations per batch.  Bit-exact with numpy
// (tests/test_cpu_host.py).
#include <stdint.h>
#include <stddef.h>

#include "../../include/ssm_b200.h"

namespace {
constexpr uint32_t kInitA = 0x43B0D7E5u, kMultA = 0x931E8875u;
constexpr uint32_t kInitB = 0x8B51F9DDu, kMultB = 0x58F38DEDu;
constexpr uint32_t kMixL = 0xCA01F9DDu, kMixR = 0x4973F715u;

struct Hasher {
  uint32_t hc = kInitA;
  uint32_t operator()(uint32_t v) {
    v ^= hc;
    hc *= kMultA;
    v *= hc;
    return v ^ (v >> 16);
  }
};

inline uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = x * kMixL - y * kMixR;
  return r ^ (r >> 16);
}
}  // namespace

extern "C" int ssm_seedseq_state(int n, int L, const uint32_t* entropy, int n_words, uint32_t* out) {
  if (n < 0 || L < 0 || n_words < 0 || (n > 0 && (!entropy || !out))) return SSM_ERR_INVALID_ARG;
  for (int s = 0; s < n; ++s) {
    const uint32_t* E = entropy + static_cast<size_t>(s) * L;
    Hasher h;
    uint32_t pool[4];
    for (int i = 0; i < 4; ++i) pool[i] = h(i < L ? E[i] : 0u);
    for (int src = 0; src < 4; ++src)
      for (int dst = 0; dst < 4; ++dst)
        if (src != dst) pool[dst] = mix(pool[dst], h(pool[src]));
    for (int src = 4; src < L; ++src)
      for (int dst = 0; dst < 4; ++dst) pool[dst] = mix(pool[dst], h(E[src]));
    uint32_t hc = kInitB;
    uint32_t* o = out + static_cast<size_t>(s) * n_words;
    for (int i = 0; i < n_words; ++i) {
      uint32_t v = pool[i % 4] ^ hc;
      hc *= kMultB;
      v *= hc;
      o[i] = v ^ (v >> 16);
    }
  }
  return SSM_OK;
}
