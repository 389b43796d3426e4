// pyrandom.hpp — a Mersenne Twister whose draws match CPython's `random.Random`.
//
// The reference generators (pkg/src/mlq_sssp/graph.py:306-420) consume
// `random.Random(seed)`.  Reproducing their graphs byte-for-byte needs
// CPython's seeding (init_by_array over the 32-bit limbs of |seed|), the standard
// MT19937 recurrence/tempering, and CPython's derived draws:
//   random()          = ((a >> 5) * 2^26 + (b >> 6)) / 2^53
//   getrandbits(k<=32)= genrand() >> (32 - k)
//   _randbelow(n)     = rejection over getrandbits(n.bit_length())
//   randint(a, b)     = a + _randbelow(b - a + 1)
// MT19937 itself is the public algorithm of Matsumoto & Nishimura (1998).
#pragma once
#include <cstdint>
#include <cstddef>

namespace mlmq {

class PyRandom {
 public:
  static constexpr int N = 624;
  static constexpr int M = 397;

  PyRandom(const uint32_t* key, size_t keylen) { seed_by_array(key, keylen); }

  // Tempered outputs are produced a whole state (624 draws) at a time: the twist and
  // the tempering then run as straight loops the compiler vectorises.
  uint32_t genrand() {
    if (mti_ >= N) refill();
    return out_[mti_++];
  }

  double random() {
    uint32_t a = genrand() >> 5, b = genrand() >> 6;
    return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
  }

  // random() as its exact 53-bit integer numerator R (random() == R / 2^53), so
  // `random() >= t` <=> `random53() >= ceil53(t)` with no floating point on the hot path.
  uint64_t random53() {
    const uint64_t a = genrand() >> 5, b = genrand() >> 6;
    return (a << 26) | b;
  }
  static uint64_t ceil53(double t) {
    const double x = t * 9007199254740992.0;  // exact: power-of-two scaling
    if (!(x > 0.0)) return 0;
    if (x >= 9007199254740992.0) return 1ull << 53;
    uint64_t c = (uint64_t)x;
    if ((double)c < x) ++c;
    return c;
  }

  uint32_t getrandbits(int k) {  // 0 < k <= 32
    return genrand() >> (32 - k);
  }

  // uniform in [0, n), n in [1, 2^32]
  uint64_t randbelow(uint64_t n) {
    int k = 0;
    for (uint64_t t = n; t; t >>= 1) ++k;  // n.bit_length()
    if (k > 32) {  // only n == 2^32 reaches here (bit_length 33)
      // CPython getrandbits(33) = low word then high word (little-endian limbs)
      for (;;) {
        uint64_t lo = genrand();
        uint64_t hi = genrand() >> (64 - 33);
        uint64_t r = lo | (hi << 32);
        if (r < n) return r;
      }
    }
    uint64_t r = getrandbits(k);
    while (r >= n) r = getrandbits(k);
    return r;
  }

  int64_t randint(int64_t a, int64_t b) { return a + (int64_t)randbelow((uint64_t)(b - a + 1)); }

 private:
  void init_genrand(uint32_t s) {
    mt_[0] = s;
    for (int i = 1; i < N; ++i)
      mt_[i] = 1812433253U * (mt_[i - 1] ^ (mt_[i - 1] >> 30)) + (uint32_t)i;
    mti_ = N;
  }

  void seed_by_array(const uint32_t* key, size_t keylen) {
    init_genrand(19650218U);
    int i = 1;
    size_t j = 0;
    size_t k = (size_t)N > keylen ? (size_t)N : keylen;
    for (; k; --k) {
      mt_[i] = (mt_[i] ^ ((mt_[i - 1] ^ (mt_[i - 1] >> 30)) * 1664525U)) + key[j] + (uint32_t)j;
      ++i;
      ++j;
      if (i >= N) { mt_[0] = mt_[N - 1]; i = 1; }
      if (j >= keylen) j = 0;
    }
    for (k = N - 1; k; --k) {
      mt_[i] = (mt_[i] ^ ((mt_[i - 1] ^ (mt_[i - 1] >> 30)) * 1566083941U)) - (uint32_t)i;
      ++i;
      if (i >= N) { mt_[0] = mt_[N - 1]; i = 1; }
    }
    mt_[0] = 0x80000000U;
  }

  static uint32_t mix(uint32_t a, uint32_t b, uint32_t m) {
    const uint32_t y = (a & 0x80000000U) | (b & 0x7fffffffU);
    return m ^ (y >> 1) ^ ((0U - (y & 1U)) & 0x9908b0dfU);
  }
  void refill() {
    int kk = 0;
    for (; kk < N - M; ++kk) mt_[kk] = mix(mt_[kk], mt_[kk + 1], mt_[kk + M]);
    for (; kk < N - 1; ++kk) mt_[kk] = mix(mt_[kk], mt_[kk + 1], mt_[kk + (M - N)]);
    mt_[N - 1] = mix(mt_[N - 1], mt_[0], mt_[M - 1]);
    for (int i = 0; i < N; ++i) {
      uint32_t y = mt_[i];
      y ^= (y >> 11);
      y ^= (y << 7) & 0x9d2c5680U;
      y ^= (y << 15) & 0xefc60000U;
      y ^= (y >> 18);
      out_[i] = y;
    }
    mti_ = 0;
  }

  uint32_t mt_[N];
  uint32_t out_[N];
  int mti_ = N + 1;
};

}  // namespace mlmq
