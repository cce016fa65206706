// host_api.cpp -- host-only part of the C ABI: error strings, launch counter,
// numpy SeedSequence / PCG64 seeding (sketch.py:51-53), jump-ahead.
//
// SeedSequence restates numpy.random.bit_generator.SeedSequence (numpy 2.3.5):
// a 4-word uint32 entropy pool mixed with hashmix/mix, then generate_state.
// PCG64 seeding restates numpy's pcg64_set_seed -> pcg_setseq_128_srandom_r.
#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"

namespace skt {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

std::atomic<uint64_t> &launch_counter() {
  static std::atomic<uint64_t> c{0};
  return c;
}

}  // namespace skt

using namespace skt;

namespace {

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr int kPool = 4;

struct HashConst {
  uint32_t v;
  uint32_t operator()(uint32_t x) {  // hashmix, advancing the hash constant
    x ^= v;
    v *= kMultA;
    x *= v;
    return x ^ (x >> 16);
  }
};

inline uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  return r ^ (r >> 16);
}

}  // namespace

extern "C" {

const char *skt_version(void) { return "sketch_b200 abi 1 (sm_100a)"; }

const char *skt_last_error(void) { return g_last_error.c_str(); }

uint64_t skt_launch_count(void) { return launch_counter().load(); }

skt_status skt_seedseq_generate(const uint32_t *entropy, int32_t n_entropy,
                                const uint32_t *spawn_key, int32_t n_spawn, uint32_t *out,
                                int32_t n_out) {
  static const char *fn = "skt_seedseq_generate";
  if (n_entropy < 0 || n_spawn < 0 || n_out < 0 || (n_entropy && !entropy) ||
      (n_spawn && !spawn_key) || (n_out && !out))
    return fail(SKT_EINVAL, fn, "bad arguments");
  // assembled entropy: run entropy, zero-padded to the pool size when a spawn
  // key follows, then the spawn key words.
  const int total = (n_spawn > 0 && n_entropy < kPool ? kPool : n_entropy) + n_spawn;
  uint32_t stackbuf[64];
  uint32_t *asm_ = total <= 64 ? stackbuf : new uint32_t[total];
  int k = 0;
  for (int i = 0; i < n_entropy; ++i) asm_[k++] = entropy[i];
  if (n_spawn > 0)
    while (k < kPool) asm_[k++] = 0u;
  for (int i = 0; i < n_spawn; ++i) asm_[k++] = spawn_key[i];

  uint32_t pool[kPool];
  HashConst hc{kInitA};
  for (int i = 0; i < kPool; ++i) pool[i] = hc(i < k ? asm_[i] : 0u);
  for (int s = 0; s < kPool; ++s)
    for (int d = 0; d < kPool; ++d)
      if (s != d) pool[d] = mix(pool[d], hc(pool[s]));
  for (int s = kPool; s < k; ++s)
    for (int d = 0; d < kPool; ++d) pool[d] = mix(pool[d], hc(asm_[s]));
  if (asm_ != stackbuf) delete[] asm_;

  uint32_t hb = kInitB;
  for (int i = 0; i < n_out; ++i) {
    uint32_t v = pool[i % kPool];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    out[i] = v ^ (v >> 16);
  }
  return SKT_OK;
}

skt_status skt_pcg64_seed(const uint32_t *entropy, int32_t n_entropy, const uint32_t *spawn_key,
                          int32_t n_spawn, skt_pcg64 *out) {
  if (!out) return fail(SKT_EINVAL, "skt_pcg64_seed", "out is NULL");
  uint32_t w[8];
  skt_status st = skt_seedseq_generate(entropy, n_entropy, spawn_key, n_spawn, w, 8);
  if (st != SKT_OK) return st;
  uint64_t v[4];
  for (int i = 0; i < 4; ++i) v[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  const u128 initstate = mk128(v[0], v[1]);
  const u128 inc = (mk128(v[2], v[3]) << 1) | 1u;
  u128 s = 0;
  s = s * pcg_mult() + inc;
  s += initstate;
  s = s * pcg_mult() + inc;
  out->state_hi = (uint64_t)(s >> 64);
  out->state_lo = (uint64_t)s;
  out->inc_hi = (uint64_t)(inc >> 64);
  out->inc_lo = (uint64_t)inc;
  return SKT_OK;
}

skt_status skt_pcg64_advance(skt_pcg64 *st, uint64_t delta) {
  if (!st) return fail(SKT_EINVAL, "skt_pcg64_advance", "state is NULL");
  const u128 inc = mk128(st->inc_hi, st->inc_lo);
  const Affine128 a = lcg_power(delta, inc);
  const u128 s = a.mult * mk128(st->state_hi, st->state_lo) + a.plus;
  st->state_hi = (uint64_t)(s >> 64);
  st->state_lo = (uint64_t)s;
  return SKT_OK;
}

}  // extern "C"
