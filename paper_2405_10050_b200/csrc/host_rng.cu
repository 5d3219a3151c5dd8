// Host-side descent streams, vectorised over starts (host code only).
//
// The reference draws every descent direction from its own stream
// numpy.random.Generator(PCG64(SeedSequence(entropy=seed,
// spawn_key=(tag, index)))) (pkg/src/voronray/rng.py:18-28, graph.py:46-85).
// Building 10,000 such Generator objects costs ~20 us each in Python (0.2 s
// of config 5's 1.1 s).  This file restates the published SeedSequence
// hashing (NumPy's bit_generator, after O'Neill's seed_seq design) and the
// PCG64 (XSL-RR 128/64) stepping over arrays of streams, and draws the
// normals with NumPy's own ziggurat sampler (random_standard_normal from
// NumPy's static libnpyrandom, linked in), so every value is bit-identical
// to the Generator's (tests/test_host.py checks it against numpy).
#include <thread>
#include <vector>
#include <cstdint>
#include <cstring>

#include "common.cuh"

extern "C" {
typedef struct bitgen {
  void* state;
  uint64_t (*next_uint64)(void* st);
  uint32_t (*next_uint32)(void* st);
  double (*next_double)(void* st);
  uint64_t (*next_raw)(void* st);
} bitgen_t;
double random_standard_normal(bitgen_t* bitgen_state);  // libnpyrandom
}

namespace {

// ---- SeedSequence (pool size 4, 32-bit words) ------------------------------
constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
constexpr uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
constexpr uint32_t MIX_MULT_L = 0xca01f9ddu, MIX_MULT_R = 0x4973f715u;
constexpr int XSHIFT = 16;
constexpr int POOL = 4;

inline uint32_t hashmix(uint32_t value, uint32_t& hc) {
  value ^= hc;
  hc *= MULT_A;
  value *= hc;
  value ^= value >> XSHIFT;
  return value;
}

inline uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = MIX_MULT_L * x - MIX_MULT_R * y;
  r ^= r >> XSHIFT;
  return r;
}

// little-endian 32-bit words of a non-negative integer (0 -> one word 0)
inline int int_words(uint64_t v, uint32_t* out) {
  int n = 0;
  do {
    out[n++] = (uint32_t)v;
    v >>= 32;
  } while (v);
  return n;
}

// entropy = seed, spawn_key = (tag, index): the assembled entropy is the run
// entropy zero-padded to the pool size, then the spawn-key words.
void seed_sequence_state(uint64_t seed, uint64_t tag, uint64_t index, uint64_t (&st)[4]) {
  uint32_t ent[16];
  int n = int_words(seed, ent);
  while (n < POOL) ent[n++] = 0u;
  n += int_words(tag, ent + n);
  n += int_words(index, ent + n);
  uint32_t pool[POOL];
  uint32_t hc = INIT_A;
  for (int i = 0; i < POOL; ++i) pool[i] = hashmix(i < n ? ent[i] : 0u, hc);
  for (int s = 0; s < POOL; ++s)
    for (int d = 0; d < POOL; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
  for (int s = POOL; s < n; ++s)
    for (int d = 0; d < POOL; ++d) pool[d] = mix(pool[d], hashmix(ent[s], hc));
  // generate_state(4, uint64): 8 words cycling the pool, then pairs of
  // little-endian words form the 64-bit values
  uint32_t w[8];
  uint32_t hb = INIT_B;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % POOL];
    v ^= hb;
    hb *= MULT_B;
    v *= hb;
    v ^= v >> XSHIFT;
    w[i] = v;
  }
  for (int i = 0; i < 4; ++i) st[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
}

// ---- PCG64: 128-bit LCG, XSL-RR output --------------------------------------
typedef unsigned __int128 u128;
constexpr u128 PCG_MULT = ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;

struct Pcg {
  u128 state, inc;
};

inline uint64_t pcg_next64(void* p) {
  Pcg* g = static_cast<Pcg*>(p);
  g->state = g->state * PCG_MULT + g->inc;
  const uint64_t hi = (uint64_t)(g->state >> 64), lo = (uint64_t)g->state;
  const unsigned rot = (unsigned)(g->state >> 122);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64 - rot) & 63));
}
inline uint32_t pcg_next32(void* p) { return (uint32_t)pcg_next64(p); }  // unused by normals
inline double pcg_next_double(void* p) {
  return (double)(pcg_next64(p) >> 11) * (1.0 / 9007199254740992.0);
}

// PCG64(SeedSequence): seed words s[0..1] (high, low) -> initstate,
// s[2..3] -> initseq; srandom: state = 0, inc = 2 initseq + 1, step,
// state += initstate, step.
void pcg_seed(Pcg& g, const uint64_t (&s)[4]) {
  const u128 initstate = ((u128)s[0] << 64) | s[1];
  const u128 initseq = ((u128)s[2] << 64) | s[3];
  g.state = 0;
  g.inc = (initseq << 1) | 1u;
  g.state = g.state * PCG_MULT + g.inc;
  g.state += initstate;
  g.state = g.state * PCG_MULT + g.inc;
}

inline void pack(const Pcg& g, uint64_t* out) {
  out[0] = (uint64_t)(g.state >> 64);
  out[1] = (uint64_t)g.state;
  out[2] = (uint64_t)(g.inc >> 64);
  out[3] = (uint64_t)g.inc;
}
inline Pcg unpack(const uint64_t* in) {
  Pcg g;
  g.state = ((u128)in[0] << 64) | in[1];
  g.inc = ((u128)in[2] << 64) | in[3];
  return g;
}

}  // namespace

// Streams stream(seed, purpose tag, index[i]) for i < n: 4 uint64 per stream
// (PCG64 state high, low, increment high, low) in `state`.
extern "C" int vr_host_streams(uint64_t seed, uint64_t tag, const int64_t* index, int64_t n,
                               uint64_t* state) {
  if (n < 0 || (n > 0 && (!index || !state))) return VR_EINVAL;
  for (int64_t i = 0; i < n; ++i) {
    if (index[i] < 0) return VR_EINVAL;
    uint64_t s[4];
    seed_sequence_state(seed, tag, (uint64_t)index[i], s);
    Pcg g;
    pcg_seed(g, s);
    pack(g, state + 4 * i);
  }
  return VR_OK;
}

// For each listed stream (rows[i], or i when rows == NULL), `count` standard
// normals in Generator.standard_normal order into out[i * count ..]; the
// stream states advance in place.
// Streams are independent, so large batches split over host threads (config
// 5's 10,000 descent streams x 88 normals: ~8 ms on one core).  Each stream
// is drawn by exactly one thread, in its own order: bitwise the serial draw.
extern "C" int vr_host_normals(uint64_t* state, const int64_t* rows, int64_t n, int64_t count,
                               double* out) {
  if (n < 0 || count < 0 || (n > 0 && (!state || !out))) return VR_EINVAL;
  auto work = [=](int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {
      uint64_t* st = state + 4 * (rows ? rows[i] : i);
      Pcg g = unpack(st);
      bitgen_t bg{&g, pcg_next64, pcg_next32, pcg_next_double, pcg_next64};
      double* o = out + i * count;
      for (int64_t k = 0; k < count; ++k) o[k] = random_standard_normal(&bg);
      pack(g, st);
    }
  };
  const int64_t total = n * count;
  unsigned hw = std::thread::hardware_concurrency();
  int64_t nt = total >= (1 << 16) ? (int64_t)(hw ? hw : 1) : 1;
  if (nt > 16) nt = 16;
  if (nt > n) nt = n;
  if (nt <= 1) {
    work(0, n);
    return VR_OK;
  }
  std::vector<std::thread> th;
  th.reserve((size_t)nt - 1);
  for (int64_t t = 1; t < nt; ++t) th.emplace_back(work, n * t / nt, n * (t + 1) / nt);
  work(0, n / nt);
  for (auto& x : th) x.join();
  return VR_OK;
}
