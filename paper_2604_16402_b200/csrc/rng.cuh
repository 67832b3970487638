// Device restatement of the numpy 2.3.5 random primitives used by the reference
// search seeding (reference searcher.py:85-87, 128, 181):
//   SeedSequence hash mixing -> PCG64 (XSL-RR 128/64) -> buffered 32-bit output
//   -> Lemire nearly-divisionless bounded draws.
// Draws are produced warp-parallel with 128-bit LCG jump-ahead, so a query's
// 4*want seed draws cost one round of 32 lanes instead of a serial chain.
// CPU twin: oracle/rng.py (pinned against numpy in tests/test_oracle_golden.py).
#pragma once
#include <stdint.h>

namespace grab {

typedef unsigned __int128 u128;

__host__ __device__ constexpr u128 pcg_mult() {
  return ((u128)2549297995355413924ull << 64) + (u128)4865540595714422341ull;
}

// Jump tables: kJumpA[j] = MULT^j, kJumpG[j] = sum_{i<j} MULT^i (mod 2^128), j=0..32.
struct PcgJump {
  uint64_t a_lo[33], a_hi[33], g_lo[33], g_hi[33];
};
void upload_pcg_jump_tables();  // host: fill the jump tables (search.cu) once per device

struct SeedSeq {
  uint32_t pool[4];
};

__host__ __device__ inline uint32_t ss_hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= 0x931E8875u;
  v *= hc;
  return v ^ (v >> 16);
}

__host__ __device__ inline uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xCA01F9DDu * x - 0x4973F715u * y;
  return r ^ (r >> 16);
}

// entropy = little-endian 32-bit words of each integer (0 -> one word 0).
__host__ __device__ inline SeedSeq seedseq_from_u64s(const uint64_t* vals, int nvals) {
  uint32_t w[8];
  int nw = 0;
  for (int i = 0; i < nvals; ++i) {
    uint64_t v = vals[i];
    w[nw++] = (uint32_t)v;
    if (v >> 32) w[nw++] = (uint32_t)(v >> 32);
  }
  SeedSeq s;
  uint32_t hc = 0x43B0D7E5u;
  for (int i = 0; i < 4; ++i) s.pool[i] = ss_hashmix(i < nw ? w[i] : 0u, hc);
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b)
      if (a != b) s.pool[b] = ss_mix(s.pool[b], ss_hashmix(s.pool[a], hc));
  for (int a = 4; a < nw; ++a)
    for (int b = 0; b < 4; ++b) s.pool[b] = ss_mix(s.pool[b], ss_hashmix(w[a], hc));
  return s;
}

// generate_state(n64, uint64)
__host__ __device__ inline void seedseq_u64(const SeedSeq& s, uint64_t* out, int n64) {
  uint32_t hc = 0x8B51F9DDu;
  for (int i = 0; i < 2 * n64; ++i) {
    uint32_t v = s.pool[i & 3] ^ hc;
    hc *= 0x58F38DEDu;
    v *= hc;
    v ^= v >> 16;
    if (i & 1)
      out[i >> 1] |= (uint64_t)v << 32;
    else
      out[i >> 1] = v;
  }
}

// derive_query_seed(base, ordinal) (searcher.py:85-87)
__host__ __device__ inline uint64_t derive_query_seed(uint64_t base, uint64_t ordinal) {
  uint64_t e[2] = {base, ordinal};
  SeedSeq s = seedseq_from_u64s(e, 2);
  uint64_t r;
  seedseq_u64(s, &r, 1);
  return r;
}

struct Pcg64 {
  u128 state;  // state before the first output
  u128 inc;
};

// default_rng(seed) -> PCG64(SeedSequence(seed))
__host__ __device__ inline Pcg64 pcg64_from_seed(uint64_t seed) {
  SeedSeq s = seedseq_from_u64s(&seed, 1);
  uint64_t v[4];
  seedseq_u64(s, v, 4);
  u128 initstate = ((u128)v[0] << 64) | v[1];
  u128 initseq = ((u128)v[2] << 64) | v[3];
  Pcg64 g;
  g.inc = (initseq << 1) | 1;
  g.state = g.inc;  // 0 * mult + inc
  g.state += initstate;
  g.state = g.state * pcg_mult() + g.inc;
  return g;
}

__host__ __device__ inline uint64_t pcg_xsl_rr(u128 s) {
  uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  unsigned r = (unsigned)(s >> 122);
  return (x >> r) | (x << ((64 - r) & 63));
}


}  // namespace grab
