// Shared helpers for the GRAB B200 kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdexcept>
#include <string>

#include "../../include/grab.h"

namespace grab {

constexpr uint32_t kSentinel = 0xFFFFFFFFu;  // reference layout.py:19
constexpr uint32_t kNoSlot = 0xFFFFFFFFu;

// Records the thread-local message for grab_last_error() and returns `code`.
int grab_set_error(int code, const char* msg);

// Error carrying one of the GRAB_ERR_* codes; converted at the C-ABI edge.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define GRAB_CUDA(call)                                                              \
  do {                                                                               \
    cudaError_t e__ = (call);                                                        \
    if (e__ != cudaSuccess)                                                          \
      throw ::grab::Error(GRAB_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e__)); \
  } while (0)

#define GRAB_CHECK_LAUNCH() GRAB_CUDA(cudaGetLastError())

// Per-phys-row attribute record: the scalar predicate and the slot id, read
// together by one 8-byte load during the scalar pre-check.
struct __align__(8) Attr {
  float s;
  uint32_t slot;  // kNoSlot for an unused phys row (headroom)
};

__host__ __device__ inline uint64_t div_up(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ float4 ldg_nc_f4(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ Attr ld_attr(const Attr* a, uint32_t p) {
  uint2 v = __ldg(reinterpret_cast<const uint2*>(a) + p);
  Attr r;
  r.s = __uint_as_float(v.x);
  r.slot = v.y;
  return r;
}

// Accumulate (x-q)^2 for one float4 in f64, ascending coordinate order.
__device__ __forceinline__ double sq4(float4 x, float4 q, double acc) {
  double a = (double)x.x - (double)q.x;
  acc = fma(a, a, acc);
  a = (double)x.y - (double)q.y;
  acc = fma(a, a, acc);
  a = (double)x.z - (double)q.z;
  acc = fma(a, a, acc);
  a = (double)x.w - (double)q.w;
  acc = fma(a, a, acc);
  return acc;
}

// Butterfly all-reduce, pairing lane i with i^16, ^8, ^4, ^2, ^1. Every
// distance in this library goes through this tree so a given (q, x) pair has
// one bit pattern regardless of which kernel computed it.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

// Reduce G per-lane partials (G candidates) at once with the SAME pairing tree
// as warp_sum (i^16, ^8, ^4, ^2, ^1): the first log2(G) levels scatter halves
// of the candidate set between partner lanes, the rest all-reduce. Lane i ends
// with the full sum of candidate (i >> (5 - log2 G)); bit-identical to
// warp_sum(p[g]) because every level adds the same operand pair.
// Shuffles: 18 (G=8), 20 (G=4), 18 (G=2) double-words vs 10*G for warp_sum.
// One level per halving (i^16 splits G -> G/2, i^8 G/2 -> G/4, ...), the
// remaining levels all-reduce.
template <int N, uint32_t OFF>
__device__ __forceinline__ double reduce_scatter_level(const double (&p)[N]) {
  const uint32_t lane = threadIdx.x & 31u;
  constexpr int H = N / 2;
  const bool hi = (lane & OFF) != 0;
  double q[H];
#pragma unroll
  for (int j = 0; j < H; ++j) {
    const double send = hi ? p[j] : p[H + j];
    const double keep = hi ? p[H + j] : p[j];
    q[j] = keep + __shfl_xor_sync(0xFFFFFFFFu, send, OFF);
  }
  if constexpr (H == 1) {
    double t = q[0];
#pragma unroll
    for (uint32_t o = OFF / 2; o > 0; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
    return t;
  } else {
    return reduce_scatter_level<H, OFF / 2>(q);
  }
}

template <int G>
__device__ __forceinline__ double reduce_scatter(double (&p)[G]) {
  static_assert(G == 1 || G == 2 || G == 4 || G == 8 || G == 16, "G: a power of two <= 16");
  if constexpr (G == 1) {
    return warp_sum(p[0]);
  } else {
    return reduce_scatter_level<G, 16>(p);
  }
}

// Total order used for every (distance, slot) decision (SPEC tie rule).
__device__ __forceinline__ bool key_less(double da, uint32_t sa, double db, uint32_t sb) {
  return da < db || (da == db && sa < sb);
}

}  // namespace grab

namespace grab {
// Growable stream-ordered device scratch buffer.
struct DBufLite {
  void* p = nullptr;
  size_t cap = 0;
  cudaStream_t st = nullptr;
  void ensure(size_t bytes, cudaStream_t s) {
    if (bytes <= cap && p) return;
    if (p) cudaFreeAsync(p, st);
    st = s;
    p = nullptr;
    GRAB_CUDA(cudaMallocAsync(&p, bytes ? bytes : 16, s));
    cap = bytes;
  }
  ~DBufLite() {
    if (p) cudaFreeAsync(p, st);
  }
};
}  // namespace grab
