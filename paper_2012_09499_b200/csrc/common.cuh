// Shared device helpers for the SRP hot-path kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace srpb {

constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs

// ---------------------------------------------------------------------------
// Packed argmax keys (srp.argmax_candidate, srp.py:107-109: lowest index
// among maxima).  key = orderable(value) << 32 | (0xFFFFFFFF - j): an
// unsigned max over keys picks the largest value, then the smallest j.
// -0.0 is canonicalised to +0.0 first (numpy treats them as equal).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t orderable_bits(float v) {
  v = v + 0.0f;  // -0 -> +0
  uint32_t b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ unsigned long long make_key(float v, uint32_t j) {
  return (static_cast<unsigned long long>(orderable_bits(v)) << 32) |
         static_cast<unsigned long long>(0xFFFFFFFFu - j);
}

__device__ __forceinline__ unsigned long long key_max(unsigned long long a,
                                                      unsigned long long b) {
  return a > b ? a : b;
}

__device__ __forceinline__ unsigned long long warp_key_max(unsigned long long k) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) k = key_max(k, __shfl_xor_sync(0xffffffffu, k, o));
  return k;
}

// ---------------------------------------------------------------------------
// Steering phase e^{j 2 pi k (i + f) / period} with the integer part reduced
// exactly: turns = ((k*i) mod period) / period + k*f / period.  `ti` arrives
// pre-reduced to [0, period) (host side), so k*ti < period^2 fits in 32 bits.
// `mask` = period-1 when period is a power of two (all BASELINE configs),
// else 0 (generic modulo).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float harmonic_turns(int k, int ti, float tf, int period,
                                                int mask, float inv_period) {
  unsigned int ki = static_cast<unsigned int>(k) * static_cast<unsigned int>(ti);
  unsigned int r = mask ? (ki & static_cast<unsigned int>(mask))
                        : (ki % static_cast<unsigned int>(period));
  return static_cast<float>(r) * inv_period + static_cast<float>(k) * tf * inv_period;
}

__device__ __forceinline__ void harmonic_phase(int k, int ti, float tf, int period, int mask,
                                               float inv_period, float* c, float* s) {
  sincospif(2.0f * harmonic_turns(k, ti, tf, period, mask, inv_period), s, c);
}

// GCC-PHAT weighting of one bin (spectral.py:258-277): raw = a conj(b),
// psi = raw / max(|raw|, floor), exact 0 where raw == 0; identity: raw.
__device__ __forceinline__ float2 phat_one(float2 a, float2 b, int weighting, double floor) {
  if (weighting != 0) {  // identity: raw product, correctly rounded from fp64
    const double re = static_cast<double>(a.x) * b.x + static_cast<double>(a.y) * b.y;
    const double im = static_cast<double>(a.y) * b.x - static_cast<double>(a.x) * b.y;
    return make_float2(static_cast<float>(re), static_cast<float>(im));
  }
  if ((a.x == 0.0f && a.y == 0.0f) || (b.x == 0.0f && b.y == 0.0f))
    return make_float2(0.0f, 0.0f);  // exact-zero product stays zero
  const float ma = hypotf(a.x, a.y), mb = hypotf(b.x, b.y);
  const double mag = static_cast<double>(ma) * mb;
  if (mag >= floor) {
    // raw/|raw| = (a/|a|) conj(b/|b|): unit modulus, no over/underflow
    const float ua = 1.0f / ma, ub = 1.0f / mb;
    const float ax = a.x * ua, ay = a.y * ua, bx = b.x * ub, by = b.y * ub;
    return make_float2(ax * bx + ay * by, ay * bx - ax * by);
  }
  const double re = static_cast<double>(a.x) * b.x + static_cast<double>(a.y) * b.y;
  const double im = static_cast<double>(a.y) * b.x - static_cast<double>(a.x) * b.y;
  return make_float2(static_cast<float>(re / floor), static_cast<float>(im / floor));
}

}  // namespace srpb
