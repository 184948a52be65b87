// Shared device helpers for the SRP hot-path kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

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
// Per-frame floor constants: the fp64 floor and its fp32 reciprocal (inf for
// a zero floor; within 1 ulp of 1/floor, it only moves the exact switch-over
// point, where both branches agree).
struct PhatFloor {
  double floor;
  float inv_floor;
};

__device__ __forceinline__ PhatFloor make_phat_floor(double floor) {
  return {floor, __frcp_rn(static_cast<float>(floor))};  // 1/0 = inf
}

static __device__ __forceinline__ float2 phat_slow(float2 a, float2 b, double floor) {
  // extreme magnitudes: normalise each factor first (no over/underflow)
  const float ma = hypotf(a.x, a.y), mb = hypotf(b.x, b.y);
  const double mag = static_cast<double>(ma) * mb;
  if (mag >= floor) {
    const float ua = 1.0f / ma, ub = 1.0f / mb;
    const float ax = a.x * ua, ay = a.y * ua, bx = b.x * ub, by = b.y * ub;
    return make_float2(ax * bx + ay * by, ay * bx - ax * by);
  }
  const double re = static_cast<double>(a.x) * b.x + static_cast<double>(a.y) * b.y;
  const double im = static_cast<double>(a.y) * b.x - static_cast<double>(a.x) * b.y;
  return make_float2(static_cast<float>(re / floor), static_cast<float>(im / floor));
}

__device__ __forceinline__ float rsqrt_approx_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Range in which the fast PHAT is exact to fp32 rounding: |y|^2 in
// (1e-30, 1e30) or exactly 0.  K1a flags frames whose every channel power
// qualifies ("clean" frames); those skip the per-bin range test.
__device__ __forceinline__ bool phat_power_clean(float pw) {
  return pw == 0.0f || (pw > 1e-30f && pw < 1e30f);
}

// Fast PHAT: 1/|raw| = rsqrt(pa) rsqrt(pb) and raw / max(|raw|, floor) =
// raw * min(1/|raw|, 1/floor).  The powers are clamped below at 1e-30 so an
// exact-zero factor gives raw = 0 times a finite scale (= 0, as required).
// Exact (to fp32 rounding) when both powers are phat_power_clean; other
// inputs must take phat_slow.
__device__ __forceinline__ float2 phat_fast(float2 a, float2 b, PhatFloor fl, float& pa,
                                            float& pb) {
  pa = fmaf(a.x, a.x, a.y * a.y);
  pb = fmaf(b.x, b.x, b.y * b.y);
  const float s = fminf(rsqrt_approx_ftz(fmaxf(pa, 1e-30f)) * rsqrt_approx_ftz(fmaxf(pb, 1e-30f)),
                        fl.inv_floor);
  const float re = fmaf(a.x, b.x, a.y * b.y), im = fmaf(a.y, b.x, -(a.x * b.y));
  return make_float2(re * s, im * s);
}

__device__ __forceinline__ float2 phat_identity(float2 a, float2 b) {
  // raw product, correctly rounded from fp64
  const double re = static_cast<double>(a.x) * b.x + static_cast<double>(a.y) * b.y;
  const double im = static_cast<double>(a.y) * b.x - static_cast<double>(a.x) * b.y;
  return make_float2(static_cast<float>(re), static_cast<float>(im));
}

// per-thread form (any thread subset)
__device__ __forceinline__ float2 phat_one(float2 a, float2 b, int weighting, PhatFloor fl) {
  if (weighting != 0) return phat_identity(a, b);
  float pa, pb;
  const float2 v = phat_fast(a, b, fl, pa, pb);
  return phat_power_clean(pa) && phat_power_clean(pb) ? v : phat_slow(a, b, fl.floor);
}

// Cross-spectrum modes of the fused lattice (CTA-uniform, compile-time):
enum PsiMode {
  kPsiStaged = 0,
  kPsiIdentity = 1,
  kPsiPhatClean = 2,
  kPsiPhatChecked = 3,
  kPsiPhatSpec = 4  // relative floor deferred: raw/|raw|, stats for the fix-up pass
};

// Speculative PHAT (kPsiPhatSpec): per-lane statistics over the bins it
// forms -- sum and min of |raw|^2 over nonzero bins, and whether any power
// left the range (1e-15, 1e15) where the fast path and |raw|^2 in fp32 are
// exact.  A frame whose min |raw|^2 could fall below floor^2 = rel^2
// mean |raw|^2, or with an out-of-range power, is recomputed exactly.
struct PhatSpecStats {
  float sum = 0.0f;
  float min = 3.0e38f;
  int bad = 0;
  __device__ __forceinline__ void add(float pa, float pb) {
    if (pa != 0.0f && pb != 0.0f) {
      const float q = pa * pb;
      sum += q;
      min = fminf(min, q);
      bad |= !(pa > 1e-15f && pa < 1e15f && pb > 1e-15f && pb < 1e15f);
    }
  }
};

// warp form (all 32 lanes active), same values as phat_one: kPsiPhatClean
// (every lane's frame flagged clean by K1a) skips the range test;
// kPsiPhatChecked enters the slow path only when some lane needs it
template <int kMode>
__device__ __forceinline__ float2 psi_warp(float2 a, float2 b, PhatFloor fl) {
  if constexpr (kMode == kPsiStaged) {
    return a;
  } else if constexpr (kMode == kPsiIdentity) {
    return phat_identity(a, b);
  } else {
    float pa, pb;
    float2 v = phat_fast(a, b, fl, pa, pb);
    if constexpr (kMode == kPsiPhatChecked) {
      const bool slow = !(phat_power_clean(pa) && phat_power_clean(pb));
      if (__any_sync(0xffffffffu, slow)) {
        if (slow) v = phat_slow(a, b, fl.floor);
      }
    }
    return v;
  }
}

// Sinc weight sinc(x - n) from the split x = i + f (|f| <= 1/2), the
// reference's normalised sinc snapped to exactly 1 / 0 at integer arguments
// (srp._sinc_kernel srp.py:250-261): with d = i - n,
//   sinc(d + f) = (-1)^d (sin(pi f) / pi) / (d + f),   exactly [d == 0] if f == 0.
// spi = sin(pi f) / pi per (candidate, pair); the reciprocal is the
// single-instruction approximation (<= 1 ulp), and the same function feeds
// both the stored table and the in-TMEM generator, so they agree bitwise.
__device__ __forceinline__ float rcp_approx_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Reciprocals of an (even, odd) column pair's denominators from one MUFU:
// P = 1 / (xe xo), 1 / xe = xo P, 1 / xo = xe P (<= ~2.5 ulp; |x| >= 0.5 or
// a normal |f| > 1e-30, so xe xo neither over- nor underflows).  odd selects
// the column.  The tensor-core generator evaluates the same expressions.
__device__ __forceinline__ float sinc_pair_rcp(float xe, float xo, int odd) {
  const float P = rcp_approx_ftz(xe * xo);
  return (odd ? xe : xo) * P;
}
__device__ __forceinline__ float sinc_spi(float f) {
  return sinpif(f) * 0.318309886183790671538f;  // sin(pi f) / pi
}
// Exact-node test: f == 0 (an integer argument, snapped by the reference),
// and |f| < 1e-30, where sin(pi f) / (pi f) is 1 and sin(pi f) / (pi d) is 0
// to fp64 rounding (and the fp32 reciprocal would see a denormal).
__device__ __forceinline__ bool sinc_is_node(float f) { return fabsf(f) < 1e-30f; }
__device__ __forceinline__ float sinc_weight_fast(int i, float f, float spi, int n) {
  const int d = i - n;
  const float w = __uint_as_float(__float_as_uint(spi * rcp_approx_ftz(static_cast<float>(d) + f)) ^
                                  (static_cast<uint32_t>(d & 1) << 31));
  return sinc_is_node(f) ? (d == 0 ? 1.0f : 0.0f) : w;
}

// Programmatic dependent launch on the lattice -> fix-up -> K4 chain (default
// on).  SRPB_NO_PDL=1 launches them as plain stream-ordered kernels: ncu's
// per-node profiling of captured graphs rejects the programmatic edges
// (LaunchFailed), so launch lists of graph replays are taken with it set.
inline int pdl_attr_value() {
  static const int v = getenv("SRPB_NO_PDL") ? 0 : 1;
  return v;
}

// Opt a kernel into dynamic shared memory.  The attribute is raised to the
// device's whole opt-in budget rather than to this launch's size: it is per
// function, and a captured graph node replayed after another launch of the
// same kernel lowered it would otherwise be refused (ncu's per-node replay of
// graphs does exactly that).  The launch's own dynamicSmemBytes still decides
// the carveout.
template <typename Kern>
inline cudaError_t allow_dynamic_smem(Kern kern, size_t need) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, kern);
  if (e != cudaSuccess) return e;
  int dev = 0, optin = 0;
  e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  const int cap = optin - static_cast<int>(fa.sharedSizeBytes);
  if (need > static_cast<size_t>(cap)) return cudaErrorInvalidValue;
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
}

}  // namespace srpb
