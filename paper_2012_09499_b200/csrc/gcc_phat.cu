// K1: GCC-PHAT cross-spectra for a batch of frames.
//
// Restates spectral.cross_spectrum (pkg/src/srpfast/spectral.py:218-285) for
// F frames at once:
//   raw    = y_m conj(y_m')                                    (:258)
//   floor  = 1e-12 * sqrt(mean_{p,k} |raw|^2) or explicit      (:268-275)
//   psi    = raw / max(|raw|, floor) where raw != 0, else 0    (:276-277)
//   identity weighting: psi = raw, floor 0                     (:259-267)
//
// Relative PHAT floor (the default): ONE HBM pass, speculative --
//   K1s psi: fully parallel over (frame, pair, bin pair), two bins per
//       thread, 16-byte loads of y_m and y_m' and a 16-byte store of psi (or
//       its fp16 operand split), computed WITHOUT the floor
//       (raw rsqrt(|y_m|^2) rsqrt(|y_m'|^2)); meanwhile each CTA reduces, in
//       fp64 from exact squares, sum |raw|^2 of its row, the minimum nonzero
//       |raw|^2 and an out-of-range flag, and adds them to per-frame totals.
//   K1f fix-up: one CTA per frame forms the floor 1e-12 sqrt(mean |raw|^2)
//       (the reference's fp64 value to rounding), writes it, and recomputes
//       the frame exactly only if some |raw| could be below it or a power
//       left the fast path's range -- otherwise every psi already equals
//       raw / max(|raw|, floor) (= raw / |raw| there) to fp32 rounding.
// Explicit floors / identity weighting: the psi pass alone.  The older
// two-pass form (K1a floor CTA per frame, then psi) stays for
// srpb_gcc_floor and SRPB_K1_TWOPASS=1.
// Algorithmic traffic: 8 (M + P) Kb bytes per frame.
#include "common.cuh"

#include <cuda_fp16.h>
#include <cstdlib>

namespace srpb {

constexpr int kFloorThreads = 512;
constexpr int kFloorSmemPowers = 4096;  // fp64 channel powers staged per pass (32 KB)
constexpr int kFloorMaxPairs = 2016;    // 64 channels

// One CTA per frame, thread <-> bin: stage |y_m[k]|^2 (fp64) for up to 4096
// (channel, bin) values per pass (all of them for M <= 8, Kb <= 512: each
// thread's M loads are in flight together), then accumulate
// sum_p pw[m_p][k] pw[m'_p][k] with pair indices broadcast from shared
// memory.  Also flags the frame "clean" when every fp32 channel power lies in
// the fast PHAT range (phat_power_clean), letting the fused lattice skip its
// per-bin range tests.
__global__ void __launch_bounds__(kFloorThreads)
gcc_floor_kernel(const float2* __restrict__ Y, int M, int Kb, const int32_t* __restrict__ pm,
                 const int32_t* __restrict__ pmp, int P, double floor_rel,
                 double* __restrict__ floor_out, int32_t* __restrict__ clean_out) {
  const int f = blockIdx.x;
  const float2* y = Y + static_cast<size_t>(f) * M * Kb;
  __shared__ double s_pow[kFloorSmemPowers];
  __shared__ int2 s_pair[kFloorMaxPairs];
  __shared__ double s_red[kFloorThreads / 32];
  for (int e = threadIdx.x; e < P; e += kFloorThreads) s_pair[e] = make_int2(pm[e], pmp[e]);
  const int kc_max = max(1, min(Kb, kFloorSmemPowers / M));
  double acc = 0.0;
  bool clean = true;
  for (int k0 = 0; k0 < Kb; k0 += kc_max) {
    const int kc = min(kc_max, Kb - k0);
    for (int kk = threadIdx.x; kk < kc; kk += kFloorThreads) {
#pragma unroll 8
      for (int m = 0; m < M; ++m) {
        const float2 v = __ldg(y + static_cast<size_t>(m) * Kb + k0 + kk);
        s_pow[m * kc + kk] = static_cast<double>(v.x) * v.x + static_cast<double>(v.y) * v.y;
        clean = clean && phat_power_clean(fmaf(v.x, v.x, v.y * v.y));
      }
    }
    __syncthreads();
    for (int kk = threadIdx.x; kk < kc; kk += kFloorThreads) {
#pragma unroll 4
      for (int pp = 0; pp < P; ++pp) {
        const int2 ab = s_pair[pp];
        acc += s_pow[ab.x * kc + kk] * s_pow[ab.y * kc + kk];
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
  const bool all_clean = __syncthreads_and(clean);
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int w = 0; w < kFloorThreads / 32; ++w) sum += s_red[w];
    if (floor_out) floor_out[f] = floor_rel * sqrt(sum / (static_cast<double>(P) * Kb));
    if (clean_out) clean_out[f] = all_clean ? 1 : 0;
  }
}

__global__ void fill_kernel(double* __restrict__ out, int n, double v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = v;
}

// One CTA per (frame, pair) row, threads along the bins: 16-byte loads of
// two bins of y_m and y_m' (L2-resident after K1a) and a 16-byte psi store.
constexpr int kPsiThreads = 128;

// fp16 operand split of scale * psi for the tensor-core K2 (hi = fp16(x),
// lo = fp16(x - hi)), written next to / instead of psi: the K2 operand
// without a separate split pass over Psi
__device__ __forceinline__ void psi_split16(float2 v, float scale, uint32_t& hi, uint32_t& lo) {
  const float xr = v.x * scale, xi = v.y * scale;
  const __half2 h = __floats2half2_rn(xr, xi);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(xr - hf.x, xi - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

// per-row statistics of the speculative pass, reduced per frame in a fixed
// order by the fix-up (deterministic floors)
struct K1Stats {
  double* sum;      // [F P] sum |raw|^2 over the row (fp64 from exact squares)
  float* min;       // [F P] min nonzero |raw|^2 (3e38: none)
  int* bad;         // [F P] some power outside the fast path's exact range
};

// Warp per (frame, pair) row, 8 rows per CTA: each lane streams its bins in
// 16-byte loads / stores (4 in flight), the row statistics reduce in-warp.
constexpr int kSpecRowsPerCta = 8;
template <bool kSplit>
__global__ void __launch_bounds__(32 * kSpecRowsPerCta)
gcc_psi_spec_kernel(const float4* __restrict__ Y, int M, int Kb2, const int32_t* __restrict__ pm,
                    const int32_t* __restrict__ pmp, int P, int rows, float4* __restrict__ Psi,
                    uint2* __restrict__ Psi_hi, uint2* __restrict__ Psi_lo, float scale,
                    K1Stats st) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * kSpecRowsPerCta + (threadIdx.x >> 5);  // f * P + p
  if (row >= rows) return;
  const int f = row / P, p = row - f * P;
  const float4* ya = Y + (static_cast<size_t>(f) * M + __ldg(pm + p)) * Kb2;
  const float4* yb = Y + (static_cast<size_t>(f) * M + __ldg(pmp + p)) * Kb2;
  const PhatFloor nofl = {0.0, __int_as_float(0x7f800000)};  // 1/floor = inf: no floor
  const size_t o = static_cast<size_t>(row) * Kb2;
  double sum = 0.0;
  float mn = 3.0e38f;
  int bad = 0;
  auto one = [&](float2 a, float2 b, float2& out) {
    float pa, pb;
    out = phat_fast(a, b, nofl, pa, pb);
    const double da = static_cast<double>(a.x) * a.x + static_cast<double>(a.y) * a.y;
    const double db = static_cast<double>(b.x) * b.x + static_cast<double>(b.y) * b.y;
    sum = fma(da, db, sum);
    if (pa != 0.0f && pb != 0.0f) mn = fminf(mn, pa * pb);
    bad |= !(phat_power_clean(pa) && phat_power_clean(pb));
  };
#pragma unroll 4
  for (int k2 = lane; k2 < Kb2; k2 += 32) {
    const float4 a = __ldg(ya + k2), b = __ldg(yb + k2);
    float2 o0, o1;
    one(make_float2(a.x, a.y), make_float2(b.x, b.y), o0);
    one(make_float2(a.z, a.w), make_float2(b.z, b.w), o1);
    if (!kSplit || Psi) __stcs(Psi + o + k2, make_float4(o0.x, o0.y, o1.x, o1.y));
    if constexpr (kSplit) {
      uint2 h, l;
      psi_split16(o0, scale, h.x, l.x);
      psi_split16(o1, scale, h.y, l.y);
      __stcs(reinterpret_cast<unsigned long long*>(Psi_hi + o + k2),
             (static_cast<unsigned long long>(h.y) << 32) | h.x);
      __stcs(reinterpret_cast<unsigned long long*>(Psi_lo + o + k2),
             (static_cast<unsigned long long>(l.y) << 32) | l.x);
    }
  }
  // fixed-order warp reduction; one entry per row
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, d);
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, d));
  }
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    st.sum[row] = sum;
    st.min[row] = mn;
    st.bad[row] = bad;
  }
}

// Frame-resident form (the frame's spectra fit shared memory, M Kb 8 bytes
// <= 200 KB: every BASELINE config): one CTA per frame loads Y_f once
// (coalesced 16-byte loads -- a row kernel re-reads each channel for each of
// its M - 1 pairs from L2), forms every pair's psi speculatively with the
// frame's statistics in registers, reduces them in a fixed order, writes the
// floor, and redoes the frame exactly from the staged spectra if needed:
// one kernel, Y read once, psi written once (twice for a flagged frame).
constexpr int kFrameThreads = 1024;
template <bool kSplit>
__global__ void __launch_bounds__(kFrameThreads)
gcc_psi_frame_kernel(const float4* __restrict__ Y, int M, int Kb2, const int32_t* __restrict__ pm,
                     const int32_t* __restrict__ pmp, int P, double floor_rel,
                     double* __restrict__ floor_out, float4* __restrict__ Psi,
                     uint2* __restrict__ Psi_hi, uint2* __restrict__ Psi_lo, float scale) {
  extern __shared__ float4 y_s[];  // [M][Kb2]
  __shared__ int2 s_pair[kFloorMaxPairs];
  __shared__ double s_sum[kFrameThreads / 32];
  __shared__ float s_mn[kFrameThreads / 32];
  __shared__ int s_redo;
  __shared__ double s_floor;
  const int f = blockIdx.x;
  const float4* yf = Y + static_cast<size_t>(f) * M * Kb2;
  for (int i = threadIdx.x; i < M * Kb2; i += kFrameThreads) y_s[i] = __ldg(yf + i);
  for (int e = threadIdx.x; e < P; e += kFrameThreads) s_pair[e] = make_int2(pm[e], pmp[e]);
  __syncthreads();
  const int n = P * Kb2;
  const size_t o = static_cast<size_t>(f) * n;
  const bool pow2 = (Kb2 & (Kb2 - 1)) == 0;
  const int sh = 31 - __clz(Kb2);
  auto store = [&](int e, float2 o0, float2 o1) {
    if (!kSplit || Psi) __stcs(Psi + o + e, make_float4(o0.x, o0.y, o1.x, o1.y));
    if constexpr (kSplit) {
      uint2 h, l;
      psi_split16(o0, scale, h.x, l.x);
      psi_split16(o1, scale, h.y, l.y);
      __stcs(reinterpret_cast<unsigned long long*>(Psi_hi + o + e),
             (static_cast<unsigned long long>(h.y) << 32) | h.x);
      __stcs(reinterpret_cast<unsigned long long*>(Psi_lo + o + e),
             (static_cast<unsigned long long>(l.y) << 32) | l.x);
    }
  };
  const PhatFloor nofl = {0.0, __int_as_float(0x7f800000)};  // 1/floor = inf: no floor
  double sum = 0.0;
  float mn = 3.0e38f;
  int bad = 0;
  auto one = [&](float2 a, float2 b, float2& out) {
    float pa, pb;
    out = phat_fast(a, b, nofl, pa, pb);
    const double da = static_cast<double>(a.x) * a.x + static_cast<double>(a.y) * a.y;
    const double db = static_cast<double>(b.x) * b.x + static_cast<double>(b.y) * b.y;
    sum = fma(da, db, sum);
    if (pa != 0.0f && pb != 0.0f) mn = fminf(mn, pa * pb);
    bad |= !(phat_power_clean(pa) && phat_power_clean(pb));
  };
  if (kSplit && !Psi && (Kb2 & 1) == 0) {
    // split only: 4 bins per thread per step, 16-byte stores of hi and lo
#pragma unroll 2
    for (int e = 2 * threadIdx.x; e < n; e += 2 * kFrameThreads) {
      const int p = pow2 ? e >> sh : e / Kb2;
      const int k2 = e - p * Kb2;
      const int2 ab = s_pair[p];
      const float4 a0 = y_s[ab.x * Kb2 + k2], b0 = y_s[ab.y * Kb2 + k2];
      const float4 a1 = y_s[ab.x * Kb2 + k2 + 1], b1 = y_s[ab.y * Kb2 + k2 + 1];
      float2 ov[4];
      one(make_float2(a0.x, a0.y), make_float2(b0.x, b0.y), ov[0]);
      one(make_float2(a0.z, a0.w), make_float2(b0.z, b0.w), ov[1]);
      one(make_float2(a1.x, a1.y), make_float2(b1.x, b1.y), ov[2]);
      one(make_float2(a1.z, a1.w), make_float2(b1.z, b1.w), ov[3]);
      uint4 h, l;
      psi_split16(ov[0], scale, h.x, l.x);
      psi_split16(ov[1], scale, h.y, l.y);
      psi_split16(ov[2], scale, h.z, l.z);
      psi_split16(ov[3], scale, h.w, l.w);
      __stcs(reinterpret_cast<uint4*>(Psi_hi + o + e), h);
      __stcs(reinterpret_cast<uint4*>(Psi_lo + o + e), l);
    }
  } else {
#pragma unroll 4
    for (int e = threadIdx.x; e < n; e += kFrameThreads) {
      const int p = pow2 ? e >> sh : e / Kb2;
      const int k2 = e - p * Kb2;
      const int2 ab = s_pair[p];
      const float4 a = y_s[ab.x * Kb2 + k2], b = y_s[ab.y * Kb2 + k2];
      float2 o0, o1;
      one(make_float2(a.x, a.y), make_float2(b.x, b.y), o0);
      one(make_float2(a.z, a.w), make_float2(b.z, b.w), o1);
      store(e, o0, o1);
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, d);
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, d));
  }
  bad = __syncthreads_or(bad);
  if ((threadIdx.x & 31) == 0) {
    s_sum[threadIdx.x >> 5] = sum;
    s_mn[threadIdx.x >> 5] = mn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    float m = 3.0e38f;
    for (int w = 0; w < kFrameThreads / 32; ++w) {
      t += s_sum[w];
      m = fminf(m, s_mn[w]);
    }
    const double floor = floor_rel * sqrt(t / (static_cast<double>(P) * 2 * Kb2));
    s_redo = bad || static_cast<double>(m) < 1.01 * floor * floor;  // fp32 |raw|^2 margin
    s_floor = floor;
    if (floor_out) floor_out[f] = floor;
  }
  __syncthreads();
  if (!s_redo) return;
  const PhatFloor fl = make_phat_floor(s_floor);
  for (int e = threadIdx.x; e < n; e += kFrameThreads) {
    const int p = pow2 ? e >> sh : e / Kb2;
    const int k2 = e - p * Kb2;
    const int2 ab = s_pair[p];
    const float4 a = y_s[ab.x * Kb2 + k2], b = y_s[ab.y * Kb2 + k2];
    store(e, phat_one(make_float2(a.x, a.y), make_float2(b.x, b.y), 0, fl),
          phat_one(make_float2(a.z, a.w), make_float2(b.z, b.w), 0, fl));
  }
}

// One CTA per frame: the floor, and the exact redo of a frame whose
// speculative psi could differ (some |raw|^2 below ~floor^2, or a power out
// of the fast path's range).  Resets the frame's statistics for the next call.
template <bool kSplit>
__global__ void __launch_bounds__(256)
gcc_psi_fixup_kernel(const float4* __restrict__ Y, int M, int Kb2, const int32_t* __restrict__ pm,
                     const int32_t* __restrict__ pmp, int P, double floor_rel,
                     double* __restrict__ floor_out, float4* __restrict__ Psi,
                     uint2* __restrict__ Psi_hi, uint2* __restrict__ Psi_lo, float scale,
                     K1Stats st) {
  const int f = blockIdx.x;
  __shared__ int s_redo;
  __shared__ double s_floor;
  __shared__ double s_sum[8];
  __shared__ float s_mn[8];
  // the frame's row statistics in a fixed order (thread t: rows t, t + 256, ..)
  double t = 0.0;
  float m = 3.0e38f;
  int bad = 0;
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    const size_t r = static_cast<size_t>(f) * P + p;
    t += st.sum[r];
    m = fminf(m, st.min[r]);
    bad |= st.bad[r];
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    t += __shfl_xor_sync(0xffffffffu, t, d);
    m = fminf(m, __shfl_xor_sync(0xffffffffu, m, d));
  }
  bad = __syncthreads_or(bad);
  if ((threadIdx.x & 31) == 0) {
    s_sum[threadIdx.x >> 5] = t;
    s_mn[threadIdx.x >> 5] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0;
    float mn = 3.0e38f;
    for (int w = 0; w < 8; ++w) {
      sum += s_sum[w];
      mn = fminf(mn, s_mn[w]);
    }
    const double floor = floor_rel * sqrt(sum / (static_cast<double>(P) * 2 * Kb2));
    // 1.01: margin for the fp32 |raw|^2 against the fp64 floor^2
    s_redo = bad || static_cast<double>(mn) < 1.01 * floor * floor;
    s_floor = floor;
    if (floor_out) floor_out[f] = floor;
  }
  __syncthreads();
  if (!s_redo) return;
  const PhatFloor fl = make_phat_floor(s_floor);
  for (int p = 0; p < P; ++p) {
    const float4* ya = Y + (static_cast<size_t>(f) * M + __ldg(pm + p)) * Kb2;
    const float4* yb = Y + (static_cast<size_t>(f) * M + __ldg(pmp + p)) * Kb2;
    const size_t o = (static_cast<size_t>(f) * P + p) * Kb2;
    for (int k2 = threadIdx.x; k2 < Kb2; k2 += blockDim.x) {
      const float4 a = __ldg(ya + k2), b = __ldg(yb + k2);
      const float2 o0 = phat_one(make_float2(a.x, a.y), make_float2(b.x, b.y), 0, fl);
      const float2 o1 = phat_one(make_float2(a.z, a.w), make_float2(b.z, b.w), 0, fl);
      if (!kSplit || Psi) Psi[o + k2] = make_float4(o0.x, o0.y, o1.x, o1.y);
      if constexpr (kSplit) {
        uint2 h, l;
        psi_split16(o0, scale, h.x, l.x);
        psi_split16(o1, scale, h.y, l.y);
        Psi_hi[o + k2] = h;
        Psi_lo[o + k2] = l;
      }
    }
  }
}

template <bool kSplit>
__global__ void __launch_bounds__(kPsiThreads)
gcc_psi_kernel(const float4* __restrict__ Y, int M, int Kb2, const int32_t* __restrict__ pm,
               const int32_t* __restrict__ pmp, int P, int weighting,
               const double* __restrict__ floors, double const_floor, float4* __restrict__ Psi,
               uint2* __restrict__ Psi_hi, uint2* __restrict__ Psi_lo, float scale) {
  const int row = blockIdx.x;  // f * P + p
  const int f = row / P, p = row - f * P;
  const float4* ya = Y + (static_cast<size_t>(f) * M + __ldg(pm + p)) * Kb2;
  const float4* yb = Y + (static_cast<size_t>(f) * M + __ldg(pmp + p)) * Kb2;
  const PhatFloor fl = make_phat_floor(floors ? __ldg(floors + f) : const_floor);
  const size_t o = static_cast<size_t>(row) * Kb2;
  for (int k2 = threadIdx.x; k2 < Kb2; k2 += kPsiThreads) {
    const float4 a = __ldg(ya + k2), b = __ldg(yb + k2);
    const float2 o0 = phat_one(make_float2(a.x, a.y), make_float2(b.x, b.y), weighting, fl);
    const float2 o1 = phat_one(make_float2(a.z, a.w), make_float2(b.z, b.w), weighting, fl);
    if (!kSplit || Psi) Psi[o + k2] = make_float4(o0.x, o0.y, o1.x, o1.y);
    if constexpr (kSplit) {
      uint2 h, l;
      psi_split16(o0, scale, h.x, l.x);
      psi_split16(o1, scale, h.y, l.y);
      Psi_hi[o + k2] = h;
      Psi_lo[o + k2] = l;
    }
  }
}

// odd Kb or unaligned buffers: one bin per thread
__global__ void __launch_bounds__(kPsiThreads)
gcc_psi1_kernel(const float2* __restrict__ Y, int M, int Kb, const int32_t* __restrict__ pm,
                const int32_t* __restrict__ pmp, int P, int weighting,
                const double* __restrict__ floors, double const_floor, float2* __restrict__ Psi) {
  const int row = blockIdx.x;
  const int f = row / P, p = row - f * P;
  const float2* ya = Y + (static_cast<size_t>(f) * M + __ldg(pm + p)) * Kb;
  const float2* yb = Y + (static_cast<size_t>(f) * M + __ldg(pmp + p)) * Kb;
  const PhatFloor fl = make_phat_floor(floors ? __ldg(floors + f) : const_floor);
  float2* out = Psi + static_cast<size_t>(row) * Kb;
  for (int k = threadIdx.x; k < Kb; k += kPsiThreads)
    out[k] = phat_one(__ldg(ya + k), __ldg(yb + k), weighting, fl);
}

cudaError_t launch_gcc_floor(const float* Y, int F, int M, int Kb, const int32_t* pm,
                             const int32_t* pmp, int P, double floor_rel, double* floor_out,
                             int32_t* clean_out, cudaStream_t stream) {
  if (F == 0) return cudaSuccess;
  gcc_floor_kernel<<<F, kFloorThreads, 0, stream>>>(reinterpret_cast<const float2*>(Y), M, Kb, pm,
                                                     pmp, P, floor_rel, floor_out, clean_out);
  return cudaGetLastError();
}

thread_local int g_gcc_kernels = 0;
int gcc_phat_last_kernels() { return g_gcc_kernels; }

cudaError_t launch_gcc_phat(const float* Y, int F, int M, int Kb, const int32_t* pm,
                            const int32_t* pmp, int P, int weighting, double floor_rel,
                            double abs_floor, float* Psi, double* floor_out,
                            cudaStream_t stream, void* Psi_hi, void* Psi_lo, float split_scale) {
  g_gcc_kernels = 0;
  if (F == 0) return cudaSuccess;
  // relative floor: per-frame values from K1a (into floor_out, or into a
  // stream-ordered scratch when the caller passed none); explicit floor and
  // identity weighting: one constant
  const bool per_frame = weighting == 0 && !(abs_floor > 0.0);
  const double const_floor = weighting == 0 ? abs_floor : 0.0;
  double* floors = nullptr;
  cudaError_t e = cudaSuccess;
  const bool vec0 = Kb % 2 == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(Psi) & 15) == 0 &&
                    ((reinterpret_cast<uintptr_t>(Psi_hi) | reinterpret_cast<uintptr_t>(Psi_lo)) & 7) == 0;
  static const bool two_pass = getenv("SRPB_K1_TWOPASS") != nullptr;
  const size_t frame_smem = size_t(M) * Kb * 8;
  if (per_frame && vec0 && !two_pass && frame_smem <= 200 * 1024 && P <= kFloorMaxPairs &&
      getenv("SRPB_K1_ROWS") == nullptr) {
    const int smem = static_cast<int>(frame_smem);
    if (Psi_hi != nullptr) {
      auto k = gcc_psi_frame_kernel<true>;
      e = allow_dynamic_smem(k, smem);
      if (e != cudaSuccess) return e;
      ++g_gcc_kernels;
      k<<<F, kFrameThreads, smem, stream>>>(
          reinterpret_cast<const float4*>(Y), M, Kb / 2, pm, pmp, P, floor_rel, floor_out,
          reinterpret_cast<float4*>(Psi), static_cast<uint2*>(Psi_hi), static_cast<uint2*>(Psi_lo),
          split_scale);
    } else {
      auto k = gcc_psi_frame_kernel<false>;
      e = allow_dynamic_smem(k, smem);
      if (e != cudaSuccess) return e;
      ++g_gcc_kernels;
      k<<<F, kFrameThreads, smem, stream>>>(
          reinterpret_cast<const float4*>(Y), M, Kb / 2, pm, pmp, P, floor_rel, floor_out,
          reinterpret_cast<float4*>(Psi), nullptr, nullptr, 0.0f);
    }
    return cudaGetLastError();
  }
  if (per_frame && vec0 && !two_pass) {
    // the stream-ordered scratch below comes from the device's default pool:
    // keep freed blocks in the pool (the default release threshold of 0
    // returns them to the driver at every synchronisation, and re-mapping
    // 32 MB per call cost ~30 ms at C4)
    static int pool_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && dev != pool_dev) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        unsigned long long keep = ~0ull;  // cudaMemPoolAttrReleaseThreshold: uint64
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      pool_dev = dev;
    }
    // speculative single pass + per-frame fix-up; row statistics in
    // stream-ordered scratch
    const int rows = F * P;
    char* scratch = nullptr;
    const size_t bytes = size_t(rows) * (sizeof(double) + sizeof(float) + sizeof(int));
    e = cudaMallocAsync(reinterpret_cast<void**>(&scratch), bytes, stream);
    if (e != cudaSuccess) return e;
    K1Stats st{reinterpret_cast<double*>(scratch),
               reinterpret_cast<float*>(scratch + size_t(rows) * sizeof(double)),
               reinterpret_cast<int*>(scratch + size_t(rows) * (sizeof(double) + sizeof(float)))};
    if (Psi_hi != nullptr) {
      ++g_gcc_kernels;
      gcc_psi_spec_kernel<true><<<(rows + kSpecRowsPerCta - 1) / kSpecRowsPerCta,
                                   32 * kSpecRowsPerCta, 0, stream>>>(
          reinterpret_cast<const float4*>(Y), M, Kb / 2, pm, pmp, P, rows,
          reinterpret_cast<float4*>(Psi), static_cast<uint2*>(Psi_hi),
          static_cast<uint2*>(Psi_lo), split_scale, st);
      ++g_gcc_kernels;
      gcc_psi_fixup_kernel<true><<<F, 256, 0, stream>>>(
          reinterpret_cast<const float4*>(Y), M, Kb / 2, pm, pmp, P, floor_rel, floor_out,
          reinterpret_cast<float4*>(Psi), static_cast<uint2*>(Psi_hi),
          static_cast<uint2*>(Psi_lo), split_scale, st);
    } else {
      ++g_gcc_kernels;
      gcc_psi_spec_kernel<false><<<(rows + kSpecRowsPerCta - 1) / kSpecRowsPerCta,
                                    32 * kSpecRowsPerCta, 0, stream>>>(
          reinterpret_cast<const float4*>(Y), M, Kb / 2, pm, pmp, P, rows,
          reinterpret_cast<float4*>(Psi), nullptr, nullptr, 0.0f, st);
      ++g_gcc_kernels;
      gcc_psi_fixup_kernel<false><<<F, 256, 0, stream>>>(
          reinterpret_cast<const float4*>(Y), M, Kb / 2, pm, pmp, P, floor_rel, floor_out,
          reinterpret_cast<float4*>(Psi), nullptr, nullptr, 0.0f, st);
    }
    e = cudaGetLastError();
    const cudaError_t e2 = cudaFreeAsync(scratch, stream);
    return e != cudaSuccess ? e : e2;
  }
  if (per_frame) {
    floors = floor_out;
    if (!floors) {
      e = cudaMallocAsync(reinterpret_cast<void**>(&floors), sizeof(double) * F, stream);
      if (e != cudaSuccess) return e;
    }
    ++g_gcc_kernels;
    gcc_floor_kernel<<<F, kFloorThreads, 0, stream>>>(reinterpret_cast<const float2*>(Y), M, Kb,
                                                       pm, pmp, P, floor_rel, floors, nullptr);
  } else if (floor_out) {
    ++g_gcc_kernels;
    fill_kernel<<<(F + 255) / 256, 256, 0, stream>>>(floor_out, F, const_floor);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const bool vec = Kb % 2 == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(Psi) & 15) == 0 &&
                   ((reinterpret_cast<uintptr_t>(Psi_hi) | reinterpret_cast<uintptr_t>(Psi_lo)) & 7) == 0;
  const int rows = F * P;
  if (Psi_hi != nullptr && !vec) return cudaErrorInvalidValue;  // split needs the 2-bin path
  ++g_gcc_kernels;  // the psi pass
  if (vec && Psi_hi != nullptr)
    gcc_psi_kernel<true><<<rows, kPsiThreads, 0, stream>>>(
        reinterpret_cast<const float4*>(Y), M, Kb / 2, pm, pmp, P, weighting, floors, const_floor,
        reinterpret_cast<float4*>(Psi), static_cast<uint2*>(Psi_hi), static_cast<uint2*>(Psi_lo),
        split_scale);
  else if (vec)
    gcc_psi_kernel<false><<<rows, kPsiThreads, 0, stream>>>(
        reinterpret_cast<const float4*>(Y), M, Kb / 2, pm, pmp, P, weighting, floors, const_floor,
        reinterpret_cast<float4*>(Psi), nullptr, nullptr, 0.0f);
  else
    gcc_psi1_kernel<<<rows, kPsiThreads, 0, stream>>>(reinterpret_cast<const float2*>(Y), M, Kb,
                                                      pm, pmp, P, weighting, floors, const_floor,
                                                      reinterpret_cast<float2*>(Psi));
  e = cudaGetLastError();
  if (per_frame && !floor_out) {
    const cudaError_t e2 = cudaFreeAsync(floors, stream);
    if (e == cudaSuccess) e = e2;
  }
  return e;
}

}  // namespace srpb
