// K1: GCC-PHAT cross-spectra for a batch of frames.
//
// Restates spectral.cross_spectrum (pkg/src/srpfast/spectral.py:218-285) for
// F frames at once:
//   raw    = y_m conj(y_m')                                    (:258)
//   floor  = 1e-12 * sqrt(mean_{p,k} |raw|^2) or explicit      (:268-275)
//   psi    = raw / max(|raw|, floor) where raw != 0, else 0    (:276-277)
//   identity weighting: psi = raw, floor 0                     (:259-267)
//
// Two HBM-bound passes:
//   K1a floor: one CTA per frame reduces sum_{p,k} |y_m|^2 |y_m'|^2 in fp64
//       from per-bin channel powers staged in shared memory (the applied
//       floor matches the reference's fp64 value to rounding); it reads Y
//       once from HBM, leaving it L2-resident for K1b.
//   K1b psi: fully parallel over (frame, pair, bin pair): two bins per
//       thread, 16-byte loads of y_m and y_m' and a 16-byte store of psi.
// Algorithmic traffic: 8 (M + P) Kb bytes per frame.
#include "common.cuh"

#include <cuda_fp16.h>

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

cudaError_t launch_gcc_phat(const float* Y, int F, int M, int Kb, const int32_t* pm,
                            const int32_t* pmp, int P, int weighting, double floor_rel,
                            double abs_floor, float* Psi, double* floor_out,
                            cudaStream_t stream, void* Psi_hi, void* Psi_lo, float split_scale) {
  if (F == 0) return cudaSuccess;
  // relative floor: per-frame values from K1a (into floor_out, or into a
  // stream-ordered scratch when the caller passed none); explicit floor and
  // identity weighting: one constant
  const bool per_frame = weighting == 0 && !(abs_floor > 0.0);
  const double const_floor = weighting == 0 ? abs_floor : 0.0;
  double* floors = nullptr;
  cudaError_t e = cudaSuccess;
  if (per_frame) {
    floors = floor_out;
    if (!floors) {
      e = cudaMallocAsync(reinterpret_cast<void**>(&floors), sizeof(double) * F, stream);
      if (e != cudaSuccess) return e;
    }
    gcc_floor_kernel<<<F, kFloorThreads, 0, stream>>>(reinterpret_cast<const float2*>(Y), M, Kb,
                                                       pm, pmp, P, floor_rel, floors, nullptr);
  } else if (floor_out) {
    fill_kernel<<<(F + 255) / 256, 256, 0, stream>>>(floor_out, F, const_floor);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const bool vec = Kb % 2 == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(Psi) & 15) == 0 &&
                   ((reinterpret_cast<uintptr_t>(Psi_hi) | reinterpret_cast<uintptr_t>(Psi_lo)) & 7) == 0;
  const int rows = F * P;
  if (Psi_hi != nullptr && !vec) return cudaErrorInvalidValue;  // split needs the 2-bin path
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
