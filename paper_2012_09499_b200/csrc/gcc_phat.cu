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

namespace srpb {

constexpr int kFloorThreads = 256;
constexpr int kFloorBinChunk = 64;
constexpr int kGccMaxSmemChannels = 64;

__global__ void __launch_bounds__(kFloorThreads)
gcc_floor_kernel(const float2* __restrict__ Y, int M, int Kb, const int32_t* __restrict__ pm,
                 const int32_t* __restrict__ pmp, int P, double floor_rel,
                 double* __restrict__ floor_out) {
  const int f = blockIdx.x;
  const float2* y = Y + static_cast<size_t>(f) * M * Kb;
  __shared__ double s_pow[kGccMaxSmemChannels][kFloorBinChunk];
  __shared__ int s_pm[1024], s_pmp[1024];
  __shared__ double s_red[kFloorThreads / 32];
  const bool pairs_in_smem = P <= 1024;
  if (pairs_in_smem)
    for (int e = threadIdx.x; e < P; e += blockDim.x) {
      s_pm[e] = pm[e];
      s_pmp[e] = pmp[e];
    }
  double acc = 0.0;
  for (int k0 = 0; k0 < Kb; k0 += kFloorBinChunk) {
    const int kc = min(kFloorBinChunk, Kb - k0);
    for (int e = threadIdx.x; e < M * kFloorBinChunk; e += blockDim.x) {
      const int m = e / kFloorBinChunk, kk = e - m * kFloorBinChunk;
      double pw = 0.0;
      if (kk < kc) {
        const float2 v = y[static_cast<size_t>(m) * Kb + k0 + kk];
        pw = static_cast<double>(v.x) * v.x + static_cast<double>(v.y) * v.y;
      }
      s_pow[m][kk] = pw;
    }
    __syncthreads();
    // thread <-> bin (kk = lane-fast): conflict-free rows of s_pow
    for (int e = threadIdx.x; e < P * kFloorBinChunk; e += blockDim.x) {
      const int p = e / kFloorBinChunk, kk = e - p * kFloorBinChunk;
      const int a = pairs_in_smem ? s_pm[p] : pm[p];
      const int b = pairs_in_smem ? s_pmp[p] : pmp[p];
      acc += s_pow[a][kk] * s_pow[b][kk];
    }
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kFloorThreads / 32; ++w) t += s_red[w];
    floor_out[f] = floor_rel * sqrt(t / (static_cast<double>(P) * Kb));
  }
}

__global__ void fill_kernel(double* __restrict__ out, int n, double v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = v;
}

// one thread per (frame, pair, 2 bins); Kb even
__global__ void __launch_bounds__(256)
gcc_psi_kernel(const float4* __restrict__ Y, int F, int M, int Kb2, const int32_t* __restrict__ pm,
               const int32_t* __restrict__ pmp, int P, int weighting,
               const double* __restrict__ floors, double const_floor, float4* __restrict__ Psi) {
  const size_t total = static_cast<size_t>(F) * P * Kb2;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t row = e / Kb2;  // f * P + p
    const int k2 = static_cast<int>(e - row * Kb2);
    const int f = static_cast<int>(row / P), p = static_cast<int>(row - static_cast<size_t>(f) * P);
    const float4* yf = Y + static_cast<size_t>(f) * M * Kb2;
    const float4 a = __ldg(yf + static_cast<size_t>(__ldg(pm + p)) * Kb2 + k2);
    const float4 b = __ldg(yf + static_cast<size_t>(__ldg(pmp + p)) * Kb2 + k2);
    const double fl = floors ? __ldg(floors + f) : const_floor;
    const float2 o0 = phat_one(make_float2(a.x, a.y), make_float2(b.x, b.y), weighting, fl);
    const float2 o1 = phat_one(make_float2(a.z, a.w), make_float2(b.z, b.w), weighting, fl);
    Psi[e] = make_float4(o0.x, o0.y, o1.x, o1.y);
  }
}

// odd Kb or unaligned buffers: one bin per thread
__global__ void __launch_bounds__(256)
gcc_psi1_kernel(const float2* __restrict__ Y, int F, int M, int Kb, const int32_t* __restrict__ pm,
                const int32_t* __restrict__ pmp, int P, int weighting,
                const double* __restrict__ floors, double const_floor, float2* __restrict__ Psi) {
  const size_t total = static_cast<size_t>(F) * P * Kb;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t row = e / Kb;
    const int k = static_cast<int>(e - row * Kb);
    const int f = static_cast<int>(row / P), p = static_cast<int>(row - static_cast<size_t>(f) * P);
    const float2* yf = Y + static_cast<size_t>(f) * M * Kb;
    const double fl = floors ? floors[f] : const_floor;
    Psi[e] = phat_one(yf[static_cast<size_t>(pm[p]) * Kb + k], yf[static_cast<size_t>(pmp[p]) * Kb + k],
                      weighting, fl);
  }
}

cudaError_t launch_gcc_floor(const float* Y, int F, int M, int Kb, const int32_t* pm,
                             const int32_t* pmp, int P, double floor_rel, double* floor_out,
                             cudaStream_t stream) {
  if (F == 0) return cudaSuccess;
  gcc_floor_kernel<<<F, kFloorThreads, 0, stream>>>(reinterpret_cast<const float2*>(Y), M, Kb, pm,
                                                     pmp, P, floor_rel, floor_out);
  return cudaGetLastError();
}

cudaError_t launch_gcc_phat(const float* Y, int F, int M, int Kb, const int32_t* pm,
                            const int32_t* pmp, int P, int weighting, double floor_rel,
                            double abs_floor, float* Psi, double* floor_out,
                            cudaStream_t stream) {
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
                                                       pm, pmp, P, floor_rel, floors);
  } else if (floor_out) {
    fill_kernel<<<(F + 255) / 256, 256, 0, stream>>>(floor_out, F, const_floor);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const bool vec = Kb % 2 == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(Psi) & 15) == 0;
  const size_t elems = static_cast<size_t>(F) * P * (vec ? Kb / 2 : Kb);
  const int blocks = static_cast<int>(std::min<size_t>((elems + 255) / 256, 16 * kNumSMs));
  if (vec)
    gcc_psi_kernel<<<blocks, 256, 0, stream>>>(reinterpret_cast<const float4*>(Y), F, M, Kb / 2, pm,
                                               pmp, P, weighting, floors, const_floor,
                                               reinterpret_cast<float4*>(Psi));
  else
    gcc_psi1_kernel<<<blocks, 256, 0, stream>>>(reinterpret_cast<const float2*>(Y), F, M, Kb, pm,
                                                pmp, P, weighting, floors, const_floor,
                                                reinterpret_cast<float2*>(Psi));
  e = cudaGetLastError();
  if (per_frame && !floor_out) {
    const cudaError_t e2 = cudaFreeAsync(floors, stream);
    if (e == cudaSuccess) e = e2;
  }
  return e;
}

}  // namespace srpb
