// K1: GCC-PHAT cross-spectra for a batch of frames.
//
// Restates spectral.cross_spectrum (pkg/src/srpfast/spectral.py:218-285) for
// F frames at once:
//   raw    = y_m conj(y_m')                                    (:258)
//   floor  = 1e-12 * sqrt(mean_{p,k} |raw|^2) or explicit      (:268-275)
//   psi    = raw / max(|raw|, floor) where raw != 0, else 0    (:276-277)
//   identity weighting: psi = raw, floor 0                     (:259-267)
//
// HBM-bound streaming kernel: one CTA per frame reads Y[f] (M x Kb complex64)
// once from HBM (the second pass hits L1/L2) and writes Psi[f] (P x Kb)
// with coalesced 8-byte stores along k.  The floor is a per-frame reduction
// over all P*Kb products, accumulated in fp64 from per-bin channel powers
// staged in shared memory, so the applied floor matches the reference's fp64
// value to rounding.  Algorithmic traffic: 8 (M + P) Kb bytes per frame.
#include "common.cuh"

namespace srpb {

constexpr int kGccThreads = 256;
constexpr int kGccBinChunk = 64;   // bins per floor-pass chunk
constexpr int kGccMaxSmemChannels = 64;

__global__ void __launch_bounds__(kGccThreads)
gcc_phat_kernel(const float2* __restrict__ Y, int M, int Kb, const int32_t* __restrict__ pm,
                const int32_t* __restrict__ pmp, int P, int weighting, double floor_rel,
                double abs_floor, float2* __restrict__ Psi, double* __restrict__ floor_out) {
  const int f = blockIdx.x;
  const float2* y = Y + static_cast<size_t>(f) * M * Kb;
  float2* psi = Psi + static_cast<size_t>(f) * P * Kb;
  __shared__ double s_pow[kGccMaxSmemChannels][kGccBinChunk];
  __shared__ double s_red[kGccThreads / 32];
  __shared__ double s_floor;

  double floor = 0.0;
  if (weighting == 0) {
    if (abs_floor > 0.0) {
      floor = abs_floor;
    } else {
      // sum_{p,k} |raw|^2 = sum_k sum_p |y_m|^2 |y_m'|^2  (fp64)
      double acc = 0.0;
      for (int k0 = 0; k0 < Kb; k0 += kGccBinChunk) {
        const int kc = min(kGccBinChunk, Kb - k0);
        for (int e = threadIdx.x; e < M * kGccBinChunk; e += blockDim.x) {
          const int m = e / kGccBinChunk, kk = e % kGccBinChunk;
          double pw = 0.0;
          if (kk < kc) {
            const float2 v = y[static_cast<size_t>(m) * Kb + k0 + kk];
            pw = static_cast<double>(v.x) * v.x + static_cast<double>(v.y) * v.y;
          }
          s_pow[m][kk] = pw;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < P * kGccBinChunk; e += blockDim.x) {
          const int p = e / kGccBinChunk, kk = e % kGccBinChunk;
          acc += s_pow[pm[p]][kk] * s_pow[pmp[p]][kk];
        }
        __syncthreads();
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kGccThreads / 32; ++w) t += s_red[w];
        s_floor = floor_rel * sqrt(t / (static_cast<double>(P) * Kb));
      }
      __syncthreads();
      floor = s_floor;
    }
  }
  if (threadIdx.x == 0 && floor_out != nullptr) floor_out[f] = floor;

  for (int p = 0; p < P; ++p) {
   const float2* ya = y + static_cast<size_t>(pm[p]) * Kb;
   const float2* yb = y + static_cast<size_t>(pmp[p]) * Kb;
   for (int k = threadIdx.x; k < Kb; k += blockDim.x) {
    const float2 a = ya[k];
    const float2 b = yb[k];
    float2 out;
    if (weighting != 0) {  // identity: raw product, correctly rounded from fp64
      const double re = static_cast<double>(a.x) * b.x + static_cast<double>(a.y) * b.y;
      const double im = static_cast<double>(a.y) * b.x - static_cast<double>(a.x) * b.y;
      out = make_float2(static_cast<float>(re), static_cast<float>(im));
    } else if ((a.x == 0.0f && a.y == 0.0f) || (b.x == 0.0f && b.y == 0.0f)) {
      out = make_float2(0.0f, 0.0f);  // exact-zero product stays zero
    } else {
      const float ma = hypotf(a.x, a.y), mb = hypotf(b.x, b.y);
      const double mag = static_cast<double>(ma) * mb;
      if (mag >= floor) {
        // raw/|raw| = (a/|a|) conj(b/|b|): unit modulus, no over/underflow
        const float ua = 1.0f / ma, ub = 1.0f / mb;
        const float ax = a.x * ua, ay = a.y * ua, bx = b.x * ub, by = b.y * ub;
        out = make_float2(ax * bx + ay * by, ay * bx - ax * by);
      } else {
        const double re = static_cast<double>(a.x) * b.x + static_cast<double>(a.y) * b.y;
        const double im = static_cast<double>(a.y) * b.x - static_cast<double>(a.x) * b.y;
        out = make_float2(static_cast<float>(re / floor), static_cast<float>(im / floor));
      }
    }
    psi[static_cast<size_t>(p) * Kb + k] = out;
   }
  }
}

cudaError_t launch_gcc_phat(const float* Y, int F, int M, int Kb, const int32_t* pm,
                            const int32_t* pmp, int P, int weighting, double floor_rel,
                            double abs_floor, float* Psi, double* floor_out,
                            cudaStream_t stream) {
  if (F == 0) return cudaSuccess;
  gcc_phat_kernel<<<F, kGccThreads, 0, stream>>>(
      reinterpret_cast<const float2*>(Y), M, Kb, pm, pmp, P, weighting, floor_rel, abs_floor,
      reinterpret_cast<float2*>(Psi), floor_out);
  return cudaGetLastError();
}

}  // namespace srpb
