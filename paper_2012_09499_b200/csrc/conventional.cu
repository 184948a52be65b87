// K2: conventional SRP maps with on-the-fly steering phases.
//
// Restates srp.srp_conventional_frames (pkg/src/srpfast/srp.py:391-429):
//   SRP[f, j] = sum_p 2 Re( e^{j w_k tau[j,p]} . psi[f, p, :] )      (:420-422)
// as one contraction over (pair, bin, re/im):
//   A[j, (p,k,0)] = cos(theta_jpk), A[j, (p,k,1)] = -sin(theta_jpk)
//   B[(p,k,c), f] = Psi[f, p, k].{re, im}   (the float view of Psi [F, P, Kb])
//   maps = 2 * A B
// The phase matrix (srp._phase_matrix, srp.py:350-373; a J x Kb complex128
// table per pair in the reference, 491 GB fp32 at C3 for all pairs) is never
// stored: every CTA generates its 128 x 16-bin A tile in shared memory and
// reuses it across its 64 frames.
//
// Harmonic bins (w_k = k w_1): theta/2pi = k (i + f) / N with the integer
// part reduced exactly (common.cuh).  Non-harmonic bins (the dense-exp branch,
// srp.py:366-367): theta = w_k tau in fp64, reduced, then fp32 sincos.
//
// Roofline: FP32 pipe, 4 P Kb flops per frame.candidate.
#include "simt_gemm.cuh"

namespace srpb {

constexpr int kBinsPerChunk = kTileK / 2;  // 16 bins -> 32 real K rows

template <bool kHarmonic>
__global__ void __launch_bounds__(kGemmThreads)
conventional_simt_kernel(const float* __restrict__ Psi, int F, int P, int Kb, int period,
                         int mask, const int32_t* __restrict__ tau_i,
                         const float* __restrict__ tau_f, const double* __restrict__ omega,
                         const double* __restrict__ tau, int J, float* __restrict__ maps,
                         unsigned long long* __restrict__ keys) {
  __shared__ __align__(16) SimtTiles s;
  const int tid = threadIdx.x;
  const int j0 = blockIdx.x * kTileJ;
  const int f0 = blockIdx.y * kTileF;
  const int tj = tid & 15, tf = tid >> 4;
  const float inv_period = 1.0f / static_cast<float>(period);

  // A-generation role: candidate jg, bins [half*8, half*8 + 8) of each chunk
  const int jg_local = tid & (kTileJ - 1);
  const int jg = j0 + jg_local;
  const int half = tid >> 7;
  // B-load role: frame fl, bins [q*4, q*4 + 4) of each chunk
  const int fl = tid & (kTileF - 1);
  const int q = tid >> 6;
  const size_t row_stride = static_cast<size_t>(P) * Kb * 2;  // floats per frame

  float acc[8][4];
  double tot[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      acc[a][c] = 0.0f;
      tot[a][c] = 0.0;
    }

  for (int p = 0; p < P; ++p) {
    int ti = 0;
    float tfr = 0.0f;
    double tau_jp = 0.0;
    if (jg < J) {
      if (kHarmonic) {
        ti = tau_i[static_cast<size_t>(p) * J + jg];
        tfr = tau_f[static_cast<size_t>(p) * J + jg];
      } else {
        tau_jp = tau[static_cast<size_t>(jg) * P + p];
      }
    }
    for (int k0 = 0; k0 < Kb; k0 += kBinsPerChunk) {
      // ---- A tile: steering phases of 128 candidates x 16 bins
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const int kl = half * 8 + b;
        const int k = k0 + kl;
        float c = 0.0f, sn = 0.0f;
        if (k < Kb) {
          if (kHarmonic) {
            harmonic_phase(k, ti, tfr, period, mask, inv_period, &c, &sn);
          } else {
            const double th = omega[k] * tau_jp;
            double sd, cd;
            sincos(th, &sd, &cd);
            c = static_cast<float>(cd);
            sn = static_cast<float>(sd);
          }
        }
        s.A[2 * kl][jg_local] = c;
        s.A[2 * kl + 1][jg_local] = -sn;
      }
      // ---- B tile: Psi[f, p, k0 .. k0+16) as 32 real rows
      {
        const int f = f0 + fl;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int kl = q * 4 + b;
          const int k = k0 + kl;
          float2 v = make_float2(0.0f, 0.0f);
          if (f < F && k < Kb)
            v = *reinterpret_cast<const float2*>(Psi + static_cast<size_t>(f) * row_stride +
                                                 (static_cast<size_t>(p) * Kb + k) * 2);
          s.B[2 * kl][fl] = v.x;
          s.B[2 * kl + 1][fl] = v.y;
        }
      }
      __syncthreads();
      simt_mma_chunk(s, tj, tf, acc);
      __syncthreads();
    }
    simt_fold(acc, tot);  // one pair done: fold into fp64
  }
  simt_epilogue(tot, 2.0, j0, f0, J, F, tj, tf, maps, keys);
}

// Few-frame batches (C5 batch 1, real-time localisation): the GEMM form
// wastes the tile's frame columns and every steering phase is generated for
// a single frame, so each thread takes one candidate and walks the bins of
// every pair with the phase recurrence -- exact anchor (integer-reduced
// turns + sincospif) every 16 bins, one-bin rotations in between (chain <=
// 15 rotations, as the tensor-core generator) -- accumulating
// 2 Re(e^{j w_k tau} psi_k) for its kF frames straight from the block's
// shared copy of the pair's cross-spectra (broadcast reads).  fp32 per pair,
// folded into fp64 (the reference's per-pair acc += order, srp.py:420-422).
constexpr int kFewThreads = 128;
constexpr int kFewMaxFrames = 4;

constexpr int kFewCands = 4;  // candidates per thread (share the spectra reads)

template <int kF>
__global__ void __launch_bounds__(kFewThreads)
conventional_few_kernel(const float2* __restrict__ Psi, int F, int P, int Kb, int period, int mask,
                        const int32_t* __restrict__ tau_i, const float* __restrict__ tau_f, int J,
                        float* __restrict__ maps, unsigned long long* __restrict__ keys) {
  extern __shared__ float2 s_psi[];  // [Kb][kF] of the current pair
  __shared__ unsigned long long s_key[kFewThreads / 32][kF];
  // candidates j0 + kFewThreads * c of this thread (coalesced per c)
  const int j0 = blockIdx.x * (kFewThreads * kFewCands) + threadIdx.x;
  const float inv_period = 1.0f / static_cast<float>(period);
  double tot[kFewCands][kF];
#pragma unroll
  for (int c = 0; c < kFewCands; ++c)
#pragma unroll
    for (int f = 0; f < kF; ++f) tot[c][f] = 0.0;
  for (int p = 0; p < P; ++p) {
    __syncthreads();  // the previous pair's spectra are consumed
    for (int e = threadIdx.x; e < Kb * kF; e += kFewThreads) {
      const int k = e / kF, f = e - (e / kF) * kF;
      s_psi[e] = f < F ? Psi[(static_cast<size_t>(f) * P + p) * Kb + k] : make_float2(0.0f, 0.0f);
    }
    __syncthreads();
    int ti[kFewCands];
    float tf[kFewCands], c1[kFewCands], s1[kFewCands];
#pragma unroll
    for (int c = 0; c < kFewCands; ++c) {
      const int j = j0 + kFewThreads * c;
      ti[c] = 0;
      tf[c] = 0.0f;
      if (j < J) {
        ti[c] = __ldg(tau_i + static_cast<size_t>(p) * J + j);
        tf[c] = __ldg(tau_f + static_cast<size_t>(p) * J + j);
      }
      harmonic_phase(1, ti[c], tf[c], period, mask, inv_period, &c1[c], &s1[c]);  // one bin
    }
    float acc[kFewCands][kF];
#pragma unroll
    for (int c = 0; c < kFewCands; ++c)
#pragma unroll
      for (int f = 0; f < kF; ++f) acc[c][f] = 0.0f;
    for (int k0 = 0; k0 < Kb; k0 += 16) {
      float cs[kFewCands], sn[kFewCands];
#pragma unroll
      for (int c = 0; c < kFewCands; ++c)
        harmonic_phase(k0, ti[c], tf[c], period, mask, inv_period, &cs[c], &sn[c]);
      const int nk = min(16, Kb - k0);
#pragma unroll 4
      for (int kk = 0; kk < nk; ++kk) {
        float2 v[kF];
#pragma unroll
        for (int f = 0; f < kF; ++f) v[f] = s_psi[(k0 + kk) * kF + f];
#pragma unroll
        for (int c = 0; c < kFewCands; ++c) {
#pragma unroll
          for (int f = 0; f < kF; ++f) {
            acc[c][f] = fmaf(cs[c], v[f].x, acc[c][f]);
            acc[c][f] = fmaf(-sn[c], v[f].y, acc[c][f]);
          }
          const float cn = cs[c] * c1[c] - sn[c] * s1[c];
          sn[c] = fmaf(cs[c], s1[c], sn[c] * c1[c]);
          cs[c] = cn;
        }
      }
    }
#pragma unroll
    for (int c = 0; c < kFewCands; ++c)
#pragma unroll
      for (int f = 0; f < kF; ++f) tot[c][f] += static_cast<double>(acc[c][f]);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int f = 0; f < kF; ++f) {
    unsigned long long k = 0ull;
#pragma unroll
    for (int c = 0; c < kFewCands; ++c) {
      const int j = j0 + kFewThreads * c;
      const float v = static_cast<float>(2.0 * tot[c][f]);
      if (j < J && f < F) {
        if (maps) __stcs(maps + static_cast<size_t>(f) * J + j, v);
        k = key_max(k, make_key(v, static_cast<uint32_t>(j)));
      }
    }
    k = warp_key_max(k);
    if (lane == 0) s_key[w][f] = k;
  }
  __syncthreads();
  if (keys && threadIdx.x < kF && threadIdx.x < F) {
    unsigned long long k = 0ull;
#pragma unroll
    for (int q = 0; q < kFewThreads / 32; ++q) k = key_max(k, s_key[q][threadIdx.x]);
    if (k != 0ull) atomicMax(keys + threadIdx.x, k);
  }
}

template <int kF>
cudaError_t launch_few(const float* Psi, int F, int P, int Kb, int period, int mask,
                       const int32_t* tau_i, const float* tau_f, int J, float* maps,
                       unsigned long long* keys, cudaStream_t stream) {
  const size_t smem = sizeof(float2) * static_cast<size_t>(Kb) * kF;
  auto kern = conventional_few_kernel<kF>;
  cudaError_t e = allow_dynamic_smem(kern, smem);
  if (e != cudaSuccess) return e;
  const int per_block = kFewThreads * kFewCands;
  kern<<<(J + per_block - 1) / per_block, kFewThreads, smem, stream>>>(
      reinterpret_cast<const float2*>(Psi), F, P, Kb, period, mask, tau_i, tau_f, J, maps, keys);
  return cudaGetLastError();
}

cudaError_t launch_conventional(const float* Psi, int F, int P, int Kb, int period,
                                const int32_t* tau_i, const float* tau_f, int J, float* maps,
                                unsigned long long* keys, cudaStream_t stream) {
  if (F == 0 || J == 0) return cudaSuccess;
  const int mask = (period & (period - 1)) == 0 ? period - 1 : 0;
  if (F <= kFewMaxFrames && static_cast<size_t>(Kb) * kFewMaxFrames * sizeof(float2) <= 200 * 1024) {
    if (F == 1) return launch_few<1>(Psi, F, P, Kb, period, mask, tau_i, tau_f, J, maps, keys, stream);
    if (F == 2) return launch_few<2>(Psi, F, P, Kb, period, mask, tau_i, tau_f, J, maps, keys, stream);
    return launch_few<4>(Psi, F, P, Kb, period, mask, tau_i, tau_f, J, maps, keys, stream);
  }
  dim3 grid((J + kTileJ - 1) / kTileJ, (F + kTileF - 1) / kTileF);
  conventional_simt_kernel<true><<<grid, kGemmThreads, 0, stream>>>(
      Psi, F, P, Kb, period, mask, tau_i, tau_f, nullptr, nullptr, J, maps, keys);
  return cudaGetLastError();
}

cudaError_t launch_conventional_general(const float* Psi, int F, int P, int Kb,
                                        const double* omega, const double* tau, int J,
                                        float* maps, unsigned long long* keys,
                                        cudaStream_t stream) {
  if (F == 0 || J == 0) return cudaSuccess;
  dim3 grid((J + kTileJ - 1) / kTileJ, (F + kTileF - 1) / kTileF);
  conventional_simt_kernel<false><<<grid, kGemmThreads, 0, stream>>>(
      Psi, F, P, Kb, 1, 0, nullptr, nullptr, omega, tau, J, maps, keys);
  return cudaGetLastError();
}

}  // namespace srpb
