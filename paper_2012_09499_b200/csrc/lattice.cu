// K3: lattice GCC samples (the paper's critically sampled IDFT) + twiddles.
//
// Restates srp.build_gcc_lattice (pkg/src/srpfast/srp.py:201-247):
//   xi_p[n] = 2 Re sum_k psi_p[k] e^{j w_k n T},  n = -(N_p+n_aux) .. N_p+n_aux
// for all F frames and P pairs at once.  The reference rebuilds the
// (T_p x Kb) exp table of every pair for every frame (:235-236); here the
// signal-independent twiddles e^{j w_k n T} (n in [-L, L], L = max reach) are
// built once per plan in fp64 and rounded to fp32, then shared by all pairs
// and frames.  Output Xi [F, T_pad] holds the concatenated per-pair rows in
// np.concatenate order (index off[p] + n + reach[p]), the K-major B operand of
// the interpolation GEMM (K4); pad columns are zero.
//
// Roofline: FP32 pipe, 4 sum_p T_p Kb flops per frame.
#include "common.cuh"

namespace srpb {

__global__ void lattice_twiddle_kernel(const double* __restrict__ omega, int Kb, double T,
                                       int L, float2* __restrict__ tw) {
  const int row = blockIdx.y;  // lag n = row - L
  const double lag = static_cast<double>(row - L) * T;  // offsets * sample_period (:235)
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < Kb; k += gridDim.x * blockDim.x) {
    double s, c;
    sincos(lag * omega[k], &s, &c);  // exp(1j * outer(lags, omega)) (:236)
    tw[static_cast<size_t>(row) * Kb + k] = make_float2(static_cast<float>(c), static_cast<float>(s));
  }
}

constexpr int kLatF = 32;   // frames per CTA (one per lane)
constexpr int kLatN = 32;   // lags per CTA (4 per warp)
constexpr int kLatK = 32;   // bins per smem chunk
constexpr int kLatThreads = 256;

__global__ void __launch_bounds__(kLatThreads)
lattice_kernel(const float2* __restrict__ Psi, int F, int P, int Kb, const float2* __restrict__ tw,
               int L, const int32_t* __restrict__ off, const int32_t* __restrict__ reach,
               int T_pad, float* __restrict__ Xi) {
  const int p = blockIdx.x;
  const int f0 = blockIdx.y * kLatF;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (p == P) {  // pad-column zero fill for this frame tile
    const int t0 = off[P];
    if (blockIdx.z != 0) return;
    for (int e = threadIdx.x; e < kLatF * (T_pad - t0); e += blockDim.x) {
      const int fl = e / (T_pad - t0), t = t0 + e % (T_pad - t0);
      if (f0 + fl < F) Xi[static_cast<size_t>(f0 + fl) * T_pad + t] = 0.0f;
    }
    return;
  }
  const int R = reach[p];
  const int Tp = 2 * R + 1;
  const int n_base = blockIdx.z * kLatN;  // local lag index (0 = lag -R)
  if (n_base >= Tp) return;

  __shared__ float2 s_psi[kLatF][kLatK + 1];
  __shared__ float2 s_tw[kLatN][kLatK];
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  const size_t frame_stride = static_cast<size_t>(P) * Kb;

  for (int k0 = 0; k0 < Kb; k0 += kLatK) {
    for (int e = threadIdx.x; e < kLatF * kLatK; e += blockDim.x) {
      const int fl = e / kLatK, kl = e % kLatK;
      const int f = f0 + fl, k = k0 + kl;
      float2 v = make_float2(0.0f, 0.0f);
      if (f < F && k < Kb) v = Psi[f * frame_stride + static_cast<size_t>(p) * Kb + k];
      s_psi[fl][kl] = v;
    }
    for (int e = threadIdx.x; e < kLatN * kLatK; e += blockDim.x) {
      const int nl = e / kLatK, kl = e % kLatK;
      const int ni = n_base + nl, k = k0 + kl;
      float2 v = make_float2(0.0f, 0.0f);
      if (ni < Tp && k < Kb) v = tw[static_cast<size_t>(L - R + ni) * Kb + k];
      s_tw[nl][kl] = v;
    }
    __syncthreads();
#pragma unroll 8
    for (int kl = 0; kl < kLatK; ++kl) {
      const float2 v = s_psi[lane][kl];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 t = s_tw[warp + 8 * i][kl];
        acc[i] = fmaf(v.x, t.x, fmaf(-v.y, t.y, acc[i]));
      }
    }
    __syncthreads();
  }
  const int f = f0 + lane;
  if (f < F) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int ni = n_base + warp + 8 * i;
      if (ni < Tp) Xi[static_cast<size_t>(f) * T_pad + off[p] + ni] = 2.0f * acc[i];
    }
  }
}

cudaError_t launch_lattice_twiddles(const double* omega, int Kb, double T, int L, float* tw,
                                    cudaStream_t stream) {
  dim3 grid((Kb + 255) / 256, 2 * L + 1);
  lattice_twiddle_kernel<<<grid, 256, 0, stream>>>(omega, Kb, T, L, reinterpret_cast<float2*>(tw));
  return cudaGetLastError();
}

cudaError_t launch_lattice(const float* Psi, int F, int P, int Kb, const float* tw, int L,
                           const int32_t* off, const int32_t* reach, int max_Tp, int T_pad,
                           float* Xi, cudaStream_t stream) {
  if (F == 0) return cudaSuccess;
  dim3 grid(P + 1, (F + kLatF - 1) / kLatF, (max_Tp + kLatN - 1) / kLatN);
  lattice_kernel<<<grid, kLatThreads, 0, stream>>>(reinterpret_cast<const float2*>(Psi), F, P, Kb,
                                                   reinterpret_cast<const float2*>(tw), L, off,
                                                   reach, T_pad, Xi);
  return cudaGetLastError();
}

}  // namespace srpb
