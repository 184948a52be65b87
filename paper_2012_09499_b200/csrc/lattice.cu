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
#include "umma.cuh"

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

// Register-tiled SIMT GEMM per pair: Xi_p[f, n] = 2 Re sum_k psi[f,p,k] tw[n,k].
// CTA = (pair p, 64 frames, 32 lags); 128 threads, each owning 4 consecutive
// frames x 4 lags (n = ng + 8 i) in 16 fp32 accumulators.  Bins stream through
// double-buffered shared memory in chunks of 32: s_psi[k][f] (row stride 66
// complex -> 16-byte aligned LDS.128 of 2 frames) and s_tw[k][n] (odd row
// stride 33 -> conflict-free transposed staging, 8 consecutive lags per
// LDS.64 wavefront).  Per bin a thread issues 2 LDS.128 + 4 LDS.64 for 32 FFMA.
// kFromY: psi is generated in the staging pass from the channel spectra Y and
// the per-frame floors (K1's psi pass fused in: the cross-spectra never
// round-trip through HBM); otherwise it is read from Psi.
constexpr int kLatF = 64;      // frames per CTA
constexpr int kLatN = 32;      // lags per CTA
constexpr int kLatK = 32;      // bins per shared-memory chunk
constexpr int kLatThreads = 128;
constexpr int kLatPsiStride = kLatF + 2;
constexpr int kLatTwStride = kLatN + 1;
constexpr int kLatPsiPerThread = kLatF * kLatK / kLatThreads;  // 16
constexpr int kLatTwPerThread = kLatN * kLatK / kLatThreads;   // 8

struct LatticeArgs {
  const float2* src;  // Psi [F, P, Kb] or Y [F, M, Kb]
  int F, P, Kb, M;
  const int32_t* pm;
  const int32_t* pmp;
  int weighting;
  const double* floors;  // per-frame floor (kFromY) or NULL -> const_floor
  double const_floor;
  const float2* tw;
  int L;
  const int32_t* off;
  const int32_t* reach;
  int T_pad;
  float* Xi;     // [F, T_pad] or NULL
  float* Xi_hi;  // optional tf32 split of Xi for the tensor-core K4 (or NULL)
  float* Xi_lo;
};

__device__ __forceinline__ void lattice_store(const LatticeArgs& a, size_t idx, float v) {
  if (a.Xi) a.Xi[idx] = v;
  if (a.Xi_hi) {
    const float h = umma::to_tf32(v);
    a.Xi_hi[idx] = h;
    a.Xi_lo[idx] = umma::to_tf32(v - h);
  }
}

template <bool kFromY>
__global__ void __launch_bounds__(kLatThreads)
lattice_kernel(const LatticeArgs a) {
  const int p = blockIdx.x;
  const int f0 = blockIdx.y * kLatF;
  const int tid = threadIdx.x;
  if (p == a.P) {  // pad-column zero fill for this frame tile
    const int t0 = __ldg(a.off + a.P);
    const int w = a.T_pad - t0;
    if (blockIdx.z != 0 || w <= 0) return;
    for (int e = tid; e < kLatF * w; e += blockDim.x) {
      const int fl = e / w, t = t0 + e - fl * w;
      if (f0 + fl < a.F) lattice_store(a, static_cast<size_t>(f0 + fl) * a.T_pad + t, 0.0f);
    }
    return;
  }
  const int R = __ldg(a.reach + p);
  const int Tp = 2 * R + 1;
  const int n_base = blockIdx.z * kLatN;  // local lag index (0 = lag -R)
  if (n_base >= Tp) return;

  extern __shared__ __align__(16) float2 s_lat[];
  auto s_psi = reinterpret_cast<float2(*)[kLatK][kLatPsiStride]>(s_lat);
  auto s_tw = reinterpret_cast<float2(*)[kLatK][kLatTwStride]>(s_lat + 2 * kLatK * kLatPsiStride);

  // staging roles: psi item j -> (k = tid%8 + 8 (j%4), f = tid/8 + 16 (j/4)):
  // per warp 4 frames x 8 consecutive bins per load; tw item j -> (k = tid%32,
  // n = tid/32 + 4 j): one 256-byte row segment per warp
  const int sk = tid & 7, sf = tid >> 3;
  const int tk = tid & 31, tn = tid >> 5;
  const float2* rowA[4];
  const float2* rowB[4];
  double fl[4];
  bool fvalid[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int f = f0 + sf + 16 * q;
    fvalid[q] = f < a.F;
    const int fc = fvalid[q] ? f : 0;
    if constexpr (kFromY) {
      const float2* y = a.src + static_cast<size_t>(fc) * a.M * a.Kb;
      rowA[q] = y + static_cast<size_t>(__ldg(a.pm + p)) * a.Kb;
      rowB[q] = y + static_cast<size_t>(__ldg(a.pmp + p)) * a.Kb;
      fl[q] = a.floors ? __ldg(a.floors + fc) : a.const_floor;
    } else {
      rowA[q] = a.src + (static_cast<size_t>(fc) * a.P + p) * a.Kb;
      rowB[q] = nullptr;
      fl[q] = 0.0;
    }
  }
  const float2* twrow[kLatTwPerThread];
  bool nvalid[kLatTwPerThread];
#pragma unroll
  for (int j = 0; j < kLatTwPerThread; ++j) {
    const int ni = n_base + tn + 4 * j;
    nvalid[j] = ni < Tp;
    twrow[j] = a.tw + static_cast<size_t>(a.L - R + (nvalid[j] ? ni : 0)) * a.Kb;
  }

  float2 ra[kLatPsiPerThread], rb[kFromY ? kLatPsiPerThread : 1];
  float2 rt[kLatTwPerThread];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int j = 0; j < kLatPsiPerThread; ++j) {
      const int k = k0 + sk + 8 * (j & 3);
      const int q = j >> 2;
      const bool ok = fvalid[q] && k < a.Kb;
      ra[j] = ok ? __ldg(rowA[q] + k) : make_float2(0.0f, 0.0f);
      if constexpr (kFromY) rb[j] = ok ? __ldg(rowB[q] + k) : make_float2(0.0f, 0.0f);
    }
#pragma unroll
    for (int j = 0; j < kLatTwPerThread; ++j) {
      const int k = k0 + tk;
      rt[j] = (nvalid[j] && k < a.Kb) ? __ldg(twrow[j] + k) : make_float2(0.0f, 0.0f);
    }
  };
  auto stage = [&](int buf) {
#pragma unroll
    for (int j = 0; j < kLatPsiPerThread; ++j) {
      float2 v = ra[j];
      if constexpr (kFromY) v = phat_one(ra[j], rb[j], a.weighting, fl[j >> 2]);
      s_psi[buf][sk + 8 * (j & 3)][sf + 16 * (j >> 2)] = v;
    }
#pragma unroll
    for (int j = 0; j < kLatTwPerThread; ++j) s_tw[buf][tk][tn + 4 * j] = rt[j];
  };

  // compute roles: frames 4 fg .. 4 fg + 3, lags ng + 8 i
  const int ng = tid & 7, fg = tid >> 3;
  float acc[4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y] = 0.0f;

  const int n_chunks = (a.Kb + kLatK - 1) / kLatK;
  fetch(0);
  stage(0);
  __syncthreads();
  for (int c = 0; c < n_chunks; ++c) {
    const int buf = c & 1;
    if (c + 1 < n_chunks) fetch((c + 1) * kLatK);
#pragma unroll 8
    for (int kk = 0; kk < kLatK; ++kk) {
      const float4 v01 = *reinterpret_cast<const float4*>(&s_psi[buf][kk][4 * fg]);
      const float4 v23 = *reinterpret_cast<const float4*>(&s_psi[buf][kk][4 * fg + 2]);
      const float2 v[4] = {make_float2(v01.x, v01.y), make_float2(v01.z, v01.w),
                           make_float2(v23.x, v23.y), make_float2(v23.z, v23.w)};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 t = s_tw[buf][kk][ng + 8 * i];
#pragma unroll
        for (int x = 0; x < 4; ++x) acc[x][i] = fmaf(v[x].x, t.x, fmaf(-v[x].y, t.y, acc[x][i]));
      }
    }
    if (c + 1 < n_chunks) stage(buf ^ 1);
    __syncthreads();
  }
  const int col0 = __ldg(a.off + p) + n_base;
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int f = f0 + 4 * fg + x;
    if (f >= a.F) continue;
    const size_t row = static_cast<size_t>(f) * a.T_pad + col0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (n_base + ng + 8 * i < Tp) lattice_store(a, row + ng + 8 * i, 2.0f * acc[x][i]);
  }
}

cudaError_t launch_lattice_twiddles(const double* omega, int Kb, double T, int L, float* tw,
                                    cudaStream_t stream) {
  dim3 grid((Kb + 255) / 256, 2 * L + 1);
  lattice_twiddle_kernel<<<grid, 256, 0, stream>>>(omega, Kb, T, L, reinterpret_cast<float2*>(tw));
  return cudaGetLastError();
}

static cudaError_t launch_lattice_args(const LatticeArgs& a, bool from_y, int max_Tp,
                                      cudaStream_t stream) {
  constexpr int smem = static_cast<int>(sizeof(float2)) * 2 * kLatK * (kLatPsiStride + kLatTwStride);
  // per launch: the attribute is per device, and setting it is cheap
  cudaError_t e = from_y ? cudaFuncSetAttribute(lattice_kernel<true>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem)
                         : cudaFuncSetAttribute(lattice_kernel<false>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  dim3 grid(a.P + 1, (a.F + kLatF - 1) / kLatF, (max_Tp + kLatN - 1) / kLatN);
  if (from_y)
    lattice_kernel<true><<<grid, kLatThreads, smem, stream>>>(a);
  else
    lattice_kernel<false><<<grid, kLatThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_lattice(const float* Psi, int F, int P, int Kb, const float* tw, int L,
                           const int32_t* off, const int32_t* reach, int max_Tp, int T_pad,
                           float* Xi, cudaStream_t stream) {
  if (F == 0) return cudaSuccess;
  LatticeArgs a{reinterpret_cast<const float2*>(Psi), F, P, Kb, 0, nullptr, nullptr, 1,
                nullptr, 0.0, reinterpret_cast<const float2*>(tw), L, off, reach, T_pad, Xi,
                nullptr, nullptr};
  return launch_lattice_args(a, false, max_Tp, stream);
}

cudaError_t launch_lattice_from_spectra(const float* Y, int F, int M, int Kb, const int32_t* pm,
                                        const int32_t* pmp, int P, int weighting,
                                        const double* floors, double abs_floor, const float* tw,
                                        int L, const int32_t* off, const int32_t* reach,
                                        int max_Tp, int T_pad, float* Xi, float* Xi_hi,
                                        float* Xi_lo, cudaStream_t stream) {
  if (F == 0) return cudaSuccess;
  LatticeArgs a{reinterpret_cast<const float2*>(Y), F, P, Kb, M, pm, pmp, weighting,
                weighting == 0 ? floors : nullptr, weighting == 0 ? abs_floor : 0.0,
                reinterpret_cast<const float2*>(tw), L, off, reach, T_pad, Xi, Xi_hi, Xi_lo};
  return launch_lattice_args(a, true, max_Tp, stream);
}

}  // namespace srpb
