// K4: sinc-interpolation maps (the paper's reconstruction step) and the
// sinc weight table.
//
// Restates srp.precompute_sinc_table (pkg/src/srpfast/srp.py:287-317) with
// the node snapping of srp._sinc_kernel (:250-261), and srp.srp_approx
// (:320-347):   SRP[f, j] = sum_p sum_n W_p[j, n] xi_p[f, n]
// as one GEMM over the concatenated lattice axis: maps = Xi W^T.
//
// With x = tau/T = i + f (host fp64 split, |f| <= 1/2) and d = i - n:
//   sinc(x - n) = (-1)^d sin(pi f) / (pi (d + f)),   exactly [d == 0] if f == 0
// which needs one sinpi per (candidate, pair) and one division per tap.
//
// Roofline: HBM (W streamed, 4 J T_pad bytes per batch) at small F; FP32 pipe
// (2 T_pad flops per frame.candidate) at large F.
#include "simt_gemm.cuh"

namespace srpb {

__device__ __forceinline__ float sinc_split(int i, float fr, float sin_pi_f, int n) {
  const int d = i - n;
  if (sinc_is_node(fr)) return d == 0 ? 1.0f : 0.0f;
  const float num = (d & 1) ? -sin_pi_f : sin_pi_f;
  return num / (3.14159265358979323846f * (static_cast<float>(d) + fr));
}

// Pair owning lattice column t (off[] ascending, off[P] = sum of T_p).
__device__ __forceinline__ int pair_of(const int32_t* s_off, int P, int t, int hint) {
  int p = hint;
  while (p + 1 <= P && s_off[p + 1] <= t) ++p;
  return p;
}

__global__ void sinc_table_kernel(const int32_t* __restrict__ sx_i, const float* __restrict__ sx_f,
                                  int J, int P, const int32_t* __restrict__ off,
                                  const int32_t* __restrict__ reach, int T_pad,
                                  float* __restrict__ W) {
  const int j = blockIdx.x;
  float* row = W + static_cast<size_t>(j) * T_pad;
  for (int p = 0; p < P; ++p) {
    const int R = reach[p], base = off[p];
    const int i = sx_i[static_cast<size_t>(p) * J + j];
    const float fr = sx_f[static_cast<size_t>(p) * J + j];
    const float spi = sinc_spi(fr);
    const int end = off[p + 1];
    for (int ni = threadIdx.x; ni < 2 * R + 1; ni += blockDim.x) {
      // the on-the-fly tensor-core generator takes the two reciprocals of an
      // (even, odd) column pair from one (sinc_pair_rcp) wherever the pair's
      // 16-column slab lies inside this pair's columns; the table follows
      // it so both kernels see the same weights bit for bit
      const int t = base + ni;
      const int s0 = t & ~15;
      if (!sinc_is_node(fr) && s0 >= base && s0 + 16 <= end) {
        const int te = t & ~1;
        const float xe = static_cast<float>(i - (te - base - R)) + fr;
        const float xo = static_cast<float>(i - (te + 1 - base - R)) + fr;
        const float r = sinc_pair_rcp(xe, xo, t & 1);
        const int d = i - (ni - R);
        row[t] = __uint_as_float(__float_as_uint(spi * r) ^ (static_cast<uint32_t>(d & 1) << 31));
      } else {
        row[t] = sinc_weight_fast(i, fr, spi, ni - R);
      }
    }
  }
  for (int t = off[P] + threadIdx.x; t < T_pad; t += blockDim.x) row[t] = 0.0f;
}

template <bool kOnTheFly>
__global__ void __launch_bounds__(kGemmThreads)
interp_simt_kernel(const float* __restrict__ W, const int32_t* __restrict__ sx_i,
                   const float* __restrict__ sx_f, int P, const int32_t* __restrict__ off,
                   const int32_t* __restrict__ reach, const float* __restrict__ Xi, int F, int J,
                   int T_pad, float* __restrict__ maps, unsigned long long* __restrict__ keys) {
  __shared__ __align__(16) SimtTiles s;
  extern __shared__ int32_t s_dyn[];  // on-the-fly: off[0..P], reach[0..P)
  const int tid = threadIdx.x;
  const int j0 = blockIdx.x * kTileJ;
  const int f0 = blockIdx.y * kTileF;
  const int tj = tid & 15, tf = tid >> 4;

  int32_t* s_off = s_dyn;
  int32_t* s_reach = s_dyn + P + 1;
  if (kOnTheFly) {
    for (int e = tid; e <= P; e += blockDim.x) s_off[e] = off[e];
    for (int e = tid; e < P; e += blockDim.x) s_reach[e] = reach[e];
    __syncthreads();
  }
  // on-the-fly generator role: candidate jg, columns [half*16, half*16+16)
  const int jg_local = tid & (kTileJ - 1);
  const int jg = j0 + jg_local;
  const int half = tid >> 7;
  int cur_p = -1, gi = 0, hint = 0;
  float gf = 0.0f, gsp = 0.0f;

  float acc[8][4];
  double tot[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      acc[a][c] = 0.0f;
      tot[a][c] = 0.0;
    }

  for (int t0 = 0; t0 < T_pad; t0 += kTileK) {
    if (kOnTheFly) {
      const int total = s_off[P];
#pragma unroll 4
      for (int b = 0; b < 16; ++b) {
        const int kl = half * 16 + b;
        const int t = t0 + kl;
        float w = 0.0f;
        if (t < total && jg < J) {
          hint = pair_of(s_off, P, t, hint);
          if (hint != cur_p) {
            cur_p = hint;
            gi = sx_i[static_cast<size_t>(cur_p) * J + jg];
            gf = sx_f[static_cast<size_t>(cur_p) * J + jg];
            gsp = sinpif(gf);
          }
          w = sinc_split(gi, gf, gsp, t - s_off[cur_p] - s_reach[cur_p]);
        }
        s.A[kl][jg_local] = w;
      }
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int e = tid + r * kGemmThreads;
        const int jl = e & (kTileJ - 1), t4 = e >> 7;
        const int j = j0 + jl;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < J) v = *reinterpret_cast<const float4*>(W + static_cast<size_t>(j) * T_pad + t0 + t4 * 4);
        s.A[t4 * 4 + 0][jl] = v.x;
        s.A[t4 * 4 + 1][jl] = v.y;
        s.A[t4 * 4 + 2][jl] = v.z;
        s.A[t4 * 4 + 3][jl] = v.w;
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int e = tid + r * kGemmThreads;
      const int fl = e & (kTileF - 1), t4 = e >> 6;
      const int f = f0 + fl;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (f < F) v = *reinterpret_cast<const float4*>(Xi + static_cast<size_t>(f) * T_pad + t0 + t4 * 4);
      s.B[t4 * 4 + 0][fl] = v.x;
      s.B[t4 * 4 + 1][fl] = v.y;
      s.B[t4 * 4 + 2][fl] = v.z;
      s.B[t4 * 4 + 3][fl] = v.w;
    }
    __syncthreads();
    simt_mma_chunk(s, tj, tf, acc);
    __syncthreads();
    if (((t0 / kTileK) & 15) == 15) simt_fold(acc, tot);  // every 512 columns
  }
  simt_fold(acc, tot);
  simt_epilogue(tot, 1.0, j0, f0, J, F, tj, tf, maps, keys);
}

cudaError_t launch_sinc_table(const int32_t* sx_i, const float* sx_f, int J, int P,
                              const int32_t* off, const int32_t* reach, int T_pad, float* W,
                              cudaStream_t stream) {
  if (J == 0) return cudaSuccess;
  sinc_table_kernel<<<J, 128, 0, stream>>>(sx_i, sx_f, J, P, off, reach, T_pad, W);
  return cudaGetLastError();
}

cudaError_t launch_interp(const float* W, const float* Xi, int F, int J, int T_pad, float* maps,
                          unsigned long long* keys, cudaStream_t stream) {
  if (F == 0 || J == 0) return cudaSuccess;
  dim3 grid((J + kTileJ - 1) / kTileJ, (F + kTileF - 1) / kTileF);
  interp_simt_kernel<false><<<grid, kGemmThreads, 0, stream>>>(
      W, nullptr, nullptr, 0, nullptr, nullptr, Xi, F, J, T_pad, maps, keys);
  return cudaGetLastError();
}

cudaError_t launch_interp_onthefly(const int32_t* sx_i, const float* sx_f, int P,
                                   const int32_t* off, const int32_t* reach, const float* Xi,
                                   int F, int J, int T_pad, float* maps,
                                   unsigned long long* keys, cudaStream_t stream) {
  if (F == 0 || J == 0) return cudaSuccess;
  dim3 grid((J + kTileJ - 1) / kTileJ, (F + kTileF - 1) / kTileF);
  const size_t smem = sizeof(int32_t) * (2 * P + 1);
  if (smem > 48 * 1024) {
    cudaError_t e = allow_dynamic_smem(interp_simt_kernel<true>, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  interp_simt_kernel<true><<<grid, kGemmThreads, smem, stream>>>(
      nullptr, sx_i, sx_f, P, off, reach, Xi, F, J, T_pad, maps, keys);
  return cudaGetLastError();
}

}  // namespace srpb
