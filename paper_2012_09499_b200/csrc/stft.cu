// K0: STFT frames on the device -- the producer of K1's input.
//
// Restates spectral.stft_analyze (pkg/src/srpfast/spectral.py:185-215) for
// every frame and channel at once: frame f covers samples [f hop, f hop + N),
// windowed by the periodic square-root Hann (FrameSpec.window_samples
// :85-90) or a rectangular window, real FFT, bins 0..N/2-1 (DC kept, Nyquist
// dropped, :211).
//
// CTA per (frame, channel).  The N-point real FFT is one N/2-point complex
// FFT of the packed sequence z[n] = x[2n] + i x[2n+1] -- a shared-memory
// Stockham radix-2 (natural-order output, no bit reversal) -- followed by the
// real-split post-pass X[k] = (Z[k] + conj Z[H-k])/2 + e^{-2 pi i k/N}
// (Z[k] - conj Z[H-k])/(2i), radix-4 stages (+ one radix-2 when log2 H is
// odd).  Twiddles come from sincospif on exact arguments; the periodic
// sqrt-Hann window is sin(pi n / N) (sinpif, exact argument).  Power-of-two N (4 ... 8192;
// every BASELINE config: 512, 1024, 2048) takes the FFT; any other even N
// (<= 4096) a direct DFT with exact integer phase reduction (k n mod N) over
// a shared twiddle table -- correct for every frame length the reference
// accepts, fast where it matters.
// Algorithmic traffic: 4 N (read, hop-overlapped) + 4 N (write) bytes per
// frame and channel; HBM-bound.
#include "common.cuh"

namespace srpb {

constexpr int kStftThreads = 256;

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// periodic sqrt-Hann: sqrt(0.5 - 0.5 cos(2 pi n / N)) = sin(pi n / N), n < N
__device__ __forceinline__ float sqrt_hann(int n, int N) {
  return sinpif(static_cast<float>(n) / static_cast<float>(N));
}

__global__ void __launch_bounds__(kStftThreads)
stft_kernel(const float* __restrict__ x, int M, int L, int N, int hop, int window,
            float2* __restrict__ Y) {
  const int f = blockIdx.x, m = blockIdx.y;
  const int H = N >> 1;  // complex FFT length
  extern __shared__ float2 s_fft[];
  float2* a = s_fft;           // [H]
  float2* b = s_fft + H;       // [H]
  float2* tw = s_fft + 2 * H;  // [H]: e^{-2 pi i t / H}
  const float* xs = x + static_cast<size_t>(m) * L + static_cast<size_t>(f) * hop;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(xs) & 7u) == 0);  // CTA-uniform
  for (int i = tid; i < H; i += nthr) {
    const float2 v = vec ? __ldg(reinterpret_cast<const float2*>(xs) + i)  // x[2i], x[2i+1]
                         : make_float2(__ldg(xs + 2 * i), __ldg(xs + 2 * i + 1));
    const float w0 = window == 0 ? sqrt_hann(2 * i, N) : 1.0f;
    const float w1 = window == 0 ? sqrt_hann(2 * i + 1, N) : 1.0f;
    a[i] = make_float2(v.x * w0, v.y * w1);
    float sn, cs;
    sincospif(2.0f * static_cast<float>(i) / static_cast<float>(H), &sn, &cs);
    tw[i] = make_float2(cs, -sn);
  }
  __syncthreads();
  // Stockham radix-4 stages, then one radix-2 stage when log2(H) is odd
  int ns = 1;
  for (; ns * 4 <= H; ns *= 4) {
    const int q = H / 4;
    for (int j = tid; j < q; j += nthr) {
      const int k = j & (ns - 1);
      const int t1 = k * (H / (4 * ns));  // twiddle e^{-2 pi i k r / (4 ns)} = tw[r t1]
      const float2 v0 = a[j];
      const float2 v1 = cmul(a[j + q], tw[t1]);
      const float2 v2 = cmul(a[j + 2 * q], tw[2 * t1]);
      const float2 v3 = cmul(a[j + 3 * q], tw[3 * t1]);
      const float2 u0 = make_float2(v0.x + v2.x, v0.y + v2.y);
      const float2 u1 = make_float2(v0.x - v2.x, v0.y - v2.y);
      const float2 u2 = make_float2(v1.x + v3.x, v1.y + v3.y);
      const float2 u3 = make_float2(v1.y - v3.y, v3.x - v1.x);  // -i (v1 - v3)
      const int idx = ((j - k) << 2) + k;
      b[idx] = make_float2(u0.x + u2.x, u0.y + u2.y);
      b[idx + ns] = make_float2(u1.x + u3.x, u1.y + u3.y);
      b[idx + 2 * ns] = make_float2(u0.x - u2.x, u0.y - u2.y);
      b[idx + 3 * ns] = make_float2(u1.x - u3.x, u1.y - u3.y);
    }
    __syncthreads();
    float2* t = a;
    a = b;
    b = t;
  }
  if (ns < H) {  // radix-2, ns = H / 2
    for (int j = tid; j < H / 2; j += nthr) {
      const int k = j & (ns - 1);
      const float2 v0 = a[j];
      const float2 v1 = cmul(a[j + H / 2], tw[k]);
      const int idx = ((j - k) << 1) + k;
      b[idx] = make_float2(v0.x + v1.x, v0.y + v1.y);
      b[idx + ns] = make_float2(v0.x - v1.x, v0.y - v1.y);
    }
    __syncthreads();
    float2* t = a;
    a = b;
    b = t;
  }
  // real split: X[k] = E[k] + e^{-2 pi i k / N} O[k], k = 0 .. H-1
  float2* out = Y + (static_cast<size_t>(f) * M + m) * H;
  for (int k = tid; k < H; k += nthr) {
    const float2 zk = a[k];
    const float2 zc = a[(H - k) & (H - 1)];  // Z[H - k], Z[H] = Z[0]
    const float2 e = make_float2(0.5f * (zk.x + zc.x), 0.5f * (zk.y - zc.y));
    const float2 d = make_float2(zk.x - zc.x, zk.y + zc.y);  // Z[k] - conj Z[H-k]
    const float2 o = make_float2(0.5f * d.y, -0.5f * d.x);   // d / (2i)
    float sn, cs;
    sincospif(static_cast<float>(k) / static_cast<float>(H), &sn, &cs);  // e^{-2 pi i k / N}
    const float2 ro = cmul(o, make_float2(cs, -sn));
    out[k] = make_float2(e.x + ro.x, e.y + ro.y);
  }
}

// any even N: X[k] = sum_n x[n] w[n] e^{-2 pi i (k n mod N) / N}
__global__ void __launch_bounds__(kStftThreads)
stft_dft_kernel(const float* __restrict__ x, int M, int L, int N, int hop, int window,
                float2* __restrict__ Y) {
  const int f = blockIdx.x, m = blockIdx.y;
  extern __shared__ float2 s_dft[];
  float* xs = reinterpret_cast<float*>(s_dft + N);  // windowed samples [N]
  float2* tw = s_dft;                                // e^{-2 pi i r / N} [N]
  const float* src = x + static_cast<size_t>(m) * L + static_cast<size_t>(f) * hop;
  const double inv_n = 1.0 / static_cast<double>(N);
  for (int n = threadIdx.x; n < N; n += kStftThreads) {
    const double w = window == 0 ? sqrt(0.5 - 0.5 * cospi(2.0 * n * inv_n)) : 1.0;
    xs[n] = static_cast<float>(static_cast<double>(__ldg(src + n)) * w);
    double sn, cs;
    sincospi(2.0 * n * inv_n, &sn, &cs);
    tw[n] = make_float2(static_cast<float>(cs), static_cast<float>(-sn));
  }
  __syncthreads();
  float2* out = Y + (static_cast<size_t>(f) * M + m) * (N / 2);
  for (int k = threadIdx.x; k < N / 2; k += kStftThreads) {
    float re = 0.0f, im = 0.0f;
    int r = 0;  // k n mod N
    for (int n = 0; n < N; ++n) {
      const float2 t = tw[r];
      re = fmaf(xs[n], t.x, re);
      im = fmaf(xs[n], t.y, im);
      r += k;
      if (r >= N) r -= N;
    }
    out[k] = make_float2(re, im);
  }
}

cudaError_t launch_stft(const float* x, int M, int L, int N, int hop, int window, int F, float* Y,
                        cudaStream_t stream) {
  if (F == 0) return cudaSuccess;
  if ((N & (N - 1)) != 0 || N < 4) {
    const int smem = static_cast<int>(sizeof(float2) * N + sizeof(float) * N);
    cudaError_t e = allow_dynamic_smem(stft_dft_kernel, smem);
    if (e != cudaSuccess) return e;
    stft_dft_kernel<<<dim3(F, M), kStftThreads, smem, stream>>>(x, M, L, N, hop, window,
                                                                reinterpret_cast<float2*>(Y));
    return cudaGetLastError();
  }
  const int H = N / 2;
  const int smem = static_cast<int>(sizeof(float2)) * 3 * H;  // a, b, twiddles
  cudaError_t e = allow_dynamic_smem(stft_kernel, smem);
  if (e != cudaSuccess) return e;
  // one thread per radix-4 butterfly (H/4), 32 ... 256 threads
  const int threads = H / 4 < 32 ? 32 : (H / 4 > kStftThreads ? kStftThreads : H / 4);
  stft_kernel<<<dim3(F, M), threads, smem, stream>>>(x, M, L, N, hop, window,
                                                     reinterpret_cast<float2*>(Y));
  return cudaGetLastError();
}

}  // namespace srpb
