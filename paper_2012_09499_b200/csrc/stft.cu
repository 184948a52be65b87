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
// (Z[k] - conj Z[H-k])/(2i).  Twiddles come from sincospif on exact
// arguments; the window is evaluated in fp64.  Power-of-two N (4 ... 8192;
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

__global__ void __launch_bounds__(kStftThreads)
stft_kernel(const float* __restrict__ x, int M, int L, int N, int hop, int window,
            float2* __restrict__ Y) {
  const int f = blockIdx.x, m = blockIdx.y;
  const int H = N >> 1;  // complex FFT length
  extern __shared__ float2 s_fft[];
  float2* a = s_fft;           // [H]
  float2* b = s_fft + H;       // [H]
  float2* tw = s_fft + 2 * H;  // [H/2]: e^{-2 pi i t / H}
  const float* xs = x + static_cast<size_t>(m) * L + static_cast<size_t>(f) * hop;
  const int tid = threadIdx.x;
  const double inv_n = 1.0 / static_cast<double>(N);
  for (int i = tid; i < H; i += kStftThreads) {
    float w0 = 1.0f, w1 = 1.0f;
    if (window == 0) {  // sqrt(0.5 - 0.5 cos(2 pi n / N)), periodic
      w0 = static_cast<float>(sqrt(0.5 - 0.5 * cospi(2.0 * (2 * i) * inv_n)));
      w1 = static_cast<float>(sqrt(0.5 - 0.5 * cospi(2.0 * (2 * i + 1) * inv_n)));
    }
    a[i] = make_float2(__ldg(xs + 2 * i) * w0, __ldg(xs + 2 * i + 1) * w1);
  }
  for (int t = tid; t < H / 2; t += kStftThreads) {
    float s, c;
    sincospif(2.0f * static_cast<float>(t) / static_cast<float>(H), &s, &c);
    tw[t] = make_float2(c, -s);
  }
  __syncthreads();
  // Stockham radix-2: stage Ns combines pairs (j, j + H/2) into (idx, idx+Ns)
  for (int ns = 1; ns < H; ns <<= 1) {
    const int tstride = H / (2 * ns);
    for (int j = tid; j < H / 2; j += kStftThreads) {
      const int k = j & (ns - 1);
      const float2 v0 = a[j];
      const float2 v1 = cmul(a[j + H / 2], tw[k * tstride]);
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
  for (int k = tid; k < H; k += kStftThreads) {
    const float2 zk = a[k];
    const float2 zc = a[(H - k) & (H - 1)];  // Z[H - k], Z[H] = Z[0]
    const float2 e = make_float2(0.5f * (zk.x + zc.x), 0.5f * (zk.y - zc.y));
    const float2 d = make_float2(zk.x - zc.x, zk.y + zc.y);  // Z[k] - conj Z[H-k]
    const float2 o = make_float2(0.5f * d.y, -0.5f * d.x);   // d / (2i)
    float s, c;
    sincospif(2.0f * static_cast<float>(k) / static_cast<float>(N), &s, &c);
    const float2 ro = cmul(o, make_float2(c, -s));
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
    cudaError_t e = cudaFuncSetAttribute(stft_dft_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    stft_dft_kernel<<<dim3(F, M), kStftThreads, smem, stream>>>(x, M, L, N, hop, window,
                                                                reinterpret_cast<float2*>(Y));
    return cudaGetLastError();
  }
  const int smem = static_cast<int>(sizeof(float2)) * (N + N / 4);  // 2H + H/2 complex
  cudaError_t e = cudaFuncSetAttribute(stft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem);
  if (e != cudaSuccess) return e;
  stft_kernel<<<dim3(F, M), kStftThreads, smem, stream>>>(x, M, L, N, hop, window,
                                                          reinterpret_cast<float2*>(Y));
  return cudaGetLastError();
}

}  // namespace srpb
