// Device-side cross-checks: the two tools the
// reference uses to judge its fast paths, run on the GPU so they reach full
// C2-C5 scale where the CPU restatement only covers subsets.
//
// 1. srp_quadform: the quadratic-form SRP map of srp.srp_oracle
//    (pkg/src/srpfast/srp.py:468-515) in fp64,
//      SRP(j) = sum_k [h_j(k)^H Psi(k) h_j(k) - tr Psi(k)],
//      h_j(k)_m = exp(-i w_k tau_{m,0}(j)),
//    evaluated from pair rows (the pair form of :432-442: Psi_{m,m'} = psi_p,
//    Psi_{m',m} = conj psi_p, zero diagonal, so the trace term vanishes):
//      SRP(j) = sum_k sum_p 2 Re(psi_p(k) conj(h_m) h_m').
//    Unlike K2 it steers per microphone (relative delays tau_{m,0}, the first
//    M-1 canonical columns, :495-498) and evaluates every exponential
//    directly with fp64 sincos -- no phase recurrence, no tensor cores -- so
//    it checks K2's algebra and its fp32/3xFP16 arithmetic independently.
//    Thread per candidate, up to four frames per CTA sharing the steering
//    vectors; psi chunks staged in shared memory (broadcast reads).
//    FP64-pipe bound: (sincos M + 4 P + 2 P F) DP ops per (candidate, bin).
//
// 2. map_error: per-frame error energy of metrics.approximation_error_db
//    (pkg/src/srpfast/metrics.py:22-41): num = sum (ref - app)^2,
//    den = sum ref^2, accumulated in fp64 in a fixed order (deterministic),
//    fp32 or fp64 maps on either side.  HBM-bound: (4|8) + (4|8) bytes per
//    frame-candidate.
#include "common.cuh"

namespace srpb {

constexpr int kQfThreads = 128;
constexpr int kQfMaxMics = 64;
constexpr int kQfSmem = 40 * 1024;

template <int kFB>
__global__ void __launch_bounds__(kQfThreads)
quadform_kernel(const float2* __restrict__ psi, int F, int P, int Kb,
                const double* __restrict__ omega, const double* __restrict__ tau_rel, int J,
                int M, const int32_t* __restrict__ pm, const int32_t* __restrict__ pmp, int kc,
                double* __restrict__ maps) {
  extern __shared__ __align__(16) unsigned char qf_smem[];
  int2* s_pair = reinterpret_cast<int2*>(qf_smem);                        // [P]
  double* s_om = reinterpret_cast<double*>(s_pair + ((P + 1) & ~1));     // [kc]
  float2* s_psi = reinterpret_cast<float2*>(s_om + kc);                  // [kc][P][kFB]
  const int j = blockIdx.x * kQfThreads + threadIdx.x;
  const int f0 = blockIdx.y * kFB;
  const int nf = min(kFB, F - f0);
  for (int p = threadIdx.x; p < P; p += kQfThreads) s_pair[p] = make_int2(pm[p], pmp[p]);
  double tr[kQfMaxMics];
  const bool live = j < J;
#pragma unroll 1
  for (int m = 0; m < M; ++m) tr[m] = live ? tau_rel[static_cast<size_t>(j) * M + m] : 0.0;
  double acc[kFB];
#pragma unroll
  for (int b = 0; b < kFB; ++b) acc[b] = 0.0;
  double2 h[kQfMaxMics];
#pragma unroll 1
  for (int k0 = 0; k0 < Kb; k0 += kc) {
    const int nk = min(kc, Kb - k0);
    __syncthreads();
    for (int i = threadIdx.x; i < nk; i += kQfThreads) s_om[i] = omega[k0 + i];
    for (int i = threadIdx.x; i < nk * P * kFB; i += kQfThreads) {
      const int b = i % kFB, p = (i / kFB) % P, kk = i / (kFB * P);
      s_psi[i] = b < nf ? psi[(static_cast<size_t>(f0 + b) * P + p) * Kb + k0 + kk]
                        : make_float2(0.0f, 0.0f);
    }
    __syncthreads();
#pragma unroll 1
    for (int kk = 0; kk < nk; ++kk) {
      const double w = s_om[kk];
#pragma unroll 1
      for (int m = 0; m < M; ++m) {
        double s, c;
        sincos(tr[m] * w, &s, &c);
        h[m] = make_double2(c, -s);  // exp(-i w tau_m)
      }
      const float2* ps = s_psi + static_cast<size_t>(kk) * P * kFB;
#pragma unroll 1
      for (int p = 0; p < P; ++p) {
        const int2 mm = s_pair[p];
        const double2 a = h[mm.x], b = h[mm.y];
        // conj(h_m) h_m'
        const double zr = a.x * b.x + a.y * b.y;
        const double zi = a.x * b.y - a.y * b.x;
#pragma unroll
        for (int q = 0; q < kFB; ++q) {
          const float2 v = ps[p * kFB + q];
          acc[q] += 2.0 * (static_cast<double>(v.x) * zr - static_cast<double>(v.y) * zi);
        }
      }
    }
  }
  if (!live) return;
#pragma unroll
  for (int q = 0; q < kFB; ++q)
    if (q < nf) maps[static_cast<size_t>(f0 + q) * J + j] = acc[q];
}

template <int kFB>
static cudaError_t launch_quadform_fb(const float2* psi, int F, int P, int Kb, const double* omega,
                                      const double* tau_rel, int J, int M, const int32_t* pm,
                                      const int32_t* pmp, double* maps, cudaStream_t stream) {
  const int fixed = static_cast<int>(sizeof(int2)) * ((P + 1) & ~1);
  const int per_bin = static_cast<int>(sizeof(double) + sizeof(float2) * P * kFB);
  int kc = (kQfSmem - fixed) / per_bin;
  kc = kc < 1 ? 1 : (kc > 32 ? 32 : kc);
  const int smem = fixed + kc * per_bin;
  cudaError_t e = allow_dynamic_smem(quadform_kernel<kFB>, smem);
  if (e != cudaSuccess) return e;
  dim3 grid((J + kQfThreads - 1) / kQfThreads, (F + kFB - 1) / kFB);
  quadform_kernel<kFB><<<grid, kQfThreads, smem, stream>>>(psi, F, P, Kb, omega, tau_rel, J, M,
                                                           pm, pmp, kc, maps);
  return cudaGetLastError();
}

cudaError_t launch_quadform(const float* psi, int F, int P, int Kb, const double* omega,
                            const double* tau_rel, int J, int M, const int32_t* pm,
                            const int32_t* pmp, double* maps, cudaStream_t stream) {
  if (F == 0 || J == 0) return cudaSuccess;
  const float2* ps = reinterpret_cast<const float2*>(psi);
  // four frames share each steering evaluation; large pair sets stage one
  if (P <= 640)
    return launch_quadform_fb<4>(ps, F, P, Kb, omega, tau_rel, J, M, pm, pmp, maps, stream);
  return launch_quadform_fb<1>(ps, F, P, Kb, omega, tau_rel, J, M, pm, pmp, maps, stream);
}

// ---------------------------------------------------------------------------
// map error energy

constexpr int kErrThreads = 256;
constexpr int kMapErrorMaxChunks = 64;  // SRPB_MAP_ERROR_SCRATCH doubles per frame / 2

template <typename T>
__device__ __forceinline__ double load_map(const void* p, size_t i) {
  return static_cast<double>(__ldcs(static_cast<const T*>(p) + i));
}

template <typename TR, typename TA>
__global__ void __launch_bounds__(kErrThreads)
map_error_partial(const void* __restrict__ ref, const void* __restrict__ app, int J, int chunks,
                  double* __restrict__ part) {
  const int f = blockIdx.y, c = blockIdx.x;
  const size_t base = static_cast<size_t>(f) * J;
  double num = 0.0, den = 0.0;
  for (int j = c * kErrThreads + threadIdx.x; j < J; j += chunks * kErrThreads) {
    const double r = load_map<TR>(ref, base + j);
    const double d = r - load_map<TA>(app, base + j);
    num = fma(d, d, num);
    den = fma(r, r, den);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
  }
  __shared__ double s[2][kErrThreads / 32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s[0][w] = num;
    s[1][w] = den;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < kErrThreads / 32; ++i) {
      a += s[0][i];
      b += s[1][i];
    }
    part[(static_cast<size_t>(f) * chunks + c) * 2] = a;
    part[(static_cast<size_t>(f) * chunks + c) * 2 + 1] = b;
  }
}

__global__ void map_error_finish(const double* __restrict__ part, int F, int chunks,
                                 double* __restrict__ num, double* __restrict__ den) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  double a = 0.0, b = 0.0;
  for (int c = 0; c < chunks; ++c) {
    a += part[(static_cast<size_t>(f) * chunks + c) * 2];
    b += part[(static_cast<size_t>(f) * chunks + c) * 2 + 1];
  }
  num[f] = a;
  den[f] = b;
}

int map_error_chunks(int F, int J) {
  const int want = (2 * kNumSMs + F - 1) / (F > 0 ? F : 1);
  const int most = (J + kErrThreads * 8 - 1) / (kErrThreads * 8);
  int c = want < most ? want : most;
  c = c > kMapErrorMaxChunks ? kMapErrorMaxChunks : c;
  return c < 1 ? 1 : c;
}

cudaError_t launch_map_error(const void* ref, int ref_f64, const void* app, int app_f64, int F,
                             int J, double* scratch, double* num, double* den,
                             cudaStream_t stream) {
  if (F == 0) return cudaSuccess;
  const int chunks = map_error_chunks(F, J);
  dim3 grid(chunks, F);
  if (ref_f64 && app_f64)
    map_error_partial<double, double><<<grid, kErrThreads, 0, stream>>>(ref, app, J, chunks, scratch);
  else if (ref_f64)
    map_error_partial<double, float><<<grid, kErrThreads, 0, stream>>>(ref, app, J, chunks, scratch);
  else if (app_f64)
    map_error_partial<float, double><<<grid, kErrThreads, 0, stream>>>(ref, app, J, chunks, scratch);
  else
    map_error_partial<float, float><<<grid, kErrThreads, 0, stream>>>(ref, app, J, chunks, scratch);
  map_error_finish<<<(F + 127) / 128, 128, 0, stream>>>(scratch, F, chunks, num, den);
  return cudaGetLastError();
}

}  // namespace srpb
