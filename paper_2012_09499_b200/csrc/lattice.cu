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

#include <cuda_fp16.h>

namespace srpb {

__host__ __device__ constexpr int twiddle_stride(int L) { return (L + 1 + 15) / 16 * 16; }

__global__ void lattice_twiddle_kernel(const double* __restrict__ omega, int Kb, double T,
                                       int L, float2* __restrict__ tw) {
  // tw [Kb, Hs]: half-lags n = 0..L of bin k contiguous (lag -n = conj),
  // zero-padded to a multiple of 16 columns (whole 128-byte windows)
  const int Hs = twiddle_stride(L);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < Kb * Hs; e += gridDim.x * blockDim.x) {
    const int k = e / Hs, n = e - k * Hs;
    double sn = 0.0, cs = 0.0;
    if (n <= L) sincos(static_cast<double>(n) * T * omega[k], &sn, &cs);  // (:235-236)
    tw[e] = make_float2(static_cast<float>(cs), static_cast<float>(sn));
  }
}

// Half-lag SIMT GEMM per pair.  With c = cos(w_k n T), s = sin(w_k n T):
//   A[n] = sum_k Re(psi_k) c,  B[n] = sum_k Im(psi_k) s,
//   Xi[+n] = 2 (A - B),  Xi[-n] = 2 (A + B)
// so only the R+1 non-negative lags are contracted (half the FMAs of the
// direct form).  CTA = (pair p, 32 frames, up to 16 half-lags), 8 warps:
// lane = frame, warp w = K-slice (bins 32c + 4w .. 32c + 4w + 3 of every
// 32-bin chunk c), each thread accumulating A and B for its half-lags in
// registers; the 8 slices are summed in a fixed order through shared memory
// at the end (deterministic, independent of the frame batching).
//
// Staging: every warp runs its own 4-stage cp.async ring over its slice (no
// CTA barrier until the final reduction, no registers held by loads in
// flight).  Sources are read in 16-byte bin pairs and land as raw[ch][pair]
// [f] (float4 = two bins of frame f), so the compute lane of frame f reads
// two bins per conflict-free LDS.128.  kFromY: the two channel rows of Y are
// staged and psi is formed in the compute loop (GCC-PHAT of K1 fused in: one
// evaluation per (frame, pair, bin), the cross-spectra never touch HBM);
// otherwise the psi row is staged.  All variants run the same arithmetic, so
// fused and two-step results agree bitwise.
constexpr int kLatF = 32;        // frames per CTA (lane = frame)
constexpr int kLatWarps = 8;     // K-slices
constexpr int kLatThreads = 32 * kLatWarps;
constexpr int kLatBinsW = 4;     // bins per warp per stage
constexpr int kLatChunk = kLatBinsW * kLatWarps;
constexpr int kLatHl = 16;       // half-lags per CTA
constexpr int kLatStages = 4;
constexpr int kLatRow = 36;      // float4 per raw row (32 frames; 36 = 4 mod 8: conflict-free copies)
constexpr int kLatRaw = 2 * (kLatBinsW / 2) * kLatRow;  // float4: [ch][pair][f]
constexpr int kLatTwW = kLatBinsW * kLatHl / 2;          // float4: [bin][h/2]
constexpr int kLatStageW = kLatRaw + kLatTwW;            // float4 per warp stage
constexpr size_t kLatSmemBytes = sizeof(float4) * kLatWarps * kLatStages * kLatStageW;
static_assert(sizeof(float4) * kLatWarps * kLatStages * kLatStageW >=
                  sizeof(float) * kLatWarps * 2 * kLatHl * kLatF,
              "reduction buffer aliases the stages");
static_assert(kLatTwW == 32 && kLatBinsW == 4, "copy mapping: one twiddle float4 per lane");

struct LatticeArgs {
  const float2* src;  // Psi [F, P, Kb] or Y [F, M, Kb]
  int F, P, Kb, M;
  const int32_t* pm;
  const int32_t* pmp;
  int weighting;
  const double* floors;  // per-frame floor (kFromY) or NULL -> const_floor
  double const_floor;
  const int32_t* clean;  // per-frame K1a range flags (kFromY) or NULL
  const float2* tw;      // [Kb, Hs]: e^{j w_k n T}, n = 0..L, zero beyond
  int Hs;                // row stride, multiple of 16
  const int32_t* off;
  const int32_t* reach;
  int T_pad;
  float* Xi;     // [F, T_pad] or NULL
  void* Xi_hi;   // optional operand split of Xi for the tensor-core K4 (or NULL):
  void* Xi_lo;   //   split_scale == 0: tf32 hi/lo floats; else fp16 hi/lo of split_scale * Xi
  float split_scale;
  int vec16;     // 16-byte copies (Kb even, 16-byte aligned source)
};

__device__ __forceinline__ void lattice_store(const LatticeArgs& a, size_t idx, float v) {
  if (a.Xi) a.Xi[idx] = v;
  if (a.Xi_hi) {
    if (a.split_scale == 0.0f) {
      const float h = umma::to_tf32(v);
      static_cast<float*>(a.Xi_hi)[idx] = h;
      static_cast<float*>(a.Xi_lo)[idx] = umma::to_tf32(v - h);
    } else {
      const float x = v * a.split_scale;
      const __half h = __float2half_rn(x);
      static_cast<__half*>(a.Xi_hi)[idx] = h;
      static_cast<__half*>(a.Xi_lo)[idx] = __float2half_rn(x - __half2float(h));
    }
  }
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(umma::smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(umma::smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// one warp's view of the CTA: its K-slice, its ring, its copy sources
struct LatticeWarp {
  float4* ring;             // [stage][kLatStageW]
  const float2* src[2][2];  // [ch][half]: row of frame (lane/2 + 16 half), clamped
  const float2* twsrc;      // this lane's twiddle column window at bin 0
  int nch, kbase;           // channels staged; first bin of the slice in chunk 0
};

template <int kNch>
__device__ __forceinline__ void lattice_issue(const LatticeArgs& a, const LatticeWarp& w, int c,
                                              int st) {
  const int lane = threadIdx.x & 31;
  float4* base = w.ring + st * kLatStageW;
  const int k0 = c * kLatChunk + w.kbase;
  // raw: lane -> (bin pair pr = lane & 1, frame lane/2 + 16 half)
  const int pr = lane & 1;
  const int kp = min(k0 + 2 * pr, a.Kb - 1);  // first bin of the pair (clamped)
#pragma unroll
  for (int ch = 0; ch < kNch; ++ch)
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      float4* dst = base + (ch * 2 + pr) * kLatRow + (lane >> 1) + 16 * half;
      const float2* s = w.src[ch][half] + kp;
      if (a.vec16) {
        cp_async16(dst, s);
      } else {
        cp_async8(dst, s);
        cp_async8(reinterpret_cast<float2*>(dst) + 1, s + (kp + 1 < a.Kb ? 1 : 0));
      }
    }
  // twiddles: lane -> (bin lane/8, half-lag pair lane%8)
  const int kt = min(k0 + (lane >> 3), a.Kb - 1);
  cp_async16(base + kLatRaw + lane, w.twsrc + static_cast<size_t>(kt) * a.Hs);
}

template <int HL>
__device__ __forceinline__ void lattice_bin(float2 v, const float4* trow, float (&A)[kLatHl],
                                            float (&B)[kLatHl]) {
#pragma unroll
  for (int q = 0; q < HL / 2; ++q) {
    const float4 t = trow[q];  // (c, s) of half-lags 2q, 2q+1
    A[2 * q] = fmaf(v.x, t.x, A[2 * q]);
    B[2 * q] = fmaf(v.y, t.y, B[2 * q]);
    A[2 * q + 1] = fmaf(v.x, t.z, A[2 * q + 1]);
    B[2 * q + 1] = fmaf(v.y, t.w, B[2 * q + 1]);
  }
}

template <int kMode, int HL>
__device__ __forceinline__ void lattice_body(const LatticeArgs& a, const LatticeWarp& w,
                                             PhatFloor fl, float (&A)[kLatHl],
                                             float (&B)[kLatHl]) {
  constexpr int kNch = kMode == kPsiStaged ? 1 : 2;
  const int lane = threadIdx.x & 31;
  const int n = (a.Kb + kLatChunk - 1) / kLatChunk;
#pragma unroll
  for (int c = 0; c < kLatStages - 1; ++c) {
    if (c < n) lattice_issue<kNch>(a, w, c, c);
    cp_async_commit();
  }
  for (int c = 0; c < n; ++c) {
    cp_async_wait<kLatStages - 2>();  // this lane's copies of chunk c landed
    __syncwarp();                     // the warp's; stage (c-1)%S is free
    if (c + kLatStages - 1 < n)
      lattice_issue<kNch>(a, w, c + kLatStages - 1, (c + kLatStages - 1) % kLatStages);
    cp_async_commit();
    const float4* stage = w.ring + (c % kLatStages) * kLatStageW;
    const int kvalid = a.Kb - (c * kLatChunk + w.kbase);  // bins of the slice inside Kb
#pragma unroll
    for (int pr = 0; pr < kLatBinsW / 2; ++pr) {
      const float4 ra = stage[pr * kLatRow + lane];
      const float4 rb = kNch == 2 ? stage[(2 + pr) * kLatRow + lane] : ra;
      float2 v0 = psi_warp<kMode>(make_float2(ra.x, ra.y), make_float2(rb.x, rb.y), fl);
      float2 v1 = psi_warp<kMode>(make_float2(ra.z, ra.w), make_float2(rb.z, rb.w), fl);
      if (2 * pr >= kvalid) v0 = make_float2(0.0f, 0.0f);  // clamped copies past Kb
      if (2 * pr + 1 >= kvalid) v1 = make_float2(0.0f, 0.0f);
      const float4* tw = stage + kLatRaw + (2 * pr) * (kLatHl / 2);
      lattice_bin<HL>(v0, tw, A, B);
      lattice_bin<HL>(v1, tw + kLatHl / 2, A, B);
    }
  }
  cp_async_wait<0>();
}

template <int HL>
__device__ __forceinline__ void lattice_reduce_store(const LatticeArgs& a, float* red, int p,
                                                     int f0, int fv, int hl0, int R,
                                                     const float (&A)[kLatHl],
                                                     const float (&B)[kLatHl]) {
  // fixed-order reduction over the 8 K-slices: red[w][acc][frame]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();  // every warp is done with its ring (aliased by red)
#pragma unroll
  for (int h = 0; h < HL; ++h) {
    red[(warp * 2 * kLatHl + h) * kLatF + lane] = A[h];
    red[(warp * 2 * kLatHl + kLatHl + h) * kLatF + lane] = B[h];
  }
  __syncthreads();
  const int col0 = __ldg(a.off + p) + R;  // column of lag 0
  for (int o = threadIdx.x; o < kLatF * HL; o += kLatThreads) {
    const int fl = o % kLatF, h = o / kLatF;
    const int f = f0 + fl, n_lag = hl0 + h;
    if (fl >= fv || n_lag > R) continue;
    float sa = 0.0f, sb = 0.0f;
#pragma unroll
    for (int w = 0; w < kLatWarps; ++w) {
      sa += red[(w * 2 * kLatHl + h) * kLatF + fl];
      sb += red[(w * 2 * kLatHl + kLatHl + h) * kLatF + fl];
    }
    const size_t row = static_cast<size_t>(f) * a.T_pad + col0;
    lattice_store(a, row + n_lag, 2.0f * (sa - sb));
    if (n_lag > 0) lattice_store(a, row - n_lag, 2.0f * (sa + sb));
  }
}

template <int kMode, int HL>
__device__ __forceinline__ void lattice_run(const LatticeArgs& a, const LatticeWarp& w,
                                         PhatFloor fl, float* red, int p, int f0, int fv,
                                         int hl0, int R) {
  float A[kLatHl], B[kLatHl];
#pragma unroll
  for (int h = 0; h < kLatHl; ++h) A[h] = B[h] = 0.0f;
  lattice_body<kMode, HL>(a, w, fl, A, B);
  lattice_reduce_store<HL>(a, red, p, f0, fv, hl0, R, A, B);
}

template <int kMode>
__device__ __forceinline__ void lattice_dispatch_hl(int hlc, const LatticeArgs& a,
                                                    const LatticeWarp& w, PhatFloor fl,
                                                    float* red, int p, int f0, int fv, int hl0,
                                                    int R) {
  if (hlc <= 8)
    lattice_run<kMode, 8>(a, w, fl, red, p, f0, fv, hl0, R);
  else if (hlc <= 12)
    lattice_run<kMode, 12>(a, w, fl, red, p, f0, fv, hl0, R);
  else
    lattice_run<kMode, 16>(a, w, fl, red, p, f0, fv, hl0, R);
}

template <bool kFromY>
__global__ void __launch_bounds__(kLatThreads, 2)
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
  const int hl0 = blockIdx.z * kLatHl;
  if (hl0 > R) return;

  extern __shared__ __align__(16) float4 s_lat[];
  const int warp = tid >> 5, lane = tid & 31;
  const int fv = min(kLatF, a.F - f0);
  LatticeWarp w;
  w.ring = s_lat + warp * kLatStages * kLatStageW;
  w.kbase = warp * kLatBinsW;
  w.twsrc = a.tw + hl0 + 2 * (lane & 7);
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const size_t f = static_cast<size_t>(f0 + min((lane >> 1) + 16 * half, fv - 1));
    if constexpr (kFromY) {
      w.src[0][half] = a.src + (f * a.M + __ldg(a.pm + p)) * a.Kb;
      w.src[1][half] = a.src + (f * a.M + __ldg(a.pmp + p)) * a.Kb;
    } else {
      w.src[0][half] = w.src[1][half] = a.src + (f * a.P + p) * a.Kb;
    }
  }
  const int hlc = min(kLatHl, R + 1 - hl0);  // half-lags this CTA owns
  float* red = reinterpret_cast<float*>(s_lat);
  if constexpr (kFromY) {
    const int f = f0 + min(lane, fv - 1);  // lane = frame
    const PhatFloor fl = make_phat_floor(a.floors ? __ldg(a.floors + f) : a.const_floor);
    // CTA-uniform: every warp sees the same 32 frames
    const bool clean = __all_sync(0xffffffffu, a.clean != nullptr && __ldg(a.clean + f) != 0);
    if (a.weighting != 0)
      lattice_dispatch_hl<kPsiIdentity>(hlc, a, w, fl, red, p, f0, fv, hl0, R);
    else if (clean)
      lattice_dispatch_hl<kPsiPhatClean>(hlc, a, w, fl, red, p, f0, fv, hl0, R);
    else
      lattice_dispatch_hl<kPsiPhatChecked>(hlc, a, w, fl, red, p, f0, fv, hl0, R);
  } else {
    lattice_dispatch_hl<kPsiStaged>(hlc, a, w, PhatFloor{0.0, 0.0f}, red, p, f0, fv, hl0, R);
  }
}

cudaError_t launch_lattice_twiddles(const double* omega, int Kb, double T, int L, float* tw,
                                    cudaStream_t stream) {
  const int blocks = (Kb * twiddle_stride(L) + 255) / 256;
  lattice_twiddle_kernel<<<blocks, 256, 0, stream>>>(omega, Kb, T, L, reinterpret_cast<float2*>(tw));
  return cudaGetLastError();
}

static cudaError_t launch_lattice_args(const LatticeArgs& a, bool from_y, int max_Tp,
                                      cudaStream_t stream) {
  constexpr int smem = static_cast<int>(kLatSmemBytes);
  // per launch: the attribute is per device, and setting it is cheap
  cudaError_t e = from_y ? cudaFuncSetAttribute(lattice_kernel<true>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem)
                         : cudaFuncSetAttribute(lattice_kernel<false>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int max_reach = (max_Tp - 1) / 2;
  dim3 grid(a.P + 1, (a.F + kLatF - 1) / kLatF, max_reach / kLatHl + 1);
  if (from_y)
    lattice_kernel<true><<<grid, kLatThreads, smem, stream>>>(a);
  else
    lattice_kernel<false><<<grid, kLatThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

cudaError_t launch_lattice(const float* Psi, int F, int P, int Kb, const float* tw, int L,
                           const int32_t* off, const int32_t* reach, int max_Tp, int T_pad,
                           float* Xi, cudaStream_t stream) {
  if (F == 0) return cudaSuccess;
  LatticeArgs a{reinterpret_cast<const float2*>(Psi), F, P, Kb, 0, nullptr, nullptr, 1,
                nullptr, 0.0, nullptr, reinterpret_cast<const float2*>(tw), twiddle_stride(L),
                off, reach, T_pad, Xi, nullptr, nullptr, 0.0f, Kb % 2 == 0 && aligned16(Psi)};
  return launch_lattice_args(a, false, max_Tp, stream);
}

cudaError_t launch_lattice_from_spectra(const float* Y, int F, int M, int Kb, const int32_t* pm,
                                        const int32_t* pmp, int P, int weighting,
                                        const double* floors, double abs_floor,
                                        const int32_t* clean, const float* tw,
                                        int L, const int32_t* off, const int32_t* reach,
                                        int max_Tp, int T_pad, float* Xi, void* Xi_hi,
                                        void* Xi_lo, float split_scale, cudaStream_t stream) {
  if (F == 0) return cudaSuccess;
  LatticeArgs a{reinterpret_cast<const float2*>(Y), F, P, Kb, M, pm, pmp, weighting,
                weighting == 0 ? floors : nullptr, weighting == 0 ? abs_floor : 0.0,
                weighting == 0 ? clean : nullptr, reinterpret_cast<const float2*>(tw),
                twiddle_stride(L), off, reach, T_pad, Xi, Xi_hi, Xi_lo, split_scale,
                Kb % 2 == 0 && aligned16(Y)};
  return launch_lattice_args(a, true, max_Tp, stream);
}

}  // namespace srpb
