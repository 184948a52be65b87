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
#include "tmap.cuh"
#include "umma.cuh"

#include <cuda_fp16.h>
#include <type_traits>

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
constexpr int kLatStageW = kLatRaw + kLatTwW;            // float4 per cp.async warp stage
// psi rows: per bin, FG/2 planes of 32/FG frame pairs; planes padded by 64
// bytes so the two planes' 8-byte stores land on different banks
constexpr int kPsiRow = 48;                               // float2 per bin row
constexpr int kLatPsiW = kLatBinsW * kPsiRow;             // float2: one chunk's psi rows
// TMA staging: per stage [raw_a 32 frames x 4 bins][raw_b][tw 4 bins x 16] in bytes
constexpr int kTmaRaw = 32 * 4 * 8;            // 1024 B per channel tile (32-byte rows, SW32)
constexpr int kTmaTwOff = 2 * kTmaRaw;         // 2048
constexpr int kTmaStageBytes = kTmaTwOff + 4 * kLatHl * 8;  // 2560
static_assert(kTmaStageBytes % 256 == 0, "stages keep the 32B-swizzle alignment");

// shared-memory geometry of the two staging variants
template <bool kTma>
struct LatGeom {
  static constexpr int kStageW = kTma ? kTmaStageBytes / 16 : kLatStageW;  // float4 per stage
  static constexpr int kRing = kLatWarps * kLatStages * kStageW;            // float4, all warps
  static constexpr size_t kSmem = 1024 /* alignment slack */ + sizeof(float4) * kRing +
                                  sizeof(float2) * kLatWarps * 2 * kLatPsiW +  // double buffered
                                  sizeof(uint64_t) * kLatWarps * kLatStages;   // TMA barriers
};
static_assert(sizeof(float4) * kLatWarps * kLatStages * (kTmaStageBytes / 16) >=
                  sizeof(float) * kLatWarps * 2 * kLatHl * 32,
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
  // speculative relative floor (kPsiPhatSpec): per (frame, pair) stats
  float* spec_sum;  // [F, P] or NULL
  float* spec_min;
  int* spec_bad;
  double floor_rel;
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
  const float2* src[2][2];  // [ch][half]: row of frame (lane/2 + 16 half), clamped (cp.async)
  const float2* twsrc;      // this lane's twiddle column window at bin 0 (cp.async)
  int nch, kbase;           // channels staged; first bin of the slice in chunk 0
  uint64_t* full;           // [stage] TMA completion barriers of this warp
  int row_c[2];             // TMA: channel (Y) or pair (Psi) coordinate per staged row set
  int f0, hl0;
  const CUtensorMap* tm_src;
  const CUtensorMap* tm_tw;
};

// TMA staging of chunk c into stage st: lane 0 issues the channel tiles
// (32 frames x 4 bins, 32-byte rows, 32-byte swizzle) and the twiddle window
// (4 bins x 16 half-lags); out-of-range frames / bins are zero-filled
template <int kNch>
__device__ __forceinline__ void lattice_issue_tma(const LatticeWarp& w, int c, int st) {
  // warp-uniform operands, one elected lane issues (no per-issue register
  // broadcasts into the uniform datapath)
  uint8_t* base = reinterpret_cast<uint8_t*>(w.ring + st * LatGeom<true>::kStageW);
  const int k0 = c * kLatChunk + w.kbase;
  if (umma::elect_one()) {
    umma::fence_proxy_async_smem();  // generic reads of this stage precede the async writes
    umma::mbar_expect_tx(&w.full[st], kNch * kTmaRaw + 4 * kLatHl * 8);
#pragma unroll
    for (int ch = 0; ch < kNch; ++ch)
      umma::tma_load_3d(base + ch * kTmaRaw, w.tm_src, &w.full[st], k0, w.row_c[ch], w.f0);
    umma::tma_load_2d(base + kTmaTwOff, w.tm_tw, &w.full[st], w.hl0, k0);
  }
  __syncwarp();
}

// raw value (two bins 2pr, 2pr+1 of frame f, channel ch) of a stage
template <bool kTma>
__device__ __forceinline__ float4 lattice_raw(const float4* stage, int ch, int pr, int f) {
  if constexpr (kTma) {
    // 32-byte swizzle: the 16-byte chunk index flips with bit 7 of the address
    const uint8_t* b = reinterpret_cast<const uint8_t*>(stage) + ch * kTmaRaw + f * 32 +
                       ((pr ^ ((f >> 2) & 1)) << 4);
    return *reinterpret_cast<const float4*>(b);
  } else {
    return stage[(ch * 2 + pr) * kLatRow + f];
  }
}
template <bool kTma>
__device__ __forceinline__ const float2* lattice_tw(const float4* stage) {
  return kTma ? reinterpret_cast<const float2*>(reinterpret_cast<const uint8_t*>(stage) + kTmaTwOff)
              : reinterpret_cast<const float2*>(stage + kLatRaw);
}

template <int kNch>
__device__ __forceinline__ void lattice_issue(const LatticeArgs& a, const LatticeWarp& w, int c,
                                              int st) {
  const int lane = threadIdx.x & 31;
  float4* base = w.ring + st * LatGeom<false>::kStageW;
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

// Compute tiling: each lane owns FG frames x HG half-lags (HL = FG * HG per
// CTA, (32 / FG) frame groups x FG half-lag groups = 32 lanes), so per bin a
// lane loads FG psi values (FG/2 LDS.128) and HG twiddles (2 LDS.128 or 3
// LDS.64) for 2 * FG * HG FFMA -- the shared-memory issue rate no longer
// bounds the loop.  Each lane still forms exactly one psi per bin (its own
// frame = lane) and shares it through a per-warp buffer laid out
// psi_w[bin][plane][frame group][2] so the LDS.128 of a frame pair is
// conflict-free.
template <int FG>
__device__ __forceinline__ int psi_slot(int f) {  // float2 offset of frame f in a bin row
  constexpr int NFG = 32 / FG;
  return ((f % FG) >> 1) * (2 * NFG + 8) + (f / FG) * 2 + (f & 1);
}

// psi of this lane's frame for the warp's 4 bins of chunk c -> psi_w row set
template <int kMode, int kNch, bool kTma>
__device__ __forceinline__ void lattice_psi(const LatticeArgs& a, const LatticeWarp& w, int c,
                                            float2* psi_dst, int my_slot, PhatFloor fl,
                                            PhatSpecStats& st) {
  const int lane = threadIdx.x & 31;
  const float4* stage = w.ring + (c % kLatStages) * LatGeom<kTma>::kStageW;
  const int kvalid = a.Kb - (c * kLatChunk + w.kbase);  // bins of the slice inside Kb
#pragma unroll
  for (int pr = 0; pr < kLatBinsW / 2; ++pr) {
    const float4 ra = lattice_raw<kTma>(stage, 0, pr, lane);
    const float4 rb = kNch == 2 ? lattice_raw<kTma>(stage, 1, pr, lane) : ra;
    float2 v0, v1;
    if constexpr (kMode == kPsiPhatSpec) {
      const PhatFloor nofloor{0.0, __int_as_float(0x7f800000)};
      float pa, pb;
      v0 = phat_fast(make_float2(ra.x, ra.y), make_float2(rb.x, rb.y), nofloor, pa, pb);
      if (kTma || 2 * pr < kvalid) st.add(pa, pb);
      v1 = phat_fast(make_float2(ra.z, ra.w), make_float2(rb.z, rb.w), nofloor, pa, pb);
      if (kTma || 2 * pr + 1 < kvalid) st.add(pa, pb);
    } else {
      v0 = psi_warp<kMode>(make_float2(ra.x, ra.y), make_float2(rb.x, rb.y), fl);
      v1 = psi_warp<kMode>(make_float2(ra.z, ra.w), make_float2(rb.z, rb.w), fl);
    }
    if (!kTma) {  // clamped copies past Kb (TMA zero-fills them, twiddles included)
      if (2 * pr >= kvalid) v0 = make_float2(0.0f, 0.0f);
      if (2 * pr + 1 >= kvalid) v1 = make_float2(0.0f, 0.0f);
    }
    psi_dst[(2 * pr) * kPsiRow + my_slot] = v0;
    psi_dst[(2 * pr + 1) * kPsiRow + my_slot] = v1;
  }
}

// FFMA of chunk c: FG frames x HG half-lags per lane, 4 bins
template <int FG, int HG, bool kTma>
__device__ __forceinline__ void lattice_fma(const LatticeWarp& w, int c, const float2* psi_src,
                                            int fgi, int hgi, float (&A)[FG * HG],
                                            float (&B)[FG * HG]) {
  const float2* twb = lattice_tw<kTma>(w.ring + (c % kLatStages) * LatGeom<kTma>::kStageW);
#pragma unroll
  for (int b = 0; b < kLatBinsW; ++b) {
    float2 v[FG];
#pragma unroll
    for (int q = 0; q < FG / 2; ++q) {
      const float4 t = *reinterpret_cast<const float4*>(psi_src + b * kPsiRow +
                                                        q * (2 * (32 / FG) + 8) + fgi * 2);
      v[2 * q] = make_float2(t.x, t.y);
      v[2 * q + 1] = make_float2(t.z, t.w);
    }
    float2 t[HG];
    const float2* trow = twb + b * kLatHl + HG * hgi;
    if constexpr (HG == 4) {
      const float4 t01 = *reinterpret_cast<const float4*>(trow);
      const float4 t23 = *reinterpret_cast<const float4*>(trow + 2);
      t[0] = make_float2(t01.x, t01.y);
      t[1] = make_float2(t01.z, t01.w);
      t[2] = make_float2(t23.x, t23.y);
      t[3] = make_float2(t23.z, t23.w);
    } else {
#pragma unroll
      for (int j = 0; j < HG; ++j) t[j] = trow[j];
    }
#pragma unroll
    for (int i = 0; i < FG; ++i)
#pragma unroll
      for (int j = 0; j < HG; ++j) {
        A[i * HG + j] = fmaf(v[i].x, t[j].x, A[i * HG + j]);
        B[i * HG + j] = fmaf(v[i].y, t[j].y, B[i * HG + j]);
      }
  }
}

// Software-pipelined over chunks: iteration c forms psi of chunk c+1 (MUFU /
// LDS latency) while the FFMAs of chunk c run; psi rows are double buffered.
template <int kMode, int FG, int HG, bool kTma>
__device__ __forceinline__ void lattice_body(const LatticeArgs& a, const LatticeWarp& w,
                                             float2* psi_w, PhatFloor fl,
                                             float (&A)[FG * HG], float (&B)[FG * HG],
                                             PhatSpecStats& st) {
  constexpr int kNch = kMode == kPsiStaged ? 1 : 2;
  constexpr int NHG = FG;  // half-lag groups
  constexpr int S = kLatStages;
  static_assert(S >= 4, "pipeline depth");
  const int lane = threadIdx.x & 31;
  const int fgi = lane / NHG, hgi = lane % NHG;
  const int my_slot = psi_slot<FG>(lane);
  const int n = (a.Kb + kLatChunk - 1) / kLatChunk;
  auto issue = [&](int c) {
    if constexpr (kTma)
      lattice_issue_tma<kNch>(w, c, c % S);
    else
      lattice_issue<kNch>(a, w, c, c % S);
  };
  auto wait_chunk = [&](int c) {  // chunk c landed and is visible to the warp
    if constexpr (kTma)
      umma::mbar_wait(&w.full[c % S], (c / S) & 1);
    else
      cp_async_wait<S - 3>();  // all but the newest group: chunks <= c
  };
#pragma unroll
  for (int c = 0; c < S - 1; ++c) {
    if (c < n) issue(c);
    if (!kTma) cp_async_commit();
  }
  if (kTma)
    umma::mbar_wait(&w.full[0], 0);
  else
    cp_async_wait<S - 2>();  // chunk 0
  __syncwarp();
  lattice_psi<kMode, kNch, kTma>(a, w, 0, psi_w, my_slot, fl, st);
  for (int c = 0; c < n; ++c) {
    // chunk c+1 landed, psi_w[c&1] written, stage (c-1)%S fully consumed
    if (c + 1 < n || !kTma) wait_chunk(c + 1);
    __syncwarp();
    if (c + S - 1 < n) issue(c + S - 1);
    if (!kTma) cp_async_commit();
    if (c + 1 < n)
      lattice_psi<kMode, kNch, kTma>(a, w, c + 1, psi_w + ((c + 1) & 1) * kLatPsiW, my_slot, fl,
                                     st);
    lattice_fma<FG, HG, kTma>(w, c, psi_w + (c & 1) * kLatPsiW, fgi, hgi, A, B);
  }
  if (!kTma) cp_async_wait<0>();
}

template <int FG, int HG>
__device__ __forceinline__ void lattice_reduce_store(const LatticeArgs& a, float* red, int p,
                                                     int f0, int fv, int hl0, int R,
                                                     const float (&A)[FG * HG],
                                                     const float (&B)[FG * HG]) {
  // fixed-order reduction over the 8 K-slices: red[w][acc][lane]
  constexpr int HL = FG * HG, NHG = FG;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();  // every warp is done with its ring (aliased by red)
#pragma unroll
  for (int e = 0; e < HL; ++e) {
    red[(warp * 2 * HL + e) * 32 + lane] = A[e];
    red[(warp * 2 * HL + HL + e) * 32 + lane] = B[e];
  }
  __syncthreads();
  const int col0 = __ldg(a.off + p) + R;  // column of lag 0
  for (int o = threadIdx.x; o < kLatF * HL; o += kLatThreads) {
    const int fl = o % kLatF, h = o / kLatF;
    const int f = f0 + fl, n_lag = hl0 + h;
    if (fl >= fv || n_lag > R) continue;
    const int src = (fl / FG) * NHG + h / HG;       // lane holding (fl, h)
    const int e = (fl % FG) * HG + h % HG;          // its accumulator
    float sa = 0.0f, sb = 0.0f;
#pragma unroll
    for (int w = 0; w < kLatWarps; ++w) {
      sa += red[(w * 2 * HL + e) * 32 + src];
      sb += red[(w * 2 * HL + HL + e) * 32 + src];
    }
    const size_t row = static_cast<size_t>(f) * a.T_pad + col0;
    lattice_store(a, row + n_lag, 2.0f * (sa - sb));
    if (n_lag > 0) lattice_store(a, row - n_lag, 2.0f * (sa + sb));
  }
}

template <int kMode, int FG, int HG, bool kTma>
__device__ __forceinline__ void lattice_run(const LatticeArgs& a, const LatticeWarp& w,
                                            float2* psi_w, PhatFloor fl, float* red, int p,
                                            int f0, int fv, int hl0, int R) {
  float A[FG * HG], B[FG * HG];
#pragma unroll
  for (int e = 0; e < FG * HG; ++e) A[e] = B[e] = 0.0f;
  PhatSpecStats st;
  lattice_body<kMode, FG, HG, kTma>(a, w, psi_w, fl, A, B, st);
  if constexpr (kMode == kPsiPhatSpec) {
    // per-frame stats over the CTA's 8 K-slices, fixed order -> [F, P]
    // (staged in the ring, which the reduction below reuses afterwards)
    float* s_sum = red;
    float* s_min = red + kLatWarps * 32;
    int* s_bad = reinterpret_cast<int*>(red + 2 * kLatWarps * 32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();  // every warp is done with its ring
    s_sum[warp * 32 + lane] = st.sum;
    s_min[warp * 32 + lane] = st.min;
    s_bad[warp * 32 + lane] = st.bad;
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x < 32 && threadIdx.x < fv) {  // half-lag group 0
      float sum = 0.0f, mn = 3.0e38f;
      int bad = 0;
#pragma unroll
      for (int q = 0; q < kLatWarps; ++q) {
        sum += s_sum[q * 32 + threadIdx.x];
        mn = fminf(mn, s_min[q * 32 + threadIdx.x]);
        bad |= s_bad[q * 32 + threadIdx.x];
      }
      const size_t o = static_cast<size_t>(f0 + threadIdx.x) * a.P + p;
      a.spec_sum[o] = sum;
      a.spec_min[o] = mn;
      a.spec_bad[o] = bad;
    }
  }
  lattice_reduce_store<FG, HG>(a, red, p, f0, fv, hl0, R, A, B);
}

template <int kMode, bool kTma>
__device__ __forceinline__ void lattice_dispatch_hl(int hlc, const LatticeArgs& a,
                                                    const LatticeWarp& w, float2* psi_w,
                                                    PhatFloor fl, float* red, int p, int f0,
                                                    int fv, int hl0, int R) {
  if (hlc <= 8)
    lattice_run<kMode, 2, 4, kTma>(a, w, psi_w, fl, red, p, f0, fv, hl0, R);
  else if (hlc <= 12)
    lattice_run<kMode, 4, 3, kTma>(a, w, psi_w, fl, red, p, f0, fv, hl0, R);
  else
    lattice_run<kMode, 4, 4, kTma>(a, w, psi_w, fl, red, p, f0, fv, hl0, R);
}

template <bool kFromY, bool kTma>
__global__ void __launch_bounds__(kLatThreads, 2)
lattice_kernel(const __grid_constant__ CUtensorMap tm_src, const __grid_constant__ CUtensorMap tm_tw,
               const LatticeArgs a) {
  // grid (half-lag group, pair, frame tile): the half-lag groups of one
  // (pair, frame tile) are adjacent in launch order and share its spectra in
  // L2 (C4: 19 groups -- pair-fastest order re-read Y from DRAM per group)
  const int p = blockIdx.y;
  const int f0 = blockIdx.z * kLatF;
  const int tid = threadIdx.x;
  if (p == a.P) {  // pad-column zero fill for this frame tile
    const int t0 = __ldg(a.off + a.P);
    const int w = a.T_pad - t0;
    if (blockIdx.x != 0 || w <= 0) return;
    for (int e = tid; e < kLatF * w; e += blockDim.x) {
      const int fl = e / w, t = t0 + e - fl * w;
      if (f0 + fl < a.F) lattice_store(a, static_cast<size_t>(f0 + fl) * a.T_pad + t, 0.0f);
    }
    return;
  }
  const int R = __ldg(a.reach + p);
  const int hl0 = blockIdx.x * kLatHl;
  if (hl0 > R) return;

  extern __shared__ __align__(1024) uint8_t s_lat_raw[];
  // 1024-align (32-byte-swizzled TMA tiles need 256-byte aligned stages)
  float4* s_lat = reinterpret_cast<float4*>(
      s_lat_raw + ((1024u - (umma::smem_u32(s_lat_raw) & 1023u)) & 1023u));
  const int warp = tid >> 5, lane = tid & 31;
  const int fv = min(kLatF, a.F - f0);
  LatticeWarp w;
  using G = LatGeom<kTma>;
  w.ring = s_lat + warp * kLatStages * G::kStageW;
  w.kbase = warp * kLatBinsW;
  w.f0 = f0;
  w.hl0 = hl0;
  w.tm_src = &tm_src;
  w.tm_tw = &tm_tw;
  w.full = reinterpret_cast<uint64_t*>(reinterpret_cast<float2*>(s_lat + G::kRing) +
                                       kLatWarps * 2 * kLatPsiW) +
           warp * kLatStages;
  if constexpr (kTma) {
    if (lane == 0) {
      for (int st = 0; st < kLatStages; ++st) umma::mbar_init(&w.full[st], 1);
      umma::fence_mbar_init();
    }
    __syncwarp();
    w.row_c[0] = kFromY ? __ldg(a.pm + p) : p;
    w.row_c[1] = kFromY ? __ldg(a.pmp + p) : p;
  } else {
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
  }
  const int hlc = min(kLatHl, R + 1 - hl0);  // half-lags this CTA owns
  float* red = reinterpret_cast<float*>(s_lat);
  float2* psi_w = reinterpret_cast<float2*>(s_lat + G::kRing) + warp * 2 * kLatPsiW;
  if constexpr (kFromY) {
    const int f = f0 + min(lane, fv - 1);  // lane = frame
    const PhatFloor fl = make_phat_floor(a.floors ? __ldg(a.floors + f) : a.const_floor);
    // CTA-uniform: every warp sees the same 32 frames
    const bool clean = __all_sync(0xffffffffu, a.clean != nullptr && __ldg(a.clean + f) != 0);
    if (a.weighting != 0)
      lattice_dispatch_hl<kPsiIdentity, kTma>(hlc, a, w, psi_w, fl, red, p, f0, fv, hl0, R);
    else if (a.spec_sum != nullptr)
      lattice_dispatch_hl<kPsiPhatSpec, kTma>(hlc, a, w, psi_w, fl, red, p, f0, fv, hl0, R);
    else if (clean)
      lattice_dispatch_hl<kPsiPhatClean, kTma>(hlc, a, w, psi_w, fl, red, p, f0, fv, hl0, R);
    else
      lattice_dispatch_hl<kPsiPhatChecked, kTma>(hlc, a, w, psi_w, fl, red, p, f0, fv, hl0, R);
  } else {
    lattice_dispatch_hl<kPsiStaged, kTma>(hlc, a, w, psi_w, PhatFloor{0.0, 0.0f}, red, p, f0, fv,
                                          hl0, R);
  }
}

// Fix-up of the speculative relative floor (kPsiPhatSpec): one CTA per frame
// combines the per-pair stats; a frame is redone exactly when some nonzero
// |raw|^2 could be below floor^2 = rel^2 mean |raw|^2 (with a margin covering
// the fp32 sums) or some power left the fast path's range.  The redo forms
// the fp64 floor like gcc_floor_kernel and recomputes every lattice sample of
// the frame directly, Xi[n] = 2 Re sum_k psi_k e^{j w_k n T} with the
// checked PHAT.  Unflagged frames (all of them on real data) exit at once:
// for them min(1/|raw|, 1/floor) = 1/|raw| and the speculative samples are
// exactly the floored ones.
constexpr int kFixThreads = 256;

// Exact redo of frame f (all kThreads threads of the CTA): fp64 floor over
// all pairs and bins, checked PHAT; s_red [kThreads / 32] doubles.
template <int kThreads>
__device__ void lattice_redo_frame(const LatticeArgs& a, int f, double* s_red);

// Flag test of frame f by one warp (lane 0's return value): the relative
// floor changes the frame iff some nonzero |raw|^2 < 1.01 floor^2, or a
// power left the fast PHAT range.
__device__ __forceinline__ bool lattice_frame_flag_warp(const LatticeArgs& a, int f, int lane) {
  double sum = 0.0;
  float mn = 3.0e38f;
  int bad = 0;
  for (int p = lane; p < a.P; p += 32) {
    const size_t o = static_cast<size_t>(f) * a.P + p;
    sum += static_cast<double>(__ldcg(a.spec_sum + o));
    mn = fminf(mn, __ldcg(a.spec_min + o));
    bad |= __ldcg(a.spec_bad + o);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  const double floor2 = a.floor_rel * a.floor_rel * sum / (static_cast<double>(a.P) * a.Kb);
  return bad || static_cast<double>(mn) < 1.01 * floor2;
}

// Flag test + exact redo of one frame (all threads of the CTA, kThreads of
// them): s_red [kThreads / 32] doubles, s_mn [kThreads / 32] floats, s_flag.
template <int kThreads>
__device__ void lattice_fixup_frame(const LatticeArgs& a, int f, double* s_red, float* s_mn,
                                    int* s_flag) {
  double sum = 0.0;
  float mn = 3.0e38f;
  int bad = 0;
  for (int p = threadIdx.x; p < a.P; p += kThreads) {
    const size_t o = static_cast<size_t>(f) * a.P + p;
    sum += static_cast<double>(__ldcg(a.spec_sum + o));
    mn = fminf(mn, __ldcg(a.spec_min + o));
    bad |= __ldcg(a.spec_bad + o);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  bad = __syncthreads_or(bad);
  if ((threadIdx.x & 31) == 0) {
    s_red[threadIdx.x >> 5] = sum;
    s_mn[threadIdx.x >> 5] = mn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    float m = 3.0e38f;
    for (int w = 0; w < kThreads / 32; ++w) {
      t += s_red[w];
      m = fminf(m, s_mn[w]);
    }
    const double floor2 = a.floor_rel * a.floor_rel * t / (static_cast<double>(a.P) * a.Kb);
    *s_flag = bad || static_cast<double>(m) < 1.01 * floor2;
  }
  __syncthreads();
  const int flagged = *s_flag;
  __syncthreads();  // s_red / s_flag reusable
  if (!flagged) return;
  lattice_redo_frame<kThreads>(a, f, s_red);
}

template <int kThreads>
__device__ void lattice_redo_frame(const LatticeArgs& a, int f, double* s_red) {
  const float2* y = a.src + static_cast<size_t>(f) * a.M * a.Kb;
  double acc = 0.0;
  for (int k = threadIdx.x; k < a.Kb; k += kThreads)
    for (int p = 0; p < a.P; ++p) {
      const float2 u = y[static_cast<size_t>(__ldg(a.pm + p)) * a.Kb + k];
      const float2 v = y[static_cast<size_t>(__ldg(a.pmp + p)) * a.Kb + k];
      acc += (static_cast<double>(u.x) * u.x + static_cast<double>(u.y) * u.y) *
             (static_cast<double>(v.x) * v.x + static_cast<double>(v.y) * v.y);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < kThreads / 32; ++w) t += s_red[w];
  __syncthreads();  // s_red reusable
  const PhatFloor fl = make_phat_floor(a.floor_rel * sqrt(t / (static_cast<double>(a.P) * a.Kb)));
  const int total = __ldg(a.off + a.P);
  for (int col = threadIdx.x; col < total; col += kThreads) {
    int p = 0;
    while (__ldg(a.off + p + 1) <= col) ++p;
    const int R = __ldg(a.reach + p);
    const int n = col - __ldg(a.off + p) - R;  // lag
    const int na = n < 0 ? -n : n;
    const float sgn = n < 0 ? -1.0f : 1.0f;     // lag -n: conjugate twiddle
    const float2* ya = y + static_cast<size_t>(__ldg(a.pm + p)) * a.Kb;
    const float2* yb = y + static_cast<size_t>(__ldg(a.pmp + p)) * a.Kb;
    float re = 0.0f;
    for (int k = 0; k < a.Kb; ++k) {
      const float2 ps = phat_one(ya[k], yb[k], 0, fl);
      const float2 tw = a.tw[static_cast<size_t>(k) * a.Hs + na];
      re = fmaf(ps.x, tw.x, fmaf(-ps.y, sgn * tw.y, re));
    }
    lattice_store(a, static_cast<size_t>(f) * a.T_pad + col, 2.0f * re);
  }
}

// One warp tests one frame (no CTA barrier in the common, unflagged case);
// a CTA redoes its flagged frames together afterwards.
constexpr int kFixFrames = kFixThreads / 32;

__global__ void __launch_bounds__(kFixThreads)
lattice_fixup_kernel(const LatticeArgs a) {
  umma::pdl_wait();  // the lattice kernel's stats and Xi are complete
  umma::pdl_launch_dependents();
  __shared__ double s_red[kFixThreads / 32];
  __shared__ int s_flag[kFixFrames];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int f = blockIdx.x * kFixFrames + w;
  const bool flag = f < a.F && lattice_frame_flag_warp(a, f, lane);
  if (lane == 0) s_flag[w] = flag;
  if (!__syncthreads_or(flag)) return;
  for (int i = 0; i < kFixFrames; ++i)
    if (s_flag[i]) lattice_redo_frame<kFixThreads>(a, blockIdx.x * kFixFrames + i, s_red);
}

cudaError_t launch_lattice_twiddles(const double* omega, int Kb, double T, int L, float* tw,
                                    cudaStream_t stream) {
  const int blocks = (Kb * twiddle_stride(L) + 255) / 256;
  lattice_twiddle_kernel<<<blocks, 256, 0, stream>>>(omega, Kb, T, L, reinterpret_cast<float2*>(tw));
  return cudaGetLastError();
}

template <bool kFromY, bool kTma>
static cudaError_t launch_lattice_kernel(const CUtensorMap& tm_src, const CUtensorMap& tm_tw,
                                         const LatticeArgs& a, dim3 grid, cudaStream_t stream) {
  constexpr int smem = static_cast<int>(LatGeom<kTma>::kSmem);
  static_assert(2 * LatGeom<kTma>::kSmem <= 227 * 1024, "two CTAs per SM");
  cudaError_t e = allow_dynamic_smem(lattice_kernel<kFromY, kTma>, smem);
  if (e != cudaSuccess) return e;
  lattice_kernel<kFromY, kTma><<<grid, kLatThreads, smem, stream>>>(tm_src, tm_tw, a);
  return cudaGetLastError();
}

static cudaError_t launch_lattice_args(const LatticeArgs& a, bool from_y, int max_Tp,
                                      cudaStream_t stream) {
  const int max_reach = (max_Tp - 1) / 2;
  dim3 grid(max_reach / kLatHl + 1, a.P + 1, (a.F + kLatF - 1) / kLatF);
  // TMA staging: 3-D map over the source rows [F][rows][Kb] of 8-byte
  // complex elements (box 4 bins x 1 row x 32 frames, 32-byte swizzle) and a
  // 2-D map over the twiddles [Kb][Hs] (box 16 half-lags x 4 bins); needs
  // even Kb and 16-byte aligned bases, else the cp.async path stages
  CUtensorMap tm_src{}, tm_tw{};
  bool tma = a.vec16 && (reinterpret_cast<uintptr_t>(a.tw) & 15) == 0;
  if (tma) {
    const cuuint64_t rows = from_y ? a.M : a.P;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(a.Kb), rows, static_cast<cuuint64_t>(a.F)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(a.Kb) * 8, rows * a.Kb * 8};
    cuuint32_t box[3] = {4, 1, kLatF};
    tma = encode_tensor_map(&tm_src, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, a.src, dims, strides, box,
                            CU_TENSOR_MAP_SWIZZLE_32B) == cudaSuccess;
    cuuint64_t tdims[2] = {static_cast<cuuint64_t>(a.Hs), static_cast<cuuint64_t>(a.Kb)};
    cuuint64_t tstrides[1] = {static_cast<cuuint64_t>(a.Hs) * 8};
    cuuint32_t tbox[2] = {kLatHl, 4};
    tma = tma && encode_tensor_map(&tm_tw, CU_TENSOR_MAP_DATA_TYPE_INT64, 2, a.tw, tdims, tstrides,
                                   tbox, CU_TENSOR_MAP_SWIZZLE_NONE) == cudaSuccess;
  }
  if (from_y)
    return tma ? launch_lattice_kernel<true, true>(tm_src, tm_tw, a, grid, stream)
               : launch_lattice_kernel<true, false>(tm_src, tm_tw, a, grid, stream);
  return tma ? launch_lattice_kernel<false, true>(tm_src, tm_tw, a, grid, stream)
             : launch_lattice_kernel<false, false>(tm_src, tm_tw, a, grid, stream);
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

cudaError_t launch_lattice(const float* Psi, int F, int P, int Kb, const float* tw, int L,
                           const int32_t* off, const int32_t* reach, int max_Tp, int T_pad,
                           float* Xi, cudaStream_t stream) {
  if (F == 0) return cudaSuccess;
  LatticeArgs a{reinterpret_cast<const float2*>(Psi), F, P, Kb, 0, nullptr, nullptr, 1,
                nullptr, 0.0, nullptr, reinterpret_cast<const float2*>(tw), twiddle_stride(L),
                off, reach, T_pad, Xi, nullptr, nullptr, 0.0f, Kb % 2 == 0 && aligned16(Psi),
                nullptr, nullptr, nullptr, 0.0};
  return launch_lattice_args(a, false, max_Tp, stream);
}

// ---------------------------------------------------------------------------
// K1b+K3 on the tensor cores (PHAT, speculative floor): one GEMM over all
// (frame, pair) rows.  The lattice twiddles e^{j w_k n T} do not depend on
// the pair, so with rows r = f P + p (the pair's PHAT cross-spectrum psi_r
// generated on the fly) and lag slots c = n + L (n in [-L, L], L = max reach):
//   C[r, c] = sum_k Re(psi_r[k]) cos(w_k n T) - Im(psi_r[k]) sin(w_k n T)
//   Xi[f, off_p + reach_p + n] = 2 C[r, n + L],   |n| <= reach_p
// A = psi rows (K = 2 Kb: Re, Im interleaved), B = [cos; -sin] rows per lag
// slot (built once per plan), both 3xFP16 split (x 2^14, |psi| <= 1 and
// |twiddle| <= 1), fp32 accumulation in TMEM.  Pairs with reach < L waste
// the unused lag slots -- free on the tensor core.
//
// CTA = 128 rows; a cluster of two CTAs splits the bins (K) and CTA 1 folds
// its partial accumulator and PHAT statistics into CTA 0 through distributed
// shared memory (fixed order: deterministic).  Warps: 0 TMA producer (B),
// 1 TMEM allocator + MMA issuer, 2..9 psi generators (16 rows each: lane =
// bin, coalesced Y loads, fast PHAT = psi_warp<kPsiPhatSpec> arithmetic,
// per-row stats for the fix-up pass); warps 4..7 (lane quarters 0..3) are the
// epilogue.  Bounded by the PHAT generation (2 MUFU + ~20 ALU per psi), not
// by the MMA (3 x 4 MMAs of 128 x N x 16 per 32-bin block).
#ifdef SRPB_TC_PROFILE
__device__ unsigned long long g_lt_prof[16];
#define LTP_T(v) const long long v = clock64()
#define LTP_ADD(i, v) atomicAdd(&g_lt_prof[i], static_cast<unsigned long long>(v))
#else
#define LTP_T(v)
#define LTP_ADD(i, v)
#endif
constexpr int kLtRows = 128;
constexpr int kLtGenWarps = 16;
constexpr int kLtRW = kLtRows / kLtGenWarps;  // rows per generator warp (8)
constexpr int kLtWarp0 = 2;  // first generator warp
constexpr int kLtThreads = 32 * (kLtWarp0 + kLtGenWarps);
constexpr int kLtStages = 4;
constexpr int kLtMaxN = 64;     // lag slots per pass
constexpr int kLtMaxPasses = 16;  // long lattices (C4: 2L + 1 = 603) run in passes of
                                  // kLtMaxN slots (grid y), the psi rows regenerated per pass
constexpr int kLtOS = kLtRows + 1;  // slot stride of the C staging (odd: conflict-free rows)
constexpr float kLtScale = 16384.0f;  // 2^14 on both operands
// TMEM accumulation drift: bin blocks go to fresh accumulators in groups of
// 4 (48 MMA steps per chain, as K2 / K4), summed in order by the epilogue
constexpr int kLtGroup = 4;
__host__ __device__ inline int lt_tmem_cols(int nkb, int N) {
  const int h = (nkb + 1) / 2;  // blocks of the larger CTA half
  const int need = (h + kLtGroup - 1) / kLtGroup * N;
  int c = 32;
  while (c < need) c <<= 1;
  return c;
}

struct LtSmem {
  uint64_t full[kLtStages];
  uint64_t empty[kLtStages];
  uint64_t yfull[kLtStages];       // the stage's spectra tile landed
  uint64_t acc_full;
  uint32_t tmem_base;
  int2 rows[kLtRows];              // (Y row of mic m, Y row of mic m') per tile row
  float st_sum[2][kLtRows];        // per-row PHAT stats: [own, partner]
  float st_min[2][kLtRows];
  int st_bad[2][kLtRows];
  // in-kernel floor fix-up (frame counters): reduction scratch, completed frames
  double fx_red[32];
  float fx_mn[32];
  int fx_flag, fx_n;
  int fx_done[kLtRows + 1];
};

// stage: A hi/lo (128 rows x 128 B), B hi/lo (N rows x 128 B), spectra tile
// Y [nF frames][M mics][32 bins] complex64 (TMA, 3-D box)
__host__ __device__ inline size_t lt_y_bytes(int nF, int M) { return size_t(nF) * M * 256; }
__host__ __device__ inline size_t lt_stage_bytes(int N, int nF, int M) {
  return (2 * 16384 + 2 * size_t(N) * 128 + lt_y_bytes(nF, M) + 1023) / 1024 * 1024;
}
// multipass: this CTA's own C lives in the idle stage ring (no Xi staging)
__host__ __device__ inline size_t lt_smem_bytes(int N, int nF, int M, int S, bool multipass = false) {
  return 1024 + S * lt_stage_bytes(N, nF, M) +
         (multipass ? 1 : 2) * size_t(kLtOS) * N * 4 /*partner (and own) C*/ +
         sizeof(LtSmem);
}
// frames a 128-row tile spans
inline int lt_frames(int P) { return (kLtRows - 1 + P - 1) / P + 1; }
// stages that fit in 227 KB (0: the tile does not fit)
inline int lt_stages(int N, int nF, int M, bool multipass = false) {
  for (int S = kLtStages; S >= 2; --S)
    if (lt_smem_bytes(N, nF, M, S, multipass) + 1024 <= 232448 &&
        (!multipass || S * lt_stage_bytes(N, nF, M) >= size_t(kLtOS) * N * 4))
      return S;
  return 0;
}

struct LtArgs {
  const float2* Y;
  int F, P, M, Kb, N, L, S, nF;
  int dbg;  // experiments (SRPB_LT_DBG): 1 skip psi math, 2 skip MMAs, 4 skip output
  const int32_t* pm;
  const int32_t* pmp;
  const int32_t* off;
  const int32_t* reach;
  int T_pad;
  float* Xi;
  __half* Xi_hi;
  __half* Xi_lo;
  float split_scale;
  float* spec_sum;
  float* spec_min;
  int* spec_bad;
  // speculative-floor fix-up inside the kernel: per-frame arrival counters
  // (zero before and after each call); NULL -> separate lattice_fixup_kernel
  int* frame_cnt;
  LatticeArgs la;  // what the exact redo of a flagged frame reads and writes
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kLtThreads, 1)
lattice_tc_kernel(const __grid_constant__ CUtensorMap tmB_hi,
                  const __grid_constant__ CUtensorMap tmB_lo,
                  const __grid_constant__ CUtensorMap tmY, const LtArgs a) {
  using namespace umma;
  LTP_T(t_entry);
  extern __shared__ __align__(1024) uint8_t lt_raw[];
  uint8_t* smem = lt_raw + ((1024u - (smem_u32(lt_raw) & 1023u)) & 1023u);
  const int N = a.N;
  const int S = a.S;
  const size_t stage_bytes = lt_stage_bytes(N, a.nF, a.M);
  // [N][129] partial C of CTA 1 and of this CTA (multipass: in the stage
  // ring, idle once this CTA's MMAs are done -- nothing is staged there)
  const bool multipass = gridDim.y > 1;
  float* s_part = reinterpret_cast<float*>(smem + S * stage_bytes);
  float* s_own = multipass ? reinterpret_cast<float*>(smem) : s_part + kLtOS * N;
  LtSmem* sm = reinterpret_cast<LtSmem*>(s_part + (multipass ? 1 : 2) * kLtOS * N);
  // pass (grid y): lag slots [cb, cb + N) of the 2L + 1
  const int cb = static_cast<int>(blockIdx.y) * N;
  auto a_hi = [&](int s) { return smem + s * stage_bytes; };
  auto a_lo = [&](int s) { return smem + s * stage_bytes + 16384; };
  auto b_hi = [&](int s) { return smem + s * stage_bytes + 32768; };
  auto b_lo = [&](int s) { return smem + s * stage_bytes + 32768 + N * 128; };
  auto y_st = [&](int s) { return smem + s * stage_bytes + 32768 + 2 * N * 128; };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int tile = blockIdx.x >> 1;
  const long long R0 = static_cast<long long>(tile) * kLtRows;
  const long long n_rows = static_cast<long long>(a.F) * a.P;
  const int f_lo = static_cast<int>(R0 / a.P);  // first frame of the tile
  // K split: rank 0 takes 32-bin blocks [0, h), rank 1 [h, nkb)
  const int nkb = a.Kb / 32;
  const int h = (nkb + 1) / 2;
  const int kb0 = rank == 0 ? 0 : h, kb1 = rank == 0 ? h : nkb;
  const int my_kb = kb1 - kb0;

  for (int r = threadIdx.x; r < kLtRows; r += blockDim.x) {
    const long long R = R0 + r;
    // byte offsets of the row's two spectra in the stage's Y tile (rows past
    // the end: tile row 0, never stored)
    int2 v = make_int2(0, 0);
    if (R < n_rows) {
      const int f = static_cast<int>(R / a.P), p = static_cast<int>(R - static_cast<long long>(f) * a.P);
      v = make_int2(((f - f_lo) * a.M + __ldg(a.pm + p)) * 256,
                    ((f - f_lo) * a.M + __ldg(a.pmp + p)) * 256);
    }
    sm->rows[r] = v;
  }
  const int tcols = lt_tmem_cols(nkb, N);
  if (warp == 1) tmem_alloc(&sm->tmem_base, tcols);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&sm->full[s], 1 + kLtGenWarps);
      mbar_init(&sm->empty[s], 1);
      mbar_init(&sm->yfull[s], 1);
    }
    mbar_init(&sm->acc_full, 1);
    fence_mbar_init();
    tma_prefetch(&tmB_hi);
    tma_prefetch(&tmB_lo);
    tma_prefetch(&tmY);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, sm->tmem_base, 0);
  // PDL: the prologue above (barriers, TMEM, row table from plan data)
  // overlaps the previous kernel; spectra reads and Xi / stats writes wait
  pdl_wait();
  pdl_launch_dependents();
  LTP_T(t_setup);
#ifdef SRPB_TC_PROFILE
  if (threadIdx.x == 0) {
    LTP_ADD(0, t_setup - t_entry);
    LTP_ADD(9, 1);
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    atomicMax(&g_lt_prof[10], ~gt);  // earliest start (complemented)
    atomicMax(&g_lt_prof[12], gt);   // latest start
  }
#endif

  if (warp == 0) {
    // ---------------------------------------------------------- B producer
    for (int i = 0; i < my_kb; ++i) {
      const int s = i % S;
      mbar_wait(&sm->empty[s], ((i / S) & 1) ^ 1);
      if (elect_one()) {
        // spectra tile first: the generators wait on it
        mbar_expect_tx(&sm->yfull[s], static_cast<uint32_t>(lt_y_bytes(a.nF, a.M)));
        tma_load_3d(y_st(s), &tmY, &sm->yfull[s], (kb0 + i) * 64, 0, f_lo);
        mbar_expect_tx(&sm->full[s], static_cast<uint32_t>(2 * N * 128));
        tma_load_2d(b_hi(s), &tmB_hi, &sm->full[s], (kb0 + i) * 64, cb);
        tma_load_2d(b_lo(s), &tmB_lo, &sm->full[s], (kb0 + i) * 64, cb);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ----------------------------------------------------------- MMA issuer
    const uint32_t idesc = idesc_f16(kLtRows, N);
    for (int i = 0; i < my_kb; ++i) {
      const int s = i % S;
      mbar_wait(&sm->full[s], (i / S) & 1);
      tc_fence_after();
      if (!(a.dbg & 2) && elect_one()) {
        const uint64_t ah = sw128_kmajor_desc(smem_u32(a_hi(s)));
        const uint64_t al = sw128_kmajor_desc(smem_u32(a_lo(s)));
        const uint64_t bh = sw128_kmajor_desc(smem_u32(b_hi(s)));
        const uint64_t bl = sw128_kmajor_desc(smem_u32(b_lo(s)));
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint32_t o = 2 * ks;  // 32 bytes of K per MMA
          const uint32_t d = tmem + static_cast<uint32_t>((i / kLtGroup) * N);
          mma_f16(d, al + o, bh + o, idesc, (i % kLtGroup > 0 || ks > 0) ? 1u : 0u);
          mma_f16(d, ah + o, bl + o, idesc, 1u);
          mma_f16(d, ah + o, bh + o, idesc, 1u);
        }
        mma_commit(&sm->empty[s]);
        if (i == my_kb - 1) mma_commit(&sm->acc_full);
      } else if ((a.dbg & 2) && elect_one()) {
        mbar_arrive(&sm->empty[s]);
        if (i == my_kb - 1) mbar_arrive(&sm->acc_full);
      }
      __syncwarp();
    }
  } else {
    // --------------------------------------------------------- psi generator
    const int g = warp - kLtWarp0;  // rows kLtRW g .. kLtRW g + kLtRW - 1
    // per-row PHAT statistics over this CTA's bins: sum and min of
    // |raw|^2 = pa pb over bins with both powers nonzero (the floor test),
    // and its maximum: the fast path below needs pa pb inside (1e-30, 1e30)
    // (rsqrt of a normal float, no overflow in the products), so a row whose
    // min or max leaves that range is flagged for the exact fix-up
    float ssum[kLtRW], smin[kLtRW], smax[kLtRW];
#pragma unroll
    for (int q = 0; q < kLtRW; ++q) {
      ssum[q] = 0.0f;
      smin[q] = 3.0e38f;
      smax[q] = 0.0f;
    }
    // swizzled 16-byte chunk of this lane's (Re, Im) pair in row r: depends
    // on r & 7 only (rows kLtRW g + q: r & 7 = q & 7)
    uint32_t xo[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      xo[q] = (static_cast<uint32_t>((lane >> 2) ^ q) << 4) + static_cast<uint32_t>(lane & 3) * 4u;
    // byte offsets of the two spectra rows in the Y tile, kept in registers
    int2 ro[kLtRW];
#pragma unroll
    for (int q = 0; q < kLtRW; ++q) ro[q] = sm->rows[kLtRW * g + q];
#ifdef SRPB_TC_PROFILE
    long long w_y = 0;
#endif
    // the floor statistics are written by pass 0 only (the fix-up after the
    // last pass redoes flagged frames in full): later passes skip them
    auto gen_loop = [&](auto stats_tag) {
    constexpr bool kStats = decltype(stats_tag)::value;
    int s = 0, ph = 0;  // stage ring position (no divisions in the loop)
    for (int i = 0; i < my_kb; ++i, s = s + 1 == S ? 0 : s + 1, ph ^= (s == 0)) {
      // the producer loads a stage only after its previous A was consumed
      LTP_T(t_w0);
      mbar_wait(&sm->yfull[s], ph);
#ifdef SRPB_TC_PROFILE
      w_y += clock64() - t_w0;
#endif
      const uint8_t* yk = y_st(s) + lane * 8;
      float2 ya[kLtRW], yb[kLtRW];
#pragma unroll
      for (int q = 0; q < kLtRW; ++q) {
        const int2 o = ro[q];
        ya[q] = *reinterpret_cast<const float2*>(yk + o.x);
        yb[q] = *reinterpret_cast<const float2*>(yk + o.y);
      }
      uint8_t* ahs = a_hi(s) + kLtRW * 128 * g;
      uint8_t* als = a_lo(s) + kLtRW * 128 * g;
#pragma unroll
      for (int q = 0; q < kLtRW; ++q) {
#ifdef SRPB_TC_PROFILE
        if (a.dbg & 1) continue;  // (a branch per row: instrumentation build only)
#endif
        const float pa = fmaf(ya[q].x, ya[q].x, ya[q].y * ya[q].y);
        const float pb = fmaf(yb[q].x, yb[q].x, yb[q].y * yb[q].y);
        const float qq = pa * pb;
        if (kStats) {
          const bool nz = fminf(pa, pb) != 0.0f;  // pa pb may underflow: test the factors
          ssum[q] += qq;
          smin[q] = fminf(smin[q], nz ? qq : 3.0e38f);
          smax[q] = fmaxf(smax[q], qq);
        }
        // 1/|raw| = rsqrt(pa pb): exact to fp32 rounding in the range above;
        // frames outside it are redone by the fix-up pass
        const float sc = rsqrt_approx_ftz(fmaxf(qq, 1e-37f)) * kLtScale;
        const float re = fmaf(ya[q].x, yb[q].x, ya[q].y * yb[q].y) * sc;
        const float im = fmaf(ya[q].y, yb[q].x, -(ya[q].x * yb[q].y)) * sc;
        const __half2 hi = __floats2half2_rn(re, im);
        const float2 hf = __half22float2(hi);
        const __half2 lo = __floats2half2_rn(re - hf.x, im - hf.y);
        *reinterpret_cast<__half2*>(ahs + q * 128 + xo[q & 7]) = hi;
        *reinterpret_cast<__half2*>(als + q * 128 + xo[q & 7]) = lo;
      }
      fence_proxy_async_smem();  // generic-proxy writes -> visible to the MMA
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm->full[s]);
    }
    };
    if (blockIdx.y == 0)
      gen_loop(std::true_type{});
    else
      gen_loop(std::false_type{});
    uint32_t sbad = 0;
#pragma unroll
    for (int q = 0; q < kLtRW; ++q)
      sbad |= (smin[q] <= 1e-30f || !(smax[q] < 1e30f) ? 1u : 0u) << q;
#ifdef SRPB_TC_PROFILE
    if (lane == 0) { LTP_ADD(3, clock64() - t_setup); LTP_ADD(4, w_y); }
#endif
    // rows past the end contributed garbage stats: dropped at the store
    // per-row stats over this CTA's bins: fixed-order warp reduction
#pragma unroll
    for (int q = 0; q < kLtRW; ++q) {
      float sum = ssum[q], mn = smin[q];
      int bad = (sbad >> q) & 1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
      }
      if (lane == 0) {
        sm->st_sum[0][kLtRW * g + q] = sum;
        sm->st_min[0][kLtRW * g + q] = mn;
        sm->st_bad[0][kLtRW * g + q] = bad;
      }
    }
  }

  // ---------------------------------------------------------------- epilogue
  const bool epi = warp >= 4 && warp < 8;
  const int quarter = warp & 3;
  const int row = 32 * quarter + lane;  // TMEM lane = tile row
  if (epi) {
    LTP_T(t_e0);
    mbar_wait(&sm->acc_full, 0);
#ifdef SRPB_TC_PROFILE
    if (lane == 0) { LTP_ADD(5, clock64() - t_e0); LTP_ADD(2, clock64() - t_setup); }
#endif
    tc_fence_after();
    const uint32_t t0 = tmem + (static_cast<uint32_t>(32 * quarter) << 16);
    const int groups = (my_kb + kLtGroup - 1) / kLtGroup;
    // CTA 0 keeps its partial C in s_own, CTA 1 sends it to CTA 0's s_part
    // (column-major [N][128]: conflict-free), 16 columns at a time
    const uint32_t dst = rank == 1 ? mapa(s_part, 0) + static_cast<uint32_t>(row) * 4u
                                   : smem_u32(s_own) + static_cast<uint32_t>(row) * 4u;
    for (int c = 0; c < N; c += 16) {
      float acc[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[e] = 0.0f;
      for (int gq = 0; gq < groups; ++gq) {
        uint32_t r16[16];
        tmem_ld16(t0 + static_cast<uint32_t>(gq * N + c), r16);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[e] += __uint_as_float(r16[e]);
      }
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const uint32_t ad = dst + 4u * kLtOS * (c + e);
        if (rank == 1)
          st_shared_cluster_u32(ad, __float_as_uint(acc[e]));
        else
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(ad), "r"(__float_as_uint(acc[e])) : "memory");
      }
    }
  }
  __syncthreads();  // stats of every generator warp are in sm->st_*[0]
  if (rank == 1) {
    for (int r = threadIdx.x; r < kLtRows; r += blockDim.x) {
      st_shared_cluster_u32(mapa(&sm->st_sum[1][r], 0), __float_as_uint(sm->st_sum[0][r]));
      st_shared_cluster_u32(mapa(&sm->st_min[1][r], 0), __float_as_uint(sm->st_min[0][r]));
      st_shared_cluster_u32(mapa(&sm->st_bad[1][r], 0), static_cast<uint32_t>(sm->st_bad[0][r]));
    }
  }
  tc_fence_before();
  LTP_T(t_c0);
  cluster_sync();  // CTA 1's partials landed in CTA 0
  LTP_T(t_c1);
#ifdef SRPB_TC_PROFILE
  if (threadIdx.x == 0) LTP_ADD(6, t_c1 - t_c0);
#endif
  if (rank == 0) {
    for (int r = threadIdx.x; r < kLtRows; r += blockDim.x) {
      const long long R = R0 + r;
      if (R < n_rows && a.spec_sum && blockIdx.y == 0) {  // statistics: pass 0
        a.spec_sum[R] = sm->st_sum[0][r] + sm->st_sum[1][r];
        a.spec_min[R] = fminf(sm->st_min[0][r], sm->st_min[1][r]);
        a.spec_bad[R] = sm->st_bad[0][r] | sm->st_bad[1][r];
      }
    }
    if (gridDim.y > 1) {
      // multi-pass: a row's slots of this pass are one contiguous run of its
      // Xi row; a warp per row, lanes over the slots (coalesced 2-byte
      // stores; the [slot][129] staging keeps the reads conflict-free)
      const float out_scale = 2.0f / (kLtScale * kLtScale);
      if (!(a.dbg & 12)) {
        for (int orow = warp; orow < kLtRows; orow += kLtThreads / 32) {
          const long long R = R0 + orow;
          if (R >= n_rows) break;
          const int f = static_cast<int>(R / a.P), p = static_cast<int>(R - static_cast<long long>(f) * a.P);
          const int Rp = __ldg(a.reach + p);
          const int lo = max(cb, a.L - Rp), hi = min(cb + N - 1, a.L + Rp);
          const size_t g0 = static_cast<size_t>(f) * a.T_pad + __ldg(a.off + p) + Rp - a.L;
          for (int c = lo + lane; c <= hi; c += 32) {
            const int cl = c - cb;
            const float v = (s_own[cl * kLtOS + orow] + s_part[cl * kLtOS + orow]) * out_scale;
            if (a.Xi) a.Xi[g0 + c] = v;
            const float x = v * a.split_scale;
            const __half hh = __float2half_rn(x);
            a.Xi_hi[g0 + c] = hh;
            a.Xi_lo[g0 + c] = __float2half_rn(x - __half2float(hh));
          }
        }
        // pad columns past the last pair's lattice: pass 0 of the frame's
        // last row writes them
        if (blockIdx.y == 0) {
          const int t_pad0 = __ldg(a.off + a.P);
          const long long R_end = min(R0 + kLtRows, n_rows);
          for (long long R = R0 + warp; R < R_end; R += kLtThreads / 32) {
            const int f = static_cast<int>(R / a.P);
            if (R - static_cast<long long>(f) * a.P != a.P - 1) continue;
            const size_t g0 = static_cast<size_t>(f) * a.T_pad;
            for (int c = t_pad0 + lane; c < a.T_pad; c += 32) {
              if (a.Xi) a.Xi[g0 + c] = 0.0f;
              a.Xi_hi[g0 + c] = __float2half_rn(0.0f);
              a.Xi_lo[g0 + c] = __float2half_rn(0.0f);
            }
          }
        }
      }
    } else {
    // Xi rows of the tile's frames are staged in shared memory (the stage
    // ring is idle now) and leave with coalesced stores: each tile row owns
    // 2 reach_p + 1 scattered columns, which as direct 2-byte global stores
    // cost one L2 sector write each
    const int nF = a.nF, Tp = a.T_pad;
    __half* xs_hi = reinterpret_cast<__half*>(smem);           // [nF][T_pad]
    __half* xs_lo = xs_hi + static_cast<size_t>(nF) * Tp;
    float* xs = reinterpret_cast<float*>(xs_lo + static_cast<size_t>(nF) * Tp);  // if a.Xi
    // 4 threads per tile row (the generator warps), lags interleaved
    const int gt = static_cast<int>(threadIdx.x) - 32 * kLtWarp0;
    if (gt >= 0 && !(a.dbg & 12)) {
      const int orow = gt >> 2, sub = gt & 3;
      const long long R = R0 + orow;
      if (R < n_rows) {
        const int f = static_cast<int>(R / a.P), p = static_cast<int>(R - static_cast<long long>(f) * a.P);
        const int Rp = __ldg(a.reach + p);
        const int col0 = (f - f_lo) * Tp + __ldg(a.off + p) + Rp;  // lag 0
        const float out_scale = 2.0f / (kLtScale * kLtScale);
        const float* part = s_part + orow;
        const float* own = s_own + orow;
        for (int c = a.L - Rp + sub; c <= a.L + Rp; c += 4) {
          const int n = c - a.L;
          {
            const float v = (own[c * kLtOS] + part[c * kLtOS]) * out_scale;
            const int idx = col0 + n;
            if (a.Xi) xs[idx] = v;
            const float x = v * a.split_scale;
            const __half hh = __float2half_rn(x);
            xs_hi[idx] = hh;
            xs_lo[idx] = __float2half_rn(x - __half2float(hh));
          }
        }
      }
    }
    __syncthreads();
    if (!(a.dbg & 20)) {
      const long long R_end = min(R0 + kLtRows, n_rows);  // rows [R0, R_end)
      const int t_pad0 = __ldg(a.off + a.P);
      for (int fl = 0; fl < nF; ++fl) {
        const long long f = f_lo + fl;
        const long long r_lo = max(R0, f * a.P), r_hi = min(R_end, (f + 1) * a.P);
        if (r_lo >= r_hi) break;
        const int p0 = static_cast<int>(r_lo - f * a.P), p1 = static_cast<int>(r_hi - f * a.P);
        const int c0 = __ldg(a.off + p0);
        const int c1 = p1 == a.P ? Tp : __ldg(a.off + p1);  // the last pair also owns the pad
        const size_t g0 = static_cast<size_t>(f) * Tp;
        for (int c = c0 + static_cast<int>(threadIdx.x); c < c1; c += blockDim.x) {
          const bool pad = c >= t_pad0;
          const int sidx = fl * Tp + c;
          if (a.Xi) a.Xi[g0 + c] = pad ? 0.0f : xs[sidx];
          if (a.Xi_hi) {
            a.Xi_hi[g0 + c] = pad ? __float2half_rn(0.0f) : xs_hi[sidx];
            a.Xi_lo[g0 + c] = pad ? __float2half_rn(0.0f) : xs_lo[sidx];
          }
        }
      }
    }
    }  // single pass
    if (a.frame_cnt) {
      // floor fix-up without a second kernel: the CTA that completes a frame
      // (its rows can span two tiles) checks the frame's statistics and, if
      // flagged, redoes the frame exactly (threadfence-reduction ordering)
      __threadfence();  // this CTA's Xi rows and statistics, device-wide
      __syncthreads();
      if (threadIdx.x == 0) {
        const long long R_end = min(R0 + kLtRows, n_rows);
        int nd = 0;
        for (int fl = 0; fl < a.nF; ++fl) {
          const long long f = f_lo + fl;
          const long long r_lo = max(R0, f * a.P), r_hi = min(R_end, (f + 1) * a.P);
          if (r_lo >= r_hi) break;
          const int rows = static_cast<int>(r_hi - r_lo);
          if (atomicAdd(a.frame_cnt + f, rows) + rows == a.P) sm->fx_done[nd++] = static_cast<int>(f);
        }
        sm->fx_n = nd;
        __threadfence();  // the other tile's rows of the completed frames
      }
      __syncthreads();
      // flag test: one warp per completed frame (no CTA barriers); counters
      // reset for the next call
      const int nd = sm->fx_n;
      int any = 0;
      for (int i = warp; i < nd; i += kLtThreads / 32) {
        const int f = sm->fx_done[i];
        const bool flag = lattice_frame_flag_warp(a.la, f, lane);
        if (lane == 0) {
          sm->fx_done[i] = flag ? f : -1;
          a.frame_cnt[f] = 0;
        }
        any |= flag;
      }
      if (__syncthreads_or(any)) {  // rare: exact redo of the flagged frames
        for (int i = 0; i < nd; ++i)
          if (sm->fx_done[i] >= 0) lattice_redo_frame<kLtThreads>(a.la, sm->fx_done[i], sm->fx_red);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
#ifdef SRPB_TC_PROFILE
  if (threadIdx.x == 0) {
    LTP_ADD(7, clock64() - t_c1);
    LTP_ADD(8, clock64() - t_entry);
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    atomicMax(&g_lt_prof[11], gt);  // latest end
  }
#endif
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, tcols);
  }
}

#ifdef SRPB_TC_PROFILE
extern "C" int srpb_lt_profile_read(unsigned long long* out) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_lt_prof, sizeof(unsigned long long) * 16);
  unsigned long long z[16] = {};
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_lt_prof, z, sizeof(z));
  return e == cudaSuccess ? 0 : 1;
}
#endif

// B operand of the tensor-core lattice: rows c = lag slot (n = c - L),
// K = 2 Kb interleaved (cos, -sin)(w_k n T) x 2^14, fp16 hi/lo split; rows
// past 2L zero.  fp64 phases, like lattice_twiddle_kernel.
__global__ void lattice_tc_twiddle_kernel(const double* __restrict__ omega, int Kb, double T,
                                          int L, int N, __half* __restrict__ bh,
                                          __half* __restrict__ bl) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < N * Kb; e += gridDim.x * blockDim.x) {
    const int c = e / Kb, k = e - c * Kb;
    double sn = 0.0, cs = 0.0;
    if (c <= 2 * L) sincos(static_cast<double>(c - L) * T * omega[k], &sn, &cs);
    const float x[2] = {static_cast<float>(cs * kLtScale), static_cast<float>(-sn * kLtScale)};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const __half hh = __float2half_rn(x[u]);
      const size_t o = static_cast<size_t>(c) * 2 * Kb + 2 * k + u;
      bh[o] = hh;
      bl[o] = __float2half_rn(x[u] - __half2float(hh));
    }
  }
}

int lattice_tc_n(int L) { return (2 * L + 1 + 15) / 16 * 16; }

cudaError_t launch_lattice_tc_twiddles(const double* omega, int Kb, double T, int L, void* bh,
                                       void* bl, cudaStream_t stream) {
  const int N = lattice_tc_n(L);
  const int total = N * Kb;
  const int blocks = (total + 255) / 256 < 4 * kNumSMs ? (total + 255) / 256 : 4 * kNumSMs;
  lattice_tc_twiddle_kernel<<<blocks, 256, 0, stream>>>(omega, Kb, T, L, N,
                                                        static_cast<__half*>(bh),
                                                        static_cast<__half*>(bl));
  return cudaGetLastError();
}

// whether the tensor-core lattice serves this shape
// slots per pass and passes of the tensor-core lattice: one pass up to 64
// slots; beyond, the widest pass whose stages fit next to the partner's C
// (psi rows are regenerated per pass, so fewer passes is the saving)
inline int lt_pass_n(int L, int P = 0, int M = 0) {
  const int n = lattice_tc_n(L);
  if (n <= kLtMaxN) return n;
  if (P > 0)
    for (int N = min(128, n); N > kLtMaxN; N -= 16)
      if (lt_stages(N, lt_frames(P), M, (n + N - 1) / N > 1) >= 2) return N;
  return kLtMaxN;
}
inline int lt_passes(int L, int P = 0, int M = 0) {
  const int N = lt_pass_n(L, P, M);
  return (lattice_tc_n(L) + N - 1) / N;
}

bool lattice_tc_ok(int Kb, int L, float split_scale, const void* Xi_hi) {
  return Kb % 32 == 0 && Kb >= 64 && lt_passes(L) <= kLtMaxPasses && split_scale != 0.0f &&
         Xi_hi != nullptr && getenv("SRPB_LATTICE_SIMT") == nullptr;
}

// shapes the tensor-core lattice serves (besides PHAT + fp16 split output)
bool lattice_tc_shape_ok(int M, int P, int Kb, int L, int T_pad) {
  if (Kb % 32 != 0 || Kb < 64 || lt_passes(L) > kLtMaxPasses || M > 256 || P < 1) return false;
  const int nF = lt_frames(P);
  if (nF > 256) return false;
  const int N = lt_pass_n(L, P, M);
  const bool multi = lt_passes(L, P, M) > 1;
  const int S = lt_stages(N, nF, M, multi);
  // the tile's spectra fit the stages, and (single pass) its Xi rows the ring
  return S >= 2 && (multi || static_cast<size_t>(nF) * T_pad * 8 <= S * lt_stage_bytes(N, nF, M));
}

static cudaError_t launch_lattice_tc(const LatticeArgs& la, int L, const void* bh, const void* bl,
                                     int* frame_cnt, cudaStream_t stream) {
  const int N = lt_pass_n(L, la.P, la.M), passes = lt_passes(L, la.P, la.M);
  if (passes > 1) frame_cnt = nullptr;  // the fix-up kernel follows (all passes done)
  CUtensorMap mh, ml;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(2 * la.Kb),
                        static_cast<cuuint64_t>(lattice_tc_n(L))};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(2 * la.Kb) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(N)};
  cudaError_t e = encode_tensor_map(&mh, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, bh, dims, strides, box,
                                    CU_TENSOR_MAP_SWIZZLE_128B);
  if (e == cudaSuccess)
    e = encode_tensor_map(&ml, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, bl, dims, strides, box,
                          CU_TENSOR_MAP_SWIZZLE_128B);
  if (e != cudaSuccess) return e;
  const int nF = lt_frames(la.P);
  const int S = lt_stages(N, nF, la.M, passes > 1);
  // spectra as [F][M][2 Kb] floats; box = 32 bins x all mics x the tile's frames
  CUtensorMap my;
  {
    cuuint64_t yd[3] = {static_cast<cuuint64_t>(2 * la.Kb), static_cast<cuuint64_t>(la.M),
                        static_cast<cuuint64_t>(la.F)};
    cuuint64_t ys[2] = {static_cast<cuuint64_t>(2 * la.Kb) * 4,
                        static_cast<cuuint64_t>(2 * la.Kb) * 4 * la.M};
    cuuint32_t yb[3] = {64, static_cast<cuuint32_t>(la.M), static_cast<cuuint32_t>(nF)};
    e = encode_tensor_map(&my, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, la.src, yd, ys, yb,
                          CU_TENSOR_MAP_SWIZZLE_NONE);
    if (e != cudaSuccess) return e;
  }
  LtArgs a{la.src, la.F, la.P, la.M, la.Kb, N, L, S, nF,
           getenv("SRPB_LT_DBG") ? atoi(getenv("SRPB_LT_DBG")) : 0,
           la.pm, la.pmp, la.off, la.reach, la.T_pad,
           la.Xi, static_cast<__half*>(la.Xi_hi), static_cast<__half*>(la.Xi_lo), la.split_scale,
           la.spec_sum, la.spec_min, la.spec_bad, frame_cnt, la};
  const size_t smem = lt_smem_bytes(N, nF, la.M, S, passes > 1);
  e = allow_dynamic_smem(lattice_tc_kernel, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const long long rows = static_cast<long long>(la.F) * la.P;
  const int tiles = static_cast<int>((rows + kLtRows - 1) / kLtRows);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * tiles, passes);
  cfg.blockDim = dim3(kLtThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_attr_value();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, lattice_tc_kernel, mh, ml, my, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_lattice_from_spectra(const float* Y, int F, int M, int Kb, const int32_t* pm,
                                        const int32_t* pmp, int P, int weighting,
                                        const double* floors, double abs_floor,
                                        const int32_t* clean, const float* tw,
                                        int L, const int32_t* off, const int32_t* reach,
                                        int max_Tp, int T_pad, float* Xi, void* Xi_hi,
                                        void* Xi_lo, float split_scale, double floor_rel,
                                        void* spec_scratch, cudaStream_t stream,
                                        const void* tc_bh, const void* tc_bl, int* frame_cnt) {
  if (F == 0) return cudaSuccess;
  // PHAT with the relative floor and no precomputed floors: speculative
  // lattice + per-frame fix-up (scratch: 12 bytes per frame and pair)
  const bool spec = weighting == 0 && floors == nullptr && !(abs_floor > 0.0);
  LatticeArgs a{reinterpret_cast<const float2*>(Y), F, P, Kb, M, pm, pmp, weighting,
                weighting == 0 ? floors : nullptr, weighting == 0 ? abs_floor : 0.0,
                weighting == 0 ? clean : nullptr, reinterpret_cast<const float2*>(tw),
                twiddle_stride(L), off, reach, T_pad, Xi, Xi_hi, Xi_lo, split_scale,
                Kb % 2 == 0 && aligned16(Y), nullptr, nullptr, nullptr, floor_rel};
  if (!spec) return launch_lattice_args(a, true, max_Tp, stream);
  void* scratch = spec_scratch;
  const size_t n = static_cast<size_t>(F) * P;
  cudaError_t e = cudaSuccess;
  if (scratch == nullptr) {  // no caller scratch: stream-ordered allocation
    e = cudaMallocAsync(&scratch, n * 12, stream);
    if (e != cudaSuccess) return e;
  }
  a.spec_sum = static_cast<float*>(scratch);
  a.spec_min = a.spec_sum + n;
  a.spec_bad = reinterpret_cast<int*>(a.spec_min + n);
  bool fixed_in_kernel = false;
  if (tc_bh && tc_bl && aligned16(Y) && lattice_tc_ok(Kb, L, split_scale, Xi_hi) &&
      lattice_tc_shape_ok(M, P, Kb, L, T_pad))
  {
    e = launch_lattice_tc(a, L, tc_bh, tc_bl, frame_cnt, stream);
    fixed_in_kernel = frame_cnt != nullptr && lt_passes(L, P, M) == 1;
  } else {
    e = launch_lattice_args(a, true, max_Tp, stream);
  }
  if (e == cudaSuccess && !fixed_in_kernel) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((F + kFixFrames - 1) / kFixFrames);
    cfg.blockDim = dim3(kFixThreads);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_attr_value();
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, lattice_fixup_kernel, a);
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  const cudaError_t e2 = spec_scratch == nullptr ? cudaFreeAsync(scratch, stream) : cudaSuccess;
  return e != cudaSuccess ? e : e2;
}

}  // namespace srpb
