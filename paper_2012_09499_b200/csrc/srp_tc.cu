// Tensor-core (tcgen05, kind::tf32, 3xTF32) SRP contractions for sm_100a.
//
//   maps[f, j] = scale * sum_kk A[j, kk] B[f, kk]
//
// K2 (conventional, srp.py:391-429): A = steering phases [cos, -sin] generated
//    on the fly by SIMT warps straight into shared memory (never stored in
//    HBM), B = Psi [F, 2 P Kb] (float view of the cross-spectra), scale 2.
// K4 (approximate, srp.py:320-347): A = W [J, T_pad] sinc weights, B = Xi
//    [F, T_pad] lattice samples, both streamed by TMA, scale 1.
//
// fp32 accuracy from TF32 tensor cores: every operand is pre-split into
// hi = tf32(x), lo = tf32(x - hi) and each K step issues three MMAs
// (hi*hi + hi*lo + lo*hi) into the same TMEM accumulator (residual ~2^-22).
// The tensor core's fp32 accumulation is not round-to-nearest: over a long
// chain the accumulator drifts toward zero (measured: -1.4e-5 relative after
// 384 K steps x 3 MMAs at C1).  The contraction is therefore cut into groups
// of a few K blocks; each group accumulates in one of two TMEM buffers
// (ping-pong) and the epilogue warps fold it into round-to-nearest fp32
// register totals while the MMA continues into the other buffer.
//
// CTA = one 128-candidate x N-frame output tile (N <= 160, multiple of 32).
//   warp 0      TMA producer (B; and A for K4)           elected lane
//   warp 1      TMEM allocator + MMA issuer              elected lane
//   warps 4..11 epilogue: TMEM drains, map store, fused argmax; for K2 they
//               also generate the A tiles (2 threads per candidate row)
// Smem: 3 stages x {A_hi, A_lo: 128 x 128 B; B_hi, B_lo: N x 128 B}, SW128.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "umma.cuh"

namespace srpb {

using namespace umma;

constexpr int kTcThreads = 384;
constexpr int kTcStages = 3;
constexpr int kTcM = 128;
constexpr int kTcMaxN = 160;
constexpr int kTcKBlock = 32;  // fp32 elements per K block = one 128-B swizzle row
constexpr int kEpiWarp0 = 4;
constexpr int kEpiWarps = 8;
constexpr int kABytes = kTcM * 128;  // one of A_hi / A_lo per stage

enum : int { kAFromTma = 0, kAPhase = 1 };

struct TcParams {
  int F, J, N;        // frames, candidates, frames per tile
  int num_kb;         // K blocks of 32
  int kb_per_group;   // TMEM drain period (K blocks)
  float scale;
  float* maps;
  unsigned long long* keys;
  // K2 phase generation
  const int32_t* tau_i;
  const float* tau_f;
  int kb_per_pair;    // Kb / 16
  int period, mask;
  float inv_period;
};

struct TcSmem {
  uint64_t full[kTcStages];
  uint64_t empty[kTcStages];
  uint64_t acc_full[2];
  uint64_t acc_empty[2];
  uint32_t tmem_base;
};

__host__ __device__ inline size_t tc_stage_bytes(int N) { return 2 * kABytes + 2 * size_t(N) * 128; }
__host__ __device__ inline size_t tc_smem_bytes(int N) {
  return 1024 /*align slack*/ + kTcStages * tc_stage_bytes(N) + sizeof(TcSmem);
}

// Fold one TMEM accumulator buffer into the register totals of this thread:
// row = 32*(warp%4) + lane, columns [half*N/2, half*N/2 + N/2).
__device__ __forceinline__ void tc_drain(const TcParams& p, TcSmem* bar, uint32_t tmem, int g,
                                         int quarter, int half, float (&tot)[kTcMaxN / 2]) {
  const int b = g & 1;
  mbar_wait(&bar->acc_full[b], (g >> 1) & 1);
  tc_fence_after();
  const uint32_t base = tmem + (static_cast<uint32_t>(32 * quarter) << 16) +
                        static_cast<uint32_t>(b * p.N + half * (p.N / 2));
  const int nchunks = p.N / 32;  // 16-column loads per half
#pragma unroll
  for (int c = 0; c < kTcMaxN / 32; ++c) {
    if (c < nchunks) {
      uint32_t r[16];
      tmem_ld16(base + 16 * c, r);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 16; ++i) tot[16 * c + i] += __uint_as_float(r[i]);
    }
  }
  tc_fence_before();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(&bar->acc_empty[b]);
}

// A tile of steering phases for K block kb: candidate row r, bins
// [k0 + 8*half, +8) of pair p, as (cos, -sin) pairs, split hi/lo, SW128.
__device__ __forceinline__ void tc_gen_phase(const TcParams& p, uint8_t* a_hi, uint8_t* a_lo,
                                             int r, int half, int kb, int j, int& cur_pair,
                                             int& ti, float& tf, float& sc, float& ss) {
  const int pair = kb / p.kb_per_pair;
  if (pair != cur_pair) {
    cur_pair = pair;
    ti = 0;
    tf = 0.0f;
    if (j < p.J) {
      ti = p.tau_i[static_cast<size_t>(pair) * p.J + j];
      tf = p.tau_f[static_cast<size_t>(pair) * p.J + j];
    }
    sincospif(2.0f * (static_cast<float>(ti) + tf) * p.inv_period, &ss, &sc);  // e^{j 2pi x/N}
  }
  const int k = (kb - pair * p.kb_per_pair) * 16 + 8 * half;
  float c, s;
  harmonic_phase(k, ti, tf, p.period, p.mask, p.inv_period, &c, &s);
  float v[16];
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    v[2 * m] = c;
    v[2 * m + 1] = -s;
    const float cn = c * sc - s * ss;  // rotate by one bin
    s = fmaf(c, ss, s * sc);
    c = cn;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float4 h, l;
    h.x = to_tf32(v[4 * q + 0]);
    h.y = to_tf32(v[4 * q + 1]);
    h.z = to_tf32(v[4 * q + 2]);
    h.w = to_tf32(v[4 * q + 3]);
    l.x = to_tf32(v[4 * q + 0] - h.x);
    l.y = to_tf32(v[4 * q + 1] - h.y);
    l.z = to_tf32(v[4 * q + 2] - h.z);
    l.w = to_tf32(v[4 * q + 3] - h.w);
    const uint32_t off = sw128_offset(r, 4 * half + q);
    *reinterpret_cast<float4*>(a_hi + off) = h;
    *reinterpret_cast<float4*>(a_lo + off) = l;
  }
}

template <int kAMode>
__global__ void __launch_bounds__(kTcThreads, 1)
srp_tc_kernel(const __grid_constant__ CUtensorMap tmA_hi, const __grid_constant__ CUtensorMap tmA_lo,
              const __grid_constant__ CUtensorMap tmB_hi, const __grid_constant__ CUtensorMap tmB_lo,
              const TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const size_t stage_bytes = tc_stage_bytes(p.N);
  TcSmem* bar = reinterpret_cast<TcSmem*>(smem + kTcStages * stage_bytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * p.N;      // first frame of the tile
  const int m0 = blockIdx.y * kTcM;     // first candidate of the tile
  const int num_groups = (p.num_kb + p.kb_per_group - 1) / p.kb_per_group;
  const uint32_t b_bytes = static_cast<uint32_t>(p.N) * 128;

  auto a_hi = [&](int s) { return smem + s * stage_bytes; };
  auto a_lo = [&](int s) { return smem + s * stage_bytes + kABytes; };
  auto b_hi = [&](int s) { return smem + s * stage_bytes + 2 * kABytes; };
  auto b_lo = [&](int s) { return smem + s * stage_bytes + 2 * kABytes + b_bytes; };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmB_hi);
    tma_prefetch(&tmB_lo);
    if (kAMode == kAFromTma) {
      tma_prefetch(&tmA_hi);
      tma_prefetch(&tmA_lo);
    }
  }
  if (warp == 1) tmem_alloc(&bar->tmem_base, 512);
  if (warp == 2 && lane == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&bar->full[s], kAMode == kAFromTma ? 1 : 1 + kEpiWarps);
      mbar_init(&bar->empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar->acc_full[b], 1);
      mbar_init(&bar->acc_empty[b], kEpiWarps);
    }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar->tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint32_t tx = 2 * b_bytes + (kAMode == kAFromTma ? 2 * kABytes : 0);
      for (int kb = 0; kb < p.num_kb; ++kb) {
        const int s = kb % kTcStages;
        mbar_wait(&bar->empty[s], ((kb / kTcStages) & 1) ^ 1);
        mbar_expect_tx(&bar->full[s], tx);
        tma_load_2d(b_hi(s), &tmB_hi, &bar->full[s], kb * kTcKBlock, n0);
        tma_load_2d(b_lo(s), &tmB_lo, &bar->full[s], kb * kTcKBlock, n0);
        if (kAMode == kAFromTma) {
          tma_load_2d(a_hi(s), &tmA_hi, &bar->full[s], kb * kTcKBlock, m0);
          tma_load_2d(a_lo(s), &tmA_lo, &bar->full[s], kb * kTcKBlock, m0);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_tf32(kTcM, p.N);
      for (int kb = 0; kb < p.num_kb; ++kb) {
        const int s = kb % kTcStages;
        const int g = kb / p.kb_per_group;
        const int in_group = kb - g * p.kb_per_group;
        const uint32_t d = tmem + static_cast<uint32_t>((g & 1) * p.N);
        if (in_group == 0) {
          mbar_wait(&bar->acc_empty[g & 1], ((g >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        mbar_wait(&bar->full[s], (kb / kTcStages) & 1);
        tc_fence_after();
        const uint32_t ah = smem_u32(a_hi(s)), al = smem_u32(a_lo(s));
        const uint32_t bh = smem_u32(b_hi(s)), bl = smem_u32(b_lo(s));
#pragma unroll
        for (int ks = 0; ks < kTcKBlock / 8; ++ks) {
          const uint32_t o = ks * 32;  // 8 tf32 = 32 bytes along K
          const uint32_t acc0 = (in_group > 0 || ks > 0) ? 1u : 0u;
          mma_tf32(d, sw128_kmajor_desc(al + o), sw128_kmajor_desc(bh + o), idesc, acc0);
          mma_tf32(d, sw128_kmajor_desc(ah + o), sw128_kmajor_desc(bl + o), idesc, 1u);
          mma_tf32(d, sw128_kmajor_desc(ah + o), sw128_kmajor_desc(bh + o), idesc, 1u);
        }
        mma_commit(&bar->empty[s]);
        if (in_group == p.kb_per_group - 1 || kb == p.num_kb - 1) mma_commit(&bar->acc_full[g & 1]);
      }
    }
  } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + kEpiWarps) {
    // ------------------------------------- epilogue (+ A generation for K2)
    const int e = warp - kEpiWarp0;  // 0..7
    const int quarter = warp & 3;    // TMEM lane quarter this warp may access
    const int half = e >> 2;         // column half of the tile
    float tot[kTcMaxN / 2];
#pragma unroll
    for (int i = 0; i < kTcMaxN / 2; ++i) tot[i] = 0.0f;
    int drained = 0;
    if (kAMode == kAPhase) {
      const int gt = e * 32 + lane;  // generator thread 0..255
      const int r = gt & (kTcM - 1), gh = gt >> 7;
      const int j = m0 + r;
      int cur_pair = -1, ti = 0;
      float tf = 0.0f, sc = 1.0f, ss = 0.0f;
      for (int kb = 0; kb < p.num_kb; ++kb) {
        const int s = kb % kTcStages;
        mbar_wait(&bar->empty[s], ((kb / kTcStages) & 1) ^ 1);
        tc_gen_phase(p, a_hi(s), a_lo(s), r, gh, kb, j, cur_pair, ti, tf, sc, ss);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar->full[s]);
        // fold finished groups a few stages behind the producer front
        const int done_kb = kb - kTcStages;
        if (done_kb >= 0 && drained < num_groups &&
            (done_kb + 1) >= (drained + 1) * p.kb_per_group) {
          tc_drain(p, bar, tmem, drained, quarter, half, tot);
          ++drained;
        }
      }
    }
    for (; drained < num_groups; ++drained) tc_drain(p, bar, tmem, drained, quarter, half, tot);

    // ---- final: scale, store maps, fused per-frame argmax (lowest j on ties)
    const int j = m0 + 32 * quarter + lane;
    const bool jv = j < p.J;
    const int cbase = n0 + half * (p.N / 2);
#pragma unroll
    for (int i = 0; i < kTcMaxN / 2; ++i) {
      if (i < p.N / 2) {
        const int f = cbase + i;
        const float v = tot[i] * p.scale;
        if (f < p.F) {
          if (jv && p.maps) p.maps[static_cast<size_t>(f) * p.J + j] = v;
          if (p.keys) {
            const uint32_t bits = jv ? orderable_bits(v) : 0u;
            const uint32_t mx = __reduce_max_sync(0xffffffffu, bits);
            const uint32_t hit = __ballot_sync(0xffffffffu, jv && bits == mx);
            if (lane == 0 && hit != 0u) {
              const uint32_t jmin = static_cast<uint32_t>(m0 + 32 * quarter + __ffs(hit) - 1);
              atomicMax(p.keys + f, (static_cast<unsigned long long>(mx) << 32) |
                                        static_cast<unsigned long long>(0xFFFFFFFFu - jmin));
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// --------------------------------------------------------------------- host
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// Row-major fp32 matrix [rows, cols] -> tensor map with a (32 x box_rows)
// box and 128-byte swizzle (K-major UMMA operand tiles).
cudaError_t make_map(CUtensorMap* m, const float* base, int rows, int cols, int box_rows) {
  auto fn = encode_fn();
  if (fn == nullptr) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * sizeof(float)};
  cuuint32_t box[2] = {kTcKBlock, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Frames per tile: N-tiles of <= 160 frames, multiple of 32.
int pick_n(int F) {
  const int tiles = (F + kTcMaxN - 1) / kTcMaxN;
  const int per = (F + tiles - 1) / tiles;
  return (per + 31) / 32 * 32;
}

template <int kAMode>
cudaError_t launch_tc(const CUtensorMap& ah, const CUtensorMap& al, const CUtensorMap& bh,
                      const CUtensorMap& bl, const TcParams& p, cudaStream_t stream) {
  const size_t smem = tc_smem_bytes(p.N);
  cudaError_t e = cudaFuncSetAttribute(srp_tc_kernel<kAMode>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  dim3 grid((p.F + p.N - 1) / p.N, (p.J + kTcM - 1) / kTcM);
  srp_tc_kernel<kAMode><<<grid, kTcThreads, smem, stream>>>(ah, al, bh, bl, p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_conventional_tc(const float* psi_hi, const float* psi_lo, int F, int P, int Kb,
                                   int period, const int32_t* tau_i, const float* tau_f, int J,
                                   float* maps, unsigned long long* keys, int kb_per_group,
                                   cudaStream_t stream) {
  if (F == 0 || J == 0) return cudaSuccess;
  TcParams p{};
  p.F = F;
  p.J = J;
  p.N = pick_n(F);
  p.kb_per_pair = Kb / 16;
  p.num_kb = P * p.kb_per_pair;
  p.kb_per_group = max(kTcStages + 1, kb_per_group);
  p.scale = 2.0f;
  p.maps = maps;
  p.keys = keys;
  p.tau_i = tau_i;
  p.tau_f = tau_f;
  p.period = period;
  p.mask = (period & (period - 1)) == 0 ? period - 1 : 0;
  p.inv_period = 1.0f / static_cast<float>(period);
  CUtensorMap bh, bl;
  const int cols = 2 * P * Kb;
  cudaError_t e = make_map(&bh, psi_hi, F, cols, p.N);
  if (e == cudaSuccess) e = make_map(&bl, psi_lo, F, cols, p.N);
  if (e != cudaSuccess) return e;
  return launch_tc<kAPhase>(bh, bl, bh, bl, p, stream);
}

cudaError_t launch_interp_tc(const float* w_hi, const float* w_lo, const float* xi_hi,
                             const float* xi_lo, int F, int J, int T_pad, float* maps,
                             unsigned long long* keys, int kb_per_group, cudaStream_t stream) {
  if (F == 0 || J == 0) return cudaSuccess;
  TcParams p{};
  p.F = F;
  p.J = J;
  p.N = pick_n(F);
  p.num_kb = T_pad / kTcKBlock;
  p.kb_per_group = max(kTcStages + 1, kb_per_group);
  p.scale = 1.0f;
  p.maps = maps;
  p.keys = keys;
  CUtensorMap ah, al, bh, bl;
  cudaError_t e = make_map(&ah, w_hi, J, T_pad, kTcM);
  if (e == cudaSuccess) e = make_map(&al, w_lo, J, T_pad, kTcM);
  if (e == cudaSuccess) e = make_map(&bh, xi_hi, F, T_pad, p.N);
  if (e == cudaSuccess) e = make_map(&bl, xi_lo, F, T_pad, p.N);
  if (e != cudaSuccess) return e;
  return launch_tc<kAFromTma>(ah, al, bh, bl, p, stream);
}

// hi = tf32(x), lo = tf32(x - hi): operand split for 3xTF32
__global__ void tf32_split_kernel(const float4* __restrict__ x, size_t n4, float4* __restrict__ hi,
                                  float4* __restrict__ lo) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4;
       i += size_t(gridDim.x) * blockDim.x) {
    const float4 v = x[i];
    float4 h, l;
    h.x = to_tf32(v.x);
    h.y = to_tf32(v.y);
    h.z = to_tf32(v.z);
    h.w = to_tf32(v.w);
    l.x = to_tf32(v.x - h.x);
    l.y = to_tf32(v.y - h.y);
    l.z = to_tf32(v.z - h.z);
    l.w = to_tf32(v.w - h.w);
    hi[i] = h;
    lo[i] = l;
  }
}

cudaError_t launch_tf32_split(const float* x, size_t n, float* hi, float* lo, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const size_t n4 = n / 4;
  const size_t want = (n4 + 255) / 256;
  const int blocks = static_cast<int>(want < size_t(8 * kNumSMs) ? want : size_t(8 * kNumSMs));
  tf32_split_kernel<<<blocks, 256, 0, stream>>>(reinterpret_cast<const float4*>(x), n4,
                                                reinterpret_cast<float4*>(hi),
                                                reinterpret_cast<float4*>(lo));
  return cudaGetLastError();
}

}  // namespace srpb
