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
// (lo*hi + hi*lo + hi*hi) into the same TMEM accumulator (residual ~2^-22).
// The tensor core's fp32 accumulation is not round-to-nearest: over a long
// chain the accumulator drifts toward zero (measured: -1.4e-5 relative after
// 384 K steps x 3 MMAs at C1).  The contraction is therefore cut into groups
// of a few K blocks; each group accumulates in one of two TMEM buffers
// (ping-pong) and the epilogue warps fold it into round-to-nearest fp32
// register totals while the MMA continues into the other buffer.
//
// Persistent: one CTA per SM loops over 128-candidate x N-frame output tiles
// (N <= 160, multiple of 32; frame tile fastest so concurrently running CTAs
// share A tiles in L2).  Stage/phase and TMEM-group counters run across
// tiles, so a tile's final map/argmax write overlaps the next tile's MMAs.
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

// Instrumentation build only (make prof -> libsrpb_prof.so, tools/tc_probe.py):
// per-role cycle counters; compiled out of libsrpb.so.
#ifdef SRPB_TC_PROFILE
__device__ unsigned long long g_tc_prof[16];
#define TCP_DECL(v) long long v = 0
#define TCP_T0() const long long _tcp0 = clock64()
#define TCP_ACC(v) (v += clock64() - _tcp0)
#define TCP_FLUSH(i, v) atomicAdd(&g_tc_prof[i], static_cast<unsigned long long>(v))
#else
#define TCP_DECL(v)
#define TCP_T0()
#define TCP_ACC(v)
#define TCP_FLUSH(i, v)
#endif

struct TcParams {
  int F, J, N;        // frames, candidates, frames per tile
  int n_tiles;        // frame tiles
  int num_tiles;      // n_tiles * candidate tiles
  int num_kb;         // K blocks of 32 per tile
  int kb_per_group;   // TMEM drain period (K blocks)
  int groups_per_tile;
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
  unsigned long long tile_keys[4 * kTcMaxN];  // per-quarter, per-frame tile argmax
  uint32_t tmem_base;
};

// K4 stages hold A and B in smem; K2 stages hold only B (A lives in TMEM).
__host__ __device__ inline size_t tc_stage_bytes(int N, bool a_in_smem) {
  return (a_in_smem ? 2 * kABytes : 0) + 2 * size_t(N) * 128;
}
__host__ __device__ inline size_t tc_smem_bytes(int N, bool a_in_smem) {
  return 1024 /*align slack*/ + kTcStages * tc_stage_bytes(N, a_in_smem) + sizeof(TcSmem);
}
// TMEM columns: accumulators [0, 2N); K2's A stages (hi 32 + lo 32 columns
// each) from column 2N: 2N + 64 * kTcStages <= 512 for N <= 160.
__host__ __device__ constexpr int tc_a_tmem_col(int N, int s) { return 2 * N + 64 * s; }

// Fold TMEM accumulator buffer of global group `g` into this thread's totals:
// row = 32*(warp%4) + lane, columns [half*N/2, half*N/2 + N/2).
__device__ __forceinline__ void tc_drain(const TcParams& p, TcSmem* bar, uint32_t tmem, int g,
                                         int quarter, int half, float (&tot)[kTcMaxN / 2]) {
  const int b = g & 1;
  mbar_wait(&bar->acc_full[b], (g >> 1) & 1);
  tc_fence_after();
  const uint32_t base = tmem + (static_cast<uint32_t>(32 * quarter) << 16) +
                        static_cast<uint32_t>(b * p.N + half * (p.N / 2));
  const int nchunks = p.N / 32;  // 16-column loads per half
  // two 16-column loads in flight per wait (register budget: 384 threads/SM)
#pragma unroll
  for (int c = 0; c < kTcMaxN / 32; c += 2) {
    if (c < nchunks) {
      uint32_t r0[16], r1[16];
      tmem_ld16(base + 16 * c, r0);
      if (c + 1 < nchunks) tmem_ld16(base + 16 * (c + 1), r1);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 16; ++i) tot[16 * c + i] += __uint_as_float(r0[i]);
      if (c + 1 < nchunks) {
#pragma unroll
        for (int i = 0; i < 16; ++i) tot[16 * (c + 1) + i] += __uint_as_float(r1[i]);
      }
    }
  }
  tc_fence_before();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(&bar->acc_empty[b]);
}

// Final output of one tile: scale, store maps, fused per-frame argmax
// (lowest j on ties), then reset the totals for the next tile.  The four
// lane-quarter warps of a column half combine their warp maxima in shared
// memory (tile_keys, double-buffered by tile parity) so each tile issues one
// global 64-bit atomicMax per frame instead of four.
__device__ __forceinline__ void tc_write_tile(const TcParams& p, TcSmem* bar, int tile_parity,
                                              int m0, int n0, int quarter, int half, int lane,
                                              float (&tot)[kTcMaxN / 2]) {
  const int j = m0 + 32 * quarter + lane;
  const bool jv = j < p.J;
  const int cbase = half * (p.N / 2);
  unsigned long long* tk = bar->tile_keys;  // [4 quarters][kTcMaxN columns]
  (void)tile_parity;
#pragma unroll
  for (int i = 0; i < kTcMaxN / 2; ++i) {
    if (i < p.N / 2) {
      const int f = n0 + cbase + i;
      const float v = tot[i] * p.scale;
      tot[i] = 0.0f;
      if (f < p.F) {
        if (jv && p.maps) p.maps[static_cast<size_t>(f) * p.J + j] = v;
        if (p.keys) {
          const uint32_t bits = jv ? orderable_bits(v) : 0u;
          const uint32_t mx = __reduce_max_sync(0xffffffffu, bits);
          const uint32_t hit = __ballot_sync(0xffffffffu, jv && bits == mx);
          if (lane == 0) {  // this quarter's best for column cbase + i (0 = none)
            const uint32_t jmin = static_cast<uint32_t>(m0 + 32 * quarter + __ffs(hit) - 1);
            tk[quarter * kTcMaxN + cbase + i] =
                hit != 0u ? (static_cast<unsigned long long>(mx) << 32) |
                                static_cast<unsigned long long>(0xFFFFFFFFu - jmin)
                          : 0ull;
          }
        }
      }
    }
  }
  if (p.keys) {
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
    const int et = threadIdx.x - kEpiWarp0 * 32;  // 0..255
    for (int c = et; c < p.N; c += kEpiWarps * 32) {
      unsigned long long k = tk[c];
#pragma unroll
      for (int q = 1; q < 4; ++q) k = key_max(k, tk[q * kTcMaxN + c]);
      const int f = n0 + c;
      if (k != 0ull && f < p.F) atomicMax(p.keys + f, k);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");  // tk reusable
  }
}

// A tile of steering phases for K block kb: candidate row j (TMEM lane of
// this thread), bins [k0 + 8*half, +8) of the block's pair, as (cos, -sin)
// pairs, split hi/lo.  a_*_tmem carry this warp's lane quarter.
__device__ __forceinline__ void tc_gen_phase(const TcParams& p, uint32_t a_hi_tmem,
                                             uint32_t a_lo_tmem, int half, int kb, int j,
                                             int& cur_pair, int& ti, float& tf, float& sc,
                                             float& ss) {
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
  // tf32 split, straight into the TMEM A operand of this stage: this thread's
  // lane (row r), columns [16*half, +16) of the 32-column K block.
  uint32_t hi[16], lo[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float h = to_tf32(v[i]);
    hi[i] = __float_as_uint(h);
    lo[i] = __float_as_uint(to_tf32(v[i] - h));
  }
  tmem_st16(a_hi_tmem + 16 * half, hi);
  tmem_st16(a_lo_tmem + 16 * half, lo);
}

// Exact round-to-nearest (ties away) of a finite fp32 to tf32, in two integer
// ops; x - tf32_rna(x) is exact in fp32.
__device__ __forceinline__ uint32_t tf32_rna_bits(float x) {
  return (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;
}

// Steering-phase generator of one A row (candidate j) and one half of every
// 32-column K block (8 bins).  Per pair: the one-bin and 16-bin rotations
// e^{j2pi x/N}, e^{j2pi 16x/N} from exact turn arithmetic; per block: the
// anchor phase, exact (integer-reduced turns + sincospif) every 4th block and
// otherwise the previous anchor rotated by 16 bins; then 7 one-bin rotations.
// Longest rotation chain: 3 x 16-bin + 7 x 1-bin, ~1e-6 relative phase error.
struct PhaseGen {
  int kbp, left;  // K blocks per pair, blocks left in the current pair
  int pair, ti;
  float tf, sc, ss, s16c, s16s, ac, as;
  int since_exact;

  __device__ __forceinline__ void start_tile(const TcParams& p) {
    kbp = p.kb_per_pair;
    left = 0;
    pair = -1;
  }

  __device__ __forceinline__ void block(const TcParams& p, int j, int half, uint32_t a_hi_tmem,
                                        uint32_t a_lo_tmem) {
    if (left == 0) {  // next pair
      ++pair;
      left = kbp;
      ti = 0;
      tf = 0.0f;
      if (j < p.J) {
        ti = p.tau_i[static_cast<size_t>(pair) * p.J + j];
        tf = p.tau_f[static_cast<size_t>(pair) * p.J + j];
      }
      sincospif(2.0f * (static_cast<float>(ti) + tf) * p.inv_period, &ss, &sc);
      const float t16 = harmonic_turns(16, ti, tf, p.period, p.mask, p.inv_period);
      sincospif(2.0f * t16, &s16s, &s16c);
      since_exact = 4;
    }
    const int k = (kbp - left) * 16 + 8 * half;
    if (since_exact >= 4) {
      harmonic_phase(k, ti, tf, p.period, p.mask, p.inv_period, &ac, &as);
      since_exact = 0;
    } else {
      const float cn = ac * s16c - as * s16s;
      as = fmaf(ac, s16s, as * s16c);
      ac = cn;
    }
    ++since_exact;
    --left;
    float c = ac, s = as;
    uint32_t hi[16], lo[16];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const float ns = -s;
      const uint32_t hc = tf32_rna_bits(c), hs = tf32_rna_bits(ns);
      hi[2 * m] = hc;
      hi[2 * m + 1] = hs;
      lo[2 * m] = __float_as_uint(c - __uint_as_float(hc));
      lo[2 * m + 1] = __float_as_uint(ns - __uint_as_float(hs));
      const float cn = c * sc - s * ss;  // rotate by one bin
      s = fmaf(c, ss, s * sc);
      c = cn;
    }
    tmem_st16(a_hi_tmem + 16 * half, hi);
    tmem_st16(a_lo_tmem + 16 * half, lo);
  }
};

template <int kAMode>
__global__ void __launch_bounds__(kTcThreads, 1)
srp_tc_kernel(const __grid_constant__ CUtensorMap tmA_hi, const __grid_constant__ CUtensorMap tmA_lo,
              const __grid_constant__ CUtensorMap tmB_hi, const __grid_constant__ CUtensorMap tmB_lo,
              const TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  constexpr bool kASmem = kAMode == kAFromTma;
  const size_t stage_bytes = tc_stage_bytes(p.N, kASmem);
  TcSmem* bar = reinterpret_cast<TcSmem*>(smem + kTcStages * stage_bytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t b_bytes = static_cast<uint32_t>(p.N) * 128;
  // tiles of this CTA: t = blockIdx.x + it * gridDim.x
  const int my_tiles =
      p.num_tiles > static_cast<int>(blockIdx.x)
          ? (p.num_tiles - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
          : 0;
  auto tile_m0 = [&](int it) {
    return ((static_cast<int>(blockIdx.x) + it * static_cast<int>(gridDim.x)) / p.n_tiles) * kTcM;
  };
  auto tile_n0 = [&](int it) {
    return ((static_cast<int>(blockIdx.x) + it * static_cast<int>(gridDim.x)) % p.n_tiles) * p.N;
  };

  const size_t a_bytes = kASmem ? 2 * kABytes : 0;
  auto a_hi = [&](int s) { return smem + s * stage_bytes; };
  auto a_lo = [&](int s) { return smem + s * stage_bytes + kABytes; };
  auto b_hi = [&](int s) { return smem + s * stage_bytes + a_bytes; };
  auto b_lo = [&](int s) { return smem + s * stage_bytes + a_bytes + b_bytes; };

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
    for (int c = 0; c < 4 * kTcMaxN; ++c) bar->tile_keys[c] = 0ull;
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // make the TMEM base provably warp-uniform (it stays in a uniform register)
  const uint32_t tmem = __shfl_sync(0xffffffffu, bar->tmem_base, 0);

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // warp-wide loop, one elected lane issues (uniform operands, no per-issue
    // register broadcasts)
    const uint32_t tx = 2 * b_bytes + (kAMode == kAFromTma ? 2 * kABytes : 0);
    int kg = 0;
    TCP_DECL(w_empty);
    TCP_DECL(t_all);
    { TCP_T0();
    for (int it = 0; it < my_tiles; ++it) {
      const int m0 = tile_m0(it), n0 = tile_n0(it);
      for (int kb = 0; kb < p.num_kb; ++kb, ++kg) {
        const int s = kg % kTcStages;
        { TCP_T0();
        mbar_wait(&bar->empty[s], ((kg / kTcStages) & 1) ^ 1);
        TCP_ACC(w_empty); }
        if (elect_one()) {
          mbar_expect_tx(&bar->full[s], tx);
          tma_load_2d(b_hi(s), &tmB_hi, &bar->full[s], kb * kTcKBlock, n0);
          tma_load_2d(b_lo(s), &tmB_lo, &bar->full[s], kb * kTcKBlock, n0);
          if (kAMode == kAFromTma) {
            tma_load_2d(a_hi(s), &tmA_hi, &bar->full[s], kb * kTcKBlock, m0);
            tma_load_2d(a_lo(s), &tmA_lo, &bar->full[s], kb * kTcKBlock, m0);
          }
        }
        __syncwarp();
      }
    }
    TCP_ACC(t_all); }
    if (lane == 0) {
      TCP_FLUSH(3, w_empty);
      TCP_FLUSH(4, t_all);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    // warp-wide loop; descriptors are base + byte-offset>>4 arithmetic on
    // uniform values; one elected lane issues the MMAs and their commits.
    const uint32_t idesc = idesc_tf32(kTcM, p.N);
    const uint64_t db0 = sw128_kmajor_desc(smem_u32(b_hi(0)));  // stage 0 B_hi
    const uint64_t da0 = sw128_kmajor_desc(smem_u32(a_hi(0)));  // stage 0 A_hi (K4)
    const uint32_t stage16 = static_cast<uint32_t>(stage_bytes >> 4);
    const uint32_t b16 = b_bytes >> 4, a16 = kABytes >> 4;
    int kg = 0;
    TCP_DECL(w_full);
    TCP_DECL(w_acc);
    TCP_DECL(t_all);
    { TCP_T0();
    for (int it = 0; it < my_tiles; ++it) {
      for (int kb = 0; kb < p.num_kb; ++kb, ++kg) {
        const int s = kg % kTcStages;
        const int gl = kb / p.kb_per_group;                 // group within the tile
        const int g = it * p.groups_per_tile + gl;          // global group
        const int in_group = kb - gl * p.kb_per_group;
        const uint32_t d = tmem + static_cast<uint32_t>((g & 1) * p.N);
        if (in_group == 0) {
          TCP_T0();
          mbar_wait(&bar->acc_empty[g & 1], ((g >> 1) & 1) ^ 1);
          TCP_ACC(w_acc);
          tc_fence_after();
        }
        { TCP_T0();
        mbar_wait(&bar->full[s], (kg / kTcStages) & 1);
        TCP_ACC(w_full); }
        tc_fence_after();
        const uint64_t bh = db0 + static_cast<uint64_t>(s * stage16);
        const uint64_t bl = bh + b16;
        if (elect_one()) {
          if (kASmem) {  // K4: A from smem (SS)
            const uint64_t ah = da0 + static_cast<uint64_t>(s * stage16);
            const uint64_t al = ah + a16;
#pragma unroll
            for (int ks = 0; ks < kTcKBlock / 8; ++ks) {
              const uint32_t o = 2 * ks;  // 32 bytes along K, in 16-byte units
              const uint32_t acc0 = (in_group > 0 || ks > 0) ? 1u : 0u;
              mma_tf32(d, al + o, bh + o, idesc, acc0);
              mma_tf32(d, ah + o, bl + o, idesc, 1u);
              mma_tf32(d, ah + o, bh + o, idesc, 1u);
            }
          } else {  // K2: A from TMEM (TS), written there by the generator warps
            const uint32_t ah = tmem + static_cast<uint32_t>(tc_a_tmem_col(p.N, s));
            const uint32_t al = ah + 32;
#pragma unroll
            for (int ks = 0; ks < kTcKBlock / 8; ++ks) {
              const uint32_t o = 2 * ks;
              const uint32_t acc0 = (in_group > 0 || ks > 0) ? 1u : 0u;
              mma_tf32_ts(d, al + 8 * ks, bh + o, idesc, acc0);
              mma_tf32_ts(d, ah + 8 * ks, bl + o, idesc, 1u);
              mma_tf32_ts(d, ah + 8 * ks, bh + o, idesc, 1u);
            }
          }
          mma_commit(&bar->empty[s]);
          if (in_group == p.kb_per_group - 1 || kb == p.num_kb - 1)
            mma_commit(&bar->acc_full[g & 1]);
        }
        __syncwarp();
      }
    }
    TCP_ACC(t_all); }
    if (lane == 0) {
      TCP_FLUSH(0, t_all);
      TCP_FLUSH(1, w_full);
      TCP_FLUSH(2, w_acc);
      TCP_FLUSH(11, 1);
    }
  } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + kEpiWarps) {
    // ------------------------------------- epilogue (+ A generation for K2)
    const int e = warp - kEpiWarp0;  // 0..7
    const int quarter = warp & 3;    // TMEM lane quarter this warp may access
    const int half = e >> 2;         // column half of the tile
    float tot[kTcMaxN / 2];
#pragma unroll
    for (int i = 0; i < kTcMaxN / 2; ++i) tot[i] = 0.0f;
    const int total_groups = my_tiles * p.groups_per_tile;
    int drained = 0;  // next global group to fold
    // incremental position of group `drained`: its tile, index in the tile,
    // and the global K block index of its last block (no divisions)
    int d_it = 0, d_gl = 0;
    int d_last_kg = min(p.kb_per_group, p.num_kb) - 1;
    TCP_DECL(c_gen_wait);
    TCP_DECL(c_gen);
    TCP_DECL(c_drain);
    TCP_DECL(c_write);
    TCP_DECL(c_all);
    auto fold_next = [&]() {
      { TCP_T0();
      tc_drain(p, bar, tmem, drained, quarter, half, tot);
      TCP_ACC(c_drain); }
      if (d_gl == p.groups_per_tile - 1) {
        TCP_T0();
        tc_write_tile(p, bar, d_it & 1, tile_m0(d_it), tile_n0(d_it), quarter, half, lane, tot);
        TCP_ACC(c_write);
        ++d_it;
        d_gl = 0;
        d_last_kg = d_it * p.num_kb + min(p.kb_per_group, p.num_kb) - 1;
      } else {
        ++d_gl;
        d_last_kg = d_it * p.num_kb + min((d_gl + 1) * p.kb_per_group, p.num_kb) - 1;
      }
      ++drained;
    };
    { TCP_T0();
    if (kAMode == kAPhase) {
      // generator thread: TMEM lane (row) 32*quarter + lane, K columns
      // [16*half, +16) of each 32-column A block
      const int r = 32 * quarter + lane;
      const uint32_t lane_base = tmem + (static_cast<uint32_t>(32 * quarter) << 16);
      PhaseGen gen;
      int kg = 0, s = 0, ph = 0;  // stage ring position
      for (int it = 0; it < my_tiles; ++it) {
        const int j = tile_m0(it) + r;
        gen.start_tile(p);
        for (int kb = 0; kb < p.num_kb; ++kb, ++kg) {
          { TCP_T0();
          mbar_wait(&bar->empty[s], ph ^ 1);
          TCP_ACC(c_gen_wait); }
          { TCP_T0();
          tc_fence_after();  // MMAs that read this stage have completed
          const uint32_t a_col = lane_base + static_cast<uint32_t>(tc_a_tmem_col(p.N, s));
          gen.block(p, j, half, a_col, a_col + 32);
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          TCP_ACC(c_gen); }
          if (lane == 0) mbar_arrive(&bar->full[s]);
          if (++s == kTcStages) {
            s = 0;
            ph ^= 1;
          }
          // fold groups whose last K block is at least kTcStages behind
          while (drained < total_groups && d_last_kg <= kg - kTcStages) fold_next();
        }
      }
    }
    while (drained < total_groups) fold_next();
    TCP_ACC(c_all); }
    if (warp == kEpiWarp0 && lane == 0) {
      TCP_FLUSH(5, c_gen_wait);
      TCP_FLUSH(6, c_gen);
      TCP_FLUSH(7, c_drain);
      TCP_FLUSH(9, c_write);
      TCP_FLUSH(10, c_all);
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

void finish_params(TcParams& p, int kb_per_group) {
  p.N = pick_n(p.F);
  p.n_tiles = (p.F + p.N - 1) / p.N;
  p.num_tiles = p.n_tiles * ((p.J + kTcM - 1) / kTcM);
  p.kb_per_group = max(kTcStages + 1, kb_per_group);
  p.groups_per_tile = (p.num_kb + p.kb_per_group - 1) / p.kb_per_group;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = kNumSMs;
  }
  return n;
}

template <int kAMode>
cudaError_t launch_tc(const CUtensorMap& ah, const CUtensorMap& al, const CUtensorMap& bh,
                      const CUtensorMap& bl, const TcParams& p, cudaStream_t stream) {
  const size_t smem = tc_smem_bytes(p.N, kAMode == kAFromTma);
  cudaError_t e = cudaFuncSetAttribute(srp_tc_kernel<kAMode>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int grid = min(p.num_tiles, num_sms());
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
  p.kb_per_pair = Kb / 16;
  p.num_kb = P * p.kb_per_pair;
  finish_params(p, kb_per_group);
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
  p.num_kb = T_pad / kTcKBlock;
  finish_params(p, kb_per_group);
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

#ifdef SRPB_TC_PROFILE
// instrumentation build only: copy out and clear the 16 role counters
extern "C" int srpb_tc_profile_read(unsigned long long* host16) {
  cudaError_t e = cudaMemcpyFromSymbol(host16, srpb::g_tc_prof, sizeof(unsigned long long) * 16);
  unsigned long long zero[16] = {};
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(srpb::g_tc_prof, zero, sizeof(zero));
  return static_cast<int>(e);
}
#endif
