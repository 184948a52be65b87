// Tensor-core (tcgen05; 3xFP16 kind::f16 or 3xTF32 kind::tf32) SRP
// contractions for sm_100a.
//
//   maps[f, j] = scale * sum_kk A[j, kk] B[f, kk]
//
// K2 (conventional, srp.py:391-429): A = steering phases [cos, -sin] generated
//    on the fly by SIMT warps straight into tensor memory (never stored in
//    HBM or smem), B = Psi [F, 2 P Kb] (float view of the cross-spectra),
//    scale 2.
// K4 (approximate, srp.py:320-347): A = W [J, T_pad] sinc weights, B = Xi
//    [F, T_pad] lattice samples, both streamed by TMA, scale 1.
//
// fp32 accuracy from 16-bit-significand tensor cores: every operand is
// pre-split into hi = r(x), lo = r(x - hi) and each K step issues three MMAs
// (lo*hi + hi*lo + hi*hi) into the same TMEM accumulator (residual ~2^-22;
// the hi*hi, hi*lo, lo*hi products are exact in fp32).  kF16: r = fp16 with
// a power-of-two prescale that keeps every operand inside fp16's range
// (steering phases and sinc weights |x| <= 1 -> 2^14; PHAT cross-spectra
// |psi| <= 1 -> 2^14; lattice samples |xi| <= 2 Kb); fp16 has tf32's 11-bit
// significand, so the split is as accurate as 3xTF32, but kind::f16 runs at
// twice the kind::tf32 rate and moves half the operand bytes.  A 128-byte
// swizzle row holds 64 fp16 (32 tf32) and each MMA consumes 32 bytes of K in
// both kinds, so descriptors, stages and TMEM A tiles are byte-identical.
// Otherwise (identity weighting: unbounded cross-spectra) r = tf32.
// The tensor core's fp32 accumulation is not round-to-nearest: over a long
// chain the accumulator drifts toward zero (measured: -1.4e-5 relative after
// 384 K steps x 3 MMAs at C1).  The contraction is therefore cut into groups
// of a few K blocks; each group accumulates in one of two TMEM buffers
// (ping-pong) and the epilogue warps fold it into round-to-nearest fp32
// register totals while the MMA continues into the other buffer.
//
// CTA pairs (cta_group::2, kPair): the per-SM TMA ingress ceiling measured on
// B200 is ~45-50 B/clk (tools/tma_bench.cu), below what a single-CTA 3xTF32
// tile needs (K2: 42 B/clk of B; K4: 75 B/clk).  A CTA pair computes a
// 256-candidate x N-frame tile with one M=256 MMA issued by the leader; each
// CTA holds its own 128 rows of A and HALF of B's rows, so per-SM B ingress
// halves.  Both CTAs' TMA loads and A-generators signal the leader's `full`
// barrier; the leader's commits multicast to both CTAs' `empty`/`acc_full`;
// both CTAs' epilogues release the leader's `acc_empty`.
//
// Persistent: one CTA (pair) per SM (pair) loops over tiles, frame tile
// fastest so concurrently running CTAs share A tiles in L2.  Stage/phase and
// TMEM-group counters run across tiles, so a tile's final map/argmax write
// overlaps the next tile's MMAs.
//   warp 0      TMA producer                              elected lane
//   warp 1      TMEM allocator + MMA issuer (leader)      elected lane
//   warps 4..11 epilogue: TMEM drains, map store, fused argmax; for K2 they
//               also generate the A tiles (2 threads per candidate row)
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "tmap.cuh"
#include "umma.cuh"

namespace srpb {

using namespace umma;

constexpr int kTcThreads = 384;
constexpr int kTcMaxStages = 8;
constexpr int kTcM = 128;            // candidate rows per CTA
constexpr int kTcMaxN = 160;
// generator modes (shared-memory totals, no register tiles): up to 192 frames
// per tile (TMEM 2 x 192 accumulators + 2 A stages)
constexpr int kTcMaxNGen = 192;
constexpr int kTcKBlock = 32;        // tf32 elements per K block = one 128-B swizzle row
constexpr int kTcKBlock16 = 64;      // fp16 elements per K block
constexpr float kF16PhaseScale = 16384.0f;  // 2^14: steering phases / sinc weights
constexpr int kEpiWarp0 = 4;
constexpr int kEpiWarps = 8;
constexpr int kABytes = kTcM * 128;  // one of A_hi / A_lo per stage

enum : int { kAFromTma = 0, kAPhase = 1, kASinc = 2, kALoad = 3 };

#ifndef SRPB_K4_STAGES
#define SRPB_K4_STAGES 4
#endif

template <int kAMode, bool kPair, bool kF16>
struct TcCfg {
  // smem stages: K4 pairs take 4 x (32 KB A + N/2 rows of B hi/lo) plus the
  // 16 KB epilogue staging (227 KB total); K2 is bounded by its A stages in
  // TMEM (2N + 64 S <= 512)
  static constexpr int kStages = (kAMode == kAFromTma && kPair) ? SRPB_K4_STAGES : 3;
  // K4 pairs: maps leave through shared memory (TMA store) and the argmax
  // reads the staged tile transposed
  static constexpr bool kEpiStage = kAMode == kAFromTma && kPair;
  static constexpr bool kASmem = kAMode == kAFromTma;
  static constexpr int kKbElems = kF16 ? kTcKBlock16 : kTcKBlock;  // elements per K block
  // generator modes keep the folded running totals in shared memory
  // (registers go to the A generator)
  static constexpr bool kTotSmem = kAMode != kAFromTma;
  // Generator teams (on-the-fly K4, single-CTA tiles): two teams of 8
  // generator warps take alternate K blocks, so two blocks' weights are in
  // production at once (one team per block: the MMA waited on a single team
  // ~20% of the time, tools/tc_probe_c4.py); each team folds and writes its
  // own 16-column accumulator chunks straight from the shared totals.  Warp
  // roles: generators 0..15 (TMEM lane quarter = warp % 4), TMA producer 16,
  // MMA issuer 17.  Otherwise: producer 0, MMA 1, epilogue warps 4..11.
  static constexpr int kTeams = kAMode != kAFromTma ? 2 : 1;
  static constexpr int kGenW0 = kTeams == 2 ? 0 : kEpiWarp0;  // first epilogue / generator warp
  static constexpr int kGenWarps = kEpiWarps * kTeams;
  static constexpr int kProdWarp = kTeams == 2 ? kGenWarps : 0;
  static constexpr int kMmaWarp = kTeams == 2 ? kGenWarps + 1 : 1;
  static constexpr int kThreads = kTeams == 2 ? 32 * (kGenWarps + 2) : kTcThreads;
  static constexpr int kItemRing = kTotSmem ? 32 : 8;  // see TcSmemT
};

// Instrumentation build only (make prof -> libsrpb_prof.so, tools/tc_probe.py):
// per-role cycle counters; compiled out of libsrpb.so.
#ifdef SRPB_TC_PROFILE
__device__ unsigned long long g_tc_prof[24];
// per-CTA event timeline (globaltimer ns): [cta][5 item + e], e = 0 producer
// starts the item, 1 first stage ready at the MMA, 2 last MMA issued, 3 drain
// starts (accumulator full), 4 item written; [cta][60] entry, [61] exit
__device__ unsigned long long g_tc_trace[160][64];
__device__ __forceinline__ void tc_trace(int it, int e) {
  if (it < 12) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tc_trace[blockIdx.x][it * 5 + e] = t;
  }
}
#define TCT(it, e) tc_trace(it, e)
#define TCP_DECL(v) long long v = 0
#define TCP_T0() const long long _tcp0 = clock64()
#define TCP_ACC(v) (v += clock64() - _tcp0)
#define TCP_FLUSH(i, v) atomicAdd(&g_tc_prof[i], static_cast<unsigned long long>(v))
#define TC_DBG(prm) ((prm).dbg)
#else
// bound-analysis switches (SRPB_TC_DBG) exist in the instrumentation build
// only: the product kernels carry no per-block flag tests
#define TC_DBG(prm) 0
#define TCP_DECL(v)
#define TCP_T0()
#define TCP_ACC(v)
#define TCP_FLUSH(i, v)
#define TCT(it, e)
#endif

struct TcParams {
  int F, J, N;        // frames, candidates, frames per tile
  int n_tiles;        // frame tiles
  int num_items;      // n_tiles * candidate tiles (of 128, or 256 per pair)
  int full_items;     // items run at full width; the tail wave's items are split
  int n_piece0;       // frames of a split item's pieces (the last: N - (k - 1) n_piece0)
  int n_pieces;       // pieces k per split item
  int n_last;         // frames of the last frame tile (multiple of 32, <= N): the
                      // tiles are N wide except the last, which covers only the
                      // remaining frames (C4: 25 x 160 + 96, not 26 x 160)
  int total_items;    // full_items + k * (num_items - full_items)
  int num_kb;         // K blocks of 32 per tile
  int maps_tma;       // staged epilogue: maps stored by TMA (J % 4 == 0), else st.global
  int stages;         // K4 (A by TMA): smem stages that fit the tile width
  int dbg;            // experiments only (SRPB_TC_DBG): 1 = A rows mod 2048
  int b_box;          // rows per B TMA box: this CTA's full B buffer (N, or N/2 per pair)
  int kb_per_group;   // TMEM drain period (K blocks)
  int groups_per_tile;  // num_kb / kb_per_group: the last group also takes the
                        // remainder (a short tail group could stall the
                        // generator modes' fold, see enforce_fold_window)
  int m_units;        // candidate tiles (of 128, or 256 per pair)
  int m_fast;         // item order: 1 = candidate tile fastest (all CTAs share a
                      // frame tile's B rows in L2), 0 = frame tile fastest
  int lockstep;       // static items only: a CTA starts round r's item once
                      // every CTA has issued its round r - 1 loads (done[1]
                      // counts them), keeping the wave within L2 of each other
  int dynamic;        // 1: items from the global cursor; 0: static round-robin
                      // (many waves: the CTAs of a wave start together and run
                      // identical items in lockstep, so they stream one B tile
                      // through L2 once instead of each reading it from DRAM)
  float scale;
  float* maps;
  unsigned long long* keys;
  // optional in-kernel argmax finish: the last CTA decodes keys -> argmax_out
  // and resets keys and the counter for the next call
  int32_t* argmax_out;
  // done[0]: CTAs finished; done[1]: dynamic item cursor (both reset to 0 by
  // the last CTA).  NULL: static round-robin items, no finish.
  unsigned int* done;
  // K2 phase generation
  const int32_t* tau_i;
  const float* tau_f;
  int kb_per_pair;    // Kb / 16
  int period, mask;
  float inv_period;
  // K4 with sinc weights generated on the fly (kASinc)
  const int32_t* sx_i;   // [P, J]
  const float* sx_f;     // [P, J]
  const int32_t* off;    // [P + 1] lattice column offsets
  const int32_t* reach;  // [P]
  int P;
  // K4 with the stored fp16 W split loaded by the generator warps into TMEM
  // (kALoad): rows of T_pad halves
  const __half* w_hi;
  const __half* w_lo;
  int T_pad;
};

// Work-item ids in flight between the roles.  A generator warp releases an
// item only when it has folded the item's last group, which may trail its
// generation by S + 2 groups, and the two teams and the MMA stay within S
// blocks of each other: with one-block tiles the producer can be 2 S + 2
// items ahead of the slowest release (S <= 8), so generator modes ring 32
// ids.  The stored-weight K4 (epilogue warps release after their drain) keeps
// 8: its 4 x 52 KB stages + staging leave no room.
template <int kRing>
struct TcSmemT {
  uint64_t full[kTcMaxStages];
  uint64_t empty[kTcMaxStages];
  uint64_t acc_full[2];
  uint64_t acc_empty[2];
  uint64_t item_full[kRing];   // ring slot holds the next item id (each CTA)
  uint64_t item_empty[kRing];  // every consumer is done with the slot (leader)
  int item_ring[kRing];
  int4 item_cache[kRing > 8 ? 16 : 1];  // generator modes: per warp, the item its fold is on
  uint32_t tmem_base;
};


// Per-CTA smem stage: A hi/lo (K4) + this CTA's B rows (all N, or N/2 per pair).
__host__ __device__ inline size_t tc_stage_bytes(int N, bool a_in_smem, bool pair) {
  return (a_in_smem ? 2 * kABytes : 0) + 2 * size_t(pair ? N / 2 : N) * 128;
}
// staged epilogue (K4 pairs): per epilogue warp two 2 KB buffers of 16
// frames x 32 candidates (fp32, TMA 128-byte swizzle)
constexpr int kEpiChunk = 8;  // frames per staged chunk (one 1 KB swizzle atom)
constexpr int kEpiStageBytes = kEpiChunk * 128;
constexpr int kEpiStageTotal = kEpiWarps * 2 * kEpiStageBytes;
// other kernels: per-quarter, per-frame tile argmax keys [4][kTcMaxN]
constexpr int kTileKeysBytes = 4 * kTcMaxNGen * 8;
// generator modes: running totals [2 halves x N / 2 columns][128 rows]
__host__ __device__ inline size_t tot_smem_bytes(int N) { return size_t(N) * kTcM * 4; }
__host__ __device__ inline size_t tc_smem_bytes(int N, bool a_in_smem, bool pair, int stages,
                                                bool epi_stage = false, bool tot_smem = false) {
  return 1024 /*align slack*/ + stages * tc_stage_bytes(N, a_in_smem, pair) +
         (tot_smem ? tot_smem_bytes(N) : 0) + (epi_stage ? kEpiStageTotal : kTileKeysBytes) +
         (tot_smem ? sizeof(TcSmemT<32>) : sizeof(TcSmemT<8>));
}
// TMEM columns: accumulators [0, 2N); K2's A stages (hi 32 + lo 32 columns
// each) from column 2N: 2N + 64 * 3 <= 512 for N <= 160.
__host__ __device__ constexpr int tc_a_tmem_col(int N, int s) { return 2 * N + 64 * s; }

// Fold TMEM accumulator buffer of global group `g` into this thread's totals:
// row = 32*(warp%4) + lane, columns [half*N/2, half*N/2 + N/2); release the
// buffer on `acc_empty_addr` (the leader's barrier for pairs).
template <class Bar>
__device__ __forceinline__ void tc_drain(const TcParams& p, Bar* bar, bool remote,
                                         uint32_t acc_empty_addr0, uint32_t tmem, int g, int nc,
                                         int quarter, int half, float (&tot)[kTcMaxN / 2]) {
  const int b = g & 1;
  mbar_wait(&bar->acc_full[b], (g >> 1) & 1);
  tc_fence_after();
  const uint32_t base = tmem + (static_cast<uint32_t>(32 * quarter) << 16) +
                        static_cast<uint32_t>(b * p.N + half * (nc / 2));
  const int nchunks = nc / 32;  // 16-column loads per half (nc: this item's frames)
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
  if ((threadIdx.x & 31) == 0) {
    if (remote)  // pair peer: the leader's barrier
      mbar_arrive_cluster(acc_empty_addr0 + 8u * b);
    else
      mbar_arrive(&bar->acc_empty[b]);
  }
}

// Shared-memory form (generator modes): chunk C folded into this thread's
// column slice of the running totals, layout [column][row] (lanes hit
// consecutive banks).
__device__ __forceinline__ void tc_drain_chunk16_smem(uint32_t base, float* tot_s, int c,
                                                      int dbg) {
  if (dbg & 16384) return;  // bound analysis only: no accumulator reads
  uint32_t r[16];
  tmem_ld16(base + 16 * c, r);
  tmem_wait_ld();
  float* t = tot_s + 16 * c * kTcM;
#pragma unroll
  for (int i = 0; i < 16; ++i) t[i * kTcM] += __uint_as_float(r[i]);
}

// One 16-column chunk C of a TMEM accumulator half folded into the totals
// (compile-time C keeps `tot` in registers).
template <int C>
__device__ __forceinline__ void tc_drain_chunk16(uint32_t base, float (&tot)[kTcMaxN / 2]) {
  if constexpr (16 * C < kTcMaxN / 2) {
    uint32_t r[16];
    tmem_ld16(base + 16 * C, r);
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 16; ++i) tot[16 * C + i] += __uint_as_float(r[i]);
  }
}

// Final output of one tile: scale, store maps, fused per-frame argmax
// (lowest j on ties), then reset the totals for the next tile.  The four
// lane-quarter warps of a column half combine their warp maxima in shared
// memory (tile_keys) so each tile issues one global 64-bit atomicMax per
// frame instead of four.  Per column a warp issues one streaming 128-byte
// store (predicated, pointer-increment addressing) and one CREDUX + VOTE for
// the argmax; full tiles (every row and column valid) take a mask-free path.
__device__ __forceinline__ void st_cs_pred(float* ptr, float v, bool pred) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p st.global.cs.f32 [%0], %1;\n}" ::"l"(ptr),
      "f"(v), "r"(static_cast<uint32_t>(pred))
      : "memory");
}

template <bool kFull>
__device__ __forceinline__ void tc_write_cols(const TcParams& p, unsigned long long* tk, int quarter,
                                              int cbase, int ncols, int lim, uint32_t jbase,
                                              int lane, float* ptr,
                                              const float (&tot)[kTcMaxN / 2]) {
  // lim: columns valid for this lane (0 when the row is past J)
  const size_t J = static_cast<size_t>(p.J);
  TCP_DECL(w_st);
  TCP_DECL(w_am);
  if (ptr != nullptr) {
    TCP_T0();
#pragma unroll
    for (int i = 0; i < kTcMaxN / 2; ++i) {
      if (kFull)
        __stcs(ptr, tot[i]);
      else
        st_cs_pred(ptr, tot[i], i < lim);
      ptr += J;
    }
    TCP_ACC(w_st);
  }
  if (p.keys) {
    TCP_T0();
    // per column, the warp's best (value, lowest row) as a 64-bit key
    // (orderable value << 32 | ~j); a 32-column butterfly transpose-reduce
    // leaves column c of each group in lane c (31 64-bit exchanges per 32
    // columns instead of a CREDUX + VOTE chain per column)
    const unsigned long long low = static_cast<unsigned long long>(0xFFFFFFFFu - (jbase + lane));
#pragma unroll
    for (int g = 0; g < (kTcMaxN / 2 + 31) / 32; ++g) {
      if (kFull || 32 * g < ncols) {  // uniform
        unsigned long long k[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int i = 32 * g + c;
          k[c] = (i < kTcMaxN / 2 && (kFull || i < lim))
                     ? (static_cast<unsigned long long>(orderable_bits(tot[i < kTcMaxN / 2 ? i : 0]))
                        << 32) | low
                     : 0ull;
        }
#pragma unroll
        for (int o = 16, n = 16; o >= 1; o >>= 1, n >>= 1) {
          const bool up = lane & o;
#pragma unroll
          for (int c = 0; c < n; ++c) {
            const unsigned long long keep = up ? k[c + n] : k[c];
            const unsigned long long send = up ? k[c] : k[c + n];
            const unsigned long long recv = __shfl_xor_sync(0xffffffffu, send, o);
            k[c] = keep > recv ? keep : recv;
          }
        }
        const int col = 32 * g + lane;
        if (col < ncols) tk[quarter * kTcMaxN + cbase + col] = k[0];  // 0 = none
      }
    }
    TCP_ACC(w_am);
  }
  if (threadIdx.x == kEpiWarp0 * 32) {
    TCP_FLUSH(14, w_st);
    TCP_FLUSH(15, w_am);
  }
}

__device__ __forceinline__ void tc_write_tile(const TcParams& p, unsigned long long* tile_keys,
                                              int m0, int n0,
                                              int nc, int quarter, int half, int lane,
                                              float (&tot)[kTcMaxN / 2]) {
  const int J = p.J;
  const uint32_t jbase = static_cast<uint32_t>(m0 + 32 * quarter);
  const int j = static_cast<int>(jbase) + lane;
  const int cbase = half * (nc / 2);
  const int ncols = nc / 2;
  const int nv = max(0, min(ncols, p.F - (n0 + cbase)));  // columns with f < F
  const int lim = j < J ? nv : 0;
  float* ptr = p.maps ? p.maps + (static_cast<size_t>(n0 + cbase) * J + j) : nullptr;
  unsigned long long* tk = tile_keys;  // [4 quarters][kTcMaxN columns]
  TCP_DECL(w_loop);
  TCP_DECL(w_flush);
  { TCP_T0();
#pragma unroll
  for (int i = 0; i < kTcMaxN / 2; ++i) tot[i] *= p.scale;
  // full: all 80 columns valid for every lane of the warp
  if (__all_sync(0xffffffffu, lim == kTcMaxN / 2))
    tc_write_cols<true>(p, tk, quarter, cbase, ncols, lim, jbase, lane, ptr, tot);
  else
    tc_write_cols<false>(p, tk, quarter, cbase, ncols, lim, jbase, lane, ptr, tot);
#pragma unroll
  for (int i = 0; i < kTcMaxN / 2; ++i) tot[i] = 0.0f;
  TCP_ACC(w_loop); }
  if (p.keys) {
    TCP_T0();
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
    const int et = threadIdx.x - kEpiWarp0 * 32;  // 0..255
    for (int c = et; c < nc; c += kEpiWarps * 32) {
      unsigned long long k = tk[c];
#pragma unroll
      for (int q = 1; q < 4; ++q) k = key_max(k, tk[q * kTcMaxN + c]);
      const int f = n0 + c;
      if (k != 0ull && f < p.F) atomicMax(p.keys + f, k);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");  // tk reusable
    TCP_ACC(w_flush);
  }
  if (threadIdx.x == kEpiWarp0 * 32) {
    TCP_FLUSH(12, w_loop);
    TCP_FLUSH(13, w_flush);
  }
}

// Team epilogue (generator teams): the warp of column half `half`, lane
// quarter `quarter` writes the 16-column chunks it owns (c0, c0 + 2, ...)
// straight from the shared running totals (zeroing them for the next tile):
// scale, streaming stores, and the fused argmax -- per chunk the warp's 32
// rows reduce to one key per column (a 16-column butterfly transpose-reduce),
// the four quarters combine in shared memory (the team's named barrier) and
// one global atomicMax per frame publishes it.
__device__ __forceinline__ void tc_write_chunks(const TcParams& p, unsigned long long* tk,
                                                float* tot_s, int m0, int n0, int nc, int quarter,
                                                int half, int lane, int team, int c0, int cstep,
                                                int et) {
  const int J = p.J;
  const uint32_t jbase = static_cast<uint32_t>(m0 + 32 * quarter);
  const int j = static_cast<int>(jbase) + lane;
  const int ncols = nc / 2;
  const int cbase = half * ncols;
  const int nv = max(0, min(ncols, p.F - (n0 + cbase)));  // columns with f < F
  const int lim = j < J ? nv : 0;
  const unsigned long long low = static_cast<unsigned long long>(0xFFFFFFFFu - (jbase + lane));
  for (int c = c0; 16 * c < ncols; c += cstep) {
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v[i] = tot_s[(16 * c + i) * kTcM] * p.scale;
      tot_s[(16 * c + i) * kTcM] = 0.0f;
    }
    if (p.maps) {
      float* ptr = p.maps + (static_cast<size_t>(n0 + cbase + 16 * c) * J + j);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        st_cs_pred(ptr, v[i], 16 * c + i < lim);
        ptr += J;
      }
    }
    if (p.keys) {
      unsigned long long k[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        k[i] = 16 * c + i < lim ? (static_cast<unsigned long long>(orderable_bits(v[i])) << 32) | low
                                : 0ull;
      // lane halves first (no transpose), then a 16-column transpose-reduce:
      // lane l < 16 ends holding column l
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const unsigned long long r = __shfl_xor_sync(0xffffffffu, k[i], 16);
        k[i] = k[i] > r ? k[i] : r;
      }
#pragma unroll
      for (int o = 8, n = 8; o >= 1; o >>= 1, n >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int i = 0; i < n; ++i) {
          const unsigned long long keep = up ? k[i + n] : k[i];
          const unsigned long long send = up ? k[i] : k[i + n];
          const unsigned long long recv = __shfl_xor_sync(0xffffffffu, send, o);
          k[i] = keep > recv ? keep : recv;
        }
      }
      if (lane < 16 && 16 * c + lane < ncols) tk[quarter * kTcMaxNGen + cbase + 16 * c + lane] = k[0];
    }
  }
  if (p.keys) {
    // the team's four quarters of each owned column -> one atomic per frame
    asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "n"(kEpiWarps * 32) : "memory");
    for (int col = et; col < nc; col += kEpiWarps * 32) {
      const int h = col >= ncols ? 1 : 0;
      const int c = (col - h * ncols) >> 4;
      if (((c + h) & 1) != team && cstep == 2) continue;  // the other team's chunk
      unsigned long long k = tk[col];
#pragma unroll
      for (int q = 1; q < 4; ++q) k = key_max(k, tk[q * kTcMaxNGen + col]);
      const int f = n0 + col;
      if (k != 0ull && f < p.F) atomicMax(p.keys + f, k);
    }
    asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "n"(kEpiWarps * 32) : "memory");  // tk reusable
  }
}

// Staged epilogue (K4 pairs).  Per 8-frame chunk the warp writes its 32 rows
// x 8 frames into a 1 KB shared buffer in the TMA 128-byte-swizzled layout
// (frame-major: one 128-byte line per frame = the warp's 32 candidates) and
// one lane stores it with a TMA bulk tensor store (no per-column st.global
// from the LSU).  The same buffer serves the argmax transposed: lane L reads
// frame L % 8's candidates [8 (L / 8), +8) with two conflict-free 16-byte
// loads, keeps the best (value, lowest j) key, merges across the four lanes
// of its frame (two shuffles) and pushes it with one global atomicMax.  Two
// buffers per warp alternate; a buffer is rewritten only after the store
// issued from it two chunks earlier has finished reading it.
__device__ __forceinline__ void tc_write_tile_staged(const TcParams& p, const CUtensorMap* tm_maps,
                                                     uint32_t sbase, int& chunk_seq, int m0, int n0,
                                                     int nc, int quarter, int half, int lane,
                                                     float (&tot)[kTcMaxN / 2]) {
  const int J = p.J;
  const uint32_t jbase = static_cast<uint32_t>(m0 + 32 * quarter);
  const int cbase = half * (nc / 2);
  const int ncols = nc / 2;
  const int f_base = n0 + cbase;
  const int j = static_cast<int>(jbase) + lane;
  const int nv = max(0, min(ncols, p.F - f_base));  // columns with f < F
  TCP_DECL(w_loop);
  TCP_DECL(w_wait);
  TCP_DECL(w_sts);
  TCP_DECL(w_am);
  { TCP_T0();
  if (p.maps && !p.maps_tma) {  // J % 4 != 0: no TMA map for the maps; direct stores
    float* ptr = p.maps + (static_cast<size_t>(f_base) * J + j);
    const int lim = j < J ? nv : 0;
#pragma unroll
    for (int i = 0; i < kTcMaxN / 2; ++i) {
      st_cs_pred(ptr, tot[i] * p.scale, i < lim);
      ptr += J;
    }
  }
  // swizzled slot of (frame row r, this lane's candidate) in an 8 x 128 B atom;
  // rows past J are staged as -inf (the TMA store clips them; the argmax
  // never picks them)
  const uint32_t lane_off = static_cast<uint32_t>(lane & 3) * 4u;
  const int lane_chunk = lane >> 2;
  uint32_t slot[kEpiChunk];
#pragma unroll
  for (int r = 0; r < kEpiChunk; ++r)
    slot[r] = static_cast<uint32_t>(r) * 128u + (static_cast<uint32_t>(lane_chunk ^ r) << 4) +
              lane_off;
  const float scale = p.scale;
  const bool row_ok = j < J;
  // argmax over a 16-frame super-chunk (both buffers): lane -> frame
  // u16 = lane % 16 (buffer u16 / 8, row u16 % 8), candidates [16 hh, +16)
  const int u16 = lane & 15;
  const int hh = lane >> 4;
  const int ur = u16 & 7;
  uint32_t rd[4];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    rd[k] = static_cast<uint32_t>(u16 >> 3) * kEpiStageBytes + static_cast<uint32_t>(ur) * 128u +
            (static_cast<uint32_t>((4 * hh + k) ^ ur) << 4);
#pragma unroll
  for (int cc = 0; cc < (kTcMaxN / 2) / 16; ++cc) {
    if (16 * cc < ncols) {  // uniform (ncols is a multiple of 16)
      { TCP_T0();
      if (chunk_seq > 0) {  // both buffers' previous stores have read them
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
      }
      TCP_ACC(w_wait); }
      chunk_seq = 1;
      { TCP_T0();
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int r = 0; r < kEpiChunk; ++r) {
          const float v = row_ok ? tot[16 * cc + 8 * b + r] * scale : -INFINITY;
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(sbase + b * kEpiStageBytes + slot[r]),
                       "f"(v)
                       : "memory");
        }
      if (p.maps && p.maps_tma) fence_proxy_async_smem();  // STS -> visible to the TMA engine
      __syncwarp();
      if (lane == 0 && p.maps && p.maps_tma) {
        tma_store_2d(tm_maps, sbase, static_cast<int>(jbase), f_base + 16 * cc);
        tma_store_2d(tm_maps, sbase + kEpiStageBytes, static_cast<int>(jbase),
                     f_base + 16 * cc + 8);
        bulk_commit();
      }
      TCP_ACC(w_sts); }
      TCP_T0();
      if (p.keys) {
        const int f_col = 16 * cc + u16;
        float vv[16];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(vv[4 * k]), "=f"(vv[4 * k + 1]), "=f"(vv[4 * k + 2]),
                         "=f"(vv[4 * k + 3])
                       : "r"(sbase + rd[k])
                       : "memory");
        // tree max with lowest-index ties: at each level keep the left
        // (lower j) element unless the right one is strictly greater (NaN
        // never selected; -inf marks rows past J)
        int id[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) id[e] = e;
#pragma unroll
        for (int w = 1; w < 16; w <<= 1)
#pragma unroll
          for (int e = 0; e < 16; e += 2 * w)
            if (vv[e + w] > vv[e]) {
              vv[e] = vv[e + w];
              id[e] = id[e + w];
            }
        unsigned long long best =
            (f_col < nv && vv[0] > -INFINITY)
                ? (static_cast<unsigned long long>(orderable_bits(vv[0])) << 32) |
                      static_cast<unsigned long long>(0xFFFFFFFFu - (jbase + 16 * hh + id[0]))
                : 0ull;
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, 16);
        best = other > best ? other : best;
        if (hh == 0 && best != 0ull) atomicMax(p.keys + f_base + f_col, best);
      }
      TCP_ACC(w_am);
    }
  }
#pragma unroll
  for (int i = 0; i < kTcMaxN / 2; ++i) tot[i] = 0.0f;
  TCP_ACC(w_loop); }
  if (threadIdx.x == kEpiWarp0 * 32) {
    TCP_FLUSH(12, w_loop);
    TCP_FLUSH(14, w_wait);
    TCP_FLUSH(13, w_sts);
    TCP_FLUSH(8, w_am);
  }
}

// Exact round-to-nearest (ties away) of a finite fp32 to tf32, in two integer
// ops; x - tf32_rna(x) is exact in fp32.
__device__ __forceinline__ uint32_t tf32_rna_bits(float x) {
  return (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;
}

// Steering-phase generator of one A row (candidate j) and one half of every
// K block it is given (kBins bins: 8 per 32-column tf32 block, 16 per
// 64-element fp16 block).  The blocks of a tile come in increasing order,
// kStride apart (generator teams take every other block).  Per pair: the
// one-bin and kStride-block rotations e^{j2pi x/N}, e^{j2pi 2 kBins kStride
// x/N} from exact turn arithmetic; per block: the anchor phase, exact
// (integer-reduced turns + sincospif) every kAnchorBlocks of this thread's
// blocks and otherwise the previous anchor rotated by kStride blocks; then
// kBins - 1 one-bin rotations.  Longest rotation chain ~ 1 block + 15 one-bin
// rotations, ~1e-6 relative phase error.
template <bool kF16, int kStride = 1>
struct PhaseGen {
  static constexpr int kBins = kF16 ? 16 : 8;                 // bins per half block
  static constexpr int kAnchorBlocks = 64 / (2 * kBins);     // exact anchor every 64 bins (per thread)
  int kbp, bip;   // K blocks per pair, block index in the current pair
  int pair, ti;
  float tf, sc, ss, sbc, sbs, ac, as;
  int since_exact;

  __device__ __forceinline__ void start_tile(const TcParams& p) {
    kbp = p.kb_per_pair;
    pair = -1;
  }

  __device__ __forceinline__ void load_pair(const TcParams& p, int j) {
    ti = 0;
    tf = 0.0f;
    if (j < p.J) {
      ti = p.tau_i[static_cast<size_t>(pair) * p.J + j];
      tf = p.tau_f[static_cast<size_t>(pair) * p.J + j];
    }
    sincospif(2.0f * (static_cast<float>(ti) + tf) * p.inv_period, &ss, &sc);
    const float tb = harmonic_turns(2 * kBins * kStride, ti, tf, p.period, p.mask, p.inv_period);
    sincospif(2.0f * tb, &sbs, &sbc);
    since_exact = kAnchorBlocks;
  }

  __device__ __forceinline__ void block(const TcParams& p, int j, int half, int kb,
                                        uint32_t a_hi_tmem, uint32_t a_lo_tmem) {
    if (pair < 0) {  // first block of the tile
      pair = kb / kbp;
      bip = kb - pair * kbp;
      load_pair(p, j);
    } else {
      bip += kStride;
      if (bip >= kbp) {  // a later pair
        do {
          bip -= kbp;
          ++pair;
        } while (bip >= kbp);
        load_pair(p, j);
      }
    }
    const int k = bip * (2 * kBins) + kBins * half;
    if (since_exact >= kAnchorBlocks) {
      harmonic_phase(k, ti, tf, p.period, p.mask, p.inv_period, &ac, &as);
      since_exact = 0;
    } else {
      const float cn = ac * sbc - as * sbs;
      as = fmaf(ac, sbs, as * sbc);
      ac = cn;
    }
    ++since_exact;
    float c = ac, s = as;
    uint32_t hi[16], lo[16];
#pragma unroll
    for (int m = 0; m < kBins; ++m) {
      const float ns = -s;
      if constexpr (kF16) {
        // one 32-bit TMEM column = half2 (cos, -sin) of one bin, prescaled
        const float xc = c * kF16PhaseScale, xs = ns * kF16PhaseScale;
        const __half2 h = __floats2half2_rn(xc, xs);
        const __half2 l = __floats2half2_rn(xc - __low2float(h), xs - __high2float(h));
        hi[m] = *reinterpret_cast<const uint32_t*>(&h);
        lo[m] = *reinterpret_cast<const uint32_t*>(&l);
      } else {
        const uint32_t hc = tf32_rna_bits(c), hs = tf32_rna_bits(ns);
        hi[2 * m] = hc;
        hi[2 * m + 1] = hs;
        lo[2 * m] = __float_as_uint(c - __uint_as_float(hc));
        lo[2 * m + 1] = __float_as_uint(ns - __uint_as_float(hs));
      }
      const float cn = c * sc - s * ss;  // rotate by one bin
      s = fmaf(c, ss, s * sc);
      c = cn;
    }
    tmem_st16(a_hi_tmem + 16 * half, hi);
    tmem_st16(a_lo_tmem + 16 * half, lo);
  }
};

// Sinc-weight generator of one A row (candidate j) for K4 without a stored
// W: columns t = 64 kb + 32 half + c (c < 32) of the lattice layout,
// W[j, t] = sinc(x_jp - n) for the pair p owning t and its lag n, computed
// with the stored table's function (sinc_weight_fast) and split like
// srpb_f16_split (v = 2^14 w, hi = half(v), lo = half(v - hi)), so the A
// operand -- and the maps -- equal the stored-W kernel's bit for bit.  The
// pair is tracked incrementally (columns only increase within an item; all
// rows of a warp share the column sequence, so pair changes are
// warp-uniform); the next pair's split is prefetched into registers one
// pair ahead, hiding its global-load latency.
//
// Cost: with d = E - t (E = i + column of lag 0, t the column), a run of 32
// columns inside one pair needs, per weight, the exact integer-valued
// denominator part (E - t0) - c, one rounding add of f, one MUFU reciprocal
// and one multiply by the pair's signed amplitude 2^14 (-1)^E sin(pi f)/pi
// (the (-1)^c alternation is compile-time) -- done two columns at a time with
// the packed f32x2 adds/multiplies -- plus the fp16 hi/lo split: ~4 ALU
// instructions and one MUFU per weight (the per-column pair tracking of a
// generic column walk cost ~20).  Runs that cross a pair boundary (C4:
// about one in nine) take one masked pass per pair.  Exact-node rows (f == 0,
// and |f| < 1e-30, where the reference's sinc is 1 / 0 to fp64 rounding) use
// amplitude 0 with a half-integer denominator and get their single 2^14
// written afterwards.
struct SincGen {
  int p, end;         // current pair, its end column (INT_MAX past the last pair)
  int E;              // split integer part + column of lag 0: d = E - t
  float f, amp;       // denominator fraction, signed 2^14 sin(pi f) / pi
  bool node;          // exact-node row: weight 2^14 at d == 0, else 0
  int nsi;            // prefetched split of pair p + 1
  float nsf;
  const int2* cols;   // shared: per pair (end column, column of lag 0)

  __device__ __forceinline__ void fetch(const TcParams& prm, int j, int q) {
    nsi = 0;
    nsf = 0.0f;
    if (q < prm.P && j < prm.J) {
      nsi = __ldg(prm.sx_i + static_cast<size_t>(q) * prm.J + j);
      nsf = __ldg(prm.sx_f + static_cast<size_t>(q) * prm.J + j);
    }
  }

  __device__ __forceinline__ void start_tile(const TcParams& prm, int j, const int2* pair_cols) {
    p = -1;
    end = 0;
    cols = pair_cols;
    fetch(prm, j, 0);
  }

  __device__ __forceinline__ void advance(const TcParams& prm, int j) {
    ++p;
    if (p < prm.P) {
      const int2 c = cols[p];
      end = c.x;
      E = nsi + c.y;
      node = sinc_is_node(nsf);
      f = node ? 0.5f : nsf;
      const float a = node ? 0.0f : sinc_spi(nsf) * kF16PhaseScale;
      amp = (E & 1) ? -a : a;
      fetch(prm, j, p + 1);
    } else {  // lattice padding columns: weight 0
      end = 0x7fffffff;
      E = 0;
      node = false;
      f = 0.5f;
      amp = 0.0f;
    }
  }

  static __device__ __forceinline__ void split2(float2 w, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __floats2half2_rn(w.x, w.y);
    const float2 hf = __half22float2(h);
    const float2 r = __fadd2_rn(w, make_float2(-hf.x, -hf.y));  // exact residual
    const __half2 l = __floats2half2_rn(r.x, r.y);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
  }

  // One 32-column run in two 16-column slabs (8 hi + 8 lo words each, one
  // tcgen05.st.x8 per half of the split): half the live weight registers of
  // a whole-run pass (the 18-warp kernel has 96 registers per thread).
  __device__ __forceinline__ void block(const TcParams& prm, int j, int half, int kb,
                                        uint32_t a_hi_tmem, uint32_t a_lo_tmem) {
    const int t0 = 64 * kb + 32 * half;
    // a thread sees 32 of every 64 columns: pairs may end in the skipped half
    while (t0 >= end) advance(prm, j);  // warp-uniform
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      constexpr int kW = 16;  // columns per slab
      const int cb = kW * q;  // first column of the slab in the run
      uint32_t hi[8], lo[8];
      // a pair may end exactly at the slab boundary: the slab's own pair
      // decides fast path vs crossing (the stored table decides the same way)
      if (q == 1)
        while (t0 + cb >= end) advance(prm, j);  // warp-uniform
      if (TC_DBG(prm) & 2048) {  // bound analysis only: no weight arithmetic
#pragma unroll
        for (int i = 0; i < 8; ++i) hi[i] = lo[i] = __float_as_uint(f) + i;
      } else if (t0 + cb + kW <= end) {
        // the slab lies in pair p: integer-valued d of columns (c, c + 1),
        // stepped by -2 (exact), then one rounding add of f = float(d) + f.
        // (Per-column immediates would go through a recycled uniform
        // register pair and serialise the loop.)
        const float Df = static_cast<float>(E - t0 - cb);
        float2 dd = make_float2(Df, Df - 1.0f);
        const float2 m2 = make_float2(-2.0f, -2.0f);
        const float2 a2 = make_float2(amp, -amp);
        const float2 f2 = make_float2(f, f);
#pragma unroll
        for (int c = 0; c < kW; c += 2) {
          const float2 x = __fadd2_rn(dd, f2);
          dd = __fadd2_rn(dd, m2);
          // both reciprocals from one MUFU (sinc_pair_rcp): the reciprocal
          // unit is the generator's largest energy item under the power cap
          // (measured: without it the kernel ran 12% faster at the same
          // cycle count)
          const float P = (TC_DBG(prm) & 1024) ? 1.0f : rcp_approx_ftz(x.x * x.y);
          const float2 r = __fmul2_rn(make_float2(x.y, x.x), make_float2(P, P));
          split2(__fmul2_rn(r, a2), hi[c >> 1], lo[c >> 1]);
        }
        if (__any_sync(0xffffffffu, node)) {
          // the node row's d == 0 column in this slab as a column bit
          // (selects per word: an `if (i == cs / 2) hi[i] = ..` becomes an
          // indexed store and moves hi[] to local memory)
          const int cs = E - t0 - cb;
          const uint32_t hit = (node && cs >= 0 && cs < kW) ? (1u << cs) : 0u;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t b2 = (hit >> (2 * i)) & 3u;
            hi[i] = b2 == 0u ? hi[i] : (b2 == 1u ? 0x00007400u : 0x74000000u);
          }
        }
      } else {
        // the slab meets several pairs: one masked pass per pair (all
        // indices compile-time, so the weights stay in registers; a rolled
        // column walk through local memory measured 11% slower at C4)
        float w[kW];
#pragma unroll
        for (int c = 0; c < kW; ++c) w[c] = 0.0f;
        int lo_c = 0;
        for (;;) {  // warp-uniform
          const int hi_c = min(end - t0 - cb, kW);
          const int cs = E - t0 - cb;
          const float Df = static_cast<float>(cs);
#pragma unroll
          for (int c = 0; c < kW; ++c) {
            const float x = (Df - static_cast<float>(c)) + f;
            float v = rcp_approx_ftz(x) * ((c & 1) ? -amp : amp);
            if (node) v = cs == c ? kF16PhaseScale : 0.0f;
            w[c] = (c >= lo_c && c < hi_c) ? v : w[c];
          }
          if (hi_c == kW) break;
          lo_c = hi_c;
          advance(prm, j);
        }
#pragma unroll
        for (int c = 0; c < kW; c += 2) split2(make_float2(w[c], w[c + 1]), hi[c >> 1], lo[c >> 1]);
      }
      if (TC_DBG(prm) & 4096) continue;  // bound analysis only: no TMEM stores
      tmem_st8(a_hi_tmem + 16 * half + 8 * q, hi);
      tmem_st8(a_lo_tmem + 16 * half + 8 * q, lo);
    }
  }
};

// Stored-weight "generator" (kALoad): the thread's 32 columns of its row of
// the fp16 W split (64 contiguous bytes of hi and of lo) loaded with 16-byte
// read-only loads and stored into the TMEM A stage -- the TS MMA then reads A
// from tensor memory, taking A off the shared-memory path (the SS kernel moves
// A through shared memory twice per stage: TMA write, two MMA reads).
struct WLoadGen {
  __device__ __forceinline__ void start_tile(const TcParams&) {}
  __device__ __forceinline__ void block(const TcParams& prm, int j, int half, int kb,
                                        uint32_t a_hi_tmem, uint32_t a_lo_tmem) {
    uint32_t hi[16], lo[16];
    const int t0 = 64 * kb + 32 * half;
    const size_t row = static_cast<size_t>(j) * prm.T_pad;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 h = make_uint4(0u, 0u, 0u, 0u), l = h;
      if (j < prm.J && t0 + 8 * q < prm.T_pad) {  // T_pad % 8 == 0: whole 16-byte chunks
        h = __ldg(reinterpret_cast<const uint4*>(prm.w_hi + row + t0 + 8 * q));
        l = __ldg(reinterpret_cast<const uint4*>(prm.w_lo + row + t0 + 8 * q));
      }
      hi[4 * q] = h.x; hi[4 * q + 1] = h.y; hi[4 * q + 2] = h.z; hi[4 * q + 3] = h.w;
      lo[4 * q] = l.x; lo[4 * q + 1] = l.y; lo[4 * q + 2] = l.z; lo[4 * q + 3] = l.w;
    }
    tmem_st16(a_hi_tmem + 16 * half, hi);
    tmem_st16(a_lo_tmem + 16 * half, lo);
  }
};

template <int kAMode, bool kPair, bool kF16>
__global__ void __launch_bounds__((TcCfg<kAMode, kPair, kF16>::kThreads), 1)
srp_tc_kernel(const __grid_constant__ CUtensorMap tmA_hi, const __grid_constant__ CUtensorMap tmA_lo,
              const __grid_constant__ CUtensorMap tmB_hi, const __grid_constant__ CUtensorMap tmB_lo,
              const __grid_constant__ CUtensorMap tmMaps, const TcParams p) {
  using Cfg = TcCfg<kAMode, kPair, kF16>;
  // K4: as many smem stages as the tile width leaves room for (narrow tiles,
  // e.g. batch 1, get more look-ahead on the W stream); generator modes:
  // their TMEM A ring
  const int S = p.stages;
  constexpr bool kASmem = Cfg::kASmem;
  constexpr int kTeams = Cfg::kTeams;
  constexpr int kGenW0 = Cfg::kGenW0;
  constexpr int kGenWarps = Cfg::kGenWarps;
  constexpr int kProdWarp = Cfg::kProdWarp;
  constexpr int kMmaWarp = Cfg::kMmaWarp;
  constexpr int KBE = Cfg::kKbElems;
  constexpr int kCta = kPair ? 2 : 1;
#ifdef SRPB_TC_PROFILE
  const long long t_entry = clock64();
  unsigned long long g_entry;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_entry));
#endif
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-align by pointer arithmetic on the shared array (keeps the shared
  // address space visible to the compiler: STS/LDS, not generic accesses)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const size_t stage_bytes = tc_stage_bytes(p.N, kASmem, kPair);
  // [stages][running totals (generator modes)][epilogue staging (K4 pairs) |
  // tile argmax keys][barriers]
  float* tot_smem = reinterpret_cast<float*>(smem + S * stage_bytes);
  uint8_t* epi_stage = smem + S * stage_bytes + (Cfg::kTotSmem ? tot_smem_bytes(p.N) : 0);
  unsigned long long* tile_keys = reinterpret_cast<unsigned long long*>(epi_stage);
  using TcSmem = TcSmemT<Cfg::kItemRing>;
  constexpr int kItemRing = Cfg::kItemRing;
  TcSmem* bar = reinterpret_cast<TcSmem*>(epi_stage +
                                          (Cfg::kEpiStage ? kEpiStageTotal : kTileKeysBytes));
  // kASinc: per pair (end column, column of lag 0), after the barriers
  int2* pair_cols = reinterpret_cast<int2*>(bar + 1);
  if (kAMode == kASinc)
    for (int q = threadIdx.x; q < p.P; q += blockDim.x)
      pair_cols[q] = make_int2(__ldg(p.off + q + 1), __ldg(p.off + q) + __ldg(p.reach + q));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b_rows = kPair ? p.N / 2 : p.N;  // B rows held by this CTA
  const uint32_t b_bytes = static_cast<uint32_t>(b_rows) * 128;
  const int rank = kPair ? static_cast<int>(cluster_ctarank()) : 0;
  const bool leader = rank == 0;

  // Work items: (frame tile, candidate tile of 128 x kCta rows); in a pair,
  // CTA `rank` owns rows [128 rank, 128 rank + 128) of the 256-row tile.
  // Scheduling is dynamic: CTA (pair) c starts with item c, then takes the
  // next id from a global cursor (done[1]) whenever its producer is ready, so
  // faster SMs take more items and the exit spread shrinks to ~one item.  The
  // leader's producer fetches ids into a shared ring (both CTAs of a pair);
  // the MMA issuer and epilogue warps read the same sequence and release
  // each slot when done with the item.  Items are computed identically
  // wherever they run, so results do not depend on the schedule.
  // The last partial wave's items are split into two frame pieces (n_piece0
  // and N - n_piece0 frames) so the wave's work spreads over more CTAs; every
  // output element accumulates over K in the same order whatever its item's
  // width, so maps are bitwise independent of the split.
  const int cid = static_cast<int>(blockIdx.x) / kCta;
  const int ncl = static_cast<int>(gridDim.x) / kCta;
  struct Item {
    int m0, n0, nc;  // candidate row base (this CTA), frame base, frames
  };
  auto item_of = [&](int g) {
    int b = g, piece = -1;
    if (g >= p.full_items) {
      const int q = g - p.full_items;
      b = p.full_items + q / p.n_pieces;
      piece = q - (q / p.n_pieces) * p.n_pieces;
    }
    Item r;
    const int mt = p.m_fast ? b % p.m_units : b / p.n_tiles;
    const int nt = p.m_fast ? b / p.m_units : b % p.n_tiles;
    r.m0 = (mt * kCta + rank) * kTcM;
    r.n0 = nt * p.N;
    r.nc = nt == p.n_tiles - 1 ? p.n_last : p.N;
    if (piece >= 0) {
      r.n0 += piece * p.n_piece0;
      r.nc = piece < p.n_pieces - 1 ? p.n_piece0 : p.N - (p.n_pieces - 1) * p.n_piece0;
    }
    return r;
  };
  unsigned int* const cursor = (p.done && p.dynamic) ? p.done + 1 : nullptr;
  // item id of the it-th item of this CTA (pair): waits for the ring slot
  // (-1 = no more items)
  auto item_id = [&](int it) -> int {
    const int slot = it % kItemRing;
    if (kPair && !leader)
      mbar_wait_acq_cluster(&bar->item_full[slot], (it / kItemRing) & 1);
    else
      mbar_wait(&bar->item_full[slot], (it / kItemRing) & 1);
    return *reinterpret_cast<volatile int*>(&bar->item_ring[slot]);
  };
  // a consumer warp is done with its it-th item (one arrive per warp)
  auto item_release = [&](int it) {
    if (lane == 0) {
      const int slot = it % kItemRing;
      if (kPair && !leader)
        mbar_arrive_cluster_relaxed(mapa(&bar->item_empty[slot], 0));
      else
        mbar_arrive(&bar->item_empty[slot]);
    }
  };
  // leader producer: publish the it-th item id to the ring of every CTA
  auto item_fetch = [&](int it) -> int {
    int g = 0;
    if (lane == 0) {
      const int slot = it % kItemRing;
      if (it >= kItemRing) mbar_wait(&bar->item_empty[slot], ((it / kItemRing) - 1) & 1);
      g = it == 0 ? cid
                  : (cursor ? ncl + static_cast<int>(atomicAdd(cursor, 1u)) : cid + it * ncl);
      if (g >= p.total_items) g = -1;
      bar->item_ring[slot] = g;
      if (kPair) {
        st_shared_cluster_u32(mapa(&bar->item_ring[slot], 1), static_cast<uint32_t>(g));
        mbar_arrive_cluster(mapa(&bar->item_full[slot], 1));
      }
      mbar_arrive(&bar->item_full[slot]);
    }
    return __shfl_sync(0xffffffffu, g, 0);
  };

  const size_t a_bytes = kASmem ? 2 * kABytes : 0;
  auto a_hi = [&](int s) { return smem + s * stage_bytes; };
  auto a_lo = [&](int s) { return smem + s * stage_bytes + kABytes; };
  auto b_hi = [&](int s) { return smem + s * stage_bytes + a_bytes; };
  auto b_lo = [&](int s) { return smem + s * stage_bytes + a_bytes + b_bytes; };

  if (warp == kProdWarp && lane == 0) {
    tma_prefetch(&tmB_hi);
    tma_prefetch(&tmB_lo);
    if (kASmem) {
      tma_prefetch(&tmA_hi);
      tma_prefetch(&tmA_lo);
    }
  }
  if (warp == kMmaWarp) {
    if (kPair)
      tmem_alloc_pair(&bar->tmem_base, 512);
    else
      tmem_alloc(&bar->tmem_base, 512);
  }
  if (warp == kProdWarp && lane == 1) {
    // full: producers (x kCta) + one team of A-generator warps (x kCta)
    // arrive on the leader's barrier; empty / acc_full: one commit from the
    // leader's MMA; acc_empty: the epilogue warps of both CTAs arrive on the
    // leader's.
    const int full_count = kCta * (1 + (kAMode != kAFromTma ? kEpiWarps : 0));
    for (int s = 0; s < S; ++s) {
      mbar_init(&bar->full[s], full_count);
      mbar_init(&bar->empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar->acc_full[b], 1);
      mbar_init(&bar->acc_empty[b], kCta * kGenWarps);
    }
    // item ring: the leader producer fills every CTA's slot; consumers are the
    // MMA issuer, all epilogue warps and the peer's producer
    for (int r = 0; r < kItemRing; ++r) {
      mbar_init(&bar->item_full[r], 1);
      mbar_init(&bar->item_empty[r], 1 + kCta * kGenWarps + (kCta - 1));
    }
    if (!Cfg::kEpiStage)
      for (int c = 0; c < 4 * kTcMaxNGen; ++c) tile_keys[c] = 0ull;
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  if (kPair) cluster_sync();  // the leader's barriers exist before peers signal them
  tc_fence_after();
#ifdef SRPB_TC_PROFILE
  if (threadIdx.x == 0) atomicAdd(&g_tc_prof[17], static_cast<unsigned long long>(clock64() - t_entry));
#endif
  // make the TMEM base provably warp-uniform (it stays in a uniform register)
  const uint32_t tmem = __shfl_sync(0xffffffffu, bar->tmem_base, 0);
  // PDL: setup above overlapped the previous kernel; operand loads, map /
  // key writes and the item cursor wait for it to complete
  pdl_wait();
  pdl_launch_dependents();
  // barriers every CTA of the pair signals live in the leader
  const uint32_t full_addr0 = kPair ? mapa(&bar->full[0], 0) : smem_u32(&bar->full[0]);
  const uint32_t acc_empty_addr0 =
      kPair ? mapa(&bar->acc_empty[0], 0) : smem_u32(&bar->acc_empty[0]);

  if (warp == kProdWarp) {
    // ------------------------------------------------------------ TMA producer
    // warp-wide loop, one elected lane issues (uniform operands, no per-issue
    // register broadcasts)
    int kg = 0;
    int ps = 0, pph = 0;  // stage ring position (no divisions)
    TCP_DECL(w_empty);
    TCP_DECL(t_all);
    { TCP_T0();
    // the leader fetches item ids one ahead: the cursor's atomic latency hides
    // behind the current item (measured: an L2 prefetch of the next item's W
    // rows from here made K4 slower, 60 -> 80 us)
    int gid_next = leader ? item_fetch(0) : 0;
    for (int it = 0;; ++it) {
      const int gid = leader ? gid_next : item_id(it);
      if (gid < 0) break;
      const Item t = item_of(gid);
      if (!leader) item_release(it);
      if (leader) gid_next = item_fetch(it + 1);
      if (p.lockstep && leader && it > 0) {  // wave barrier (static schedule)
        // bounded: CTAs that are not co-resident (another kernel holding
        // SMs) must not deadlock the wave -- after 2 ms a CTA goes on alone
        if (lane == 0) {
          const unsigned need = static_cast<unsigned>(min(p.total_items, it * ncl));
          unsigned long long t0, t1;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
          unsigned got;
          for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(got) : "l"(p.done + 1));
            if (got >= need) break;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            if (t1 - t0 > 2000000ull) break;
          }
        }
        __syncwarp();
      }
      if (lane == 0) TCT(it, 0);
      const int m0 = (TC_DBG(p) & 1) ? t.m0 % 2048 : t.m0;
      const int rows = kPair ? t.nc / 2 : t.nc;    // this CTA's B rows (multiple of 16)
      const int nb = t.n0 + rank * rows;
      // one box per B buffer: b_box = the buffer's rows, so a narrower
      // (split) item loads unused tail rows -- never past the buffer
      const int nbox = (rows + p.b_box - 1) / p.b_box;
      const uint32_t tx = static_cast<uint32_t>(kCta) *
                          (((TC_DBG(p) & 4) ? 1 : 2) * static_cast<uint32_t>(nbox * p.b_box) * 128 +
                           (kASmem ? ((TC_DBG(p) & 2) ? 1 : 2) * kABytes : 0));
      for (int kb = 0; kb < p.num_kb; ++kb, ++kg, ps = ps + 1 == S ? 0 : ps + 1, pph ^= (ps == 0)) {
        const int s = ps;
        { TCP_T0();
        mbar_wait(&bar->empty[s], pph ^ 1);
        TCP_ACC(w_empty); }
        if (elect_one()) {
          const uint32_t fb = full_addr0 + 8u * s;
          if (kPair) {
            // leader arms the pair's byte count, the peer arrives remotely
            if (leader)
              mbar_expect_tx(&bar->full[s], (TC_DBG(p) & 256) ? 0u : tx);
            else
              mbar_arrive_cluster_relaxed(fb);
            for (int r = 0; r < rows && !(TC_DBG(p) & 256); r += p.b_box) {
              tma_load_2d_pair(b_hi(s) + r * 128, &tmB_hi, fb, kb * KBE, nb + r);
              if (!(TC_DBG(p) & 4)) tma_load_2d_pair(b_lo(s) + r * 128, &tmB_lo, fb, kb * KBE, nb + r);
            }
            if (kASmem && !(TC_DBG(p) & 256)) {
              tma_load_2d_pair(a_hi(s), &tmA_hi, fb, kb * KBE, m0);
              if (!(TC_DBG(p) & 2)) tma_load_2d_pair(a_lo(s), &tmA_lo, fb, kb * KBE, m0);
            }
          } else {
            mbar_expect_tx(&bar->full[s], (TC_DBG(p) & 256) ? 0u : tx);
            for (int r = 0; r < rows && !(TC_DBG(p) & 256); r += p.b_box) {
              // (bound analysis: 32 = every block loads K block 0's B)
              const int kx = (TC_DBG(p) & 32) ? 0 : kb * KBE;
              tma_load_2d(b_hi(s) + r * 128, &tmB_hi, &bar->full[s], kx, nb + r);
              tma_load_2d(b_lo(s) + r * 128, &tmB_lo, &bar->full[s], kx, nb + r);
            }
            if (kASmem && !(TC_DBG(p) & 256)) {
              tma_load_2d(a_hi(s), &tmA_hi, &bar->full[s], kb * KBE, m0);
              tma_load_2d(a_lo(s), &tmA_lo, &bar->full[s], kb * KBE, m0);
            }
          }
        }
        __syncwarp();
      }
      if (p.lockstep && leader && lane == 0) atomicAdd(p.done + 1, 1u);
    }
    // tail: every stage's last release has landed before this CTA may exit
    for (int t = 0; t < S; ++t, ps = ps + 1 == S ? 0 : ps + 1, pph ^= (ps == 0))
      mbar_wait(&bar->empty[ps], pph ^ 1);
    TCP_ACC(t_all); }
    if (lane == 0) {
      TCP_FLUSH(3, w_empty);
      TCP_FLUSH(4, t_all);
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------- MMA issuer
    // warp-wide loop (leader CTA only for pairs); descriptors are base +
    // byte-offset>>4 arithmetic on uniform values; one elected lane issues
    // the MMAs and their commits.
    if (leader) {
      const uint64_t db0 = sw128_kmajor_desc(smem_u32(b_hi(0)));  // stage 0 B_hi
      const uint64_t da0 = sw128_kmajor_desc(smem_u32(a_hi(0)));  // stage 0 A_hi (K4)
      const uint32_t stage16 = static_cast<uint32_t>(stage_bytes >> 4);
      const uint32_t b16 = b_bytes >> 4, a16 = kABytes >> 4;
      int kg = 0;
      int ms = 0, mph = 0;  // stage ring position
      TCP_DECL(w_full);
      TCP_DECL(w_acc);
      TCP_DECL(t_all);
      { TCP_T0();
      for (int it = 0;; ++it) {
        const int gid = item_id(it);
        if (gid < 0) break;
        const int nc = item_of(gid).nc;
        item_release(it);
        const uint32_t idesc = kF16 ? idesc_f16(kTcM * kCta, nc) : idesc_tf32(kTcM * kCta, nc);
        for (int kb = 0; kb < p.num_kb; ++kb, ++kg, ms = ms + 1 == S ? 0 : ms + 1, mph ^= (ms == 0)) {
          const int s = ms;
          const int gl = min(kb / p.kb_per_group, p.groups_per_tile - 1);  // group in the tile
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
          mbar_wait(&bar->full[s], mph);
          TCP_ACC(w_full); }
          if (kb == 0 && lane == 0) TCT(it, 1);
          if (kb == p.num_kb - 1 && lane == 0) TCT(it, 2);
          tc_fence_after();
          const uint64_t bh = db0 + static_cast<uint64_t>(s * stage16);
          const uint64_t bl = bh + b16;
          if (elect_one()) {
            if (kASmem) {  // K4: A from smem (SS)
              const uint64_t ah = da0 + static_cast<uint64_t>(s * stage16);
              const uint64_t al = ah + a16;
#pragma unroll
              for (int ks = 0; ks < 4; ++ks) {  // 4 MMAs x 32 bytes of K
                const uint32_t o = 2 * ks;      // in 16-byte units
                const uint32_t acc0 = (in_group > 0 || ks > 0) ? 1u : 0u;
                if constexpr (kPair && kF16) {
                  if (!(TC_DBG(p) & 8)) {
                    mma_f16_pair(d, al + o, bh + o, idesc, acc0);
                    mma_f16_pair(d, ah + o, bl + o, idesc, 1u);
                  }
                  mma_f16_pair(d, ah + o, bh + o, idesc, (TC_DBG(p) & 8) ? acc0 : 1u);
                } else if constexpr (kPair) {
                  mma_tf32_pair(d, al + o, bh + o, idesc, acc0);
                  mma_tf32_pair(d, ah + o, bl + o, idesc, 1u);
                  mma_tf32_pair(d, ah + o, bh + o, idesc, 1u);
                } else if constexpr (kF16) {
                  mma_f16(d, al + o, bh + o, idesc, acc0);
                  mma_f16(d, ah + o, bl + o, idesc, 1u);
                  mma_f16(d, ah + o, bh + o, idesc, 1u);
                } else {
                  mma_tf32(d, al + o, bh + o, idesc, acc0);
                  mma_tf32(d, ah + o, bl + o, idesc, 1u);
                  mma_tf32(d, ah + o, bh + o, idesc, 1u);
                }
              }
            } else {  // K2: A from TMEM (TS), written there by the generator warps
              const uint32_t ah = tmem + static_cast<uint32_t>(tc_a_tmem_col(p.N, s));
              const uint32_t al = ah + 32;
#pragma unroll
              for (int ks = 0; ks < 4; ++ks) {  // 8 TMEM columns (32 bytes) of K each
                const uint32_t o = 2 * ks;
                const uint32_t acc0 = (in_group > 0 || ks > 0) ? 1u : 0u;
                if constexpr (kPair && kF16) {
                  mma_f16_ts_pair(d, al + 8 * ks, bh + o, idesc, acc0);
                  mma_f16_ts_pair(d, ah + 8 * ks, bl + o, idesc, 1u);
                  mma_f16_ts_pair(d, ah + 8 * ks, bh + o, idesc, 1u);
                } else if constexpr (kPair) {
                  mma_tf32_ts_pair(d, al + 8 * ks, bh + o, idesc, acc0);
                  mma_tf32_ts_pair(d, ah + 8 * ks, bl + o, idesc, 1u);
                  mma_tf32_ts_pair(d, ah + 8 * ks, bh + o, idesc, 1u);
                } else if constexpr (kF16) {
                  mma_f16_ts(d, al + 8 * ks, bh + o, idesc, acc0);
                  mma_f16_ts(d, ah + 8 * ks, bl + o, idesc, 1u);
                  mma_f16_ts(d, ah + 8 * ks, bh + o, idesc, 1u);
                } else {
                  mma_tf32_ts(d, al + 8 * ks, bh + o, idesc, acc0);
                  mma_tf32_ts(d, ah + 8 * ks, bl + o, idesc, 1u);
                  mma_tf32_ts(d, ah + 8 * ks, bh + o, idesc, 1u);
                }
              }
            }
            const bool last_in_group =
                (in_group == p.kb_per_group - 1 && gl < p.groups_per_tile - 1) || kb == p.num_kb - 1;
            if (kPair) {
              mma_commit_pair_mc(&bar->empty[s], 0x3);
              if (last_in_group) mma_commit_pair_mc(&bar->acc_full[g & 1], 0x3);
            } else {
              mma_commit(&bar->empty[s]);
              if (last_in_group) mma_commit(&bar->acc_full[g & 1]);
            }
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
    }
  } else if (warp >= kGenW0 && warp < kGenW0 + kGenWarps) {
    // ---------------------- epilogue (+ A generation for the generator modes)
    const int e = warp - kGenW0;       // 0..8 kTeams - 1
    const int team = e >> 3;           // generator team: K blocks kg = team (mod kTeams)
    const int quarter = warp & 3;      // TMEM lane quarter this warp may access
    const int half = (e >> 2) & 1;     // column half of the tile
    // accumulator chunks (16 columns of this half) folded and written by this
    // warp: all of them, or with two teams every other one (alternating
    // between the halves so each team owns half of the tile's columns)
    const int c0 = kTeams == 2 ? ((team + half) & 1) : 0;
    float tot[kTcMaxN / 2];
#pragma unroll
    for (int i = 0; i < kTcMaxN / 2; ++i) tot[i] = 0.0f;
    int drained = 0;  // next global group to fold
    // incremental position of group `drained`: its tile, index in the tile,
    // and the global K block index of its last block (no divisions)
    int d_it = 0, d_gl = 0;
    // last K block of group gl of a tile (the last group takes the remainder)
    auto group_last = [&](int gl) {
      return gl == p.groups_per_tile - 1 ? p.num_kb - 1 : (gl + 1) * p.kb_per_group - 1;
    };
    int d_last_kg = group_last(0);
    // generator modes: tiles shorter than the fold window
    const bool fold_all = p.num_kb < p.kb_per_group;
    TCP_DECL(c_gen_wait);
    TCP_DECL(c_gen);
    TCP_DECL(c_drain);
    TCP_DECL(c_write);
    TCP_DECL(c_all);
    // incremental fold (generator modes): one 16-column chunk per generated K
    // block, so a drain never stalls the A generation for long; the buffer
    // is released when the group is complete (the ping-pong leaves the MMA
    // kb_per_group blocks of slack)
    int d_chunk = -1;  // chunk of group `drained` next to fold (-1: not started)
    // generator modes: this thread's slice of the shared running totals
    float* tot_s = tot_smem + half * (p.N / 2) * kTcM + 32 * quarter + lane;
    if constexpr (Cfg::kTotSmem) {
      for (int c = c0; c < p.N / 32; c += kTeams)
#pragma unroll
        for (int i = 0; i < 16; ++i) tot_s[(16 * c + i) * kTcM] = 0.0f;
    }
    auto finish_group = [&](const Item& t) {
      if (d_gl == p.groups_per_tile - 1) {
        TCP_T0();
        if constexpr (kTeams == 2) {
          tc_write_chunks(p, tile_keys, tot_s, t.m0, t.n0, t.nc, quarter, half, lane, team, c0,
                          kTeams, (e & 7) * 32 + lane);
        } else {
          if constexpr (Cfg::kTotSmem) {
#pragma unroll
            for (int i = 0; i < kTcMaxN / 2; ++i) {
              tot[i] = tot_s[i * kTcM];
              tot_s[i * kTcM] = 0.0f;
            }
          }
          tc_write_tile(p, tile_keys, t.m0, t.n0, t.nc, quarter, half, lane, tot);
        }
        TCP_ACC(c_write);
        item_release(d_it);
        ++d_it;
        d_gl = 0;
        d_last_kg = d_it * p.num_kb + group_last(0);
      } else {
        ++d_gl;
        d_last_kg = d_it * p.num_kb + group_last(d_gl);
      }
      ++drained;
    };
    // item of the group being folded, cached per warp in shared memory
    // (item_of divides; registers are scarce in the 18-warp kernels)
    int f_it = -1;
    int4* const f_cache = &bar->item_cache[Cfg::kItemRing > 8 ? (warp - kGenW0) & 15 : 0];
    auto fold_step = [&]() {
      if (f_it != d_it) {
        const Item ti = item_of(item_id(d_it));
        if (lane == 0) *f_cache = make_int4(ti.m0, ti.n0, ti.nc, 0);
        __syncwarp();
        f_it = d_it;
      }
      const volatile int* fcv = reinterpret_cast<volatile int*>(f_cache);
      const Item t{fcv[0], fcv[1], fcv[2]};
      TCP_T0();
      const int b = drained & 1;
      if (d_chunk < 0) {
        mbar_wait(&bar->acc_full[b], (drained >> 1) & 1);
        tc_fence_after();
        d_chunk = c0;
      }
      // (shared-memory totals: the chunk is a runtime offset, one code copy)
      if (d_chunk < t.nc / 32) {
        const uint32_t d_base = tmem + (static_cast<uint32_t>(32 * quarter) << 16) +
                                static_cast<uint32_t>(b * p.N + half * (t.nc / 2));
        tc_drain_chunk16_smem(d_base, tot_s, d_chunk, TC_DBG(p));
        d_chunk += kTeams;
      }
      if (d_chunk >= t.nc / 32) {  // this warp's chunks folded: release its share
        tc_fence_before();
        __syncwarp();
        if ((threadIdx.x & 31) == 0) {
          if (!leader)
            mbar_arrive_cluster(acc_empty_addr0 + 8u * b);
          else
            mbar_arrive(&bar->acc_empty[b]);
        }
        d_chunk = -1;
        TCP_ACC(c_drain);
        finish_group(t);
      } else {
        TCP_ACC(c_drain);
      }
    };
    const uint32_t epi_sbase =
        smem_u32(epi_stage) + static_cast<uint32_t>(e) * 2u * kEpiStageBytes;
    int chunk_seq = 0;  // staged chunks written by this warp (buffer parity)
    auto fold_next = [&](const Item& t) {
      { TCP_T0();
      tc_drain(p, bar, !leader, acc_empty_addr0, tmem, drained, t.nc, quarter, half, tot);
      TCP_ACC(c_drain); }
      if (warp == kGenW0 && lane == 0) TCT(d_it, 3);
      if (d_gl == p.groups_per_tile - 1) {
        TCP_T0();
        if constexpr (Cfg::kEpiStage)
          tc_write_tile_staged(p, &tmMaps, epi_sbase, chunk_seq, t.m0, t.n0, t.nc, quarter,
                               half, lane, tot);
        else
          tc_write_tile(p, tile_keys, t.m0, t.n0, t.nc, quarter, half, lane, tot);
        TCP_ACC(c_write);
        if (warp == kGenW0 && lane == 0) TCT(d_it, 4);
        item_release(d_it);
        ++d_it;
        d_gl = 0;
        d_last_kg = d_it * p.num_kb + group_last(0);
      } else {
        ++d_gl;
        d_last_kg = d_it * p.num_kb + group_last(d_gl);
      }
      ++drained;
    };
    { TCP_T0();
    if constexpr (kAMode != kAFromTma) {
      // generator thread: TMEM lane (row) 32*quarter + lane, K columns
      // [16*half, +16) of each 32-column A block
      const int r = 32 * quarter + lane;
      const uint32_t lane_base = tmem + (static_cast<uint32_t>(32 * quarter) << 16);
      using Gen = typename std::conditional<
          kAMode == kASinc, SincGen,
          typename std::conditional<kAMode == kALoad, WLoadGen, PhaseGen<kF16, kTeams>>::type>::type;
      Gen gen;
      // global K block kg (across items) and its stage ring position; a team
      // takes every kTeams-th block (S >= 2 >= kTeams)
      int kg = team, s = team, ph = 0;
      int n_items = 0;            // items seen so far (the fold trails them)
      for (int it = 0;; ++it) {
        const int gid = item_id(it);
        if (gid < 0) break;
        n_items = it + 1;
        const int j = item_of(gid).m0 + r;
        if constexpr (kAMode == kASinc)
          gen.start_tile(p, j, pair_cols);
        else
          gen.start_tile(p);
        const int kg_base = it * p.num_kb;
        for (; kg < kg_base + p.num_kb; kg += kTeams) {
          const int kb = kg - kg_base;
          { TCP_T0();
          mbar_wait(&bar->empty[s], ph ^ 1);
          TCP_ACC(c_gen_wait); }
          { TCP_T0();
          tc_fence_after();  // MMAs that read this stage have completed
          const uint32_t a_col = lane_base + static_cast<uint32_t>(tc_a_tmem_col(p.N, s));
          if constexpr (kAMode == kASinc)
            gen.block(p, j, half, (TC_DBG(p) & 64) ? 0 : kb, a_col, a_col + 32);  // 64: A of block 0
          else
            gen.block(p, j, half, kb, a_col, a_col + 32);
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          TCP_ACC(c_gen); }
          if (lane == 0) {
            if (leader)
              mbar_arrive(&bar->full[s]);
            else  // pair peer: its TMEM A tile is complete (wait::st + fence above)
              mbar_arrive_cluster_relaxed(full_addr0 + 8u * s);
          }
          s += kTeams;
          if (s >= S) {
            s -= S;
            ph ^= 1;
          }
          // fold one chunk of the oldest group whose last K block is at
          // least S behind; with tiles shorter than the fold window (one
          // group of fewer blocks, groups arriving faster than a team's
          // blocks) every such group is folded at once, or the MMA of group
          // g + 2 would wait on a fold that waits for blocks it holds up
          auto fold_due = [&]() {
            return d_chunk >= 0 || (d_it < n_items && d_last_kg <= kg - S);
          };
          if (fold_due()) {
            do {
              fold_step();
            } while (fold_all && fold_due());
          }
        }
      }
      while (d_it < n_items) fold_step();
    } else {
      for (;;) {
        const int gid = item_id(d_it);
        if (gid < 0) break;
        fold_next(item_of(gid));
      }
      if (Cfg::kEpiStage && lane == 0) bulk_wait_all();  // maps written, staging free
    }
    TCP_ACC(c_all); }
    if (warp == kGenW0 && lane == 0) {
      TCP_FLUSH(5, c_gen_wait);
      TCP_FLUSH(6, c_gen);
      TCP_FLUSH(7, c_drain);
      TCP_FLUSH(9, c_write);
      TCP_FLUSH(10, c_all);
    }
  }
#ifdef SRPB_TC_PROFILE
  const long long t_work = clock64();
#endif
  // in-kernel argmax finish: every thread's key atomics are visible device-wide
  // before its CTA counts itself done (one fence per thread, at exit)
  if (p.argmax_out) __threadfence();
  tc_fence_before();
  __syncthreads();
  if (kPair) cluster_sync();  // the pair leaves together (remote arrivals landed)
  if (p.done) {
    // last CTA: keys -> argmax (srpb_keys_to_index), keys, counter and item
    // cursor reset (srpb_argmax_keys_reset) for the next call -- two launches
    // saved
    __shared__ unsigned int s_last;
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(p.done, 1u) == gridDim.x - 1 ? 1u : 0u;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      if (p.argmax_out) {
        for (int f = threadIdx.x; f < p.F; f += blockDim.x) {
          const unsigned long long k = __ldcg(p.keys + f);
          p.argmax_out[f] = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(k));
          p.keys[f] = 0ull;
        }
      }
      if (threadIdx.x == 0) {
        p.done[0] = 0u;  // every CTA has fetched its last (sentinel) item id
        p.done[1] = 0u;
      }
    }
  }
#ifdef SRPB_TC_PROFILE
  if (threadIdx.x == 0) {
    atomicAdd(&g_tc_prof[16], static_cast<unsigned long long>(clock64() - t_entry));
    atomicAdd(&g_tc_prof[18], static_cast<unsigned long long>(clock64() - t_work));
    atomicAdd(&g_tc_prof[19], 1ull);
    unsigned long long g_exit;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_exit));
    g_tc_trace[blockIdx.x][60] = g_entry;
    g_tc_trace[blockIdx.x][61] = g_exit;
    atomicMax(&g_tc_prof[20], ~g_entry);  // earliest entry (complemented)
    atomicMax(&g_tc_prof[21], g_exit);    // latest exit
    atomicMax(&g_tc_prof[22], ~g_exit);   // earliest exit (complemented)
    atomicMax(&g_tc_prof[23], g_entry);   // latest entry
  }
#endif
  if (warp == kMmaWarp) {
    tc_fence_after();
    if (kPair)
      tmem_dealloc_pair(tmem, 512);
    else
      tmem_dealloc(tmem, 512);
  }
}

// --------------------------------------------------------------------- host
namespace {

// Row-major fp32 / fp16 matrix [rows, cols] -> tensor map with a 128-byte
// (32 fp32 or 64 fp16) x box_rows box and 128-byte swizzle (K-major UMMA
// operand tiles); columns past `cols` read as zero.
cudaError_t make_map(CUtensorMap* m, const void* base, int rows, int cols, int box_rows,
                     bool f16) {
  const size_t esz = f16 ? 2 : 4;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * esz};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / esz), static_cast<cuuint32_t>(box_rows)};
  return encode_tensor_map(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                           2, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
}

// Frames per tile: N-tiles of <= 160 frames, multiple of 32.
int pick_n(int F, int hard_cap = kTcMaxN) {
  static int env = -1;  // SRPB_TC_NMAX (experiments): narrower frame tiles
  if (env < 0) {
    const char* e = getenv("SRPB_TC_NMAX");
    env = e ? max(32, atoi(e) / 32 * 32) : 0;
  }
  const int cap = env ? min(env, hard_cap) : hard_cap;
  const int tiles = (F + cap - 1) / cap;
  const int per = (F + tiles - 1) / tiles;
  return (per + 31) / 32 * 32;
}

// CTA pairs by default when there are >= 2 candidate tiles; SRPB_TC_PAIR=0
// forces single-CTA tiles (tuning / A-B comparison).
// Measured on B200 (C2): K4 108.5 us paired vs 116 us single; K2 with one
// generator team 4.36 ms paired vs 3.60 ms single (its 3-stage TMEM A ring
// could not absorb the cross-SM signalling latency) -- with two teams pairs
// win for K2 as well (see conventional_tc).
bool use_pair(int m_tiles, bool default_on) {
  static int env = -2;
  if (env == -2) {
    const char* s = getenv("SRPB_TC_PAIR");
    env = s ? atoi(s) : -1;
  }
  if (m_tiles < 2 || env == 0) return false;
  return env == 1 || default_on;
}

// on-the-fly K4: CTA pairs unless SRPB_OTF_PAIR=0.  With two generator
// teams the kernel is power-bound (sw_power_cap; tensor pipe busy), and the
// Xi stream from L2 is the largest non-MMA energy item (measured at C4,
// F = 320: without B loads the same cycle count ran at 1.61 instead of
// 1.37 GHz); a pair halves each SM's B rows: 143 -> 137 ms (single-team
// round: 148 single vs 151 ms paired).
bool use_pair_otf(int m_tiles) {
  static int env = -2;
  if (env == -2) {
    const char* s = getenv("SRPB_OTF_PAIR");
    env = s ? atoi(s) : -1;
  }
  return m_tiles >= 2 && env != 0;
}

int num_sms();
// Generator modes stream only B (the A operand is generated): with many
// waves, order items candidate tile fastest and schedule them statically so
// a wave's CTAs share each B block in L2 (SRPB_TC_DYNAMIC=1 / 0 overrides;
// measured at C4: K2 read 38.9 TB of DRAM per launch with the dynamic cursor).
void lockstep_items(TcParams& p, bool pair) {
  const int units = max(1, num_sms() / (pair ? 2 : 1));
  const char* e = getenv("SRPB_TC_DYNAMIC");
  const bool many = p.num_items >= 4 * units;
  p.dynamic = e ? (atoi(e) != 0) : !many;
  if (!p.dynamic) {
    p.m_fast = 1;
    p.lockstep = p.done != nullptr && getenv("SRPB_TC_NOLOCKSTEP") == nullptr;
  }
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

// Generator modes fold one 16-column accumulator chunk per generated K block
// (c = N / 32 chunks per group), starting S blocks after the group's last
// block.  The MMA of group g + 2 needs group g folded, and the generator can
// run at most S blocks ahead of the MMA, so every group after the first must
// span at least c - 1 blocks or the generator stalls on a stage the MMA never
// frees (measured: a 2-block tail group hung the kernel).  Groups are at
// least c + 1 blocks and the tile's remainder joins its last group.
// With two generator teams a warp folds every other chunk, one per block of
// its own team (every second block): groups of >= 2 ceil(c / 2) + 1 blocks.
void enforce_fold_window(TcParams& p, int teams = 1) {
  const int c = p.N / 32;
  p.kb_per_group = max(p.kb_per_group, teams == 2 ? 2 * ((c + 1) / 2) + 1 : c + 1);
  p.groups_per_tile = max(1, p.num_kb / p.kb_per_group);
}

// frame-tile cap of the generator kernels (SRPB_TC_GEN_NMAX: 160 or 192)
int gen_nmax() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SRPB_TC_GEN_NMAX");
    v = e ? max(32, min(kTcMaxNGen, atoi(e) / 32 * 32)) : kTcMaxN;
  }
  return v;
}

void finish_params(TcParams& p, int kb_per_group, bool pair, bool f16, int nmax = kTcMaxN) {
  p.N = pick_n(p.F, nmax);
  p.n_tiles = (p.F + p.N - 1) / p.N;
  const int m_tiles = (p.J + kTcM - 1) / kTcM;
  const int cta = pair ? 2 : 1;
  p.m_units = (m_tiles + cta - 1) / cta;
  p.num_items = p.n_tiles * p.m_units;
  p.m_fast = 0;
  p.dynamic = 1;
  p.lockstep = 0;
  // tail-wave split: items beyond the last full wave of `units` CTAs (pairs)
  // run as two frame pieces (widths multiples of 32: the epilogue drains
  // 16-column chunks per column half)
  const int units = max(1, min(p.num_items, num_sms() / cta));
  p.n_piece0 = (p.N / 2 + 31) / 32 * 32;
  p.n_last = getenv("SRPB_TC_NOLAST") ? p.N
                                      : min(p.N, (p.F - (p.n_tiles - 1) * p.N + 31) / 32 * 32);
  // (a narrower last tile already shortens the tail wave: no piece split)
  const bool split = p.N >= 64 && p.n_piece0 < p.N && p.n_last == p.N && p.num_items > units &&
                     p.num_items % units != 0 && getenv("SRPB_TC_NOSPLIT") == nullptr;
  p.full_items = split ? p.num_items / units * units : p.num_items;
  p.n_pieces = 2;
  p.total_items = p.full_items + 2 * (p.num_items - p.full_items);
  p.kb_per_group = max(f16 ? 2 : 4, kb_per_group);
  p.b_box = getenv("SRPB_TC_BOX16") ? 16 : (pair ? p.N / 2 : p.N);
  p.dbg = getenv("SRPB_TC_DBG") ? atoi(getenv("SRPB_TC_DBG")) : 0;
  p.groups_per_tile = max(1, p.num_kb / p.kb_per_group);
}

template <int kAMode, bool kPair, bool kF16>
cudaError_t launch_tc(const CUtensorMap& ah, const CUtensorMap& al, const CUtensorMap& bh,
                      const CUtensorMap& bl, const TcParams& p, cudaStream_t stream,
                      const CUtensorMap* maps_map = nullptr) {
  using Cfg = TcCfg<kAMode, kPair, kF16>;
  TcParams q = p;
  int S = Cfg::kStages;
  if (!Cfg::kASmem) {  // generator modes: as many TMEM A stages as 2N + 64 S <= 512 allows
    S = min(kTcMaxStages, (512 - 2 * p.N) / 64);
    if (getenv("SRPB_TC_GSTAGES")) S = min(S, max(2, atoi(getenv("SRPB_TC_GSTAGES"))));
  } else {  // K4: fill the 227 KB (static 1 KB included)
    S = kTcMaxStages;
    while (S > Cfg::kStages && tc_smem_bytes(p.N, true, kPair, S, Cfg::kEpiStage) + 1024 > 232448)
      --S;
  }
  q.stages = S;
  const size_t smem = tc_smem_bytes(p.N, Cfg::kASmem, kPair, S, Cfg::kEpiStage, Cfg::kTotSmem) +
                      (kAMode == kASinc ? sizeof(int2) * static_cast<size_t>(p.P) : 0);
  auto kern = srp_tc_kernel<kAMode, kPair, kF16>;
  cudaError_t e = allow_dynamic_smem(kern, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  constexpr int cta = kPair ? 2 : 1;
  const int units = min(p.total_items, num_sms() / cta);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(units * cta);
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cta;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_attr_value();
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  // kernels without a staged epilogue never touch the maps map
  e = cudaLaunchKernelEx(&cfg, kern, ah, al, bh, bl, maps_map ? *maps_map : bh, q);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

// K2: B = psi split (fp32 tf32-split or fp16 prescaled by psi_scale)
static cudaError_t conventional_tc(const void* psi_hi, const void* psi_lo, bool f16, float psi_scale,
                                   int F, int P, int Kb, int period, const int32_t* tau_i,
                                   const float* tau_f, int J, float* maps,
                                   unsigned long long* keys, int kb_per_group,
                                   cudaStream_t stream, int32_t* argmax_out = nullptr,
                                   unsigned int* done = nullptr) {
  if (F == 0 || J == 0) return cudaSuccess;
  TcParams p{};
  p.F = F;
  p.J = J;
  p.kb_per_pair = Kb / (f16 ? 32 : 16);  // K blocks per pair: 2 Kb elements
  p.num_kb = P * p.kb_per_pair;
  // CTA pairs by default: with two generator teams the pair's cross-SM
  // signalling is absorbed (measured C4 shapes, F = 320, J = 148k: 125.5 ms
  // single-team single-CTA, 124.5 two teams, 117 two teams + pairs)
  const bool pair = use_pair((J + kTcM - 1) / kTcM, true);
  finish_params(p, kb_per_group, pair, f16, gen_nmax());
  enforce_fold_window(p, TcCfg<kAPhase, false, true>::kTeams);
  p.scale = f16 ? 2.0f / (kF16PhaseScale * psi_scale) : 2.0f;
  p.maps = maps;
  p.keys = keys;
  p.argmax_out = argmax_out;
  p.done = done;
  lockstep_items(p, pair);
  p.tau_i = tau_i;
  p.tau_f = tau_f;
  p.period = period;
  p.mask = (period & (period - 1)) == 0 ? period - 1 : 0;
  p.inv_period = 1.0f / static_cast<float>(period);
  CUtensorMap bh, bl;
  const int cols = 2 * P * Kb;
  cudaError_t e = make_map(&bh, psi_hi, F, cols, p.b_box, f16);
  if (e == cudaSuccess) e = make_map(&bl, psi_lo, F, cols, p.b_box, f16);
  if (e != cudaSuccess) return e;
  if (f16)
    return pair ? launch_tc<kAPhase, true, true>(bh, bl, bh, bl, p, stream)
                : launch_tc<kAPhase, false, true>(bh, bl, bh, bl, p, stream);
  return pair ? launch_tc<kAPhase, true, false>(bh, bl, bh, bl, p, stream)
              : launch_tc<kAPhase, false, false>(bh, bl, bh, bl, p, stream);
}

// K4: A = W split, B = Xi split; maps = (W_hi + W_lo)(Xi_hi + Xi_lo)^T * scale.
// (Measured: splitting the argmax into a K5 pass over the stored maps saves
// 6 us of K4 epilogue but costs 16 us of K5, so it stays fused.)
static cudaError_t interp_tc(const void* w_hi, const void* w_lo, const void* xi_hi,
                             const void* xi_lo, bool f16, float scale, int F, int J, int T_pad,
                             float* maps, unsigned long long* keys, int kb_per_group,
                             cudaStream_t stream, int32_t* argmax_out = nullptr,
                             unsigned int* done = nullptr) {
  if (F == 0 || J == 0) return cudaSuccess;
  TcParams p{};
  p.F = F;
  p.J = J;
  const int kbe = f16 ? kTcKBlock16 : kTcKBlock;
  p.num_kb = (T_pad + kbe - 1) / kbe;  // partial last block: TMA zero-fills
  const bool pair = use_pair((J + kTcM - 1) / kTcM, true);
  finish_params(p, kb_per_group, pair, f16);
  // K4's pieces cost only their MMAs (W is re-read, mostly from L2): split
  // the tail items finer than the generator kernels can afford
  if (p.full_items < p.num_items) {
    const char* e = getenv("SRPB_TC_SPLITK");
    const int k = e ? atoi(e) : 2;
    if (k > 2) {
      p.n_piece0 = max(32, (p.N / k + 31) / 32 * 32);
      p.n_pieces = (p.N + p.n_piece0 - 1) / p.n_piece0;
      p.total_items = p.full_items + p.n_pieces * (p.num_items - p.full_items);
    }
  }
  p.scale = scale;
  p.maps = maps;
  p.keys = keys;
  p.argmax_out = argmax_out;
  p.done = done;
  static const bool ts = getenv("SRPB_K4_TS") != nullptr;
  if (f16 && ts && T_pad % 8 == 0) {
    // A (W split) loaded into TMEM by the generator warps: TS MMA
    p.kb_per_group = max(p.kb_per_group, 2);
    enforce_fold_window(p, TcCfg<kALoad, false, true>::kTeams);
    p.full_items = p.num_items;  // no piece split (generator-mode schedule)
    p.total_items = p.num_items;
    p.w_hi = static_cast<const __half*>(w_hi);
    p.w_lo = static_cast<const __half*>(w_lo);
    p.T_pad = T_pad;
    CUtensorMap bh, bl;
    cudaError_t e = make_map(&bh, xi_hi, F, T_pad, p.b_box, true);
    if (e == cudaSuccess) e = make_map(&bl, xi_lo, F, T_pad, p.b_box, true);
    if (e != cudaSuccess) return e;
    return pair ? launch_tc<kALoad, true, true>(bh, bl, bh, bl, p, stream)
                : launch_tc<kALoad, false, true>(bh, bl, bh, bl, p, stream);
  }
  CUtensorMap ah, al, bh, bl;
  cudaError_t e = make_map(&ah, w_hi, J, T_pad, kTcM, f16);
  if (e == cudaSuccess) e = make_map(&al, w_lo, J, T_pad, kTcM, f16);
  if (e == cudaSuccess) e = make_map(&bh, xi_hi, F, T_pad, p.b_box, f16);
  if (e == cudaSuccess) e = make_map(&bl, xi_lo, F, T_pad, p.b_box, f16);
  if (e != cudaSuccess) return e;
  // staged epilogue (pairs): maps [F, J] fp32 leave by TMA in 32 x 16 boxes
  // (needs a 16-byte row pitch: J % 4 == 0; otherwise direct stores)
  CUtensorMap mm;
  p.maps_tma = 0;
  if (pair && maps && J % 4 == 0 && (reinterpret_cast<uintptr_t>(maps) & 15) == 0 &&
      !(TC_DBG(p) & 512)) {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(J), static_cast<cuuint64_t>(F)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(J) * 4};
    cuuint32_t box[2] = {32, static_cast<cuuint32_t>(kEpiChunk)};
    e = encode_tensor_map(&mm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, maps, dims, strides, box,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE);
    if (e != cudaSuccess) return e;
    p.maps_tma = 1;
  }
  const CUtensorMap* mmp = p.maps_tma ? &mm : nullptr;
  if (f16)
    return pair ? launch_tc<kAFromTma, true, true>(ah, al, bh, bl, p, stream, mmp)
                : launch_tc<kAFromTma, false, true>(ah, al, bh, bl, p, stream);
  return pair ? launch_tc<kAFromTma, true, false>(ah, al, bh, bl, p, stream, mmp)
              : launch_tc<kAFromTma, false, false>(ah, al, bh, bl, p, stream);
}

// K4 with the sinc weights generated in TMEM (no stored W): B = Xi fp16 split
cudaError_t launch_interp_tc16_onthefly(const int32_t* sx_i, const float* sx_f, int P,
                                        const int32_t* off, const int32_t* reach,
                                        const void* xi_hi, const void* xi_lo, float xi_scale,
                                        int F, int J, int T_pad, float* maps,
                                        unsigned long long* keys, int kb_per_group,
                                        int32_t* argmax_out, unsigned int* done,
                                        cudaStream_t stream) {
  if (F == 0 || J == 0) return cudaSuccess;
  TcParams p{};
  p.argmax_out = argmax_out;
  p.done = done;
  p.F = F;
  p.J = J;
  p.num_kb = (T_pad + kTcKBlock16 - 1) / kTcKBlock16;
  // CTA pairs: each SM streams half of the tile's B rows (Xi is re-read from
  // L2 by every candidate tile; the weights are generated, not loaded)
  const bool pair = use_pair_otf((J + kTcM - 1) / kTcM);
  finish_params(p, kb_per_group, pair, true, gen_nmax());
  enforce_fold_window(p, pair ? TcCfg<kASinc, true, true>::kTeams : TcCfg<kASinc, false, true>::kTeams);
  // candidate tiles fastest: the CTAs in flight share one frame tile's Xi
  // rows in L2 instead of streaming every frame tile's
  // (dynamic items: the tile's Xi rows fit L2, 92 MB at C4; measured with
  // the static lockstep schedule: 2.13 vs 2.06 s per C4 step)
  p.m_fast = getenv("SRPB_OTF_NFAST") ? 0 : 1;
  // SRPB_OTF_LOCKSTEP=1 (experiments): static items with the wave barrier, as K2
  if (getenv("SRPB_OTF_LOCKSTEP") && done) {
    p.dynamic = 0;
    p.lockstep = 1;
  }
  p.scale = 1.0f / (kF16PhaseScale * xi_scale);
  p.maps = maps;
  p.keys = keys;
  p.sx_i = sx_i;
  p.sx_f = sx_f;
  p.off = off;
  p.reach = reach;
  p.P = P;
  CUtensorMap bh, bl;
  cudaError_t e = make_map(&bh, xi_hi, F, T_pad, p.b_box, true);
  if (e == cudaSuccess) e = make_map(&bl, xi_lo, F, T_pad, p.b_box, true);
  if (e != cudaSuccess) return e;
  return pair ? launch_tc<kASinc, true, true>(bh, bl, bh, bl, p, stream)
              : launch_tc<kASinc, false, true>(bh, bl, bh, bl, p, stream);
}

cudaError_t launch_conventional_tc(const float* psi_hi, const float* psi_lo, int F, int P, int Kb,
                                   int period, const int32_t* tau_i, const float* tau_f, int J,
                                   float* maps, unsigned long long* keys, int kb_per_group,
                                   cudaStream_t stream) {
  return conventional_tc(psi_hi, psi_lo, false, 1.0f, F, P, Kb, period, tau_i, tau_f, J, maps,
                         keys, kb_per_group, stream);
}

cudaError_t launch_conventional_tc16(const void* psi_hi, const void* psi_lo, float psi_scale, int F,
                                     int P, int Kb, int period, const int32_t* tau_i,
                                     const float* tau_f, int J, float* maps,
                                     unsigned long long* keys, int kb_per_group,
                                     int32_t* argmax_out, unsigned int* done,
                                     cudaStream_t stream) {
  return conventional_tc(psi_hi, psi_lo, true, psi_scale, F, P, Kb, period, tau_i, tau_f, J, maps,
                         keys, kb_per_group, stream, argmax_out, done);
}

cudaError_t launch_interp_tc(const float* w_hi, const float* w_lo, const float* xi_hi,
                             const float* xi_lo, int F, int J, int T_pad, float* maps,
                             unsigned long long* keys, int kb_per_group, cudaStream_t stream) {
  return interp_tc(w_hi, w_lo, xi_hi, xi_lo, false, 1.0f, F, J, T_pad, maps, keys, kb_per_group,
                   stream);
}

cudaError_t launch_interp_tc16(const void* w_hi, const void* w_lo, float w_scale,
                               const void* xi_hi, const void* xi_lo, float xi_scale, int F, int J,
                               int T_pad, float* maps, unsigned long long* keys, int kb_per_group,
                               int32_t* argmax_out, unsigned int* done, cudaStream_t stream) {
  return interp_tc(w_hi, w_lo, xi_hi, xi_lo, true, 1.0f / (w_scale * xi_scale), F, J, T_pad, maps,
                   keys, kb_per_group, stream, argmax_out, done);
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

// hi = fp16(s x), lo = fp16(s x - hi): operand split for 3xFP16 (s a power
// of two chosen so that |s x| < 65504)
__global__ void f16_split_kernel(const float* __restrict__ x, size_t n, float scale,
                                 __half* __restrict__ hi, __half* __restrict__ lo) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const float v = x[i] * scale;
    const __half h = __float2half_rn(v);
    hi[i] = h;
    lo[i] = __float2half_rn(v - __half2float(h));
  }
}

cudaError_t launch_f16_split(const float* x, size_t n, float scale, void* hi, void* lo,
                             cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const size_t want = (n + 255) / 256;
  const int blocks = static_cast<int>(want < size_t(8 * kNumSMs) ? want : size_t(8 * kNumSMs));
  f16_split_kernel<<<blocks, 256, 0, stream>>>(x, n, scale, static_cast<__half*>(hi),
                                               static_cast<__half*>(lo));
  return cudaGetLastError();
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
extern "C" int srpb_tc_trace_read(unsigned long long* host) {
  cudaError_t e = cudaMemcpyFromSymbol(host, srpb::g_tc_trace, sizeof(unsigned long long) * 160 * 64);
  return static_cast<int>(e);
}
extern "C" int srpb_tc_profile_read(unsigned long long* host16) {
  cudaError_t e = cudaMemcpyFromSymbol(host16, srpb::g_tc_prof, sizeof(unsigned long long) * 24);
  unsigned long long zero[24] = {};
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(srpb::g_tc_prof, zero, sizeof(zero));
  return static_cast<int>(e);
}
#endif
