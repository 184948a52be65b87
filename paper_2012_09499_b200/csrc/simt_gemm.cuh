// Register-tiled FP32 (SIMT) contraction core shared by K2 and K4:
//
//   maps[f, j] = scale * sum_kk A[j, kk] * B[kk, f]
//
// CTA tile 128 candidates x 64 frames, 256 threads, 8 x 4 outputs per
// thread, K staged through shared memory 32 rows at a time.  The caller
// fills the A tile (generated steering phases for K2, sinc weights for K4)
// and the B tile (frame data); this header provides the inner product and
// the epilogue (optional map store + fused per-frame argmax on packed keys).
#pragma once

#include "common.cuh"

namespace srpb {

constexpr int kTileJ = 128;
constexpr int kTileF = 64;
constexpr int kTileK = 32;
constexpr int kGemmThreads = 256;

struct SimtTiles {
  float A[kTileK][kTileJ];  // A^T tile: row kk, column j
  float B[kTileK][kTileF];  // B tile: row kk, column f
};

// acc[a][b]: candidate j = tj*8 + a, frame f = tf*4 + b.
__device__ __forceinline__ void simt_mma_chunk(const SimtTiles& s, int tj, int tf,
                                               float (&acc)[8][4]) {
#pragma unroll 8
  for (int kk = 0; kk < kTileK; ++kk) {
    const float4 a0 = *reinterpret_cast<const float4*>(&s.A[kk][tj * 8]);
    const float4 a1 = *reinterpret_cast<const float4*>(&s.A[kk][tj * 8 + 4]);
    const float4 b = *reinterpret_cast<const float4*>(&s.B[kk][tf * 4]);
    const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][c] = fmaf(av[a], bv[c], acc[a][c]);
  }
}

// Fold the fp32 partial sums into the fp64 totals and restart them.  K2
// folds once per pair, K4 every 512 lattice columns: the fp32 partials then
// sum at most ~2K terms, and the long reduction over pairs (C4: 496 pairs x
// 1024 terms) runs in fp64 like the reference's per-pair accumulation
// (srp.py:422, srp.py:342).
__device__ __forceinline__ void simt_fold(float (&acc)[8][4], double (&tot)[8][4]) {
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      tot[a][c] += static_cast<double>(acc[a][c]);
      acc[a][c] = 0.0f;
    }
}

// Epilogue: scale, store maps (row-major [F, J]) and fold the per-frame
// argmax of this tile into keys[f] (lowest j on ties).
__device__ __forceinline__ void simt_epilogue(const double (&acc)[8][4], double scale, int j0,
                                              int f0, int J, int F, int tj, int tf,
                                              float* __restrict__ maps,
                                              unsigned long long* __restrict__ keys) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int f = f0 + tf * 4 + c;
    unsigned long long best = 0ull;
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int j = j0 + tj * 8 + a;
      const float v = static_cast<float>(acc[a][c] * scale);
      if (j < J && f < F) {
        if (maps) maps[static_cast<size_t>(f) * J + j] = v;
        best = key_max(best, make_key(v, static_cast<uint32_t>(j)));
      }
    }
    if (keys) {
      // reduce over the 16 lanes (tj = 0..15) that share this frame
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) best = key_max(best, __shfl_xor_sync(0xffffffffu, best, o));
      if (tj == 0 && f < F && best != 0ull) atomicMax(keys + f, best);
    }
  }
}

}  // namespace srpb
