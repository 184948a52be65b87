// K5: per-frame argmax over stored maps, lowest index on ties
// (srp.argmax_candidate, pkg/src/srpfast/srp.py:107-109).
//
// HBM-bound: 4 J bytes per frame.  Grid = frames x candidate slices sized to
// fill the 148 SMs; each CTA reduces its slice with float4 loads into one
// packed key (common.cuh) and folds it into keys[f] with a 64-bit atomicMax.
// The K2/K4 kernels fuse the same reduction into their epilogues, so this
// kernel only runs for externally supplied maps.
#include "common.cuh"

namespace srpb {

constexpr int kArgThreads = 256;

__global__ void __launch_bounds__(kArgThreads)
argmax_kernel(const float* __restrict__ maps, int J, int slice, unsigned long long* __restrict__ keys) {
  const int f = blockIdx.y;
  const int j_begin = blockIdx.x * slice;
  const int j_end = min(J, j_begin + slice);
  const float* row = maps + static_cast<size_t>(f) * J;
  // per thread: best orderable bits and its (lowest, ascending scan) index;
  // strict > keeps the first maximum; keys combine across threads
  uint32_t bb = 0u;
  int bj = 0;
  // scalar head until 16-byte alignment of the row pointer
  int j = j_begin;
  while (j < j_end && (reinterpret_cast<uintptr_t>(row + j) & 15u) != 0) {
    if (threadIdx.x == 0) {
      const uint32_t b = orderable_bits(row[j]);
      if (b > bb) { bb = b; bj = j; }
    }
    ++j;
  }
  const int nvec = (j_end - j) / 4;
  const float4* v4 = reinterpret_cast<const float4*>(row + j);
#pragma unroll 4
  for (int e = threadIdx.x; e < nvec; e += blockDim.x) {
    const float4 v = __ldcs(v4 + e);
    const int jj = j + 4 * e;
    const uint32_t b0 = orderable_bits(v.x), b1 = orderable_bits(v.y);
    const uint32_t b2 = orderable_bits(v.z), b3 = orderable_bits(v.w);
    if (b0 > bb) { bb = b0; bj = jj; }
    if (b1 > bb) { bb = b1; bj = jj + 1; }
    if (b2 > bb) { bb = b2; bj = jj + 2; }
    if (b3 > bb) { bb = b3; bj = jj + 3; }
  }
  for (int jj = j + 4 * nvec + threadIdx.x; jj < j_end; jj += blockDim.x) {
    const uint32_t b = orderable_bits(row[jj]);
    if (b > bb) { bb = b; bj = jj; }
  }
  unsigned long long best =
      bb != 0u ? (static_cast<unsigned long long>(bb) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(bj))
               : 0ull;
  best = warp_key_max(best);
  __shared__ unsigned long long s_best[kArgThreads / 32];
  if ((threadIdx.x & 31) == 0) s_best[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kArgThreads / 32; ++w) best = key_max(best, s_best[w]);
    best = key_max(best, s_best[0]);
    if (best != 0ull) atomicMax(keys + f, best);
  }
}

// fp64 maps (host-built SrpMap values): one CTA per frame, (value, index)
// reduction with numpy's rule (first maximum wins).
__global__ void __launch_bounds__(kArgThreads)
argmax_f64_kernel(const double* __restrict__ maps, int J, int32_t* __restrict__ idx) {
  const int f = blockIdx.x;
  const double* row = maps + static_cast<size_t>(f) * J;
  double bv = -INFINITY;
  int bj = -1;
  for (int j = threadIdx.x; j < J; j += blockDim.x) {
    const double v = row[j];
    if (bj < 0 || v > bv) { bv = v; bj = j; }  // strided j ascending: first max kept
  }
  __shared__ double s_v[kArgThreads];
  __shared__ int s_j[kArgThreads];
  s_v[threadIdx.x] = bv;
  s_j[threadIdx.x] = bj;
  __syncthreads();
  for (int w = kArgThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double ov = s_v[threadIdx.x + w];
      const int oj = s_j[threadIdx.x + w];
      const double mv = s_v[threadIdx.x];
      const int mj = s_j[threadIdx.x];
      if (oj >= 0 && (mj < 0 || ov > mv || (ov == mv && oj < mj))) {
        s_v[threadIdx.x] = ov;
        s_j[threadIdx.x] = oj;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) idx[f] = s_j[0];
}

__global__ void keys_reset_kernel(unsigned long long* keys, int F) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < F) keys[f] = 0ull;
}

__global__ void keys_to_index_kernel(const unsigned long long* __restrict__ keys, int F,
                                     int32_t* __restrict__ idx) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f < F) idx[f] = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(keys[f] & 0xFFFFFFFFull));
}

cudaError_t launch_argmax(const float* maps, int F, int J, unsigned long long* keys,
                          cudaStream_t stream) {
  if (F == 0 || J == 0) return cudaSuccess;
  // about 8 CTAs per SM in total, slices of >= 4096 candidates
  int slices = (8 * kNumSMs + F - 1) / F;
  int slice = (J + slices - 1) / slices;
  slice = max(4096, (slice + 3) & ~3);
  slices = (J + slice - 1) / slice;
  dim3 grid(slices, F);
  argmax_kernel<<<grid, kArgThreads, 0, stream>>>(maps, J, slice, keys);
  return cudaGetLastError();
}

cudaError_t launch_argmax_f64(const double* maps, int F, int J, int32_t* idx,
                              cudaStream_t stream) {
  if (F == 0 || J == 0) return cudaSuccess;
  argmax_f64_kernel<<<F, kArgThreads, 0, stream>>>(maps, J, idx);
  return cudaGetLastError();
}

cudaError_t launch_keys_reset(unsigned long long* keys, int F, cudaStream_t stream) {
  if (F == 0) return cudaSuccess;
  keys_reset_kernel<<<(F + 255) / 256, 256, 0, stream>>>(keys, F);
  return cudaGetLastError();
}

cudaError_t launch_keys_to_index(const unsigned long long* keys, int F, int32_t* idx,
                                 cudaStream_t stream) {
  if (F == 0) return cudaSuccess;
  keys_to_index_kernel<<<(F + 255) / 256, 256, 0, stream>>>(keys, F, idx);
  return cudaGetLastError();
}

}  // namespace srpb
