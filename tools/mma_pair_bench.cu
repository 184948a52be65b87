// Microbenchmark: tcgen05.mma.cta_group::2 kind::f16 (M = 256) issue rate
// with resident shared-memory operands, as K4 issues them (SS, 128-byte
// swizzled K-major tiles), for several N.  One cluster of 2 CTAs per SM pair,
// the whole chip busy.  Reports cycles per MMA (K = 16) against the
// max(M,128) N / (256 cta_group) floor.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/mma_pair_bench tools/mma_pair_bench.cu
#include <cstdio>

#include "../paper_2012_09499_b200/csrc/umma.cuh"

using namespace srpb::umma;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
bench(int N, int iters, int random_data, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  // A: 128 rows x 128 B; B: N/2 rows x 128 B (per CTA), 4 copies (stages)
  const int a_bytes = 128 * 128, b_bytes = (N / 2) * 128;
  const int stage = a_bytes + b_bytes;
  for (int i = threadIdx.x; i < 4 * stage / 4; i += blockDim.x) {
    uint32_t h = (i + 1) * 2654435761u;
    h ^= h >> 13;
    reinterpret_cast<uint32_t*>(smem)[i] = random_data ? ((h & 0x83FF83FFu) | 0x34003400u) : 0u;
  }
  if (warp == 0) tmem_alloc_pair(&tbase, 512);
  if (threadIdx.x == 32) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const bool leader = cluster_ctarank() == 0;
  long long t0 = clock64();
  if (leader && warp == 1) {
    const uint32_t idesc = idesc_f16(256, N);
    for (int it = 0; it < iters; ++it) {
      const int s = it & 3;
      const uint64_t da = sw128_kmajor_desc(smem_u32(smem + s * stage));
      const uint64_t db = sw128_kmajor_desc(smem_u32(smem + s * stage + a_bytes));
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint32_t o = 2 * ks;
          mma_f16_pair(tmem + (it & 1) * N, da + o, db + o, idesc, (it > 1 || ks > 0) ? 1u : 0u);
        }
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit_pair_mc(&bar, 0x3);
    __syncwarp();
  }
  if (warp == 1) {
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (leader && threadIdx.x == 32) atomicAdd(out, static_cast<unsigned long long>(t1 - t0));
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) tmem_dealloc_pair(tmem, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int ns[] = {64, 128, 160, 192, 256};
  for (int rnd = 0; rnd < 2; ++rnd)
    for (int N : ns) {
      const int stage = 128 * 128 + (N / 2) * 128;
      const size_t smem = 1024 + 4 * size_t(stage);
      cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int iters = 4000;
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(d, 0, 8);
        bench<<<148, 128, smem>>>(N, iters, rnd, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h = 0;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        const double per = double(h) / 74.0 / (4.0 * iters);
        if (rep == 1)
          printf("%s N=%3d: %6.1f cycles/MMA (floor %.0f) %s\n", rnd ? "random" : "zeros ", N,
                 per, 256.0 * N / 512.0, cudaGetErrorString(e));
      }
    }
  return 0;
}
