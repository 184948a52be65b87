// Microbenchmark: single-CTA tcgen05.mma kind::f16 (M = 128) issue rate with
// A from TMEM (TS, as K2 issues it) vs A from shared memory (SS), N = 160.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/mma_ts_bench tools/mma_ts_bench.cu
#include <cstdio>
#include <cstdlib>

#include "../paper_2012_09499_b200/csrc/umma.cuh"

using namespace srpb::umma;

template <bool kTS>
__global__ void __launch_bounds__(384, 1) bench(int N, int iters, unsigned long long* out, int mode) {
  __shared__ uint64_t sbar[4];
  __shared__ uint64_t sfull[3], sempty[3];
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint64_t spin_done;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  const int a_bytes = 128 * 128, b_bytes = N * 128;
  const int stage = a_bytes + b_bytes;
  for (int i = threadIdx.x; i < 4 * stage / 4; i += blockDim.x) {
    uint32_t h = (i + 1) * 2654435761u;
    h ^= h >> 13;
    reinterpret_cast<uint32_t*>(smem)[i] = (h & 0x83FF83FFu) | 0x34003400u;
  }
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (threadIdx.x == 32) {
    for (int i = 0; i < 4; ++i) mbar_init(&sbar[i], 1);
    mbar_init(&bar, 1);
    mbar_init(&spin_done, 1);
    for (int i = 0; i < 3; ++i) {
      mbar_init(&sfull[i], 1 + 8);
      mbar_init(&sempty[i], 1);
    }
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  long long t0 = clock64();
  if (warp == 1) {
    const uint32_t idesc = idesc_f16(128, N);
    for (int it = 0; it < iters; ++it) {
      const int s = it & 3;
      if (mode == 11) {  // the kernel's ring: wait for the stage's producers
        mbar_wait(&sfull[it % 3], (it / 3) & 1);
        tc_fence_after();
      }
      const uint64_t da = sw128_kmajor_desc(smem_u32(smem + s * stage));
      const uint64_t db = sw128_kmajor_desc(smem_u32(smem + s * stage + a_bytes));
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint32_t o = 2 * ks;
          if (mode >= 7) {
            // the kernel's operands: distinct B_hi / B_lo (B_lo = the next
            // stage's B region), 3 TMEM A stages; 7: (lo,hi) (hi,lo) (hi,hi)
            // as K2/K4 issue them; 8: (lo,hi) (hi,hi) (hi,lo) -- consecutive
            // MMAs on the same B; 9: (hi,hi) (lo,hi) (hi,lo); 10: as 7, A
            // from smem (SS)
            const int s3 = it % 3;
            const uint64_t bh = db + o;
            const uint64_t bl = sw128_kmajor_desc(smem_u32(smem + ((s + 1) & 3) * stage + a_bytes)) + o;
            const uint32_t ah = tmem + 2 * N + 64 * s3 + 8 * ks, al = ah + 32;
            const uint32_t d = tmem + ((it / 10) & 1) * N;
            const uint32_t a0 = (it % 10 > 0 || ks > 0) ? 1u : 0u;
            if (mode == 7 || mode == 11) {
              mma_f16_ts(d, al, bh, idesc, a0);
              mma_f16_ts(d, ah, bl, idesc, 1u);
              mma_f16_ts(d, ah, bh, idesc, 1u);
            } else if (mode == 8) {
              mma_f16_ts(d, al, bh, idesc, a0);
              mma_f16_ts(d, ah, bh, idesc, 1u);
              mma_f16_ts(d, ah, bl, idesc, 1u);
            } else if (mode == 9) {
              mma_f16_ts(d, ah, bh, idesc, a0);
              mma_f16_ts(d, al, bh, idesc, 1u);
              mma_f16_ts(d, ah, bl, idesc, 1u);
            } else {
              const uint64_t sah = da + o, sal = sw128_kmajor_desc(smem_u32(smem + ((s + 1) & 3) * stage)) + o;
              mma_f16(d, sal, bh, idesc, a0);
              mma_f16(d, sah, bl, idesc, 1u);
              mma_f16(d, sah, bh, idesc, 1u);
            }
          } else if (mode >= 2) {  // the K4/K2 pattern: lo*hi + hi*lo + hi*hi, A from TMEM
            const uint32_t ah = tmem + 2 * N + 64 * (s & 1) + 8 * ks, al = ah + 32;
            const uint32_t d = tmem + ((it / 10) & 1) * N;
            mma_f16_ts(d, al, db + o, idesc, (it % 10 > 0 || ks > 0) ? 1u : 0u);
            mma_f16_ts(d, ah, db + o, idesc, 1u);
            mma_f16_ts(d, ah, db + o, idesc, 1u);
          } else if (kTS)  // A: 8 TMEM columns (32 bytes of K) per MMA, columns 2N..
            mma_f16_ts(tmem + (it & 1) * N, tmem + 2 * N + 32 * (it & 1) + 8 * ks, db + o, idesc,
                       (it > 1 || ks > 0) ? 1u : 0u);
          else
            mma_f16(tmem + (it & 1) * N, da + o, db + o, idesc, (it > 1 || ks > 0) ? 1u : 0u);
        }
        if (mode == 11)
          mma_commit(&sempty[it % 3]);
        else if (mode >= 1)
          mma_commit(&sbar[s]);
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 32) mbar_arrive(&spin_done);
    if (threadIdx.x == 32) atomicAdd(out, static_cast<unsigned long long>(t1 - t0));
  }
  if (mode == 11 && (warp == 0 || warp >= 4)) {
    // producer + 8 generator warps: wait for the stage to drain, arrive
    for (int it = 0; it < iters; ++it) {
      if (it >= 3) mbar_wait(&sempty[it % 3], ((it / 3) - 1) & 1);
      tc_fence_after();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&sfull[it % 3]);
    }
  }
  if (warp >= 4 && mode == 4) {  // 8 warps issue ALU work (FFMA chains + MUFU) throughout
    float x0 = threadIdx.x, x1 = x0 + 1.f, x2 = x0 + 2.f, x3 = x0 + 3.f;
    while (!mbar_try_wait(smem_u32(&spin_done), 0)) {
#pragma unroll 16
      for (int i = 0; i < 64; ++i) {
        x0 = fmaf(x0, 0.999f, 0.5f);
        x1 = fmaf(x1, 0.999f, 0.5f);
        x2 = __frcp_rn(x2 + 1.f);
        x3 = fmaf(x3, 0.999f, x0);
      }
    }
    if (x0 + x1 + x2 + x3 == 1234.5f) out[1] = 1;
  } else if (warp >= 4 && (mode == 5 || mode == 6)) {
    // 8 warps stream tcgen05.st (5) / tcgen05.ld (6) to the A columns of the
    // stage the MMAs are not reading (columns 2N + 128.. : a third A slot)
    const uint32_t q = static_cast<uint32_t>(warp & 3) << 21;  // lane quarter (<<16 * 32)
    const uint32_t col = tmem + 2 * N + 128 + 16 * ((warp >> 2) & 1);
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 16 + i;
    while (!mbar_try_wait(smem_u32(&spin_done), 0)) {
      for (int i = 0; i < 8; ++i) {
        if (mode == 5) {
          tmem_st16(col + q, r);
          tmem_wait_st();
        } else {
          tmem_ld16(col + q, r);
          tmem_wait_ld();
          r[0] += r[15];
        }
      }
    }
    if (r[0] == 12345u) out[1] = 1;
  }
  tc_fence_before();
  if (warp >= 4 && mode != 11) mbar_wait(&spin_done, 0);  // mode 3: 8 warps poll a barrier throughout
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main(int argc, char** argv) {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  for (int N : {128, 160}) {
    const int stage = 128 * 128 + N * 128;
    const size_t smem = 1024 + 4 * size_t(stage);
    cudaFuncSetAttribute(bench<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(bench<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int iters = argc > 1 ? atoi(argv[1]) : 4000;
    for (int mode = (argc > 2 ? atoi(argv[2]) : 0); mode < (argc > 2 ? atoi(argv[2]) + 1 : 12); ++mode)
    for (int ts = 0; ts < 2; ++ts)
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(d, 0, 8);
        if (ts)
          bench<true><<<148, mode >= 3 ? 384 : 128, smem>>>(N, iters, d, mode);
        else
          bench<false><<<148, mode >= 3 ? 384 : 128, smem>>>(N, iters, d, mode);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h = 0;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        if (rep == 1)
          printf("mode %d %s N=%3d: %6.1f cycles/MMA (floor %.0f) %s\n", mode, ts ? "TS" : "SS", N,
                 double(h) / 148.0 / ((mode >= 2 ? 12.0 : 4.0) * iters), 128.0 * N / 256.0,
                 cudaGetErrorString(e));
      }
  }
  return 0;
}
