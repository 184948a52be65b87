// Throughput of warp cross-lane ops on sm_100a: REDUX.MAX (u32), SHFL.BFLY,
// VOTE.ballot, with 8 warps per SM (the SRP epilogue configuration).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/xlane_bench tools/xlane_bench.cu
#include <cstdio>

template <int kOp>
__global__ void __launch_bounds__(256) xl(int iters, unsigned* out) {
  unsigned v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * 977u + i * 131u;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (kOp == 0) v[i] = __reduce_max_sync(0xffffffffu, v[i]) + (unsigned)i;
      if (kOp == 1) v[i] = max(v[i], __shfl_xor_sync(0xffffffffu, v[i], 1 << (i & 4))) + 1u;
      if (kOp == 2) v[i] = __ballot_sync(0xffffffffu, v[i] & 1u) + v[i] * 3u;
    }
  }
  long long t1 = clock64();
  unsigned acc = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) acc ^= v[i];
  if (acc == 0x12345u) out[1] = acc;
  if (threadIdx.x == 0) atomicAdd(out, (unsigned)((t1 - t0) / iters));
}

int main() {
  unsigned* d;
  cudaMalloc(&d, 8);
  const char* names[] = {"REDUX.MAX.u32", "SHFL.BFLY+IMNMX", "VOTE.ballot"};
  for (int op = 0; op < 3; ++op) {
    cudaMemset(d, 0, 8);
    if (op == 0) xl<0><<<148, 256>>>(1000, d);
    if (op == 1) xl<1><<<148, 256>>>(1000, d);
    if (op == 2) xl<2><<<148, 256>>>(1000, d);
    cudaDeviceSynchronize();
    unsigned h;
    cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    // per block: cycles per iteration (16 ops per warp, 8 warps)
    printf("%-18s %.1f cycles per 16 ops/warp with 8 warps -> %.2f cycles per warp-op per SM\n",
           names[op], h / 148.0, h / 148.0 / (16.0 * 8.0));
  }
  return 0;
}
