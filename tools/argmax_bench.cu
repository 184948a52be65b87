// Per-column argmax over the 32 lanes of a warp, 80 columns per lane (the
// tcgen05 epilogue's fused K5), 8 warps per SM.  Variants:
//   0: per column CREDUX.max + ballot + lane-0 STS (the current epilogue)
//   1: butterfly transpose-reduce of 64-bit (value, ~row) keys: 31 64-bit
//      exchanges per 32 columns, lane c ends with column c's key
//   2: butterfly on 32-bit values for the max, then per column shfl of the
//      max + ballot for the lowest matching row
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/argmax_bench tools/argmax_bench.cu
#include <cstdint>
#include <cstdio>

constexpr int kCols = 80;

__device__ __forceinline__ uint32_t orderable(float v) {
  uint32_t b = __float_as_uint(v + 0.0f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// 32-column butterfly: in v[0..31] (this lane's row), out: lane l holds the
// reduced value of column l.  Round with offset o keeps the half of the
// columns selected by lane bit o and exchanges the other half.
template <typename T, typename Op>
__device__ __forceinline__ T butterfly32(T (&v)[32], Op op) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16, n = 16; o >= 1; o >>= 1, n >>= 1) {
    const bool up = lane & o;
#pragma unroll
    for (int k = 0; k < n; ++k) {
      const T keep = up ? v[k + n] : v[k];
      const T send = up ? v[k] : v[k + n];
      const T recv = __shfl_xor_sync(0xffffffffu, send, o);
      v[k] = op(keep, recv);
    }
  }
  return v[0];
}

template <int kV>
__global__ void __launch_bounds__(256) am(int iters, const float* in, unsigned long long* out,
                                          long long* cyc) {
  __shared__ unsigned long long tk[8][kCols];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float tot[kCols];
#pragma unroll
  for (int i = 0; i < kCols; ++i) tot[i] = in[(blockIdx.x * 256 + threadIdx.x) * 3 + i % 7];
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (kV == 0) {
#pragma unroll
      for (int i = 0; i < kCols; ++i) {
        const uint32_t bits = orderable(tot[i]);
        const uint32_t mx = __reduce_max_sync(0xffffffffu, bits);
        const uint32_t hit = __ballot_sync(0xffffffffu, bits == mx);
        if (lane == 0)
          tk[warp][i] = (static_cast<unsigned long long>(mx) << 32) | (0xFFFFFFFFu - (__ffs(hit) - 1));
      }
    } else {
#pragma unroll
      for (int g = 0; g < (kCols + 31) / 32; ++g) {
        if (kV == 1) {
          unsigned long long k[32];
#pragma unroll
          for (int c = 0; c < 32; ++c)
            k[c] = g * 32 + c < kCols
                       ? (static_cast<unsigned long long>(orderable(tot[(g * 32 + c) % kCols])) << 32) |
                             (0xFFFFFFFFu - lane)
                       : 0ull;
          const unsigned long long r =
              butterfly32(k, [](unsigned long long a, unsigned long long b) { return a > b ? a : b; });
          if (g * 32 + lane < kCols) tk[warp][g * 32 + lane] = r;
        } else {
          uint32_t b[32], v[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            b[c] = g * 32 + c < kCols ? orderable(tot[(g * 32 + c) % kCols]) : 0u;
            v[c] = b[c];
          }
          const uint32_t mx = butterfly32(v, [](uint32_t a, uint32_t c) { return a > c ? a : c; });
          unsigned long long mine = 0;
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const uint32_t m = __shfl_sync(0xffffffffu, mx, c);
            const uint32_t hit = __ballot_sync(0xffffffffu, b[c] == m);
            if (lane == c) mine = (static_cast<unsigned long long>(m) << 32) | (0xFFFFFFFFu - (__ffs(hit) - 1));
          }
          if (g * 32 + lane < kCols) tk[warp][g * 32 + lane] = mine;
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < kCols; ++i) tot[i] += 1.0f;  // new values each iteration
  }
  long long t1 = clock64();
  if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(cyc), (unsigned long long)(t1 - t0));
  __syncthreads();  // warp 0's last keys are visible to the threads copying them out
  if (threadIdx.x < kCols) out[blockIdx.x * kCols + threadIdx.x] = tk[0][threadIdx.x];
}

int main() {
  const int blocks = 148, iters = 200;
  float* in;
  unsigned long long* out[3];
  long long* cyc;
  cudaMalloc(&in, blocks * 256 * 3 * sizeof(float) + 4096);
  cudaMemset(in, 0, blocks * 256 * 3 * sizeof(float));
  // distinct values per lane
  float* h = new float[blocks * 256 * 3];
  for (int i = 0; i < blocks * 256 * 3; ++i) h[i] = static_cast<float>((i * 7919) % 10007) - 5000.0f;
  cudaMemcpy(in, h, blocks * 256 * 3 * sizeof(float), cudaMemcpyHostToDevice);
  cudaMalloc(&cyc, 8);
  const char* names[] = {"CREDUX+ballot per column", "butterfly 64-bit keys", "butterfly max + ballot"};
  unsigned long long* hres[3];
  for (int v = 0; v < 3; ++v) {
    cudaMalloc(&out[v], blocks * kCols * 8);
    cudaMemset(cyc, 0, 8);
    if (v == 0) am<0><<<blocks, 256>>>(iters, in, out[v], cyc);
    if (v == 1) am<1><<<blocks, 256>>>(iters, in, out[v], cyc);
    if (v == 2) am<2><<<blocks, 256>>>(iters, in, out[v], cyc);
    cudaError_t e = cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    hres[v] = new unsigned long long[blocks * kCols];
    cudaMemcpy(hres[v], out[v], blocks * kCols * 8, cudaMemcpyDeviceToHost);
    const double per_tile = static_cast<double>(c) / (blocks * 8) / iters;
    printf("%-28s %s  %.0f cycles per 80-column tile per warp (%.1f per column)\n", names[v],
           cudaGetErrorString(e), per_tile, per_tile / kCols);
  }
  int bad1 = 0, bad2 = 0;
  for (int i = 0; i < blocks * kCols; ++i) {
    bad1 += hres[1][i] != hres[0][i];
    bad2 += hres[2][i] != hres[0][i];
  }
  printf("mismatches vs variant 0: butterfly64 %d, butterfly+ballot %d\n", bad1, bad2);
  for (int i = 0, shown = 0; i < blocks * kCols && shown < 6; ++i)
    if (hres[1][i] != hres[0][i]) {
      printf("  col %d: v0 %016llx v1 %016llx v2 %016llx\n", i, hres[0][i], hres[1][i], hres[2][i]);
      ++shown;
    }
  return 0;
}
