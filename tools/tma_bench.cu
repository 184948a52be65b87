// Per-SM TMA ingress throughput on sm_100a: a 3-stage ring of SW128 2D tensor
// loads (32 fp32 x R rows per box, like the SRP kernels' operand tiles), the
// consumer releasing each stage as soon as it lands.  148 CTAs, data L2-resident.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tma_bench tools/tma_bench.cu
#include <cudaTypedefs.h>

#include <cstdio>

#include "../paper_2012_09499_b200/csrc/umma.cuh"

using namespace srpb::umma;

__global__ void __launch_bounds__(64, 1) ring(const __grid_constant__ CUtensorMap m, int rows_per_box,
                                              int boxes_per_stage, int iters, int src_rows, int S,
                                              unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[8], empty[8];
  const int warp = threadIdx.x >> 5;
  const uint32_t box_bytes = rows_per_box * 128;
  const uint32_t stage_bytes = box_bytes * boxes_per_stage;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  long long t0 = clock64();
  if (warp == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % S;
      mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
      if (elect_one()) {
        mbar_expect_tx(&full[s], stage_bytes);
        for (int b = 0; b < boxes_per_stage; ++b)
          tma_load_2d(smem + s * stage_bytes + b * box_bytes, &m, &full[s], (it % 19) * 32,
                      ((blockIdx.x * 7 + b * 3 + it) * rows_per_box) % src_rows);
      }
      __syncwarp();
    }
  } else {
    for (int it = 0; it < iters; ++it) {
      const int s = it % S;
      mbar_wait(&full[s], (it / S) & 1);
      if (elect_one()) mbar_arrive(&empty[s]);
      __syncwarp();
    }
    long long t1 = clock64();
    if (threadIdx.x == 32) atomicAdd(out, static_cast<unsigned long long>(t1 - t0));
  }
}

int main() {
  const int cols = 608, src_rows = 65536;
  float* src;
  cudaMalloc(&src, size_t(cols) * src_rows * 4);
  cudaMemset(src, 0, size_t(cols) * src_rows * 4);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  unsigned long long* d;
  cudaMalloc(&d, 8);
  struct Cfg { int rows, boxes; const char* what; } cfgs[] = {
      {128, 4, "K4 A stage (4 x 128 rows)"}, {160, 2, "B stage N=160 (2 x 160)"},
      {80, 4, "4 x 80 rows"}, {256, 2, "2 x 256 rows"}, {64, 8, "8 x 64 rows"}};
  for (int S = 2; S <= 6; ++S)
  for (auto c : cfgs) {
    if (size_t(S) * c.rows * 128 * c.boxes > 220000) continue;
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(src_rows)};
    cuuint64_t strides[1] = {cuuint64_t(cols) * 4};
    cuuint32_t box[2] = {32, cuuint32_t(c.rows)};
    cuuint32_t es[2] = {1, 1};
    fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int stage = c.rows * 128 * c.boxes;
    const size_t smem = 1024 + S * size_t(stage);
    cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int iters = 3000;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(d, 0, 8);
      ring<<<148, 64, smem>>>(m, c.rows, c.boxes, iters, src_rows, S, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h = 0;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      const double cyc = double(h) / 148.0;
      if (rep == 1)
        printf("S=%d %-28s stage %6d B: %.1f B/cycle/SM (%s)\n", S, c.what, stage,
               double(stage) * iters / cyc, cudaGetErrorString(e));
    }
  }
  return 0;
}
