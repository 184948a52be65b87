// Does TMA multicast raise the per-SM operand ingress the K4 stage ring sees?
// 148 CTAs in clusters of C (1, 2, 4); every CTA runs a 4-stage ring of
// 52 KB stages (K4's pair stage: 4 boxes of 128 rows x 128 B + 2 of 80 rows).
// With C > 1 the CTAs of a cluster need the same data: CTA r loads 1/C of
// each stage and multicasts it to all, so L2 serves each byte once per
// cluster.  Reports bytes landed per cycle per SM.  L2-resident source.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tma_mc_bench tools/tma_mc_bench.cu -lcuda
#include <cudaTypedefs.h>

#include <cstdio>

#include "../paper_2012_09499_b200/csrc/umma.cuh"

using namespace srpb::umma;

constexpr int kS = 4;
constexpr int kBoxRows = 128;                // 16 KB boxes (fp16 rows of 128 B)
constexpr int kBoxes = 3;                    // 48 KB per stage (~K4's 52 KB)
constexpr int kStage = kBoxes * kBoxRows * 128;

template <int C>
__global__ void __launch_bounds__(64, 1) ring(const __grid_constant__ CUtensorMap m, int iters,
                                              int src_rows, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kS], empty[kS];
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = C > 1 ? cluster_ctarank() : 0;
  const int cl = blockIdx.x / C;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C);  // every CTA of the cluster must release it
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (C > 1) cluster_sync();
  long long t0 = clock64();
  if (warp == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % kS;
      mbar_wait(&empty[s], ((it / kS) & 1) ^ 1);
      if (elect_one()) {
        mbar_expect_tx(&full[s], kStage);
        for (int b = 0; b < kBoxes; ++b) {
          if (C > 1 && (b % C) != static_cast<int>(rank)) continue;  // another CTA loads it
          const int row = ((cl * 7 + b * 3 + it) * kBoxRows) % src_rows;
          uint8_t* dst = smem + s * kStage + b * kBoxRows * 128;
          if (C > 1)
            tma_load_2d_mc(dst, &m, &full[s], (it % 5) * 64, row, (1u << C) - 1);
          else
            tma_load_2d(dst, &m, &full[s], (it % 5) * 64, row);
        }
      }
      __syncwarp();
    }
  } else {
    for (int it = 0; it < iters; ++it) {
      const int s = it % kS;
      mbar_wait(&full[s], (it / kS) & 1);
      if (elect_one()) {
        // release the stage in every CTA of the cluster (their producers
        // multicast into it)
        for (int c = 0; c < C; ++c) {
          if (C > 1)
            mbar_arrive_cluster(mapa(&empty[s], c));
          else
            mbar_arrive(&empty[s]);
        }
      }
      __syncwarp();
    }
    const long long t1 = clock64();
    if (threadIdx.x == 32) atomicAdd(out, static_cast<unsigned long long>(t1 - t0));
  }
  __syncthreads();
  if (C > 1) cluster_sync();
}

template <int C>
void run(const CUtensorMap& m, unsigned long long* d, int src_rows) {
  const size_t smem = 1024 + kS * size_t(kStage);
  cudaFuncSetAttribute(ring<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 3000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(d, 0, 8);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148 / C * C);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, ring<C>, m, iters, src_rows, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double cyc = double(h) / (148 / C * C);
    if (rep == 1)
      printf("cluster %d: %.1f B/cycle/SM landed (%s)\n", C, double(kStage) * iters / cyc,
             cudaGetErrorString(e));
  }
}

int main() {
  const int cols = 640, src_rows = 16384;  // fp16 [16384, 640]: 20 MB, L2-resident
  void* src;
  cudaMalloc(&src, size_t(cols) * src_rows * 2);
  cudaMemset(src, 0, size_t(cols) * src_rows * 2);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  CUtensorMap m;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(src_rows)};
  cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
  cuuint32_t box[2] = {64, cuuint32_t(kBoxRows)};
  cuuint32_t es[2] = {1, 1};
  fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, src, dims, strides, box, es,
     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long* d;
  cudaMalloc(&d, 8);
  run<1>(m, d, src_rows);
  run<2>(m, d, src_rows);
  run<4>(m, d, src_rows);
  return 0;
}
