// Issue throughput of the weight generator's instructions on B200 (sm_100a):
// MUFU.RCP, F2FP.F16.F32.PACK_AB, HADD2.F32 (f16 -> f32), FADD2, FFMA.
// 1 CTA/SM x 8 warps, 16 independent chains per thread, inline PTX so the
// compiler keeps exactly one instruction per chain per step; prints lanes per
// cycle per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/xu_bench tools/xu_bench.cu
#include <cstdint>
#include <cstdio>

constexpr int kChains = 16;

template <int OP>
__global__ void __launch_bounds__(256) bench(uint32_t* out, int iters, unsigned long long* cyc) {
  uint32_t r[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) r[i] = 0x3f800000u + threadIdx.x * 7u + i;  // ~1.0f
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      if (OP == 0)
        asm volatile("{\n .reg .f32 t;\n rcp.approx.ftz.f32 t, %0;\n mov.b32 %0, t;\n}" : "+r"(r[i]));
      else if (OP == 1)  // pack two fp32 into f16x2 (second operand: the next chain)
        asm volatile("cvt.rn.f16x2.f32 %0, %0, %1;" : "+r"(r[i]) : "r"(r[(i + 1) % kChains]));
      else if (OP == 2) {  // f16 (low half) -> f32
        asm volatile("{\n .reg .b16 lo, hi;\n mov.b32 {lo, hi}, %0;\n cvt.f32.f16 %0, lo;\n}"
                     : "+r"(r[i]));
      } else if (OP == 3) {  // packed f32x2 add on (r[i], r[i+1]) pairs
        if ((i & 1) == 0)
          asm volatile("{\n .reg .b64 a, b;\n mov.b64 a, {%0, %1};\n add.rn.f32x2 a, a, a;\n"
                       " mov.b64 {%0, %1}, a;\n}"
                       : "+r"(r[i]), "+r"(r[i + 1]));
      } else {
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+r"(r[i]));
      }
    }
  }
  const long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s ^= r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) atomicAdd(cyc, static_cast<unsigned long long>(t1 - t0));
}

int main() {
  uint32_t* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 148 * 256 * 4);
  cudaMalloc(&cyc, 8);
  const char* names[5] = {"MUFU.RCP", "F2FP.PACK_AB", "cvt f16->f32", "FADD2", "FFMA"};
  const int iters = 4000;
  for (int op = 0; op < 5; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(cyc, 0, 8);
      if (op == 0) bench<0><<<148, 256>>>(out, iters, cyc);
      if (op == 1) bench<1><<<148, 256>>>(out, iters, cyc);
      if (op == 2) bench<2><<<148, 256>>>(out, iters, cyc);
      if (op == 3) bench<3><<<148, 256>>>(out, iters, cyc);
      if (op == 4) bench<4><<<148, 256>>>(out, iters, cyc);
      cudaDeviceSynchronize();
      unsigned long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double cyc_per_cta = double(c) / 148.0;
      const double ops = 256.0 * iters * (op == 3 ? kChains / 2 : kChains);  // thread-ops per CTA
      if (rep == 1) printf("%-14s %7.1f lanes/cycle/SM\n", names[op], ops / cyc_per_cta);
    }
  }
  return 0;
}
