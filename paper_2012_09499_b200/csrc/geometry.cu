// Plan build on the device: candidate TDOAs and their phase / sinc splits.
//
// Restates geometry.build_tdoa_table (pkg/src/srpfast/geometry.py:365-398)
// fused with the host-side splits the plan needs:
//   near field  tau[j,p] = (|q_j - p_m| - |q_j - p_m'|) / c   (:383-389)
//   far field   tau[j,p] = (p_m - p_m') . r_j / c             (:375-381)
//   conventional phase split  x = (w_1 tau) N / 2pi = i + f, i mod N
//   sinc split                x = tau / T = i + f            (srp.py:310)
// (rint, |f| <= 1/2; i int32, f float32), plus the bound check
// |tau| <= d/c + slack (:390-392) reported through a flag.  All arithmetic
// is fp64 with explicit round-to-nearest operations in the reference's
// order (no FMA contraction), so the splits match the host restatement.
// Thread per (candidate, pair), candidates fastest ([P, J] outputs).
#include "common.cuh"

namespace srpb {

struct TdoaSplitArgs {
  const double* pos;  // [M, 3]
  const double* pts;  // [J, 3]: points (near) or unit directions (far)
  int J, P, far_field;
  const int32_t* pm;
  const int32_t* pmp;
  double c, omega1, two_pi, sample_period, slack;
  int period;
  const double* bounds;  // [P]
  int32_t* conv_ti;      // [P, J] or NULL
  float* conv_tf;
  int32_t* sx_i;         // [P, J] or NULL
  float* sx_f;
  double* tau;           // [J, P] or NULL (non-harmonic conventional kernel)
  int* violation;        // set to 1 when a bound is exceeded
};

__device__ __forceinline__ double dist3(const double* q, const double* p) {
  const double dx = __dsub_rn(q[0], p[0]), dy = __dsub_rn(q[1], p[1]),
               dz = __dsub_rn(q[2], p[2]);
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

__global__ void tdoa_split_kernel(const TdoaSplitArgs a) {
  const int p = blockIdx.y;
  const int m = __ldg(a.pm + p), mp = __ldg(a.pmp + p);
  const double* pa = a.pos + 3 * m;
  const double* pb = a.pos + 3 * mp;
  const double bound = __dadd_rn(__ldg(a.bounds + p), a.slack);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < a.J; j += gridDim.x * blockDim.x) {
    const double* q = a.pts + 3 * static_cast<size_t>(j);
    double tau;
    if (a.far_field) {
      const double d0 = __dsub_rn(pa[0], pb[0]), d1 = __dsub_rn(pa[1], pb[1]),
                   d2 = __dsub_rn(pa[2], pb[2]);
      const double dot =
          __dadd_rn(__dadd_rn(__dmul_rn(q[0], d0), __dmul_rn(q[1], d1)), __dmul_rn(q[2], d2));
      tau = __ddiv_rn(dot, a.c);
    } else {
      tau = __ddiv_rn(__dsub_rn(dist3(q, pa), dist3(q, pb)), a.c);
    }
    if (fabs(tau) > bound) atomicOr(a.violation, 1);
    const size_t o = static_cast<size_t>(p) * a.J + j;
    if (a.conv_ti) {
      const double x = __ddiv_rn(__dmul_rn(__dmul_rn(a.omega1, tau), static_cast<double>(a.period)),
                                 a.two_pi);
      const double i = rint(x);
      long long ii = static_cast<long long>(i) % a.period;
      if (ii < 0) ii += a.period;
      a.conv_ti[o] = static_cast<int32_t>(ii);
      a.conv_tf[o] = static_cast<float>(__dsub_rn(x, i));
    }
    if (a.sx_i) {
      const double x = __ddiv_rn(tau, a.sample_period);
      const double i = rint(x);
      a.sx_i[o] = static_cast<int32_t>(i);
      a.sx_f[o] = static_cast<float>(__dsub_rn(x, i));
    }
    if (a.tau) a.tau[static_cast<size_t>(j) * a.P + p] = tau;
  }
}

cudaError_t launch_tdoa_split(const double* pos, const double* pts, int J, const int32_t* pm,
                              const int32_t* pmp, int P, int far_field, double c, double omega1,
                              int period, double sample_period, const double* bounds,
                              double slack, int32_t* conv_ti, float* conv_tf, int32_t* sx_i,
                              float* sx_f, double* tau, int* violation, cudaStream_t stream) {
  if (J == 0) return cudaSuccess;
  TdoaSplitArgs a{pos,   pts,    J,      P,     far_field, pm,   pmp,     c,   omega1,
                  6.283185307179586476925286766559, sample_period, slack, period, bounds,
                  conv_ti, conv_tf, sx_i, sx_f, tau, violation};
  const int blocks = (J + 255) / 256 < 4 * kNumSMs ? (J + 255) / 256 : 4 * kNumSMs;
  tdoa_split_kernel<<<dim3(blocks, P), 256, 0, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace srpb
