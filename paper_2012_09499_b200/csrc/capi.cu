// C ABI of libsrpb.so (declared in include/srpb.h): argument validation,
// thread-local error messages, and stream-ordered launches.
#include <cstdarg>
#include <cstdio>

#include <cmath>
#include "../../include/srpb.h"
#include "common.cuh"

namespace srpb {
cudaError_t launch_gcc_phat(const float*, int, int, int, const int32_t*, const int32_t*, int, int,
                            double, double, float*, double*, cudaStream_t, void* = nullptr, void* = nullptr, float = 0.0f);
cudaError_t launch_stft(const float*, int, int, int, int, int, int, float*, cudaStream_t);
cudaError_t launch_tdoa_split(const double*, const double*, int, const int32_t*, const int32_t*,
                              int, int, double, double, int, double, const double*, double,
                              int32_t*, float*, int32_t*, float*, double*, int*, cudaStream_t);
int gcc_phat_last_kernels();
cudaError_t launch_gcc_floor(const float*, int, int, int, const int32_t*, const int32_t*, int,
                             double, double*, int32_t*, cudaStream_t);
cudaError_t launch_lattice_from_spectra(const float*, int, int, int, const int32_t*,
                                        const int32_t*, int, int, const double*, double,
                                        const int32_t*, const float*, int, const int32_t*,
                                        const int32_t*, int, int, float*, void*, void*, float,
                                        double, void*, cudaStream_t, const void*, const void*, int*);
int lattice_tc_n(int L);
bool lattice_tc_shape_ok(int M, int P, int Kb, int L, int T_pad);
cudaError_t launch_lattice_tc_twiddles(const double*, int, double, int, void*, void*,
                                       cudaStream_t);
cudaError_t launch_conventional(const float*, int, int, int, int, const int32_t*, const float*,
                                int, float*, unsigned long long*, cudaStream_t);
cudaError_t launch_conventional_general(const float*, int, int, int, const double*,
                                        const double*, int, float*, unsigned long long*,
                                        cudaStream_t);
cudaError_t launch_lattice_twiddles(const double*, int, double, int, float*, cudaStream_t);
cudaError_t launch_lattice(const float*, int, int, int, const float*, int, const int32_t*,
                           const int32_t*, int, int, float*, cudaStream_t);
cudaError_t launch_sinc_table(const int32_t*, const float*, int, int, const int32_t*,
                              const int32_t*, int, float*, cudaStream_t);
cudaError_t launch_interp(const float*, const float*, int, int, int, float*,
                          unsigned long long*, cudaStream_t);
cudaError_t launch_interp_onthefly(const int32_t*, const float*, int, const int32_t*,
                                   const int32_t*, const float*, int, int, int, float*,
                                   unsigned long long*, cudaStream_t);
cudaError_t launch_argmax(const float*, int, int, unsigned long long*, cudaStream_t);
cudaError_t launch_conventional_tc(const float*, const float*, int, int, int, int, const int32_t*,
                                   const float*, int, float*, unsigned long long*, int,
                                   cudaStream_t);
cudaError_t launch_interp_tc(const float*, const float*, const float*, const float*, int, int, int,
                             float*, unsigned long long*, int, cudaStream_t);
cudaError_t launch_tf32_split(const float*, size_t, float*, float*, cudaStream_t);
cudaError_t launch_f16_split(const float*, size_t, float, void*, void*, cudaStream_t);
cudaError_t launch_conventional_tc16(const void*, const void*, float, int, int, int, int,
                                     const int32_t*, const float*, int, float*,
                                     unsigned long long*, int, int32_t*, unsigned int*,
                                     cudaStream_t);
cudaError_t launch_interp_tc16(const void*, const void*, float, const void*, const void*, float,
                               int, int, int, float*, unsigned long long*, int, int32_t*,
                               unsigned int*, cudaStream_t);
cudaError_t launch_interp_tc16_onthefly(const int32_t*, const float*, int, const int32_t*,
                                        const int32_t*, const void*, const void*, float, int, int,
                                        int, float*, unsigned long long*, int, int32_t*,
                                        unsigned int*, cudaStream_t);
cudaError_t launch_argmax_f64(const double*, int, int, int32_t*, cudaStream_t);
cudaError_t launch_keys_reset(unsigned long long*, int, cudaStream_t);
cudaError_t launch_keys_to_index(const unsigned long long*, int, int32_t*, cudaStream_t);
cudaError_t launch_quadform(const float*, int, int, int, const double*, const double*, int, int,
                            const int32_t*, const int32_t*, double*, cudaStream_t);
cudaError_t launch_map_error(const void*, int, const void*, int, int, int, double*, double*,
                             double*, cudaStream_t);
}  // namespace srpb

namespace {

thread_local char g_err[512] = "";

int fail(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return -1;
}

int status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return 0;
  snprintf(g_err, sizeof(g_err), "%s: CUDA error %d (%s)", what, static_cast<int>(e),
           cudaGetErrorString(e));
  return static_cast<int>(e);
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define REQUIRE(cond, ...) \
  do {                     \
    if (!(cond)) return fail(__VA_ARGS__); \
  } while (0)

}  // namespace

extern "C" {

static bool pow2_scale(float s) {
  int e;
  return s > 0.0f && std::isfinite(s) && std::frexp(s, &e) == 0.5f;
}

int srpb_abi_version(void) { return 13; }

// kernels launched by this thread's last srpb_gcc_phat / srpb_gcc_phat_split16
// call (1: the frame-resident single pass; 2: two-pass or row pass + fix-up)
int srpb_last_gcc_kernels(void) { return srpb::gcc_phat_last_kernels(); }

const char* srpb_last_error(void) { return g_err; }

int srpb_stft(const float* x, int M, int L, int frame_length, int hop, int window, int F,
              float* Y, void* stream) {
  REQUIRE(M >= 1 && L >= 1, "srpb_stft: bad shape M=%d L=%d", M, L);
  REQUIRE(frame_length >= 2 && frame_length % 2 == 0,
          "srpb_stft: frame_length must be an even integer >= 2, got %d", frame_length);
  REQUIRE((frame_length & (frame_length - 1)) == 0 ? frame_length <= 8192 : frame_length <= 4096,
          "srpb_stft: frame_length %d too large (power of two <= 8192, else <= 4096)",
          frame_length);
  REQUIRE(hop >= 1, "srpb_stft: hop_length must be >= 1, got %d", hop);
  REQUIRE(window == 0 || window == 1, "srpb_stft: unknown window %d", window);
  REQUIRE(L >= frame_length, "srpb_stft: signal of %d samples is shorter than one frame (%d)", L,
          frame_length);
  REQUIRE(F == (L - frame_length) / hop + 1, "srpb_stft: F=%d, expected %d frames", F,
          (L - frame_length) / hop + 1);
  REQUIRE(x && Y, "srpb_stft: null pointer");
  return status(srpb::launch_stft(x, M, L, frame_length, hop, window, F, Y, S(stream)),
                "srpb_stft");
}

int srpb_tdoa_split(const double* mic_pos, int M, const double* points, int J,
                    const int32_t* pair_m, const int32_t* pair_mp, int P, int far_field,
                    double speed_of_sound, double omega1, int period, double sample_period,
                    const double* bounds, double slack, int32_t* conv_ti, float* conv_tf,
                    int32_t* sx_i, float* sx_f, double* tau, int* violation, void* stream) {
  REQUIRE(M >= 2 && J >= 0 && P >= 1, "srpb_tdoa_split: bad shape M=%d J=%d P=%d", M, J, P);
  REQUIRE(speed_of_sound > 0.0, "srpb_tdoa_split: speed_of_sound must be positive");
  REQUIRE(!conv_ti == !conv_tf && !sx_i == !sx_f, "srpb_tdoa_split: split outputs go in pairs");
  REQUIRE(!conv_ti || (period >= 1 && period <= 46340 && omega1 > 0.0),
          "srpb_tdoa_split: conventional split needs period in [1, 46340] and omega1 > 0");
  REQUIRE(!sx_i || sample_period > 0.0, "srpb_tdoa_split: sinc split needs sample_period > 0");
  REQUIRE(J == 0 || (mic_pos && points && pair_m && pair_mp && bounds && violation),
          "srpb_tdoa_split: null pointer");
  return status(srpb::launch_tdoa_split(mic_pos, points, J, pair_m, pair_mp, P, far_field,
                                        speed_of_sound, omega1, period, sample_period, bounds,
                                        slack, conv_ti, conv_tf, sx_i, sx_f, tau, violation,
                                        S(stream)),
                "srpb_tdoa_split");
}

int srpb_gcc_phat(const float* Y, int F, int M, int Kb, const int32_t* pair_m,
                  const int32_t* pair_mp, int P, int weighting, double floor_rel,
                  double abs_floor, float* Psi, double* floor_out, void* stream) {
  REQUIRE(F >= 0 && M >= 1 && Kb >= 1 && P >= 1, "srpb_gcc_phat: bad shape F=%d M=%d Kb=%d P=%d",
          F, M, Kb, P);
  REQUIRE(M <= 64, "srpb_gcc_phat: at most 64 channels supported, got %d", M);
  REQUIRE(P <= 2016, "srpb_gcc_phat: at most 2016 pairs supported, got %d", P);
  REQUIRE(weighting == SRPB_WEIGHT_PHAT || weighting == SRPB_WEIGHT_IDENTITY,
          "srpb_gcc_phat: unknown weighting %d", weighting);
  REQUIRE(F == 0 || (Y && Psi && pair_m && pair_mp), "srpb_gcc_phat: null pointer");
  REQUIRE(static_cast<long long>(F) * P <= 2147483647LL, "srpb_gcc_phat: F*P too large");
  return status(srpb::launch_gcc_phat(Y, F, M, Kb, pair_m, pair_mp, P, weighting, floor_rel,
                                      abs_floor, Psi, floor_out, S(stream)),
                "srpb_gcc_phat");
}

int srpb_gcc_phat_split16(const float* Y, int F, int M, int Kb, const int32_t* pair_m,
                          const int32_t* pair_mp, int P, int weighting, double floor_rel,
                          double abs_floor, float* Psi, void* Psi_hi, void* Psi_lo,
                          float split_scale, double* floor_out, void* stream) {
  REQUIRE(F >= 0 && M >= 1 && Kb >= 2 && P >= 1,
          "srpb_gcc_phat_split16: bad shape F=%d M=%d Kb=%d P=%d", F, M, Kb, P);
  REQUIRE(Kb % 2 == 0, "srpb_gcc_phat_split16: Kb must be even, got %d", Kb);
  REQUIRE(M <= 64, "srpb_gcc_phat_split16: at most 64 channels supported, got %d", M);
  REQUIRE(P <= 2016, "srpb_gcc_phat_split16: at most 2016 pairs supported, got %d", P);
  REQUIRE(weighting == SRPB_WEIGHT_PHAT,
          "srpb_gcc_phat_split16: the fp16 split needs PHAT-bounded psi (weighting %d)", weighting);
  REQUIRE(pow2_scale(split_scale), "srpb_gcc_phat_split16: split_scale must be a power of two");
  REQUIRE(F == 0 || (Y && Psi_hi && Psi_lo && pair_m && pair_mp),
          "srpb_gcc_phat_split16: null pointer");
  REQUIRE(((reinterpret_cast<uintptr_t>(Y) | reinterpret_cast<uintptr_t>(Psi)) & 15) == 0 &&
              ((reinterpret_cast<uintptr_t>(Psi_hi) | reinterpret_cast<uintptr_t>(Psi_lo)) & 7) == 0,
          "srpb_gcc_phat_split16: Y / Psi must be 16-byte and Psi_hi / Psi_lo 8-byte aligned");
  REQUIRE(static_cast<long long>(F) * P <= 2147483647LL, "srpb_gcc_phat_split16: F*P too large");
  return status(srpb::launch_gcc_phat(Y, F, M, Kb, pair_m, pair_mp, P, weighting, floor_rel,
                                      abs_floor, Psi, floor_out, S(stream), Psi_hi, Psi_lo,
                                      split_scale),
                "srpb_gcc_phat_split16");
}

int srpb_gcc_floor(const float* Y, int F, int M, int Kb, const int32_t* pair_m,
                   const int32_t* pair_mp, int P, double floor_rel, double* floor_out,
                   int32_t* clean_out, void* stream) {
  REQUIRE(F >= 0 && M >= 1 && Kb >= 1 && P >= 1, "srpb_gcc_floor: bad shape F=%d M=%d Kb=%d P=%d",
          F, M, Kb, P);
  REQUIRE(M <= 64, "srpb_gcc_floor: at most 64 channels supported, got %d", M);
  REQUIRE(P <= 2016, "srpb_gcc_floor: at most 2016 pairs supported, got %d", P);
  REQUIRE(floor_out || clean_out, "srpb_gcc_floor: need floor_out and/or clean_out");
  REQUIRE(F == 0 || (Y && pair_m && pair_mp), "srpb_gcc_floor: null pointer");
  return status(srpb::launch_gcc_floor(Y, F, M, Kb, pair_m, pair_mp, P, floor_rel, floor_out,
                                       clean_out, S(stream)),
                "srpb_gcc_floor");
}

int srpb_conventional(const float* Psi, int F, int P, int Kb, int period, const int32_t* tau_i,
                      const float* tau_f, int J, float* maps, unsigned long long* keys,
                      void* stream) {
  REQUIRE(F >= 0 && P >= 1 && Kb >= 1 && J >= 0, "srpb_conventional: bad shape");
  REQUIRE(period >= 1 && period <= 46340, "srpb_conventional: period %d out of range", period);
  REQUIRE(F == 0 || J == 0 || (Psi && tau_i && tau_f), "srpb_conventional: null pointer");
  REQUIRE(maps || keys, "srpb_conventional: need maps and/or keys output");
  return status(srpb::launch_conventional(Psi, F, P, Kb, period, tau_i, tau_f, J, maps, keys,
                                          S(stream)),
                "srpb_conventional");
}

int srpb_conventional_general(const float* Psi, int F, int P, int Kb, const double* omega,
                              const double* tau, int J, float* maps, unsigned long long* keys,
                              void* stream) {
  REQUIRE(F >= 0 && P >= 1 && Kb >= 1 && J >= 0, "srpb_conventional_general: bad shape");
  REQUIRE(F == 0 || J == 0 || (Psi && omega && tau), "srpb_conventional_general: null pointer");
  REQUIRE(maps || keys, "srpb_conventional_general: need maps and/or keys output");
  return status(srpb::launch_conventional_general(Psi, F, P, Kb, omega, tau, J, maps, keys,
                                                  S(stream)),
                "srpb_conventional_general");
}

int srpb_lattice_twiddles(const double* omega, int Kb, double sample_period, int L, float* tw,
                          void* stream) {
  REQUIRE(Kb >= 1 && L >= 0 && omega && tw, "srpb_lattice_twiddles: bad argument");
  REQUIRE(sample_period > 0.0, "srpb_lattice_twiddles: sample_period must be positive");
  return status(srpb::launch_lattice_twiddles(omega, Kb, sample_period, L, tw, S(stream)),
                "srpb_lattice_twiddles");
}

int srpb_lattice(const float* Psi, int F, int P, int Kb, const float* tw, int L,
                 const int32_t* off, const int32_t* reach, int T_pad, float* Xi, void* stream) {
  REQUIRE(F >= 0 && P >= 1 && Kb >= 1 && L >= 0 && T_pad >= 1, "srpb_lattice: bad shape");
  REQUIRE(F == 0 || (Psi && tw && off && reach && Xi), "srpb_lattice: null pointer");
  REQUIRE((reinterpret_cast<uintptr_t>(tw) & 15) == 0, "srpb_lattice: tw must be 16-byte aligned");
  return status(srpb::launch_lattice(Psi, F, P, Kb, tw, L, off, reach, 2 * L + 1, T_pad, Xi,
                                     S(stream)),
                "srpb_lattice");
}

static int lattice_from_spectra(const float* Y, int F, int M, int Kb, const int32_t* pair_m,
                                const int32_t* pair_mp, int P, int weighting,
                                const double* floors, double abs_floor, const int32_t* clean,
                                const float* tw, int L, const int32_t* off, const int32_t* reach,
                                int T_pad, float* Xi, void* Xi_hi, void* Xi_lo, float split_scale,
                                double floor_rel, void* spec_scratch, const void* tc_b_hi,
                                const void* tc_b_lo, int* frame_counters, void* stream) {
  REQUIRE(F >= 0 && M >= 1 && P >= 1 && Kb >= 1 && L >= 0 && T_pad >= 1,
          "srpb_lattice_from_spectra: bad shape");
  REQUIRE(weighting == SRPB_WEIGHT_PHAT || weighting == SRPB_WEIGHT_IDENTITY,
          "srpb_lattice_from_spectra: unknown weighting %d", weighting);
  REQUIRE(weighting != SRPB_WEIGHT_PHAT || floors || abs_floor > 0.0 || floor_rel > 0.0,
          "srpb_lattice_from_spectra: PHAT needs floors, abs_floor > 0 or floor_rel > 0");
  REQUIRE((Xi_hi == nullptr) == (Xi_lo == nullptr),
          "srpb_lattice_from_spectra: Xi_hi and Xi_lo go together");
  REQUIRE(Xi || Xi_hi, "srpb_lattice_from_spectra: need Xi and/or Xi_hi/Xi_lo output");
  REQUIRE(split_scale == 0.0f || pow2_scale(split_scale),
          "srpb_lattice_from_spectra: split_scale must be 0 (tf32) or a power of two (fp16)");
  REQUIRE(F == 0 || (Y && pair_m && pair_mp && tw && off && reach),
          "srpb_lattice_from_spectra: null pointer");
  REQUIRE((reinterpret_cast<uintptr_t>(tw) & 15) == 0,
          "srpb_lattice_from_spectra: tw must be 16-byte aligned");
  return status(srpb::launch_lattice_from_spectra(Y, F, M, Kb, pair_m, pair_mp, P, weighting,
                                                  floors, abs_floor, clean, tw, L, off, reach,
                                                  2 * L + 1,
                                                  T_pad, Xi, Xi_hi, Xi_lo, split_scale, floor_rel,
                                                  spec_scratch, S(stream), tc_b_hi, tc_b_lo,
                                                  frame_counters),
                "srpb_lattice_from_spectra");
}

int srpb_lattice_from_spectra(const float* Y, int F, int M, int Kb, const int32_t* pair_m,
                              const int32_t* pair_mp, int P, int weighting, const double* floors,
                              double abs_floor, const int32_t* clean, const float* tw, int L,
                              const int32_t* off, const int32_t* reach, int T_pad, float* Xi,
                              void* Xi_hi, void* Xi_lo, float split_scale, double floor_rel,
                              void* spec_scratch, void* stream) {
  return lattice_from_spectra(Y, F, M, Kb, pair_m, pair_mp, P, weighting, floors, abs_floor,
                              clean, tw, L, off, reach, T_pad, Xi, Xi_hi, Xi_lo, split_scale,
                              floor_rel, spec_scratch, nullptr, nullptr, nullptr, stream);
}

int srpb_lattice_tc_cols(int L) { return L >= 0 ? srpb::lattice_tc_n(L) : -1; }

int srpb_lattice_tc_supported(int M, int P, int Kb, int L, int T_pad) {
  return M >= 1 && L >= 0 && T_pad >= 1 && getenv("SRPB_LATTICE_SIMT") == nullptr &&
                 srpb::lattice_tc_shape_ok(M, P, Kb, L, T_pad)
             ? 1
             : 0;
}

int srpb_lattice_tc_twiddles(const double* omega, int Kb, double sample_period, int L, void* b_hi,
                             void* b_lo, void* stream) {
  REQUIRE(Kb >= 1 && L >= 0 && omega && b_hi && b_lo, "srpb_lattice_tc_twiddles: bad argument");
  REQUIRE(sample_period > 0.0, "srpb_lattice_tc_twiddles: sample_period must be positive");
  REQUIRE(((reinterpret_cast<uintptr_t>(b_hi) | reinterpret_cast<uintptr_t>(b_lo)) & 15) == 0,
          "srpb_lattice_tc_twiddles: operands must be 16-byte aligned");
  return status(srpb::launch_lattice_tc_twiddles(omega, Kb, sample_period, L, b_hi, b_lo,
                                                 S(stream)),
                "srpb_lattice_tc_twiddles");
}

int srpb_lattice_from_spectra_tc(const float* Y, int F, int M, int Kb, const int32_t* pair_m,
                                 const int32_t* pair_mp, int P, int weighting,
                                 const double* floors, double abs_floor, const int32_t* clean,
                                 const float* tw, int L, const int32_t* off, const int32_t* reach,
                                 int T_pad, float* Xi, void* Xi_hi, void* Xi_lo, float split_scale,
                                 double floor_rel, void* spec_scratch, const void* tc_b_hi,
                                 const void* tc_b_lo, int* frame_counters, void* stream) {
  REQUIRE(!tc_b_hi == !tc_b_lo, "srpb_lattice_from_spectra_tc: tc_b_hi and tc_b_lo go together");
  REQUIRE(((reinterpret_cast<uintptr_t>(tc_b_hi) | reinterpret_cast<uintptr_t>(tc_b_lo)) & 15) == 0,
          "srpb_lattice_from_spectra_tc: tensor-core twiddles must be 16-byte aligned");
  return lattice_from_spectra(Y, F, M, Kb, pair_m, pair_mp, P, weighting, floors, abs_floor,
                              clean, tw, L, off, reach, T_pad, Xi, Xi_hi, Xi_lo, split_scale,
                              floor_rel, spec_scratch, tc_b_hi, tc_b_lo, frame_counters, stream);
}

int srpb_sinc_table(const int32_t* sx_i, const float* sx_f, int J, int P, const int32_t* off,
                    const int32_t* reach, int T_pad, float* W, void* stream) {
  REQUIRE(J >= 0 && P >= 1 && T_pad >= 1, "srpb_sinc_table: bad shape");
  REQUIRE(J == 0 || (sx_i && sx_f && off && reach && W), "srpb_sinc_table: null pointer");
  return status(srpb::launch_sinc_table(sx_i, sx_f, J, P, off, reach, T_pad, W, S(stream)),
                "srpb_sinc_table");
}

int srpb_interp(const float* W, const float* Xi, int F, int J, int T_pad, float* maps,
                unsigned long long* keys, void* stream) {
  REQUIRE(F >= 0 && J >= 0 && T_pad >= 1, "srpb_interp: bad shape");
  REQUIRE(T_pad % 32 == 0, "srpb_interp: T_pad must be a multiple of 32, got %d", T_pad);
  REQUIRE(F == 0 || J == 0 || (W && Xi), "srpb_interp: null pointer");
  REQUIRE(maps || keys, "srpb_interp: need maps and/or keys output");
  return status(srpb::launch_interp(W, Xi, F, J, T_pad, maps, keys, S(stream)), "srpb_interp");
}

int srpb_interp_onthefly(const int32_t* sx_i, const float* sx_f, int P, const int32_t* off,
                         const int32_t* reach, const float* Xi, int F, int J, int T_pad,
                         float* maps, unsigned long long* keys, void* stream) {
  REQUIRE(F >= 0 && J >= 0 && P >= 1 && T_pad >= 1, "srpb_interp_onthefly: bad shape");
  REQUIRE(T_pad % 32 == 0, "srpb_interp_onthefly: T_pad must be a multiple of 32");
  REQUIRE(F == 0 || J == 0 || (sx_i && sx_f && off && reach && Xi),
          "srpb_interp_onthefly: null pointer");
  REQUIRE(maps || keys, "srpb_interp_onthefly: need maps and/or keys output");
  return status(srpb::launch_interp_onthefly(sx_i, sx_f, P, off, reach, Xi, F, J, T_pad, maps,
                                             keys, S(stream)),
                "srpb_interp_onthefly");
}

int srpb_tf32_split(const float* x, size_t n, float* hi, float* lo, void* stream) {
  REQUIRE(n % 4 == 0, "srpb_tf32_split: n must be a multiple of 4, got %zu", n);
  REQUIRE(n == 0 || (x && hi && lo), "srpb_tf32_split: null pointer");
  REQUIRE((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(hi) |
           reinterpret_cast<uintptr_t>(lo)) % 16 == 0, "srpb_tf32_split: pointers must be 16-byte aligned");
  return status(srpb::launch_tf32_split(x, n, hi, lo, S(stream)), "srpb_tf32_split");
}

int srpb_conventional_tc(const float* psi_hi, const float* psi_lo, int F, int P, int Kb, int period,
                         const int32_t* tau_i, const float* tau_f, int J, float* maps,
                         unsigned long long* keys, int kb_per_group, void* stream) {
  REQUIRE(F >= 0 && P >= 1 && Kb >= 16 && J >= 0, "srpb_conventional_tc: bad shape");
  REQUIRE(Kb % 16 == 0, "srpb_conventional_tc: Kb must be a multiple of 16, got %d", Kb);
  REQUIRE(period >= 1 && period <= 46340, "srpb_conventional_tc: period %d out of range", period);
  REQUIRE(kb_per_group >= 1, "srpb_conventional_tc: kb_per_group must be >= 1");
  REQUIRE(F == 0 || J == 0 || (psi_hi && psi_lo && tau_i && tau_f),
          "srpb_conventional_tc: null pointer");
  REQUIRE(maps || keys, "srpb_conventional_tc: need maps and/or keys output");
  return status(srpb::launch_conventional_tc(psi_hi, psi_lo, F, P, Kb, period, tau_i, tau_f, J,
                                             maps, keys, kb_per_group, S(stream)),
                "srpb_conventional_tc");
}


int srpb_f16_split(const float* x, size_t n, float scale, void* hi, void* lo, void* stream) {
  REQUIRE(n == 0 || (x && hi && lo), "srpb_f16_split: null pointer");
  REQUIRE(pow2_scale(scale), "srpb_f16_split: scale must be a positive power of two");
  return status(srpb::launch_f16_split(x, n, scale, hi, lo, S(stream)), "srpb_f16_split");
}

int srpb_conventional_tc16(const void* psi_hi, const void* psi_lo, float psi_scale, int F, int P,
                           int Kb, int period, const int32_t* tau_i, const float* tau_f, int J,
                           float* maps, unsigned long long* keys, int kb_per_group,
                           int32_t* argmax_out, unsigned int* done_counter, void* stream) {
  REQUIRE(F >= 0 && P >= 1 && Kb >= 1 && J >= 0, "srpb_conventional_tc16: bad shape");
  REQUIRE(!argmax_out || (keys && done_counter),
          "srpb_conventional_tc16: argmax_out needs keys and done_counter");
  REQUIRE(Kb % 32 == 0, "srpb_conventional_tc16: Kb must be a multiple of 32, got %d", Kb);
  REQUIRE(period >= 1 && period <= 46340, "srpb_conventional_tc16: period %d out of range",
          period);
  REQUIRE(pow2_scale(psi_scale), "srpb_conventional_tc16: psi_scale must be a power of two");
  REQUIRE(F == 0 || J == 0 || (psi_hi && psi_lo && tau_i && tau_f),
          "srpb_conventional_tc16: null pointer");
  REQUIRE(maps || keys, "srpb_conventional_tc16: need maps and/or keys output");
  return status(srpb::launch_conventional_tc16(psi_hi, psi_lo, psi_scale, F, P, Kb, period, tau_i,
                                               tau_f, J, maps, keys, kb_per_group, argmax_out,
                                               done_counter, S(stream)),
                "srpb_conventional_tc16");
}

int srpb_interp_tc16_onthefly(const int32_t* sx_i, const float* sx_f, int P, const int32_t* off,
                              const int32_t* reach, const void* xi_hi, const void* xi_lo,
                              float xi_scale, int F, int J, int T_pad, float* maps,
                              unsigned long long* keys, int kb_per_group, int32_t* argmax_out,
                              unsigned int* done_counter, void* stream) {
  REQUIRE(F >= 0 && J >= 0 && P >= 1 && T_pad >= 1, "srpb_interp_tc16_onthefly: bad shape");
  REQUIRE(!argmax_out || (keys && done_counter),
          "srpb_interp_tc16_onthefly: argmax_out needs keys and done_counter");
  REQUIRE(T_pad % 8 == 0, "srpb_interp_tc16_onthefly: T_pad must be a multiple of 8, got %d",
          T_pad);
  REQUIRE(pow2_scale(xi_scale), "srpb_interp_tc16_onthefly: xi_scale must be a power of two");
  REQUIRE(F == 0 || J == 0 || (sx_i && sx_f && off && reach && xi_hi && xi_lo),
          "srpb_interp_tc16_onthefly: null pointer");
  REQUIRE(maps || keys, "srpb_interp_tc16_onthefly: need maps and/or keys output");
  return status(srpb::launch_interp_tc16_onthefly(sx_i, sx_f, P, off, reach, xi_hi, xi_lo,
                                                  xi_scale, F, J, T_pad, maps, keys, kb_per_group,
                                                  argmax_out, done_counter, S(stream)),
                "srpb_interp_tc16_onthefly");
}

int srpb_interp_tc16(const void* w_hi, const void* w_lo, float w_scale, const void* xi_hi,
                     const void* xi_lo, float xi_scale, int F, int J, int T_pad, float* maps,
                     unsigned long long* keys, int kb_per_group, int32_t* argmax_out,
                     unsigned int* done_counter, void* stream) {
  REQUIRE(F >= 0 && J >= 0 && T_pad >= 1, "srpb_interp_tc16: bad shape");
  REQUIRE(!argmax_out || (keys && done_counter),
          "srpb_interp_tc16: argmax_out needs keys and done_counter");
  REQUIRE(T_pad % 8 == 0, "srpb_interp_tc16: T_pad must be a multiple of 8, got %d", T_pad);
  REQUIRE(pow2_scale(w_scale) && pow2_scale(xi_scale),
          "srpb_interp_tc16: scales must be powers of two");
  REQUIRE(F == 0 || J == 0 || (w_hi && w_lo && xi_hi && xi_lo), "srpb_interp_tc16: null pointer");
  REQUIRE(maps || keys, "srpb_interp_tc16: need maps and/or keys output");
  return status(srpb::launch_interp_tc16(w_hi, w_lo, w_scale, xi_hi, xi_lo, xi_scale, F, J, T_pad,
                                         maps, keys, kb_per_group, argmax_out, done_counter,
                                         S(stream)),
                "srpb_interp_tc16");
}

int srpb_interp_tc(const float* w_hi, const float* w_lo, const float* xi_hi, const float* xi_lo,
                   int F, int J, int T_pad, float* maps, unsigned long long* keys,
                   int kb_per_group, void* stream) {
  REQUIRE(F >= 0 && J >= 0 && T_pad >= 32, "srpb_interp_tc: bad shape");
  REQUIRE(T_pad % 32 == 0, "srpb_interp_tc: T_pad must be a multiple of 32, got %d", T_pad);
  REQUIRE(kb_per_group >= 1, "srpb_interp_tc: kb_per_group must be >= 1");
  REQUIRE(F == 0 || J == 0 || (w_hi && w_lo && xi_hi && xi_lo), "srpb_interp_tc: null pointer");
  REQUIRE(maps || keys, "srpb_interp_tc: need maps and/or keys output");
  return status(srpb::launch_interp_tc(w_hi, w_lo, xi_hi, xi_lo, F, J, T_pad, maps, keys,
                                       kb_per_group, S(stream)),
                "srpb_interp_tc");
}

int srpb_argmax(const float* maps, int F, int J, unsigned long long* keys, void* stream) {
  REQUIRE(F >= 0 && J >= 0, "srpb_argmax: bad shape");
  REQUIRE(F == 0 || J == 0 || (maps && keys), "srpb_argmax: null pointer");
  return status(srpb::launch_argmax(maps, F, J, keys, S(stream)), "srpb_argmax");
}

int srpb_argmax_f64(const double* maps, int F, int J, int32_t* idx, void* stream) {
  REQUIRE(F >= 0 && J >= 0, "srpb_argmax_f64: bad shape");
  REQUIRE(F == 0 || J == 0 || (maps && idx), "srpb_argmax_f64: null pointer");
  return status(srpb::launch_argmax_f64(maps, F, J, idx, S(stream)), "srpb_argmax_f64");
}

int srpb_argmax_keys_reset(unsigned long long* keys, int F, void* stream) {
  REQUIRE(F >= 0 && (F == 0 || keys), "srpb_argmax_keys_reset: bad argument");
  return status(srpb::launch_keys_reset(keys, F, S(stream)), "srpb_argmax_keys_reset");
}

int srpb_keys_to_index(const unsigned long long* keys, int F, int32_t* idx, void* stream) {
  REQUIRE(F >= 0 && (F == 0 || (keys && idx)), "srpb_keys_to_index: bad argument");
  return status(srpb::launch_keys_to_index(keys, F, idx, S(stream)), "srpb_keys_to_index");
}

int srpb_copy_rows_h2d(void* dst, size_t dst_pitch, const void* src, size_t src_pitch,
                       size_t row_bytes, int rows, void* stream) {
  REQUIRE(rows >= 0 && row_bytes <= dst_pitch && row_bytes <= src_pitch,
          "srpb_copy_rows_h2d: bad geometry");
  REQUIRE(rows == 0 || row_bytes == 0 || (dst && src), "srpb_copy_rows_h2d: null pointer");
  if (rows == 0 || row_bytes == 0) return 0;
  return status(cudaMemcpy2DAsync(dst, dst_pitch, src, src_pitch, row_bytes,
                                  static_cast<size_t>(rows), cudaMemcpyHostToDevice, S(stream)),
                "srpb_copy_rows_h2d");
}

int srpb_srp_quadform(const float* Psi, int F, int P, int Kb, const double* omega,
                      const double* tau_rel, int J, int M, const int32_t* pair_m,
                      const int32_t* pair_mp, double* maps, void* stream) {
  REQUIRE(F >= 0 && P >= 1 && Kb >= 1 && J >= 0 && M >= 2,
          "srpb_srp_quadform: bad shape F=%d P=%d Kb=%d J=%d M=%d", F, P, Kb, J, M);
  REQUIRE(M <= 64, "srpb_srp_quadform: at most 64 channels supported, got %d", M);
  REQUIRE(P <= 2016, "srpb_srp_quadform: at most 2016 pairs supported, got %d", P);
  REQUIRE(F == 0 || J == 0 || (Psi && omega && tau_rel && pair_m && pair_mp && maps),
          "srpb_srp_quadform: null pointer");
  return status(srpb::launch_quadform(Psi, F, P, Kb, omega, tau_rel, J, M, pair_m, pair_mp, maps,
                                      S(stream)),
                "srpb_srp_quadform");
}

int srpb_map_error(const void* ref, int ref_f64, const void* app, int app_f64, int F, int J,
                   double* scratch, double* num, double* den, void* stream) {
  REQUIRE(F >= 0 && J >= 1, "srpb_map_error: bad shape F=%d J=%d", F, J);
  REQUIRE(F == 0 || (ref && app && scratch && num && den), "srpb_map_error: null pointer");
  return status(srpb::launch_map_error(ref, ref_f64, app, app_f64, F, J, scratch, num, den,
                                       S(stream)),
                "srpb_map_error");
}

}  // extern "C"
