// Host build of coot_crmath.cuh for development checks (tools/crmath_check.py):
// the same source the device compiles, run on x86-64 with -ffp-contract=off.
#include "../paper_2508_11385_b200/csrc/coot_crmath.cuh"
using namespace coot::crm;
extern "C" {
void crm_exp(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = cr_exp(x[i]); }
void crm_log(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = cr_log(x[i]); }
void crm_expf(const float* x, float* y, long n) { for (long i = 0; i < n; ++i) y[i] = cr_expf(x[i]); }
void crm_logf(const float* x, float* y, long n) { for (long i = 0; i < n; ++i) y[i] = cr_logf(x[i]); }
// fast phase vs accurate phase: relative difference (hi+lo) and whether decided
void crm_exp_phases(const double* x, double* rel, int* decided, long n) {
  for (long i = 0; i < n; ++i) {
    int m1, m2;
    dd a = exp_fast(x[i], &m1), b = exp_accurate(x[i], &m2);
    rel[i] = ((a.hi - b.hi) + (a.lo - b.lo)) / b.hi;
    decided[i] = f64_decided(a, kRoundC64);
  }
}
void crm_log_phases(const double* x, double* rel, int* decided, long n) {
  for (long i = 0; i < n; ++i) {
    dd a = log_fast(x[i]), b = log_accurate(x[i]);
    rel[i] = b.hi == 0 ? 0 : ((a.hi - b.hi) + (a.lo - b.lo)) / b.hi;
    decided[i] = f64_decided(a, kRoundC64);
  }
}
}
extern "C" {
void crm_exp_batched(const double* x, double* y, long n) {
  for (long i = 0; i < n; ++i) { bool ok; double v = exp_fast_ok(x[i], ok); y[i] = ok ? v : cr_exp_slow(x[i]); }
}
void crm_log_batched(const double* x, double* y, long n) {
  for (long i = 0; i < n; ++i) { bool ok; double v = log_fast_ok(x[i], ok); y[i] = ok ? v : cr_log_slow(x[i]); }
}
}
extern "C" {
// the device's vectorised f32 path (coot_device.cuh un_vec): fast value when
// in range and clear of a midpoint, else the scalar correctly rounded function
void crm_expf_vec(const float* x, float* y, long n) {
  for (long i = 0; i < n; ++i) {
    const double v = exp_f64_of_f32_core((double)x[i]);
    y[i] = (expf_fast_range(x[i]) && f32_mid_clear(v, kF32Margin)) ? (float)v : cr_expf(x[i]);
  }
}
void crm_logf_vec(const float* x, float* y, long n) {
  for (long i = 0; i < n; ++i) {
    const double v = logf_fast_core(x[i]);
    y[i] = (logf_fast_range(x[i]) && f32_mid_clear(v, kF32Margin)) ? (float)v : cr_logf(x[i]);
  }
}
}
