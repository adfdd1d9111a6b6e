// Common device helpers for the SubApSnap online-phase kernels (sm_100a).
//
// * cplx: complex128 with the exact operation order numpy uses for complex128
//   (a+bi)(c+di) = (ac - bd) + (ad + bc)i, evaluated without FMA contraction
//   where bitwise agreement with the reference's affine combine matters
//   (online.py:108-112).
// * Scalar traits so the least-squares kernel is one template for f64 and c128.
// * 2048-entry-table FP64 exponentials for the kernel-row contraction (K3) and
//   the stencil residual checker (K6): 5-9 FP64-pipe ops instead of the
//   ~24-DFMA-equivalent libdevice exp (measured on B200,
//   profiles/r01_fp64_peaks.jsonl).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define SAS_HD __host__ __device__ __forceinline__

struct cplx {
  double re, im;
};

SAS_HD cplx mk(double re, double im) { return cplx{re, im}; }

// ---- exact (no-FMA) complex ops, matching numpy complex128 ufuncs ----------
SAS_HD cplx cmul_exact(cplx a, cplx b) {
#ifdef __CUDA_ARCH__
  return cplx{__dsub_rn(__dmul_rn(a.re, b.re), __dmul_rn(a.im, b.im)),
              __dadd_rn(__dmul_rn(a.re, b.im), __dmul_rn(a.im, b.re))};
#else
  volatile double t0 = a.re * b.re, t1 = a.im * b.im, t2 = a.re * b.im, t3 = a.im * b.re;
  return cplx{t0 - t1, t2 + t3};
#endif
}
SAS_HD cplx cadd_exact(cplx a, cplx b) {
#ifdef __CUDA_ARCH__
  return cplx{__dadd_rn(a.re, b.re), __dadd_rn(a.im, b.im)};
#else
  return cplx{a.re + b.re, a.im + b.im};
#endif
}
SAS_HD double dmul_exact(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  volatile double t = a * b;
  return t;
#endif
}
SAS_HD double dadd_exact(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  volatile double t = a + b;
  return t;
#endif
}
SAS_HD double dsub_exact(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  volatile double t = a - b;
  return t;
#endif
}

// ---- scalar traits ----------------------------------------------------------
template <typename T>
struct Sc;

template <>
struct Sc<double> {
  static SAS_HD double zero() { return 0.0; }
  static SAS_HD double from(double re, double) { return re; }
  static SAS_HD double conj(double a) { return a; }
  static SAS_HD double abs2(double a) { return a * a; }
  static SAS_HD double abs(double a) { return fabs(a); }
  static SAS_HD double re(double a) { return a; }
  static SAS_HD double im(double) { return 0.0; }
  // acc + conj(a) * b
  static SAS_HD double fma_conj(double a, double b, double acc) { return fma(a, b, acc); }
  // acc - a * b
  static SAS_HD double fms(double a, double b, double acc) { return fma(-a, b, acc); }
  static SAS_HD double mul(double a, double b) { return a * b; }
  static SAS_HD double mulr(double a, double b) { return a * b; }  // scalar * real
  static SAS_HD double add(double a, double b) { return a + b; }
  static SAS_HD double sub(double a, double b) { return a - b; }
  static SAS_HD double div(double a, double b) { return a / b; }
  static SAS_HD bool finite(double a) { return isfinite(a); }
  static SAS_HD double mul_exact(double a, double b) { return dmul_exact(a, b); }
  static SAS_HD double add_exact(double a, double b) { return dadd_exact(a, b); }
};

template <>
struct Sc<cplx> {
  static SAS_HD cplx zero() { return cplx{0.0, 0.0}; }
  static SAS_HD cplx from(double re, double im) { return cplx{re, im}; }
  static SAS_HD cplx conj(cplx a) { return cplx{a.re, -a.im}; }
  static SAS_HD double abs2(cplx a) { return a.re * a.re + a.im * a.im; }
  static SAS_HD double abs(cplx a) { return hypot(a.re, a.im); }
  static SAS_HD double re(cplx a) { return a.re; }
  static SAS_HD double im(cplx a) { return a.im; }
  static SAS_HD cplx fma_conj(cplx a, cplx b, cplx acc) {
    // conj(a) * b = (ar br + ai bi) + i (ar bi - ai br)
    acc.re = fma(a.re, b.re, acc.re);
    acc.re = fma(a.im, b.im, acc.re);
    acc.im = fma(a.re, b.im, acc.im);
    acc.im = fma(-a.im, b.re, acc.im);
    return acc;
  }
  static SAS_HD cplx fms(cplx a, cplx b, cplx acc) {
    acc.re = fma(-a.re, b.re, acc.re);
    acc.re = fma(a.im, b.im, acc.re);
    acc.im = fma(-a.re, b.im, acc.im);
    acc.im = fma(-a.im, b.re, acc.im);
    return acc;
  }
  static SAS_HD cplx mul(cplx a, cplx b) {
    return cplx{fma(a.re, b.re, -a.im * b.im), fma(a.re, b.im, a.im * b.re)};
  }
  static SAS_HD cplx mulr(cplx a, double b) { return cplx{a.re * b, a.im * b}; }
  static SAS_HD cplx add(cplx a, cplx b) { return cplx{a.re + b.re, a.im + b.im}; }
  static SAS_HD cplx sub(cplx a, cplx b) { return cplx{a.re - b.re, a.im - b.im}; }
  static SAS_HD cplx div(cplx a, cplx b) {
    // Smith's algorithm (robust against overflow)
    if (fabs(b.re) >= fabs(b.im)) {
      double rt = b.im / b.re, den = b.re + b.im * rt;
      return cplx{(a.re + a.im * rt) / den, (a.im - a.re * rt) / den};
    } else {
      double rt = b.re / b.im, den = b.re * rt + b.im;
      return cplx{(a.re * rt + a.im) / den, (a.im * rt - a.re) / den};
    }
  }
  static SAS_HD bool finite(cplx a) { return isfinite(a.re) && isfinite(a.im); }
  static SAS_HD cplx mul_exact(cplx a, cplx b) { return cmul_exact(a, b); }
  static SAS_HD cplx add_exact(cplx a, cplx b) { return cadd_exact(a, b); }
};

// ---- fast FP64 exp ----------------------------------------------------------
#define SAS_EXP_MAGIC 0x1.8p52

// 2^(j/2048), j = 0..2047 (correctly rounded), copied to shared memory by K3/K6.
__device__ const double g_exp2_tab2048[2048] = {
#include "exp2_table2048.inc"
};

// General form (K6 stencil checker): 2048-entry table in shared memory, degree-3 polynomial.
//   k = rint(x 2048/ln2), r = x - k ln2/2048 (two-constant, |r| <= ln2/4096),
//   e^r - 1 = r (1 + r/2 + r^2/6) (truncation r^4/24 <= 3.4e-17),
//   e^x = 2^(k mod 2048 / 2048) (1 + q) 2^(k div 2048).
// 9 FP64-pipe ops per value.  k < -2093055
// (x < -708.39) flushes to +0.
#define SAS_INVLN2X2K 0x1.71547652b82fep+11
#define SAS_LN2D2K_HI 0x1.62e42fec00000p-12
#define SAS_LN2D2K_LO 0x1.d1cf79abc9e3bp-43
#define SAS_EXP2K_KMIN (-2093055)

__device__ __forceinline__ double sas_exp64_t2k(double x, const double* __restrict__ tab_s) {
  const double kd = fma(x, SAS_INVLN2X2K, SAS_EXP_MAGIC);
  const int ki = __double2loint(kd);
  const double kf = kd - SAS_EXP_MAGIC;
  double r = fma(-kf, SAS_LN2D2K_HI, x);
  r = fma(-kf, SAS_LN2D2K_LO, r);
  double q = fma(r, 1.0 / 6.0, 0.5);
  q = fma(q, r, 1.0);
  q = q * r;
  const double t = tab_s[ki & 2047];
  const double res = fma(t, q, t);
  const int hi = __double2hiint(res) + ((ki >> 11) << 20);
  const int keep = (ki >= SAS_EXP2K_KMIN) ? -1 : 0;
  return __hiloint2double(hi & keep, __double2loint(res) & keep);
}

#define SAS_EXP2K_A1 0x1.62e42fefa39efp-12
#define SAS_EXP2K_A2 0x1.ebfbdff82c58fp-25
#define SAS_EXP2K_A3 0x1.c6b08d704a0c0p-38

// K3 exponentials in "table units": e^(a*b) for a = D' >= 0 (kernel-row
// distance pre-scaled by 2048/ln2 at plan time) and b = -1/(2 p^2) < 0, with
// bf = (float)b.  tabn holds the table NEGATED (-2^(j/2048)): the final
// fma then yields -t(1+q) and the sign is cleared by the same integer add
// that applies 2^(k div 2048) (see below), saving an instruction per value.
//
// sas_exp64_t2k_fr: k = rint(a*b) from an FP32 product of truncated copies
// (integer bit ops give float(a)); |k - a*b| <= 1/2 + 2^-22 |a*b|, so with the
// clamp below (|k| < 2^22) the reduced argument r = a*b + |k| (one FMA on the
// exact product, |k| rebuilt as an exact double from the float's bits) has
// |r| <= 0.52, where the degree-3 polynomial's truncation is 4e-17.
// 2^(r/2048) - 1 = r (a1 + r (a2 + r a3)), a_i = (ln2/2048)^i / i!.  5 FP64-pipe
// ops.  k = 0 yields |k| = 2^-127 instead of 0, which perturbs r by 2^-127
// (below half an ulp of any nonzero r) and leaves a = 0 exactly the selected
// table value.  k < -2093055 (x < -708.39) flushes to +0.  ridx >= 0 selects
// tabn[ridx] instead of the table (the kernel-row ridge on the diagonal).
__device__ __forceinline__ double sas_exp64_t2k_fr(double a, double b, float bf, const double* __restrict__ tabn,
                                                   int ridx) {
  const int ah = max(__double2hiint(a), 0x38000000);
  const float af = __int_as_float((ah - 0x38000000) << 3);  // float(a) truncated; a < 2^-126 -> 0
  const float pf = fmaxf(af * bf, -3.0e6f);                  // below KMIN: flushed to 0 at the end
  const float kd32 = pf + 0x1.8p23f;
  const int ki = __float_as_int(kd32) - 0x4B400000;          // k = rint(pf)
  const int kb = __float_as_int(0x1.8p23f - kd32);           // bits of float(|k|), exact
  const double kabs = __hiloint2double((kb >> 3) + 0x38000000, kb << 29);
  const double r = fma(a, b, kabs);
  double q = fma(r, SAS_EXP2K_A3, SAS_EXP2K_A2);
  q = fma(q, r, SAS_EXP2K_A1);
  q = q * r;
  const double tv = tabn[ridx >= 0 ? ridx : (ki & 2047)];
  const double res = fma(tv, q, tv);  // -t (1 + q)
  const int hi = (__double2hiint(res) + ((ki >> 11) << 20)) ^ (int)0x80000000;
  const int keep = (ki >= SAS_EXP2K_KMIN) ? -1 : 0;
  return __hiloint2double(hi & keep, __double2loint(res) & keep);
}

// sas_exp64_t2k_fast: the same arithmetic for a CTA whose arguments all satisfy
// |a b| < 2.0e6 (x > -677: nothing underflows, no clamp or flush; the caller
// checks the bound per CTA), with fewer integer instructions: k from one FFMA
// on the magic constant (exactly rint of the FP32 product), the table index
// straight from the float's low bits (the magic constant is a multiple of
// 2048), and sign + 2^(k div 2048) in one add: the float bits kdb = 0x4B400000
// + k give (kdb >> 11) << 20 = 0x80000000 + (k div 2048) << 20 (mod 2^32), and
// the 0x80000000 clears the sign of -t(1+q).  a = 0 gives exactly 1.0.  No
// ridge select: K3 adds lam X[S_i] after the contraction.
__device__ __forceinline__ double sas_exp64_t2k_fast(double a, double b, float bf, const double* __restrict__ tabn) {
  const int ah = max(__double2hiint(a), 0x38000000);
  const float af = __int_as_float(ah * 8 + 0x40000000);   // (ah - 0x38000000) << 3 mod 2^32: float(a) truncated
  const float kd32 = fmaf(af, bf, 0x1.8p23f);            // 1.5 2^23 + k, k = rint(af bf) <= 0
  const int kdb = __float_as_int(kd32);
  const int kb = __float_as_int(0x1.8p23f - kd32);        // bits of float(|k|), exact
  const double kabs = __hiloint2double((kb >> 3) + 0x38000000, kb << 29);
  const double r = fma(a, b, kabs);
  double q = fma(r, SAS_EXP2K_A3, SAS_EXP2K_A2);
  q = fma(q, r, SAS_EXP2K_A1);
  q = q * r;
  const double tv = tabn[kdb & 2047];
  const double res = fma(tv, q, tv);  // -t (1 + q)
  const int hi = __double2hiint(res) + ((kdb >> 11) << 20);
  return __hiloint2double(hi, __double2loint(res));
}
#define SAS_EXP2K_FAST_MAX 2.0e6

// Host reference of the same algorithm (for the CPU accuracy test).
double sas_exp64_host(double x);

#define SAS_CUDA_CHECK(expr)                                                   \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      sas_set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e),        \
                    __FILE__, __LINE__, cudaGetErrorString(_e));               \
      return SAS_ERR_CUDA;                                                     \
    }                                                                          \
  } while (0)

void sas_set_error(const char* fmt, ...);
