// glibc's log1p restated for the device (and host, for the CPU test).
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define NENMF_HD __host__ __device__
#else
#define NENMF_HD
#endif

#ifdef __CUDA_ARCH__
#define L1P_FMA(a, b, c) __fma_rn(a, b, c)
#define L1P_MUL(a, b) __dmul_rn(a, b)
#define L1P_ADD(a, b) __dadd_rn(a, b)
#define L1P_SUB(a, b) __dsub_rn(a, b)
#define L1P_DIV(a, b) __ddiv_rn(a, b)
NENMF_HD inline int l1p_hi(double x) { return __double2hiint(x); }
NENMF_HD inline int l1p_lo(double x) { return __double2loint(x); }
NENMF_HD inline double l1p_make(int hi, int lo) { return __hiloint2double(hi, lo); }
#else  // host: plain IEEE operations; build with -ffp-contract=off
#define L1P_FMA(a, b, c) fma(a, b, c)
#define L1P_MUL(a, b) ((a) * (b))
#define L1P_ADD(a, b) ((a) + (b))
#define L1P_SUB(a, b) ((a) - (b))
#define L1P_DIV(a, b) ((a) / (b))
inline int l1p_hi(double x) {
  uint64_t b;
  memcpy(&b, &x, 8);
  return (int)(uint32_t)(b >> 32);
}
inline int l1p_lo(double x) {
  uint64_t b;
  memcpy(&b, &x, 8);
  return (int)(uint32_t)b;
}
inline double l1p_make(int hi, int lo) {
  const uint64_t b = ((uint64_t)(uint32_t)hi << 32) | (uint32_t)lo;
  double x;
  memcpy(&x, &b, 8);
  return x;
}
#endif

// log1p exactly as the C library NumPy links against computes it (glibc
// 2.39, x86-64, the FMA variant its ifunc selects on the hosts of this pool):
// the classic argument reduction 1 + x = 2^k (1 + f), s = f / (2 + f), and
// the degree-7 polynomial in z = s^2 evaluated in Estrin form with the
// contractions that build performs.  Every operation is spelled with an
// explicit rounding intrinsic so nvcc cannot re-associate or fuse anything
// else.  Checked against the host libm on 4.1e8 arguments in (-1, 0]
// (tests/test_log1p_restatement.py compiles this header on the host and
// compares it with libm).
NENMF_HD inline double glibc_log1p(double x) {
  constexpr double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  constexpr double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
                   Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
                   Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
                   Lp7 = 1.479819860511658591e-01;
  const int hx = l1p_hi(x), ax = hx & 0x7fffffff;
  int k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -HUGE_VAL : NAN;
    if (ax < 0x3e200000) {
      if (ax < 0x3c900000) return x;
      return L1P_FMA(-L1P_MUL(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= (int)0xbfd2bec3) {
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return L1P_ADD(x, x);
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = L1P_ADD(1.0, x);
      hu = l1p_hi(u);
      k = (hu >> 20) - 1023;
      c = k > 0 ? L1P_SUB(1.0, L1P_SUB(u, x)) : L1P_SUB(x, L1P_SUB(u, 1.0));
      c = L1P_DIV(c, u);
    } else {
      u = x;
      hu = l1p_hi(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = l1p_make(hu | 0x3ff00000, l1p_lo(u));
    } else {
      ++k;
      u = l1p_make(hu | 0x3fe00000, l1p_lo(u));
      hu = (0x00100000 - hu) >> 2;
    }
    f = L1P_SUB(u, 1.0);
  }
  const double dk = (double)k;
  const double hfsq = L1P_MUL(L1P_MUL(0.5, f), f);
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = L1P_FMA(dk, ln2_lo, c);
      return L1P_FMA(dk, ln2_hi, c);
    }
    const double R = L1P_MUL(hfsq, L1P_FMA(-0.66666666666666666, f, 1.0));
    if (k == 0) return L1P_SUB(f, R);
    return L1P_FMA(dk, ln2_hi, -L1P_SUB(L1P_SUB(R, L1P_FMA(dk, ln2_lo, c)), f));
  }
  const double s = L1P_DIV(f, L1P_ADD(2.0, f));
  const double z = L1P_MUL(s, s);
  const double z2 = L1P_MUL(z, z), z4 = L1P_MUL(z2, z2), z6 = L1P_MUL(z4, z2);
  const double R2 = L1P_FMA(z, Lp3, Lp2), R3 = L1P_FMA(z, Lp5, Lp4), R4 = L1P_FMA(z, Lp7, Lp6);
  const double R = L1P_FMA(z6, R4, L1P_FMA(z4, R3, L1P_FMA(z, Lp1, L1P_MUL(z2, R2))));
  const double sp = L1P_MUL(s, L1P_ADD(hfsq, R));
  if (k == 0) return L1P_SUB(f, L1P_SUB(hfsq, sp));
  return L1P_FMA(dk, ln2_hi, -L1P_SUB(L1P_SUB(hfsq, L1P_ADD(L1P_FMA(dk, ln2_lo, c), sp)), f));
}
