// semd_libm.cuh -- glibc 2.39 log and sincos restated for the device (and the host checker).
//
// The reference's white_noise (emd.cpp:181-200) maps mt19937_64 draws through std::log and
// std::cos / std::sin; g++ -O2 fuses the pair into one glibc sincos call, and on an FMA-capable
// x86-64 host glibc's ifunc dispatch runs the FMA builds of both. Reproducing the reference's
// noise bit-for-bit therefore means evaluating exactly those two algorithms in exactly that
// operation order:
//   log    -- glibc sysdeps/ieee754/dbl-64/e_log.c (the Arm optimized-routines table log):
//             log(x) = k ln2 + log(c) + log1p(z/c - 1), 128 subintervals, degree-5 polynomial;
//             inputs within [1 - 2^-4, 1 + 0x1.09p-4) use a degree-11 polynomial in r = x - 1
//             with a hi/lo split of the quadratic term.
//   sincos -- glibc sysdeps/ieee754/dbl-64/s_sincos.c over s_sin.c's do_sin / do_cos (the IBM
//             Accurate Mathematical Library): |x| < 0.855469 direct; |x| < 2.426265 via
//             hp0 - |x| (106-bit pi/2); larger via reduce_sincos (x n pi/2, 3-part pi/2).
//             Each kernel looks up sin/cos of the nearest k/128 as double-double pairs and
//             corrects with short polynomials; |a| < 0.126 uses a Taylor polynomial instead.
// Every multiply-add below is an explicit single-rounding fma exactly where the FMA build of
// glibc contracts one; everything else is a separately rounded IEEE operation (the engine is
// compiled with -fmad=false, the host checker with -ffp-contract=off). The constants and
// tables are glibc's data, read from the installed libm by gen_libm_tables.py.
// tests/test_libm_restatement.py checks these functions against the system libm bit-for-bit.
#pragma once

#include <stdint.h>

#include <cmath>
#include <cstring>

#include "semd_libm_tables.h"

#ifdef __CUDACC__
#define SEMD_LIBM_HD __host__ __device__ __forceinline__
#else
#define SEMD_LIBM_HD inline
#endif

namespace semd {
namespace libm {

constexpr uint64_t kSign = 0x8000000000000000ULL;

SEMD_LIBM_HD uint64_t as_u64(double v) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(v);
#else
    uint64_t u;
    std::memcpy(&u, &v, 8);
    return u;
#endif
}

SEMD_LIBM_HD double as_f64(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double v;
    std::memcpy(&v, &u, 8);
    return v;
#endif
}

SEMD_LIBM_HD double fma_rn(double a, double b, double c) {
#ifdef __CUDA_ARCH__
    return __fma_rn(a, b, c);
#else
    return std::fma(a, b, c);
#endif
}

SEMD_LIBM_HD double neg(double v) { return as_f64(as_u64(v) ^ kSign); }
SEMD_LIBM_HD double with_sign_of(double v, double s) { return as_f64((as_u64(v) & ~kSign) | (as_u64(s) & kSign)); }

// ---- log (e_log.c), valid for normal x > 0 (the Box-Muller input is in [2^-53, 1]) ------------
// tab: kLogTab ({1/c, log c} pairs), passed so device callers can serve it from shared memory.
SEMD_LIBM_HD double log(double x, const double* tab) {
    const uint64_t ix = as_u64(x);
    if (ix - 0x3fee000000000000ULL <= 0x308ffffffffffULL) {  // 1 - 2^-4 <= x < 1 + 0x1.09p-4
        if (ix == 0x3ff0000000000000ULL) return 0.0;
        const double r = x - 1.0;
        double p2 = fma_rn(r, kLogB2, kLogB1);
        double p5 = fma_rn(r, kLogB5, kLogB4);
        const double r2 = r * r;
        const double p8 = fma_rn(r, kLogB8, kLogB7);
        p2 = fma_rn(r2, kLogB3, p2);
        p5 = fma_rn(r2, kLogB6, p5);
        const double r3 = r * r2;
        double q = fma_rn(r2, kLogB9, p8);
        q = fma_rn(r3, kLogB10, q);
        q = fma_rn(q, r3, p5);
        q = fma_rn(q, r3, p2);
        const double w = fma_rn(r, 0x1p27, r);       // r + r 2^27
        const double rhi = fma_rn(-0x1p27, r, w);     // (r + w) - w: the top 26 bits of r
        const double rhi2 = rhi * rhi;
        const double rlo = r - rhi;
        const double hi = fma_rn(rhi2, kLogB0, r);    // r - rhi^2 / 2
        const double lo0 = fma_rn(rhi2, kLogB0, r - hi);
        const double lo = fma_rn(kLogB0 * rlo, rhi + r, lo0);
        return hi + fma_rn(q, r3, lo);
    }
    const uint64_t tmp = ix - 0x3fe6000000000000ULL;  // subinterval of [0x1.6p-1, 0x1.6p0) and exponent
    const int i = (int)((tmp >> 45) & 0x7f);
    const int k = (int)((int64_t)tmp >> 52);
    const double z = as_f64(ix - (tmp & 0xfff0000000000000ULL));
    const double invc = tab[2 * i], logc = tab[2 * i + 1];
    const double kd = (double)k;
    const double w = fma_rn(kd, kLn2hi, logc);
    const double r = fma_rn(z, invc, -1.0);           // z/c - 1
    const double p21 = fma_rn(r, kLogA2, kLogA1);
    const double hi = r + w;
    const double r2 = r * r;
    double lo = (w - hi) + r;
    lo = fma_rn(kd, kLn2lo, lo);
    const double r3 = r * r2;
    const double p43 = fma_rn(r, kLogA4, kLogA3);
    lo = fma_rn(r2, kLogA0, lo);
    const double p = fma_rn(p43, r2, p21);
    return fma_rn(r3, p, lo) + hi;
}

// ---- sincos (s_sincos.c / s_sin.c) -----------------------------------------------------------
// Table row of |a|: u = big + |a| rounds |a| to the nearest 1/128; xa = |a| - k/128.
struct Row {
    double sn, ssn, cs, ccs, xa;
};

SEMD_LIBM_HD Row row(double abs_a, const double* sct) {
    const double u = kBig + abs_a;
    const int k4 = (int)((uint32_t)as_u64(u) << 2);
    Row t;
    t.xa = abs_a - (u - kBig);
    t.sn = sct[k4];
    t.ssn = sct[k4 + 1];
    t.cs = sct[k4 + 2];
    t.ccs = sct[k4 + 3];
    return t;
}

// TAYLOR_SIN: a + ((P(xx) a - da/2) xx + da)
SEMD_LIBM_HD double taylor_sin(double a, double da) {
    const double xx = a * a;
    double p = fma_rn(xx, kTaylorS5, kTaylorS4);
    p = fma_rn(xx, p, kTaylorS3);
    p = fma_rn(xx, p, kTaylorS2);
    p = fma_rn(xx, p, kTaylorS1);
    const double t1 = fma_rn(p, a, neg(da * 0.5));  // p a - da/2, one rounding
    return a + fma_rn(xx, t1, da);
}

// do_sin past its Taylor branch: dx carries do_sin's sign rule; the result takes sign_src's sign
SEMD_LIBM_HD double do_sin_tab(const Row& t, double dx, double sign_src) {
    const double x = t.xa;
    const double xx = x * x;
    const double p = fma_rn(xx, kSn5, kSn3);
    const double s = fma_rn(x * xx, p, dx) + x;
    const double q = fma_rn(fma_rn(xx, kCs6, kCs4), xx, kCs2);
    const double c = fma_rn(dx, x, xx * q);
    double cor = fma_rn(s, t.ccs, t.ssn);
    cor = fma_rn(neg(c), t.sn, cor);
    cor = fma_rn(s, t.cs, cor);
    return with_sign_of(cor + t.sn, sign_src);
}

// do_cos: x = xa + dx (dx with do_cos's sign rule)
SEMD_LIBM_HD double do_cos_tab(const Row& t, double x) {
    const double xx = x * x;
    const double p = fma_rn(xx, kSn5, kSn3);
    const double s = fma_rn(x * xx, p, x);
    const double q = fma_rn(fma_rn(xx, kCs6, kCs4), xx, kCs2);
    const double c = xx * q;
    double cor = fma_rn(neg(t.ssn), s, t.ccs);
    cor = fma_rn(neg(c), t.cs, cor);
    cor = fma_rn(neg(s), t.sn, cor);
    return t.cs + cor;
}

// sincos for finite |x| < 105414350 (the Box-Muller angle is in (0, 2 pi]); sct: kSinCosTab.
SEMD_LIBM_HD void sincos(double x, const double* sct, double* sinx, double* cosx) {
    const uint32_t k = (uint32_t)(as_u64(x) >> 32) & 0x7fffffffu;
    if (k < 0x3e400000u) {  // |x| < 2^-27
        *sinx = x;
        *cosx = 1.0;
        return;
    }
    if (k < 0x3feb6000u) {  // |x| < 0.855469: do_sin(x, 0), do_cos(x, 0)
        const double ax = with_sign_of(x, 0.0);
        const Row t = row(ax, sct);
        if (kSmall > ax) {
            *sinx = taylor_sin(x, 0.0);
        } else {
            *sinx = do_sin_tab(t, x > 0.0 ? 0.0 : -0.0, x);
        }
        *cosx = do_cos_tab(t, (x >= 0.0 ? 0.0 : -0.0) + t.xa);
        return;
    }
    if (k < 0x400368fdu) {  // |x| < 2.426265: a + da = pi/2 - |x| to 106 bits
        const double y = kHp0 - with_sign_of(x, 0.0);
        const double a = y + kHp1;
        const double da = (y - a) + kHp1;
        const double aa = with_sign_of(a, 0.0);
        const Row t = row(aa, sct);
        // sin x = copysign(do_cos(a, da), x)
        *sinx = with_sign_of(do_cos_tab(t, t.xa + (0.0 > a ? neg(da) : da)), x);
        // cos x = do_sin(a, da)
        if (kSmall > aa) *cosx = taylor_sin(a, da);
        else *cosx = do_sin_tab(t, a <= 0.0 ? neg(da) : da, a);
        return;
    }
    // reduce_sincos: x = n pi/2 + (a + da)
    const double tq = fma_rn(x, kHpInv, kToInt);
    const double xn = tq - kToInt;
    const int n = (int)(as_u64(tq) & 3);
    double y = fma_rn(neg(xn), kMp1, x);
    y = fma_rn(neg(xn), kMp2, y);
    const double t2 = fma_rn(neg(xn), kPp3, y);
    double db = fma_rn(neg(xn), kPp3, y - t2);
    double a = fma_rn(neg(xn), kPp4, t2);
    db = db + fma_rn(neg(xn), kPp4, t2 - a);
    if (n == 1 || n == 2) {
        a = neg(a);
        db = neg(db);
    }
    const double aa = with_sign_of(a, 0.0);
    const Row t = row(aa, sct);
    const double s1 = kSmall > aa ? taylor_sin(a, db) : do_sin_tab(t, a > 0.0 ? db : neg(db), a);
    double c1 = do_cos_tab(t, (a < 0.0 ? neg(db) : db) + t.xa);
    if (n & 2) c1 = neg(c1);
    if (n & 1) {
        *cosx = s1;
        *sinx = c1;
    } else {
        *sinx = s1;
        *cosx = c1;
    }
}

}  // namespace libm
}  // namespace semd
