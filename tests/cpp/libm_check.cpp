// Checks the restatement of glibc's log and sincos (paper_2106_15319_b200/csrc/semd_libm.cuh)
// against the system libm, bit for bit, on the inputs the reference's white_noise feeds them
// (emd.cpp:189-198): u = ((draw >> 11) + 1) 2^-53 in (0, 1] for log, theta = 2 pi u for sincos.
//   libm_check <random pairs> <seed>   -> prints "mismatches <log> <sin> <cos> of <n>"; exit 1 on any
#define _GNU_SOURCE 1
#include <math.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "semd_libm.cuh"

static long nlog = 0, nsin = 0, ncos = 0, total = 0;

static bool same(double a, double b) { return std::memcmp(&a, &b, 8) == 0; }

static void check_log(double u) {
    volatile double v = u;
    const double ref = ::log(v);
    const double got = semd::libm::log(u, semd::libm::kLogTab);
    if (!same(ref, got)) {
        if (nlog < 5) std::printf("log(%a): libm %a restated %a\n", u, ref, got);
        ++nlog;
    }
}

static void check_sincos(double th) {
    volatile double v = th;
    double rs, rc, s, c;
    ::sincos(v, &rs, &rc);
    semd::libm::sincos(th, semd::libm::kSinCosTab, &s, &c);
    if (!same(rs, s)) {
        if (nsin < 5) std::printf("sin(%a): libm %a restated %a\n", th, rs, s);
        ++nsin;
    }
    if (!same(rc, c)) {
        if (ncos < 5) std::printf("cos(%a): libm %a restated %a\n", th, rc, c);
        ++ncos;
    }
}

int main(int argc, char** argv) {
    const long n = argc > 1 ? std::atol(argv[1]) : 1000000;
    const uint64_t seed = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1;
    const double two_pi = 6.283185307179586476925286766559;
    std::mt19937_64 eng(seed);
    auto unit = [&eng]() { return static_cast<double>((eng() >> 11) + 1) * 0x1.0p-53; };
    for (long i = 0; i < n; ++i) {  // the white_noise draw pattern
        check_log(unit());
        check_sincos(two_pi * unit());
        total += 1;
    }
    // edges of the log paths: near 1, the near-one window [1 - 2^-4, 1 + 0x1.09p-4), the smallest u
    for (long j = 1; j <= 200000; ++j) {
        check_log(1.0 - j * 0x1.0p-53);
        check_log(0.9375 + (j - 100000) * 0x1.0p-53);
        check_log(j * 0x1.0p-53);
        check_log(0.5 + (j - 100000) * 0x1.0p-53);
    }
    check_log(1.0);
    // edges of the sincos paths over theta = 2 pi u, u = j 2^-53
    const double edges[] = {0x1.0p-27, 0.126, 0.855469, 1.5707963267948966, 2.426265, 3.141592653589793,
                            4.71238898038469, 6.283185307179586, 0.78539816339744828, 2.356194490192345,
                            3.9269908169872414, 5.497787143782138};
    for (double e : edges)
        for (long j = -100000; j <= 100000; ++j) {
            const double u = std::nearbyint(e / two_pi * 0x1.0p53 + j) * 0x1.0p-53;
            if (u > 0.0 && u <= 1.0) check_sincos(two_pi * u);
        }
    for (long j = 1; j <= 200000; ++j) check_sincos(two_pi * (j * 0x1.0p-53));
    // every 1/128 table cell of |a| in [0, 0.86), through all three sincos paths
    for (int k = 0; k < 110; ++k)
        for (int q = -300; q <= 300; ++q) {
            const double a = k / 128.0 + q * 0x1.0p-17;
            if (a <= 0) continue;
            check_sincos(a);
            check_sincos(1.5707963267948966 - a);
            check_sincos(3.141592653589793 + a);
            check_sincos(4.71238898038469 - a);
            check_sincos(6.283185307179586 - a);
        }
    std::printf("mismatches %ld %ld %ld of %ld random pairs + edge sweeps\n", nlog, nsin, ncos, total);
    return (nlog || nsin || ncos) ? 1 : 0;
}
