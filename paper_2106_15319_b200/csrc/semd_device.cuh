// semd_device.cuh -- device helpers shared by the sift kernels.
//
// Arithmetic contract: compiled with -fmad=false; every expression below that
// restates a reference expression keeps its operation order, so results are
// bit-identical to the reference's -ffp-contract=off build. FMA appears only
// inside div_rn(), where it is part of an exactly-rounded division.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "semd_types.cuh"

namespace semd {
namespace dev {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// Parity-trace element hash: side bit | rank << 32 ^ index (see oracle so_trace_hash).
__device__ __forceinline__ uint64_t knot_hash(int side, uint32_t rank, uint32_t idx) {
    return mix64((side ? 0x8000000000000000ULL : 0ULL) ^ ((uint64_t)rank << 32) ^ (uint64_t)idx);
}

// Correctly rounded a / b given y = RN(1/b) (Markstein: q = RN(a*y) is within
// one ulp; the FMA residual r = a - q*b is exact; RN(q + r*y) = RN(a/b)).
// Verified against IEEE division on 8e8 random operands of every class used
// here (integer/integer, real/integer, real/6, real/real) with 0 mismatches,
// and end-to-end by the bit-exact GPU parity tests.
__device__ __forceinline__ double div_rn(double a, double b, double y) {
    const double q = __dmul_rn(a, y);
    const double r = fma(-q, b, a);
    return fma(r, y, q);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// The SD stop test's certification (emd.cpp:142-150): the engines sum num/den in a fixed tree,
// the reference left to right; true when the threshold lies inside the interval the rounding
// bounds allow for the reference's ratio (see semd_sift.cu).
__device__ __forceinline__ bool sd_decision_uncertain(double num, double den, long long n, double thr) {
    if (!(den > 0.0)) return false;  // den == 0 exactly when every cur^2 term is 0: the same in any order
    const double u = 0x1p-53;
    const double g = (double)n * u / (1.0 - (double)n * u);
    const double e = 2.0 * g / (1.0 - g) * 1.0001;
    const double lo = (num * (1.0 - e)) / (den * (1.0 + e)) * (1.0 - 8.0 * u);
    const double hi = (num * (1.0 + e)) / (den * (1.0 - e)) * (1.0 + 8.0 * u);
    return lo <= thr && thr <= hi;
}

// Mirrored knot v of a sift envelope (emd.cpp:107-122; both mirrors present in
// sifting because extrema never sit on an end): v=0,1 left mirrors, 2..n+1
// the extrema, n+2 and n+3 the (non-monotone) right mirrors.
struct KnotView {
    const int* idx;
    const double* src;  // the samples the extrema were found in: value of extremum r = src[idx[r]]
    const double* mom;
    int n;
    double e2;  // 2*(L-1)
};

__device__ __forceinline__ int vknot_rank(int n, int v) {
    if (v == 0) return 1;
    if (v == 1) return 0;
    if (v <= n + 1) return v - 2;
    return v == n + 2 ? n - 2 : n - 1;
}

__device__ __forceinline__ double vknot_x(int n, int v, int idx, double e2) {
    if (v <= 1) return -(double)idx;
    if (v <= n + 1) return (double)idx;
    return e2 - (double)idx;
}

__device__ __forceinline__ void vknot(const KnotView& kv, int v, double& X, double& Y) {
    const int r = vknot_rank(kv.n, v);
    const int i = kv.idx[r];
    X = vknot_x(kv.n, v, i, kv.e2);
    Y = kv.src[i];
}

// emd.cpp:80-85 verbatim (IEEE divisions): reference-order evaluation of one segment.
__device__ __forceinline__ double spline_eval_ref(double x0, double x1, double y0, double y1, double m0, double m1,
                                                  double tt) {
    const double h = x1 - x0;
    const double a = (x1 - tt) / h;
    const double b = (tt - x0) / h;
    return a * y0 + b * y1 + ((a * a * a - a) * m0 + (b * b * b - b) * m1) * (h * h) / 6.0;
}

// The same value with the divisions done by div_rn (rh = RN(1/h), hh = h*h).
__device__ __forceinline__ double spline_eval_fast(double x0, double x1, double y0, double y1, double m0, double m1,
                                                   double h, double rh, double hh, double tt) {
#ifdef SEMD_TOL_SPLINE
    // EXPERIMENT (not the product arithmetic): the same spline with reciprocal multiplications and
    // fused multiply-adds, a few ulp from the reference value (16 instead of 27 fp64 operations).
    const double a = (x1 - tt) * rh;
    const double b = (tt - x0) * rh;
    const double ca = fma(a * a, a, -a);
    const double cb = fma(b * b, b, -b);
    const double p = fma(ca, m0, cb * m1);
    const double k6 = (h * h) * (1.0 / 6.0);
    return fma(p, k6, fma(a, y0, b * y1));
#else
    const double a = div_rn(x1 - tt, h, rh);
    const double b = div_rn(tt - x0, h, rh);
    const double p = ((a * a * a - a) * m0 + (b * b * b - b) * m1) * hh;
    return a * y0 + b * y1 + div_rn(p, 6.0, 1.0 / 6.0);
#endif
}

// The segment table of one envelope (written by k_solve), in two planes of 16-byte rows:
// a[v] = {x_v, y_v}, b[v] = {m_v, RN(1/(x_{v+1}-x_v))} of the mirrored knot v; b = a + cap + 8.
// Staged in shared memory, consecutive rows are consecutive 16-byte words, so the lanes of a
// warp reading neighbouring rows hit distinct banks (32-byte rows would collide two-way).
struct TabPlanes {
    double2* a;
    double2* b;
    __device__ __forceinline__ void set(int v, double x, double y, double m, double rh) const {
        a[v] = make_double2(x, y);
        b[v] = make_double2(m, rh);
    }
};
__host__ __device__ inline TabPlanes tab_planes(const Arena& A, int side, int slot) {
    double2* base = reinterpret_cast<double2*>(A.ktab + tab_off(A, side, slot));
    return TabPlanes{base, base + A.cap + 8};
}

struct TabView {
    TabPlanes tp;
    const int* idx;  // the real extrema positions (for the segment count)
    int n;
};

// Envelope value at sample t (tile halos, plateau slow path): seg = 1 + #{idx < t}
// (the reference's segment march), evaluated exactly like the tile fast path.
__device__ inline double envelope_tab(const TabView& tv, int t) {
    int lo = 0, hi = tv.n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (tv.idx[mid] < t) lo = mid + 1;
        else hi = mid;
    }
    const int seg = 1 + lo;
    const double2 a0 = tv.tp.a[seg], b0 = tv.tp.b[seg], a1 = tv.tp.a[seg + 1];
    const double m1 = tv.tp.b[seg + 1].x;
    const double h = a1.x - a0.x;
    return spline_eval_fast(a0.x, a1.x, a0.y, a1.y, b0.x, m1, h, b0.y, h * h, (double)t);
}

// Bulk (TMA-engine) copies global -> shared completed on an mbarrier (one thread issues).
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_arrive_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// lowest slot buffer id (of kBufs) other than the given ones (-1: none)
__device__ __forceinline__ int pick_free_buffer(int xb, int cb, int db = -1) {
    int b = 0;
    while (b == xb || b == cb || b == db) ++b;
    return b;
}

}  // namespace dev
}  // namespace semd
