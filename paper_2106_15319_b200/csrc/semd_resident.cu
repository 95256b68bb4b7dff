// semd_resident.cu -- the resident sift engine for short signals (C1-C3 sizes).
//
// north_star: "One persistent CTA per signal or realization keeps the serialized signal resident
// in shared memory." One CTA of kResThreads threads (one per SM: the candidate and both envelopes'
// segment tables fill the SM's shared memory) takes whole jobs from a queue -- a plain EMD, an
// EEMD realization x + beta*w_m, a CEEMDAN noise-mode or first-mode task -- and runs the IMF loop
// of emd() (emd.cpp:155-172) around extract_imf() (:127-153) to the end without leaving the SM.
// Per sift, block-cooperative passes over the shared-memory candidate:
//   detect   find_extrema (emd.cpp:10-35): per 4-sample group flags, ballot-free block scan of
//            the per-group counts -> ordered extrema ranks (no knot lists are materialised: a
//            group's knots are rows 2 + prefix + j)
//   tables   the mirrored knot system of envelope() (:91-125) for both sides, rows {x, y}
//   solve    the natural-spline moments (:53-73), bit-exact: speculative chains (one thread per
//            chain, both sides at once) verified at every chain boundary; any mismatch re-solves
//            that side sequentially (the reference's own loop)
//   eval     the envelopes at every sample (:75-86) from the group prefix (no search), the mean
//            subtraction and the SD partials (:142-148) -- in place
//   SD test  fixed-tree sums, certified against the reference's left-to-right order (the
//            lockstep engine's bound); uncertified decisions redo the sums in the reference order
// The IMF, the residue update (:167) and the optional per-task outputs go to HBM once per IMF.
// Ensemble sums are formed afterwards by k_res_accum in job (= realization) order, so results
// are bit-identical to the lockstep engine and the reference.
//
// Arithmetic contract as in semd_device.cuh (-fmad=false, reference operation order).
#include <cuda_runtime.h>

#include <cstdint>

#include "semd_device.cuh"
#include "semd_launch.h"
#include "semd_types.cuh"

namespace semd {
namespace dev {

constexpr int kResWarps = kResThreads / 32;
constexpr int kResChains = kResThreads / 2;  // chains per side (both sides solve concurrently)
constexpr int kResWarm = 40;                 // speculative warm-up rows of a chain (forward and back)
constexpr int kResChainMin = 8;              // rows per chain at least (R <= 8 * kResChains uses more chains' worth)

struct ResShared {
    double red[2][kResWarps];
    int scan[kResWarps];
    unsigned long long hred[kResWarps];
    int job;
    int bad;  // bit s: side s's speculative solve disagreed at a chain boundary
    int unc;
};

__device__ __forceinline__ bool same_bits(double a, double b) {
    return __double_as_longlong(a) == __double_as_longlong(b);
}

// Exclusive block scan of one int per thread; *tot = block total. Three barriers.
__device__ __forceinline__ int res_excl_scan(int v, int* tot, ResShared& sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) sh.scan[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int x = lane < kResWarps ? sh.scan[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane < kResWarps) sh.scan[lane] = x;
    }
    __syncthreads();
    const int off = wid ? sh.scan[wid - 1] : 0;
    *tot = sh.scan[kResWarps - 1];
    __syncthreads();
    return off + incl - v;
}

// Fixed-order block sum of two doubles (warp trees, then warps in order by one thread).
__device__ __forceinline__ void res_sum2(double& a, double& b, ResShared& sh) {
    a = warp_sum(a);
    b = warp_sum(b);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        sh.red[0][wid] = a;
        sh.red[1][wid] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double x = 0.0, y = 0.0;
        for (int w = 0; w < kResWarps; ++w) {
            x += sh.red[0][w];
            y += sh.red[1][w];
        }
        sh.red[0][0] = x;
        sh.red[1][0] = y;
    }
    __syncthreads();
    a = sh.red[0][0];
    b = sh.red[1][0];
    __syncthreads();
}

__device__ __forceinline__ unsigned long long res_sum_u64(unsigned long long v, ResShared& sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) sh.hred[wid] = v;
    __syncthreads();
    unsigned long long s = 0;
    for (int w = 0; w < kResWarps; ++w) s += sh.hred[w];
    __syncthreads();
    return s;
}

// find_extrema flags of the 4 samples of group g (emd.cpp:16-33): bit k max, bit 4+k min.
__device__ __forceinline__ unsigned res_group_flags(const double* cur, int L, int g) {
    unsigned f = 0;
    const int t0 = 4 * g;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int t = t0 + k;
        if (t < 1 || t > L - 2) continue;
        const double v = cur[t], l = cur[t - 1], r = cur[t + 1];
        if (v == l || v == r) {  // plateau: the maximal run of samples equal to v, extremum at its middle
            int rs = t, re = t;
            while (rs > 0 && cur[rs - 1] == v) --rs;
            while (re < L - 1 && cur[re + 1] == v) ++re;
            if (rs > 0 && re < L - 1 && t == (rs + re) / 2) {
                const double lv = cur[rs - 1], rv = cur[re + 1];
                if (v > lv && v > rv) f |= 1u << k;
                else if (v < lv && v < rv) f |= 16u << k;
            }
        } else if (v > l && v > r) {
            f |= 1u << k;
        } else if (v < l && v < r) {
            f |= 16u << k;
        }
    }
    return f;
}

struct ResCtx {
    const ResArgs* P;
    int L, Lp, NG;
    double* cur;               // shared: the candidate (in place)
    unsigned short* pre[2];    // shared: extrema of side s before group g
    unsigned char* fl;         // shared: group flags
    double2* tab;              // shared: segment tables (rows {x, y} then {m, 1/h}, side 0 then side 1)
    int tab_rows;              // capacity in double2 rows
    double* xg;                // global (this CTA): the IMF input X (the running residue)
    double* oldc;              // global (this CTA): the candidate before the last eval (SD recheck)
    int n[2];                  // extrema counts of the last detection
    double2 *A[2], *B[2];      // table planes of the current sift
    int N[2];
};

// find_extrema over the candidate: group flags and prefix counts; returns the trace hash (when
// tracing) = sum over extrema of knot_hash(side, rank, index), the lockstep engine's definition.
__device__ unsigned long long res_detect(ResCtx& C, ResShared& sh, bool tracing) {
    int base0 = 0, base1 = 0;
    unsigned long long h = 0;
    for (int g0 = 0; g0 < C.NG; g0 += kResThreads) {
        const int g = g0 + (int)threadIdx.x;
        const unsigned f = g < C.NG ? res_group_flags(C.cur, C.L, g) : 0u;
        const int c = __popc(f & 15u) | (__popc(f >> 4) << 16);
        int tot;
        const int ex = res_excl_scan(c, &tot, sh);
        if (g < C.NG) {
            const int r0 = base0 + (ex & 0xFFFF), r1 = base1 + (ex >> 16);
            C.pre[0][g] = (unsigned short)r0;
            C.pre[1][g] = (unsigned short)r1;
            C.fl[g] = (unsigned char)f;
            if (tracing && f) {
                unsigned q = (unsigned)r0;
                for (unsigned m = f & 15u; m; m &= m - 1u) h += knot_hash(0, q++, (unsigned)(4 * g + __ffs(m) - 1));
                q = (unsigned)r1;
                for (unsigned m = f >> 4; m; m &= m - 1u) h += knot_hash(1, q++, (unsigned)(4 * g + __ffs(m) - 1));
            }
        }
        base0 += tot & 0xFFFF;
        base1 += tot >> 16;
    }
    C.n[0] = base0;
    C.n[1] = base1;
    return tracing ? res_sum_u64(h, sh) : 0ull;
}

// Mirrored knot rows {x, y} of both envelopes (envelope(), emd.cpp:107-122). Sifting always has
// both mirror pairs: find_extrema never reports index 0 or L-1. Returns false when the tables do
// not fit the shared-memory capacity (the host reruns the call on the lockstep engine).
__device__ bool res_tables(ResCtx& C) {
    C.N[0] = C.n[0] + 4;
    C.N[1] = C.n[1] + 4;
    if (2 * (C.N[0] + C.N[1]) > C.tab_rows) return false;
    C.A[0] = C.tab;
    C.B[0] = C.A[0] + C.N[0];
    C.A[1] = C.B[0] + C.N[0];
    C.B[1] = C.A[1] + C.N[1];
    for (int g = threadIdx.x; g < C.NG; g += kResThreads) {
        const unsigned f = C.fl[g];
        if (!f) continue;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            int q = 2 + C.pre[s][g];
            for (unsigned m = (f >> (4 * s)) & 15u; m; m &= m - 1u) {
                const int t = 4 * g + __ffs(m) - 1;
                C.A[s][q++] = make_double2((double)t, C.cur[t]);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        const int s = threadIdx.x, n = C.n[s];
        double2* A = C.A[s];
        const double e2 = 2.0 * (double)(C.L - 1);
        const double2 k0 = A[2], k1 = A[3], kn2 = A[n], kn1 = A[n + 1];
        A[0] = make_double2(-k1.x, k1.y);  // descending source order: -idx[1], -idx[0]
        A[1] = make_double2(-k0.x, k0.y);
        A[n + 2] = make_double2(e2 - kn2.x, kn2.y);  // 2*end - idx[n-2], 2*end - idx[n-1]
        A[n + 3] = make_double2(e2 - kn1.x, kn1.y);
    }
    __syncthreads();
    return true;
}

// Both envelopes' moments (emd.cpp:53-73, bit-exact); B[s] ends as {m_v, RN(1/(x_{v+1} - x_v))}.
// Threads [0, kResChains) solve side 0, the rest side 1, one chain of CH rows each:
//   1. rhs_i (emd.cpp:62, IEEE divisions) once per row into A[i].y (y is restored from the
//      candidate at the end: A[v].y = cur[index of knot v])
//   2. forward sweep (:64-69) from a guessed state kResWarm rows before the chain (exact from
//      row 1), {diag, rhs} of the chain's rows into B
//   3. back substitution (:70-73) from a guessed moment kResWarm rows above the chain, m into A.y
// Each boundary is verified bitwise (the guessed state at a chain's start against its
// predecessor's stored end); a mismatch replays the chains from there in order (one thread per
// side) until the recomputed rows agree with the stored ones. Returns the number of replays.
__device__ int res_solve(ResCtx& C, ResShared& sh, int& replays_out) {
    const int side = threadIdx.x >= kResChains ? 1 : 0;
    const int c = threadIdx.x - side * kResChains;
    double2* A = C.A[side];
    double2* B = C.B[side];
    const int N = C.N[side];
    const int R = N - 2;  // rows 1 .. N-2
    const int CH = max(kResChainMin, (R + kResChains - 1) / kResChains);
    const int nch = (R + CH - 1) / CH;
    const bool mine = c < nch;
    const int s = 1 + c * CH, e = min(s + CH, N - 1);
    const int warm = (C.P->debug & 1) ? 2 : kResWarm;  // test hook: short warm-ups force the replays
    if (threadIdx.x == 0) sh.bad = 0;
    // ---- 1. rhs per row (parked in B.x, then moved to A.y once every y has been read)
    for (int i = c + 1; i <= R; i += kResChains) {
        const double2 p = A[i - 1], q = A[i], n = A[i + 1];
        const double h0 = q.x - p.x, h1 = n.x - q.x;
        B[i].x = 6.0 * ((n.y - q.y) / h1 - (q.y - p.y) / h0);
    }
    __syncthreads();
    for (int i = c + 1; i <= R; i += kResChains) A[i].y = B[i].x;
    __syncthreads();
    // ---- 2. forward sweep
    double gd = 0.0, gr = 0.0;
    const int i0 = max(1, s - warm);
    if (mine) {
        double xp = A[i0 - 1].x, xc = A[i0].x, xn = A[i0 + 1].x;
        double h0 = xc - xp, h1 = xn - xc;
        double d = 2.0 * (h0 + h1);  // row i0 as if it were row 1 (exact when i0 == 1)
        double r = A[i0].y;
        if (i0 == s) B[s] = make_double2(d, r);
        for (int i = i0 + 1; i < e; ++i) {
            if (i == s) {
                gd = d;  // the guessed state at row s-1
                gr = r;
            }
            xp = xc;
            xc = xn;
            xn = A[i + 1].x;
            h0 = h1;
            h1 = xn - xc;
            const double w = h0 / d;
            d = 2.0 * (h0 + h1) - w * h0;
            r = A[i].y - w * r;
            if (i >= s) B[i] = make_double2(d, r);
        }
    }
    __syncthreads();
    if (mine && i0 < s) {
        const double2 t = B[s - 1];  // the predecessor chain's state at row s-1
        if (!same_bits(t.x, gd) || !same_bits(t.y, gr)) atomicOr(&sh.bad, 1 << side);
    }
    __syncthreads();
    int replays = 0;
    if (((sh.bad >> side) & 1) && c == 0) {  // replay chain heads in order until they agree
        for (int cc = 1; cc < nch; ++cc) {
            const int s2 = 1 + cc * CH, e2 = min(s2 + CH, N - 1);
            double d = B[s2 - 1].x, r = B[s2 - 1].y;
            for (int i = s2; i < e2; ++i) {
                const double h0 = A[i].x - A[i - 1].x, h1 = A[i + 1].x - A[i].x;
                const double w = h0 / d;
                d = 2.0 * (h0 + h1) - w * h0;
                r = A[i].y - w * r;
                const double2 st = B[i];
                if (same_bits(st.x, d) && same_bits(st.y, r)) break;  // the rest of the chain agrees
                B[i] = make_double2(d, r);
                ++replays;
            }
        }
    }
    __syncthreads();
    // ---- 3. back substitution: m_i into A[i].y (rhs is consumed; chains read only B and A.x)
    double mg = 0.0;
    const int top = min(e + warm, N - 1);
    if (mine) {
        double m = 0.0;  // exact when top == N-1
        for (int i = top - 1; i >= e; --i) {
            const double2 dr = B[i];
            m = (dr.y - (A[i + 1].x - A[i].x) * m) / dr.x;
        }
        mg = m;  // guessed m_e
        for (int i = e - 1; i >= s; --i) {
            const double2 dr = B[i];
            m = (dr.y - (A[i + 1].x - A[i].x) * m) / dr.x;
            A[i].y = m;
        }
    }
    if (threadIdx.x == 0) sh.bad = 0;
    __syncthreads();
    if (mine && top < N - 1 && !same_bits(mg, A[e].y)) atomicOr(&sh.bad, 1 << side);
    __syncthreads();
    if (((sh.bad >> side) & 1) && c == 0) {  // replay from the top chain down
        for (int cc = nch - 2; cc >= 0; --cc) {
            const int s2 = 1 + cc * CH, e2 = min(s2 + CH, N - 1);
            double m = A[e2].y;
            for (int i = e2 - 1; i >= s2; --i) {
                const double2 dr = B[i];
                m = (dr.y - (A[i + 1].x - A[i].x) * m) / dr.x;
                if (same_bits(A[i].y, m)) break;
                A[i].y = m;
                ++replays;
            }
        }
    }
    __syncthreads();
    // ---- the segment table {m, 1/h}; y back from the candidate
    const double e2 = 2.0 * (double)(C.L - 1);
    for (int v = c; v < N; v += kResChains) {
        const double x = A[v].x;
        const double h = v + 1 < N ? A[v + 1].x - x : 0.0;
        B[v] = make_double2(v == 0 || v == N - 1 ? 0.0 : A[v].y, v + 1 < N ? 1.0 / h : 0.0);
    }
    __syncthreads();
    for (int v = c; v < N; v += kResChains) {
        const double x = A[v].x;
        const int t = v <= 1 ? (int)(-x) : (v <= N - 3 ? (int)x : (int)(e2 - x));
        A[v].y = C.cur[t];
    }
    __syncthreads();
    replays_out = replays;
    return 0;
}

// Envelope value of side s at sample t whose segment row is q (spline_eval_fast, emd.cpp:80-85).
__device__ __forceinline__ double res_env(const double2* A, const double2* B, int q, double tt) {
    const double2 a0 = A[q], b0 = B[q], a1 = A[q + 1];
    const double m1 = B[q + 1].x;
    const double h = a1.x - a0.x;
    return spline_eval_fast(a0.x, a1.x, a0.y, a1.y, b0.x, m1, h, b0.y, h * h, tt);
}

// One sift pass (emd.cpp:142-148) in place; the candidate before it goes to oldc (SD recheck).
__device__ void res_eval(ResCtx& C, double& num, double& den) {
    double x = 0.0, y = 0.0;
    const double2 *A0 = C.A[0], *B0 = C.B[0], *A1 = C.A[1], *B1 = C.B[1];
    for (int g = threadIdx.x; g < C.NG; g += kResThreads) {
        const int t0 = 4 * g;
        const unsigned f = C.fl[g];
        const int q0 = 1 + C.pre[0][g], q1 = 1 + C.pre[1][g];
        const double2 v01 = *reinterpret_cast<const double2*>(C.cur + t0);
        const double2 v23 = *reinterpret_cast<const double2*>(C.cur + t0 + 2);
        const double cv[4] = {v01.x, v01.y, v23.x, v23.y};
        double nv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int t = t0 + k;
            const double tt = (double)t;
            const unsigned below = (1u << k) - 1u;  // extrema at t0 .. t-1 precede t
            const double u = res_env(A0, B0, q0 + __popc(f & below), tt);
            const double l = res_env(A1, B1, q1 + __popc((f >> 4) & below), tt);
            const double mean = 0.5 * (u + l);
            if (t < C.L) {
                x += mean * mean;
                y += cv[k] * cv[k];
                nv[k] = cv[k] - mean;
            } else {
                nv[k] = 0.0;
            }
        }
        *reinterpret_cast<double2*>(C.cur + t0) = make_double2(nv[0], nv[1]);
        *reinterpret_cast<double2*>(C.cur + t0 + 2) = make_double2(nv[2], nv[3]);
        *reinterpret_cast<double2*>(C.oldc + t0) = v01;
        *reinterpret_cast<double2*>(C.oldc + t0 + 2) = v23;
    }
    num = x;
    den = y;
}

// The reference's own left-to-right sums (emd.cpp:142-148) over the current tables and the
// candidate before the pass (oldc); one thread, only for uncertified SD decisions.
__device__ __noinline__ void res_sd_sequential(const ResCtx& C, double* num, double* den) {
    int seg[2] = {0, 0};
    double x = 0.0, y = 0.0;
    for (int t = 0; t < C.L; ++t) {
        const double tt = (double)t;
        double e[2];
        for (int k = 0; k < 2; ++k) {
            while (seg[k] + 2 < C.N[k] && tt > C.A[k][seg[k] + 1].x) ++seg[k];
            e[k] = res_env(C.A[k], C.B[k], seg[k], tt);
        }
        const double mean = 0.5 * (e[0] + e[1]);
        const double cv = C.oldc[t];
        x += mean * mean;
        y += cv * cv;
    }
    *num = x;
    *den = y;
}

__device__ void res_trace(const ResArgs& P, const RJob& J, int k, int iter, unsigned n0, unsigned n1,
                          unsigned long long h) {
    const int pos = atomicAdd(P.trace_count, 1);
    if (pos < P.trace_cap) {
        TraceRec r;
        r.task = J.task;
        r.m = J.m;
        r.k = k;
        r.iter = iter;
        r.n_max = n0;
        r.n_min = n1;
        r.hash = h;
        P.trace[pos] = r;
    }
}

#define RES_PROF(k)                                                     \
    do {                                                                \
        if (prof_on && threadIdx.x == 0) {                              \
            const long long now_ = clock64();                           \
            atomicAdd(&P.prof[k], (unsigned long long)(now_ - prof_t)); \
            prof_t = now_;                                              \
        }                                                               \
    } while (0)

// One job: emd()'s IMF loop (emd.cpp:155-172) with extract_imf (:127-153).
__device__ void res_job(ResCtx& C, ResShared& sh, int j) {
    const ResArgs& P = *C.P;
    const RJob J = P.jobs[j];
    RResult out{};
    out.k = J.k;
    const int L = C.L;
    const bool tracing = P.trace != nullptr;
    const bool prof_on = (P.debug & 2) && P.prof;
    long long prof_t = clock64();
    // X = the job's input (emd.cpp:238-240: x + beta*w), into the candidate and the residue copy
    for (int t = threadIdx.x; t < C.Lp; t += kResThreads) {
        double v = 0.0;
        if (t < L) v = J.init_kind == 1 ? J.a[t] + J.beta * J.b[t] : J.a[t];
        C.cur[t] = v;
        C.xg[t] = v;
    }
    __syncthreads();
    RES_PROF(6);
    int produced = 0;
    int* sifts = P.sifts + (size_t)j * P.kc;
    while (true) {
        if (J.kmax > 0 && out.k >= J.kmax) break;
        // ---- extract_imf(X): iteration 0's find_extrema (emd.cpp:133-140, :164)
        int iter = 0;
        if (P.max_iters > 0 || J.detect_only) {
            const unsigned long long h = res_detect(C, sh, tracing);
            if (tracing && threadIdx.x == 0) res_trace(P, J, out.k, 0, C.n[0], C.n[1], h);
            RES_PROF(0);
            out.n0 = C.n[0];
            out.n1 = C.n[1];
            if (J.detect_only) break;
            if (C.n[0] < 2 || C.n[1] < 2) {  // InsufficientExtrema on X: the decomposition ends
                out.ended_insufficient = 1;
                break;
            }
            while (true) {
                if (!res_tables(C)) {
                    out.smem_overflow = 1;
                    goto done;
                }
                RES_PROF(1);
                {
                    int rp = 0;
                    res_solve(C, sh, rp);
                    out.hazards += rp > 0;
                }
                RES_PROF(2);
                double num, den;
                res_eval(C, num, den);
                __syncthreads();
                RES_PROF(3);
                res_sum2(num, den, sh);
                ++iter;
                out.sifted += L;
                const bool unc = (P.debug & 4) || sd_decision_uncertain(num, den, L, P.sd_thr);
                if (unc) {  // the reference's sequential sums decide (rare)
                    if (threadIdx.x == 0) {
                        res_sd_sequential(C, &num, &den);
                        sh.red[0][0] = num;
                        sh.red[1][0] = den;
                        atomicAdd(P.sd_rechecks, 1);
                    }
                    __syncthreads();
                    num = sh.red[0][0];
                    den = sh.red[1][0];
                    __syncthreads();
                }
                RES_PROF(4);
                if (den == 0.0 || num / den < P.sd_thr || iter >= P.max_iters) break;  // emd.cpp:150, :131
                const unsigned long long h = res_detect(C, sh, tracing);
                if (tracing && threadIdx.x == 0) res_trace(P, J, out.k, iter, C.n[0], C.n[1], h);
                RES_PROF(0);
                if (C.n[0] < 2 || C.n[1] < 2) break;  // envelope throws: the candidate is the IMF
            }
        }
        // ---- the IMF is the candidate: store it, residue -= imf (emd.cpp:167)
        if (J.write_imf && produced >= P.kc) {
            out.k_overflow = 1;
            break;
        }
        if (threadIdx.x == 0 && produced < P.kc) sifts[produced] = iter;
        double* row = J.write_imf ? P.store + ((size_t)j * P.kc + produced) * C.Lp : nullptr;
        for (int t = threadIdx.x; t < L; t += kResThreads) {
            const double imf = C.cur[t];
            const double rv = C.xg[t] - imf;
            if (row) row[t] = imf;
            if (J.imf_out) J.imf_out[t] = imf;
            if (J.res_out) J.res_out[t] = rv;
            C.xg[t] = rv;
            C.cur[t] = rv;
        }
        __syncthreads();
        RES_PROF(5);
        ++produced;
        ++out.k;
    }
done:
    if (J.res_final)
        for (int t = threadIdx.x; t < L; t += kResThreads) J.res_final[t] = C.xg[t];
    out.produced = produced;
    if (threadIdx.x == 0) P.res[j] = out;
    __syncthreads();
}

__global__ void __launch_bounds__(kResThreads, 1) k_resident(ResArgs P) {
    extern __shared__ __align__(16) unsigned char res_smem[];
    __shared__ ResShared sh;
    ResCtx C;
    C.P = &P;
    C.L = P.L;
    C.Lp = (P.L + 3) & ~3;
    C.NG = C.Lp / 4;
    unsigned char* p = res_smem;
    C.cur = reinterpret_cast<double*>(p);
    p += (size_t)C.Lp * 8;
    C.tab = reinterpret_cast<double2*>(p);
    p += (size_t)P.tab_rows * 16;
    C.pre[0] = reinterpret_cast<unsigned short*>(p);
    C.pre[1] = C.pre[0] + C.NG;
    p += (size_t)C.NG * 4;
    C.fl = p;
    C.tab_rows = P.tab_rows;
    C.xg = P.scratch + (size_t)blockIdx.x * 2 * C.Lp;
    C.oldc = C.xg + C.Lp;
    while (true) {
        if (threadIdx.x == 0) sh.job = (int)atomicAdd(P.ticket, 1u);
        __syncthreads();
        const int j = sh.job;
        __syncthreads();
        if (j >= P.njobs) break;
        res_job(C, sh, j);
    }
}

// shared-memory bytes of k_resident for a signal of length L with `rows` table rows
size_t resident_smem_bytes(int L, int rows) {
    const size_t Lp = (size_t)((L + 3) & ~3);
    return Lp * 8 + (size_t)rows * 16 + (Lp / 4) * 5 + 16;
}

int resident_max_smem() {
    static int v = [] {
        int dev = 0, x = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&x, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        return x - (int)sizeof(ResShared) - 64;
    }();
    return v;
}

void launch_resident(const ResArgs& P, int grid, cudaStream_t st) {
    const size_t smem = resident_smem_bytes(P.L, P.tab_rows);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_resident, cudaFuncAttributeMaxDynamicSharedMemorySize, resident_max_smem());
        attr = true;
    }
    k_resident<<<grid, kResThreads, smem, st>>>(P);
    count_launches(1);
}

// sums[r][t] += store rows of every write_imf job in job order (emd.cpp:246-251 / :301-306):
// job j's IMF kk lands in row rowbase_j + kk. One thread per (row, sample).
__global__ void __launch_bounds__(256) k_res_accum(const RJob* jobs, const RResult* res, int njobs, const double* store,
                                                   int kc, long long Lp, int L, double* sums, int rows) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)rows * L) return;
    const int r = (int)(i / L), t = (int)(i % L);
    double* dst = sums + (size_t)r * L + t;
    double acc = *dst;
    bool any = false;
    for (int j = 0; j < njobs; ++j) {
        if (!jobs[j].write_imf) continue;
        const int kk = r - (jobs[j].k0 + jobs[j].k);
        if (kk < 0 || kk >= res[j].produced) continue;
        acc = acc + store[((size_t)j * kc + kk) * Lp + t];
        any = true;
    }
    if (any) *dst = acc;
}

void launch_res_accum(const RJob* jobs, const RResult* res, int njobs, const double* store, int kc, long long Lp,
                      int L, double* sums, int rows, cudaStream_t st) {
    const long long n = (long long)rows * L;
    if (n <= 0) return;
    k_res_accum<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(jobs, res, njobs, store, kc, Lp, L, sums, rows);
    count_launches(1);
}

}  // namespace dev
}  // namespace semd
