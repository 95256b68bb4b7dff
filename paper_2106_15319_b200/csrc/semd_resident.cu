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
constexpr int kResWarm = 32;      // speculative warm-up rows of a chain (forward and back), as the lockstep solve
constexpr int kResChainMin = 8;   // rows per chain at least
constexpr int kResChainDiv = 96;  // chains per side aimed at: longer chains cost latency, more chains redundant warm-up rows

extern __shared__ __align__(16) unsigned char res_smem[];
__device__ __forceinline__ double* sm_d(int off) { return reinterpret_cast<double*>(res_smem + off); }
__device__ __forceinline__ double2* sm_d2(int off) { return reinterpret_cast<double2*>(res_smem + off); }
__device__ __forceinline__ unsigned short* sm_u16(int off) { return reinterpret_cast<unsigned short*>(res_smem + off); }
__device__ __forceinline__ unsigned char* sm_u8(int off) { return res_smem + off; }

constexpr int kResRcpTab = 64;
struct ResShared {
    double red[2][kResWarps];
    int scan4[4][kResWarps];  // res_detect's four-round block scan
    unsigned long long hred[kResWarps];
    int job;
    bool moved[kResThreads];  // solve replay rounds: the chain's end changed
    int unc;  // a control word broadcast to the CTA
    double rtab[kResRcpTab + 1];  // RN(1/h) of small integer knot spacings (the IEEE quotients themselves)
};
// 1/h of a knot spacing (an integer >= 1, except across the reference's non-monotone right mirror
// knots): from the table when small, else the IEEE division
__device__ __forceinline__ double res_rcp_h(const ResShared& sh, double h) {
    return h >= 1.0 && h <= (double)kResRcpTab ? sh.rtab[(int)h] : 1.0 / h;
}
__device__ __forceinline__ void res_rcp_init(ResShared& sh) {  // visible after the next __syncthreads
    for (int i = threadIdx.x + 1; i <= kResRcpTab; i += blockDim.x) sh.rtab[i] = 1.0 / (double)i;
}

__device__ __forceinline__ bool same_bits(double a, double b) {
    return __double_as_longlong(a) == __double_as_longlong(b);
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
// The window t0-2 .. t0+5 arrives as four aligned 16-byte loads; each neighbour pair is compared
// once; samples equal to a neighbour take the reference's plateau rule (rare, out of line).
__device__ __noinline__ unsigned res_plateau_flags(const double* cur, int L, int t0, unsigned f, unsigned plat) {
    for (int k = 0; k < 4; ++k) {
        if (!((plat >> k) & 1u)) continue;
        const int t = t0 + k;
        const double v = cur[t];
        int rs = t, re = t;
        while (rs > 0 && cur[rs - 1] == v) --rs;
        while (re < L - 1 && cur[re + 1] == v) ++re;
        if (rs > 0 && re < L - 1 && t == (rs + re) / 2) {
            const double lv = cur[rs - 1], rv = cur[re + 1];
            if (v > lv && v > rv) f |= 1u << k;
            else if (v < lv && v < rv) f |= 16u << k;
        }
    }
    return f;
}
__device__ __forceinline__ unsigned res_group_flags(const double* cur, int L, int g) {
    const int t0 = 4 * g;
    double w[8];  // t0-2 .. t0+5 (padding beyond L reads zeros or the next group: masked below)
    if (t0 >= 4 && t0 + 8 <= ((L + 3) & ~3)) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 v = *reinterpret_cast<const double2*>(cur + t0 - 2 + 2 * q);
            w[2 * q] = v.x;
            w[2 * q + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int t = t0 - 2 + q;
            w[q] = t >= 0 && t < L ? cur[t] : 0.0;
        }
    }
    // pair j compares w[j+1] (sample t0-1+j) with w[j+2]
    unsigned up = 0, dn = 0;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        up |= (unsigned)(w[j + 2] > w[j + 1]) << j;
        dn |= (unsigned)(w[j + 2] < w[j + 1]) << j;
    }
    unsigned inm = 0;  // samples t0 .. t0+3 inside [1, L-2]
#pragma unroll
    for (int k = 0; k < 4; ++k) inm |= (unsigned)(t0 + k >= 1 && t0 + k <= L - 2) << k;
    const unsigned eq = ~(up | dn) & 31u;   // pair j equal (or unordered)
    unsigned fmax = up & (dn >> 1) & inm;   // v > l (pair k up) and v > r (pair k+1 down)
    unsigned fmin = dn & (up >> 1) & inm;
    unsigned f = fmax | (fmin << 4);
    const unsigned plat = (eq | (eq >> 1)) & inm;  // v == l or v == r
    if (plat) {
        // an unordered pair (NaN) is not a plateau: the reference's run logic never extends a run
        // over NaN and its strict comparisons fail, exactly like the fast path's bits
        unsigned real = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double v = w[k + 2];
            real |= (unsigned)(v == w[k + 1] || v == w[k + 3]) << k;
        }
        real &= inm;
        if (real) f = res_plateau_flags(cur, L, t0, f & ~(real | (real << 4)), real);
    }
    return f;
}

// Per-CTA context. Shared-memory arrays are byte offsets into res_smem (pointers rebuilt from the
// __shared__ symbol keep the compiler on LDS/STS; pointers loaded from this stack struct would
// be generic loads).
struct ResCtx {
    const ResArgs* P;
    int L, Lp, NG;
    int o_cur;                 // double[Lp]: the candidate (in place)
    int o_pre0, o_pre1;        // ushort[NG]: extrema of side s before group g
    int o_fl;                  // uchar[NG]: group flags
    int o_tab;                 // segment tables (rows {x, y} then {m, 1/h}, side 0 then side 1)
    int tab_rows;              // capacity in double2 rows
    double* xg;                // global (this CTA): the IMF input X (the running residue)
    double* oldc;              // global (this CTA): the candidate before the last eval (SD recheck)
    int n[2];                  // extrema counts of the last detection
    int o_A[2], o_B[2];        // table planes of the current sift
    int N[2];
};

// find_extrema over the candidate: group flags and prefix counts; returns the trace hash (when
// tracing) = sum over extrema of knot_hash(side, rank, index), the lockstep engine's definition.
__device__ __forceinline__ unsigned long long res_detect(ResCtx& C, ResShared& sh, bool tracing) {
    const double* const cur = sm_d(C.o_cur);
    unsigned short* const pre0 = sm_u16(C.o_pre0);
    unsigned short* const pre1 = sm_u16(C.o_pre1);
    unsigned char* const fl = sm_u8(C.o_fl);
    const int NG = C.NG, L = C.L;
    static_assert(kResMaxL <= 4 * 4 * kResThreads, "at most four groups per thread");
    // group g = i * kResThreads + tid, i < 4: flags and packed counts (max | min << 16) per round
    unsigned f[4];
    int cnt[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int g = i * kResThreads + (int)threadIdx.x;
        f[i] = g < NG ? res_group_flags(cur, L, g) : 0u;
        cnt[i] = __popc(f[i] & 15u) | (__popc(f[i] >> 4) << 16);
    }
    // one block scan of the four rounds at once: within-round exclusive prefixes + round totals
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) incl[i] = cnt[i];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int y = __shfl_up_sync(0xffffffffu, incl[i], o);
            if (lane >= o) incl[i] += y;
        }
    }
    if (lane == 31) {
#pragma unroll
        for (int i = 0; i < 4; ++i) sh.scan4[i][wid] = incl[i];
    }
    __syncthreads();
    if (wid < 4) {  // warp i scans round i's warp totals
        int x = lane < kResWarps ? sh.scan4[wid][lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane < kResWarps) sh.scan4[wid][lane] = x;
    }
    __syncthreads();
    int base = 0;  // packed running total of the earlier rounds
    unsigned long long h = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int g = i * kResThreads + (int)threadIdx.x;
        const int ex = base + (wid ? sh.scan4[i][wid - 1] : 0) + incl[i] - cnt[i];
        if (g < NG) {
            const int r0 = ex & 0xFFFF, r1 = ex >> 16;
            pre0[g] = (unsigned short)r0;
            pre1[g] = (unsigned short)r1;
            fl[g] = (unsigned char)f[i];
            if (tracing && f[i]) {
                unsigned q = (unsigned)r0;
                for (unsigned m = f[i] & 15u; m; m &= m - 1u) h += knot_hash(0, q++, (unsigned)(4 * g + __ffs(m) - 1));
                q = (unsigned)r1;
                for (unsigned m = f[i] >> 4; m; m &= m - 1u) h += knot_hash(1, q++, (unsigned)(4 * g + __ffs(m) - 1));
            }
        }
        base += sh.scan4[i][kResWarps - 1];
    }
    C.n[0] = base & 0xFFFF;
    C.n[1] = base >> 16;
    SEMD_ASSERT(C.n[0] <= C.L / 2 && C.n[1] <= C.L / 2);
    __syncthreads();
    return tracing ? res_sum_u64(h, sh) : 0ull;
}

// Mirrored knot rows {x, y} of both envelopes (envelope(), emd.cpp:107-122). Sifting always has
// both mirror pairs: find_extrema never reports index 0 or L-1. Returns false when the tables do
// not fit the shared-memory capacity (the host reruns the call on the lockstep engine).
__device__ __forceinline__ bool res_tables(ResCtx& C) {
    C.N[0] = C.n[0] + 4;
    C.N[1] = C.n[1] + 4;
    if (2 * (C.N[0] + C.N[1]) > C.tab_rows) return false;
    C.o_A[0] = C.o_tab;
    C.o_B[0] = C.o_A[0] + 16 * C.N[0];
    C.o_A[1] = C.o_B[0] + 16 * C.N[0];
    C.o_B[1] = C.o_A[1] + 16 * C.N[1];
    for (int g = threadIdx.x; g < C.NG; g += kResThreads) {
        const unsigned f = sm_u8(C.o_fl)[g];
        if (!f) continue;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            int q = 2 + sm_u16(s ? C.o_pre1 : C.o_pre0)[g];
            for (unsigned m = (f >> (4 * s)) & 15u; m; m &= m - 1u) {
                const int t = 4 * g + __ffs(m) - 1;
                sm_d2(C.o_A[s])[q++] = make_double2((double)t, sm_d(C.o_cur)[t]);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        const int s = threadIdx.x, n = C.n[s];
        SEMD_ASSERT(n >= 2 && C.o_B[1] + 16 * C.N[1] <= C.o_tab + 16 * C.tab_rows);
        double2* A = sm_d2(C.o_A[s]);
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
#define SOLVE_SUB(k)                                                        \
    do {                                                                    \
        if (sprof && threadIdx.x == 0) {                                    \
            const long long now_ = clock64();                               \
            atomicAdd(&C.P->prof[k], (unsigned long long)(now_ - sprof_t)); \
            sprof_t = now_;                                                 \
        }                                                                   \
    } while (0)
__device__ __forceinline__ int res_solve(ResCtx& C, ResShared& sh, int& replays_out) {
    const bool sprof = (C.P->debug & 2) && C.P->prof;
    long long sprof_t = clock64();
    const int side = threadIdx.x >= kResChains ? 1 : 0;
    const int c = threadIdx.x - side * kResChains;
    double2* A = sm_d2(C.o_A[side]);
    double2* B = sm_d2(C.o_B[side]);
    const int N = C.N[side];
    const int R = N - 2;  // rows 1 .. N-2
    const int cdiv = C.P->chain_div > 0 ? C.P->chain_div : kResChainDiv;
    const int CH = max(kResChainMin, max((R + kResChains - 1) / kResChains, (R + cdiv - 1) / cdiv));
    const int nch = (R + CH - 1) / CH;
    const bool mine = c < nch;
    const int s = 1 + c * CH, e = min(s + CH, N - 1);
    const int warm = (C.P->debug & 1) ? 2 : kResWarm;  // test hook: short warm-ups force the replays
    SEMD_ASSERT(!mine || (s >= 1 && s < e && e <= N - 1));
    // ---- 1. rhs per row: the slope (y[i+1]-y[i])/h_i of every segment once (exactly rounded:
    // div_rn with RN(1/h)), parked in B.x; then rhs_i = 6 (slope_i - slope_{i-1}) into A.y, once
    // every y has been read
    for (int i = c; i <= R; i += kResChains) {
        const double2 q = A[i], n = A[i + 1];
        const double h = n.x - q.x;
        B[i].x = div_rn(n.y - q.y, h, res_rcp_h(sh, h));
    }
    __syncthreads();
    for (int i = c + 1; i <= R; i += kResChains) A[i].y = 6.0 * (B[i].x - B[i - 1].x);
    __syncthreads();
    SOLVE_SUB(8);
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
    // Boundary check and replay rounds: a chain whose guessed start state differs from its
    // predecessor's stored end replays its rows from that end until a recomputed row equals the
    // stored one (from there on the stored rows are the sequential ones); a replay that reaches the
    // chain's end moved that end, and the successor is checked in the next round.
    int replays = 0;
    bool dirty = false;
    if (mine && i0 < s) {
        const double2 t = B[s - 1];  // the predecessor chain's state at row s-1
        dirty = !same_bits(t.x, gd) || !same_bits(t.y, gr);
    }
    while (__syncthreads_or(dirty)) {
        bool moved = false;
        if (dirty) {
            double d = B[s - 1].x, r = B[s - 1].y;
            moved = true;
            for (int i = s; i < e; ++i) {
                const double h0 = A[i].x - A[i - 1].x, h1 = A[i + 1].x - A[i].x;
                const double w = h0 / d;
                d = 2.0 * (h0 + h1) - w * h0;
                r = A[i].y - w * r;
                const double2 st = B[i];
                if (same_bits(st.x, d) && same_bits(st.y, r)) {
                    moved = false;
                    break;
                }
                B[i] = make_double2(d, r);
                ++replays;
            }
        }
        sh.moved[threadIdx.x] = moved;
        __syncthreads();
        dirty = mine && c > 0 && sh.moved[threadIdx.x - 1];
    }
    SOLVE_SUB(9);
    // ---- 3. back substitution. rhs is consumed: A[i].y = RN(1/diag_i), so each row is the exactly
    // rounded div_rn (r - h m) / diag (Markstein, as the lockstep solve) off a 5-op critical path.
    // Phase a: every chain runs its warm-up rows (reading other chains' rows); phase b: its own
    // rows from the guessed m_e, writing m_i over A[i].y row by row (only its own rows).
    for (int i = c + 1; i <= R; i += kResChains) A[i].y = 1.0 / B[i].x;
    __syncthreads();
    SOLVE_SUB(12);
    double mg = 0.0;
    const int top = min(e + warm, N - 1);
    if (mine) {
        double m = 0.0;  // exact when top == N-1
        for (int i = top - 1; i >= e; --i) {
            const double2 dr = B[i];
            const double2 a0 = A[i];
            m = div_rn(dr.y - (A[i + 1].x - a0.x) * m, dr.x, a0.y);
        }
        mg = m;  // guessed m_e
    }
    __syncthreads();
    if (mine) {
        double m = mg;
        for (int i = e - 1; i >= s; --i) {
            const double2 dr = B[i];
            const double2 a0 = A[i];
            m = div_rn(dr.y - (A[i + 1].x - a0.x) * m, dr.x, a0.y);
            A[i].y = m;
        }
    }
    __syncthreads();
    // the same rounds downwards: chain c starts from m_e = A[e].y (chain c+1's first row); own
    // rows hold m now, so replays divide exactly (IEEE)
    dirty = mine && top < N - 1 && !same_bits(mg, A[e].y);
    while (__syncthreads_or(dirty)) {
        bool moved = false;
        if (dirty) {
            double m = A[e].y;
            moved = true;
            for (int i = e - 1; i >= s; --i) {
                const double2 dr = B[i];
                m = (dr.y - (A[i + 1].x - A[i].x) * m) / dr.x;
                if (same_bits(A[i].y, m)) {
                    moved = false;
                    break;
                }
                A[i].y = m;
                ++replays;
            }
        }
        sh.moved[threadIdx.x] = moved;
        __syncthreads();
        dirty = mine && c + 1 < nch && sh.moved[threadIdx.x + 1];
    }
    SOLVE_SUB(10);
    // ---- the segment table {m, 1/h}; y back from the candidate
    const double* const cur = sm_d(C.o_cur);
    const double e2 = 2.0 * (double)(C.L - 1);
    for (int v = c; v < N; v += kResChains) {
        const double x = A[v].x;
        const double h = v + 1 < N ? A[v + 1].x - x : 0.0;
        B[v] = make_double2(v == 0 || v == N - 1 ? 0.0 : A[v].y, v + 1 < N ? res_rcp_h(sh, h) : 0.0);
    }
    __syncthreads();
    for (int v = c; v < N; v += kResChains) {
        const double x = A[v].x;
        const int t = v <= 1 ? (int)(-x) : (v <= N - 3 ? (int)x : (int)(e2 - x));
        A[v].y = cur[t];
    }
    __syncthreads();
    SOLVE_SUB(11);
    replays_out = replays;
    return 0;
}

// Envelope value of side s at sample t whose segment row is q (spline_eval_fast, emd.cpp:80-85).
__device__ __forceinline__ double res_env(const double2* A, const double2* B, int q, double tt) {
    SEMD_ASSERT(q >= 0 && A + q + 1 < B);  // rows q, q+1 of the {x, y} plane (B follows A)
    const double2 a0 = A[q], b0 = B[q], a1 = A[q + 1];
    const double m1 = B[q + 1].x;
    const double h = a1.x - a0.x;
    return spline_eval_fast(a0.x, a1.x, a0.y, a1.y, b0.x, m1, h, b0.y, h * h, tt);
}

// One sift pass (emd.cpp:142-148) in place; the candidate before it goes to oldc (SD recheck).
__device__ __forceinline__ void res_eval(ResCtx& C, double& num, double& den) {
    double x = 0.0, y = 0.0;
    const double2 *const A0 = sm_d2(C.o_A[0]), *const B0 = sm_d2(C.o_B[0]), *const A1 = sm_d2(C.o_A[1]),
                  *const B1 = sm_d2(C.o_B[1]);
    double* const cur = sm_d(C.o_cur);
    double* const oldc = C.oldc;
    const unsigned char* const fl = sm_u8(C.o_fl);
    const unsigned short* const pre0 = sm_u16(C.o_pre0);
    const unsigned short* const pre1 = sm_u16(C.o_pre1);
    const int NG = C.NG, L = C.L;
    // items of 2 samples (half a detection group): the rounds over the CTA are better filled
    for (int hg = threadIdx.x; hg < 2 * NG; hg += kResThreads) {
        const int g = hg >> 1, kb = (hg & 1) * 2;
        const int t0 = 4 * g + kb;
        const unsigned f = fl[g];
        const int q0 = 1 + pre0[g], q1 = 1 + pre1[g];
        const double2 v = *reinterpret_cast<const double2*>(cur + t0);
        const double cv[2] = {v.x, v.y};
        double nv[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int t = t0 + k;
            const double tt = (double)t;
            const unsigned below = (1u << (kb + k)) - 1u;  // the group's extrema before t precede t
            const double u = res_env(A0, B0, q0 + __popc(f & below), tt);
            const double l = res_env(A1, B1, q1 + __popc((f >> 4) & below), tt);
            const double mean = 0.5 * (u + l);
            if (t < L) {
                x += mean * mean;
                y += cv[k] * cv[k];
                nv[k] = cv[k] - mean;
            } else {
                nv[k] = 0.0;
            }
        }
        *reinterpret_cast<double2*>(cur + t0) = make_double2(nv[0], nv[1]);
        *reinterpret_cast<double2*>(oldc + t0) = v;
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
            while (seg[k] + 2 < C.N[k] && tt > sm_d2(C.o_A[k])[seg[k] + 1].x) ++seg[k];
            e[k] = res_env(sm_d2(C.o_A[k]), sm_d2(C.o_B[k]), seg[k], tt);
        }
        const double mean = 0.5 * (e[0] + e[1]);
        const double cv = C.oldc[t];
        x += mean * mean;
        y += cv * cv;
    }
    *num = x;
    *den = y;
}

__device__ void res_trace(const ResArgs& P, int task, int m, int k, int iter, unsigned n0, unsigned n1,
                          unsigned long long h) {
    const int pos = atomicAdd(P.trace_count, 1);
    if (pos < P.trace_cap) {
        TraceRec r;
        r.task = task;
        r.m = m;
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

enum { RX_IMF = 0, RX_INSUFFICIENT = 1, RX_OVERFLOW = 2 };
struct RxStats {
    long long sifted;
    int hazards;
    unsigned n0, n1;  // extrema counts of the last detection
};

// extract_imf (emd.cpp:127-153) on the shared-memory candidate X: RX_IMF leaves the IMF in cur
// after *iter sifts; RX_INSUFFICIENT: X itself has fewer than 2 maxima or minima (emd.cpp:138,
// cur = X untouched); RX_OVERFLOW: the segment tables outgrew the shared memory. Trace records
// (task, m, k, iter) of every find_extrema call, as the lockstep engine writes them.
__device__ __forceinline__ int res_extract(ResCtx& C, ResShared& sh, int task, int m, int k, int* iter_out, RxStats& st) {
    const ResArgs& P = *C.P;
    const int L = C.L;
    const bool tracing = P.trace != nullptr;
    const bool prof_on = (P.debug & 2) && P.prof;
    long long prof_t = clock64();
    int iter = 0;
    *iter_out = 0;
    if (P.max_iters <= 0) return RX_IMF;  // the sift loop never runs: the IMF is X
    {
        const unsigned long long h = res_detect(C, sh, tracing);
        if (tracing && threadIdx.x == 0) res_trace(P, task, m, k, 0, C.n[0], C.n[1], h);
        RES_PROF(0);
    }
    st.n0 = C.n[0];
    st.n1 = C.n[1];
    if (C.n[0] < 2 || C.n[1] < 2) return RX_INSUFFICIENT;
    while (true) {
        if (!res_tables(C)) return RX_OVERFLOW;
        RES_PROF(1);
        {
            int rp = 0;
            res_solve(C, sh, rp);
            st.hazards += rp > 0;
        }
        RES_PROF(2);
        double num, den;
        res_eval(C, num, den);
        __syncthreads();
        RES_PROF(3);
        res_sum2(num, den, sh);
        ++iter;
        st.sifted += L;
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
        if (tracing && threadIdx.x == 0) res_trace(P, task, m, k, iter, C.n[0], C.n[1], h);
        RES_PROF(0);
        st.n0 = C.n[0];
        st.n1 = C.n[1];
        if (C.n[0] < 2 || C.n[1] < 2) break;  // envelope throws: the candidate is the IMF
    }
    *iter_out = iter;
    return RX_IMF;
}

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
        sm_d(C.o_cur)[t] = v;
        C.xg[t] = v;
    }
    __syncthreads();
    RES_PROF(6);
    int produced = 0;
    int* sifts = P.sifts + (size_t)j * P.kc;
    RxStats st{};
    while (true) {
        if (J.kmax > 0 && out.k >= J.kmax) break;
        if (J.detect_only) {  // one find_extrema (the CEEMDAN stage check, emd.cpp:311)
            const unsigned long long h = res_detect(C, sh, tracing);
            if (tracing && threadIdx.x == 0) res_trace(P, J.task, J.m, out.k, 0, C.n[0], C.n[1], h);
            st.n0 = C.n[0];
            st.n1 = C.n[1];
            break;
        }
        int iter = 0;
        const int rc = res_extract(C, sh, J.task, J.m, out.k, &iter, st);
        if (rc == RX_OVERFLOW) {
            out.smem_overflow = 1;
            break;
        }
        if (rc == RX_INSUFFICIENT) {  // InsufficientExtrema on X: the decomposition ends (emd.cpp:164)
            out.ended_insufficient = 1;
            break;
        }
        // ---- the IMF is the candidate: store it, residue -= imf (emd.cpp:167)
        if (J.write_imf && produced >= P.kc) {
            out.k_overflow = 1;
            break;
        }
        prof_t = clock64();
        if (threadIdx.x == 0 && produced < P.kc) sifts[produced] = iter;
        double* row = J.write_imf ? P.store + ((size_t)j * P.kc + produced) * C.Lp : nullptr;
        for (int t = threadIdx.x; t < L; t += kResThreads) {
            const double imf = sm_d(C.o_cur)[t];
            const double rv = C.xg[t] - imf;
            if (row) row[t] = imf;
            if (J.imf_out) J.imf_out[t] = imf;
            if (J.res_out) J.res_out[t] = rv;
            C.xg[t] = rv;
            sm_d(C.o_cur)[t] = rv;
        }
        __syncthreads();
        RES_PROF(5);
        ++produced;
        ++out.k;
    }
    if (J.res_final)
        for (int t = threadIdx.x; t < L; t += kResThreads) J.res_final[t] = C.xg[t];
    out.produced = produced;
    out.sifted = st.sifted;
    out.hazards = st.hazards;
    out.n0 = st.n0;
    out.n1 = st.n1;
    if (threadIdx.x == 0) P.res[j] = out;
    __syncthreads();
}

// Shared-memory carve-up common to the resident kernels.
__device__ __forceinline__ void res_setup(ResCtx& C, const ResArgs& P) {
    C.P = &P;
    C.L = P.L;
    C.Lp = (P.L + 3) & ~3;
    C.NG = C.Lp / 4;
    int o = 0;
    C.o_cur = o;
    o += C.Lp * 8;
    C.o_tab = o;
    o += P.tab_rows * 16;
    C.o_pre0 = o;
    C.o_pre1 = o + C.NG * 2;
    o += C.NG * 4;
    C.o_fl = o;
    C.tab_rows = P.tab_rows;
    C.xg = P.scratch + (size_t)blockIdx.x * 2 * C.Lp;
    C.oldc = C.xg + C.Lp;
}

__global__ void __launch_bounds__(kResThreads, 1) k_resident(ResArgs P) {
    __shared__ ResShared sh;
    ResCtx C;
    res_setup(C, P);
    res_rcp_init(sh);
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

__global__ void __launch_bounds__(kResThreads, 1) k_res_ceemdan(ResArgs P, CeeArgs Q);

// the kernels' dynamic shared-memory limit (a per-device function attribute; launch_setup() runs
// this for every context's device)
cudaError_t resident_setup() {
    cudaError_t e = cudaFuncSetAttribute(k_resident, cudaFuncAttributeMaxDynamicSharedMemorySize, resident_max_smem());
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_res_ceemdan, cudaFuncAttributeMaxDynamicSharedMemorySize, resident_max_smem());
}

void launch_resident(const ResArgs& P, int grid, cudaStream_t st) {
    const size_t smem = resident_smem_bytes(P.L, P.tab_rows);
    k_resident<<<grid, kResThreads, smem, st>>>(P);
    count_launches(1);
}

// ---------------------------------------------------------------- CEEMDAN on the device
//
// emd.cpp:264-344 in one cooperative launch (every CTA resident): stage K runs one job per
// realization m -- the next mode of the noise residue (task 1, emd.cpp:316-325; the mode stays in
// shared memory) and the first mode of r_K + beta_K E_K(w_m) (task 2, :326-329), or of
// x + beta_0 w_m at K = 0 (:296-300) -- then a grid barrier, the ordered mean of the first modes
// (:301-306 / :331-338, realization order), the all-zero test and the residue update. The residue
// check (find_extrema(residue).total() < 3, :311) and beta_K = nstd * signal_std(r_K) (:312, the
// reference's two sequential passes) run in CTA 0 while the other CTAs start their noise modes.

// GPU-scope acquire loads for flags other CTAs publish (volatile would make them system-scope)
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_acquire(const int* p) { return (int)ld_acquire(reinterpret_cast<const unsigned*>(p)); }

__device__ __forceinline__ void grid_sync(CeeCtl* ctl) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire(&ctl->bar_gen);
        __threadfence();
        if (atomicAdd(&ctl->bar_count, 1u) == gridDim.x - 1) {
            ctl->bar_count = 0;
            __threadfence();
            atomicAdd(&ctl->bar_gen, 1u);
        } else {
            while (ld_acquire(&ctl->bar_gen) == g) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}
// a control word read once per CTA after a grid barrier and broadcast through shared memory
__device__ __forceinline__ int cta_flag(const int* p, ResShared& sh) {
    if (threadIdx.x == 0) sh.unc = ld_acquire(p);
    __syncthreads();
    const int v = sh.unc;
    __syncthreads();
    return v;
}

// emd.cpp:209-217 on the shared-memory copy (one thread; two sequential passes)
__device__ double res_std_seq(const double* v, int n) {
    double mean = 0.0;
    for (int i = 0; i < n; ++i) mean += v[i];
    mean /= (double)n;
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += (v[i] - mean) * (v[i] - mean);
    return sqrt(acc / (double)n);
}

__global__ void __launch_bounds__(kResThreads, 1) k_res_ceemdan(ResArgs P, CeeArgs Q) {
    __shared__ ResShared sh;
    ResCtx C;
    res_setup(C, P);
    res_rcp_init(sh);
    __syncthreads();
    CeeCtl* ctl = Q.ctl;
    const int L = C.L;
    const bool tracing = P.trace != nullptr;
    RxStats st{};
    int K = 0;
    for (;; ++K) {
        if (K >= Q.kcap || K >= 64) {  // the host grows the rows and reruns the call
            if (blockIdx.x == 0 && threadIdx.x == 0) ctl->status = 2;
            break;
        }
        if (K > 0) {
            if (blockIdx.x == 0) {  // emd.cpp:310-311
                int stop = Q.max_imfs > 0 && K >= Q.max_imfs;
                if (!stop) {
                    for (int t = threadIdx.x; t < C.Lp; t += kResThreads) sm_d(C.o_cur)[t] = t < L ? __ldcg(Q.residue + t) : 0.0;
                    __syncthreads();
                    const unsigned long long h = res_detect(C, sh, tracing);
                    if (tracing && threadIdx.x == 0) res_trace(P, 3, -1, K, 0, C.n[0], C.n[1], h);
                    stop = C.n[0] + C.n[1] < 3;
                }
                if (threadIdx.x == 0) ctl->stop[K] = stop;
            }
            grid_sync(ctl);
            if (cta_flag(&ctl->stop[K], sh)) break;
            if (blockIdx.x == 0 && threadIdx.x == 0) {  // beta_K (emd.cpp:312); cur holds the residue
                ctl->beta[K] = Q.nstd * res_std_seq(sm_d(C.o_cur), L);
                __threadfence();
                atomicMax(&ctl->beta_stage, K);
            }
        }
        // items: K == 0: the nr first modes; K > 0: the nr noise modes, then the nr first modes
        // (a first mode waits for its noise mode, handed over through Q.E and the stage-tagged
        // Q.edone flag) -- finer items shorten the stage's tail
        const int nitems = K == 0 ? Q.nr : 2 * Q.nr;
        while (true) {
            if (threadIdx.x == 0) sh.job = (int)atomicAdd(&ctl->ticket[K], 1u);
            __syncthreads();
            const int item = sh.job;
            __syncthreads();
            if (item >= nitems) break;
            const bool noise_item = K > 0 && item < Q.nr;
            const int j = K > 0 && item >= Q.nr ? item - Q.nr : item;
            const int m = Q.m0 + j;
            double* w = Q.nres + (size_t)j * Q.Ls;
            double* E = Q.E + (size_t)j * C.Lp;
            int iter = 0;
            if (noise_item) {  // E_K(w_m): the next mode of the noise residue (emd.cpp:316-325)
                int have = 0;
                if (__ldcg(Q.alive + j)) {
                    for (int t = threadIdx.x; t < C.Lp; t += kResThreads) sm_d(C.o_cur)[t] = t < L ? __ldcg(w + t) : 0.0;
                    __syncthreads();
                    const int rc = res_extract(C, sh, 1, m, K, &iter, st);
                    if (rc == RX_OVERFLOW) {
                        if (threadIdx.x == 0) ctl->status = 1;
                    } else if (rc == RX_INSUFFICIENT) {
                        if (threadIdx.x == 0) Q.alive[j] = 0;
                    } else {
                        for (int t = threadIdx.x; t < L; t += kResThreads) {
                            const double e = sm_d(C.o_cur)[t];
                            w[t] = __ldcg(w + t) - e;
                            E[t] = e;
                        }
                        have = 1;
                    }
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    Q.e_have[j] = have;
                    __threadfence();
                    atomicExch(Q.edone + j, K);
                }
                continue;
            }
            if (K == 0) {  // x + beta_0 w (emd.cpp:297-298)
                for (int t = threadIdx.x; t < C.Lp; t += kResThreads)
                    sm_d(C.o_cur)[t] = t < L ? Q.x[t] + Q.beta0 * __ldcg(w + t) : 0.0;
                __syncthreads();
            } else {
                if (threadIdx.x == 0) {
                    while (ld_acquire(Q.edone + j) < K) __nanosleep(128);
                    while (ld_acquire(&ctl->beta_stage) < K) __nanosleep(256);
                    sh.red[0][0] = __ldcg(&ctl->beta[K]);
                    sh.unc = __ldcg(Q.e_have + j);
                }
                __syncthreads();
                const double beta = sh.red[0][0];
                const bool have = sh.unc != 0;
                __syncthreads();
                for (int t = threadIdx.x; t < C.Lp; t += kResThreads)  // r + beta * E (zeros when exhausted)
                    sm_d(C.o_cur)[t] = t < L ? __ldcg(Q.residue + t) + beta * (have ? __ldcg(E + t) : 0.0) : 0.0;
                __syncthreads();
            }
            const int rc = res_extract(C, sh, 2, m, K, &iter, st);  // first_mode (emd.cpp:285-290)
            if (rc == RX_OVERFLOW) {
                if (threadIdx.x == 0) ctl->status = 1;
                continue;
            }
            double* row = Q.e1 + (size_t)j * C.Lp;
            if (rc == RX_IMF)
                for (int t = threadIdx.x; t < L; t += kResThreads) row[t] = sm_d(C.o_cur)[t];
            if (threadIdx.x == 0) Q.e1_ok[j] = rc == RX_IMF;
            __syncthreads();
        }
        grid_sync(ctl);
        if (cta_flag(&ctl->status, sh)) break;
        // the stage mean in realization order (emd.cpp:301-306, :331-338)
        int nz = 0;
        for (int t = blockIdx.x * kResThreads + threadIdx.x; t < L; t += gridDim.x * kResThreads) {
            double acc = 0.0;
            for (int j = 0; j < Q.nr; ++j)
                if (__ldcg(Q.e1_ok + j)) acc += __ldcg(Q.e1 + (size_t)j * C.Lp + t);
            const double mode = acc * Q.inv_nr;
            Q.modes[(size_t)K * L + t] = mode;
            if (K == 0) Q.residue[t] -= mode;
            nz |= mode != 0.0;
        }
        if (K > 0) {
            if (__syncthreads_or(nz) && threadIdx.x == 0) ctl->nonzero[K] = 1;
            grid_sync(ctl);
            if (!cta_flag(&ctl->nonzero[K], sh)) break;  // nothing extractable anywhere (emd.cpp:336)
            for (int t = blockIdx.x * kResThreads + threadIdx.x; t < L; t += gridDim.x * kResThreads)
                Q.residue[t] -= Q.modes[(size_t)K * L + t];
        }
        grid_sync(ctl);
    }
    if (threadIdx.x == 0) {
        atomicAdd(&ctl->sifted, (unsigned long long)st.sifted);
        atomicAdd(&ctl->hazards, st.hazards);
        if (blockIdx.x == 0) ctl->K = K;
    }
}

int launch_res_ceemdan(const ResArgs& P, const CeeArgs& Q, int grid, cudaStream_t st) {
    const size_t smem = resident_smem_bytes(P.L, P.tab_rows);
    ResArgs p = P;
    CeeArgs q = Q;
    void* args[] = {&p, &q};
    count_launches(1);
    return (int)cudaLaunchCooperativeKernel((const void*)k_res_ceemdan, dim3(grid), dim3(kResThreads), args, smem, st);
}

// sums[r][t] += store rows of every write_imf job in job order (emd.cpp:246-251 / :301-306;
// baseline.cpp:14 per channel): job j's IMF kk lands in row rowbase_j + kk. One thread per
// (row, sample); the jobs that can write row r are the range rowj[2r] .. rowj[2r+1] (job rows are
// non-decreasing in job order in every driver).
__global__ void __launch_bounds__(256) k_res_accum(const RJob* jobs, const RResult* res, const int* rowj,
                                                   const double* store, int kc, long long Lp, int L, double* sums,
                                                   int rows) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)rows * L) return;
    const int r = (int)(i / L), t = (int)(i % L);
    const int j0 = rowj[2 * r], j1 = rowj[2 * r + 1];
    if (j0 >= j1) return;
    double* dst = sums + (size_t)r * L + t;
    double acc = *dst;
    bool any = false;
    for (int j = j0; j < j1; ++j) {
        if (!jobs[j].write_imf) continue;
        const int kk = r - (jobs[j].k0 + jobs[j].k);
        if (kk < 0 || kk >= res[j].produced) continue;
        SEMD_ASSERT(kk < kc);
        acc = acc + store[((size_t)j * kc + kk) * Lp + t];
        any = true;
    }
    if (any) *dst = acc;
}

void launch_res_accum(const RJob* jobs, const RResult* res, const int* rowj, const double* store, int kc, long long Lp,
                      int L, double* sums, int rows, cudaStream_t st) {
    const long long n = (long long)rows * L;
    if (n <= 0) return;
    k_res_accum<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(jobs, res, rowj, store, kc, Lp, L, sums, rows);
    count_launches(1);
}

}  // namespace dev
}  // namespace semd
