// semd_eval.cu -- k_eval, the sift pass (the dominant kernel).
//
// Per tile of kEvalTile samples of one slot:
//   new = cur - 0.5*(upper + lower)      (emd.cpp:142-148; spline evaluation :75-86)
//   SD partials sum(mean^2), sum(cur^2)  (emd.cpp:145-146)
//   extrema of `new` + tile-local ordered lists for the next sift (emd.cpp:10-35)
//
// Work unit: a warp owns a strip of kStripTiles consecutive tiles of one slot.
// Slot constants (buffers, table, knot offsets of the 17 tile boundaries) are
// set up once per strip, lane-parallel; the new values at the tile boundary
// are carried in registers. Each tile's inputs -- its samples and the two
// envelopes' segment-table rows {x, y, m, 1/h} written by k_solve -- are
// contiguous in HBM and arrive by bulk (TMA-engine) copies issued by one lane,
// double-buffered per warp behind an mbarrier, so tile i+1 streams in while
// tile i is computed.
//
// Arithmetic contract: -fmad=false; spline_eval_fast is the reference
// expression bit-for-bit (div_rn = correctly rounded division, semd_device.cuh).
#include <cuda_runtime.h>

#include <cstdint>

#include "semd_device.cuh"
#include "semd_launch.h"
#include "semd_types.cuh"

namespace semd {
namespace dev {

// ------------------------------------------------------- global recomputation
// (rare paths: the two values before a strip in INIT mode, plateau runs that
// leave the lane's window)

struct EvalCtx {
    int mode, L, init_kind;
    const double* src;
    const double* x;  // EM_SPEC: the IMF input X (R' = X - new)
    const double* a;
    const double* b;
    double beta;
    TabView tv[2];
};

__device__ EvalCtx make_ctx(const Arena& A, int slot, int mode) {
    const Slot& sl = A.slots[slot];
    EvalCtx J;
    J.mode = mode;
    J.L = A.L;
    J.init_kind = sl.init_kind;
    J.a = sl.init_a;
    J.b = sl.init_b;
    J.beta = sl.beta;
    // the samples the pass reads: the candidate (SIFT, SPEC; DETECT of ST_REDETECT) or X
    const bool cand = (mode == EM_SIFT || mode == EM_SPEC || sl.state == ST_REDETECT) && sl.cb >= 0;
    J.src = A.bufs + buf_off(A, slot, cand ? sl.cb : sl.xb);
    J.x = A.bufs + buf_off(A, slot, sl.xb);
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        J.tv[s].tp = tab_planes(A, s, slot);
        J.tv[s].idx = A.kidx + knot_off(A, sl.par, s, slot);
        J.tv[s].n = (int)sl.n[s];
    }
    return J;
}

// new value at sample t from global data (reference formula)
__device__ double new_value_global(const EvalCtx& J, int t) {
    if (J.mode == EM_INIT) return J.init_kind == 1 ? J.a[t] + J.beta * J.b[t] : J.a[t];
    if (J.mode == EM_DETECT) return J.src[t];
    const double u = envelope_tab(J.tv[0], t);
    const double l = envelope_tab(J.tv[1], t);
    const double mean = 0.5 * (u + l);
    const double nv = J.src[t] - mean;
    return J.mode == EM_SPEC ? J.x[t] - nv : nv;  // EM_SPEC detects R' = X - new (emd.cpp:167)
}

__device__ __noinline__ double init_value(const Arena& A, int slot, int t) {
    return new_value_global(make_ctx(A, slot, EM_INIT), t);
}

// Extrema flags of one lane's detection sample t given the window values t0-2..t0+3
// (find_extrema, emd.cpp:16-33): the maximal run of samples exactly equal to v.
struct Win6 {
    double w[kSpt + 2];
};
__device__ __noinline__ unsigned plateau_flags(const Arena& A, int slot, int mode, int t, Win6 win, int t0, double v,
                                               int& ismin) {
    const EvalCtx J = make_ctx(A, slot, mode);
    auto val = [&](int u) -> double {
        const int li = u - (t0 - 2);
        if (li >= 0 && li < kSpt + 2 && u < J.L) return win.w[li];
        return new_value_global(J, u);
    };
    const int L = J.L;
    int rs = t, re = t;
    while (rs > 0 && val(rs - 1) == v) --rs;
    while (re < L - 1 && val(re + 1) == v) ++re;
    ismin = 0;
    if (rs > 0 && re < L - 1 && t == (rs + re) / 2) {
        const double lv = val(rs - 1), rv = val(re + 1);
        ismin = v < lv && v < rv;
        return v > lv && v > rv;
    }
    return 0;
}

// ------------------------------------------------------------- staging

constexpr int kWarpRows = kEvalTile / 2 + 6;  // table rows one tile can touch per side
// A stage holds one group of g consecutive tiles, laid out
//   samples [base-2, base + g*T)  |  g x 32 detection words (SIFT)  |  rows side 0  |  rows side 1
//   |  (SPEC: X [base-2, base + g*T))
// (one bulk copy each). SIFT groups take as many tiles (<= kGroupMax) as fit; one tile
// always fits (kWarpRows rows per side).
constexpr int kStageBytes = 6912;
constexpr int kGroupMax = 4;
struct alignas(16) WarpStage {
    double flat[kStageBytes / 8];
    unsigned long long bar;  // mbarrier: the group's bulk copies have landed
};
__host__ __device__ constexpr int group_bytes(int g, int rows, bool spec = false) {
    return (g * kEvalTile + 2) * 8 * (spec ? 2 : 1) + g * 32 * 4 + rows * 32;
}
static_assert(group_bytes(1, 2 * kWarpRows, true) <= kStageBytes, "one SPEC tile fits a stage");

constexpr int kStripTiles = 16;  // longest strip (A.strip tiles): consecutive tiles one warp walks

// Per-strip constants of one warp.
struct Strip {
    int slot, j0, nt, mode, par;
    double* dst;           // where new values go (INIT: X, SIFT: the candidate; DETECT: none)
    unsigned* nw;          // tflags words of tile j0 (parity of the new detection)
    unsigned* cnt0;        // scnt of tile j0, side 0 (side 1 at + A.G * tiles4)
    int to[2];             // lane l <= nt: knot offset (toff) of tile j0 + l, per side (SIFT)
};

// The global sources of a strip's bulk copies, only ever read by the lane that issues them.
// They live in the warp's shared memory, not in registers: held across the strip in registers
// they were spilled, and every group's copies then waited on local-memory reloads from L2.
struct alignas(16) CopySrc {
    const double* src;     // the samples this pass reads (SIFT, DETECT)
    const double* xsrc;    // SPEC: X
    const unsigned* ow;    // SIFT: tflags words of tile j0 (current knot parity)
    const double2* tab0;   // side-0 segment table, {x, y} plane ({m, 1/h} plane at + cap + 8)
    const double2* tab1;   // side-1 segment table
};

template <int ST>
__device__ __forceinline__ Strip strip_setup(const Arena& A, unsigned item, unsigned strips, CopySrc& cs) {
    const int lane = threadIdx.x & 31;
    Strip S;
    const unsigned sx = item % strips;
    S.slot = A.eval_list[item / strips];
    S.j0 = (int)sx * ST;
    S.nt = min(ST, A.tiles - S.j0);
    const Slot& sl = A.slots[S.slot];
    const int state = sl.state;
    S.mode = state == ST_INIT ? EM_INIT
           : (state == ST_DETECT || state == ST_REDETECT) ? EM_DETECT
           : state == ST_SIFT ? (sl.spec ? EM_SPEC : EM_SIFT)
                              : EM_NONE;
    const int cb = sl.cb, xb = sl.xb;
    S.par = sl.par;
    const bool sifting = S.mode == EM_SIFT || S.mode == EM_SPEC;
    S.dst = S.mode == EM_INIT ? A.bufs + buf_off(A, S.slot, xb)
                              : (sifting ? A.bufs + buf_off(A, S.slot, sl.db) : nullptr);
    if (lane == 0) {
        const bool cand = (sifting || state == ST_REDETECT) && cb >= 0;
        cs.src = A.bufs + buf_off(A, S.slot, cand ? cb : xb);
        cs.xsrc = A.bufs + buf_off(A, S.slot, xb);
        cs.tab0 = tab_planes(A, 0, S.slot).a;
        cs.tab1 = tab_planes(A, 1, S.slot).a;
        cs.ow = A.tflags + tfl_off(A, S.par, S.slot) + (size_t)S.j0 * 32;
    }
    S.nw = A.tflags + tfl_off(A, 1 - S.par, S.slot) + (size_t)S.j0 * 32;
    S.cnt0 = A.scnt + scnt_off(A, 0, S.slot) + S.j0;
    S.to[0] = S.to[1] = 0;
    if (sifting) {
        const int j = S.j0 + min(lane, S.nt);
#pragma unroll
        for (int s = 0; s < 2; ++s) S.to[s] = (int)toff_view(A, sl.par, s, S.slot)[j];
    }
    return S;
}

// The next strip, set up during the current strip's last group (its first bulk copy issued into
// the free stage), parked in shared memory so it does not hold registers meanwhile.
struct alignas(16) StripStash {
    int to[2][32];
    int slot, mode, par, dstb, g, pad[3];
};
template <int ST>
__device__ __forceinline__ void stash_strip(const Arena& A, const Strip& S, int g, StripStash& st) {
    const int lane = threadIdx.x & 31;
    st.to[0][lane] = S.to[0];
    st.to[1][lane] = S.to[1];
    if (lane == 0) {
        const Slot& sl = A.slots[S.slot];
        st.slot = S.slot;
        st.mode = S.mode;
        st.par = S.par;
        st.dstb = S.mode == EM_INIT ? sl.xb : sl.db;
        st.g = g;
    }
    __syncwarp();
}
template <int ST>
__device__ __forceinline__ Strip strip_from(const Arena& A, unsigned item, unsigned strips, const StripStash& st) {
    const int lane = threadIdx.x & 31;
    Strip S;
    S.slot = st.slot;
    S.j0 = (int)(item % strips) * ST;
    S.nt = min(ST, A.tiles - S.j0);
    S.mode = st.mode;
    S.par = st.par;
    S.dst = S.mode == EM_DETECT ? nullptr : A.bufs + buf_off(A, S.slot, st.dstb);

    S.nw = A.tflags + tfl_off(A, 1 - S.par, S.slot) + (size_t)S.j0 * 32;
    S.cnt0 = A.scnt + scnt_off(A, 0, S.slot) + S.j0;
    S.to[0] = st.to[0][lane];
    S.to[1] = st.to[1][lane];
    return S;
}

// SIFT group of tiles i .. i+g-1: as many tiles (<= kGroupMax, <= the strip) as fit a stage.
// Tile j's extrema are those of window [base-1, base+T-1); its samples [base-2, base+T) need
// table rows [toff[j], toff[j+1]+2], so the group needs rows [toff[j_i], toff[j_i+g]+2].
__device__ __forceinline__ int group_tiles(const Strip& S, int i) {
    // lane l holds toff of tile j0 + min(l, nt): it rates the group of c = l - i tiles i .. l-1
    // (bytes grow with c, so the largest fitting c is the highest lane that fits; c = 1 always does)
    const int lane = threadIdx.x & 31;
    const int lo0 = __shfl_sync(0xffffffffu, S.to[0], i), lo1 = __shfl_sync(0xffffffffu, S.to[1], i);
    const int c = lane - i;
    const int rows = S.to[0] - lo0 + S.to[1] - lo1 + 6;
    const bool fit = c >= 1 && c <= kGroupMax && lane <= S.nt &&
                     (c == 1 || group_bytes(c, rows, S.mode == EM_SPEC) <= kStageBytes);
    return 31 - __clz((int)__ballot_sync(0xffffffffu, fit)) - i;
}

// One lane of the converged warp (elect.sync: the compiler then knows the region is single-lane).
__device__ __forceinline__ bool elect_one() {
    unsigned pred;
    asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(pred));
    return pred != 0;
}

// Issue group (i, g)'s copies: samples, detection words, both sides' rows (lane 0 arms the barrier).
__device__ __forceinline__ void issue_group(const Strip& S, int i, int g, WarpStage& st, int bofs,
                                            const CopySrc& cs) {
    const int lo0 = __shfl_sync(0xffffffffu, S.to[0], i), lo1 = __shfl_sync(0xffffffffu, S.to[1], i);
    const int n0 = __shfl_sync(0xffffffffu, S.to[0], i + g) + 3 - lo0;
    const int n1 = __shfl_sync(0xffffffffu, S.to[1], i + g) + 3 - lo1;
    if (!elect_one()) return;  // one lane issues (every operand is warp-uniform)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of the stage
    const int base = (S.j0 + i) * kEvalTile;
    const int e0 = base > 0 ? base - 2 : 0;  // 16-byte aligned; Lp = whole tiles
    const unsigned sb = (unsigned)(base + g * kEvalTile - e0) * 8u;
    const bool spec = S.mode == EM_SPEC;
    double* f = st.flat;
    unsigned* ow = reinterpret_cast<unsigned*>(f + g * kEvalTile + 2);
    double2* r0 = reinterpret_cast<double2*>(ow + g * 32);  // {x,y} side 0 | side 1, then {m,1/h} side 0 | side 1
    const CopySrc c = cs;
    bar_arrive_tx(&st.bar, sb * (spec ? 2u : 1u) + (unsigned)g * 128u + (unsigned)(n0 + n1) * 32u);
    bulk_g2s(f + (e0 - (base - 2)), c.src + e0, sb, &st.bar);
    if (spec) bulk_g2s(reinterpret_cast<double*>(r0 + 2 * (n0 + n1)) + (e0 - (base - 2)), c.xsrc + e0, sb, &st.bar);
    bulk_g2s(ow, c.ow + i * 32, (unsigned)g * 128u, &st.bar);
    bulk_g2s(r0, c.tab0 + lo0, (unsigned)n0 * 16u, &st.bar);
    bulk_g2s(r0 + n0, c.tab1 + lo1, (unsigned)n1 * 16u, &st.bar);
    bulk_g2s(r0 + n0 + n1, c.tab0 + bofs + lo0, (unsigned)n0 * 16u, &st.bar);
    bulk_g2s(r0 + 2 * n0 + n1, c.tab1 + bofs + lo1, (unsigned)n1 * 16u, &st.bar);
}

// DETECT passes stream samples only: the stage's row area holds kDetChunk tiles, so one bulk
// copy (staged from the chunk's base - 2) feeds kDetChunk tiles and the per-tile copy latency
// is amortised.
constexpr int kDetChunk = 6;
static_assert((kDetChunk * kEvalTile + 2) * 8 <= kStageBytes, "a DETECT chunk fits one stage");
__device__ __forceinline__ double* stage_flat(WarpStage& st) { return st.flat; }
__device__ __forceinline__ void issue_chunk(const Strip& S, int c, WarpStage& st, const CopySrc& cs) {
    if (!elect_one()) return;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of the stage
    const int base = (S.j0 + c * kDetChunk) * kEvalTile;
    const int end = (S.j0 + min(S.nt, (c + 1) * kDetChunk)) * kEvalTile;  // <= Lp (whole tiles)
    const int e0 = base > 0 ? base - 2 : 0;                                 // 16-byte aligned
    const unsigned sb = (unsigned)(end - e0) * 8u;
    bar_arrive_tx(&st.bar, sb);
    bulk_g2s(stage_flat(st) + (e0 - (base - 2)), cs.src + e0, sb, &st.bar);
}

__device__ __forceinline__ int smem_search(const double2* R, int hi, double t) {  // last q <= hi with x_q < t
    int lo = 0;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (R[mid].x < t) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// ---------------------------------------------------------------- one tile
// kSpt = 4 consecutive samples per lane; c2/c1 carry the new values at base-2/base-1.
// Interior: the whole tile and its detection windows lie inside [1, L-2] (every tile but the
// first and the last of a slot) -- no per-sample bound checks.
// SPEC (a speculative last sift): as SIFT, and also R' = X - new (emd.cpp:167) from the staged X
// (xsamp, aligned like samp) into S.rdst; the extrema detected are R''s, not new's.
template <bool Interior, int M>
__device__ __forceinline__ void eval_tile(const Arena& A, const Strip& S, int i, const double* samp,
                                          const unsigned* ows, const double2* R0, const double2* R1, int nab, double& c2,
                                          double& c1, double& snum, double& sden, const double* xsamp = nullptr) {
    const int lane = threadIdx.x & 31;
    constexpr int mode = M;  // the pass's mode (each loop instantiates its own)
    const bool spec = mode == EM_SIFT && xsamp != nullptr;  // a speculative last sift (warp-uniform)
    const int L = A.L;
    const int j = S.j0 + i;
    const int base = j * kEvalTile;
    const int t0 = base + lane * kSpt;
    int qmax[2] = {0, 0};
    if (mode == EM_SIFT) {
#pragma unroll
        for (int s = 0; s < 2; ++s)
            qmax[s] = __shfl_sync(0xffffffffu, S.to[s], i + 1) + 1 - __shfl_sync(0xffffffffu, S.to[s], i);
    }
    if (i == 0 && base > 0) {  // strip start: the new values at base-2, base-1 (staged rows cover them)
        double cc[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int t = base - 2 + u;
            if (mode == EM_INIT) {
                cc[u] = init_value(A, S.slot, t);
            } else if (mode == EM_DETECT) {
                cc[u] = samp[u];
            } else {
                const double tt = (double)t;
                double e[2];
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const double2* R = s ? R1 : R0;
                    // rows 0 and 1 are the two knots before the tile's detection window [base-1, ..):
                    // x_1 <= base-2 and x_2 >= base-1, so the last row with x < t is row 1, or row 0
                    // when t = base-2 sits on knot 1 (what the search over the staged rows returns)
                    const int qq = R[1].x < tt ? 1 : 0;
                    SEMD_ASSERT(qq == smem_search(R, qmax[s], tt));
                    const double2 a0 = R[qq], b0 = R[nab + qq], a1 = R[qq + 1];
                    const double m1 = R[nab + qq + 1].x;
                    const double h = a1.x - a0.x;
                    e[s] = spline_eval_fast(a0.x, a1.x, a0.y, a1.y, b0.x, m1, h, b0.y, h * h, tt);
                }
                cc[u] = samp[u] - 0.5 * (e[0] + e[1]);
                if (spec) cc[u] = xsamp[u] - cc[u];
            }
        }
        c2 = cc[0];
        c1 = cc[1];
    }
    double cv[kSpt];
    if (mode == EM_INIT) {
        const Slot& sl = A.slots[S.slot];
        const double* a = sl.init_a;
        const double* b = sl.init_b;
        const double beta = sl.beta;
        const int kind = sl.init_kind;
#pragma unroll
        for (int k = 0; k < kSpt; ++k) {
            const int t = t0 + k;
            cv[k] = t < L ? (kind == 1 ? a[t] + beta * b[t] : a[t]) : 0.0;
        }
    } else {
        const double* sp = samp + 2 + lane * kSpt;
#pragma unroll
        for (int k = 0; k < kSpt; k += 2) {
            const double2 v = *reinterpret_cast<const double2*>(sp + k);
            cv[k] = Interior || t0 + k < L ? v.x : 0.0;
            cv[k + 1] = Interior || t0 + k + 1 < L ? v.y : 0.0;
        }
    }

    double nv[kSpt];
    if (mode == EM_SIFT) {
        // seg(t) = last staged row q with x_q < t (the reference's march, emd.cpp:79). Rows 0-1
        // precede the tile's detection window and rows 2.. are its extrema in order, so
        // seg(t) = 1 + #(window extrema at positions < t): the previous detection stored, per
        // lane, its flags for window positions t0-1 .. t0+2 and its rank among the tile's
        // extrema of each side; each further sample adds the extrema it passes.
        const unsigned ow = ows[lane];
        double env0[kSpt];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const double2* R = s ? R1 : R0;
            const unsigned fl = (ow >> (4 * s)) & 0xFu;  // window positions t0-1 .. t0+2
            const int q0 = 1 + (int)((ow >> (8 + 8 * s)) & 0xFFu) + (int)(fl & 1u);
#pragma unroll
            for (int k = 0; k < kSpt; ++k) {
                const double tt = (double)(t0 + k);
                const int q = q0 + __popc((fl >> 1) & ((1u << k) - 1u));
                SEMD_ASSERT(q >= 0 && q <= qmax[s]);  // the tile's staged rows (k_solve's table, toff)
                const double2 a0 = R[q], b0 = R[nab + q], a1 = R[q + 1];
                const double m1 = R[nab + q + 1].x;
                const double h = a1.x - a0.x;
                const double e = spline_eval_fast(a0.x, a1.x, a0.y, a1.y, b0.x, m1, h, b0.y, h * h, tt);
                if (s == 0) {
                    env0[k] = e;
                } else {
                    const double mean = 0.5 * (env0[k] + e);  // emd.cpp:144-147
                    if (Interior || t0 + k < L) {
                        snum += mean * mean;
                        sden += cv[k] * cv[k];
                        nv[k] = cv[k] - mean;
                    } else {
                        nv[k] = 0.0;
                    }
                }
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < kSpt; ++k) nv[k] = cv[k];
    }
    if (S.dst) {
        if (Interior || t0 + kSpt <= L) {
#pragma unroll
            for (int k = 0; k < kSpt; k += 2)
                __stcs(reinterpret_cast<double2*>(S.dst + t0 + k), make_double2(nv[k], nv[k + 1]));
        } else {
            for (int k = 0; k < kSpt; ++k)
                if (t0 + k < L) S.dst[t0 + k] = nv[k];
        }
    }
    if (spec) {  // R' = X - new (emd.cpp:167); the detection below runs on R'
        // (R''s buffer is looked up per tile rather than held in a register across the strip)
        double* const rdst = A.bufs + buf_off(A, S.slot, __ldg(&A.slots[S.slot].rb));
        const double* xp = xsamp + 2 + lane * kSpt;
#pragma unroll
        for (int k = 0; k < kSpt; k += 2) {
            const double2 v = *reinterpret_cast<const double2*>(xp + k);
            nv[k] = Interior || t0 + k < L ? v.x - nv[k] : 0.0;
            nv[k + 1] = Interior || t0 + k + 1 < L ? v.y - nv[k + 1] : 0.0;
        }
        if (Interior || t0 + kSpt <= L) {
#pragma unroll
            for (int k = 0; k < kSpt; k += 2)
                __stcs(reinterpret_cast<double2*>(rdst + t0 + k), make_double2(nv[k], nv[k + 1]));
        } else {
            for (int k = 0; k < kSpt; ++k)
                if (t0 + k < L) rdst[t0 + k] = nv[k];
        }
    }
    // detection window t0-1 .. t0+2 needs values t0-2 .. t0+3
    // One rotation by a lane serves both the window's left values (lane l takes lane l-1's last two
    // values) and the carry across tiles: lane 31 sends its last two values of the PREVIOUS tile
    // (c2, c1: each lane keeps its own), which lane 0 -- the only reader of lane 31 -- needs.
    double w[kSpt + 2];
    const int from = (lane + 31) & 31;
    w[0] = __shfl_sync(0xffffffffu, lane == 31 ? c2 : nv[kSpt - 2], from);
    w[1] = __shfl_sync(0xffffffffu, lane == 31 ? c1 : nv[kSpt - 1], from);
#pragma unroll
    for (int k = 0; k < kSpt; ++k) w[k + 2] = nv[k];
    c2 = nv[kSpt - 2];  // (lane 31's: the values at base+T-2, base+T-1 for the next tile of the strip)
    c1 = nv[kSpt - 1];

    // extrema flags branch-free (find_extrema, emd.cpp:16-33); samples equal to a neighbour
    // take the reference's plateau rule in a warp-uniform slow path
    // Each neighbour pair (w[j], w[j+1]) is compared once (up: w[j+1] > w[j], dn: w[j+1] < w[j])
    // and shared by the two samples it borders: v > r of sample k is dn of pair k+1. Equality is
    // "neither up nor dn"; a NaN neighbour lands in the plateau path, which compares exactly.
    unsigned up = 0, dn = 0;
#pragma unroll
    for (int j = 0; j <= kSpt; ++j) {
        up |= (unsigned)(w[j + 1] > w[j]) << j;
        dn |= (unsigned)(w[j + 1] < w[j]) << j;
    }
    unsigned inm = (1u << kSpt) - 1u;
    if (!Interior) {
        inm = 0;
#pragma unroll
        for (int k = 0; k < kSpt; ++k) {
            const int t = t0 - 1 + k;
            inm |= (unsigned)(t >= 1 && t <= L - 2) << k;
        }
    }
    const unsigned eq = ~(up | dn);  // bit j: w[j+1] == w[j] (or unordered)
    unsigned fmax = up & (dn >> 1) & inm;  // v > l (up_k) and v > r (dn_{k+1})
    unsigned fmin = dn & (up >> 1) & inm;  // v < l (dn_k) and v < r (up_{k+1})
    const unsigned plat = (eq | (eq >> 1)) & inm;  // v == l or v == r
    if (__any_sync(0xffffffffu, plat != 0u)) {
        for (int k = 0; k < kSpt; ++k) {
            if (!(plat & (1u << k))) continue;
            int mn;
            Win6 win;
#pragma unroll
            for (int z = 0; z < kSpt + 2; ++z) win.w[z] = w[z];
            if (plateau_flags(A, S.slot, spec ? EM_SPEC : mode, t0 - 1 + k, win, t0, w[k + 1], mn)) fmax |= 1u << k;
            if (mn) fmin |= 1u << k;
        }
    }

    // tile-local ranks: with the flags they are the tile's ordered extrema lists, expanded into
    // the knot lists by k_compact and read back by the next sift. A lane holds at most 2 extrema
    // of a side (no two maxima or minima are adjacent), so the exclusive prefix of the per-lane
    // counts is two ballots per side (count bits 0 and 1) instead of a shuffle scan.
    const unsigned nmax = (unsigned)__popc(fmax), nmin = (unsigned)__popc(fmin);
    const unsigned a0 = __ballot_sync(0xffffffffu, nmax & 1u), a1 = __ballot_sync(0xffffffffu, nmax >> 1);
    const unsigned b0 = __ballot_sync(0xffffffffu, nmin & 1u), b1 = __ballot_sync(0xffffffffu, nmin >> 1);
    const unsigned lt = (1u << lane) - 1u;
    const unsigned emax = (unsigned)__popc(a0 & lt) + 2u * (unsigned)__popc(a1 & lt);
    const unsigned emin = (unsigned)__popc(b0 & lt) + 2u * (unsigned)__popc(b1 & lt);
    S.nw[i * 32 + lane] = fmax | (fmin << 4) | (emax << 8) | (emin << 16);
    if (lane == 0) {
        S.cnt0[i] = (unsigned)__popc(a0) + 2u * (unsigned)__popc(a1);
        S.cnt0[i + (size_t)A.G * tiles4(A)] = (unsigned)__popc(b0) + 2u * (unsigned)__popc(b1);
    }
}

// Warp-level software pipeline over two stages: a group of tiles (SIFT) or a chunk (DETECT) is
// computed while the next one's bulk copies are in flight; during a strip's last group the next
// strip is set up and its first copy issued. SD partials are summed per lane over the strip and
// reduced once per strip (tnum/tden are indexed by strip).

// ST: tiles per strip (A.strip), a compile-time constant of each instantiation
template <int ST>
__global__ void __launch_bounds__(kEvalThreads, 2) k_eval(Arena A) {
    pdl_begin();
    if (A.ctrl->finished) return;  // a step launched past the run's end
    extern __shared__ __align__(16) unsigned char eval_smem[];
    const int kstep_ = A.ctrl->step;
    if (threadIdx.x == 0) {
        atomicMin(&A.ctrl->ev_t0, gtimer());
        span_begin(A.ctrl, KID_EVAL);
    }
    const int lane = threadIdx.x & 31;
    WarpStage* stage = reinterpret_cast<WarpStage*>(eval_smem) + 2 * (threadIdx.x >> 5);
    const unsigned strips = ((unsigned)A.tiles + ST - 1) / ST;
    const unsigned nstrips = (unsigned)A.ctrl->n_eval_pass * strips;  // ST_PRIMED slots have no pass
    if (lane == 0) {
        bar_init(&stage[0].bar);
        bar_init(&stage[1].bar);
    }
    __syncwarp();
    unsigned phase = 0;  // bit b: parity of stage b's next completion
    int b = 0;           // stage of the next tile
    // dynamic strip tickets (C->ticket[0], reset by k_scan): a CTA that starts late -- e.g.
    // next to the noise generator on the side stream -- just takes fewer strips. The next
    // ticket is fetched one strip ahead.
    unsigned* tk = &A.ctrl->ticket[0];
    unsigned item = 0, next = 0;
    if (lane == 0) item = atomicAdd(tk, 1u);
    item = __shfl_sync(0xffffffffu, item, 0);
    StripStash& stash = reinterpret_cast<StripStash*>(reinterpret_cast<WarpStage*>(eval_smem) +
                                                      2 * (kEvalThreads / 32))[threadIdx.x >> 5];
    CopySrc* csrc = reinterpret_cast<CopySrc*>(reinterpret_cast<StripStash*>(reinterpret_cast<WarpStage*>(eval_smem) +
                                                                            2 * (kEvalThreads / 32)) +
                                               kEvalThreads / 32) +
                    2 * (threadIdx.x >> 5);  // [2] per warp: this strip's and the prefetched one's
    int ci = 0;
    bool pre = false;  // this strip was set up (and its first copy issued) by the previous one
    while (item < nstrips) {
        if (lane == 0) next = atomicAdd(tk, 1u);
        const Strip S = pre ? strip_from<ST>(A, item, strips, stash) : strip_setup<ST>(A, item, strips, csrc[ci]);
        __syncwarp();  // csrc[ci] written by lane 0
        const int g_pre = pre ? stash.g : 0;
        bool pre_next = false;
        // during this strip's last group: set up the next strip and issue its first copy into
        // the free stage (SIFT / DETECT strips; INIT strips stage nothing)
        auto prefetch_next = [&](int fb) {
            const unsigned nx = __shfl_sync(0xffffffffu, next, 0);
            if (nx >= nstrips) return;
            const Strip S2 = strip_setup<ST>(A, nx, strips, csrc[ci ^ 1]);
            if (S2.mode == EM_INIT || S2.mode == EM_NONE) return;
            __syncwarp();
            int g2 = 0;
            if (S2.mode == EM_SIFT || S2.mode == EM_SPEC) {
                g2 = group_tiles(S2, 0);
                issue_group(S2, 0, g2, stage[fb], A.cap + 8, csrc[ci ^ 1]);
            } else {
                issue_chunk(S2, 0, stage[fb], csrc[ci ^ 1]);
            }
            stash_strip<ST>(A, S2, g2, stash);
            pre_next = true;
        };
        const long long cyc0 = clock64();
        double c2 = 0.0, c1 = 0.0, snum = 0.0, sden = 0.0;
        if (S.mode == EM_DETECT) {
            const int nch = (S.nt + kDetChunk - 1) / kDetChunk;
            if (!pre) issue_chunk(S, 0, stage[b], csrc[ci]);
            for (int c = 0; c < nch; ++c) {
                if (c + 1 < nch) issue_chunk(S, c + 1, stage[b ^ 1], csrc[ci]);
                else prefetch_next(b ^ 1);
                bar_wait(&stage[b].bar, (phase >> b) & 1u);
                phase ^= 1u << b;
                const double* flat = stage_flat(stage[b]);
                const int i1 = min(S.nt, (c + 1) * kDetChunk);
                for (int i = c * kDetChunk; i < i1; ++i) {
                    const int base = (S.j0 + i) * kEvalTile;
                    const double* sp = flat + (i - c * kDetChunk) * kEvalTile;
                    if (base >= kEvalTile && base + 2 * kEvalTile <= A.L)
                        eval_tile<true, EM_DETECT>(A, S, i, sp, nullptr, nullptr, nullptr, 0, c2, c1, snum, sden);
                    else
                        eval_tile<false, EM_DETECT>(A, S, i, sp, nullptr, nullptr, nullptr, 0, c2, c1, snum, sden);
                }
                __syncwarp();  // stage b is refilled next
                b ^= 1;
            }
        } else if (S.mode == EM_SIFT || S.mode == EM_SPEC) {
            const bool spec = S.mode == EM_SPEC;
            int g = pre ? g_pre : group_tiles(S, 0);
            if (!pre) issue_group(S, 0, g, stage[b], A.cap + 8, csrc[ci]);
            for (int i = 0; i < S.nt;) {
                const int gn = i + g < S.nt ? group_tiles(S, i + g) : 0;
                if (gn) issue_group(S, i + g, gn, stage[b ^ 1], A.cap + 8, csrc[ci]);
                else prefetch_next(b ^ 1);
                bar_wait(&stage[b].bar, (phase >> b) & 1u);
                phase ^= 1u << b;
                const double* flat = stage_flat(stage[b]);
                const unsigned* ows = reinterpret_cast<const unsigned*>(flat + g * kEvalTile + 2);
                const double2* R0 = reinterpret_cast<const double2*>(ows + g * 32);
                const int lo0 = __shfl_sync(0xffffffffu, S.to[0], i), lo1 = __shfl_sync(0xffffffffu, S.to[1], i);
                const int n0 = __shfl_sync(0xffffffffu, S.to[0], i + g) + 3 - lo0;
                const double2* R1 = R0 + n0;
                const int nab = n0 + __shfl_sync(0xffffffffu, S.to[1], i + g) + 3 - lo1;  // rows of both sides
                for (int u = 0; u < g; ++u) {
                    const int t = i + u;
                    const int base = (S.j0 + t) * kEvalTile;
                    const double2* T0 = R0 + (__shfl_sync(0xffffffffu, S.to[0], t) - lo0);
                    const double2* T1 = R1 + (__shfl_sync(0xffffffffu, S.to[1], t) - lo1);
                    const double* sp = flat + u * kEvalTile;
                    const double* xp = spec ? reinterpret_cast<const double*>(R0 + 2 * nab) + u * kEvalTile : nullptr;
                    if (base >= kEvalTile && base + 2 * kEvalTile <= A.L)
                        eval_tile<true, EM_SIFT>(A, S, t, sp, ows + u * 32, T0, T1, nab, c2, c1, snum, sden, xp);
                    else
                        eval_tile<false, EM_SIFT>(A, S, t, sp, ows + u * 32, T0, T1, nab, c2, c1, snum, sden, xp);
                }
                __syncwarp();  // stage b is refilled next
                b ^= 1;
                i += g;
                g = gn;
            }
        } else if (S.mode == EM_INIT) {  // values computed from the job's inputs, nothing staged
            for (int i = 0; i < S.nt; ++i)
                eval_tile<false, EM_INIT>(A, S, i, nullptr, nullptr, nullptr, nullptr, 0, c2, c1, snum, sden);
        }
        if (S.mode == EM_SIFT || S.mode == EM_SPEC) {
            snum = warp_sum(snum);
            sden = warp_sum(sden);
            if (lane == 0) {
                A.tnum[tsd_off(A, S.slot) + S.j0 / ST] = snum;
                A.tden[tsd_off(A, S.slot) + S.j0 / ST] = sden;
            }
        }
        if (lane == 0) {
            const int sx = S.mode == EM_SIFT || S.mode == EM_SPEC;
            atomicAdd(&A.ctrl->strips[sx], 1ull);
            atomicAdd(&A.ctrl->strip_cyc[sx], (unsigned long long)(clock64() - cyc0));
        }
        item = __shfl_sync(0xffffffffu, next, 0);
        pre = pre_next;
        if (pre_next) ci ^= 1;  // the prefetched strip's copy sources are in the other slot
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicMax(&A.ctrl->ev_t1, gtimer());
        span_end(A.ctrl, KID_EVAL, kstep_);
    }
}

size_t eval_smem_bytes() {
    return (sizeof(WarpStage) * 2 + sizeof(StripStash) + 2 * sizeof(CopySrc)) * (kEvalThreads / 32);
}
cudaError_t eval_setup() {
    const cudaError_t e = cudaFuncSetAttribute(k_eval<kStripTiles>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)eval_smem_bytes());
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_eval<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)eval_smem_bytes());
}

void launch_eval(const Arena& A, int sms, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(sms * 2));
    cfg.blockDim = dim3((unsigned)kEvalThreads);
    cfg.dynamicSmemBytes = eval_smem_bytes();
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (A.strip == 4)
        cudaLaunchKernelEx(&cfg, k_eval<4>, A);
    else
        cudaLaunchKernelEx(&cfg, k_eval<kStripTiles>, A);
}

}  // namespace dev
}  // namespace semd
