// semd_kernels.cu -- sm_100a kernels of the serial-EMD sift engine.
//
// Reference behaviour being reproduced (paths relative to /root/reference/proj):
//   find_extrema        src/emd.cpp:10-35   -> k_eval detection + ordered compaction
//   envelope / spline   src/emd.cpp:41-125  -> k_solve (moments) + k_eval (evaluation)
//   extract_imf         src/emd.cpp:127-153 -> k_eval subtract + SD partials, decide1
//   emd residue update  src/emd.cpp:167     -> k_final
//   eemd accumulation   src/emd.cpp:246-251 -> k_final (realization order within a step)
//   white_noise         src/emd.cpp:181-200 -> k_mt19937_64 + k_box_muller
//
// Arithmetic contract: this translation unit is compiled with -fmad=false so
// that every expression that mirrors the reference rounds exactly like the
// reference's -ffp-contract=off build; all spline / sift arithmetic is
// bit-identical to the CPU reference. The only non-bitwise parts are the
// SD-criterion sums (a deterministic tree reduction instead of a sequential
// sum; they only feed the stop comparison) and libm log/sin/cos in the noise.
#include <cuda_runtime.h>

#include <cstdint>

#include "semd_launch.h"
#include "semd_types.cuh"

namespace semd {
namespace dev {

// ------------------------------------------------------------------ helpers

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t knot_hash(int side, uint32_t rank, uint32_t idx) {
    return mix64((side ? 0x8000000000000000ULL : 0ULL) ^ ((uint64_t)rank << 32) ^ (uint64_t)idx);
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// emd.cpp:80-85: one natural-spline segment evaluated at tt (same operation order).
__device__ __forceinline__ double spline_eval(double x0, double x1, double y0, double y1, double m0, double m1,
                                              double tt) {
    const double h = x1 - x0;
    const double a = (x1 - tt) / h;
    const double b = (tt - x0) / h;
    return a * y0 + b * y1 + ((a * a * a - a) * m0 + (b * b * b - b) * m1) * (h * h) / 6.0;
}

// Mirrored knot v of a sift envelope (emd.cpp:107-122; both mirrors present in
// sifting because extrema never sit on an end): v=0,1 left mirrors, 2..n+1
// the extrema, n+2 and n+3 the (non-monotone) right mirrors.
struct KnotView {
    const int* idx;
    const double* val;
    const double* mom;
    int n;
    double e2;  // 2*(L-1)
};

__device__ __forceinline__ void vknot(const KnotView& kv, int v, double& X, double& Y) {
    const int n = kv.n;
    int r;
    if (v == 0) {
        r = 1;
        X = -(double)kv.idx[r];
    } else if (v == 1) {
        r = 0;
        X = -(double)kv.idx[r];
    } else if (v <= n + 1) {
        r = v - 2;
        X = (double)kv.idx[r];
    } else {
        r = (v == n + 2) ? n - 2 : n - 1;
        X = kv.e2 - (double)kv.idx[r];
    }
    Y = kv.val[r];
}

// Envelope value at sample t from global knots (slow path: plateau runs that
// leave the tile halo). seg = 1 + #{idx < t} (the reference's segment march).
__device__ double envelope_at_global(const KnotView& kv, int t) {
    int lo = 0, hi = kv.n;  // count of idx < t
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (kv.idx[mid] < t) lo = mid + 1;
        else hi = mid;
    }
    const int seg = 1 + lo;
    double x0, y0, x1, y1;
    vknot(kv, seg, x0, y0);
    vknot(kv, seg + 1, x1, y1);
    return spline_eval(x0, x1, y0, y1, kv.mom[seg], kv.mom[seg + 1], (double)t);
}

struct TileJob {
    int slot, mode, L;
    const double* src;  // current signal (EM_DETECT / EM_SIFT)
    const double* a;    // EM_INIT inputs
    const double* b;
    double beta;
    int init_kind;
    KnotView kv[2];
};

// The value the tile job produces at sample t (identical arithmetic to the
// fast path; used for plateau runs that extend past the tile halo).
__device__ double new_value_at(const TileJob& J, int t) {
    if (J.mode == EM_INIT) return J.init_kind == 1 ? J.a[t] + J.beta * J.b[t] : J.a[t];
    if (J.mode == EM_DETECT) return J.src[t];
    const double u = envelope_at_global(J.kv[0], t);
    const double l = envelope_at_global(J.kv[1], t);
    const double mean = 0.5 * (u + l);
    return J.src[t] - mean;
}

// ---------------------------------------------------------- block utilities

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block reduction of two doubles (fixed tree order).
__device__ void block_sum2(double& a, double& b, double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    a = warp_sum(a);
    b = warp_sum(b);
    __syncthreads();
    if (lane == 0) {
        red[wid] = a;
        red[32 + wid] = b;
    }
    __syncthreads();
    if (wid == 0) {
        a = lane < nw ? red[lane] : 0.0;
        b = lane < nw ? red[32 + lane] : 0.0;
        a = warp_sum(a);
        b = warp_sum(b);
    }
}

// Decoupled look-back over the tiles of one slot (one warp). Returns the
// exclusive prefix of `agg` for tile j. Status word: epoch<<32 | flag<<30 | value.
__device__ unsigned lookback(unsigned long long* status, int j, unsigned epoch, unsigned agg) {
    const int lane = threadIdx.x & 31;
    const unsigned long long ep = (unsigned long long)epoch << 32;
    if (j == 0) {
        if (lane == 0) st_volatile_u64(&status[0], ep | (2ULL << 30) | agg);
        return 0;
    }
    if (lane == 0) st_volatile_u64(&status[j], ep | (1ULL << 30) | agg);
    unsigned excl = 0;
    int look = j - 1;
    while (true) {
        const int idx = look - lane;
        unsigned long long w = 0;
        unsigned flag = 2, val = 0;
        if (idx >= 0) {
            do {
                w = ld_volatile_u64(&status[idx]);
            } while ((w >> 32) != epoch || ((w >> 30) & 3ULL) == 0);
            flag = (unsigned)((w >> 30) & 3ULL);
            val = (unsigned)(w & 0x3FFFFFFFULL);
        }
        // idx < 0 behaves as an inclusive prefix of 0 (flag 2, val 0)
        const unsigned incl_mask = __ballot_sync(0xffffffffu, flag == 2);
        if (incl_mask) {
            const int pos = __ffs(incl_mask) - 1;
            unsigned contrib = lane <= pos ? val : 0;
            excl += warp_sum(contrib);
            break;
        }
        excl += warp_sum(val);
        look -= 32;
    }
    if (lane == 0) st_volatile_u64(&status[j], ep | (2ULL << 30) | (excl + agg));
    return excl;
}

// ------------------------------------------------------------ eval kernel
//
// One work item = one tile of one slot. Modes:
//   EM_INIT   X[t] = a[t] (+ beta*b[t]) written to buffer xb, then detect
//   EM_DETECT detect extrema of X (first find_extrema of an IMF)
//   EM_SIFT   new = cur - 0.5*(upper+lower) (emd.cpp:143-147) written to db,
//             SD partials, then detect extrema of `new` for the next sift
// Detection + compaction reproduce find_extrema exactly (ordered lists).

struct EvalShared {
    unsigned ticket;
    int last;
    unsigned scan[kEvalThreads / 32];
    unsigned gbase[2];
    double red[64];
};

__device__ void eval_tile(const Arena& A, int slot, int j, double* sv, double* nv, double* kX, double* kY,
                          double* kM, EvalShared& sh) {
    const int tid = threadIdx.x;
    const Slot& S = A.slots[slot];
    const int L = A.L;
    const int state = S.state;
    TileJob J;
    J.slot = slot;
    J.L = L;
    J.mode = state == ST_INIT ? EM_INIT : (state == ST_DETECT ? EM_DETECT : EM_SIFT);
    J.a = S.init_a;
    J.b = S.init_b;
    J.beta = S.beta;
    J.init_kind = S.init_kind;
    double* bufs = A.bufs;
    const int xb = S.xb, cb = S.cb;
    J.src = bufs + buf_off(A, slot, (J.mode == EM_SIFT && cb >= 0) ? cb : xb);
    double* dst = nullptr;
    if (J.mode == EM_INIT) dst = bufs + buf_off(A, slot, xb);
    if (J.mode == EM_SIFT) dst = bufs + buf_off(A, slot, S.db);
    const int par = S.par;
    const double e2 = 2.0 * (double)(L - 1);
    for (int s = 0; s < 2; ++s) {
        J.kv[s].idx = A.kidx + knot_off(A, par, s, slot);
        J.kv[s].val = A.kval + knot_off(A, par, s, slot);
        J.kv[s].mom = A.mom + mom_off(A, s, slot);
        J.kv[s].n = (int)S.n[s];
        J.kv[s].e2 = e2;
    }

    const int base = j * kEvalTile;
    const int tlen = min(kEvalTile, L - base);

    // 1. stage the source values (tile + one halo sample each side)
    for (int i = tid; i < kEvalTile + 2; i += kEvalThreads) {
        const int t = base - 1 + i;
        double v = 0.0;
        if (t >= 0 && t < L && i <= tlen + 1) {
            if (J.mode == EM_INIT) v = J.init_kind == 1 ? J.a[t] + J.beta * J.b[t] : J.a[t];
            else v = J.src[t];
        }
        sv[i] = v;
    }
    int vlo[2] = {0, 0}, vcnt[2] = {0, 0};
    if (J.mode == EM_SIFT) {
        // 2. knots touching this tile: virtual v in [toff[j], toff[j+1]+2]
        for (int s = 0; s < 2; ++s) {
            const unsigned* to = A.toff + toff_off(A, par, s, slot);
            vlo[s] = (int)to[j];
            vcnt[s] = (int)to[j + 1] + 2 - vlo[s] + 1;
            for (int q = tid; q < vcnt[s]; q += kEvalThreads) {
                double X, Y;
                vknot(J.kv[s], vlo[s] + q, X, Y);
                kX[s * kKnotCapTile + q] = X;
                kY[s * kKnotCapTile + q] = Y;
                kM[s * kKnotCapTile + q] = J.kv[s].mom[vlo[s] + q];
            }
        }
    }
    __syncthreads();

    // 3. new values (fast path) for the thread's consecutive samples
    double num = 0.0, den = 0.0;
    if (J.mode == EM_SIFT) {
        // samples handled by this thread: local i in [1+tid*kSpt, ...], plus halos by edge threads
        int i_begin = 1 + tid * kSpt, i_end = i_begin + kSpt;
        if (tid == 0) i_begin = 0;                           // left halo t = base-1
        if (tid == kEvalThreads - 1) i_end = kEvalTile + 2;  // right halo t = base+T
        int p[2] = {-1, -1};
        for (int i = i_begin; i < i_end; ++i) {
            const int t = base - 1 + i;
            if (t < 0 || t >= L || i > tlen + 1) continue;
            const double tt = (double)t;
            double env[2];
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const double* X = kX + s * kKnotCapTile;
                int q = p[s];
                if (q < 0) {  // binary search: last q with X[q] < tt
                    int lo = 0, hi = vcnt[s] - 2;
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (X[mid] < tt) lo = mid;
                        else hi = mid - 1;
                    }
                    q = lo;
                }
                while (q + 1 < vcnt[s] - 1 && X[q + 1] < tt) ++q;
                p[s] = q;
                env[s] = spline_eval(X[q], X[q + 1], kY[s * kKnotCapTile + q], kY[s * kKnotCapTile + q + 1],
                                     kM[s * kKnotCapTile + q], kM[s * kKnotCapTile + q + 1], tt);
            }
            const double cur = sv[i];
            const double mean = 0.5 * (env[0] + env[1]);
            const double nw = cur - mean;
            nv[i] = nw;
            if (i >= 1 && i <= tlen) {
                num += mean * mean;
                den += cur * cur;
                dst[t] = nw;
            }
        }
    } else {
        for (int i = tid; i < kEvalTile + 2; i += kEvalThreads) {
            nv[i] = sv[i];
            const int t = base - 1 + i;
            if (dst && i >= 1 && i <= tlen) dst[t] = sv[i];
        }
    }
    if (J.mode == EM_SIFT) {
        block_sum2(num, den, sh.red);
        if (tid == 0) {
            A.tnum[(size_t)slot * A.tiles + j] = num;
            A.tden[(size_t)slot * A.tiles + j] = den;
        }
    }
    __syncthreads();

    // 4. extrema of the new values (find_extrema, emd.cpp:16-33)
    unsigned fmax = 0, fmin = 0;  // bit k: sample k of this thread
    for (int k = 0; k < kSpt; ++k) {
        const int i = 1 + tid * kSpt + k;
        const int t = base - 1 + i;
        if (i > tlen || t < 1 || t > L - 2) continue;
        const double v = nv[i], l = nv[i - 1], r = nv[i + 1];
        bool ismax = false, ismin = false;
        if (v != l && v != r) {
            ismax = v > l && v > r;
            ismin = v < l && v < r;
        } else {
            // plateau: find the maximal run of samples equal to v
            auto val = [&](int u) -> double {
                const int li = u - base + 1;
                if (li >= 0 && li <= tlen + 1) return nv[li];
                return new_value_at(J, u);
            };
            int rs = t, re = t;
            while (rs > 0 && val(rs - 1) == v) --rs;
            while (re < L - 1 && val(re + 1) == v) ++re;
            if (rs > 0 && re < L - 1 && t == (rs + re) / 2) {
                const double lv = val(rs - 1), rv = val(re + 1);
                ismax = v > lv && v > rv;
                ismin = v < lv && v < rv;
            }
        }
        if (ismax) fmax |= 1u << k;
        if (ismin) fmin |= 1u << k;
    }
    // 5. ordered compaction: block scan of packed counts, look-back for the tile base
    const unsigned packed = (unsigned)__popc(fmax) | ((unsigned)__popc(fmin) << 16);
    const int lane = tid & 31, wid = tid >> 5;
    unsigned incl = packed;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) sh.scan[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        unsigned w = lane < kEvalThreads / 32 ? sh.scan[lane] : 0;
        unsigned wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < kEvalThreads / 32) sh.scan[lane] = wi - w;  // exclusive warp offsets
        const unsigned total = __shfl_sync(0xffffffffu, wi, kEvalThreads / 32 - 1);
        // two look-backs: warp 0 does max then min (cheap: tiles are few in flight)
        const unsigned tmax = total & 0xFFFF, tmin = total >> 16;
        const unsigned epoch = S.epoch;
        const unsigned gmax = lookback(A.status + status_off(A, 0, slot), j, epoch, tmax);
        const unsigned gmin = lookback(A.status + status_off(A, 1, slot), j, epoch, tmin);
        if (lane == 0) {
            sh.gbase[0] = gmax;
            sh.gbase[1] = gmin;
            const int np = 1 - par;
            unsigned* to0 = A.toff + toff_off(A, np, 0, slot);
            unsigned* to1 = A.toff + toff_off(A, np, 1, slot);
            to0[j] = gmax;
            to1[j] = gmin;
            if (j == A.tiles - 1) {
                to0[A.tiles] = gmax + tmax;
                to1[A.tiles] = gmin + tmin;
            }
        }
    }
    __syncthreads();
    const unsigned excl = sh.scan[wid] + incl - packed;
    unsigned omax = sh.gbase[0] + (excl & 0xFFFF), omin = sh.gbase[1] + (excl >> 16);
    const int np = 1 - par;
    int* kidx0 = A.kidx + knot_off(A, np, 0, slot);
    int* kidx1 = A.kidx + knot_off(A, np, 1, slot);
    double* kval0 = A.kval + knot_off(A, np, 0, slot);
    double* kval1 = A.kval + knot_off(A, np, 1, slot);
    uint64_t h = 0;
    for (int k = 0; k < kSpt; ++k) {
        const int i = 1 + tid * kSpt + k;
        const int t = base - 1 + i;
        if (fmax & (1u << k)) {
            kidx0[omax] = t;
            kval0[omax] = nv[i];
            h += knot_hash(0, omax, (unsigned)t);
            ++omax;
        }
        if (fmin & (1u << k)) {
            kidx1[omin] = t;
            kval1[omin] = nv[i];
            h += knot_hash(1, omin, (unsigned)t);
            ++omin;
        }
    }
    h = warp_sum(h);
    __syncthreads();
    unsigned long long* hred = reinterpret_cast<unsigned long long*>(sh.red);
    if (lane == 0) hred[wid] = h;
    __syncthreads();
    if (tid == 0) {
        uint64_t hs = 0;
        for (int w = 0; w < kEvalThreads / 32; ++w) hs += hred[w];
        A.thash[(size_t)slot * A.tiles + j] = hs;
    }
    __syncthreads();
}

__device__ __forceinline__ int pick_free_buffer(int xb, int cb) {
    if (cb < 0) return xb == 0 ? 1 : 0;
    return 3 - xb - cb;
}

__device__ void emit_trace(const Arena& A, const Slot& S, int iter, unsigned nmax, unsigned nmin, uint64_t h) {
    if (!A.trace) return;
    const int pos = atomicAdd(&A.ctrl->trace_count, 1);
    if (pos < A.trace_cap) {
        TraceRec r;
        r.task = S.task;
        r.m = S.m;
        r.k = S.k;
        r.iter = iter;
        r.n_max = nmax;
        r.n_min = nmin;
        r.hash = h;
        A.trace[pos] = r;
    }
}

// Rebuild the per-step work lists (one CTA). Lockstep rule: IMF k is
// finalised for every slot in the same step, once no slot is still sifting.
__device__ void build_lists(const Arena& A, bool allow_final) {
    __shared__ int s_cnt[4];
    Ctrl* C = A.ctrl;
    const int tid = threadIdx.x;
    if (tid < 4) s_cnt[tid] = 0;
    __syncthreads();
    // pass 1: are all unfinished slots waiting?
    for (int s = tid; s < A.G; s += blockDim.x) {
        const int st = A.slots[s].state;
        if (st == ST_INIT || st == ST_DETECT || st == ST_SIFT) atomicAdd(&s_cnt[0], 1);
        if (st == ST_WAITK) atomicAdd(&s_cnt[1], 1);
    }
    __syncthreads();
    const bool finalize = allow_final && s_cnt[0] == 0 && s_cnt[1] > 0;
    __syncthreads();
    if (tid == 0) {
        // ordered lists (slot order fixes the accumulation order)
        int ne = 0, nf = 0, ns = 0, nb = 0, act = 0;
        for (int s = 0; s < A.G; ++s) {
            Slot& S = A.slots[s];
            if (finalize && S.state == ST_WAITK) S.state = ST_FINAL;
            const int st = S.state;
            if (st == ST_INIT || st == ST_DETECT || st == ST_SIFT) A.eval_list[ne++] = s;
            if (st == ST_FINAL) A.final_list[nf++] = s;
            if (st != ST_FREE && st != ST_DONE) ++act;
            if (st == ST_SIFT) {
                if (S.iter == 0 || S.cb >= 0) S.db = pick_free_buffer(S.xb, S.cb);
                for (int side = 0; side < 2; ++side) {
                    const int rows = (int)S.n[side] + 2;
                    const int blocks = rows <= kSolveSeqMax ? 1 : (rows + kSolveBlock - 1) / kSolveBlock;
                    A.solve_item[ns] = (s << 1) | side;
                    A.solve_off[ns] = nb;
                    ++ns;
                    nb += blocks;
                }
            }
        }
        A.solve_off[ns] = nb;
        C->n_eval = ne;
        C->n_final = nf;
        C->n_solve = ns;
        C->solve_blocks = nb;
        C->active = act;
    }
    __syncthreads();
}

// decide1: after the eval pass (emd.cpp:131-151 control flow).
__device__ void decide_after_eval(const Arena& A) {
    Ctrl* C = A.ctrl;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int ne = C->n_eval;
    for (int li = wid; li < ne; li += nw) {
        const int s = A.eval_list[li];
        Slot& S = A.slots[s];
        const int state = S.state;
        double num = 0.0, den = 0.0;
        uint64_t h = 0;
        for (int j = lane; j < A.tiles; j += 32) {
            if (state == ST_SIFT) {
                num += A.tnum[(size_t)s * A.tiles + j];
                den += A.tden[(size_t)s * A.tiles + j];
            }
            h += A.thash[(size_t)s * A.tiles + j];
        }
        num = warp_sum(num);
        den = warp_sum(den);
        h = warp_sum(h);
        if (lane != 0) continue;
        const int np = 1 - S.par;
        const unsigned nmax = A.toff[toff_off(A, np, 0, s) + A.tiles];
        const unsigned nmin = A.toff[toff_off(A, np, 1, s) + A.tiles];
        S.epoch += 1;
        if (state == ST_INIT || state == ST_DETECT) {
            // iteration 0 of IMF k: extract_imf's first find_extrema
            if (A.max_sift_iters <= 0 && !S.detect_only) {  // loop body never runs: IMF = input, 0 sifts
                S.cb = -1;
                S.iter = 0;
                S.state = ST_WAITK;
                if (S.k0 + S.k < A.kcap && A.imf_sifts) A.imf_sifts[S.k0 + S.k] = 0;
                continue;
            }
            emit_trace(A, S, 0, nmax, nmin, h);
            if (S.detect_only) {
                S.n[0] = nmax;
                S.n[1] = nmin;
                S.state = ST_DONE;
                continue;
            }
            S.par = np;
            S.n[0] = nmax;
            S.n[1] = nmin;
            S.iter = 0;
            S.cb = -1;
            if (nmax < 2 || nmin < 2) {  // InsufficientExtrema on the unsifted input
                S.ended_insufficient = 1;
                S.state = ST_DONE;
            } else {
                S.state = ST_SIFT;
            }
        } else if (state == ST_SIFT) {
            S.iter += 1;
            S.sifted += A.L;
            S.cb = S.db;
            S.num = num;
            S.den = den;
            bool stop = (den == 0.0 || num / den < A.sd_threshold) || S.iter >= A.max_sift_iters;
            if (!stop) {
                emit_trace(A, S, S.iter, nmax, nmin, h);
                if (nmax < 2 || nmin < 2) {
                    stop = true;  // envelope throws; the candidate is the IMF (emd.cpp:137-140)
                } else {
                    S.par = np;
                    S.n[0] = nmax;
                    S.n[1] = nmin;
                }
            }
            if (stop) {
                S.state = ST_WAITK;
                if (S.k0 + S.k < A.kcap && A.imf_sifts) A.imf_sifts[S.k0 + S.k] = S.iter;
            }
        }
    }
    __syncthreads();
    build_lists(A, true);
}

__global__ void __launch_bounds__(kEvalThreads, 2) k_eval(Arena A) {
    extern __shared__ double smem[];
    double* sv = smem;
    double* nv = sv + (kEvalTile + 2);
    double* kX = nv + (kEvalTile + 2);
    double* kY = kX + 2 * kKnotCapTile;
    double* kM = kY + 2 * kKnotCapTile;
    __shared__ EvalShared sh;
    Ctrl* C = A.ctrl;
    const int nitems = C->n_eval * A.tiles;
    while (true) {
        if (threadIdx.x == 0) sh.ticket = atomicAdd(&C->ticket[0], 1u);
        __syncthreads();
        const unsigned q = sh.ticket;
        __syncthreads();
        if (q >= (unsigned)nitems) break;
        const int li = (int)(q / (unsigned)A.tiles), j = (int)(q % (unsigned)A.tiles);
        eval_tile(A, A.eval_list[li], j, sv, nv, kX, kY, kM, sh);
    }
    if (threadIdx.x == 0) {
        __threadfence();
        sh.last = atomicAdd(&C->done[0], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (sh.last) {
        __threadfence();
        decide_after_eval(A);
        if (threadIdx.x == 0) {
            C->ticket[0] = 0;
            C->done[0] = 0;
        }
    }
}

// ----------------------------------------------------------- solve kernel
//
// Natural-spline moments (emd.cpp:53-73) for the mirrored knot system of one
// envelope, reproducing the reference's sequential Thomas algorithm
// BIT-FOR-BIT with parallel chains: each chain restarts the recurrence from a
// guessed state at its chunk start; because the recurrences are contractive,
// the speculative chain becomes bitwise identical to the true chain after a
// few dozen rows. Every chain then replays its head from its predecessor's
// end state until it meets its own stored values bitwise ("convergence"),
// which makes the result exactly the sequential one. Chunk boundaries that do
// not converge inside the chunk are repaired sequentially. Across CTA blocks
// a 64-row warm-up is used and the boundary values are cross-checked
// (mismatches are counted as hazards).

struct RowCtx {
    const double* X;  // window arrays indexed by v - wa
    const double* Y;
    int wa;
};

__device__ __forceinline__ void row_coef(const RowCtx& w, int i, double& h0, double& diag, double& rhs) {
    const double* X = w.X - w.wa;
    const double* Y = w.Y - w.wa;
    h0 = X[i] - X[i - 1];
    const double h1 = X[i + 1] - X[i];
    diag = 2.0 * (h0 + h1);
    rhs = 6.0 * ((Y[i + 1] - Y[i]) / h1 - (Y[i] - Y[i - 1]) / h0);
}

__device__ __forceinline__ void fwd_step(const RowCtx& w, int i, double& d, double& r) {
    double h0, diag, rhs;
    row_coef(w, i, h0, diag, rhs);
    const double wgt = h0 / d;
    d = diag - wgt * h0;
    r = rhs - wgt * r;
}

__device__ __forceinline__ void fwd_start(const RowCtx& w, int i, double& d, double& r) {
    double h0;
    row_coef(w, i, h0, d, r);
}

__device__ __forceinline__ double back_step(const RowCtx& w, int i, double dp, double rp, double mnext) {
    const double* X = w.X - w.wa;
    const double upper = X[i + 1] - X[i];
    return (rp - upper * mnext) / dp;
}

struct SolveShared {
    unsigned ticket;
    int last;
    int flag;
    int item, b;
};

__global__ void __launch_bounds__(kSolveThreads + 32, 1) k_solve(Arena A) {
    extern __shared__ double smem[];
    __shared__ SolveShared sh;
    Ctrl* C = A.ctrl;
    const int tid = threadIdx.x;
    const int nblocks = C->solve_blocks;
    const int nitems = C->n_solve;
    while (true) {
        if (tid == 0) {
            sh.ticket = atomicAdd(&C->ticket[1], 1u);
            sh.flag = 0;
            if (sh.ticket < (unsigned)nblocks) {
                int lo = 0, hi = nitems - 1;  // last item with off <= ticket
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if ((unsigned)A.solve_off[mid] <= sh.ticket) lo = mid;
                    else hi = mid - 1;
                }
                sh.item = lo;
                sh.b = (int)sh.ticket - A.solve_off[lo];
            }
        }
        __syncthreads();
        const unsigned q = sh.ticket;
        if (q >= (unsigned)nblocks) break;
        const int code = A.solve_item[sh.item];
        const int slot = code >> 1, side = code & 1, b = sh.b;
        const Slot& S = A.slots[slot];
        KnotView kv;
        kv.idx = A.kidx + knot_off(A, S.par, side, slot);
        kv.val = A.kval + knot_off(A, S.par, side, slot);
        kv.n = (int)S.n[side];
        kv.e2 = 2.0 * (double)(A.L - 1);
        double* mom = A.mom + mom_off(A, side, slot);
        const int N = kv.n + 4;
        const int rows = N - 2;
        if (rows <= kSolveSeqMax) {
            // small system: one thread runs the reference Thomas algorithm verbatim
            double* X = smem;
            double* Y = X + (kSolveSeqMax + 2);
            double* dp = Y + (kSolveSeqMax + 2);
            double* rp = dp + (kSolveSeqMax + 2);
            for (int v = tid; v < N; v += blockDim.x) vknot(kv, v, X[v], Y[v]);
            __syncthreads();
            if (tid == 0) {
                RowCtx w{X, Y, 0};
                double d, r;
                fwd_start(w, 1, d, r);
                dp[1] = d;
                rp[1] = r;
                for (int i = 2; i <= N - 2; ++i) {
                    fwd_step(w, i, d, r);
                    dp[i] = d;
                    rp[i] = r;
                }
                double m = 0.0;
                mom[N - 1] = 0.0;
                for (int i = N - 2; i >= 1; --i) {
                    m = back_step(w, i, dp[i], rp[i], m);
                    mom[i] = m;
                }
                mom[0] = 0.0;
            }
            __syncthreads();
            continue;
        }
        const int H = kSolveHalo, B = kSolveBlock, CH = kSolveChunk, NT = kSolveThreads;
        const int r0 = 1 + b * B;
        const int r1 = min(r0 + B, N - 1);
        const int r1e = min(r1 + H, N - 1);
        const int wa = max(0, r0 - H - 1);
        const int wb = min(N - 1, r1 + H);
        const int wn = wb - wa + 1;
        double* X = smem;
        double* Y = X + (B + 2 * H + 2);
        double* dp = Y + (B + 2 * H + 2);
        double* rp = dp + (B + H);
        double* mm = rp + (B + H);
        for (int v = tid; v < wn; v += blockDim.x) vknot(kv, wa + v, X[v], Y[v]);
        __syncthreads();
        RowCtx w{X, Y, wa};
        // chains: c in [0, NT) own [r0+c*CH, ...) ; c == NT owns the back halo [r1, r1e)
        const int c = tid;
        int cs, ce;
        if (c < NT) {
            cs = min(r0 + c * CH, r1);
            ce = min(cs + CH, r1);
        } else if (c == NT) {
            cs = r1;
            ce = r1e;
        } else {
            cs = ce = 0;
        }
        // --- phase A: forward, speculative
        if (c <= NT && cs < ce) {
            double d, r;
            int i = cs;
            if (c == 0 && r0 > 1) {
                const int ws = max(1, r0 - H);
                fwd_start(w, ws, d, r);
                for (int k = ws + 1; k < r0; ++k) fwd_step(w, k, d, r);
                double* rec = A.sb + (((size_t)side * A.G + slot) * A.max_blocks + b) * 6;
                rec[0] = d;  // state at row r0-1 reached by the warm-up
                rec[1] = r;
                fwd_step(w, i, d, r);
            } else {
                fwd_start(w, i, d, r);  // exact when i == 1, a guess otherwise
            }
            dp[i - r0] = d;
            rp[i - r0] = r;
            for (++i; i < ce; ++i) {
                fwd_step(w, i, d, r);
                dp[i - r0] = d;
                rp[i - r0] = r;
            }
        }
        __syncthreads();
        // --- phase B: replay each chain head from the predecessor's end state
        if (c >= 1 && c <= NT && cs < ce) {
            double d = dp[cs - 1 - r0], r = rp[cs - 1 - r0];
            bool conv = false;
            for (int i = cs; i < ce; ++i) {
                fwd_step(w, i, d, r);
                if (d == dp[i - r0] && r == rp[i - r0]) {
                    conv = true;
                    break;
                }
                dp[i - r0] = d;
                rp[i - r0] = r;
            }
            if (!conv) sh.flag = 1;
        }
        __syncthreads();
        if (sh.flag) {
            if (tid == 0) {
                for (int cc = 1; cc <= NT; ++cc) {
                    const int s0 = cc < NT ? min(r0 + cc * CH, r1) : r1;
                    const int e0 = cc < NT ? min(s0 + CH, r1) : r1e;
                    if (s0 >= e0) continue;
                    double d = dp[s0 - 1 - r0], r = rp[s0 - 1 - r0];
                    for (int i = s0; i < e0; ++i) {
                        fwd_step(w, i, d, r);
                        if (d == dp[i - r0] && r == rp[i - r0]) break;
                        dp[i - r0] = d;
                        rp[i - r0] = r;
                    }
                }
                sh.flag = 0;
            }
            __syncthreads();
        }
        // --- phase C: back substitution, speculative (m_{N-1} = 0 is exact)
        auto mget = [&](int i) -> double { return i >= N - 1 ? 0.0 : mm[i - r0]; };
        if (c <= NT && cs < ce) {
            double m = 0.0;  // guess for m[ce] unless ce == N-1 (exact)
            for (int i = ce - 1; i >= cs; --i) {
                m = back_step(w, i, dp[i - r0], rp[i - r0], m);
                mm[i - r0] = m;
            }
        }
        __syncthreads();
        // --- phase D: replay chain tails from the successor's first value
        if (c < NT && cs < ce && ce < N - 1) {
            double m = mget(ce);
            bool conv = false;
            for (int i = ce - 1; i >= cs; --i) {
                m = back_step(w, i, dp[i - r0], rp[i - r0], m);
                if (m == mm[i - r0]) {
                    conv = true;
                    break;
                }
                mm[i - r0] = m;
            }
            if (!conv) sh.flag = 1;
        }
        __syncthreads();
        if (sh.flag) {
            if (tid == 0) {
                for (int cc = NT - 1; cc >= 0; --cc) {
                    const int s0 = min(r0 + cc * CH, r1);
                    const int e0 = min(s0 + CH, r1);
                    if (s0 >= e0 || e0 >= N - 1) continue;
                    double m = mget(e0);
                    for (int i = e0 - 1; i >= s0; --i) {
                        m = back_step(w, i, dp[i - r0], rp[i - r0], m);
                        if (m == mm[i - r0]) break;
                        mm[i - r0] = m;
                    }
                }
            }
            __syncthreads();
        }
        // --- outputs + cross-block check values. Record per block (6 doubles):
        // [0,1] warm-up forward state at row r0-1, [2,3] this block's forward
        // state at row r1-1, [4] m at row r0, [5] the m at row r1 this block used.
        for (int i = r0 + tid; i < r1; i += blockDim.x) mom[i] = mm[i - r0];
        if (tid == 0) {
            if (r0 == 1) mom[0] = 0.0;
            if (r1 == N - 1) mom[N - 1] = 0.0;
            double* rec = A.sb + (((size_t)side * A.G + slot) * A.max_blocks + b) * 6;
            rec[2] = dp[r1 - 1 - r0];
            rec[3] = rp[r1 - 1 - r0];
            rec[4] = mm[0];
            rec[5] = mget(r1);
        }
        __syncthreads();
    }
    if (tid == 0) {
        __threadfence();
        sh.last = atomicAdd(&C->done[1], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (sh.last) {
        __threadfence();
        // cross-block consistency of the speculative chains (hazard = a block
        // whose warm-up did not reach the neighbour's exact boundary state)
        for (int it = tid; it < nitems; it += blockDim.x) {
            const int code = A.solve_item[it];
            const int slot = code >> 1, side = code & 1;
            const int nb = A.solve_off[it + 1] - A.solve_off[it];
            const int rows = (int)A.slots[slot].n[side] + 2;
            if (rows <= kSolveSeqMax) continue;
            const double* base = A.sb + ((size_t)side * A.G + slot) * A.max_blocks * 6;
            int bad = 0;
            for (int b = 1; b < nb; ++b) {
                const double* p = base + (size_t)(b - 1) * 6;
                const double* q = base + (size_t)b * 6;
                if (q[0] != p[2] || q[1] != p[3] || p[5] != q[4]) ++bad;
            }
            if (bad) {
                atomicAdd(&A.slots[slot].hazards, bad);
                atomicAdd(&C->hazards, bad);
            }
        }
        if (tid == 0) {
            C->ticket[1] = 0;
            C->done[1] = 0;
        }
    }
}

// ----------------------------------------------------------- final kernel
//
// IMF k is complete for every slot in final_list (lockstep). Per sample:
//   sums[k0+k][t] += imf_s[t]   in slot order (eemd accumulation, emd.cpp:249-251)
//   R_s[t] = X_s[t] - imf_s[t]  (emd.cpp:167 residue update)

__device__ void decide_after_final(const Arena& A) {
    Ctrl* C = A.ctrl;
    const int tid = threadIdx.x;
    const int nf = C->n_final;
    for (int li = tid; li < nf; li += blockDim.x) {
        const int s = A.final_list[li];
        Slot& S = A.slots[s];
        const int rb = pick_free_buffer(S.xb, S.cb);
        S.last_imf_b = S.cb >= 0 ? S.cb : S.xb;
        S.xb = rb;
        S.cb = -1;
        S.k += 1;
        S.iter = 0;
        if (S.kmax > 0 && S.k >= S.kmax) S.state = ST_DONE;
        else S.state = ST_DETECT;
    }
    __syncthreads();
    build_lists(A, false);
    if (tid == 0 && A.status_host) {
        C->step += 1;
        volatile int* hs = A.status_host;
        hs[0] = C->active;
        hs[1] = C->step;
    }
}

__global__ void __launch_bounds__(256) k_final(Arena A) {
    __shared__ unsigned s_ticket;
    __shared__ int s_last;
    Ctrl* C = A.ctrl;
    const int nf = C->n_final;
    const int tiles = (A.L + kFinalTile - 1) / kFinalTile;
    const int nitems = nf > 0 ? tiles : 0;
    while (true) {
        if (threadIdx.x == 0) s_ticket = atomicAdd(&C->ticket[2], 1u);
        __syncthreads();
        const unsigned q = s_ticket;
        __syncthreads();
        if (q >= (unsigned)nitems) break;
        for (int i = threadIdx.x; i < kFinalTile; i += blockDim.x) {
            const size_t t = (size_t)q * kFinalTile + i;
            if (t >= (size_t)A.L) break;
            int row = -1;
            double acc = 0.0;
            for (int li = 0; li < nf; ++li) {
                const int s = A.final_list[li];
                const Slot& S = A.slots[s];
                const double x = A.bufs[buf_off(A, s, S.xb) + t];
                const double imf = S.cb >= 0 ? A.bufs[buf_off(A, s, S.cb) + t] : x;
                const int rb = pick_free_buffer(S.xb, S.cb);
                const double res = x - imf;
                A.bufs[buf_off(A, s, rb) + t] = res;
                if (S.imf_out) S.imf_out[t] = imf;
                if (S.res_out) S.res_out[t] = res;
                if (S.write_imf) {
                    const int r = S.k0 + S.k;
                    if (r < A.kcap) {
                        if (r != row) {
                            if (row >= 0) A.sums[(size_t)row * A.L + t] = acc;
                            row = r;
                            acc = A.sums[(size_t)row * A.L + t];
                        }
                        acc = acc + imf;
                    }
                }
            }
            if (row >= 0) A.sums[(size_t)row * A.L + t] = acc;
        }
    }
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&C->done[2], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        if (threadIdx.x == 0) {
            for (int li = 0; li < nf; ++li) {
                const Slot& S = A.slots[A.final_list[li]];
                if (S.write_imf && S.k0 + S.k >= A.kcap) atomicAdd(&C->k_overflow, 1);
            }
        }
        decide_after_final(A);
        if (threadIdx.x == 0) {
            C->ticket[2] = 0;
            C->done[2] = 0;
        }
    }
}

// -------------------------------------------------------------- RNG
//
// std::mt19937_64 ([rand.predef]) for one realization per CTA: the 312-word
// twist is done in three data-parallel phases, then tempering; draws are
// written as raw u64. k_box_muller maps draw pairs exactly like
// white_noise (emd.cpp:189-198).

__device__ __forceinline__ uint64_t mt_twist(uint64_t a, uint64_t b) {
    const uint64_t x = (a & 0xFFFFFFFF80000000ULL) | (b & 0x7FFFFFFFULL);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
    return xa;
}

__global__ void __launch_bounds__(320) k_mt19937_64(const RngJob* jobs) {
    __shared__ uint64_t mt[312];
    const RngJob J = jobs[blockIdx.x];
    const int t = threadIdx.x;
    if (t == 0) {
        mt[0] = J.seed;
        for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
    }
    __syncthreads();
    const long long ndraw = 2 * ((J.n + 1) / 2);
    for (long long base = 0; base < ndraw; base += 312) {
        uint64_t a = 0, b = 0, c = 0;
        if (t < 312) {
            a = mt[t];
            b = mt[(t + 1) % 312];
            c = mt[(t + 156) % 312];
        }
        __syncthreads();
        if (t < 156) mt[t] = c ^ mt_twist(a, b);
        __syncthreads();
        if (t >= 156 && t < 311) mt[t] = mt[t - 156] ^ mt_twist(a, b);
        if (t == 311) mt[311] = mt[155] ^ mt_twist(a, mt[0]);
        __syncthreads();
        if (t < 312 && base + t < ndraw) {
            uint64_t y = mt[t];
            y ^= (y >> 29) & 0x5555555555555555ULL;
            y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
            y ^= (y << 37) & 0xFFF7EEE000000000ULL;
            y ^= y >> 43;
            J.out[base + t] = y;
        }
    }
}

// In place: draws (u64 pairs) -> Gaussian samples (f64), emd.cpp:189-198.
__global__ void k_box_muller(uint64_t* draws, long long n, double stdv) {
    const long long pairs = (n + 1) / 2;
    const double two_pi = 6.283185307179586476925286766559;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < pairs;
         p += (long long)gridDim.x * blockDim.x) {
        const uint64_t d1 = draws[2 * p], d2 = draws[2 * p + 1];
        const double u1 = (double)((d1 >> 11) + 1) * 0x1.0p-53;
        const double r = stdv * sqrt(-2.0 * log(u1));
        const double u2 = (double)((d2 >> 11) + 1) * 0x1.0p-53;
        const double theta = two_pi * u2;
        double* out = reinterpret_cast<double*>(draws);
        out[2 * p] = r * cos(theta);
        if (2 * p + 1 < n) out[2 * p + 1] = r * sin(theta);
    }
}

// ------------------------------------------------------------ small kernels

// emd.cpp:209-217 verbatim (sequential two-pass sums): one thread.
__global__ void k_signal_std(const double* x, long long n, double* out, double scale) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (n == 0) {
        *out = 0.0;
        return;
    }
    double mean = 0.0;
    for (long long i = 0; i < n; ++i) mean += x[i];
    mean /= (double)n;
    double acc = 0.0;
    for (long long i = 0; i < n; ++i) acc += (x[i] - mean) * (x[i] - mean);
    *out = scale * sqrt(acc / (double)n);
}

// eemd finish (emd.cpp:252-260): imfs *= 1/nr ; residue = x - sum_k imf_k (k order).
__global__ void k_ensemble_finish(double* sums, int K, long long L, const double* x, double* residue, double inv) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < L; t += (long long)gridDim.x * blockDim.x) {
        double r = x[t];
        for (int k = 0; k < K; ++k) {
            const double v = sums[(size_t)k * L + t] * inv;
            sums[(size_t)k * L + t] = v;
            r -= v;
        }
        residue[t] = r;
    }
}

// serialize.cpp:30-50: channel copy + blended transitions (2 mul + 1 add, no FMA).
__global__ void k_concatenate(const double* x, long long M, long long N, long long D, const double* a, double* out,
                              int naive) {
    const long long L = M * N + D * (N - 1);
    const long long stride = M + D;
    for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < L; o += (long long)gridDim.x * blockDim.x) {
        const long long j = o / stride, p = o % stride;
        if (p < M) {
            out[o] = x[j * M + p];
        } else {
            const long long t = p - M;  // transition sample t of block j
            const double* ch = x + j * M;
            const double* next = x + (j + 1) * M;
            if (!naive) {
                out[o] = next[D - 1 - t] * a[t] + ch[M - 1 - t] * a[D - 1 - t];
            } else {  // serialize.cpp:64-67, i = t + 1
                const long long i = t + 1;
                const double wg = (double)i / (double)(D + 1);
                const double wf = (double)(D + 1 - i) / (double)(D + 1);
                out[o] = wg * next[D - i] + wf * ch[M - i];
            }
        }
    }
}

// serialize.cpp:7-13
__global__ void k_transition_weights(long long d, double* a) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < d; i += (long long)gridDim.x * blockDim.x)
        a[i] = (double)(i + 1) / (double)(d + 1);
}

// serialize.cpp:86-93: out[(k*N+j)*M+i] = modes[k][j*(M+D)+i]
__global__ void k_deconcatenate(const double* modes, long long K, long long Lm, long long M, long long N, long long D,
                                double* out) {
    const long long total = K * N * M;
    for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < total;
         o += (long long)gridDim.x * blockDim.x) {
        const long long i = o % M, kj = o / M, j = kj % N, k = kj / N;
        out[o] = modes[k * Lm + j * (M + D) + i];
    }
}

// General envelope (emd.cpp:91-125) for the standalone envelope() entry:
// conditional mirrors, the two-knot line (:46-51), sequential Thomas in one
// thread, parallel evaluation. xs/ys built on the host side of the kernel.
__global__ void k_envelope_solve(const double* xs, const double* ys, int n, double* mom, double* work) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (n == 2) return;
    double* dp = work;
    double* rp = work + n;
    RowCtx w{xs, ys, 0};
    double d, r;
    fwd_start(w, 1, d, r);
    dp[1] = d;
    rp[1] = r;
    for (int i = 2; i + 1 < n; ++i) {
        fwd_step(w, i, d, r);
        dp[i] = d;
        rp[i] = r;
    }
    double m = 0.0;
    mom[n - 1] = 0.0;
    for (int i = n - 2; i >= 1; --i) {
        m = back_step(w, i, dp[i], rp[i], m);
        mom[i] = m;
    }
    mom[0] = 0.0;
}

__global__ void k_envelope_eval(const double* xs, const double* ys, const double* mom, int n, long long length,
                                double* out) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < length;
         t += (long long)gridDim.x * blockDim.x) {
        const double tt = (double)t;
        if (n == 2) {
            const double slope = (ys[1] - ys[0]) / (xs[1] - xs[0]);
            out[t] = ys[0] + slope * (tt - xs[0]);
            continue;
        }
        // seg = the reference's march result: largest seg <= n-2 with seg==0 or tt > xs[seg]
        int lo = 0, hi = n - 2;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            bool passed = true;  // the march passes xs[1..mid] iff tt > xs[q] for all q <= mid
            passed = tt > xs[mid];
            if (passed) lo = mid;
            else hi = mid - 1;
        }
        // the march stops at the first seg with tt <= xs[seg+1]; with increasing xs on the
        // evaluated range this is the largest seg with tt > xs[seg] (or 0)
        const int seg = lo;
        out[t] = spline_eval(xs[seg], xs[seg + 1], ys[seg], ys[seg + 1], mom[seg], mom[seg + 1], tt);
    }
}

// CEEMDAN stage mean (emd.cpp:301-304 / :331-336): mode *= inv, flag any nonzero.
__global__ void k_stage_scale(double* mode, long long n, double inv, int* nonzero) {
    int nz = 0;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
        const double v = mode[t] * inv;
        mode[t] = v;
        if (v != 0.0) nz = 1;
    }
    if (__syncthreads_or(nz) && threadIdx.x == 0) atomicOr(nonzero, 1);
}

// residue -= mode (emd.cpp:304 / :338)
__global__ void k_sub(double* residue, const double* mode, long long n) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
        residue[t] = residue[t] - mode[t];
}

// Knot vector of a general envelope() call (emd.cpp:98-122): optional mirrors.
__global__ void k_envelope_knots(const unsigned long long* idx, const double* val, long long n, long long length,
                                 double* xs, double* ys) {
    const bool left = idx[0] != 0, right = idx[n - 1] != (unsigned long long)(length - 1);
    const long long off = left ? 2 : 0;
    const long long N = n + off + (right ? 2 : 0);
    const double end = (double)(length - 1);
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < N; v += (long long)gridDim.x * blockDim.x) {
        if (v < off) {  // descending source order: k = 1 then 0
            const long long k = 1 - v;
            xs[v] = -(double)idx[k];
            ys[v] = val[k];
        } else if (v < off + n) {
            xs[v] = (double)idx[v - off];
            ys[v] = val[v - off];
        } else {
            const long long k = n - 2 + (v - off - n);
            xs[v] = 2.0 * end - (double)idx[k];
            ys[v] = val[k];
        }
    }
}

__global__ void k_fill(double* p, long long n, double v) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
        p[t] = v;
}

// Copy one slot buffer (e.g. the final residue) out.
__global__ void k_copy(const double* src, double* dst, long long n) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
        dst[t] = src[t];
}

// X = a + beta * b (CEEMDAN first-mode input, emd.cpp:297 / :327)
__global__ void k_axpy(const double* a, const double* b, double beta, double* out, long long n) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
        out[t] = a[t] + beta * b[t];
}

}  // namespace dev
}  // namespace semd

// ------------------------------------------------------------ launchers
namespace semd {
namespace dev {

size_t eval_smem_bytes() { return (size_t)(2 * (kEvalTile + 2) + 6 * kKnotCapTile) * sizeof(double); }
size_t solve_smem_bytes() {
    const size_t chunked = (size_t)(2 * (kSolveBlock + 2 * kSolveHalo + 2) + 3 * (kSolveBlock + kSolveHalo)) * 8;
    const size_t seq = (size_t)4 * (kSolveSeqMax + 2) * 8;
    return chunked > seq ? chunked : seq;
}

cudaError_t launch_setup() {
    cudaError_t e = cudaFuncSetAttribute(k_eval, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)eval_smem_bytes());
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)solve_smem_bytes());
}

void launch_step(const Arena& A, int sms, cudaStream_t st) {
    k_solve<<<sms, kSolveThreads + 32, solve_smem_bytes(), st>>>(A);
    k_eval<<<2 * sms, kEvalThreads, eval_smem_bytes(), st>>>(A);
    k_final<<<2 * sms, 256, 0, st>>>(A);
}

void launch_rng(const RngJob* jobs, int njobs, cudaStream_t st) { k_mt19937_64<<<njobs, 320, 0, st>>>(jobs); }
void launch_box_muller(uint64_t* draws, long long n, double stdv, cudaStream_t st) {
    const long long pairs = (n + 1) / 2;
    const int grid = (int)((pairs + 255) / 256 < 4096 ? (pairs + 255) / 256 : 4096);
    k_box_muller<<<grid > 0 ? grid : 1, 256, 0, st>>>(draws, n, stdv);
}
void launch_signal_std(const double* x, long long n, double* out, double scale, cudaStream_t st) {
    k_signal_std<<<1, 32, 0, st>>>(x, n, out, scale);
}
static int grid_for(long long n) {
    long long g = (n + 255) / 256;
    if (g > 8192) g = 8192;
    return g < 1 ? 1 : (int)g;
}
void launch_ensemble_finish(double* sums, int K, long long L, const double* x, double* residue, double inv,
                            cudaStream_t st) {
    k_ensemble_finish<<<grid_for(L), 256, 0, st>>>(sums, K, L, x, residue, inv);
}
void launch_concatenate(const double* x, long long M, long long N, long long D, const double* a, double* out,
                        int naive, cudaStream_t st) {
    k_concatenate<<<grid_for(M * N + D * (N - 1)), 256, 0, st>>>(x, M, N, D, a, out, naive);
}
void launch_transition_weights(long long d, double* a, cudaStream_t st) {
    k_transition_weights<<<grid_for(d), 256, 0, st>>>(d, a);
}
void launch_deconcatenate(const double* modes, long long K, long long Lm, long long M, long long N, long long D,
                          double* out, cudaStream_t st) {
    k_deconcatenate<<<grid_for(K * N * M), 256, 0, st>>>(modes, K, Lm, M, N, D, out);
}
void launch_envelope(const double* xs, const double* ys, int n, double* mom, double* work, long long length,
                     double* out, cudaStream_t st) {
    k_envelope_solve<<<1, 32, 0, st>>>(xs, ys, n, mom, work);
    k_envelope_eval<<<grid_for(length), 256, 0, st>>>(xs, ys, mom, n, length, out);
}
void launch_stage_scale(double* mode, long long n, double inv, int* nonzero, cudaStream_t st) {
    k_stage_scale<<<grid_for(n), 256, 0, st>>>(mode, n, inv, nonzero);
}
void launch_sub(double* residue, const double* mode, long long n, cudaStream_t st) {
    k_sub<<<grid_for(n), 256, 0, st>>>(residue, mode, n);
}
void launch_envelope_knots(const unsigned long long* idx, const double* val, long long n, long long length,
                           double* xs, double* ys, cudaStream_t st) {
    k_envelope_knots<<<grid_for(n + 4), 256, 0, st>>>(idx, val, n, length, xs, ys);
}
void launch_fill(double* p, long long n, double v, cudaStream_t st) { k_fill<<<grid_for(n), 256, 0, st>>>(p, n, v); }
void launch_copy(const double* src, double* dst, long long n, cudaStream_t st) {
    k_copy<<<grid_for(n), 256, 0, st>>>(src, dst, n);
}
void launch_axpy(const double* a, const double* b, double beta, double* out, long long n, cudaStream_t st) {
    k_axpy<<<grid_for(n), 256, 0, st>>>(a, b, beta, out, n);
}

}  // namespace dev
}  // namespace semd
