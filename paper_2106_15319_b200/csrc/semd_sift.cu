// semd_sift.cu -- the sm_100a sift engine: one lockstep step =
//   k_solve   spline moments of every sifting slot's envelopes   (emd.cpp:53-73)
//   k_eval    mean-envelope subtraction + SD partials + extrema  (emd.cpp:10-35, :75-86, :142-148)
//   k_scan    per-slot tile prefix of the new extrema + SD sums; epilogue = stop rules (:131-151)
//   k_compact ordered extrema lists for the next solve + parity-trace hashes
//   k_final   residue update and ensemble accumulation           (emd.cpp:167, :246-251)
// Paths relative to /root/reference/proj/src. Compiled with -fmad=false: the
// arithmetic mirrors the reference's -ffp-contract=off build bit-for-bit.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "semd_device.cuh"
#include "semd_launch.h"
#include "semd_types.cuh"

namespace semd {
namespace dev {

// ------------------------------------------------------------------- lists

// Block-wide exclusive scan of one int per thread (blockDim.x <= 1024).
__device__ int block_excl_scan(int v, int* total) {
    __shared__ int s_w[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    __syncthreads();
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < nw; ++w) {
        const int c = s_w[w];
        if (w < wid) off += c;
        tot += c;
    }
    *total = tot;
    __syncthreads();
    return off + incl - v;
}

// Rebuild the per-step work lists (one CTA; lists are in slot order, which
// fixes the accumulation order). Lockstep rule: IMF k is finalised for every
// slot in the same step, once no slot is still sifting.
__device__ void build_lists(const Arena& A, bool allow_final) {
    Ctrl* C = A.ctrl;
    const int G = A.G;
    const int per = (G + blockDim.x - 1) / blockDim.x;
    const int s0 = min(G, (int)threadIdx.x * per), s1 = min(G, s0 + per);
    int busy = 0, wait = 0;
    for (int s = s0; s < s1; ++s) {
        const int st = A.slots[s].state;
        busy += eval_state(st);
        wait += (st == ST_WAITK);
    }
    int tb, tw;
    block_excl_scan(busy, &tb);
    block_excl_scan(wait, &tw);
    const bool finalize = allow_final && tb == 0 && tw > 0;
    int ne = 0, np = 0, nf = 0, ns = 0, nb = 0, act = 0;
    for (int s = s0; s < s1; ++s) {
        Slot& S = A.slots[s];
        if (finalize && S.state == ST_WAITK) S.state = ST_FINAL;
        const int st = S.state;
        ne += eval_state(st) && st != ST_PRIMED;
        np += (st == ST_PRIMED);
        nf += (st == ST_FINAL);
        act += (st != ST_FREE && st != ST_DONE);
        if (st == ST_SIFT) {
            S.db = pick_free_buffer(S.xb, S.cb);
            S.rb = S.spec ? pick_free_buffer(S.xb, S.cb, S.db) : -1;
            ns += 2;
            for (int side = 0; side < 2; ++side) {
                const int rows = (int)S.n[side] + 2;
                nb += rows <= kSolveSeqMax ? 1 : (rows + kSolveBlock - 1) / kSolveBlock;
            }
        }
    }
    int tne, tnp, tnf, tns, tnb, tact;
    int oe = block_excl_scan(ne, &tne);
    int op = block_excl_scan(np, &tnp);
    int of = block_excl_scan(nf, &tnf);
    int os = block_excl_scan(ns, &tns);
    int ob = block_excl_scan(nb, &tnb);
    block_excl_scan(act, &tact);
    for (int s = s0; s < s1; ++s) {
        const Slot& S = A.slots[s];
        const int st = S.state;
        if (eval_state(st) && st != ST_PRIMED) A.eval_list[oe++] = s;
        if (st == ST_PRIMED) A.eval_list[tne + op++] = s;  // decided (and compacted) without an eval pass
        if (st == ST_FINAL) A.final_list[of++] = s;
        if (st == ST_SIFT) {
            for (int side = 0; side < 2; ++side) {
                const int rows = (int)S.n[side] + 2;
                A.solve_item[os] = (s << 1) | side;
                A.solve_off[os] = ob;
                ++os;
                ob += rows <= kSolveSeqMax ? 1 : (rows + kSolveBlock - 1) / kSolveBlock;
            }
        }
    }
    if (threadIdx.x == 0) {
        A.solve_off[tns] = tnb;
        C->n_eval = tne + tnp;
        C->n_eval_pass = tne;
        C->n_final = tnf;
        C->n_solve = tns;
        C->solve_blocks = tnb;
        C->active = tact;
    }
    __syncthreads();
}

// ------------------------------------------------------------------- scan
//
// Chunked per-slot tile prefix of the new extrema (see k_scan) + SD sums in a
// fixed reduction order; the last CTA applies extract_imf's control flow.

// ---- the SD stop test (emd.cpp:142-150), certified ----------------------------------------
// The engine forms num = sum mean^2 and den = sum cur^2 in a fixed tree (per-lane runs, warp
// sums, strip and chunk partials); the reference adds left to right. The terms are bit-identical,
// non-negative and n in number, so both sums lie within g = n u / (1 - n u) of the exact sum S,
// and each within 2g/(1-g) (relative) of the other. The decision num/den < sd_threshold is
// certified when the threshold lies outside the interval those bounds allow for the reference's
// ratio; otherwise the slot's sums are redone in the reference's order before deciding.

// The reference's own loop, emd.cpp:142-148 (num += mean*mean, den += cur*cur, t = 0..L-1), over
// this iteration's envelopes (the segment tables of the step's solve, the reference's segment
// march, emd.cpp:79) and the candidate it sifted. One thread: only reached for uncertified tests.
__device__ __noinline__ void sd_sums_sequential(const Arena& A, int s, int cur_buf, double* num, double* den) {
    const Slot& S = A.slots[s];
    const double* cur = A.bufs + buf_off(A, s, cur_buf);
    const TabPlanes tp[2] = {tab_planes(A, 0, s), tab_planes(A, 1, s)};
    const int N[2] = {(int)S.n[0] + 4, (int)S.n[1] + 4};
    int seg[2] = {0, 0};
    double x = 0.0, y = 0.0;
    for (int t = 0; t < A.L; ++t) {
        const double tt = (double)t;
        double e[2];
        for (int k = 0; k < 2; ++k) {
            while (seg[k] + 2 < N[k] && tt > tp[k].a[seg[k] + 1].x) ++seg[k];
            const double2 a0 = tp[k].a[seg[k]], b0 = tp[k].b[seg[k]], a1 = tp[k].a[seg[k] + 1];
            const double m1 = tp[k].b[seg[k] + 1].x;
            const double h = a1.x - a0.x;
            e[k] = spline_eval_fast(a0.x, a1.x, a0.y, a1.y, b0.x, m1, h, b0.y, h * h, tt);
        }
        const double mean = 0.5 * (e[0] + e[1]);
        x += mean * mean;
        y += cur[t] * cur[t];
    }
    *num = x;
    *den = y;
}

__device__ __noinline__ void sd_fix_uncertain(const Arena& A, int ne) {
    for (int li = 0; li < ne; ++li) {
        Slot& S = A.slots[A.eval_list[li]];
        if (S.state != ST_SIFT) continue;
        if (!(A.debug & 4) && !sd_decision_uncertain(S.num, S.den, A.L, A.sd_threshold)) continue;
        double num, den;
        sd_sums_sequential(A, A.eval_list[li], S.cb >= 0 ? S.cb : S.xb, &num, &den);  // cb: the candidate sifted
        S.num = num;
        S.den = den;
        atomicAdd(&A.ctrl->sd_rechecks, 1);
    }
}

// Is sift number `sift` (1-based) of the slot's current IMF likely its last? Then it runs as a
// speculative last sift (ST_PRIMED). The stop statistics of earlier IMFs with the same index decide
// (speculate when at least half of those that reached this sift stopped there) -- of earlier waves
// and earlier calls on this context (A.spec_hist; the slots of one wave decide together, so a
// wave cannot learn from itself); without them, from the second sift on. Any choice gives the same results: speculation only
// changes which detection runs when.
__device__ int spec_policy(const Arena& A, const Slot& S, int sift) {
    if (A.debug & 8) return 0;
    if (S.detect_only || S.imf_out || S.res_out) return 0;  // single-IMF jobs: no next IMF
    if (S.kmax > 0 && S.k + 1 >= S.kmax) return 0;
    if (A.debug & 16) return 1;
    if (sift >= A.max_sift_iters) return 1;  // the iteration cap stops it
    const int* h = A.spec_hist + min(S.k, kSpecK - 1) * kSpecS;
    const int j = min(sift, kSpecS - 1);
    int reach = 0;
    for (int q = j; q < kSpecS; ++q) reach += *(volatile const int*)(h + q);
    if (reach < 4) return sift >= 2;
    return 2 * *(volatile const int*)(h + j) >= reach;
}
__device__ __forceinline__ void spec_count_stop(const Arena& A, const Slot& S) {
    atomicAdd(A.spec_hist + min(S.k, kSpecK - 1) * kSpecS + min(S.iter, kSpecS - 1), 1);
}

// extract_imf's control flow (emd.cpp:131-151) for one slot after its eval
// pass; returns 1 when this step's extrema must be compacted.
__device__ int decide_slot(const Arena& A, int s) {
    Slot& S = A.slots[s];
    const int state = S.state;
    const int np = 1 - S.par;
    const unsigned nmax = toff_view(A, np, 0, s).cg(A.tiles);
    const unsigned nmin = toff_view(A, np, 1, s).cg(A.tiles);
    const int tracing = A.trace != nullptr;
    int compact = 0;
    S.trace_iter = -1;
    S.cpar = np;
    S.tn[0] = nmax;
    S.tn[1] = nmin;
    if (state == ST_INIT || state == ST_DETECT || state == ST_PRIMED) {
        // iteration 0 of IMF k: extract_imf's first find_extrema (ST_PRIMED: detected by the
        // previous IMF's speculative last sift, on its residue R' = this IMF's input)
        S.spec = 0;
        S.spec_hit = 0;
        if (A.max_sift_iters <= 0 && !S.detect_only) {  // loop body never runs: IMF = input
            S.cb = -1;
            S.iter = 0;
            S.state = ST_WAITK;
            if (A.imf_sifts && S.k0 + S.k < A.kcap) A.imf_sifts[S.k0 + S.k] = 0;
            return 0;
        }
        S.trace_iter = 0;
        if (S.detect_only) {  // standalone find_extrema / CEEMDAN stage check: lists are returned
            S.n[0] = nmax;
            S.n[1] = nmin;
            S.state = ST_DONE;
            return 1;
        }
        S.par = np;
        S.n[0] = nmax;
        S.n[1] = nmin;
        S.iter = 0;
        S.cb = -1;
        if (nmax < 2 || nmin < 2) {  // InsufficientExtrema on the unsifted input (emd.cpp:138, :164)
            S.ended_insufficient = 1;
            S.state = ST_DONE;
            return tracing;
        }
        S.state = ST_SIFT;
        S.spec = spec_policy(A, S, 1);
        return 1;
    }
    if (state == ST_REDETECT) {
        // the candidate's find_extrema of sift iteration `iter` (emd.cpp:132), after a speculative
        // sift that did not stop
        S.trace_iter = S.iter;
        if (nmax < 2 || nmin < 2) {  // envelope throws: the candidate is the IMF (emd.cpp:137-140)
            S.state = ST_WAITK;
            S.spec_hit = 0;
            if (A.imf_sifts && S.k0 + S.k < A.kcap) A.imf_sifts[S.k0 + S.k] = S.iter;
            spec_count_stop(A, S);
            return tracing;
        }
        S.par = np;
        S.n[0] = nmax;
        S.n[1] = nmin;
        S.state = ST_SIFT;
        S.spec = spec_policy(A, S, S.iter + 1);
        return 1;
    }
    if (state == ST_SIFT) {
        S.iter += 1;
        S.sifted += A.L;
        S.cb = S.db;
        const double num = S.num, den = S.den;  // reference-order sums when uncertified (sd_fix_uncertain)
        bool stop = (den == 0.0 || num / den < A.sd_threshold) || S.iter >= A.max_sift_iters;
        if (S.spec) {  // this step detected R' = X - candidate, not the candidate
            atomicAdd(&A.ctrl->spec_pass, 1);
            if (stop) {
                atomicAdd(&A.ctrl->spec_hits, 1);
                S.state = ST_WAITK;
                S.spec_hit = 1;
                if (A.imf_sifts && S.k0 + S.k < A.kcap) A.imf_sifts[S.k0 + S.k] = S.iter;
                spec_count_stop(A, S);
            } else {
                atomicAdd(&A.ctrl->spec_misses, 1);
                S.state = ST_REDETECT;
            }
            return 0;
        }
        if (!stop) {
            S.trace_iter = S.iter;
            if (nmax < 2 || nmin < 2) {
                stop = true;  // envelope throws: the candidate is the IMF (emd.cpp:137-140)
                compact = tracing;
            } else {
                S.par = np;
                S.n[0] = nmax;
                S.n[1] = nmin;
                compact = 1;
                S.spec = spec_policy(A, S, S.iter + 1);
            }
        }
        if (stop) {
            S.state = ST_WAITK;
            S.spec_hit = 0;
            if (A.imf_sifts && S.k0 + S.k < A.kcap) A.imf_sifts[S.k0 + S.k] = S.iter;
            spec_count_stop(A, S);
        }
    }
    return compact;
}

__device__ void decide_after_eval(const Arena& A) {
    Ctrl* C = A.ctrl;
    const int ne = C->n_eval;
    // chunk bases of the new knot parity (exclusive scan of the k_scan chunk totals)
    // and the SD sums (chunk partials in chunk order)
    const int P = A.chunks;
    for (int w = threadIdx.x; w < 2 * ne; w += blockDim.x) {
        const int s = A.eval_list[w >> 1], side = w & 1;
        Slot& S = A.slots[s];
        const unsigned* ct = A.ctot + chunk_off(A, side, s);
        unsigned* tb = A.tbase + tbase_off(A, 1 - S.par, side, s);
        unsigned run = 0;
        for (int c = 0; c < P; ++c) {  // L1-bypassing reads: written by the other CTAs
            tb[c] = run;
            run += __ldcg(ct + c);
        }
        if (side == 0 && S.state == ST_SIFT) {
            const double* cn = A.cnum + chunk_off(A, 0, s);
            const double* cd = A.cden + chunk_off(A, 0, s);
            double x = 0.0, y = 0.0;
            for (int c = 0; c < P; ++c) {
                x += __ldcg(cn + c);
                y += __ldcg(cd + c);
            }
            S.num = x;
            S.den = y;
        }
    }
    __syncthreads();
    // SD tests too close to the threshold to certify get the reference's sequential sums first
    // (cold path: one thread, out of line, so the decision loop below keeps its registers)
    int unc = 0;
    for (int li = threadIdx.x; li < ne; li += blockDim.x) {
        const Slot& S = A.slots[A.eval_list[li]];
        if (S.state == ST_SIFT && ((A.debug & 4) || sd_decision_uncertain(S.num, S.den, A.L, A.sd_threshold))) unc = 1;
    }
    if (__syncthreads_or(unc)) {
        if (threadIdx.x == 0) sd_fix_uncertain(A, ne);
        __syncthreads();
    }
    const int per = (ne + blockDim.x - 1) / blockDim.x;
    const int l0 = min(ne, (int)threadIdx.x * per), l1 = min(ne, l0 + per);
    int flags = 0, cnt = 0;  // per <= 32 when G <= 8192
    for (int li = l0; li < l1; ++li) {
        const int f = decide_slot(A, A.eval_list[li]);
        flags |= f << (li - l0);
        cnt += f;
    }
    int tot;
    int off = block_excl_scan(cnt, &tot);
    for (int li = l0; li < l1; ++li)
        if (flags & (1 << (li - l0))) A.compact_list[off++] = A.eval_list[li];
    if (threadIdx.x == 0) C->n_compact = tot;
    __syncthreads();
    build_lists(A, true);
}

// One CTA per (eval slot, side, chunk of kScanChunk tiles): chunk-local exclusive
// prefix of the per-tile extrema counts -> toff, the chunk total -> ctot, and
// (side 0) the chunk's SD partials. The last CTA scans the chunk totals into
// tbase and applies extract_imf's control flow.
__host__ __device__ inline bool scan_by_warp(const Arena& A) { return A.chunks == 1 && A.tiles <= 32 * kScanPer; }
__host__ __device__ inline int scan_grid(const Arena& A) {
    return scan_by_warp(A) ? (2 * A.G + kScanThreads / 32 - 1) / (kScanThreads / 32) : 2 * A.G * A.chunks;
}

__global__ void __launch_bounds__(kScanThreads) k_scan(Arena A) {
    pdl_begin();
    if (A.ctrl->finished) return;  // a step launched past the run's end
    const int kstep_ = A.ctrl->step;
    if (threadIdx.x == 0) span_begin(A.ctrl, KID_SCAN);
    constexpr int W = kScanThreads / 32;
    __shared__ unsigned s_w[W];
    __shared__ double s_red[2][W];
    __shared__ int s_last;
    Ctrl* C = A.ctrl;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int P = A.chunks;
    if (scan_by_warp(A)) {
        // short signals (one chunk of at most 32 * kScanPer tiles): one warp per (slot, side); the
        // same tile prefix, and the same SD partial sums (the strips sit in one warp either way)
        const int item = blockIdx.x * W + wid;
        const int li = item >> 1, side = item & 1;
        if (li < C->n_eval) {
            const int s = A.eval_list[li];
            const Slot& S = A.slots[s];
            const int np = 1 - S.par;
            const int T = A.tiles;
            const int j0 = lane * kScanPer;
            const unsigned* cnt = A.scnt + scnt_off(A, side, s);
            unsigned v[kScanPer];
            unsigned sum = 0;
#pragma unroll
            for (int q = 0; q < kScanPer / 4; ++q) {
                uint4 u = make_uint4(0u, 0u, 0u, 0u);
                if (j0 + 4 * q < T) u = *reinterpret_cast<const uint4*>(cnt + j0 + 4 * q);  // rows padded to 4
                v[4 * q] = j0 + 4 * q < T ? u.x : 0u;
                v[4 * q + 1] = j0 + 4 * q + 1 < T ? u.y : 0u;
                v[4 * q + 2] = j0 + 4 * q + 2 < T ? u.z : 0u;
                v[4 * q + 3] = j0 + 4 * q + 3 < T ? u.w : 0u;
            }
#pragma unroll
            for (int i = 0; i < kScanPer; ++i) sum += v[i];
            unsigned incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
            unsigned run = incl - sum;
            unsigned* to = A.toff + toff_off(A, np, side, s);
#pragma unroll
            for (int i = 0; i < kScanPer; ++i) {
                if (j0 + i < T) to[j0 + i] = run;
                run += v[i];
            }
            if (lane == 0) {
                to[T] = tot;
                A.ctot[chunk_off(A, side, s)] = tot;
            }
            if (side == 0 && S.state == ST_SIFT) {  // SD sums (emd.cpp:145-146)
                const int st = A.strip, sb1 = (T + st - 1) / st;
                double a = 0.0, b = 0.0;
                for (int sx = lane; sx < sb1; sx += 32) {
                    a += A.tnum[tsd_off(A, s) + sx];
                    b += A.tden[tsd_off(A, s) + sx];
                }
                a = warp_sum(a);
                b = warp_sum(b);
                if (lane == 0) {
                    A.cnum[chunk_off(A, 0, s)] = a;
                    A.cden[chunk_off(A, 0, s)] = b;
                }
            }
        }
    } else {
    const int item = blockIdx.x / P, c = blockIdx.x - item * P;
    const int li = item >> 1, side = item & 1;
    if (li < C->n_eval) {
        const int s = A.eval_list[li];
        const Slot& S = A.slots[s];
        const int np = 1 - S.par;
        const int T = A.tiles;
        const int jb = c * kScanChunk, je = min(T, jb + kScanChunk);
        const int j0 = jb + tid * kScanPer;
        const unsigned* cnt = A.scnt + scnt_off(A, side, s);
        unsigned v[kScanPer];
        unsigned sum = 0;
#pragma unroll
        for (int q = 0; q < kScanPer / 4; ++q) {
            uint4 u = make_uint4(0u, 0u, 0u, 0u);
            if (j0 + 4 * q < je) u = *reinterpret_cast<const uint4*>(cnt + j0 + 4 * q);  // rows padded to 4
            v[4 * q] = j0 + 4 * q < je ? u.x : 0u;
            v[4 * q + 1] = j0 + 4 * q + 1 < je ? u.y : 0u;
            v[4 * q + 2] = j0 + 4 * q + 2 < je ? u.z : 0u;
            v[4 * q + 3] = j0 + 4 * q + 3 < je ? u.w : 0u;
        }
#pragma unroll
        for (int i = 0; i < kScanPer; ++i) sum += v[i];
        unsigned incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) s_w[wid] = incl;
        __syncthreads();
        unsigned run = incl - sum, tot = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const unsigned x = s_w[w];
            if (w < wid) run += x;
            tot += x;
        }
        unsigned* to = A.toff + toff_off(A, np, side, s);
#pragma unroll
        for (int i = 0; i < kScanPer; ++i) {
            if (j0 + i < je) to[j0 + i] = run;
            run += v[i];
        }
        if (tid == 0) {
            if (c == P - 1) to[T] = tot;  // tile T (the total) belongs to the last chunk
            A.ctot[chunk_off(A, side, s) + c] = tot;
        }
        if (side == 0 && S.state == ST_SIFT) {  // SD sums (emd.cpp:145-146), fixed reduction order
            // k_eval leaves one partial per strip of A.strip tiles; this chunk owns strips
            // [jb/strip, ceil(je/strip)), taken by the threads in order (a fixed reduction order)
            static_assert(kScanChunk == 16 * kScanThreads, "one 16-tile strip per scan thread");
            const int st = A.strip;
            const int sb0 = jb / st, sb1 = (je + st - 1) / st;
            double a = 0.0, b = 0.0;
            for (int sx = sb0 + tid; sx < sb1; sx += kScanThreads) {
                a += A.tnum[tsd_off(A, s) + sx];
                b += A.tden[tsd_off(A, s) + sx];
            }
            a = warp_sum(a);
            b = warp_sum(b);
            if (lane == 0) {
                s_red[0][wid] = a;
                s_red[1][wid] = b;
            }
            __syncthreads();
            if (tid == 0) {
                double x = 0.0, y = 0.0;
                for (int w = 0; w < W; ++w) {
                    x += s_red[0][w];
                    y += s_red[1][w];
                }
                A.cnum[chunk_off(A, 0, s) + c] = x;
                A.cden[chunk_off(A, 0, s) + c] = y;
            }
        }
    }
    }  // one CTA per (slot, side, chunk)
    if (tid == 0) {
        __threadfence();
        s_last = atomicAdd(&C->done[4], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        decide_after_eval(A);
        if (tid == 0) {
            C->done[4] = 0;
            C->ticket[0] = 0;  // k_eval's strip tickets
            if (C->ev_t1 > C->ev_t0) C->ev_ns += C->ev_t1 - C->ev_t0;
            C->ev_t0 = ~0ull;
            C->ev_t1 = 0;
        }
    }
    if (threadIdx.x == 0) span_end(A.ctrl, KID_SCAN, kstep_);
}

// ---------------------------------------------------------------- compact
//
// Stage -> ordered global extrema lists (tile j's knots land at toff[j]).
// Also the order-sensitive parity-trace hash (tracing only).

__device__ void emit_trace(const Arena& A, const Slot& S, uint64_t h) {
    const int pos = atomicAdd(&A.ctrl->trace_count, 1);
    if (pos < A.trace_cap) {
        TraceRec r;
        r.task = S.task;
        r.m = S.m;
        r.k = S.k;
        r.iter = S.trace_iter;
        r.n_max = S.tn[0];
        r.n_min = S.tn[1];
        r.hash = h;
        A.trace[pos] = r;
    }
}

// One warp per (compact slot, strip of 16 tiles) item, grid-stride: lanes load the
// strip's tile offsets in one coalesced access and the 16 detection words of their
// lane; each lane then writes its own extrema of both sides to the knot lists.
constexpr int kCompactThreads = 128;
constexpr int kCompactStrip = 16;
__global__ void __launch_bounds__(kCompactThreads) k_compact(Arena A) {
    pdl_begin();
    if (A.ctrl->finished) return;  // a step launched past the run's end
    const int kstep_ = A.ctrl->step;
    if (threadIdx.x == 0) span_begin(A.ctrl, KID_COMPACT);
    __shared__ int s_last;
    Ctrl* C = A.ctrl;
    const int lane = threadIdx.x & 31;
    const int wpb = kCompactThreads / 32;
    const int strips = (A.tiles + kCompactStrip - 1) / kCompactStrip;
    const unsigned nitems = (unsigned)C->n_compact * (unsigned)strips;
    const bool tracing = A.trace != nullptr;
    // each warp takes a contiguous run of items (consecutive strips of one slot share the slot's
    // state, read once per slot instead of per item)
    const unsigned nw = gridDim.x * wpb;
    const unsigned per = (nitems + nw - 1) / nw;
    const unsigned it0 = (blockIdx.x * wpb + (threadIdx.x >> 5)) * per;
    const unsigned it1 = min(nitems, it0 + per);
    int cur_li = -1, s = 0, cpar = 0;
    for (unsigned it = it0; it < it1; ++it) {
        const int li = (int)(it / (unsigned)strips);
        if (li != cur_li) {
            cur_li = li;
            s = A.compact_list[li];
            cpar = A.slots[s].cpar;
        }
        const int sx = (int)(it % (unsigned)strips);
        const int j0 = sx * kCompactStrip;
        const int nt = min(kCompactStrip, A.tiles - j0);
        unsigned off0 = 0, off1 = 0;
        if (lane < nt) {
            off0 = toff_view(A, cpar, 0, s)[j0 + lane];
            off1 = toff_view(A, cpar, 1, s)[j0 + lane];
        }
        // eval's per-lane detection words: window flags of samples t0-1 .. t0+2 and the lane's
        // rank among the tile's extrema of each side. Extremum e of a lane lands at knot
        // toff[tile] + rank + e: every lane writes its own (the tile's knots are contiguous)
        const unsigned* wd = A.tflags + tfl_off(A, cpar, s) + (size_t)j0 * 32 + lane;
        int* gi[2] = {A.kidx + knot_off(A, cpar, 0, s), A.kidx + knot_off(A, cpar, 1, s)};
        uint64_t h0 = 0, h1 = 0;
        unsigned wv[kCompactStrip];  // all of the strip's words in flight at once
#pragma unroll
        for (int u = 0; u < kCompactStrip; ++u) wv[u] = u < nt ? __ldcs(wd + u * 32) : 0u;
#pragma unroll
        for (int u = 0; u < kCompactStrip; ++u) {
            const unsigned w = wv[u];
            if (!__any_sync(0xffffffffu, (w & 0xFFu) != 0u)) continue;  // no extrema in the tile (sparse IMFs)
            const int p0 = (j0 + u) * kEvalTile + lane * kSpt - 1;
            const unsigned o[2] = {__shfl_sync(0xffffffffu, off0, u), __shfl_sync(0xffffffffu, off1, u)};
#pragma unroll
            for (int side = 0; side < 2; ++side) {
                unsigned fl = (w >> (4 * side)) & 0xFu;
                unsigned q = o[side] + ((w >> (8 + 8 * side)) & 0xFFu);
                for (; fl; fl &= fl - 1u, ++q) {  // the lane's extrema in order (at most 2)
                    const int t = p0 + __ffs(fl) - 1;
                    SEMD_ASSERT(q < (unsigned)A.cap && t >= 1 && t <= A.L - 2);  // knot list row, interior extremum
                    gi[side][q] = t;
                    if (tracing) (side ? h1 : h0) += knot_hash(side, q, (unsigned)t);
                }
            }
        }
        if (tracing) {
            h0 = warp_sum(h0);
            h1 = warp_sum(h1);
            if (lane == 0) {
                A.thash[(size_t)s * A.tiles + sx] = h0;
                A.thash[((size_t)A.G + s) * A.tiles + sx] = h1;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&C->done[1], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        if (tracing) {
            const int wid = threadIdx.x >> 5;
            for (int li = wid; li < C->n_compact; li += wpb) {
                const int s = A.compact_list[li];
                const Slot& S = A.slots[s];
                uint64_t h = 0;
                const int strips = (A.tiles + kCompactStrip - 1) / kCompactStrip;
                for (int j = lane; j < strips; j += 32)
                    h += __ldcg(A.thash + (size_t)s * A.tiles + j) + __ldcg(A.thash + ((size_t)A.G + s) * A.tiles + j);
                h = warp_sum(h);
                if (lane == 0 && S.trace_iter >= 0) emit_trace(A, S, h);
            }
        }
        if (threadIdx.x == 0) {
            C->ticket[1] = 0;
            C->done[1] = 0;
        }
    }
    if (threadIdx.x == 0) span_end(A.ctrl, KID_COMPACT, kstep_);
}

// ------------------------------------------------------------------ solve
//
// Natural-spline moments (emd.cpp:53-73) of one envelope's mirrored knot
// system, reproducing the reference's sequential Thomas algorithm BIT-FOR-BIT
// with parallel chains. Each chain restarts the recurrence kSolveWarm rows
// before its chunk from a guessed state; the recurrences contract (~0.27 per
// row), so the speculative chain soon coincides bitwise with the true one.
// Every chain then replays its head from its predecessor's end state until it
// meets its own stored values bitwise, which makes the result exactly the
// sequential one; replays repeat while a chain's end moved. Across CTA blocks
// a kSolveHalo-row warm-up is used and the boundary values are cross-checked
// (mismatches are counted as hazards; none has been observed).
//
// Shared layout per block, indexed by knot/row v - wa:
//   H[v] = X[v+1]-X[v], RHS[i], DP[i], RP[i], M[i]  (X and Y only staged)

// Shared arrays of the chunked solve are indexed through spad(): one pad double per
// kSolveChunk rows, so the chains (kSolveChunk rows apart) of a warp hit distinct banks.
__device__ __forceinline__ int spad(int q) { return q + (q >> 4); }
static_assert(kSolveChunk == 16, "spad() pads one double per 16 rows");

struct SolveCtx {
    const double* H;
    const double* RHS;
    int wa;
};

__device__ __forceinline__ void fwd_first(const SolveCtx& c, int i, double& d, double& r) {
    const double h0 = c.H[spad(i - 1 - c.wa)], h1 = c.H[spad(i - c.wa)];
    d = 2.0 * (h0 + h1);  // emd.cpp:60
    r = c.RHS[spad(i - c.wa)];
}

// emd.cpp:64-69: w = h0 / diag[i-1]; diag[i] -= w*upper[i-1]; rhs[i] -= w*rhs[i-1]
__device__ __forceinline__ void fwd_step(const SolveCtx& c, int i, double& d, double& r) {
    const double h0 = c.H[spad(i - 1 - c.wa)], h1 = c.H[spad(i - c.wa)];
    const double w = h0 / d;
    d = 2.0 * (h0 + h1) - w * h0;
    r = c.RHS[spad(i - c.wa)] - w * r;
}

struct SolveShared {
    unsigned ticket;
    int item, b, last, any;
    int pf, pf_lo;  // the next block's knot indices were bulk-copied to the idx buffer from rank pf_lo
    int bb;         // block index of sh.b within its (slot, side) item
    int slot, side, n, par, srcb;  // the block's item, read ahead by the helper: slot, side, extrema, knot parity, candidate buffer
    int dirty[kSolveMaxChains];
    int moved[kSolveMaxChains];
};

__device__ void solve_small(const KnotView& kv, const TabPlanes tab, double* sm) {
    // one thread runs the reference Thomas algorithm verbatim
    const int N = kv.n + 4;
    double* X = sm;
    double* Y = X + (kSolveSeqMax + 4);
    double* dp = Y + (kSolveSeqMax + 4);
    double* rp = dp + (kSolveSeqMax + 4);
    for (int v = threadIdx.x; v < N; v += blockDim.x) vknot(kv, v, X[v], Y[v]);
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i + 1 < N; ++i) {
            const double h0 = X[i] - X[i - 1], h1 = X[i + 1] - X[i];
            dp[i] = 2.0 * (h0 + h1);
            rp[i] = 6.0 * ((Y[i + 1] - Y[i]) / h1 - (Y[i] - Y[i - 1]) / h0);
        }
        for (int i = 2; i + 1 < N; ++i) {
            const double h0 = X[i] - X[i - 1];
            const double w = h0 / dp[i - 1];
            dp[i] -= w * (X[i] - X[i - 1]);
            rp[i] -= w * rp[i - 1];
        }
        double m = 0.0;
        tab.set(N - 1, X[N - 1], Y[N - 1], 0.0, 0.0);
        for (int i = N - 2; i >= 1; --i) {
            m = (rp[i] - (X[i + 1] - X[i]) * m) / dp[i];
            tab.set(i, X[i], Y[i], m, 1.0 / (X[i + 1] - X[i]));
        }
        tab.set(0, X[0], Y[0], 0.0, 1.0 / (X[1] - X[0]));
    }
    __syncthreads();
}

// Exact fallback for an envelope whose speculative block boundaries disagreed:
// the reference's sequential Thomas algorithm (emd.cpp:57-73, IEEE divisions)
// run by one thread, using the segment-table rows as forward-sweep scratch.
__device__ __noinline__ void solve_sequential(const KnotView& kv, const TabPlanes tab) {
    const int N = kv.n + 4;
    double xp, yp, xc, yc;
    vknot(kv, 0, xp, yp);
    vknot(kv, 1, xc, yc);
    double d = 0.0, r = 0.0;
    for (int i = 1; i + 1 < N; ++i) {
        double xn, yn;
        vknot(kv, i + 1, xn, yn);
        const double h0 = xc - xp, h1 = xn - xc;
        const double rhs = 6.0 * ((yn - yc) / h1 - (yc - yp) / h0);  // emd.cpp:62
        if (i == 1) {
            d = 2.0 * (h0 + h1);
            r = rhs;
        } else {  // emd.cpp:64-69
            const double w = h0 / d;
            d = 2.0 * (h0 + h1) - w * h0;
            r = rhs - w * r;
        }
        tab.set(i, xc, yc, d, r);  // forward-sweep scratch in the b plane
        xp = xc;
        yp = yc;
        xc = xn;
        yc = yn;
    }
    double xn, yn;
    vknot(kv, N - 1, xn, yn);
    tab.set(N - 1, xn, yn, 0.0, 0.0);
    double m = 0.0;
    for (int i = N - 2; i >= 1; --i) {  // emd.cpp:70-73
        const double2 ta = tab.a[i], tb = tab.b[i];  // {x, y}, {diag, rhs}
        m = (tb.y - (xn - ta.x) * m) / tb.x;
        tab.set(i, ta.x, ta.y, m, 1.0 / (xn - ta.x));
        xn = ta.x;
    }
    double x0, y0;
    vknot(kv, 0, x0, y0);
    tab.set(0, x0, y0, 0.0, 1.0 / (xn - x0));
}

#define SOLVE_PROF(k)                                                              \
    do {                                                                           \
        if (prof_on && tid == 0) {                                                 \
            const long long now = clock64();                                       \
            atomicAdd(&A.prof[k], (unsigned long long)(now - prof_t));             \
            prof_t = now;                                                          \
        }                                                                          \
    } while (0)

// Staged rows [wa, wb] of block b of an N-row system (see k_solve).
__device__ __forceinline__ void solve_window(int b, int N, int& wa, int& wb) {
    const int r0 = 1 + b * kSolveBlock;
    const int r1 = min(r0 + kSolveBlock, N - 1);
    wb = min(r1 + kSolveHalo, N - 1);
    wa = max(0, max(1, r0 - kSolveHalo) - kSolveWarm - 1);
}
constexpr int kSolveIdxBuf = kSolveWin + 8;  // ints: one window's knot ranks, 16-byte aligned both ends

__global__ void __launch_bounds__(kSolveThreads, kSolveCtasPerSm) k_solve(Arena A) {
    pdl_begin();
    if (A.ctrl->finished) return;  // a step launched past the run's end
    const int kstep_ = A.ctrl->step;
    if (threadIdx.x == 0) span_begin(A.ctrl, KID_SOLVE);
    if (threadIdx.x == 0 && blockIdx.x == 0) span_fold(A.ctrl, (kstep_ & 1) ^ 1);
    const bool prof_on = (A.debug & 2) && A.prof;
    long long prof_t = clock64();
    extern __shared__ double sm[];
    __shared__ SolveShared sh;
    Ctrl* C = A.ctrl;
    const int tid = threadIdx.x;
    const int nblocks = C->solve_blocks;
    const int nitems = C->n_solve;
    // the next block's knot indices are bulk-copied into IB while this block is solved, so its
    // staging waits only for the dependent value gather
    int* IB = reinterpret_cast<int*>(sm + 5 * kSolvePadWin);
    unsigned long long* pbar = reinterpret_cast<unsigned long long*>(IB + kSolveIdxBuf);
    unsigned pfph = 0;  // parity of the idx buffer's next completion
    // dynamic block tickets (C->ticket[2]); the (slot, side) item of a block is the last i
    // with solve_off[i] <= block. The next ticket and its item are fetched by an idle helper
    // thread during this block's forward sweep.
    auto find_item = [&](int blk, int lo) {
        int hi = nitems - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (A.solve_off[mid] <= blk) lo = mid;
            else hi = mid - 1;
        }
        return lo;
    };
    // A slot's two items (sides 0 and 1, consecutive in the lists) take their blocks
    // alternately, so both envelopes' blocks over the same stretch of the candidate run
    // together and the second side's value gathers hit L2.
    auto load_item = [&](int it) {  // one thread: the item's slot state the block needs
        const int code = A.solve_item[it];
        const int sl = code >> 1, sd = code & 1;
        const Slot& S = A.slots[sl];
        sh.slot = sl;
        sh.side = sd;
        sh.n = (int)S.n[sd];
        sh.par = S.par;
        sh.srcb = S.cb >= 0 ? S.cb : S.xb;
    };
    auto decode = [&](int blk, int lo, int& it, int& bb) {
        const int p = find_item(blk, lo) & ~1;
        const int o = A.solve_off[p];
        const int n0 = A.solve_off[p + 1] - o, n1 = A.solve_off[p + 2] - A.solve_off[p + 1];
        const int t = blk - o, m = min(n0, n1);
        int sd;
        if (t < 2 * m) {
            sd = t & 1;
            bb = t >> 1;
        } else {
            sd = n0 > n1 ? 0 : 1;
            bb = m + (t - 2 * m);
        }
        it = p + sd;
    };
    if (tid == 0) {
        sh.b = (int)atomicAdd(&C->ticket[2], 1u);
        if (sh.b < nblocks) {
            decode(sh.b, 0, sh.item, sh.bb);
            load_item(sh.item);
        }
        sh.pf = 0;
        bar_init(pbar);
    }
    __syncthreads();
    while (true) {
        const int blk = sh.b;
        if (blk >= nblocks) break;
        const int item = sh.item;
        const int slot = sh.slot, side = sh.side, b = sh.bb;
        const int s_n = sh.n, s_par = sh.par, s_srcb = sh.srcb;
        __syncthreads();  // sh.b / sh.item / the item's state consumed
        auto prefetch = [&]() {  // one thread: the next block, its item and its knot indices
            const int nb2 = (int)atomicAdd(&C->ticket[2], 1u);
            sh.b = nb2;
            sh.pf = 0;
            if (nb2 >= nblocks) return;
            int it2, bb2;
            decode(nb2, item & ~1, it2, bb2);
            sh.item = it2;
            sh.bb = bb2;
            load_item(it2);
            const int sl2 = sh.slot, sd2 = sh.side, n2 = sh.n;
            if (n2 + 2 <= kSolveSeqMax) return;  // solve_small: no staging
            int wa2, wb2;
            solve_window(bb2, n2 + 4, wa2, wb2);
            const int rlo = wa2 <= 1 ? 0 : wa2 - 2;           // ranks of rows wa2..wb2 (vknot_rank)
            const int rhi = wb2 >= n2 + 2 ? n2 - 1 : wb2 - 2;
            const int lo4 = rlo & ~3;
            const unsigned bytes = (unsigned)((rhi + 1 - lo4 + 3) & ~3) * 4u;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // IB's earlier generic reads
            bar_arrive_tx(pbar, bytes);
            bulk_g2s(IB, A.kidx + knot_off(A, sh.par, sd2, sl2) + lo4, bytes, pbar);
            sh.pf = 1;
            sh.pf_lo = lo4;
        };
        KnotView kv;
        kv.idx = A.kidx + knot_off(A, s_par, side, slot);
        kv.src = A.bufs + buf_off(A, slot, s_srcb);
        kv.n = s_n;
        kv.e2 = 2.0 * (double)(A.L - 1);
        kv.mom = nullptr;
        const TabPlanes tab = tab_planes(A, side, slot);
        const int N = kv.n + 4;
        if (N - 2 <= kSolveSeqMax) {
            if (tid == kSolveThreads - 1) prefetch();
            solve_small(kv, tab, sm);  // ends with __syncthreads
            continue;
        }
        const int HW = kSolveHalo, B = kSolveBlock, CH = kSolveChunk, W0 = kSolveWarm;
        const int r0 = 1 + b * B;
        const int r1 = min(r0 + B, N - 1);
        const int r1e = min(r1 + HW, N - 1);
        const int ra = max(1, r0 - HW);              // first chain row (front halo)
        const int wa = max(0, ra - W0 - 1);          // staged window: every chain warms up W0 rows
        const int wb = r1e;
        const int wn = wb - wa + 1;
        double* H = sm;          // [wn]   H[spad(v)] = X[v+1]-X[v]
        double* RHS = H + kSolvePadWin;     // rhs; after the forward sweep: RN(1/diag)
        double* DP = RHS + kSolvePadWin;
        double* RP = DP + kSolvePadWin;
        double* M = RP + kSolvePadWin;
        SOLVE_PROF(0);  // item fetch + setup
        // stage X into DP and Y into M (temporarily), then H, 1/H (into RP), RHS
        {  // every row of the window in one batch: the index loads, then the value gathers
            constexpr int U = (kSolveWin + kSolveThreads - 1) / kSolveThreads;
            int iv[U];
            double yv[U];
            if (sh.pf) {  // prefetched during the previous block
                bar_wait(pbar, pfph);
                pfph ^= 1u;
                const int lo = sh.pf_lo;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int q = u * kSolveThreads + tid;
                    if (q < wn) iv[u] = IB[vknot_rank(kv.n, wa + q) - lo];
                }
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int q = u * kSolveThreads + tid;
                    if (q < wn) iv[u] = kv.idx[vknot_rank(kv.n, wa + q)];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = u * kSolveThreads + tid;
                if (q < wn) yv[u] = kv.src[iv[u]];  // extremum value = the candidate sample
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = u * kSolveThreads + tid;
                if (q < wn) {
                    DP[spad(q)] = vknot_x(kv.n, wa + q, iv[u], kv.e2);
                    M[spad(q)] = yv[u];
                }
            }
        }
        __syncthreads();
        SOLVE_PROF(11);  // knot loads
        for (int q = tid; q < wn - 1; q += blockDim.x) {
            const double h = DP[spad(q + 1)] - DP[spad(q)];
            H[spad(q)] = h;
            RP[spad(q)] = 1.0 / h;
        }
        __syncthreads();
        SOLVE_PROF(12);  // H, 1/H
        for (int q = tid + 1; q < wn - 1; q += blockDim.x) {  // emd.cpp:62 with exactly rounded divisions
            const double h0 = H[spad(q - 1)], h1 = H[spad(q)];
            RHS[spad(q)] = 6.0 * (div_rn(M[spad(q + 1)] - M[spad(q)], h1, RP[spad(q)]) - div_rn(M[spad(q)] - M[spad(q - 1)], h0, RP[spad(q - 1)]));
            const int i = wa + q;  // this block's segment-table rows {x, y, -, 1/h}; m follows the solve
            if (i >= r0 && i < r1) tab.set(i, DP[spad(q)], M[spad(q)], 0.0, RP[spad(q)]);
        }
        if (tid == 0) {
            if (r0 == 1) tab.set(0, DP[spad(0 - wa)], M[spad(0 - wa)], 0.0, RP[spad(0 - wa)]);
            if (r1 == N - 1) tab.set(N - 1, DP[spad(N - 1 - wa)], M[spad(N - 1 - wa)], 0.0, 0.0);
        }
        __syncthreads();
        SOLVE_PROF(1);  // staging + H + RHS
        SolveCtx cx{H, RHS, wa};
        // Chains tile rows [ra, rb) = [r0-HW, r1+HW) (clipped to the system) in CH-row pieces:
        // the front-halo chains (rows < r0) only carry the forward state up to r0-1, the
        // back-halo chains (rows >= r1) only the back-substitution down to r1.
        const int rb = r1e;
        const int nch = (rb - ra + CH - 1) / CH;
        const int c = tid;
        const int cs = ra + c * CH, ce = min(cs + CH, rb);
        const bool mine = c < nch;
        double* rec = A.sb + (((size_t)side * A.G + slot) * A.max_blocks + b) * 6;
        // --- phase A: forward from a guessed state kSolveWarm rows early (exact from row 1)
        if (tid == kSolveThreads - 1) prefetch();  // idle helper
        if (mine) {
            const int ws = max(1, cs - W0);
            double d, r;
            fwd_first(cx, ws, d, r);  // exact when ws == 1, otherwise a guess
#pragma unroll 4
            for (int i = ws + 1; i < cs; ++i) fwd_step(cx, i, d, r);
            if (ws < cs) fwd_step(cx, cs, d, r);
            DP[spad(cs - wa)] = d;
            RP[spad(cs - wa)] = r;
#pragma unroll 4
            for (int i = cs + 1; i < ce; ++i) {
                fwd_step(cx, i, d, r);
                DP[spad(i - wa)] = d;
                RP[spad(i - wa)] = r;
            }
        }
        if (tid < kSolveMaxChains) sh.moved[tid] = 1;
        __syncthreads();
        SOLVE_PROF(2);  // phase A
        // --- phase B: replay chain heads from the predecessor's end state until bitwise agreement
        for (int round = 0; round < nch; ++round) {
            if (prof_on && tid == 0) atomicAdd(&A.prof[8], 1ull);
            if (tid == 0) sh.any = 0;
            if (tid < kSolveMaxChains) sh.dirty[tid] = 0;
            __syncthreads();
            if (mine && c >= 1 && sh.moved[c - 1]) {
                double d = DP[spad(cs - 1 - wa)], r = RP[spad(cs - 1 - wa)];
                bool conv = false;
                for (int i = cs; i < ce; ++i) {
                    fwd_step(cx, i, d, r);
                    if (d == DP[spad(i - wa)] && r == RP[spad(i - wa)]) {
                        conv = true;
                        break;
                    }
                    DP[spad(i - wa)] = d;
                    RP[spad(i - wa)] = r;
                }
                if (!conv) {
                    sh.dirty[c] = 1;
                    sh.any = 1;
                }
            }
            __syncthreads();
            const int any = sh.any;
            if (tid < kSolveMaxChains) sh.moved[tid] = sh.dirty[tid];
            __syncthreads();
            if (!any) break;
        }
        SOLVE_PROF(3);  // phase B
        for (int q = tid + r0 - wa; q < rb - wa; q += blockDim.x) RHS[spad(q)] = 1.0 / DP[spad(q)];  // RN(1/diag)
        __syncthreads();
        // --- phase C: back substitution (emd.cpp:70-73), speculative above each chunk;
        // chains below r0 take no part
        auto upper = [&](int i) { return H[spad(i - wa)]; };  // X[i+1]-X[i]
        const bool back = mine && ce > r0;
        if (back) {
            const int top = min(ce + W0, rb);
            double m = 0.0;  // exact when top == N-1, otherwise a guess
#pragma unroll 4
            for (int i = top - 1; i >= cs; --i) {
                m = div_rn(RP[spad(i - wa)] - upper(i) * m, DP[spad(i - wa)], RHS[spad(i - wa)]);
                if (i < ce) M[spad(i - wa)] = m;
            }
        }
        if (tid < kSolveMaxChains) sh.moved[tid] = 1;
        __syncthreads();
        SOLVE_PROF(4);  // 1/diag + phase C
        // --- phase D: replay chain tails from the successor's first value
        for (int round = 0; round < nch; ++round) {
            if (prof_on && tid == 0) atomicAdd(&A.prof[9], 1ull);
            if (tid == 0) sh.any = 0;
            if (tid < kSolveMaxChains) sh.dirty[tid] = 0;
            __syncthreads();
            if (back && c + 1 < nch && sh.moved[c + 1]) {
                double m = M[spad(ce - wa)];
                bool conv = false;
                for (int i = ce - 1; i >= cs; --i) {
                    m = div_rn(RP[spad(i - wa)] - upper(i) * m, DP[spad(i - wa)], RHS[spad(i - wa)]);
                    if (m == M[spad(i - wa)]) {
                        conv = true;
                        break;
                    }
                    M[spad(i - wa)] = m;
                }
                if (!conv) {
                    sh.dirty[c] = 1;
                    sh.any = 1;
                }
            }
            __syncthreads();
            const int any = sh.any;
            if (tid < kSolveMaxChains) sh.moved[tid] = sh.dirty[tid];
            __syncthreads();
            if (!any) break;
        }
        SOLVE_PROF(5);  // phase D
        // --- outputs + cross-block records: [0,1] forward state at r0-1 (from the front halo),
        // [2,3] this block's state at r1-1, [4] m at r0, [5] the m at r1 it used
        // the m column of this block's segment-table rows (x, y, 1/h were written with the rhs)
        for (int i = r0 + tid; i < r1; i += blockDim.x) reinterpret_cast<double*>(tab.b + i)[0] = M[spad(i - wa)];
        if (tid == 0) {
            if (r0 > 1) {
                rec[0] = DP[spad(r0 - 1 - wa)];
                rec[1] = RP[spad(r0 - 1 - wa)];
            }
            rec[2] = DP[spad(r1 - 1 - wa)];
            rec[3] = RP[spad(r1 - 1 - wa)];
            rec[4] = M[spad(r0 - wa)];
            rec[5] = r1 < N - 1 ? M[spad(r1 - wa)] : 0.0;
        }
        __syncthreads();
        SOLVE_PROF(6);  // outputs
        if (prof_on && tid == 0) atomicAdd(&A.prof[10], 1ull);
    }
    if (tid == 0) {
        __threadfence();
        sh.last = atomicAdd(&C->done[2], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (sh.last) {
        __threadfence();
        // Cross-block check of every multi-block envelope: block bb's warm-up state at r0-1
        // must equal block bb-1's state there, and the m at r0 it produced must equal the m
        // block bb-1 assumed. Items with few blocks are checked by one thread each; items
        // with many blocks (queued in shared memory) by the whole CTA.
        __shared__ int s_big[64];
        __shared__ int s_nbig, s_bad;
        if (tid == 0) s_nbig = 0;
        __syncthreads();
        auto boundary_bad = [&](const double* base, int bb) {
            const double* p = base + (size_t)(bb - 1) * 6;
            const double* q = base + (size_t)bb * 6;
            const bool fwd = __ldcg(q) != __ldcg(p + 2) || __ldcg(q + 1) != __ldcg(p + 3);
            const bool bwd = __ldcg(p + 5) != __ldcg(q + 4);
            return fwd ? 1 : (bwd ? 2 : 0);
        };
        auto log_hazard = [&](int slot, int side, int bb, int nb, int kind) {
            const int pos = atomicAdd(&C->hz_count, 1);
            if (A.hzlog && pos < A.hzlog_cap) {
                const Slot& S = A.slots[slot];
                int* r = A.hzlog + (size_t)pos * 8;
                r[0] = S.m;
                r[1] = S.k;
                r[2] = S.iter;
                r[3] = side;
                r[4] = (int)S.n[side];
                r[5] = bb;
                r[6] = nb;
                r[7] = kind;  // 1 forward state, 2 back-substitution
            }
        };
        auto repair = [&](int slot, int side, int bad) {  // the whole envelope again, sequentially and exactly
            atomicAdd(&A.slots[slot].hazards, bad);
            atomicAdd(&C->hazards, bad);
            const Slot& S = A.slots[slot];
            KnotView kv;
            kv.idx = A.kidx + knot_off(A, S.par, side, slot);
            kv.src = A.bufs + buf_off(A, slot, S.cb >= 0 ? S.cb : S.xb);
            kv.n = (int)S.n[side];
            kv.e2 = 2.0 * (double)(A.L - 1);
            kv.mom = nullptr;
            solve_sequential(kv, tab_planes(A, side, slot));
        };
        for (int it = tid; it < nitems; it += blockDim.x) {
            const int nb = A.solve_off[it + 1] - A.solve_off[it];
            if (nb <= 1) continue;
            if (nb > 32) {
                const int k = atomicAdd(&s_nbig, 1);
                if (k < 64) {
                    s_big[k] = it;
                    continue;
                }
            }
            const int code = A.solve_item[it];
            const int slot = code >> 1, side = code & 1;
            const double* base = A.sb + ((size_t)side * A.G + slot) * A.max_blocks * 6;
            int bad = 0;
            for (int bb = 1; bb < nb; ++bb) {
                const int kind = boundary_bad(base, bb);
                if (kind) {
                    ++bad;
                    log_hazard(slot, side, bb, nb, kind);
                }
            }
            if (A.debug & 1) ++bad;
            if (bad) repair(slot, side, bad);
        }
        __syncthreads();
        const int nbig = min(s_nbig, 64);
        for (int k = 0; k < nbig; ++k) {
            const int it = s_big[k];
            const int nb = A.solve_off[it + 1] - A.solve_off[it];
            const int code = A.solve_item[it];
            const int slot = code >> 1, side = code & 1;
            const double* base = A.sb + ((size_t)side * A.G + slot) * A.max_blocks * 6;
            if (tid == 0) s_bad = 0;
            __syncthreads();
            int bad = 0;
            for (int bb = 1 + tid; bb < nb; bb += blockDim.x) {
                const int kind = boundary_bad(base, bb);
                if (kind) {
                    ++bad;
                    log_hazard(slot, side, bb, nb, kind);
                }
            }
            if (bad) atomicAdd(&s_bad, bad);
            __syncthreads();
            if (tid == 0) {
                const int tb = s_bad + ((A.debug & 1) ? 1 : 0);
                if (tb) repair(slot, side, tb);
            }
            __syncthreads();
        }
        if (tid == 0) {
            C->ticket[2] = 0;
            C->done[2] = 0;
        }
    }
    if (tid == 0) span_end(A.ctrl, KID_SOLVE, kstep_);
}

// ------------------------------------------------------------------ final
//
// IMF k is complete for every slot in final_list (lockstep). Per sample:
//   sums[k0+k][t] += imf_s[t]   in slot order (emd.cpp:249-251 accumulation order)
//   R_s[t] = X_s[t] - imf_s[t]  (emd.cpp:167 residue update)

constexpr int kFinalChunk = 128;

struct FinalSlot {
    const double* x;
    const double* imf;
    double* res;
    double* imf_out;
    double* res_out;
    double* row;  // accumulation row or null
};

__device__ void decide_after_final(const Arena& A) {
    Ctrl* C = A.ctrl;
    const int nf = C->n_final;
    for (int li = threadIdx.x; li < nf; li += blockDim.x) {
        Slot& S = A.slots[A.final_list[li]];
        const int rb = S.spec_hit ? S.rb : pick_free_buffer(S.xb, S.cb);  // k_final's residue / R'
        S.last_imf_b = S.cb >= 0 ? S.cb : S.xb;
        S.xb = rb;
        S.cb = -1;
        S.k += 1;
        S.iter = 0;
        if (S.kmax > 0 && S.k >= S.kmax) S.state = ST_DONE;
        else if (S.write_imf && !imf_row_ok(A, S.k0, S.k - 1)) S.state = ST_DONE;  // overflowed (counted): host grows kcap
        else S.state = S.spec_hit ? ST_PRIMED : ST_DETECT;
    }
    __syncthreads();
    build_lists(A, false);
    if (threadIdx.x == 0 && A.status_host) {
        C->step += 1;
        volatile int* hs = A.status_host;
        hs[0] = C->active;
        __threadfence_system();  // the host reads the step counter, then `active`
        hs[1] = C->step;
    }
    // the host launches up to LAG steps past the last one: those return at once
    if (threadIdx.x == 0 && C->active == 0) C->finished = 1;
}

__global__ void __launch_bounds__(256) k_final(Arena A) {
    pdl_begin();
    if (A.ctrl->finished) return;  // a step launched past the run's end
    const int kstep_ = A.ctrl->step;
    if (threadIdx.x == 0) span_begin(A.ctrl, KID_FINAL);
    __shared__ unsigned s_ticket;
    __shared__ int s_last;
    __shared__ FinalSlot tab[kFinalChunk];
    Ctrl* C = A.ctrl;
    const int nf = C->n_final;
    const int tiles = (A.L + kFinalTile - 1) / kFinalTile;
    const unsigned nitems = nf > 0 ? (unsigned)tiles : 0u;
    static_assert(kFinalTile == 4 * 256, "4 consecutive samples per thread");
    const size_t L = (size_t)A.L;
    // Short signals with many slots (C2/C3: 6k samples x 500 slots): too few tiles to keep the GPU
    // busy, so the residue updates run per (slot, tile) and the ordered accumulation per element
    // (each thread: one element, every finalising slot in slot order).
    const bool split = nf > 1 && tiles * 2 < (int)gridDim.x;
    if (split) {
        // Static assignment (no ticket atomics: thousands of short items would serialise on one
        // counter): CTAs [0, nS) take one element block each -- the long, ordered accumulations
        // start first -- and the remaining CTAs stride over the (slot, tile) residue items.
        const unsigned nR = (unsigned)nf * (unsigned)tiles;
        const unsigned nS = (unsigned)((L + 255) / 256);
        const unsigned G = gridDim.x;
        const bool sep = nS < G;  // else every CTA strides over all items
        const unsigned rb = sep ? nS : 0u, rs = sep ? G - nS : G;
        for (unsigned k = 0;; ++k) {
            unsigned q;
            if (sep && blockIdx.x < nS) {
                if (k > 0) break;
                q = nR + blockIdx.x;
            } else {
                const unsigned r = (blockIdx.x - rb) + k * rs;
                if (sep) {
                    if (r >= nR) break;
                    q = r;
                } else {
                    if (r >= nR + nS) break;
                    q = r;
                }
            }
            if (q < nR) {  // R = X - imf (emd.cpp:167), imf_out / res_out copies
                const int li = (int)(q / (unsigned)tiles), tq = (int)(q % (unsigned)tiles);
                const int sl = A.final_list[li];
                const Slot& S = A.slots[sl];
                if (S.spec_hit) continue;  // R' was written by the speculative last sift
                const double* x = A.bufs + buf_off(A, sl, S.xb);
                const double* imf = S.cb >= 0 ? A.bufs + buf_off(A, sl, S.cb) : x;
                double* res = A.bufs + buf_off(A, sl, pick_free_buffer(S.xb, S.cb));
                double* const io = S.imf_out;
                double* const ro = S.res_out;
                // all of the item's loads first (the stores may alias them as far as the compiler
                // knows, which would serialise the iterations on the load latency)
                constexpr int kPer = kFinalTile / 256;
                double iv[kPer], xv[kPer];
#pragma unroll
                for (int e = 0; e < kPer; ++e) {
                    const size_t t = (size_t)tq * kFinalTile + (size_t)e * 256 + threadIdx.x;
                    iv[e] = t < L ? imf[t] : 0.0;
                    xv[e] = t < L ? x[t] : 0.0;
                }
#pragma unroll
                for (int e = 0; e < kPer; ++e) {
                    const size_t t = (size_t)tq * kFinalTile + (size_t)e * 256 + threadIdx.x;
                    if (t >= L) break;
                    const double rv = xv[e] - iv[e];  // emd.cpp:167
                    res[t] = rv;
                    if (io) io[t] = iv[e];
                    if (ro) ro[t] = rv;
                }
            } else {  // sums[k0+k][t] += imf_s[t] in slot order (emd.cpp:249-251)
                const size_t t = (size_t)(q - nR) * 256 + threadIdx.x;
                double acc = 0.0;
                double* accrow = nullptr;
                for (int c0 = 0; c0 < nf; c0 += kFinalChunk) {
                    const int cn = min(kFinalChunk, nf - c0);
                    __syncthreads();
                    for (int li = threadIdx.x; li < cn; li += blockDim.x) {
                        const int sl = A.final_list[c0 + li];
                        const Slot& S = A.slots[sl];
                        FinalSlot f;
                        f.x = A.bufs + buf_off(A, sl, S.xb);
                        f.imf = S.cb >= 0 ? A.bufs + buf_off(A, sl, S.cb) : f.x;
                        f.res = nullptr;
                        f.imf_out = f.res_out = nullptr;
                        const int r = S.k0 + S.k;
                        f.row = (S.write_imf && imf_row_ok(A, S.k0, S.k)) ? A.sums + (size_t)r * A.L : nullptr;
                        tab[li] = f;
                    }
                    __syncthreads();
                    if (t >= L) continue;
                    for (int g = 0; g < cn; g += 8) {
                        double iv[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) iv[u] = g + u < cn && tab[g + u].row ? tab[g + u].imf[t] : 0.0;
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            if (g + u >= cn) break;
                            double* row = tab[g + u].row;
                            if (!row) continue;
                            if (row != accrow) {
                                if (accrow) accrow[t] = acc;
                                accrow = row;
                                acc = accrow[t];
                            }
                            acc = acc + iv[u];
                        }
                    }
                }
                if (accrow && t < L) accrow[t] = acc;
            }
        }
    }
    while (!split) {
        if (threadIdx.x == 0) s_ticket = atomicAdd(&C->ticket[3], 1u);
        __syncthreads();
        const unsigned q = s_ticket;
        __syncthreads();
        if (q >= nitems) break;
        const size_t tb = (size_t)q * kFinalTile + 4 * threadIdx.x;  // this thread's 4 samples
        const bool full = tb + 4 <= L;  // slot rows are whole tiles: 32-byte aligned vector access
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        double* accrow = nullptr;
        for (int c0 = 0; c0 < nf; c0 += kFinalChunk) {
            const int cn = min(kFinalChunk, nf - c0);
            __syncthreads();
            for (int li = threadIdx.x; li < cn; li += blockDim.x) {
                const Slot& S = A.slots[A.final_list[c0 + li]];
                FinalSlot f;
                f.x = A.bufs + buf_off(A, A.final_list[c0 + li], S.xb);
                f.imf = S.cb >= 0 ? A.bufs + buf_off(A, A.final_list[c0 + li], S.cb) : f.x;
                f.res = S.spec_hit ? nullptr  // R' was written by the speculative last sift
                                   : A.bufs + buf_off(A, A.final_list[c0 + li], pick_free_buffer(S.xb, S.cb));
                f.imf_out = S.imf_out;
                f.res_out = S.res_out;
                const int r = S.k0 + S.k;
                f.row = (S.write_imf && imf_row_ok(A, S.k0, S.k)) ? A.sums + (size_t)r * A.L : nullptr;
                tab[li] = f;
            }
            __syncthreads();
            if (tb >= L) continue;
            // groups of 4 slots: all loads in flight first, then the adds in slot order
            for (int g = 0; g < cn; g += 4) {
                double xv[4][4], iv[4][4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (g + u >= cn) break;
                    const FinalSlot& f = tab[g + u];
                    if (full) {
                        if (f.res) {
                            const double2 a0 = __ldcs(reinterpret_cast<const double2*>(f.x + tb));
                            const double2 a1 = __ldcs(reinterpret_cast<const double2*>(f.x + tb) + 1);
                            xv[u][0] = a0.x; xv[u][1] = a0.y; xv[u][2] = a1.x; xv[u][3] = a1.y;
                        }
                        const double2 b0 = __ldcs(reinterpret_cast<const double2*>(f.imf + tb));
                        const double2 b1 = __ldcs(reinterpret_cast<const double2*>(f.imf + tb) + 1);
                        iv[u][0] = b0.x; iv[u][1] = b0.y; iv[u][2] = b1.x; iv[u][3] = b1.y;
                    } else {
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            xv[u][e] = tb + e < L ? f.x[tb + e] : 0.0;
                            iv[u][e] = tb + e < L ? f.imf[tb + e] : 0.0;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (g + u >= cn) break;
                    const FinalSlot& f = tab[g + u];
                    double rv[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) rv[e] = xv[u][e] - iv[u][e];  // emd.cpp:167
                    if (!f.res) {
                    } else if (full) {
                        reinterpret_cast<double2*>(f.res + tb)[0] = make_double2(rv[0], rv[1]);
                        reinterpret_cast<double2*>(f.res + tb)[1] = make_double2(rv[2], rv[3]);
                    } else {
                        for (int e = 0; e < 4; ++e)
                            if (tb + e < L) f.res[tb + e] = rv[e];
                    }
                    if (f.imf_out || f.res_out) {
                        for (int e = 0; e < 4; ++e) {
                            if (tb + e >= L) break;
                            if (f.imf_out) f.imf_out[tb + e] = iv[u][e];
                            if (f.res_out) f.res_out[tb + e] = rv[e];
                        }
                    }
                    if (f.row) {
                        if (f.row != accrow) {
                            if (accrow)
                                for (int e = 0; e < 4; ++e)
                                    if (tb + e < L) accrow[tb + e] = acc[e];
                            accrow = f.row;
#pragma unroll
                            for (int e = 0; e < 4; ++e) acc[e] = tb + e < L ? accrow[tb + e] : 0.0;
                        }
#pragma unroll
                        for (int e = 0; e < 4; ++e) acc[e] = acc[e] + iv[u][e];  // emd.cpp:249-251, slot order
                    }
                }
            }
        }
        if (accrow)
            for (int e = 0; e < 4; ++e)
                if (tb + e < L) accrow[tb + e] = acc[e];
    }
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&C->done[3], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        for (int li = threadIdx.x; li < nf; li += blockDim.x) {  // (one thread per slot: 500-slot waves)
            const Slot& S = A.slots[A.final_list[li]];
            if (S.write_imf && !imf_row_ok(A, S.k0, S.k)) atomicAdd(&C->k_overflow, 1);
        }
        __syncthreads();
        decide_after_final(A);
        if (threadIdx.x == 0) {
            C->ticket[3] = 0;
            C->done[3] = 0;
        }
    }
    if (threadIdx.x == 0) span_end(A.ctrl, KID_FINAL, kstep_);
}

// --------------------------------------------------------------- launchers

size_t solve_smem_bytes() {
    const size_t chunked = (size_t)5 * kSolvePadWin * sizeof(double) + kSolveIdxBuf * sizeof(int) + 8;
    const size_t seq = (size_t)4 * (kSolveSeqMax + 4) * sizeof(double);
    return chunked > seq ? chunked : seq;
}

// The speculation statistics fade: halved at the start of every decomposition, so a context
// follows a change of input within a call or two.
__global__ void k_spec_decay(int* h) {
    const int i = threadIdx.x;
    if (i < kSpecK * kSpecS) h[i] >>= 1;
}
void launch_spec_decay(int* h, cudaStream_t st) {
    k_spec_decay<<<1, kSpecK * kSpecS, 0, st>>>(h);
    count_launches(1);
}

cudaError_t launch_setup() {
    cudaError_t e = resident_setup();
    if (e != cudaSuccess) return e;
    e = eval_setup();
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)solve_smem_bytes());
}

static unsigned long long g_launches = 0;
unsigned long long launch_count() { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }
void count_launches(int n) { __atomic_fetch_add(&g_launches, (unsigned long long)n, __ATOMIC_RELAXED); }

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SEMD_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <typename Kernel>
static void launch_pdl(Kernel kernel, int grid, int block, size_t smem, cudaStream_t st, const Arena& A) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, A);
}

void launch_step(const Arena& A, int sms, cudaStream_t st) {
    launch_pdl(k_solve, kSolveCtasPerSm * sms, kSolveThreads, solve_smem_bytes(), st, A);
    launch_eval(A, sms, st);
    launch_pdl(k_scan, scan_grid(A), kScanThreads, 0, st, A);
    launch_pdl(k_compact, sms * 8, kCompactThreads, 0, st, A);
    launch_pdl(k_final, 2 * sms, 256, 0, st, A);
    count_launches(5);
}

}  // namespace dev
}  // namespace semd
