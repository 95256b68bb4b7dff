// semd_eval.cu -- k_eval, the sift pass (the dominant kernel).
//
// Per tile of kEvalTile samples of one slot:
//   new = cur - 0.5*(upper + lower)      (emd.cpp:142-148; spline evaluation :75-86)
//   SD partials sum(mean^2), sum(cur^2)  (emd.cpp:145-146)
//   extrema of `new` + tile-local ordered lists for the next sift (emd.cpp:10-35)
//
// The envelopes are read from the segment table k_solve writes for every
// mirrored knot v: {x_v, y_v, m_v, 1/(x_{v+1}-x_v)}. A thread owns kSpt
// consecutive samples: one bounded binary search finds its first segment in
// the tile's knot range (toff), the reference's march advances it, and the
// arithmetic of the kSpt samples and two envelopes is branch-free and
// independent (ILP). No shared-memory staging: the table rows a tile needs
// are contiguous and L1/L2-resident, so many small CTAs per SM hide latency.
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

struct EvalCtx {
    int mode, L, init_kind;
    const double* src;
    const double* a;
    const double* b;
    double beta;
    TabView tv[2];
};

// new value at sample t from global data (reference formula; halos and plateau slow path)
__device__ double new_value_global(const EvalCtx& J, int t) {
    if (J.mode == EM_INIT) return J.init_kind == 1 ? J.a[t] + J.beta * J.b[t] : J.a[t];
    if (J.mode == EM_DETECT) return J.src[t];
    const double u = envelope_tab(J.tv[0], t);
    const double l = envelope_tab(J.tv[1], t);
    const double mean = 0.5 * (u + l);
    return J.src[t] - mean;
}

constexpr int kTabRows = kEvalTile / 2 + 4;  // table rows a tile can touch per side

__device__ __forceinline__ double4 ld_row(const double4* p) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

// last table row q in [lo, hi] with x_q < t (x_lo < t holds for the tile's range)
__device__ __forceinline__ int tab_search(const double4* tab, int lo, int hi, double t) {
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(&tab[mid].x) < t) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Envelope value at t whose segment is known to lie in rows [lo, hi] of the table.
__device__ __forceinline__ double env_in(const double4* tab, int lo, int hi, double tt) {
    const int q = tab_search(tab, lo, hi, tt);
    const double4 r0 = ld_row(tab + q), r1 = ld_row(tab + q + 1);
    const double h = r1.x - r0.x;
    return spline_eval_fast(r0.x, r1.x, r0.y, r1.y, r0.z, r1.z, h, r0.w, h * h, tt);
}

constexpr int kWarpRows = kEvalTile / 2 + 6;  // table rows one warp tile can touch per side
constexpr int kWarpSamp = kEvalTile + 8;      // staged samples [base-2, base+T+2)

// One warp's staging buffer for one tile.
struct alignas(16) WarpStage {
    double4 rows[2][kWarpRows];
    double samp[kWarpSamp];
    int qmap[2][32];          // per-lane first segment (bucket map, SIFT mode)
    unsigned long long bar;   // mbarrier: the tile's bulk copies have landed
};

// What a warp needs to know about a tile before issuing its copies.
struct WarpMeta {
    int valid, slot, j, mode, src_b, par, fresh;  // fresh: first tile of a strip (no carried values)
    int vlo[2], vmax[2];
};

constexpr int kStripTiles = 16;  // consecutive tiles one warp walks, carrying boundary values

// Tile number `seq` of this warp's sequence (strips q0, q0+stride, ...; 16 tiles each).
__device__ __forceinline__ WarpMeta fetch_meta(const Arena& A, unsigned q0, unsigned stride, unsigned seq,
                                               unsigned nstrips_total) {
    WarpMeta m;
    const unsigned strips = ((unsigned)A.tiles + kStripTiles - 1) / kStripTiles;
    const unsigned k = seq / kStripTiles, within = seq % kStripTiles;
    const unsigned item = q0 + k * stride;
    m.valid = 0;
    if (item >= nstrips_total) return m;
    const unsigned strip = item % strips;
    const int j = (int)(strip * kStripTiles + within);
    if (j >= A.tiles) {  // short last strip: skip to the next strip of this warp
        m.valid = 2;
        return m;
    }
    m.valid = 1;
    m.slot = A.eval_list[item / strips];
    m.j = j;
    m.fresh = within == 0;
    const Slot& sl = A.slots[m.slot];
    const int state = sl.state;
    m.mode = state == ST_INIT ? EM_INIT : (state == ST_DETECT ? EM_DETECT : EM_SIFT);
    m.src_b = (m.mode == EM_SIFT && sl.cb >= 0) ? sl.cb : sl.xb;
    m.par = sl.par;
    if (m.mode == EM_SIFT) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const ToffView to = toff_view(A, m.par, s, m.slot);
            // tile j's extrema are those of window [base-1, base+T-1); samples [base-2, base+T)
            // need segments in [toff[j], toff[j+1]+1] (plus the right row of the last one)
            m.vlo[s] = (int)to[j];
            m.vmax[s] = (int)to[j + 1] + 1;
        }
    }
    return m;
}

// Bulk (TMA-engine) copies: one lane per warp issues a tile's contiguous
// segments -- the samples and the two envelopes' table rows -- signalling the
// stage's mbarrier with the byte count (cp.async.bulk ... complete_tx).
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

// Issue the tile's copies (lane 0). Every call completes one phase of the stage's barrier.
__device__ __forceinline__ void issue_stage(const Arena& A, const WarpMeta& m, WarpStage& st) {
    if ((threadIdx.x & 31) != 0) return;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of the stage
    if (m.valid == 1 && m.mode != EM_INIT) {
        const double* src = A.bufs + buf_off(A, m.slot, m.src_b);
        const int base = m.j * kEvalTile;
        const int e0 = base > 0 ? base - 2 : 0;  // samples [base-2, base+T) (16-byte aligned; Lp = whole tiles)
        const unsigned sb = (unsigned)(base + kEvalTile - e0) * 8u;
        unsigned rb[2] = {0u, 0u};
        if (m.mode == EM_SIFT) {
#pragma unroll
            for (int s = 0; s < 2; ++s) rb[s] = (unsigned)(m.vmax[s] + 2 - m.vlo[s]) * 32u;
        }
        bar_arrive_tx(&st.bar, sb + rb[0] + rb[1]);
        bulk_g2s(&st.samp[e0 - (base - 2)], src + e0, sb, &st.bar);
        if (m.mode == EM_SIFT) {
#pragma unroll
            for (int s = 0; s < 2; ++s)
                bulk_g2s(st.rows[s], A.ktab + tab_off(A, s, m.slot) + m.vlo[s], rb[s], &st.bar);
        }
    } else {
        bar_arrive_tx(&st.bar, 0u);
    }
}

__device__ __forceinline__ int smem_search(const double4* R, int hi, double t) {  // last q <= hi with x_q < t
    int lo = 0;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (R[mid].x < t) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Extrema flags of one lane's detection window t0-1..t0+2 given v[-2..3] (find_extrema, emd.cpp:16-33).
struct Win6 {
    double w[kSpt + 2];
};
__device__ __noinline__ unsigned plateau_flags(const EvalCtx& J, int t, Win6 win, int t0, double v, int& ismin) {
    // the maximal run of samples exactly equal to v; win holds values t0-2 .. t0+3
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

// One warp evaluates one 128-sample tile (kSpt = 4 consecutive samples per lane)
// from its staged rows/samples; c2/c1 carry the new values at base-2/base-1.
__device__ void eval_warp_tile(const Arena& A, const WarpMeta& m, WarpStage& st, double& c2, double& c1) {
    const int lane = threadIdx.x & 31;
    const int slot = m.slot, j = m.j, mode = m.mode;
    const Slot& sl = A.slots[slot];
    const int L = A.L;
    EvalCtx J;
    J.mode = mode;
    J.L = L;
    J.init_kind = sl.init_kind;
    J.a = sl.init_a;
    J.b = sl.init_b;
    J.beta = sl.beta;
    J.src = A.bufs + buf_off(A, slot, m.src_b);
    double* dst = mode == EM_INIT ? A.bufs + buf_off(A, slot, sl.xb)
                                  : (mode == EM_SIFT ? A.bufs + buf_off(A, slot, sl.db) : nullptr);
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        J.tv[s].tab = A.ktab + tab_off(A, s, slot);
        J.tv[s].idx = A.kidx + knot_off(A, m.par, s, slot);
        J.tv[s].n = (int)sl.n[s];
    }
    const int base = j * kEvalTile;
    const int t0 = base + lane * kSpt;
    const bool inside = t0 + kSpt <= L;
    if (m.fresh && base > 0) {  // strip start: the new values at base-2, base-1 (staged rows cover them)
        double cc[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int t = base - 2 + u;
            if (mode == EM_INIT) {
                cc[u] = new_value_global(J, t);
            } else if (mode == EM_DETECT) {
                cc[u] = st.samp[u];
            } else {
                const double tt = (double)t;
                double e[2];
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const double4* R = st.rows[s];
                    const int qq = smem_search(R, m.vmax[s] - m.vlo[s], tt);
                    const double4 r0 = R[qq], r1 = R[qq + 1];
                    const double h = r1.x - r0.x;
                    e[s] = spline_eval_fast(r0.x, r1.x, r0.y, r1.y, r0.z, r1.z, h, r0.w, h * h, tt);
                }
                cc[u] = st.samp[u] - 0.5 * (e[0] + e[1]);
            }
        }
        c2 = cc[0];
        c1 = cc[1];
    }
    double cv[kSpt], nv[kSpt];
    if (mode == EM_INIT) {
#pragma unroll
        for (int k = 0; k < kSpt; ++k) {
            const int t = t0 + k;
            cv[k] = t < L ? (J.init_kind == 1 ? J.a[t] + J.beta * J.b[t] : J.a[t]) : 0.0;
        }
    } else {
        const double* sp = st.samp + 2 + lane * kSpt;
#pragma unroll
        for (int k = 0; k < kSpt; k += 2) {
            const double2 v = *reinterpret_cast<const double2*>(sp + k);
            cv[k] = t0 + k < L ? v.x : 0.0;
            cv[k + 1] = t0 + k + 1 < L ? v.y : 0.0;
        }
    }

    double num = 0.0, den = 0.0;
    if (mode == EM_SIFT) {
        // seg(t) = last staged row q <= qmax with x_q < t (the reference's march, emd.cpp:79).
        // Knot positions are distinct integers, so at most one row boundary lies between
        // consecutive samples: the warp finds each lane's first segment with a bucket map
        // (row r -> first lane whose t0 exceeds x_r; prefix max over lanes), and the lane's
        // kSpt segments follow from kSpt-1 independent compares -- no data-dependent branches.
        double env[2][kSpt];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const double4* R = st.rows[s];
            const int qmax = m.vmax[s] - m.vlo[s];
            int* qm = st.qmap[s];
            qm[lane] = 0;
            __syncwarp();
#pragma unroll
            for (int i = 0; i < (kWarpRows + 31) / 32; ++i) {
                const int r = 1 + lane + 32 * i;
                if (r <= qmax) {
                    const int d = (int)R[r].x - base;  // x integral; bucket = first lane with t0 > x
                    const int b = d < 0 ? 0 : (d >> 2) + 1;
                    if (b < 32) atomicMax(&qm[b], r);
                }
            }
            __syncwarp();
            int q0 = qm[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, q0, o);
                if (lane >= o) q0 = max(q0, y);
            }
            double xa[kSpt - 1];
#pragma unroll
            for (int i = 1; i < kSpt; ++i) xa[i - 1] = q0 + i <= qmax ? R[q0 + i].x : 1e300;
#pragma unroll
            for (int k = 0; k < kSpt; ++k) {
                const double tt = (double)(t0 + k);
                int q = q0;
#pragma unroll
                for (int i = 1; i <= k; ++i) q += xa[i - 1] < tt;
                const double4 r0 = R[q], r1 = R[q + 1];
                const double h = r1.x - r0.x;
                env[s][k] = spline_eval_fast(r0.x, r1.x, r0.y, r1.y, r0.z, r1.z, h, r0.w, h * h, tt);
            }
        }
#pragma unroll
        for (int k = 0; k < kSpt; ++k) {
            const double mean = 0.5 * (env[0][k] + env[1][k]);  // emd.cpp:144-147
            if (t0 + k < L) {
                num += mean * mean;
                den += cv[k] * cv[k];
                nv[k] = cv[k] - mean;
            } else {
                nv[k] = 0.0;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < kSpt; ++k) nv[k] = cv[k];
    }
    if (dst) {
        if (inside) {
#pragma unroll
            for (int k = 0; k < kSpt; k += 2)
                __stcs(reinterpret_cast<double2*>(dst + t0 + k), make_double2(nv[k], nv[k + 1]));
        } else {
            for (int k = 0; k < kSpt; ++k)
                if (t0 + k < L) dst[t0 + k] = nv[k];
        }
    }
    // detection window t0-1 .. t0+2 needs values t0-2 .. t0+3
    double w[kSpt + 2];
    w[0] = __shfl_up_sync(0xffffffffu, nv[kSpt - 2], 1);
    w[1] = __shfl_up_sync(0xffffffffu, nv[kSpt - 1], 1);
    if (lane == 0) {
        w[0] = c2;
        w[1] = c1;
    }
#pragma unroll
    for (int k = 0; k < kSpt; ++k) w[k + 2] = nv[k];
    c2 = __shfl_sync(0xffffffffu, nv[kSpt - 2], 31);  // carried into the next tile of the strip
    c1 = __shfl_sync(0xffffffffu, nv[kSpt - 1], 31);

    unsigned fmax = 0, fmin = 0;
#pragma unroll
    for (int k = 0; k < kSpt; ++k) {
        const int t = t0 - 1 + k;
        if (t < 1 || t > L - 2) continue;
        const double l = w[k], v = w[k + 1], r = w[k + 2];
        if (v != l && v != r) {
            if (v > l && v > r) fmax |= 1u << k;
            if (v < l && v < r) fmin |= 1u << k;
        } else {
            int mn;
            Win6 win;
#pragma unroll
            for (int z = 0; z < kSpt + 2; ++z) win.w[z] = w[z];
            if (plateau_flags(J, t, win, t0, v, mn)) fmax |= 1u << k;
            if (mn) fmin |= 1u << k;
        }
    }

    // tile-local ordered compaction (warp scan of packed counts)
    const unsigned packed = (unsigned)__popc(fmax) | ((unsigned)__popc(fmin) << 16);
    unsigned incl = packed;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
    const unsigned excl = incl - packed;
    unsigned omax = excl & 0xFFFF, omin = excl >> 16;
    if (fmax | fmin) {
        int* si0 = A.sidx + stage_off(A, 0, slot) + (size_t)j * kTileKnots;
        int* si1 = A.sidx + stage_off(A, 1, slot) + (size_t)j * kTileKnots;
        double* sv0 = A.sval + stage_off(A, 0, slot) + (size_t)j * kTileKnots;
        double* sv1 = A.sval + stage_off(A, 1, slot) + (size_t)j * kTileKnots;
#pragma unroll
        for (int k = 0; k < kSpt; ++k) {
            if (fmax & (1u << k)) {
                si0[omax] = t0 - 1 + k;
                sv0[omax] = w[k + 1];
                ++omax;
            }
            if (fmin & (1u << k)) {
                si1[omin] = t0 - 1 + k;
                sv1[omin] = w[k + 1];
                ++omin;
            }
        }
    }
    if (mode == EM_SIFT) {
        num = warp_sum(num);
        den = warp_sum(den);
    }
    if (lane == 0) {
        A.scnt[scnt_off(A, 0, slot) + j] = total & 0xFFFF;
        A.scnt[scnt_off(A, 1, slot) + j] = total >> 16;
        if (mode == EM_SIFT) {
            A.tnum[tsd_off(A, slot) + j] = num;
            A.tden[tsd_off(A, slot) + j] = den;
        }
    }
}

// Warp-level software pipeline over the warp's strips: tile i is computed while
// the copies of tile i+1 are in flight and the metadata of tile i+2 is loading.
__global__ void __launch_bounds__(kEvalThreads, 2) k_eval(Arena A) {
    extern __shared__ __align__(16) unsigned char eval_smem[];
    WarpStage* stage = reinterpret_cast<WarpStage*>(eval_smem) + 2 * (threadIdx.x >> 5);
    const unsigned strips = ((unsigned)A.tiles + kStripTiles - 1) / kStripTiles;
    const unsigned nstrips = (unsigned)A.ctrl->n_eval * strips;
    const unsigned wpb = kEvalThreads / 32;
    const unsigned stride = gridDim.x * wpb;
    const unsigned q0 = blockIdx.x * wpb + (threadIdx.x >> 5);
    // tile `seq` of this warp's sequence; a short last strip jumps to the next strip
    auto meta = [&](unsigned& sq) {
        WarpMeta m = fetch_meta(A, q0, stride, sq, nstrips);
        while (m.valid == 2) {
            sq = (sq / kStripTiles + 1) * kStripTiles;
            m = fetch_meta(A, q0, stride, sq, nstrips);
        }
        return m;
    };
    if ((threadIdx.x & 31) == 0) {
        bar_init(&stage[0].bar);
        bar_init(&stage[1].bar);
    }
    __syncwarp();
    unsigned phase = 0;  // bit b: parity of stage b's next completion
    unsigned seq0 = 0;
    WarpMeta cur = meta(seq0);
    issue_stage(A, cur, stage[0]);
    unsigned seq1 = seq0 + 1;
    WarpMeta nxt = meta(seq1);
    double c2 = 0.0, c1 = 0.0;
    for (unsigned i = 0; cur.valid; ++i) {
        issue_stage(A, nxt, stage[(i + 1) & 1]);
        unsigned seq2 = seq1 + 1;
        const WarpMeta after = meta(seq2);
        const unsigned b = i & 1;
        bar_wait(&stage[b].bar, (phase >> b) & 1u);
        phase ^= 1u << b;
        eval_warp_tile(A, cur, stage[b], c2, c1);
        __syncwarp();  // stage b is refilled next iteration
        cur = nxt;
        nxt = after;
        seq1 = seq2;
    }
    // the last issue was for an invalid tile (arrive only): no copies are in flight
}

size_t eval_smem_bytes() { return sizeof(WarpStage) * 2 * (kEvalThreads / 32); }
cudaError_t eval_setup() {
    return cudaFuncSetAttribute(k_eval, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)eval_smem_bytes());
}

void launch_eval(const Arena& A, int sms, cudaStream_t st) {
    k_eval<<<sms * 2, kEvalThreads, eval_smem_bytes(), st>>>(A);
}

}  // namespace dev
}  // namespace semd
