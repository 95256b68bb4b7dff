// semd_aux.cu -- sm_100a kernels around the sift engine: the noise streams
// (std::mt19937_64 + Box-Muller, emd.cpp:181-200), the exact signal_std
// (emd.cpp:209-217), ensemble finish (:252-260), CEEMDAN stage means
// (:301-306, :331-338), the serializer / deserializer (serialize.cpp:7-95) and
// the standalone envelope() entry (emd.cpp:41-125).
// Compiled with -fmad=false (reference rounding, see semd_device.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "semd_device.cuh"
#include "semd_launch.h"
#include "semd_libm.cuh"
#include "semd_types.cuh"

namespace semd {
namespace dev {

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

// One CTA per realization m0 + blockIdx.x of an ensemble: seed = derive_seed(base, m)
// (emd.cpp:174-179, :238), draws into out + blockIdx.x * stride.
__global__ void __launch_bounds__(320) k_mt19937_64_ens(uint64_t base, long long m0, uint64_t* out, long long stride,
                                                       long long n) {
    __shared__ uint64_t mt[312];
    const int t = threadIdx.x;
    uint64_t* dst = out + blockIdx.x * stride;
    if (t == 0) {
        uint64_t z = base + 0x9E3779B97F4A7C15ULL * ((uint64_t)(m0 + blockIdx.x) + 1);
        mt[0] = mix64(z);
        for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
    }
    __syncthreads();
    const long long ndraw = 2 * ((n + 1) / 2);
    for (long long b0 = 0; b0 < ndraw; b0 += 312) {
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
        if (t < 312 && b0 + t < ndraw) {
            uint64_t y = mt[t];
            y ^= (y >> 29) & 0x5555555555555555ULL;
            y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
            y ^= (y << 37) & 0xFFF7EEE000000000ULL;
            y ^= y >> 43;
            dst[b0 + t] = y;
        }
    }
}

// In place: draws (u64 pairs) -> Gaussian samples (f64), emd.cpp:189-198.
// white_noise's Box-Muller (emd.cpp:189-198) with glibc's own log and sincos restated
// (semd_libm.cuh), so every noise sample equals the reference's bit-for-bit. The two glibc
// tables (2 KB log, 3.5 KB sin/cos) are served from shared memory.
__global__ void __launch_bounds__(256) k_box_muller(uint64_t* draws, long long n, double stdv) {
    __shared__ double logtab[256];
    __shared__ double sctab[440];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) logtab[i] = libm::kLogTab[i];
    for (int i = threadIdx.x; i < 440; i += blockDim.x) sctab[i] = libm::kSinCosTab[i];
    __syncthreads();
    const long long pairs = (n + 1) / 2;
    const double two_pi = 6.283185307179586476925286766559;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < pairs;
         p += (long long)gridDim.x * blockDim.x) {
        const uint64_t d1 = draws[2 * p], d2 = draws[2 * p + 1];
        const double u1 = (double)((d1 >> 11) + 1) * 0x1.0p-53;
        const double r = stdv * __dsqrt_rn(-2.0 * libm::log(u1, logtab));
        const double u2 = (double)((d2 >> 11) + 1) * 0x1.0p-53;
        double sn, cs;
        libm::sincos(two_pi * u2, sctab, &sn, &cs);
        double* out = reinterpret_cast<double*>(draws);
        out[2 * p] = r * cs;
        if (2 * p + 1 < n) out[2 * p + 1] = r * sn;
    }
}

// ------------------------------------------------------------ small kernels

// emd.cpp:209-217 verbatim: two passes of SEQUENTIAL sums (the reference's
// rounding), fed through shared memory. Warp 1 streams chunks (pass 2: the
// squared deviations) while lane 0 of warp 0 performs the dependent additions,
// so the cost is one fp64 add latency per sample and pass.
constexpr int kStdChunk = 2048;
// (every length: beta = nstd * signal_std seeds every realization's noise, so
// it must carry the reference's rounding; ~4.4 ns per sample, once per call)
__global__ void __launch_bounds__(64) k_signal_std(const double* x, long long n, double* out, double scale) {
    __shared__ double buf[2][kStdChunk];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (n == 0) {
        if (threadIdx.x == 0) *out = 0.0;
        return;
    }
    const long long nch = (n + kStdChunk - 1) / kStdChunk;
    double mean = 0.0, acc = 0.0;
    for (int pass = 0; pass < 2; ++pass) {
        auto fill = [&](long long c) {
            const long long o = c * kStdChunk;
            const int len = (int)min((long long)kStdChunk, n - o);
            double* d = buf[c & 1];
            for (int i = lane; i < len; i += 32) {
                const double v = x[o + i];
                d[i] = pass == 0 ? v : (v - mean) * (v - mean);
            }
        };
        if (warp == 1) fill(0);
        __syncthreads();
        double s = 0.0;
        for (long long c = 0; c < nch; ++c) {
            if (warp == 1 && c + 1 < nch) fill(c + 1);
            if (warp == 0 && lane == 0) {
                const double* d = buf[c & 1];
                const int len = (int)min((long long)kStdChunk, n - c * kStdChunk);
                int i = 0;
                for (; i + 8 <= len; i += 8) {
                    const double v0 = d[i], v1 = d[i + 1], v2 = d[i + 2], v3 = d[i + 3];
                    const double v4 = d[i + 4], v5 = d[i + 5], v6 = d[i + 6], v7 = d[i + 7];
                    s += v0; s += v1; s += v2; s += v3; s += v4; s += v5; s += v6; s += v7;
                }
                for (; i < len; ++i) s += d[i];
            }
            __syncthreads();
        }
        if (warp == 0 && lane == 0) {
            if (pass == 0) buf[0][0] = s / (double)n;  // mean /= n
            else acc = s;
        }
        __syncthreads();
        if (pass == 0) mean = buf[0][0];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = scale * sqrt(acc / (double)n);
}

// ---- the same sequential sums, computed in parallel and still bit-identical ("binade-locked"
// integer accumulation), for long signals.
//
// s_{i+1} = RN(s_i + v_i) is not associative, but while the running sum stays inside one binade
// [2^e, 2^(e+1)) (same sign) every s_i is an integer multiple S_i of u = 2^(e-52), and
//     RN(s_i + v_i) = (S_i + rint(v_i / u)) * u
// because the rounding grid is u throughout: the additions become exact INTEGER additions of
// k_i = rint(v_i / u), which are associative. A tie (v_i / u = k + 1/2) rounds to even, which depends
// on the parity of S_i only, so each piece of the sum is a function of the entry parity p:
//     p -> (K_p = sum of k_i, min and max over the running prefixes)
// and pieces compose in order: (f ; g)(p) = f(p) followed by g((p + K_p(f)) & 1).
// The signal is cut into segments of kSeqSeg terms (one warp each). A segment's binade is guessed
// from tree-summed approximate prefix sums; a single warp then walks the segments in order with
// the EXACT running sum: when the guess matches the sum's sign and exponent, no term was too
// large, and entry + min/max stay inside [2^52 + 1, 2^53 - 1] (so every exact intermediate lies
// strictly inside the binade), the segment is one integer addition; otherwise the segment is
// added term by term in fp64, as the reference does. Any input gives the reference's bits; the
// guesses only decide how many segments take the slow path (C5: 526 of 33,280 in the mean pass,
// 16 in the variance pass).
constexpr int kSeqSeg = 512;
constexpr long long kSeqMinLen = 1 << 16;  // shorter signals: the single-thread kernel (fewer launches)
constexpr int kSeqLane = kSeqSeg / 32;  // consecutive terms per lane
constexpr long long kSeqBig = 1ll << 61;
struct alignas(16) SeqRec {
    long long K[2], mn[2], mx[2];  // per entry parity
    int guess;                     // sign << 11 | biased exponent of the guessed running sum
    int bad;                       // a term too large for the binade's integers (or NaN): slow path
};
struct SeqHead {       // workspace header
    double mean;       // pass 0's result: sum / n
    unsigned slow[2];  // segments added term by term, per pass
    unsigned pad[2];
};

__device__ __forceinline__ double seq_term(const double* x, long long i, int pass, double mean) {
    const double v = x[i];
    return pass == 0 ? v : (v - mean) * (v - mean);  // emd.cpp:212 / :215
}

// approximate segment sums (any order)
__global__ void __launch_bounds__(256) k_seq_segsum(const double* x, long long n, int pass, const SeqHead* hd,
                                                    double* segsum, long long nseg) {
    const int lane = threadIdx.x & 31;
    const double mean = pass ? hd->mean : 0.0;
    for (long long sg = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); sg < nseg;
         sg += (long long)gridDim.x * (blockDim.x >> 5)) {
        const long long o = sg * kSeqSeg;
        double a = 0.0;
#pragma unroll 4
        for (int j = 0; j < kSeqLane; ++j) {
            const long long i = o + j * 32 + lane;
            if (i < n) a += seq_term(x, i, pass, mean);
        }
        a = warp_sum(a);
        if (lane == 0) segsum[sg] = a;
    }
}

// guess[c] = sign and exponent of the approximate sum of segments 0..c-1 (one CTA)
__global__ void __launch_bounds__(1024) k_seq_guess(const double* segsum, long long nseg, int* guess) {
    __shared__ double wsum[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long per = (nseg + blockDim.x - 1) / blockDim.x;
    const long long c0 = min(nseg, tid * per), c1 = min(nseg, c0 + per);
    double a = 0.0;
    for (long long c = c0; c < c1; ++c) a += segsum[c];
    double inc = a;  // inclusive scan over the CTA
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        double w = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += t;
        }
        wsum[lane] = w;
    }
    __syncthreads();
    double run = (inc - a) + (warp ? wsum[warp - 1] : 0.0);
    for (long long c = c0; c < c1; ++c) {
        guess[c] = (int)((unsigned long long)__double_as_longlong(run) >> 52);
        run += segsum[c];
    }
}

struct SeqFn {
    long long K[2], mn[2], mx[2];
};
__device__ __forceinline__ SeqFn seq_compose(const SeqFn& f, const SeqFn& g) {  // f first, then g
    SeqFn r;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const int q = (int)((p + f.K[p]) & 1);
        const long long gk = q ? g.K[1] : g.K[0], gmn = q ? g.mn[1] : g.mn[0], gmx = q ? g.mx[1] : g.mx[0];
        r.K[p] = f.K[p] + gk;
        r.mn[p] = min(f.mn[p], f.K[p] + gmn);
        r.mx[p] = max(f.mx[p], f.K[p] + gmx);
    }
    return r;
}

// one warp per segment: the segment as a function of the entry parity, for the guessed binade
__global__ void __launch_bounds__(256) k_seq_records(const double* x, long long n, int pass, const SeqHead* hd,
                                                     const int* guess, SeqRec* rec, long long nseg) {
    const int lane = threadIdx.x & 31;
    const double mean = pass ? hd->mean : 0.0;
    for (long long sg = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); sg < nseg;
         sg += (long long)gridDim.x * (blockDim.x >> 5)) {
        const int g = guess[sg];
        const int eb = g & 0x7ff;
        // 1/u = 2^(52-e) (sign folded in: a negative running sum is mirrored); exponents where
        // that power is not a normal double take the slow path
        int bad = eb < 60 || eb > 2040;
        const double scale =
            __longlong_as_double(((long long)(g >> 11) << 63) | ((long long)(bad ? 1023 : 1023 + 52 - (eb - 1023)) << 52));
        SeqFn f;
        f.K[0] = f.K[1] = 0;
        f.mn[0] = f.mn[1] = kSeqBig;
        f.mx[0] = f.mx[1] = -kSeqBig;
        const long long o = sg * kSeqSeg + lane * kSeqLane;
#pragma unroll 4
        for (int j = 0; j < kSeqLane; ++j) {
            if (o + j >= n) break;
            const double t = seq_term(x, o + j, pass, mean) * scale;  // v / u, exact
            if (!(fabs(t) < 0x1p53)) {
                bad = 1;
                break;
            }
            const double fl = floor(t);
            const double fr = t - fl;  // exact
            const long long kf = (long long)fl;
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                long long k = kf;
                if (fr > 0.5) k += 1;
                else if (fr == 0.5) k += (p + f.K[p] + kf) & 1;  // tie: to the even S
                f.K[p] += k;
                f.mn[p] = min(f.mn[p], f.K[p]);
                f.mx[p] = max(f.mx[p], f.K[p]);
            }
        }
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {  // in-order fold: lane l takes lanes l .. l+2d-1
            SeqFn h;
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                h.K[p] = __shfl_down_sync(0xffffffffu, f.K[p], d);
                h.mn[p] = __shfl_down_sync(0xffffffffu, f.mn[p], d);
                h.mx[p] = __shfl_down_sync(0xffffffffu, f.mx[p], d);
            }
            if (lane + d < 32) f = seq_compose(f, h);
        }
        bad = __any_sync(0xffffffffu, bad);
        if (lane == 0) {
            SeqRec r;
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                r.K[p] = f.K[p];
                r.mn[p] = f.mn[p];
                r.mx[p] = f.mx[p];
            }
            r.guess = g;
            r.bad = bad;
            rec[sg] = r;
        }
    }
}

// one warp walks the segments in order with the exact running sum (every lane computes the same)
__global__ void __launch_bounds__(32) k_seq_stitch(const double* x, long long n, int pass, SeqHead* hd,
                                                   const SeqRec* rec, long long nseg, double* out, double scale) {
    __shared__ double buf[kSeqSeg];
    __shared__ SeqRec rs[2][32];
    const int lane = threadIdx.x;
    const double mean = pass ? hd->mean : 0.0;
    double s = 0.0;
    unsigned slow = 0;
    if (lane < nseg) rs[0][lane] = rec[lane];
    __syncwarp();
    for (long long b = 0; b * 32 < nseg; ++b) {
        const SeqRec* cur = rs[b & 1];
        SeqRec nxt;  // the next 32 records travel while these are walked
        const long long c2 = (b + 1) * 32 + lane;
        if (c2 < nseg) nxt = rec[c2];
        const int cnt = (int)min(32ll, nseg - b * 32);
        for (int j = 0; j < cnt; ++j) {
            const SeqRec r = cur[j];
            const long long bits = __double_as_longlong(s);
            const long long S = (bits & ((1ll << 52) - 1)) | (1ll << 52);
            const int p = (int)(S & 1);
            const long long K = p ? r.K[1] : r.K[0], mn = p ? r.mn[1] : r.mn[0], mx = p ? r.mx[1] : r.mx[0];
            const bool fast = !r.bad && (int)((unsigned long long)bits >> 52) == r.guess && S + mn >= (1ll << 52) + 1 &&
                              S + mx <= (1ll << 53) - 1;
            if (fast) {
                s = __longlong_as_double((bits & ~((1ll << 52) - 1)) | ((S + K) & ((1ll << 52) - 1)));
            } else {  // the reference's additions, term by term
                ++slow;
                const long long o = (b * 32 + j) * kSeqSeg;
                const int len = (int)min((long long)kSeqSeg, n - o);
                for (int i = lane; i < len; i += 32) buf[i] = seq_term(x, o + i, pass, mean);
                __syncwarp();
                int i = 0;
                for (; i + 8 <= len; i += 8) {
                    const double v0 = buf[i], v1 = buf[i + 1], v2 = buf[i + 2], v3 = buf[i + 3];
                    const double v4 = buf[i + 4], v5 = buf[i + 5], v6 = buf[i + 6], v7 = buf[i + 7];
                    s += v0; s += v1; s += v2; s += v3; s += v4; s += v5; s += v6; s += v7;
                }
                for (; i < len; ++i) s += buf[i];
                __syncwarp();
            }
        }
        if (c2 < nseg) rs[(b + 1) & 1][lane] = nxt;
        __syncwarp();
    }
    if (lane == 0) {
        hd->slow[pass] = slow;
        if (pass == 0) hd->mean = s / (double)n;       // emd.cpp:213
        else *out = scale * sqrt(s / (double)n);       // emd.cpp:216
    }
}

// signal_std of B signals of length n (row b contiguous), one thread per signal:
// emd.cpp:209-217's two sequential passes verbatim; out[b] = scale * std(x_b).
__global__ void k_signal_std_batch(const double* x, long long n, int B, double* out, double scale) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const double* v = x + (size_t)b * n;
    if (n == 0) {
        out[b] = 0.0;
        return;
    }
    double mean = 0.0;
    for (long long i = 0; i < n; ++i) mean += v[i];
    mean /= (double)n;
    double acc = 0.0;
    for (long long i = 0; i < n; ++i) acc += (v[i] - mean) * (v[i] - mean);
    out[b] = scale * sqrt(acc / (double)n);
}

// slicewise tensor (baseline.cpp:17-27, layout types.hpp:105-110): mode k of channel j at
// (k*N + j)*M + i; IMF rows k < K_j from sums row j*kc + k (scaled by `scale`), the residue
// at k = common-1, zeros in between.
__global__ void k_slicewise_tensor(const double* sums, int kc, const int* kj, const double* res, long long M, int N,
                                   int common, double scale, int scaled, double* out) {
    const long long total = (long long)common * N * M;
    for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < total;
         o += (long long)gridDim.x * blockDim.x) {
        const long long i = o % M;
        const long long kjn = o / M;
        const int j = (int)(kjn % N), k = (int)(kjn / N);
        double v = 0.0;
        if (k == common - 1) v = res[(size_t)j * M + i];
        else if (k < kj[j]) {
            v = sums[((size_t)j * kc + k) * M + i];
            if (scaled) v *= scale;
        }
        out[o] = v;
    }
}

// EEMD residue per channel: res = x - sum_k (sums_k * inv) over the channel's kc rows
// (emd.cpp:252-260; rows beyond K_j are +0.0 and leave every value unchanged)
__global__ void k_slicewise_finish(const double* x, const double* sums, int kc, long long M, int N, double inv,
                                   double* res) {
    const long long total = (long long)N * M;
    for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < total;
         o += (long long)gridDim.x * blockDim.x) {
        const long long j = o / M, i = o % M;
        double r = x[o];
        for (int k = 0; k < kc; ++k) r -= sums[((size_t)j * kc + k) * M + i] * inv;
        res[o] = r;
    }
}

// out[i] = src[idx[i]] (find_extrema's values: the samples at the extrema)
__global__ void k_gather(const int* idx, unsigned n, const double* src, double* out) {
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = src[idx[i]];
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
    double* diag = work;
    double* rhs = work + n;
    for (int i = 1; i + 1 < n; ++i) {  // emd.cpp:57-63
        const double h0 = xs[i] - xs[i - 1];
        const double h1 = xs[i + 1] - xs[i];
        diag[i] = 2.0 * (h0 + h1);
        rhs[i] = 6.0 * ((ys[i + 1] - ys[i]) / h1 - (ys[i] - ys[i - 1]) / h0);
    }
    for (int i = 2; i + 1 < n; ++i) {  // :64-69
        const double h0 = xs[i] - xs[i - 1];
        const double w = h0 / diag[i - 1];
        diag[i] -= w * (xs[i] - xs[i - 1]);
        rhs[i] -= w * rhs[i - 1];
    }
    double m = 0.0;  // :70-73
    mom[n - 1] = 0.0;
    for (int i = n - 2; i >= 1; --i) {
        m = (rhs[i] - (xs[i + 1] - xs[i]) * m) / diag[i];
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
        out[t] = spline_eval_ref(xs[seg], xs[seg + 1], ys[seg], ys[seg + 1], mom[seg], mom[seg + 1], tt);
    }
}

// CEEMDAN stage mean (emd.cpp:301-304 / :331-336): mode *= inv, flag any nonzero.
// Number of maxima and minima find_extrema (emd.cpp:10-35) reports for x: runs of exactly
// equal samples with both neighbours, strictly above (below) both; the thread at each run's
// first sample decides (CEEMDAN's residue test, emd.cpp:311, needs only the total).
__global__ void k_count_extrema(const double* x, long long n, unsigned long long* cnt) {
    unsigned long long mx = 0, mn = 0;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
        const double v = x[t];
        if (t == 0 || x[t - 1] == v) continue;  // runs touching index 0 never count; not a run start
        long long re = t;
        while (re + 1 < n && x[re + 1] == v) ++re;
        if (re == n - 1) continue;
        const double l = x[t - 1], r = x[re + 1];
        mx += (v > l && v > r) ? 1ull : 0ull;
        mn += (v < l && v < r) ? 1ull : 0ull;
    }
    for (int o = 16; o > 0; o >>= 1) {
        mx += __shfl_xor_sync(0xffffffffu, mx, o);
        mn += __shfl_xor_sync(0xffffffffu, mn, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (mx) atomicAdd(&cnt[0], mx);
        if (mn) atomicAdd(&cnt[1], mn);
    }
}

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

void launch_rng(const RngJob* jobs, int njobs, cudaStream_t st) { k_mt19937_64<<<njobs, 320, 0, st>>>(jobs); }
void launch_rng_ensemble(uint64_t base, long long m0, int count, uint64_t* out, long long stride, long long n,
                         cudaStream_t st) {
    k_mt19937_64_ens<<<count, 320, 0, st>>>(base, m0, out, stride, n);
    count_launches(1);
}
void launch_box_muller(uint64_t* draws, long long n, double stdv, cudaStream_t st) {
    const long long pairs = (n + 1) / 2;
    const int grid = (int)((pairs + 255) / 256 < 4096 ? (pairs + 255) / 256 : 4096);
    k_box_muller<<<grid > 0 ? grid : 1, 256, 0, st>>>(draws, n, stdv);
    count_launches(1);
}
size_t signal_std_workspace(long long n) {
    if (n < kSeqMinLen) return 0;
    const size_t nseg = (size_t)((n + kSeqSeg - 1) / kSeqSeg);
    return sizeof(SeqHead) + 32 + nseg * (sizeof(SeqRec) + sizeof(double) + sizeof(int));
}
// ws: signal_std_workspace(n) bytes (16-byte aligned), or null for the single-thread kernel
void launch_signal_std(const double* x, long long n, double* out, double scale, cudaStream_t st, void* ws) {
    if (!ws || n < kSeqMinLen) {
        k_signal_std<<<1, 64, 0, st>>>(x, n, out, scale);
        count_launches(1);
        return;
    }
    const long long nseg = (n + kSeqSeg - 1) / kSeqSeg;
    SeqHead* hd = reinterpret_cast<SeqHead*>(ws);
    SeqRec* rec = reinterpret_cast<SeqRec*>(reinterpret_cast<unsigned char*>(ws) + 32);
    double* segsum = reinterpret_cast<double*>(rec + nseg);
    int* guess = reinterpret_cast<int*>(segsum + nseg);
    const int grid = (int)std::min<long long>((nseg + 7) / 8, 148 * 8);
    for (int pass = 0; pass < 2; ++pass) {
        k_seq_segsum<<<grid, 256, 0, st>>>(x, n, pass, hd, segsum, nseg);
        k_seq_guess<<<1, 1024, 0, st>>>(segsum, nseg, guess);
        k_seq_records<<<grid, 256, 0, st>>>(x, n, pass, hd, guess, rec, nseg);
        k_seq_stitch<<<1, 32, 0, st>>>(x, n, pass, hd, rec, nseg, out, scale);
    }
    count_launches(8);
}
static int grid_for(long long n);
void launch_signal_std_batch(const double* x, long long n, int B, double* out, double scale, cudaStream_t st) {
    k_signal_std_batch<<<(B + 127) / 128, 128, 0, st>>>(x, n, B, out, scale);
    count_launches(1);
}
void launch_slicewise_tensor(const double* sums, int kc, const int* kj, const double* res, long long M, int N,
                             int common, double scale, int scaled, double* out, cudaStream_t st) {
    k_slicewise_tensor<<<grid_for((long long)common * N * M), 256, 0, st>>>(sums, kc, kj, res, M, N, common, scale,
                                                                           scaled, out);
    count_launches(1);
}
void launch_slicewise_finish(const double* x, const double* sums, int kc, long long M, int N, double inv, double* res,
                             cudaStream_t st) {
    k_slicewise_finish<<<grid_for((long long)N * M), 256, 0, st>>>(x, sums, kc, M, N, inv, res);
    count_launches(1);
}
void launch_gather(const int* idx, unsigned n, const double* src, double* out, cudaStream_t st) {
    if (!n) return;
    k_gather<<<grid_for(n), 256, 0, st>>>(idx, n, src, out);
    count_launches(1);
}
static int grid_for(long long n) {
    long long g = (n + 255) / 256;
    if (g > 8192) g = 8192;
    return g < 1 ? 1 : (int)g;
}
void launch_ensemble_finish(double* sums, int K, long long L, const double* x, double* residue, double inv,
                            cudaStream_t st) {
    k_ensemble_finish<<<grid_for(L), 256, 0, st>>>(sums, K, L, x, residue, inv);
    count_launches(1);
}
void launch_concatenate(const double* x, long long M, long long N, long long D, const double* a, double* out,
                        int naive, cudaStream_t st) {
    k_concatenate<<<grid_for(M * N + D * (N - 1)), 256, 0, st>>>(x, M, N, D, a, out, naive);
    count_launches(1);
}
void launch_transition_weights(long long d, double* a, cudaStream_t st) {
    k_transition_weights<<<grid_for(d), 256, 0, st>>>(d, a);
    count_launches(1);
}
void launch_deconcatenate(const double* modes, long long K, long long Lm, long long M, long long N, long long D,
                          double* out, cudaStream_t st) {
    k_deconcatenate<<<grid_for(K * N * M), 256, 0, st>>>(modes, K, Lm, M, N, D, out);
    count_launches(1);
}
void launch_envelope(const double* xs, const double* ys, int n, double* mom, double* work, long long length,
                     double* out, cudaStream_t st) {
    k_envelope_solve<<<1, 32, 0, st>>>(xs, ys, n, mom, work);
    count_launches(1);
    k_envelope_eval<<<grid_for(length), 256, 0, st>>>(xs, ys, mom, n, length, out);
    count_launches(1);
}
void launch_count_extrema(const double* x, long long n, unsigned long long* cnt, cudaStream_t st) {
    k_count_extrema<<<grid_for(n), 256, 0, st>>>(x, n, cnt);
    count_launches(1);
}
void launch_stage_scale(double* mode, long long n, double inv, int* nonzero, cudaStream_t st) {
    k_stage_scale<<<grid_for(n), 256, 0, st>>>(mode, n, inv, nonzero);
    count_launches(1);
}
void launch_sub(double* residue, const double* mode, long long n, cudaStream_t st) {
    k_sub<<<grid_for(n), 256, 0, st>>>(residue, mode, n);
    count_launches(1);
}
void launch_envelope_knots(const unsigned long long* idx, const double* val, long long n, long long length,
                           double* xs, double* ys, cudaStream_t st) {
    k_envelope_knots<<<grid_for(n + 4), 256, 0, st>>>(idx, val, n, length, xs, ys);
    count_launches(1);
}
__global__ void k_fill_i32(int* p, long long n, int v) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = v;
}
void launch_fill_i32(int* p, long long n, int v, cudaStream_t st) {
    k_fill_i32<<<(unsigned)std::min<long long>((n + 255) / 256, 1024), 256, 0, st>>>(p, n, v);
    count_launches(1);
}
void launch_fill(double* p, long long n, double v, cudaStream_t st) { k_fill<<<grid_for(n), 256, 0, st>>>(p, n, v); }
void launch_copy(const double* src, double* dst, long long n, cudaStream_t st) {
    k_copy<<<grid_for(n), 256, 0, st>>>(src, dst, n);
    count_launches(1);
}
void launch_axpy(const double* a, const double* b, double beta, double* out, long long n, cudaStream_t st) {
    k_axpy<<<grid_for(n), 256, 0, st>>>(a, b, beta, out, n);
    count_launches(1);
}

}  // namespace dev
}  // namespace semd
