// Row (f).3: the run's random streams on the device.
//
// The reference draws every random number from numpy Generators seeded with
// default_rng([seed, k]) (workload.py:88-90 trace, :186-187 SLO scales,
// engine.py:267 predictor noise).  This file reproduces those streams bit for
// bit on the GPU so a 512K-request trace never has to be generated on the host:
//
// * SeedSequence + PCG64 seeding (host, a few hundred integer ops);
// * the raw PCG64 stream: 128-bit LCG, one thread per word class with a
//   T-step jump (coalesced stores), XSL-RR output;
// * numpy's ziggurat samplers (exponential, normal) whose word consumption
//   varies per sample (1 word ~99 %, 2+ on the wedge / tail / rejection
//   paths).  Every stream position p is evaluated as if a sample started
//   there (consumption len(p), accept flag, value); the samples are then the
//   accepting positions on the orbit of 0 under p -> p + len(p).  The orbit is
//   resolved per 1024-position chunk speculatively (each chunk chases from
//   its own first position), and a sequential pass over the chunks repairs
//   each chunk's entry: a chase from the true entry merges with the
//   speculative orbit after a step or two, because orbits that meet coincide
//   from then on.  An ordered compaction writes the accepted values.
// * Lemire's bounded integers on the bit generator's 32-bit half-word buffer
//   (predictor noise, estimation.py:76-83): closed-form positions assuming no
//   rejection (probability (2^32 mod range) / 2^32 per draw, ~1e-8 at the
//   reference's scales), and an exact sequential re-run from the first
//   rejecting arrival if there is one.
//
// Floating-point: every expression is evaluated in numpy's operation order
// with explicit round-to-nearest intrinsics (no FMA contraction).  exp / log1p
// are CUDA's (<= 1 ulp from glibc's); the integer outputs (arrival_us, token
// lengths, SLOs, error draws) can differ only if such an ulp straddles a
// rounding boundary, which the device parity tests check does not happen on
// the traces they generate.
#pragma once
#include <cstdint>
#include <vector>
#include "zig_tables.cuh"

namespace co {

typedef unsigned __int128 u128;
constexpr u128 PCG_MULT128 = ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;

struct U128 {  // kernel-argument form
    uint64_t hi, lo;
};
__host__ __device__ __forceinline__ u128 from_u(U128 v) { return ((u128)v.hi << 64) | (u128)v.lo; }
__host__ __device__ __forceinline__ U128 to_u(u128 v) { return U128{(uint64_t)(v >> 64), (uint64_t)v}; }

__device__ __forceinline__ uint64_t pcg_out(u128 st) {
    const uint64_t x = (uint64_t)(st >> 64) ^ (uint64_t)st;
    const unsigned rot = (unsigned)(st >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}
__device__ __forceinline__ double u53(uint64_t w) { return (double)(w >> 11) * (1.0 / 9007199254740992.0); }

// (mult, plus) of k LCG steps: state_k = mult * state + plus
__host__ __device__ inline void pcg_jump(u128 inc, uint64_t k, u128& mult, u128& plus) {
    u128 am = 1, ap = 0, cm = PCG_MULT128, cp = inc;
    while (k) {
        if (k & 1) { am *= cm; ap = ap * cm + cp; }
        cp = (cm + 1) * cp;
        cm *= cm;
        k >>= 1;
    }
    mult = am; plus = ap;
}

// word i of the stream = output of the (i+1)-th step from `state`
__global__ void k_pcg_fill(U128 state, U128 inc, U128 jm, U128 jp, int64_t count, uint64_t* out) {
    const int64_t T = (int64_t)gridDim.x * blockDim.x, t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count) return;
    u128 m, p;
    pcg_jump(from_u(inc), (uint64_t)t + 1, m, p);
    u128 st = m * from_u(state) + p;
    const u128 JM = from_u(jm), JP = from_u(jp);
    for (int64_t i = t; i < count; i += T) {
        out[i] = pcg_out(st);
        st = JM * st + JP;
    }
}

// -- ziggurat local step ------------------------------------------------------

constexpr double ZIG_NOR_R_D = 3.6541528853610088;
constexpr double ZIG_NOR_INV_R_D = 0.27366123732975828;
constexpr double ZIG_EXP_R_D = 7.69711747013104972;
enum { ZIG_EXP = 0, ZIG_NOR = 1 };
constexpr int ORB_CHUNK = 1024;  // positions per speculative chunk (32 bitmap words)

// len[p]: words a sample starting at p consumes (+ `extra` trailing words when
// it accepts), 0 if that would read past the raw buffer; acc bitmap; value.
template <int KIND>
__global__ void k_zig_local(const uint64_t* __restrict__ raw, int64_t R, int64_t M, int extra, uint8_t* len,
                            uint32_t* accw, double* val) {
    __shared__ uint64_t sk[256];
    __shared__ double sw[256], sf[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        sk[i] = KIND == ZIG_EXP ? ZIG_ke[i] : ZIG_ki[i];
        sw[i] = __longlong_as_double((long long)(KIND == ZIG_EXP ? ZIG_we[i] : ZIG_wi[i]));
        sf[i] = __longlong_as_double((long long)(KIND == ZIG_EXP ? ZIG_fe[i] : ZIG_fi[i]));
    }
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p - threadIdx.x % 32 < M; p += stride) {
        int c = 0;
        bool acc = false;
        double v = 0.0;
        if (p < M) {
            if (KIND == ZIG_EXP) {
                uint64_t ri = raw[p] >> 3;
                const int idx = (int)(ri & 0xFF);
                ri >>= 8;
                const double x = __dmul_rn((double)ri, sw[idx]);
                if (ri < sk[idx]) {
                    c = 1; acc = true; v = x;
                } else if (p + 1 < R) {
                    const double u = u53(raw[p + 1]);
                    c = 2;
                    if (idx == 0) {
                        acc = true; v = __dsub_rn(ZIG_EXP_R_D, log1p(-u));
                    } else if (__dadd_rn(__dmul_rn(__dsub_rn(sf[idx - 1], sf[idx]), u), sf[idx]) < exp(-x)) {
                        acc = true; v = x;
                    }
                }
            } else {
                uint64_t r = raw[p];
                const int idx = (int)(r & 0xFF);
                r >>= 8;
                const uint64_t rabs = (r >> 1) & 0x000FFFFFFFFFFFFFull;
                double x = __dmul_rn((double)rabs, sw[idx]);
                if (r & 1) x = -x;
                if (rabs < sk[idx]) {
                    c = 1; acc = true; v = x;
                } else if (idx == 0) {
                    int64_t q = p + 1;
                    while (q + 1 < R) {
                        const double xx = __dmul_rn(-ZIG_NOR_INV_R_D, log1p(-u53(raw[q])));
                        const double yy = -log1p(-u53(raw[q + 1]));
                        q += 2;
                        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
                            const double t = __dadd_rn(ZIG_NOR_R_D, xx);
                            acc = true; v = ((rabs >> 8) & 1) ? -t : t;
                            break;
                        }
                    }
                    c = acc ? (int)(q - p) : 0;
                } else if (p + 1 < R) {
                    const double u = u53(raw[p + 1]);
                    c = 2;
                    if (__dadd_rn(__dmul_rn(__dsub_rn(sf[idx - 1], sf[idx]), u), sf[idx]) <
                        exp(__dmul_rn(__dmul_rn(-0.5, x), x))) {
                        acc = true; v = x;
                    }
                }
            }
            if (acc) c += extra;
            if (p + c > R || c > 255) c = 0, acc = false;  // invalid: the orbit must never reach it
            len[p] = (uint8_t)c;
            val[p] = v;
        }
        const unsigned b = __ballot_sync(0xffffffffu, acc);
        if ((threadIdx.x & 31) == 0 && p < M) accw[p >> 5] = b;
    }
}

// speculative orbits of each chunk from its first ORB_K positions (the true
// orbit enters a chunk at most a sample's length past its start, so one of
// them almost always IS the true orbit there; with a trailing word per
// sample, entries at odd offsets are as common as even ones).  One warp per
// chunk: the warp stages the chunk's lens in shared memory, lane v chases
// from position v.  exit[k][v] = the first orbit position past the chunk
// (-1: the chase ran into an invalid position).
constexpr int ORB_WARPS = 4, ORB_K = 4;
__global__ void __launch_bounds__(ORB_WARPS * 32) k_orbit_spec(const uint8_t* __restrict__ len, int64_t M,
                                                                int64_t nch, uint32_t* vis, int64_t* exit_) {
    __shared__ uint8_t sl[ORB_WARPS][ORB_CHUNK];
    __shared__ uint32_t sw[ORB_WARPS][ORB_K][ORB_CHUNK / 32];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t k = (int64_t)blockIdx.x * ORB_WARPS + wid;
    if (k >= nch) return;
    const int64_t s = k * ORB_CHUNK;
    const uint4* src = reinterpret_cast<const uint4*>(len + s);
    for (int i = lane; i < ORB_CHUNK / 16; i += 32) reinterpret_cast<uint4*>(sl[wid])[i] = src[i];
#pragma unroll
    for (int v = 0; v < ORB_K; v++) sw[wid][v][lane] = 0;
    __syncwarp();
    if (lane < ORB_K) {
        int p = lane;
        int64_t ex = 0;
        for (;;) {
            if (p >= ORB_CHUNK) { ex = s + p; break; }
            const int c = sl[wid][p];
            if (c == 0) { ex = -1; break; }
            sw[wid][lane][p >> 5] |= 1u << (p & 31);
            p += c;
        }
        exit_[k * ORB_K + lane] = ex;
    }
    __syncwarp();
#pragma unroll
    for (int v = 0; v < ORB_K; v++) vis[(k * ORB_K + v) * 32 + lane] = sw[wid][v][lane];
}

// true entries, chunk by chunk (one thread walks; the block stages the
// speculative exits in shared memory a tile at a time): choice[k] = the
// variant whose orbit is the true one, -1 for a chunk the orbit skips.  An
// entry past the first ORB_K positions (not seen in practice) is repaired in
// variant 0's bitmap by a chase from the entry until it merges.
__global__ void k_orbit_fix(const uint8_t* __restrict__ len, int64_t nch, uint32_t* vis, const int64_t* exit_,
                            int8_t* choice, int32_t* bad) {
    constexpr int TILE = 1024;
    __shared__ int64_t se[TILE * ORB_K];
    __shared__ int64_t t_s;
    if (threadIdx.x == 0) t_s = 0;
    for (int64_t k0 = 0; k0 < nch; k0 += TILE) {
        const int m = (int)(nch - k0 < TILE ? nch - k0 : TILE);
        __syncthreads();
        for (int i = threadIdx.x; i < m * ORB_K; i += blockDim.x) se[i] = exit_[k0 * ORB_K + i];
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t t = t_s;
            for (int i = 0; i < m; i++) {
                const int64_t k = k0 + i, s = k * ORB_CHUNK, e = s + ORB_CHUNK;
                const int64_t off = t - s;
                if (t >= 0 && off >= 0 && off < ORB_K) {
                    choice[k] = (int8_t)off;
                    t = se[i * ORB_K + off];
                    continue;
                }
                if (t < 0 || t >= e) { choice[k] = -1; continue; }
                choice[k] = 0;
                uint32_t* w = vis + k * ORB_K * 32;
                for (int64_t q = s; q < t; q++) w[(q - s) >> 5] &= ~(1u << (q & 31));
                int64_t p = t;
                for (;;) {
                    if (p >= e) { t = p; break; }
                    if (w[(p - s) >> 5] >> (p & 31) & 1) { t = se[i * ORB_K]; break; }
                    const int c = len[p];
                    if (c == 0) { t = -1; break; }
                    w[(p - s) >> 5] |= 1u << (p & 31);
                    const int64_t q_end = p + c < e ? p + c : e;
                    for (int64_t q = p + 1; q < q_end; q++) w[(q - s) >> 5] &= ~(1u << (q & 31));
                    p += c;
                }
            }
            t_s = t;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && t_s < 0) *bad = 1;
}

__device__ __forceinline__ uint32_t orbit_word(const uint32_t* vis, const int8_t* choice, int64_t k, int lane) {
    const int c = choice[k];
    return c < 0 ? 0u : vis[(k * ORB_K + c) * 32 + lane];
}

// accepted samples per chunk (warp per chunk)
__global__ void k_orbit_count(const uint32_t* __restrict__ vis, const int8_t* __restrict__ choice,
                              const uint32_t* __restrict__ accw, int64_t nch, int64_t* cnt) {
    const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (k >= nch) return;
    int c = __popc(orbit_word(vis, choice, k, lane) & accw[k * 32 + lane]);
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[k] = c;
}

// exclusive prefix over the chunk counts (one block)
__global__ void k_orbit_scan(int64_t* cnt, int64_t nch, int64_t* total) {
    __shared__ int64_t part[1024];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int64_t per = (nch + nt - 1) / nt, b = tid * per, e = b + per < nch ? b + per : nch;
    int64_t s = 0;
    for (int64_t i = b; i < e; i++) s += cnt[i];
    part[tid] = s;
    __syncthreads();
    if (tid == 0) {
        int64_t a = 0;
        for (int i = 0; i < nt; i++) { const int64_t x = part[i]; part[i] = a; a += x; }
        *total = a;
    }
    __syncthreads();
    int64_t a = part[tid];
    for (int64_t i = b; i < e; i++) { const int64_t x = cnt[i]; cnt[i] = a; a += x; }
}

// ordered compaction: sample j = j-th accepting orbit position; `ex` gets the
// u53 of the trailing word when extra > 0
__global__ void k_orbit_emit(const uint32_t* __restrict__ vis, const int8_t* __restrict__ choice,
                             const uint32_t* __restrict__ accw,
                             const int64_t* __restrict__ off, const uint8_t* __restrict__ len,
                             const double* __restrict__ val, const uint64_t* __restrict__ raw, int64_t nch, int64_t n,
                             int extra, double* out, double* ex) {
    const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (k >= nch) return;
    uint32_t m = orbit_word(vis, choice, k, lane) & accw[k * 32 + lane];
    const int c = __popc(m);
    int inc = c;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    int64_t j = off[k] + inc - c;
    while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        const int64_t p = k * ORB_CHUNK + lane * 32 + b;
        if (j < n) {
            out[j] = val[p];
            if (extra) ex[j] = u53(raw[p + len[p] - 1]);
        }
        j++;
    }
}

// -- consumers of the samples --------------------------------------------------

// workload.py:92-93: gaps = scale * E; arrival_us = floor(cumsum(gaps) * 1e6 + 0.5).
//
// np.cumsum is the left-to-right running sum s_i = fl(s_{i-1} + g_i).  It is
// evaluated exactly in parallel: while s stays in one binade [2^e, 2^(e+1))
// every partial sum is an integer multiple of u = ulp(s) = 2^(e-52), and
// fl(x + g) = x + u * rne(g / u) -- an INTEGER increment independent of x --
// unless g / u sits exactly on a half (a tie: round-half-even then depends on
// the parity of x / u) or the sum leaves the binade.  So one CTA sweeps the
// array in tiles: increments k_i = rint(g_i / u) and a block-wide int64 prefix
// give every s_i = (x/u + P_i) * u exactly up to the first tie or binade exit;
// that one element is added in double the sequential way, and the sweep
// resumes after it.  Rounds = tiles + binades (~20) + ties (~1 per 2^19
// elements at config-2 magnitudes).
constexpr int ARR_T = 1024, ARR_I = 8;
__global__ void __launch_bounds__(ARR_T) k_arrivals(const double* __restrict__ e, int64_t n, double scale,
                                                    int64_t* arrival) {
    __shared__ long long wsum[ARR_T / 32];
    __shared__ int64_t s_f;
    __shared__ double s_x;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (n <= 0) return;
    double x = __dmul_rn(scale, e[0]);  // s_0 = g_0
    if (tid == 0) arrival[0] = (int64_t)floor(__dadd_rn(__dmul_rn(x, 1000000.0), 0.5));
    int64_t pos = 1;
    while (pos < n) {
        const int64_t end = pos + (int64_t)ARR_T * ARR_I < n ? pos + (int64_t)ARR_T * ARR_I : n;
        int ex = 0;
        const double m = frexp(x, &ex);  // x = m 2^ex, m in [0.5, 1): u = 2^(ex-53), X = m 2^53
        const long long X = (long long)ldexp(m, 53);
        const bool xok = x > 0.0;
        // this thread's items: pos + tid*ARR_I + j
        long long k[ARR_I];
        bool bad[ARR_I];
        double g[ARR_I];
        long long tsum = 0;
#pragma unroll
        for (int j = 0; j < ARR_I; j++) {
            const int64_t i = pos + (int64_t)tid * ARR_I + j;
            g[j] = i < end ? __dmul_rn(scale, e[i]) : 0.0;
            const double q = ldexp(g[j], 53 - ex);
            const double fq = floor(q);
            bad[j] = i < end && (!xok || q - fq == 0.5 || q >= 4.0e18);
            k[j] = (i < end && !bad[j]) ? (long long)rint(q) : 0;
            tsum += k[j];
        }
        // block exclusive scan of the thread sums
        long long inc = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) wsum[w] = inc;
        if (tid == 0) s_f = end;
        __syncthreads();
        if (w == 0) {
            long long v = wsum[lane], z = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(0xffffffffu, z, o);
                if (lane >= o) z += y;
            }
            wsum[lane] = z - v;
        }
        __syncthreads();
        long long P = wsum[w] + inc - tsum;  // prefix before this thread's first item
        // first exception: a tie / unrepresentable increment, or leaving the binade
        int64_t my_f = end;
        {
            long long Q = P;
#pragma unroll
            for (int j = 0; j < ARR_I; j++) {
                const int64_t i = pos + (int64_t)tid * ARR_I + j;
                if (i >= end) break;
                if (bad[j]) { my_f = i; break; }
                Q += k[j];
                if (X + Q >= (1ll << 53)) { my_f = i; break; }
            }
        }
        if (my_f < end) atomicMin((unsigned long long*)&s_f, (unsigned long long)my_f);
        __syncthreads();
        const int64_t f = s_f;
        // exact partial sums before the exception
        {
            long long Q = P;
#pragma unroll
            for (int j = 0; j < ARR_I; j++) {
                const int64_t i = pos + (int64_t)tid * ARR_I + j;
                Q += k[j];
                if (i < f) {
                    const double si = ldexp((double)(X + Q), ex - 53);
                    arrival[i] = (int64_t)floor(__dadd_rn(__dmul_rn(si, 1000000.0), 0.5));
                    if (i == f - 1 && f == end) s_x = si;
                }
                if (i == f - 1 && f < end) s_x = ldexp((double)(X + Q), ex - 53);
            }
        }
        __syncthreads();
        if (f < end) {
            // the exception element, the sequential way (thread owning it)
            const int64_t rel = f - pos;
            if (tid == (int)(rel / ARR_I)) {
                const double prev = f == pos ? x : s_x;
                const double sf = __dadd_rn(prev, g[rel % ARR_I]);
                arrival[f] = (int64_t)floor(__dadd_rn(__dmul_rn(sf, 1000000.0), 0.5));
                s_x = sf;
            }
            __syncthreads();
            x = s_x;
            pos = f + 1;
        } else {
            x = s_x;
            pos = end;
        }
        __syncthreads();
    }
}

// workload.py:96-99: clip(rint(exp(mu + sigma * z)), lo, hi)
__global__ void k_lognormal_len(const double* __restrict__ z, int64_t n, double mu, double sigma, int32_t lo,
                                int32_t hi, int32_t* out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double v = rint(exp(__dadd_rn(mu, __dmul_rn(sigma, z[i]))));
        v = v < (double)lo ? (double)lo : (v > (double)hi ? (double)hi : v);
        out[i] = (int32_t)v;
    }
}

// workload.py:181-194: u = lo + (hi - lo) * U; slo = max(1, round(base * u * f))
__global__ void k_slos(const uint64_t* __restrict__ ra, const uint64_t* __restrict__ rb, const int32_t* prompt,
                       int64_t n, double lo, double range, int64_t base_ttft, int64_t base_tbt, int32_t chunk,
                       int64_t* ttft, int64_t* tbt) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double ut = __dadd_rn(lo, __dmul_rn(range, u53(ra[i])));
        const double ub = __dadd_rn(lo, __dmul_rn(range, u53(rb[i])));
        const int64_t f = prompt[i] <= chunk ? 1 : ((int64_t)prompt[i] + chunk - 1) / chunk;
        const double a = rint(__dmul_rn(__dmul_rn((double)base_ttft, ut), (double)f));
        const double b = rint(__dmul_rn((double)base_tbt, ub));
        ttft[i] = a < 1.0 ? 1 : (int64_t)a;
        tbt[i] = b < 1.0 ? 1 : (int64_t)b;
    }
}

// estimation.py:80-83 / :97: err = floor(0 + scale * z + 0.5); flip = U < 1 - acc
__global__ void k_pred_normal(const double* __restrict__ z, const double* __restrict__ u, int64_t n, double scale,
                              double miss, int flip_on, int32_t* err, uint8_t* flip) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        err[i] = (int32_t)floor(__dadd_rn(__dadd_rn(0.0, __dmul_rn(scale, z[i])), 0.5));
        flip[i] = flip_on ? (u[i] < miss ? 1 : 0) : 0;
    }
}

// estimation.py:80 integers(-s, s + 1) (+ random() per arrival when
// flip_on), closed-form stream positions assuming no Lemire rejection; the
// first rejecting arrival (if any) goes to *first_rej
__device__ __forceinline__ void pred_uni_pos(int64_t k, int flip_on, int64_t& word, int& hi_half, int64_t& fword) {
    if (flip_on) {
        const int64_t m = k >> 1;
        word = 3 * m; hi_half = (int)(k & 1); fword = 3 * m + 1 + (k & 1);
    } else {
        word = k >> 1; hi_half = (int)(k & 1); fword = -1;
    }
}
__global__ void k_pred_uniform(const uint64_t* __restrict__ raw, int64_t n, uint32_t s, double miss, int flip_on,
                               int32_t* err, uint8_t* flip, unsigned long long* first_rej) {
    const uint32_t excl = 2u * s + 1u, rng = 2u * s;
    const uint32_t thr = (uint32_t)((0xFFFFFFFFull - rng) % excl);
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        int64_t w, fw;
        int hh;
        pred_uni_pos(k, flip_on, w, hh, fw);
        const uint32_t u = hh ? (uint32_t)(raw[w] >> 32) : (uint32_t)raw[w];
        const uint64_t m = (uint64_t)u * excl;
        if ((uint32_t)m < thr) atomicMin(first_rej, (unsigned long long)k);
        err[k] = (int32_t)((int64_t)(m >> 32) - (int64_t)s);
        flip[k] = flip_on ? (u53(raw[fw]) < miss ? 1 : 0) : 0;
    }
}
// exact sequential re-run from the first rejecting arrival (one thread)
__global__ void k_pred_uniform_fix(const uint64_t* __restrict__ raw, int64_t R, int64_t n, uint32_t s, double miss,
                                   int flip_on, int32_t* err, uint8_t* flip, const unsigned long long* first_rej,
                                   int32_t* bad) {
    const unsigned long long k0 = *first_rej;
    if (k0 >= (unsigned long long)n) return;
    const uint32_t excl = 2u * s + 1u, rng = 2u * s;
    const uint32_t thr = (uint32_t)((0xFFFFFFFFull - rng) % excl);
    int64_t w, fw;
    int hh;
    pred_uni_pos((int64_t)k0, flip_on, w, hh, fw);
    // stream state before arrival k0: the next fresh word, and the buffered high half
    int has = 0;
    uint32_t buf = 0;
    int64_t next;
    if (hh) { has = 1; buf = (uint32_t)(raw[w] >> 32); next = flip_on ? w + 2 : w + 1; }
    else next = w;
    auto u32 = [&](bool& ok) -> uint32_t {
        if (has) { has = 0; return buf; }
        if (next >= R) { ok = false; return 0; }
        const uint64_t v = raw[next++];
        has = 1; buf = (uint32_t)(v >> 32);
        return (uint32_t)v;
    };
    bool ok = true;
    for (int64_t k = (int64_t)k0; k < n && ok; k++) {
        uint64_t m = (uint64_t)u32(ok) * excl;
        if ((uint32_t)m < excl)
            while (ok && (uint32_t)m < thr) m = (uint64_t)u32(ok) * excl;
        err[k] = (int32_t)((int64_t)(m >> 32) - (int64_t)s);
        if (flip_on) {
            if (next >= R) { ok = false; break; }
            flip[k] = u53(raw[next++]) < miss ? 1 : 0;
        } else flip[k] = 0;
    }
    if (!ok) *bad = 1;
}

// estimation.py:97 with error_dist "zero": one random() per arrival
__global__ void k_pred_flip_only(const uint64_t* __restrict__ raw, int64_t n, double miss, int32_t* err,
                                 uint8_t* flip) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        err[k] = 0;
        flip[k] = u53(raw[k]) < miss ? 1 : 0;
    }
}

// -- host side ---------------------------------------------------------------

// numpy SeedSequence(entropy).generate_state(4, uint64) -> PCG64 seeding
// (pcg_setseq_128_srandom_r), restated; entropy = the integers of
// default_rng([seed, k]), each split into little-endian 32-bit words.
inline void seed_pcg64(const uint64_t* ent, int n_ent, u128& state, u128& inc) {
    std::vector<uint32_t> w;
    for (int i = 0; i < n_ent; i++) {
        uint64_t v = ent[i];
        w.push_back((uint32_t)v);
        for (v >>= 32; v; v >>= 32) w.push_back((uint32_t)v);
    }
    uint32_t hc = 0x43B0D7E5u;
    auto hashmix = [&](uint32_t v) {
        v ^= hc;
        hc *= 0x931E8875u;
        v *= hc;
        return v ^ (v >> 16);
    };
    auto mix = [](uint32_t x, uint32_t y) {
        uint32_t r = 0xCA01F9DDu * x - 0x4973F715u * y;
        return r ^ (r >> 16);
    };
    uint32_t pool[4];
    for (int i = 0; i < 4; i++) pool[i] = hashmix(i < (int)w.size() ? w[i] : 0u);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
    for (size_t s = 4; s < w.size(); s++)
        for (int d = 0; d < 4; d++) pool[d] = mix(pool[d], hashmix(w[s]));
    uint32_t h = 0x8B51F9DDu, o[8];
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i % 4] ^ h;
        h *= 0x58F38DEDu;
        v *= h;
        o[i] = v ^ (v >> 16);
    }
    uint64_t q[4];
    for (int i = 0; i < 4; i++) q[i] = (uint64_t)o[2 * i] | ((uint64_t)o[2 * i + 1] << 32);
    const u128 initstate = ((u128)q[0] << 64) | q[1], initseq = ((u128)q[2] << 64) | q[3];
    inc = (initseq << 1) | 1;
    state = inc;  // 0 * mult + inc
    state += initstate;
    state = state * PCG_MULT128 + inc;
}

}  // namespace co
