// Row (f).1: compute_metrics (engine.py:132-211) on the device.
//
// k_met_rows makes one pass over the request table: attainment counts, exact
// int64 sums (every integer-valued mean is sum / count, exact below 2^53 in
// any order), and the four percentile lists as uint64 keys -- the IEEE bits
// of the non-negative doubles the reference takes percentiles of (monotone
// as unsigned integers): TTFT and normalized latency of completed requests,
// every inter-token gap of completed requests (from the token-time slab), and
// the preemption time of preempted requests.  Order statistics come from an
// MSB-first 8-bit radix select over those keys (k_rs_hist / k_rs_pick), so
// no list is ever sorted or read back.  The one floating-point mean whose
// value depends on summation order (normalized latency) is summed with
// numpy's pairwise algorithm in the caller's request order (k_met_norm).
#pragma once
#include "engine_state.cuh"

namespace co {

constexpr int MET_LISTS = 4;  // ttft, tbt gaps, normalized, preemption time
constexpr int MET_RANKS = 7;  // p50 lo/hi, p90 lo/hi, p99 lo/hi, max

struct MetScratch {
    unsigned long long* cnt;   // [16] counters and int64 sums (see co_metrics)
    uint64_t* keys[MET_LISTS];
    double* normc;             // normalized latency by caller position
    uint8_t* flagc;            // caller position is a completed request
    double* norm_list;         // completed, caller order
    const int32_t* perm;       // sorted position -> caller position
    unsigned int* hist;        // [MET_RANKS][256]
    uint64_t* pre;             // [MET_RANKS] radix-select prefix
    long long* rem;            // [MET_RANKS] remaining rank within the prefix
    double* out_norm_sum;
};
enum MetCnt { MC_DONE = 0, MC_OK_TTFT, MC_OK_TBT, MC_GEN, MC_PRE_TOTAL, MC_PREEMPTED, MC_SUM_TTFT, MC_SUM_GAP,
              MC_SUM_WAIT, MC_SUM_EXEC, MC_SUM_PDEC, MC_SUM_PTIME, MC_N0, MC_N1, MC_N2, MC_N3 };

__device__ __forceinline__ uint64_t dbits(double v) { return (uint64_t)__double_as_longlong(v); }

__global__ void k_met_rows(Dev d, MetScratch m) {
    unsigned long long* c = m.cnt;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < d.n; i += gridDim.x * blockDim.x) {
        const int64_t arr = d.arr[i], ft = d.first_tok[i];
        if (ft >= 0 && ft - arr <= d.slo_ttft[i]) atomicAdd(&c[MC_OK_TTFT], 1ull);
        const int32_t g = d.gen[i], pc = d.pcount[i];
        atomicAdd(&c[MC_GEN], (unsigned long long)g);
        if (pc > 0) {
            atomicAdd(&c[MC_PRE_TOTAL], (unsigned long long)pc);
            atomicAdd(&c[MC_PREEMPTED], 1ull);
            atomicAdd(&c[MC_SUM_PTIME], (unsigned long long)d.ptime[i]);
            m.keys[3][atomicAdd(&c[MC_N3], 1ull)] = dbits((double)d.ptime[i]);
        }
        const int32_t cp = m.perm[i];
        if (d.state[i] != ST_COMPLETED) { m.flagc[cp] = 0; continue; }
        atomicAdd(&c[MC_DONE], 1ull);
        if (d.max_tbt[i] <= d.slo_tbt[i]) atomicAdd(&c[MC_OK_TBT], 1ull);  // all(gaps <= slo): max gap
        const int64_t comp = d.completion[i], fs = d.first_start[i], pt = d.ptime[i];
        atomicAdd(&c[MC_SUM_TTFT], (unsigned long long)(ft - arr));
        atomicAdd(&c[MC_SUM_WAIT], (unsigned long long)(fs - arr));
        atomicAdd(&c[MC_SUM_EXEC], (unsigned long long)(comp - fs - pt));
        atomicAdd(&c[MC_SUM_PDEC], (unsigned long long)pt);
        m.keys[0][atomicAdd(&c[MC_N0], 1ull)] = dbits((double)(ft - arr));
        const double nv = (double)(comp - arr) / (double)d.tout[i];  // int/int true division, both < 2^53
        m.keys[2][atomicAdd(&c[MC_N2], 1ull)] = dbits(nv);
        m.normc[cp] = nv;
        m.flagc[cp] = 1;
        if (g >= 2) {
            const int64_t* t = d.tok_times + d.tok_off[i];
            atomicAdd(&c[MC_SUM_GAP], (unsigned long long)(t[g - 1] - t[0]));
            const unsigned long long base = atomicAdd(&c[MC_N1], (unsigned long long)(g - 1));
            for (int32_t k = 1; k < g; k++) m.keys[1][base + k - 1] = dbits((double)(t[k] - t[k - 1]));
        }
    }
}

// numpy's pairwise summation (pairwise_sum in loops_utils.h.src): 8-way
// unrolled blocks of <= 128, halves rounded down to a multiple of 8 above
__device__ double np_pairwise(const double* a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; i++) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
}

// order-preserving compaction of the completed requests' normalized
// latencies in caller order (one CTA), then the pairwise sum (one thread)
__global__ void k_met_norm(MetScratch m, int32_t n) {
    __shared__ int32_t warp_tot[32];
    __shared__ int32_t base_s;
    if (threadIdx.x == 0) base_s = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int32_t c0 = 0; c0 < n; c0 += blockDim.x) {
        const int32_t p = c0 + threadIdx.x;
        const int32_t f = p < n ? m.flagc[p] : 0;
        int32_t x = f;
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_tot[w] = x;
        __syncthreads();
        if (w == 0) {
            int32_t y = lane < nw ? warp_tot[lane] : 0, z = y;
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t q = __shfl_up_sync(0xffffffffu, z, o);
                if (lane >= o) z += q;
            }
            if (lane < nw) warp_tot[lane] = z - y;
        }
        __syncthreads();
        const int32_t pos = base_s + warp_tot[w] + x - f;
        if (f) m.norm_list[pos] = m.normc[p];
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) base_s = pos + f;
        __syncthreads();
    }
    if (threadIdx.x == 0) *m.out_norm_sum = np_pairwise(m.norm_list, base_s);
}

// radix select, one 8-bit digit per pass from the MSB: histogram the keys
// that match each rank's prefix ...
__global__ void k_rs_hist(const uint64_t* keys, int64_t n, int k, const uint64_t* pre, uint64_t mask, int shift,
                          unsigned int* hist) {
    __shared__ unsigned int h[MET_RANKS][256];
    for (int q = threadIdx.x; q < MET_RANKS * 256; q += blockDim.x) h[q / 256][q % 256] = 0;
    __syncthreads();
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t v = keys[j];
        const int dg = (int)((v >> shift) & 255);
        for (int q = 0; q < k; q++)
            if ((v & mask) == pre[q]) atomicAdd(&h[q][dg], 1u);
    }
    __syncthreads();
    for (int q = threadIdx.x; q < k * 256; q += blockDim.x)
        if (h[q / 256][q % 256]) atomicAdd(&hist[q], h[q / 256][q % 256]);
}
// ... and pick the digit holding each rank (warp q, lane = 8 digits)
__global__ void k_rs_pick(int k, uint64_t* pre, long long* rem, int shift, unsigned int* hist) {
    const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (q >= k) return;
    unsigned int* hq = hist + q * 256;
    unsigned int part = 0;
    for (int j = 0; j < 8; j++) part += hq[lane * 8 + j];
    unsigned int inc = part;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    const long long r = rem[q];
    const unsigned int before = inc - part;
    const bool mine = (long long)before <= r && r < (long long)inc;
    const unsigned int who = __ballot_sync(0xffffffffu, mine);
    if (mine) {
        long long acc = before;
        int dg = lane * 8;
        for (int j = 0; j < 8; j++) {
            if (r < acc + (long long)hq[lane * 8 + j]) { dg = lane * 8 + j; break; }
            acc += hq[lane * 8 + j];
        }
        pre[q] |= (uint64_t)dg << shift;
        rem[q] = r - acc;
    }
    (void)who;
    __syncwarp();
    for (int j = lane; j < 256; j += 32) hq[j] = 0;
}

}  // namespace co
