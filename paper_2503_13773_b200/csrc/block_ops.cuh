// Single-CTA (1024-thread) cooperative primitives used by the planner and
// apply kernels: reductions, exclusive scans, order-preserving compaction and
// a rank sort for the small totally-ordered sets the reference sorts with
// Python's sorted() (every key there ends in req_id, so keys are unique).
#pragma once
#include <cstdint>
#include "engine_state.cuh"

namespace co {

struct BlkShared {
    int64_t red[32];
    uint64_t ured[32];
    int32_t scan[32];
    // rank-sort tile
    static constexpr int TILE = 512;
    uint64_t t0[TILE], t1[TILE], t2[TILE];
    int32_t it[TILE];
};

__device__ __forceinline__ int64_t warp_sum64(int64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

// all threads must call; every thread receives the block total
__device__ __forceinline__ int64_t blk_sum(int64_t v, BlkShared& s) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum64(v);
    if (lane == 0) s.red[w] = v;
    __syncthreads();
    if (w == 0) {
        int64_t x = lane < (int)(blockDim.x >> 5) ? s.red[lane] : 0;
        x = warp_sum64(x);
        if (lane == 0) s.red[0] = x;
    }
    __syncthreads();
    int64_t r = s.red[0];
    __syncthreads();
    return r;
}

// three sums in one reduction (same barrier count as one)
__device__ __forceinline__ void blk_sum3(int64_t& a, int64_t& b, int64_t& c, BlkShared& s) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
    a = warp_sum64(a); b = warp_sum64(b); c = warp_sum64(c);
    if (lane == 0) { s.red[w] = a; s.ured[w] = (uint64_t)b; s.t0[w] = (uint64_t)c; }
    __syncthreads();
    if (w == 0) {
        int64_t x = lane < nw ? s.red[lane] : 0, y = lane < nw ? (int64_t)s.ured[lane] : 0,
                z = lane < nw ? (int64_t)s.t0[lane] : 0;
        x = warp_sum64(x); y = warp_sum64(y); z = warp_sum64(z);
        if (lane == 0) { s.red[0] = x; s.ured[0] = (uint64_t)y; s.t0[0] = (uint64_t)z; }
    }
    __syncthreads();
    a = s.red[0]; b = (int64_t)s.ured[0]; c = (int64_t)s.t0[0];
    __syncthreads();
}

__device__ __forceinline__ uint64_t blk_min(uint64_t v, BlkShared& s) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_min_u64(v);
    if (lane == 0) s.ured[w] = v;
    __syncthreads();
    if (w == 0) {
        uint64_t x = lane < (int)(blockDim.x >> 5) ? s.ured[lane] : ~0ull;
        x = warp_min_u64(x);
        if (lane == 0) s.ured[0] = x;
    }
    __syncthreads();
    uint64_t r = s.ured[0];
    __syncthreads();
    return r;
}

// exclusive prefix of a 0/1 (or small int) value across the block
__device__ __forceinline__ int32_t blk_excl_scan(int32_t v, int32_t* total, BlkShared& s) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s.scan[w] = x;
    __syncthreads();
    if (w == 0) {
        int32_t y = lane < (int)(blockDim.x >> 5) ? s.scan[lane] : 0;
        int32_t z = y;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int32_t q = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += q;
        }
        s.scan[lane] = z - y;  // exclusive warp offsets
        if (lane == 31) s.red[0] = z;
    }
    __syncthreads();
    int32_t r = s.scan[w] + x - v;
    *total = (int32_t)s.red[0];
    __syncthreads();
    return r;
}

// In-place exclusive prefix sum of a[0..n) in shared memory (any n); returns
// the total to every thread.
__device__ __forceinline__ int32_t blk_scan_smem(int32_t* a, int32_t n, BlkShared& s) {
    const int32_t bd = (int32_t)blockDim.x, per = (n + bd - 1) / bd;
    const int32_t lo = threadIdx.x * per, hi = min(n, lo + per);
    int32_t t = 0;
    for (int32_t k = lo; k < hi; k++) t += a[k];
    int32_t total;
    int32_t run = blk_excl_scan(t, &total, s);
    for (int32_t k = lo; k < hi; k++) { const int32_t v = a[k]; a[k] = run; run += v; }
    __syncthreads();
    return total;
}

// Order-preserving compaction of src[0..m) (or of 0..m when src == nullptr)
// by predicate pred(item) into dst, returning the count (all threads).
// m <= 32 (the common case on the step's small sets): warp 0 alone, ballot
// + popcount, two barriers instead of the two-level scan's four or five --
// less code fetched and fewer barriers on the single-CTA critical path
template <class Item, class Pred>
__device__ __forceinline__ int32_t blk_compact_warp(int32_t m, int32_t* dst, Item item_of, Pred pred, BlkShared& s) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        int32_t item = 0;
        bool f = false;
        if (lane < m) {
            item = item_of(lane);
            f = pred(lane, item);
        }
        const unsigned b = __ballot_sync(0xffffffffu, f);
        if (f) dst[__popc(b & ((1u << lane) - 1u))] = item;
        if (lane == 0) s.scan[0] = __popc(b);
    }
    __syncthreads();
    const int32_t r = s.scan[0];
    __syncthreads();
    return r;
}

template <class Pred>
__device__ __forceinline__ int32_t blk_compact(const int32_t* src, int32_t m, int32_t* dst, Pred pred, BlkShared& s) {
    if (m <= 32)
        return blk_compact_warp(m, dst, [&](int32_t k) { return src ? src[k] : k; },
                                [&](int32_t, int32_t item) { return pred(item); }, s);
    int32_t base = 0;
    for (int32_t c = 0; c < m; c += (int)blockDim.x) {
        int32_t k = c + (int32_t)threadIdx.x;
        int32_t item = 0;
        int32_t f = 0;
        if (k < m) {
            item = src ? src[k] : k;
            f = pred(item) ? 1 : 0;
        }
        int32_t tot;
        int32_t p = blk_excl_scan(f, &tot, s);
        if (f) dst[base + p] = item;
        base += tot;
    }
    __syncthreads();
    return base;
}

// Order-preserving compaction over positions k of src[0..m) with a predicate
// that sees (k, src[k]); writes src[k].
template <class Pred>
__device__ __forceinline__ int32_t blk_compact_at(const int32_t* src, int32_t m, int32_t* dst, Pred pred, BlkShared& s) {
    if (m <= 32) return blk_compact_warp(m, dst, [&](int32_t k) { return src[k]; }, pred, s);
    int32_t base = 0;
    for (int32_t c = 0; c < m; c += (int)blockDim.x) {
        int32_t k = c + (int32_t)threadIdx.x;
        int32_t item = 0, f = 0;
        if (k < m) {
            item = src[k];
            f = pred(k, item) ? 1 : 0;
        }
        int32_t tot;
        int32_t p = blk_excl_scan(f, &tot, s);
        if (f) dst[base + p] = item;
        base += tot;
    }
    __syncthreads();
    return base;
}

// Sort items[0..m) by the unique 192-bit key kf(item, k0, k1, k2),
// lexicographic ascending, in place (rank sort, O(m^2 / NT)).
template <class KeyFn>
__device__ __forceinline__ void blk_sort(int32_t* items, int32_t m, KeyFn kf, const Dev& d, BlkShared& s) {
    if (m <= 1) return;
    if (m <= 32) {
        // warp 0 alone: each lane ranks its key against the others by shuffles
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            uint64_t a0 = ~0ull, b0 = ~0ull, c0 = ~0ull;
            int32_t it = 0;
            if (lane < m) {
                it = items[lane];
                kf(it, a0, b0, c0);
            }
            int32_t rank = 0;
            for (int j = 0; j < m; j++) {
                const uint64_t a = __shfl_sync(0xffffffffu, a0, j), b = __shfl_sync(0xffffffffu, b0, j),
                               c = __shfl_sync(0xffffffffu, c0, j);
                rank += (a < a0 || (a == a0 && (b < b0 || (b == b0 && c < c0)))) ? 1 : 0;
            }
            __syncwarp();
            if (lane < m) items[rank] = it;
        }
        __syncthreads();
        return;
    }
    if (m <= BlkShared::TILE) {
        // small set: keys and items live in shared memory, one rank per thread
        for (int32_t k = threadIdx.x; k < m; k += (int)blockDim.x) {
            uint64_t a, b, c;
            kf(items[k], a, b, c);
            s.t0[k] = a; s.t1[k] = b; s.t2[k] = c;
            s.it[k] = items[k];
        }
        __syncthreads();
        for (int32_t k = threadIdx.x; k < m; k += (int)blockDim.x) {
            const uint64_t a0 = s.t0[k], b0 = s.t1[k], c0 = s.t2[k];
            int32_t rank = 0;
            for (int32_t j = 0; j < m; j++) {
                const uint64_t a = s.t0[j], b = s.t1[j], c = s.t2[j];
                rank += (a < a0 || (a == a0 && (b < b0 || (b == b0 && c < c0)))) ? 1 : 0;
            }
            items[rank] = s.it[k];
        }
        __syncthreads();
        return;
    }
    for (int32_t k = threadIdx.x; k < m; k += (int)blockDim.x) {
        uint64_t a, b, c;
        kf(items[k], a, b, c);
        d.sk0[k] = a; d.sk1[k] = b; d.sk2[k] = c;
        d.sk_item[k] = items[k];
    }
    __syncthreads();
    constexpr int Q = 4;
    for (int32_t base = 0; base < m; base += Q * (int)blockDim.x) {
        int32_t rank[Q];
        uint64_t m0[Q], m1[Q], m2[Q];
#pragma unroll
        for (int q = 0; q < Q; q++) {
            int32_t k = base + q * (int)blockDim.x + threadIdx.x;
            rank[q] = 0;
            if (k < m) { m0[q] = d.sk0[k]; m1[q] = d.sk1[k]; m2[q] = d.sk2[k]; }
            else { m0[q] = m1[q] = m2[q] = 0; }
        }
        for (int32_t t = 0; t < m; t += BlkShared::TILE) {
            int32_t tn = m - t < BlkShared::TILE ? m - t : BlkShared::TILE;
            for (int32_t j = threadIdx.x; j < tn; j += (int)blockDim.x) {
                s.t0[j] = d.sk0[t + j]; s.t1[j] = d.sk1[t + j]; s.t2[j] = d.sk2[t + j];
            }
            __syncthreads();
            for (int32_t j = 0; j < tn; j++) {
                uint64_t a = s.t0[j], b = s.t1[j], c = s.t2[j];
#pragma unroll
                for (int q = 0; q < Q; q++) {
                    bool lt = a < m0[q] || (a == m0[q] && (b < m1[q] || (b == m1[q] && c < m2[q])));
                    rank[q] += lt ? 1 : 0;
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int q = 0; q < Q; q++) {
            int32_t k = base + q * (int)blockDim.x + threadIdx.x;
            if (k < m) items[rank[q]] = d.sk_item[k];
        }
    }
    __syncthreads();
}

// blk_sort for a unique 64-bit key; the small case compares one word
template <class KeyFn>
__device__ __forceinline__ void blk_sort_u64(int32_t* items, int32_t m, KeyFn kf, const Dev& d, BlkShared& s) {
    if (m <= 1) return;
    if (m <= 32) {
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            uint64_t a0 = ~0ull;
            int32_t it = 0;
            if (lane < m) {
                it = items[lane];
                a0 = kf(it);
            }
            int32_t rank = 0;
            for (int j = 0; j < m; j++) rank += __shfl_sync(0xffffffffu, a0, j) < a0 ? 1 : 0;
            __syncwarp();
            if (lane < m) items[rank] = it;
        }
        __syncthreads();
        return;
    }
    if (m > BlkShared::TILE) {
        blk_sort(items, m, [&](int32_t i, uint64_t& k0, uint64_t& k1, uint64_t& k2) {
            k0 = kf(i); k1 = 0; k2 = 0;
        }, d, s);
        return;
    }
    for (int32_t k = threadIdx.x; k < m; k += (int)blockDim.x) {
        const int32_t it = items[k];
        s.t0[k] = kf(it);
        s.it[k] = it;
    }
    __syncthreads();
    for (int32_t k = threadIdx.x; k < m; k += (int)blockDim.x) {
        const uint64_t a0 = s.t0[k];
        int32_t rank = 0;
        for (int32_t j = 0; j < m; j++) rank += s.t0[j] < a0 ? 1 : 0;
        items[rank] = s.it[k];
    }
    __syncthreads();
}

}  // namespace co
