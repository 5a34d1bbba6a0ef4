// N3 paged decode on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// Work item = (decode member, layer, kv head, split of `split` tokens), as in
// the split-KV layout k_decode_reduce combines.  One persistent CTA per SM
// streams its items' KV in 128-position tiles through a 3-stage TMA ring and
// runs both products of every tile as single-thread-issued tcgen05.mma with
// the 128 positions of the tile on the M axis and the <= 16 query heads that
// share the KV head on the N axis (so the padding is at most 16/G, not the
// 128/G an M-axis of heads would cost):
//
//   S^T[pos][h]  = K_tile[pos][:] . Q[h][:]       (A = K, K-major, SW128;
//                                                  B = Q, K-major, SW128)
//   O^T[dim][h]  = V_tile^T[dim][pos] . P^T[pos][h] (A = V, MN-major, SW128;
//                                                  B = P, K-major, SW128)
//
// S and O accumulate in TMEM (fp32, 16 columns each, double-buffered).  A
// softmax group of four warps owns the 128 TMEM lanes: lane = position when
// it reads S (online-softmax max across positions = a 16-shuffle butterfly +
// one 128-thread named barrier per tile), lane = head dim when it reads O,
// which it folds into a register accumulator with the running correction
// (the O buffer in TMEM is overwritten per tile: no TMEM read-modify-write).
//
// Two softmax groups ping-pong: group g owns every other item of the CTA and
// the tile stream alternates between the groups' items, so one group's
// softmax overlaps the other's and the MMAs of both (FA4-style).
//
// Roles (416 threads): warps 0 / 3 = TMA producers of the K / V rings (lanes
// 0..7 issue the boxes of one 16-position group each), warp 1 = TMEM owner +
// S = K Q^T issuer (lane 0), warp 2 = query producer (the synthetic q of each
// group's next item, double buffered), warps 4..7 = softmax group 0, 8..11 =
// group 1, warp 12 = O = V^T P issuer (lane 0).
#pragma once
#include <cuda.h>
#include "decode_common.cuh"

namespace co {

constexpr int T5_TILE = 128;                          // positions per tile (MMA M)
constexpr int T5_NH = 16;                             // MMA N: query heads per KV head, padded
#ifndef T5_KS_DEF
#define T5_KS_DEF 3
#endif
#ifndef T5_VS_DEF
#define T5_VS_DEF 3
#endif
// K and V rings of their own depth (a K slot frees as soon as its S product
// completes, a V slot only after the softmax and the O product); measured on
// config 5: 3/3 = 84.9 %, 2/4 = 84.6 %, 1/5 = 64.9 % of HBM
constexpr int T5_KS = T5_KS_DEF;
constexpr int T5_VS = T5_VS_DEF;
constexpr int T5_GROUPS = 2;                          // softmax groups
constexpr int T5_SM_WARP0 = 4;                        // first softmax warp
constexpr int T5_O_WARP = T5_SM_WARP0 + 4 * T5_GROUPS;  // the PV (O) issuer
constexpr int T5_THREADS = 32 * (T5_O_WARP + 1);
constexpr int T5_KV_BYTES = T5_TILE * 128 * 2;        // one K (or V) tile: 32 KB
constexpr int T5_QP_BYTES = T5_NH * 128 * 2;          // one Q or P operand: 4 KB
constexpr int T5_OFF_Q = (T5_KS + T5_VS) * T5_KV_BYTES;  // Q [group][2]
constexpr int T5_OFF_P = T5_OFF_Q + 2 * T5_GROUPS * T5_QP_BYTES;  // P [group][2]
constexpr int T5_OFF_BAR = T5_OFF_P + 2 * T5_GROUPS * T5_QP_BYTES;
constexpr int T5_GBAR = 14;                           // per group: q, s, o full/empty + p full, x2
constexpr int T5_NBAR = 2 * (T5_KS + T5_VS) + T5_GROUPS * T5_GBAR;  // K full/empty, V full/empty + groups
constexpr int T5_OFF_RED = (T5_OFF_BAR + T5_NBAR * 8 + 8 + 15) & ~15;  // + TMEM base slot, 16 B aligned
constexpr int T5_RED_FLOATS = 2 * T5_NH * 4 + 4 * T5_NH;  // max [2][16 heads][4 warps], l [4 warps][16]
constexpr int T5_SMEM = T5_OFF_RED + T5_GROUPS * T5_RED_FLOATS * 4 + 1024;  // + alignment slack
constexpr uint32_t T5_TMEM_COLS = 128;                // group g: S[2] at 32g+{0,16}, O[2] at 64+32g+{0,16}
static_assert(T5_SMEM <= 232448, "tcgen05 decode shared memory exceeds 227 KB");

// ---- tcgen05 / descriptor helpers ------------------------------------------

// shared-memory matrix descriptor, SWIZZLE_128B, Blackwell version bits
__device__ __forceinline__ uint64_t t5_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3fff);
    d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
    d |= 1ull << 46;  // version = 1 (sm_100)
    d |= 2ull << 61;  // layout = SWIZZLE_128B
    return d;
}
// instruction descriptor: bf16 x bf16 -> fp32, M = 128, N = 16
__device__ __forceinline__ constexpr uint32_t t5_idesc(bool a_mn_major) {
    return (1u << 4)                        // D format f32
           | (1u << 7)                      // A bf16
           | (1u << 10)                     // B bf16
           | ((a_mn_major ? 1u : 0u) << 15) // A major
           | (0u << 16)                     // B K-major
           | ((uint32_t)(T5_NH >> 3) << 17) // N >> 3
           | ((uint32_t)(T5_TILE >> 4) << 24);  // M >> 4
}
__device__ __forceinline__ void t5_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void t5_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void t5_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void t5_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void t5_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int k = 0; k < 16; k++) v[k] = __uint_as_float(r[k]);
}
template <int N>
__device__ __forceinline__ void t5_ld(uint32_t taddr, float* v) {  // N = 8 or 16 columns of this lane
    if constexpr (N == 16) {
        t5_ld16(taddr, v);
    } else {
        uint32_t r[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = __uint_as_float(r[k]);
    }
}
// max of each of N values over the 32 lanes of a warp: halving exchanges at
// lane offsets 16, 8, ... leave lane l with head (l >> (5 - log2 N)) & (N - 1),
// reduced over the remaining low lane bits
template <int N>
__device__ __forceinline__ float t5_butterfly_max(const float* v, int lane) {
    float a[N];
#pragma unroll
    for (int k = 0; k < N; k++) a[k] = v[k];
    int off = 16;
#pragma unroll
    for (int cnt = N; cnt > 1; cnt >>= 1, off >>= 1) {
        const bool hi = lane & off;
#pragma unroll
        for (int k = 0; k < cnt / 2; k++) {
            const float keep = hi ? a[k + cnt / 2] : a[k], send = hi ? a[k] : a[k + cnt / 2];
            a[k] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, off));
        }
    }
#pragma unroll
    for (; off > 0; off >>= 1) a[0] = fmaxf(a[0], __shfl_xor_sync(0xffffffffu, a[0], off));
    return a[0];
}
__device__ __forceinline__ float t5_ex2(float v) {  // 2^v, MUFU.EX2 (ex2(-inf) = +0)
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void t5_named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// byte offset of element (row, k) in a K-major SW128 operand of 64-element
// (128 B) rows, chunks of 64 k at chunk_stride
__device__ __forceinline__ uint32_t t5_kmaj(int row, int k, uint32_t chunk_stride) {
    return (uint32_t)(k >> 6) * chunk_stride + (uint32_t)row * 128u +
           ((uint32_t)(((k & 63) >> 3) ^ (row & 7)) << 4) + (uint32_t)(k & 7) * 2u;
}

// The CTA's tile stream: group g owns items blockIdx.x + (2m + g) * gridDim.x;
// tiles alternate between the two groups' current items (one group's tiles
// only once the other has no items left).  Every role walks it identically.
struct T5Cursor {
    // two groups as separate scalars: a runtime-indexed array would live in
    // local memory
    DecItem w0, w1;
    int32_t it0, it1, t0, t1, nt0, nt1;
    int turn, g;  // g: group of the current tile (after next())
    __device__ __forceinline__ static void load(const Dev& d, const DataCfg& x, const DataCtl* dc, int32_t item,
                                                int32_t nitems, DecItem& w, int32_t& it, int32_t& t, int32_t& nt) {
        it = item;
        t = 0;
        nt = 0;
        if (item < nitems) {
            dec_item(d, x, dc, item, w);
            nt = (w.pos_hi - w.nt0 + T5_TILE - 1) / T5_TILE;
        }
    }
    __device__ __forceinline__ void init(const Dev& d, const DataCfg& x, const DataCtl* dc, int32_t nitems) {
        load(d, x, dc, (int32_t)blockIdx.x, nitems, w0, it0, t0, nt0);
        load(d, x, dc, (int32_t)(blockIdx.x + gridDim.x), nitems, w1, it1, t1, nt1);
        turn = 0;
    }
    __device__ __forceinline__ bool next(int32_t nitems) {
        const bool v0 = it0 < nitems, v1 = it1 < nitems;
        if (turn == 0) g = v0 ? 0 : (v1 ? 1 : -1);
        else g = v1 ? 1 : (v0 ? 0 : -1);
        if (g < 0) return false;
        turn = g ^ 1;
        return true;
    }
    __device__ __forceinline__ const DecItem& w() const { return g ? w1 : w0; }
    __device__ __forceinline__ int32_t t() const { return g ? t1 : t0; }
    __device__ __forceinline__ int32_t nt() const { return g ? nt1 : nt0; }
    __device__ __forceinline__ void advance(const Dev& d, const DataCfg& x, const DataCtl* dc, int32_t nitems) {
        const int32_t step = T5_GROUPS * (int32_t)gridDim.x;
        if (g == 0) {
            if (++t0 == nt0) load(d, x, dc, it0 + step, nitems, w0, it0, t0, nt0);
        } else {
            if (++t1 == nt1) load(d, x, dc, it1 + step, nitems, w1, it1, t1, nt1);
        }
    }
};

// NHR = query heads per KV head the softmax handles (G rounded up to 8 or
// 16): the MMA N stays 16 (its minimum at M = 128, padded rows are zero) but
// the softmax, its reductions and the TMEM loads skip the padding.
template <int NHR>
__global__ void __launch_bounds__(T5_THREADS, 1)
    k_decode_tc05(Dev d, DataCfg x, DataCtl* dc, const __grid_constant__ CUtensorMap kvmap) {
    const Ctl& c = *d.ctl;
    if (!c.active || !x.decode_on || !dc->decode_enabled) return;
    extern __shared__ __align__(1024) uint8_t dsm5[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm5) + 1023) & ~uintptr_t(1023));
    const uint32_t sb = smem_u32(base);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bar0 = sb + T5_OFF_BAR;
    // K and V rings are separate: a K slot is free again as soon as its S
    // product completes, a V slot only after the O product (after softmax)
    // barriers: K full[KS], K empty[KS], V full[VS], V empty[VS], then the groups'
    auto FULL = [&](int kv, int s) { return bar0 + 8u * (kv ? 2 * T5_KS + s : s); };
    auto EMPTY = [&](int kv, int s) { return bar0 + 8u * (kv ? 2 * T5_KS + T5_VS + s : T5_KS + s); };
    auto GB = [&](int g, int k, int b) { return bar0 + 8u * (2 * (T5_KS + T5_VS) + g * T5_GBAR + 2 * k + b); };
    auto QF = [&](int g, int b) { return GB(g, 0, b); };
    auto QE = [&](int g, int b) { return GB(g, 1, b); };
    auto SF = [&](int g, int b) { return GB(g, 2, b); };
    auto SE = [&](int g, int b) { return GB(g, 3, b); };
    auto PF = [&](int g, int b) { return GB(g, 4, b); };
    auto OF = [&](int g, int b) { return GB(g, 5, b); };
    auto OE = [&](int g, int b) { return GB(g, 6, b); };
    auto QBUF = [&](int g, int b) { return (uint32_t)(T5_OFF_Q + (2 * g + b) * T5_QP_BYTES); };
    auto PBUF = [&](int g, int b) { return (uint32_t)(T5_OFF_P + (2 * g + b) * T5_QP_BYTES); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + T5_OFF_BAR + T5_NBAR * 8);

    // zero the KV ring and the Q/P operands once: boxes past a tile's last
    // position are never loaded, and their stale bytes must be finite
    for (uint32_t o = threadIdx.x * 16; o < (uint32_t)T5_OFF_BAR; o += blockDim.x * 16)
        *reinterpret_cast<uint4*>(base + o) = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < T5_KS; s++) { mbar_init(FULL(0, s), 1); mbar_init(EMPTY(0, s), 1); }
        for (int s = 0; s < T5_VS; s++) { mbar_init(FULL(1, s), 1); mbar_init(EMPTY(1, s), 1); }
        for (int g = 0; g < T5_GROUPS; g++)
            for (int b = 0; b < 2; b++) {
                mbar_init(QF(g, b), 1); mbar_init(QE(g, b), 1);
                mbar_init(SF(g, b), 1); mbar_init(SE(g, b), 4);
                mbar_init(PF(g, b), 4);
                mbar_init(OF(g, b), 1); mbar_init(OE(g, b), 4);
            }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(T5_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    t5_fence_before();
    __syncthreads();
    t5_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int32_t nitems = dc->dec_items;
    const int G = x.Hq / x.Hkv;
    const int bs = d.bs;

    if (warp == 0 || warp == 3) {
        // ---------------- TMA producers: warp 0 = K ring, warp 3 = V ring ----------------
        const int kv = warp == 0 ? 0 : 1;
        T5Cursor cur;
        cur.init(d, x, dc, nitems);
        const int box = bs < 16 ? bs : 16;
        const int nbox_grp = 16 / box;  // boxes per 16-position group
        uint32_t T = 0;
        while (cur.next(nitems)) {
            const DecItem& w = cur.w();
            const uint32_t NS = kv ? T5_VS : T5_KS;
            const int s = (int)(T % NS);
            const int32_t P0 = w.nt0 + cur.t() * T5_TILE;
            int32_t ngrp = (w.pos_hi - P0 + 15) / 16;
            if (ngrp > T5_TILE / 16) ngrp = T5_TILE / 16;
            const int32_t row = (w.layer * 2 + kv) * x.Hkv + w.kh;
            // addresses first (page lookups overlap the wait for the slot)
            int32_t rr = 0, off = 0;
            const bool mine = lane < ngrp * nbox_grp;
            if (mine) {
                off = lane * box;
                const int32_t pos = P0 + off;
                const int32_t pi = pos / bs;
                const int32_t page = pi < d.tab_len[w.owner] ? page_of(d, w.owner, pi) : 0;
                rr = (page * x.rows + row) * bs + pos % bs;
            }
            if (lane == 0) {
                mbar_wait(EMPTY(kv, s), ((T / NS) & 1) ^ 1);
                mbar_expect(FULL(kv, s), (uint32_t)ngrp * 16 * 128 * 2);
            }
            __syncwarp();
            if (mine) {
                const uint32_t dst = sb + (uint32_t)((kv ? T5_KS : 0) + s) * T5_KV_BYTES + (uint32_t)off * 128;
                tma_2d(dst, &kvmap, 0, rr, FULL(kv, s));
                tma_2d(dst + T5_KV_BYTES / 2, &kvmap, 64, rr, FULL(kv, s));
            }
            __syncwarp();
            T++;
            cur.advance(d, x, dc, nitems);
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            constexpr uint32_t ID_S = t5_idesc(false);
            T5Cursor cur;
            cur.init(d, x, dc, nitems);
            uint32_t T = 0, Tg0 = 0, Tg1 = 0, Ig0 = 0, Ig1 = 0;
            while (cur.next(nitems)) {
                const int g = cur.g;
                const int s = (int)(T % T5_KS);
                const uint32_t tg = g ? Tg1 : Tg0, ig = g ? Ig1 : Ig0;
                const int sbuf = (int)(tg & 1), qb = (int)(ig & 1);
                const bool first = cur.t() == 0, last = cur.t() == cur.nt() - 1;
                if (first) mbar_wait(QF(g, qb), (ig >> 1) & 1);
                mbar_wait(FULL(0, s), (T / T5_KS) & 1);
                mbar_wait(SE(g, sbuf), ((tg >> 1) & 1) ^ 1);
                t5_fence_after();
                const uint32_t kb = sb + (uint32_t)s * T5_KV_BYTES;
                const uint32_t qbase = sb + QBUF(g, qb);
#pragma unroll
                for (int kk = 0; kk < 8; kk++) {
                    const uint64_t a = t5_desc(kb + (kk >> 2) * (T5_KV_BYTES / 2) + (kk & 3) * 32, 16, 1024);
                    const uint64_t b = t5_desc(qbase + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024);
                    t5_mma(tmem + 32 * g + 16 * sbuf, a, b, ID_S, kk > 0 ? 1u : 0u);
                }
                t5_commit(SF(g, sbuf));
                t5_commit(EMPTY(0, s));
                if (last) t5_commit(QE(g, qb));
                if (g) { Tg1++; Ig1 += last; } else { Tg0++; Ig0 += last; }
                T++;
                cur.advance(d, x, dc, nitems);
            }
        }
        __syncwarp();
    } else if (warp == T5_O_WARP) {
        // ---------------- PV issuer: O = V^T P per tile, in stream order ----------------
        // A thread of its own so that a group's O never waits behind the
        // next S (and its K load) of the issuer above: a softmax group folds
        // its previous tile's O right after producing this tile's P.
        if (lane == 0) {
            constexpr uint32_t ID_O = t5_idesc(true);
            T5Cursor cur;
            cur.init(d, x, dc, nitems);
            uint32_t T = 0, Tg0 = 0, Tg1 = 0;
            while (cur.next(nitems)) {
                const int og = cur.g;
                const uint32_t tg = og ? Tg1 : Tg0;
                const int st = (int)(T % T5_VS);
                const int ob = (int)(tg & 1);
                mbar_wait(PF(og, ob), (tg >> 1) & 1);
                mbar_wait(OE(og, ob), ((tg >> 1) & 1) ^ 1);
                mbar_wait(FULL(1, st), (T / T5_VS) & 1);
                t5_fence_after();
                const uint32_t vb = sb + (uint32_t)(T5_KS + st) * T5_KV_BYTES;
                const uint32_t pb = sb + PBUF(og, ob);
#pragma unroll
                for (int kk = 0; kk < T5_TILE / 16; kk++) {
                    // A = V^T: M = head dim (MN-major, 64-dim halves 16 KB apart),
                    // K = 16 positions = 2048 B of rows
                    const uint64_t a = t5_desc(vb + kk * 2048, T5_KV_BYTES / 2, 1024);
                    const uint64_t b = t5_desc(pb + (kk >> 2) * 2048 + (kk & 3) * 32, 16, 1024);
                    t5_mma(tmem + 64 + 32 * og + 16 * ob, a, b, ID_O, kk > 0 ? 1u : 0u);
                }
                t5_commit(OF(og, ob));
                t5_commit(EMPTY(1, st));
                if (og) Tg1++; else Tg0++;
                T++;
                cur.advance(d, x, dc, nitems);
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // ---------------- query producer (stream order) ----------------
        const uint32_t step = (uint32_t)c.steps;
        const float qscale = rsqrtf((float)x.D) * 1.4426950408889634f;  // exp2 domain
        T5Cursor cur;
        cur.init(d, x, dc, nitems);
        uint32_t Ig0 = 0, Ig1 = 0;
        while (cur.next(nitems)) {
            const int g = cur.g;
            if (cur.t() == 0) {
                const DecItem& w = cur.w();
                const uint32_t rid = (uint32_t)d.rid[w.i];
                const uint32_t ig = g ? Ig1++ : Ig0++;
                const int qb = (int)(ig & 1);
                if (lane == 0) mbar_wait(QE(g, qb), ((ig >> 1) & 1) ^ 1);
                __syncwarp();
                uint8_t* qs = base + QBUF(g, qb);
                // lane owns dims [4*lane, 4*lane+4) of every head; rows >= G are zero
                for (int h = 0; h < T5_NH; h++) {
                    float v[4] = {0.f, 0.f, 0.f, 0.f};
                    if (h < G) {
#pragma unroll
                        for (int e = 0; e < 4; e++)
                            v[e] = q_value(rid, step, w.layer, w.kh * G + h, 4 * lane + e) * qscale;
                    }
                    *reinterpret_cast<uint2*>(qs + t5_kmaj(h, 4 * lane, 2048)) =
                        make_uint2(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]));
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(QF(g, qb));
            }
            cur.advance(d, x, dc, nitems);
        }
    } else if (warp >= T5_SM_WARP0 && warp < T5_O_WARP) {
        // ---------------- softmax + output (group g) ----------------
        const int g = (warp - T5_SM_WARP0) >> 2, q4 = warp & 3;
        const int r = q4 * 32 + lane;  // TMEM lane: tile position (S) / head dim (O)
        const uint32_t tl = tmem + ((uint32_t)(q4 * 32) << 16);
        float* red = reinterpret_cast<float*>(base + T5_OFF_RED) + g * T5_RED_FLOATS;
        constexpr int LSH = NHR == 16 ? 1 : 2;  // lanes per head after the butterfly = 1 << LSH
        const int hme = (lane >> LSH) & (NHR - 1);  // the head this lane reduces in the butterfly
        uint32_t T = 0;
        for (int32_t it = (int32_t)(blockIdx.x + g * gridDim.x); it < nitems; it += T5_GROUPS * (int32_t)gridDim.x) {
            DecItem w;
            dec_item(d, x, dc, it, w);
            const int32_t nt = (w.pos_hi - w.nt0 + T5_TILE - 1) / T5_TILE;
            float mrun[NHR], lpart[NHR], oacc[NHR], cprev[NHR];
#pragma unroll
            for (int h = 0; h < NHR; h++) { mrun[h] = -INFINITY; lpart[h] = 0.f; oacc[h] = 0.f; cprev[h] = 1.f; }
            for (int32_t t = 0; t < nt; t++, T++) {
                const int b = (int)(T & 1);
                mbar_wait(SF(g, b), (T >> 1) & 1);
                t5_fence_after();
                float sv[NHR];
                t5_ld<NHR>(tl + 32 * g + 16 * b, sv);
                t5_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(SE(g, b));
                const int32_t pos = w.nt0 + t * T5_TILE + r;
                const bool valid = pos >= w.pos_lo && pos < w.pos_hi;
#pragma unroll
                for (int h = 0; h < NHR; h++) sv[h] = valid ? sv[h] : -INFINITY;
                // butterfly max: NHR heads over 32 lanes (NHR shuffles); lane
                // ends with head hme
                const float m1 = t5_butterfly_max<NHR>(sv, lane);
                float* rb = red + b * T5_NH * 4;  // [head][warp]
                if (!(lane & ((1 << LSH) - 1))) rb[hme * 4 + q4] = m1;
                t5_named_sync(1 + g, 128);
                float corr[NHR];
                uint8_t* pbuf = base + PBUF(g, b);
#pragma unroll
                for (int h = 0; h < NHR; h++) {
                    const float4 q = *reinterpret_cast<const float4*>(rb + h * 4);
                    const float m = fmaxf(mrun[h], fmaxf(fmaxf(q.x, q.y), fmaxf(q.z, q.w)));
                    corr[h] = t5_ex2(mrun[h] - m);  // mrun = -inf -> 0
                    mrun[h] = m;
                    const float p = t5_ex2(sv[h] - m);  // masked -> 0
                    lpart[h] = lpart[h] * corr[h] + p;
                    *reinterpret_cast<__nv_bfloat16*>(pbuf + t5_kmaj(h, r, 2048)) = __float2bfloat16_rn(p);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(PF(g, b));
                // fold the previous tile's O, and this tile's at the item end
#pragma unroll 1
                for (int f = (t > 0 ? 0 : 1); f < (t == nt - 1 ? 2 : 1); f++) {
                    const uint32_t To = T - 1 + f;
                    const int ob = (int)(To & 1);
                    mbar_wait(OF(g, ob), (To >> 1) & 1);
                    t5_fence_after();
                    float ov[NHR];
                    t5_ld<NHR>(tl + 64 + 32 * g + 16 * ob, ov);
                    t5_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(OE(g, ob));
#pragma unroll
                    for (int h = 0; h < NHR; h++) oacc[h] = oacc[h] * (f ? corr[h] : cprev[h]) + ov[h];
                }
#pragma unroll
                for (int h = 0; h < NHR; h++) cprev[h] = corr[h];
            }
            // item result: O (lane = dim), m (exp2 domain -> natural log), l
            float* out = x.dec_part + (int64_t)it * G * (x.D + 2);
#pragma unroll
            for (int h = 0; h < NHR; h++)  // unrolled: the accumulators stay in registers
                if (h < G) out[h * (x.D + 2) + r] = oacc[h];
            float* lb = red + 2 * T5_NH * 4;  // [4 warps][16 heads]
#pragma unroll
            for (int h = 0; h < NHR; h++) {
                if (h >= G) break;
                float l = lpart[h];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
                if (lane == 0) lb[q4 * T5_NH + h] = l;
            }
            t5_named_sync(1 + g, 128);
            if (r < G) {
                const float l = lb[r] + lb[T5_NH + r] + lb[2 * T5_NH + r] + lb[3 * T5_NH + r];
                float m = 0.f;
#pragma unroll
                for (int h = 0; h < NHR; h++) m = h == r ? mrun[h] : m;
                out[r * (x.D + 2) + x.D] = m * 0.6931471805599453f;  // exp2 domain -> natural log
                out[r * (x.D + 2) + x.D + 1] = l;
            }
        }
    }
    t5_fence_before();
    __syncthreads();
    if (warp == 1) {
        t5_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(T5_TMEM_COLS));
    }
}

}  // namespace co
