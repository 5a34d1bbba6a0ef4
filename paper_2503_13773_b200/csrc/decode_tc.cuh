// N3 paged decode on tensor cores.
//
// Work item = (decode member, layer, kv head, split of `split` tokens), one
// WARP per item (8 independent warps per CTA).  The KV pool is addressed by
// TMA as a 2-D tensor [n_pages * rows * bs][128] bf16: a 16-position tile of
// one (layer, K|V, kv head) is 1 box of 16 rows (bs >= 16) or 16/bs boxes of
// bs rows, split into two 64-column halves, 128B-swizzled.  Each warp runs a
// 3-stage mbarrier pipeline of K+V tiles (8 KB per stage); the G query heads
// that share the KV head are the M rows (padded to 16) of
//   S = Q K^T   (mma.sync m16n8k16 bf16 -> fp32, 16 per tile)
//   O += P V    (16 per tile; P re-packed from S's accumulator fragments)
// with the online softmax in registers (FlashAttention-2 style).  Partial
// (O, m, l) per item go to dec_part; k_decode_reduce combines the splits.
#pragma once
#include <cuda.h>
#include "data_plane.cuh"

namespace co {

constexpr int TC_WARPS = 8;
constexpr int TC_STAGES = 3;
constexpr int TC_TILE_BYTES = 16 * 128 * 2;                 // one K or V tile
constexpr int TC_STAGE_BYTES = 2 * TC_TILE_BYTES;           // K + V
constexpr int TC_SMEM = TC_WARPS * TC_STAGES * TC_STAGE_BYTES + 1024 + TC_WARPS * TC_STAGES * 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
    }
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
// byte offset of (tile row t, 16B chunk c) in a 64-column, 128B-swizzled half
__device__ __forceinline__ uint32_t swz(int t, int c) { return (uint32_t)(t * 128 + ((c ^ (t & 7)) << 4)); }

struct DecItem {
    int32_t m, i, layer, kh, owner, pos_lo, pos_hi, nt0;
};

__device__ __forceinline__ bool dec_item(const Dev& d, const DataCfg& x, const DataCtl* dc, int32_t it, DecItem& o) {
    int32_t lo = 0, hi = dc->n_dec;
    while (hi - lo > 1) {
        int32_t mid = (lo + hi) >> 1;
        if (x.dec_item_off[mid] <= it) lo = mid; else hi = mid;
    }
    o.m = lo;
    o.i = x.dec_idx[lo];
    const int32_t ctx = x.dec_ctx[lo];
    const int32_t nsplit = (ctx + x.split - 1) / x.split;
    const int32_t rel = it - x.dec_item_off[lo];
    const int32_t lh = rel / nsplit, sp = rel % nsplit;
    o.layer = lh / x.Hkv;
    o.kh = lh % x.Hkv;
    const int32_t t0 = sp * x.split, t1 = min(ctx, t0 + x.split);
    const int32_t host = d.host[o.i];
    if (host >= 0) {  // guest: token k at host position end-1-k
        const int32_t end = d.off[o.i] + d.granted[o.i];
        o.owner = host;
        o.pos_lo = end - t1;
        o.pos_hi = end - t0;
    } else {
        o.owner = o.i;
        o.pos_lo = t0;
        o.pos_hi = t1;
    }
    o.nt0 = o.pos_lo & ~15;
    return true;
}

// issue the K and V boxes of the 16-position tile starting at P
__device__ __forceinline__ void dec_issue(const Dev& d, const DataCfg& x, const CUtensorMap* map, const DecItem& w,
                                         int32_t P, uint32_t kdst, uint32_t bar) {
    const int bs = d.bs;
    const int box = bs < 16 ? bs : 16;
    const int32_t rowK = (w.layer * 2 + 0) * x.Hkv + w.kh, rowV = rowK + x.Hkv;
    const int32_t npg = d.tab_len[w.owner];
    mbar_expect(bar, TC_STAGE_BYTES);
    for (int32_t s = 0; s < 16; s += box) {
        const int32_t pos = P + s;
        int32_t pi = pos / bs;
        int32_t page = pi < npg ? page_of(d, w.owner, pi) : 0;  // past the table: any valid page, masked
        const int32_t slot = pos % bs;
        const int32_t rk = (page * x.rows + rowK) * bs + slot;
        const int32_t rv = (page * x.rows + rowV) * bs + slot;
        const uint32_t off = (uint32_t)s * 128;
        tma_2d(kdst + off, map, 0, rk, bar);
        tma_2d(kdst + 2048 + off, map, 64, rk, bar);
        tma_2d(kdst + TC_TILE_BYTES + off, map, 0, rv, bar);
        tma_2d(kdst + TC_TILE_BYTES + 2048 + off, map, 64, rv, bar);
    }
}

__global__ void __launch_bounds__(TC_WARPS * 32, 1)
    k_decode_tc(Dev d, DataCfg x, DataCtl* dc, const __grid_constant__ CUtensorMap kvmap) {
    const Ctl& c = *d.ctl;
    if (!c.active || !x.decode_on || !dc->decode_enabled) return;
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tiles = smem_u32(base) + warp * TC_STAGES * TC_STAGE_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + TC_WARPS * TC_STAGES * TC_STAGE_BYTES) + warp * TC_STAGES;
    if (lane == 0)
        for (int s = 0; s < TC_STAGES; s++) mbar_init(smem_u32(&bars[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int32_t nitems = dc->dec_items;
    const int G = x.Hq / x.Hkv;
    const uint32_t step = (uint32_t)c.steps;
    const int r = lane >> 2, cq = lane & 3;  // fragment row / column pair
    const float qscale = rsqrtf((float)x.D) * 1.4426950408889634f;  // exp2 domain
    uint32_t fill = 0, use = 0;  // tiles issued / consumed by this warp (ring position + phase)
    for (int32_t it = blockIdx.x * TC_WARPS + warp; it < nitems; it += gridDim.x * TC_WARPS) {
        DecItem w;
        dec_item(d, x, dc, it, w);
        const uint32_t rid = (uint32_t)d.rid[w.i];
        // Q as A fragments (rows >= G are zero padding)
        uint32_t qa[8][4];
#pragma unroll
        for (int kk = 0; kk < 8; kk++) {
#pragma unroll
            for (int h = 0; h < 2; h++) {  // h: row r / r+8
                const int row = r + 8 * h;
                float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f;
                if (row < G) {
                    const int qh = w.kh * G + row;
                    const int d0 = kk * 16 + 2 * cq;
                    v0 = q_value(rid, step, w.layer, qh, d0) * qscale;
                    v1 = q_value(rid, step, w.layer, qh, d0 + 1) * qscale;
                    v2 = q_value(rid, step, w.layer, qh, d0 + 8) * qscale;
                    v3 = q_value(rid, step, w.layer, qh, d0 + 9) * qscale;
                }
                qa[kk][h] = pack_bf16(v0, v1);
                qa[kk][h + 2] = pack_bf16(v2, v3);
            }
        }
        float o[16][4];
#pragma unroll
        for (int j = 0; j < 16; j++) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
        float mrow = -INFINITY, lrow = 0.f;
        const int32_t ntiles = (w.pos_hi - w.nt0 + 15) / 16;
        // prologue
        for (int32_t t = 0; t < ntiles && t < TC_STAGES; t++) {
            const uint32_t s = (fill + t) % TC_STAGES;
            if (lane == 0) dec_issue(d, x, &kvmap, w, w.nt0 + 16 * t, tiles + s * TC_STAGE_BYTES, smem_u32(&bars[s]));
        }
        const uint32_t fill0 = fill;
        fill += ntiles;
        for (int32_t t = 0; t < ntiles; t++) {
            const uint32_t s = (use) % TC_STAGES;
            const uint32_t ph = (use / TC_STAGES) & 1;
            mbar_wait(smem_u32(&bars[s]), ph);
            use++;
            const uint32_t kt = tiles + s * TC_STAGE_BYTES, vt = kt + TC_TILE_BYTES;
            // ---- S = Q K^T : two n8 tiles of tokens ----
            float sacc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
            for (int kk = 0; kk < 8; kk++) {
                // matrices: (tok 0-7, dims 16kk..+7), (tok 0-7, +8..15), (tok 8-15, ..), (tok 8-15, +8)
                const int mi = lane >> 3, rr = lane & 7;
                const int tok = rr + ((mi >> 1) << 3);
                const int chunk = kk * 2 + (mi & 1);   // 16B chunk within 256 B of dims
                const int half = chunk >> 3;            // which 64-column half
                uint32_t b0, b1, b2, b3;
                ldsm_x4(kt + half * 2048 + swz(tok, chunk & 7), b0, b1, b2, b3);
                mma_bf16(sacc[0], qa[kk], b0, b1);
                mma_bf16(sacc[1], qa[kk], b2, b3);
            }
            // ---- mask + online softmax over the 16 positions of this tile ----
            const int32_t P = w.nt0 + 16 * t;
            float sv[4];
#pragma unroll
            for (int j = 0; j < 2; j++)
#pragma unroll
                for (int e = 0; e < 2; e++) {
                    const int32_t pos = P + 8 * j + 2 * cq + e;
                    sv[2 * j + e] = (pos >= w.pos_lo && pos < w.pos_hi) ? sacc[j][e] : -INFINITY;
                }
            float mx = fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3]));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float mnew = fmaxf(mrow, mx);
            const float corr = exp2f(mrow - mnew);
            float p[4], ps = 0.f;
#pragma unroll
            for (int e = 0; e < 4; e++) { p[e] = exp2f(sv[e] - mnew); ps += p[e]; }
            ps += __shfl_xor_sync(0xffffffffu, ps, 1);
            ps += __shfl_xor_sync(0xffffffffu, ps, 2);
            lrow = lrow * corr + ps;
            mrow = mnew;
#pragma unroll
            for (int j = 0; j < 16; j++) { o[j][0] *= corr; o[j][1] *= corr; }
            // P as the A fragment of a k16 step (rows r+8 are padding)
            uint32_t pa[4];
            pa[0] = pack_bf16(p[0], p[1]);
            pa[1] = 0u;
            pa[2] = pack_bf16(p[2], p[3]);
            pa[3] = 0u;
            // ---- O += P V : 16 n8 tiles of dims ----
#pragma unroll
            for (int jj = 0; jj < 8; jj++) {
                // matrices (transposed): (tok 0-7, dims 16jj..+7), (tok 8-15, same), (tok 0-7, +8..15), (tok 8-15, +8)
                const int mi = lane >> 3, rr = lane & 7;
                const int tok = rr + ((mi & 1) << 3);
                const int chunk = jj * 2 + (mi >> 1);
                const int half = chunk >> 3;
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(vt + half * 2048 + swz(tok, chunk & 7), b0, b1, b2, b3);
                mma_bf16(o[2 * jj], pa, b0, b1);
                mma_bf16(o[2 * jj + 1], pa, b2, b3);
            }
            __syncwarp();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            // refill this stage with tile t + STAGES of the same item
            if (t + TC_STAGES < ntiles && lane == 0)
                dec_issue(d, x, &kvmap, w, w.nt0 + 16 * (t + TC_STAGES), kt, smem_u32(&bars[s]));
        }
        (void)fill0;
        // partial result of this item: rows r < G
        if (r < G) {
            float* out = x.dec_part + ((int64_t)it * G + r) * (x.D + 2);
#pragma unroll
            for (int j = 0; j < 16; j++) {
                out[8 * j + 2 * cq] = o[j][0];
                out[8 * j + 2 * cq + 1] = o[j][1];
            }
            if (cq == 0) {
                // store m in the natural-log domain like k_decode (exp2 domain / log2 e)
                out[x.D] = mrow * 0.6931471805599453f;
                out[x.D + 1] = lrow;
            }
        }
    }
}

}  // namespace co
