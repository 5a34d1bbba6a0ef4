// Shared pieces of the paged-decode path: mbarrier / TMA primitives and the
// split-KV work-item decomposition (member, layer, kv head, split) whose
// partial results k_decode_reduce combines.
#pragma once
#include <cuda.h>
#include <cstdio>
#include "data_plane.cuh"

namespace co {

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
#ifdef CO_MBAR_WATCHDOG  // development aid: report a stuck wait, then trap
    long long spins = 0;
#endif
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
#ifdef CO_MBAR_WATCHDOG
        if (++spins == (1ll << 22))
            printf("mbar watchdog: block %d thread %d bar smem+0x%x parity %u\n", blockIdx.x, threadIdx.x, bar & 0x3ffff,
                   phase);
        if (spins == (1ll << 24)) __trap();
#endif
    }
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
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

}  // namespace co
