// The reference's pure scheduling ops (scheduler.py:129-279, preemption.py:
// 46-75) over a caller's view table, on the device, through the planner's own
// device code: the criticality predicate and queue keys k_plan sorts by, the
// block compaction / rank sort of block_ops.cuh, the token-budget prefix, the
// exact integer amortize() (largest remainder over u64/u128 weights), the
// provider argmin of pair_release and the victim key.  One single-CTA kernel
// per call; the reference's own scheduler/preemption tests drive it
// (tests/test_sched_ops_device.py).  Included by cacheopt.cu.
//
// rows: int64 [n][8], columns per op (see include/cacheopt.h CO_SOP_*);
// `rank` is the row's position in ascending req_id order (every reference
// key ends in req_id, so ranks break ties exactly like ids).
#pragma once

namespace co {

__global__ void __launch_bounds__(NT, 1) k_sched_op(Dev d, int32_t op, int32_t n, const int64_t* __restrict__ rows,
                                                    const int64_t* __restrict__ prm, int64_t* out) {
    extern __shared__ __align__(16) uint8_t sop_smem[];
    PlanSh& S = *reinterpret_cast<PlanSh*>(sop_smem);
    const int tid = threadIdx.x;
    auto R = [&](int32_t k, int c) -> int64_t { return rows[8 * k + c]; };
    switch (op) {
        case CO_SOP_CLASSIFY: {
            // scheduler.py:129-163.  row: rank, list (0 waiting, 1 running),
            // rt (waiting: rt_us(v); running: remaining_tbt), returned, arrival
            const int64_t ti = prm[0], eps = prm[1];
            auto crit_rt = [&](int64_t r) { return r >= -eps && r - ti < eps; };  // as k_plan's
            int32_t* lists[4] = {d.l_part, d.l_grp, d.l_pro, d.l_ful};
            int32_t cnt[4];
            for (int cls = 0; cls < 4; cls++) {
                cnt[cls] = blk_compact(nullptr, n, lists[cls], [&](int32_t k) {
                    const bool running = R(k, 1) != 0;
                    if (running && !R(k, 3)) return false;  // only returned running requests classify
                    const int c = (running ? 1 : 0) + (crit_rt(R(k, 2)) ? 0 : 2);
                    return c == cls;
                }, S.b);
                if (cls < 2) {  // n_w / n_r by (rt, id)
                    blk_sort(lists[cls], cnt[cls], [&](int32_t k, uint64_t& k0, uint64_t& k1, uint64_t& k2) {
                        k0 = (uint64_t)(R(k, 2) + (1ll << 62)); k1 = (uint64_t)R(k, 0); k2 = 0;
                    }, d, S.b);
                } else {        // queue_key: (0, rt, id) or blown (1, arrival, id)
                    blk_sort(lists[cls], cnt[cls], [&](int32_t k, uint64_t& k0, uint64_t& k1, uint64_t& k2) {
                        const int64_t r = R(k, 2);
                        k0 = r < 0 ? 1 : 0;
                        k1 = r < 0 ? (uint64_t)(R(k, 4) + (1ll << 62)) : (uint64_t)r;
                        k2 = (uint64_t)R(k, 0);
                    }, d, S.b);
                }
            }
            int64_t base = 4;
            for (int cls = 0; cls < 4; cls++) {
                if (tid == 0) out[cls] = cnt[cls];
                for (int32_t k = tid; k < cnt[cls]; k += (int)blockDim.x) out[base + k] = lists[cls][k];
                base += cnt[cls];
            }
            return;
        }
        case CO_SOP_FILL_BUDGET: {
            // scheduler.py:182-200: row: chunk; prm: budget, consumed
            const int64_t budget = prm[0];
            int64_t used_base = prm[1];
            int32_t ksel = n;
            for (int32_t base = 0; base < n; base += (int)blockDim.x) {
                const int32_t k = base + tid;
                const int32_t ch = k < n ? (int32_t)R(k, 0) : 0;
                int32_t tot;
                const int32_t ex = blk_excl_scan(ch, &tot, S.b);
                const bool over = k < n && used_base + ex + ch > budget;
                const uint64_t mk = blk_min(over ? (uint64_t)k : ~0ull, S.b);
                if (mk != ~0ull) { ksel = (int32_t)mk; break; }
                used_base += tot;
            }
            if (tid == 0) { out[0] = ksel; out[1] = prm[1] > budget ? 1 : 0; }
            return;
        }
        case CO_SOP_ALLOCATE_REMAINING: {
            // scheduler.py:211-243 through k_plan's amortize() with block
            // size 1 (no block flooring).  row: rank, m_tokens, rt_us, prompt_len
            for (int32_t p = tid; p < n; p += (int)blockDim.x) {
                PV v{};
                v.i = p;
                v.rt = R(p, 2);
                const int64_t pr = R(p, 3);
                v.kvn = (int32_t)(pr > 0x7fffffff ? 0x7fffffff : pr);
                v.idrank = (int32_t)R(p, 0);
                S.pv[p] = v;
                S.pneed[p] = (int32_t)R(p, 1);
                d.l_part[p] = p;
                const_cast<int32_t*>(d.idrank)[p] = (int32_t)R(p, 0);
                d.l_grp[p] = p;
            }
            __syncthreads();
            int64_t tot = 0;
            if (d.inv) amortize<true>(d, S, d.l_grp, n, prm[0], 0, &tot);
            else amortize<false>(d, S, d.l_grp, n, prm[0], 0, &tot);
            __syncthreads();
            for (int32_t p = tid; p < n; p += (int)blockDim.x) out[p] = R(p, 1) > 0 ? (int64_t)S.pgrant[p] : -1;
            return;
        }
        case CO_SOP_PAIR_RELEASE: {
            // scheduler.py:253-266 (k_plan's provider argmin).  row: rank,
            // est_remaining_iters, release_gain; prm: residual, runway
            const int64_t resid = prm[0], runway = prm[1];
            uint64_t best = ~0ull;
            for (int32_t k = tid; k < n; k += (int)blockDim.x) {
                const int64_t er = R(k, 1);
                if (er > runway || R(k, 2) < resid) continue;
                const uint64_t key = ((uint64_t)(er + (1ll << 31)) << 32) | (uint64_t)(uint32_t)R(k, 0);
                best = key < best ? key : best;
            }
            best = blk_min(best, S.b);
            if (tid == 0) {
                out[0] = -1;
                if (best != ~0ull)
                    for (int32_t k = 0; k < n; k++)
                        if ((uint32_t)R(k, 0) == (uint32_t)best) out[0] = k;
            }
            return;
        }
        case CO_SOP_ORDER_VICTIMS: {
            // preemption.py:46-75 with k_plan's victim key.  row: rank,
            // slo_tbt_us, remaining_tokens, occupancy; prm: token_step, n_edges, edges...
            const int64_t step = prm[0];
            const int32_t ne = (int32_t)prm[1];
            for (int32_t k = tid; k < n; k += (int)blockDim.x) d.l_part[k] = k;
            __syncthreads();
            blk_sort(d.l_part, n, [&](int32_t k, uint64_t& k0, uint64_t& k1, uint64_t& k2) {
                uint64_t sb = 0;
                for (int e = 0; e < ne; e++) sb += R(k, 1) >= prm[2 + e] ? 1 : 0;
                const int64_t rem = R(k, 2) > 0 ? R(k, 2) : 0;
                const uint64_t rb = (uint64_t)(rem / step);
                k0 = ((15ull - sb) << 32) | (0x7fffffffull - rb);
                k1 = (uint64_t)(R(k, 3) + (1ll << 62));
                k2 = (uint64_t)R(k, 0);
            }, d, S.b);
            for (int32_t k = tid; k < n; k += (int)blockDim.x) out[k] = d.l_part[k];
            return;
        }
        case CO_SOP_PROACTIVE_INCLUDE: {
            // scheduler.py:269-279 (k_plan's n_pro predicate and key).  row:
            // rank, returned, allocated, target_alloc, est_remaining; prm: m
            const int64_t m = prm[0];
            const int32_t np = blk_compact(nullptr, n, d.l_part, [&](int32_t k) {
                return !R(k, 1) && R(k, 2) < R(k, 3) && R(k, 4) <= m;
            }, S.b);
            blk_sort(d.l_part, np, [&](int32_t k, uint64_t& k0, uint64_t& k1, uint64_t& k2) {
                k0 = (uint64_t)R(k, 4); k1 = (uint64_t)R(k, 0); k2 = 0;
            }, d, S.b);
            if (tid == 0) out[0] = np;
            for (int32_t k = tid; k < np; k += (int)blockDim.x) out[1 + k] = d.l_part[k];
            return;
        }
        default:
            if (tid == 0) out[0] = -1;
    }
}

}  // namespace co

extern "C" int co_sched_op(int32_t op, int32_t n, const int64_t* rows, const int64_t* params, int64_t* out,
                           int32_t device) {
    if (n < 0 || (n > 0 && !rows) || !params || !out) return fail(CO_EINVAL, "bad arguments");
    if (op == CO_SOP_ALLOCATE_REMAINING && n > co::PV_CAP)
        return fail(CO_EINVAL, "allocate_remaining on the device takes at most 1024 demands");
    if (op == CO_SOP_ORDER_VICTIMS && (params[1] < 0 || params[1] > 6 || params[0] < 1))
        return fail(CO_EINVAL, "order_victims: 0..6 SLO edges and token_step >= 1");
    CK(cudaSetDevice(device));
    static bool attr = false;
    if (!attr) {
        CK(cudaFuncSetAttribute(co::k_sched_op, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(co::PlanSh)));
        attr = true;
    }
    const int64_t m = std::max<int32_t>(n, 1);
    std::vector<void*> bufs;
    auto al = [&](auto** p, int64_t count) -> cudaError_t {
        void* q = nullptr;
        cudaError_t e = cudaMalloc(&q, std::max<int64_t>(count, 1) * sizeof(**p));
        if (e == cudaSuccess) bufs.push_back(q);
        *p = static_cast<std::remove_reference_t<decltype(*p)>>(q);
        return e;
    };
    co::Dev d{};
    int64_t *drows = nullptr, *dprm = nullptr, *dout = nullptr;
    const int64_t nout = 2 * m + 8;
    cudaError_t e = cudaSuccess;
    for (cudaError_t x : {al(&drows, 8 * m), al(&dprm, 16), al(&dout, nout), al(&d.l_part, m), al(&d.l_grp, 2 * m),
                          al(&d.l_ful, m), al(&d.l_pro, m), al(const_cast<int32_t**>(&d.idrank), m), al(&d.am_rhi, m), al(&d.am_rlo, m), al(&d.sk0, m),
                          al(&d.sk1, m), al(&d.sk2, m), al(&d.sk_item, m), al(&d.l_part_need, m),
                          al(&d.l_part_grant, m), al(&d.big, 5 * (int64_t)co::INV_LIMBS)})
        if (x != cudaSuccess) e = x;
    int r = CO_OK;
    if (e != cudaSuccess) {
        r = fail(CO_ECUDA, std::string("sched op buffers: ") + cudaGetErrorString(e));
    } else {
        d.bs = 1;  // allocate_remaining: no block flooring
        d.inv = op == CO_SOP_ALLOCATE_REMAINING && params[1] ? 1 : 0;  // scheduler.py:212 invert
        if (n) e = cudaMemcpy(drows, rows, 8 * n * sizeof(int64_t), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(dprm, params, 16 * sizeof(int64_t), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemset(dout, 0, nout * sizeof(int64_t));
        if (e == cudaSuccess) {
            co::k_sched_op<<<1, co::NT, sizeof(co::PlanSh)>>>(d, op, n, drows, dprm, dout);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaMemcpy(out, dout, nout * sizeof(int64_t), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) r = fail(CO_ECUDA, std::string("sched op: ") + cudaGetErrorString(e));
    }
    for (void* p : bufs) cudaFree(p);
    return r;
}
