// Grid-wide (data-parallel) phases of one engine step:
//   k_begin     engine.py:606-614 guards, clock jump and the arrival window
//   k_admit     engine.py:344-353 + estimation.py:85-128 (row a1)
//   k_classify  engine.py:284-334 snapshot + scheduler.py:129-163 (rows a2/a3):
//               one 64-bit composite sort key per request so ONE radix sort
//               yields N_w (by rt,id), N'_w (by queue key) and the running
//               set in arrival order as contiguous segments.
#pragma once
#include "engine_state.cuh"
#include "pool_ops.cuh"

namespace co {

__global__ void k_begin(Dev d, int32_t guard) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    Ctl& c = *d.ctl;
    c.active = 0;
    if (d.result) d.result[0] = -1;
    if (c.done) { c.last_result = 0; return; }
    if (c.paused || c.error) return;
    // append-buffer headroom for the worst case of this step: pause (the host
    // drains and relaunches) before touching any state
    {
        int64_t now = c.now;
        if (c.n_live == 0 && c.next_pending < d.n && d.arr[c.next_pending] > now) now = d.arr[c.next_pending];
        int32_t lo = c.next_pending, hi = d.n;
        while (lo < hi) {
            int32_t mid = lo + (hi - lo) / 2;
            if (d.arr[mid] <= now) lo = mid + 1; else hi = mid;
        }
        int64_t live_after = (int64_t)c.n_live + (lo - c.next_pending);
        bool full = c.sample_count + 1 > d.sample_cap;
        if (d.record_events)
            full = full || c.ev_count + (lo - c.next_pending) + 4 * live_after + 8 > d.ev_cap ||
                   c.mem_count + live_after + 8 > d.mem_cap;
        if (full) { c.paused = 1; return; }
    }
    c.last_result = 0;
    c.sid += 1;
    if (d.dp.on) { d.dctl->n_dec = 0; d.dctl->dec_items = 0; }
    c.cnt_nw = c.cnt_nwp = c.cnt_run = 0;
    if (guard) {
        // engine.py:644-659 no-progress guard, evaluated before each step()
        int64_t m[5] = {c.now, c.gen_total, c.n_live, (int64_t)(d.n - c.next_pending), c.fp_sum};
        bool same = c.has_mark;
        for (int k = 0; k < 5; k++) same = same && m[k] == c.mark[k];
        if (same) {
            c.streak += 1;
            if (c.streak > 1000000) { c.error = 3; c.done = 1; return; }
        } else {
            c.streak = 0;
        }
        for (int k = 0; k < 5; k++) c.mark[k] = m[k];
        c.has_mark = 1;
    }
    c.steps += 1;
    if (c.n_live == 0 && c.next_pending >= d.n) { c.done = 1; return; }
    if (c.now > c.horizon) { c.done = 1; return; }
    if (c.n_live == 0 && d.arr[c.next_pending] > c.now) c.now = d.arr[c.next_pending];
    int32_t lo = c.next_pending, hi = d.n;
    while (lo < hi) {
        int32_t mid = lo + (hi - lo) / 2;
        if (d.arr[mid] <= c.now) lo = mid + 1; else hi = mid;
    }
    int32_t adm = lo - c.next_pending;
    c.adm_lo = c.next_pending;
    c.adm_hi = lo;
    c.next_pending = lo;
    c.n_live += adm;
    c.decisions += c.n_live;  // one decision per live request per step
    if (d.record_events) c.ev_count += adm;  // arrive records written by k_admit
    c.active = 1;
}

// estimation.py:92-99 + 122-128 with the host-drawn noise, and the arrive
// event (engine.py:353); runs inside k_classify for the admission window
__device__ __forceinline__ void admit_one(const Dev& d, int32_t i, int32_t lo, int64_t ev0) {
    int32_t t = d.tout[i];
    int32_t p = t - d.err[i];
    if (p < 1) p = 1;
    bool under = t >= p;
    if (d.flip[i]) under = !under;
    int32_t e = under ? p + d.pad : (p - d.pad > 1 ? p - d.pad : 1);
    d.pred[i] = p;
    d.est[i] = e;
    d.state[i] = ST_WAITING;
    if (d.record_events) {
        co_event ev;
        ev.kind = CO_EV_ARRIVE; ev.idx = i; ev.t = d.arr[i]; ev.a = ev.b = ev.c = 0;
        d.events[ev0 + (i - lo)] = ev;
    }
}

// class codes in the top two key bits: [class:2][blown:1][time].  Keys are
// written at position idrank[i], so the sort's input is in req_id order and
// the (stable) radix sort breaks every tie by id without id-rank key bits.
constexpr uint64_t K_NW = 0, K_NWP = 1, K_RUN = 2;

__global__ void k_classify(Dev d) {
    const Ctl& c = *d.ctl;
    if (!c.active) return;
    const int64_t now = c.now, ti = c.t_i, eps = d.eps;
    const int cs = d.key_bits - 2, fs = d.key_bits - 3;  // class / blown-flag bit positions
    int32_t cw = 0, cwp = 0, cr = 0;
    const int32_t hi_live = c.next_pending;
    const int32_t alo = c.adm_lo, ahi = c.adm_hi;
    const int64_t ev0 = c.ev_count - (ahi - alo);
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < d.n; i += gridDim.x * blockDim.x) {
        uint64_t key = ~0ull;
        if (i >= alo && i < ahi) admit_one(d, i, alo, ev0);
        if (i < hi_live) {
            int8_t s = d.state[i];
            if (s >= ST_WAITING && s <= ST_PREEMPTED) {
                const PV v = make_pv(d, i, now);  // the planner's snapshot view
                uint4* dst = reinterpret_cast<uint4*>(d.views + i);
                const uint4* src = reinterpret_cast<const uint4*>(&v);
                dst[0] = src[0]; dst[1] = src[1]; dst[2] = src[2]; dst[3] = src[3];
            }
            if (s == ST_WAITING || s == ST_PREEMPTED) {
                // every waiting view is ready (engine.py:311-312); rt = D - now
                int64_t D = d.first_tok[i] < 0 ? d.arr[i] + d.slo_ttft[i] : d.last_tok[i] + d.slo_tbt[i];
                int64_t rt = D - now;
                if (rt >= -eps && rt - ti < eps) {
                    key = (K_NW << cs) | (uint64_t)D;
                    cw++;
                } else {
                    // queue_key (scheduler.py:151-157): (0, rt, id) / (1, arrival, id)
                    uint64_t flag = rt < 0 ? 1 : 0;
                    uint64_t v = flag ? (uint64_t)d.arr[i] : (uint64_t)D;
                    key = (K_NWP << cs) | (flag << fs) | v;
                    cwp++;
                }
            } else if (s == ST_RUNNING) {
                key = (K_RUN << cs) | (uint64_t)i;
                cr++;
            }
        }
        const int32_t pos = d.idrank[i];
        d.keys_in[pos] = key;
        d.vals_in[pos] = (uint32_t)i;
    }
    // warp-aggregated counters
    for (int o = 16; o > 0; o >>= 1) {
        cw += __shfl_xor_sync(0xffffffffu, cw, o);
        cwp += __shfl_xor_sync(0xffffffffu, cwp, o);
        cr += __shfl_xor_sync(0xffffffffu, cr, o);
    }
    if ((threadIdx.x & 31) == 0) {
        Ctl* cm = d.ctl;
        if (cw) atomicAdd(&cm->cnt_nw, cw);
        if (cwp) atomicAdd(&cm->cnt_nwp, cwp);
        if (cr) atomicAdd(&cm->cnt_run, cr);
    }
}

}  // namespace co
