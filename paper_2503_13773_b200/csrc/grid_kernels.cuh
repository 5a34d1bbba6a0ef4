// Grid-wide (data-parallel) phases of one engine step:
//   begin_*     engine.py:606-614 guards, clock jump and the arrival window
//               (evaluated by every k_classify CTA, committed by k_serial)
//   admit_one   engine.py:344-353 + estimation.py:85-128 (row a1), in k_classify
//   k_classify  engine.py:284-334 snapshot + scheduler.py:129-163 (rows a2/a3):
//               one 64-bit composite sort key per request so ONE radix sort
//               yields N_w (by rt,id), N'_w (by queue key) and the running
//               set in arrival order as contiguous segments.
#pragma once
#include "engine_state.cuh"
#include "pool_ops.cuh"

namespace co {

// engine.py:606-614 step guards, the clock jump and the arrival window, as a
// PURE function of the control block at the step's start: every k_classify
// CTA evaluates it to know the step's clock and admission window, and
// k_serial's thread 0 evaluates it again and commits it (begin_commit)
// before planning -- so no kernel of its own runs ahead of classify, and no
// CTA ever reads a half-updated control block.  reset = 1: the host consumed
// the whole append log from the step mirror, so it restarts empty.
struct BeginR {
    int32_t active, paused, done, err3, adm_lo, adm_hi;
    int64_t now, ev0;  // ev0: where this step's arrive records start
};
__device__ __forceinline__ int32_t arrivals_upto(const Dev& d, int32_t lo, int64_t now) {
    // first index >= lo with arr > now: gallop from lo (the window is usually
    // short), then binary search
    int32_t hi = d.n;
    if (lo >= hi || d.arr[lo] > now) return lo;
    int32_t step = 1, prev = lo;
    while (true) {
        const int32_t probe = lo + step;
        if (probe >= hi) break;
        if (d.arr[probe] > now) { hi = probe; break; }
        prev = probe;
        step <<= 1;
    }
    lo = prev + 1;
    while (lo < hi) {
        const int32_t mid = lo + (hi - lo) / 2;
        if (d.arr[mid] <= now) lo = mid + 1; else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ BeginR begin_eval(const Dev& d, const Ctl& c, int32_t guard, int32_t reset) {
    BeginR r{};
    r.active = 0;
    const int64_t ev_count = reset ? 0 : c.ev_count, mem_count = reset ? 0 : c.mem_count,
                  sample_count = reset ? 0 : c.sample_count;
    const int32_t paused = reset ? 0 : c.paused;
    r.ev0 = ev_count;
    r.now = c.now;
    if (c.done) { r.done = 1; return r; }
    if (paused || c.error) { r.paused = paused; return r; }
    // append-buffer headroom for the worst case of this step: pause (the host
    // drains and relaunches) before touching any state
    {
        int64_t now = c.now;
        if (c.n_live == 0 && c.next_pending < d.n && d.arr[c.next_pending] > now) now = d.arr[c.next_pending];
        const int32_t lo = arrivals_upto(d, c.next_pending, now);
        const int64_t live_after = (int64_t)c.n_live + (lo - c.next_pending);
        bool full = sample_count + 1 > d.sample_cap;
        if (d.record_events)
            full = full || ev_count + (lo - c.next_pending) + 4 * live_after + 8 > d.ev_cap ||
                   mem_count + live_after + 8 > d.mem_cap;
        if (full) { r.paused = 1; return r; }
    }
    if (guard) {
        // engine.py:644-659 no-progress guard, evaluated before each step()
        const int64_t m[5] = {c.now, c.gen_total, c.n_live, (int64_t)(d.n - c.next_pending), c.fp_sum};
        bool same = c.has_mark;
        for (int k = 0; k < 5; k++) same = same && m[k] == c.mark[k];
        if (same && c.streak + 1 > 1000000) { r.err3 = 1; r.done = 1; return r; }
    }
    if (c.n_live == 0 && c.next_pending >= d.n) { r.done = 1; return r; }
    if (c.now > c.horizon) { r.done = 1; return r; }
    int64_t now = c.now;
    if (c.n_live == 0 && d.arr[c.next_pending] > now) now = d.arr[c.next_pending];
    r.now = now;
    r.adm_lo = c.next_pending;
    r.adm_hi = arrivals_upto(d, c.next_pending, now);
    r.active = 1;
    return r;
}
// k_serial thread 0: apply the step's begin to the control block (what the
// round-1 k_begin kernel wrote), given the classify CTAs' counts untouched
__device__ __forceinline__ void begin_commit(const Dev& d, int32_t guard, int32_t reset) {
    Ctl& c = *d.ctl;
    const BeginR r = begin_eval(d, c, guard, reset);
    if (reset) { c.ev_count = 0; c.mem_count = 0; c.sample_count = 0; c.paused = 0; }
    c.active = 0;
    if (d.result) d.result[0] = -1;
    if (c.done) { c.last_result = 0; return; }
    if (c.paused || c.error) return;
    if (r.paused) { c.paused = 1; return; }
    c.last_result = 0;
    c.sid += 1;
    if (d.dp.on) { d.dctl->n_dec = 0; d.dctl->dec_items = 0; }
    if (guard) {
        const int64_t m[5] = {c.now, c.gen_total, c.n_live, (int64_t)(d.n - c.next_pending), c.fp_sum};
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
    if (r.done) { c.done = 1; return; }
    c.now = r.now;
    const int32_t adm = r.adm_hi - r.adm_lo;
    c.adm_lo = r.adm_lo;
    c.adm_hi = r.adm_hi;
    c.next_pending = r.adm_hi;
    c.n_live += adm;
    c.decisions += c.n_live;  // one decision per live request per step
    if (d.record_events) c.ev_count += adm;  // arrive records written by k_classify
    c.active = 1;
}
// the classify counters for the NEXT step (k_serial's tail, after the
// planner consumed this step's)
__device__ __forceinline__ void classify_counters_reset(const Dev& d) {
    Ctl& c = *d.ctl;
    c.cnt_nw = c.cnt_nwp = c.cnt_run = c.cnt_blown = c.cnt_cand = 0;
    c.kmin = ~0ull;
    c.kmax = 0;
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
    d.key0[i] = wait_key(d, i);
    if (d.record_events) {
        co_event ev;
        ev.kind = CO_EV_ARRIVE; ev.idx = i; ev.t = d.arr[i]; ev.a = ev.b = ev.c = 0;
        d.events[ev0 + (i - lo)] = ev;
    }
}

// k_classify (contiguous index chunk per block): admission, and the
// classification of scheduler.py:129-163 into
//   running (index order)              -> run_tmp   (block-ordered)
//   critical N_w                       -> crit_idx  (unordered; sorted by the planner)
//   N'_w blown, rt < 0 (arrival order) -> blown_tmp (block-ordered; SoA order IS (arrival, id))
//   N'_w rt >= 0 ordered by (D, id)    -> counted (key range kmin..kmax); the head
//                                         (key < thr) is appended to cand[]
// The planner's 64-byte views are written for the running, critical, blown
// and candidate requests only: a waiting request outside the head costs one
// state byte and one key read per step.
__global__ void __launch_bounds__(256) k_classify(Dev d, int32_t guard, int32_t reset) {
    pdl_enter();
    __shared__ int32_t sc[32];
    __shared__ uint64_t kr[2][8];
    __shared__ int32_t tot_s[2];
    __shared__ BeginR br;
    const Ctl& c = *d.ctl;
    // this thread's first slot: its state and waiting key are loaded before
    // the begin's control-block round trip, so the two overlap (admitted
    // slots are rewritten below and take admit_one's values instead)
    const int32_t i0 = blockIdx.x * d.chunk + (int32_t)threadIdx.x;
    int8_t s_pre = ST_PENDING;
    uint64_t k_pre = 0;
    const uint64_t thr_pre = c.thr;  // (not changed by the begin)
    if (i0 < d.n) { s_pre = d.state[i0]; k_pre = d.key0[i0]; }
    if (threadIdx.x == 0) {
        br = begin_eval(d, c, guard, reset);  // the step's begin, read-only
    } else if (i0 < d.n && (s_pre == ST_RUNNING ||
                            ((s_pre == ST_WAITING || s_pre == ST_PREEMPTED) && k_pre < thr_pre))) {
        pv_prefetch(d, i0);  // running slots and the N'_w head always get a view
    }
    __syncthreads();
    if (!br.active) return;
    const int64_t now = br.now, ti = c.t_i, eps = d.eps;
    const uint64_t thr = c.thr;
    const int32_t hi_live = br.adm_hi;
    const int32_t alo = br.adm_lo, ahi = br.adm_hi;
    const int64_t ev0 = br.ev0;
    const int32_t lo = blockIdx.x * d.chunk, hi = min(d.n, lo + d.chunk);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t run_base = 0, blown_base = 0, ncrit = 0, nf0 = 0;
    uint64_t kmin = ~0ull, kmax = 0;
    for (int32_t c0 = lo; c0 < hi; c0 += 256) {
        const int32_t i = c0 + (int32_t)threadIdx.x;
        int32_t is_run = 0, is_blown = 0, is_cand = 0;
        if (i < hi) {
            int8_t s;
            uint64_t k;
            if (i >= alo && i < ahi) {
                admit_one(d, i, alo, ev0);
                s = ST_WAITING;
                k = d.key0[i];
            } else if (c0 == lo) {
                s = s_pre;
                k = k_pre;
            } else {
                s = d.state[i];
                k = d.key0[i];
            }
            if (i < hi_live) {
                bool view = false;
                if (s == ST_WAITING || s == ST_PREEMPTED) {
                    const int32_t wc = wait_class(d, s, k, now, ti, eps);
                    if (wc == WC_CRIT) {
                        d.crit_idx[atomicAdd(&d.ctl->cnt_nw, 1)] = i;
                        ncrit++;
                        view = true;
                    } else if (wc == WC_BLOWN) {
                        is_blown = 1;  // queue key (1, arrival, id)
                        view = true;
                    } else {
                        nf0++;
                        kmin = k < kmin ? k : kmin;
                        kmax = k > kmax ? k : kmax;
                        if (k < thr) { is_cand = 1; view = true; }
                    }
                } else if (s == ST_RUNNING) {
                    is_run = 1;
                    view = true;
                }
                if (view) {
                    const PV v = make_pv(d, i, now);  // the planner's snapshot view
                    uint4* dst = reinterpret_cast<uint4*>(d.views + i);
                    const uint4* src = reinterpret_cast<const uint4*>(&v);
                    dst[0] = src[0]; dst[1] = src[1]; dst[2] = src[2]; dst[3] = src[3];
                }
            }
        }
        // the head candidates: one atomic per warp
        const unsigned cb = __ballot_sync(0xffffffffu, is_cand);
        if (cb) {
            int32_t base = 0;
            if (lane == 0) base = atomicAdd(&d.ctl->cnt_cand, __popc(cb));
            base = __shfl_sync(0xffffffffu, base, 0);
            const int32_t pos = base + __popc(cb & ((1u << lane) - 1));
            if (is_cand && pos < CAND_CAP) d.cand[pos] = i;
        }
        // order-preserving block compaction of the running and blown flags
        int32_t packed = is_run | (is_blown << 16), x = packed;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) sc[w] = x;
        __syncthreads();
        if (w == 0) {
            int32_t y = lane < 8 ? sc[lane] : 0, z = y;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int32_t q = __shfl_up_sync(0xffffffffu, z, o);
                if (lane >= o) z += q;
            }
            if (lane < 8) sc[lane] = z - y;
            if (lane == 7) { tot_s[0] = z & 0xffff; tot_s[1] = z >> 16; }
        }
        __syncthreads();
        const int32_t ex = sc[w] + x - packed;
        if (is_run) d.run_tmp[lo + run_base + (ex & 0xffff)] = i;
        if (is_blown) d.blown_tmp[lo + blown_base + (ex >> 16)] = i;
        run_base += tot_s[0];
        blown_base += tot_s[1];
        __syncthreads();
    }
    // block totals: counts, key range
    for (int o = 16; o > 0; o >>= 1) {
        ncrit += __shfl_xor_sync(0xffffffffu, ncrit, o);
        nf0 += __shfl_xor_sync(0xffffffffu, nf0, o);
        uint64_t a = __shfl_xor_sync(0xffffffffu, kmin, o), b = __shfl_xor_sync(0xffffffffu, kmax, o);
        kmin = a < kmin ? a : kmin;
        kmax = b > kmax ? b : kmax;
    }
    if (lane == 0) { kr[0][w] = kmin; kr[1][w] = kmax; sc[w] = nf0; }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t mn = ~0ull, mx = 0;
        int32_t f = 0;
        for (int k = 0; k < 8; k++) {
            mn = kr[0][k] < mn ? kr[0][k] : mn;
            mx = kr[1][k] > mx ? kr[1][k] : mx;
            f += sc[k];
        }
        Ctl* cm = d.ctl;
        if (f) {
            atomicAdd(&cm->cnt_nwp, f);
            atomicMin((unsigned long long*)&cm->kmin, (unsigned long long)mn);
            atomicMax((unsigned long long*)&cm->kmax, (unsigned long long)mx);
        }
        if (run_base) atomicAdd(&cm->cnt_run, run_base);
        if (blown_base) atomicAdd(&cm->cnt_blown, blown_base);
        d.blk_cnt[2 * blockIdx.x] = run_base;
        d.blk_cnt[2 * blockIdx.x + 1] = blown_base;
    }
}

}  // namespace co
