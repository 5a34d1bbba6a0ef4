// KV pool record operations (kvc.py:156-332) and request lifecycle mechanics
// (engine.py:360-433) as device functions.  They run on ONE thread (thread 0
// of the single-CTA apply kernel): the reference applies a plan strictly in
// list order and every later operation observes the earlier ones, so these
// are ordered by construction.  A reference ValueError (contract violation)
// is a `false` return exactly where the engine swallows it
// (engine.py:448-467); the ones the engine does not swallow set ctl->error.
#pragma once
#include "engine_state.cuh"
#include "data_plane.cuh"

namespace co {

// -- N1 block tables ----------------------------------------------------------
// Pages 0..P-1 (P = capacity // block_size) live on a LIFO free stack; the
// pool pops exactly Delta(footprint)/block_size pages whenever a standalone
// record's footprint grows and pushes a record's pages back in reverse table
// order when it is released, so sum(tab_len) == footprint_sum / block_size.
__device__ __forceinline__ void pop_pages(const Dev& d, int i, int64_t k) {
    Ctl& c = *d.ctl;
    if (k <= 0) return;
    int32_t len = d.tab_len[i];
    if (k > c.free_top || (len + k + TCHUNK - 1) / TCHUNK > d.dir_w) {
        c.error = 5; c.err_info[0] = i; c.err_info[1] = (int32_t)k;
        return;
    }
    int32_t* dir = d.dir + (int64_t)i * d.dir_w;
    const int32_t top = c.free_top;
    for (int64_t j = 0; j < k; j++, len++) {
        if (len % TCHUNK == 0) dir[len / TCHUNK] = d.chunk_stack[--c.chunk_top];
        d.chunk_pool[(int64_t)dir[len / TCHUNK] * TCHUNK + len % TCHUNK] = d.free_stack[top - 1 - j];
    }
    c.free_top = top - (int32_t)k;
    d.tab_len[i] = len;
}
__device__ __forceinline__ void push_table(const Dev& d, int i) {
    Ctl& c = *d.ctl;
    const int32_t len = d.tab_len[i];
    const int32_t* dir = d.dir + (int64_t)i * d.dir_w;
    const int32_t top = c.free_top;
    for (int32_t j = 0; j < len; j++) {
        int32_t k = len - 1 - j;
        d.free_stack[top + j] = d.chunk_pool[(int64_t)dir[k / TCHUNK] * TCHUNK + k % TCHUNK];
        if (k % TCHUNK == 0) d.chunk_stack[c.chunk_top++] = dir[k / TCHUNK];
    }
    c.free_top = top + len;
    d.tab_len[i] = 0;
}

__device__ __forceinline__ void new_record(const Dev& d, int i, int32_t granted, int32_t host, int32_t off) {
    d.holds[i] = 1;
    d.granted[i] = granted;
    d.host[i] = host;
    d.off[i] = off;
    d.rsv[i] = 0;
    d.guest[i] = -1;
    d.gnext[i] = -1;
    d.rec_seq[i] = ++d.ctl->seq;  // dict insertion order (kvc.py:82)
}
__device__ __forceinline__ void drop_record(const Dev& d, int i) {
    d.holds[i] = 0;
    d.ctl->used_sum -= d.used[i];
}

// kvc.py:156-167
__device__ __forceinline__ bool pool_allocate(const Dev& d, int i, int64_t n) {
    if (n < 1 || d.holds[i]) return false;
    int64_t fp = fp_tokens(n, d.bs);
    if (fp > free_tokens(d)) return false;
    new_record(d, i, (int32_t)n, -1, 0);
    d.ctl->fp_sum += fp;
    d.ctl->granted_sum += n;
    pop_pages(d, i, fp / d.bs);
    return true;
}

// unlink guest i from host h's list (kvc.py:294 / :306 `host.guests.remove`)
__device__ __forceinline__ void guest_unlink(const Dev& d, int h, int i) {
    int32_t prev = -1;
    for (int32_t g = d.guest[h]; g >= 0; prev = g, g = d.gnext[g]) {
        if (g != i) continue;
        if (prev < 0) d.guest[h] = d.gnext[g]; else d.gnext[prev] = d.gnext[g];
        d.gnext[g] = -1;
        d.ctl->n_guests -= 1;
        return;
    }
}

// kvc.py:202-227
__device__ __forceinline__ bool pool_embed(const Dev& d, int i, int64_t n, int h, int64_t start) {
    if (n < 1 || d.holds[i] || !d.holds[h]) return false;
    if (d.host[h] >= 0 || i == h) return false;
    if (d.guest[h] >= 0 && !d.stacking) return false;
    if (start < 0 || start + n > d.granted[h]) return false;
    int32_t tail = -1;
    for (int32_t g = d.guest[h]; g >= 0; tail = g, g = d.gnext[g])  // no overlap with an existing guest
        if (!(start + n <= d.off[g] || (int64_t)d.off[g] + d.granted[g] <= start)) return false;
    new_record(d, i, (int32_t)n, h, (int32_t)start);
    if (tail < 0) d.guest[h] = i; else d.gnext[tail] = i;  // guests.append
    d.ctl->n_guests += 1;
    d.ctl->granted_sum += n;
    return true;
}

// kvc.py:229-249
__device__ __forceinline__ bool pool_draw_reserved(const Dev& d, int i, int32_t nb) {
    Ctl& c = *d.ctl;
    if (nb < 1 || nb > c.rsv_cur) return false;
    if (!d.holds[i]) new_record(d, i, 0, -1, 0);
    if (d.host[i] >= 0) return false;
    int64_t tokens = (int64_t)nb * d.bs;
    c.rsv_cur -= nb;
    d.rsv[i] += nb;
    int64_t g = d.granted[i];
    int64_t old = g ? fp_tokens(g, d.bs) : 0;
    d.granted[i] = (int32_t)(g + tokens);
    const int64_t dfp = fp_tokens(g + tokens, d.bs) - old;
    c.fp_sum += dfp;
    c.granted_sum += tokens;
    pop_pages(d, i, dfp / d.bs);
    return true;
}

// kvc.py:251-281
__device__ __forceinline__ bool pool_grow(const Dev& d, int i, int64_t n) {
    if (n < 1 || !d.holds[i]) return false;
    Ctl& c = *d.ctl;
    int64_t g = d.granted[i];
    int32_t h = d.host[i];
    if (h < 0) {
        int64_t delta = fp_tokens(g + n, d.bs) - fp_tokens(g, d.bs);
        if (delta > free_tokens(d)) return false;
        d.granted[i] = (int32_t)(g + n);
        c.fp_sum += delta;
        c.granted_sum += n;
        pop_pages(d, i, delta / d.bs);
        return true;
    }
    // guests grow downward to the host's used region plus the buffer, or to
    // the top of the guest below them
    int64_t floor_ = (int64_t)d.used[h] + d.buffer_b;
    for (int32_t g = d.guest[h]; g >= 0; g = d.gnext[g])
        if (g != i && d.off[g] < d.off[i]) {
            const int64_t top = (int64_t)d.off[g] + d.granted[g];
            floor_ = top > floor_ ? top : floor_;
        }
    if (n > (int64_t)d.off[i] - floor_) return false;
    d.off[i] -= (int32_t)n;
    d.granted[i] = (int32_t)(g + n);
    c.granted_sum += n;
    return true;
}

// kvc.py:283-297
__device__ __forceinline__ bool pool_promote(const Dev& d, int i) {
    int64_t fp = fp_tokens(d.granted[i], d.bs);
    if (fp > free_tokens(d)) return false;
    int32_t h = d.host[i];
    int64_t vsnap = 0;
    int32_t vend = 0;
    const int32_t gused = d.used[i];
    if (d.dp.on && gused > 0) vsnap = snap_view(d, d.dp, h, d.off[i] + d.granted[i], gused, &vend);
    guest_unlink(d, h, i);
    d.host[i] = -1;
    d.off[i] = 0;
    d.ctl->fp_sum += fp;
    pop_pages(d, i, fp / d.bs);
    if (d.dp.on && gused > 0) log_move(d, d.dp, i, gused, vsnap, vend);  // N2: the guest's KV follows it
    return true;
}

// kvc.py:299-324
__device__ __forceinline__ void pool_release(const Dev& d, int i) {
    Ctl& c = *d.ctl;
    int32_t h = d.host[i];
    if (h >= 0) {
        if (d.holds[h]) guest_unlink(d, h, i);
        c.granted_sum -= d.granted[i];
        d.host[i] = -1;
        drop_record(d, i);
        return;
    }
    // every guest is re-homed (kvc.py:311-317), in embed order, into pages
    // of its own; their views are snapshotted before the host's pages go back
    constexpr int MAXG = 32;
    int64_t vsnap[MAXG];
    int32_t vend[MAXG], gused[MAXG];
    int32_t ng = 0;
    for (int32_t g = d.guest[i]; g >= 0; g = d.gnext[g], ng++) {
        if (ng == MAXG) { c.error = 11; c.err_info[0] = i; return; }
        gused[ng] = d.used[g];
        vsnap[ng] = 0;
        vend[ng] = 0;
        if (d.dp.on && gused[ng] > 0) vsnap[ng] = snap_view(d, d.dp, i, d.off[g] + d.granted[g], gused[ng], &vend[ng]);
    }
    push_table(d, i);
    int32_t k = 0;
    for (int32_t g = d.guest[i]; g >= 0; k++) {
        const int32_t nx = d.gnext[g];
        d.host[g] = -1;
        d.off[g] = 0;
        d.gnext[g] = -1;
        c.n_guests -= 1;
        const int64_t gfp = fp_tokens(d.granted[g], d.bs);
        c.fp_sum += gfp;
        pop_pages(d, g, gfp / d.bs);
        if (d.dp.on && gused[k] > 0) log_move(d, d.dp, g, gused[k], vsnap[k], vend[k]);
        g = nx;
    }
    d.guest[i] = -1;
    c.fp_sum -= fp_tokens(d.granted[i], d.bs);
    c.granted_sum -= d.granted[i];
    int64_t room = (int64_t)d.rsv_target - c.rsv_cur;
    int64_t refill = d.rsv[i] < room ? d.rsv[i] : room;
    c.rsv_cur += (int32_t)refill;
    drop_record(d, i);
}

// kvc.py:326-332; the engine never expects this to raise
__device__ __forceinline__ void set_used(const Dev& d, int i, int32_t u) {
    if (u < 0 || u > d.granted[i]) {
        d.ctl->error = 2;
        d.ctl->err_info[0] = i;
        d.ctl->err_info[1] = u;
    }
    d.ctl->used_sum += (int64_t)u - d.used[i];
    d.used[i] = u;
}

// -- events ---------------------------------------------------------------

__device__ __forceinline__ void emit_event(const Dev& d, int32_t kind, int32_t idx, int64_t t, int64_t a = 0,
                                           int64_t b = 0, int64_t c = 0) {
    if (!d.record_events) return;
    int64_t p = d.ctl->ev_count++;
    co_event e;
    e.kind = kind; e.idx = idx; e.t = t; e.a = a; e.b = b; e.c = c;
    d.events[p] = e;
}

// -- lifecycle ------------------------------------------------------------

__device__ __forceinline__ bool live_state(int8_t s) { return s >= ST_WAITING && s <= ST_PREEMPTED; }

// engine.py:360-384
__device__ __forceinline__ void do_preempt(const Dev& d, int i, int32_t strat, int64_t now, int32_t cause) {
    if (d.state[i] != ST_RUNNING) return;
    d.state[i] = ST_PREEMPTED;
    d.key0[i] = wait_key(d, i);  // its waiting-queue key (D = last token + TBT SLO)
    d.pcount[i] += 1;
    d.last_strat[i] = (int8_t)strat;
    int32_t u = d.used[i];
    int64_t restored = u > 1 ? u : 1;
    d.pstart[i] = now;
    d.prefill[i] = u;
    if (u > d.kv_need[i]) d.kv_need[i] = u;
    d.swap_done[i] = strat == CO_SWAP ? now + lut(d.lut_swap_half, restored, d.s_max) : 0;
    if (strat == CO_SWAP) log_swap_out(d, d.dp, i);  // N2: KV leaves before its pages do
    if (d.holds[i]) pool_release(d, i);
    d.used[i] = 0;
    d.alloc_kvc[i] = 0;
    d.claim_w[i] = -1;     // _claims.pop(rid) as provider
    d.epoch[i] += 1;       // entries naming rid as waiter are dead
    emit_event(d, CO_EV_PREEMPT, i, now, restored, strat, cause);
}

// engine.py:386-402
__device__ __forceinline__ void do_readmit(const Dev& d, int i) {
    const int64_t now = d.ctl->now;
    d.state[i] = ST_RUNNING;
    int64_t restored = d.prefill[i] > 1 ? d.prefill[i] : 1;
    int64_t ra;
    if (d.last_strat[i] == CO_SWAP) {
        int64_t base = now > d.swap_done[i] ? now : d.swap_done[i];
        ra = base + lut(d.lut_swap_half, restored, d.s_max);
    } else {
        ra = now + lut(d.lut_rec, restored, d.s_max);
    }
    d.ready_at[i] = ra;
    d.ptime[i] += ra - d.pstart[i];
    int32_t u = d.prefill[i] < d.granted[i] ? d.prefill[i] : d.granted[i];
    set_used(d, i, u);
    log_readmit(d, d.dp, i, d.last_strat[i] == CO_SWAP);  // N2: swap-in or recompute fill
    emit_event(d, CO_EV_READMIT, i, now, ra);
}

__device__ __forceinline__ bool claim_valid(const Dev& d, int p) {
    int32_t w = d.claim_w[p];
    return w >= 0 && d.claim_ep[p] == d.epoch[w];
}

// engine.py:419-433
__device__ __forceinline__ void fulfill_claim(const Dev& d, int w) {
    if (d.state[w] != ST_RUNNING || !d.holds[w]) return;
    int64_t target = target_of(d, w);
    int64_t residual = target - d.granted[w];
    if (residual > 0 && pool_grow(d, w, residual)) d.alloc_kvc[w] = d.granted[w];
}

// engine.py:404-417
__device__ __forceinline__ void do_complete(const Dev& d, int i, int64_t now) {
    d.state[i] = ST_COMPLETED;
    d.completion[i] = now;
    if (d.holds[i]) pool_release(d, i);
    d.ctl->n_live -= 1;
    emit_event(d, CO_EV_COMPLETE, i, now);
    d.epoch[i] += 1;  // providers promised to i are dropped
    if (claim_valid(d, i)) {
        int32_t w = d.claim_w[i];
        d.claim_w[i] = -1;
        if (live_state(d.state[w])) fulfill_claim(d, w);
    }
    d.claim_w[i] = -1;
}

}  // namespace co
