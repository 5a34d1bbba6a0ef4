// k_apply: plan application and the rest of one engine step (rows a11/a12):
// engine.py:437-536 (_apply_plan), 619-625 (idle jump to the next event),
// 627-633 (iteration charge + event), 553-571 (_emit), 404-433
// (_complete/_fulfill_claim), 573-591 (_resolve_collisions), 636-640.
// Pool mutations happen in plan order on thread 0; token emission is a
// block-parallel pass over the (distinct) surviving members, and
// completions, whose claim hand-offs are order dependent, are then replayed
// in member order.
#pragma once
#include "block_ops.cuh"
#include "pool_ops.cuh"

namespace co {

// kvc.py:336-375 check_invariants over every record (validate_every)
__device__ __forceinline__ void check_pool(const Dev& d, BlkShared& sb) {
    Ctl& c = *d.ctl;
    int64_t fp = 0, bad = 0;
    for (int32_t i = threadIdx.x; i < d.n; i += (int)blockDim.x) {
        if (!d.holds[i]) continue;
        if (d.host[i] < 0) fp += fp_tokens(d.granted[i], d.bs);
        if (d.used[i] > d.granted[i]) bad |= 1;
        int32_t h = d.host[i];
        if (h >= 0) {
            if (d.guest[i] >= 0) bad |= 2;
            bool listed = false;
            if (d.holds[h])
                for (int32_t g = d.guest[h]; g >= 0 && !listed; g = d.gnext[g]) listed = g == i;
            if (!listed) bad |= 4;
            else if (d.off[i] < 0 || (int64_t)d.off[i] + d.granted[i] > d.granted[h]) bad |= 8;
        } else if (d.tab_len[i] * (int64_t)d.bs != fp_tokens(d.granted[i], d.bs)) {
            bad |= 32;  // N1: the table covers exactly the footprint
        }
        // guest spans above the host's used region, pairwise disjoint (kvc.py:365-375)
        for (int32_t g = d.guest[i]; g >= 0; g = d.gnext[g]) {
            if (d.off[g] < d.used[i]) bad |= 16;
            for (int32_t q = d.gnext[g]; q >= 0; q = d.gnext[q])
                if (!((int64_t)d.off[g] + d.granted[g] <= d.off[q] || (int64_t)d.off[q] + d.granted[q] <= d.off[g]))
                    bad |= 16;
        }
    }
    fp = blk_sum(fp, sb);
    bad = blk_sum(bad ? 1 : 0, sb);
    if (threadIdx.x == 0) {
        if (fp != c.fp_sum) bad += 1;
        if (free_tokens(d) < 0) bad += 1;
        if (c.rsv_cur < 0 || c.rsv_cur > d.rsv_target) bad += 1;
        if ((int64_t)c.free_top * d.bs != (int64_t)d.n_pages * d.bs - c.fp_sum) bad += 1;
        if (bad) { c.error = 4; c.done = 1; }
    }
}

struct ApplySh {
    BlkShared b;
    int64_t batch, end;
    int32_t n_surv, n_acted, idle;
};

// plan application + step remainder (run by k_serial after plan_body; S
// aliases the planner's shared memory, which is dead by then)
__device__ __forceinline__ void apply_body(const Dev& d, ApplySh& S) {
    Ctl& c = *d.ctl;
    const int tid = threadIdx.x;
    const int64_t now = c.now;
    const int32_t sid = c.sid;
    const PlanHdr& P = *d.plan;
    const int32_t n_run = c.cnt_run;
    const int32_t* RUN = d.l_run;  // running set in arrival order (built by k_plan)

    prof_mark(d, 32);
    if (tid == 0) {
        for (int32_t k = 0; k < P.n_pre; k++) do_preempt(d, d.pre_idx[k], d.pre_strat[k], now, CO_CAUSE_PLAN);
        int32_t n_acted = 0;
        for (int32_t a = 0; a < P.n_act; a++) {
            const int32_t i = d.act_idx[a];
            if (d.st_failed[i] == sid || !live_state(d.state[i])) continue;
            const int32_t kind = d.act_kind[a];
            const int64_t tok = d.act_tok[a];
            bool ok;
            if (kind == A_ALLOCATE) ok = pool_allocate(d, i, tok);
            else if (kind == A_GROW) ok = pool_grow(d, i, tok);
            else if (kind == A_RESERVE) ok = pool_draw_reserved(d, i, d.act_nb[a]);
            else ok = pool_embed(d, i, tok, d.act_host[a], d.act_start[a]);
            if (ok) {
                if (d.st_acted[i] != sid) { d.st_acted[i] = sid; d.l_acted[n_acted++] = i; }
                d.alloc_kvc[i] = d.granted[i];
                continue;
            }
            // a guest out of room is promoted when the pool covers it,
            // squeezed out otherwise (engine.py:474-494)
            if (kind == A_GROW && d.holds[i] && d.host[i] >= 0 && d.state[i] == ST_RUNNING) {
                if (pool_promote(d, i)) {
                    if (pool_grow(d, i, tok)) {
                        if (d.st_acted[i] != sid) { d.st_acted[i] = sid; d.l_acted[n_acted++] = i; }
                        d.alloc_kvc[i] = d.granted[i];
                        continue;
                    }
                    d.st_failed[i] = sid;
                    continue;
                }
                do_preempt(d, i, strategy_of(d, i), now, CO_CAUSE_SQUEEZE);
            }
            d.st_failed[i] = sid;
        }
        for (int32_t k = 0; k < n_acted; k++) {
            int32_t i = d.l_acted[k];
            if (d.state[i] == ST_PREEMPTED) do_readmit(d, i);
        }
        S.n_acted = n_acted;
    }
    __syncthreads();

    prof_mark(d, 33);
    // ---- member filter (engine.py:500-531), block-parallel ------------------
    // A position is examined iff its request is not failed and it is the
    // request's first position (the reference's `seen`); each examined member's
    // outcome depends only on its own post-action state, and admit events and
    // survivors keep member order through ordered compactions.
    const int32_t nm = P.n_mem;
    const uint64_t stamp = (uint64_t)(uint32_t)sid << 24;
    for (int32_t m = tid; m < nm; m += (int)blockDim.x) atomicMax((unsigned long long*)&d.seen64[d.mem_idx[m]],
                                                      (unsigned long long)(stamp | (0xFFFFFFu - (uint32_t)m)));
    __syncthreads();
    int32_t my_i = -1, my_tok = 0, my_f = 0;  // this thread's member when nm <= blockDim.x
    for (int32_t m = tid; m < nm; m += (int)blockDim.x) {
        const int32_t i = d.mem_idx[m];
        const int32_t tok = d.mem_tok[m];
        // every field the decision reads, loaded up front: one round trip
        // instead of one per branch (the guest's offset is the only dependent load)
        const int32_t failed = d.st_failed[i];
        const uint64_t seen = d.seen64[i];
        const int8_t st = d.state[i];
        const uint8_t holds = d.holds[i];
        const int32_t granted = d.granted[i], prefill = d.prefill[i], kvn = d.kv_need[i], used = d.used[i];
        const int32_t gu = d.guest[i];
        const int64_t ready = d.ready_at[i], fstart = d.first_start[i];
        int32_t f = 0;  // bit0 survive, bit1 admit event
        if (failed != sid && seen == (stamp | (0xFFFFFFu - (uint32_t)m))) {
            bool go = live_state(st);
            if (go && st == ST_WAITING) {
                if (!holds || granted < prefill + tok) {
                    go = false;
                } else {
                    f |= 4;  // becomes RUNNING
                    if (fstart < 0) f |= 2;
                }
            } else if (go && st != ST_RUNNING) {
                go = false;
            }
            if (go && ready > now) go = false;
            if (go) {
                if (prefill >= kvn) {
                    int32_t eff = holds ? granted : 0;  // eff_of (engine.py:275-282)
                    if (holds && gu >= 0) { const int32_t o = d.off[gu]; eff = o < granted ? o : granted; }
                    if (eff < used + 1) go = false;
                } else if (granted < prefill + tok) {
                    go = false;
                }
            }
            if (go) f |= 1;
        }
        d.l_mflag[m] = f;
        if (m == tid) { my_i = i; my_tok = tok; my_f = f; }
    }
    int32_t n_admit = 0, ns0 = 0;
    int64_t bsum = 0;
    if (nm <= (int)blockDim.x) {
        // one member per thread, decisions in registers: the state changes,
        // then ONE scan placing admit events (high half) and survivors (low
        // half) in member order
        if (my_f & 4) {
            d.state[my_i] = ST_RUNNING;
            if (my_f & 2) d.first_start[my_i] = now;
        }
        const int32_t packed = ((my_f & 2) ? (1 << 16) : 0) | (my_f & 1);
        int32_t tot;
        const int32_t ex = blk_excl_scan(packed, &tot, S.b);
        if (d.record_events) {
            if (my_f & 2) {
                co_event e;
                e.kind = CO_EV_ADMIT; e.idx = my_i; e.t = now; e.a = e.b = e.c = 0;
                d.events[c.ev_count + (ex >> 16)] = e;
            }
            n_admit = tot >> 16;
        }
        if (my_f & 1) { d.l_surv_idx[ex & 0xffff] = my_i; d.l_surv_tok[ex & 0xffff] = my_tok; }
        ns0 = tot & 0xffff;
        bsum = blk_sum((my_f & 1) ? my_tok : 0, S.b);  // (its barriers publish the survivor lists)
    } else {
    __syncthreads();
    for (int32_t m = tid; m < nm; m += (int)blockDim.x) {
        const int32_t f = d.l_mflag[m];
        if (f & 4) {
            const int32_t i = d.mem_idx[m];
            d.state[i] = ST_RUNNING;
            if (f & 2) d.first_start[i] = now;
        }
    }
    if (d.record_events) {
        const int64_t ev_base = c.ev_count;
        int32_t base = 0;
        for (int32_t c0 = 0; c0 < nm; c0 += (int)blockDim.x) {
            const int32_t m = c0 + tid;
            const int32_t fl = (m < nm && (d.l_mflag[m] & 2)) ? 1 : 0;
            int32_t tot;
            const int32_t p = blk_excl_scan(fl, &tot, S.b);
            if (fl) {
                co_event e;
                e.kind = CO_EV_ADMIT; e.idx = d.mem_idx[m]; e.t = now; e.a = e.b = e.c = 0;
                d.events[ev_base + base + p] = e;
            }
            base += tot;
        }
        n_admit = base;
    }
    // survivors in member order: positions first, then (idx, tokens)
    ns0 = blk_compact(nullptr, nm, d.l_surv_tok, [&](int32_t m) { return (d.l_mflag[m] & 1) != 0; }, S.b);
    for (int32_t k = tid; k < ns0; k += (int)blockDim.x) bsum += d.mem_tok[d.l_surv_tok[k]];
    bsum = blk_sum(bsum, S.b);
    for (int32_t k = tid; k < ns0; k += (int)blockDim.x) {
        const int32_t m = d.l_surv_tok[k];
        d.l_surv_idx[k] = d.mem_idx[m];
    }
    __syncthreads();
    for (int32_t k = tid; k < ns0; k += (int)blockDim.x) d.l_surv_tok[k] = d.mem_tok[d.l_surv_tok[k]];  // position -> tokens
    }
    __syncthreads();
    if (tid == 0) {
        const int32_t ns = ns0;
        const int64_t batch = bsum;
        c.ev_count += n_admit;
        // claims (engine.py:533-535): setdefault(provider, waiter)
        for (int32_t k = 0; k < P.n_cl; k++) {
            int32_t w = d.cl_w[k], p = d.cl_p[k];
            if (live_state(d.state[w]) && live_state(d.state[p]) && !claim_valid(d, p)) {
                d.claim_w[p] = w;
                d.claim_ep[p] = d.epoch[w];
            }
        }
        S.n_surv = ns;
        S.batch = batch;
        S.idle = (ns == 0 && P.n_act == 0 && P.n_pre == 0) ? 1 : 0;
    }
    __syncthreads();

    if (S.idle) {
        // engine.py:619-625 / 593-602: jump to the next arrival or resume
        // barrier; nothing changed state in this step, so the classify-time
        // running set is current
        uint64_t best = ~0ull;
        for (int32_t k = tid; k < n_run; k += (int)blockDim.x) {
            int32_t i = RUN[k];
            if (d.state[i] == ST_RUNNING && d.ready_at[i] > now) {
                uint64_t v = (uint64_t)d.ready_at[i];
                best = v < best ? v : best;
            }
        }
        best = blk_min(best, S.b);
        if (tid == 0) {
            if (c.next_pending < d.n) {
                uint64_t a = (uint64_t)d.arr[c.next_pending];
                best = a < best ? a : best;
            }
            if (best == ~0ull) {
                c.stalled = 1; c.done = 1; c.last_result = 0;
            } else {
                c.now = (int64_t)best;
                c.last_result = 1;
            }
            if (d.result) d.result[0] = 0;
        }
        return;
    }

    prof_mark(d, 34);
    // ---- iteration charge and event (engine.py:627-633) -------------------
    const int32_t ns = S.n_surv;
    int64_t mem0 = 0;
    if (tid == 0) {
        int64_t il = to_us_d(iter_ms(d, S.batch));
        S.end = now + il;
        c.t_i = il;
        if (d.record_events) {
            mem0 = c.mem_count;
            emit_event(d, CO_EV_ITER, ns, now, S.end, S.batch, mem0);
            c.mem_count += ns;
        }
        d.plan->batch_tokens = S.batch;  // keep the applied batch for readers
        S.n_acted = (int32_t)mem0;       // stash member-stream offset
    }
    __syncthreads();
    const int64_t end = S.end;
    if (d.record_events) {
        const int64_t off = S.n_acted;
        for (int32_t k = tid; k < ns; k += (int)blockDim.x) {
            d.members[2 * (off + k)] = d.l_surv_idx[k];
            d.members[2 * (off + k) + 1] = d.l_surv_tok[k];
        }
    }
    if (d.result) {  // the iteration's result straight into mapped host memory
        const int32_t nr = ns < d.result_cap ? ns : (int32_t)d.result_cap;
        for (int32_t k = tid; k < nr; k += (int)blockDim.x) {
            d.result[4 + 2 * k] = d.l_surv_idx[k];
            d.result[4 + 2 * k + 1] = d.l_surv_tok[k];
        }
        if (tid == 0) {
            d.result[0] = nr;
            *reinterpret_cast<int64_t*>(d.result + 2) = S.end;
        }
    }

    prof_mark(d, 35);
    // ---- emission (engine.py:553-571), members are distinct ---------------
    int64_t dused = 0, dgen = 0;
    for (int32_t k = tid; k < ns; k += (int)blockDim.x) {
        const int32_t i = d.l_surv_idx[k];
        const int32_t tok = d.l_surv_tok[k];
        // the member's fields up front (members are distinct: no other thread writes them)
        const int32_t prefill = d.prefill[i], kvn = d.kv_need[i], used = d.used[i], gen = d.gen[i];
        const int32_t granted = d.granted[i];
        const int64_t ftok = d.first_tok[i], ltok = d.last_tok[i], mtbt = d.max_tbt[i], toff = d.tok_off[i];
        bool token = false;
        int32_t nu;
        if (prefill < kvn) {
            d.l_fill_t0[k] = prefill;  // N2: the chunk's KV is written this iteration
            d.l_fill_n[k] = tok;
            nu = prefill + tok;
            d.prefill[i] = nu;
            token = nu >= kvn && gen == 0;
        } else {
            d.l_fill_t0[k] = used;     // decode writes the KV of position used
            d.l_fill_n[k] = -1;        // (negative: decode member)
            nu = used + 1;
            token = true;
        }
        if (nu < 0 || nu > granted) { c.error = 2; c.err_info[0] = i; c.err_info[1] = nu; }
        dused += (int64_t)nu - used;
        d.used[i] = nu;
        if (token) {
            const int32_t g = gen + 1;
            d.gen[i] = g;
            dgen += 1;
            if (ftok < 0) {
                d.first_tok[i] = end;
            } else {
                const int64_t gap = end - ltok;
                if (gap > mtbt) d.max_tbt[i] = gap;
            }
            d.last_tok[i] = end;
            d.tok_times[toff + g - 1] = end;
        }
    }
    dused = blk_sum(dused, S.b);
    dgen = blk_sum(dgen, S.b);
    const int32_t n_done = blk_compact(d.l_surv_idx, ns, d.l_done, [&](int32_t i) { return d.gen[i] >= d.tout[i]; }, S.b);
    if (tid == 0) {
        c.used_sum += dused;
        c.gen_total += dgen;
        if (d.dp.on) {
            // guests' KV goes into their host's pages now, before a completing
            // host re-homes them or a colliding host evicts them
            for (int32_t k = 0; k < ns; k++) {
                const int32_t i = d.l_surv_idx[k];
                if (d.host[i] >= 0) {
                    int32_t n = d.l_fill_n[k];
                    log_fill(d, d.dp, i, d.l_fill_t0[k], n < 0 ? 1 : n);
                    d.l_fill_n[k] = n < 0 ? -2 : 0;  // logged
                }
            }
        }
        for (int32_t k = 0; k < n_done; k++) do_complete(d, d.l_done[k], end);
    }
    __syncthreads();

    prof_mark(d, 36);
    // ---- collisions (engine.py:573-591), hosts in record-creation order ----
    int32_t n_coll = 0;
    if (c.n_guests > 0) {  // (no guest record: nothing can collide)
        n_coll = blk_compact(RUN, n_run, d.l_coll, [&](int32_t h) {
            if (d.state[h] != ST_RUNNING || !d.holds[h] || d.host[h] >= 0) return false;
            for (int32_t g = d.guest[h]; g >= 0; g = d.gnext[g])
                if (d.used[h] >= d.off[g]) return true;
            return false;
        }, S.b);
        blk_sort(d.l_coll, n_coll, [&](int32_t h, uint64_t& k0, uint64_t& k1, uint64_t& k2) {
            k0 = (uint64_t)d.rec_seq[h]; k1 = 0; k2 = 0;
        }, d, S.b);
    }
    if (tid == 0) {
        for (int32_t k = 0; k < n_coll; k++) {
            int32_t h = d.l_coll[k];
            if (d.state[h] != ST_RUNNING || !d.holds[h]) continue;
            // the host's guests by offset ascending (engine.py:585), a copy:
            // promotions and preemptions unlink them as the loop goes
            constexpr int MAXG = 32;
            int32_t gl[MAXG];
            int32_t ng = 0;
            for (int32_t g = d.guest[h]; g >= 0 && ng < MAXG; g = d.gnext[g]) {
                int32_t p = ng++;
                while (p > 0 && d.off[gl[p - 1]] > d.off[g]) { gl[p] = gl[p - 1]; p--; }
                gl[p] = g;
            }
            for (int32_t q = 0; q < ng; q++) {
                const int32_t g = gl[q];
                if (d.used[h] < d.off[g]) continue;
                if (pool_promote(d, g)) continue;
                if (d.state[g] == ST_RUNNING) do_preempt(d, g, strategy_of(d, g), end, CO_CAUSE_COLLISION);
            }
        }
        if (d.dp.on) {
            // standalone members' KV at their final pages, then this
            // iteration's decode set (members that decoded and still hold)
            DataCtl& dc = *d.dctl;
            int32_t nd = 0, items = 0;
            for (int32_t k = 0; k < ns; k++) {
                const int32_t i = d.l_surv_idx[k];
                const int32_t n = d.l_fill_n[k];
                if (!d.holds[i] || d.state[i] != ST_RUNNING) continue;
                if (n > 0 || n == -1) log_fill(d, d.dp, i, d.l_fill_t0[k], n < 0 ? 1 : n);
                if ((n == -1 || n == -2) && d.dp.decode_on && dc.decode_enabled) {
                    if (nd == d.dp.dec_cap) { c.error = 9; c.err_info[0] = nd; break; }
                    const int32_t ctx = d.used[i];
                    const int32_t need = ((ctx + d.dp.split - 1) / d.dp.split) * d.dp.L * d.dp.Hkv;
                    if (items + need > d.dp.dec_item_cap) { c.error = 8; break; }
                    d.dp.dec_idx[nd] = i;
                    d.dp.dec_ctx[nd] = ctx;
                    d.dp.dec_item_off[nd] = items;
                    items += need;
                    nd++;
                }
            }
            d.dp.dec_item_off[nd] = items;
            dc.n_dec = nd;
            dc.dec_items = items;
            if (nd) { dc.dec_steps += 1; dc.dec_members += nd; }
            for (int32_t k = 0; k < nd; k++) dc.dec_tokens += d.dp.dec_ctx[k];
        }
        // engine.py:636-640
        int64_t sp = c.sample_count++;
        d.samples[2 * sp] = c.fp_sum;
        d.samples[2 * sp + 1] = c.used_sum;
        c.iters += 1;
        c.check_due = (d.validate_every && c.iters % d.validate_every == 0) ? 1 : 0;
        c.now = end;
        c.last_result = 1;
    }
    __syncthreads();
    prof_mark(d, 37);
    if (c.check_due) check_pool(d, S.b);
}

__global__ void __launch_bounds__(NT, 1) k_check(Dev d) {
    __shared__ BlkShared sb;
    check_pool(d, sb);
}

}  // namespace co
