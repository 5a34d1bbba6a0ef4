// Device-resident CacheOPT engine state: a structure-of-arrays request table
// in HBM indexed by arrival rank (engine.py:241 orders requests by
// (arrival_us, id); that rank is also the reference's _live iteration order,
// engine.py:242/352), the KV pool records of kvc.py:44-52 as parallel arrays,
// and a small control block of engine scalars (engine.py:243-270).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/cacheopt.h"
#include "dp_types.cuh"

namespace co {

// Programmatic dependent launch inside the step graph: a step kernel waits
// for its predecessor's completion (and memory) here, then lets its own
// successor launch, so each launch's latency overlaps the previous kernel's
// tail.  A no-op when the kernel was launched without the PDL attribute.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

constexpr int NT = 256;   // threads of the single-CTA planner / apply kernels (max; 256 measured best)
constexpr int TCHUNK = 64;  // pages per block-table chunk
constexpr int CAND_CAP = 1024;    // candidate head of the keyed N'_w collected by k_classify
constexpr int CAND_TARGET = 128;  // head size the planner aims the next step's threshold at
constexpr int XNB = 2048;         // histogram bins of the planner's queue extension
constexpr int XCHUNK = 2048;      // at most this many items per extension
constexpr int ST_PENDING = CO_PENDING, ST_WAITING = CO_WAITING, ST_RUNNING = CO_RUNNING,
              ST_PREEMPTED = CO_PREEMPTED, ST_COMPLETED = CO_COMPLETED;

enum ActKind : int32_t { A_ALLOCATE = 0, A_GROW = 1, A_RESERVE = 2, A_EMBED = 3 };

// Engine scalars shared by every kernel of a step (device memory).
struct Ctl {
    int64_t now, horizon, first_arrival, t_i;
    int64_t fp_sum, granted_sum, used_sum;          // kvc.py:83-84, used_tokens kvc.py:109
    int64_t gen_total, iters, steps, seq, decisions;
    int64_t ev_count, mem_count, sample_count;      // undrained append-buffer fill
    int64_t mark[5];                                 // engine.py:647-650 progress mark
    int64_t streak;
    int32_t has_mark, guard;                         // guard: run() semantics active
    int32_t rsv_cur, n_live, next_pending, adm_lo, adm_hi;
    int32_t done, stalled, error, paused;
    int32_t active;                                   // this step proceeds past begin
    int32_t last_result;                              // step() return value
    int32_t cnt_nw, cnt_nwp, cnt_run;                 // classify counts (N_w, non-blown N'_w, running)
    int32_t cnt_blown;                                // blown N'_w (arrival order)
    int32_t cnt_cand;                                 // non-blown N'_w with key < thr (k_classify)
    uint64_t thr;                                     // candidate key bound, set by the planner per step
    uint64_t kmin, kmax;                              // range of the non-blown N'_w keys
    int32_t sid;                                      // stamp id of the current step
    int32_t check_due;
    int32_t free_top;                                 // N1: pages on the free stack
    int32_t chunk_top;                                // N1: free table chunks
    int32_t err_info[4];
    uint64_t mir_seq;                                 // step mirrors written (mapped completion flag)
    int32_t n_guests;                                 // live guest records (apply skips collisions at 0)
};

// The plan of one step (scheduler.py:295-323 BatchPlan) as device lists.
struct PlanHdr {
    int32_t n_mem, n_act, n_pre, n_cl, n_def, overflow, sated, k_sel;
    int64_t batch_tokens;
};

struct Dev {
    // configuration (co_config + derived)
    int32_t n, bs, B, buffer_b, token_budget, prealloc_m, runway_iters, fcfs;
    int32_t record_events, validate_every, pad, idbits, n_edges, token_step, rsv_target;
    int32_t key_bits;            // composite sort key width: class(2) | blown(1) | time | idrank
    int32_t policy, vbt, s3b, rlp_pad;  // planner (CO_POLICY_*) and the baselines' parameters
    int32_t inv;                 // invert_amortization (scheduler.py:43): exact serial path, planner.cuh
    uint64_t* big;               // its multi-precision scratch: 5 numbers of INV_LIMBS limbs
    int64_t eps, capacity, s_star, s_max, ev_cap, mem_cap, sample_cap;
    int64_t edges[CO_MAX_SLO_EDGES];
    double base_ms, per_token_ms;
    // trace (sorted order)
    const int64_t *rid, *arr, *slo_ttft, *slo_tbt;
    const int32_t *prompt, *tout, *idrank, *err;
    const uint8_t* flip;
    // LUTs
    const int64_t *lut_swap_half, *lut_rec, *lut_surv_swap, *lut_surv_rec;
    // runtime (core.py:72-94)
    int8_t *state, *last_strat;
    int32_t *gen, *used, *kv_need, *prefill, *pcount, *pred, *est, *alloc_kvc;
    int64_t *first_tok, *last_tok, *max_tbt, *ready_at, *pstart, *swap_done, *first_start,
        *completion, *ptime;
    const int64_t* tok_off;
    int64_t* tok_times;
    // pool records (kvc.py:44-52).  A host's guests (kvc.py:52 `guests`, in
    // embed order) are a singly linked list: guest[h] = first, gnext[g] =
    // next.  Without stacking the list has at most one entry.
    uint8_t* holds;
    int32_t *granted, *host, *off, *rsv, *guest, *gnext;
    int32_t stacking;  // BlockPool.allow_stacking (kvc.py:64, 187-192, 212)
    int64_t* rec_seq;
    // N1 physical block tables (standalone records only; a guest is a view
    // into its host's pages).  Request i's k-th page is
    //   chunk_pool[dir[i * dir_w + k / TCHUNK] * TCHUNK + k % TCHUNK]
    // with 64-page chunks drawn from a shared chunk stack, because a grant
    // can be as large as the whole supply (scheduler.py:237 shares are not
    // capped by the demand).
    int32_t* chunk_pool;
    int32_t* chunk_stack;
    int32_t* dir;
    int32_t* tab_len;
    int32_t* free_stack;
    int32_t n_pages, dir_w;
    // claims provider -> waiter (engine.py:246) with lazy invalidation epochs
    int32_t *claim_w, *claim_ep, *epoch;
    // per-step membership stamps (compared with Ctl::sid, never cleared)
    int32_t *st_nr, *st_crit, *st_removed, *st_embedded, *st_resumed, *st_stalled, *st_parts,
        *st_claimed, *st_failed, *st_acted, *st_deferred;
    uint64_t* seen64;            // member-filter first occurrence: (sid << 24) | (2^24-1-pos)
    // classify + bucketed ordering (no full sort): classify block b owns the
    // index range [b*chunk, (b+1)*chunk) and compacts its running / blown
    // requests in index order; non-blown N'_w requests get the unique key
    // (D << idbits | idrank) and are bucketed by a range-adaptive histogram
    int32_t nblk, chunk;
    int32_t *run_tmp, *blown_tmp, *blk_cnt;
    int32_t* crit_idx;
    uint64_t* key0;    // waiting-queue key, set when a request starts waiting (wait_key)
    int32_t* cand;     // this step's candidate head of N'_w (unordered, <= CAND_CAP)
    int32_t *l_run, *l_blown, *l_nw, *l_nwp;
    // plan buffers
    PlanHdr* plan;
    int32_t *mem_idx, *mem_tok, *act_kind, *act_idx, *act_tok, *act_nb, *act_host, *act_start;
    int32_t *pre_idx, *pre_strat, *cl_w, *cl_p, *def_idx;
    // planner / apply scratch (n-sized unless noted)
    int32_t *l_nr, *l_nrp, *l_pend, *l_tri, *l_tri_taken, *l_vict, *l_defer, *l_pro, *l_ful,
        *l_part, *l_part_need, *l_part_grant, *l_mready, *l_gm_idx, *l_gm_tok, *l_acted,
        *l_surv_idx, *l_surv_tok, *l_done, *l_coll, *l_grp, *l_fill_t0, *l_fill_n, *l_mflag;
    int64_t* l_tri_key;
    uint64_t *am_rhi, *am_rlo;   // amortize remainders (128-bit), by participant position
    int32_t* rank_to_idx;        // inverse of idrank
    uint64_t *sk0, *sk1, *sk2;   // generic sort keys
    int32_t* sk_item;
    // N2/N3 data plane
    DataCfg dp;
    DataCtl* dctl;
    // outputs
    co_event* events;
    int32_t* members;   // (idx, tok) pairs
    int64_t* samples;   // (footprint, used) pairs
    Ctl* ctl;
    struct PV* views;  // per-request planner snapshot (k_classify -> k_plan)
    int64_t* prof;   // optional phase timestamps (ns, %globaltimer), 64 slots per kernel
    // per-step result in mapped pinned host memory (co_step_result):
    // [0] member count (-1 while the step is idle/ended), [1] unused,
    // [2..3] iteration end (int64), then (idx, tokens) pairs
    int32_t* result;
    int64_t result_cap;
};

// ---------------------------------------------------------------------------
// per-request view quantities (engine.py:284-317, scheduler.py:99-118);
// valid while the pool is not mutated (planning phase) or at the instant read

__device__ __forceinline__ int32_t page_of(const Dev& d, int i, int32_t k) {
    return d.chunk_pool[(int64_t)d.dir[(int64_t)i * d.dir_w + k / TCHUNK] * TCHUNK + k % TCHUNK];
}

__device__ __forceinline__ int64_t fp_tokens(int64_t t, int bs) { return ((t + bs - 1) / bs) * bs; }

__device__ __forceinline__ int64_t rt_of(const Dev& d, int i, int64_t now) {
    return d.first_tok[i] < 0 ? d.slo_ttft[i] - (now - d.arr[i]) : d.slo_tbt[i] - (now - d.last_tok[i]);
}
// engine.py:275-282: min(granted, lowest guest offset)
__device__ __forceinline__ int32_t eff_of(const Dev& d, int i) {
    if (!d.holds[i]) return 0;
    int32_t g = d.granted[i];
    for (int32_t gu = d.guest[i]; gu >= 0; gu = d.gnext[gu]) {
        const int32_t o = d.off[gu];
        g = o < g ? o : g;
    }
    return g;
}
__device__ __forceinline__ bool guest_of(const Dev& d, int i) { return d.holds[i] && d.host[i] >= 0; }
__device__ __forceinline__ int32_t est_rem(const Dev& d, int i) {
    int32_t r = d.est[i] - d.gen[i];
    return r > 0 ? r : 0;
}
__device__ __forceinline__ int32_t target_of(const Dev& d, int i) {
    int32_t a = d.used[i] > d.kv_need[i] ? d.used[i] : d.kv_need[i];
    return a + est_rem(d, i);
}
__device__ __forceinline__ bool returned_of(const Dev& d, int i) {
    return d.state[i] == ST_RUNNING && eff_of(d, i) < d.used[i] + 1;
}
__device__ __forceinline__ bool ready_of(const Dev& d, int i, int64_t now) {
    return d.state[i] != ST_RUNNING || now >= d.ready_at[i];
}
// _FreeTracker.alloc_cost (scheduler.py:350-354)
__device__ __forceinline__ int64_t cost_of(const Dev& d, int i, int64_t grant) {
    if (guest_of(d, i)) return 0;
    int64_t h = d.holds[i] ? d.granted[i] : 0;
    return fp_tokens(h + grant, d.bs) - fp_tokens(h, d.bs);
}
__device__ __forceinline__ int64_t free_tokens(const Dev& d) {
    const Ctl& c = *d.ctl;
    return d.capacity - (int64_t)c.rsv_cur * d.bs - c.fp_sum;
}
// BlockPool.net_release_gain (kvc.py:142-152)
__device__ __forceinline__ int64_t gain_of(const Dev& d, int i) {
    if (d.host[i] >= 0) return 0;
    int64_t freed = fp_tokens(d.granted[i], d.bs);
    for (int32_t g = d.guest[i]; g >= 0; g = d.gnext[g]) freed -= fp_tokens(d.granted[g], d.bs);
    int64_t room = (int64_t)d.rsv_target - d.ctl->rsv_cur;
    int64_t refill = d.rsv[i] < room ? d.rsv[i] : room;
    return freed - refill * d.bs;
}
// preemption.py:198-200 via engine.py:355-358
__device__ __forceinline__ int32_t strategy_of(const Dev& d, int i) {
    int64_t s = d.used[i] > 1 ? d.used[i] : 1;
    return s > d.s_star ? CO_SWAP : CO_RECOMPUTE;
}
__device__ __forceinline__ int64_t lut(const int64_t* t, int64_t s, int64_t smax) {
    return t[s < smax ? s : smax];
}
// %globaltimer phase stamps (tools/phase_timeline.py); compiled in only for
// development builds (CACHEOPT_NVCC_EXTRA=-DCO_PHASE_PROF): every stamp site
// is executed code the step fetches after an L2 flush
__device__ __forceinline__ void prof_mark(const Dev& d, int slot) {
#ifdef CO_PHASE_PROF
    if (d.prof && threadIdx.x == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        d.prof[slot] = (int64_t)t;
    }
#endif
}
// costmodel.py:51-55 iteration_latency in IEEE double, no contraction
__device__ __forceinline__ double iter_ms(const Dev& d, int64_t tokens) {
    return __dadd_rn(d.base_ms, __dmul_rn(d.per_token_ms, (double)tokens));
}
// core.py:21-23 to_us
__device__ __forceinline__ int64_t to_us_d(double ms) { return (int64_t)floor(__dadd_rn(__dmul_rn(ms, 1000.0), 0.5)); }

// The waiting-queue key of a request, fixed while it waits: set when it
// becomes WAITING (admission) or PREEMPTED, the only transitions into the
// waiting states.  CacheOPT (scheduler.py:151-157): (D << idbits | id rank)
// with D = the deadline, so rt = D - now; the baselines: FCFS by id rank, or
// rlp's (max(1, predicted - generated) / 50, arrival, id) (scheduler.py:869-873).
__device__ __forceinline__ uint64_t wait_key(const Dev& d, int32_t i) {
    if (d.policy == CO_POLICY_CACHEOPT) {
        const int64_t D = d.first_tok[i] < 0 ? d.arr[i] + d.slo_ttft[i] : d.last_tok[i] + d.slo_tbt[i];
        return ((uint64_t)D << d.idbits) | (uint64_t)d.idrank[i];
    }
    if (d.policy == CO_POLICY_RLP) {
        const int32_t r = d.pred[i] - d.gen[i];
        return ((uint64_t)((r > 1 ? r : 1) / 50) << d.idbits) | (uint64_t)d.idrank[i];
    }
    return (uint64_t)d.idrank[i];
}

// Classification of a waiting request (scheduler.py:129-163; baselines
// scheduler.py:760-766, 869-873) shared by k_classify and the planner's
// queue extension: N_w (critical), blown N'_w (arrival order) or the keyed
// N'_w (key order).
enum WaitClass : int32_t { WC_CRIT = 0, WC_BLOWN = 1, WC_KEYED = 2 };
__device__ __forceinline__ int32_t wait_class(const Dev& d, int8_t s, uint64_t key, int64_t now, int64_t ti,
                                              int64_t eps) {
    if (d.policy != CO_POLICY_CACHEOPT)
        return (s == ST_PREEMPTED && d.policy != CO_POLICY_RLP) ? WC_BLOWN : WC_KEYED;
    // every waiting view is ready (engine.py:311-312); rt = D - now
    const int64_t rt = (int64_t)(key >> d.idbits) - now;
    if (rt >= -eps && rt - ti < eps) return WC_CRIT;
    return rt < 0 ? WC_BLOWN : WC_KEYED;
}

// Planner view of one request (engine.py:284-317 fields the planner reads):
// one 64-byte record per live request written by k_classify, so the
// latency-bound planner reads one line per request instead of a dozen SoA
// arrays; hot lists are further staged into shared memory.  The pool is not
// mutated while planning, so a view stays valid for the whole plan.
struct __align__(16) PV {
    int32_t i, eff, target, er, kvn, pre, used, granted, pcount, pg, idrank, flags;
    int64_t rt, gain;
};
enum : int32_t { PV_HOLDS = 1, PV_GUEST = 2, PV_RETURNED = 4, PV_RUNNING = 8, PV_WAITING = 16, PV_READY = 32 };

__device__ __forceinline__ PV make_pv(const Dev& d, int32_t i, int64_t now) {
    PV v;
    v.i = i;
    v.eff = eff_of(d, i);
    v.er = est_rem(d, i);
    v.kvn = d.kv_need[i];
    v.pre = d.prefill[i];
    v.used = d.used[i];
    v.target = (v.used > v.kvn ? v.used : v.kvn) + v.er;
    v.granted = d.holds[i] ? d.granted[i] : 0;
    v.pcount = d.pcount[i];
    v.pg = d.pred[i] - d.gen[i];
    v.idrank = d.idrank[i];
    const int8_t st = d.state[i];
    v.flags = (d.holds[i] ? PV_HOLDS : 0) | (guest_of(d, i) ? PV_GUEST : 0) |
              (st == ST_RUNNING ? PV_RUNNING : 0) | (st == ST_WAITING ? PV_WAITING : 0) |
              ((st == ST_RUNNING && v.eff < v.used + 1) ? PV_RETURNED : 0);
    v.flags |= (st != ST_RUNNING || now >= d.ready_at[i]) ? PV_READY : 0;
    v.rt = rt_of(d, i, now);
    v.gain = (d.holds[i] && d.host[i] < 0) ? gain_of(d, i) : 0;
    return v;
}
// L1 prefetch of the fields make_pv reads (k_classify issues it for a slot
// it already knows needs a view, ahead of the step's begin round trip)
__device__ __forceinline__ void pv_prefetch(const Dev& d, int32_t i) {
#define CO_PF(ptr) asm volatile("prefetch.global.L1 [%0];" ::"l"(ptr))
    CO_PF(d.granted + i); CO_PF(d.used + i); CO_PF(d.holds + i); CO_PF(d.host + i); CO_PF(d.guest + i);
    CO_PF(d.kv_need + i); CO_PF(d.prefill + i); CO_PF(d.est + i); CO_PF(d.gen + i); CO_PF(d.pred + i);
    CO_PF(d.pcount + i); CO_PF(d.idrank + i); CO_PF(d.ready_at + i); CO_PF(d.first_tok + i);
    CO_PF(d.last_tok + i); CO_PF(d.slo_tbt + i); CO_PF(d.rsv + i);
#undef CO_PF
}
// the step's snapshot view, written by k_classify for every live request
__device__ __forceinline__ PV view_of(const Dev& d, int32_t i) {
    const uint4* src = reinterpret_cast<const uint4*>(d.views + i);
    PV v;
    uint4* dst = reinterpret_cast<uint4*>(&v);
    dst[0] = src[0]; dst[1] = src[1]; dst[2] = src[2]; dst[3] = src[3];
    return v;
}

}  // namespace co
