// k_plan: the CacheOPT planner (scheduler.py:408-753, rows a4-a10) on one
// 1024-thread CTA.  The reference's greedy loops are order dependent and
// operate on a running free counter, so they run in reference order on
// thread 0 over staged lists, while every N-wide pass (set construction,
// demand sums, decode membership, the token-budget prefix, the case-2 extras
// walk, the pair-release provider search, the amortized split's ranking) is
// a block-cooperative scan / reduction / compaction / rank sort.
#pragma once
#include "block_ops.cuh"
#include "pool_ops.cuh"

namespace co {

__device__ __forceinline__ int64_t pv_cost(const PV& v, int64_t grant, int bs) {  // scheduler.py:350-354
    if (v.flags & PV_GUEST) return 0;
    return fp_tokens(v.granted + grant, bs) - fp_tokens(v.granted, bs);
}

constexpr int PV_CAP = 1024;
constexpr int INV_CAP = 1024;            // live demands per group on the inverted-weight path
constexpr int INV_LIMBS = INV_CAP + 8;   // 64-bit limbs per multi-precision number there
struct FV {  // fulfilled provider candidate (scheduler.py:685-689, 711-716)
    int64_t gain;
    int32_t er, idrank, i, _pad;
};
constexpr int FV_CAP = 1024;
constexpr int RV_CAP = 1024;

struct PlanSh {
    BlkShared b;
    PV pv[PV_CAP];
    FV fv[FV_CAP];
    int32_t pneed[PV_CAP], pgrant[PV_CAP];
    int64_t tri_key[PV_CAP];     // host triples (a_j - u_j), cached when n_tri <= PV_CAP
    int32_t tri_idx[PV_CAP], tri_taken[PV_CAP];
    int32_t n_tri_cached;
    PV rv[RV_CAP];               // the running set's views, staged once per plan
    int32_t blkoff[2][1288];     // prefix of the classify blocks' running / blown counts
    int32_t mat, any_feasible;
    unsigned __int128 wsum;
    int64_t free, shortfall, runway, batch_now, gm_tokens, probe_tok;
    int64_t f_total, a_total, f_supply, a_supply, tbt_floor, lim, resid;
    int32_t rsvb, n_mem, n_act, n_pre, n_cl, n_def, n_gm, n_pend, n_mready, n_part;
    int32_t k_sel, search, cur, pos, stop, sated, overflow, g_nlive, g_left;
    // the keyed N'_w materialized so far: l_nwp[0..mat) in key order holds
    // every keyed item with key < lo_key (then the blown tail)
    uint64_t lo_key;
    int32_t cand_done, xcnt, xbest;
    int32_t any_flags;  // over the running views: 1 returned, 2 proactive candidate, 4 top-up candidate
    int32_t ndec0;      // running views past prefill and not guests (the decode runway before victims)
    int32_t xh[XNB];
};

// Appends to l_nwp[S.mat..) the next keyed N'_w items in key order: every
// item with key in [S.lo_key, hi), hi chosen from a histogram so that about
// `want` (at most XCHUNK) items come in.  A block-wide pass over the live
// slots re-derives membership with k_classify's own wait_class; used when
// the step needs more of the queue than k_classify's candidate head.
__device__ __forceinline__ int32_t nwp_extend(const Dev& d, PlanSh& S, int32_t want, int64_t now, int64_t ti, int64_t eps) {
    const Ctl& c = *d.ctl;
    const int tid = threadIdx.x, bd = (int)blockDim.x;
    const uint64_t lo = S.lo_key;
    if (c.cnt_nwp == 0 || lo > c.kmax) return 0;
    const int32_t n = c.next_pending;
    uint64_t top = c.kmax, hi;
    auto keyed = [&](int32_t i, uint64_t& k) -> bool {
        const int8_t s = d.state[i];
        if (s != ST_WAITING && s != ST_PREEMPTED) return false;
        k = d.key0[i];
        return wait_class(d, s, k, now, ti, eps) == WC_KEYED;
    };
    while (true) {
        const uint64_t range = top - lo;
        const int bits = range ? 64 - __clzll((long long)range) : 0;
        const int sh = bits > 11 ? bits - 11 : 0;  // (range >> sh) < XNB
        for (int k = tid; k < XNB; k += bd) S.xh[k] = 0;
        __syncthreads();
        for (int32_t i = tid; i < n; i += bd) {
            uint64_t k;
            if (keyed(i, k) && k >= lo && k <= top) atomicAdd(&S.xh[(k - lo) >> sh], 1);
        }
        __syncthreads();
        const int32_t total = blk_scan_smem(S.xh, XNB, S.b);  // exclusive prefix in place
        uint64_t bst = ~0ull;
        for (int b = tid; b < XNB; b += bd) {
            const int32_t incl = b + 1 < XNB ? S.xh[b + 1] : total;
            if (incl >= want && (uint64_t)b < bst) bst = (uint64_t)b;
        }
        bst = blk_min(bst, S.b);
        const int bs_ = bst == ~0ull ? XNB - 1 : (int)bst;
        const int32_t incl = bs_ + 1 < XNB ? S.xh[bs_ + 1] : total, excl = S.xh[bs_];
        __syncthreads();
        if (incl <= XCHUNK) {
            hi = bs_ == XNB - 1 ? top + 1 : lo + ((uint64_t)(bs_ + 1) << sh);
            break;
        }
        if (excl > 0) { hi = lo + ((uint64_t)bs_ << sh); break; }
        top = lo + ((uint64_t)(bs_ + 1) << sh) - 1;  // everything below is empty: refine inside this bin
    }
    if (tid == 0) S.xcnt = 0;
    __syncthreads();
    const int32_t m0 = S.mat;
    for (int32_t i = tid; i < n; i += bd) {
        uint64_t k;
        if (keyed(i, k) && k >= lo && k < hi) {
            d.l_nwp[m0 + atomicAdd(&S.xcnt, 1)] = i;
            const PV v = make_pv(d, i, now);  // its view, as k_classify writes the head's
            uint4* dst = reinterpret_cast<uint4*>(d.views + i);
            const uint4* src = reinterpret_cast<const uint4*>(&v);
            dst[0] = src[0]; dst[1] = src[1]; dst[2] = src[2]; dst[3] = src[3];
        }
    }
    __syncthreads();
    const int32_t got = S.xcnt;
    blk_sort_u64(d.l_nwp + m0, got, [&](int32_t i) { return d.key0[i]; }, d, S.b);
    if (tid == 0) { S.mat = m0 + got; S.lo_key = hi; }
    __syncthreads();
    return got;
}

// the candidate bound for the next step: the key just above the first
// CAND_TARGET keyed items of this step's queue (thread 0, end of the plan)
__device__ __forceinline__ void set_next_threshold(const Dev& d, const PlanSh& S, int32_t n_f0) {
    if (!S.cand_done) return;
    const int32_t keyed = S.mat < n_f0 ? S.mat : n_f0;
    uint64_t t;
    if (keyed >= CAND_TARGET) t = d.key0[d.l_nwp[CAND_TARGET - 1]] + 1;
    else if (S.lo_key > d.ctl->kmax) t = ~0ull;  // the whole keyed queue is the head
    else t = S.lo_key;
    d.ctl->thr = t;
}

__device__ __forceinline__ void push_act(const Dev& d, PlanSh& S, int32_t kind, int32_t i, int64_t tok,
                                         int32_t nb = 0, int32_t h = -1, int64_t start = 0) {
    int32_t p = S.n_act++;
    d.act_kind[p] = kind; d.act_idx[p] = i; d.act_tok[p] = (int32_t)tok;
    d.act_nb[p] = nb; d.act_host[p] = h; d.act_start[p] = (int32_t)start;
}
__device__ __forceinline__ void push_mem(const Dev& d, PlanSh& S, int32_t i, int64_t tok) {
    int32_t p = S.n_mem++;
    d.mem_idx[p] = i; d.mem_tok[p] = (int32_t)tok;
    S.batch_now += tok;
}

// scheduler.py:432-449 try_embed + kvc.py:169-200 find_embedding_host.
// A guest-free host is feasible iff (a_j - u_j) >= b + need + out, so with
// the hosts sorted by (a_j - u_j, id) the argmin is the first free entry at
// or after a lower bound.  With stacking a host that already carries guests
// places the new one below its lowest guest (end = min offset <= a_j), so it
// additionally needs (end - u_j) >= b + need + out; every entry before the
// lower bound is infeasible either way, so the scan stays exact.
__device__ __forceinline__ bool try_embed(const Dev& d, PlanSh& S, const PV& v, int32_t n_tri, int32_t sid) {
    const int32_t i = v.i;
    if (v.eff > 0 || v.pcount > 0) return false;
    int32_t out = v.er > v.pg ? v.er : v.pg;
    if (out < 1) out = 1;
    int64_t need = (int64_t)v.kvn + out;
    int64_t thr = (int64_t)d.buffer_b + need + out;
    const bool cached = S.n_tri_cached;
    int32_t lo = 0, hi = n_tri;
    while (lo < hi) {
        int32_t mid = (lo + hi) >> 1;
        if ((cached ? S.tri_key[mid] : d.l_tri_key[mid]) < thr) lo = mid + 1; else hi = mid;
    }
    int64_t end = 0;
    for (; lo < n_tri; lo++) {
        const int32_t hh = cached ? S.tri_idx[lo] : d.l_tri[lo];
        if ((cached ? S.tri_taken[lo] : d.l_tri_taken[lo]) || d.st_removed[hh] == sid) continue;
        end = (cached ? S.tri_key[lo] : d.l_tri_key[lo]) + d.used[hh];  // a_j
        if (d.guest[hh] >= 0) {  // stacking: below the lowest guest
            end = eff_of(d, hh);
            if (end - d.used[hh] < thr) continue;
        }
        break;
    }
    if (lo >= n_tri) return false;
    int32_t h = cached ? S.tri_idx[lo] : d.l_tri[lo];
    push_act(d, S, A_EMBED, i, need, 0, h, end - need);
    d.st_embedded[i] = sid;
    if (cached) S.tri_taken[lo] = 1; else d.l_tri_taken[lo] = 1;  // one guest per host per plan (scheduler.py:446-448)
    return true;
}

__device__ __forceinline__ int64_t nw_need(const Dev& d, int32_t i) {  // scheduler.py:166-167
    int64_t v = (int64_t)d.kv_need[i] + d.B - eff_of(d, i);
    return v > 0 ? v : 0;
}

// participant view by position: cached for p < PV_CAP, recomputed beyond
__device__ __forceinline__ PV part_pv(const Dev& d, const PlanSh& S, int32_t p, int64_t now) {
    return p < PV_CAP ? S.pv[p] : view_of(d, d.l_part[p]);
}
// exact floor(x / W) and x mod W for x = supply * w with supply < 2^31 (so
// the quotient is < 2^31): double-precision estimate, then exact u128
// multiply corrections (no software 128-bit division)
__device__ __forceinline__ void divmod_small_q(unsigned __int128 x, unsigned __int128 W, uint64_t& q,
                                               unsigned __int128& r) {
    double est = (double)x / (double)W;
    uint64_t qe = est < 0 ? 0 : (uint64_t)est;
    unsigned __int128 prod = (unsigned __int128)qe * W;
    while (prod > x) { qe--; prod -= W; }
    while (prod + W <= x) { qe++; prod += W; }
    q = qe;
    r = x - prod;
}
__device__ __forceinline__ uint64_t amort_weight(const PV& v) {
    int64_t rt = v.rt < 1 ? 1 : v.rt;  // scheduler.py:645: max(1, rt_us), max(1, kv_need)
    int64_t pr = v.kvn < 1 ? 1 : v.kvn;
    return (uint64_t)rt * (uint64_t)pr;
}

// allocate_remaining (scheduler.py:211-243) + block flooring
// (scheduler.py:642-660) over participant positions grp[0..m).  Exact
// integer restatement of the Fraction arithmetic: every share has the common
// denominator W, so floor(share_i) = q_i and the fractional order is the
// order of r_i = supply*w_i mod W (unsigned 128-bit).
__device__ __forceinline__ int32_t& part_need(const Dev& d, PlanSh& S, int32_t p) {
    return p < PV_CAP ? S.pneed[p] : d.l_part_need[p];
}
__device__ __forceinline__ int32_t& part_grant(const Dev& d, PlanSh& S, int32_t p) {
    return p < PV_CAP ? S.pgrant[p] : d.l_part_grant[p];
}

// The exact share computation of a warp of demands with a 128-bit weight sum
// (some weight >= 2^57; never on realistic traces).
__device__ __forceinline__ int64_t amortize_lane_wide(const Dev& d, const PV& v, bool live, int64_t supply,
                                                   int64_t tot, int32_t m) {
    const uint64_t w = live ? amort_weight(v) : 0;
    uint64_t lo = w, hi = 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t lo2 = __shfl_xor_sync(0xffffffffu, lo, o), hi2 = __shfl_xor_sync(0xffffffffu, hi, o);
        uint64_t nl = lo + lo2;
        hi = hi + hi2 + (nl < lo ? 1 : 0);
        lo = nl;
    }
    const unsigned __int128 W = ((unsigned __int128)hi << 64) | lo;
    uint64_t q = 0;
    unsigned __int128 r = 0;
    if (live) divmod_small_q((unsigned __int128)(uint64_t)supply * w, W, q, r);
    int64_t g = (int64_t)q;
    const int64_t left = supply - warp_sum64(g);
    const uint64_t rhi = (uint64_t)(r >> 64), rlo = (uint64_t)r;
    const uint32_t id = live ? (uint32_t)v.idrank : 0xffffffffu;
    int32_t rank = 0;
    for (int j = 0; j < m; j++) {
        const uint64_t jhi = __shfl_sync(0xffffffffu, rhi, j), jlo = __shfl_sync(0xffffffffu, rlo, j);
        const uint32_t jid = __shfl_sync(0xffffffffu, id, j);
        const bool jlive = __shfl_sync(0xffffffffu, live ? 1 : 0, j);
        const bool before = jhi > rhi || (jhi == rhi && (jlo > rlo || (jlo == rlo && jid < id)));
        rank += (jlive && before) ? 1 : 0;
    }
    if (live && rank < left) g += 1;
    if (tot > supply) {
        const int bs = d.bs;
        const int64_t fl = (g / bs) * bs;
        const int64_t left_blocks = (supply - warp_sum64(live ? fl : 0)) / bs;
        const uint64_t rem = (uint64_t)(g - fl);
        int32_t rk = 0;
        for (int j = 0; j < m; j++) {
            const uint64_t jr = __shfl_sync(0xffffffffu, rem, j);
            const uint32_t jid = __shfl_sync(0xffffffffu, id, j);
            const bool jlive = __shfl_sync(0xffffffffu, live ? 1 : 0, j);
            rk += (jlive && (jr > rem || (jr == rem && jid < id))) ? 1 : 0;
        }
        g = fl + ((live && rk < left_blocks) ? bs : 0);
    }
    return live ? g : 0;
}

// amortize() for groups of at most 32 demands, entirely in warp 0 (lane =
// demand): same exact integer arithmetic, ranks by pairwise shuffles, one
// block barrier at the end.  With every weight below 2^57 the weight sum W
// fits 62 bits, so q = floor(supply w / W) (< supply < 2^31) comes from a
// double estimate corrected by exact 64-bit wrap-around remainders (the true
// remainder lies in (-2W, 2W)): no 128-bit arithmetic, no 64-bit division.
__device__ __forceinline__ void amortize_warp(const Dev& d, PlanSh& S, int32_t* grp, int32_t m, int64_t supply, int64_t now,
                              int64_t* total_out) {
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
        const bool in = lane < m;
        const int32_t p = in ? grp[lane] : 0;
        const int64_t need = in ? part_need(d, S, p) : 0;
        const bool live = in && need > 0;
        int64_t tot = need, live_tot = live ? need : 0, nlive = live ? 1 : 0;
        tot = warp_sum64(tot); live_tot = warp_sum64(live_tot); nlive = warp_sum64(nlive);
        int64_t g = 0;
        if (nlive > 0 && supply > 0) {
            if (live_tot <= supply) {
                g = live ? need : 0;
            } else {
                const PV v = live ? part_pv(d, S, p, now) : PV{};
                const uint64_t w = live ? amort_weight(v) : 0;
                if (__any_sync(0xffffffffu, w >= (1ull << 57))) {
                    g = amortize_lane_wide(d, v, live, supply, tot, m);
                } else {
                    uint64_t W = w;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) W += __shfl_xor_sync(0xffffffffu, W, o);
                    int64_t q = 0;
                    uint64_t r = 0;
                    if (live) {
                        int64_t qe = (int64_t)((double)supply * (double)w / (double)W);
                        int64_t rr = (int64_t)((uint64_t)supply * w - (uint64_t)qe * W);
                        while (rr < 0) { qe--; rr += (int64_t)W; }
                        while (rr >= (int64_t)W) { qe++; rr -= (int64_t)W; }
                        q = qe;
                        r = (uint64_t)rr;
                    }
                    const int32_t sup = (int32_t)supply;
                    int32_t gi = (int32_t)q;
                    int32_t sq = gi;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
                    const int32_t left = sup - sq;
                    const uint32_t id = live ? (uint32_t)v.idrank : 0xffffffffu;
                    // largest remainder first, ties by id (scheduler.py:240-242)
                    int32_t rank = 0;
#pragma unroll 4
                    for (int j = 0; j < m; j++) {
                        const uint64_t jr = __shfl_sync(0xffffffffu, r, j);
                        const uint32_t jid = __shfl_sync(0xffffffffu, id, j);
                        const bool jlive = __shfl_sync(0xffffffffu, live ? 1 : 0, j);
                        rank += (jlive && (jr > r || (jr == r && jid < id))) ? 1 : 0;
                    }
                    if (live && rank < left) gi += 1;
                    if (tot > supply) {  // block flooring, leftover blocks by remainder (scheduler.py:653-659)
                        const int32_t bs = d.bs;
                        const int32_t fl = (gi / bs) * bs;
                        int32_t sfl = live ? fl : 0;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) sfl += __shfl_xor_sync(0xffffffffu, sfl, o);
                        const int32_t left_blocks = (sup - sfl) / bs;
                        const int32_t rem = gi - fl;
                        int32_t rk = 0;
#pragma unroll 4
                        for (int j = 0; j < m; j++) {
                            const int32_t jr = __shfl_sync(0xffffffffu, rem, j);
                            const uint32_t jid = __shfl_sync(0xffffffffu, id, j);
                            const bool jlive = __shfl_sync(0xffffffffu, live ? 1 : 0, j);
                            rk += (jlive && (jr > rem || (jr == rem && jid < id))) ? 1 : 0;
                        }
                        gi = fl + ((live && rk < left_blocks) ? bs : 0);
                    }
                    g = live ? gi : 0;
                }
            }
        }
        if (in) part_grant(d, S, p) = (int32_t)g;
        if (lane == 0) S.b.red[0] = tot;
    }
    __syncthreads();
    *total_out = S.b.red[0];
    __syncthreads();
}

// ---------------------------------------------------------------------------
// invert_amortization=True (scheduler.py:43, :229-243 with weights 1/w_i,
// w_i = max(1,rt)*max(1,prompt), :233).  The shares a'*(1/w_i)/S, S = sum
// 1/w_j, have no small common denominator, so this path is exact
// multi-precision arithmetic on one thread (an ablation mode: no fast path).
//   S = p/q with q = prod w_j, p = sum_j prod_{k!=j} w_k  (unreduced; exact)
//   T = a'/S = a'q/p,  F = floor(T) (< 2^128),  phi = T - F = R/p, R = a'q - F p
//   floor(share_i) = floor(T/w_i) = floor(F/w_i),  rho_i = F mod w_i
//   frac_i = (rho_i + phi)/w_i, so frac_i - frac_k has the sign of
//   c*p - D*R with c = rho_i w_k - rho_k w_i and D = w_i - w_k.
// Most comparisons are settled by a double estimate (error < 2^-50); the rest
// are exact.  Limbs are little-endian uint64.
struct Big { uint64_t* l; int n; };

__device__ inline void big_set1(Big& a, uint64_t v) { a.l[0] = v; a.n = v ? 1 : 0; }
__device__ inline void big_trim(Big& a) { while (a.n > 0 && a.l[a.n - 1] == 0) a.n--; }
// o = a * m (m < 2^128); o must not alias a
__device__ inline void big_mul_u128(Big& o, const Big& a, unsigned __int128 m) {
    const uint64_t m0 = (uint64_t)m, m1 = (uint64_t)(m >> 64);
    for (int k = 0; k < a.n + 2; k++) o.l[k] = 0;
    for (int t = 0; t < 2; t++) {
        const uint64_t mm = t ? m1 : m0;
        if (!mm) continue;
        uint64_t carry = 0;
        for (int k = 0; k < a.n; k++) {
            unsigned __int128 x = (unsigned __int128)a.l[k] * mm + o.l[k + t] + carry;
            o.l[k + t] = (uint64_t)x;
            carry = (uint64_t)(x >> 64);
        }
        for (int k = a.n + t; carry; k++) {
            unsigned __int128 x = (unsigned __int128)o.l[k] + carry;
            o.l[k] = (uint64_t)x;
            carry = (uint64_t)(x >> 64);
        }
    }
    o.n = a.n + 2;
    big_trim(o);
}
// a = a * m + b (in place; m < 2^64)
__device__ inline void big_muladd(Big& a, uint64_t m, const Big& b) {
    uint64_t carry = 0;
    const int n = a.n > b.n ? a.n : b.n;
    for (int k = 0; k < n; k++) {
        const uint64_t ak = k < a.n ? a.l[k] : 0, bk = k < b.n ? b.l[k] : 0;
        unsigned __int128 x = (unsigned __int128)ak * m + bk + carry;
        a.l[k] = (uint64_t)x;
        carry = (uint64_t)(x >> 64);
    }
    a.n = n;
    if (carry) a.l[a.n++] = carry;
    big_trim(a);
}
__device__ inline int big_cmp(const Big& a, const Big& b) {
    if (a.n != b.n) return a.n < b.n ? -1 : 1;
    for (int k = a.n - 1; k >= 0; k--)
        if (a.l[k] != b.l[k]) return a.l[k] < b.l[k] ? -1 : 1;
    return 0;
}
// a -= b (a >= b)
__device__ inline void big_sub(Big& a, const Big& b) {
    uint64_t borrow = 0;
    for (int k = 0; k < a.n; k++) {
        const uint64_t bk = k < b.n ? b.l[k] : 0;
        const uint64_t d1 = a.l[k] - bk, b1 = a.l[k] < bk ? 1 : 0;
        a.l[k] = d1 - borrow;
        borrow = b1 | (d1 < borrow ? 1 : 0);
    }
    big_trim(a);
}
// a / b as a double (b > 0): the top limbs of both
__device__ inline double big_ratio(const Big& a, const Big& b) {
    auto top = [](const Big& x, int n) {
        double v = 0;
        for (int k = n - 1; k >= 0 && k >= n - 3; k--) v = v * 18446744073709551616.0 + (k < x.n ? (double)x.l[k] : 0.0);
        return v;
    };
    const int n = a.n > b.n ? a.n : b.n;
    return n ? top(a, n) / top(b, n) : 0.0;
}

struct InvCtx {
    Big p, R, X, Y;
    double phi;
};
// sign of frac_i - frac_k (see above); w = weights, rho = F mod w
__device__ inline int inv_frac_cmp(InvCtx& C, uint64_t wi, uint64_t ri, uint64_t wk, uint64_t rk) {
    if (wi == wk) return ri == rk ? 0 : (ri > rk ? 1 : -1);
    const double fi = ((double)ri + C.phi) / (double)wi, fk = ((double)rk + C.phi) / (double)wk;
    if (fi - fk > 0x1p-40) return 1;
    if (fk - fi > 0x1p-40) return -1;
    const unsigned __int128 a = (unsigned __int128)ri * wk, b = (unsigned __int128)rk * wi;
    const int sc = a == b ? 0 : (a > b ? 1 : -1);
    const unsigned __int128 cm = a >= b ? a - b : b - a;
    const int sd = wi > wk ? 1 : -1;
    const uint64_t dm = wi > wk ? wi - wk : wk - wi;
    if (sc == 0) return C.R.n == 0 ? 0 : -sd;
    if (sc != sd) return sc;  // c*p and -D*R share the sign of c
    big_mul_u128(C.X, C.p, cm);
    big_mul_u128(C.Y, C.R, dm);
    const int s = big_cmp(C.X, C.Y);
    return sc > 0 ? s : -s;
}

// amortize() with inverted weights: thread 0 computes every grant; the block
// waits at one barrier.  Errors (code 12) when a group holds more than
// INV_CAP live demands.
__device__ __noinline__ void amortize_inverted(const Dev& d, PlanSh& S, int32_t* grp, int32_t m, int64_t supply, int64_t now,
                                  int64_t* total_out) {
    if (threadIdx.x == 0) {
        int64_t tot = 0, live_tot = 0;
        int32_t L = 0;
        int32_t* live = d.sk_item;
        for (int32_t k = 0; k < m; k++) {
            const int32_t p = grp[k];
            const int64_t need = part_need(d, S, p);
            tot += need;
            part_grant(d, S, p) = 0;
            if (need > 0) { live_tot += need; live[L++] = p; }
        }
        S.b.red[0] = tot;
        if (L > 0 && supply > 0 && live_tot <= supply) {
            for (int32_t k = 0; k < L; k++) part_grant(d, S, live[k]) = part_need(d, S, live[k]);
        } else if (L > INV_CAP && supply > 0) {
            if (d.ctl) { d.ctl->error = 12; d.ctl->err_info[0] = L; }
        } else if (L > 0 && supply > 0) {
            Big q{d.big, 0}, A{d.big + INV_LIMBS, 0};
            InvCtx C{{d.big + 2 * INV_LIMBS, 0}, {d.big + INV_LIMBS, 0}, {d.big + 3 * INV_LIMBS, 0},
                     {d.big + 4 * INV_LIMBS, 0}, 0.0};
            uint64_t* w = d.am_rhi;   // weights by live position
            uint64_t* rho = d.am_rlo;
            big_set1(q, 1);
            C.p.n = 0;
            for (int32_t k = 0; k < L; k++) {
                w[k] = amort_weight(part_pv(d, S, live[k], now));
                big_muladd(C.p, w[k], q);    // p = p*w + q
                Big z{C.X.l, 0};
                big_muladd(q, w[k], z);      // q = q*w
            }
            big_mul_u128(A, q, (unsigned __int128)(uint64_t)supply);  // A = a' q
            // F = floor(A / p) by bits (F <= a' * min w < 2^128)
            unsigned __int128 F = 0;
            for (int b = 127; b >= 0; b--) {
                const unsigned __int128 cand = F | ((unsigned __int128)1 << b);
                big_mul_u128(C.X, C.p, cand);
                if (big_cmp(C.X, A) <= 0) F = cand;
            }
            big_mul_u128(C.X, C.p, F);
            big_sub(A, C.X);  // A becomes R = a'q - F p (C.R aliases it)
            C.R.n = A.n;
            C.phi = big_ratio(C.R, C.p);
            int64_t sq = 0;
            for (int32_t k = 0; k < L; k++) {
                const uint64_t g = (uint64_t)(F / w[k]);
                rho[k] = (uint64_t)(F % w[k]);
                part_grant(d, S, live[k]) = (int32_t)g;
                sq += (int64_t)g;
            }
            // largest remainder first, ties by req_id (scheduler.py:240-242):
            // partial selection of the `left` best positions to the front
            const int64_t left = supply - sq;
            auto id_of = [&](int32_t k) { return part_pv(d, S, live[k], now).idrank; };
            for (int32_t t = 0; t < left && t < L; t++) {
                int32_t best = t;
                for (int32_t k = t + 1; k < L; k++) {
                    const int c = inv_frac_cmp(C, w[k], rho[k], w[best], rho[best]);
                    if (c > 0 || (c == 0 && id_of(k) < id_of(best))) best = k;
                }
                if (best != t) {
                    int32_t ti = live[t]; live[t] = live[best]; live[best] = ti;
                    uint64_t tw = w[t]; w[t] = w[best]; w[best] = tw;
                    uint64_t tr = rho[t]; rho[t] = rho[best]; rho[best] = tr;
                }
                part_grant(d, S, live[t]) += 1;
            }
            if (tot > supply) {  // block flooring (scheduler.py:653-659)
                const int32_t bs = d.bs;
                int64_t fsum = 0;
                for (int32_t k = 0; k < L; k++) {
                    const int32_t g = part_grant(d, S, live[k]);
                    fsum += (g / bs) * bs;
                }
                const int64_t left_blocks = (supply - fsum) / bs;
                for (int32_t t = 0; t < L; t++) {
                    int32_t best = t;
                    if (t < left_blocks) {
                        for (int32_t k = t + 1; k < L; k++) {
                            const int32_t gk = part_grant(d, S, live[k]), gb = part_grant(d, S, live[best]);
                            const int32_t rk = gk - (gk / bs) * bs, rb = gb - (gb / bs) * bs;
                            if (rk > rb || (rk == rb && id_of(k) < id_of(best))) best = k;
                        }
                        int32_t ti = live[t]; live[t] = live[best]; live[best] = ti;
                    }
                    int32_t& g = part_grant(d, S, live[t]);
                    g = (g / bs) * bs + (t < left_blocks ? bs : 0);
                }
            }
        }
    }
    __syncthreads();
    *total_out = S.b.red[0];
    __syncthreads();
}

// INV: invert_amortization (a separate k_serial instantiation, so the
// default planner's code carries no trace of the inverted path)
template <bool INV>
__device__ __forceinline__ void amortize(const Dev& d, PlanSh& S, int32_t* grp, int32_t m, int64_t supply, int64_t now,
                         int64_t* total_out) {
    const int tid = threadIdx.x;
    if (m == 0) { *total_out = 0; return; }  // block-uniform: nothing to split
    if (INV) { amortize_inverted(d, S, grp, m, supply, now, total_out); return; }
    if (m <= 32) { amortize_warp(d, S, grp, m, supply, now, total_out); return; }
    int64_t tot = 0, live_tot = 0, nlive = 0;
    for (int32_t k = tid; k < m; k += (int)blockDim.x) {
        int32_t p = grp[k];
        int64_t need = part_need(d, S, p);
        tot += need;
        if (need > 0) { live_tot += need; nlive += 1; }
        part_grant(d, S, p) = 0;
    }
    blk_sum3(tot, live_tot, nlive, S.b);
    *total_out = tot;
    if (nlive == 0) return;
    if (supply == 0) {
        // a' = 0: every share a'*w/W and remainder is 0, nothing is left over
        // and the block floor keeps 0 (scheduler.py:229-243, 653-659)
        return;
    }
    if (live_tot <= supply) {
        for (int32_t k = tid; k < m; k += (int)blockDim.x) {
            int32_t p = grp[k];
            int64_t need = part_need(d, S, p);
            if (need > 0) part_grant(d, S, p) = (int32_t)need;
        }
        __syncthreads();
        return;
    }
    // live demands only, order-preserving (the ranking below is total)
    const int32_t w = blk_compact(grp, m, d.sk_item, [&](int32_t p) { return part_need(d, S, p) > 0; }, S.b);
    for (int32_t k = tid; k < w; k += (int)blockDim.x) grp[k] = d.sk_item[k];
    if (tid == 0) S.wsum = 0;
    __syncthreads();
    // W = sum of weights (u128): per-thread partial sums, then one atomic-free
    // serial fold of the 32 warp totals
    unsigned __int128 part = 0;
    for (int32_t k = tid; k < w; k += (int)blockDim.x) part += (unsigned __int128)amort_weight(part_pv(d, S, grp[k], now));
    {
        uint64_t lo = (uint64_t)part, hi = (uint64_t)(part >> 64);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            uint64_t lo2 = __shfl_xor_sync(0xffffffffu, lo, o), hi2 = __shfl_xor_sync(0xffffffffu, hi, o);
            uint64_t nl = lo + lo2;
            hi = hi + hi2 + (nl < lo ? 1 : 0);
            lo = nl;
        }
        if ((tid & 31) == 0) { S.b.ured[tid >> 5] = lo; S.b.red[tid >> 5] = (int64_t)hi; }
    }
    __syncthreads();
    if (tid == 0) {
        unsigned __int128 W = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); k++)
            W += ((unsigned __int128)(uint64_t)S.b.red[k] << 64) | (unsigned __int128)S.b.ured[k];
        S.wsum = W;
    }
    __syncthreads();
    const unsigned __int128 W = S.wsum;
    int64_t sq = 0;
    for (int32_t k = tid; k < w; k += (int)blockDim.x) {
        const int32_t p = grp[k];
        uint64_t q;
        unsigned __int128 r;
        divmod_small_q((unsigned __int128)(uint64_t)supply * amort_weight(part_pv(d, S, p, now)), W, q, r);
        part_grant(d, S, p) = (int32_t)q;
        sq += (int64_t)q;
        d.am_rhi[p] = (uint64_t)(r >> 64);
        d.am_rlo[p] = (uint64_t)r;
    }
    sq = blk_sum(sq, S.b);
    const int64_t left = supply - sq;
    // largest remainder first, ties by req_id (scheduler.py:240-242)
    blk_sort(grp, w, [&](int32_t p, uint64_t& k0, uint64_t& k1, uint64_t& k2) {
        k0 = ~d.am_rhi[p];
        k1 = ~d.am_rlo[p];
        k2 = (uint64_t)d.idrank[d.l_part[p]];
    }, d, S.b);
    for (int32_t k = tid; k < left && k < w; k += (int)blockDim.x) part_grant(d, S, grp[k]) += 1;
    __syncthreads();
    if (tot > supply) {
        const int bs = d.bs;
        int64_t fsum = 0;
        for (int32_t k = tid; k < w; k += (int)blockDim.x) {
            int64_t g = part_grant(d, S, grp[k]);
            fsum += (g / bs) * bs;
        }
        fsum = blk_sum(fsum, S.b);
        const int64_t left_blocks = (supply - fsum) / bs;
        blk_sort(grp, w, [&](int32_t p, uint64_t& k0, uint64_t& k1, uint64_t& k2) {
            int64_t g = part_grant(d, S, p);
            k0 = 0x7fffffffull - (uint64_t)(g - (g / bs) * bs);
            k1 = (uint64_t)d.idrank[d.l_part[p]];
            k2 = 0;
        }, d, S.b);
        for (int32_t k = tid; k < w; k += (int)blockDim.x) {
            int32_t p = grp[k];
            int64_t g = part_grant(d, S, p);
            g = (g / bs) * bs;
            if (k < left_blocks) g += bs;
            part_grant(d, S, p) = (int32_t)g;
        }
        __syncthreads();
    }
}

// The reference's baseline planners (scheduler.py:760-936): vllm_block and
// sarathi_chunked (one function, `chunked`), rlp and s3.  They are short
// ordered greedy loops over the running set (arrival order) and the waiting
// queue (classify keyed it FCFS, preempted first, or by rlp's bucket), so
// thread 0 runs them; the queue is materialized in 256-item groups.
template <class Ensure>
__device__ __forceinline__ void plan_baseline(const Dev& d, PlanSh& S, const int32_t* RUN, int32_t n_run, int32_t n_f0,
                              int32_t n_blown, bool rcached, int32_t sid, Ensure& ensure) {
    const int tid = threadIdx.x, bs = d.bs, pol = d.policy;
    const bool vllm = pol == CO_POLICY_VLLM_BLOCK || pol == CO_POLICY_SARATHI_CHUNKED;
    const bool chunked = pol == CO_POLICY_SARATHI_CHUNKED;
    auto RV = [&](int32_t k) -> PV { return rcached ? S.rv[k] : view_of(d, RUN[k]); };
    auto returned = [&](const PV& v) { return (v.flags & PV_RUNNING) && v.eff < v.used + 1; };
    auto admit_one = [&](int32_t i, int64_t& budget) -> bool {  // false: stop admitting
        const PV v = view_of(d, i);
        int64_t chunk = (int64_t)v.kvn - v.pre, alloc, cost;
        if (vllm) {  // scheduler.py:820-835: round_up(kv_need + 1), costed as a fresh footprint
            alloc = (((int64_t)v.kvn + 1 + d.vbt - 1) / d.vbt) * d.vbt;
            cost = fp_tokens(alloc, bs);
        } else if (pol == CO_POLICY_RLP) {  // scheduler.py:874-877 rlp_demand
            int64_t rem = (int64_t)d.pred[i] - d.gen[i];
            alloc = (int64_t)v.kvn + (rem > 1 ? rem : 1) + d.rlp_pad - v.eff;
            cost = pv_cost(v, alloc, bs);
        } else {  // scheduler.py:917-921 s3_demand, doubling per preemption
            const int64_t p = d.pred[i] > 1 ? d.pred[i] : 1;
            const int64_t nb = (p + d.s3b - 1) / d.s3b;
            const int32_t pc = d.pcount[i];
            int64_t out = (nb > 1 ? nb : 1) * d.s3b;
            out = pc >= 40 ? ((int64_t)1 << 62) : out << pc;  // beyond any pool: the loop breaks
            alloc = (int64_t)v.kvn + out - v.eff;
            if (alloc < 0) alloc = 0;
            cost = alloc >= ((int64_t)1 << 61) ? alloc : pv_cost(v, alloc, bs);
        }
        if (cost > S.free) return false;
        if (chunk > 0) {
            if (chunked) {
                chunk = chunk < budget ? chunk : budget;
                if (chunk < 1) return false;
            } else if (budget < chunk) {
                return false;
            }
            push_mem(d, S, i, chunk);
            budget -= chunk;
        }
        push_act(d, S, vllm ? A_ALLOCATE : ((v.flags & PV_HOLDS) ? A_GROW : A_ALLOCATE), i, alloc);
        S.free -= cost;
        return true;
    };
    if (tid == 0) {
        int64_t budget = d.token_budget;
        if (vllm) {
            // grow exhausted decodes one block, evicting the newest holder (scheduler.py:781-802)
            int32_t vp = n_run - 1;
            for (int32_t k = 0; k < n_run; k++) {
                const PV v = RV(k);
                const int32_t i = RUN[k];
                if (!(v.flags & PV_READY) || !returned(v) || d.st_removed[i] == sid) continue;
                while (true) {
                    const int64_t cost = pv_cost(v, d.vbt, bs);
                    if (cost <= S.free) {
                        push_act(d, S, A_GROW, i, d.vbt);
                        S.free -= cost;
                        d.st_embedded[i] = sid;  // grown this plan
                        break;
                    }
                    while (vp >= 0) {
                        const PV x = RV(vp);
                        if ((x.flags & PV_READY) && d.st_removed[RUN[vp]] != sid && (x.flags & PV_HOLDS)) break;
                        vp--;
                    }
                    if (vp < 0) break;
                    const int32_t victim = RUN[vp];
                    d.pre_idx[S.n_pre] = victim; d.pre_strat[S.n_pre] = CO_RECOMPUTE; S.n_pre++;
                    d.st_removed[victim] = sid;
                    S.free += gain_of(d, victim);
                    if (victim == i) break;
                }
            }
        } else {
            // returned requests evict themselves (scheduler.py:848-851, 900-903)
            for (int32_t k = 0; k < n_run; k++) {
                const PV v = RV(k);
                if (!(v.flags & PV_READY) || !returned(v)) continue;
                d.pre_idx[S.n_pre] = RUN[k];
                d.pre_strat[S.n_pre] = pol == CO_POLICY_RLP ? CO_RECOMPUTE : CO_SWAP;
                S.n_pre++;
                d.st_removed[RUN[k]] = sid;
            }
        }
        // decode (and, chunked, prefill-continuation) members in running order
        for (int32_t k = 0; k < n_run; k++) {
            const PV v = RV(k);
            const int32_t i = RUN[k];
            if (!(v.flags & PV_READY) || d.st_removed[i] == sid) continue;
            if (v.pre < v.kvn) {
                if (!chunked) continue;
                int64_t chunk = (int64_t)v.kvn - v.pre;
                chunk = chunk < budget ? chunk : budget;
                if (chunk > 0) { push_mem(d, S, i, chunk); budget -= chunk; }
                continue;
            }
            if (vllm && returned(v) && d.st_embedded[i] != sid) continue;
            if (budget >= 1) { push_mem(d, S, i, 1); budget -= 1; }
        }
        // admissions: preempted first (FCFS), until the first that does not fit
        S.stop = 0;
        for (int32_t k = 0; k < n_blown; k++)
            if (!admit_one(d.l_blown[k], budget)) { S.stop = 1; break; }
        S.resid = budget;
    }
    __syncthreads();
    for (int32_t base = 0; base < n_f0 && !S.stop; base += (int)blockDim.x) {
        ensure(base + (int)blockDim.x);  // materializes at least [0, base + NT) of the keyed queue
        if (tid == 0) {
            int64_t budget = S.resid;
            const int32_t end = base + (int)blockDim.x < n_f0 ? base + (int)blockDim.x : n_f0;
            for (int32_t k = base; k < end; k++)
                if (!admit_one(d.l_nwp[k], budget)) { S.stop = 1; break; }
            S.resid = budget;
        }
        __syncthreads();
    }
    if (tid == 0) {
        PlanHdr& P = *d.plan;
        P.n_mem = S.n_mem; P.n_act = S.n_act; P.n_pre = S.n_pre; P.n_cl = 0; P.n_def = 0;
        P.batch_tokens = S.batch_now;
        P.overflow = S.batch_now > d.token_budget ? 1 : 0;
        P.sated = 0;
        P.k_sel = 0;
        set_next_threshold(d, S, n_f0);
    }
}

// the planner body (run by k_serial, csrc/cacheopt.cu); all threads call it
// when the step is active
// PLAN: which planner this k_serial instantiation carries -- PLAN_CACHEOPT,
// PLAN_INVERTED (cacheopt with invert_amortization) or PLAN_BASELINES (the
// four baseline policies); the host launches the one matching the config
// (csrc/cacheopt.cu serial_kernel), so each carries only its own code.
enum : int { PLAN_CACHEOPT = 0, PLAN_INVERTED = 1, PLAN_BASELINES = 2 };
template <int PLAN>
__device__ __forceinline__ void plan_body(const Dev& d, PlanSh& S) {
    const Ctl& c = *d.ctl;
    const int tid = threadIdx.x;
    const int64_t now = c.now, ti = c.t_i, eps = d.eps;
    const int32_t sid = c.sid;
    const int32_t n_nw = c.cnt_nw, n_f0 = c.cnt_nwp, n_blown = c.cnt_blown, n_run = c.cnt_run;
    const int32_t n_nwp = n_f0 + n_blown;
    const int32_t* NW = d.crit_idx;   // sorted below by (rt, id)
    const int32_t* NWP = d.l_nwp;     // N'_w queue order, materialized on demand
    const int32_t* RUN = d.l_run;     // running set in arrival order
    const int B = d.B, bs = d.bs;
    if (tid == 0) {
        S.free = free_tokens(d);
        S.rsvb = c.rsv_cur;
        S.n_mem = S.n_act = S.n_pre = S.n_cl = S.n_def = S.n_gm = S.n_pend = S.n_mready = S.n_part = 0;
        S.batch_now = 0; S.gm_tokens = 0; S.overflow = 0; S.sated = 0;
        S.any_flags = 0;
        S.ndec0 = 0;
    }
    __syncthreads();

    prof_mark(d, 0);
    // running set and the blown N'_w tail: concatenate the classify blocks'
    // ordered lists (block b owns indices [b*chunk, (b+1)*chunk))
    for (int32_t b = tid; b < d.nblk; b += (int)blockDim.x) {
        S.blkoff[0][b] = d.blk_cnt[2 * b];
        S.blkoff[1][b] = d.blk_cnt[2 * b + 1];
    }
    if (tid == 0) {
        S.blkoff[0][d.nblk] = 0; S.blkoff[1][d.nblk] = 0;
    }
    __syncthreads();
    blk_scan_smem(S.blkoff[0], d.nblk + 1, S.b);
    blk_scan_smem(S.blkoff[1], d.nblk + 1, S.b);
    // one thread per classify block: the lists are short per block, so all
    // blocks' copies are in flight at once
    for (int32_t b = tid; b < d.nblk; b += (int)blockDim.x) {
        const int32_t r0 = S.blkoff[0][b], nr = S.blkoff[0][b + 1] - r0;
        const int32_t b0 = S.blkoff[1][b], nb = S.blkoff[1][b + 1] - b0, src = b * d.chunk;
#pragma unroll 4
        for (int32_t k = 0; k < nr; k++) d.l_run[r0 + k] = d.run_tmp[src + k];
#pragma unroll 4
        for (int32_t k = 0; k < nb; k++) d.l_blown[b0 + k] = d.blown_tmp[src + k];
    }
    __syncthreads();
    // N_w by (rt, id) (scheduler.py:159); D = rt + now, unique with the id rank
    blk_sort(d.crit_idx, n_nw, [&](int32_t i, uint64_t& k0, uint64_t& k1, uint64_t& k2) {
        k0 = (uint64_t)(view_of(d, i).rt + (1ll << 62)); k1 = (uint64_t)d.idrank[i]; k2 = 0;
    }, d, S.b);
    // N'_w (scheduler.py:151-160): rt >= 0 by (D, id) -- k_classify's
    // candidate head sorted on first use, then extensions -- followed by the
    // blown requests in arrival order.  l_nwp[0..S.mat) is always exact.
    if (tid == 0) { S.cand_done = 0; S.lo_key = 0; S.mat = 0; }
    __syncthreads();
    auto ensure = [&](int32_t target) {
        if (target > n_nwp) target = n_nwp;
        if (S.mat >= target) return;
        if (!S.cand_done) {
            const int32_t nc = c.cnt_cand;
            if (nc <= CAND_CAP) {
                for (int32_t k = tid; k < nc; k += (int)blockDim.x) d.l_nwp[k] = d.cand[k];
                __syncthreads();
                blk_sort_u64(d.l_nwp, nc, [&](int32_t i) { return d.key0[i]; }, d, S.b);
                if (tid == 0) { S.mat = nc; S.lo_key = c.thr; }
            }  // (an overflowed head is ignored: extensions start from key 0)
            if (tid == 0) S.cand_done = 1;
            __syncthreads();
        }
        while (S.mat < target) {
            const int32_t m0 = S.mat;
            if (m0 < n_f0) {
                int32_t want = target - m0;
                const int32_t geo = m0 > CAND_TARGET ? m0 : CAND_TARGET;  // geometric growth
                want = want > geo ? want : geo;
                want = want < XCHUNK ? want : XCHUNK;
                if (nwp_extend(d, S, want, now, ti, eps) == 0) {
                    if (tid == 0) { d.ctl->error = 10; d.ctl->err_info[0] = m0; d.ctl->err_info[1] = n_f0; }
                    __syncthreads();
                    return;
                }
            } else {
                for (int32_t k = tid; k < n_blown; k += (int)blockDim.x) d.l_nwp[m0 + k] = d.l_blown[k];
                if (tid == 0) S.mat = m0 + n_blown;
            }
            __syncthreads();
        }
    };

    const bool rcached = n_run <= RV_CAP;
    // which later phases can have members at all (supersets of their
    // predicates, from the staged views): the empty ones are skipped whole
    const int64_t mpre = d.prealloc_m;
    int fl = 0;
    if (rcached) {
        unsigned nd = 0;
        for (int32_t k = tid; k < n_run; k += (int)blockDim.x) {
            const PV v = view_of(d, RUN[k]);
            S.rv[k] = v;
            const bool ret = (v.flags & PV_RETURNED) != 0;
            fl |= (ret ? 1 : 0) | ((!ret && v.eff < v.target && v.er <= mpre) ? 2 : 0) |
                  ((!ret && !(v.flags & PV_GUEST) && (v.flags & PV_READY) && v.pre >= v.kvn &&
                    (int64_t)v.eff - v.used <= mpre) ? 4 : 0);
            nd += (!(v.flags & PV_GUEST) && v.pre >= v.kvn) ? 1u : 0u;
        }
        fl = (int)__reduce_or_sync(0xffffffffu, (unsigned)fl);
        nd = __reduce_add_sync(0xffffffffu, nd);
        if ((tid & 31) == 0 && fl) atomicOr(&S.any_flags, fl);
        if ((tid & 31) == 0 && nd) atomicAdd(&S.ndec0, (int32_t)nd);
    }
    __syncthreads();
    fl = rcached ? S.any_flags : 7;
    const bool any_ret = (fl & 1) != 0;
    auto RV = [&](int32_t k) -> PV { return rcached ? S.rv[k] : view_of(d, RUN[k]); };

    if (PLAN == PLAN_BASELINES) {
        plan_baseline(d, S, RUN, n_run, n_f0, n_blown, rcached, sid, ensure);
        return;
    }

    // ---- returned running (scheduler.py:142-150, 161-162) ------------------
    auto crit_rt = [&](int64_t r) { return r >= -eps && r - ti < eps; };
    int32_t n_nr = 0, n_nrp = 0;
    if (any_ret) {
        n_nr = blk_compact_at(RUN, n_run, d.l_nr, [&](int32_t k, int32_t i) {
            const PV v = RV(k);
            return (v.flags & PV_READY) && (v.flags & PV_RETURNED) && crit_rt(v.rt);
        }, S.b);
        n_nrp = blk_compact_at(RUN, n_run, d.l_nrp, [&](int32_t k, int32_t i) {
            const PV v = RV(k);
            return (v.flags & PV_READY) && (v.flags & PV_RETURNED) && !crit_rt(v.rt);
        }, S.b);
        blk_sort(d.l_nr, n_nr, [&](int32_t i, uint64_t& k0, uint64_t& k1, uint64_t& k2) {
            k0 = (uint64_t)(rt_of(d, i, now) + (1ll << 62)); k1 = (uint64_t)d.idrank[i]; k2 = 0;
        }, d, S.b);
        blk_sort(d.l_nrp, n_nrp, [&](int32_t i, uint64_t& k0, uint64_t& k1, uint64_t& k2) {
            int64_t r = rt_of(d, i, now);
            k0 = r < 0 ? 1 : 0; k1 = r < 0 ? (uint64_t)d.arr[i] : (uint64_t)r; k2 = (uint64_t)d.idrank[i];
        }, d, S.b);
        for (int32_t k = tid; k < n_nr; k += (int)blockDim.x) d.st_nr[d.l_nr[k]] = sid;
    }

    prof_mark(d, 1);
    // ---- embedding hosts (scheduler.py:425-430) sorted by (a_j - u_j, id) --
    const int32_t n_tri = blk_compact_at(RUN, n_run, d.l_tri, [&](int32_t k, int32_t i) {
        const PV v = RV(k);
        return !(v.flags & PV_GUEST) && (v.flags & PV_HOLDS) && v.pre >= v.kvn;
    }, S.b);
    blk_sort(d.l_tri, n_tri, [&](int32_t i, uint64_t& k0, uint64_t& k1, uint64_t& k2) {
        const PV v = view_of(d, i);
        k0 = (uint64_t)((int64_t)v.granted - v.used + (1ll << 40)); k1 = (uint64_t)v.idrank; k2 = 0;
    }, d, S.b);
    const bool tri_cached = n_tri <= PV_CAP;
    for (int32_t k = tid; k < n_tri; k += (int)blockDim.x) {
        int32_t h = d.l_tri[k];
        const int64_t key = (int64_t)d.granted[h] - d.used[h];
        const int32_t taken = (d.guest[h] >= 0 && !d.stacking) ? 1 : 0;  // already hosting: skipped without stacking
        if (tri_cached) {
            S.tri_key[k] = key; S.tri_idx[k] = h; S.tri_taken[k] = taken;
        } else {
            d.l_tri_key[k] = key; d.l_tri_taken[k] = taken;
        }
    }
    if (tid == 0) S.n_tri_cached = tri_cached ? 1 : 0;
    __syncthreads();

    prof_mark(d, 2);
    // ---- critical waiting: embed first (scheduler.py:451-457) -------------
    if (n_nw > 0) {
        if (tid == 0) {
            for (int32_t k = 0; k < n_nw; k++) {
                int32_t i = NW[k];
                if (try_embed(d, S, view_of(d, i), n_tri, sid)) {
                    int32_t ch = d.kv_need[i] - d.prefill[i];
                    d.l_gm_idx[S.n_gm] = i; d.l_gm_tok[S.n_gm] = ch; S.n_gm++;
                    S.gm_tokens += ch;
                } else {
                    d.l_pend[S.n_pend++] = i;
                }
            }
        }
        __syncthreads();
    }
    const int32_t n_pend0 = S.n_pend;

    prof_mark(d, 3);
    // ---- exact-consumption demand and reserve (scheduler.py:459-472) ------
    int64_t dem = 0;
    if (n_pend0 + n_nr > 0) {  // (block-uniform; nothing to sum in a step without critical requests)
        for (int32_t k = tid; k < n_pend0; k += (int)blockDim.x) {
            const PV v = view_of(d, d.l_pend[k]);
            int64_t need = (int64_t)v.kvn + B - v.eff;
            dem += pv_cost(v, need > 0 ? need : 0, bs);
        }
        for (int32_t k = tid; k < n_nr; k += (int)blockDim.x) {
            const PV v = view_of(d, d.l_nr[k]);
            if (!(v.flags & PV_GUEST)) dem += pv_cost(v, B, bs);
        }
        dem = blk_sum(dem, S.b);
    }
    if (tid == 0) {
        int64_t sf = dem - S.free;
        if (sf < 0) sf = 0;
        if (sf > 0) { int64_t r = (int64_t)S.rsvb * bs; sf -= sf < r ? sf : r; }
        S.shortfall = sf;
    }
    __syncthreads();

    prof_mark(d, 4);
    // ---- victims and deferral (scheduler.py:474-507) ----------------------
    if (S.shortfall > 0) {
        for (int32_t k = tid; k < n_pend0; k += (int)blockDim.x) d.st_crit[d.l_pend[k]] = sid;
        for (int32_t k = tid; k < n_nr; k += (int)blockDim.x) d.st_crit[d.l_nr[k]] = sid;
        __syncthreads();
        const bool fcfs = d.fcfs;
        const int32_t n_v = blk_compact(RUN, n_run, d.l_vict, [&](int32_t i) {
            return !guest_of(d, i) && d.st_crit[i] != sid && d.holds[i] && gain_of(d, i) > 0 &&
                   (fcfs || d.prefill[i] >= d.kv_need[i]);
        }, S.b);
        blk_sort(d.l_vict, n_v, [&](int32_t i, uint64_t& k0, uint64_t& k1, uint64_t& k2) {
            if (fcfs) {  // scheduler.py:397-398: (-arrival, id)
                k0 = (uint64_t)((1ll << 62) - d.arr[i]); k1 = (uint64_t)d.idrank[i]; k2 = 0;
            } else {     // preemption.py:54-64: (-slo bucket, -remaining bucket, occupancy, id)
                uint64_t sb = 0;
                for (int e = 0; e < d.n_edges; e++) sb += d.slo_tbt[i] >= d.edges[e] ? 1 : 0;
                uint64_t rb = (uint64_t)(est_rem(d, i) / d.token_step);
                k0 = ((15ull - sb) << 32) | (0x7fffffffull - rb);
                k1 = (uint64_t)(uint32_t)d.used[i];
                k2 = (uint64_t)d.idrank[i];
            }
        }, d, S.b);
        if (tid == 0) {
            const int64_t queued = (int64_t)n_nw + n_nwp;  // every waiting view is ready
            for (int32_t k = 0; k < n_v && S.shortfall > 0; k++) {
                int32_t i = d.l_vict[k];
                int32_t strat = strategy_of(d, i);
                if (!fcfs) {  // _survives_eviction (scheduler.py:362-375)
                    int64_t s = d.used[i] > 1 ? d.used[i] : 1;
                    int64_t charge = lut(strat == CO_SWAP ? d.lut_surv_swap : d.lut_surv_rec, s, d.s_max) +
                                     ti * (1 + queued);
                    if (!(rt_of(d, i, now) > charge)) continue;
                }
                int64_t g = gain_of(d, i);
                d.pre_idx[S.n_pre] = i; d.pre_strat[S.n_pre] = strat; S.n_pre++;
                d.st_removed[i] = sid;
                S.free += g;
                S.shortfall -= g;
            }
        }
        __syncthreads();
        if (S.shortfall > 0) {
            for (int32_t k = tid; k < n_pend0; k += (int)blockDim.x) d.l_defer[k] = d.l_pend[k];
            __syncthreads();
            blk_sort(d.l_defer, n_pend0, [&](int32_t i, uint64_t& k0, uint64_t& k1, uint64_t& k2) {
                k0 = (uint64_t)((1ll << 62) - rt_of(d, i, now)); k1 = (uint64_t)d.idrank[i]; k2 = 0;
            }, d, S.b);
            if (tid == 0) {
                for (int32_t k = 0; k < n_pend0 && S.shortfall > 0; k++) {
                    int32_t i = d.l_defer[k];
                    S.shortfall -= cost_of(d, i, nw_need(d, i));
                    d.st_deferred[i] = sid;
                    d.def_idx[S.n_def++] = i;
                }
            }
            __syncthreads();
        }
    }

    prof_mark(d, 5);
    // ---- continuation, resumption, critical admission (scheduler.py:515-574)
    if (n_nr + n_nrp + n_pend0 > 0) {
        if (tid == 0) {
            const int32_t nb_B = (B + bs - 1) / bs;
            for (int32_t k = 0; k < n_nr; k++) {
                int32_t i = d.l_nr[k];
                if (d.st_removed[i] == sid) continue;
                int64_t cst = cost_of(d, i, B);
                if (guest_of(d, i)) {
                    push_act(d, S, A_GROW, i, B);
                } else if (cst <= S.free) {
                    push_act(d, S, A_GROW, i, B);
                    S.free -= cst;
                } else if (S.rsvb >= nb_B) {
                    push_act(d, S, A_RESERVE, i, 0, nb_B);
                    S.rsvb -= nb_B;
                } else {
                    d.st_stalled[i] = sid;
                }
            }
            for (int32_t k = 0; k < n_nrp; k++) {
                int32_t i = d.l_nrp[k];
                if (d.st_removed[i] == sid) continue;
                if (guest_of(d, i)) {
                    push_act(d, S, A_GROW, i, B);
                    d.st_resumed[i] = sid;
                    continue;
                }
                int64_t cst = cost_of(d, i, B);
                if (cst <= S.free) {
                    push_act(d, S, A_GROW, i, B);
                    S.free -= cst;
                    d.st_resumed[i] = sid;
                }
            }
            for (int32_t k = 0; k < n_pend0; k++) {
                int32_t i = d.l_pend[k];
                if (d.st_deferred[i] == sid) continue;
                int64_t need = nw_need(d, i);
                int64_t cst = cost_of(d, i, need);
                if (cst <= S.free) {
                    push_act(d, S, d.holds[i] ? A_GROW : A_ALLOCATE, i, need);
                    S.free -= cst;
                } else if (!guest_of(d, i)) {
                    int32_t nb = (int32_t)((need + bs - 1) / bs);
                    if (nb <= S.rsvb) {
                        push_act(d, S, A_RESERVE, i, 0, nb);
                        S.rsvb -= nb;
                    } else {
                        d.def_idx[S.n_def++] = i;
                        continue;
                    }
                } else {
                    d.def_idx[S.n_def++] = i;
                    continue;
                }
                int32_t ch = d.kv_need[i] - d.prefill[i];
                if (ch > 0) {
                    d.l_gm_idx[S.n_gm] = i; d.l_gm_tok[S.n_gm] = ch; S.n_gm++;
                    S.gm_tokens += ch;
                }
            }
        }
        __syncthreads();
    }

    prof_mark(d, 6);
    // ---- decode members in running order (scheduler.py:576-593) -----------
    const int32_t n_dec_mem = blk_compact_at(RUN, n_run, d.mem_idx, [&](int32_t k, int32_t i) {
        const PV v = RV(k);
        if (d.st_removed[i] == sid || !(v.flags & PV_READY) || v.pre < v.kvn) return false;
        if (v.flags & PV_RETURNED) {
            if (d.st_stalled[i] == sid) return false;
            if (d.st_nr[i] != sid && d.st_resumed[i] != sid) return false;
        }
        return true;
    }, S.b);
    for (int32_t k = tid; k < n_dec_mem; k += (int)blockDim.x) d.mem_tok[k] = 1;
    const int32_t n_gm = S.n_gm;
    for (int32_t k = tid; k < n_gm; k += (int)blockDim.x) {
        d.mem_idx[n_dec_mem + k] = d.l_gm_idx[k];
        d.mem_tok[n_dec_mem + k] = d.l_gm_tok[k];
    }
    __syncthreads();
    if (tid == 0) {
        S.n_mem = n_dec_mem + n_gm;
        S.batch_now = n_dec_mem + S.gm_tokens;
    }
    __syncthreads();
    const int64_t consumed = S.batch_now;

    prof_mark(d, 7);
    // ---- token-budget fill over N'_w (scheduler.py:182-200, 596-598) ------
    {
        const int64_t budget = d.token_budget;
        int64_t used_base = consumed;
        int32_t ksel = n_nwp;
        // warp probe of the queue head first: the budget usually fills within
        // a few prompts, so only the first (small) group is materialized
        int32_t base0 = 0;
        if (n_nwp > 0) {
            ensure(32);
            if (tid < 32) {
                const int32_t k = tid;
                int64_t ch = 0;
                if (k < n_nwp) { const PV v = view_of(d, NWP[k]); ch = v.kvn - v.pre; }
                int64_t inc = ch;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (tid >= o) inc += y;
                }
                const unsigned over = __ballot_sync(0xffffffffu, k < n_nwp && used_base + inc > budget);
                const int64_t tot = __shfl_sync(0xffffffffu, inc, 31);
                if (tid == 0) { S.k_sel = over ? __ffs(over) - 1 : -1; S.probe_tok = tot; }
            }
            __syncthreads();
            if (S.k_sel >= 0) ksel = S.k_sel;
            used_base += S.probe_tok;
            base0 = S.k_sel >= 0 ? n_nwp : 32;
            __syncthreads();
        }
        for (int32_t base = base0; base < n_nwp; base += (int)blockDim.x) {
            ensure(base + (int)blockDim.x);
            int32_t k = base + tid;
            int32_t ch = 0;
            if (k < n_nwp) { const PV v = view_of(d, NWP[k]); ch = v.kvn - v.pre; }
            int32_t tot;
            int32_t ex = blk_excl_scan(ch, &tot, S.b);
            bool over = k < n_nwp && used_base + ex + ch > budget;
            uint64_t mk = blk_min(over ? (uint64_t)k : ~0ull, S.b);
            if (mk != ~0ull) { ksel = (int32_t)mk; break; }
            used_base += tot;
        }
        if (tid == 0) {
            S.k_sel = ksel;
            S.overflow = consumed > budget ? 1 : 0;
        }
    }
    __syncthreads();
    const int32_t k_sel = S.k_sel;

    prof_mark(d, 8);
    // ---- participants (scheduler.py:600-638) ------------------------------
    for (int32_t k = tid; k < k_sel && k < PV_CAP; k += (int)blockDim.x) S.pv[k] = view_of(d, NWP[k]);
    __syncthreads();
    if (tid == 0) {
        for (int32_t k = 0; k < k_sel; k++) {
            const PV v = k < PV_CAP ? S.pv[k] : view_of(d, NWP[k]);
            const int32_t i = v.i;
            if (try_embed(d, S, v, n_tri, sid)) { d.l_mready[S.n_mready++] = i; continue; }
            int64_t t = v.target, f = (int64_t)v.kvn + 1;
            int64_t need = (t > f ? t : f) - v.eff;
            if (need <= 0) {
                d.l_mready[S.n_mready++] = i;
            } else {
                d.l_part[S.n_part] = i; d.l_part_need[S.n_part] = (int32_t)need; S.n_part++;
                d.st_parts[i] = sid;
            }
        }
        for (int32_t k = 0; k < n_nrp; k++) {
            int32_t i = d.l_nrp[k];
            if (d.st_removed[i] == sid || guest_of(d, i) || d.st_resumed[i] != sid) continue;
            int64_t res = (int64_t)target_of(d, i) - eff_of(d, i) - B;
            if (res > 0) {
                d.l_part[S.n_part] = i; d.l_part_need[S.n_part] = (int32_t)res; S.n_part++;
                d.st_parts[i] = sid;
            }
        }
    }
    __syncthreads();
    prof_mark(d, 9);
    // proactive_include (scheduler.py:269-279) over the post-eviction running set
    if (fl & 2) {
        const int32_t n_pro = blk_compact_at(RUN, n_run, d.l_pro, [&](int32_t k, int32_t i) {
            const PV v = RV(k);
            return d.st_removed[i] != sid && !(v.flags & PV_RETURNED) && v.eff < v.target && v.er <= mpre;
        }, S.b);
        blk_sort(d.l_pro, n_pro, [&](int32_t i, uint64_t& k0, uint64_t& k1, uint64_t& k2) {
            const PV v = view_of(d, i);
            k0 = (uint64_t)v.er; k1 = (uint64_t)v.idrank; k2 = 0;
        }, d, S.b);
        if (tid == 0) {
            for (int32_t k = 0; k < n_pro; k++) {
                int32_t i = d.l_pro[k];
                if (guest_of(d, i) || d.st_parts[i] == sid) continue;
                d.l_part[S.n_part] = i; d.l_part_need[S.n_part] = target_of(d, i) - eff_of(d, i); S.n_part++;
                d.st_parts[i] = sid;
            }
        }
        __syncthreads();
    }
    prof_mark(d, 10);
    // pre-exhaust top-up, running order (scheduler.py:625-638)
    if (fl & 4) {
        const int32_t base = S.n_part;
        const int32_t n_top = blk_compact_at(RUN, n_run, d.l_part + base, [&](int32_t k, int32_t i) {
            const PV v = RV(k);
            return d.st_removed[i] != sid && !(v.flags & PV_GUEST) && (v.flags & PV_READY) && v.pre >= v.kvn &&
                   !(v.flags & PV_RETURNED) && (int64_t)v.eff - v.used <= mpre && d.st_parts[i] != sid;
        }, S.b);
        for (int32_t k = tid; k < n_top; k += (int)blockDim.x) {
            const PV v = view_of(d, d.l_part[base + k]);
            int64_t t = v.target, f = (int64_t)v.used + 1 + B;
            d.l_part_need[base + k] = (int32_t)((t > f ? t : f) - v.eff);
        }
        __syncthreads();
        if (tid == 0) S.n_part = base + n_top;
        __syncthreads();
    }
    const int32_t n_part = S.n_part;
    prof_mark(d, 11);
    // participant views, cached
    for (int32_t p = tid; p < n_part && p < PV_CAP; p += (int)blockDim.x) {
        S.pv[p] = view_of(d, d.l_part[p]);
        S.pneed[p] = d.l_part_need[p];
    }
    __syncthreads();

    prof_mark(d, 12);
    // ---- amortized round (scheduler.py:662-682) ---------------------------
    int64_t ndec = 0;
    if (rcached && S.n_pre == 0) {  // no victims: the count taken while staging the views
        ndec = S.ndec0;
    } else {
        for (int32_t k = tid; k < n_run; k += (int)blockDim.x) {
            int32_t i = RUN[k];
            const PV v = RV(k);
            if (d.st_removed[i] != sid && !(v.flags & PV_GUEST) && v.pre >= v.kvn) ndec++;
        }
        ndec = blk_sum(ndec, S.b);
    }
    prof_mark(d, 16);
    auto part_running = [&](int32_t p) { return (part_pv(d, S, p, now).flags & PV_RUNNING) != 0; };
    const int32_t n_fl = blk_compact(nullptr, n_part, d.l_grp, [&](int32_t p) { return part_running(p); }, S.b);
    const int32_t n_ad = blk_compact(nullptr, n_part, d.l_grp + n_part, [&](int32_t p) { return !part_running(p); },
                                     S.b);
    if (tid == 0) {
        S.runway = (int64_t)d.runway_iters * ndec;
        S.f_supply = (S.free / bs) * bs;  // free >= 0 throughout planning
    }
    __syncthreads();
    prof_mark(d, 17);
    int64_t ftot;
    amortize<PLAN == PLAN_INVERTED>(d, S, d.l_grp, n_fl, S.f_supply, now, &ftot);
    prof_mark(d, 18);
    int64_t spent = 0;  // sum of the in-flight grants (amortize compacts grp in place)
    if (n_fl > 0) {
        for (int32_t p = tid; p < n_part; p += (int)blockDim.x)
            if (part_running(p)) spent += part_grant(d, S, p);
        spent = blk_sum(spent, S.b);
    }
    if (tid == 0) {
        int64_t a = S.free - spent - S.runway;
        if (a < 0) a = 0;
        S.a_supply = (a / bs) * bs;
        S.f_total = ftot;
    }
    __syncthreads();
    prof_mark(d, 19);
    int64_t atot;
    amortize<PLAN == PLAN_INVERTED>(d, S, d.l_grp + n_part, n_ad, S.a_supply, now, &atot);
    prof_mark(d, 20);
    if (tid == 0) {
        S.a_total = atot;
        S.sated = (S.f_total <= S.f_supply && S.a_total <= S.a_supply) ? 1 : 0;
    }
    __syncthreads();

    prof_mark(d, 13);
    // ---- grant application + pair-release claims (scheduler.py:684-720) ---
    const int32_t n_ful = blk_compact_at(RUN, n_run, d.l_ful, [&](int32_t k, int32_t i) {
        const PV v = RV(k);
        return !(v.flags & PV_GUEST) && !(v.flags & PV_RETURNED) && v.eff >= v.target && d.st_removed[i] != sid;
    }, S.b);
    const bool ful_cached = n_ful <= FV_CAP;
    if (ful_cached) {
        for (int32_t k = tid; k < n_ful; k += (int)blockDim.x) {
            const int32_t q = d.l_ful[k];
            const PV v = view_of(d, q);
            FV f;
            f.gain = v.gain;
            f.er = v.er;
            f.idrank = v.idrank;
            f.i = q;
            f._pad = 0;  // claimed this plan
            S.fv[k] = f;
        }
    }
    __syncthreads();
    // one participant's grant (thread 0); returns whether a provider search is due
    auto grant_one = [&](int32_t p) -> bool {
        const PV v = part_pv(d, S, p, now);
        const int32_t i = v.i;
        const int64_t need = p < PV_CAP ? S.pneed[p] : d.l_part_need[p];
        const int64_t g = part_grant(d, S, p);
        const int64_t eff = v.eff;
        if (!(v.flags & PV_RUNNING)) {
            if (eff + g < (int64_t)v.kvn + 1) return false;  // a partial grant that cannot start prefill
            push_act(d, S, (v.flags & PV_HOLDS) ? A_GROW : A_ALLOCATE, i, g);
            S.free -= pv_cost(v, g, bs);
            d.l_mready[S.n_mready++] = i;
        } else if (g > 0) {
            push_act(d, S, A_GROW, i, g);
            S.free -= pv_cost(v, g, bs);
            if ((v.flags & PV_RETURNED) && eff + g >= (int64_t)v.used + 1) push_mem(d, S, i, 1);
        }
        if (g < need) {
            // scheduler.py:710 rebinds `runway`; the extras gate below sees it
            S.runway = eff + g - v.used;
            S.lim = S.runway > 0 ? S.runway : 0;
            S.resid = need - g;
            S.cur = i;
            return true;
        }
        return false;
    };
    if (ful_cached) {
        // every provider candidate is in shared memory: thread 0 runs the
        // whole ordered loop, pair_release (scheduler.py:253-266) as a scan
        if (tid == 0) {
            for (int32_t p = 0; p < n_part; p++) {
                if (!grant_one(p)) continue;
                int32_t best = -1;
                uint64_t bkey = ~0ull;
                for (int32_t k = 0; k < n_ful; k++) {
                    const FV& f = S.fv[k];
                    if (f._pad || f.er > S.lim || f.gain < S.resid) continue;
                    uint64_t key = ((uint64_t)f.er << 32) | (uint64_t)(uint32_t)f.idrank;
                    if (key < bkey) { bkey = key; best = k; }
                }
                if (best >= 0) {
                    d.cl_w[S.n_cl] = S.cur; d.cl_p[S.n_cl] = S.fv[best].i; S.n_cl++;
                    S.fv[best]._pad = 1;
                }
            }
        }
        __syncthreads();
    } else {
        for (int32_t p = 0; p < n_part; p++) {
            if (tid == 0) S.search = grant_one(p) ? 1 : 0;
            __syncthreads();
            if (S.search) {
                const int64_t lim = S.lim, resid = S.resid;
                uint64_t best = ~0ull;
                for (int32_t k = tid; k < n_ful; k += (int)blockDim.x) {
                    int32_t q = d.l_ful[k];
                    if (d.st_claimed[q] == sid) continue;
                    int64_t er = est_rem(d, q);
                    if (er > lim || gain_of(d, q) < resid) continue;
                    uint64_t key = ((uint64_t)er << 32) | (uint64_t)(uint32_t)d.idrank[q];
                    best = key < best ? key : best;
                }
                best = blk_min(best, S.b);
                if (tid == 0 && best != ~0ull) {
                    int32_t q = d.rank_to_idx[(uint32_t)best];
                    d.cl_w[S.n_cl] = S.cur; d.cl_p[S.n_cl] = q; S.n_cl++;
                    d.st_claimed[q] = sid;
                }
                __syncthreads();
            }
        }
    }
    if (tid == 0) {
        for (int32_t k = 0; k < S.n_mready; k++) {
            int32_t i = d.l_mready[k];
            if (d.state[i] == ST_WAITING) push_mem(d, S, i, d.kv_need[i] - d.prefill[i]);
        }
    }
    __syncthreads();

    prof_mark(d, 14);
    // ---- case 2: extras while sated (scheduler.py:726-748) ----------------
    if (S.sated) {
        uint64_t fl = ~0ull;
        for (int32_t k = tid; k < n_run; k += (int)blockDim.x) {
            int32_t x = RUN[k];
            if (d.st_removed[x] == sid || d.last_tok[x] < 0 || returned_of(d, x)) continue;
            if (d.max_tbt[x] > d.slo_tbt[x]) continue;
            if (d.slo_tbt[x] - (now - d.last_tok[x]) < 0) continue;
            uint64_t v = (uint64_t)d.slo_tbt[x];
            fl = v < fl ? v : fl;
        }
        fl = blk_min(fl, S.b);
        if (tid == 0) { S.tbt_floor = (int64_t)fl; S.stop = 0; S.pos = k_sel; }
        __syncthreads();
        // exact early exit: the loop only ever takes items with need > 0 and
        // cost <= free - runway, and free only decreases, so if no remaining
        // N'_w item qualifies now the walk cannot act (scheduler.py:737-741)
        {
            const int64_t room0 = S.free - S.runway;
            auto feas = [&](int32_t i) {
                const PV v = view_of(d, i);
                const int64_t t = (int64_t)v.target - v.eff;
                return t > 0 && pv_cost(v, t, bs) <= room0;
            };
            int f = 0;
            for (int32_t k = k_sel + tid; k < S.mat; k += (int)blockDim.x) f |= feas(NWP[k]);
            if (S.mat < n_f0) {
                // the keyed items not materialized yet (key >= lo_key): no views
                // were written for them, so they are derived on the spot
                const uint64_t lo = S.lo_key;
                for (int32_t i = tid; i < c.next_pending; i += (int)blockDim.x) {
                    const int8_t s = d.state[i];
                    if (s != ST_WAITING && s != ST_PREEMPTED) continue;
                    const uint64_t k = d.key0[i];
                    if (k < lo || wait_class(d, s, k, now, ti, eps) != WC_KEYED) continue;
                    const PV v = make_pv(d, i, now);
                    const int64_t t = (int64_t)v.target - v.eff;
                    f |= t > 0 && pv_cost(v, t, bs) <= room0;
                }
            }
            if (S.mat <= n_f0)
                for (int32_t k = tid; k < n_blown; k += (int)blockDim.x) f |= feas(d.l_blown[k]);
            if (!__syncthreads_or(f) && tid == 0) S.stop = 1;
            __syncthreads();
        }
        const int64_t batch_now = S.batch_now;
        const bool has_floor = fl != ~0ull;
        for (int32_t base = k_sel; base < n_nwp && !S.stop; base += (int)blockDim.x) {
            ensure(base + (int)blockDim.x);
            int32_t k = base + tid;
            int64_t need = 0, cst = 0;
            if (k < n_nwp) {
                const PV v = view_of(d, NWP[k]);
                int64_t t = (int64_t)v.target - v.eff;
                need = t > 0 ? t : 0;
                cst = pv_cost(v, need, bs);
            }
            while (true) {
                const int64_t room = S.free - S.runway;
                const int32_t pos = S.pos;
                bool ok = k < n_nwp && k >= pos && need > 0 && cst <= room;
                uint64_t mk = blk_min(ok ? (uint64_t)k : ~0ull, S.b);
                if (mk == ~0ull) break;
                if (tid == 0) {
                    int32_t i = NWP[(int32_t)mk];
                    if (has_floor) {
                        double proj = iter_ms(d, batch_now + d.kv_need[i]);
                        if (__dmul_rn(proj, 1000.0) > (double)S.tbt_floor) S.stop = 1;
                    }
                    if (!S.stop) {
                        int64_t t = (int64_t)target_of(d, i) - eff_of(d, i);
                        int64_t nd = t > 0 ? t : 0;
                        push_act(d, S, d.holds[i] ? A_GROW : A_ALLOCATE, i, nd);
                        S.free -= cost_of(d, i, nd);
                        S.pos = (int32_t)mk + 1;
                    }
                }
                __syncthreads();
                if (S.stop) break;
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        PlanHdr& P = *d.plan;
        P.n_mem = S.n_mem; P.n_act = S.n_act; P.n_pre = S.n_pre; P.n_cl = S.n_cl; P.n_def = S.n_def;
        P.batch_tokens = S.batch_now;
        P.overflow = (S.overflow || S.batch_now > d.token_budget) ? 1 : 0;
        P.sated = S.sated;
        P.k_sel = k_sel;
        set_next_threshold(d, S, n_f0);
    }
    prof_mark(d, 15);
}

}  // namespace co
