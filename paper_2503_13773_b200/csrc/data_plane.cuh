// N2/N3: the KV data plane that rides on the N1 block tables.
//
// The reference moves no data (kvc.py:1-16, engine.py:9-14: swap and
// recompute are time charges).  Here every pool mutation that moves KV is
// recorded by the (sequential) apply kernel into a per-step data-op log, with
// its physical addresses snapshotted at the moment the reference would move
// the data; k_data then executes the log in order on the whole GPU:
//   GATHER   swap-out of a preempted request's KV into mapped pinned host
//            pages (engine.py:371-373, strategy SWAP)
//   SCATTER  swap-in of the restored prefix into its new pages
//            (engine.py:391-394)
//   MOVE     guest promotion / re-homing (kvc.py:283-297, 310-317) through an
//            HBM staging buffer (source and destination pages may alias)
//   FILL     the KV a token writes: prefill chunks and decode tokens of this
//            iteration's members, recompute restores (engine.py:395-397).
// Synthetic KV content is a hash of (request id, token, row, dim) so any
// token's bytes can be checked anywhere (k_kv_verify) and the decode can be
// checked against an fp32 reference computed from the same formula.
//
// Pool layout, per page: [layer][K|V][kv_head][slot][head_dim] bf16, so one
// page of one (layer, K|V, head) is a contiguous bs*head_dim tile.  A guest's
// token k lives at host position end-1-k, end = embed_offset + granted.
#pragma once
#include "engine_state.cuh"

namespace co {

// ---- synthetic content ------------------------------------------------------

__device__ __forceinline__ uint32_t mix32(uint32_t h) {
    h ^= h >> 16; h *= 0x7feb352du;
    h ^= h >> 15; h *= 0x846ca68bu;
    h ^= h >> 16;
    return h;
}
// KV element = int8(hash) / 128, exactly representable in bf16
__device__ __forceinline__ uint16_t kv_value(uint32_t rid, uint32_t tok, uint32_t row, uint32_t dim) {
    uint32_t h = mix32(rid * 0x9E3779B1u ^ mix32(tok * 0x85EBCA77u + row * 0xC2B2AE3Du + dim * 0x27D4EB2Fu));
    float v = (float)(int8_t)(h >> 24) * (1.0f / 128.0f);
    return (uint16_t)(__float_as_uint(v) >> 16);
}
// decode query element, fp32
__device__ __forceinline__ float q_value(uint32_t rid, uint32_t step, uint32_t layer, uint32_t qh, uint32_t dim) {
    uint32_t h = mix32(rid * 0x2545F491u ^ mix32(step * 0x9E3779B9u + layer * 0x632BE5ABu + qh * 0x85157AF5u +
                                                dim * 0x4CF5AD43u));
    return (float)(int32_t)(h >> 20) * (1.0f / 2048.0f) - 1.0f;
}

// ---- logging (thread 0 of k_apply) -----------------------------------------

__device__ __forceinline__ DataCtl& dctl(const Dev& d) { return *d.dctl; }

__device__ __forceinline__ int64_t snap_alloc(const Dev& d, const DataCfg& x, int64_t n) {
    DataCtl& c = dctl(d);
    int64_t o = c.n_snap;
    if (o + n > x.snap_cap) { d.ctl->error = 6; return -1; }
    c.n_snap = o + n;
    return o;
}
__device__ __forceinline__ void log_op(const Dev& d, const DataCfg& x, const DOp& op) {
    DataCtl& c = dctl(d);
    if (c.n_ops >= x.op_cap) { d.ctl->error = 6; return; }
    x.ops[c.n_ops++] = op;
}
// snapshot of a standalone request's first npages pages
__device__ __forceinline__ int64_t snap_table(const Dev& d, const DataCfg& x, int i, int32_t npages) {
    int64_t o = snap_alloc(d, x, npages);
    if (o < 0) return 0;
    for (int32_t k = 0; k < npages; k++) x.snap[o + k] = page_of(d, i, k);
    return o;
}
// snapshot of the host pages holding a guest view [end-ntok, end);
// returns the offset, *end_rel = end relative to the first snapshotted page
__device__ __forceinline__ int64_t snap_view(const Dev& d, const DataCfg& x, int h, int32_t end, int32_t ntok, int32_t* end_rel) {
    const int bs = d.bs;
    int32_t p0 = (end - ntok) / bs, p1 = (end - 1) / bs;
    int64_t o = snap_alloc(d, x, p1 - p0 + 1);
    if (o < 0) return 0;
    for (int32_t k = p0; k <= p1; k++) x.snap[o + (k - p0)] = page_of(d, h, k);
    *end_rel = end - p0 * bs;
    return o;
}
// where a request's tokens [0, ntok) live right now
__device__ __forceinline__ void snap_location(const Dev& d, const DataCfg& x, int i, int32_t ntok, int32_t* where, int64_t* snap,
                              int32_t* end) {
    const int32_t h = d.host[i];
    *where = W_DEV;
    if (h >= 0) {
        *snap = snap_view(d, x, h, d.off[i] + d.granted[i], ntok, end);
    } else {
        *end = -1;
        *snap = snap_table(d, x, i, (ntok + d.bs - 1) / d.bs);
    }
}

// swap-out at preemption (before the pool release)
__device__ __forceinline__ void log_swap_out(const Dev& d, const DataCfg& x, int i) {
    const int32_t ntok = d.used[i];
    if (!x.on || ntok <= 0 || !d.holds[i]) return;
    DataCtl& c = dctl(d);
    const int32_t hp = (ntok + d.bs - 1) / d.bs;
    if (hp > c.htop || hp > x.hdir_w) { d.ctl->error = 7; return; }
    DOp op;
    op.kind = D_GATHER; op.req = i; op.ntok = ntok; op.t0 = 0;
    snap_location(d, x, i, ntok, &op.src_where, &op.src_snap, &op.src_end);
    int64_t o = snap_alloc(d, x, hp);
    if (o < 0) return;
    for (int32_t k = 0; k < hp; k++) {
        int32_t pg = x.hstack[--c.htop];
        x.hdir[(int64_t)i * x.hdir_w + k] = pg;
        x.snap[o + k] = pg;
    }
    x.hsaved[i] = hp;
    op.dst_where = W_HOST; op.dst_snap = o; op.dst_end = -1;
    op.io = 0; op.hp = 0; op.stage_off = -1;
    if (x.split_io) {  // k_data stages the pages in HBM; k_swapio sends them over the link
        if (c.stage_fill + ntok > x.gstage_tokens) { d.ctl->error = 6; return; }
        op.io = 1;
        op.stage_off = c.stage_fill;
        c.stage_fill += ntok;
        c.n_io += 1;
    }
    log_op(d, x, op);
}
// readmission: swap-in of the restored prefix or its recompute
__device__ __forceinline__ void log_readmit(const Dev& d, const DataCfg& x, int i, bool swap) {
    if (!x.on) return;
    DataCtl& c = dctl(d);
    const int32_t ntok = d.used[i];
    const int32_t hp = x.hsaved[i];
    if (ntok > 0) {
        DOp op;
        op.req = i; op.ntok = ntok; op.t0 = 0;
        op.dst_where = W_TABLE; op.dst_snap = 0; op.dst_end = -1;
        op.io = 0; op.hp = 0; op.stage_off = -1;
        if (swap && hp > 0) {
            op.kind = D_SCATTER;
            int64_t o = snap_alloc(d, x, hp);
            if (o < 0) return;
            for (int32_t k = 0; k < hp; k++) x.snap[o + k] = x.hdir[(int64_t)i * x.hdir_w + k];
            op.src_where = W_HOST; op.src_snap = o; op.src_end = -1;
            if (x.split_io) {
                // k_swapio reads the host pages after this step's apply, so
                // they return to the swap pool only once it has (below)
                op.io = 1;
                op.hp = hp;
                c.n_io += 1;
                log_op(d, x, op);
                x.hsaved[i] = 0;
                return;
            }
        } else {
            op.kind = D_FILL;
            op.src_where = W_DEV; op.src_snap = 0; op.src_end = -1;
        }
        log_op(d, x, op);
    }
    for (int32_t k = hp - 1; k >= 0; k--) x.hstack[c.htop++] = x.hdir[(int64_t)i * x.hdir_w + k];
    x.hsaved[i] = 0;
}
// guest g leaves the view (end) in host h's pages for its own table:
// call with the view snapshot taken BEFORE the pages moved
__device__ __forceinline__ void log_move(const Dev& d, const DataCfg& x, int g, int32_t ntok, int64_t src_snap, int32_t src_end) {
    if (!x.on || ntok <= 0) return;
    DOp op;
    op.kind = D_MOVE; op.req = g; op.ntok = ntok; op.t0 = 0;
    op.io = 0; op.hp = 0; op.stage_off = -1;
    op.src_where = W_DEV; op.src_snap = src_snap; op.src_end = src_end;
    op.dst_where = W_DEV; op.dst_end = -1;
    op.dst_snap = snap_table(d, x, g, (ntok + d.bs - 1) / d.bs);
    log_op(d, x, op);
}
// KV written by this iteration for tokens [t0, t0+n) of request i
__device__ __forceinline__ void log_fill(const Dev& d, const DataCfg& x, int i, int32_t t0, int32_t n) {
    if (!x.on || n <= 0) return;
    DOp op;
    op.kind = D_FILL; op.req = i; op.ntok = n; op.t0 = t0;
    op.io = 0; op.hp = 0; op.stage_off = -1;
    op.src_where = W_DEV; op.src_snap = 0; op.src_end = -1;
    if (d.host[i] >= 0) {
        op.dst_where = W_DEV;
        op.dst_snap = snap_view(d, x, d.host[i], d.off[i] + d.granted[i], t0 + n, &op.dst_end);
    } else {
        op.dst_where = W_TABLE; op.dst_snap = 0; op.dst_end = -1;
    }
    log_op(d, x, op);
}

// ---- execution ---------------------------------------------------------------

// software grid barrier (every CTA of k_data is co-resident: one per SM)
__device__ __forceinline__ void grid_barrier(uint32_t* bar, uint32_t nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile uint32_t* gen = bar + 1;
        uint32_t g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == nblocks - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) { __nanosleep(64); }
        }
        __threadfence();
    }
    __syncthreads();
}

// element offset of (token, row) of a location
__device__ __forceinline__ int64_t loc_elem(const Dev& d, const DataCfg& x, int32_t where, int64_t snap, int32_t end,
                                            int32_t req, int32_t tok, int32_t row) {
    const int bs = d.bs;
    int32_t page, slot;
    if (where == W_TABLE) {
        page = page_of(d, req, tok / bs);
        slot = tok % bs;
    } else if (end >= 0) {
        int32_t p = end - 1 - tok;
        page = x.snap[snap + p / bs];
        slot = p % bs;
    } else {
        page = x.snap[snap + tok / bs];
        slot = tok % bs;
    }
    return (int64_t)page * x.page_elems + ((int64_t)row * bs + slot) * x.D;
}

// tokens an op moves inside k_data (a split SCATTER is k_swapio's entirely)
__device__ __forceinline__ int64_t kdata_tokens(const DOp& op) {
    return (op.kind == D_SCATTER && op.io) ? 0 : op.ntok;
}

__global__ void __launch_bounds__(512, 1) k_data(Dev d, DataCfg x, DataCtl* dc, int force = 0) {
    const Ctl& c = *d.ctl;
    if (!(c.active || force) || !x.on) return;
    const int32_t nops = dc->n_ops;
    if (nops == 0) return;
    const int64_t units_per_tok = (int64_t)x.rows * (x.D / 8);  // 16-byte units
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsz = (int64_t)gridDim.x * blockDim.x;
    int32_t a = 0;
    while (a < nops) {
        const int32_t kind = x.ops[a].kind;
        int32_t b = a + 1;
        if (kind != D_MOVE) {
            while (b < nops && x.ops[b].kind == kind) b++;
        } else if (x.group_moves) {
            int64_t tk = x.ops[a].ntok;
            while (b < nops && x.ops[b].kind == D_MOVE && tk + x.ops[b].ntok <= x.stage_tokens) tk += x.ops[b++].ntok;
        }
        // ops [a, b): independent, same kind; flat work over their units
        int64_t total = 0;
        for (int32_t o = a; o < b; o++) total += kdata_tokens(x.ops[o]) * units_per_tok;
        const int passes = kind == D_MOVE ? 2 : 1;
        for (int pass = 0; pass < passes; pass++) {
            int32_t o = a;
            int64_t obase = 0;
            for (int64_t u = gtid; u < total; u += gsz) {
                while (u >= obase + kdata_tokens(x.ops[o]) * units_per_tok) {
                    obase += kdata_tokens(x.ops[o]) * units_per_tok;
                    o++;
                }
                const DOp& op = x.ops[o];
                const int64_t w = u - obase;
                const int32_t j = (int32_t)(w / units_per_tok);
                const int32_t r = (int32_t)((w % units_per_tok) / (x.D / 8));
                const int32_t ch = (int32_t)(w % (x.D / 8));
                const int32_t tok = op.t0 + j;
                uint4 v;
                if (op.kind == D_FILL) {
                    uint32_t rid = (uint32_t)d.rid[op.req];
                    uint16_t e[8];
#pragma unroll
                    for (int q = 0; q < 8; q++) e[q] = kv_value(rid, tok, r, ch * 8 + q);
                    v.x = e[0] | ((uint32_t)e[1] << 16); v.y = e[2] | ((uint32_t)e[3] << 16);
                    v.z = e[4] | ((uint32_t)e[5] << 16); v.w = e[6] | ((uint32_t)e[7] << 16);
                    uint16_t* dst = x.kv + loc_elem(d, x, op.dst_where, op.dst_snap, op.dst_end, op.req, tok, r) + ch * 8;
                    *reinterpret_cast<uint4*>(dst) = v;
                    continue;
                }
                const uint16_t* src;
                uint16_t* dst;
                const int64_t so = obase / units_per_tok + j;  // staging slot: token offset within the group
                if (op.kind == D_MOVE && pass == 1) {
                    src = x.stage + (so * x.rows + r) * x.D + ch * 8;
                } else {
                    const uint16_t* base = op.src_where == W_HOST ? x.hkv : x.kv;
                    src = base + loc_elem(d, x, op.src_where, op.src_snap, op.src_end, op.req, tok, r) + ch * 8;
                }
                if (op.kind == D_MOVE && pass == 0) {
                    dst = x.stage + (so * x.rows + r) * x.D + ch * 8;
                } else if (op.kind == D_GATHER && op.io) {  // split I/O: stage in HBM
                    dst = x.gstage + ((op.stage_off + j) * x.rows + r) * x.D + ch * 8;
                } else {
                    uint16_t* base = op.dst_where == W_HOST ? x.hkv : x.kv;
                    dst = base + loc_elem(d, x, op.dst_where, op.dst_snap, op.dst_end, op.req, tok, r) + ch * 8;
                }
                v = __ldcv(reinterpret_cast<const uint4*>(src));  // host pages: no stale cached copy
                *reinterpret_cast<uint4*>(dst) = v;
            }
            __threadfence_system();
            grid_barrier(x.gbar, gridDim.x);
        }
        a = b;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        int64_t tb = (int64_t)x.rows * x.D * 2;
        for (int32_t o = 0; o < nops; o++) {
            int64_t bytes = (int64_t)x.ops[o].ntok * tb;
            switch (x.ops[o].kind) {
                case D_GATHER: dc->bytes_out += bytes; break;
                case D_SCATTER: dc->bytes_in += bytes; break;
                case D_MOVE: dc->bytes_move += bytes; break;
                default: dc->bytes_fill += bytes;
            }
        }
        if (dc->n_io == 0) {  // else k_swapio still reads the log and the snapshots
            dc->n_ops = 0;
            dc->n_snap = 0;
        }
    }
}

// The host-link half of the split swap I/O, on a side stream while the
// decode runs: staged swap-outs to the pinned host pool, swap-ins from it
// into the restored request's pages.  Every such op touches its own pages
// (fresh host pages, the staging slot, or pages of a request that is not a
// decode member before its ready time), so they are independent: one flat
// grid-stride pass, no barrier, an ordinary launch of `io_ctas` small CTAs
// that fit beside the decode's one-CTA-per-SM residency.  The last CTA out
// returns the swap-ins' host pages to the pool and clears the log.
constexpr int IO_T = 256;
__global__ void __launch_bounds__(IO_T) k_swapio(Dev d, DataCfg x, DataCtl* dc) {
    const int32_t nops = dc->n_ops;
    if (dc->n_io == 0) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        dc->io_t0 = (int64_t)t;
    }
    const int64_t upt = (int64_t)x.rows * (x.D / 8);
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gsz = (int64_t)gridDim.x * blockDim.x;
    int64_t obase = 0;
    for (int32_t o = 0; o < nops; o++) {
        const DOp& op = x.ops[o];
        if (!op.io) continue;
        const int64_t units = (int64_t)op.ntok * upt;
        // this thread's first unit of the op (units are numbered across io ops)
        int64_t u0 = gtid - obase % gsz;
        if (u0 < 0) u0 += gsz;
        for (int64_t w = u0; w < units; w += gsz) {
            const int32_t j = (int32_t)(w / upt);
            const int32_t r = (int32_t)((w % upt) / (x.D / 8));
            const int32_t ch = (int32_t)(w % (x.D / 8));
            const uint16_t* src;
            uint16_t* dst;
            if (op.kind == D_GATHER) {
                src = x.gstage + ((op.stage_off + j) * x.rows + r) * x.D + ch * 8;
                dst = x.hkv + loc_elem(d, x, W_HOST, op.dst_snap, -1, op.req, j, r) + ch * 8;
            } else {
                src = x.hkv + loc_elem(d, x, W_HOST, op.src_snap, -1, op.req, j, r) + ch * 8;
                dst = x.kv + loc_elem(d, x, W_TABLE, 0, -1, op.req, j, r) + ch * 8;
            }
            *reinterpret_cast<uint4*>(dst) = __ldcv(reinterpret_cast<const uint4*>(src));
        }
        obase += units;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&dc->io_done, 1) == (int)gridDim.x - 1) {
            __threadfence();
            DataCtl& c = *dc;
            const int64_t tb = (int64_t)x.rows * x.D * 2;
            for (int32_t o = 0; o < nops; o++) {
                const DOp& op = x.ops[o];
                if (!op.io) continue;
                if (op.kind == D_GATHER) {
                    c.io_bytes_out += (int64_t)op.ntok * tb;
                } else {
                    c.io_bytes_in += (int64_t)op.ntok * tb;
                    for (int32_t k = op.hp - 1; k >= 0; k--) x.hstack[c.htop++] = x.snap[op.src_snap + k];
                }
            }
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            c.io_ns += (int64_t)t - c.io_t0;
            c.io_launches += 1;
            c.n_io = 0;
            c.io_done = 0;
            c.stage_fill = 0;
            c.n_ops = 0;
            c.n_snap = 0;
        }
    }
}

// ---- paged decode (split-KV flash decoding) --------------------------------
// work item = (member, layer, kv_head, split of `split` tokens); a 128-thread
// CTA stages one page tile (bs x D of K and of V) at a time and keeps the
// online-softmax state of the G = Hq/Hkv query heads that share the KV head.

constexpr int DEC_T = 128;
constexpr int DEC_GMAX = 16;

__global__ void __launch_bounds__(DEC_T) k_decode(Dev d, DataCfg x, DataCtl* dc) {
    const Ctl& c = *d.ctl;
    if (!c.active || !x.decode_on || !dc->decode_enabled) return;
    const int32_t nitems = dc->dec_items;
    const int G = x.Hq / x.Hkv;
    const int D = x.D;  // 128
    const int bs = d.bs;
    __shared__ float qs[DEC_GMAX][128];
    __shared__ float ks[64][129];
    __shared__ float ps[DEC_GMAX][64];
    __shared__ int32_t pages_sh[64];
    const int tid = threadIdx.x;
    const uint32_t step = (uint32_t)c.steps;
    for (int32_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        // locate (member, lh, split)
        int32_t lo = 0, hi = dc->n_dec;
        while (hi - lo > 1) {
            int32_t mid = (lo + hi) >> 1;
            if (x.dec_item_off[mid] <= it) lo = mid; else hi = mid;
        }
        const int32_t m = lo;
        const int32_t i = x.dec_idx[m];
        const int32_t ctx = x.dec_ctx[m];
        const int32_t nsplit = (ctx + x.split - 1) / x.split;
        const int32_t rel = it - x.dec_item_off[m];
        const int32_t lh = rel / nsplit, sp = rel % nsplit;
        const int32_t layer = lh / x.Hkv, kh = lh % x.Hkv;
        const int32_t t_begin = sp * x.split;
        const int32_t t_end = min(ctx, t_begin + x.split);
        const uint32_t rid = (uint32_t)d.rid[i];
        const float scale = rsqrtf((float)D);
        for (int e = tid; e < G * D; e += DEC_T) {
            int g = e / D, dd = e % D;
            qs[g][dd] = q_value(rid, step, layer, kh * G + g, dd) * scale;
        }
        // owner of the pages: standalone table or guest view in the host
        const int32_t host = d.host[i];
        const int32_t end = host >= 0 ? d.off[i] + d.granted[i] : -1;
        float mrun[DEC_GMAX], lrun[DEC_GMAX];
        float accg[DEC_GMAX];
#pragma unroll
        for (int g = 0; g < DEC_GMAX; g++) { mrun[g] = -INFINITY; lrun[g] = 0.f; accg[g] = 0.f; }
        const int rowK = (layer * 2 + 0) * x.Hkv + kh, rowV = (layer * 2 + 1) * x.Hkv + kh;
        __syncthreads();
        for (int32_t t0 = t_begin; t0 < t_end; t0 += 64) {
            const int32_t nt = min(64, t_end - t0);
            // K tile -> smem (fp32), one token row of D per iteration
            for (int e = tid; e < nt * (D / 8); e += DEC_T) {
                int tt = e / (D / 8), ch = e % (D / 8);
                int32_t tok = t0 + tt;
                int32_t page, slot;
                if (end >= 0) { int32_t p = end - 1 - tok; page = page_of(d, host, p / bs); slot = p % bs; }
                else { page = page_of(d, i, tok / bs); slot = tok % bs; }
                if (ch == 0) pages_sh[tt] = page * bs + slot;
                const uint4 v = *reinterpret_cast<const uint4*>(x.kv + (int64_t)page * x.page_elems +
                                                                ((int64_t)rowK * bs + slot) * D + ch * 8);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    ks[tt][ch * 8 + 2 * q] = __uint_as_float(w[q] << 16);
                    ks[tt][ch * 8 + 2 * q + 1] = __uint_as_float(w[q] & 0xffff0000u);
                }
            }
            __syncthreads();
            // scores: thread handles (g, token) pairs
            for (int e = tid; e < G * nt; e += DEC_T) {
                int g = e / nt, tt = e % nt;
                float s = 0.f;
#pragma unroll 8
                for (int dd = 0; dd < 128; dd++) s += qs[g][dd] * ks[tt][dd];
                ps[g][tt] = s;
            }
            __syncthreads();
            // online softmax per g (each thread redundantly computes the tile max/sum for all g)
            float corr[DEC_GMAX];
            for (int g = 0; g < G; g++) {
                float mx = mrun[g];
                for (int tt = 0; tt < nt; tt++) mx = fmaxf(mx, ps[g][tt]);
                corr[g] = __expf(mrun[g] - mx);
                mrun[g] = mx;
            }
            __syncthreads();
            for (int e = tid; e < G * nt; e += DEC_T) {
                int g = e / nt, tt = e % nt;
                ps[g][tt] = __expf(ps[g][tt] - mrun[g]);
            }
            // V tile -> reuse ks
            for (int e = tid; e < nt * (D / 8); e += DEC_T) {
                int tt = e / (D / 8), ch = e % (D / 8);
                int32_t ps_ = pages_sh[tt];
                int32_t page = ps_ / bs, slot = ps_ % bs;
                const uint4 v = *reinterpret_cast<const uint4*>(x.kv + (int64_t)page * x.page_elems +
                                                                ((int64_t)rowV * bs + slot) * D + ch * 8);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    ks[tt][ch * 8 + 2 * q] = __uint_as_float(w[q] << 16);
                    ks[tt][ch * 8 + 2 * q + 1] = __uint_as_float(w[q] & 0xffff0000u);
                }
            }
            __syncthreads();
            for (int g = 0; g < G; g++) {
                float sum = 0.f, a2 = 0.f;
                for (int tt = 0; tt < nt; tt++) {
                    float p = ps[g][tt];
                    sum += p;
                    a2 += p * ks[tt][tid];
                }
                lrun[g] = lrun[g] * corr[g] + sum;
                accg[g] = accg[g] * corr[g] + a2;
            }
            __syncthreads();
        }
        // partial result: [it][g][D + 2] = acc..., m, l
        float* out = x.dec_part + (int64_t)it * G * (D + 2);
        for (int g = 0; g < G; g++) {
            out[g * (D + 2) + tid] = accg[g];
            if (tid == 0) { out[g * (D + 2) + D] = mrun[g]; out[g * (D + 2) + D + 1] = lrun[g]; }
        }
        __syncthreads();
    }
}

// combine the splits of every (member, layer, q head)
// Split-KV combine: one WARP per work unit = (member, layer, KV head), all G
// query heads of it at once, so a split's partial rows (G x (D + 2) floats)
// are read contiguously and an SM keeps dozens of units in flight (the
// combine is latency-bound: a few KB per unit).  The per-split maxima go
// through the warp's shared-memory slice; each lane then folds four outputs
// at a time over the splits with independent loads.
constexpr int RED_T = 256, RED_W = RED_T / 32, RED_CAP = 128;  // split x head slots per warp
__global__ void __launch_bounds__(RED_T) k_decode_reduce(Dev d, DataCfg x, DataCtl* dc) {
    const Ctl& c = *d.ctl;
    if (!c.active || !x.decode_on || !dc->decode_enabled) return;
    __shared__ float ssc[RED_W][RED_CAP];  // [split][head]: m, then the scale
    __shared__ float sL[RED_W][16];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = x.Hq / x.Hkv, D = x.D, W = D + 2;
    const int32_t nm = dc->n_dec;
    const int64_t total = (int64_t)nm * x.L * x.Hkv;
    float* sc = ssc[wid];
    for (int64_t w = (int64_t)blockIdx.x * RED_W + wid; w < total; w += (int64_t)gridDim.x * RED_W) {
        const int32_t m = (int32_t)(w / ((int64_t)x.L * x.Hkv));
        const int32_t lk = (int32_t)(w % ((int64_t)x.L * x.Hkv));
        const int32_t layer = lk / x.Hkv, kh = lk % x.Hkv;
        const int32_t ctx = x.dec_ctx[m];
        const int32_t nsplit = (ctx + x.split - 1) / x.split;
        const int64_t base_item = x.dec_item_off[m] + (int64_t)(layer * x.Hkv + kh) * nsplit;
        const float* part = x.dec_part + base_item * G * W;  // [split][head][W]
        float* out = x.dec_out + (((int64_t)m * x.L + layer) * x.Hq + (int64_t)kh * G) * D;
        const int ns = nsplit * G;
        if (ns <= RED_CAP && G <= 16) {
            for (int k = lane; k < ns; k += 32) sc[k] = part[(int64_t)k * W + D];
            __syncwarp();
            if (lane < G) {
                float M = -INFINITY;
                for (int s2 = 0; s2 < nsplit; s2++) M = fmaxf(M, sc[s2 * G + lane]);
                float L = 0.f;
                for (int s2 = 0; s2 < nsplit; s2++) {
                    const float e = __expf(sc[s2 * G + lane] - M);
                    sc[s2 * G + lane] = e;
                    L += part[((int64_t)s2 * G + lane) * W + D + 1] * e;
                }
                sL[wid][lane] = L;
            }
            __syncwarp();
            const int64_t SW = (int64_t)G * W;  // floats per split
            if ((D & 1) == 0) {
                // float2 lanes: W = D + 2 is even, so every (split, head) row is 8-B aligned
                const int H2 = D >> 1, GD2 = G * H2;
                for (int f0 = lane; f0 < GD2; f0 += 128) {
                    const float2* pp[4];
                    int gg[4];
                    bool ok[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const int f = f0 + 32 * u;
                        ok[u] = f < GD2;
                        const int g = ok[u] ? f / H2 : 0;
                        gg[u] = g;
                        pp[u] = reinterpret_cast<const float2*>(part + (int64_t)g * W) + (ok[u] ? f - g * H2 : 0);
                    }
                    float2 acc[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) acc[u] = make_float2(0.f, 0.f);
                    for (int s2 = 0; s2 < nsplit; s2++) {
                        float2 v[4];
#pragma unroll
                        for (int u = 0; u < 4; u++) v[u] = ok[u] ? pp[u][s2 * (SW >> 1)] : make_float2(0.f, 0.f);
                        const float* scs = sc + s2 * G;
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            const float e = scs[gg[u]];
                            acc[u].x += v[u].x * e;
                            acc[u].y += v[u].y * e;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 4; u++)
                        if (ok[u]) {
                            const float inv = sL[wid][gg[u]];
                            reinterpret_cast<float2*>(out)[f0 + 32 * u] = make_float2(acc[u].x / inv, acc[u].y / inv);
                        }
                }
            } else {
                const int GD = G * D;
                for (int o0 = lane; o0 < GD; o0 += 128) {
                    const float* pp[4];
                    int gg[4];
                    bool ok[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const int o = o0 + 32 * u;
                        ok[u] = o < GD;
                        const int g = ok[u] ? o / D : 0;
                        gg[u] = g;
                        pp[u] = part + (int64_t)g * W + (ok[u] ? o - g * D : 0);
                    }
                    float acc[4] = {0.f, 0.f, 0.f, 0.f};
                    for (int s2 = 0; s2 < nsplit; s2++) {
                        float v[4];
#pragma unroll
                        for (int u = 0; u < 4; u++) v[u] = ok[u] ? pp[u][s2 * SW] : 0.f;
                        const float* scs = sc + s2 * G;
#pragma unroll
                        for (int u = 0; u < 4; u++) acc[u] += v[u] * scs[gg[u]];
                    }
#pragma unroll
                    for (int u = 0; u < 4; u++)
                        if (ok[u]) out[o0 + 32 * u] = acc[u] / sL[wid][gg[u]];
                }
            }
            __syncwarp();
        } else {
            // more splits x heads than the warp's slice holds: per output, two passes
            for (int o = lane; o < G * D; o += 32) {
                const int g = o / D, j = o - g * D;
                float M = -INFINITY;
                for (int s2 = 0; s2 < nsplit; s2++) M = fmaxf(M, part[((int64_t)s2 * G + g) * W + D]);
                float L = 0.f, acc = 0.f;
                for (int s2 = 0; s2 < nsplit; s2++) {
                    const float* q = part + ((int64_t)s2 * G + g) * W;
                    const float e = __expf(q[D] - M);
                    L += q[D + 1] * e;
                    acc += q[j] * e;
                }
                out[o] = acc / L;
            }
        }
    }
}

// KV integrity: every holder's tokens [0, used) carry their synthetic values
__global__ void k_kv_verify(Dev d, DataCfg x, unsigned long long* bad, unsigned long long* checked) {
    const int64_t units_per_tok = (int64_t)x.rows * x.D;
    for (int32_t i = blockIdx.x; i < d.n; i += gridDim.x) {
        if (!d.holds[i]) continue;
        const int32_t used = d.used[i];
        const int32_t host = d.host[i];
        const int32_t end = host >= 0 ? d.off[i] + d.granted[i] : -1;
        const uint32_t rid = (uint32_t)d.rid[i];
        unsigned long long nb = 0, nc = 0;
        for (int64_t u = threadIdx.x; u < (int64_t)used * units_per_tok; u += blockDim.x) {
            int32_t tok = (int32_t)(u / units_per_tok);
            int32_t r = (int32_t)((u % units_per_tok) / x.D), dim = (int32_t)(u % x.D);
            int32_t page, slot;
            if (end >= 0) { int32_t p = end - 1 - tok; page = page_of(d, host, p / d.bs); slot = p % d.bs; }
            else { page = page_of(d, i, tok / d.bs); slot = tok % d.bs; }
            uint16_t v = x.kv[(int64_t)page * x.page_elems + ((int64_t)r * d.bs + slot) * x.D + dim];
            nb += v != kv_value(rid, tok, r, dim);
            nc++;
        }
        atomicAdd(bad, nb);
        atomicAdd(checked, nc);
    }
}

}  // namespace co
