// kvc.BlockPool (kvc.py:55-375) as a standalone device object: the SAME pool
// functions the engine step runs (csrc/pool_ops.cuh: pool_allocate,
// pool_embed, pool_draw_reserved, pool_grow, pool_promote, pool_release,
// set_used, gain_of, and the N1 block tables under them) applied to a record
// table in HBM, one operation per single-thread kernel.  The kernel also
// evaluates the reference's contract checks in the reference's order and
// reports which one failed (the host raises the matching ValueError) and the
// Grant / Shortfall payload, so the reference's own BlockPool tests run
// against device code (tests/test_pool_device.py).  Included by cacheopt.cu.
#pragma once

namespace co {

enum PoolOp : int32_t {
    PO_ALLOCATE = 0, PO_EMBED = 1, PO_DRAW_RESERVED = 2, PO_GROW = 3, PO_PROMOTE = 4, PO_RELEASE = 5,
    PO_SET_USED = 6, PO_GAIN = 7
};
// out[0]: >0 Grant, 0 Shortfall, <0 contract violation (CO_PV_*, include/cacheopt.h)
// out[1], out[2]: Grant(tokens, footprint) / Shortfall(missing) / release's int

__device__ __forceinline__ void pool_new_slot(const Dev& d, int i) {
    // a fresh AllocationRecord starts with used = 0 (kvc.py:51); the slot may
    // hold a stale value from an earlier record of the same request
    d.used[i] = 0;
}

__global__ void k_pool_op(Dev d, int32_t op, int32_t i, int64_t a, int64_t b, int64_t c3, int64_t* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    Ctl& c = *d.ctl;
    out[0] = 1; out[1] = 0; out[2] = 0;
    const int bs = d.bs;
    switch (op) {
        case PO_ALLOCATE: {  // kvc.py:156-167
            if (a < 1) { out[0] = -CO_PV_TOKENS; return; }
            if (d.holds[i]) { out[0] = -CO_PV_HOLDS; return; }
            const int64_t fp = fp_tokens(a, bs), fr = free_tokens(d);
            if (fp > fr) { out[0] = 0; out[1] = fp - fr; return; }
            pool_new_slot(d, i);
            pool_allocate(d, i, a);
            out[1] = a; out[2] = fp;
            return;
        }
        case PO_EMBED: {  // kvc.py:202-227: n = a, host = b, start = c3
            const int h = (int)b;
            if (a < 1) { out[0] = -CO_PV_TOKENS; return; }
            if (d.holds[i]) { out[0] = -CO_PV_HOLDS; return; }
            if (h < 0 || !d.holds[h]) { out[0] = -CO_PV_NO_RECORD_HOST; return; }
            if (d.host[h] >= 0) { out[0] = -CO_PV_HOST_EMBEDDED; return; }
            if (i == h) { out[0] = -CO_PV_SELF_HOST; return; }
            if (d.guest[h] >= 0 && !d.stacking) { out[0] = -CO_PV_HAS_GUEST; return; }
            if (c3 < 0 || c3 + a > d.granted[h]) { out[0] = -CO_PV_EMBED_RANGE; return; }
            for (int32_t g = d.guest[h]; g >= 0; g = d.gnext[g])
                if (!(c3 + a <= d.off[g] || (int64_t)d.off[g] + d.granted[g] <= c3)) {
                    out[0] = -CO_PV_EMBED_OVERLAP;
                    return;
                }
            pool_new_slot(d, i);
            pool_embed(d, i, a, h, c3);
            out[1] = a; out[2] = 0;
            return;
        }
        case PO_DRAW_RESERVED: {  // kvc.py:229-249: nb = a
            if (a < 1) { out[0] = -CO_PV_BLOCKS; return; }
            if (a > c.rsv_cur) { out[0] = 0; out[1] = (a - c.rsv_cur) * bs; return; }
            if (d.holds[i] && d.host[i] >= 0) { out[0] = -CO_PV_GUEST_RESERVE; return; }
            if (!d.holds[i]) pool_new_slot(d, i);
            pool_draw_reserved(d, i, (int32_t)a);
            out[1] = a * bs; out[2] = a * bs;
            return;
        }
        case PO_GROW: {  // kvc.py:251-281
            if (a < 1) { out[0] = -CO_PV_TOKENS; return; }
            if (!d.holds[i]) { out[0] = -CO_PV_NO_RECORD; return; }
            const int32_t h = d.host[i];
            if (h < 0) {
                const int64_t g = d.granted[i];
                const int64_t delta = fp_tokens(g + a, bs) - fp_tokens(g, bs), fr = free_tokens(d);
                if (delta > fr) { out[0] = 0; out[1] = delta - fr; return; }
                pool_grow(d, i, a);
                out[1] = a; out[2] = delta;
                return;
            }
            int64_t floor_ = (int64_t)d.used[h] + d.buffer_b;
            for (int32_t g = d.guest[h]; g >= 0; g = d.gnext[g])
                if (g != i && d.off[g] < d.off[i]) {
                    const int64_t top = (int64_t)d.off[g] + d.granted[g];
                    floor_ = top > floor_ ? top : floor_;
                }
            const int64_t allowed = (int64_t)d.off[i] - floor_;
            if (a > allowed) { out[0] = 0; out[1] = a - (allowed > 0 ? allowed : 0); return; }
            pool_grow(d, i, a);
            out[1] = a; out[2] = 0;
            return;
        }
        case PO_PROMOTE: {  // kvc.py:283-297
            if (!d.holds[i]) { out[0] = -CO_PV_NO_RECORD; return; }
            if (d.host[i] < 0) { out[0] = -CO_PV_NOT_EMBEDDED; return; }
            const int64_t fp = fp_tokens(d.granted[i], bs), fr = free_tokens(d);
            if (fp > fr) { out[0] = 0; out[1] = fp - fr; return; }
            pool_promote(d, i);
            out[1] = 0; out[2] = fp;
            return;
        }
        case PO_RELEASE: {  // kvc.py:299-324: returns the net tokens freed
            if (!d.holds[i]) { out[0] = -CO_PV_NO_RECORD; return; }
            out[1] = gain_of(d, i);  // = the release's return value (kvc.py:142-152)
            pool_release(d, i);
            return;
        }
        case PO_SET_USED: {  // kvc.py:326-332
            if (!d.holds[i]) { out[0] = -CO_PV_NO_RECORD; return; }
            if (a < 0 || a > d.granted[i]) { out[0] = -CO_PV_USED_RANGE; out[1] = d.granted[i]; return; }
            set_used(d, i, (int32_t)a);
            return;
        }
        case PO_GAIN: {  // kvc.py:142-152
            if (!d.holds[i]) { out[0] = -CO_PV_NO_RECORD; return; }
            out[1] = gain_of(d, i);
            return;
        }
        default:
            out[0] = -CO_PV_TOKENS;
    }
}

// kvc.py:169-200 find_embedding_host over caller triples (slot, id, a_j, u_j):
// feasible hosts hold a standalone record (stacking: below their lowest
// guest), the argmin is by (a_j - u_j, id).  out = {found, slot, start, slack}
__global__ void k_pool_find_host(Dev d, int32_t n, const int64_t* tri, int64_t prompt, int64_t outlen,
                                 int64_t buffer_b, int64_t* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int64_t need = prompt + outlen;
    int64_t bk = 0, bid = 0, bstart = 0, bslack = 0;
    int32_t best = -1;
    for (int32_t k = 0; k < n; k++) {
        const int32_t h = (int32_t)tri[4 * k];
        const int64_t id = tri[4 * k + 1], aj = tri[4 * k + 2], uj = tri[4 * k + 3];
        if (h < 0 || !d.holds[h] || d.host[h] >= 0) continue;
        if (d.guest[h] >= 0 && !d.stacking) continue;
        int64_t end = aj;
        if (d.guest[h] >= 0) {
            end = INT64_MAX;
            for (int32_t g = d.guest[h]; g >= 0; g = d.gnext[g]) end = d.off[g] < end ? d.off[g] : end;
        }
        const int64_t slack = end - (uj + outlen) - need;
        if (slack < buffer_b) continue;
        const int64_t key = aj - uj;
        if (best < 0 || key < bk || (key == bk && id < bid)) {
            best = h; bk = key; bid = id; bstart = end - need; bslack = slack;
        }
    }
    out[0] = best >= 0 ? 1 : 0;
    out[1] = best;
    out[2] = bstart;
    out[3] = bslack;
}

}  // namespace co

struct co_pool {
    co::Dev d{};
    int device = 0;
    cudaStream_t stream = nullptr;
    std::vector<void*> allocs;
    int64_t* out = nullptr;   // device result slots
    int64_t* tri = nullptr;   // find_host triples (grown on demand)
    int64_t tri_cap = 0;
    int32_t n = 0;
};

extern "C" {

int co_pool_destroy(co_pool* P) {
    if (!P) return CO_OK;
    if (P->stream) cudaStreamSynchronize(P->stream);
    for (void* p : P->allocs) cudaFree(p);
    if (P->tri) cudaFree(P->tri);
    if (P->stream) cudaStreamDestroy(P->stream);
    delete P;
    return CO_OK;
}

int co_pool_create(int64_t capacity, int32_t block_size, int32_t reserved_blocks, int32_t buffer_b,
                   int32_t allow_stacking, int32_t max_records, int32_t device, co_pool** out) {
    if (!out) return fail(CO_EINVAL, "null argument");
    *out = nullptr;
    // kvc.py:66-77 validation, same order and messages
    if (capacity < 1) return fail(CO_EINVAL, "capacity must be >= 1");
    if (block_size < 1) return fail(CO_EINVAL, "block_size must be >= 1");
    if (buffer_b < 0) return fail(CO_EINVAL, "buffer_b must be >= 0");
    if (reserved_blocks < 0) return fail(CO_EINVAL, "reserved_blocks must be >= 0");
    if ((int64_t)reserved_blocks * block_size > capacity) return fail(CO_EINVAL, "reserve exceeds capacity");
    if (max_records < 1) return fail(CO_EINVAL, "max_records must be >= 1");
    co_pool* P = new co_pool();
    P->device = device;
    P->n = max_records;
    if (cudaSetDevice(device) != cudaSuccess) { delete P; return fail(CO_ECUDA, "cudaSetDevice"); }
    if (cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete P;
        return fail(CO_ECUDA, "stream");
    }
    co::Dev& d = P->d;
    const int64_t n = max_records;
    const int32_t n_pages = (int32_t)(capacity / block_size);
    const int32_t dir_w = (n_pages + co::TCHUNK - 1) / co::TCHUNK + 1;
    const int64_t n_chunks = (int64_t)n_pages / co::TCHUNK + n + 2;
    auto al = [&](auto** p, int64_t count) -> bool {
        void* q = nullptr;
        if (cudaMalloc(&q, std::max<int64_t>(count, 1) * sizeof(**p)) != cudaSuccess) return false;
        P->allocs.push_back(q);
        *p = static_cast<std::remove_reference_t<decltype(*p)>>(q);
        return cudaMemsetAsync(q, 0, std::max<int64_t>(count, 1) * sizeof(**p), P->stream) == cudaSuccess;
    };
    bool ok = al(&d.ctl, 1) && al(&d.holds, n) && al(&d.granted, n) && al(&d.host, n) && al(&d.off, n) &&
              al(&d.rsv, n) && al(&d.guest, n) && al(&d.gnext, n) && al(&d.rec_seq, n) && al(&d.used, n) &&
              al(&d.tab_len, n) && al(&d.dir, n * dir_w) && al(&d.chunk_pool, n_chunks * co::TCHUNK) &&
              al(&d.chunk_stack, n_chunks) && al(&d.free_stack, n_pages) && al(&P->out, 4);
    if (!ok) { co_pool_destroy(P); return fail(CO_ECUDA, "pool allocation"); }
    for (int32_t* p : {d.host, d.guest, d.gnext}) cudaMemsetAsync(p, 0xff, n * sizeof(int32_t), P->stream);
    std::vector<int32_t> fs(n_pages), cs(n_chunks);
    for (int32_t k = 0; k < n_pages; k++) fs[k] = n_pages - 1 - k;  // pop order 0, 1, 2, ...
    for (int64_t k = 0; k < n_chunks; k++) cs[k] = (int32_t)(n_chunks - 1 - k);
    co::Ctl c0;
    std::memset(&c0, 0, sizeof(c0));
    c0.rsv_cur = reserved_blocks;
    c0.free_top = n_pages;
    c0.chunk_top = (int32_t)n_chunks;
    if ((n_pages && cudaMemcpyAsync(d.free_stack, fs.data(), fs.size() * 4, cudaMemcpyHostToDevice, P->stream)) ||
        cudaMemcpyAsync(d.chunk_stack, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice, P->stream) ||
        cudaMemcpyAsync(d.ctl, &c0, sizeof(c0), cudaMemcpyHostToDevice, P->stream) ||
        cudaStreamSynchronize(P->stream)) {
        co_pool_destroy(P);
        return fail(CO_ECUDA, "pool initialisation");
    }
    d.n = max_records;
    d.bs = block_size;
    d.B = block_size;
    d.buffer_b = buffer_b;
    d.capacity = capacity;
    d.rsv_target = reserved_blocks;
    d.stacking = allow_stacking ? 1 : 0;
    d.n_pages = n_pages;
    d.dir_w = dir_w;
    *out = P;
    return CO_OK;
}

int co_pool_op(co_pool* P, int32_t op, int32_t slot, int64_t a, int64_t b, int64_t c, int64_t* out) {
    if (!P || !out) return fail(CO_EINVAL, "null argument");
    if (slot < 0 || slot >= P->n) return fail(CO_EINVAL, "record slot out of range");
    if (op == co::PO_EMBED && (b < -1 || b >= P->n)) return fail(CO_EINVAL, "host slot out of range");
    co::k_pool_op<<<1, 1, 0, P->stream>>>(P->d, op, slot, a, b, c, P->out);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, P->out, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost, P->stream));
    CK(cudaStreamSynchronize(P->stream));
    co::Ctl c0;
    CK(cudaMemcpy(&c0, P->d.ctl, sizeof(c0), cudaMemcpyDeviceToHost));
    if (c0.error) return fail(CO_EDEVICE, "pool operation left the device pool inconsistent (code " +
                                              std::to_string(c0.error) + ")");
    return CO_OK;
}

int co_pool_find_host(co_pool* P, int32_t n, const int64_t* triples, int64_t prompt, int64_t out_len,
                      int64_t buffer_b, int64_t* out) {
    if (!P || !out || (n > 0 && !triples)) return fail(CO_EINVAL, "null argument");
    if (n > P->tri_cap) {
        if (P->tri) cudaFree(P->tri);
        P->tri = nullptr;
        P->tri_cap = 0;
        CK(cudaMalloc(&P->tri, (size_t)n * 4 * sizeof(int64_t)));
        P->tri_cap = n;
    }
    if (n) CK(cudaMemcpyAsync(P->tri, triples, (size_t)n * 4 * sizeof(int64_t), cudaMemcpyHostToDevice, P->stream));
    co::k_pool_find_host<<<1, 1, 0, P->stream>>>(P->d, n, P->tri, prompt, out_len, buffer_b, P->out);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, P->out, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, P->stream));
    CK(cudaStreamSynchronize(P->stream));
    return CO_OK;
}

int co_pool_state(co_pool* P, int64_t* scalars, int64_t* records) {
    if (!P || !scalars) return fail(CO_EINVAL, "null argument");
    co::Ctl c0;
    CK(cudaMemcpyAsync(&c0, P->d.ctl, sizeof(c0), cudaMemcpyDeviceToHost, P->stream));
    const int64_t n = P->n;
    std::vector<int32_t> buf;
    std::vector<uint8_t> holds;
    std::vector<int64_t> seq;
    if (records) {
        buf.resize((size_t)n * 7);
        holds.resize((size_t)n);
        seq.resize((size_t)n);
        const co::Dev& d = P->d;
        int32_t* cols[7] = {d.granted, d.host, d.off, d.rsv, d.guest, d.gnext, d.used};
        for (int k = 0; k < 7; k++)
            CK(cudaMemcpyAsync(buf.data() + (size_t)k * n, cols[k], n * 4, cudaMemcpyDeviceToHost, P->stream));
        CK(cudaMemcpyAsync(holds.data(), d.holds, n, cudaMemcpyDeviceToHost, P->stream));
        CK(cudaMemcpyAsync(seq.data(), d.rec_seq, n * 8, cudaMemcpyDeviceToHost, P->stream));
    }
    CK(cudaStreamSynchronize(P->stream));
    scalars[0] = P->d.capacity - (int64_t)c0.rsv_cur * P->d.bs - c0.fp_sum;  // free_tokens
    scalars[1] = c0.fp_sum;
    scalars[2] = c0.granted_sum;
    scalars[3] = c0.used_sum;
    scalars[4] = c0.rsv_cur;
    scalars[5] = c0.free_top;
    if (records) {
        // per slot: holds, granted, host, offset, reserved, first guest, next guest, used, record seq
        for (int64_t i = 0; i < n; i++) {
            int64_t* r = records + 9 * i;
            r[0] = holds[i];
            for (int k = 0; k < 7; k++) r[1 + k] = buf[(size_t)k * n + i];
            r[8] = seq[i];
        }
    }
    return CO_OK;
}

int co_pool_check(co_pool* P) {
    if (!P) return fail(CO_EINVAL, "null argument");
    co::k_check<<<1, co::NT, 0, P->stream>>>(P->d);
    CK(cudaGetLastError());
    co::Ctl c0;
    CK(cudaMemcpyAsync(&c0, P->d.ctl, sizeof(c0), cudaMemcpyDeviceToHost, P->stream));
    CK(cudaStreamSynchronize(P->stream));
    if (c0.error == 4) return fail(CO_EDEVICE, "pool invariant violated (kvc.py:336-375)");
    if (c0.error) return fail(CO_EDEVICE, "device pool error code " + std::to_string(c0.error));
    return CO_OK;
}

int co_pool_read_tables(co_pool* P, int32_t* lens, int32_t* pages, int64_t max_pages, int32_t* free_pages,
                        int32_t* n_free) {
    if (!P || !lens || !n_free) return fail(CO_EINVAL, "null argument");
    const co::Dev& d = P->d;
    const int64_t n = P->n;
    const int64_t n_chunks = (int64_t)d.n_pages / co::TCHUNK + n + 2;
    std::vector<int32_t> dir((size_t)n * d.dir_w), pool((size_t)n_chunks * co::TCHUNK);
    co::Ctl c0;
    CK(cudaMemcpyAsync(&c0, d.ctl, sizeof(c0), cudaMemcpyDeviceToHost, P->stream));
    CK(cudaMemcpyAsync(lens, d.tab_len, n * 4, cudaMemcpyDeviceToHost, P->stream));
    CK(cudaMemcpyAsync(dir.data(), d.dir, dir.size() * 4, cudaMemcpyDeviceToHost, P->stream));
    CK(cudaMemcpyAsync(pool.data(), d.chunk_pool, pool.size() * 4, cudaMemcpyDeviceToHost, P->stream));
    CK(cudaStreamSynchronize(P->stream));
    *n_free = c0.free_top;
    if (free_pages && c0.free_top)
        CK(cudaMemcpy(free_pages, d.free_stack, (size_t)c0.free_top * 4, cudaMemcpyDeviceToHost));
    int64_t w = 0;
    for (int64_t i = 0; i < n; i++) {
        if (w + lens[i] > max_pages) return fail(CO_EINVAL, "page buffer too small");
        for (int32_t k = 0; k < lens[i]; k++)
            if (pages) pages[w + k] = pool[(size_t)dir[(size_t)i * d.dir_w + k / co::TCHUNK] * co::TCHUNK + k % co::TCHUNK];
        w += lens[i];
    }
    return CO_OK;
}

}  // extern "C"
