// Types of the KV data plane (see data_plane.cuh).
#pragma once
#include <cstdint>

namespace co {

enum DKind : int32_t { D_GATHER = 0, D_SCATTER = 1, D_MOVE = 2, D_FILL = 3 };
enum DWhere : int32_t { W_DEV = 0, W_HOST = 1, W_TABLE = 2 };

struct DOp {
    int32_t kind, req, ntok, t0;
    int32_t src_where, dst_where, src_end, dst_end;
    int64_t src_snap, dst_snap;
    // split swap I/O (DataCfg::split_io): io = 1 marks a GATHER / SCATTER whose
    // host-link half runs in k_swapio (side stream, overlapping the decode);
    // a GATHER's pages are first staged at gstage[stage_off ..) by k_data
    int64_t stage_off;
    int32_t io, hp;  // hp: host pages a deferred SCATTER returns to the swap pool
};

struct DataCfg {
    uint16_t* kv;        // device pool
    uint16_t* hkv;       // mapped pinned host swap pool (device pointer)
    uint16_t* stage;     // MOVE staging, token-major
    int64_t page_elems;  // elements per page
    int32_t rows;        // layers * 2 * kv_heads
    int32_t D;           // head_dim
    int32_t L, Hkv, Hq, split;
    DOp* ops;
    int32_t* snap;
    int32_t* hstack;
    int32_t* hdir;
    int32_t* hsaved;
    int64_t op_cap, snap_cap, stage_tokens;
    int32_t h_pages, hdir_w;
    // decode
    int32_t* dec_idx;     // decode members of the step
    int32_t* dec_ctx;
    int32_t* dec_item_off;  // prefix of split counts
    float* dec_part;      // [items][G][D + 2]
    float* dec_out;       // [members][L][Hq][D]
    int32_t dec_cap;
    int64_t dec_item_cap;
    uint32_t* gbar;       // grid barrier {count, generation}
    int32_t on, decode_on;
    // stacking: a host release re-homes several guests, and an earlier guest's
    // new pages can be the pages that still hold a later guest's KV, so a run
    // of MOVEs is staged as one group (all reads, then all writes)
    int32_t group_moves;
    // swap-out staging (HBM, token-major, `gstage_tokens` = the pool's tokens:
    // every victim's KV of one step was resident at once) for the split I/O
    uint16_t* gstage;
    int64_t gstage_tokens;
    int32_t split_io, io_ctas;
};

struct DataCtl {
    int32_t n_ops, n_dec, htop, dec_items, decode_enabled;
    int64_t n_snap;
    int64_t bytes_out, bytes_in, bytes_fill, bytes_move;
    int64_t dec_steps, dec_members, dec_tokens;
    int64_t last_bytes_out, last_bytes_in;
    // split swap I/O: ops pending for k_swapio, staged tokens, and its
    // device-timed totals (%globaltimer, first CTA in -> last CTA out)
    int32_t n_io, io_done;
    int64_t stage_fill, io_t0, io_ns, io_bytes_out, io_bytes_in, io_launches;
};

}  // namespace co
