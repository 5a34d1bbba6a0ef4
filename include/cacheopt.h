/*
 * cacheopt.h -- C ABI of the B200-native CacheOPT hot path.
 *
 * The reference (`/root/reference/pkg/src/kvcsim`, pure Python) has no FFI:
 * its "operator" boundary is the engine object (engine.py:222-672) that owns
 * the request table and the KV pool and calls `plan_batch` once per step
 * (engine.py:616, scheduler.py:939).  This header is the boundary a
 * maintainer would bind instead (ctypes stub in INTEGRATION.md): one opaque
 * engine instance per (device, stream), plain pointers and sizes only, no
 * torch types, no C++ exceptions across the ABI.  Every entry point names the
 * reference interface it replaces.
 *
 * Status codes: CO_OK (0), CO_EINVAL (unsupported / invalid input, see
 * co_last_error), CO_ECUDA (a CUDA error), CO_EDEVICE (the device engine
 * raised the equivalent of a reference exception, e.g. the no-progress guard
 * engine.py:653-656).
 */
#ifndef CACHEOPT_H
#define CACHEOPT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CO_OK 0
#define CO_EINVAL 1
#define CO_ECUDA 2
#define CO_EDEVICE 3
#define CO_EAGAIN 4  /* caller buffers too small; the sizes needed were returned */

/* lifecycle codes (core.py:26-30); PENDING = not yet arrived */
#define CO_PENDING 0
#define CO_WAITING 1
#define CO_RUNNING 2
#define CO_PREEMPTED 3
#define CO_COMPLETED 4

#define CO_SWAP 0
#define CO_RECOMPUTE 1

/* event kinds (engine.py:338-340 and its call sites) */
#define CO_EV_ARRIVE 0   /* engine.py:353 */
#define CO_EV_ADMIT 1    /* engine.py:520 */
#define CO_EV_ITER 2     /* engine.py:630-633 */
#define CO_EV_PREEMPT 3  /* engine.py:383-384 */
#define CO_EV_READMIT 4  /* engine.py:401-402 */
#define CO_EV_COMPLETE 5 /* engine.py:412 */

#define CO_CAUSE_PLAN 0
#define CO_CAUSE_SQUEEZE 1
#define CO_CAUSE_COLLISION 2

#define CO_MAX_SLO_EDGES 8

/* Scalars of EngineConfig (engine.py:66-79), SchedulerConfig
 * (scheduler.py:34-48), BucketConfig (preemption.py:19-28) and the
 * per-run constants the reference derives from floats at engine init.
 * The host evaluates every float expression with Python's own IEEE double
 * semantics and passes the results; the device only does integer work plus
 * the two double expressions it evaluates with round-to-nearest intrinsics
 * (iteration latency, costmodel.py:51-55). */
typedef struct co_config {
    int64_t capacity_tokens;        /* engine.py:67 */
    int32_t reserved_blocks;        /* engine.py:68 */
    int32_t allow_stacking;         /* engine.py:69, kvc.py:64: several guests per host */
    int32_t block_size;             /* small_block_b, engine.py:236 */
    int32_t buffer_b;               /* scheduler.py:41 */
    int32_t token_budget;           /* scheduler.py:39 */
    int32_t preallocate_m;          /* scheduler.py:40 */
    int32_t decode_runway_iters;    /* scheduler.py:44 */
    int32_t victim_rule_fcfs;       /* scheduler.py:42: 0 = "slo", 1 = "fcfs" */
    int64_t epsilon_us;             /* scheduler.py:38 */
    int32_t n_slo_edges;            /* preemption.py:21-26 */
    int32_t token_step;             /* preemption.py:27 */
    int64_t slo_edges_us[CO_MAX_SLO_EDGES];
    double iter_base_ms;            /* costmodel.py:21 */
    double iter_per_token_ms;       /* costmodel.py:22 */
    int64_t horizon_factor;         /* engine.py:76 */
    int32_t validate_every;         /* engine.py:77 */
    int32_t record_events;          /* engine.py:78 */
    int32_t padding;                /* estimation.py:139-142 for the run's confidence */
    int32_t invert_amortization;    /* scheduler.py:43, :233: amortization weights 1/(rt*p) */
    int64_t s_star;                 /* scheduler.py:381-393 sweet spot */
    int64_t t_i_init_us;            /* engine.py:268-270 */
    /* N2/N3 KV data plane (no reference counterpart; 0 layers = off).
     * Page layout [layer][K|V][kv_head][slot][head_dim] bf16. */
    int32_t kv_layers;
    int32_t kv_heads;
    int32_t q_heads;                /* multiple of kv_heads, <= 16 per kv head */
    int32_t head_dim;               /* must be 128 */
    int64_t host_swap_pages;        /* pinned host swap pool, in pages */
    int32_t decode;                 /* run the paged decode for each step's decode members */
    int32_t decode_split;           /* tokens per split-KV work item */
    /* planner (scheduler.py:30 POLICIES; plan_batch dispatch :939-950) */
    int32_t policy;                 /* CO_POLICY_* */
    int32_t vllm_block_tokens;      /* scheduler.py:45 */
    int32_t s3_bucket_tokens;       /* scheduler.py:46 */
    int32_t rlp_padding;            /* scheduler.py:47 */
} co_config;

enum { CO_POLICY_CACHEOPT = 0, CO_POLICY_VLLM_BLOCK = 1, CO_POLICY_SARATHI_CHUNKED = 2, CO_POLICY_RLP = 3,
       CO_POLICY_S3 = 4 };

/* One trace, any order (the library sorts by (arrival_us, id) like
 * engine.py:241).  err_draw/flip_draw are the predictor noise draws of
 * estimation.py:76-99 in (arrival, id) order, i.e. aligned with the SORTED
 * order; the host produces them from numpy's default_rng([seed, 3]) stream
 * exactly as engine.py:267/348 consumes it. */
typedef struct co_trace {
    int64_t n;
    const int64_t* req_id;
    const int64_t* arrival_us;
    const int32_t* prompt_len;
    const int32_t* true_output_len;
    const int64_t* slo_ttft_us;
    const int64_t* slo_tbt_us;
    const int32_t* err_draw;        /* sorted order */
    const uint8_t* flip_draw;       /* sorted order */
} co_trace;

/* Host-evaluated integer lookup tables over sequence length S in [0, s_max]
 * (index 0 unused): the float cost models of costmodel.py:58-69 /
 * preemption.py:94-116 rounded exactly as the reference rounds them. */
typedef struct co_luts {
    int64_t s_max;
    const int64_t* swap_half_us;    /* to_us(swap_latency(S)/2)      engine.py:372,392 */
    const int64_t* recompute_us;    /* to_us(recompute_latency(S))   engine.py:395-397 */
    const int64_t* survive_swap_us; /* int(L_s(S)*1000+0.5)          scheduler.py:368-374 */
    const int64_t* survive_rec_us;  /* int(L_r(S)*1000+0.5)          scheduler.py:368-374 */
} co_luts;

/* Engine-level scalars (engine.py:243-270 state), read back after a step. */
typedef struct co_scalars {
    int64_t now_us;
    int64_t horizon_us;
    int64_t first_arrival_us;
    int64_t t_i_max_us;
    int64_t footprint_tokens;       /* kvc.py:101 */
    int64_t granted_tokens;         /* kvc.py:105 */
    int64_t used_tokens;            /* kvc.py:109 */
    int64_t generated_total;
    int64_t iterations;
    int64_t steps;
    int64_t record_seq;
    int64_t n_events;               /* undrained events on the device */
    int64_t n_samples;
    int64_t decisions;              /* sum over steps of live requests (BASELINE.md unit) */
    int32_t reserved_blocks_current;/* kvc.py:79 */
    int32_t n_live;
    int32_t n_pending;
    int32_t done;
    int32_t stalled;
    int32_t last_step_result;       /* return value of engine.py:606 step() */
    int32_t error;
    int32_t _pad0;
} co_scalars;

/* Fixed-size event record; host turns it into the reference dict. */
typedef struct co_event {
    int32_t kind;
    int32_t idx;        /* request index (sorted order); ITER: member count */
    int64_t t;
    int64_t a;          /* ITER: end; PREEMPT: kv; READMIT: ready_at */
    int64_t b;          /* ITER: tokens; PREEMPT: strategy */
    int64_t c;          /* ITER: offset into the member stream; PREEMPT: cause */
} co_event;

/* Per-request state readback (sorted order), field by field. */
typedef enum co_field {
    CO_F_STATE = 0, CO_F_GENERATED, CO_F_USED, CO_F_KV_NEED, CO_F_PREFILL_DONE,
    CO_F_PREEMPTION_COUNT, CO_F_PREEMPTION_TIME, CO_F_FIRST_TOKEN, CO_F_LAST_TOKEN,
    CO_F_MAX_TBT, CO_F_READY_AT, CO_F_PREEMPT_STARTED, CO_F_SWAP_OUT_DONE,
    CO_F_LAST_STRATEGY, CO_F_FIRST_START, CO_F_COMPLETION, CO_F_ALLOCATED_KVC,
    CO_F_PREDICTED, CO_F_ESTIMATED, CO_F_HOLDS, CO_F_GRANTED, CO_F_HOST,
    CO_F_EMBED_OFFSET, CO_F_RESERVED_DRAWN, CO_F_RECORD_SEQ, CO_F_CLAIM_WAITER,
    CO_F_SORTED_ORDER, CO_F_COUNT
} co_field;

typedef struct co_engine co_engine;

/* engine.py:225-271 Engine.__init__ (plus the host-derived constants).
 * device < 0 keeps the current device. */
int co_create(const co_config* cfg, const co_trace* trace, const co_luts* luts,
              int device, co_engine** out);
/* releases every device/pinned buffer of the instance */
int co_destroy(co_engine* eng);

/* engine.py:606-641 Engine.step(): one scheduling round on the device.
 * *result receives step()'s boolean. */
int co_step(co_engine* eng, int32_t* result);

/* step() with the iteration's result in the same call and one device sync:
 * *result = step()'s bool, members = the (idx, tokens) pairs that ran this
 * iteration (engine.py:630-633 `members`), *iter_end_us its end time (-1 when
 * the step idled).  The members are written by the device straight into
 * mapped pinned host memory. */
int co_step_result(co_engine* eng, int32_t* result, int32_t* members, int64_t max_members,
                   int64_t* n_members, int64_t* iter_end_us);

/* allocates step_result's mapped result buffer and instantiates the
 * single-step graph without running a step (so a timed loop of
 * co_step_result calls starts warm). */
int co_prepare_step(co_engine* eng);

/* engine.py:643-661 Engine.run() loop including the no-progress guard,
 * executed as CUDA-graph launches of `steps_per_launch` device steps.
 * max_steps <= 0 means until done.  *steps_done = step() calls made. */
int co_run(co_engine* eng, int64_t max_steps, int32_t steps_per_launch, int64_t* steps_done);

/* engine.py:360-384 Engine._preempt(rid, strategy, now, cause) on the device
 * (white-box hook used by the reference's own engine tests). */
int co_preempt(co_engine* eng, int64_t idx, int32_t strategy, int64_t now_us, int32_t cause);

/* Blocking readbacks into caller-owned host buffers. */
int co_get_scalars(co_engine* eng, co_scalars* out);
int co_read_field(co_engine* eng, int32_t field, int64_t* out /* n values */);
/* co_step_result followed by co_drain_log in one call (the per-step API with
 * the step's event log taken along; CO_EAGAIN as co_drain_log when the log
 * buffers are too small -- the step has run, drain again with larger ones). */
int co_step_result_log(co_engine* eng, int32_t* result, int32_t* members, int64_t max_members,
                       int64_t* n_members, int64_t* iter_end_us, co_event* events, int64_t max_events,
                       int32_t* log_members, int64_t max_log_members, int64_t* samples, int64_t max_samples,
                       int64_t* counts);
/* The same with every argument in one caller-owned struct (filled once and
 * reused: a binding then passes a single pointer per step). */
typedef struct co_step_args {
    co_engine* eng;
    int32_t* result;
    int32_t* members;
    int64_t max_members;
    int64_t* n_members;
    int64_t* iter_end_us;
    co_event* events;
    int64_t max_events;
    int32_t* log_members;
    int64_t max_log_members;
    int64_t* samples;
    int64_t max_samples;
    int64_t* counts;
    int32_t drain;  /* 0: co_step_result, 1: co_step_result_log */
    int32_t _pad;
    /* optional: with both set, the iteration's members are also written as
     * (ids[idx], tokens) int64 pairs (the caller's request ids by sorted
     * position), max_members pairs at most; members may then be NULL */
    const int64_t* ids;
    int64_t* members_ids;
} co_step_args;
int co_step_packed(const co_step_args* args);
/* Undrained append-log sizes in one call: out[0] events, out[1] iteration
 * members, out[2] utilization samples (the counts co_pending_events and
 * co_get_scalars' n_samples report). */
int co_pending_log(co_engine* eng, int64_t* out /* 3 */);
/* Drains up to max_events events (and their iter member streams) into the
 * caller's buffers; returns counts.  members: (idx, tokens) int32 pairs. */
int co_drain_events(co_engine* eng, co_event* events, int64_t max_events,
                    int32_t* members, int64_t max_members,
                    int64_t* n_events, int64_t* n_members);
int co_pending_events(co_engine* eng, int64_t* n_events, int64_t* n_members);
/* The whole append log in one call: events (+ their iteration members) and
 * utilization samples.  counts[3] = {events, members, samples} drained; if a
 * buffer is too small nothing is drained, counts holds the sizes needed and
 * the return is CO_EAGAIN. */
int co_drain_log(co_engine* eng, co_event* events, int64_t max_events, int32_t* members, int64_t max_members,
                 int64_t* samples, int64_t max_samples, int64_t* counts);
/* per-iteration (footprint, used) samples (engine.py:636), drained */
int co_drain_samples(co_engine* eng, int64_t* out /* 2 per sample */, int64_t max, int64_t* n);
/* token timestamps: offsets[n+1] and the Σ true_output_len slab; callers
 * use generated[i] to know how many entries of request i are valid. */
int co_read_token_times(co_engine* eng, int64_t* offsets, int64_t* times);
/* N1 physical block tables (no reference counterpart):
 * lens[n] pages per request (sorted order), their page ids concatenated in
 * request order into pages[], and the free stack bottom..top. */
int co_read_block_tables(co_engine* eng, int32_t* lens, int32_t* pages, int64_t max_pages,
                         int32_t* free_pages, int32_t* n_free);
/* N2/N3 data plane readbacks (CO_EINVAL when the data plane is off):
 * stats[8] = {swap-out bytes, swap-in bytes, fill bytes, move bytes,
 *             decode steps, decode member-steps, decode context tokens, 0} */
int co_data_stats(co_engine* eng, int64_t* stats);
/* counts KV elements of every holder's tokens [0, used) that differ from the
 * synthetic content (0 = the data path never lost or misplaced a byte) */
/* plan_batch(PlannerInputs, cfg) (scheduler.py:939-950) on a snapshot: the
 * engine must have been created over the snapshot's requests (sorted order)
 * without data plane or communicator.  cols [n][20] per request (sorted order):
 * state, generated, used, kv_need, prefill_done, preemption_count, predicted,
 * estimated, first_token_us (-1 = none), last_token_us, max_tbt_us, ready_at_us,
 * holds, granted, host (index or -1), embed_offset, reserved_drawn, first guest,
 * next guest, record creation seq; scal[8] = {now, t_i_max, reserved_current,
 * footprint_sum, granted_sum, used_sum, record seq, live count}.  hdr[8] =
 * {members, actions, preempt, claims, deferred, overflow, batch_tokens, active};
 * lists = members (idx[], tokens[]), actions (kind[], idx[], tokens[], blocks[],
 * host[], start[]), preempt (idx[], strategy[]), claims (waiter[], provider[]),
 * deferred (idx[]) -- each array of its count, concatenated. */
int co_plan_snapshot(co_engine* eng, const int64_t* cols, const int64_t* scal, int64_t* hdr, int32_t* lists,
                     int64_t cap);
/* Split swap I/O totals (k_swapio, the host-link half of swap-out/in, run on
 * a side stream beside the decode): out[6] = {bytes to host, bytes from host,
 * device ns from its first CTA in to its last CTA out, summed over launches,
 * launches that moved data, split on (0 = copies inside k_data), CTAs}. */
int co_swap_io_stats(co_engine* eng, int64_t* out);
int co_kv_verify(co_engine* eng, int64_t* mismatches, int64_t* checked);
/* the last step's paged-decode outputs: member indices (sorted order),
 * context lengths, and out[member][layer][q_head][head_dim] fp32 */
int co_read_decode(co_engine* eng, int32_t* members, int32_t* ctx, float* out, int64_t max_members,
                   int64_t* n_members, int64_t* step_id);
/* turn the per-step decode on/off at run time (configured with decode = 1) */
int co_set_decode(co_engine* eng, int32_t on);
/* swap micro-benchmark: one gather (HBM pages -> pinned host) and one scatter
 * (back) of ntok tokens through the engine's own data kernel; mean device
 * ms of each over `iters` rounds.  Clobbers KV contents. */
int co_swap_bench(co_engine* eng, int64_t ntok, int32_t iters, double* out_ms, double* in_ms);
/* N4 (no reference counterpart; kvc.py:76-79 is one instance): a 128-byte
 * ncclUniqueId for rank 0 to broadcast, and attaching the instance to an
 * NCCL communicator, after which every step all-reduces (sum) the instance's
 * [free_tokens, reserved_blocks_current] on a side stream captured into the
 * step graph.  Telemetry only: decisions never read it, so each instance stays
 * bit-exact against its own CPU reference.  Every rank must then launch the
 * same number of steps (co_run requires max_steps > 0). */
int co_nccl_unique_id(uint8_t* out /* 128 bytes */);
int co_attach_nccl(co_engine* eng, const uint8_t* uid, int32_t nranks, int32_t rank);
/* last all-reduced totals {free_tokens, reserved_blocks_current} and how
 * many all-reduces were enqueued */
int co_global_reserve(co_engine* eng, int64_t* out /* 2 */, int64_t* calls);
/* pinned-memory cudaMemcpyAsync bandwidth of this GPU's host link (GB/s) */
int co_host_link_gbs(int64_t bytes, double* d2h, double* h2d);
/* kvc.py:336-375 BlockPool.check_invariants on the device; CO_EDEVICE on
 * a violation with the reason in co_last_error(). */
int co_check_invariants(co_engine* eng);

/* Device time of the last co_run/co_step launch sequence (CUDA events on
 * the engine stream), milliseconds.  co_step / co_step_result record their
 * per-step events only after the first call of this function (the events
 * cost a few microseconds of every step otherwise). */
int co_last_device_ms(co_engine* eng, double* ms);
/* development aid: phase timestamps (ns) of the planner/apply kernels of
 * the last step; enable = 1 allocates the stamp buffer */
int co_phase_profile(co_engine* eng, int32_t enable, int64_t* out /* 64 */);
/* Number of kernels one device step launches (for gpu_launches accounting). */
int co_kernels_per_step(co_engine* eng, int32_t* n);

/* Benchmark helper: runs k engine steps (run() semantics) as one CUDA graph
 * with CUDA events between the stages of every step, optionally preceded per
 * step by an L2 flush (a memset of flush_bytes), and returns the device time
 * of each step (step_ms[k], flush excluded) and the summed device time of
 * each stage over the k steps (stage_ms[CO_NSTAGES]).  Stages: begin+admit,
 * classify, bucket, plan, apply, check, data (N2 moves + KV fills), decode (N3).
 * stage_ms may be NULL: then only the step boundaries carry events, and the
 * step kernels chain through programmatic-dependent-launch edges. */
#define CO_NSTAGES 8
int co_time_steps(co_engine* eng, int32_t k, int64_t flush_bytes, double* step_ms, double* stage_ms);

/* engine.py:132-211 compute_metrics on the device: counts,
 * exact integer sums, numpy-pairwise sum of the normalized latencies in the
 * caller's request order, and the order statistics the percentiles
 * interpolate between (np.percentile 'linear': ranks floor/ceil of
 * (count-1)*q for q = .50/.90/.99, and the max), per list: 0 TTFT and 2
 * normalized latency of completed requests, 1 every inter-token gap of
 * completed requests, 3 preemption time of preempted requests. */
typedef struct co_metrics_raw {
    int64_t completed, ok_ttft, ok_tbt, generated, preemption_total, preempted;
    int64_t sum_ttft, sum_gap, sum_wait, sum_exec, sum_pdec, sum_ptime;
    int64_t count[4];
    double norm_sum;
    double order_stat[4][7]; /* p50 lo, p50 hi, p90 lo, p90 hi, p99 lo, p99 hi, max */
} co_metrics_raw;
int co_metrics(co_engine* eng, co_metrics_raw* out);

/* ---- the run's random streams on the device --------------
 * Bit-exact device versions of the reference's numpy draws (default_rng
 * ([seed, k]) = SeedSequence + PCG64, numpy's ziggurat exponential / normal,
 * uniform, Lemire bounded integers).  Output pointers are DEVICE pointers on
 * `device` (< 0: current device); every call is synchronous. */

/* default_rng(entropy) -> PCG64 (state_hi, state_lo, inc_hi, inc_lo) */
int co_pcg64_seed(const uint64_t* entropy, int32_t n_entropy, uint64_t out[4]);
/* the first `count` raw 64-bit outputs of default_rng([seed, stream]) */
int co_gen_raw(uint64_t seed, uint64_t stream, int64_t count, int device, uint64_t* out);
/* n draws of default_rng([seed, stream]).standard_exponential (kind 0) or
 * .standard_normal (kind 1) */
int co_gen_std(int32_t kind, uint64_t seed, uint64_t stream, int64_t n, int device, double* out);

/* workload.py:85-109 generate(spec, seed): arrivals from exponential gaps of
 * default_rng([seed, 0]), prompt / output lengths from the lognormals of
 * default_rng([seed, 1]) / ([seed, 2]), clipped.  mu / sigma are the host's
 * _lognormal_params (workload.py:79-82); gap_scale = 1.0 / arrival_rate. */
typedef struct co_trace_spec {
    int64_t n;
    double gap_scale;
    double mu_in, sigma_in;
    double mu_out, sigma_out;
    int32_t input_min, input_max;
    int32_t output_min, output_max;
} co_trace_spec;
int co_gen_trace(const co_trace_spec* spec, uint64_t seed, int device, int64_t* arrival_us, int32_t* prompt_len,
                 int32_t* output_len);

/* workload.py:181-194 assign_slos(requests, base_ttft, base_tbt, policy, seed) */
typedef struct co_slo_spec {
    int64_t base_ttft_us, base_tbt_us;
    double scale_lo, scale_hi;
    int32_t chunk_budget;
    int32_t _pad;
} co_slo_spec;
int co_gen_slos(int64_t n, const int32_t* prompt_len /* device */, const co_slo_spec* spec, uint64_t seed,
                int device, int64_t* slo_ttft_us, int64_t* slo_tbt_us);

/* estimation.py:76-99 predictor draws for n arrivals in admission order from
 * default_rng([seed, 3]) (engine.py:267): err = _sample_error, flip = the
 * direction-flip test (1 - direction_accuracy). */
enum { CO_ERR_ZERO = 0, CO_ERR_UNIFORM = 1, CO_ERR_NORMAL = 2 };
typedef struct co_predictor_spec {
    int32_t error_dist;
    int32_t _pad;
    double error_scale;
    double direction_accuracy;
} co_predictor_spec;
int co_gen_predictor(int64_t n, const co_predictor_spec* spec, uint64_t seed, int device, int32_t* err_draw,
                     uint8_t* flip_draw);

const char* co_last_error(void);
const char* co_version(void);

/* ---- kvc.BlockPool on the device (kvc.py:55-375) ---------------------------
 * A standalone record table in HBM driven by the engine's own pool functions
 * (csrc/pool_api.cuh); records are addressed by slot (the host maps request
 * ids to slots).  co_pool_op: op = CO_POOL_*, a/b/c as listed; out[3]:
 * out[0] > 0 Grant(out[1] tokens, out[2] footprint) or release's net tokens
 * in out[1]; out[0] == 0 Shortfall(missing = out[1]); out[0] < 0 the
 * contract violation -CO_PV_* (the reference's ValueError). */
typedef struct co_pool co_pool;
enum { CO_POOL_ALLOCATE = 0,        /* a = n_tokens                       kvc.py:156 */
       CO_POOL_EMBED = 1,           /* a = n_tokens, b = host slot, c = start_offset  :202 */
       CO_POOL_DRAW_RESERVED = 2,   /* a = n_blocks                       :229 */
       CO_POOL_GROW = 3,            /* a = n_tokens                       :251 */
       CO_POOL_PROMOTE = 4,         /*                                    :283 */
       CO_POOL_RELEASE = 5,         /* out[1] = net tokens returned       :299 */
       CO_POOL_SET_USED = 6,        /* a = used_tokens                    :326 */
       CO_POOL_NET_RELEASE_GAIN = 7 /* out[1]                             :142 */ };
enum { CO_PV_TOKENS = 1,            /* "n_tokens must be >= 1" */
       CO_PV_HOLDS = 2,             /* "request {id} already holds an allocation" */
       CO_PV_NO_RECORD = 3,         /* "no allocation for request {id}" */
       CO_PV_NO_RECORD_HOST = 4,    /* "no allocation for request {host}" */
       CO_PV_HOST_EMBEDDED = 5,     /* "host {host} is itself embedded" */
       CO_PV_SELF_HOST = 6,         /* "a request cannot host itself" */
       CO_PV_HAS_GUEST = 7,         /* "host {host} already has a guest" */
       CO_PV_EMBED_RANGE = 8,       /* "embed region exceeds host allocation" */
       CO_PV_EMBED_OVERLAP = 9,     /* "embed region overlaps an existing guest" */
       CO_PV_BLOCKS = 10,           /* "n_blocks must be >= 1" */
       CO_PV_GUEST_RESERVE = 11,    /* "guests cannot draw from the reserve" */
       CO_PV_NOT_EMBEDDED = 12,     /* "request {id} is not embedded" */
       CO_PV_USED_RANGE = 13        /* "request {id}: used {u} outside [0, {granted}]" (out[1] = granted) */ };
int co_pool_create(int64_t capacity, int32_t block_size, int32_t reserved_blocks, int32_t buffer_b,
                   int32_t allow_stacking, int32_t max_records, int32_t device, co_pool** out);
int co_pool_destroy(co_pool* pool);
int co_pool_op(co_pool* pool, int32_t op, int32_t slot, int64_t a, int64_t b, int64_t c, int64_t* out /* 3 */);
/* kvc.py:169-200: triples[4n] = (host slot or -1, request id, allocated a_j,
 * used u_j); out[4] = {found, host slot, start_offset, feasible_slack} */
int co_pool_find_host(co_pool* pool, int32_t n, const int64_t* triples, int64_t cand_prompt, int64_t cand_out,
                      int64_t buffer_b, int64_t* out);
/* scalars[6] = {free, footprint, granted, used, reserved_current, free pages};
 * records (optional) [max_records][9] = {holds, granted, host slot, offset,
 * reserved drawn, first guest slot, next guest slot, used, creation seq} */
int co_pool_state(co_pool* pool, int64_t* scalars, int64_t* records);
int co_pool_check(co_pool* pool);  /* kvc.py:336-375 + N1 page conservation */
int co_pool_read_tables(co_pool* pool, int32_t* lens, int32_t* pages, int64_t max_pages, int32_t* free_pages,
                        int32_t* n_free);

/* ---- the reference's pure scheduling ops on the device -------------------
 * (scheduler.py:129-279, preemption.py:46-75) through the planner's own
 * device code (csrc/sched_ops.cuh).  rows: int64 [n][8]; column 0 is always
 * the row's rank in ascending req_id order (the ids' tie-break).
 *   CLASSIFY           rows (rank, list 0 waiting / 1 running, rt, returned, arrival)
 *                      params (t_i_max_us, epsilon_us); out = 4 counts, then the
 *                      row indices of n_w, n_r, n_w', n_r' in the reference's order
 *   FILL_BUDGET        rows (chunk); params (token_budget, consumed); out (k, overflow)
 *   ALLOCATE_REMAINING rows (rank, m_tokens, rt_us, prompt_len), n <= 1024;
 *                      params (a_prime, invert: scheduler.py:212/:233 weights 1/(rt*p));
 *                      out[k] = grant, -1 for m_tokens <= 0
 *   PAIR_RELEASE       rows (rank, est_remaining_iters, release_gain);
 *                      params (residual_tokens, runway_iters); out[0] = row or -1
 *   ORDER_VICTIMS      rows (rank, slo_tbt_us, remaining_tokens, occupancy);
 *                      params (token_step, n_edges <= 6, edges...); out = order
 *   PROACTIVE_INCLUDE  rows (rank, returned, allocated, target_alloc, est_remaining);
 *                      params (m); out = count, then the rows in order
 * out holds 2n + 8 values. */
enum { CO_SOP_CLASSIFY = 0, CO_SOP_FILL_BUDGET = 1, CO_SOP_ALLOCATE_REMAINING = 2, CO_SOP_PAIR_RELEASE = 3,
       CO_SOP_ORDER_VICTIMS = 4, CO_SOP_PROACTIVE_INCLUDE = 5 };
int co_sched_op(int32_t op, int32_t n, const int64_t* rows, const int64_t* params /* 16 */, int64_t* out,
                int32_t device);

#ifdef __cplusplus
}
#endif
#endif /* CACHEOPT_H */
