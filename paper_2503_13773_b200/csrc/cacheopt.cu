// libcacheopt: the B200-native CacheOPT engine behind the C ABI of
// include/cacheopt.h.  One translation unit so every device helper inlines.
//
// Per engine step the stream runs:
//   k_classify (grid: the step's begin evaluated per CTA, admission, views, classes,
//   block-ordered running/blown lists, the N'_w candidate head) -> k_serial
//   (1 CTA x 256: the planner, then plan application + the rest of the step,
//   gated invariant check inside) [-> NCCL reserve all-reduce
//   on a side stream] [-> k_data -> k_decode_tc05 + k_decode_reduce]
// co_run captures `steps_per_launch` steps into one CUDA graph and relaunches
// it; every kernel early-exits once the device control block says the run is
// done or paused (an append buffer needs draining), so no host round trip is
// needed inside a launch.
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>
#include <dlfcn.h>

#include <algorithm>
#include <type_traits>
#include <climits>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>
#include <map>
#include <mutex>

#include "engine_state.cuh"
#include "block_ops.cuh"
#include "pool_ops.cuh"
#include "grid_kernels.cuh"
#include "planner.cuh"
#include "apply.cuh"
#include "data_plane.cuh"
#include "decode_tc05.cuh"
#include "metrics.cuh"
#include "trace_gen.cuh"
#include <cudaTypedefs.h>

using namespace co;

static thread_local std::string g_err;

// NCCL is resolved at first use (N4 only), never at load time: a process that
// loads this library before torch must still get torch's own libnccl
// (dlopen of the soname returns an already-loaded copy).
struct NcclApi {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
    bool ok = false;
};
static NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(h, "ncclCommInitRank"));
        a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(h, "ncclAllReduce"));
        a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.errorString = reinterpret_cast<decltype(a.errorString)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.getUniqueId && a.commInitRank && a.allReduce && a.commDestroy && a.errorString;
        return a;
    }();
    return api;
}

// NVTX ranges around the C-ABI entry points (header-only nvtx3: a no-op
// unless a profiler is attached), so an nsys/ncu timeline shows which host
// call issued which kernels
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
#define CO_RANGE(name) NvtxRange nvtx_range_(name)

static int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess)                                                             \
            return fail(CO_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));         \
    } while (0)

__global__ void k_preempt_one(Dev d, int32_t i, int32_t strat, int64_t now, int32_t cause) {
    if (threadIdx.x == 0 && blockIdx.x == 0) do_preempt(d, i, strat, now, cause);
}
__global__ void k_reset_drained(Dev d, int64_t ev, int64_t mem, int64_t smp) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        d.ctl->ev_count -= ev;
        d.ctl->mem_count -= mem;
        d.ctl->sample_count -= smp;
        d.ctl->paused = 0;
    }
}

// The step graph's last kernel copies the control block and the (undrained)
// append log into mapped pinned memory, so after a step() the host can serve
// scalars, events, members and samples with no further device round trip.
constexpr int MIR_EV = 256, MIR_MEM = 4096, MIR_S = 64;
struct LogMirror {
    Ctl ctl;
    co_event ev[MIR_EV];
    int32_t mem[2 * MIR_MEM];
    int64_t smp[2 * MIR_S];
    volatile uint64_t seq;  // written last: the host's completion flag for a step() launch
};

__device__ __forceinline__ void mirror_body(const Dev& d, LogMirror* m) {
    const Ctl& c = *d.ctl;
    const uint64_t seq = c.mir_seq + 1;
    if (threadIdx.x == 0) {
        m->ctl = c;
        m->ctl.mir_seq = seq;
    }
    const int64_t ne = c.ev_count, nm = c.mem_count, ns = c.sample_count;
    if (ne <= MIR_EV && nm <= MIR_MEM && ns <= MIR_S) {  // else the host drains the slow way
        for (int64_t k = threadIdx.x; k < ne; k += blockDim.x) m->ev[k] = d.events[k];
        for (int64_t k = threadIdx.x; k < 2 * nm; k += blockDim.x) m->mem[k] = d.members[k];
        for (int64_t k = threadIdx.x; k < 2 * ns; k += blockDim.x) m->smp[k] = d.samples[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        d.ctl->mir_seq = seq;
        __threadfence_system();  // the mirror's bytes reach host memory before the flag
        m->seq = seq;
    }
}

// The step's single-CTA part: MODE 0 = planner only, 1 = apply only (the
// per-stage timing replay), 2 = planner then apply in one launch; then, when
// `mir` is set (the step() graph), the control block and the append log into
// mapped pinned memory.
// `pack` (a communicator is attached): N4's send slot for this step, filled
// with the instance's [free_tokens, reserved_blocks_current] (kvc.py:92-98,
// :79) after apply, every step whether or not it ran.
template <int MODE, int PLAN = PLAN_CACHEOPT>
__global__ void __launch_bounds__(NT, 1) k_serial(Dev d, LogMirror* mir, int64_t* pack, int32_t guard,
                                                  int32_t reset) {
    pdl_enter();
    extern __shared__ __align__(16) uint8_t serial_smem[];
    if (MODE != 1) {  // the step's begin (engine.py:606-614), evaluated read-only by k_classify
        if (threadIdx.x == 0) begin_commit(d, guard, reset);
        __syncthreads();
    }
    if (d.ctl->active) {
        if (MODE != 1) plan_body<PLAN>(d, *reinterpret_cast<PlanSh*>(serial_smem));
        if (MODE == 2) __syncthreads();
        if (MODE != 0) apply_body(d, *reinterpret_cast<ApplySh*>(serial_smem));
    }
    if (MODE != 0) {
        __syncthreads();
        if (threadIdx.x == 0) classify_counters_reset(d);  // for the next step's k_classify
    }
    if (mir || (pack && MODE != 0)) __syncthreads();
    if (pack && MODE != 0 && threadIdx.x == 0) {
        pack[0] = free_tokens(d);
        pack[1] = d.ctl->rsv_cur;
    }
    if (mir) mirror_body(d, mir);
}

// the k_serial instantiation for a planning MODE (0 = plan only, 2 = plan +
// apply) and the engine's planner configuration
using SerialKernel = void (*)(Dev, LogMirror*, int64_t*, int32_t, int32_t);
static SerialKernel serial_kernel(int mode, const Dev& d) {
    const int plan = d.policy != CO_POLICY_CACHEOPT ? PLAN_BASELINES : d.inv ? PLAN_INVERTED : PLAN_CACHEOPT;
    if (mode == 0)
        return plan == PLAN_BASELINES ? k_serial<0, PLAN_BASELINES>
             : plan == PLAN_INVERTED  ? k_serial<0, PLAN_INVERTED> : k_serial<0, PLAN_CACHEOPT>;
    return plan == PLAN_BASELINES ? k_serial<2, PLAN_BASELINES>
         : plan == PLAN_INVERTED  ? k_serial<2, PLAN_INVERTED> : k_serial<2, PLAN_CACHEOPT>;
}

struct co_engine {
    Dev d{};
    int device = 0;
    cudaStream_t stream = nullptr;
    std::vector<void*> allocs;
    Ctl* h_ctl = nullptr;  // pinned mirror
    cudaGraphExec_t graph = nullptr;
    int32_t graph_k = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    double last_ms = 0.0;
    bool timing = false;  // per-step events for co_last_device_ms (on after its first call)
    int grid = 1;
    int64_t n = 0;
    int64_t tok_total = 0;
    std::vector<int64_t> perm;         // sorted position -> caller position
    std::vector<int64_t> tok_off_host;
    int64_t n_chunks = 0;
    int sms = 148;
    int plan_threads = NT;  // CTA size of the single-CTA planner / apply kernels (256 measured best)
    void* host_pool = nullptr;
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join[2] = {nullptr, nullptr};
    cudaStream_t io = nullptr;                           // split swap I/O (k_swapio)
    cudaEvent_t io_fork = nullptr, io_join = nullptr;
    bool io_pending = false;                             // k_swapio not yet joined by the compute stream
    int64_t* red = nullptr;  // two slots of [send 2][recv 2]; step j of a sequence uses slot j & 1
    int join_pending = -1;   // slot whose all-reduce the compute stream has not joined yet
    int last_slot = 0;       // slot of the last all-reduce enqueued (co_global_reserve)
    int64_t reduce_calls = 0;
    CUtensorMap kvmap;
    cudaGraphExec_t graph1 = nullptr;   // one step, step() semantics
    cudaGraphExec_t graph1r = nullptr;  // the same, starting with an emptied append log
    LogMirror* mir = nullptr;           // mapped pinned (host view)
    uint64_t mir_expect = 0;            // mirror sequence number the next step() launch writes
    LogMirror* mir_dev = nullptr;       // its device alias
    bool ctl_fresh = false;             // h_ctl == the logical device state (no sync needed)
    bool reset_pending = false;         // log consumed from the mirror; device counts not yet reset
    int64_t pend_ev = 0, pend_mem = 0, pend_s = 0;
    void* result_host = nullptr;
    bool pdl = true;         // programmatic dependent launch between step kernels (CACHEOPT_PDL=0: off)
    bool tc_decode = false;  // tcgen05 (k_decode_tc05) when the block size tiles by 16; else CUDA cores
    int64_t page_bytes = 0;
    std::vector<co_event> st_events;   // host staging of drained device events
    std::vector<int32_t> st_members;
    std::vector<int64_t> st_samples;

    template <class T>
    int alloc(T** p, size_t count) {
        void* q = nullptr;
        size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
        cudaError_t e = cudaMalloc(&q, bytes);
        if (e != cudaSuccess) return fail(CO_ECUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
        allocs.push_back(q);
        *p = static_cast<T*>(q);
        return CO_OK;
    }
};

#define AL(ptr, cnt)                                  \
    do {                                              \
        int r_ = E->alloc(&(ptr), (size_t)(cnt));     \
        if (r_) { co_destroy(E); return r_; }         \
    } while (0)

template <class T>
static int upload(co_engine* E, T* dst, const std::vector<T>& src) {
    if (src.empty()) return CO_OK;
    CK(cudaMemcpyAsync(dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, E->stream));
    return CO_OK;
}

// ev (optional): CO_NSTAGES + 1 events recorded at the stage boundaries
static inline void mark(cudaEvent_t e, cudaStream_t s) {
    // an external event node when captured into a graph (a plain record
    // inside capture is only a dependency edge and cannot be timed)
    cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
}

// a step kernel launched with programmatic stream serialization (see pdl_enter)
template <typename... KArgs, typename... Args>
static void launch_pdl(bool pdl, void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t s,
                       Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, args...);
}

// k_data's software grid barrier needs every CTA resident at once: launch it
// cooperatively (the driver then refuses a grid that cannot be co-resident,
// instead of letting the resident CTAs spin behind a concurrent kernel)
template <typename... KArgs, typename... Args>
static void launch_coop(void (*kern)(KArgs...), int grid, int block, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, args...);
}

// N4's all-reduce runs on the side stream; with `defer` the compute stream
// joins it only at the end of the NEXT step (the totals never
// feed a decision), so a step's collective latency hides behind the next
// step.  Every sequence ends with flush_join (a capture must rejoin its fork).
static void flush_n4(co_engine* E) {
    if (E->comm && E->join_pending >= 0) cudaStreamWaitEvent(E->stream, E->join[E->join_pending], 0);
    E->join_pending = -1;
}
// The split swap I/O (k_swapio) of a step overlaps that step's decode; the
// compute stream joins it before the next step's planner/apply (which may
// preempt or release the pages it writes), or at the end of the step/sequence.
static bool flush_io(co_engine* E) {
    if (!E->io_pending) return false;
    cudaStreamWaitEvent(E->stream, E->io_join, 0);
    E->io_pending = false;
    return true;
}
static void flush_join(co_engine* E) {
    flush_n4(E);
    flush_io(E);
}

static int launch_step(co_engine* E, int32_t guard, cudaEvent_t* ev = nullptr, int32_t reset = 0,
                       LogMirror* mir = nullptr, int slot = 0, bool defer = false) {
    Dev& d = E->d;
    cudaStream_t s = E->stream;
    int64_t* pack = E->comm ? E->red + 4 * slot : nullptr;
    if (ev) mark(ev[0], s);
    if (ev) mark(ev[1], s);  // (no begin kernel: k_classify evaluates it, k_serial commits it)
    // PDL edges only between back-to-back kernels (an event node in between
    // is a full dependency anyway)
    const bool pdl = E->pdl;
    launch_pdl(pdl && !ev, k_classify, d.nblk, 256, 0, s, d, guard, reset);
    if (ev) mark(ev[2], s);
    if (ev) mark(ev[3], s);  // (no bucket stage: k_classify collects the N'_w head)
    const bool io_waited = flush_io(E);  // the previous step's swap I/O, before this apply
    if (ev) {
        launch_pdl(false, serial_kernel(0, d), 1, E->plan_threads, sizeof(PlanSh), s, d, (LogMirror*)nullptr,
                   (int64_t*)nullptr, guard, reset);
        mark(ev[4], s);
        launch_pdl(false, k_serial<1>, 1, E->plan_threads, sizeof(PlanSh), s, d, (LogMirror*)nullptr, pack,
                   guard, reset);
        mark(ev[5], s);
    } else {
        launch_pdl(pdl && !io_waited, serial_kernel(2, d), 1, E->plan_threads, sizeof(PlanSh), s, d, mir, pack,
                   guard, reset);
    }
    if (ev) mark(ev[6], s);  // (the validate_every check runs inside k_apply)
    if (E->comm) {
        // global reserve telemetry: overlaps the data plane on a side stream
        cudaEventRecord(E->fork, s);
        cudaStreamWaitEvent(E->side, E->fork, 0);
        ncclResult_t nr = nccl().allReduce(pack, pack + 2, 2, ncclInt64, ncclSum, E->comm, E->side);
        if (nr != ncclSuccess) return fail(CO_ECUDA, std::string("ncclAllReduce: ") + nccl().errorString(nr));
        cudaEventRecord(E->join[slot], E->side);
        E->last_slot = slot;
    }
    if (d.dp.on) {
        launch_coop(k_data, E->sms, 512, s, d, d.dp, d.dctl, 0);
        if (d.dp.split_io) {
            cudaEventRecord(E->io_fork, s);
            cudaStreamWaitEvent(E->io, E->io_fork, 0);
            k_swapio<<<d.dp.io_ctas, IO_T, 0, E->io>>>(d, d.dp, d.dctl);
            cudaEventRecord(E->io_join, E->io);
            E->io_pending = true;
        }
        if (ev) mark(ev[7], s);
        if (d.dp.decode_on) {
            if (E->tc_decode) {
                if (d.dp.Hq / d.dp.Hkv <= 8)
                    k_decode_tc05<8><<<E->sms, T5_THREADS, T5_SMEM, s>>>(d, d.dp, d.dctl, E->kvmap);
                else
                    k_decode_tc05<16><<<E->sms, T5_THREADS, T5_SMEM, s>>>(d, d.dp, d.dctl, E->kvmap);
            } else {
                k_decode<<<E->sms * 8, DEC_T, 0, s>>>(d, d.dp, d.dctl);
            }
            k_decode_reduce<<<E->sms * 8, RED_T, 0, s>>>(d, d.dp, d.dctl);
        }
        if (ev) mark(ev[8], s);
    } else if (ev) {
        mark(ev[7], s);
        mark(ev[8], s);
    }
    if (E->comm) {
        flush_n4(E);  // the previous step's collective (deferred) ...
        E->join_pending = slot;
        if (!defer) flush_n4(E);  // ... and this one's unless deferred to the next step
    }
    if (!defer) flush_io(E);  // (after the decode it overlapped)
    return CO_OK;
}

// device work that changes the control block is about to be enqueued
static inline void touch(co_engine* E) { E->ctl_fresh = false; }

static int apply_pending_reset(co_engine* E) {
    if (!E->reset_pending) return CO_OK;
    k_reset_drained<<<1, 1, 0, E->stream>>>(E->d, E->pend_ev, E->pend_mem, E->pend_s);
    CK(cudaGetLastError());
    E->reset_pending = false;
    return CO_OK;
}

// before enqueueing device work outside the step graphs
static int begin_work(co_engine* E) {
    touch(E);
    return apply_pending_reset(E);
}

static int sync_ctl(co_engine* E) {
    if (E->ctl_fresh) return CO_OK;
    int r = apply_pending_reset(E);
    if (r) return r;
    CK(cudaMemcpyAsync(E->h_ctl, E->d.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, E->stream));
    CK(cudaStreamSynchronize(E->stream));
    return CO_OK;
}

static void stage_log(co_engine* E, const co_event* ev, int64_t ne, const int32_t* mem, int64_t nm,
                      const int64_t* smp, int64_t ns) {
    const size_t base = E->st_events.size();
    const int64_t mbase = (int64_t)E->st_members.size() / 2;
    E->st_events.insert(E->st_events.end(), ev, ev + ne);
    for (size_t k = base; k < E->st_events.size(); k++)
        if (E->st_events[k].kind == CO_EV_ITER) E->st_events[k].c += mbase;
    E->st_members.insert(E->st_members.end(), mem, mem + 2 * nm);
    E->st_samples.insert(E->st_samples.end(), smp, smp + 2 * ns);
}

// move device append buffers into host staging and reset the device fill
static int drain_device(co_engine* E) {
    int r = sync_ctl(E);
    if (r) return r;
    Ctl& c = *E->h_ctl;
    int64_t ne = c.ev_count, nm = c.mem_count, ns = c.sample_count;
    if (ne == 0 && nm == 0 && ns == 0 && !c.paused) return CO_OK;
    if (E->ctl_fresh && E->mir && ne <= MIR_EV && nm <= MIR_MEM && ns <= MIR_S) {
        // fast path: the step graph mirrored the whole log; the device counts
        // are reset by the next step graph (graph1r) or before any other use
        stage_log(E, E->mir->ev, ne, E->mir->mem, nm, E->mir->smp, ns);
        E->pend_ev = ne; E->pend_mem = nm; E->pend_s = ns;
        E->reset_pending = true;
        c.ev_count = c.mem_count = c.sample_count = 0;
        c.paused = 0;
        return CO_OK;
    }
    touch(E);
    if (ne > 0) {
        size_t base = E->st_events.size();
        int64_t mbase = (int64_t)E->st_members.size() / 2;
        E->st_events.resize(base + ne);
        CK(cudaMemcpyAsync(E->st_events.data() + base, E->d.events, ne * sizeof(co_event), cudaMemcpyDeviceToHost,
                           E->stream));
        if (nm > 0) {
            size_t mb = E->st_members.size();
            E->st_members.resize(mb + 2 * nm);
            CK(cudaMemcpyAsync(E->st_members.data() + mb, E->d.members, 2 * nm * sizeof(int32_t),
                               cudaMemcpyDeviceToHost, E->stream));
        }
        CK(cudaStreamSynchronize(E->stream));
        for (size_t k = base; k < E->st_events.size(); k++)
            if (E->st_events[k].kind == CO_EV_ITER) E->st_events[k].c += mbase;
    }
    if (ns > 0) {
        size_t sb = E->st_samples.size();
        E->st_samples.resize(sb + 2 * ns);
        CK(cudaMemcpyAsync(E->st_samples.data() + sb, E->d.samples, 2 * ns * sizeof(int64_t), cudaMemcpyDeviceToHost,
                           E->stream));
    }
    k_reset_drained<<<1, 1, 0, E->stream>>>(E->d, ne, nm, ns);
    CK(cudaGetLastError());
    return sync_ctl(E);
}

template <class T>
static int read_arr(co_engine* E, const T* src, int64_t* out) {
    std::vector<T> h(E->n);
    if (E->n) {
        CK(cudaMemcpyAsync(h.data(), src, E->n * sizeof(T), cudaMemcpyDeviceToHost, E->stream));
        CK(cudaStreamSynchronize(E->stream));
    }
    for (int64_t k = 0; k < E->n; k++) out[k] = (int64_t)h[k];
    return CO_OK;
}

extern "C" {

const char* co_last_error(void) { return g_err.c_str(); }
int co_drain_log(co_engine* E, co_event* events, int64_t max_events, int32_t* members, int64_t max_members,
                 int64_t* samples, int64_t max_samples, int64_t* counts);
const char* co_version(void) { return "cacheopt-b200 0.1 (sm_100a)"; }

int co_destroy(co_engine* E) {
    if (!E) return CO_OK;
    if (E->graph) cudaGraphExecDestroy(E->graph);
    if (E->graph1) cudaGraphExecDestroy(E->graph1);
    if (E->graph1r) cudaGraphExecDestroy(E->graph1r);
    if (E->mir) cudaFreeHost(E->mir);
    if (E->result_host) cudaFreeHost(E->result_host);
    if (E->comm) nccl().commDestroy(E->comm);
    if (E->side) cudaStreamDestroy(E->side);
    if (E->io) { cudaStreamSynchronize(E->io); cudaStreamDestroy(E->io); }
    if (E->io_fork) cudaEventDestroy(E->io_fork);
    if (E->io_join) cudaEventDestroy(E->io_join);
    if (E->fork) cudaEventDestroy(E->fork);
    for (cudaEvent_t j : E->join)
        if (j) cudaEventDestroy(j);
    if (E->red) cudaFree(E->red);
    if (E->d.prof) cudaFree(E->d.prof);
    for (void* p : E->allocs) cudaFree(p);
    if (E->host_pool) cudaFreeHost(E->host_pool);
    if (E->h_ctl) cudaFreeHost(E->h_ctl);
    if (E->ev0) cudaEventDestroy(E->ev0);
    if (E->ev1) cudaEventDestroy(E->ev1);
    if (E->stream) cudaStreamDestroy(E->stream);
    delete E;
    return CO_OK;
}

int co_create(const co_config* cfg, const co_trace* tr, const co_luts* lu, int device, co_engine** out) {
    CO_RANGE("co_create");
    if (!cfg || !tr || !lu || !out) return fail(CO_EINVAL, "null argument");
    *out = nullptr;
    if (cfg->block_size < 1 || cfg->buffer_b < 0 || cfg->token_budget < 1 || cfg->preallocate_m < 0 ||
        cfg->decode_runway_iters < 0 || cfg->epsilon_us < 0 || cfg->token_step < 1 || cfg->capacity_tokens < 1 ||
        cfg->reserved_blocks < 0 || cfg->n_slo_edges < 0 || cfg->n_slo_edges > CO_MAX_SLO_EDGES)
        return fail(CO_EINVAL, "invalid configuration scalar");
    if ((int64_t)cfg->reserved_blocks * cfg->block_size > cfg->capacity_tokens)
        return fail(CO_EINVAL, "reserve exceeds capacity");
    if (cfg->policy < CO_POLICY_CACHEOPT || cfg->policy > CO_POLICY_S3 || cfg->vllm_block_tokens < 1 ||
        cfg->s3_bucket_tokens < 1 || cfg->rlp_padding < 0)
        return fail(CO_EINVAL, "invalid policy or policy parameter");
    if (cfg->capacity_tokens > (1ll << 30)) return fail(CO_EINVAL, "capacity_tokens too large for int32 records");
    const int64_t n = tr->n;
    if (n < 0 || n > (1ll << 30)) return fail(CO_EINVAL, "bad trace size");
    if (lu->s_max < 1) return fail(CO_EINVAL, "LUTs must cover S >= 1");
    // sorted order (engine.py:241) and uniqueness (engine.py:226-228)
    std::vector<int64_t> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    std::sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) {
        if (tr->arrival_us[a] != tr->arrival_us[b]) return tr->arrival_us[a] < tr->arrival_us[b];
        return tr->req_id[a] < tr->req_id[b];
    });
    for (int64_t k = 1; k < n; k++)
        if (tr->req_id[perm[k]] == tr->req_id[perm[k - 1]]) return fail(CO_EINVAL, "request ids must be unique");
    std::vector<int64_t> by_id(n);
    std::iota(by_id.begin(), by_id.end(), 0);
    std::sort(by_id.begin(), by_id.end(),
              [&](int64_t a, int64_t b) { return tr->req_id[perm[a]] < tr->req_id[perm[b]]; });
    std::vector<int32_t> idrank(n), rank_to_idx(n);
    for (int64_t r = 0; r < n; r++) { idrank[by_id[r]] = (int32_t)r; rank_to_idx[r] = (int32_t)by_id[r]; }
    if (std::adjacent_find(by_id.begin(), by_id.end(), [&](int64_t a, int64_t b) {
            return tr->req_id[perm[a]] == tr->req_id[perm[b]];
        }) != by_id.end())
        return fail(CO_EINVAL, "request ids must be unique");

    std::vector<int64_t> rid(n), arr(n), sttft(n), stbt(n), tok_off(n + 1, 0);
    std::vector<int32_t> prompt(n), tout(n), err(n);
    std::vector<uint8_t> flip(n);
    int64_t maxD = 0, max_tbt_slo = 0, tot_tokens = 0, max_s = 1;
    for (int64_t k = 0; k < n; k++) {
        int64_t p = perm[k];
        rid[k] = tr->req_id[p]; arr[k] = tr->arrival_us[p]; prompt[k] = tr->prompt_len[p];
        tout[k] = tr->true_output_len[p]; sttft[k] = tr->slo_ttft_us[p]; stbt[k] = tr->slo_tbt_us[p];
        err[k] = tr->err_draw[k]; flip[k] = tr->flip_draw[k];
        if (arr[k] < 0 || prompt[k] < 1 || tout[k] < 1 || sttft[k] <= 0 || stbt[k] <= 0)
            return fail(CO_EINVAL, "invalid request (core.py:59-69 rules)");
        tok_off[k + 1] = tok_off[k] + tout[k];
        maxD = std::max(maxD, arr[k] + sttft[k]);
        max_tbt_slo = std::max(max_tbt_slo, stbt[k]);
        tot_tokens += (int64_t)prompt[k] + tout[k] + 1;
        max_s = std::max<int64_t>(max_s, (int64_t)prompt[k] + tout[k]);
    }
    if (lu->s_max < max_s) return fail(CO_EINVAL, "LUTs do not cover max(prompt_len + true_output_len)");
    const int32_t n_pages = (int32_t)(cfg->capacity_tokens / cfg->block_size);
    const int32_t dir_w = (n_pages + TCHUNK - 1) / TCHUNK + 1;
    const int64_t n_chunks = (int64_t)n_pages / TCHUNK + n + 2;
    int64_t first = n ? arr[0] : 0, horizon = 0;
    if (n) {
        int64_t span = arr[n - 1] - first;
        horizon = arr[n - 1] + cfg->horizon_factor * std::max<int64_t>(span, 1000000);
    }
    // composite classify key: [class:2][flag:1][time:61-idbits][idrank:idbits]
    int idbits = 1;
    while ((1ll << idbits) < n) idbits++;
    double max_iter_ms = cfg->iter_base_ms + cfg->iter_per_token_ms * (double)tot_tokens;
    double bound = std::max((double)maxD, (double)horizon + max_iter_ms * 1000.0 + 2.0 + (double)max_tbt_slo);
    // non-blown N'_w key = deadline << idbits | id rank (unique u64)
    if (bound >= std::ldexp(1.0, 62 - idbits)) return fail(CO_EINVAL, "trace time range exceeds the key budget");
    const int key_bits = 64;

    co_engine* E = new co_engine();
    E->n = n;
    E->perm = perm;
    E->tok_off_host = tok_off;
    E->tok_total = tok_off[n];
    if (device >= 0) {
        cudaError_t e = cudaSetDevice(device);
        if (e != cudaSuccess) { delete E; return fail(CO_ECUDA, cudaGetErrorString(e)); }
    }
    cudaGetDevice(&E->device);
    if (cudaStreamCreateWithFlags(&E->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete E;
        return fail(CO_ECUDA, "stream create failed");
    }
    cudaEventCreate(&E->ev0);
    cudaEventCreate(&E->ev1);
    if (cudaMallocHost(&E->h_ctl, sizeof(Ctl)) != cudaSuccess) { co_destroy(E); return fail(CO_ECUDA, "pinned alloc"); }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, E->device);
    E->grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8));
    E->sms = sms;
    if (const char* pv = std::getenv("CACHEOPT_PDL")) E->pdl = std::atoi(pv) != 0;
    if (const char* pt = std::getenv("CACHEOPT_PLAN_THREADS")) {
        int v = std::atoi(pt);
        if (v >= 64 && v <= NT && v % 32 == 0) E->plan_threads = v;
    }

    Dev& d = E->d;
    d.n = (int32_t)n; d.bs = cfg->block_size; d.B = cfg->block_size; d.buffer_b = cfg->buffer_b;
    d.stacking = cfg->allow_stacking ? 1 : 0;
    d.token_budget = cfg->token_budget; d.prealloc_m = cfg->preallocate_m; d.runway_iters = cfg->decode_runway_iters;
    d.fcfs = cfg->victim_rule_fcfs; d.record_events = cfg->record_events; d.validate_every = cfg->validate_every;
    d.pad = cfg->padding; d.idbits = idbits; d.key_bits = key_bits; d.n_edges = cfg->n_slo_edges; d.token_step = cfg->token_step;
    d.rsv_target = cfg->reserved_blocks; d.eps = cfg->epsilon_us; d.capacity = cfg->capacity_tokens;
    d.s_star = cfg->s_star; d.s_max = lu->s_max;
    d.policy = cfg->policy; d.vbt = cfg->vllm_block_tokens; d.s3b = cfg->s3_bucket_tokens; d.rlp_pad = cfg->rlp_padding;
    d.inv = cfg->invert_amortization ? 1 : 0;
    for (int k = 0; k < CO_MAX_SLO_EDGES; k++) d.edges[k] = k < cfg->n_slo_edges ? cfg->slo_edges_us[k] : 0;
    d.base_ms = cfg->iter_base_ms; d.per_token_ms = cfg->iter_per_token_ms;
    d.ev_cap = std::max<int64_t>(1 << 16, 8 * n + 4096);
    d.mem_cap = std::max<int64_t>(1 << 16, 4 * n + 4096);
    d.sample_cap = 1 << 16;
    const int64_t n2 = 2 * n + 64, n3 = 3 * n + 64;

    int64_t *p_rid, *p_arr, *p_sttft, *p_stbt, *p_tok_off;
    int32_t *p_prompt, *p_tout, *p_idrank, *p_err;
    uint8_t* p_flip;
    int64_t *l0, *l1, *l2, *l3;
    AL(p_rid, n); AL(p_arr, n); AL(p_sttft, n); AL(p_stbt, n); AL(p_tok_off, n + 1);
    AL(p_prompt, n); AL(p_tout, n); AL(p_idrank, n); AL(p_err, n); AL(p_flip, n);
    const int64_t L = lu->s_max + 1;
    AL(l0, L); AL(l1, L); AL(l2, L); AL(l3, L);
    d.rid = p_rid; d.arr = p_arr; d.slo_ttft = p_sttft; d.slo_tbt = p_stbt; d.tok_off = p_tok_off;
    d.prompt = p_prompt; d.tout = p_tout; d.idrank = p_idrank; d.err = p_err; d.flip = p_flip;
    d.lut_swap_half = l0; d.lut_rec = l1; d.lut_surv_swap = l2; d.lut_surv_rec = l3;
    AL(d.state, n); AL(d.last_strat, n);
    AL(d.gen, n); AL(d.used, n); AL(d.kv_need, n); AL(d.prefill, n); AL(d.pcount, n); AL(d.pred, n); AL(d.est, n);
    AL(d.alloc_kvc, n);
    AL(d.first_tok, n); AL(d.last_tok, n); AL(d.max_tbt, n); AL(d.ready_at, n); AL(d.pstart, n);
    AL(d.swap_done, n); AL(d.first_start, n); AL(d.completion, n); AL(d.ptime, n);
    AL(d.tok_times, E->tok_total);
    AL(d.holds, n); AL(d.granted, n); AL(d.host, n); AL(d.off, n); AL(d.rsv, n); AL(d.guest, n); AL(d.gnext, n); AL(d.rec_seq, n);
    AL(d.claim_w, n); AL(d.claim_ep, n); AL(d.epoch, n);
    AL(d.chunk_pool, n_chunks * TCHUNK); AL(d.chunk_stack, n_chunks); AL(d.dir, (int64_t)n * dir_w);
    AL(d.tab_len, n); AL(d.free_stack, n_pages);
    d.n_pages = n_pages;
    d.dir_w = dir_w;
    E->n_chunks = n_chunks;
    AL(d.st_nr, n); AL(d.st_crit, n); AL(d.st_removed, n); AL(d.st_embedded, n); AL(d.st_resumed, n);
    AL(d.st_stalled, n); AL(d.st_parts, n); AL(d.st_claimed, n); AL(d.st_failed, n); AL(d.seen64, n);
    AL(d.st_acted, n); AL(d.st_deferred, n);
    {
        int64_t nb = std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8));
        int64_t chunk = ((n + nb - 1) / nb + 255) / 256 * 256;
        if (chunk < 256) chunk = 256;
        nb = std::max<int64_t>(1, (n + chunk - 1) / chunk);
        d.nblk = (int32_t)nb;
        d.chunk = (int32_t)chunk;
    }
    AL(d.run_tmp, n); AL(d.blown_tmp, n); AL(d.blk_cnt, 2 * d.nblk + 2); AL(d.crit_idx, n); AL(d.key0, n);
    AL(d.cand, CAND_CAP);
    AL(d.l_run, n); AL(d.l_blown, n); AL(d.l_nw, n); AL(d.l_nwp, n);
    AL(d.plan, 1);
    AL(d.mem_idx, n3); AL(d.mem_tok, n3);
    AL(d.act_kind, n3); AL(d.act_idx, n3); AL(d.act_tok, n3); AL(d.act_nb, n3); AL(d.act_host, n3); AL(d.act_start, n3);
    AL(d.pre_idx, n); AL(d.pre_strat, n); AL(d.cl_w, n2); AL(d.cl_p, n2); AL(d.def_idx, n2);
    AL(d.l_nr, n); AL(d.l_nrp, n); AL(d.l_pend, n); AL(d.l_tri, n); AL(d.l_tri_taken, n); AL(d.l_vict, n);
    AL(d.l_defer, n); AL(d.l_pro, n); AL(d.l_ful, n); AL(d.l_part, n3); AL(d.l_part_need, n3);
    AL(d.l_part_grant, n3); AL(d.l_mready, n2); AL(d.l_gm_idx, n); AL(d.l_gm_tok, n); AL(d.l_acted, n3);
    AL(d.l_surv_idx, n3); AL(d.l_surv_tok, n3); AL(d.l_done, n3); AL(d.l_coll, n); AL(d.l_grp, 2 * n3);
    AL(d.l_fill_t0, n3); AL(d.l_fill_n, n3); AL(d.l_mflag, n3);
    AL(d.views, n);
    AL(d.dctl, 1);
    std::memset(&d.dp, 0, sizeof(d.dp));
    if (cfg->kv_layers > 0) {
        DataCfg& x = d.dp;
        if (cfg->head_dim != 128) { co_destroy(E); return fail(CO_EINVAL, "head_dim must be 128"); }
        if (cfg->kv_heads < 1 || cfg->q_heads % cfg->kv_heads || cfg->q_heads / cfg->kv_heads > DEC_GMAX) {
            co_destroy(E);
            return fail(CO_EINVAL, "q_heads must be a multiple (<= 16x) of kv_heads");
        }
        int coop = 0, per_sm = 0;
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, E->device);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_data, 512, 0);
        if (!coop || per_sm < 1) {
            co_destroy(E);
            return fail(CO_ECUDA, "k_data needs a cooperative launch with one 512-thread CTA per SM");
        }
        x.on = 1;
        x.decode_on = cfg->decode;
        x.L = cfg->kv_layers; x.Hkv = cfg->kv_heads; x.Hq = cfg->q_heads; x.D = cfg->head_dim;
        x.rows = x.L * 2 * x.Hkv;
        x.page_elems = (int64_t)x.rows * cfg->block_size * x.D;
        x.split = cfg->decode_split > 0 ? cfg->decode_split : 512;
        const int64_t page_bytes = x.page_elems * 2;
        AL(x.kv, (int64_t)n_pages * x.page_elems);
        x.h_pages = (int32_t)std::max<int64_t>(cfg->host_swap_pages, 1);
        cudaError_t he = cudaHostAlloc(&E->host_pool, (size_t)x.h_pages * page_bytes, cudaHostAllocMapped);
        if (he != cudaSuccess) { co_destroy(E); return fail(CO_ECUDA, "pinned host swap pool allocation failed"); }
        void* hdev = nullptr;
        cudaHostGetDevicePointer(&hdev, E->host_pool, 0);
        x.hkv = static_cast<uint16_t*>(hdev);
        // every guest moves at most once per step and all their KV fits the
        // pool, so with stacking the whole step's MOVE group fits `capacity`
        x.group_moves = cfg->allow_stacking ? 1 : 0;
        x.stage_tokens = cfg->allow_stacking ? std::max<int64_t>(max_s, cfg->capacity_tokens) + 1 : max_s + 1;
        AL(x.stage, x.stage_tokens * x.rows * x.D);
        // split swap I/O (default on; CACHEOPT_SPLIT_IO=0 runs the host-link
        // copies inside k_data, before the decode, as round 1 did)
        x.split_io = 1;
        if (const char* sv = std::getenv("CACHEOPT_SPLIT_IO")) x.split_io = std::atoi(sv) != 0;
        x.io_ctas = 32;
        if (const char* cv = std::getenv("CACHEOPT_IO_CTAS")) x.io_ctas = std::max(1, std::atoi(cv));
        x.gstage_tokens = x.split_io ? cfg->capacity_tokens + 1 : 0;
        if (x.split_io) {
            AL(x.gstage, x.gstage_tokens * x.rows * x.D);
            if (cudaStreamCreateWithFlags(&E->io, cudaStreamNonBlocking) != cudaSuccess ||
                cudaEventCreateWithFlags(&E->io_fork, cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&E->io_join, cudaEventDisableTiming) != cudaSuccess) {
                co_destroy(E);
                return fail(CO_ECUDA, "swap I/O stream");
            }
        }
        x.op_cap = 8 * n + 4096;
        x.snap_cap = 16 * (int64_t)n_pages + 8 * n + 65536;
        AL(x.ops, x.op_cap); AL(x.snap, x.snap_cap); AL(x.hstack, x.h_pages);
        x.hdir_w = (int32_t)((max_s + cfg->block_size - 1) / cfg->block_size + 1);
        AL(x.hdir, (int64_t)n * x.hdir_w); AL(x.hsaved, n);
        x.dec_cap = (int32_t)std::min<int64_t>(n, 4096);
        x.dec_item_cap = 1 << 20;
        AL(x.dec_idx, x.dec_cap + 1); AL(x.dec_ctx, x.dec_cap + 1); AL(x.dec_item_off, x.dec_cap + 1);
        const int G = x.Hq / x.Hkv;
        if (x.decode_on) {
            AL(x.dec_part, x.dec_item_cap * G * (x.D + 2));
            AL(x.dec_out, (int64_t)x.dec_cap * x.L * x.Hq * x.D);
        }
        AL(x.gbar, 2);
        E->page_bytes = page_bytes;
        const int bs = cfg->block_size;
        if (x.decode_on && (16 % bs == 0 || bs % 16 == 0)) {
            // TMA view of the pool: [n_pages * rows * bs][128] bf16, 128B-swizzled boxes
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
                co_destroy(E);
                return fail(CO_ECUDA, "cuTensorMapEncodeTiled unavailable");
            }
            cuuint64_t gdim[2] = {(cuuint64_t)x.D, (cuuint64_t)n_pages * x.rows * bs};
            cuuint64_t gstride[1] = {(cuuint64_t)x.D * 2};
            cuuint32_t box[2] = {64, (cuuint32_t)(bs < 16 ? bs : 16)};
            cuuint32_t estride[2] = {1, 1};
            CUresult cr = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn)(
                &E->kvmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x.kv, gdim, gstride, box, estride,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (cr != CUDA_SUCCESS) { co_destroy(E); return fail(CO_ECUDA, "tensor map encode failed"); }
            cudaFuncSetAttribute(k_decode_tc05<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, T5_SMEM);
            cudaFuncSetAttribute(k_decode_tc05<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, T5_SMEM);
            E->tc_decode = true;
        }
    }
    AL(d.l_tri_key, n); AL(d.am_rhi, n3); AL(d.am_rlo, n3); AL(d.rank_to_idx, n);
    AL(d.sk0, n3); AL(d.sk1, n3); AL(d.sk2, n3); AL(d.sk_item, n3);
    if (d.inv) AL(d.big, 5 * (int64_t)INV_LIMBS);
    AL(d.events, d.ev_cap); AL(d.members, 2 * d.mem_cap); AL(d.samples, 2 * d.sample_cap);
    AL(d.ctl, 1);

    int r = 0;
    std::vector<int64_t> lut_v(L);
    auto up_lut = [&](int64_t* dst, const int64_t* src) {
        CK(cudaMemcpyAsync(dst, src, L * sizeof(int64_t), cudaMemcpyHostToDevice, E->stream));
        return CO_OK;
    };
    if ((r = upload(E, p_rid, rid)) || (r = upload(E, p_arr, arr)) || (r = upload(E, p_sttft, sttft)) ||
        (r = upload(E, p_stbt, stbt)) || (r = upload(E, p_tok_off, tok_off)) || (r = upload(E, p_prompt, prompt)) ||
        (r = upload(E, p_tout, tout)) || (r = upload(E, p_idrank, idrank)) || (r = upload(E, p_err, err)) ||
        (r = upload(E, p_flip, flip)) || (r = upload(E, d.rank_to_idx, rank_to_idx)) ||
        (r = upload(E, d.kv_need, prompt)) || (r = up_lut(l0, lu->swap_half_us)) || (r = up_lut(l1, lu->recompute_us)) ||
        (r = up_lut(l2, lu->survive_swap_us)) || (r = up_lut(l3, lu->survive_rec_us))) {
        co_destroy(E);
        return r;
    }
    auto memset_all = [&](void* p, int v, size_t bytes) { return cudaMemsetAsync(p, v, bytes, E->stream); };
    const size_t n8 = n * 8, n4 = n * 4;
    memset_all(d.state, 0, n); memset_all(d.last_strat, 0xff, n);
    for (int32_t* p : {d.gen, d.used, d.prefill, d.pcount, d.pred, d.est, d.alloc_kvc, d.granted, d.off, d.rsv,
                       d.claim_ep, d.epoch})
        memset_all(p, 0, n4);
    for (int32_t* p : {d.host, d.guest, d.gnext, d.claim_w}) memset_all(p, 0xff, n4);
    for (int32_t* p : {d.st_nr, d.st_crit, d.st_removed, d.st_embedded, d.st_resumed, d.st_stalled, d.st_parts,
                       d.st_claimed, d.st_failed, d.st_acted, d.st_deferred})
        memset_all(p, 0, n4);
    for (int64_t* p : {d.max_tbt, d.ready_at, d.pstart, d.swap_done, d.ptime, d.rec_seq}) memset_all(p, 0, n8);
    for (int64_t* p : {d.first_tok, d.last_tok, d.first_start, d.completion}) memset_all(p, 0xff, n8);
    memset_all(d.holds, 0, n);
    memset_all(d.seen64, 0, n8);
    memset_all(d.dctl, 0, sizeof(DataCtl));
    if (d.dp.on) {
        memset_all(d.dp.gbar, 0, 8);
        memset_all(d.dp.kv, 0, (size_t)d.n_pages * d.dp.page_elems * 2);
        memset_all(d.dp.hsaved, 0, n4);
        std::vector<int32_t> hs(d.dp.h_pages);
        for (int32_t k = 0; k < d.dp.h_pages; k++) hs[k] = d.dp.h_pages - 1 - k;
        if ((r = upload(E, d.dp.hstack, hs))) { co_destroy(E); return r; }
        DataCtl dc0;
        std::memset(&dc0, 0, sizeof(dc0));
        dc0.htop = d.dp.h_pages;
        dc0.decode_enabled = d.dp.decode_on;
        // on the engine stream, after the memset above (a legacy-stream copy
        // is not ordered with the non-blocking stream's async memset)
        CK(cudaMemcpyAsync(d.dctl, &dc0, sizeof(dc0), cudaMemcpyHostToDevice, E->stream));
        CK(cudaStreamSynchronize(E->stream));
    }
    memset_all(d.tab_len, 0, n4);
    {
        std::vector<int32_t> fs(n_pages);
        for (int32_t k = 0; k < n_pages; k++) fs[k] = n_pages - 1 - k;  // pop order 0, 1, 2, ...
        if ((r = upload(E, d.free_stack, fs))) { co_destroy(E); return r; }
        std::vector<int32_t> cs(n_chunks);
        for (int64_t k = 0; k < n_chunks; k++) cs[k] = (int32_t)(n_chunks - 1 - k);
        if ((r = upload(E, d.chunk_stack, cs))) { co_destroy(E); return r; }
    }
    memset_all(d.plan, 0, sizeof(PlanHdr));
    Ctl c0;
    std::memset(&c0, 0, sizeof(c0));
    c0.now = first; c0.horizon = horizon; c0.first_arrival = first; c0.t_i = cfg->t_i_init_us;
    c0.rsv_cur = cfg->reserved_blocks;
    c0.kmin = ~0ull;  // classify key range, reset after every step by k_serial
    c0.free_top = n_pages;
    c0.chunk_top = (int32_t)n_chunks;
    *E->h_ctl = c0;
    if (cudaMemcpyAsync(d.ctl, E->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, E->stream) != cudaSuccess) {
        co_destroy(E);
        return fail(CO_ECUDA, "ctl upload");
    }
    for (auto k : {serial_kernel(0, d), k_serial<1>, serial_kernel(2, d)})
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PlanSh));
    cudaError_t e = cudaStreamSynchronize(E->stream);
    if (e != cudaSuccess) { co_destroy(E); return fail(CO_ECUDA, cudaGetErrorString(e)); }
    *out = E;
    return CO_OK;
}

static int check_device_error(co_engine* E) {
    int32_t err = E->h_ctl->error;
    if (!err) return CO_OK;
    char buf[256];
    const char* what = err == 3 ? "no progress after 1000000 rounds (engine.py:653-656)"
                     : err == 4 ? "pool invariant violated (kvc.py:336-375)"
                     : err == 2 ? "set_used outside [0, granted] (kvc.py:326-332)"
                     : err == 5 ? "block table capacity exceeded"
                     : err == 6 ? "data-op log or snapshot buffer full"
                     : err == 7 ? "host swap pool exhausted (raise KVLayout.host_swap_pages)"
                     : err == 8 ? "decode work-item buffer full"
                     : err == 9 ? "more decode members than the decode output buffer holds (4096)"
                     : err == 10 ? "N'_w queue extension found no candidates"
                     : err == 11 ? "more than 32 stacked guests on one released host"
                     : err == 12 ? "invert_amortization: more live participants in one amortized group than the "
                                   "exact serial path takes (1024)"
                                : "device engine error";
    snprintf(buf, sizeof(buf), "%s [code %d, info %d %d]", what, err, E->h_ctl->err_info[0], E->h_ctl->err_info[1]);
    return fail(CO_EDEVICE, buf);
}

// Drain the append buffers before a single step when its worst case could
// overflow them, so the step never pauses (a paused-and-retried step would
// enqueue one extra all-reduce on this rank only when a communicator is attached).
static int predrain(co_engine* E) {
    const Ctl& c = *E->h_ctl;
    const int64_t need_ev = 5 * E->n + 16, need_mem = E->n + 16;
    if (c.ev_count + need_ev > E->d.ev_cap || c.mem_count + need_mem > E->d.mem_cap ||
        c.sample_count + 1 > E->d.sample_cap)
        return drain_device(E);
    return CO_OK;
}

static int ensure_step_graph(co_engine* E) {
    if (E->graph1 && E->graph1r) return CO_OK;
    if (!E->mir) {
        CK(cudaHostAlloc(&E->mir, sizeof(LogMirror), cudaHostAllocMapped));
        void* dev = nullptr;
        CK(cudaHostGetDevicePointer(&dev, E->mir, 0));
        E->mir_dev = static_cast<LogMirror*>(dev);
    }
    for (int32_t reset = 0; reset < 2; reset++) {
        cudaGraphExec_t& ge = reset ? E->graph1r : E->graph1;
        if (ge) continue;
        cudaGraph_t g;
        int r;
        CK(cudaStreamBeginCapture(E->stream, cudaStreamCaptureModeThreadLocal));
        // the control block and the step's log come back inside the graph
        // (k_serial's tail): one launch + one sync per step
        if ((r = launch_step(E, 0, nullptr, reset, E->mir_dev))) {
            flush_join(E);
            cudaStreamEndCapture(E->stream, &g);
            return r;
        }
        CK(cudaStreamEndCapture(E->stream, &g));
        CK(cudaGraphInstantiate(&ge, g, 0));
        cudaGraphDestroy(g);
    }
    return CO_OK;
}

// one step through graph1 (which ends with the mirror kernel); per-step
// device timing only once co_last_device_ms has been asked for
static int launch_step1(co_engine* E) {
    touch(E);
    if (E->timing) CK(cudaEventRecord(E->ev0, E->stream));
    CK(cudaGraphLaunch(E->reset_pending ? E->graph1r : E->graph1, E->stream));
    E->last_slot = 0;
    E->reset_pending = false;
    E->mir_expect += 1;
    if (E->comm) E->reduce_calls += 1;
    if (E->timing) CK(cudaEventRecord(E->ev1, E->stream));
    // When k_serial (whose tail writes the mirror) is the graph's last node --
    // no data plane, no collective -- the step is complete once the mapped
    // flag shows this launch's sequence number: spin on host memory instead
    // of a stream synchronize (no driver round trip).  A stuck or failed step
    // falls back to the synchronize, which reports the error.
    bool seen = false;
    if (!E->d.dp.on && !E->comm && !E->timing) {
        const auto t0 = std::chrono::steady_clock::now();
        for (uint32_t spin = 0;; spin++) {
            if (E->mir->seq == E->mir_expect) { seen = true; break; }
            if ((spin & 1023) == 1023 &&
                std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(50))
                break;
        }
        std::atomic_thread_fence(std::memory_order_acquire);
    }
    if (!seen) CK(cudaStreamSynchronize(E->stream));
    if (E->mir->seq != E->mir_expect) return fail(CO_EDEVICE, "step mirror sequence mismatch");
    std::memcpy(E->h_ctl, &E->mir->ctl, sizeof(Ctl));
    E->ctl_fresh = true;
    if (E->timing) {
        float ms = 0;
        cudaEventElapsedTime(&ms, E->ev0, E->ev1);
        E->last_ms = ms;
    }
    return CO_OK;
}

// the mapped iteration-result buffer step_result reads (graphs captured
// before it existed are dropped and recaptured with it)
static int ensure_result_buffer(co_engine* E) {
    if (E->result_host) return CO_OK;
    const int64_t cap = 3 * E->n + 64;
    CK(cudaHostAlloc(&E->result_host, (4 + 2 * cap) * sizeof(int32_t), cudaHostAllocMapped));
    void* dev = nullptr;
    CK(cudaHostGetDevicePointer(&dev, E->result_host, 0));
    E->d.result = static_cast<int32_t*>(dev);
    E->d.result_cap = cap;
    if (E->graph) { cudaGraphExecDestroy(E->graph); E->graph = nullptr; }
    if (E->graph1) { cudaGraphExecDestroy(E->graph1); E->graph1 = nullptr; }
        if (E->graph1r) { cudaGraphExecDestroy(E->graph1r); E->graph1r = nullptr; }
    return CO_OK;
}

int co_prepare_step(co_engine* E) {
    if (!E) return fail(CO_EINVAL, "null argument");
    int r = ensure_result_buffer(E);
    if (r) return r;
    return ensure_step_graph(E);
}

int co_step_result(co_engine* E, int32_t* result, int32_t* members, int64_t max_members, int64_t* n_members,
                   int64_t* iter_end_us) {
    CO_RANGE("co_step_result");
    if (!E || !result || !n_members) return fail(CO_EINVAL, "null argument");
    int r;
    if ((r = ensure_result_buffer(E))) return r;
    if ((r = ensure_step_graph(E))) return r;
    if ((r = predrain(E))) return r;
    const int32_t* res = static_cast<const int32_t*>(E->result_host);
    for (int attempt = 0; attempt < 3; attempt++) {
        if ((r = launch_step1(E))) return r;
        if ((r = check_device_error(E))) return r;
        if (E->h_ctl->paused) {
            if (E->comm) return fail(CO_EDEVICE, "step paused with a communicator attached");
            if ((r = drain_device(E))) return r;
            continue;
        }
        *result = E->h_ctl->done ? 0 : E->h_ctl->last_result;
        int64_t n = res[0] > 0 ? res[0] : 0;
        if (n > max_members) return fail(CO_EINVAL, "member buffer too small");
        if (n && members) std::memcpy(members, res + 4, 2 * n * sizeof(int32_t));
        *n_members = n;
        if (iter_end_us) *iter_end_us = n ? *reinterpret_cast<const int64_t*>(res + 2) : -1;
        return CO_OK;
    }
    return fail(CO_EDEVICE, "step could not make buffer headroom");
}

int co_step_result_log(co_engine* E, int32_t* result, int32_t* members, int64_t max_members, int64_t* n_members,
                       int64_t* iter_end_us, co_event* events, int64_t max_events, int32_t* log_members,
                       int64_t max_log_members, int64_t* samples, int64_t max_samples, int64_t* counts) {
    CO_RANGE("co_step_result_log");
    int r = co_step_result(E, result, members, max_members, n_members, iter_end_us);
    if (r) return r;
    return co_drain_log(E, events, max_events, log_members, max_log_members, samples, max_samples, counts);
}

int co_step_packed(const co_step_args* a) {
    if (!a) return fail(CO_EINVAL, "null argument");
    // the step itself; a CO_EAGAIN from the log drain still leaves the step's result valid
    const int r = !a->drain
        ? co_step_result(a->eng, a->result, a->members, a->max_members, a->n_members, a->iter_end_us)
        : co_step_result_log(a->eng, a->result, a->members, a->max_members, a->n_members, a->iter_end_us,
                             a->events, a->max_events, a->log_members, a->max_log_members, a->samples,
                             a->max_samples, a->counts);
    if ((r == CO_OK || r == CO_EAGAIN) && a->ids && a->members_ids) {
        // (req_id, tokens) pairs straight from the mapped result (valid until the next step)
        const int32_t* res = static_cast<const int32_t*>(a->eng->result_host) + 4;
        const int64_t n = *a->n_members;
        for (int64_t j = 0; j < n; j++) {
            a->members_ids[2 * j] = a->ids[res[2 * j]];
            a->members_ids[2 * j + 1] = res[2 * j + 1];
        }
    }
    return r;
}

int co_step(co_engine* E, int32_t* result) {
    CO_RANGE("co_step");
    if (!E || !result) return fail(CO_EINVAL, "null argument");
    int r = ensure_step_graph(E);
    if (r) return r;
    if ((r = predrain(E))) return r;
    for (int attempt = 0; attempt < 3; attempt++) {
        if ((r = launch_step1(E))) return r;
        if ((r = check_device_error(E))) return r;
        if (E->h_ctl->paused) {
            if (E->comm) return fail(CO_EDEVICE, "step paused with a communicator attached");
            if ((r = drain_device(E))) return r;
            continue;
        }
        *result = E->h_ctl->done ? 0 : E->h_ctl->last_result;
        return CO_OK;
    }
    return fail(CO_EDEVICE, "step could not make buffer headroom");
}

int co_run(co_engine* E, int64_t max_steps, int32_t K, int64_t* steps_done) {
    CO_RANGE("co_run");
    if (!E) return fail(CO_EINVAL, "null argument");
    { int rw_ = begin_work(E); if (rw_) return rw_; }
    if (E->comm && max_steps <= 0)
        return fail(CO_EINVAL, "with a communicator every rank must run the same fixed number of steps");
    if (K < 1) K = 1;
    int r = sync_ctl(E);
    if (r) return r;
    const int64_t steps0 = E->h_ctl->steps;
    if (E->graph && E->graph_k != K) { cudaGraphExecDestroy(E->graph); E->graph = nullptr; }
    if (!E->graph) {
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(E->stream, cudaStreamCaptureModeThreadLocal));
        for (int k = 0; k < K; k++) {
            if ((r = launch_step(E, 1, nullptr, 0, nullptr, k & 1, true))) {
                flush_join(E);
                cudaStreamEndCapture(E->stream, &g);
                return r;
            }
        }
        flush_join(E);
        CK(cudaStreamEndCapture(E->stream, &g));
        CK(cudaGraphInstantiate(&E->graph, g, 0));
        cudaGraphDestroy(g);
        E->graph_k = K;
    }
    double total_ms = 0;
    // With a communicator every rank must enqueue the same number of steps
    // (each carries one all-reduce), so progress is counted in launched steps
    // there, and in executed steps otherwise.
    int64_t launched = 0;
    while (true) {
        const int64_t done_steps = E->comm ? launched : E->h_ctl->steps - steps0;
        if (max_steps > 0 && done_steps >= max_steps) break;
        const bool single = max_steps > 0 && max_steps - done_steps < K;
        CK(cudaEventRecord(E->ev0, E->stream));
        if (single) {
            if ((r = launch_step(E, 1))) return r;
            launched += 1;
        } else {
            CK(cudaGraphLaunch(E->graph, E->stream));
            E->last_slot = (K - 1) & 1;
            launched += K;
        }
        if (E->comm) E->reduce_calls += single ? 1 : K;
        CK(cudaEventRecord(E->ev1, E->stream));
        if ((r = sync_ctl(E))) return r;
        float ms = 0;
        cudaEventElapsedTime(&ms, E->ev0, E->ev1);
        total_ms += ms;
        if ((r = check_device_error(E))) return r;
        if (E->h_ctl->paused) {
            if ((r = drain_device(E))) return r;
            continue;
        }
        if (E->h_ctl->done && !E->comm) break;
    }
    E->last_ms = total_ms;
    if (steps_done) *steps_done = E->h_ctl->steps - steps0;
    return CO_OK;
}

int co_preempt(co_engine* E, int64_t idx, int32_t strategy, int64_t now_us, int32_t cause) {
    CO_RANGE("co_preempt");
    if (!E || idx < 0 || idx >= E->n) return fail(CO_EINVAL, "bad request index");
    { int rw_ = begin_work(E); if (rw_) return rw_; }
    k_preempt_one<<<1, 1, 0, E->stream>>>(E->d, (int32_t)idx, strategy, now_us, cause);
    CK(cudaGetLastError());
    return sync_ctl(E);
}

int co_get_scalars(co_engine* E, co_scalars* o) {
    if (!E || !o) return fail(CO_EINVAL, "null argument");
    int r = sync_ctl(E);
    if (r) return r;
    const Ctl& c = *E->h_ctl;
    std::memset(o, 0, sizeof(*o));
    o->now_us = c.now; o->horizon_us = c.horizon; o->first_arrival_us = c.first_arrival; o->t_i_max_us = c.t_i;
    o->footprint_tokens = c.fp_sum; o->granted_tokens = c.granted_sum; o->used_tokens = c.used_sum;
    o->generated_total = c.gen_total; o->iterations = c.iters; o->steps = c.steps; o->record_seq = c.seq;
    o->n_events = c.ev_count + (int64_t)E->st_events.size(); o->n_samples = c.sample_count + E->st_samples.size() / 2;
    o->decisions = c.decisions;
    o->reserved_blocks_current = c.rsv_cur; o->n_live = c.n_live; o->n_pending = (int32_t)(E->n - c.next_pending);
    o->done = c.done; o->stalled = c.stalled; o->last_step_result = c.done ? 0 : c.last_result; o->error = c.error;
    return CO_OK;
}

int co_read_field(co_engine* E, int32_t f, int64_t* out) {
    if (!E || !out) return fail(CO_EINVAL, "null argument");
    Dev& d = E->d;
    switch (f) {
        case CO_F_STATE: return read_arr(E, d.state, out);
        case CO_F_GENERATED: return read_arr(E, d.gen, out);
        case CO_F_USED: return read_arr(E, d.used, out);
        case CO_F_KV_NEED: return read_arr(E, d.kv_need, out);
        case CO_F_PREFILL_DONE: return read_arr(E, d.prefill, out);
        case CO_F_PREEMPTION_COUNT: return read_arr(E, d.pcount, out);
        case CO_F_PREEMPTION_TIME: return read_arr(E, d.ptime, out);
        case CO_F_FIRST_TOKEN: return read_arr(E, d.first_tok, out);
        case CO_F_LAST_TOKEN: return read_arr(E, d.last_tok, out);
        case CO_F_MAX_TBT: return read_arr(E, d.max_tbt, out);
        case CO_F_READY_AT: return read_arr(E, d.ready_at, out);
        case CO_F_PREEMPT_STARTED: return read_arr(E, d.pstart, out);
        case CO_F_SWAP_OUT_DONE: return read_arr(E, d.swap_done, out);
        case CO_F_LAST_STRATEGY: return read_arr(E, d.last_strat, out);
        case CO_F_FIRST_START: return read_arr(E, d.first_start, out);
        case CO_F_COMPLETION: return read_arr(E, d.completion, out);
        case CO_F_ALLOCATED_KVC: return read_arr(E, d.alloc_kvc, out);
        case CO_F_PREDICTED: return read_arr(E, d.pred, out);
        case CO_F_ESTIMATED: return read_arr(E, d.est, out);
        case CO_F_HOLDS: return read_arr(E, d.holds, out);
        case CO_F_GRANTED: return read_arr(E, d.granted, out);
        case CO_F_HOST: return read_arr(E, d.host, out);
        case CO_F_EMBED_OFFSET: return read_arr(E, d.off, out);
        case CO_F_RESERVED_DRAWN: return read_arr(E, d.rsv, out);
        case CO_F_RECORD_SEQ: return read_arr(E, d.rec_seq, out);
        case CO_F_CLAIM_WAITER: {
            std::vector<int64_t> w(E->n), ep(E->n), epo(E->n);
            int r;
            if ((r = read_arr(E, d.claim_w, w.data())) || (r = read_arr(E, d.claim_ep, ep.data())) ||
                (r = read_arr(E, d.epoch, epo.data())))
                return r;
            for (int64_t k = 0; k < E->n; k++) out[k] = (w[k] >= 0 && ep[k] == epo[w[k]]) ? w[k] : -1;
            return CO_OK;
        }
        case CO_F_SORTED_ORDER:
            for (int64_t k = 0; k < E->n; k++) out[k] = E->perm[k];
            return CO_OK;
        default: return fail(CO_EINVAL, "unknown field");
    }
}

int co_pending_events(co_engine* E, int64_t* ne, int64_t* nm) {
    if (!E) return fail(CO_EINVAL, "null argument");
    int r = sync_ctl(E);
    if (r) return r;
    if (ne) *ne = (int64_t)E->st_events.size() + E->h_ctl->ev_count;
    if (nm) *nm = (int64_t)E->st_members.size() / 2 + E->h_ctl->mem_count;
    return CO_OK;
}

int co_drain_log(co_engine* E, co_event* events, int64_t max_events, int32_t* members, int64_t max_members,
                 int64_t* samples, int64_t max_samples, int64_t* counts) {
    CO_RANGE("co_drain_log");
    if (!E || !counts) return fail(CO_EINVAL, "null argument");
    int r = drain_device(E);
    if (r) return r;
    const int64_t ne = (int64_t)E->st_events.size(), nm = (int64_t)E->st_members.size() / 2,
                  ns = (int64_t)E->st_samples.size() / 2;
    counts[0] = ne; counts[1] = nm; counts[2] = ns;
    if (ne > max_events || nm > max_members || ns > max_samples) return CO_EAGAIN;  // counts = sizes needed
    if (ne) std::memcpy(events, E->st_events.data(), ne * sizeof(co_event));
    if (nm) std::memcpy(members, E->st_members.data(), 2 * nm * sizeof(int32_t));
    if (ns) std::memcpy(samples, E->st_samples.data(), 2 * ns * sizeof(int64_t));
    E->st_events.clear();
    E->st_members.clear();
    E->st_samples.clear();
    return CO_OK;
}

int co_pending_log(co_engine* E, int64_t* out) {
    if (!E || !out) return fail(CO_EINVAL, "null argument");
    int r = sync_ctl(E);
    if (r) return r;
    out[0] = (int64_t)E->st_events.size() + E->h_ctl->ev_count;
    out[1] = (int64_t)E->st_members.size() / 2 + E->h_ctl->mem_count;
    out[2] = (int64_t)E->st_samples.size() / 2 + E->h_ctl->sample_count;
    return CO_OK;
}

int co_drain_events(co_engine* E, co_event* events, int64_t max_events, int32_t* members, int64_t max_members,
                    int64_t* n_events, int64_t* n_members) {
    if (!E) return fail(CO_EINVAL, "null argument");
    int r = drain_device(E);
    if (r) return r;
    int64_t ne = (int64_t)E->st_events.size(), nm = (int64_t)E->st_members.size() / 2;
    if (ne > max_events || nm > max_members) return fail(CO_EINVAL, "drain buffers too small");
    if (ne) std::memcpy(events, E->st_events.data(), ne * sizeof(co_event));
    if (nm) std::memcpy(members, E->st_members.data(), 2 * nm * sizeof(int32_t));
    E->st_events.clear();
    E->st_members.clear();
    if (n_events) *n_events = ne;
    if (n_members) *n_members = nm;
    return CO_OK;
}

int co_drain_samples(co_engine* E, int64_t* out, int64_t max, int64_t* n) {
    if (!E) return fail(CO_EINVAL, "null argument");
    int r = drain_device(E);
    if (r) return r;
    int64_t ns = (int64_t)E->st_samples.size() / 2;
    if (ns > max) return fail(CO_EINVAL, "sample buffer too small");
    if (ns) std::memcpy(out, E->st_samples.data(), 2 * ns * sizeof(int64_t));
    E->st_samples.clear();
    if (n) *n = ns;
    return CO_OK;
}

int co_read_token_times(co_engine* E, int64_t* offsets, int64_t* times) {
    if (!E) return fail(CO_EINVAL, "null argument");
    if (offsets) std::memcpy(offsets, E->tok_off_host.data(), (E->n + 1) * sizeof(int64_t));
    if (times && E->tok_total) {
        CK(cudaMemcpyAsync(times, E->d.tok_times, E->tok_total * sizeof(int64_t), cudaMemcpyDeviceToHost, E->stream));
        CK(cudaStreamSynchronize(E->stream));
    }
    return CO_OK;
}

int co_metrics(co_engine* E, co_metrics_raw* out) {
    CO_RANGE("co_metrics");
    if (!E || !out) return fail(CO_EINVAL, "null argument");
    { int rw_ = begin_work(E); if (rw_) return rw_; }
    const int64_t n = E->n, ntok = std::max<int64_t>(E->tok_total, 1);
    std::memset(out, 0, sizeof(*out));
    if (n == 0) return CO_OK;
    std::vector<void*> tmp;
    auto get = [&](size_t bytes) -> void* {
        void* p = nullptr;
        if (cudaMalloc(&p, std::max<size_t>(bytes, 8)) != cudaSuccess) return nullptr;
        tmp.push_back(p);
        return p;
    };
    auto release = [&]() { for (void* p : tmp) cudaFree(p); };
    MetScratch m;
    m.cnt = (unsigned long long*)get(16 * 8);
    m.keys[0] = (uint64_t*)get(n * 8); m.keys[1] = (uint64_t*)get(ntok * 8);
    m.keys[2] = (uint64_t*)get(n * 8); m.keys[3] = (uint64_t*)get(n * 8);
    m.normc = (double*)get(n * 8); m.flagc = (uint8_t*)get(n); m.norm_list = (double*)get(n * 8);
    int32_t* perm = (int32_t*)get(n * 4);
    m.perm = perm;
    m.hist = (unsigned int*)get(MET_RANKS * 256 * 4);
    m.pre = (uint64_t*)get(MET_RANKS * 8); m.rem = (long long*)get(MET_RANKS * 8);
    m.out_norm_sum = (double*)get(8);
    for (void* p : tmp)
        if (!p) { release(); return fail(CO_ECUDA, "metrics scratch allocation failed"); }
    std::vector<int32_t> ph(n);
    for (int64_t k = 0; k < n; k++) ph[k] = (int32_t)E->perm[k];
    cudaStream_t s = E->stream;
    int r = CO_OK;
    auto ck = [&](cudaError_t e) { if (e != cudaSuccess && r == CO_OK) r = fail(CO_ECUDA, cudaGetErrorString(e)); };
    ck(cudaMemcpyAsync(perm, ph.data(), n * 4, cudaMemcpyHostToDevice, s));
    ck(cudaMemsetAsync(m.cnt, 0, 16 * 8, s));
    ck(cudaMemsetAsync(m.hist, 0, MET_RANKS * 256 * 4, s));
    k_met_rows<<<E->grid, 256, 0, s>>>(E->d, m);
    k_met_norm<<<1, 1024, 0, s>>>(m, (int32_t)n);
    ck(cudaGetLastError());
    unsigned long long cnt[16];
    ck(cudaMemcpyAsync(cnt, m.cnt, sizeof(cnt), cudaMemcpyDeviceToHost, s));
    ck(cudaMemcpyAsync(&out->norm_sum, m.out_norm_sum, 8, cudaMemcpyDeviceToHost, s));
    ck(cudaStreamSynchronize(s));
    if (r) { release(); return r; }
    out->completed = cnt[MC_DONE]; out->ok_ttft = cnt[MC_OK_TTFT]; out->ok_tbt = cnt[MC_OK_TBT];
    out->generated = cnt[MC_GEN]; out->preemption_total = cnt[MC_PRE_TOTAL]; out->preempted = cnt[MC_PREEMPTED];
    out->sum_ttft = cnt[MC_SUM_TTFT]; out->sum_gap = cnt[MC_SUM_GAP]; out->sum_wait = cnt[MC_SUM_WAIT];
    out->sum_exec = cnt[MC_SUM_EXEC]; out->sum_pdec = cnt[MC_SUM_PDEC]; out->sum_ptime = cnt[MC_SUM_PTIME];
    for (int l = 0; l < MET_LISTS; l++) out->count[l] = (int64_t)cnt[MC_N0 + l];
    const double qs[3] = {50.0 / 100.0, 90.0 / 100.0, 99.0 / 100.0};
    for (int l = 0; l < MET_LISTS && !r; l++) {
        const int64_t c = out->count[l];
        if (c == 0) continue;
        // np.percentile 'linear': virtual index (c - 1) * q, floor / +1, clamped to the last
        long long rk[MET_RANKS];
        for (int q = 0; q < 3; q++) {
            const double v = (double)(c - 1) * qs[q];
            if (v >= (double)(c - 1)) { rk[2 * q] = rk[2 * q + 1] = c - 1; }
            else { rk[2 * q] = (long long)std::floor(v); rk[2 * q + 1] = rk[2 * q] + 1; }
        }
        rk[6] = c - 1;
        std::vector<uint64_t> zero(MET_RANKS, 0);
        ck(cudaMemcpyAsync(m.pre, zero.data(), MET_RANKS * 8, cudaMemcpyHostToDevice, s));
        ck(cudaMemcpyAsync(m.rem, rk, MET_RANKS * 8, cudaMemcpyHostToDevice, s));
        const int grid = (int)std::min<int64_t>((c + 255) / 256, (int64_t)E->sms * 4);
        for (int pass = 0; pass < 8; pass++) {
            const int shift = 56 - 8 * pass;
            const uint64_t mask = pass == 0 ? 0ull : (~0ull << (64 - 8 * pass));
            k_rs_hist<<<grid, 256, 0, s>>>(m.keys[l], c, MET_RANKS, m.pre, mask, shift, m.hist);
            k_rs_pick<<<1, 32 * MET_RANKS, 0, s>>>(MET_RANKS, m.pre, m.rem, shift, m.hist);
        }
        uint64_t bits[MET_RANKS];
        ck(cudaMemcpyAsync(bits, m.pre, sizeof(bits), cudaMemcpyDeviceToHost, s));
        ck(cudaStreamSynchronize(s));
        for (int q = 0; q < MET_RANKS; q++) std::memcpy(&out->order_stat[l][q], &bits[q], 8);
    }
    release();
    return r;
}

int co_check_invariants(co_engine* E) {
    if (!E) return fail(CO_EINVAL, "null argument");
    { int rw_ = begin_work(E); if (rw_) return rw_; }
    k_check<<<1, NT, 0, E->stream>>>(E->d);
    CK(cudaGetLastError());
    int r = sync_ctl(E);
    if (r) return r;
    return check_device_error(E);
}

int co_last_device_ms(co_engine* E, double* ms) {
    if (!E || !ms) return fail(CO_EINVAL, "null argument");
    *ms = E->last_ms;
    E->timing = true;
    return CO_OK;
}

int co_time_steps(co_engine* E, int32_t k, int64_t flush_bytes, double* step_ms, double* stage_ms) {
    CO_RANGE("co_time_steps");
    if (!E || k < 1) return fail(CO_EINVAL, "bad arguments");
    { int rw_ = begin_work(E); if (rw_) return rw_; }
    const int NE = CO_NSTAGES + 1;
    std::vector<cudaEvent_t> evs((size_t)k * NE);
    for (auto& e : evs) CK(cudaEventCreate(&e));
    void* flush = nullptr;
    if (flush_bytes > 0) CK(cudaMalloc(&flush, flush_bytes));
    cudaGraph_t g;
    cudaGraphExec_t ge = nullptr;
    int r = CO_OK;
    CK(cudaStreamBeginCapture(E->stream, cudaStreamCaptureModeThreadLocal));
    const bool stages = stage_ms != nullptr;  // stage events split the graph; without them the
                                              // step kernels chain through PDL edges
    for (int32_t j = 0; j < k && !r; j++) {
        if (flush) cudaMemsetAsync(flush, j & 0xff, flush_bytes, E->stream);
        cudaEvent_t* e = evs.data() + (size_t)j * NE;
        if (stages) {
            r = launch_step(E, 1, e, 0, nullptr, j & 1, true);
        } else {
            mark(e[0], E->stream);
            r = launch_step(E, 1, nullptr, 0, nullptr, j & 1, true);
            mark(e[NE - 1], E->stream);
        }
    }
    flush_join(E);  // (the last step's collective is joined after its end event)
    CK(cudaStreamEndCapture(E->stream, &g));
    if (!r) {
        CK(cudaGraphInstantiate(&ge, g, 0));
        CK(cudaGraphLaunch(ge, E->stream));
        E->last_slot = (k - 1) & 1;
        if (E->comm) E->reduce_calls += k;
        CK(cudaStreamSynchronize(E->stream));
        if (stages)
            for (int q = 0; q < CO_NSTAGES; q++) stage_ms[q] = 0;
        for (int32_t j = 0; j < k; j++) {
            cudaEvent_t* e = evs.data() + (size_t)j * NE;
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e[0], e[NE - 1]));
            step_ms[j] = ms;
            for (int q = 0; q < CO_NSTAGES && stages; q++) {
                float x = 0;
                CK(cudaEventElapsedTime(&x, e[q], e[q + 1]));
                stage_ms[q] += x;
            }
        }
        cudaGraphExecDestroy(ge);
    }
    cudaGraphDestroy(g);
    for (auto& e : evs) cudaEventDestroy(e);
    if (flush) cudaFree(flush);
    if (r) return r;
    if ((r = sync_ctl(E))) return r;
    if (E->h_ctl->paused) return fail(CO_EDEVICE, "append buffers filled during a timed run; drain first");
    return check_device_error(E);
}

int co_read_block_tables(co_engine* E, int32_t* lens, int32_t* pages, int64_t max_pages, int32_t* free_pages,
                         int32_t* n_free) {
    CO_RANGE("co_read_block_tables");
    if (!E || !lens || !n_free) return fail(CO_EINVAL, "null argument");
    int r = sync_ctl(E);
    if (r) return r;
    const int64_t n = E->n;
    const int32_t W = E->d.dir_w;
    std::vector<int32_t> dir((size_t)n * W), pool((size_t)E->n_chunks * TCHUNK);
    if (n) {
        CK(cudaMemcpyAsync(lens, E->d.tab_len, n * sizeof(int32_t), cudaMemcpyDeviceToHost, E->stream));
        CK(cudaMemcpyAsync(dir.data(), E->d.dir, dir.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, E->stream));
    }
    CK(cudaMemcpyAsync(pool.data(), E->d.chunk_pool, pool.size() * sizeof(int32_t), cudaMemcpyDeviceToHost,
                       E->stream));
    const int32_t nf = E->h_ctl->free_top;
    if (free_pages && nf)
        CK(cudaMemcpyAsync(free_pages, E->d.free_stack, nf * sizeof(int32_t), cudaMemcpyDeviceToHost, E->stream));
    CK(cudaStreamSynchronize(E->stream));
    *n_free = nf;
    int64_t w = 0;
    for (int64_t i = 0; i < n; i++) {
        if (w + lens[i] > max_pages) return fail(CO_EINVAL, "page buffer too small");
        for (int32_t k = 0; k < lens[i]; k++)
            if (pages) pages[w + k] = pool[(size_t)dir[(size_t)i * W + k / TCHUNK] * TCHUNK + k % TCHUNK];
        w += lens[i];
    }
    return CO_OK;
}

int co_data_stats(co_engine* E, int64_t* st) {
    if (!E || !st) return fail(CO_EINVAL, "null argument");
    if (!E->d.dp.on) return fail(CO_EINVAL, "data plane is off (kv_layers = 0)");
    DataCtl dc;
    CK(cudaMemcpyAsync(&dc, E->d.dctl, sizeof(dc), cudaMemcpyDeviceToHost, E->stream));
    CK(cudaStreamSynchronize(E->stream));
    st[0] = dc.bytes_out; st[1] = dc.bytes_in; st[2] = dc.bytes_fill; st[3] = dc.bytes_move;
    st[4] = dc.dec_steps; st[5] = dc.dec_members; st[6] = dc.dec_tokens; st[7] = 0;
    return CO_OK;
}

// ---- snapshot planning: plan_batch(PlannerInputs, cfg) (scheduler.py:939-950)
// The caller's views and pool records are written into the engine's SoA (the
// request space of a co_create over the views' ids) and ONE planner pass runs
// -- k_classify, then k_serial in plan-only mode -- with the plan read back.
constexpr int SNAP_COLS = 20;
__global__ void k_load_snapshot(Dev d, const int64_t* __restrict__ col, int32_t n) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int64_t* r = col + (int64_t)i * SNAP_COLS;
        d.state[i] = (int8_t)r[0];
        d.gen[i] = (int32_t)r[1]; d.used[i] = (int32_t)r[2]; d.kv_need[i] = (int32_t)r[3];
        d.prefill[i] = (int32_t)r[4]; d.pcount[i] = (int32_t)r[5]; d.pred[i] = (int32_t)r[6];
        d.est[i] = (int32_t)r[7];
        d.first_tok[i] = r[8]; d.last_tok[i] = r[9]; d.max_tbt[i] = r[10]; d.ready_at[i] = r[11];
        d.holds[i] = (uint8_t)r[12]; d.granted[i] = (int32_t)r[13]; d.host[i] = (int32_t)r[14];
        d.off[i] = (int32_t)r[15]; d.rsv[i] = (int32_t)r[16]; d.guest[i] = (int32_t)r[17];
        d.gnext[i] = (int32_t)r[18]; d.rec_seq[i] = r[19];
        const int8_t s = d.state[i];
        if (s == ST_WAITING || s == ST_PREEMPTED) d.key0[i] = wait_key(d, i);
    }
}
__global__ void k_load_snapshot_ctl(Dev d, int64_t now, int64_t ti, int32_t rsv, int64_t fp, int64_t gsum,
                                    int64_t usum, int64_t seq, int32_t n_live) {
    Ctl& c = *d.ctl;
    c.now = now; c.t_i = ti; c.rsv_cur = rsv; c.fp_sum = fp; c.granted_sum = gsum; c.used_sum = usum;
    c.seq = seq; c.n_live = n_live; c.next_pending = d.n; c.horizon = INT64_MAX / 4;
    c.done = 0; c.paused = 0; c.error = 0; c.has_mark = 0; c.streak = 0; c.thr = 0;
    c.cnt_nw = c.cnt_nwp = c.cnt_run = c.cnt_blown = c.cnt_cand = 0;
    c.kmin = ~0ull; c.kmax = 0;
    c.ev_count = c.mem_count = c.sample_count = 0;
}

int co_plan_snapshot(co_engine* E, const int64_t* cols, const int64_t* scal, int64_t* hdr, int32_t* lists,
                     int64_t cap) {
    CO_RANGE("co_plan_snapshot");
    if (!E || !cols || !scal || !hdr || !lists) return fail(CO_EINVAL, "null argument");
    if (E->comm || E->d.dp.on) return fail(CO_EINVAL, "snapshot planning needs a plain engine (no data plane / NCCL)");
    { int rw_ = begin_work(E); if (rw_) return rw_; }
    const int32_t n = (int32_t)E->n;
    int64_t* dcol = nullptr;
    CK(cudaMalloc(&dcol, std::max<int64_t>(1, (int64_t)n * SNAP_COLS) * sizeof(int64_t)));
    int r = CO_OK;
    cudaError_t e = n ? cudaMemcpyAsync(dcol, cols, (size_t)n * SNAP_COLS * sizeof(int64_t), cudaMemcpyHostToDevice,
                                        E->stream)
                      : cudaSuccess;
    if (e == cudaSuccess) {
        k_load_snapshot<<<std::max(1, std::min(E->sms * 4, (n + 255) / 256)), 256, 0, E->stream>>>(E->d, dcol, n);
        k_load_snapshot_ctl<<<1, 1, 0, E->stream>>>(E->d, scal[0], scal[1], (int32_t)scal[2], scal[3], scal[4],
                                                    scal[5], scal[6], (int32_t)scal[7]);
        k_classify<<<E->d.nblk, 256, 0, E->stream>>>(E->d, 0, 1);
        serial_kernel(0, E->d)<<<1, E->plan_threads, sizeof(PlanSh), E->stream>>>(E->d, (LogMirror*)nullptr,
                                                                               (int64_t*)nullptr, 0, 1);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(E->stream);
    cudaFree(dcol);
    if (e != cudaSuccess) return fail(CO_ECUDA, std::string("snapshot plan: ") + cudaGetErrorString(e));
    if ((r = sync_ctl(E))) return r;
    if ((r = check_device_error(E))) return r;
    PlanHdr P;
    CK(cudaMemcpy(&P, E->d.plan, sizeof(P), cudaMemcpyDeviceToHost));
    hdr[0] = P.n_mem; hdr[1] = P.n_act; hdr[2] = P.n_pre; hdr[3] = P.n_cl; hdr[4] = P.n_def;
    hdr[5] = P.overflow; hdr[6] = P.batch_tokens; hdr[7] = E->h_ctl->active;
    const int64_t need = 2LL * P.n_mem + 6LL * P.n_act + 2LL * P.n_pre + 2LL * P.n_cl + P.n_def;
    if (need > cap) return fail(CO_EINVAL, "plan buffer too small");
    const Dev& d = E->d;
    int32_t* w = lists;
    auto get = [&](const int32_t* src, int32_t cnt) -> cudaError_t {
        cudaError_t x = cnt ? cudaMemcpy(w, src, cnt * sizeof(int32_t), cudaMemcpyDeviceToHost) : cudaSuccess;
        w += cnt;
        return x;
    };
    for (auto x : {get(d.mem_idx, P.n_mem), get(d.mem_tok, P.n_mem), get(d.act_kind, P.n_act), get(d.act_idx, P.n_act),
                   get(d.act_tok, P.n_act), get(d.act_nb, P.n_act), get(d.act_host, P.n_act),
                   get(d.act_start, P.n_act), get(d.pre_idx, P.n_pre), get(d.pre_strat, P.n_pre),
                   get(d.cl_w, P.n_cl), get(d.cl_p, P.n_cl), get(d.def_idx, P.n_def)})
        if (x != cudaSuccess) return fail(CO_ECUDA, "plan readback");
    touch(E);
    return CO_OK;
}

int co_swap_io_stats(co_engine* E, int64_t* out) {
    if (!E || !out) return fail(CO_EINVAL, "null argument");
    if (!E->d.dp.on) return fail(CO_EINVAL, "data plane is off (kv_layers = 0)");
    CK(cudaStreamSynchronize(E->stream));
    DataCtl dc;
    CK(cudaMemcpyAsync(&dc, E->d.dctl, sizeof(dc), cudaMemcpyDeviceToHost, E->stream));
    CK(cudaStreamSynchronize(E->stream));
    out[0] = dc.io_bytes_out; out[1] = dc.io_bytes_in; out[2] = dc.io_ns; out[3] = dc.io_launches;
    out[4] = E->d.dp.split_io; out[5] = E->d.dp.io_ctas;
    return CO_OK;
}

int co_kv_verify(co_engine* E, int64_t* bad, int64_t* checked) {
    CO_RANGE("co_kv_verify");
    if (!E || !bad || !checked) return fail(CO_EINVAL, "null argument");
    { int rw_ = begin_work(E); if (rw_) return rw_; }
    if (!E->d.dp.on) return fail(CO_EINVAL, "data plane is off (kv_layers = 0)");
    unsigned long long* cnt = nullptr;
    CK(cudaMalloc(&cnt, 16));
    CK(cudaMemsetAsync(cnt, 0, 16, E->stream));
    k_kv_verify<<<E->sms * 4, 256, 0, E->stream>>>(E->d, E->d.dp, cnt, cnt + 1);
    unsigned long long h[2];
    CK(cudaMemcpyAsync(h, cnt, 16, cudaMemcpyDeviceToHost, E->stream));
    CK(cudaStreamSynchronize(E->stream));
    cudaFree(cnt);
    *bad = (int64_t)h[0];
    *checked = (int64_t)h[1];
    return CO_OK;
}

int co_read_decode(co_engine* E, int32_t* members, int32_t* ctx, float* out, int64_t max_members, int64_t* n,
                   int64_t* step_id) {
    if (!E || !n) return fail(CO_EINVAL, "null argument");
    const DataCfg& x = E->d.dp;
    if (!x.on || !x.decode_on) return fail(CO_EINVAL, "decode is off");
    DataCtl dc;
    CK(cudaMemcpyAsync(&dc, E->d.dctl, sizeof(dc), cudaMemcpyDeviceToHost, E->stream));
    int r = sync_ctl(E);
    if (r) return r;
    *n = dc.n_dec;
    if (step_id) *step_id = E->h_ctl->steps;
    if (dc.n_dec > max_members) return fail(CO_EINVAL, "decode buffers too small");
    if (dc.n_dec) {
        if (members) CK(cudaMemcpyAsync(members, x.dec_idx, dc.n_dec * 4, cudaMemcpyDeviceToHost, E->stream));
        if (ctx) CK(cudaMemcpyAsync(ctx, x.dec_ctx, dc.n_dec * 4, cudaMemcpyDeviceToHost, E->stream));
        if (out)
            CK(cudaMemcpyAsync(out, x.dec_out, (size_t)dc.n_dec * x.L * x.Hq * x.D * sizeof(float),
                               cudaMemcpyDeviceToHost, E->stream));
        CK(cudaStreamSynchronize(E->stream));
    }
    return CO_OK;
}

int co_host_link_gbs(int64_t bytes, double* d2h, double* h2d) {
    if (bytes <= 0 || !d2h || !h2d) return fail(CO_EINVAL, "bad arguments");
    void *dev = nullptr, *host = nullptr;
    cudaStream_t s;
    cudaEvent_t a, b;
    CK(cudaMalloc(&dev, bytes));
    CK(cudaHostAlloc(&host, bytes, cudaHostAllocDefault));
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best_d2h = 1e30f, best_h2d = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        float ms;
        cudaEventRecord(a, s);
        cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        best_d2h = std::min(best_d2h, ms);
        cudaEventRecord(a, s);
        cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        best_h2d = std::min(best_h2d, ms);
    }
    *d2h = bytes / (best_d2h * 1e-3) / 1e9;
    *h2d = bytes / (best_h2d * 1e-3) / 1e9;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaStreamDestroy(s);
    cudaFree(dev);
    cudaFreeHost(host);
    return CO_OK;
}

int co_set_decode(co_engine* E, int32_t on) {
    if (!E || !E->d.dp.on || !E->d.dp.decode_on) return fail(CO_EINVAL, "decode is not configured");
    { int rw_ = begin_work(E); if (rw_) return rw_; }
    int32_t v = on ? 1 : 0;
    CK(cudaMemcpyAsync(&E->d.dctl->decode_enabled, &v, 4, cudaMemcpyHostToDevice, E->stream));
    CK(cudaStreamSynchronize(E->stream));
    return CO_OK;
}

// Swap data path micro-benchmark: ONE GATHER (device pages -> pinned host
// pages) and ONE SCATTER (back) of ntok tokens through k_data, the same
// kernel the engine runs, on the first pages of the pool.  Clobbers KV
// contents: use a dedicated instance.
int co_swap_bench(co_engine* E, int64_t ntok, int32_t iters, double* out_ms, double* in_ms) {
    CO_RANGE("co_swap_bench");
    if (!E || !out_ms || !in_ms || iters < 1) return fail(CO_EINVAL, "bad arguments");
    { int rw_ = begin_work(E); if (rw_) return rw_; }
    DataCfg& x = E->d.dp;
    if (!x.on) return fail(CO_EINVAL, "data plane is off");
    const int bs = E->d.bs;
    const int64_t np = (ntok + bs - 1) / bs;
    if (np > E->d.n_pages || np > x.h_pages || ntok > (1ll << 30)) return fail(CO_EINVAL, "ntok too large");
    std::vector<int32_t> snap(2 * np);
    for (int64_t k = 0; k < np; k++) { snap[k] = (int32_t)k; snap[np + k] = (int32_t)k; }
    CK(cudaMemcpyAsync(x.snap, snap.data(), snap.size() * 4, cudaMemcpyHostToDevice, E->stream));
    DOp ops[2] = {};
    for (int q = 0; q < 2; q++) {
        ops[q].kind = q == 0 ? D_GATHER : D_SCATTER; ops[q].req = 0; ops[q].ntok = (int32_t)ntok; ops[q].t0 = 0;
        ops[q].src_end = ops[q].dst_end = -1;
        ops[q].src_where = q == 0 ? W_DEV : W_HOST; ops[q].dst_where = q == 0 ? W_HOST : W_DEV;
        ops[q].src_snap = q == 0 ? 0 : np; ops[q].dst_snap = q == 0 ? np : 0;
    }
    DataCtl saved;
    CK(cudaMemcpyAsync(&saved, E->d.dctl, sizeof(saved), cudaMemcpyDeviceToHost, E->stream));
    CK(cudaStreamSynchronize(E->stream));
    float t_out = 0, t_in = 0;
    for (int it = 0; it < iters + 1; it++) {
        for (int q = 0; q < 2; q++) {
            CK(cudaMemcpyAsync(x.ops, &ops[q], sizeof(DOp), cudaMemcpyHostToDevice, E->stream));
            int32_t one = 1;
            CK(cudaMemcpyAsync(&E->d.dctl->n_ops, &one, 4, cudaMemcpyHostToDevice, E->stream));
            CK(cudaEventRecord(E->ev0, E->stream));
            launch_coop(k_data, E->sms, 512, E->stream, E->d, x, E->d.dctl, 1);
            CK(cudaEventRecord(E->ev1, E->stream));
            CK(cudaEventSynchronize(E->ev1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, E->ev0, E->ev1));
            if (it > 0) (q == 0 ? t_out : t_in) += ms;  // first round is warm-up
        }
    }
    CK(cudaMemcpyAsync(E->d.dctl, &saved, sizeof(saved), cudaMemcpyHostToDevice, E->stream));
    CK(cudaStreamSynchronize(E->stream));
    *out_ms = t_out / iters;
    *in_ms = t_in / iters;
    return CO_OK;
}

int co_nccl_unique_id(uint8_t* out) {
    if (!out) return fail(CO_EINVAL, "null argument");
    if (!nccl().ok) return fail(CO_ECUDA, "libnccl.so.2 not loadable");
    ncclUniqueId id;
    ncclResult_t r = nccl().getUniqueId(&id);
    if (r != ncclSuccess) return fail(CO_ECUDA, std::string("ncclGetUniqueId: ") + nccl().errorString(r));
    std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
    return CO_OK;
}

int co_attach_nccl(co_engine* E, const uint8_t* uid, int32_t nranks, int32_t rank) {
    if (!E || !uid || nranks < 1 || rank < 0 || rank >= nranks) return fail(CO_EINVAL, "bad arguments");
    { int rw_ = begin_work(E); if (rw_) return rw_; }
    if (E->comm) return fail(CO_EINVAL, "already attached");
    if (!nccl().ok) return fail(CO_ECUDA, "libnccl.so.2 not loadable");
    ncclUniqueId id;
    std::memcpy(id.internal, uid, NCCL_UNIQUE_ID_BYTES);
    cudaSetDevice(E->device);
    ncclResult_t r = nccl().commInitRank(&E->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        E->comm = nullptr;
        return fail(CO_ECUDA, std::string("ncclCommInitRank: ") + nccl().errorString(r));
    }
    CK(cudaStreamCreateWithFlags(&E->side, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&E->fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&E->join[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&E->join[1], cudaEventDisableTiming));
    CK(cudaMalloc(&E->red, 8 * sizeof(int64_t)));
    CK(cudaMemset(E->red, 0, 8 * sizeof(int64_t)));
    E->nranks = nranks;
    E->rank = rank;
    if (E->graph) { cudaGraphExecDestroy(E->graph); E->graph = nullptr; }  // recapture with the collective
    if (E->graph1) { cudaGraphExecDestroy(E->graph1); E->graph1 = nullptr; }
        if (E->graph1r) { cudaGraphExecDestroy(E->graph1r); E->graph1r = nullptr; }
    return CO_OK;
}

int co_global_reserve(co_engine* E, int64_t* out, int64_t* calls) {
    if (!E || !out) return fail(CO_EINVAL, "null argument");
    if (!E->comm) return fail(CO_EINVAL, "no communicator attached");
    CK(cudaStreamSynchronize(E->side));
    CK(cudaMemcpy(out, E->red + 4 * E->last_slot + 2, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (calls) *calls = E->reduce_calls;
    return CO_OK;
}

// development aid: enable/read the %globaltimer phase stamps of k_plan/k_apply
int co_phase_profile(co_engine* E, int32_t enable, int64_t* out /* 64 */) {
    if (!E) return fail(CO_EINVAL, "null argument");
    { int rw_ = begin_work(E); if (rw_) return rw_; }
    if (enable && !E->d.prof) {
        CK(cudaMalloc(&E->d.prof, 64 * sizeof(int64_t)));
        CK(cudaMemset(E->d.prof, 0, 64 * sizeof(int64_t)));
        if (E->graph) { cudaGraphExecDestroy(E->graph); E->graph = nullptr; }
        if (E->graph1) { cudaGraphExecDestroy(E->graph1); E->graph1 = nullptr; }
        if (E->graph1r) { cudaGraphExecDestroy(E->graph1r); E->graph1r = nullptr; }
    }
    if (out && E->d.prof) {
        CK(cudaMemcpyAsync(out, E->d.prof, 64 * sizeof(int64_t), cudaMemcpyDeviceToHost, E->stream));
        CK(cudaStreamSynchronize(E->stream));
    }
    return CO_OK;
}

int co_kernels_per_step(co_engine* E, int32_t* n) {
    if (!E || !n) return fail(CO_EINVAL, "null argument");
    // begin, classify(+admit, N'_w head), serial (plan + apply + check
    // [+ mirror]); the data plane adds k_data (+ k_swapio, + decode + combine)
    *n = 2 + (E->d.dp.on ? 1 + (E->d.dp.split_io ? 1 : 0) + (E->d.dp.decode_on ? 2 : 0) : 0);
    return CO_OK;
}

}  // extern "C"

// ---- random streams on the device (csrc/trace_gen.cuh) -----

namespace {
// Scratch and stream of the generator calls: grow-only per-device slots,
// reused call after call (slot i = the i-th buffer a call asks for), so a
// generation costs kernels, not cudaMalloc / cudaFree / stream creation.
// Calls are serialized by a process-wide mutex and end with a stream sync.
struct GenArena {
    cudaStream_t s = nullptr;
    std::vector<std::pair<void*, size_t>> slots;
};
std::mutex g_gen_mu;
std::map<int, GenArena> g_gen_arena;

struct GenCtx {
    std::lock_guard<std::mutex> lk{g_gen_mu};
    GenArena* A = nullptr;
    cudaStream_t s = nullptr;
    int sms = 148;
    int r = CO_OK;
    size_t slot = 0;
    bool ck(cudaError_t e) {
        if (e != cudaSuccess && r == CO_OK) r = fail(CO_ECUDA, cudaGetErrorString(e));
        return r == CO_OK;
    }
    template <class T>
    T* get(int64_t n) {
        const size_t bytes = (size_t)std::max<int64_t>(n, 1) * sizeof(T);
        if (r) return nullptr;
        if (A->slots.size() <= slot) A->slots.push_back({nullptr, 0});
        auto& sl = A->slots[slot++];
        if (sl.second < bytes) {
            if (sl.first) cudaFree(sl.first);
            sl = {nullptr, 0};
            const size_t want = bytes + bytes / 4;
            if (!ck(cudaMalloc(&sl.first, want))) return nullptr;
            sl.second = want;
        }
        return (T*)sl.first;
    }
    int init(int device) {
        if (device >= 0 && !ck(cudaSetDevice(device))) return r;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        A = &g_gen_arena[dev];
        if (!A->s) ck(cudaStreamCreateWithFlags(&A->s, cudaStreamNonBlocking));
        s = A->s;
        return r;
    }
    int grid(int64_t n, int threads = 256) const {
        return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, (int64_t)sms * 8));
    }
};

void stream_seed(uint64_t seed, uint64_t stream, u128& st, u128& inc) {
    const uint64_t ent[2] = {seed, stream};
    seed_pcg64(ent, 2, st, inc);
}

void pcg_fill(GenCtx& G, u128 st, u128 inc, int64_t count, uint64_t* out) {
    const int grid = G.grid(count);
    u128 jm, jp;
    pcg_jump(inc, (uint64_t)grid * 256, jm, jp);
    k_pcg_fill<<<grid, 256, 0, G.s>>>(to_u(st), to_u(inc), to_u(jm), to_u(jp), count, out);
    G.ck(cudaGetLastError());
}

// n ziggurat samples (+ the u53 of `extra` trailing words per sample)
int zig_stream(GenCtx& G, int kind, u128 st, u128 inc, int64_t n, int extra, double* out, double* ex) {
    if (n == 0) return CO_OK;
    const int64_t M = ((n * (1 + extra) + n / 8 + 8192) + ORB_CHUNK - 1) / ORB_CHUNK * ORB_CHUNK, R = M + 4096,
                  nch = M / ORB_CHUNK;
    uint64_t* raw = G.get<uint64_t>(R);
    uint8_t* len = G.get<uint8_t>(M);
    uint32_t* accw = G.get<uint32_t>(M / 32);
    uint32_t* vis = G.get<uint32_t>(nch * ORB_K * 32);
    double* val = G.get<double>(M);
    int64_t* ex_ = G.get<int64_t>(nch * ORB_K);
    int8_t* choice = G.get<int8_t>(nch);
    int64_t* cnt = G.get<int64_t>(nch);
    int64_t* total = G.get<int64_t>(1);
    int32_t* bad = G.get<int32_t>(1);
    if (G.r) return G.r;
    pcg_fill(G, st, inc, R, raw);
    if (kind == ZIG_EXP) k_zig_local<ZIG_EXP><<<G.grid(M), 256, 0, G.s>>>(raw, R, M, extra, len, accw, val);
    else k_zig_local<ZIG_NOR><<<G.grid(M), 256, 0, G.s>>>(raw, R, M, extra, len, accw, val);
    k_orbit_spec<<<(int)((nch + ORB_WARPS - 1) / ORB_WARPS), ORB_WARPS * 32, 0, G.s>>>(len, M, nch, vis, ex_);
    k_orbit_fix<<<1, 256, 0, G.s>>>(len, nch, vis, ex_, choice, bad);
    k_orbit_count<<<(int)((nch * 32 + 255) / 256), 256, 0, G.s>>>(vis, choice, accw, nch, cnt);
    k_orbit_scan<<<1, 1024, 0, G.s>>>(cnt, nch, total);
    k_orbit_emit<<<(int)((nch * 32 + 255) / 256), 256, 0, G.s>>>(vis, choice, accw, cnt, len, val, raw, nch, n,
                                                                  extra, out, ex);
    G.ck(cudaGetLastError());
    int64_t got = 0;
    G.ck(cudaMemcpyAsync(&got, total, 8, cudaMemcpyDeviceToHost, G.s));
    G.ck(cudaStreamSynchronize(G.s));
    if (G.r) return G.r;
    if (got < n) return fail(CO_EDEVICE, "ziggurat stream budget exhausted");
    return CO_OK;
}
}  // namespace

extern "C" {

int co_pcg64_seed(const uint64_t* entropy, int32_t n, uint64_t out[4]) {
    if (!entropy || !out || n < 1) return fail(CO_EINVAL, "bad entropy");
    u128 st, inc;
    seed_pcg64(entropy, n, st, inc);
    out[0] = (uint64_t)(st >> 64); out[1] = (uint64_t)st;
    out[2] = (uint64_t)(inc >> 64); out[3] = (uint64_t)inc;
    return CO_OK;
}

int co_gen_raw(uint64_t seed, uint64_t stream, int64_t count, int device, uint64_t* out) {
    if (count < 0 || (count && !out)) return fail(CO_EINVAL, "bad arguments");
    GenCtx G;
    if (G.init(device)) return G.r;
    u128 st, inc;
    stream_seed(seed, stream, st, inc);
    if (count) pcg_fill(G, st, inc, count, out);
    G.ck(cudaStreamSynchronize(G.s));
    return G.r;
}

int co_gen_std(int32_t kind, uint64_t seed, uint64_t stream, int64_t n, int device, double* out) {
    if (n < 0 || (n && !out) || (kind != ZIG_EXP && kind != ZIG_NOR)) return fail(CO_EINVAL, "bad arguments");
    GenCtx G;
    if (G.init(device)) return G.r;
    u128 st, inc;
    stream_seed(seed, stream, st, inc);
    return zig_stream(G, kind, st, inc, n, 0, out, nullptr);
}

int co_gen_trace(const co_trace_spec* sp, uint64_t seed, int device, int64_t* arrival_us, int32_t* prompt_len,
                 int32_t* output_len) {
    CO_RANGE("co_gen_trace");
    if (!sp || sp->n < 0 || sp->n > (1ll << 30)) return fail(CO_EINVAL, "bad trace spec");
    const int64_t n = sp->n;
    if (n && (!arrival_us || !prompt_len || !output_len)) return fail(CO_EINVAL, "null output");
    if (!(sp->gap_scale > 0) || sp->input_min < 1 || sp->input_min > sp->input_max || sp->output_min < 1 ||
        sp->output_min > sp->output_max)
        return fail(CO_EINVAL, "invalid trace spec (workload.py:33-47 rules)");
    if (n == 0) return CO_OK;
    GenCtx G;
    if (G.init(device)) return G.r;
    double* z = G.get<double>(n);
    if (G.r) return G.r;
    u128 st, inc;
    stream_seed(seed, 0, st, inc);
    if (int r = zig_stream(G, ZIG_EXP, st, inc, n, 0, z, nullptr)) return r;
    k_arrivals<<<1, ARR_T, 0, G.s>>>(z, n, sp->gap_scale, arrival_us);
    G.ck(cudaStreamSynchronize(G.s));  // z is reused below
    stream_seed(seed, 1, st, inc);
    if (int r = zig_stream(G, ZIG_NOR, st, inc, n, 0, z, nullptr)) return r;
    k_lognormal_len<<<G.grid(n), 256, 0, G.s>>>(z, n, sp->mu_in, sp->sigma_in, sp->input_min, sp->input_max,
                                                prompt_len);
    G.ck(cudaStreamSynchronize(G.s));
    stream_seed(seed, 2, st, inc);
    if (int r = zig_stream(G, ZIG_NOR, st, inc, n, 0, z, nullptr)) return r;
    k_lognormal_len<<<G.grid(n), 256, 0, G.s>>>(z, n, sp->mu_out, sp->sigma_out, sp->output_min, sp->output_max,
                                                output_len);
    G.ck(cudaGetLastError());
    G.ck(cudaStreamSynchronize(G.s));
    return G.r;
}

int co_gen_slos(int64_t n, const int32_t* prompt_len, const co_slo_spec* sp, uint64_t seed, int device,
                int64_t* slo_ttft_us, int64_t* slo_tbt_us) {
    CO_RANGE("co_gen_slos");
    if (!sp || n < 0 || (n && (!prompt_len || !slo_ttft_us || !slo_tbt_us))) return fail(CO_EINVAL, "bad arguments");
    if (sp->base_ttft_us <= 0 || sp->base_tbt_us <= 0) return fail(CO_EINVAL, "baselines must be > 0");
    if (!(0 < sp->scale_lo && sp->scale_lo <= sp->scale_hi) || sp->chunk_budget < 1)
        return fail(CO_EINVAL, "invalid SloPolicy (workload.py:156-166 rules)");
    if (n == 0) return CO_OK;
    GenCtx G;
    if (G.init(device)) return G.r;
    uint64_t* ra = G.get<uint64_t>(n);
    uint64_t* rb = G.get<uint64_t>(n);
    if (G.r) return G.r;
    u128 st, inc;
    stream_seed(seed, 10, st, inc);
    pcg_fill(G, st, inc, n, ra);
    stream_seed(seed, 11, st, inc);
    pcg_fill(G, st, inc, n, rb);
    k_slos<<<G.grid(n), 256, 0, G.s>>>(ra, rb, prompt_len, n, sp->scale_lo, sp->scale_hi - sp->scale_lo,
                                       sp->base_ttft_us, sp->base_tbt_us, sp->chunk_budget, slo_ttft_us, slo_tbt_us);
    G.ck(cudaGetLastError());
    G.ck(cudaStreamSynchronize(G.s));
    return G.r;
}

int co_gen_predictor(int64_t n, const co_predictor_spec* sp, uint64_t seed, int device, int32_t* err,
                     uint8_t* flip) {
    CO_RANGE("co_gen_predictor");
    if (!sp || n < 0 || (n && (!err || !flip))) return fail(CO_EINVAL, "bad arguments");
    if (sp->error_dist < CO_ERR_ZERO || sp->error_dist > CO_ERR_NORMAL || !(sp->error_scale >= 0) ||
        !(sp->direction_accuracy >= 0.0 && sp->direction_accuracy <= 1.0))
        return fail(CO_EINVAL, "invalid PredictorConfig (estimation.py:29-42 rules)");
    if (n == 0) return CO_OK;
    GenCtx G;
    if (G.init(device)) return G.r;
    const int flip_on = sp->direction_accuracy < 1.0;
    const double miss = 1.0 - sp->direction_accuracy;
    u128 st, inc;
    stream_seed(seed, 3, st, inc);
    const int64_t s_int = (int64_t)sp->error_scale;  // int(cfg.error_scale)
    if (sp->error_dist == CO_ERR_NORMAL) {
        double* z = G.get<double>(n);
        double* u = flip_on ? G.get<double>(n) : nullptr;
        if (G.r) return G.r;
        if (int r = zig_stream(G, ZIG_NOR, st, inc, n, flip_on, z, u)) return r;
        k_pred_normal<<<G.grid(n), 256, 0, G.s>>>(z, u, n, sp->error_scale, miss, flip_on, err, flip);
    } else if (sp->error_dist == CO_ERR_UNIFORM && s_int > 0) {
        if (s_int >= (1ll << 31) - 1) return fail(CO_EINVAL, "error_scale too large for int32 draws");
        const int64_t R = (flip_on ? 3 * ((n + 1) / 2) + 2 : (n + 1) / 2 + 1) + 4096;
        uint64_t* raw = G.get<uint64_t>(R);
        unsigned long long* rej = G.get<unsigned long long>(1);
        int32_t* bad = G.get<int32_t>(1);
        if (G.r) return G.r;
        pcg_fill(G, st, inc, R, raw);
        G.ck(cudaMemsetAsync(rej, 0xff, 8, G.s));
        G.ck(cudaMemsetAsync(bad, 0, 4, G.s));
        k_pred_uniform<<<G.grid(n), 256, 0, G.s>>>(raw, n, (uint32_t)s_int, miss, flip_on, err, flip, rej);
        k_pred_uniform_fix<<<1, 1, 0, G.s>>>(raw, R, n, (uint32_t)s_int, miss, flip_on, err, flip, rej, bad);
        int32_t hb = 0;
        G.ck(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, G.s));
        G.ck(cudaStreamSynchronize(G.s));
        if (!G.r && hb) return fail(CO_EDEVICE, "predictor stream budget exhausted");
    } else if (flip_on) {
        uint64_t* raw = G.get<uint64_t>(n);
        if (G.r) return G.r;
        pcg_fill(G, st, inc, n, raw);
        k_pred_flip_only<<<G.grid(n), 256, 0, G.s>>>(raw, n, miss, err, flip);
    } else {
        G.ck(cudaMemsetAsync(err, 0, n * 4, G.s));
        G.ck(cudaMemsetAsync(flip, 0, n, G.s));
    }
    G.ck(cudaGetLastError());
    G.ck(cudaStreamSynchronize(G.s));
    return G.r;
}

}  // extern "C"

#include "pool_api.cuh"
#include "sched_ops.cuh"
