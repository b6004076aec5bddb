// coop_api.cu -- host side of libcoop: the C ABI declared in include/coop.h.
//
// Each blocking call: validate -> size the persistent grid from the occupancy
// API (co-residency) -> stage the control block -> one
// cooperative-attribute launch (co-residency is guaranteed or the launch
// fails; grid.sync is never used) -> read back the control block -> map the
// device error word to a coop_status.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <sched.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "../../include/coop.h"
#include "apps.cuh"
#include "part_app.cuh"
#include "part_sssp.cuh"

using namespace coop;

// ------------------------------------------------------------------ errors
static thread_local char g_err[512];
// shared with coop_dev_api.cu (the device-API half of the ABI)
char *coop_internal_errbuf() { return g_err; }

static coop_status fail(coop_status s, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return s;
}
#define CUDA_TRY(x)                                                                          \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess) {                                                             \
            cudaGetLastError();                                                              \
            return fail(COOP_ERR_CUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                 \
        }                                                                                    \
    } while (0)

extern "C" int coop_abi_version(void) { return COOP_ABI_VERSION; }

extern "C" const char *coop_status_string(coop_status s) {
    switch (s) {
        case COOP_OK: return "COOP_OK";
        case COOP_ERR_INVALID_ARG: return "COOP_ERR_INVALID_ARG";
        case COOP_ERR_CUDA: return "COOP_ERR_CUDA";
        case COOP_ERR_NOT_CORESIDENT: return "COOP_ERR_NOT_CORESIDENT";
        case COOP_ERR_FORK_BOUND: return "COOP_ERR_FORK_BOUND";
        case COOP_ERR_NO_CAPACITY: return "COOP_ERR_NO_CAPACITY";
        case COOP_ERR_TIMEOUT: return "COOP_ERR_TIMEOUT";
        case COOP_ERR_OVERFLOW: return "COOP_ERR_OVERFLOW";
        case COOP_ERR_NCCL: return "COOP_ERR_NCCL";
        case COOP_ERR_INVARIANT: return "COOP_ERR_INVARIANT";
        case COOP_ERR_BUSY: return "COOP_ERR_BUSY";
    }
    return "COOP_ERR_UNKNOWN";
}

extern "C" const char *coop_last_error(void) { return g_err; }

// ------------------------------------------------------------------ kernels
#ifndef COOP_THREADS_PER_SM
#define COOP_THREADS_PER_SM 1024
#endif
template <class App, int BLOCK>
static void *kernel_ptr() {
    // CTAs per SM the register allocation targets: 1024 threads per SM (64 registers per
    // thread) by default; COOP_THREADS_PER_SM=1536 asks for 48 warps (<= 40 registers)
    constexpr int MINB = BLOCK >= COOP_THREADS_PER_SM ? 1 : COOP_THREADS_PER_SM / BLOCK;
    return reinterpret_cast<void *>(&coop_kernel<App, BLOCK, MINB>);
}

template <class App>
static void *pick_block(uint32_t threads) {
    switch (threads) {
        case 256: return kernel_ptr<App, 256>();
        case 512: return kernel_ptr<App, 512>();
        case 1024: return kernel_ptr<App, 1024>();
        default: return nullptr;
    }
}

// the scheduler-armed specialisation (SCHEDULER + query: mid-interval offer_kill with
// hand-back), BFS and SSSP at 256 and 512 threads per workgroup; other block sizes run the
// general kernel, whose mid-interval instance is out of line
template <class App, int BLOCK>
static void *armed_kernel_ptr() {
    constexpr int MINB = BLOCK >= COOP_THREADS_PER_SM ? 1 : COOP_THREADS_PER_SM / BLOCK;
    return reinterpret_cast<void *>(&coop_kernel<App, BLOCK, MINB, true>);
}
template <class App>
static void *pick_block_armed(uint32_t threads) {
    switch (threads) {
        case 256: return armed_kernel_ptr<App, 256>();
        case 512: return armed_kernel_ptr<App, 512>();
        default: return pick_block<App>(threads);
    }
}

// plain (COOP_BARRIER_PLAIN): the separately compiled non-cooperative persistent
// kernel of the same traversal (kCoop = false: no scheduler, pool, mailboxes,
// kill/fork or chunk-claim code), the T2 baseline
static void *select_kernel(uint32_t app, int off64, uint32_t threads, bool plain, bool armed = false) {
    if (app == APP_PBFS) return off64 ? pick_block<PartBfsApp<int64_t>>(threads) : pick_block<PartBfsApp<uint32_t>>(threads);
    if (app == APP_PSSSP) return off64 ? pick_block<PartSsspApp<int64_t>>(threads) : pick_block<PartSsspApp<uint32_t>>(threads);
    if (app == APP_BFS) {
        if (plain) return off64 ? pick_block<BfsApp<int64_t, false>>(threads) : pick_block<BfsApp<uint32_t, false>>(threads);
        if (armed) return off64 ? pick_block_armed<BfsApp<int64_t>>(threads) : pick_block_armed<BfsApp<uint32_t>>(threads);
        return off64 ? pick_block<BfsApp<int64_t>>(threads) : pick_block<BfsApp<uint32_t>>(threads);
    }
    if (app == APP_SSSP) {
        if (plain) return off64 ? pick_block<SsspApp<int64_t, false>>(threads) : pick_block<SsspApp<uint32_t, false>>(threads);
        if (armed) return off64 ? pick_block_armed<SsspApp<int64_t>>(threads) : pick_block_armed<SsspApp<uint32_t>>(threads);
        return off64 ? pick_block<SsspApp<int64_t>>(threads) : pick_block<SsspApp<uint32_t>>(threads);
    }
    switch (threads) {
        case 128: return kernel_ptr<BarrierApp, 128>();
        case 256: return kernel_ptr<BarrierApp, 256>();
        case 512: return kernel_ptr<BarrierApp, 512>();
        case 1024: return kernel_ptr<BarrierApp, 1024>();
    }
    return nullptr;
}

// control block + mailboxes of one call: zero, then the generation-0 words and the pool
__global__ void ctl_init_kernel(Ctl *c, uint32_t P, uint32_t M0) {
    unsigned long long *w = reinterpret_cast<unsigned long long *>(c);
    const uint32_t n = (uint32_t)((sizeof(Ctl) + sizeof(Mailbox) * P) / 8);   // mailboxes follow the block
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) w[i] = 0ull;
    __syncthreads();
    if (threadIdx.x == 0) {
        c->W = pack_w(0, M0, 0);
        c->R = pack_w(0, M0, 0);
        c->mhist[0] = M0;
        c->min_m = M0;
        c->max_m = M0;
        c->task_next = 0xFFFFFFFFu;
    }
    for (uint32_t b = M0 + threadIdx.x; b < P; b += blockDim.x) atomicOr(&c->pool[b >> 5], 1u << (b & 31));
}

__global__ void max_u32_kernel(const uint32_t *w, int64_t n, uint32_t *out) {
    uint32_t m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, w[i]);
    for (int s = 16; s; s >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, s));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// probe records {degree << 32 | first neighbour} (coop_csr_probe): coalesced offsets in,
// one column per vertex, coalesced records out
template <typename OffT>
__global__ void probe_kernel(const OffT *ro, const int32_t *col, int64_t V, unsigned long long *out) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
        const OffT b = ro[v], e = ro[v + 1];
        const uint32_t d = (uint32_t)(e - b);
        const uint32_t f = d ? (uint32_t)__ldg(col + b) : 0xFFFFFFFFu;
        out[v] = ((unsigned long long)d << 32) | f;
    }
}

// degree-zero bitmap (coop_csr_isolated): warp per 32-vertex word, one coalesced offsets load
template <typename OffT>
__global__ void isolated_kernel(const OffT *ro, int64_t V, uint32_t *bits) {
    const uint32_t lane = threadIdx.x & 31;
    const int64_t nw = (V + 31) / 32;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; w < nw;
         w += (int64_t)gridDim.x * blockDim.x / 32) {
        const int64_t v = w * 32 + lane;
        const bool iso = v < V && ro[v + 1] == ro[v];
        const uint32_t m = __ballot_sync(0xffffffffu, iso);
        if (lane == 0) bits[w] = m;
    }
}

// L2 round-trip microbenchmark (the barrier's latency denominator): one thread on each
// of 8 SMs spread over both dies (picked by %smid, the first CTA landing on the SM) runs
// a dependent chain of `iters` operations on its own 128-B line; kinds:
//   0 atom.relaxed.gpu.add.u64   1 atom.relaxed.gpu.add.u32   2 atom.acq_rel.gpu.add.u64
//   3 ld.acquire.gpu.u64
// out_ns[kind * 8 + k] = ns per operation on the k-th chosen SM.
__global__ void l2_rtt_kernel(unsigned long long *words, uint32_t *claimed, uint64_t iters, double *out_ns) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const uint32_t nsm = gridDim.x;
    int k = -1;
    for (int j = 0; j < 8; ++j)
        if (smid == (uint32_t)j * (nsm / 8)) k = j;
    if (k < 0 || threadIdx.x != 0 || atomicCAS(claimed + k, 0u, 1u) != 0u) return;
    unsigned long long *w = words + 16 * k;                       // own 128-B line
    for (int kind = 0; kind < 4; ++kind) {
        unsigned long long v = 0;
        const uint64_t t0 = globaltimer();
        for (uint64_t i = 0; i < iters; ++i) {
            unsigned long long *a = w + (v >> 63);                 // dependent address (v < 2^63)
            if (kind == 0) v = atomicAdd(a, 1ull);
            else if (kind == 1) v = atomicAdd(reinterpret_cast<unsigned int *>(a), 1u) & 0x7FFFFFFFu;
            else if (kind == 2) v = coop_proto::atom_add_acq_rel64(a, 1ull);
            else v = coop_proto::ld_acquire64(a) & 0x7FFFFFFFFFFFFFFFull;
        }
        const uint64_t t1 = globaltimer();
        out_ns[kind * 8 + k] = (double)(t1 - t0) / (double)iters + (v == ~0ull ? 1.0 : 0.0);
    }
}

// ------------------------------------------------------------------ scratch
// Scratch grows with stream-ordered allocations on the call's stream: a
// cudaFree/cudaMalloc would synchronise the device and deadlock against a
// running persistent kernel of another rank sharing the GPU (tests).
static thread_local cudaStream_t g_alloc_stream = nullptr;

struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t n) {
        if (n <= cap) return cudaSuccess;
        if (p) cudaFreeAsync(p, g_alloc_stream);
        p = nullptr;
        cap = 0;
        size_t want = std::max<size_t>(n, 256);
        cudaError_t e = cudaMallocAsync(&p, want, g_alloc_stream);
        if (e == cudaSuccess) cap = want;
        return e;
    }
};

struct Scratch {
    int device = -1;
    DevBuf ctl, lt, mb, visited, qlev, ql0, ql1, qh0, qh1, stamp, mtrace, lsizes, events, script, wmax, fb0, fb1, fb2,
        far0, far1;
    DevBuf h_ro, h_col, h_w, h_out;   // end-to-end (host-pointer) calls
    DevBuf nccl_aux;                  // NCCL data plane: ready, gathered, count send/recv slots
    DevBuf runt;                      // source loop: end time of every run
    DevBuf rep;                       // hand-back entries of mid-interval offer_kill [P][W]
    DevBuf lv8;                       // BFS: one level byte per vertex during the traversal
    cudaEvent_t done_ev = nullptr;    // handle API: the control block's copy back has landed
    volatile uint32_t *nccl_host = nullptr;     // mapped host mirror of `ready`
    void *nccl_warm = nullptr;                  // communicator already warmed up on nccl_stream
    cudaStream_t nccl_stream = nullptr;         // the comm stream (waits, all-gathers, writes)
    cudaEvent_t nccl_ev = nullptr;
    Ctl *host_ctl = nullptr;          // pinned, host-mapped: the kernel's last CTA mirrors the control block here
    Ctl *host_ctl_dev = nullptr;      // its device pointer
    std::mutex mu;
};

constexpr uint32_t kWorkspaces = 8;
constexpr uint32_t kNcclReserve = 16;     // CTA slots left to NCCL kernels (coop_bfs_part_nccl)
constexpr uint32_t kDefaultAlpha = 14;   // Beamer et al.'s direction-switch thresholds (reading R14)
constexpr uint32_t kDefaultBeta = 24;
static Scratch g_scratch[16][kWorkspaces];

static coop_status get_scratch(Scratch **out, uint32_t ws) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 16) return fail(COOP_ERR_INVALID_ARG, "device %d out of range", dev);
    if (ws >= kWorkspaces) return fail(COOP_ERR_INVALID_ARG, "workspace %u out of range [0, %u)", ws, kWorkspaces);
    Scratch *s = &g_scratch[dev][ws];
    if (!s->host_ctl) {   // all workspaces of the device at once (no allocation while a kernel runs)
        for (uint32_t k = 0; k < kWorkspaces; ++k)
            if (!g_scratch[dev][k].host_ctl) {
                // control block + zeroed mailboxes: one pinned staging buffer, one H2D copy per call
                const size_t bytes = sizeof(Ctl) + sizeof(Mailbox) * kMaxCtas;
                CUDA_TRY(cudaHostAlloc((void **)&g_scratch[dev][k].host_ctl, bytes, cudaHostAllocMapped));
                memset((void *)g_scratch[dev][k].host_ctl, 0, bytes);
                CUDA_TRY(cudaHostGetDevicePointer((void **)&g_scratch[dev][k].host_ctl_dev,
                                                  (void *)g_scratch[dev][k].host_ctl, 0));
            }
    }
    s->device = dev;
    *out = s;
    return COOP_OK;
}

// ------------------------------------------------------------------ device info
// co-residency capacity, cached per (device, kernel, block size): the occupancy query is a
// host-side cost on every call otherwise (the GPU idles while the next call prepares)
static coop_status occupancy(void *kern, uint32_t threads, int *sm_count, int *per_sm) {
    struct Entry { int dev; void *kern; uint32_t threads; int sms, per; };
    static std::mutex mu;
    static std::vector<Entry> cache;
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(mu);
        for (const Entry &e : cache)
            if (e.dev == dev && e.kern == kern && e.threads == threads) {
                *sm_count = e.sms;
                *per_sm = e.per;
                return COOP_OK;
            }
    }
    CUDA_TRY(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev));
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kern, (int)threads, 0));
    std::lock_guard<std::mutex> lk(mu);
    cache.push_back(Entry{dev, kern, threads, *sm_count, *per_sm});
    return COOP_OK;
}

extern "C" coop_status coop_csr_probe(const coop_csr *g, uint64_t *probe_out, void *stream) {
    if (!g || !probe_out || !g->row_offsets || (!g->col_idx && g->num_edges > 0))
        return fail(COOP_ERR_INVALID_ARG, "NULL graph / output");
    if (g->num_vertices < 1 || g->num_vertices > (int64_t)INT32_MAX) return fail(COOP_ERR_INVALID_ARG, "bad V");
    if (g->offset_bits != 32 && g->offset_bits != 64) return fail(COOP_ERR_INVALID_ARG, "offset_bits must be 32 or 64");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    unsigned long long *out = reinterpret_cast<unsigned long long *>(probe_out);
    int dev = 0, sms = 148;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (g->offset_bits == 32)
        probe_kernel<<<sms * 8, 256, 0, s>>>(static_cast<const uint32_t *>(g->row_offsets), g->col_idx, g->num_vertices, out);
    else
        probe_kernel<<<sms * 8, 256, 0, s>>>(static_cast<const unsigned long long *>(g->row_offsets), g->col_idx,
                                             g->num_vertices, out);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(s));
    return COOP_OK;
}

extern "C" coop_status coop_csr_isolated(const coop_csr *g, uint32_t *bits_out, void *stream) {
    if (!g || !bits_out || !g->row_offsets) return fail(COOP_ERR_INVALID_ARG, "NULL graph / output");
    if (g->num_vertices < 1 || g->num_vertices > (int64_t)INT32_MAX) return fail(COOP_ERR_INVALID_ARG, "bad V");
    if (g->offset_bits != 32 && g->offset_bits != 64) return fail(COOP_ERR_INVALID_ARG, "offset_bits must be 32 or 64");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int dev = 0, sms = 148;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (g->offset_bits == 32)
        isolated_kernel<<<sms * 8, 256, 0, s>>>(static_cast<const uint32_t *>(g->row_offsets), g->num_vertices, bits_out);
    else
        isolated_kernel<<<sms * 8, 256, 0, s>>>(static_cast<const unsigned long long *>(g->row_offsets),
                                                g->num_vertices, bits_out);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(s));
    return COOP_OK;
}

extern "C" coop_status coop_device_query(int device, uint32_t threads_per_wg, coop_device_info *out) {
    if (!out) return fail(COOP_ERR_INVALID_ARG, "out is NULL");
    if (threads_per_wg == 0) threads_per_wg = 512;
    void *k = select_kernel(APP_BFS, 0, threads_per_wg, false);
    if (!k) return fail(COOP_ERR_INVALID_ARG, "threads_per_wg %u not supported (256/512/1024)", threads_per_wg);
    int cur = 0;
    CUDA_TRY(cudaGetDevice(&cur));
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    int sms = 0, per = 0;
    coop_status st = occupancy(k, threads_per_wg, &sms, &per);
    cudaFuncAttributes fa;
    CUDA_TRY(cudaFuncGetAttributes(&fa, k));
    CUDA_TRY(cudaSetDevice(cur));
    if (st != COOP_OK) return st;
    out->device = device;
    out->sm_count = sms;
    out->max_ctas_per_sm = per;
    out->max_coresident = sms * per;
    out->regs_per_thread = fa.numRegs;
    out->l2_bytes = (size_t)prop.l2CacheSize;
    out->hbm_bytes = prop.totalGlobalMem;
    return COOP_OK;
}

// ------------------------------------------------------------------ launch core
// buffers of the NCCL data plane (per workspace; see coop_bfs_part_nccl)
struct NcclExt {
    uint32_t *ready, *gathered;
    unsigned long long *cnt_send, *cnt_recv;
    volatile uint32_t *host_ready;     // device pointer of the mapped host word
    uint64_t slice_words;
};

struct RunReq {
    uint32_t app;
    const coop_csr *g;
    const coop_part *part;      // APP_PBFS
    int64_t source;
    void *out;
    const coop_opts *opts;
    coop_stats *stats;
    uint64_t iters;             // barrier bench
    HostChannel *host;          // handle API (device pointer of mapped host memory)
    bool async;                 // do not synchronise (handle API)
    const NcclExt *nx;          // APP_PBFS with the NCCL data plane (coop_bfs_part_nccl)
    const uint32_t *part_w;     // APP_PSSSP: weights of the local edges
    const int64_t *sources;     // APP_BFS source loop (coop_bfs_loop): device array
    uint32_t n_src;
    uint64_t loop_ns;
    uint32_t run_cap;
};

static coop_status fill_stats(const Ctl &c, const KParams &kp, coop_stats *st, cudaStream_t stream) {
    if (!st) return COOP_OK;
    st->kernel_ns = c.t_end > c.t_start ? c.t_end - c.t_start : 0;
    st->edges_scanned = c.edges_scanned;
    st->frontier_total = c.frontier_total;
    st->reached = c.reached;
    st->levels = c.levels;
    st->episodes = c.episode;
    st->kills = c.kills;
    st->forks = c.forks;
    st->min_m = c.min_m;
    st->max_m = c.max_m;
    st->n_wgs = kp.P;
    st->tasks_posted = c.tasks_posted;
    st->tasks_completed = c.tasks_completed;
    st->bottom_up_levels = c.n_bu_levels;
    st->mid_kills = c.mid_kills;
    st->handbacks = c.handbacks;
    st->replays = c.replays;
    bool pending = false;   // async copies to wait for (only then: a pipelined caller's next
                            // kernel may already be queued on this stream)
    if (st->m_trace && st->m_trace_cap) {
        uint32_t n = std::min(st->m_trace_cap, std::min(c.episode, kp.m_trace_cap));
        if (n) CUDA_TRY(cudaMemcpyAsync(st->m_trace, kp.m_trace, n * 4, cudaMemcpyDeviceToHost, stream));
        pending |= n != 0;
    }
    if (st->level_sizes && st->level_sizes_cap) {
        uint32_t n = std::min(st->level_sizes_cap, std::min(c.levels + 1, kp.level_cap));
        if (n) CUDA_TRY(cudaMemcpyAsync(st->level_sizes, kp.level_sizes, n * 4, cudaMemcpyDeviceToHost, stream));
        pending |= n != 0;
    }
    if (st->level_end_ns && st->level_end_ns_cap) {
        uint32_t n = std::min(st->level_end_ns_cap, std::min(c.levels, kp.level_cap));
        std::vector<unsigned long long> tmp(n);
        if (n) {
            CUDA_TRY(cudaMemcpyAsync(tmp.data(), kp.level_t, n * 8, cudaMemcpyDeviceToHost, stream));
            CUDA_TRY(cudaStreamSynchronize(stream));
        }
        for (uint32_t i = 0; i < n; ++i) st->level_end_ns[i] = tmp[i] > c.t_start ? tmp[i] - c.t_start : 0;
    }
    if (st->task_events && st->task_events_cap) {
        uint32_t n = std::min(st->task_events_cap, c.n_events);
        std::vector<TaskEventDev> tmp(n);
        if (n) {
            CUDA_TRY(cudaMemcpyAsync(tmp.data(), kp.events, n * sizeof(TaskEventDev), cudaMemcpyDeviceToHost, stream));
            CUDA_TRY(cudaStreamSynchronize(stream));
        }
        for (uint32_t i = 0; i < n; ++i) {
            st->task_events[i].t_arrive = tmp[i].t_arrive;
            st->task_events[i].t_first_surrender = tmp[i].t_first_surrender;
            st->task_events[i].t_last_surrender = tmp[i].t_last_surrender;
            st->task_events[i].t_first_start = tmp[i].t_first_start;
            st->task_events[i].t_end = tmp[i].t_end;
            st->task_events[i].demanded = tmp[i].demanded;
            st->task_events[i].surrendered = tmp[i].surrendered;
        }
    }
    if (pending) CUDA_TRY(cudaStreamSynchronize(stream));
    return COOP_OK;
}

static coop_status map_err(const Ctl &c) {
    switch (c.err) {
        case DERR_NONE: return COOP_OK;
        case DERR_TIMEOUT: return fail(COOP_ERR_TIMEOUT, "in-kernel watchdog fired (episode %u)", c.episode);
        case DERR_INVARIANT: return fail(COOP_ERR_INVARIANT, "barrier invariant violated (%u violations)", c.violations);
        case DERR_OVERFLOW: return fail(COOP_ERR_OVERFLOW, "distance overflow");
    }
    return fail(COOP_ERR_INVARIANT, "unknown device error %u", c.err);
}

struct Prepared {
    KParams kp;
    void *kern;
    uint32_t grid, threads;
    cudaStream_t stream;
    Scratch *s;
    cudaEvent_t ev0, ev1;
    bool ctl_copied = false;    // handle API: the control block's D2H copy is already enqueued
};

static coop_status prepare(const RunReq &r, Prepared *pr) {
    static const coop_opts kDefault = {};
    const coop_opts &o = r.opts ? *r.opts : kDefault;
    g_alloc_stream = static_cast<cudaStream_t>(o.stream);
    Scratch *s = nullptr;
    coop_status st = get_scratch(&s, o.workspace);
    if (st != COOP_OK) return st;
    KParams kp;
    memset(&kp, 0, sizeof kp);
    kp.app = r.app;
    const uint32_t threads = o.threads_per_wg ? o.threads_per_wg : (r.app == APP_BARRIER ? 128u : 512u);
    int off64 = 0;
    if (r.app == APP_PBFS || r.app == APP_PSSSP) {
        const coop_part *pt = r.part;
        if (!pt) return fail(COOP_ERR_INVALID_ARG, "part is NULL");
        if (pt->num_vertices < 1 || pt->num_vertices > (int64_t)INT32_MAX)
            return fail(COOP_ERR_INVALID_ARG, "num_vertices out of range");
        if (pt->nranks < 1 || pt->nranks > COOP_MAX_RANKS || pt->rank < 0 || pt->rank >= pt->nranks)
            return fail(COOP_ERR_INVALID_ARG, "rank %d / nranks %d invalid", pt->rank, pt->nranks);
        if (pt->v_begin < 0 || pt->v_end > pt->num_vertices || pt->v_begin > pt->v_end ||
            ((pt->v_begin & 31) && pt->v_begin != pt->num_vertices))   // an empty trailing rank may start at V
            return fail(COOP_ERR_INVALID_ARG, "owned range [%lld, %lld) invalid (v_begin %% 32 == 0 required)",
                        (long long)pt->v_begin, (long long)pt->v_end);
        if (pt->offset_bits != 32 && pt->offset_bits != 64) return fail(COOP_ERR_INVALID_ARG, "offset_bits");
        if (!pt->row_offsets || (!pt->col_local && pt->num_edges > 0)) return fail(COOP_ERR_INVALID_ARG, "CSR NULL");
        if (pt->num_hubs && (!pt->hub_ids || !pt->hub_prefix || !pt->hub_degree))
            return fail(COOP_ERR_INVALID_ARG, "hub arrays NULL");
        for (int q = 0; q < pt->nranks; ++q)   // the NCCL data plane uses only this rank's bitmaps
            if ((!r.nx || q == pt->rank) && (!pt->frontier[q][0] || !pt->frontier[q][1] || (!r.nx && !pt->flags[q])))
                return fail(COOP_ERR_INVALID_ARG, "exchange buffers of rank %d NULL", q);
        if (r.source < 0 || r.source >= pt->num_vertices) return fail(COOP_ERR_INVALID_ARG, "source out of range");
        if (!r.out) return fail(COOP_ERR_INVALID_ARG, "output buffer is NULL");
        off64 = pt->offset_bits == 64;
        kp.V = pt->num_vertices;
        kp.ro = pt->row_offsets;
        kp.off64 = off64;
        kp.col = pt->col_local;
        kp.source = r.source;
        kp.E = pt->num_edges;
        kp.level_out = static_cast<int32_t *>(r.out);
        PartParams &pp = kp.part;
        pp.vb = pt->v_begin;
        pp.ve = pt->v_end;
        pp.rank = pt->rank;
        pp.nranks = pt->nranks;
        pp.seq = pt->seq;
        pp.nhub = pt->num_hubs;
        pp.hub_deg = pt->hub_degree;
        pp.hub_ids = pt->hub_ids;
        pp.hub_prefix = reinterpret_cast<const unsigned long long *>(pt->hub_prefix);
        for (int q = 0; q < pt->nranks; ++q) {
            pp.F[q][0] = pt->frontier[q][0];
            pp.F[q][1] = pt->frontier[q][1];
            pp.flags[q] = reinterpret_cast<unsigned long long *>(pt->flags[q]);
        }
        if (r.nx) {
            pp.nccl = 1;
            pp.ready = r.nx->ready;
            pp.gathered = r.nx->gathered;
            pp.cnt_send = r.nx->cnt_send;
            pp.cnt_recv = r.nx->cnt_recv;
            pp.host_ready = r.nx->host_ready;
            pp.slice_words = r.nx->slice_words;
        }
        if (r.app == APP_PSSSP) {
            if (!r.part_w && pt->num_edges > 0) return fail(COOP_ERR_INVALID_ARG, "partitioned SSSP needs weights");
            // inbox offsets of every source rank: the uniform slices of graphgen.part_bounds
            const uint64_t nw = ((uint64_t)pt->num_vertices + 31) / 32, sw = (nw + pt->nranks - 1) / pt->nranks;
            for (int q = 0; q <= pt->nranks; ++q)
                pp.qvb[q] = std::min<int64_t>(pt->num_vertices, (int64_t)(32 * sw * q));
            pp.qvb[pt->nranks] = pt->num_vertices;
            if (pp.qvb[pt->rank] != pt->v_begin || pp.qvb[pt->rank + 1] != pt->v_end)
                return fail(COOP_ERR_INVALID_ARG, "partitioned SSSP needs the uniform slices of graphgen.part_bounds");
            kp.w = r.part_w;
            kp.dist_out = static_cast<uint32_t *>(r.out);
            kp.level_out = nullptr;
        }
        if (o.flags & COOP_FLAG_DIROPT && r.app == APP_PBFS) {
            if (!pt->rows_offsets || (!pt->rows_col && pt->v_end > pt->v_begin) || pt->num_edges_global <= 0)
                return fail(COOP_ERR_INVALID_ARG, "COOP_FLAG_DIROPT needs rows_offsets / rows_col / num_edges_global");
            pp.rro = pt->rows_offsets;
            pp.rcol = pt->rows_col;
            pp.E_global = pt->num_edges_global;
            kp.dopt = 1;
        }
    } else if (r.app != APP_BARRIER) {
        const coop_csr *g = r.g;
        if (!g) return fail(COOP_ERR_INVALID_ARG, "graph is NULL");
        if (g->num_vertices < 1 || g->num_vertices > (int64_t)INT32_MAX)
            return fail(COOP_ERR_INVALID_ARG, "num_vertices %lld out of range [1, 2^31-1]", (long long)g->num_vertices);
        if (g->num_edges < 0) return fail(COOP_ERR_INVALID_ARG, "num_edges < 0");
        if (g->offset_bits != 32 && g->offset_bits != 64) return fail(COOP_ERR_INVALID_ARG, "offset_bits must be 32 or 64");
        if (g->offset_bits == 32 && g->num_edges > (int64_t)UINT32_MAX)
            return fail(COOP_ERR_INVALID_ARG, "num_edges needs 64-bit offsets");
        if (!g->row_offsets || (!g->col_idx && g->num_edges > 0))
            return fail(COOP_ERR_INVALID_ARG, "row_offsets/col_idx NULL");
        if (r.source < 0 || r.source >= g->num_vertices)
            return fail(COOP_ERR_INVALID_ARG, "source %lld out of range [0, %lld)", (long long)r.source, (long long)g->num_vertices);
        if (!r.out) return fail(COOP_ERR_INVALID_ARG, "output buffer is NULL");
        if (r.app == APP_SSSP && !g->weights && g->num_edges > 0) return fail(COOP_ERR_INVALID_ARG, "SSSP needs weights");
        off64 = g->offset_bits == 64;
        kp.V = g->num_vertices;
        kp.ro = g->row_offsets;
        kp.off64 = off64;
        kp.col = g->col_idx;
        kp.w = g->weights;
        kp.probe = reinterpret_cast<const unsigned long long *>(g->probe);
        kp.iso = g->isolated;
        kp.source = r.source;
        kp.E = g->num_edges;
        if (r.app == APP_BFS) kp.level_out = static_cast<int32_t *>(r.out);
        else kp.dist_out = static_cast<uint32_t *>(r.out);
    }
    void *kern = select_kernel(r.app, off64, threads, o.barrier_mode == COOP_BARRIER_PLAIN,
                               o.policy == COOP_POLICY_SCHEDULER && o.barrier_mode == COOP_BARRIER_QUERY);
    if (!kern) return fail(COOP_ERR_INVALID_ARG, "threads_per_wg %u not supported", threads);
    int sms = 0, per = 0;
    st = occupancy(kern, threads, &sms, &per);
    if (st != COOP_OK) return st;
    const uint32_t cap = (uint32_t)(sms * per);
    const bool plain = o.barrier_mode == COOP_BARRIER_PLAIN;
    if (o.barrier_mode > COOP_BARRIER_NAIVE) return fail(COOP_ERR_INVALID_ARG, "bad barrier_mode %u", o.barrier_mode);
    if (o.policy > COOP_POLICY_SCHEDULER) return fail(COOP_ERR_INVALID_ARG, "bad policy %u", o.policy);
    const bool sched = !plain && (o.policy == COOP_POLICY_SCHEDULER);
    // the NCCL data plane needs free CTA slots for NCCL's own kernels while the
    // persistent kernel waits for the gather (kNcclReserve slots left free by default)
    const uint32_t reserve = (r.nx && cap > 2 * kNcclReserve) ? kNcclReserve : 0u;
    uint32_t P = o.max_wgs ? o.max_wgs : cap - (sched ? 1 : 0) - reserve;
    if (P < 1 || P > kMaxCtas) return fail(COOP_ERR_INVALID_ARG, "max_wgs %u out of range [1, %u]", P, kMaxCtas);
    if (P + (sched ? 1 : 0) > cap)
        return fail(COOP_ERR_NOT_CORESIDENT, "%u workgroups%s exceed the co-resident capacity %u (%d SMs x %d)",
                    P, sched ? " + scheduler" : "", cap, sms, per);
    uint32_t M0 = o.init_wgs ? o.init_wgs : P;
    if (M0 < 1 || M0 > P) return fail(COOP_ERR_INVALID_ARG, "init_wgs %u not in [1, %u]", M0, P);
    if (plain) M0 = P;
    const uint32_t bpl = (r.app == APP_PBFS || r.app == APP_PSSSP) ? 2u : (o.barriers_per_level ? o.barriers_per_level : 1);
    if (bpl != 1 && bpl != 2) return fail(COOP_ERR_INVALID_ARG, "barriers_per_level must be 1 or 2");
    if (o.policy == COOP_POLICY_SCRIPTED && o.script_len && !o.script) return fail(COOP_ERR_INVALID_ARG, "script NULL");
    if (o.resize_prob < 0 || o.resize_prob > 1) return fail(COOP_ERR_INVALID_ARG, "resize_prob not in [0,1]");
    if (sched && (o.task_period_ns || r.host)) {
        if (o.task_period_ns && (o.task_wgs < 1 || o.task_wgs > P - 1))
            return fail(COOP_ERR_NO_CAPACITY, "task_wgs %u not in [1, N-1=%u] (WG 0 is never killed, P:543)", o.task_wgs, P - 1);
    }
    if (r.app == APP_SSSP) {
        uint32_t wmax = r.g->max_weight;
        if (!wmax && r.g->num_edges > 0) {
            CUDA_TRY(s->wmax.ensure(4));
            cudaStream_t st0 = static_cast<cudaStream_t>(o.stream);
            CUDA_TRY(cudaMemsetAsync(s->wmax.p, 0, 4, st0));
            max_u32_kernel<<<296, 256, 0, st0>>>(r.g->weights, r.g->num_edges, static_cast<uint32_t *>(s->wmax.p));
            CUDA_TRY(cudaGetLastError());
            CUDA_TRY(cudaMemcpyAsync(&wmax, s->wmax.p, 4, cudaMemcpyDeviceToHost, st0));
            CUDA_TRY(cudaStreamSynchronize(st0));
        }
        if ((uint64_t)(r.g->num_vertices - 1) * wmax >= 0xFFFFFFFFull)
            return fail(COOP_ERR_OVERFLOW, "(V-1)*max_weight = %llu >= 2^32-1", (unsigned long long)(r.g->num_vertices - 1) * wmax);
    }

    // ---- scratch
    const uint64_t V = r.app == APP_BARRIER ? 0 : (uint64_t)kp.V;
    const uint64_t E = (r.app == APP_BARRIER || r.app == APP_PBFS || r.app == APP_PSSSP) ? 0 : (uint64_t)r.g->num_edges;
    CUDA_TRY(s->ctl.ensure(sizeof(Ctl) + sizeof(Mailbox) * kMaxCtas));   // mailboxes follow the control block
    CUDA_TRY(s->stamp.ensure(4ull * kMaxCtas));
    const uint32_t mcap = 1u << 16, lcap = 1u << 16, ecap = 4096;
    CUDA_TRY(s->mtrace.ensure(4ull * mcap));
    CUDA_TRY(s->lsizes.ensure(4ull * lcap));
    CUDA_TRY(s->lt.ensure(8ull * lcap));
    CUDA_TRY(s->events.ensure(sizeof(TaskEventDev) * ecap));
    if (r.app == APP_BFS) {
        const size_t le = off64 ? sizeof(LightEntry64) : sizeof(LightEntry);
        // light queues: per-warp reservations of 256 slots may leave holes (empty
        // entries): at most one partly used reservation per refill (< 128 unused
        // slots, refills hold >= 128 entries) plus one open reservation per warp
        const size_t qcap = 2 * V + (size_t)P * (threads / 32) * 256;
        CUDA_TRY(s->visited.ensure(4 * ((V + 31) / 32)));
        CUDA_TRY(s->lv8.ensure(4 * ((V + 3) / 4)));
        kp.lv8 = static_cast<uint8_t *>(s->lv8.p);
        CUDA_TRY(s->ql0.ensure(le * qcap));
        CUDA_TRY(s->ql1.ensure(le * qcap));
        const size_t nh = E / kHeavyDeg + 1;
        CUDA_TRY(s->qh0.ensure(sizeof(HeavyEntry) * nh));
        CUDA_TRY(s->qh1.ensure(sizeof(HeavyEntry) * nh));
        kp.visited = static_cast<uint32_t *>(s->visited.p);
        if (o.flags & COOP_FLAG_DIROPT) {
            const size_t fbytes = 4 * ((V + 31) / 32);
            CUDA_TRY(s->fb0.ensure(fbytes));
            CUDA_TRY(s->fb1.ensure(fbytes));
            CUDA_TRY(s->fb2.ensure(fbytes));
            kp.fbits[0] = static_cast<uint32_t *>(s->fb0.p);
            kp.fbits[1] = static_cast<uint32_t *>(s->fb1.p);
            kp.fbits[2] = static_cast<uint32_t *>(s->fb2.p);
            kp.dopt = 1;
        }
        kp.qheavy[0] = static_cast<HeavyEntry *>(s->qh0.p);
        kp.qheavy[1] = static_cast<HeavyEntry *>(s->qh1.p);
    } else if (r.app == APP_PBFS) {
        const uint64_t nown = (uint64_t)(kp.part.ve - kp.part.vb);
        CUDA_TRY(s->visited.ensure(4 * ((nown + 31) / 32) + 4));
        kp.visited = static_cast<uint32_t *>(s->visited.p);
    } else if (r.app == APP_PSSSP) {
        const uint64_t nown = (uint64_t)(kp.part.ve - kp.part.vb);
        CUDA_TRY(s->qlev.ensure(8 * nown + 8));
        CUDA_TRY(s->ql0.ensure(4 * nown + 4));
        CUDA_TRY(s->ql1.ensure(4 * nown + 4));
        kp.dq = static_cast<unsigned long long *>(s->qlev.p);
        kp.part.list[0] = static_cast<uint32_t *>(s->ql0.p);
        kp.part.list[1] = static_cast<uint32_t *>(s->ql1.p);
    } else if (r.app == APP_SSSP) {
        CUDA_TRY(s->qlev.ensure(8 * V));
        CUDA_TRY(s->ql0.ensure(4 * V));
        CUDA_TRY(s->ql1.ensure(4 * V));
        kp.dq = static_cast<unsigned long long *>(s->qlev.p);
        if (o.sssp_delta) {   // far piles: every entry is one distance improvement, so <= E + V
            CUDA_TRY(s->far0.ensure(4 * (E + V)));
            CUDA_TRY(s->far1.ensure(4 * (E + V)));
            kp.far[0] = static_cast<uint32_t *>(s->far0.p);
            kp.far[1] = static_cast<uint32_t *>(s->far1.p);
            kp.delta = o.sssp_delta;
            kp.far_cap = (uint32_t)std::min<uint64_t>(E + V, 0xFFFFFFFFull);
        }
    }
    kp.qlight[0] = s->ql0.p;
    kp.qlight[1] = s->ql1.p;
    kp.ctl = static_cast<Ctl *>(s->ctl.p);
    kp.mb = reinterpret_cast<Mailbox *>(static_cast<char *>(s->ctl.p) + sizeof(Ctl));
    kp.stamp = static_cast<uint32_t *>(s->stamp.p);
    if (sched && o.barrier_mode == COOP_BARRIER_QUERY) {   // mid-interval offer_kill hands items back
        CUDA_TRY(s->rep.ensure(sizeof(RepEntry) * (size_t)P * (threads / 32)));
        kp.rep = static_cast<RepEntry *>(s->rep.p);
    }
    kp.m_trace = static_cast<uint32_t *>(s->mtrace.p);
    kp.m_trace_cap = mcap;
    kp.level_sizes = static_cast<uint32_t *>(s->lsizes.p);
    kp.level_t = static_cast<unsigned long long *>(s->lt.p);
    kp.level_cap = lcap;
    kp.events = static_cast<TaskEventDev *>(s->events.p);
    kp.events_cap = ecap;
    cudaStream_t stream = static_cast<cudaStream_t>(o.stream);
    if (o.policy == COOP_POLICY_SCRIPTED && o.script_len) {
        CUDA_TRY(s->script.ensure(4ull * o.script_len));
        CUDA_TRY(cudaMemcpyAsync(s->script.p, o.script, 4ull * o.script_len, cudaMemcpyHostToDevice, stream));
        kp.script = static_cast<const uint32_t *>(s->script.p);
        kp.script_len = o.script_len;
    }
    kp.host = r.host;
    kp.alpha = o.bfs_alpha ? o.bfs_alpha : kDefaultAlpha;   // direction-switch thresholds (Beamer et al.)
    kp.beta = o.bfs_beta ? o.bfs_beta : kDefaultBeta;
    kp.P = P;
    kp.M0 = M0;
    kp.policy = plain ? COOP_POLICY_NEVER : o.policy;
    kp.barrier_mode = o.barrier_mode;
    kp.bpl = bpl;
    kp.flags = o.flags;
    kp.has_sched = sched ? 1 : 0;
    kp.seed = o.seed;
    kp.resize_thresh = (uint32_t)std::min(4294967295.0, o.resize_prob * 4294967296.0);
    kp.timeout_ns = o.timeout_ns ? o.timeout_ns : 20000000000ull;
    kp.iters = r.iters;
    kp.task_wgs = o.task_wgs;
    kp.task_blocks = o.task_blocks ? o.task_blocks : 1;
    kp.task_max = o.task_max;
    kp.task_block_ns = o.task_block_ns;
    kp.task_period_ns = sched ? o.task_period_ns : 0;
    kp.task_first_ns = o.task_first_ns;
    if (r.sources) {
        CUDA_TRY(s->runt.ensure(8ull * std::max(1u, r.run_cap)));
        kp.sources = r.sources;
        kp.n_src = r.n_src;
        kp.loop_ns = r.loop_ns;
        kp.run_t = static_cast<unsigned long long *>(s->runt.p);
        kp.run_cap = r.run_cap;
        if (!o.timeout_ns) kp.timeout_ns = r.loop_ns + 20000000000ull;
    }

    // ---- control block
    // the control block and the P mailboxes behind it, initialised on the device (no
    // host-to-device copy per call); the kernel's last CTA mirrors the block back
    kp.ctl_mirror = s->host_ctl_dev;
    ctl_init_kernel<<<1, 512, 0, stream>>>(kp.ctl, P, M0);
    CUDA_TRY(cudaGetLastError());
    if (sched) CUDA_TRY(cudaMemsetAsync(kp.events, 0, sizeof(TaskEventDev) * ecap, stream));
    pr->kp = kp;
    pr->kern = kern;
    pr->grid = P + (sched ? 1 : 0);
    pr->threads = threads;
    pr->stream = stream;
    pr->s = s;
    pr->ev0 = static_cast<cudaEvent_t>(o.ev_kernel_start);
    pr->ev1 = static_cast<cudaEvent_t>(o.ev_kernel_end);
    return COOP_OK;
}

static coop_status launch(Prepared &pr) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pr.grid);
    cfg.blockDim = dim3(pr.threads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = pr.stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;   // co-residency guarantee only; no grid.sync anywhere
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void *args[] = {&pr.kp};
    if (pr.ev0) CUDA_TRY(cudaEventRecord(pr.ev0, pr.stream));
    CUDA_TRY(cudaLaunchKernelExC(&cfg, pr.kern, args));
    if (pr.ev1) CUDA_TRY(cudaEventRecord(pr.ev1, pr.stream));
    return COOP_OK;
}

static coop_status finish(Prepared &pr, coop_stats *stats) {
    Ctl *h = pr.s->host_ctl;          // mirrored by the kernel's last CTA (mapped memory)
    if (pr.ctl_copied) CUDA_TRY(cudaEventSynchronize(pr.s->done_ev));   // recorded right behind the kernel
    else CUDA_TRY(cudaStreamSynchronize(pr.stream));
    coop_status st = map_err(*h);
    Ctl copy = *h;
    if (stats) {
        stats->threads_per_wg = pr.threads;
        coop_status s2 = fill_stats(copy, pr.kp, stats, pr.stream);
        if (st == COOP_OK) st = s2;
    }
    return st;
}

// The per-device scratch belongs to one call at a time; never block on it (a
// handle that was launched but not waited owns it until coop_wait/destroy).
#define SCRATCH_LOCK(s)                                                                           \
    std::unique_lock<std::mutex> lk((s)->mu, std::try_to_lock);                                   \
    if (!lk.owns_lock())                                                                          \
        return fail(COOP_ERR_BUSY, "device scratch in use by another call or an un-waited handle")

static coop_status run_blocking(const RunReq &r) {
    Prepared pr;
    Scratch *s = nullptr;
    coop_status st = get_scratch(&s, r.opts ? r.opts->workspace : 0);
    if (st != COOP_OK) return st;
    SCRATCH_LOCK(s);
    st = prepare(r, &pr);
    if (st != COOP_OK) return st;
    st = launch(pr);
    if (st != COOP_OK) return st;
    return finish(pr, r.stats);
}

extern "C" coop_status coop_bfs(const coop_csr *g, int64_t source, int32_t *levels_out, const coop_opts *opts,
                                coop_stats *stats) {
    RunReq r = {APP_BFS, g, nullptr, source, levels_out, opts, stats, 0, nullptr, false};
    return run_blocking(r);
}

extern "C" coop_status coop_sssp(const coop_csr *g, int64_t source, uint32_t *dist_out, const coop_opts *opts,
                                 coop_stats *stats) {
    RunReq r = {APP_SSSP, g, nullptr, source, dist_out, opts, stats, 0, nullptr, false};
    return run_blocking(r);
}

// BFS looped over sources inside ONE persistent launch (the paper's multitasking
// workload: "BFS ... in a loop"): run r traverses from sources[r % n_sources];
// a new run starts while less than loop_ns has elapsed since the kernel started.
extern "C" coop_status coop_bfs_loop(const coop_csr *g, const int64_t *sources, uint32_t n_sources,
                                     uint64_t loop_ns, int32_t *levels_out, uint64_t *run_end_ns,
                                     uint32_t run_cap, uint32_t *runs_out, const coop_opts *opts,
                                     coop_stats *stats) {
    if (!g || !sources || !n_sources || !runs_out) return fail(COOP_ERR_INVALID_ARG, "bad arguments");
    std::vector<int64_t> hs(n_sources);
    CUDA_TRY(cudaMemcpy(hs.data(), sources, 8ull * n_sources, cudaMemcpyDeviceToHost));
    for (int64_t v : hs)
        if (v < 0 || v >= g->num_vertices) return fail(COOP_ERR_INVALID_ARG, "source %lld out of range", (long long)v);
    RunReq r = {APP_BFS, g, nullptr, hs[0], levels_out, opts, stats, 0, nullptr, false, nullptr, nullptr,
                sources, n_sources, loop_ns, run_cap};
    Prepared pr;
    Scratch *s = nullptr;
    coop_status st = get_scratch(&s, opts ? opts->workspace : 0);
    if (st != COOP_OK) return st;
    SCRATCH_LOCK(s);
    st = prepare(r, &pr);
    if (st != COOP_OK) return st;
    st = launch(pr);
    if (st != COOP_OK) return st;
    st = finish(pr, stats);
    const Ctl &c = *pr.s->host_ctl;
    const uint32_t runs = c.run & 0x7FFFFFFFu;
    *runs_out = runs;
    if (run_end_ns && run_cap) {
        const uint32_t n = std::min(runs, run_cap);
        std::vector<unsigned long long> t(n);
        if (n) CUDA_TRY(cudaMemcpy(t.data(), pr.kp.run_t, 8ull * n, cudaMemcpyDeviceToHost));
        for (uint32_t i = 0; i < n; ++i) run_end_ns[i] = t[i] > c.t_start ? t[i] - c.t_start : 0;
    }
    return st;
}

// ------------------------------------------------------------------ end-to-end (host pointers)
static coop_status run_host(uint32_t app, int64_t V, const void *ro, int32_t offset_bits, const int32_t *col,
                            const uint32_t *w, uint32_t max_weight, int64_t source, void *out,
                            const coop_opts *opts, coop_stats *stats) {
    if (V < 1 || !ro || !out) return fail(COOP_ERR_INVALID_ARG, "bad host arguments");
    if (offset_bits != 32 && offset_bits != 64) return fail(COOP_ERR_INVALID_ARG, "offset_bits must be 32 or 64");
    Scratch *s = nullptr;
    coop_status st = get_scratch(&s, opts ? opts->workspace : 0);
    if (st != COOP_OK) return st;
    const size_t ob = offset_bits / 8;
    uint64_t E = 0;
    if (offset_bits == 32) E = static_cast<const uint32_t *>(ro)[V];
    else E = (uint64_t) static_cast<const int64_t *>(ro)[V];
    if (E && !col) return fail(COOP_ERR_INVALID_ARG, "col_idx NULL");
    if (app == APP_SSSP && E && !w) return fail(COOP_ERR_INVALID_ARG, "SSSP needs weights");
    cudaStream_t stream = opts ? static_cast<cudaStream_t>(opts->stream) : nullptr;
    g_alloc_stream = stream;
    {
        SCRATCH_LOCK(s);
        CUDA_TRY(s->h_ro.ensure(ob * (V + 1)));
        CUDA_TRY(s->h_col.ensure(4 * std::max<uint64_t>(E, 1)));
        if (app == APP_SSSP) CUDA_TRY(s->h_w.ensure(4 * std::max<uint64_t>(E, 1)));
        CUDA_TRY(s->h_out.ensure(4 * V));
        CUDA_TRY(cudaMemcpyAsync(s->h_ro.p, ro, ob * (V + 1), cudaMemcpyHostToDevice, stream));
        if (E) CUDA_TRY(cudaMemcpyAsync(s->h_col.p, col, 4 * E, cudaMemcpyHostToDevice, stream));
        if (app == APP_SSSP && E) CUDA_TRY(cudaMemcpyAsync(s->h_w.p, w, 4 * E, cudaMemcpyHostToDevice, stream));
    }
    coop_csr g = {V, (int64_t)E, s->h_ro.p, offset_bits, static_cast<const int32_t *>(s->h_col.p),
                  app == APP_SSSP ? static_cast<const uint32_t *>(s->h_w.p) : nullptr, max_weight};
    RunReq r = {app, &g, nullptr, source, s->h_out.p, opts, stats, 0, nullptr, false};
    st = run_blocking(r);
    if (st != COOP_OK) return st;
    CUDA_TRY(cudaMemcpyAsync(out, s->h_out.p, 4 * V, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    return COOP_OK;
}

extern "C" coop_status coop_bfs_host(int64_t num_vertices, const void *row_offsets, int32_t offset_bits,
                                     const int32_t *col_idx, int64_t source, int32_t *levels_out,
                                     const coop_opts *opts, coop_stats *stats) {
    return run_host(APP_BFS, num_vertices, row_offsets, offset_bits, col_idx, nullptr, 0, source, levels_out,
                    opts, stats);
}

extern "C" coop_status coop_sssp_host(int64_t num_vertices, const void *row_offsets, int32_t offset_bits,
                                      const int32_t *col_idx, const uint32_t *weights, uint32_t max_weight,
                                      int64_t source, uint32_t *dist_out, const coop_opts *opts, coop_stats *stats) {
    return run_host(APP_SSSP, num_vertices, row_offsets, offset_bits, col_idx, weights, max_weight, source,
                    dist_out, opts, stats);
}

// ------------------------------------------------------------------ microbenchmarks
extern "C" coop_status coop_barrier_bench(uint32_t n_ctas, uint32_t threads, uint64_t iters, double resize_prob,
                                          uint64_t seed, uint32_t barrier_mode, uint32_t flags,
                                          coop_barrier_stats *out) {
    if (!out) return fail(COOP_ERR_INVALID_ARG, "out is NULL");
    if (iters == 0) return fail(COOP_ERR_INVALID_ARG, "iters must be > 0");
    if (barrier_mode != COOP_BARRIER_QUERY && barrier_mode != COOP_BARRIER_PLAIN)
        return fail(COOP_ERR_INVALID_ARG, "barrier_mode must be QUERY or PLAIN");
    coop_opts o = {};
    o.max_wgs = n_ctas;
    o.threads_per_wg = threads ? threads : 128;
    o.barrier_mode = barrier_mode;
    o.policy = (resize_prob > 0 && barrier_mode == COOP_BARRIER_QUERY) ? COOP_POLICY_RANDOM : COOP_POLICY_NEVER;
    o.resize_prob = resize_prob;
    o.seed = seed;
    o.flags = flags;
    o.timeout_ns = 60000000000ull;
    coop_stats st = {};
    Scratch *s = nullptr;
    coop_status rc = get_scratch(&s, 0);
    if (rc != COOP_OK) return rc;
    SCRATCH_LOCK(s);
    RunReq r = {APP_BARRIER, nullptr, nullptr, 0, nullptr, &o, &st, iters, nullptr, false};
    Prepared pr;
    rc = prepare(r, &pr);
    if (rc != COOP_OK) return rc;
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    CUDA_TRY(cudaEventRecord(e0, pr.stream));
    rc = launch(pr);
    CUDA_TRY(cudaEventRecord(e1, pr.stream));
    if (rc != COOP_OK) return rc;
    rc = finish(pr, &st);
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    out->iters = iters;
    out->ns_per_barrier = ms * 1e6 / (double)iters;
    out->kernel_ns = st.kernel_ns;
    out->kills = st.kills;
    out->forks = st.forks;
    out->violations = pr.s->host_ctl->violations;
    return rc;
}

extern "C" coop_status coop_debug_trace(uint64_t *out16) {
    if (!out16) return fail(COOP_ERR_INVALID_ARG, "NULL argument");
    Scratch *s = nullptr;
    coop_status st = get_scratch(&s, 0);
    if (st != COOP_OK) return st;
    memcpy(out16, s->host_ctl->trace, sizeof(s->host_ctl->trace));
    return COOP_OK;
}

#if COOP_LTRACE
// debug builds only (not part of the ABI in include/coop.h): the per-level stamps
extern "C" coop_status coop_debug_ltrace(uint64_t *out, size_t n) {
    if (!out) {   // clear
        void *a = nullptr;
        CUDA_TRY(cudaGetSymbolAddress(&a, coop::g_ltrace));
        CUDA_TRY(cudaMemset(a, 0, sizeof(coop::g_ltrace)));
        return COOP_OK;
    }
    n = std::min(n, sizeof(coop::g_ltrace) / sizeof(uint64_t));
    CUDA_TRY(cudaMemcpyFromSymbol(out, coop::g_ltrace, n * sizeof(uint64_t)));
    return COOP_OK;
}
#endif

static coop_status l2_profile(uint64_t iters, double *out32) {
    unsigned long long *d = nullptr;
    CUDA_TRY(cudaMalloc(&d, 16 * 8 * sizeof(unsigned long long) + 64 + 32 * sizeof(double)));
    CUDA_TRY(cudaMemset(d, 0, 16 * 8 * sizeof(unsigned long long) + 64 + 32 * sizeof(double)));
    uint32_t *claimed = reinterpret_cast<uint32_t *>(d + 16 * 8);
    double *out = reinterpret_cast<double *>(d + 16 * 8 + 8);
    int dev = 0, sms = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    l2_rtt_kernel<<<sms, 32>>>(d, claimed, iters, out);             // one CTA per SM
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpy(out32, out, 32 * sizeof(double), cudaMemcpyDeviceToHost));
    cudaFree(d);
    return COOP_OK;
}

extern "C" coop_status coop_l2_atomic_rtt(uint64_t iters, double *ns_per_atomic) {
    if (!ns_per_atomic || iters == 0) return fail(COOP_ERR_INVALID_ARG, "bad arguments");
    double t[32];
    coop_status st = l2_profile(iters, t);
    if (st != COOP_OK) return st;
    std::vector<double> v;
    for (int k = 0; k < 8; ++k)
        if (t[k] > 0) v.push_back(t[k]);
    if (v.empty()) return fail(COOP_ERR_CUDA, "no SM measured");
    std::sort(v.begin(), v.end());
    *ns_per_atomic = v[v.size() / 2];                               // median over the SMs
    return COOP_OK;
}

extern "C" coop_status coop_l2_latency_profile(uint64_t iters, double *ns_out) {
    if (!ns_out || iters == 0) return fail(COOP_ERR_INVALID_ARG, "bad arguments");
    return l2_profile(iters, ns_out);
}

// The competing task as a standalone (non-cooperative) kernel: `blocks` CTAs each
// occupy their SM slot for block_ns (the same synthetic task the megakernel's pool
// runs, K11).  Used for the kernel-level preemption comparison (T3,
// P:1258-1313): the task is enqueued between compute launches, i.e. it preempts the
// compute work at kernel granularity.
__global__ void spin_task_kernel(unsigned long long block_ns) {
    if (threadIdx.x == 0) {
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 >= block_ns) break;
            __nanosleep(100);
        }
    }
    __syncthreads();
}

extern "C" coop_status coop_spin_task(uint32_t blocks, uint32_t threads, uint64_t block_ns, void *stream) {
    if (!blocks || !threads || threads > 1024) return fail(COOP_ERR_INVALID_ARG, "bad arguments");
    spin_task_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(block_ns);
    CUDA_TRY(cudaGetLastError());
    return COOP_OK;
}

// ------------------------------------------------------------------ handle API
struct coop_handle {
    Prepared pr;
    HostChannel *hc = nullptr;      // host view (mapped pinned)
    HostChannel *dc = nullptr;      // device view
    uint32_t seq = 0;
    bool waited = false;
    uint64_t next_task_id = 0;
};

static coop_status launch_handle(const RunReq &r0, const coop_opts *opts, bool channel, coop_handle **handle) {
    coop_handle *h = new (std::nothrow) coop_handle();
    if (!h) return fail(COOP_ERR_INVALID_ARG, "out of host memory");
    if (channel) {
        cudaError_t e = cudaHostAlloc((void **)&h->hc, sizeof(HostChannel), cudaHostAllocMapped);
        if (e != cudaSuccess) { delete h; return fail(COOP_ERR_CUDA, "cudaHostAlloc: %s", cudaGetErrorString(e)); }
        memset((void *)h->hc, 0, sizeof(HostChannel));
        e = cudaHostGetDevicePointer((void **)&h->dc, h->hc, 0);
        if (e != cudaSuccess) { cudaFreeHost(h->hc); delete h; return fail(COOP_ERR_CUDA, "cudaHostGetDevicePointer"); }
    }
    RunReq r = r0;
    r.host = h->dc;
    Scratch *s = nullptr;
    coop_status st = get_scratch(&s, opts ? opts->workspace : 0);
    if (st == COOP_OK) {
        if (!s->mu.try_lock()) {   // held until coop_wait/destroy: the scratch belongs to this launch
            st = fail(COOP_ERR_BUSY, "device scratch in use by another call or an un-waited handle");
        } else {
            st = prepare(r, &h->pr);
            if (st == COOP_OK) st = launch(h->pr);
            if (st == COOP_OK && !channel) {
                // the control block comes back right behind the kernel, so coop_wait of this
                // call does not queue behind the kernels launched after it on the same stream
                // (channel handles keep copying at wait: their kernel runs until the host says)
                cudaError_t e = s->done_ev ? cudaSuccess : cudaEventCreateWithFlags(&s->done_ev, cudaEventDisableTiming);
                if (e == cudaSuccess) e = cudaEventRecord(s->done_ev, h->pr.stream);
                if (e != cudaSuccess) st = fail(COOP_ERR_CUDA, "control block copy: %s", cudaGetErrorString(e));
                else h->pr.ctl_copied = true;
            }
            if (st != COOP_OK) s->mu.unlock();
        }
    }
    if (st != COOP_OK) {
        if (h->hc) cudaFreeHost(h->hc);
        delete h;
        return st;
    }
    *handle = h;
    return COOP_OK;
}

extern "C" coop_status coop_launch(int kind, const coop_csr *g, int64_t source, void *out, const coop_opts *opts,
                                   coop_handle **handle) {
    if (!handle || !opts) return fail(COOP_ERR_INVALID_ARG, "handle/opts NULL");
    if (kind != 0 && kind != 1) return fail(COOP_ERR_INVALID_ARG, "kind must be 0 (BFS) or 1 (SSSP)");
    if (opts->policy != COOP_POLICY_SCHEDULER || opts->barrier_mode == COOP_BARRIER_PLAIN)
        return fail(COOP_ERR_INVALID_ARG, "coop_launch needs policy SCHEDULER and a cooperative barrier");
    RunReq r = {kind == 0 ? APP_BFS : APP_SSSP, g, nullptr, source, out, opts, nullptr, 0, nullptr, true};
    return launch_handle(r, opts, true, handle);
}

// asynchronous BFS / SSSP with any policy (finish with coop_wait): back-to-back calls on one
// stream, each with its own opts->workspace, overlap the host preparation of call i+1 with
// the kernel of call i
extern "C" coop_status coop_bfs_launch(const coop_csr *g, int64_t source, int32_t *levels_out, const coop_opts *opts,
                                       coop_handle **handle) {
    if (!handle) return fail(COOP_ERR_INVALID_ARG, "handle NULL");
    RunReq r = {APP_BFS, g, nullptr, source, levels_out, opts, nullptr, 0, nullptr, true};
    const bool chan = opts && opts->policy == COOP_POLICY_SCHEDULER;
    return launch_handle(r, opts, chan, handle);
}

// ------------------------------------------------------------------ partitioned BFS
extern "C" coop_status coop_bfs_part(const coop_part *part, int64_t source, int32_t *levels_owned_out,
                                     const coop_opts *opts, coop_stats *stats) {
    RunReq r = {APP_PBFS, nullptr, part, source, levels_owned_out, opts, stats, 0, nullptr, false};
    return run_blocking(r);
}

extern "C" coop_status coop_bfs_part_launch(const coop_part *part, int64_t source, int32_t *levels_owned_out,
                                            const coop_opts *opts, coop_handle **handle) {
    if (!handle) return fail(COOP_ERR_INVALID_ARG, "handle NULL");
    RunReq r = {APP_PBFS, nullptr, part, source, levels_owned_out, opts, nullptr, 0, nullptr, true};
    const bool chan = opts && opts->policy == COOP_POLICY_SCHEDULER;
    return launch_handle(r, opts, chan, handle);
}

extern "C" coop_status coop_sssp_part(const coop_part *part, const uint32_t *weights_local, int64_t source,
                                      uint32_t *dist_owned_out, const coop_opts *opts, coop_stats *stats) {
    RunReq r = {APP_PSSSP, nullptr, part, source, dist_owned_out, opts, stats, 0, nullptr, false, nullptr, weights_local};
    return run_blocking(r);
}

extern "C" coop_status coop_sssp_part_launch(const coop_part *part, const uint32_t *weights_local, int64_t source,
                                             uint32_t *dist_owned_out, const coop_opts *opts, coop_handle **handle) {
    if (!handle) return fail(COOP_ERR_INVALID_ARG, "handle NULL");
    RunReq r = {APP_PSSSP, nullptr, part, source, dist_owned_out, opts, nullptr, 0, nullptr, true, nullptr, weights_local};
    const bool chan = opts && opts->policy == COOP_POLICY_SCHEDULER;
    return launch_handle(r, opts, chan, handle);
}

extern "C" coop_status coop_exchange_alloc(uint64_t bytes, void **dptr) {
    if (!dptr || !bytes) return fail(COOP_ERR_INVALID_ARG, "bad arguments");
    CUDA_TRY(cudaMalloc(dptr, bytes));
    CUDA_TRY(cudaMemset(*dptr, 0, bytes));
    return COOP_OK;
}

extern "C" coop_status coop_exchange_free(void *dptr) {
    if (!dptr) return fail(COOP_ERR_INVALID_ARG, "NULL argument");
    CUDA_TRY(cudaFree(dptr));
    return COOP_OK;
}

extern "C" coop_status coop_ipc_get_handle(const void *dptr, void *handle64) {
    if (!dptr || !handle64) return fail(COOP_ERR_INVALID_ARG, "NULL argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, const_cast<void *>(dptr)));
    memcpy(handle64, &h, sizeof h);
    return COOP_OK;
}

extern "C" coop_status coop_ipc_open(const void *handle64, void **dptr) {
    if (!dptr || !handle64) return fail(COOP_ERR_INVALID_ARG, "NULL argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof h);
    CUDA_TRY(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
    return COOP_OK;
}

extern "C" coop_status coop_ipc_close(void *dptr) {
    if (!dptr) return fail(COOP_ERR_INVALID_ARG, "NULL argument");
    CUDA_TRY(cudaIpcCloseMemHandle(dptr));
    return COOP_OK;
}

// ------------------------------------------------------------------ NCCL data plane
// north_star's bring-up exchange for the partitioned BFS: the
// persistent cooperative kernel runs on the caller's stream; a comm stream holds,
// per level L, cuStreamWaitValue32(ready >= L+1) -> ncclAllGather of the own
// bitmap slice (in place) + the counts -> cuStreamWriteValue32(gathered = L+1).
// The kernel publishes `ready` in RB1's serial section and waits for `gathered`
// in RB2's.  The host enqueues levels ahead of the kernel (kNcclAhead) from a
// mapped mirror of `ready`; every rank enqueues exactly final + kNcclAhead
// gathers, so the collectives match across ranks.
struct NcclSyms {
    bool ok = false;
    char why[256] = {0};
    ncclResult_t (*get_unique_id)(ncclUniqueId *);
    ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*comm_destroy)(ncclComm_t);
    ncclResult_t (*all_gather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*group_start)();
    ncclResult_t (*group_end)();
    const char *(*error_string)(ncclResult_t);
    CUresult (*wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
    CUresult (*write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
};

static NcclSyms &nccl_syms() {
    static NcclSyms S;
    static std::once_flag once;
    std::call_once(once, [] {
        // the process's NCCL if one is loaded already (torch's), else the system library
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) { snprintf(S.why, sizeof S.why, "libnccl.so.2 not found: %s", dlerror()); return; }
#define NSYM(f, n)                                                                   \
    *reinterpret_cast<void **>(&S.f) = dlsym(h, n);                                  \
    if (!S.f) { snprintf(S.why, sizeof S.why, "NCCL symbol %s missing", n); return; }
        NSYM(get_unique_id, "ncclGetUniqueId");
        NSYM(comm_init_rank, "ncclCommInitRank");
        NSYM(comm_destroy, "ncclCommDestroy");
        NSYM(all_gather, "ncclAllGather");
        NSYM(group_start, "ncclGroupStart");
        NSYM(group_end, "ncclGroupEnd");
        NSYM(error_string, "ncclGetErrorString");
#undef NSYM
        // the CUDA 12 ABI of the stream memory operations (the _v2 entry points; the v1
        // ones need a driver option and fail at enqueue on this image)
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", reinterpret_cast<void **>(&S.wait32), 12000,
                                             cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
            S.wait32 = nullptr;
        if (cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", reinterpret_cast<void **>(&S.write32), 12000,
                                             cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
            S.write32 = nullptr;
        S.ok = true;
    });
    return S;
}

#define NCCL_TRY(x)                                                                                  \
    do {                                                                                             \
        ncclResult_t r_ = (x);                                                                       \
        if (r_ != ncclSuccess) return fail(COOP_ERR_NCCL, "%s: %s", #x, N.error_string(r_));          \
    } while (0)
#define CU_TRY(x)                                                                                    \
    do {                                                                                             \
        CUresult r_ = (x);                                                                           \
        if (r_ != CUDA_SUCCESS) return fail(COOP_ERR_CUDA, "%s: CUresult %d", #x, (int)r_);          \
    } while (0)

extern "C" coop_status coop_nccl_get_unique_id(void *uid128) {
    NcclSyms &N = nccl_syms();
    if (!N.ok) return fail(COOP_ERR_NCCL, "%s", N.why);
    if (!uid128) return fail(COOP_ERR_INVALID_ARG, "NULL argument");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    NCCL_TRY(N.get_unique_id(&id));
    memcpy(uid128, &id, sizeof id);
    return COOP_OK;
}

extern "C" coop_status coop_nccl_comm_init(int32_t nranks, const void *uid128, int32_t rank, void **comm) {
    NcclSyms &N = nccl_syms();
    if (!N.ok) return fail(COOP_ERR_NCCL, "%s", N.why);
    if (!uid128 || !comm || nranks < 1 || rank < 0 || rank >= nranks) return fail(COOP_ERR_INVALID_ARG, "bad arguments");
    ncclUniqueId id;
    memcpy(&id, uid128, sizeof id);
    ncclComm_t c = nullptr;
    NCCL_TRY(N.comm_init_rank(&c, nranks, id, rank));
    *comm = c;
    return COOP_OK;
}

extern "C" coop_status coop_nccl_comm_destroy(void *comm) {
    NcclSyms &N = nccl_syms();
    if (!N.ok) return fail(COOP_ERR_NCCL, "%s", N.why);
    if (!comm) return fail(COOP_ERR_INVALID_ARG, "NULL comm");
    NCCL_TRY(N.comm_destroy(static_cast<ncclComm_t>(comm)));
    return COOP_OK;
}

constexpr uint32_t kNcclAhead = 2;            // levels of gathers enqueued ahead of the kernel

extern "C" coop_status coop_bfs_part_nccl(const coop_part *part, int64_t source, int32_t *levels_owned_out,
                                          void *nccl_comm, const coop_opts *opts, coop_stats *stats) {
    NcclSyms &N = nccl_syms();
    if (!N.ok) return fail(COOP_ERR_NCCL, "%s", N.why);
    if (!part || !nccl_comm) return fail(COOP_ERR_INVALID_ARG, "part / nccl_comm NULL");
    if (part->nranks < 1 || part->nranks > COOP_MAX_RANKS || part->rank < 0 || part->rank >= part->nranks)
        return fail(COOP_ERR_INVALID_ARG, "rank %d / nranks %d invalid", part->rank, part->nranks);
    const int P = part->nranks, me = part->rank;
    const uint64_t nw = ((uint64_t)part->num_vertices + 31) / 32;
    const uint64_t sw = (nw + P - 1) / P;                       // uniform slice: in-place all-gather
    const int64_t vb = std::min<int64_t>(part->num_vertices, (int64_t)(32 * sw * me));
    const int64_t ve = std::min<int64_t>(part->num_vertices, (int64_t)(32 * sw * (me + 1)));
    if (part->v_begin != vb || part->v_end != ve)
        return fail(COOP_ERR_INVALID_ARG, "NCCL data plane needs uniform slices: rank %d must own [%lld, %lld)", me,
                    (long long)vb, (long long)ve);
    if (!part->frontier[me][0] || !part->frontier[me][1])
        return fail(COOP_ERR_INVALID_ARG, "frontier[rank][0..1] (nranks * slice words each) NULL");
    Scratch *s = nullptr;
    coop_status st = get_scratch(&s, opts ? opts->workspace : 0);
    if (st != COOP_OK) return st;
    SCRATCH_LOCK(s);
    cudaStream_t ks = opts ? static_cast<cudaStream_t>(opts->stream) : nullptr;
    // per-workspace comm stream, mapped host mirror, small device buffer
    if (!s->nccl_stream) {
        CUDA_TRY(cudaStreamCreateWithFlags(&s->nccl_stream, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&s->nccl_ev, cudaEventDisableTiming));
        CUDA_TRY(cudaHostAlloc((void **)&s->nccl_host, 64, cudaHostAllocMapped));   // [0] mirror, [1..8] values
    }
    const size_t aux = 256 + 8 * 4 * 2 + 8 * 4 * 2 * COOP_MAX_RANKS + 64 * COOP_MAX_RANKS;
    g_alloc_stream = ks;
    CUDA_TRY(s->nccl_aux.ensure(aux));
    char *base = static_cast<char *>(s->nccl_aux.p);
    if (s->nccl_warm != nccl_comm) {
        // a first collective on a new communicator may set up NCCL state with calls that
        // synchronise with the device; that must not happen while the persistent kernel
        // waits for a gather: warm the communicator up before any launch (collective:
        // every rank makes its first call with this comm at the same point)
        CUDA_TRY(cudaStreamSynchronize(ks));
        uint32_t *scratch = reinterpret_cast<uint32_t *>(base + aux - 64 * COOP_MAX_RANKS);
        NCCL_TRY(N.all_gather(scratch + me, scratch, 1, ncclUint32, static_cast<ncclComm_t>(nccl_comm),
                              s->nccl_stream));
        CUDA_TRY(cudaStreamSynchronize(s->nccl_stream));
        s->nccl_warm = nccl_comm;
    }
    NcclExt nx;
    nx.ready = reinterpret_cast<uint32_t *>(base);
    nx.gathered = reinterpret_cast<uint32_t *>(base + 128);
    nx.cnt_send = reinterpret_cast<unsigned long long *>(base + 256);
    nx.cnt_recv = nx.cnt_send + 8;
    volatile uint32_t *hdev = nullptr;
    CUDA_TRY(cudaHostGetDevicePointer((void **)&hdev, (void *)s->nccl_host, 0));
    nx.host_ready = hdev;
    nx.slice_words = sw;
    s->nccl_host[0] = 0;
    CUDA_TRY(cudaMemsetAsync(base, 0, 256, ks));                  // ready = gathered = 0
    CUDA_TRY(cudaEventRecord(s->nccl_ev, ks));
    CUDA_TRY(cudaStreamWaitEvent(s->nccl_stream, s->nccl_ev, 0));  // no wait may see the previous call's values
    RunReq r = {APP_PBFS, nullptr, part, source, levels_owned_out, opts, stats, 0, nullptr, false, &nx};
    Prepared pr;
    st = prepare(r, &pr);
    if (st != COOP_OK) return st;
    st = launch(pr);
    if (st != COOP_OK) return st;
    CUDA_TRY(cudaEventRecord(s->nccl_ev, ks));                    // kernel done (abort detection)
    ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
    cudaStream_t cs = s->nccl_stream;
    auto enqueue = [&](uint32_t i) -> coop_status {               // gather i: frontier of level i + 1
        const uint32_t b = (i + 1) & 1;
        uint32_t *F = part->frontier[me][b];
        CU_TRY(N.wait32((CUstream)cs, (CUdeviceptr)nx.ready, i + 1, CU_STREAM_WAIT_VALUE_GEQ));
        NCCL_TRY(N.group_start());
        NCCL_TRY(N.all_gather(F + sw * me, F, sw, ncclUint32, comm, cs));
        NCCL_TRY(N.all_gather(nx.cnt_send + 4 * b, nx.cnt_recv + (size_t)4 * P * b, 4, ncclUint64, comm, cs));
        NCCL_TRY(N.group_end());
        CU_TRY(N.write32((CUstream)cs, (CUdeviceptr)nx.gathered, i + 1, CU_STREAM_WRITE_VALUE_DEFAULT));
        return COOP_OK;
    };
    // Two ways to order the gathers against the persistent kernel:
    //  relay (default): the host polls the mapped mirror of `ready` and enqueues gather L
    //    when the kernel has published level L -- the comm stream never blocks, so NCCL's
    //    host-side enqueue never waits on a stalled stream (measured: with gathers
    //    enqueued ahead behind cuStreamWaitValue32 the NCCL launch blocked the host while
    //    the kernel waited for the gather -- a deadlock until the watchdog);
    //  COOP_NCCL_MEMOP=1: gathers enqueued kNcclAhead levels ahead, each behind
    //    cuStreamWaitValue32(ready >= L+1) (no host on the critical path).
    static const bool memop = getenv("COOP_NCCL_MEMOP") && getenv("COOP_NCCL_MEMOP")[0] == '1' && N.wait32 && N.write32;
    auto enqueue_now = [&](uint32_t i) -> coop_status {            // relay: gather i, then `gathered`
        const uint32_t b = (i + 1) & 1;
        uint32_t *F = part->frontier[me][b];
        NCCL_TRY(N.group_start());
        NCCL_TRY(N.all_gather(F + sw * me, F, sw, ncclUint32, comm, cs));
        NCCL_TRY(N.all_gather(nx.cnt_send + 4 * b, nx.cnt_recv + (size_t)4 * P * b, 4, ncclUint64, comm, cs));
        NCCL_TRY(N.group_end());
        // `gathered` = i+1 by a copy from pinned host memory behind the gathers (copy engine;
        // the slot is rewritten only after the kernel has seen it: the kernel publishes
        // level i+1 only after observing gathered >= i+1)
        volatile uint32_t *slot = s->nccl_host + 1 + (i & 7);
        *slot = i + 1;
        CUDA_TRY(cudaMemcpyAsync(nx.gathered, (const void *)slot, 4, cudaMemcpyHostToDevice, cs));
        return COOP_OK;
    };
    uint32_t enq = 0;
    coop_status est = COOP_OK;
    if (memop)
        for (; enq < kNcclAhead && est == COOP_OK; ++enq) est = enqueue(enq);
    bool aborted = false;
    static const bool dbg = getenv("COOP_NCCL_DEBUG") != nullptr;
    auto t_dbg = std::chrono::steady_clock::now();
    while (est == COOP_OK) {
        if (dbg && std::chrono::steady_clock::now() - t_dbg > std::chrono::milliseconds(500)) {
            t_dbg = std::chrono::steady_clock::now();
            fprintf(stderr, "[coop nccl] enq=%u host_ready=%#x comm stream %s\n", enq, s->nccl_host[0],
                    cudaGetErrorString(cudaStreamQuery(cs)));
        }
        const uint32_t hr = s->nccl_host[0];
        if (hr & 0x80000000u) {                                     // final: (hr & ~bit) gathers used
            if (memop) {
                const uint32_t target = (hr & 0x7FFFFFFFu) + kNcclAhead;
                while (enq < target && est == COOP_OK) est = enqueue(enq++);
            }
            break;
        }
        if (memop) {
            while (enq < hr + kNcclAhead && est == COOP_OK) est = enqueue(enq++);
        } else {
            while (enq < hr && est == COOP_OK) est = enqueue_now(enq++);
        }
        const cudaError_t eq = cudaEventQuery(s->nccl_ev);
        if (eq == cudaSuccess) {                                    // kernel ended without the final mark
            if (s->nccl_host[0] & 0x80000000u) continue;
            aborted = true;
            if (dbg) fprintf(stderr, "[coop nccl] kernel ended without the final mark: enq=%u host_ready=%#x\n", enq,
                             s->nccl_host[0]);
            break;
        } else if (eq != cudaErrorNotReady) {
            est = fail(COOP_ERR_CUDA, "event query: %s", cudaGetErrorString(eq));
            break;
        }
        if (memop) sched_yield();
    }
    if (dbg) fprintf(stderr, "[coop nccl] host loop done: enq=%u host_ready=%#x est=%d\n", enq, s->nccl_host[0], (int)est);
    if (aborted || est != COOP_OK) {
        // release any wait still enqueued so the comm stream drains (the kernel has ended)
        static const uint32_t big = 0xFFFFFFFFu;
        cudaMemcpyAsync(nx.ready, &big, 4, cudaMemcpyHostToDevice, ks);
        cudaStreamSynchronize(ks);
    }
    char msg[sizeof g_err];
    memcpy(msg, g_err, sizeof msg);                                 // the host loop's own error, if any
    coop_status fst = finish(pr, stats);
    cudaError_t ce = cudaStreamSynchronize(cs);
    if (est != COOP_OK) {
        memcpy(g_err, msg, sizeof msg);
        return est;
    }
    if (fst != COOP_OK) return fst;
    if (ce != cudaSuccess) return fail(COOP_ERR_CUDA, "comm stream: %s", cudaGetErrorString(ce));
    return COOP_OK;
}

static coop_status post(coop_handle *h, uint32_t kind, uint32_t a, uint32_t b, uint64_t c) {
    if (h->waited) return fail(COOP_ERR_BUSY, "handle already waited");
    if (!h->hc) return fail(COOP_ERR_BUSY, "handle has no host channel (policy is not SCHEDULER)");
    // single-slot channel: wait until the scheduler CTA consumed the previous packet
    for (long spins = 0; h->hc->ack != h->seq; ++spins) {
        if (h->hc->done_mirror) return fail(COOP_ERR_BUSY, "kernel already terminated");
        if (spins > 200000000L) return fail(COOP_ERR_TIMEOUT, "scheduler CTA did not consume the packet");
    }
    h->hc->kind = kind;
    h->hc->a = a;
    h->hc->b = b;
    h->hc->c = c;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    h->hc->seq = ++h->seq;
    return COOP_OK;
}

extern "C" coop_status coop_submit_task(coop_handle *h, uint32_t task_wgs, uint32_t task_blocks,
                                        uint64_t task_block_ns, uint64_t *task_id) {
    if (!h) return fail(COOP_ERR_INVALID_ARG, "handle NULL");
    if (task_wgs < 1 || task_wgs > h->pr.kp.P - 1)
        return fail(COOP_ERR_NO_CAPACITY, "task_wgs %u not in [1, N-1=%u]", task_wgs, h->pr.kp.P - 1);
    coop_status st = post(h, 1, task_wgs, task_blocks ? task_blocks : 1, task_block_ns);
    if (st == COOP_OK && task_id) *task_id = h->next_task_id;
    if (st == COOP_OK) h->next_task_id++;
    return st;
}

extern "C" coop_status coop_demand(coop_handle *h, uint32_t kills) {
    if (!h) return fail(COOP_ERR_INVALID_ARG, "handle NULL");
    if (kills > h->pr.kp.P - 1) return fail(COOP_ERR_NO_CAPACITY, "demand %u > N-1", kills);
    return post(h, 2, kills, 0, 0);
}

extern "C" coop_status coop_grant(coop_handle *h, uint32_t forks) {
    if (!h) return fail(COOP_ERR_INVALID_ARG, "handle NULL");
    if (forks > h->pr.kp.P) return fail(COOP_ERR_FORK_BOUND, "grant %u > N=%u (k <= N-M, P:565)", forks, h->pr.kp.P);
    return post(h, 3, forks, 0, 0);
}

extern "C" coop_status coop_query(coop_handle *h, uint32_t *W) {
    if (!h || !W) return fail(COOP_ERR_INVALID_ARG, "NULL argument");
    if (!h->hc) return fail(COOP_ERR_BUSY, "handle has no host channel");
    *W = h->hc->demand_mirror;
    return COOP_OK;
}

extern "C" coop_status coop_current_m(coop_handle *h, uint32_t *M) {
    if (!h || !M) return fail(COOP_ERR_INVALID_ARG, "NULL argument");
    if (!h->hc) return fail(COOP_ERR_BUSY, "handle has no host channel");
    *M = h->hc->cur_m;
    return COOP_OK;
}

extern "C" coop_status coop_wait(coop_handle *h, coop_stats *stats) {
    if (!h) return fail(COOP_ERR_INVALID_ARG, "handle NULL");
    if (h->waited) return fail(COOP_ERR_BUSY, "already waited");
    h->waited = true;
    coop_status st = finish(h->pr, stats);
    h->pr.s->mu.unlock();
    return st;
}

extern "C" void coop_destroy(coop_handle *h) {
    if (!h) return;
    if (!h->waited) {
        cudaStreamSynchronize(h->pr.stream);
        h->pr.s->mu.unlock();
    }
    if (h->hc) cudaFreeHost(h->hc);
    delete h;
}
