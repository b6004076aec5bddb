// coop_dev_api.cu -- host half of the device API (include/coop_device.cuh) and
// two cooperative kernels written on it:
//   * fig4_kernel : the paper's Fig. 4 cooperative graph traversal, literally
//                   (PAPER.md:709-729), as BFS;
//   * ws_kernel   : cooperative work stealing, Fig. 2 adapted per §3.2
//                   (PAPER.md:341-385, 666-680).
// Both use only the public device API, exactly as a user kernel would.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "../../include/coop.h"
#include "../../include/coop_device.cuh"

char *coop_internal_errbuf();

namespace {

coop_status dfail(coop_status s, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(coop_internal_errbuf(), 512, fmt, ap);
    va_end(ap);
    return s;
}
#define DCUDA(x)                                                                             \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess) {                                                             \
            cudaGetLastError();                                                              \
            return dfail(COOP_ERR_CUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                         __FILE__, __LINE__);                                                \
        }                                                                                    \
    } while (0)

uint32_t prob_thresh(double p) {
    if (p <= 0.0) return 0u;
    if (p >= 1.0) return 0xFFFFFFFFu;
    return (uint32_t)(p * 4294967296.0);
}

}  // namespace

struct coop_dev_handle {
    coop_dev_opts opts;
    std::vector<uint32_t> script;
    coop_dev *d = nullptr;              // device control block
    coop_dev_mailbox *mb = nullptr;     // device mailboxes [COOP_DEV_MAX_CTAS]
    uint32_t *script_d = nullptr;
    uint32_t *trace_d = nullptr;
    uint32_t *posted_h = nullptr;       // pinned {demand_posted, grant_posted}
    cudaStream_t side = nullptr;        // resource messages while a kernel runs
    cudaEvent_t armed = nullptr;        // recorded after arm's control-block copy
    std::mutex mu;
    uint32_t n_wgs = 0;
    int device = 0;
};

extern "C" coop_status coop_dev_create(const coop_dev_opts *opts, coop_dev_handle **handle) {
    if (!opts || !handle) return dfail(COOP_ERR_INVALID_ARG, "null argument");
    if (opts->policy > COOP_POLICY_SCHEDULER) return dfail(COOP_ERR_INVALID_ARG, "unknown policy %u", opts->policy);
    if (opts->max_fork > 32) return dfail(COOP_ERR_INVALID_ARG, "max_fork %u > 32", opts->max_fork);
    if (opts->policy == COOP_POLICY_SCRIPTED && (!opts->script || !opts->script_len))
        return dfail(COOP_ERR_INVALID_ARG, "SCRIPTED policy needs a script");
    coop_dev_handle *h = new (std::nothrow) coop_dev_handle();
    if (!h) return dfail(COOP_ERR_INVALID_ARG, "out of host memory");
    h->opts = *opts;
    if (opts->script && opts->script_len) h->script.assign(opts->script, opts->script + opts->script_len);
    auto bail = [&](cudaError_t e, const char *what) {
        coop_dev_destroy(h);
        cudaGetLastError();
        return dfail(COOP_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    };
    cudaError_t e = cudaGetDevice(&h->device);
    if (e != cudaSuccess) return bail(e, "cudaGetDevice");
    if ((e = cudaMalloc((void **)&h->d, sizeof(coop_dev))) != cudaSuccess) return bail(e, "cudaMalloc(coop_dev)");
    if ((e = cudaMalloc((void **)&h->mb, sizeof(coop_dev_mailbox) * COOP_DEV_MAX_CTAS)) != cudaSuccess)
        return bail(e, "cudaMalloc(mailboxes)");
    if (!h->script.empty()) {
        if ((e = cudaMalloc((void **)&h->script_d, 4 * h->script.size())) != cudaSuccess) return bail(e, "cudaMalloc");
        if ((e = cudaMemcpy(h->script_d, h->script.data(), 4 * h->script.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
            return bail(e, "cudaMemcpy(script)");
    }
    if (opts->m_trace_cap) {
        if ((e = cudaMalloc((void **)&h->trace_d, 4ull * opts->m_trace_cap)) != cudaSuccess) return bail(e, "cudaMalloc");
    }
    if ((e = cudaHostAlloc((void **)&h->posted_h, 64, cudaHostAllocDefault)) != cudaSuccess) return bail(e, "cudaHostAlloc");
    memset(h->posted_h, 0, 64);
    if ((e = cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking)) != cudaSuccess) return bail(e, "cudaStreamCreate");
    if ((e = cudaEventCreateWithFlags(&h->armed, cudaEventDisableTiming)) != cudaSuccess) return bail(e, "cudaEventCreate");
    *handle = h;
    return COOP_OK;
}

extern "C" void coop_dev_destroy(coop_dev_handle *h) {
    if (!h) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(h->device);
    if (h->side) cudaStreamSynchronize(h->side), cudaStreamDestroy(h->side);
    if (h->armed) cudaEventDestroy(h->armed);
    cudaFree(h->d);
    cudaFree(h->mb);
    cudaFree(h->script_d);
    cudaFree(h->trace_d);
    if (h->posted_h) cudaFreeHost(h->posted_h);
    cudaSetDevice(cur);
    cudaGetLastError();
    delete h;
}

extern "C" coop_status coop_dev_arm(coop_dev_handle *h, uint32_t n_wgs, void *stream, coop_dev **dev_out) {
    if (!h || !dev_out) return dfail(COOP_ERR_INVALID_ARG, "null argument");
    if (n_wgs == 0 || n_wgs > COOP_DEV_MAX_CTAS) return dfail(COOP_ERR_INVALID_ARG, "n_wgs %u out of [1, %u]", n_wgs, COOP_DEV_MAX_CTAS);
    const coop_dev_opts &o = h->opts;
    const uint32_t M0 = o.init_wgs ? o.init_wgs : n_wgs;
    if (M0 > n_wgs) return dfail(COOP_ERR_INVALID_ARG, "init_wgs %u > N %u", M0, n_wgs);
    if (M0 > 0xFFFF || n_wgs > 0xFFFF) return dfail(COOP_ERR_INVALID_ARG, "too many workgroups");
    std::lock_guard<std::mutex> lk(h->mu);
    cudaStream_t s = (cudaStream_t)stream;
    coop_dev hd;
    memset(&hd, 0, sizeof hd);
    hd.W = ((unsigned long long)M0 << 16);             // {gen 0, M0, 0}
    hd.R = ((unsigned long long)M0 << 16);
    hd.N = n_wgs;
    hd.M0 = M0;
    hd.policy = o.policy;
    hd.flags = o.flags;
    hd.seed = o.seed;
    hd.kill_thresh = prob_thresh(o.kill_prob);
    hd.fork_thresh = prob_thresh(o.fork_prob);
    hd.resize_thresh = prob_thresh(o.resize_prob);
    hd.max_fork = o.max_fork ? o.max_fork : 4u;
    hd.script = h->script_d;
    hd.script_len = (uint32_t)h->script.size();
    hd.m_trace = h->trace_d;
    hd.m_trace_cap = o.m_trace_cap;
    hd.timeout_ns = o.timeout_ns ? o.timeout_ns : 20000000000ull;
    hd.mb = h->mb;
    hd.min_m = M0;
    hd.max_m = M0;
    // the host's resource messages so far count as already taken: a new launch starts clean
    hd.demand_posted = hd.demand_taken = h->posted_h[0];
    hd.grant_posted = hd.grant_taken = h->posted_h[1];
    for (uint32_t p = M0; p < n_wgs; ++p) hd.pool[p >> 5] |= 1u << (p & 31u);
    // pageable source: cudaMemcpyAsync stages it before returning, so `hd` may go out of scope
    DCUDA(cudaMemcpyAsync(h->d, &hd, sizeof hd, cudaMemcpyHostToDevice, s));
    DCUDA(cudaMemsetAsync(h->mb, 0, sizeof(coop_dev_mailbox) * n_wgs, s));
    // a resource message posted after arm returns must land after this copy, or the
    // copy's older posted counts would overwrite it (post() waits on this event)
    DCUDA(cudaEventRecord(h->armed, s));
    h->n_wgs = n_wgs;
    *dev_out = h->d;
    return COOP_OK;
}

static coop_status post(coop_dev_handle *h, int which, uint32_t n) {
    if (!h) return dfail(COOP_ERR_INVALID_ARG, "null handle");
    std::lock_guard<std::mutex> lk(h->mu);
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != h->device) DCUDA(cudaSetDevice(h->device));
    h->posted_h[which] += n;
    // one monotone 32-bit store into the running kernel's control block (copy engine,
    // non-blocking stream: it does not wait for the persistent kernel)
    uint32_t *dst = which == 0 ? &h->d->demand_posted : &h->d->grant_posted;
    cudaError_t e = cudaStreamWaitEvent(h->side, h->armed, 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dst, &h->posted_h[which], 4, cudaMemcpyHostToDevice, h->side);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->side);
    if (cur != h->device) cudaSetDevice(cur);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return dfail(COOP_ERR_CUDA, "posting a resource message: %s", cudaGetErrorString(e));
    }
    return COOP_OK;
}
extern "C" coop_status coop_dev_demand(coop_dev_handle *h, uint32_t kills) { return post(h, 0, kills); }
extern "C" coop_status coop_dev_grant(coop_dev_handle *h, uint32_t forks) {
    if (h && forks > COOP_DEV_MAX_CTAS) return dfail(COOP_ERR_FORK_BOUND, "grant %u > N", forks);
    return post(h, 1, forks);
}

extern "C" coop_status coop_dev_collect(coop_dev_handle *h, void *stream, coop_dev_stats *st) {
    if (!h) return dfail(COOP_ERR_INVALID_ARG, "null handle");
    DCUDA(cudaStreamSynchronize((cudaStream_t)stream));
    coop_dev hd;
    DCUDA(cudaMemcpy(&hd, h->d, sizeof hd, cudaMemcpyDeviceToHost));
    if (st) {
        st->kernel_ns = hd.t_end > hd.t_start ? hd.t_end - hd.t_start : 0;
        st->n_wgs = h->n_wgs;
        st->kills = hd.kills;
        st->forks = hd.forks;
        st->episodes = hd.episodes;
        st->barriers = hd.barriers;
        st->offers = hd.offers;
        st->fork_calls = hd.fork_calls;
        st->min_m = hd.min_m;
        st->max_m = hd.max_m;
        st->final_m = (uint32_t)(hd.W >> 16) & 0xFFFFu;
        st->violations = hd.violations;
        if (st->m_trace && st->m_trace_cap && h->trace_d) {
            const uint32_t n = std::min(std::min(st->m_trace_cap, h->opts.m_trace_cap), hd.episodes);
            if (n) DCUDA(cudaMemcpy(st->m_trace, h->trace_d, 4ull * n, cudaMemcpyDeviceToHost));
        }
    }
    switch (hd.err) {
        case COOP_DEV_ERR_NONE: break;
        case COOP_DEV_ERR_TIMEOUT: return dfail(COOP_ERR_TIMEOUT, "cooperative kernel watchdog fired");
        case COOP_DEV_ERR_OVERFLOW: return dfail(COOP_ERR_OVERFLOW, "a fixed-capacity queue overflowed");
        default: return dfail(COOP_ERR_INVARIANT, "device error %u (violations %u)", hd.err, hd.violations);
    }
    if (hd.violations) return dfail(COOP_ERR_INVARIANT, "%u barrier invariant violations", hd.violations);
    return COOP_OK;
}

// ==================================================================== Fig. 4
namespace {

struct F4Params {
    const uint32_t *ro;
    const int32_t *col;
    int32_t *level;
    int32_t *q[2];      // in_nodes / out_nodes
    uint32_t *size;     // size[2]
};
struct F4Tx {           // the transmit-annotated variables of Fig. 4
    uint32_t level;
    uint32_t in_sel;    // in_nodes = q[in_sel], out_nodes = q[in_sel ^ 1]
};
enum : uint32_t { F4_START = 0, F4_AFTER_RB1 = 1, F4_AFTER_RB2 = 2 };

template <int BLOCK>
__device__ void fig4_body(coop_ctx *ctx, const F4Params &p) {
    F4Tx t;
    const uint32_t entry = coop_entry(ctx);
    if (entry == F4_START) { t.level = 0; t.in_sel = 0; }
    else coop_get_transmit(ctx, &t, sizeof t);
    bool resume_rb1 = entry == F4_AFTER_RB1;
    for (;;) {
        if (!resume_rb1) {
            const uint32_t n = *(volatile uint32_t *)&p.size[t.in_sel];
            if (n == 0) return;                                   // while (in_nodes.size > 0)
            // re-chunk after every resizing barrier
            const uint32_t tid = coop_group_id(ctx) * BLOCK + threadIdx.x;
            const uint32_t stride = coop_num_groups(ctx) * BLOCK;
            const int32_t *in = p.q[t.in_sel];
            int32_t *out = p.q[t.in_sel ^ 1u];
            uint32_t *osize = &p.size[t.in_sel ^ 1u];
            const int32_t nl = (int32_t)t.level + 1;
            for (uint32_t i = tid; i < n; i += stride) {          // process_node
                const int32_t u = in[i];
                for (uint32_t e = p.ro[u], end = p.ro[u + 1]; e < end; ++e) {
                    const int32_t v = p.col[e];
                    if (p.level[v] == -1 && atomicCAS(&p.level[v], -1, nl) == -1) out[atomicAdd(osize, 1u)] = v;
                }
            }
            t.in_sel ^= 1u;                                       // swap(&in_nodes, &out_nodes)
            if (!coop_resizing_global_barrier(ctx, &t, sizeof t, F4_AFTER_RB1)) return;
        }
        resume_rb1 = false;
        if (coop_group_id(ctx) == 0 && threadIdx.x == 0) p.size[t.in_sel ^ 1u] = 0;   // reset(out_nodes)
        t.level += 1;                                             // level++
        if (!coop_resizing_global_barrier(ctx, &t, sizeof t, F4_AFTER_RB2)) return;
    }
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) fig4_kernel(coop_dev *d, const __grid_constant__ F4Params p) {
    coop_run(d, [&](coop_ctx *ctx) { fig4_body<BLOCK>(ctx, p); });
}

// ==================================================================== work stealing
constexpr uint32_t kTW = 256;   // lanes of work per task (R19)

struct WsTask {
    unsigned long long id;
    uint32_t depth, pad;
};
struct __align__(128) WsQueue {
    uint32_t lock, head, tail;
    uint32_t pad[29];
};
struct WsParams {
    WsQueue *q;
    WsTask *tasks;              // [N][cap]
    unsigned long long *acc;    // [0] outstanding [1] count [2] total [3] steals, [8 + d] hist
    unsigned long long seed;
    uint32_t D, B, fixed, rounds, cap;
};

__device__ __forceinline__ unsigned long long splitmix(unsigned long long x) { return coop_proto::mix64(x); }

__device__ __forceinline__ void q_lock(WsQueue *q) {
    while (atomicCAS(&q->lock, 0u, 1u) != 0u) __nanosleep(32);
    __threadfence();
}
__device__ __forceinline__ void q_unlock(WsQueue *q) {
    __threadfence();
    atomicExch(&q->lock, 0u);
}

// pop_or_steal by warp 0: own queue LIFO, else the first non-empty
// victim in a scan of 32 queues at a time from a random start.
__device__ bool pop_or_steal(const WsParams &p, coop_ctx *ctx, uint32_t qid, uint32_t N, uint32_t salt,
                             WsTask *out, bool *stolen) {
    const uint32_t lane = threadIdx.x & 31u;
    bool ok = false;
    if (lane == 0) {
        WsQueue *q = p.q + qid;
        if (*(volatile uint32_t *)&q->tail != *(volatile uint32_t *)&q->head) {
            q_lock(q);
            if (q->tail != q->head) {
                q->tail -= 1;
                *out = p.tasks[(size_t)qid * p.cap + (q->tail & (p.cap - 1))];
                ok = true;
            }
            q_unlock(q);
        }
    }
    ok = __shfl_sync(0xffffffffu, ok, 0);
    if (ok) { *stolen = false; return true; }
    const uint32_t start = (uint32_t)(splitmix(((unsigned long long)ctx->phys << 32) ^ salt) % N);
    for (uint32_t base = 0; base < N; base += 32u) {
        const uint32_t v = (start + base + lane) % N;
        bool ne = false;
        if (base + lane < N && v != qid) {
            WsQueue *q = p.q + v;
            ne = *(volatile uint32_t *)&q->tail != *(volatile uint32_t *)&q->head;
        }
        uint32_t m = __ballot_sync(0xffffffffu, ne);
        while (m) {
            const uint32_t l = __ffs(m) - 1u;
            m &= m - 1u;
            bool got = false;
            if (lane == l) {
                WsQueue *q = p.q + v;
                q_lock(q);
                if (q->tail != q->head) {                       // steal the oldest (FIFO end)
                    *out = p.tasks[(size_t)v * p.cap + (q->head & (p.cap - 1))];
                    q->head += 1;
                    got = true;
                }
                q_unlock(q);
            }
            const uint32_t gl = __ballot_sync(0xffffffffu, got);
            if (gl) {
                const uint32_t src = __ffs(gl) - 1u;
                out->id = __shfl_sync(0xffffffffu, out->id, src);
                out->depth = __shfl_sync(0xffffffffu, out->depth, src);
                *stolen = true;
                return true;
            }
        }
    }
    return false;
}

template <int BLOCK>
__device__ void ws_body(coop_ctx *ctx, const WsParams &p) {
    __shared__ WsTask t_sh;
    __shared__ uint32_t have_sh;
    __shared__ unsigned long long red[BLOCK / 32];
    uint32_t iter = 0;
    for (;;) {
        // §3.2: offer to be killed, then to fork, before each task
        if (coop_offer_kill(ctx)) return;
        coop_request_fork(ctx, nullptr, 0, 1);
        if (threadIdx.x < 32) {
            uint32_t have = 0;
            if (threadIdx.x == 0)
                have = *(volatile unsigned long long *)&p.acc[0] == 0ull ? 2u : 0u;   // more_work
            have = __shfl_sync(0xffffffffu, have, 0);
            if (have == 0) {
                // the queue id is read after the fork point
                const uint32_t qid = coop_group_id(ctx);
                WsTask t;
                bool stolen = false;
                if (pop_or_steal(p, ctx, qid, ctx->d->N, iter, &t, &stolen)) {
                    have = 1;
                    if (threadIdx.x == 0) {
                        t_sh = t;
                        if (stolen) atomicAdd(&p.acc[3], 1ull);
                    }
                }
            }
            if (threadIdx.x == 0) have_sh = have;
        }
        coop_detail::cta_sync_after_t0();
        const uint32_t have = have_sh;
        ++iter;
        if (have == 2) return;                                   // no more work: finished
        if (have == 0) {
            if (threadIdx.x == 0) __nanosleep(256);
            continue;
        }
        // process_task: TW lanes of `rounds` splitmix64 applications
        const WsTask t = t_sh;
        const unsigned long long h = splitmix(t.id);
        unsigned long long s = 0;
        for (uint32_t l = threadIdx.x; l < kTW; l += BLOCK) {
            unsigned long long x = h ^ l;
            for (uint32_t r = 0; r < p.rounds; ++r) x = splitmix(x);
            s += x;
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = s;
        coop_detail::cta_sync_after_t0();
        if (threadIdx.x == 0) {
            unsigned long long tot = 0;
            for (int w = 0; w < BLOCK / 32; ++w) tot += red[w];
            const uint32_t nch = t.depth >= p.D ? 0u : (p.fixed ? p.B : (uint32_t)((h >> 32) % (p.B + 1u)));
            if (nch) {
                // count the children before they become visible (termination detection)
                atomicAdd(&p.acc[0], (unsigned long long)nch);
                const uint32_t qid = coop_group_id(ctx);
                WsQueue *q = p.q + qid;
                q_lock(q);
                if (q->tail - q->head + nch > p.cap) {
                    q_unlock(q);
                    coop_abort(ctx, COOP_DEV_ERR_OVERFLOW);
                } else {
                    for (uint32_t j = 0; j < nch; ++j) {
                        WsTask c;
                        c.id = h + j + 1ull;
                        c.depth = t.depth + 1u;
                        c.pad = 0;
                        p.tasks[(size_t)qid * p.cap + (q->tail & (p.cap - 1))] = c;
                        q->tail += 1;
                    }
                    q_unlock(q);
                }
            }
            atomicAdd(&p.acc[1], 1ull);
            atomicAdd(&p.acc[2], tot);
            atomicAdd(&p.acc[8 + t.depth], 1ull);
            __threadfence();
            atomicAdd(&p.acc[0], ~0ull);                         // this task is done (-1)
        }
        coop_detail::cta_sync_after_t0();
    }
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) ws_kernel(coop_dev *d, const __grid_constant__ WsParams p) {
    coop_run(d, [&](coop_ctx *ctx) { ws_body<BLOCK>(ctx, p); });
}

template <class K>
coop_status pick_n(coop_dev_handle *h, K kernel, uint32_t threads, uint32_t *n) {
    uint32_t cap = 0;
    DCUDA(coop_dev_max_wgs(kernel, (int)threads, 0, &cap));
    if (cap == 0) return dfail(COOP_ERR_NOT_CORESIDENT, "kernel cannot be resident");
    cap = std::min(cap, COOP_DEV_MAX_CTAS);
    if (h->opts.max_wgs > cap)
        return dfail(COOP_ERR_NOT_CORESIDENT, "max_wgs %u exceeds the co-resident capacity %u", h->opts.max_wgs, cap);
    *n = h->opts.max_wgs ? h->opts.max_wgs : cap;
    return COOP_OK;
}

}  // namespace

extern "C" coop_status coop_fig4_bfs(coop_dev_handle *h, const coop_csr *g, int64_t source, int32_t *levels_out,
                                     uint32_t threads, coop_dev_stats *stats) {
    if (!h || !g || !levels_out) return dfail(COOP_ERR_INVALID_ARG, "null argument");
    if (g->offset_bits != 32) return dfail(COOP_ERR_INVALID_ARG, "coop_fig4_bfs takes 32-bit offsets");
    if (g->num_vertices < 1 || g->num_vertices >= (1ll << 31)) return dfail(COOP_ERR_INVALID_ARG, "bad V");
    if (source < 0 || source >= g->num_vertices) return dfail(COOP_ERR_INVALID_ARG, "source out of range");
    if (threads == 0) threads = 256;
    void (*k)(coop_dev *, F4Params);
    if (threads == 128) k = fig4_kernel<128>;
    else if (threads == 256) k = fig4_kernel<256>;
    else if (threads == 512) k = fig4_kernel<512>;
    else return dfail(COOP_ERR_INVALID_ARG, "threads_per_wg %u not in {128, 256, 512}", threads);
    uint32_t N = 0;
    coop_status st = pick_n(h, k, threads, &N);
    if (st != COOP_OK) return st;
    const int64_t V = g->num_vertices;
    F4Params p;
    p.ro = (const uint32_t *)g->row_offsets;
    p.col = g->col_idx;
    p.level = levels_out;
    int32_t *qbuf = nullptr;
    DCUDA(cudaMalloc((void **)&qbuf, sizeof(int32_t) * (2 * V + 32)));
    p.q[0] = qbuf;
    p.q[1] = qbuf + V;
    p.size = (uint32_t *)(qbuf + 2 * V);
    const int32_t src = (int32_t)source, zero = 0;
    const uint32_t sizes[2] = {1u, 0u};
    cudaStream_t s = nullptr;
    cudaError_t e = cudaMemsetAsync(levels_out, 0xFF, sizeof(int32_t) * V, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(levels_out + source, &zero, 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p.q[0], &src, 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p.size, sizes, 8, cudaMemcpyHostToDevice, s);
    coop_dev *d = nullptr;
    if (e == cudaSuccess) {
        st = coop_dev_arm(h, N, s, &d);
        if (st == COOP_OK) e = coop_dev_launch(k, N, threads, 0, s, d, p);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        cudaFree(qbuf);
        return dfail(COOP_ERR_CUDA, "fig4 launch: %s", cudaGetErrorString(e));
    }
    if (st == COOP_OK) st = coop_dev_collect(h, s, stats);
    cudaFree(qbuf);
    return st;
}

extern "C" coop_status coop_work_steal(coop_dev_handle *h, const coop_ws_tree *tree, uint32_t threads,
                                       coop_ws_result *res, coop_dev_stats *stats) {
    if (!h || !tree || !res) return dfail(COOP_ERR_INVALID_ARG, "null argument");
    if (tree->depth > 62) return dfail(COOP_ERR_INVALID_ARG, "depth %u > 62", tree->depth);
    const uint32_t cap = tree->queue_cap ? tree->queue_cap : 1024u;
    if (cap & (cap - 1)) return dfail(COOP_ERR_INVALID_ARG, "queue_cap %u not a power of two", cap);
    if (threads == 0) threads = 256;
    void (*k)(coop_dev *, WsParams);
    if (threads == 128) k = ws_kernel<128>;
    else if (threads == 256) k = ws_kernel<256>;
    else if (threads == 512) k = ws_kernel<512>;
    else return dfail(COOP_ERR_INVALID_ARG, "threads_per_wg %u not in {128, 256, 512}", threads);
    uint32_t N = 0;
    coop_status st = pick_n(h, k, threads, &N);
    if (st != COOP_OK) return st;
    WsParams p;
    p.seed = tree->seed;
    p.D = tree->depth;
    p.B = tree->max_fanout;
    p.fixed = tree->fixed ? 1u : 0u;
    p.rounds = tree->rounds;
    p.cap = cap;
    const size_t qbytes = sizeof(WsQueue) * N, tbytes = sizeof(WsTask) * (size_t)N * cap, abytes = 8 * 72;
    char *buf = nullptr;
    DCUDA(cudaMalloc((void **)&buf, qbytes + tbytes + abytes));
    p.q = (WsQueue *)buf;
    p.tasks = (WsTask *)(buf + qbytes);
    p.acc = (unsigned long long *)(buf + qbytes + tbytes);
    cudaStream_t s = nullptr;
    // initial state: the root task in queue 0 (the host-initialised queues of Fig. 2)
    WsQueue q0;
    memset(&q0, 0, sizeof q0);
    q0.tail = 1;
    WsTask root = {tree->seed, 0u, 0u};
    unsigned long long one = 1;
    cudaError_t e = cudaMemsetAsync(p.q, 0, qbytes, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(p.acc, 0, abytes, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p.q, &q0, sizeof q0, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p.tasks, &root, sizeof root, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p.acc, &one, 8, cudaMemcpyHostToDevice, s);
    coop_dev *d = nullptr;
    if (e == cudaSuccess) {
        st = coop_dev_arm(h, N, s, &d);
        if (st == COOP_OK) e = coop_dev_launch(k, N, threads, 0, s, d, p);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        cudaFree(buf);
        return dfail(COOP_ERR_CUDA, "work-stealing launch: %s", cudaGetErrorString(e));
    }
    if (st == COOP_OK) st = coop_dev_collect(h, s, stats);
    unsigned long long acc[72];
    cudaError_t e2 = cudaMemcpy(acc, p.acc, abytes, cudaMemcpyDeviceToHost);
    cudaFree(buf);
    if (e2 != cudaSuccess) return dfail(COOP_ERR_CUDA, "reading results: %s", cudaGetErrorString(e2));
    memset(res, 0, sizeof *res);
    res->count = acc[1];
    res->total = acc[2];
    res->steals = acc[3];
    for (int i = 0; i < 64; ++i) res->hist[i] = acc[8 + i];
    return st;
}

// ==================================================================== Pannotia apps (Table 1)
// color, mis and p-sssp ported to cooperative kernels on the
// device API, with the resizing-barrier counts of Table 1 (color 2/2, mis 3/3,
// p-sssp 3/3): vertex-strided loops re-chunked after every resizing barrier
// (P:695-705); the only transmitted state is the iteration counter.  Algorithms:
// DESIGN.md reading R23 (Jones-Plassmann colouring and Luby's MIS with fixed
// priorities prio(v) = (splitmix64(seed ^ v), v); Bellman-Ford over all vertices).
namespace {

struct PnParams {
    const uint32_t *ro;
    const int32_t *col;
    const uint32_t *w;
    int32_t *a;                 // colour / MIS state / distance (u32 bits)
    uint32_t *b;                // p-sssp: next distances
    uint32_t *flag;             // [2]: work remains in iteration parity p
    uint32_t *iters;            // out
    unsigned long long seed;
    uint32_t V;
};
struct PnTx {
    uint32_t it;
};
enum : uint32_t { PN_START = 0, PN_B = 1, PN_C = 2, PN_NEXT = 3 };
constexpr int32_t PN_UNC = -1, PN_UND = 0, PN_IN = 1, PN_OUT = 2;
constexpr uint32_t PN_INF = 0xFFFFFFFFu;

// (splitmix64(seed ^ v), v) > (splitmix64(seed ^ u), u)
__device__ __forceinline__ bool prio_gt(unsigned long long seed, uint32_t v, uint32_t u) {
    const unsigned long long pv = coop_proto::mix64(seed ^ v), pu = coop_proto::mix64(seed ^ u);
    return pv > pu || (pv == pu && v > u);
}

template <int BLOCK>
__device__ void color_body(coop_ctx *ctx, const PnParams &p) {
    PnTx t;
    uint32_t entry = coop_entry(ctx);
    if (entry == PN_START) t.it = 0;
    else coop_get_transmit(ctx, &t, sizeof t);
    for (;;) {
        if (entry != PN_B) {
            // A: an uncoloured vertex above every neighbour uncoloured at the start of the
            // iteration takes colour it (a neighbour coloured `it` right now still counts)
            const uint32_t tid = coop_group_id(ctx) * BLOCK + threadIdx.x, stride = coop_num_groups(ctx) * BLOCK;
            const int32_t it = (int32_t)t.it;
            for (uint32_t v = tid; v < p.V; v += stride) {
                if (*(volatile int32_t *)&p.a[v] != PN_UNC) continue;
                bool top = true;
                for (uint32_t e = p.ro[v], end = p.ro[v + 1]; e < end && top; ++e) {
                    const uint32_t u = (uint32_t)p.col[e];
                    const int32_t cu = *(volatile int32_t *)&p.a[u];
                    if ((cu == PN_UNC || cu == it) && prio_gt(p.seed, u, v)) top = false;
                }
                if (top) p.a[v] = it;
                else atomicOr(&p.flag[t.it & 1u], 1u);
            }
            if (!coop_resizing_global_barrier(ctx, &t, sizeof t, PN_B)) return;
        }
        // B: the iteration's flag is final after the barrier; recycle the other parity
        if (coop_group_id(ctx) == 0 && threadIdx.x == 0) p.flag[(t.it + 1u) & 1u] = 0u;
        const bool done = *(volatile uint32_t *)&p.flag[t.it & 1u] == 0u;
        if (done) {
            if (coop_group_id(ctx) == 0 && threadIdx.x == 0) *p.iters = t.it + 1u;
            return;
        }
        t.it += 1u;
        if (!coop_resizing_global_barrier(ctx, &t, sizeof t, PN_NEXT)) return;
        entry = PN_NEXT;
    }
}

template <int BLOCK>
__device__ void mis_body(coop_ctx *ctx, const PnParams &p) {
    PnTx t;
    uint32_t entry = coop_entry(ctx);
    if (entry == PN_START) t.it = 0;
    else coop_get_transmit(ctx, &t, sizeof t);
    for (;;) {
        if (entry != PN_B && entry != PN_C) {
            // A: an undecided vertex below every undecided neighbour joins (an earlier member
            // has no undecided neighbour, so IN here means "joined this iteration")
            const uint32_t tid = coop_group_id(ctx) * BLOCK + threadIdx.x, stride = coop_num_groups(ctx) * BLOCK;
            for (uint32_t v = tid; v < p.V; v += stride) {
                if (*(volatile int32_t *)&p.a[v] != PN_UND) continue;
                bool low = true;
                for (uint32_t e = p.ro[v], end = p.ro[v + 1]; e < end && low; ++e) {
                    const uint32_t u = (uint32_t)p.col[e];
                    const int32_t su = *(volatile int32_t *)&p.a[u];
                    if ((su == PN_UND || su == PN_IN) && prio_gt(p.seed, v, u)) low = false;
                }
                if (low) p.a[v] = PN_IN;
            }
            if (!coop_resizing_global_barrier(ctx, &t, sizeof t, PN_B)) return;
        }
        if (entry != PN_C) {
            // B: an undecided neighbour of a member leaves; the rest remain
            const uint32_t tid = coop_group_id(ctx) * BLOCK + threadIdx.x, stride = coop_num_groups(ctx) * BLOCK;
            for (uint32_t v = tid; v < p.V; v += stride) {
                if (p.a[v] != PN_UND) continue;
                bool out = false;
                for (uint32_t e = p.ro[v], end = p.ro[v + 1]; e < end && !out; ++e)
                    out = p.a[p.col[e]] == PN_IN;
                if (out) p.a[v] = PN_OUT;
                else atomicOr(&p.flag[t.it & 1u], 1u);
            }
            if (!coop_resizing_global_barrier(ctx, &t, sizeof t, PN_C)) return;
        }
        // C: termination test
        if (coop_group_id(ctx) == 0 && threadIdx.x == 0) p.flag[(t.it + 1u) & 1u] = 0u;
        const bool done = *(volatile uint32_t *)&p.flag[t.it & 1u] == 0u;
        if (done) {
            if (coop_group_id(ctx) == 0 && threadIdx.x == 0) *p.iters = t.it + 1u;
            return;
        }
        t.it += 1u;
        if (!coop_resizing_global_barrier(ctx, &t, sizeof t, PN_NEXT)) return;
        entry = PN_NEXT;
    }
}

template <int BLOCK>
__device__ void psssp_body(coop_ctx *ctx, const PnParams &p) {
    PnTx t;
    uint32_t entry = coop_entry(ctx);
    if (entry == PN_START) t.it = 0;
    else coop_get_transmit(ctx, &t, sizeof t);
    uint32_t *d = reinterpret_cast<uint32_t *>(p.a);
    for (;;) {
        if (entry != PN_B && entry != PN_C) {
            // A: pull relaxation of every vertex over its in-edges (symmetric graph)
            const uint32_t tid = coop_group_id(ctx) * BLOCK + threadIdx.x, stride = coop_num_groups(ctx) * BLOCK;
            for (uint32_t v = tid; v < p.V; v += stride) {
                uint32_t nd = d[v];
                for (uint32_t e = p.ro[v], end = p.ro[v + 1]; e < end; ++e) {
                    const uint32_t du = d[p.col[e]];
                    if (du != PN_INF && du + p.w[e] < nd) nd = du + p.w[e];
                }
                p.b[v] = nd;
            }
            if (!coop_resizing_global_barrier(ctx, &t, sizeof t, PN_B)) return;
        }
        if (entry != PN_C) {
            // B: publish the improvements
            const uint32_t tid = coop_group_id(ctx) * BLOCK + threadIdx.x, stride = coop_num_groups(ctx) * BLOCK;
            for (uint32_t v = tid; v < p.V; v += stride) {
                const uint32_t nd = p.b[v];
                if (nd != d[v]) {
                    d[v] = nd;
                    atomicOr(&p.flag[t.it & 1u], 1u);
                }
            }
            if (!coop_resizing_global_barrier(ctx, &t, sizeof t, PN_C)) return;
        }
        if (coop_group_id(ctx) == 0 && threadIdx.x == 0) p.flag[(t.it + 1u) & 1u] = 0u;
        const bool done = *(volatile uint32_t *)&p.flag[t.it & 1u] == 0u;
        if (done) {
            if (coop_group_id(ctx) == 0 && threadIdx.x == 0) *p.iters = t.it + 1u;
            return;
        }
        t.it += 1u;
        if (!coop_resizing_global_barrier(ctx, &t, sizeof t, PN_NEXT)) return;
        entry = PN_NEXT;
    }
}

template <int BLOCK, int APP>
__global__ void __launch_bounds__(BLOCK) pannotia_kernel(coop_dev *d, const __grid_constant__ PnParams p) {
    coop_run(d, [&](coop_ctx *ctx) {
        if (APP == 0) color_body<BLOCK>(ctx, p);
        else if (APP == 1) mis_body<BLOCK>(ctx, p);
        else psssp_body<BLOCK>(ctx, p);
    });
}

template <int APP>
coop_status pannotia_run(coop_dev_handle *h, const coop_csr *g, uint64_t seed_or_source, int32_t *out,
                         uint32_t threads, uint32_t *iters_out, coop_dev_stats *stats) {
    if (!h || !g || !out || !iters_out) return dfail(COOP_ERR_INVALID_ARG, "null argument");
    if (g->offset_bits != 32) return dfail(COOP_ERR_INVALID_ARG, "Pannotia apps take 32-bit offsets");
    if (g->num_vertices < 1 || g->num_vertices >= (1ll << 31)) return dfail(COOP_ERR_INVALID_ARG, "bad V");
    if (APP == 2) {
        if (!g->weights && g->num_edges) return dfail(COOP_ERR_INVALID_ARG, "p-sssp needs weights");
        if ((int64_t)seed_or_source >= g->num_vertices) return dfail(COOP_ERR_INVALID_ARG, "source out of range");
        if (g->max_weight && (uint64_t)(g->num_vertices - 1) * g->max_weight >= 0xFFFFFFFFull)
            return dfail(COOP_ERR_OVERFLOW, "(V-1)*max_weight >= 2^32-1");
    }
    if (threads == 0) threads = 256;
    void (*k)(coop_dev *, PnParams);
    if (threads == 128) k = pannotia_kernel<128, APP>;
    else if (threads == 256) k = pannotia_kernel<256, APP>;
    else if (threads == 512) k = pannotia_kernel<512, APP>;
    else return dfail(COOP_ERR_INVALID_ARG, "threads_per_wg %u not in {128, 256, 512}", threads);
    uint32_t N = 0;
    coop_status st = pick_n(h, k, threads, &N);
    if (st != COOP_OK) return st;
    const int64_t V = g->num_vertices;
    PnParams p;
    p.ro = (const uint32_t *)g->row_offsets;
    p.col = g->col_idx;
    p.w = g->weights;
    p.a = out;
    p.V = (uint32_t)V;
    p.seed = seed_or_source;
    uint32_t *buf = nullptr;
    DCUDA(cudaMalloc((void **)&buf, sizeof(uint32_t) * ((APP == 2 ? V : 0) + 8)));
    p.b = buf + 8;
    p.flag = buf;
    p.iters = buf + 4;
    cudaStream_t s = nullptr;
    cudaError_t e = cudaMemsetAsync(buf, 0, 32, s);
    if (e == cudaSuccess) {
        if (APP == 0) e = cudaMemsetAsync(out, 0xFF, sizeof(int32_t) * V, s);           // uncoloured
        else if (APP == 1) e = cudaMemsetAsync(out, 0, sizeof(int32_t) * V, s);        // undecided
        else {
            e = cudaMemsetAsync(out, 0xFF, sizeof(int32_t) * V, s);                    // INF
            const uint32_t zero = 0;
            if (e == cudaSuccess) e = cudaMemcpyAsync(out + seed_or_source, &zero, 4, cudaMemcpyHostToDevice, s);
        }
    }
    coop_dev *d = nullptr;
    if (e == cudaSuccess) {
        st = coop_dev_arm(h, N, s, &d);
        if (st == COOP_OK) e = coop_dev_launch(k, N, threads, 0, s, d, p);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        cudaFree(buf);
        return dfail(COOP_ERR_CUDA, "pannotia launch: %s", cudaGetErrorString(e));
    }
    if (st == COOP_OK) st = coop_dev_collect(h, s, stats);
    if (st == COOP_OK) {
        cudaError_t e2 = cudaMemcpy(iters_out, p.iters, 4, cudaMemcpyDeviceToHost);
        if (e2 != cudaSuccess) st = dfail(COOP_ERR_CUDA, "iterations: %s", cudaGetErrorString(e2));
    }
    cudaFree(buf);
    return st;
}

}  // namespace

extern "C" coop_status coop_color(coop_dev_handle *h, const coop_csr *g, uint64_t seed, int32_t *colors_out,
                                  uint32_t threads, uint32_t *iters_out, coop_dev_stats *stats) {
    return pannotia_run<0>(h, g, seed, colors_out, threads, iters_out, stats);
}
extern "C" coop_status coop_mis(coop_dev_handle *h, const coop_csr *g, uint64_t seed, int32_t *state_out,
                                uint32_t threads, uint32_t *iters_out, coop_dev_stats *stats) {
    return pannotia_run<1>(h, g, seed, state_out, threads, iters_out, stats);
}
extern "C" coop_status coop_psssp(coop_dev_handle *h, const coop_csr *g, int64_t source, uint32_t *dist_out,
                                  uint32_t threads, uint32_t *iters_out, coop_dev_stats *stats) {
    if (source < 0) return dfail(COOP_ERR_INVALID_ARG, "source out of range");
    return pannotia_run<2>(h, g, (uint64_t)source, reinterpret_cast<int32_t *>(dist_out), threads, iters_out, stats);
}
