/*
 * coop_device.cuh -- device half of libcoop: the cooperative-kernel
 * programming model (Sorensen, Evrard, Donaldson, arXiv 1707.01989, §3) for
 * kernels written by the user, on NVIDIA B200 (sm_100a).
 *
 * A cooperative kernel is launched with N co-resident CTAs (the paper's
 * occupancy-bound execution); M of them are ACTIVE with
 * contiguous logical ids [0, M), the rest wait in the
 * library's worker loop (the megakernel pool) until a fork
 * gives them an id.  The body calls, CTA-collectively (every thread of the CTA,
 * uniform control flow):
 *
 *   coop_offer_kill(ctx)                  PAPER.md:529-550.  True => the
 *        scheduler accepted: the CTA has left the active set and the body must
 *        `return` at once (its id was M-1; only M-1 > 0 can leave).
 *   coop_request_fork(ctx, tx, bytes, e)  PAPER.md:553-592.  Returns k >= 0:
 *        k parked CTAs joined with ids [M, M+k) (M before the call) and will
 *        start the body at entry point e with `bytes` of transmitted state
 *        copied from `tx`.  k = 0 when M = N.
 *   coop_global_barrier(ctx)              PAPER.md:600-610.  Barrier over the
 *        M active CTAs.  False => abort (watchdog / error): return.
 *   coop_resizing_global_barrier(ctx, tx, bytes, e)   PAPER.md:612-638 in
 *        the query form: the scheduler may kill ids >= M' or fork
 *        ids [M, M'), which start at entry point e with workgroup 0's `tx`
 *        (P:622-624).  False => this CTA was killed (or abort): return.
 *   coop_group_id(ctx) / coop_num_groups(ctx)   get_group_id / get_num_groups
 *        (P:519-522); M as of this CTA's last cooperative call -- stable within
 *        a resizing-barrier interval when the body makes no bare kill/fork
 *        calls.
 *   coop_query_dev(ctx)                   outstanding demand W (query).
 *   coop_entry(ctx), coop_get_transmit(ctx, dst, bytes)   where a forked CTA
 *        starts and the state it received (0 = kernel start, never forked).
 *
 * The kernel itself is written as
 *
 *   __global__ void my_kernel(coop_dev *d, ...) {
 *       coop_run(d, [&](coop_ctx *ctx) { ...body...; });
 *   }
 *
 * and launched through coop_dev_launch() below with a control block from the
 * host ABI in coop.h (coop_dev_create / coop_dev_arm / coop_dev_collect).
 * coop_run starts CTAs [0, M0) in the body at entry 0, parks the others, and
 * re-enters forked CTAs at their entry point.  Killed CTAs return to the pool
 * and can be forked again; when a CTA returns from the body without being
 * killed the computation is finished and parked CTAs exit.
 *
 * Scheduler decisions (coop_dev_opts.policy, the paper's nondeterministic
 * choices P:545-548):
 *   COOP_POLICY_NEVER     never kill or fork;
 *   COOP_POLICY_SCRIPTED  resizing barrier e sets M' = script[e] (0 = unchanged);
 *   COOP_POLICY_RANDOM    counter RNG keyed by (seed, episode) at resizing
 *                         barriers (resize_prob, M' ~ U[1, N]) and by (seed, CTA,
 *                         call) at bare calls (kill_prob; fork_prob with k ~ U[1, max_fork]);
 *   COOP_POLICY_SCHEDULER resource messages from the host (coop_dev_demand /
 *                         coop_dev_grant): kill while demand is outstanding, fork
 *                         up to the granted count.
 *
 * Protocol (model-checked in oracle/barrier_model.py): a packed
 * arrival word W = {gen:32 | M:16 | arrived:16} and a release word R on its own
 * 128-B line.  Arrival = fence + atomicAdd(W, 1); the CTA completing
 * arrived == M runs the serial section (policy, forks, statistics) and
 * releases R = {gen+1, M'}.  Bare offer_kill = CAS W {g, M, a} -> {g, M-1, a}
 * by id M-1 (completing the episode on the waiters' behalf if a == M-1); bare
 * request_fork claims parked CTAs from the pool bitmap, then CAS
 * W {g, M, a} -> {g, M+k, a} and hands out ids [M, M+k) through mailboxes.
 * Every spin is bounded by a %globaltimer watchdog (coop_dev_opts.timeout_ns).
 *
 * Memory ordering: the barrier is a release/acquire point at gpu scope
 * (all writes before it by any active CTA are visible after it to all).
 */
#ifndef COOP_DEVICE_CUH
#define COOP_DEVICE_CUH

#include <stdint.h>

#include "coop.h"
#include "coop_protocol.cuh"

#define COOP_TX_MAX 64u                 /* bytes of transmitted state */
#define COOP_DEV_MAX_CTAS 4096u
#define COOP_DEV_POOL_WORDS (COOP_DEV_MAX_CTAS / 32u)

/* coop_dev error word values (coop_dev_collect maps them to coop_status) */
#define COOP_DEV_ERR_NONE 0u
#define COOP_DEV_ERR_TIMEOUT 1u
#define COOP_DEV_ERR_INVARIANT 2u
#define COOP_DEV_ERR_APP 3u            /* set by the body through coop_abort(ctx, COOP_DEV_ERR_APP) */
#define COOP_DEV_ERR_OVERFLOW 4u       /* an app's fixed-capacity structure overflowed */

typedef struct __align__(64) {
    uint32_t flag;                      /* assignments so far (parked CTA consumed them when equal) */
    uint32_t lid, gen, entry;
    uint8_t tx[COOP_TX_MAX];
} coop_dev_mailbox;

/* Control block (device memory; created and armed by the host ABI). */
typedef struct __align__(128) coop_dev {
    unsigned long long W;               /* arrivals {gen:32 | M:16 | arrived:16} */
    unsigned long long pad_w[15];
    unsigned long long R;               /* release {gen:32 | M':16 | 0} */
    unsigned long long pad_r[15];
    uint32_t demand_posted, grant_posted;   /* host-written, monotone (resource messages) */
    uint32_t demand_taken, grant_taken;     /* device atomics */
    uint32_t pad_c[28];
    uint32_t done, err;
    uint32_t pad_s[30];
    /* configuration (immutable during a launch) */
    uint32_t N, M0, policy, flags;
    unsigned long long seed;
    uint32_t kill_thresh, fork_thresh, resize_thresh, max_fork;
    const uint32_t *script;
    uint32_t script_len, m_trace_cap;
    uint32_t *m_trace;
    unsigned long long timeout_ns;
    coop_dev_mailbox *mb;
    uint32_t pad_g[10];
    /* workgroup 0's transmit at the barrier in progress */
    uint32_t tx0_kind, tx0_entry, tx0_bytes, pad_t;
    uint8_t tx0[COOP_TX_MAX];
    uint32_t pad_t2[12];
    /* statistics */
    uint32_t kills, forks, episodes, barriers, offers, fork_calls, min_m, max_m, violations, finished;
    uint32_t pad_x[2];
    unsigned long long t_start, t_end;
    /* COOP_FLAG_CHECK */
    uint32_t chk_arr[2];
    uint32_t idmap[2][COOP_DEV_POOL_WORDS];
    /* parked, forkable physical CTAs */
    uint32_t pool[COOP_DEV_POOL_WORDS];
} coop_dev;

#ifdef __CUDACC__

/* Per-CTA state, in shared memory (owned by coop_run). */
typedef struct {
    coop_dev *d;
    uint32_t lid, M, gen, entry, phys, consumed, state, last, bar_M, calls, bcast, offers;
    unsigned long long deadline;
    uint8_t tx[COOP_TX_MAX];
} coop_ctx;

enum { COOP_ST_ACTIVE = 0, COOP_ST_KILLED = 1, COOP_ST_ABORT = 2 };

namespace coop_detail {

/* ordered accesses, the packed words and the generator come from the shared
 * protocol header (the same steps the BFS/SSSP runtime uses) */
using namespace coop_proto;

/* CTA barrier after a region only some lanes of a warp execute (thread-0
 * blocks, spin loops).  Measured on sm_100a (tools/fork_repro.cu): when ptxas
 * lays out a straight-line `if (threadIdx.x == 0) {...}` as a plain forward
 * branch with no reconvergence point, lanes 1..31 reach the (warp-aligned) CTA
 * barrier before lane 0; the warp is counted for them and again when lane 0
 * arrives, so the NEXT barrier releases the other warps early.  ptxas believes
 * the warp is converged there and deletes a plain __syncwarp(), so the
 * reconvergence uses a mask it cannot see through (a __constant__ word). */
__constant__ uint32_t coop_full_mask = 0xffffffffu;   /* constant cache: no memory round trip */
__device__ __forceinline__ void cta_sync_after_t0() {
    __syncwarp(coop_full_mask);
    asm volatile("barrier.sync 0;" ::: "memory");
}

/* thread-level: true => abort (error word set by someone, or watchdog) */
__device__ __forceinline__ bool abort_check(coop_ctx *c, uint32_t &spins) {
    if ((++spins & 63u) != 0) return false;
    coop_dev *d = c->d;
    if (ld_relaxed32(&d->err) != COOP_DEV_ERR_NONE) return true;
    if (globaltimer() > c->deadline) {
        atomicCAS(&d->err, COOP_DEV_ERR_NONE, COOP_DEV_ERR_TIMEOUT);
        st_release32(&d->done, 1u);
        return true;
    }
    return false;
}

__device__ __forceinline__ void copy_tx(uint8_t *dst, const uint8_t *src, uint32_t bytes) {
    for (uint32_t i = 0; i < bytes; ++i) dst[i] = src[i];
}

/* hand id `lid`, generation `gen`, entry point and transmit to parked CTA `phys` */
__device__ __forceinline__ void assign(coop_dev *d, uint32_t phys, uint32_t lid, uint32_t gen, uint32_t entry,
                                      const uint8_t *tx, uint32_t bytes) {
    coop_dev_mailbox *mb = d->mb + phys;
    const uint32_t f = mb->flag;        // only the claimer of `phys` writes its mailbox
    mb->lid = lid;
    mb->gen = gen;
    mb->entry = entry;
    copy_tx(mb->tx, tx, bytes);
    __threadfence();
    st_release32(&mb->flag, f + 1u);
}

/* Warp-collective (warp 0): claim up to k parked CTAs from the pool bitmap.
 * With out_phys == nullptr each claimed CTA is assigned at once the id
 * base + i (generation gen, entry point, transmit); otherwise the physical ids
 * are stored to out_phys[0, got).  With `wait`, retries until k are found
 * (killed CTAs park promptly). */
__device__ __noinline__ uint32_t claim_pool(coop_ctx *c, uint32_t k, bool wait, uint32_t *out_phys, uint32_t base,
                                            uint32_t gen, uint32_t entry, const uint8_t *tx, uint32_t bytes) {
    coop_dev *d = c->d;
    uint32_t spins = 0;
    return claim_idle(d->pool, (d->N + 31u) / 32u, k, wait,
        [&](uint32_t phys, uint32_t i) {
            if (out_phys) out_phys[i] = phys;
            else assign(d, phys, base + i, gen, entry, tx, bytes);
        },
        [&]() { return abort_check(c, spins); });
}

/* Serial section of episode g (warp 0 of the CTA completing it; all M active
 * CTAs wait).  Returns M' (broadcast to the warp).  `behalf`: the caller is a
 * CTA that just left by offer_kill and completes the episode for the waiters;
 * it is not in the pool yet, so at most N-M-1 CTAs can be forked (a waiting
 * fork of N-M would never finish: oracle/barrier_model.py bug
 * "no_cap_on_behalf"). */
__device__ __noinline__ uint32_t serial_section(coop_ctx *c, uint32_t g, uint32_t M, bool behalf = false) {
    coop_dev *d = c->d;
    const uint32_t lane = threadIdx.x & 31u;
    const bool resizing = d->tx0_kind != 0u;
    uint32_t Mp = M, take = 0, fork_want = 0;
    bool wait = false, sched = false;
    if (lane == 0 && resizing) {
        const uint32_t ep = d->episodes;
        if (d->policy == COOP_POLICY_SCRIPTED) {
            uint32_t s = ep < d->script_len ? d->script[ep] : 0u;
            if (s) Mp = s;
            wait = true;
        } else if (d->policy == COOP_POLICY_RANDOM) {
            unsigned long long h = mix64(d->seed * 0x2545F4914F6CDD1Dull + ep);
            if ((uint32_t)h < d->resize_thresh) Mp = 1u + (uint32_t)((h >> 32) % d->N);
            wait = true;
        } else if (d->policy == COOP_POLICY_SCHEDULER) {
            /* query(): W = outstanding demand, satisfied up to M-1 in one episode */
            uint32_t t = ld_relaxed32(&d->demand_taken);
            for (;;) {
                const uint32_t posted = ld_relaxed32(&d->demand_posted);
                if (posted <= t || M <= 1) break;
                const uint32_t want = min(posted - t, M - 1u);
                const uint32_t old = atomicCAS(&d->demand_taken, t, t + want);
                if (old == t) { take = want; break; }
                t = old;
            }
            if (take) {
                Mp = M - take;
            } else if (M < d->N) {
                uint32_t gt = ld_relaxed32(&d->grant_taken);
                for (;;) {
                    const uint32_t posted = ld_relaxed32(&d->grant_posted);
                    if (posted <= gt) break;
                    const uint32_t want = min(posted - gt, d->N - M);
                    const uint32_t old = atomicCAS(&d->grant_taken, gt, gt + want);
                    if (old == gt) { Mp = M + want; sched = true; break; }
                    gt = old;
                }
            }
        }
        Mp = max(1u, min(Mp, d->N));
        if (behalf && wait) Mp = min(Mp, d->N - 1u);
        fork_want = Mp > M ? Mp - M : 0u;
    }
    fork_want = __shfl_sync(0xffffffffu, fork_want, 0);
    wait = __shfl_sync(0xffffffffu, (uint32_t)wait, 0) != 0u;
    uint32_t got = 0;
    if (fork_want) {
        /* new ids [M, M+got) join generation g+1 at WG 0's entry point with WG 0's transmit */
        got = claim_pool(c, fork_want, wait, nullptr, M, g + 1u, d->tx0_entry, d->tx0, d->tx0_bytes);
    }
    if (lane == 0) {
        if (fork_want) {
            if (sched && got < fork_want) atomicSub(&d->grant_taken, fork_want - got);
            Mp = M + got;
        }
        if (resizing) {
            const uint32_t ep = d->episodes;
            if (ep < d->m_trace_cap) d->m_trace[ep] = Mp;
            d->episodes = ep + 1u;
        }
        d->barriers += 1u;
        if (Mp < M) atomicAdd(&d->kills, M - Mp);
        if (got) atomicAdd(&d->forks, got);
        if (Mp != M) {
            atomicMin(&d->min_m, Mp);
            atomicMax(&d->max_m, Mp);
        }
        if (d->flags & COOP_FLAG_CHECK) {   /* every active CTA arrived once, ids exactly [0, M) */
            bool bad = atomicExch(&d->chk_arr[g & 1u], 0u) != M;
            const uint32_t nw = (d->N + 31u) / 32u;
            for (uint32_t w = 0; w < nw; ++w) {
                const uint32_t bits = atomicExch(&d->idmap[g & 1u][w], 0u), lo = w * 32u;
                const uint32_t expect = M >= lo + 32u ? 0xffffffffu : (M > lo ? ((1u << (M - lo)) - 1u) : 0u);
                bad |= bits != expect;
            }
            if (bad) {
                atomicAdd(&d->violations, 1u);
                atomicCAS(&d->err, COOP_DEV_ERR_NONE, COOP_DEV_ERR_INVARIANT);
            }
        }
        publish(&d->W, &d->R, g + 1u, Mp);
    }
    return __shfl_sync(0xffffffffu, Mp, 0);
}

/* CTA-collective barrier; kind 0 = global_barrier, 1 = resizing_global_barrier */
__device__ __noinline__ bool barrier(coop_ctx *c, uint32_t kind, const void *tx, uint32_t bytes, uint32_t entry) {
    coop_dev *d = c->d;
    coop_detail::cta_sync_after_t0();
    if (threadIdx.x == 0) {
        const uint32_t g = c->gen;
        if (c->lid == 0) {   /* publish WG 0's transmit and the barrier kind (released by the arrival) */
            d->tx0_kind = kind;
            d->tx0_entry = entry;
            d->tx0_bytes = bytes;
            copy_tx(d->tx0, (const uint8_t *)tx, bytes);
        }
        if (d->flags & COOP_FLAG_CHECK) {
            atomicAdd(&d->chk_arr[g & 1u], 1u);
            atomicOr(&d->idmap[g & 1u][c->lid >> 5], 1u << (c->lid & 31u));
        }
        const unsigned long long old = arrive_fenced(&d->W);
        const uint32_t last = is_last(old);
        if (w_gen(old) != g) {
            atomicCAS(&d->err, COOP_DEV_ERR_NONE, COOP_DEV_ERR_INVARIANT);
            st_release32(&d->done, 1u);
        }
        c->last = last;
        c->bar_M = w_M(old);
        if (!last) {
            uint32_t spins = 0;
            unsigned long long r;
            for (;;) {
                r = ld_acquire64(&d->R);
                if (w_gen(r) != g) break;
                if (abort_check(c, spins)) { c->state = COOP_ST_ABORT; break; }
            }
            if (c->state != COOP_ST_ABORT) {
                if (fate(r, g, c->lid) == FATE_KILLED) c->state = COOP_ST_KILLED;
                else { c->M = w_M(r); c->gen = g + 1u; }
            }
        }
    }
    cta_sync_after_t0();
    if (c->last) {
        if (threadIdx.x < 32) {
            const uint32_t Mp = serial_section(c, c->gen, c->bar_M);
            if (threadIdx.x == 0) {
                if (c->lid >= Mp) c->state = COOP_ST_KILLED;
                else { c->M = Mp; c->gen += 1u; }
            }
        }
        coop_detail::cta_sync_after_t0();
    }
    return c->state == COOP_ST_ACTIVE;
}

}  // namespace coop_detail

__device__ __forceinline__ uint32_t coop_group_id(const coop_ctx *c) { return c->lid; }
__device__ __forceinline__ uint32_t coop_num_groups(const coop_ctx *c) { return c->M; }
__device__ __forceinline__ uint32_t coop_entry(const coop_ctx *c) { return c->entry; }
__device__ __forceinline__ void coop_get_transmit(const coop_ctx *c, void *dst, uint32_t bytes) {
    coop_detail::copy_tx((uint8_t *)dst, c->tx, bytes < COOP_TX_MAX ? bytes : COOP_TX_MAX);
}
/* outstanding demand (query), capped at M-1 */
__device__ __forceinline__ uint32_t coop_query_dev(const coop_ctx *c) {
    const uint32_t p = coop_detail::ld_relaxed32(&c->d->demand_posted), t = coop_detail::ld_relaxed32(&c->d->demand_taken);
    const uint32_t w = p > t ? p - t : 0u;
    return c->M > 1u ? min(w, c->M - 1u) : 0u;
}
/* body-detected error: every CTA leaves, the host call returns COOP_ERR_INVARIANT/... */
__device__ __forceinline__ void coop_abort(coop_ctx *c, uint32_t code) {
    atomicCAS(&c->d->err, COOP_DEV_ERR_NONE, code);
    coop_detail::st_release32(&c->d->done, 1u);
}

__device__ __forceinline__ bool coop_global_barrier(coop_ctx *c) {
    return coop_detail::barrier(c, 0u, nullptr, 0u, 0u);
}
__device__ __forceinline__ bool coop_resizing_global_barrier(coop_ctx *c, const void *tx, uint32_t bytes,
                                                             uint32_t entry) {
    return coop_detail::barrier(c, 1u, tx, bytes < COOP_TX_MAX ? bytes : COOP_TX_MAX, entry);
}

/* offer_kill.  CTA-collective.  True => killed (or abort): return. */
__device__ __noinline__ bool coop_offer_kill(coop_ctx *c) {
    using namespace coop_detail;
    coop_dev *d = c->d;
    coop_detail::cta_sync_after_t0();
    if (threadIdx.x == 0) {
        c->last = 0;
        c->offers += 1u;
        bool accept = false, took = false;
        if (c->lid != 0u && ld_relaxed32(&d->err) == COOP_DEV_ERR_NONE) {
            if (d->policy == COOP_POLICY_RANDOM) {
                const unsigned long long h = mix64(d->seed ^ ((unsigned long long)c->phys << 40) ^ (c->calls++ * 2u));
                accept = (uint32_t)h < d->kill_thresh;
            } else if (d->policy == COOP_POLICY_SCHEDULER) {
                accept = ld_relaxed32(&d->demand_posted) > ld_relaxed32(&d->demand_taken);
            }
        } else if (ld_relaxed32(&d->err) != COOP_DEV_ERR_NONE) {
            c->state = COOP_ST_ABORT;
        }
        if (accept) {
            unsigned long long w = ld_relaxed64(&d->W);
            if (c->lid + 1u == w_M(w) && w_M(w) > 1u) {   /* only the top id can go */
                if (d->policy == COOP_POLICY_SCHEDULER) {
                    uint32_t t = ld_relaxed32(&d->demand_taken);
                    for (;;) {
                        if (ld_relaxed32(&d->demand_posted) <= t) break;
                        const uint32_t old = atomicCAS(&d->demand_taken, t, t + 1u);
                        if (old == t) { took = true; break; }
                        t = old;
                    }
                    accept = took;
                }
                if (accept) {
                    __threadfence();                       /* release this CTA's work */
                    uint32_t M = 0, a = 0;
                    const bool ok = kill_top(&d->W, w, c->lid, c->gen, &a, &M);   /* fails if M/gen moved */
                    if (ok) {
                        c->state = COOP_ST_KILLED;
                        atomicAdd(&d->kills, 1u);
                        atomicMin(&d->min_m, M - 1u);
                        if (a == M - 1u) {                 /* all others wait: complete the episode */
                            __threadfence();
                            c->last = 1;
                            c->bar_M = M - 1u;
                        }
                    } else if (took) {
                        atomicSub(&d->demand_taken, 1u);
                    }
                }
            }
        }
    }
    cta_sync_after_t0();
    if (c->state == COOP_ST_KILLED && c->last) {
        if (threadIdx.x < 32) (void)serial_section(c, c->gen, c->bar_M, /*behalf=*/true);
        coop_detail::cta_sync_after_t0();
    }
    return c->state != COOP_ST_ACTIVE;
}

/* request_fork.  CTA-collective.  Returns k: ids [M, M+k) start at
 * `entry` with `bytes` of `tx`.  (The serial-section fork buffer bounds k by 32.) */
__device__ __noinline__ uint32_t coop_request_fork(coop_ctx *c, const void *tx, uint32_t bytes, uint32_t entry) {
    using namespace coop_detail;
    __shared__ uint32_t phys_buf_f[32];
    coop_dev *d = c->d;
    if (bytes > COOP_TX_MAX) bytes = COOP_TX_MAX;
    coop_detail::cta_sync_after_t0();
    if (threadIdx.x == 0) {
        uint32_t k = 0;
        const uint32_t M = w_M(ld_relaxed64(&d->W));
        if (M < d->N && ld_relaxed32(&d->err) == COOP_DEV_ERR_NONE) {
            if (d->policy == COOP_POLICY_RANDOM) {
                const unsigned long long h = mix64(d->seed ^ ((unsigned long long)c->phys << 40) ^ (c->calls++ * 2u + 1u));
                if ((uint32_t)h < d->fork_thresh) k = 1u + (uint32_t)((h >> 32) % d->max_fork);
            } else if (d->policy == COOP_POLICY_SCHEDULER) {
                uint32_t t = ld_relaxed32(&d->grant_taken);
                for (;;) {
                    const uint32_t posted = ld_relaxed32(&d->grant_posted);
                    if (posted <= t) break;
                    const uint32_t want = min(min(posted - t, d->N - M), 32u);
                    const uint32_t old = atomicCAS(&d->grant_taken, t, t + want);
                    if (old == t) { k = want; break; }
                    t = old;
                }
            }
        }
        c->bcast = min(k, 32u);
        atomicAdd(&d->fork_calls, 1u);
    }
    cta_sync_after_t0();
    const uint32_t want = c->bcast;
    if (want && threadIdx.x < 32) {
        const uint32_t got = claim_pool(c, want, false, phys_buf_f, 0u, 0u, 0u, nullptr, 0u);
        const uint32_t lane = threadIdx.x & 31u;
        uint32_t base = 0;
        if (lane == 0 && got) {
            /* publish the new active count: W {g, M, a} -> {g, M + got, a} */
            base = add_forks(&d->W, got);
            atomicAdd(&d->forks, got);
            atomicMax(&d->max_m, base + got);
            c->M = base + got;
        }
        if (lane == 0 && d->policy == COOP_POLICY_SCHEDULER && got < want) atomicSub(&d->grant_taken, want - got);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (lane < got) assign(d, phys_buf_f[lane], base + lane, c->gen, entry, (const uint8_t *)tx, bytes);
        if (lane == 0) c->bcast = got;
    }
    cta_sync_after_t0();
    return c->bcast;
}

/* The megakernel wrapper.  body(coop_ctx*) is CTA-collective. */
template <class Body>
__device__ void coop_run(coop_dev *d, Body &&body) {
    using namespace coop_detail;
    __shared__ coop_ctx ctx;
    coop_ctx *c = &ctx;
    const uint32_t phys = blockIdx.x;
    {
        /* every thread stores the same values: no divergent branch before the first barrier */
        const unsigned long long t0 = globaltimer();
        const uint32_t M0 = d->M0;
        const unsigned long long to = d->timeout_ns;
        if (threadIdx.x == 0) {
            c->d = d; c->phys = phys; c->lid = phys; c->M = M0; c->gen = 0; c->entry = 0; c->consumed = 0;
            c->calls = 0; c->offers = 0; c->state = COOP_ST_ACTIVE; c->deadline = t0 + to;
        }
        if (phys == 0 && threadIdx.x == 0) d->t_start = t0;
    }
    coop_detail::cta_sync_after_t0();
    bool run = phys < d->M0;
    for (;;) {
        if (run) {
            body(c);
            coop_detail::cta_sync_after_t0();
            /* read before the next CTA barrier: thread 0 rewrites c->state as soon as it is forked again */
            const uint32_t st = c->state;
            if (threadIdx.x == 0) {
                if (c->state == COOP_ST_ACTIVE) {          /* finished: release the pool */
                    if (atomicExch(&d->finished, 1u) == 0u) d->t_end = globaltimer();
                    __threadfence();
                    st_release32(&d->done, 1u);
                } else if (c->state == COOP_ST_KILLED) {   /* back to the worker pool */
                    __threadfence();
                    atomicOr(&d->pool[phys >> 5], 1u << (phys & 31u));
                }
            }
            cta_sync_after_t0();
            if (st != COOP_ST_KILLED) { break; }   /* finished or aborted: leave the kernel */
        }
        /* parked: wait for a fork assignment; exit once finished and not claimed.
         * Warp 0 spins as a whole (lane 0 polls, the decision is broadcast with a
         * shuffle): a lone spinning lane whose siblings wait at the CTA barrier
         * let the other warps through early (measured: tools/fork_repro.cu). */
        if (threadIdx.x < 32) {
            const uint32_t lane = threadIdx.x;
            uint32_t spins = 0, act = 0;   /* 1 = run, 2 = exit */
            coop_dev_mailbox *mb = d->mb + phys;
            for (;;) {
                uint32_t r = 0;
                if (lane == 0) {
                    const uint32_t f = ld_acquire32(&mb->flag);
                    if (f != c->consumed) {
                        c->consumed = f;
                        c->lid = mb->lid;
                        c->gen = mb->gen;
                        c->entry = mb->entry;
                        copy_tx(c->tx, mb->tx, COOP_TX_MAX);
                        r = 1;
                    } else if (ld_acquire32(&d->done)) {
                        const uint32_t bit = 1u << (phys & 31u);
                        if (ld_relaxed32(&d->err) != COOP_DEV_ERR_NONE) r = 2;
                        else if (atomicAnd(&d->pool[phys >> 5], ~bit) & bit) r = 2;   /* not claimed: leave */
                        /* else claimed by a forker: the assignment is on its way */
                    }
                    if (!r && abort_check(c, spins)) r = 2;
                }
                r = __shfl_sync(0xffffffffu, r, 0);
                if (r) { act = r; break; }
                __nanosleep(64);
            }
            if (act == 1) {   /* join generation gen once it is released */
                for (;;) {
                    uint32_t r = 0;
                    if (lane == 0) {
                        if (w_gen(ld_acquire64(&d->R)) == c->gen) r = 1;
                        else if (abort_check(c, spins)) r = 2;
                    }
                    r = __shfl_sync(0xffffffffu, r, 0);
                    if (r == 2) act = 2;
                    if (r) break;
                }
                if (lane == 0 && act == 1) {
                    c->M = w_M(ld_relaxed64(&d->W));
                    c->state = COOP_ST_ACTIVE;
                }
            }
            if (lane == 0) c->bcast = act;
        }
        cta_sync_after_t0();
        if (c->bcast != 1u) break;
        run = true;
    }
    if (threadIdx.x == 0 && c->offers) atomicAdd(&d->offers, c->offers);
}

/* ---- host helpers (compiled in the user's translation unit) ---- */
#include <cuda_runtime.h>

/* N = co-resident capacity of `kernel`: SMs x CTAs per SM. */
template <class K>
static inline cudaError_t coop_dev_max_wgs(K kernel, int threads, size_t smem, uint32_t *n) {
    int dev = 0, sms = 0, per = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem);
    *n = (uint32_t)(sms * per);
    return e;
}

/* Launch `kernel(coop_dev*, args...)` with n_wgs CTAs under the cooperative
 * launch attribute: the launch fails rather than run CTAs that are not
 * co-resident (no grid.sync is used; the attribute is only the residency guarantee). */
template <class... KArgs, class... Args>
static inline cudaError_t coop_dev_launch(void (*kernel)(coop_dev *, KArgs...), uint32_t n_wgs, uint32_t threads,
                                          size_t smem, cudaStream_t stream, coop_dev *d, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_wgs);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, d, static_cast<KArgs>(args)...);
}

#endif /* __CUDACC__ */
#endif /* COOP_DEVICE_CUH */
