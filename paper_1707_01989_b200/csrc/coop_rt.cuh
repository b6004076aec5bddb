// coop_rt.cuh -- device runtime of the cooperative-kernel model on sm_100a.
//
// One persistent launch = the paper's megakernel: P worker
// CTAs (the N workgroups) + optionally one scheduler CTA.  A
// worker is either ACTIVE in the cooperative body with a logical id in
// [0, M) or PARKED in the worker loop, where it runs blocks of the competing
// non-cooperative task and waits to be forked.
//
// Resizing global barrier = one episode on a packed word
//   W = {gen:32 | M:16 | arrived:16}      (modelled in oracle/barrier_model.py)
//   arrive : thread 0: fence; old = atomicAdd(W, 1); last iff old.arrived+1 == old.M
//   serial : warp 0 of the last arriver, while all M CTAs wait: query the
//            scheduler (W_q = min(demand, M-1)), pick M', fork new
//            ids [M, M') onto idle parked CTAs (mailbox + transmit of WG 0,
//            P:892-903), run the app's serial work (Fig. 4 reset(out)),
//            record M' in mhist[gen+1], then release W := {gen+1, M', 0}.
//   waiters: spin on the release word R until R.gen != gen; killed iff
//            R.gen != gen+1 or id >= M' (ids >= M' leave: the query barrier's
//            "ids >= M-W").  R sits on its own line so the polls do
//            not queue behind the arrival atomics on W.
// NAIVE mode: on entry the top WG (id M-1 > 0) offers kill; if the
// scheduler has demand it leaves by CAS W {g,M,a} -> {g,M-1,a}.
#pragma once
#include <stdint.h>
#include "coop_internal.h"
#include "../../include/coop_protocol.cuh"
#include "../../include/coop.h"

// Barrier implementation switches (A/B measured with tools/barrier_variants.sh;
// the defaults are the measured best that keeps the acquire/release pairing):
//   COOP_POLL_ACQUIRE : 1 = poll with ld.acquire; 0 = poll relaxed, one fence after
//   COOP_POST_FENCE   : extra __threadfence() after the poll (L1 invalidation)
//   COOP_ERR_RELOAD   : re-read the error word after the serial section
//   COOP_ARRIVE_ACQREL: 1 = atom.acq_rel arrival; 0 = fence.sc + relaxed atom (+ fence if
//                       last).  Every warp that issues fire-and-forget reductions the serial
//                       section reads fences them itself before the CTA barrier (flush_counts,
//                       drain_group, the partitioned expand), so the cumulative release of
//                       the acq_rel arrival suffices: 148 CTAs 3192 -> 2746 ns per barrier,
//                       0 violations under COOP_FLAG_CHECK (profiles/r02_variants.log)
#ifndef COOP_POLL_ACQUIRE
#define COOP_POLL_ACQUIRE 1
#endif
#ifndef COOP_POST_FENCE
#define COOP_POST_FENCE 0
#endif
#ifndef COOP_ERR_RELOAD
#define COOP_ERR_RELOAD 0
#endif
#ifndef COOP_ARRIVE_ACQREL
#define COOP_ARRIVE_ACQREL 1
#endif
#ifndef COOP_ARRIVE_REL
#define COOP_ARRIVE_REL 0     // 1: release-only arrival, fence.acq_rel by the last arriver only (measured
                              // slower: 3.14 vs 2.76 us per plain barrier at 148 CTAs, profiles/r02g_variants.log)
#endif

// bisection switches (A/B of the cooperative machinery's cost; 1 = shipped code)
#ifndef COOP_BIS_SERIAL
#define COOP_BIS_SERIAL 1
#endif
#ifndef COOP_BIS_BARRIER
#define COOP_BIS_BARRIER 1
#endif
#ifndef COOP_BIS_CLAIM
#define COOP_BIS_CLAIM 1
#endif
#ifndef COOP_BIS_PARK
#define COOP_BIS_PARK 1
#endif
#ifndef COOP_TAIL_DYN
#define COOP_TAIL_DYN 0       // static intervals (measured: 4/16 and 8/16 slower on RMAT-24 direction-optimising)
//: the last TAIL_DYN/16 of the items are claimed dynamically
#endif
#ifndef COOP_RUNBODY_NOINLINE
#define COOP_RUNBODY_NOINLINE 0
#endif
#ifndef COOP_RUNBODY_INLINE
#define COOP_RUNBODY_INLINE 0 // 1: force run_body inline at both call sites (kernel body, park loop)
#endif
#if COOP_RUNBODY_NOINLINE
#define COOP_RUNBODY_ATTR __noinline__
#elif COOP_RUNBODY_INLINE
#define COOP_RUNBODY_ATTR __forceinline__
#else
#define COOP_RUNBODY_ATTR
#endif
#ifndef COOP_WARP_WAIT
#define COOP_WARP_WAIT 1      // waiters poll the release word with all of warp 0 (converged at the CTA barrier)
#endif

#ifndef COOP_POLL_CYCLES
#define COOP_POLL_CYCLES 2000 // DIST_MID: a CTA reads the demand word at most once per this many SM
                              // cycles (~1 us; every warp reading it with every item: 4736 warps on
                              // one L2 line, +12 % kernel time on RMAT-24)
#endif
#ifndef COOP_MID_INLINE
#define COOP_MID_INLINE 0     // 1: the DIST_MID / DIST_REPLAY expand instances inlined into run_body
#endif
#ifndef COOP_MID_NOCHECK
#define COOP_MID_NOCHECK 0    // measurement only: the mid-interval instance without its per-item checks
#endif
#ifndef COOP_MID_UNIFIED
#define COOP_MID_UNIFIED 0    // 1: every policy runs the DIST_MID instance (inline), its checks gated at run time
#endif

#ifndef COOP_TRACE
#define COOP_TRACE 0          // 1: clock64 breakdown of the barrier, CTA 0 (coop_debug_trace)
#endif

#ifndef COOP_LTRACE
#define COOP_LTRACE 0         // 1: per-level per-CTA %globaltimer stamps (tools/level_trace.py)
#endif

namespace coop {

#if COOP_LTRACE
// [level][blockIdx][expand start, expand end, after RB1, after RB2, app stamps 4..7,
//                   barrier: 8 arrival done, 9 serial section before publish (last arriver),
//                   10 after publish (last arriver), 11 release seen (waiter)]
constexpr int kLtraceSlots = 12;
__device__ unsigned long long g_ltrace[64][1184][kLtraceSlots];
#define LTRACE(k)                                                                         \
    do {                                                                                  \
        if (threadIdx.x == 0 && cs.level < 64 && blockIdx.x < 1184)                       \
            g_ltrace[cs.level][blockIdx.x][k] = globaltimer();                            \
    } while (0)
#define LTRACE_RB2(l) (g_ltrace[l][blockIdx.x][3] = globaltimer())
#else
#define LTRACE(k) do {} while (0)
#define LTRACE_RB2(l) ((void)0)
#endif

constexpr unsigned FULL = 0xffffffffu;

// CTA barrier that is safe after thread-0-only regions.  Measured on sm_100a
// (tools/fork_repro.cu, the device-API twin of this runtime): when ptxas lays a
// straight-line `if (threadIdx.x == 0) {...}` out as a plain forward branch
// with no reconvergence point, lanes 1..31 reach the warp-aligned bar.sync
// before lane 0, the warp is counted twice and the NEXT barrier releases the
// other warps early.  ptxas deletes a plain __syncwarp() there (it believes the
// warp converged), so the reconvergence takes a mask it cannot fold, and the
// barrier is the non-aligned barrier.sync.
// (a __constant__ word: the constant cache, not an L2 round trip as a volatile global load would be)
__constant__ uint32_t c_full_mask = 0xffffffffu;
// COOP_ALIGNED_SYNC=1 restores plain __syncthreads() (A/B only: measured 2.95 vs 3.73 us per
// plain barrier at 148 CTAs, but test_handle_api_host_channel timed out in 1 of 8 runs with it
// and in none of 14 without; __syncwarp(mask) + __syncthreads() crashes ptxas 12.9)
#if defined(COOP_ALIGNED_SYNC)
__device__ __forceinline__ void cta_sync() { __syncthreads(); }
#else
__device__ __forceinline__ void cta_sync() {
    __syncwarp(c_full_mask);
    asm volatile("barrier.sync 0;" ::: "memory");
}
#endif

// ---------------------------------------------------------------- PTX helpers
// ordered accesses, the packed words and the generator: the shared protocol header
// (include/coop_protocol.cuh, also used by the device API)
using coop_proto::globaltimer;
using coop_proto::ld_acquire64;
using coop_proto::ld_acquire32;
using coop_proto::ld_relaxed32;
using coop_proto::ld_relaxed64;
using coop_proto::st_release32;
using coop_proto::st_release64;
using coop_proto::st_relaxed64;
using coop_proto::st_relaxed32;
using coop_proto::atom_add_acq_rel64;
using coop_proto::w_gen;
using coop_proto::w_M;
using coop_proto::w_arr;
using coop_proto::mix64;
__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_sys32(const volatile uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}


__device__ __forceinline__ void prefetch_l2(const void *a) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
}
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        uint32_t n = __shfl_up_sync(FULL, v, s);
        if (lane >= (uint32_t)s) v += n;
    }
    return v;
}
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
// lowest `n` set bits of `w`
__device__ __forceinline__ uint32_t lowest_bits(uint32_t w, uint32_t n) {
    uint32_t m = 0;
    for (uint32_t i = 0; i < n && w; ++i) {
        uint32_t b = w & (0u - w);
        m |= b;
        w ^= b;
    }
    return m;
}

// ---------------------------------------------------------------- CTA state
struct CtaState {
    uint32_t lid, M, gen, level, in_sel;
    uint32_t action, last, entry, block, consumed;
    uint64_t deadline;
    unsigned long long edges, frontier, reached;   // per-CTA stats, flushed at body exit
    uint32_t bar_M, bar_naive;                     // barrier: M of the episode, killed on entry (NAIVE)
    uint32_t wait_rel;                             // barrier: this CTA waits for the release word
    uint32_t stop, nostop;                         // DIST_MID: asked to surrender / stop offering this interval
    uint32_t resume;                               // DIST_MID: expand re-entered after an offer that did not kill
    uint64_t hb_n, hb_tw;                          // DIST_MID: static items / warp stride of the interval (hand-back)
    uint32_t replay, rep_M;                        // a replay interval follows this barrier; survivors' M in it
    uint32_t rk[32];                               // DIST_MID: next static item index per warp (~0u: none left)
    uint32_t nextc[32];                            // DIST_MID: per-warp clock of the next stop/poll check
    unsigned long long poll_t;                     // DIST_MID: %globaltimer of the CTA's last demand poll
#if COOP_TRACE
    unsigned long long tr[12];
    long long tr_last;
#endif
    const KParams *sp;                             // the CTA's shared-memory copy of the kernel parameters:
                                                   // what the out-of-line functions read (a generic load
                                                   // through the __grid_constant__ parameter's address
                                                   // is slow; inlined code keeps the constant bank)
    unsigned long long acc[2];                     // app per-CTA level counters (BFS: nf, mf), added to the
    uint32_t acc_sel;                              //   control block by pre_arrive; their parity
    uint32_t app_u32[8];                           // app broadcast scratch
};

__device__ __forceinline__ bool set_abort(const KParams &p, uint32_t code) {
    atomicCAS(&p.ctl->err, DERR_NONE, code);
    st_release32(&p.ctl->done, 1);
    return true;
}
// watchdog for spin loops (thread-level); true => abort
__device__ __forceinline__ bool spin_check(const KParams &p, const CtaState &cs, uint32_t &spins) {
    if ((++spins & 127u) != 0) return false;
    if (ld_relaxed32(&p.ctl->err) != DERR_NONE) return true;
    if (globaltimer() > cs.deadline) return set_abort(p, DERR_TIMEOUT);
    return false;
}

__device__ __forceinline__ uint32_t mhist_get(const KParams &p, uint32_t gen);

// ---------------------------------------------------------------- forks
// Warp-collective: claim up to k idle parked CTAs from the pool and assign
// them logical ids M, M+1, ... with the transmit state of WG 0.
// With `wait`, keeps trying until k are found (killed CTAs park promptly).
__device__ __noinline__ uint32_t fork_from_pool(const KParams &p, const CtaState &cs, uint32_t gnext, uint32_t M,
                                   uint32_t k, uint32_t entry, const Transmit &tx0, bool wait) {
    uint32_t spins = 0;
    return coop_proto::claim_idle(p.ctl->pool, (p.P + 31) / 32, k, wait,
        [&](uint32_t phys, uint32_t i) {                    // mailbox: id M+i, generation, WG 0's state
            Mailbox *mb = p.mb + phys;
            Transmit t = tx0;
            t.gen = gnext;
            t.lid = M + i;
            t.entry = entry;
            mb->tx = t;
            __threadfence();
            st_release32(&mb->flag, gnext);
        },
        [&]() { return spin_check(p, cs, spins); });
}

// ---------------------------------------------------------------- barrier
template <class App>
__device__ void serial_section(const KParams &p, CtaState &cs, App &app, uint32_t g, uint32_t M,
                               bool resizing, uint32_t entry, uint32_t *out_mp, uint32_t *out_flags) {
    const uint32_t lane = threadIdx.x & 31;
    Ctl *c = p.ctl;
    // every app passes exactly one non-resizing barrier (the init global_barrier at
    // generation 0), so the resizing episode of generation g is g - 1 (no load)
    const uint32_t ep = g - 1;
    uint32_t Mp = M, take = 0;
    bool sched_fork = false, wait_fork = false;
    // hand-back (SCHEDULER + query, barrier #1): items handed back by CTAs that left inside
    // the interval make this episode the start of a replay interval -- the level is not
    // over: no policy decision, no forks, no app serial work, M' = M
    uint32_t replay = 0;
    // the scheduler channel and the hand-back word: one batch of independent plain loads
    // (after the arrival's acquire; the asm-volatile relaxed loads would serialise one
    // round trip each on this critical path)
    uint32_t d0 = 0, gr0 = 0;
    if constexpr (App::kCoop) {
        if (lane == 0 && resizing && p.policy == COOP_POLICY_SCHEDULER) {
            const volatile Ctl *vc = c;
            d0 = c->demand;
            gr0 = c->grant;
            if (entry == ENTRY_AFTER_RB1 && p.barrier_mode == COOP_BARRIER_QUERY) {
                const unsigned long long dw = vc->don;
                if (dw) {
                    c->don = 0ull;
                    if (dw & kMask44) { c->rep = dw; replay = 1; }
                }
            }
        }
        replay = __shfl_sync(FULL, replay, 0);
    }
    if ((App::kCoop && COOP_BIS_SERIAL) && lane == 0 && !replay) {
        if (resizing && p.barrier_mode != COOP_BARRIER_PLAIN) {
            if (p.policy == COOP_POLICY_SCRIPTED) {
                uint32_t s = ep < p.script_len ? p.script[ep] : 0u;
                if (s) Mp = s;
                wait_fork = true;
            } else if (p.policy == COOP_POLICY_RANDOM) {
                uint64_t h = mix64(p.seed * 0x2545F4914F6CDD1Dull + ep);
                if ((uint32_t)h < p.resize_thresh) Mp = 1 + (uint32_t)((h >> 32) % p.P);
                wait_fork = true;
            } else if (p.policy == COOP_POLICY_SCHEDULER) {
                if (p.barrier_mode == COOP_BARRIER_QUERY) {
                    // query(): W = demand, satisfied up to M-1 in this episode (reading R5)
                    uint32_t d = d0;
                    while (d > 0 && M > 1) {
                        uint32_t t = min(d, M - 1);
                        uint32_t old = atomicCAS(&c->demand, d, d - t);
                        if (old == d) { take = t; break; }
                        d = old;
                    }
                }
                if (take > 0) {
                    Mp = M - take;
                } else {
                    const uint32_t gr = gr0;
                    if (gr > 0 && M < p.P) { Mp = M + min(gr, p.P - M); sched_fork = true; }
                }
            }
            Mp = max(1u, min(Mp, p.P));
        }
    }
    Mp = __shfl_sync(FULL, Mp, 0);
    wait_fork = __shfl_sync(FULL, (uint32_t)wait_fork, 0) != 0;
    uint32_t got = 0;
    if ((App::kCoop && COOP_BIS_SERIAL) && Mp > M) {
        // the transmit-annotated state is uniform over the workgroups at a barrier
        // (PAPER.md:1731-1742), so the serial section's own copy IS WG 0's
        // (checked against WG 0's published copy under COOP_FLAG_CHECK)
        Transmit tx0;
        tx0.level = cs.level;
        tx0.in_sel = cs.in_sel;
        got = fork_from_pool(*cs.sp, cs, g + 1, M, Mp - M, entry, tx0, wait_fork);
        Mp = M + got;
    }
    if (lane == 0) {
        if (!replay) app.serial(p, cs, entry, resizing);
        else atomicAdd(&c->replays, 1u);
        if (p.flags & COOP_FLAG_CHECK) {
            // every active WG arrived exactly once and ids were exactly [0, M)
            uint32_t a = atomicExch(&c->chk_arr[g & 1], 0u);
            bool bad = a != M;
            const uint32_t nw = (p.P + 31) / 32;
            for (uint32_t w = 0; w < nw; ++w) {
                uint32_t bits = atomicExch(&c->idmap[g & 1][w], 0u);
                uint32_t lo = w * 32;
                uint32_t expect = M >= lo + 32 ? 0xffffffffu : (M > lo ? ((1u << (M - lo)) - 1u) : 0u);
                bad |= bits != expect;
            }
            if (resizing && (c->tx0.level != cs.level || c->tx0.in_sel != cs.in_sel)) bad = true;
            if (bad) { atomicAdd(&c->violations, 1u); atomicCAS(&c->err, DERR_NONE, DERR_INVARIANT); }
        }
        // M' of generation g+1 for NAIVE mode and forked CTAs (NAIVE kills may lower
        // W.M during g+1); the release store publishes it with everything above
        if ((App::kCoop && COOP_BIS_SERIAL)) st_relaxed32(&c->mhist[(g + 1) & 7], Mp);
        // the grant consumed by these forks is channel state the next serial section reads
        if ((App::kCoop && COOP_BIS_SERIAL) && sched_fork && got) atomicSub(&c->grant, got);
        // reset the arrival word for generation g+1, then release on the separate
        // release line R (waiters poll R, arrivals hit W: no polling traffic on the
        // line the arrival atomics serialise on)
        LTRACE(9);
        coop_proto::publish(&c->W, &c->R, g + 1, Mp, replay);
        LTRACE(10);
        // statistics after the release: nobody waits for them (the host reads them at the end)
        if constexpr ((App::kCoop && COOP_BIS_SERIAL)) {
            if (take > 0) {   // gather bookkeeping of the task instance in flight
                const uint64_t now = globaltimer();
                uint32_t cur = c->cur_task;
                if (cur && cur - 1 < p.events_cap) {
                    TaskEventDev *e = p.events + (cur - 1);
                    const uint32_t before = atomicAdd(&e->surrendered, take);
                    if (before == 0) e->t_first_surrender = now;
                    if (before + take >= e->demanded) e->t_last_surrender = now;
                }
            }
            if (Mp < M) atomicAdd(&c->kills, M - Mp);
            if (got) atomicAdd(&c->forks, got);
            if (Mp != M) {
                atomicMin(&c->min_m, Mp);
                atomicMax(&c->max_m, Mp);
            }
        }
        if (resizing) {
            if (ep < p.m_trace_cap) p.m_trace[ep] = Mp;
            c->episode = ep + 1;                       // plain store: statistics only
        }
    }
    *out_mp = Mp;
    *out_flags = replay;
}

__device__ __forceinline__ uint32_t mhist_get(const KParams &p, uint32_t gen) {
    return ld_relaxed32(&p.ctl->mhist[gen & 7]);
}

// Resizing (or plain, resizing=false) global barrier for the whole CTA.
// Returns ACT_CONT (survived; cs.M / cs.gen updated), ACT_KILLED or ACT_ABORT.
template <class App>
__device__ uint32_t barrier(const KParams &p, CtaState &cs, App &app, bool resizing, uint32_t entry,
                            bool swap = false) {
#if COOP_TRACE
    long long tr0 = clock64();
#endif
    cta_sync();
    // Fig. 4's swap(&in_nodes, &out_nodes) before barrier #1: after the entry CTA barrier every
    // warp is done reading the interval's in_sel (no CTA barrier of its own)
    if (swap && threadIdx.x == 0) {
        LTRACE(1);
        cs.in_sel ^= 1u;
    }
    Ctl *c = p.ctl;
#if COOP_TRACE
    long long tr1 = clock64(), tr2 = 0, tr3 = 0;
#endif
    if (threadIdx.x == 0) {
        const uint32_t g = cs.gen;
        app.pre_arrive(p, cs);                           // the CTA's counters, released by the arrival
        if (cs.lid == 0 && (p.flags & COOP_FLAG_CHECK)) {  // WG 0's transmit state, for the check
            c->tx0.level = cs.level;
            c->tx0.in_sel = cs.in_sel;
        }
        if (p.flags & COOP_FLAG_CHECK) {
            atomicAdd(&c->chk_arr[g & 1], 1u);
            atomicOr(&c->idmap[g & 1][cs.lid >> 5], 1u << (cs.lid & 31));
        }
        uint32_t action = ACT_CONT, last = 0, killed_naive = 0;
        unsigned long long old;
        if ((App::kCoop && COOP_BIS_BARRIER) && resizing && p.barrier_mode == COOP_BARRIER_NAIVE && p.policy == COOP_POLICY_SCHEDULER &&
            cs.lid != 0) {
            // naive barrier: the slave offers kill on entry; only id M-1 can go
            __threadfence();
            old = ld_relaxed64(&c->W);
            for (;;) {
                uint32_t Mw = w_M(old);
                if (cs.lid != Mw - 1 || Mw <= 1) break;
                uint32_t d = ld_relaxed32(&c->demand);
                if (d == 0) break;
                if (atomicCAS(&c->demand, d, d - 1) != d) continue;
                // W: {g, M, a} -> {g, M-1, a} (retried on concurrent arrivals)
                uint32_t a_k = 0, M_k = 0;
                if (!coop_proto::kill_top(&c->W, old, cs.lid, g, &a_k, &M_k)) {
                    atomicAdd(&c->demand, 1u);                  // W moved: give the unit back, arrive
                    break;
                }
                old = pack_w(g, M_k, a_k);
                Mw = M_k;
                killed_naive = 1;
                atomicAdd(&c->kills, 1u);
                uint32_t cur = c->cur_task;
                uint64_t now = globaltimer();
                if (cur && cur - 1 < p.events_cap) {
                    TaskEventDev *e = p.events + (cur - 1);
                    const uint32_t before = atomicAdd(&e->surrendered, 1u);
                    if (before == 0) e->t_first_surrender = now;
                    if (before + 1 >= e->demanded) e->t_last_surrender = now;
                }
                if (p.flags & COOP_FLAG_CHECK) {  // withdraw from the arrival check
                    atomicSub(&c->chk_arr[g & 1], 1u);
                    atomicAnd(&c->idmap[g & 1][cs.lid >> 5], ~(1u << (cs.lid & 31)));
                }
                if (w_arr(old) == Mw - 1) last = 1;   // everybody else already waits: complete on their behalf
                break;
            }
            if (!killed_naive) {
                old = coop_proto::arrive(&c->W);
                last = coop_proto::is_last(old) ? 1u : 0u;
            }
        } else {
            // arrive: release the CTA's writes of this interval (bar.sync + cumulative
            // release) and, for the last arriver, acquire everybody else's
#if COOP_ARRIVE_REL
            old = coop_proto::arrive_release(&c->W);
            last = coop_proto::is_last(old) ? 1u : 0u;
#elif COOP_ARRIVE_ACQREL
            old = coop_proto::arrive(&c->W);
            last = coop_proto::is_last(old) ? 1u : 0u;
#else
            old = coop_proto::arrive_fenced(&c->W);
            last = coop_proto::is_last(old) ? 1u : 0u;
#endif
        }
#if COOP_TRACE
        tr2 = clock64();
#endif
        if (resizing) LTRACE(8);
        if (w_gen(old) != g) { atomicCAS(&c->err, DERR_NONE, DERR_INVARIANT); set_abort(p, DERR_INVARIANT); }
        cs.last = last;
        cs.bar_M = killed_naive ? w_M(old) - 1 : w_M(old);   // M of the episode for the serial section
        cs.bar_naive = killed_naive;
        if (!last) {
            if (killed_naive) action = ACT_KILLED;
            else cs.wait_rel = 1u;                       // wait for the release below (warp 0)
        }
        cs.action = action;
    }
#if COOP_WARP_WAIT
    // Waiters poll the release word with the whole of warp 0 (lane 0 loads, the
    // decision is shuffled): warp 0 is converged when it reaches the CTA barrier,
    // so the divergence-safe barrier takes its fast path.
    if (threadIdx.x < 32) {
        __syncwarp();
        // every lane reads the shared flags before lane 0 rewrites them (racecheck-clean)
        const uint32_t waiting = cs.wait_rel, g = cs.gen;
        __syncwarp();
        if (waiting) {
            uint32_t spins = 0, stop = 0;
            unsigned long long w = 0;
            for (;;) {
                if (threadIdx.x == 0) {
                    w = ld_acquire64(&c->R);
                    stop = w_gen(w) != g ? 1u : (spin_check(p, cs, spins) ? 2u : 0u);
                }
                if (__shfl_sync(FULL, stop, 0)) break;
            }
            if (threadIdx.x == 0) {
                cs.wait_rel = 0u;
                if (resizing) LTRACE(11);
                if (stop == 2u) {
                    cs.action = ACT_ABORT;
                } else if (w_gen(w) != g + 1) {
                    cs.action = ACT_KILLED;                // W moved on without us => we were killed at g
                } else {
                    // W.M is M' unless NAIVE kills of generation g+1 already lowered it
                    const uint32_t Mn = (App::kCoop && COOP_BIS_BARRIER) && p.barrier_mode == COOP_BARRIER_NAIVE ? mhist_get(p, g + 1) : w_M(w);
                    if ((App::kCoop && COOP_BIS_BARRIER) && cs.lid >= Mn) cs.action = ACT_KILLED;
                    else { cs.M = Mn; cs.gen = g + 1; cs.replay = w_arr(w) & 1u; }
                }
            }
            __syncwarp();
        }
    }
#else
    if (threadIdx.x == 0 && cs.wait_rel) {
        const uint32_t g = cs.gen;
        uint32_t spins = 0;
        unsigned long long w;
        cs.wait_rel = 0u;
        for (;;) {
            w = ld_acquire64(&c->R);
            if (w_gen(w) != g) break;
            if (spin_check(p, cs, spins)) { cs.action = ACT_ABORT; break; }
        }
        if (cs.action != ACT_ABORT) {
            if (w_gen(w) != g + 1) {
                cs.action = ACT_KILLED;                    // W moved on without us => we were killed at g
            } else {
                const uint32_t Mn = p.barrier_mode == COOP_BARRIER_NAIVE ? mhist_get(p, g + 1) : w_M(w);
                if (cs.lid >= Mn) cs.action = ACT_KILLED;
                else { cs.M = Mn; cs.gen = g + 1; cs.replay = w_arr(w) & 1u; }
            }
        }
    }
#endif
#if COOP_TRACE
    if (threadIdx.x == 0) tr3 = clock64();
#endif
    cta_sync();
    if (cs.last) {  // uniform
        if (threadIdx.x < 32) {
            uint32_t Mp, fl;
            serial_section(p, cs, app, cs.gen, cs.bar_M, resizing, entry, &Mp, &fl);
            if (threadIdx.x == 0) {
                if (cs.bar_naive || cs.lid >= Mp) cs.action = ACT_KILLED;
                else { cs.M = Mp; cs.gen = cs.gen + 1; cs.action = ACT_CONT; cs.replay = fl; }
#if COOP_ERR_RELOAD
                if (ld_relaxed32(&c->err) != DERR_NONE) cs.action = ACT_ABORT;
#endif
            }
        }
        cta_sync();
    }
#if COOP_TRACE
    if (threadIdx.x == 0 && blockIdx.x == 0) {               // shared-memory sums: no global traffic
        long long tr4 = clock64();
        unsigned long long *T = cs.tr;
        const int o = cs.last ? 6 : 0;                       // [0..5] waiter, [6..11] last arriver
        T[o + 0] += tr1 - tr0;                               // entry __syncthreads
        T[o + 1] += tr2 - tr1;                               // arrival (fence + atomic)
        T[o + 2] += tr3 - tr2;                               // wait for release
        T[o + 3] += tr4 - tr3;                               // serial section + exit sync
        if (cs.tr_last) T[o + 4] += tr0 - cs.tr_last;        // interval before the barrier
        T[o + 5] += 1;
        cs.tr_last = tr4;
    }
#endif
    return cs.action;
}

// ---------------------------------------------------------------- mid-interval offer_kill
// SCHEDULER + query: a CTA may leave inside an interval (the paper's remedy
// for wide graphs whose barriers are rare) without any dynamic claiming.
// Work stays split statically by (id, M) exactly as in Fig. 4; every warp
// reads the demand word with each item, and a CTA asked to surrender (id >= M - demand,
// query style P:940-947) stops after the items in hand, HANDS BACK the rest of its
// static share (hand_back below) and offers itself.  Only the current top id M-1 can go
// (P:541-548), by CAS on the arrival word {g, M, a} -> {g, M-1, a}; if everybody else
// already waits at the barrier, the leaver completes the episode on their behalf.  The
// serial section of the barrier sees the handed-back items and releases the survivors
// into a replay interval that runs them (the level ends only after it).  Returns
// ACT_KILLED, ACT_CONT (resume the static share) or ACT_ABORT; `flush` is called
// (CTA-collective) before the CTA can be counted out.

// the static slot of warp w of CTA lid among the M*W warps of an interval.  COOP_CTA_INTERLEAVE:
// consecutive items go to consecutive CTAs (warp-major), so a small interval's few items spread
// over the SMs instead of filling the warps of the first CTAs
#ifndef COOP_CTA_INTERLEAVE
#define COOP_CTA_INTERLEAVE 0
#endif
template <int WPB>
__device__ __forceinline__ uint64_t warp_slot(uint32_t lid, uint32_t M, uint32_t w) {
    return COOP_CTA_INTERLEAVE ? (uint64_t)w * M + lid : (uint64_t)lid * WPB + w;
}

// thread 0: hand back what is left of this CTA's static share (cs.rk[w] = the next
// item index of warp w; warp w's items are gw, gw + TW, ... below n); returns the donor
// index, or ~0u when nothing is left
template <int BLOCK>
__device__ __forceinline__ uint32_t hand_back(const KParams &p, CtaState &cs, uint64_t n, uint64_t TW) {
    constexpr uint32_t WPB = BLOCK / 32;
    uint64_t start[WPB], cnt[WPB], tot = 0;
#pragma unroll
    for (uint32_t w = 0; w < WPB; ++w) {
        start[w] = warp_slot<WPB>(cs.lid, (uint32_t)(TW / WPB), w) + (uint64_t)cs.rk[w] * TW;
        cnt[w] = start[w] < n ? (n - start[w] + TW - 1) / TW : 0;
        tot += cnt[w];
    }
    if (tot == 0) return ~0u;
    Ctl *c = p.ctl;
    const unsigned long long old = atomicAdd(&c->don, (1ull << 44) | tot);
    const uint32_t idx = (uint32_t)(old >> 44);
    uint64_t pre = old & kMask44;
    RepEntry *e = p.rep + (uint64_t)idx * WPB;
#pragma unroll
    for (uint32_t w = 0; w < WPB; ++w) {
        e[w].start = start[w];
        e[w].prefix = pre;
        e[w].count = (uint32_t)cnt[w];
        pre += cnt[w];
    }
    st_relaxed64(&c->rep_tw, TW);          // the same value from every donor of the interval
    atomicAdd(&c->handbacks, 1u);
    return idx;
}

// (the caller flushes the CTA's counters first, inline: a flush lambda handed to this
// out-of-line function would make the warps' per-item accumulators address-taken, i.e.
// live on the stack through every item -- measured: +16 M L2 sectors, +13 % kernel time)
template <int BLOCK, class App>
__device__ __noinline__ uint32_t offer_kill_mid(const KParams &p, CtaState &cs, App &app) {
    constexpr uint32_t WPB = BLOCK / 32;
    Ctl *c = p.ctl;
    const uint64_t n = cs.hb_n, TW = cs.hb_tw;
    for (uint32_t spins = 0;;) {
        if (threadIdx.x == 0) {
            uint32_t act = ACT_CONT, serial = 0, Mnew = 0;
            app.pre_arrive(p, cs);
            __threadfence();                               // release this CTA's work of the interval
            unsigned long long w = ld_relaxed64(&c->W);
            for (;;) {
                const uint32_t M = w_M(w);
                const uint32_t d = ld_relaxed32(&c->demand);
                if (d == 0 || cs.lid == 0 || cs.lid + d < M || w_gen(w) != cs.gen) { act = ACT_CONT; break; }
                // the ids above go first; but once some CTA has arrived at the barrier the top
                // id may be among them and can no longer leave mid-interval: then stop offering
                // for the rest of the interval and let the query barrier take the demand
                // (waiting here would deadlock; re-offering at every item would thrash)
                if (cs.lid != M - 1) {
                    if (w_arr(w)) { act = ACT_CONT; cs.nostop = 1; } else act = ACT_IDLE;
                    break;
                }
                if (atomicCAS(&c->demand, d, d - 1) != d) { w = ld_relaxed64(&c->W); continue; }
                const uint32_t idx = hand_back<BLOCK>(p, cs, n, TW);
                __threadfence();                           // the entries before the kill-CAS
                uint32_t a = 0, M_k = 0;
                if (!coop_proto::kill_top(&c->W, w, cs.lid, cs.gen, &a, &M_k)) {   // W moved: not the top now
                    if (idx != ~0u)                        // withdraw: this CTA keeps its items
                        for (uint32_t k = 0; k < WPB; ++k) p.rep[(uint64_t)idx * WPB + k].start |= kRepVoid;
                    __threadfence();
                    atomicAdd(&c->demand, 1u);
                    act = ACT_CONT;
                    break;
                }
                atomicAdd(&c->kills, 1u);
                atomicAdd(&c->mid_kills, 1u);
                const uint32_t cur = c->cur_task;
                const uint64_t now = globaltimer();
                if (cur && cur - 1 < p.events_cap) {
                    TaskEventDev *e = p.events + (cur - 1);
                    const uint32_t before = atomicAdd(&e->surrendered, 1u);
                    if (before == 0) e->t_first_surrender = now;
                    if (before + 1 >= e->demanded) e->t_last_surrender = now;
                }
                act = ACT_KILLED;
                if (a == M - 1) { serial = 1; Mnew = M - 1; }          // all others wait: complete for them
                break;
            }
            if (act == ACT_CONT) cs.stop = 0;
            cs.action = act;
            cs.last = serial;
            cs.bar_M = Mnew;
        }
        cta_sync();
        const uint32_t act = cs.action;
        if (act == ACT_KILLED) {
            if (cs.last) {
                // the episode is that of resizing barrier #1, after Fig. 4's swap
                if (threadIdx.x == 0) cs.in_sel ^= 1u;
                cta_sync();
                if (threadIdx.x < 32) {
                    uint32_t Mp, fl;
                    serial_section(p, cs, app, cs.gen, cs.bar_M, true, ENTRY_AFTER_RB1, &Mp, &fl);
                }
                cta_sync();
            }
            return ACT_KILLED;
        }
        if (act == ACT_CONT) return ACT_CONT;
        if (threadIdx.x == 0) {
            if (spin_check(p, cs, spins)) cs.action = ACT_ABORT;
            else __nanosleep(64);
        }
        cta_sync();
        if (cs.action == ACT_ABORT) return ACT_ABORT;
    }
}

// Work distribution of an interval over `n_items` warp-sized items; fn(item) is
// warp-collective.  DIST:
//  DIST_STATIC (no scheduler can ask for workgroups inside this interval): Fig. 4's
//          distribution, item i to warp i mod (M*W) -- no atomics, no syncs;
//          the last tail16/16 of the items are claimed one at a time from the level's
//          counter by warps that finished their share (top-down levels: evens out the end
//          of the level without any CTA barrier)
//  DIST_MID (SCHEDULER + query): the same split; each item also reads the demand word
//          (lane 0, the load overlaps the item), a CTA asked to surrender stops after the
//          items in hand and offers itself with its remaining static items handed back
//          (offer_kill_mid).  Tail items are claimed, so none is ever stranded.
//  DIST_REPLAY: the survivors run the items handed back in the interval just ended,
//          flattened (RepEntry prefixes) and split statically over the survivors' warps.
enum : int { DIST_STATIC = 0, DIST_MID = 1, DIST_REPLAY = 2 };

template <int BLOCK, int DIST, class App, class Fn, class Flush>
__device__ uint32_t claim_items(const KParams &p, CtaState &cs, App &app, uint32_t *counter, uint64_t n_items,
                                Fn &&fn, Flush &&flush, uint32_t tail16 = COOP_TAIL_DYN) {
    constexpr uint32_t WPB = BLOCK / 32;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t n_static = tail16 ? n_items - n_items * tail16 / 16 : n_items;
    if constexpr (DIST == DIST_REPLAY) {
        // cs.rep_M = survivors; the items were numbered by the donors' interval
        const Ctl *c = p.ctl;
        const unsigned long long rw = __ldcg(&c->rep);
        const uint64_t total = rw & kMask44, npairs = (rw >> 44) * WPB;
        const uint64_t TWi = __ldcg(&c->rep_tw);
        const uint64_t TWs = (uint64_t)cs.rep_M * WPB;
        for (uint64_t f = warp_slot<WPB>(cs.lid, cs.rep_M, warp); f < total; f += TWs) {
            uint64_t lo = 0, hi = npairs - 1;                 // last entry with prefix <= f
            while (lo < hi) {
                const uint64_t mid = (lo + hi + 1) >> 1;
                if (__ldcg(&p.rep[mid].prefix) <= f) lo = mid; else hi = mid - 1;
            }
            const uint64_t st = __ldcg(&p.rep[lo].start), pre = __ldcg(&p.rep[lo].prefix);
            if (st & kRepVoid) continue;                      // withdrawn: its donor ran it
            fn(st + (f - pre) * TWi);
        }
        (void)counter; (void)app; (void)flush; (void)n_static;
        return ACT_CONT;
    } else {
        constexpr bool mid = DIST == DIST_MID && App::kCoop && COOP_BIS_CLAIM;
        const uint64_t TW = (uint64_t)cs.M * WPB;
        const uint64_t gw = warp_slot<WPB>(cs.lid, cs.M, warp);
        if constexpr (!mid) {
            for (uint64_t it = gw; it < n_static; it += TW) fn(it);
            if (tail16 && n_static < n_items) {
                uint32_t t = 0;
                if (lane == 0) t = atomicAdd(counter, 1u);
                for (;;) {
                    const uint64_t it = n_static + __shfl_sync(FULL, t, 0);
                    if (it >= n_items) break;
                    if (lane == 0) t = atomicAdd(counter, 1u);        // next claim in flight
                    fn(it);
                }
            }
            (void)app; (void)flush;
            return ACT_CONT;
        } else {
            volatile uint32_t *stopf = &cs.stop;
            const bool resumed = cs.resume != 0;
            if (threadIdx.x == 0) {
                cs.stop = 0;
                if (!resumed) cs.nostop = 0;                       // kept by a resumed interval
                cs.poll_t = clock64();
            }
            if (lane == 0) cs.nextc[warp] = (uint32_t)clock() + COOP_POLL_CYCLES;
            cta_sync();
            // After an item, each warp checks at most once per COOP_POLL_CYCLES of the SM clock
            // (its next check time in shared memory: the item loop keeps exactly the static
            // loop's registers -- anything more live across the item spilled the bottom-up item
            // body, +9 % kernel time): the CTA's stop flag and, lane 0 if COOP_POLL_CYCLES passed
            // since the CTA's last read, the demand word (raising the stop flag if this id is
            // asked to surrender, query style).  Only a polling warp waits for that load.
            auto check = [&]() -> bool {                             // warp-uniform
                if (COOP_MID_NOCHECK) return false;                     // measurement only: no kills
                if (!(p.policy == COOP_POLICY_SCHEDULER && p.barrier_mode == COOP_BARRIER_QUERY)) return false;
                volatile uint32_t *nx = &cs.nextc[warp];
                uint32_t due = (int32_t)((uint32_t)clock() - *nx) >= 0 ? 1u : 0u;
                if (!__shfl_sync(FULL, due, 0)) return false;
                if (lane == 0) {
                    const unsigned long long now = clock64();
                    *nx = (uint32_t)now + COOP_POLL_CYCLES;
                    volatile unsigned long long *pollt = &cs.poll_t;
                    if (cs.lid != 0 && !cs.nostop && now - *pollt >= COOP_POLL_CYCLES) {
                        *pollt = now;
                        const uint32_t d = ld_relaxed32(&p.ctl->demand);
                        if (d && cs.lid + d >= w_M(ld_relaxed64(&p.ctl->W))) *stopf = 1u;
                    }
                }
                return __shfl_sync(FULL, lane == 0 ? *stopf : 0u, 0) != 0;
            };
            {
                uint64_t it = resumed ? gw + (uint64_t)cs.rk[warp] * TW : gw;
                bool halted = false;
                for (; it < n_static; it += TW) {
                    fn(it);
                    if (check()) { halted = true; it += TW; break; }
                }
                // next static item of this warp (all done: past the end)
                if (lane == 0)
                    cs.rk[warp] = halted ? (uint32_t)((it - gw) / TW) : 0xFFFFFFFFu;
                if (tail16 && n_static < n_items && !halted) {
                    uint32_t t = 0;
                    if (lane == 0) t = atomicAdd(counter, 1u);
                    for (;;) {
                        const uint64_t ti = n_static + __shfl_sync(FULL, t, 0);
                        if (ti >= n_items) break;
                        uint32_t more = 0;
                        if (lane == 0) {
                            more = *stopf ? 0u : 1u;
                            if (more) t = atomicAdd(counter, 1u);     // next claim in flight
                        }
                        fn(ti);                                       // a claimed item is always run
                        check();
                        if (!__shfl_sync(FULL, more, 0)) break;
                    }
                }
                cta_sync();
                if (!cs.stop) return ACT_CONT;
                // asked to surrender: counters out, then run_body offers this CTA (out of line,
                // outside the item loops: a call in here would constrain their registers) and
                // re-enters the expand with cs.resume if it is not taken
                flush();
                if (threadIdx.x == 0) { cs.hb_n = n_static; cs.hb_tw = TW; }
                cta_sync();
                (void)app;
                return ACT_STOP;
            }
        }
    }
}

// ---------------------------------------------------------------- body
// the expand instances of the scheduler-armed path (DIST_MID, DIST_REPLAY) out of line
#if COOP_MID_INLINE
#define COOP_EXPAND_DIST_ATTR __forceinline__
#else
#define COOP_EXPAND_DIST_ATTR __noinline__
#endif
template <class App, int BLOCK, int DIST>
__device__ COOP_EXPAND_DIST_ATTR uint32_t expand_dist(const KParams &p, CtaState &cs, App &app) {
    return app.template expand<BLOCK, DIST>(p, cs);
}

// Fig. 4 with the app's process_node; entry points are the
// program points after each resizing barrier (forked CTAs start there).
template <class App, int BLOCK, bool ARMED = false>
__device__ COOP_RUNBODY_ATTR uint32_t run_body(const KParams &p, CtaState &cs, App &app, uint32_t entry) {
    uint32_t r;
    app.enter(p, cs);
    if (entry == ENTRY_START) {
#if COOP_LTRACE
        if (threadIdx.x == 0 && blockIdx.x < 1184) g_ltrace[63][blockIdx.x][1] = globaltimer();   // init start
#endif
        app.template init<BLOCK>(*cs.sp, cs);
#if COOP_LTRACE
        cta_sync();
        if (threadIdx.x == 0 && blockIdx.x < 1184) g_ltrace[63][blockIdx.x][2] = globaltimer();   // init done
#endif
        r = barrier(p, cs, app, /*resizing=*/false, ENTRY_AFTER_RB2);   // global_barrier
        if (r != ACT_CONT) return r;
        entry = ENTRY_AFTER_RB2;
    }
    bool skip_to_rb1 = entry == ENTRY_AFTER_RB1;
    for (;;) {
        if (!skip_to_rb1) {
            if (app.empty(p, cs)) {                           // while (in_nodes.size > 0)
                if (!app.next_run(p, cs)) return ACT_DONE;
                // BFS looped over sources inside the launch: the next run's init by
                // the active CTAs, then a resizing barrier (forked CTAs join at the loop head)
                if (threadIdx.x == 0) { cs.level = 0; cs.in_sel = 0; }
                cta_sync();
                app.template init<BLOCK>(*cs.sp, cs);
                r = barrier(p, cs, app, /*resizing=*/true, ENTRY_RESTART);
                if (r != ACT_CONT) return r;
                continue;
            }
            LTRACE(0);
            // for (i = tid; ...) process_node -- the chunked instance when a scheduler may ask
            // for workgroups mid-interval (offer_kill at chunk boundaries), else the static one
            const bool midk = App::kCoop && p.policy == COOP_POLICY_SCHEDULER && p.barrier_mode == COOP_BARRIER_QUERY;
            if constexpr (App::kCoop) {
                // one call site of the expand: asked to surrender inside the interval (ACT_STOP,
                // counters flushed), the CTA offers itself out of line; not taken, it re-enters
                // the expand to finish its share (cs.resume)
                for (;;) {
                    if constexpr (ARMED) {
                        // the scheduler-armed kernel (SCHEDULER + query): the mid-interval instance
                        // inlined in a kernel of its own -- its own register allocation, parameters
                        // from the constant bank -- while the NEVER kernel keeps only the static one
                        r = app.template expand<BLOCK, DIST_MID>(p, cs);
                    } else {
#if COOP_MID_UNIFIED
                        r = app.template expand<BLOCK, DIST_MID>(p, cs);      // checks gated at run time
#else
                        if (midk)
                            r = expand_dist<App, BLOCK, DIST_MID>(*cs.sp, cs, app); // out of line: keeps the
                        else                                                        // static instance as tight
                            r = app.template expand<BLOCK, DIST_STATIC>(p, cs);     // as the non-coop kernel's
#endif
                    }
                    if (r != ACT_STOP) break;
                    r = offer_kill_mid<BLOCK>(*cs.sp, cs, app);
                    if (r != ACT_CONT) break;                  // killed (its rest handed back) / abort
                    if (threadIdx.x == 0) cs.resume = 1;
                    cta_sync();
                }
                if (threadIdx.x == 0) cs.resume = 0;
            } else {
                r = app.template expand<BLOCK, DIST_STATIC>(p, cs);
            }
            if (r != ACT_CONT) return r;                       // killed inside the interval (offer_kill)
            r = barrier(p, cs, app, true, ENTRY_AFTER_RB1, /*swap=*/true);   // swap; resizing_global_barrier() #1
            if constexpr (App::kCoop) {
                // hand-back: workgroups left inside the interval with static items undone; the
                // survivors run them (items numbered by the donors' interval: cs.M = its M for
                // the app's item parameters, cs.rep_M = the survivors) before the level ends
                while (midk && r == ACT_CONT && cs.replay) {
                    if (threadIdx.x == 0) {
                        cs.in_sel ^= 1u;
                        cs.rep_M = cs.M;
                        cs.M = (uint32_t)(__ldcg(&p.ctl->rep_tw) / (BLOCK / 32));
                    }
                    cta_sync();
                    r = expand_dist<App, BLOCK, DIST_REPLAY>(*cs.sp, cs, app);
                    if (r != ACT_CONT) return r;
                    cta_sync();
                    if (threadIdx.x == 0) { cs.M = cs.rep_M; cs.in_sel ^= 1u; }
                    r = barrier(p, cs, app, true, ENTRY_AFTER_RB1);
                }
            }
            if (r != ACT_CONT) return r;
            LTRACE(2);
        }
        skip_to_rb1 = false;
        if constexpr (App::kBetween) {
            app.template between<BLOCK>(p, cs);               // CTA work between Fig. 4's two barriers
            cta_sync();                                       // every warp is done with it
        }
        if (threadIdx.x == 0) cs.level += 1;                  // reset(out_nodes) done in serial; level++
        if (p.bpl == 2) {
            r = barrier(p, cs, app, true, ENTRY_AFTER_RB2);   // resizing_global_barrier() #2
            if (r != ACT_CONT) return r;
            if (threadIdx.x == 0 && cs.level >= 1 && cs.level <= 64 && blockIdx.x < 1184 && COOP_LTRACE)
                LTRACE_RB2(cs.level - 1);
        } else {
            cta_sync();
        }
    }
}

__device__ __forceinline__ void flush_stats(const KParams &p, CtaState &cs) {
    if (threadIdx.x == 0) {
        if (cs.edges) atomicAdd(&p.ctl->edges_scanned, cs.edges);
        if (cs.frontier) atomicAdd(&p.ctl->frontier_total, cs.frontier);
        if (cs.reached) atomicAdd(&p.ctl->reached, cs.reached);
        cs.edges = cs.frontier = cs.reached = 0;
    }
}

// ---------------------------------------------------------------- tasks
// One block of the synthetic non-cooperative task (K11: occupies a workgroup
// for a fixed time).  Thread 0 spins on %globaltimer.
__device__ __noinline__ void run_task_block(const KParams &p, CtaState &cs) {
    if (threadIdx.x == 0) {
        Ctl *c = p.ctl;
        uint64_t t0 = globaltimer();
        uint32_t cur = ld_relaxed32(&c->cur_task);
        if (cur && cur - 1 < p.events_cap) atomicCAS(&p.events[cur - 1].t_first_start, 0ull, (unsigned long long)t0);
        unsigned long long ns = ld_relaxed64(&c->task_block_ns);
        uint32_t spins = 0;
        while (globaltimer() - t0 < ns) {
            if (spin_check(p, cs, spins)) break;
            __nanosleep(100);
        }
        __threadfence();
        uint32_t total = ld_relaxed32(&c->task_total);
        if (atomicAdd(&c->task_done, 1u) + 1 == total && cur && cur - 1 < p.events_cap)
            p.events[cur - 1].t_end = globaltimer();
    }
    cta_sync();
}

// ---------------------------------------------------------------- scheduler CTA
__device__ __noinline__ void scheduler_loop(const KParams &p, CtaState &cs) {
    if (threadIdx.x != 0) return;
    Ctl *c = p.ctl;
    const uint64_t t0 = globaltimer();
    uint64_t next = t0 + p.task_first_ns;
    uint32_t posted = 0, inflight = 0, cur = 0, spins = 0;
    uint32_t pend_task = 0, pend_wgs = 0, pend_blocks = 0;
    unsigned long long pend_ns = 0;
    for (;;) {
        if (ld_relaxed32(&c->err) != DERR_NONE) break;
        const uint64_t now = globaltimer();
        const uint32_t done = ld_acquire32(&c->done);
        if (p.host) {  // host packets (SVM-style channel)
            uint32_t s = ld_sys32(&p.host->seq);
            if (s != c->host_seq_seen) {
                uint32_t kind = ld_sys32(&p.host->kind);
                if (kind == 1) { pend_task = 1; pend_wgs = p.host->a; pend_blocks = p.host->b; pend_ns = p.host->c; }
                else if (kind == 2) atomicAdd(&c->demand, (uint32_t)p.host->a);
                else if (kind == 3) atomicAdd(&c->grant, (uint32_t)p.host->a);
                c->host_seq_seen = s;
                __threadfence_system();
                p.host->ack = s;
            }
            p.host->cur_m = w_M(ld_relaxed64(&c->W));
            p.host->demand_mirror = ld_relaxed32(&c->demand);
        }
        if (inflight) {
            if (ld_acquire32(&c->task_done) >= c->task_total) {
                st_relaxed32(&c->task_next, 0xFFFFFFFFu);
                uint32_t rem = atomicExch(&c->demand, 0u);
                TaskEventDev *e = cur < p.events_cap ? p.events + cur : nullptr;
                uint32_t surrendered = e ? e->surrendered : (c->task_wgs - min(rem, c->task_wgs));
                if (surrendered) atomicAdd(&c->grant, surrendered);   // fork them back
                c->tasks_completed += 1;
                c->cur_task = 0;
                inflight = 0;
            }
        } else if (!done) {
            bool periodic = p.task_period_ns && (p.task_max == 0 || posted < p.task_max) && now >= next;
            if (periodic || pend_task) {
                uint32_t q = pend_task ? pend_wgs : p.task_wgs;
                uint32_t b = pend_task ? pend_blocks : p.task_blocks;
                unsigned long long ns = pend_task ? pend_ns : p.task_block_ns;
                pend_task = 0;
                cur = posted++;
                if (cur < p.events_cap) {
                    TaskEventDev *e = p.events + cur;
                    e->t_arrive = now;
                    e->demanded = q;
                }
                c->task_total = b;
                c->task_done = 0;
                c->task_block_ns = ns;
                c->task_wgs = q;
                c->cur_task = cur + 1;
                c->tasks_posted = posted;
                c->n_events = min(posted, p.events_cap);
                __threadfence();
                st_release32(&c->task_next, 0u);       // blocks become claimable
                atomicAdd(&c->demand, q);               // resource message: surrender q WGs
                inflight = 1;
                if (periodic) next += p.task_period_ns;
            }
        }
        if (done && !inflight) break;
        if (spin_check(p, cs, spins)) break;
        __nanosleep(400);
    }
    if (p.host) p.host->done_mirror = 1;
}

// ---------------------------------------------------------------- park loop
// The megakernel worker pool: wait for a fork assignment,
// otherwise run blocks of the competing task; exit at termination.
template <class App, int BLOCK, bool ARMED>
__device__ __noinline__ void park_loop(const KParams &p, CtaState &cs, App &app) {
    Ctl *c = p.ctl;
    const uint32_t phys = blockIdx.x;
    const uint32_t wi = phys >> 5, bit = 1u << (phys & 31);
    for (;;) {
        if (threadIdx.x == 0) {
            uint32_t action = ACT_IDLE, spins = 0;
            Mailbox *mb = p.mb + phys;
            for (;;) {
                uint32_t f = ld_acquire32(&mb->flag);
                if (f != cs.consumed) {
                    cs.consumed = f;
                    Transmit t = mb->tx;
                    cs.lid = t.lid; cs.gen = t.gen; cs.level = t.level; cs.in_sel = t.in_sel; cs.entry = t.entry;
                    action = ACT_RUN_BODY;
                    break;
                }
                if (ld_acquire32(&c->done)) {
                    if (ld_acquire32(&mb->flag) != cs.consumed) continue;   // a final fork happened-before done
                    if (ld_relaxed32(&c->task_next) >= c->task_total) { action = ACT_EXIT; break; }
                }
                if (ld_relaxed32(&c->err) != DERR_NONE) { action = ACT_EXIT; break; }
                if (ld_relaxed32(&c->task_next) < ld_relaxed32(&c->task_total)) {
                    uint32_t old = atomicAnd(&c->pool[wi], ~bit);     // leave the forkable set
                    if (old & bit) {
                        // claim a block by CAS: never advance task_next past task_total (the
                        // scheduler's 0xFFFFFFFF "finished" mark must not wrap to 0 and
                        // re-open the finished instance's blocks)
                        uint32_t b = ld_relaxed32(&c->task_next), got = 0;
                        while (b < ld_relaxed32(&c->task_total)) {
                            const uint32_t prev = atomicCAS(&c->task_next, b, b + 1u);
                            if (prev == b) { got = 1; break; }
                            b = prev;
                        }
                        if (got) { cs.block = b; action = ACT_RUN_TASK; break; }
                        atomicOr(&c->pool[wi], bit);
                    }
                }
                if (spin_check(p, cs, spins)) { action = ACT_EXIT; break; }
                __nanosleep(128);
            }
            cs.action = action;
        }
        cta_sync();
        const uint32_t act = cs.action;
        if (act == ACT_EXIT) return;
        if (act == ACT_RUN_TASK) {
            run_task_block(*cs.sp, cs);
            if (threadIdx.x == 0) { __threadfence(); atomicOr(&c->pool[wi], bit); }
            continue;
        }
        // forked: join generation cs.gen once W reaches it (the release of the fork episode)
        // (the result goes to cs.stop, not cs.action: other warps may still be reading
        // cs.action above -- racecheck)
        if (threadIdx.x == 0) {
            uint32_t spins = 0;
            cs.stop = 0;
            while (w_gen(ld_acquire64(&c->R)) != cs.gen) {
                if (spin_check(p, cs, spins)) { cs.stop = 1; break; }
            }
            cs.M = mhist_get(p, cs.gen);
            __threadfence();
        }
        cta_sync();
        if (cs.stop) return;
        uint32_t r = run_body<App, BLOCK, ARMED>(p, cs, app, cs.entry);
        flush_stats(p, cs);
        if (r == ACT_DONE) {
            if (threadIdx.x == 0 && cs.lid == 0) {
                c->t_end = globaltimer();
                st_release32(&c->done, 1);
            }
        }
        if (r == ACT_ABORT) return;
        // killed (offer_kill accepted) or finished: back to the worker pool, where the
        // CTA can run task blocks and be forked again
        if (threadIdx.x == 0) { __threadfence(); atomicOr(&c->pool[wi], bit); }
        cta_sync();
    }
}

// ---------------------------------------------------------------- kernel
template <class App, int BLOCK, bool ARMED>
__device__ __forceinline__ void kernel_body(const KParams &p, CtaState &cs, App &app) {
    if (threadIdx.x == 0) {
        const uint64_t t0 = globaltimer();
#if COOP_TRACE
        for (int i = 0; i < 12; ++i) cs.tr[i] = 0;
        cs.tr_last = 0;
#endif
        cs.deadline = t0 + p.timeout_ns;
#if COOP_LTRACE
        if (blockIdx.x < 1184) g_ltrace[63][blockIdx.x][0] = t0;                                 // kernel entry
#endif
        cs.edges = cs.frontier = cs.reached = 0;
        cs.consumed = 0;
        cs.wait_rel = 0;
        cs.lid = blockIdx.x; cs.M = p.M0; cs.gen = 0; cs.level = 0; cs.in_sel = 0;
        cs.acc[0] = cs.acc[1] = 0; cs.acc_sel = 0;
        cs.resume = 0; cs.stop = 0; cs.nostop = 0;
        if (blockIdx.x == 0) p.ctl->t_start = t0;
    }
    cta_sync();
    if constexpr ((App::kCoop && COOP_BIS_PARK)) {
        if (p.has_sched && blockIdx.x == p.P) { scheduler_loop(*cs.sp, cs); return; }
    }
    if (blockIdx.x < p.M0) {
        uint32_t r = run_body<App, BLOCK, ARMED>(p, cs, app, ENTRY_START);
        flush_stats(p, cs);
        if (r == ACT_DONE) {
            if (threadIdx.x == 0 && cs.lid == 0) {
                p.ctl->t_end = globaltimer();
                st_release32(&p.ctl->done, 1);
            }
        }
        if (r == ACT_ABORT) return;
        // killed or finished: join the pool -- unless no CTA can ever be forked or run a task
        // (NEVER: no scheduler, no resize), then leave the kernel at once
        if ((App::kCoop && COOP_BIS_PARK) && p.barrier_mode != COOP_BARRIER_PLAIN && p.policy != COOP_POLICY_NEVER &&
            threadIdx.x == 0) {
            __threadfence();
            atomicOr(&p.ctl->pool[blockIdx.x >> 5], 1u << (blockIdx.x & 31));
        }
        cta_sync();
    }
    if constexpr ((App::kCoop && COOP_BIS_PARK)) {
        if (p.barrier_mode != COOP_BARRIER_PLAIN && p.policy != COOP_POLICY_NEVER)
            park_loop<App, BLOCK, ARMED>(*cs.sp, cs, app);
    }
#if COOP_TRACE
    if (threadIdx.x == 0 && blockIdx.x == 0)
        for (int i = 0; i < 12; ++i) p.ctl->trace[i + (i >= 6 ? 2 : 0)] = cs.tr[i];
#endif
}


// __grid_constant__: the parameter block is addressed in place by the out-of-line runtime
// functions (const KParams &), so no thread copies the ~0.9 KB struct to its stack at launch
// (without it every thread of the grid did: ~140 MB of local-memory stores per launch)
template <class App, int BLOCK, int MINB, bool ARMED = false>
__global__ void __launch_bounds__(BLOCK, MINB) coop_kernel(const __grid_constant__ KParams p) {
    __shared__ CtaState cs;
    __shared__ uint32_t s_last;
    __shared__ __align__(16) KParams s_p;
    {
        static_assert(sizeof(KParams) % 8 == 0, "KParams copy by 8-byte words");
        const unsigned long long *src = reinterpret_cast<const unsigned long long *>(&p);
        unsigned long long *dst = reinterpret_cast<unsigned long long *>(&s_p);
        for (uint32_t i = threadIdx.x; i < sizeof(KParams) / 8; i += BLOCK) dst[i] = src[i];
        if (threadIdx.x == 0) cs.sp = &s_p;
    }
    App app;
    kernel_body<App, BLOCK, ARMED>(p, cs, app);
    // epilogue: the last CTA out mirrors the control block into host-mapped memory, so the
    // host reads status and statistics without a device-to-host copy operation per call
    if (p.ctl_mirror) {
        cta_sync();
        if (threadIdx.x == 0) {
            __threadfence();
            s_last = atomicAdd(&p.ctl->exits, 1u) + 1u == gridDim.x ? 1u : 0u;
            if (s_last) __threadfence();
        }
        cta_sync();
        if (s_last) {
            const unsigned long long *src = reinterpret_cast<const unsigned long long *>(p.ctl);
            unsigned long long *dst = reinterpret_cast<unsigned long long *>(p.ctl_mirror);
            for (uint32_t i = threadIdx.x; i < sizeof(Ctl) / 8; i += BLOCK) dst[i] = __ldcg(src + i);
            __threadfence_system();
        }
    }
}

}  // namespace coop
