// apps.cuh -- the process_node of Fig. 4 for BFS and
// worklist SSSP, plus the empty app of the barrier microbenchmark.
//
// Each app provides, for the generic cooperative body in coop_rt.cuh:
//   enter(p, cs)        -- per-CTA state at (re)entry into the body
//   init<BLOCK>(p, cs)  -- interval 0: initialise outputs, seed the frontier
//   empty(p, cs)        -- while (in_nodes.size > 0) test (CTA-uniform)
//   expand<BLOCK>(p,cs) -- for (i = tid; i < in.size; i += stride) process_node
//   serial(p, cs, e, r) -- work between the two barriers of Fig. 4 (reset(out)),
//                          run once by the serial section of the barrier
//
// Frontier work is distributed exactly as in Fig. 4 -- a stride that depends
// only on (id, M) of the current resizing-barrier interval -- at
// warp granularity, plus an edge-balanced split of high-degree vertices that is
// likewise a pure function of (id, M).
#pragma once
#include <type_traits>
#include "coop_rt.cuh"

#ifndef COOP_BU_KW
#define COOP_BU_KW 4          // bottom-up: 32-vertex words per warp item
#endif
#ifndef COOP_BU_EPS
#define COOP_BU_EPS 1         // bottom-up: edges probed per list per step (first hits dominate)
#endif
#ifndef COOP_INIT_DEAD
#define COOP_INIT_DEAD 1      // direction-optimising BFS: close degree-0 vertices in init
#endif
#ifndef COOP_BU_COMPACT
#define COOP_BU_COMPACT 1     // bottom-up: compacted candidates over 32-word items (else lane per vertex)
#endif
#ifndef COOP_BU_K
#define COOP_BU_K 3           // bottom-up (compacted): candidates per lane per round (hub-first layout sweep: profiles/r01c_bu_hubfirst_variants.log)
#endif
#ifndef COOP_BU_SOLO
#define COOP_BU_SOLO 8        // bottom-up (compacted): per-lane steps before the warp takes a list over (same sweep)
#endif
#ifndef COOP_L2_HINTS
#define COOP_L2_HINTS 1       // streaming reads (probe records, row offsets, columns of the bottom-up
                              // scan) carry an L2 evict_first policy so the hot bitmaps stay resident
#endif
#ifndef COOP_TD_TAIL
#define COOP_TD_TAIL 8        // top-down levels: the last TD_TAIL/16 of the items are claimed dynamically
#endif
#ifndef COOP_SSSP_MIN_SZ
#define COOP_SSSP_MIN_SZ 8    // SSSP: smallest worklist group per warp item (32 = fixed groups)
#endif
#ifndef COOP_SSSP_PRECHECK
#define COOP_SSSP_PRECHECK 0  // SSSP: read dist[v] before the atomicMin (fewer atomics, one more dependent round trip: 73.4 vs 68.4 ms on the 2048^2 grid without it)
#endif
#ifndef COOP_SERIAL_INLINE
#define COOP_SERIAL_INLINE 1  // BFS serial-section work inlined (out of line, its parameter reads are generic
                              // loads through the __grid_constant__ pointer, on the barrier's critical path)
#endif
#if COOP_SERIAL_INLINE
#define COOP_SERIAL_ATTR __forceinline__
#else
#define COOP_SERIAL_ATTR __noinline__
#endif
#ifndef COOP_TD_SPEC_RO
#define COOP_TD_SPEC_RO 0     // top-down claims: load the candidate's offsets alongside the claim atomic
#endif
#ifndef COOP_PROBE_NO_LEVELS
#define COOP_PROBE_NO_LEVELS 0   // measurement only (wrong output): drop the level stores of claims
#endif
#ifndef COOP_BU_DENSE_W
#define COOP_BU_DENSE_W 16    // bottom-up (compacted): words per item in the first (dense) level
#endif

namespace coop {

template <typename T>
__device__ __forceinline__ T ldcg(const T *p) { return __ldcg(p); }

// ============================================================== BFS
// Level L reads frontier parity in = L & 1 (the transmitted in_sel) and fills
// parity out.  Modes (chosen by the serial section at the end of each level):
//   TDQ  top-down over the light/heavy frontier queues (process_node of Fig. 4)
//   TDB  top-down over the frontier bitmap (the level after a bottom-up level)
//   BU   bottom-up: every unvisited vertex looks for a parent in the frontier
//        bitmap (direction optimisation; only with COOP_FLAG_DIROPT)
// Every mode produces the same level values (BFS levels are unique).
// kCoop = false compiles the non-cooperative persistent baseline of the same
// traversal (the paper's T2 comparison): plain generation barrier,
// static work split, no scheduler, pool, mailboxes or kill/fork code.
// claim counters of a level parity back to 0 (serial section)
__device__ __forceinline__ void reset_claims(Ctl *c, uint32_t parity) {
#pragma unroll
    for (uint32_t r = 0; r < kClaimShards; ++r) c->claim[parity][r][0] = 0;
}

// read-only loads with an L2 eviction-priority hint (createpolicy + ld.L2::cache_hint)
__device__ __forceinline__ unsigned long long l2_evict_first_policy() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ int32_t ld_hint(const int32_t *a, unsigned long long pol) {
    int32_t v;
    asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ld_hint(const uint32_t *a, unsigned long long pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ int64_t ld_hint(const int64_t *a, unsigned long long pol) {
    int64_t v;
    asm volatile("ld.global.nc.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ unsigned long long ld_hint(const unsigned long long *a, unsigned long long pol) {
    unsigned long long v;
    asm volatile("ld.global.nc.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
    return v;
}
#if COOP_L2_HINTS
#define LDS(ptr) ld_hint((ptr), pol_stream)
#else
#define LDS(ptr) __ldg(ptr)
#endif

// BFS levels during the traversal: one byte per vertex (lv8[v] = level + 1, 0 = not
// reached, 255 = level >= 254, whose int32 is stored directly), 16 MB at RMAT-24 and so
// L2-resident -- the claims' scattered stores no longer read-modify-write sectors of the
// 67 MB int32 output in HBM (7 % of the kernel, build variant COOP_PROBE_NO_LEVELS).  The
// output is written once, coalesced, when the frontier empties (BfsApp::empty).
__device__ __forceinline__ void store_level(const KParams &p, int64_t v, uint32_t L) {
    if (COOP_PROBE_NO_LEVELS) return;
    p.lv8[v] = (uint8_t)(L < 254u ? L + 1u : 255u);
    if (L >= 254u) p.level_out[v] = (int32_t)L;
}

template <typename OffT, bool KCOOP = true>
struct BfsApp {
    static constexpr bool kCoop = KCOOP;
    static constexpr bool kBetween = false;          // no CTA work between Fig. 4's barriers
    using LE = typename std::conditional<sizeof(OffT) == 4, LightEntry, LightEntry64>::type;
    static constexpr int KB = 4;   // 32-edge windows per warp iteration (32*KB <= kHeavyDeg)

    __device__ void enter(const KParams &, CtaState &) {}
    template <int BLOCK>
    __device__ void between(const KParams &, CtaState &) {}

    template <int BLOCK>
    __device__ __noinline__ void init(const KParams &p, CtaState &cs) {
        const uint64_t tid = (uint64_t)cs.lid * BLOCK + threadIdx.x;
        const uint64_t nth = (uint64_t)cs.M * BLOCK;
        const int64_t V = p.V, s = run_source(p);
        // lv8[v] = 0 (not reached), lv8[s] = 1 (level 0): 4 bytes per thread, the mapping the
        // output pass of empty() uses, so a source-loop restart never races a slower CTA's pass
        uint32_t *l4 = reinterpret_cast<uint32_t *>(p.lv8);
        const uint64_t n4 = ((uint64_t)V + 3) / 4;
        for (uint64_t i = tid; i < n4; i += nth) l4[i] = (uint64_t)(s >> 2) == i ? 1u << (8 * (s & 3)) : 0u;
        const uint64_t nw = ((uint64_t)V + 31) / 32;
        const uint32_t sw = (uint32_t)(s >> 5), sb = 1u << (s & 31);
        const bool dead_from_iso = p.dopt && COOP_INIT_DEAD && p.iso != nullptr;
        if (dead_from_iso) {
            // the graph's degree-zero bitmap (a layout step done once per graph): 2 MB copied
            // instead of the 67 MB of row offsets read below
            for (uint64_t i = tid; i < nw; i += nth) {
                const uint32_t m = __ldg(p.iso + i) & ~(i == sw ? sb : 0u);
                p.visited[i] = m | (i == sw ? sb : 0u);
            }
        } else if (p.dopt && COOP_INIT_DEAD && sizeof(OffT) == 4 && ((uintptr_t)p.ro & 15) == 0) {
            // symmetric CSR: a degree-0 vertex is never a neighbour, so it starts
            // closed and the bottom-up levels do not enumerate it (about half of
            // an R-MAT graph's vertices).  Thread per word: the 33 offsets of its
            // 32 vertices as 8 independent 16-B loads + 1.
            const uint32_t *ro = reinterpret_cast<const uint32_t *>(p.ro);
            for (uint64_t i = tid; i < nw; i += nth) {
                uint32_t m = 0;
                if ((i + 1) * 32 <= (uint64_t)V) {
                    const uint4 *r4 = reinterpret_cast<const uint4 *>(ro + i * 32);
                    uint4 q[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) q[k] = __ldg(r4 + k);
                    const uint32_t last = __ldg(ro + i * 32 + 32);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint32_t nx = k < 7 ? q[k + 1].x : last;
                        m |= (q[k].x == q[k].y ? 1u : 0u) << (4 * k);
                        m |= (q[k].y == q[k].z ? 1u : 0u) << (4 * k + 1);
                        m |= (q[k].z == q[k].w ? 1u : 0u) << (4 * k + 2);
                        m |= (q[k].w == nx ? 1u : 0u) << (4 * k + 3);
                    }
                } else {
                    for (uint64_t v = i * 32; v < (uint64_t)V; ++v)
                        if (__ldg(ro + v + 1) == __ldg(ro + v)) m |= 1u << (v - i * 32);
                }
                if (i == sw) m = (m & ~sb) | sb;   // the source is reached, not closed-as-isolated
                p.visited[i] = m | (i == sw ? sb : 0u);
            }
        }
        for (uint64_t i = tid; i < nw; i += nth) {
            if (!dead_from_iso && !(p.dopt && COOP_INIT_DEAD && sizeof(OffT) == 4 && ((uintptr_t)p.ro & 15) == 0))
                p.visited[i] = i == sw ? sb : 0u;
            if (p.dopt) {
                p.fbits[0][i] = i == sw ? sb : 0u;
                p.fbits[1][i] = 0u;
                p.fbits[2][i] = 0u;
            }
        }
        // the frontier counters: here for the first run; for a restart of the source loop in
        // the serial section of the restart barrier (slower CTAs may still be reading the
        // previous run's counters in empty() until they arrive there)
        if (cs.lid == 0 && threadIdx.x == 0 && ld_relaxed32(&p.ctl->run) == 0) init_ctl(p, s);
        if (cs.lid == 0 && threadIdx.x == 0) cs.reached += 1;
    }

    __device__ void init_ctl(const KParams &p, int64_t s) {
        {
            const OffT *ro = static_cast<const OffT *>(p.ro);
            const OffT b = ro[s], e = ro[s + 1];
            const uint32_t deg = (uint32_t)(e - b);
            if (deg >= kHeavyDeg) {
                p.qheavy[0][0] = HeavyEntry{(uint64_t)b, 0ull, deg, 0u};
                p.ctl->heavy[0] = (1ull << 40) | deg;
            } else if (deg > 0) {
                LE le;
                le.beg = b;
                le.deg = deg;
                static_cast<LE *>(p.qlight[0])[0] = le;
                p.ctl->qsize[0] = 1;
            }
            p.ctl->nf[0] = 1;
            p.ctl->mf[0] = deg;
            p.ctl->vis_edges = deg;
            p.ctl->bmode[0] = BFS_TDQ;
            if (p.level_cap) p.level_sizes[0] = 1;
            p.ctl->frontier_total = 1;
            p.ctl->levels = 1;
        }
    }

    // BFS looped over sources (coop_bfs_loop): the source of the current run
    __device__ __forceinline__ static int64_t run_source(const KParams &p) {
        return p.n_src ? __ldg(p.sources + (ld_relaxed32(&p.ctl->run) % p.n_src)) : p.source;
    }
    // after an empty frontier: does another run start? (uniform: read after the release)
    __device__ bool next_run(const KParams &p, CtaState &cs) {
        if (!p.n_src) return false;
        if (threadIdx.x == 0) cs.app_u32[7] = ld_relaxed32(&p.ctl->run) & 0x80000000u ? 0u : 1u;
        cta_sync();
        return cs.app_u32[7] != 0;
    }

    __device__ bool empty(const KParams &p, CtaState &cs) {
        if (threadIdx.x == 0) {
            const uint32_t in = cs.in_sel;
            // plain loads after the barrier's acquire: independent, so they overlap
            // (the asm-volatile relaxed loads serialise one round trip each)
            const Ctl *c = p.ctl;
            const unsigned long long hv = c->heavy[in];
            const uint64_t Eh = hv & kMask40;
            cs.app_u32[0] = c->qsize[in];
            cs.app_u32[1] = (uint32_t)(hv >> 40);
            cs.app_u32[2] = (uint32_t)Eh;
            cs.app_u32[3] = (uint32_t)(Eh >> 32);
            cs.app_u32[4] = c->nf[in] ? 1u : 0u;
            cs.app_u32[5] = c->bmode[in];
            cs.app_u32[6] = c->n_bu_levels;                  // 1 during the first bottom-up level
        }
        cta_sync();
        const bool done = cs.app_u32[4] == 0;
        if (done) {
            // the traversal's output, once: levels = lv8 - 1 (-1 unreached, reading R10); every
            // active CTA its stride, 4 vertices per thread (one coalesced 4-B load, 16-B store)
            const uint64_t V = (uint64_t)p.V, n4 = (V + 3) / 4, nth = (uint64_t)cs.M * blockDim.x;
            const uint32_t *l4 = reinterpret_cast<const uint32_t *>(p.lv8);
            for (uint64_t i = (uint64_t)cs.lid * blockDim.x + threadIdx.x; i < n4; i += nth) {
                const uint32_t b = __ldcg(l4 + i);
                int32_t o[4];
                bool direct = false;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t x = (b >> (8 * k)) & 0xFFu;
                    o[k] = (int32_t)x - 1;
                    direct |= x == 255u && 4 * i + k < V;
                }
                if (!direct && 4 * i + 4 <= V && ((uintptr_t)p.level_out & 15) == 0) {
                    *reinterpret_cast<int4 *>(p.level_out + 4 * i) = make_int4(o[0], o[1], o[2], o[3]);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (4 * i + k < V && ((b >> (8 * k)) & 0xFFu) != 255u) p.level_out[4 * i + k] = o[k];
                }
            }
        }
        return done;
    }

    static constexpr uint32_t kQueueRes = 256;   // per-warp queue reservation (>= 2 * 32 * KB)

    // empty entries in the unused reserved slots [res.x, res.y) (warp-collective)
    __device__ __forceinline__ static void fill_holes(LE *q, uint2 &res) {
        const uint32_t lane = threadIdx.x & 31;
        for (uint32_t i = res.x + lane; i < res.y; i += 32) {
            LE z;
            z.beg = 0;
            z.deg = 0;
            q[i] = z;
        }
        res = make_uint2(0, 0);
    }

    // ---------------------------------------------------------- top-down claim
    // Claim a batch of K candidates per lane at level L1 and push the winners to
    // the next frontier (warp-collective; u < 0 = no candidate).  The K probes,
    // the K atomics and the K offset reads are independent, so each warp keeps
    // K memory operations of each kind in flight.
    template <int K>
    __device__ __forceinline__ void visit_batch(const KParams &p, const int32_t (&u)[K], uint32_t L1,
                                                uint32_t out, uint32_t *fnext, uint32_t &reached,
                                                uint64_t &mfsum, uint2 &res) {
        const uint32_t lane = threadIdx.x & 31;
        uint32_t *vis = p.visited;
        uint32_t cur[K];
#pragma unroll
        for (int k = 0; k < K; ++k) cur[k] = u[k] >= 0 ? vis[(uint32_t)u[k] >> 5] : 0xFFFFFFFFu;  // pre-check
        bool win[K];
        const OffT *ro = static_cast<const OffT *>(p.ro);
        OffT nb[K], ne[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            win[k] = false;
            nb[k] = ne[k] = 0;
            if (u[k] >= 0) {
                const uint32_t bit = 1u << (u[k] & 31);
                if (!(cur[k] & bit)) {
                    win[k] = !(atomicOr(vis + ((uint32_t)u[k] >> 5), bit) & bit);   // claim
#if COOP_TD_SPEC_RO
                    // the candidate's offsets alongside the claim (independent of its result):
                    // one dependent round trip less per batch for the winners
                    nb[k] = __ldg(ro + u[k]);
                    ne[k] = __ldg(ro + u[k] + 1);
#endif
                }
            }
        }
        uint32_t nd[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            nd[k] = 0;
            if (win[k]) {
                store_level(p, u[k], L1);
#if !COOP_TD_SPEC_RO
                nb[k] = __ldg(ro + u[k]);
                ne[k] = __ldg(ro + u[k] + 1);
#endif
                nd[k] = (uint32_t)(ne[k] - nb[k]);
                mfsum += nd[k];
                if (fnext) atomicOr(fnext + ((uint32_t)u[k] >> 5), 1u << (u[k] & 31));
            }
        }
        // contract: warp ballots, one queue atomic per warp for the whole batch
        uint32_t m[K], off[K], tot = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            reached += __popc(__ballot_sync(FULL, win[k]));
            m[k] = __ballot_sync(FULL, win[k] && nd[k] > 0 && nd[k] < kHeavyDeg);
            off[k] = tot;
            tot += __popc(m[k]);
        }
        if (tot) {
            // slots come from a per-warp reservation of kQueueRes entries (one queue
            // atomic per kQueueRes appends instead of one per batch: the single counter
            // serialises every warp of the grid); unused slots are filled with empty
            // entries (deg 0), which expand to nothing
            LE *q = static_cast<LE *>(p.qlight[out]);
            if (res.x + tot > res.y) {
                fill_holes(q, res);
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(&p.ctl->qsize[out], kQueueRes);
                base = __shfl_sync(FULL, base, 0);
                res = make_uint2(base, base + kQueueRes);
            }
            const uint32_t pos = res.x;
            res.x += tot;
            const uint32_t lt = lanemask_lt();
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if ((m[k] >> lane) & 1u) {
                    LE le;
                    le.beg = nb[k];
                    le.deg = nd[k];
                    q[pos + off[k] + __popc(m[k] & lt)] = le;
                }
            }
        }
        // heavy winners: one packed {count, edges} atomic per warp batch (per-winner
        // atomics on the single counter serialise: hub levels push 1e4-1e5 of them);
        // entries take indices in (lane, k) order with prefix = running edge offset
        uint32_t hcnt = 0;
        uint64_t hdeg = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (win[k] && nd[k] >= kHeavyDeg) {
                hcnt += 1;
                hdeg += nd[k];
            }
        }
        if (__any_sync(FULL, hcnt != 0)) {
            uint32_t ci = hcnt;
            uint64_t di = hdeg;
#pragma unroll
            for (int s = 1; s < 32; s <<= 1) {
                const uint32_t cn = __shfl_up_sync(FULL, ci, s);
                const uint64_t dn = __shfl_up_sync(FULL, di, s);
                if (lane >= (uint32_t)s) { ci += cn; di += dn; }
            }
            const uint32_t ctot = __shfl_sync(FULL, ci, 31);
            const uint64_t dtot = __shfl_sync(FULL, di, 31);
            unsigned long long old = 0;
            if (lane == 0) old = atomicAdd(&p.ctl->heavy[out], ((unsigned long long)ctot << 40) | dtot);
            old = __shfl_sync(FULL, old, 0);
            uint64_t idx = (old >> 40) + (ci - hcnt), pre = (old & kMask40) + (di - hdeg);
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (win[k] && nd[k] >= kHeavyDeg) {
                    p.qheavy[out][idx] = HeavyEntry{(uint64_t)nb[k], pre, nd[k], 0u};
                    idx += 1;
                    pre += nd[k];
                }
            }
        }
    }

    // warp-wide neighbour gather over up to 32 lists (one per lane): prefix sum
    // of the degrees, then 32*KB edges per iteration, owner found by a shuffle
    // binary search (warp-level load balancing of short lists)
    __device__ __forceinline__ uint32_t gather(const KParams &p, OffT beg, uint32_t deg, uint32_t L1, uint32_t out,
                                               uint32_t *fnext, uint32_t &reached, uint64_t &mfsum, uint2 &res) {
        const uint32_t lane = threadIdx.x & 31;
        const int32_t *__restrict__ col = p.col;
#if COOP_L2_HINTS
        const unsigned long long pol_stream = l2_evict_first_policy();
#endif
        const uint32_t incl = warp_incl_scan(deg), excl = incl - deg;
        const uint32_t total = __shfl_sync(FULL, incl, 31);
        for (uint32_t e0 = 0; e0 < total; e0 += 32 * KB) {
            int32_t u[KB];
#pragma unroll
            for (int k = 0; k < KB; ++k) {
                const uint32_t e = e0 + 32 * k + lane;
                uint32_t j = 0;   // owner lane: largest j with excl_j <= e
#pragma unroll
                for (uint32_t s = 16; s >= 1; s >>= 1) {
                    const uint32_t c = j + s;
                    const uint32_t ex = __shfl_sync(FULL, excl, c);
                    if (ex <= e) j = c;
                }
                const OffT b = __shfl_sync(FULL, beg, j);
                const uint32_t ex = __shfl_sync(FULL, excl, j);
                u[k] = e < total ? LDS(col + b + (e - ex)) : -1;
            }
            visit_batch<KB>(p, u, L1, out, fnext, reached, mfsum, res);
        }
        return total;
    }

    // ---------------------------------------------------------- top-down, heavy entries
    // The edge range [0, Eh) of the high-degree frontier entries split evenly
    // over the M*W warps of the interval (static: done before any chunk claim,
    // so a CTA that later leaves at a chunk boundary has finished its slice).
    __device__ void expand_heavy(const KParams &p, CtaState &cs, uint64_t gw, uint64_t TW, uint32_t *fnext,
                                 uint64_t &edges, uint32_t &reached, uint64_t &mfsum, uint2 &res) {
        const uint32_t lane = threadIdx.x & 31;
        const uint32_t nh = cs.app_u32[1];
        const uint64_t Eh = ((uint64_t)cs.app_u32[3] << 32) | cs.app_u32[2];
        if (!nh) return;
        const uint32_t in = cs.in_sel, out = in ^ 1u;
        const uint32_t L1 = cs.level + 1;
        const int32_t *__restrict__ col = p.col;
#if COOP_L2_HINTS
        const unsigned long long pol_stream = l2_evict_first_policy();
#endif
        const HeavyEntry *hq = p.qheavy[in];
        const uint64_t s0 = Eh * gw / TW, s1 = Eh * (gw + 1) / TW;
        if (s0 >= s1) return;
        uint32_t lo = 0, hi = nh - 1;
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (ldcg(&hq[mid].prefix) <= s0) lo = mid; else hi = mid - 1;
        }
        uint32_t j = lo;
        uint64_t hb = ldcg(&hq[j].beg), hp = ldcg(&hq[j].prefix);
        uint32_t hd = ldcg(&hq[j].deg);
        constexpr uint32_t WIN = 32 * KB;   // <= kHeavyDeg: a window crosses at most one entry end
        for (uint64_t ws = s0; ws < s1; ws += WIN) {
            const uint64_t hend = hp + hd;
            uint64_t hb2 = hb, hp2 = hp;
            uint32_t hd2 = hd;
            if (ws + WIN >= hend && j + 1 < nh) {   // window reaches the next entry
                hb2 = ldcg(&hq[j + 1].beg); hp2 = ldcg(&hq[j + 1].prefix); hd2 = ldcg(&hq[j + 1].deg);
            }
            int32_t u[KB];
#pragma unroll
            for (int k = 0; k < KB; ++k) {
                const uint64_t e = ws + 32 * k + lane;
                u[k] = e < s1 ? LDS(col + (e < hend ? hb + (e - hp) : hb2 + (e - hp2))) : -1;
            }
            visit_batch<KB>(p, u, L1, out, fnext, reached, mfsum, res);
            if (ws + WIN >= hend) { ++j; hb = hb2; hp = hp2; hd = hd2; }
        }
        edges += s1 - s0;          // warp-uniform, added by every lane (x32 convention)
    }

    // ---------------------------------------------------------- top-down, queue input (one group)
    // warp group g: light entries [sz*g, sz*g + sz), sz <= 32 (one per lane)
    __device__ __forceinline__ void tdq_group(const KParams &p, CtaState &cs, uint64_t g, uint32_t sz, uint32_t *fnext,
                              uint64_t &edges, uint32_t &reached, uint64_t &mfsum, uint2 &res) {
        const uint32_t lane = threadIdx.x & 31;
        const uint32_t nl = cs.app_u32[0];
        const uint32_t in = cs.in_sel, out = in ^ 1u;
        const LE *inq = static_cast<const LE *>(p.qlight[in]);
        const uint64_t i = g * sz + lane;
        OffT beg = 0;
        uint32_t deg = 0;
        if (lane < sz && i < nl) {
            LE e = inq[i];
            beg = e.beg;
            deg = e.deg;
        }
        edges += (uint64_t)gather(p, beg, deg, cs.level + 1, out, fnext, reached, mfsum, res);
    }

    // ---------------------------------------------------------- top-down, bitmap input (one group)
    // lane l owns frontier word 32g+l and pops one vertex per round
    __device__ __forceinline__ void tdb_group(const KParams &p, CtaState &cs, uint64_t g, uint32_t *fnext, uint64_t &edges,
                              uint32_t &reached, uint64_t &mfsum, uint2 &res) {
        const uint32_t lane = threadIdx.x & 31;
        const uint32_t out = cs.in_sel ^ 1u;
        const uint32_t L1 = cs.level + 1;
        const uint32_t *fcur = p.fbits[cs.level % 3];
        const OffT *ro = static_cast<const OffT *>(p.ro);
        const uint64_t nw = ((uint64_t)p.V + 31) / 32;
        const uint64_t wi = g * 32 + lane;
        uint32_t word = wi < nw ? ldcg(fcur + wi) : 0u;
        while (__any_sync(FULL, word != 0)) {
            OffT beg = 0;
            uint32_t deg = 0;
            if (word) {
                const uint32_t b = __ffs(word) - 1;
                word &= word - 1;
                const uint64_t v = wi * 32 + b;
                beg = __ldg(ro + v);
                deg = (uint32_t)(__ldg(ro + v + 1) - beg);
            }
            edges += (uint64_t)gather(p, beg, deg, L1, out, fnext, reached, mfsum, res);
        }
    }

    // ---------------------------------------------------------- bottom-up (KW 32-vertex words)
    // each unvisited vertex scans its list (4 per step) for a parent in the
    // frontier bitmap and stops at the first hit.  The warp owns the visited /
    // next-frontier words, so no atomics.
    // Lane-per-vertex variant (COOP_BU_COMPACT=0): KW consecutive words per warp
    // item, lane l owns vertex (w0+k)*32 + l of each word k, all KW lists advance
    // together (EPS column loads and probes per list per step); an item is a load
    // half (bu_load: visited words, then the offsets of open words) and a process
    // half (bu_process).
    template <int KW>
    struct BuItem {
        uint32_t vw[KW];   // visited words
        OffT b[KW];        // ro[v] of this lane's vertex (v <= V)
        OffT e31[KW];      // lane 31: ro[v + 1] (other lanes take the next lane's b)
    };

    // offsets of the words with an unvisited lane, after the visited words arrive
    template <int KW>
    __device__ __forceinline__ void bu_load(const KParams &p, uint64_t w0, uint64_t nw, BuItem<KW> &x) {
        const uint32_t lane = threadIdx.x & 31;
        const OffT *ro = static_cast<const OffT *>(p.ro);
        const uint64_t V = (uint64_t)p.V;
#pragma unroll
        for (int k = 0; k < KW; ++k) x.vw[k] = w0 + k < nw ? p.visited[w0 + k] : 0xFFFFFFFFu;
#pragma unroll
        for (int k = 0; k < KW; ++k) {
            const uint64_t v = (w0 + k) * 32 + lane;
            const bool want = x.vw[k] != 0xFFFFFFFFu;
            x.b[k] = (want && v <= V) ? __ldg(ro + v) : (OffT)0;
            x.e31[k] = (want && lane == 31 && v < V) ? __ldg(ro + v + 1) : (OffT)0;
        }
    }

    static constexpr int EPS = COOP_BU_EPS;

    template <int KW>
    __device__ __forceinline__ void bu_process(const KParams &p, CtaState &cs, uint64_t w0, const BuItem<KW> &x,
                                               uint64_t &edges, uint32_t &reached, uint64_t &mfsum) {
        const uint32_t lane = threadIdx.x & 31;
        const uint32_t L1 = cs.level + 1;
        const uint32_t *fcur = p.fbits[cs.level % 3];
        uint32_t *fnext = p.fbits[L1 % 3];
        const int32_t *__restrict__ col = p.col;
        const uint64_t V = (uint64_t)p.V;
        bool any_open = false;
#pragma unroll
        for (int k = 0; k < KW; ++k) any_open |= x.vw[k] != 0xFFFFFFFFu;
        if (!any_open) return;                                 // warp-uniform
        OffT b[KW], e[KW];
        bool found[KW];
        uint32_t deg[KW], dead[KW];
#pragma unroll
        for (int k = 0; k < KW; ++k) {
            const uint64_t v = (w0 + k) * 32 + lane;
            const OffT nx = __shfl_down_sync(FULL, x.b[k], 1);
            const bool open = v < V && !((x.vw[k] >> lane) & 1u);
            b[k] = open ? x.b[k] : (OffT)0;
            e[k] = open ? (lane == 31 ? x.e31[k] : nx) : (OffT)0;
            found[k] = false;
            deg[k] = (uint32_t)(e[k] - b[k]);
            // unvisited and degree 0: never a neighbour (symmetric CSR), so it is
            // retired here once and later bottom-up levels skip it
            dead[k] = __ballot_sync(FULL, open && deg[k] == 0);
        }
        uint32_t scanned = 0;
        for (;;) {
            bool more = false;
#pragma unroll
            for (int k = 0; k < KW; ++k) more |= (b[k] < e[k] && !found[k]);
            if (!more) break;
            int32_t u[KW][EPS];
#pragma unroll
            for (int k = 0; k < KW; ++k) {
                const bool act = b[k] < e[k] && !found[k];
#pragma unroll
                for (int j = 0; j < EPS; ++j) u[k][j] = (act && b[k] + j < e[k]) ? __ldg(col + b[k] + j) : -1;
            }
#pragma unroll
            for (int k = 0; k < KW; ++k) {
                const bool act = b[k] < e[k] && !found[k];
#pragma unroll
                for (int j = 0; j < EPS; ++j)
                    if (u[k][j] >= 0 && ((fcur[(uint32_t)u[k][j] >> 5] >> (u[k][j] & 31)) & 1u)) found[k] = true;
                if (act) {
                    const uint32_t n = (uint32_t)min((OffT)EPS, (OffT)(e[k] - b[k]));
                    scanned += n;
                    b[k] += n;
                }
            }
        }
        edges += (uint64_t)scanned * 32;
#pragma unroll
        for (int k = 0; k < KW; ++k) {
            const uint32_t wins = __ballot_sync(FULL, found[k]);
            if (found[k]) {
                store_level(p, (int64_t)((w0 + k) * 32 + lane), L1);
                mfsum += deg[k];
            }
            if (wins | dead[k]) {
                if (lane == 0) {
                    p.visited[w0 + k] = x.vw[k] | wins | dead[k];
                    if (wins) fnext[w0 + k] = wins;
                }
                reached += __popc(wins);
            }
        }
    }

    template <int KW>
    __device__ __forceinline__ void bu_words(const KParams &p, CtaState &cs, uint64_t w0, uint64_t nw,
                                             uint64_t &edges, uint32_t &reached, uint64_t &mfsum) {
        BuItem<KW> x;
        bu_load<KW>(p, w0, nw, x);
        bu_process<KW>(p, cs, w0, x, edges, reached, mfsum);
    }

    // ---------------------------------------------------------- bottom-up, compacted candidates
    // Warp item = 32 visited words (lane l owns word w0 + l, one load for all).
    // The unvisited vertices of the 32 words are enumerated densely (warp prefix
    // sum of the per-word counts, then select the r-th open bit of the owner
    // word) and handed out K per lane per round, so every lane checks a real
    // candidate: sparse levels cost one visited load per 1024 vertices instead of
    // one per 128, and dense ones keep all lanes busy.  Found / degree-0 bits are
    // merged into the owner lane's word in shared memory (per-warp slots).
    __device__ __forceinline__ static uint32_t select_bit(uint32_t m, uint32_t r) {   // r-th set bit (0-based)
        uint32_t pos = 0;
#pragma unroll
        for (uint32_t w = 16; w; w >>= 1) {
            const uint32_t c = __popc(m & ((1u << w) - 1u));
            if (r >= c) { r -= c; m >>= w; pos += w; }
        }
        return pos;
    }

    template <int K>
    __device__ __forceinline__ void bu_compact(const KParams &p, CtaState &cs, uint64_t w0, uint64_t nw,
                                               uint32_t nwords, uint32_t *s_found, uint32_t *s_dead,
                                               uint64_t &edges, uint32_t &reached, uint64_t &mfsum) {
        const uint32_t lane = threadIdx.x & 31;
        const uint32_t L1 = cs.level + 1;
#if COOP_L2_HINTS
        const unsigned long long pol_stream = l2_evict_first_policy();
#endif
        const uint32_t *fcur = p.fbits[cs.level % 3];
        uint32_t *fnext = p.fbits[L1 % 3];
        const OffT *ro = static_cast<const OffT *>(p.ro);
        const int32_t *__restrict__ col = p.col;
        const uint64_t V = (uint64_t)p.V;
        const uint64_t w = w0 + lane;
        uint32_t vw = 0xFFFFFFFFu;
        if (lane < nwords && w < nw) {
            vw = p.visited[w];
            const uint64_t vend = (w + 1) * 32;
            if (vend > V) vw |= ~((1u << (uint32_t)(32 - (vend - V))) - 1u);   // bits past V: closed
        }
        const uint32_t open = ~vw;
        const uint32_t cnt = __popc(open);
        const uint32_t incl = warp_incl_scan(cnt), excl = incl - cnt;
        const uint32_t total = __shfl_sync(FULL, incl, 31);
        if (total == 0) return;                                  // warp-uniform
        s_found[lane] = 0u;
        s_dead[lane] = 0u;
        __syncwarp();
        uint32_t scanned = 0;
        for (uint32_t base = 0; base < total; base += 32 * K) {
            uint32_t own[K], bit[K];
            OffT b[K], e[K];
            bool found[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const uint32_t j = base + 32 * k + lane;
                uint32_t o = 0;   // owner lane: largest o with excl_o <= j
#pragma unroll
                for (uint32_t st = 16; st >= 1; st >>= 1) {
                    const uint32_t ex = __shfl_sync(FULL, excl, o + st);
                    if (ex <= j) o += st;
                }
                const uint32_t om = __shfl_sync(FULL, open, o), oe = __shfl_sync(FULL, excl, o);
                own[k] = o;
                bit[k] = j < total ? select_bit(om, j - oe) : 32u;
                b[k] = 0;
                e[k] = 0;
                found[k] = false;
                if (bit[k] < 32 && !p.probe) {
                    const uint64_t v = (w0 + o) * 32 + bit[k];
                    b[k] = LDS(ro + v);
                    e[k] = LDS(ro + v + 1);
                }
            }
            uint32_t deg[K];
            if (p.probe) {
                // probe records {degree | first neighbour}: one coalesced 8-B load decides
                // degree-0 vertices and first-neighbour hits (most candidates of a dense
                // level) without the row offsets or a random column sector
                unsigned long long rec[K];
                OffT b0[K];
#pragma unroll
                for (int k = 0; k < K; ++k) {   // the offset is loaded alongside (coalesced, independent)
                    const uint64_t v = (w0 + own[k]) * 32 + bit[k];
                    rec[k] = bit[k] < 32 ? LDS(p.probe + v) : 0ull;
                    b0[k] = bit[k] < 32 ? LDS(ro + v) : (OffT)0;
                }
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    deg[k] = (uint32_t)(rec[k] >> 32);
                    const uint32_t f = (uint32_t)rec[k];
                    if (bit[k] < 32 && deg[k] == 0) atomicOr(&s_dead[own[k]], 1u << bit[k]);   // never a neighbour
                    if (deg[k]) {
                        found[k] = (fcur[f >> 5] >> (f & 31)) & 1u;
                        scanned += 1;
                    }
                }
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    if (deg[k] > 1 && !found[k]) {   // the rest of the list from the second entry
                        b[k] = b0[k] + 1;
                        e[k] = b0[k] + deg[k];
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    deg[k] = (uint32_t)(e[k] - b[k]);
                    if (bit[k] < 32 && deg[k] == 0) atomicOr(&s_dead[own[k]], 1u << bit[k]);   // never a neighbour
                }
            }
            for (int step = 0; step < COOP_BU_SOLO; ++step) {   // per-lane: the first hits dominate
                bool more = false;
#pragma unroll
                for (int k = 0; k < K; ++k) more |= (b[k] < e[k] && !found[k]);
                if (!__any_sync(FULL, more)) break;
                int32_t u[K][EPS];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const bool act = b[k] < e[k] && !found[k];
#pragma unroll
                    for (int jj = 0; jj < EPS; ++jj) u[k][jj] = (act && b[k] + jj < e[k]) ? LDS(col + b[k] + jj) : -1;
                }
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const bool act = b[k] < e[k] && !found[k];
#pragma unroll
                    for (int jj = 0; jj < EPS; ++jj)
                        if (u[k][jj] >= 0 && ((fcur[(uint32_t)u[k][jj] >> 5] >> (u[k][jj] & 31)) & 1u)) found[k] = true;
                    if (act) {
                        const uint32_t n = (uint32_t)min((OffT)EPS, (OffT)(e[k] - b[k]));
                        scanned += n;
                        b[k] += n;
                    }
                }
            }
            // the rest of the long lists: one list at a time, 32 edges per warp step
            // (a lane walking a long list alone would hold the whole warp)
#pragma unroll
            for (int k = 0; k < K; ++k) {
                uint32_t m = __ballot_sync(FULL, b[k] < e[k] && !found[k]);
                while (m) {
                    const uint32_t ld = __ffs(m) - 1;
                    m &= m - 1;
                    const OffT lb = __shfl_sync(FULL, b[k], ld), le = __shfl_sync(FULL, e[k], ld);
                    bool hit = false;
                    for (OffT x = lb; x < le; x += 32) {
                        const OffT xe = x + lane;
                        const int32_t uu = xe < le ? LDS(col + xe) : -1;
                        const bool h = uu >= 0 && ((fcur[(uint32_t)uu >> 5] >> (uu & 31)) & 1u);
                        const uint32_t hm = __ballot_sync(FULL, h);
                        const OffT lim = min((OffT)32, (OffT)(le - x));
                        if (hm) {
                            scanned += lane == ld ? (uint32_t)(__ffs(hm)) : 0u;
                            hit = true;
                            break;
                        }
                        scanned += lane == ld ? (uint32_t)lim : 0u;
                    }
                    if (lane == ld) {
                        found[k] = hit;
                        b[k] = e[k];
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (found[k]) {
                    store_level(p, (int64_t)((w0 + own[k]) * 32 + bit[k]), L1);
                    atomicOr(&s_found[own[k]], 1u << bit[k]);
                    mfsum += deg[k];
                }
            }
        }
        edges += (uint64_t)scanned * 32;
        __syncwarp();
        const uint32_t f = s_found[lane], d = s_dead[lane];
        if (f | d) {   // only lanes that own an in-range word can have bits
            p.visited[w] = vw | f | d;
            if (f) fnext[w] = f;
        }
        reached += __reduce_add_sync(FULL, __popc(f));   // warp-uniform, like the other modes
        __syncwarp();
    }

    static constexpr uint32_t BU_KW = COOP_BU_KW;  // bottom-up: words per warp item

    // per-warp counters -> the CTA's shared accumulators (before a mid-interval kill and at
    // the end of the interval); thread 0 adds them to the control block right before the
    // CTA's arrival / kill-CAS (pre_arrive), whose release orders them -- one global atomic
    // per counter per CTA instead of one per warp plus a fence per warp (4736 warps hit the
    // same line at the end of every level)
    __device__ __forceinline__ void flush_counts(const KParams &p, CtaState &cs, uint32_t out, uint64_t &edges,
                                                 uint32_t &reached, uint64_t &mfsum) {
        const uint32_t lane = threadIdx.x & 31;
        uint64_t e = edges, m = mfsum;
#pragma unroll
        for (int s = 16; s; s >>= 1) {
            e += __shfl_xor_sync(FULL, e, s);
            m += __shfl_xor_sync(FULL, m, s);
        }
        if (lane == 0) {
            if (e) atomicAdd(&cs.edges, (unsigned long long)(e / 32));
            if (reached) {
                atomicAdd(&cs.reached, (unsigned long long)reached);
                atomicAdd(&cs.acc[0], (unsigned long long)reached);
            }
            if (m) atomicAdd(&cs.acc[1], (unsigned long long)m);
            cs.acc_sel = out;
        }
        edges = 0;
        reached = 0;
        mfsum = 0;
    }

    // thread 0, after the CTA barrier that follows every warp's flush_counts, before the
    // arrival or kill-CAS (both release): the level's counters (nf decides termination)
    __device__ __forceinline__ void pre_arrive(const KParams &p, CtaState &cs) {
        const unsigned long long nf = cs.acc[0], mf = cs.acc[1];
        if (nf | mf) {
            if (nf) atomicAdd(&p.ctl->nf[cs.acc_sel], nf);
            if (mf) atomicAdd(&p.ctl->mf[cs.acc_sel], mf);
            cs.acc[0] = cs.acc[1] = 0;
        }
    }

    template <int BLOCK, int DIST = DIST_STATIC>
    __device__ uint32_t expand(const KParams &p, CtaState &cs) {
        constexpr uint32_t WPB = BLOCK / 32;
        const uint32_t warp = threadIdx.x >> 5;
        const uint64_t gw = (uint64_t)cs.lid * WPB + warp;        // get_global_id at warp granularity
        const uint64_t TW = (uint64_t)cs.M * WPB;                 // get_global_size / 32
        const uint32_t in = cs.in_sel;
        // per-lane accumulators; edges are kept x32 (top-down counts are warp-uniform and
        // added by every lane; bottom-up counts are per lane and added x32)
        uint64_t edges = 0, mfsum = 0;
        uint32_t reached = 0;
        const uint32_t mode = cs.app_u32[5];
        uint32_t *fnext = p.dopt ? p.fbits[(cs.level + 1) % 3] : nullptr;
        // (a DIST_MID expand resumed after an offer_kill that did not take this CTA skips
        // the static-split steps it has done already)
        const bool first = DIST == DIST_STATIC || (DIST == DIST_MID && !cs.resume);
        if (p.dopt && first) {   // recycle the bitmap of level L-1 as the next-next frontier (static split)
            uint32_t *fold = p.fbits[(cs.level + 2) % 3];
            const uint64_t nw = ((uint64_t)p.V + 31) / 32;
            for (uint64_t i = (uint64_t)cs.lid * BLOCK + threadIdx.x; i < nw; i += (uint64_t)cs.M * BLOCK) fold[i] = 0u;
        }
        LTRACE(4);
        const uint32_t out = in ^ 1u;                             // parity filled by this level
        uint2 res = make_uint2(0, 0);
        auto flush = [&]() {
            fill_holes(static_cast<LE *>(p.qlight[out]), res);
            flush_counts(p, cs, out, edges, reached, mfsum);
        };
        const uint64_t nw = ((uint64_t)p.V + 31) / 32;
        uint32_t r;
        if (COOP_BU_COMPACT && mode == BFS_BU) {          // item = 32 words, compacted candidates
            __shared__ uint32_t s_bits[2][BLOCK];
            const uint32_t wb = (threadIdx.x >> 5) * 32;
            // the first bottom-up level is dense (most vertices still open): smaller
            // items so the static split stays balanced; later levels: 32 words
            const uint32_t W = cs.app_u32[6] <= 1 ? COOP_BU_DENSE_W : 32u;
            // chunk = items claimed per CTA claim; only used when a scheduler can ask for workgroups
            // mid-interval (static split otherwise): it bounds the offer_kill latency
            r = claim_items<BLOCK, DIST>(p, cs, *this, &p.ctl->claim[in][0][0], (nw + W - 1) / W, [&](uint64_t it) {
                bu_compact<COOP_BU_K>(p, cs, it * W, nw, W, &s_bits[0][wb], &s_bits[1][wb], edges, reached, mfsum);
            }, flush);
        } else if (mode == BFS_BU) {                          // item = BU_KW 32-vertex words
            r = claim_items<BLOCK, DIST>(p, cs, *this, &p.ctl->claim[in][0][0], (nw + BU_KW - 1) / BU_KW, [&](uint64_t it) {
                bu_words<BU_KW>(p, cs, it * BU_KW, nw, edges, reached, mfsum);
            }, flush);
        } else if (mode == BFS_TDB) {                         // item = 32 frontier words
            r = claim_items<BLOCK, DIST>(p, cs, *this, &p.ctl->claim[in][0][0], (nw + 31) / 32, [&](uint64_t g) {
                tdb_group(p, cs, g, fnext, edges, reached, mfsum, res);
            }, flush, COOP_TD_TAIL);
        } else {                                              // item = 32 light frontier entries
            if (first) expand_heavy(p, cs, gw, TW, fnext, edges, reached, mfsum, res);
            LTRACE(5);
            // entries per warp item: 32 (a full gather) when there are enough items for
            // every warp, else fewer, down to one list per warp -- a small frontier of
            // lists just under the heavy threshold would otherwise sit on a few warps
            const uint64_t nl = cs.app_u32[0];
            uint32_t sz = 32;
            while (sz > 1 && (nl + sz - 1) / sz < TW) sz >>= 1;
            r = claim_items<BLOCK, DIST>(p, cs, *this, &p.ctl->claim[in][0][0], (nl + sz - 1) / sz,
                            [&](uint64_t g) { tdq_group(p, cs, g, sz, fnext, edges, reached, mfsum, res); }, flush,
                            COOP_TD_TAIL);
        }
        LTRACE(6);
        if (r == ACT_CONT) flush();
        LTRACE(7);
        return r;
    }

    // Fig. 4 between the barriers: reset(out_nodes); per-level statistics; the
    // direction of the next level (Beamer: TD->BU if m_f > m_u/alpha, BU->TD if
    // n_f < V/beta)
    __device__ COOP_SERIAL_ATTR void serial(const KParams &p, CtaState &cs, uint32_t entry, bool resizing) {
        if (resizing && entry == ENTRY_RESTART) { init_ctl(p, run_source(p)); return; }
        if (!resizing || entry != ENTRY_AFTER_RB1) return;
        Ctl *c = p.ctl;
        const uint32_t in = cs.in_sel, out = in ^ 1u;        // post-swap selectors
        // every load first, as one batch of independent round trips (this runs on
        // the critical path of the barrier, while all other CTAs wait)
        const uint32_t prev = c->bmode[out];
        const unsigned long long nf = c->nf[in], mf = c->mf[in];
        const unsigned long long vis = c->vis_edges + mf, ftot = c->frontier_total;
        const uint32_t nlev = c->levels, nbu = c->n_bu_levels;
        c->qsize[out] = 0;
        c->heavy[out] = 0;
        reset_claims(c, out);
        c->nf[out] = 0;
        c->mf[out] = 0;
        c->vis_edges = vis;
        uint32_t mode = BFS_TDQ;
        if (p.dopt) {
            const unsigned long long mu = (unsigned long long)p.E - min((unsigned long long)p.E, vis);
            if (prev == BFS_BU) mode = nf * p.beta < (unsigned long long)p.V ? BFS_TDB : BFS_BU;
            else mode = mf * p.alpha > mu ? BFS_BU : BFS_TDQ;
            if (mode == BFS_BU) c->n_bu_levels = nbu + 1;
        }
        c->bmode[in] = mode;
        const unsigned long long now = globaltimer();
        if (cs.level < p.level_cap) p.level_t[cs.level] = now;   // level L's expand done
        if (nf) {
            const uint32_t L = cs.level + 1;
            if (L < p.level_cap) p.level_sizes[L] = (uint32_t)nf;
            c->frontier_total = ftot + nf;
            c->levels = nlev + 1;
        } else if (p.n_src) {
            // end of a run of the source loop: stamp it, and either stop (bit 31) or
            // reset the per-traversal counters for the next run (its init follows)
            const uint32_t r = c->run;
            if (r < p.run_cap) p.run_t[r] = now;
            const bool more = now - c->t_start < p.loop_ns;
            c->run = more ? r + 1 : ((r + 1) | 0x80000000u);
            if (more) {
                c->qsize[0] = c->qsize[1] = 0;
                c->heavy[0] = c->heavy[1] = 0;
                reset_claims(c, 0);
                reset_claims(c, 1);
                c->nf[0] = c->nf[1] = 0;
                c->mf[0] = c->mf[1] = 0;
                c->bmode[0] = c->bmode[1] = BFS_TDQ;
                c->n_bu_levels = 0;
            }
        }
    }
};

// ============================================================== SSSP
// Worklist SSSP (l-sssp of Table 1, reading R8): each interval relaxes the
// out-edges of the current worklist with atomicMin and appends every improved
// vertex once per round (atomicMax stamp).  With delta > 0 the worklist is
// split near/far (Davidson et al.'s near-far pile, a Delta-stepping variant):
// a relaxation with new distance < T goes to the next near worklist, others to
// the far pile; when the near worklist runs dry a DRAIN interval moves far
// entries with dist < T + delta to near (T += delta) and compacts the rest.
// The fixpoint -- and so every distance -- is the same as plain Bellman-Ford.
enum : uint32_t { SSSP_RELAX = 0, SSSP_DRAIN = 1, SSSP_DONE = 2 };
constexpr uint32_t kNoRound = 0xFFFFFFFFu;   // low word of an SSSP key not pushed to a near worklist

template <typename OffT, bool KCOOP = true>
struct SsspApp {
    static constexpr bool kCoop = KCOOP;
    static constexpr bool kBetween = false;
    __device__ void pre_arrive(const KParams &, CtaState &) {}
    __device__ bool next_run(const KParams &, CtaState &) { return false; }
    __device__ void enter(const KParams &, CtaState &) {}
    template <int BLOCK>
    __device__ void between(const KParams &, CtaState &) {}

    template <int BLOCK>
    __device__ void init(const KParams &p, CtaState &cs) {
        const uint64_t tid = (uint64_t)cs.lid * BLOCK + threadIdx.x;
        const uint64_t nth = (uint64_t)cs.M * BLOCK;
        const int64_t V = p.V, s = p.source;
        // key[v] = {dist:32 | ~round:32}: one 64-bit atomicMin both relaxes dist[v] and tells
        // whether v was already pushed to the near worklist of this round (low word ~r1; far
        // improvements and the initial state carry ~0 = "no round"); dist_out is written at the end
        for (uint64_t i = tid; i < (uint64_t)V; i += nth)
            p.dq[i] = (int64_t)i == s ? (unsigned long long)kNoRound : ~0ull;
        if (cs.lid == 0 && threadIdx.x == 0) {
            Ctl *c = p.ctl;
            static_cast<uint32_t *>(p.qlight[0])[0] = (uint32_t)s;
            c->qsize[0] = 1;
            c->smode[0] = SSSP_RELAX;
            c->T = p.delta ? p.delta : 0xFFFFFFFFull;
            if (p.level_cap) p.level_sizes[0] = 1;
            c->frontier_total = 1;
            c->levels = 1;
        }
    }

    __device__ bool empty(const KParams &p, CtaState &cs) {
        if (threadIdx.x == 0) {
            const Ctl *c = p.ctl;
            // plain loads after the barrier's acquire (overlapping round trips)
            const uint32_t q = c->qsize[cs.in_sel], m = c->smode[cs.in_sel], fs = c->far_sel;
            const uint32_t f0 = c->far_size[0], f1 = c->far_size[1];
            const unsigned long long T = c->T, Tlo = c->T_lo;
            cs.app_u32[0] = q;
            cs.app_u32[5] = m;
            cs.app_u32[1] = fs;
            cs.app_u32[2] = min(fs ? f1 : f0, p.far_cap);
            cs.app_u32[3] = (uint32_t)T;
            cs.app_u32[4] = (uint32_t)(T >> 32);
            cs.app_u32[6] = (uint32_t)Tlo;
            cs.app_u32[7] = (uint32_t)(Tlo >> 32);
        }
        cta_sync();
        const bool done = cs.app_u32[5] == SSSP_DONE;
        if (done) {   // every active CTA copies its stride of the distances out (the kernel's output)
            const uint64_t nth = (uint64_t)cs.M * blockDim.x;
            for (uint64_t i = (uint64_t)cs.lid * blockDim.x + threadIdx.x; i < (uint64_t)p.V; i += nth)
                p.dist_out[i] = (uint32_t)(ldcg(p.dq + i) >> 32);
        }
        return done;
    }

    uint32_t r1_cur;
    __device__ __forceinline__ uint32_t r1_of(const KParams &) const { return r1_cur; }

    // push v into the next near worklist (once per round) or into the far pile;
    // warp-collective, `who` = lane pushes somewhere, `near` selects the pile
    __device__ __forceinline__ void push(const KParams &p, bool who, bool near, uint32_t v, uint32_t dval,
                                         uint32_t out, uint32_t fout) {
        const uint32_t lane = threadIdx.x & 31;
        const uint32_t lt = lanemask_lt();
        const uint32_t mn = __ballot_sync(FULL, who && near);
        if (mn) {
            uint32_t pos = 0;
            if (lane == __ffs(mn) - 1) pos = atomicAdd(&p.ctl->qsize[out], (uint32_t)__popc(mn));
            pos = __shfl_sync(FULL, pos, __ffs(mn) - 1);
            if (who && near) static_cast<uint32_t *>(p.qlight[out])[pos + __popc(mn & lt)] = v;
        }
        const uint32_t mf = __ballot_sync(FULL, who && !near);
        if (mf) {
            uint32_t pos = 0;
            if (lane == __ffs(mf) - 1) pos = atomicAdd(&p.ctl->far_size[fout], (uint32_t)__popc(mf));
            pos = __shfl_sync(FULL, pos, __ffs(mf) - 1);
            if (who && !near) {
                const uint32_t slot = pos + __popc(mf & lt);
                if (slot < p.far_cap) {
                    p.far[fout][slot] = v;
                } else {                                                   // far pile full: relax it early
                    const uint32_t mark = ~r1_of(p);
                    const unsigned long long o = atomicMin(p.dq + v, ((unsigned long long)dval << 32) | mark);
                    if ((uint32_t)o != mark && (uint32_t)(o >> 32) >= dval)
                        static_cast<uint32_t *>(p.qlight[out])[atomicAdd(&p.ctl->qsize[out], 1u)] = v;
                }
            }
        }
    }

    // worklist entries [sz*g, sz*g+sz): relax their out-edges (warp-wide gather).  sz < 32
    // when the worklist is small (a road-like graph's wavefront: a few thousand entries),
    // so that every warp gets an item and a group's edges fit one 32-lane pass -- the
    // episode then costs one dependent chain of loads/atomics instead of several
    __device__ __forceinline__ void relax_group(const KParams &p, CtaState &cs, uint64_t g, uint32_t sz,
                                                uint64_t &edges) {
        const uint32_t lane = threadIdx.x & 31;
        const uint32_t in = cs.in_sel, out = in ^ 1u;
        const uint32_t r1 = cs.level + 1;
        const uint32_t fsel = cs.app_u32[1];
        const unsigned long long T = ((unsigned long long)cs.app_u32[4] << 32) | cs.app_u32[3];
        const uint32_t n = cs.app_u32[0];
        const uint32_t *inq = static_cast<const uint32_t *>(p.qlight[in]);
        const OffT *ro = static_cast<const OffT *>(p.ro);
        const int32_t *__restrict__ col = p.col;
        const uint32_t *__restrict__ wt = p.w;
        const uint64_t i = g * sz + lane;
        OffT beg = 0;
        uint32_t deg = 0, du = 0;
        if (lane < sz && i < n) {
            const uint32_t v = ldcg(inq + i);
            beg = __ldg(ro + v);
            deg = (uint32_t)(__ldg(ro + v + 1) - beg);
            du = (uint32_t)(ldcg(p.dq + v) >> 32);             // current dist[u] (reading R8)
        }
        const uint32_t incl = warp_incl_scan(deg), excl = incl - deg;
        const uint32_t total = __shfl_sync(FULL, incl, 31);
        edges += total;
        for (uint32_t e0 = 0; e0 < total; e0 += 32) {
            const uint32_t e = e0 + lane;
            uint32_t j = 0;
#pragma unroll
            for (uint32_t s = 16; s >= 1; s >>= 1) {
                const uint32_t c = j + s;
                const uint32_t ex = __shfl_sync(FULL, excl, c);
                if (ex <= e) j = c;
            }
            const OffT b = __shfl_sync(FULL, beg, j);
            const uint32_t ex = __shfl_sync(FULL, excl, j);
            const uint32_t dsrc = __shfl_sync(FULL, du, j);
            bool who = false, near = true;
            int32_t v = -1;
            uint32_t nd = 0;
            if (e < total) {
                const OffT k = b + (e - ex);
                v = __ldg(col + k);
                nd = dsrc + __ldg(wt + k);
                if (!COOP_SSSP_PRECHECK || nd < (uint32_t)(ldcg(p.dq + v) >> 32)) {   // pre-check
                    near = nd < T;
                    const uint32_t mark = near ? ~r1 : kNoRound;
                    const unsigned long long old = atomicMin(p.dq + v, ((unsigned long long)nd << 32) | mark);
                    const uint32_t od = (uint32_t)(old >> 32);
                    if (nd < od)                                        // relaxed; near: once per round
                        who = near ? (uint32_t)old != mark : true;
                    else if (near && nd == od && (uint32_t)old != mark)
                        // an equal distance replaced an older round mark with this round's:
                        // v now looks queued for this round, so queue it (a harmless extra
                        // expansion; otherwise a later improvement this round would skip it)
                        who = true;
                }
            }
            push(p, who, near, (uint32_t)v, nd, out, fsel);
        }
    }

    // far entries [32g, 32g+32) -> near worklist for Tlo <= dist < T (the serial
    // section raised T from Tlo); dist < Tlo means the vertex already went through a
    // near worklist after its last improvement (stale copy: dropped); the rest is
    // compacted into the other far buffer
    __device__ __forceinline__ void drain_group(const KParams &p, CtaState &cs, uint64_t g) {
        const uint32_t lane = threadIdx.x & 31;
        const uint32_t out = cs.in_sel ^ 1u;
        const uint32_t r1 = cs.level + 1;
        const uint32_t fsel = cs.app_u32[1];
        const unsigned long long T = ((unsigned long long)cs.app_u32[4] << 32) | cs.app_u32[3];
        const unsigned long long Tlo = ((unsigned long long)cs.app_u32[7] << 32) | cs.app_u32[6];
        const uint32_t nf = cs.app_u32[2];
        const uint32_t *fin = p.far[fsel];
        const uint64_t i = g * 32 + lane;
        uint32_t v = 0, d = 0xFFFFFFFFu;
        bool have = i < nf;
        if (have) {
            v = ldcg(fin + i);
            d = (uint32_t)(ldcg(p.dq + v) >> 32);
        }
        have = have && d >= Tlo;
        const bool near = have && d < T;
        bool who = have && !near;
        if (near) {                                          // once per round
            const unsigned long long o = atomicMin(p.dq + v, ((unsigned long long)d << 32) | ~r1);
            who = (uint32_t)o != ~r1;
        }
        if (have && !near) atomicMin(&p.ctl->far_min, d);
        push(p, who, near, v, d, out, fsel ^ 1u);
        __threadfence();   // far_min (RED) is read by the serial section
    }

    template <int BLOCK, int DIST = DIST_STATIC>
    __device__ uint32_t expand(const KParams &p, CtaState &cs) {
        constexpr uint32_t WPB = BLOCK / 32;
        const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        r1_cur = cs.level + 1;
        uint64_t edges = 0;
        auto flush = [&]() {
            if (lane == 0 && edges) atomicAdd(&cs.edges, (unsigned long long)edges);
            edges = 0;
        };
        const bool drain = cs.app_u32[5] == SSSP_DRAIN;
        const uint64_t items = drain ? cs.app_u32[2] : cs.app_u32[0];
        uint32_t sz = 32;                                   // worklist entries per warp item
        if (!drain) {
            const uint64_t TW = (uint64_t)cs.M * WPB;
            while (sz > COOP_SSSP_MIN_SZ && (items + sz - 1) / sz < TW) sz >>= 1;
        }
        const uint32_t r = claim_items<BLOCK, DIST>(p, cs, *this, &p.ctl->claim[cs.in_sel][0][0], (items + sz - 1) / sz,
                                                    [&](uint64_t g) {
            if (drain) drain_group(p, cs, g);
            else relax_group(p, cs, g, sz, edges);
        }, flush);
        if (r == ACT_CONT) flush();
        return r;
    }

    // between the barriers: reset(out); choose the next interval (relax, drain, done)
    __device__ void serial(const KParams &p, CtaState &cs, uint32_t entry, bool resizing) {
        if (!resizing || entry != ENTRY_AFTER_RB1) return;
        Ctl *c = p.ctl;
        const uint32_t in = cs.in_sel, out = in ^ 1u;        // post-swap selectors
        // every load first, one batch of independent round trips (critical path)
        const uint32_t done_mode = c->smode[out];
        uint32_t fsel = c->far_sel;
        const uint32_t n = c->qsize[in];
        const uint32_t fs0 = c->far_size[0], fs1 = c->far_size[1], fmin = c->far_min;
        const unsigned long long T0 = c->T, ftot = c->frontier_total;
        const uint32_t nlev = c->levels;
        c->qsize[out] = 0;
        reset_claims(c, out);
        if (done_mode == SSSP_DRAIN) {                        // kept entries now live in the other buffer
            c->far_size[fsel] = 0;
            fsel ^= 1u;
            c->far_sel = fsel;
        }
        const uint32_t nfar = min(fsel ? fs1 : fs0, p.far_cap);
        uint32_t mode = SSSP_RELAX;
        if (n == 0) {
            if (nfar == 0) {
                mode = SSSP_DONE;
            } else {
                // raise the threshold; skip empty bands using the smallest kept distance
                unsigned long long T = T0 + p.delta;
                if (done_mode == SSSP_DRAIN && fmin != 0xFFFFFFFFu && fmin >= T) T = (unsigned long long)fmin + 1;
                c->T_lo = T0;
                c->T = T;
                c->far_min = 0xFFFFFFFFu;
                mode = SSSP_DRAIN;
            }
        }
        c->smode[in] = mode;
        if (cs.level < p.level_cap) p.level_t[cs.level] = globaltimer();
        if (n) {
            const uint32_t L = cs.level + 1;
            if (L < p.level_cap) p.level_sizes[L] = n;
            c->frontier_total = ftot + n;
            c->levels = nlev + 1;
        }
    }
};

// ============================================================== barrier microbench
// Each interval: store stamp[id] = gen; after the barrier check that the
// stamp of a peer from the previous interval is visible (message passing
// across the barrier).  iters resizing barriers in total.
struct BarrierApp {
    static constexpr bool kCoop = true;
    static constexpr bool kBetween = false;
    __device__ void pre_arrive(const KParams &, CtaState &) {}
    __device__ bool next_run(const KParams &, CtaState &) { return false; }
    __device__ void enter(const KParams &, CtaState &cs) {
        if (threadIdx.x == 0) cs.app_u32[4] = 0;   // no previous interval for a (re)entered CTA
    }
    template <int BLOCK>
    __device__ void init(const KParams &, CtaState &) {}
    template <int BLOCK>
    __device__ void between(const KParams &, CtaState &) {}
    __device__ bool empty(const KParams &p, CtaState &cs) {
        return (uint64_t)cs.level >= p.iters;
    }
    template <int BLOCK, int DIST = DIST_STATIC>
    __device__ uint32_t expand(const KParams &p, CtaState &cs) {
        if (threadIdx.x == 0 && (p.flags & COOP_FLAG_CHECK)) {
            if (cs.app_u32[4]) {
                const uint32_t pm = cs.app_u32[5], pg = cs.app_u32[6];
                const uint32_t peer = (cs.lid + 1) % pm;
                if (ld_relaxed32(p.stamp + peer) < pg) {
                    atomicAdd(&p.ctl->violations, 1u);
                    atomicCAS(&p.ctl->err, DERR_NONE, DERR_INVARIANT);
                }
            }
            st_relaxed32(p.stamp + cs.lid, cs.gen);
            cs.app_u32[4] = 1;
            cs.app_u32[5] = cs.M;
            cs.app_u32[6] = cs.gen;
        }
        return ACT_CONT;
    }
    __device__ void serial(const KParams &, CtaState &, uint32_t, bool) {}
};

}  // namespace coop
