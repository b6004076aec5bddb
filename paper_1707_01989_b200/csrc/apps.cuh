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

namespace coop {

template <typename T>
__device__ __forceinline__ T ldcg(const T *p) { return __ldcg(p); }

// ============================================================== BFS
template <typename OffT>
struct BfsApp {
    using LE = typename std::conditional<sizeof(OffT) == 4, LightEntry, LightEntry64>::type;

    __device__ void enter(const KParams &, CtaState &) {}

    template <int BLOCK>
    __device__ void init(const KParams &p, CtaState &cs) {
        const uint64_t tid = (uint64_t)cs.lid * BLOCK + threadIdx.x;
        const uint64_t nth = (uint64_t)cs.M * BLOCK;
        const int64_t V = p.V, s = p.source;
        int32_t *lv = p.level_out;
        // level[v] = -1 (unreached, reading R10), level[s] = 0; 16-B vector stores on the aligned body
        const uint64_t head = ((16 - ((uintptr_t)lv & 15)) & 15) / 4;
        const uint64_t h = head < (uint64_t)V ? head : (uint64_t)V;
        for (uint64_t i = tid; i < h; i += nth) lv[i] = (int64_t)i == s ? 0 : -1;
        const uint64_t nvec = ((uint64_t)V - h) / 4;
        int4 *lv4 = reinterpret_cast<int4 *>(lv + h);
        for (uint64_t i = tid; i < nvec; i += nth) {
            int4 x = make_int4(-1, -1, -1, -1);
            const int64_t b = (int64_t)(h + 4 * i);
            if (s >= b && s < b + 4) {
                if (s == b) x.x = 0; else if (s == b + 1) x.y = 0; else if (s == b + 2) x.z = 0; else x.w = 0;
            }
            lv4[i] = x;
        }
        for (uint64_t i = h + 4 * nvec + tid; i < (uint64_t)V; i += nth) lv[i] = (int64_t)i == s ? 0 : -1;
        const uint64_t nw = ((uint64_t)V + 31) / 32;
        for (uint64_t i = tid; i < nw; i += nth) p.visited[i] = i == (uint64_t)(s >> 5) ? (1u << (s & 31)) : 0u;
        if (cs.lid == 0 && threadIdx.x == 0) {
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
            cs.reached += 1;
            if (p.level_cap) p.level_sizes[0] = 1;
            p.ctl->frontier_total = 1;
            p.ctl->levels = 1;
        }
    }

    __device__ bool empty(const KParams &p, CtaState &cs) {
        if (threadIdx.x == 0) {
            const uint32_t in = cs.in_sel;
            const uint32_t nl = ld_relaxed32(&p.ctl->qsize[in]);
            const unsigned long long hv = ld_relaxed64(&p.ctl->heavy[in]);
            cs.app_u32[0] = nl;
            cs.app_u32[1] = (uint32_t)(hv >> 40);
            const uint64_t Eh = hv & kMask40;
            cs.app_u32[2] = (uint32_t)Eh;
            cs.app_u32[3] = (uint32_t)(Eh >> 32);
        }
        __syncthreads();
        return cs.app_u32[0] == 0 && cs.app_u32[1] == 0;
    }

    // claim u at level L1 (atomic on the visited bitmap, reading R8) and push it
    // to the next frontier; warp-collective (every lane calls, u < 0 = nothing)
    __device__ __forceinline__ void visit(const KParams &p, int32_t u, uint32_t L1, uint32_t out,
                                          uint32_t &reached) {
        const uint32_t lane = threadIdx.x & 31;
        bool win = false;
        OffT nb = 0;
        uint32_t nd = 0;
        if (u >= 0) {
            const uint32_t wd = (uint32_t)u >> 5, bit = 1u << (u & 31);
            const uint32_t cur = p.visited[wd];                 // non-atomic pre-check (stale 0 is safe)
            if (!(cur & bit)) {
                const uint32_t old = atomicOr(&p.visited[wd], bit);
                if (!(old & bit)) {
                    win = true;
                    p.level_out[u] = (int32_t)L1;
                    const OffT *ro = static_cast<const OffT *>(p.ro);
                    nb = __ldg(ro + u);
                    nd = (uint32_t)(__ldg(ro + u + 1) - nb);
                }
            }
        }
        const uint32_t wins = __ballot_sync(FULL, win);
        reached += __popc(wins);
        const bool lw = win && nd > 0 && nd < kHeavyDeg;
        const uint32_t m = __ballot_sync(FULL, lw);
        if (m) {   // warp-aggregated append: one atomic per warp (ballot + popc)
            const uint32_t leader = __ffs(m) - 1;
            uint32_t pos = 0;
            if (lane == leader) pos = atomicAdd(&p.ctl->qsize[out], (uint32_t)__popc(m));
            pos = __shfl_sync(FULL, pos, leader);
            if (lw) {
                LE le;
                le.beg = nb;
                le.deg = nd;
                static_cast<LE *>(p.qlight[out])[pos + __popc(m & lanemask_lt())] = le;
            }
        }
        if (win && nd >= kHeavyDeg) {
            const unsigned long long old = atomicAdd(&p.ctl->heavy[out], (1ull << 40) | nd);
            p.qheavy[out][old >> 40] = HeavyEntry{(uint64_t)nb, old & kMask40, nd, 0u};
        }
    }

    template <int BLOCK>
    __device__ void expand(const KParams &p, CtaState &cs) {
        constexpr uint32_t WPB = BLOCK / 32;
        const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const uint64_t gw = (uint64_t)cs.lid * WPB + warp;        // get_global_id at warp granularity
        const uint64_t TW = (uint64_t)cs.M * WPB;                 // get_global_size / 32
        const uint32_t nl = cs.app_u32[0], nh = cs.app_u32[1];
        const uint64_t Eh = ((uint64_t)cs.app_u32[3] << 32) | cs.app_u32[2];
        const uint32_t in = cs.in_sel, out = in ^ 1u;
        const uint32_t L1 = cs.level + 1;
        const LE *inq = static_cast<const LE *>(p.qlight[in]);
        const int32_t *__restrict__ col = p.col;
        uint64_t edges = 0;
        uint32_t reached = 0;

        // ---- light entries: 32 per warp, Fig. 4 stride over warps
        for (uint64_t base = gw * 32; base < nl; base += TW * 32) {
            const uint64_t i = base + lane;
            OffT beg = 0;
            uint32_t deg = 0;
            if (i < nl) {
                LE e = inq[i];
                beg = e.beg;
                deg = e.deg;
            }
            const uint32_t incl = warp_incl_scan(deg), excl = incl - deg;
            const uint32_t total = __shfl_sync(FULL, incl, 31);
            edges += total;
            for (uint32_t e0 = 0; e0 < total; e0 += 32) {
                const uint32_t e = e0 + lane;
                uint32_t j = 0;   // owner lane: largest j with excl_j <= e
#pragma unroll
                for (uint32_t s = 16; s >= 1; s >>= 1) {
                    const uint32_t c = j + s;
                    const uint32_t ex = __shfl_sync(FULL, excl, c);
                    if (ex <= e) j = c;
                }
                const OffT b = __shfl_sync(FULL, beg, j);
                const uint32_t ex = __shfl_sync(FULL, excl, j);
                const int32_t u = e < total ? __ldg(col + b + (e - ex)) : -1;
                visit(p, u, L1, out, reached);
            }
        }

        // ---- heavy entries: the edge range [0, Eh) split evenly over the M*WPB warps
        if (nh) {
            const HeavyEntry *hq = p.qheavy[in];
            const uint64_t s0 = Eh * gw / TW, s1 = Eh * (gw + 1) / TW;
            if (s0 < s1) {
                uint32_t lo = 0, hi = nh - 1;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi + 1) >> 1;
                    if (ldcg(&hq[mid].prefix) <= s0) lo = mid; else hi = mid - 1;
                }
                uint32_t j = lo;
                uint64_t hb = ldcg(&hq[j].beg), hp = ldcg(&hq[j].prefix);
                uint32_t hd = ldcg(&hq[j].deg);
                for (uint64_t ws = s0; ws < s1; ws += 32) {
                    const uint64_t hend = hp + hd;
                    uint64_t hb2 = hb, hp2 = hp;
                    uint32_t hd2 = hd;
                    if (ws + 32 >= hend && j + 1 < nh) {   // window reaches the next entry
                        hb2 = ldcg(&hq[j + 1].beg); hp2 = ldcg(&hq[j + 1].prefix); hd2 = ldcg(&hq[j + 1].deg);
                    }
                    const uint64_t e = ws + lane;
                    int32_t u = -1;
                    if (e < s1) u = __ldg(col + (e < hend ? hb + (e - hp) : hb2 + (e - hp2)));
                    visit(p, u, L1, out, reached);
                    if (ws + 32 >= hend) { ++j; hb = hb2; hp = hp2; hd = hd2; }
                }
                edges += s1 - s0;
            }
        }
        if (lane == 0) {
            if (edges) atomicAdd(&cs.edges, (unsigned long long)edges);
            if (reached) atomicAdd(&cs.reached, (unsigned long long)reached);
        }
    }

    // Fig. 4 between the barriers: reset(out_nodes); per-level statistics
    __device__ void serial(const KParams &p, CtaState &cs, uint32_t entry, bool resizing) {
        if (!resizing || entry != ENTRY_AFTER_RB1) return;
        Ctl *c = p.ctl;
        const uint32_t in = cs.in_sel, out = in ^ 1u;        // post-swap selectors
        c->qsize[out] = 0;
        c->heavy[out] = 0;
        const uint32_t n = ld_relaxed32(&c->qsize[in]) + (uint32_t)(ld_relaxed64(&c->heavy[in]) >> 40);
        if (n) {
            const uint32_t L = cs.level + 1;
            if (L < p.level_cap) p.level_sizes[L] = n;
            c->frontier_total += n;
            c->levels += 1;
        }
    }
};

// ============================================================== SSSP
template <typename OffT>
struct SsspApp {
    __device__ void enter(const KParams &, CtaState &) {}

    template <int BLOCK>
    __device__ void init(const KParams &p, CtaState &cs) {
        const uint64_t tid = (uint64_t)cs.lid * BLOCK + threadIdx.x;
        const uint64_t nth = (uint64_t)cs.M * BLOCK;
        const int64_t V = p.V, s = p.source;
        for (uint64_t i = tid; i < (uint64_t)V; i += nth) {
            p.dist_out[i] = (int64_t)i == s ? 0u : 0xFFFFFFFFu;
            p.qlev[i] = 0u;
        }
        if (cs.lid == 0 && threadIdx.x == 0) {
            static_cast<uint32_t *>(p.qlight[0])[0] = (uint32_t)s;
            p.ctl->qsize[0] = 1;
            if (p.level_cap) p.level_sizes[0] = 1;
            p.ctl->frontier_total = 1;
            p.ctl->levels = 1;
        }
    }

    __device__ bool empty(const KParams &p, CtaState &cs) {
        if (threadIdx.x == 0) cs.app_u32[0] = ld_relaxed32(&p.ctl->qsize[cs.in_sel]);
        __syncthreads();
        return cs.app_u32[0] == 0;
    }

    template <int BLOCK>
    __device__ void expand(const KParams &p, CtaState &cs) {
        constexpr uint32_t WPB = BLOCK / 32;
        const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const uint64_t gw = (uint64_t)cs.lid * WPB + warp;
        const uint64_t TW = (uint64_t)cs.M * WPB;
        const uint32_t n = cs.app_u32[0];
        const uint32_t in = cs.in_sel, out = in ^ 1u;
        const uint32_t r1 = cs.level + 1;                         // round counter (transmitted "level")
        const uint32_t *inq = static_cast<const uint32_t *>(p.qlight[in]);
        uint32_t *outq = static_cast<uint32_t *>(p.qlight[out]);
        const OffT *ro = static_cast<const OffT *>(p.ro);
        const int32_t *__restrict__ col = p.col;
        const uint32_t *__restrict__ wt = p.w;
        uint64_t edges = 0;
        for (uint64_t base = gw * 32; base < n; base += TW * 32) {
            const uint64_t i = base + lane;
            OffT beg = 0;
            uint32_t deg = 0, du = 0;
            if (i < n) {
                const uint32_t v = ldcg(inq + i);
                beg = __ldg(ro + v);
                deg = (uint32_t)(__ldg(ro + v + 1) - beg);
                du = ldcg(p.dist_out + v);                         // current dist[u] (reading R8)
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
                bool push = false;
                int32_t v = -1;
                if (e < total) {
                    const OffT k = b + (e - ex);
                    v = __ldg(col + k);
                    const uint32_t nd = dsrc + __ldg(wt + k);
                    if (nd < ldcg(p.dist_out + v)) {                      // pre-check
                        const uint32_t old = atomicMin(p.dist_out + v, nd);   // relax
                        if (nd < old) push = atomicMax(p.qlev + v, r1) < r1;  // once per round
                    }
                }
                const uint32_t m = __ballot_sync(FULL, push);
                if (m) {
                    const uint32_t leader = __ffs(m) - 1;
                    uint32_t pos = 0;
                    if (lane == leader) pos = atomicAdd(&p.ctl->qsize[out], (uint32_t)__popc(m));
                    pos = __shfl_sync(FULL, pos, leader);
                    if (push) outq[pos + __popc(m & lanemask_lt())] = (uint32_t)v;
                }
            }
        }
        if (lane == 0 && edges) atomicAdd(&cs.edges, (unsigned long long)edges);
    }

    __device__ void serial(const KParams &p, CtaState &cs, uint32_t entry, bool resizing) {
        if (!resizing || entry != ENTRY_AFTER_RB1) return;
        Ctl *c = p.ctl;
        const uint32_t in = cs.in_sel, out = in ^ 1u;
        c->qsize[out] = 0;
        const uint32_t n = ld_relaxed32(&c->qsize[in]);
        if (n) {
            const uint32_t L = cs.level + 1;
            if (L < p.level_cap) p.level_sizes[L] = n;
            c->frontier_total += n;
            c->levels += 1;
        }
    }
};

// ============================================================== barrier microbench
// Each interval: store stamp[id] = gen; after the barrier check that the
// stamp of a peer from the previous interval is visible (message passing
// across the barrier).  iters resizing barriers in total.
struct BarrierApp {
    __device__ void enter(const KParams &, CtaState &cs) {
        if (threadIdx.x == 0) cs.app_u32[4] = 0;   // no previous interval for a (re)entered CTA
    }
    template <int BLOCK>
    __device__ void init(const KParams &, CtaState &) {}
    __device__ bool empty(const KParams &p, CtaState &cs) {
        return (uint64_t)cs.level >= p.iters;
    }
    template <int BLOCK>
    __device__ void expand(const KParams &p, CtaState &cs) {
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
    }
    __device__ void serial(const KParams &, CtaState &, uint32_t, bool) {}
};

}  // namespace coop
