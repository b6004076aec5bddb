// part_sssp.cuh -- 1-D vertex-partitioned cooperative SSSP (SURVEY §8(e) "SSSP
// multi-GPU: needs (vertex, dist) exchange"; §8(f) rank 2).  Not in the paper.
//
// Same partition as PartBfsApp: rank p owns [vb, ve) and stores every edge
// (u, v, w) with v owned, indexed by the global source u.  The frontier is not
// a bitmap but a list of (vertex, distance) pairs: the vertices whose distance
// improved in the previous round, each rank contributing its owned ones.
// Round r (two resizing barriers, Fig. 4):
//   expand : for every source rank q, every pair (u, du) of q's list in this
//            rank's inbox (parity r&1): relax the local edges (u, v, w) --
//            one 64-bit atomicMin on key[v] = {dist:32 | ~round:32} (the SSSP
//            relaxation of reading R8); an owned v whose distance dropped is
//            appended to the own next list once per round
//   RB1
//   between: the own list becomes pairs (v, dist(v)) -- read AFTER every
//            relaxation of the round, so a vertex improved twice carries its
//            final distance -- stored into every rank's inbox (parity (r+1)&1)
//            at offset vb (disjoint per source rank) with NVLink peer stores
//   RB2    : its serial section is the cross-GPU barrier: every rank publishes
//            its list length and reads every peer's (the inbox counts of the
//            next round); the sum 0 terminates every rank at the same round.
// Plain data-driven Bellman-Ford per round (no near-far bands): the fixpoint is
// the shortest-path distance, so every schedule and rank count gives the same
// output (tests compare with Dijkstra).
#pragma once
#include "part_app.cuh"

namespace coop {

template <typename OffT>
struct PartSsspApp {
    static constexpr bool kCoop = true;
    static constexpr bool kBetween = true;           // the exchange step between the two barriers
    __device__ void pre_arrive(const KParams &, CtaState &) {}
    __device__ bool next_run(const KParams &, CtaState &) { return false; }
    __device__ void enter(const KParams &, CtaState &) {}

    // pair (global vertex, distance) of the inbox slot of source rank q, parity b
    __device__ __forceinline__ static unsigned long long *inbox(const KParams &p, int rank, uint32_t b) {
        return reinterpret_cast<unsigned long long *>(p.part.F[rank][b]);
    }

    template <int BLOCK>
    __device__ void init(const KParams &p, CtaState &cs) {
        const PartParams &pp = p.part;
        const uint64_t tid = (uint64_t)cs.lid * BLOCK + threadIdx.x, nth = (uint64_t)cs.M * BLOCK;
        const uint64_t nown = (uint64_t)(pp.ve - pp.vb);
        const int64_t s = p.source;
        for (uint64_t i = tid; i < nown; i += nth) p.dq[i] = (int64_t)i + pp.vb == s ? (unsigned long long)kNoRound : ~0ull;
        if (cs.lid == 0 && threadIdx.x == 0) {
            Ctl *c = p.ctl;
            // round 0's frontier {(s, 0)} is known to every rank: its owner's inbox slot
            int owner = 0;
            while (owner + 1 < pp.nranks && s >= pp.qvb[owner + 1]) ++owner;
            inbox(p, pp.rank, 0)[pp.qvb[owner]] = ((unsigned long long)s << 32) | 0ull;
            for (int q = 0; q < kMaxRanks; ++q) c->qcnt[q] = q == owner ? 1u : 0u;
            c->list_n[0] = c->list_n[1] = 0;
            c->gcount = 1;
            c->frontier_total = 1;
            c->levels = 1;
            if (p.level_cap) p.level_sizes[0] = 1;
        }
    }

    __device__ bool empty(const KParams &p, CtaState &cs) {
        if (threadIdx.x == 0) cs.app_u32[0] = p.ctl->gcount ? 1u : 0u;
        cta_sync();
        const bool done = cs.app_u32[0] == 0;
        if (done) {   // every active CTA writes its stride of the owned distances
            const uint64_t nown = (uint64_t)(p.part.ve - p.part.vb);
            const uint64_t nth = (uint64_t)cs.M * blockDim.x;
            for (uint64_t i = (uint64_t)cs.lid * blockDim.x + threadIdx.x; i < nown; i += nth)
                p.dist_out[i] = (uint32_t)(ldcg(p.dq + i) >> 32);
        }
        return done;
    }

    template <int BLOCK, int DIST = DIST_STATIC>
    __device__ uint32_t expand(const KParams &p, CtaState &cs) {
        constexpr uint32_t WPB = BLOCK / 32;
        const PartParams &pp = p.part;
        const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const uint64_t gw = (uint64_t)cs.lid * WPB + warp, TW = (uint64_t)cs.M * WPB;
        const uint32_t r1 = cs.level + 1, in = cs.level & 1u, out = r1 & 1u;
        const OffT *ro = static_cast<const OffT *>(p.ro);
        const int32_t *__restrict__ col = p.col;
        const uint32_t *__restrict__ wt = p.w;
        const unsigned long long *ib = inbox(p, pp.rank, in);
        uint32_t *list = pp.list[out];
        uint64_t edges = 0;
        for (int q = 0; q < pp.nranks; ++q) {
            const uint32_t n = (uint32_t)ldcg(&p.ctl->qcnt[q]);
            const unsigned long long *src = ib + pp.qvb[q];
            for (uint64_t g = gw; g * 32 < n; g += TW) {
                const uint64_t i = g * 32 + lane;
                OffT beg = 0;
                uint32_t deg = 0, du = 0;
                if (i < n) {
                    const unsigned long long e = ldcg(src + i);
                    const uint32_t u = (uint32_t)(e >> 32);
                    du = (uint32_t)e;
                    beg = __ldg(ro + u);
                    deg = (uint32_t)(__ldg(ro + u + 1) - beg);
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
                    bool who = false;
                    int32_t v = -1;
                    if (e < total) {
                        const OffT k = b + (e - ex);
                        v = __ldg(col + k);                          // rank-local destination
                        const uint32_t nd = dsrc + __ldg(wt + k);
                        const uint32_t mark = ~r1;
                        const unsigned long long old = atomicMin(p.dq + v, ((unsigned long long)nd << 32) | mark);
                        const uint32_t od = (uint32_t)(old >> 32);
                        // dropped: queue once per round; equal distance over an older mark: queue
                        // too (the mark now claims "queued this round", reading R8)
                        who = (nd < od && (uint32_t)old != mark) || (nd == od && (uint32_t)old != mark);
                    }
                    const uint32_t m = __ballot_sync(FULL, who);
                    if (m) {
                        uint32_t pos = 0;
                        if (lane == __ffs(m) - 1) pos = atomicAdd(&p.ctl->list_n[out], (uint32_t)__popc(m));
                        pos = __shfl_sync(FULL, pos, __ffs(m) - 1);
                        if (who) list[pos + __popc(m & lanemask_lt())] = (uint32_t)v;
                    }
                }
            }
        }
        if (lane == 0 && edges) atomicAdd(&cs.edges, (unsigned long long)edges);
        return ACT_CONT;
    }

    // between RB1 and RB2: the own list as (vertex, final distance of the round) pairs into
    // every rank's inbox (own included), at offset vb
    template <int BLOCK>
    __device__ void between(const KParams &p, CtaState &cs) {
        const PartParams &pp = p.part;
        const uint64_t tid = (uint64_t)cs.lid * BLOCK + threadIdx.x, nth = (uint64_t)cs.M * BLOCK;
        const uint32_t out = (cs.level + 1) & 1u;
        const uint32_t n = (uint32_t)ldcg(&p.ctl->list_n[out]);
        const uint32_t *list = pp.list[out];
        for (uint64_t i = tid; i < n; i += nth) {
            const uint32_t v = ldcg(list + i);
            const unsigned long long pair =
                ((unsigned long long)(pp.vb + v) << 32) | (uint32_t)(ldcg(p.dq + v) >> 32);
            for (int q = 0; q < pp.nranks; ++q) inbox(p, q, out)[pp.vb + i] = pair;
        }
        __threadfence_system();
    }

    __device__ void serial(const KParams &p, CtaState &cs, uint32_t entry, bool resizing) {
        Ctl *c = p.ctl;
        const PartParams &pp = p.part;
        const uint32_t base = pp.seq << 16;
        if (!resizing) {   // init barrier: every rank's inbox slot of round 0 is written locally
            unsigned long long cnt[kMaxRanks];
            exchange_counts(p, cs, base | 1u, 0, cnt);
            return;
        }
        if (entry != ENTRY_AFTER_RB2) return;
        const uint32_t L = cs.level;                 // level++ done: the round whose lists were built
        const uint32_t b = L & 1u;
        unsigned long long cnt[kMaxRanks];
        if (!exchange_counts(p, cs, base | (L + 1), c->list_n[b], cnt)) return;
        unsigned long long tot = 0;
        for (int q = 0; q < kMaxRanks; ++q) {
            const unsigned long long x = q < pp.nranks ? cnt[q] : 0ull;
            c->qcnt[q] = x;
            tot += x;
        }
        c->list_n[b] = 0;
        c->gcount = tot;
        if (tot) {
            if (L < p.level_cap) p.level_sizes[L] = (uint32_t)tot;
            c->frontier_total += tot;
            c->levels += 1;
        }
    }

    // cross-GPU barrier of the serial section: publish this rank's count, read every
    // rank's (flag block slot [rank][epoch & 1] of every peer, as PartBfsApp::exchange)
    __device__ bool exchange_counts(const KParams &p, const CtaState &cs, uint32_t epoch, unsigned long long count,
                                    unsigned long long *out) {
        const PartParams &pp = p.part;
        __threadfence_system();
        const unsigned long long word = ((unsigned long long)epoch << 32) | (count & 0xFFFFFFFFull);
        const uint32_t slot = (uint32_t)pp.rank * 4 + (epoch & 1) * 2;
        for (int q = 0; q < pp.nranks; ++q) st_release_sys64(pp.flags[q] + slot, word);
        const unsigned long long *mine = pp.flags[pp.rank];
        uint32_t spins = 0;
        for (int q = 0; q < pp.nranks; ++q) {
            const uint32_t qs = (uint32_t)q * 4 + (epoch & 1) * 2;
            unsigned long long v;
            while (((v = ld_acquire_sys64(mine + qs)) >> 32) != epoch)
                if (spin_check(p, cs, spins)) return false;
            out[q] = v & 0xFFFFFFFFull;
        }
        return true;
    }
};

}  // namespace coop
