// part_app.cuh -- 1-D vertex-partitioned cooperative BFS (BASELINE.json
// configs[4]).  Not in the paper (single iGPU): the paper's
// cooperative kernel runs unchanged on every GPU, and the per-level frontier
// exchange is fused into it as a direct NVLink peer-memory all-gather.
//
// Rank p owns vertices [vb, ve) (vb a multiple of 32) and stores every edge
// (u, v) with v owned, indexed by the global source u (row_offsets over all V,
// col = v - vb).  Per level L (two resizing barriers, Fig. 4):
//   expand : read the global frontier bitmap F[L&1] (own copy), scan the
//            local rows of its vertices, claim owned targets in the local
//            visited bitmap, write level L+1 and set their bit in the own
//            slice of F[(L+1)&1]
//   RB1    : resizing barrier
//   between: clear the consumed F[L&1]; store the own slice of F[(L+1)&1]
//            into every peer's copy (NVLink stores, 16 B each)
//   RB2    : resizing barrier whose serial section is also the cross-GPU
//            barrier: fence.sys, then publish (epoch, discovered count) into
//            every peer's flag block and wait for every peer's; the sum is
//            the size of the next global frontier (0 = terminate everywhere)
// Static hubs (local degree >= hub_deg) are processed edge-balanced over
// all warps so one hub cannot stall a level.
// With COOP_FLAG_DIROPT (and the owned rows of the symmetric graph) a level
// can run bottom-up instead: each owned unvisited vertex scans its neighbours
// for one in the (complete) global frontier bitmap.  The direction is chosen
// by Beamer's rule from the GLOBAL n_f / m_f exchanged with the counts, so
// every rank picks the same one.
#pragma once
#include "apps.cuh"

namespace coop {

template <typename OffT>
struct PartBfsApp {
    static constexpr bool kCoop = true;
    static constexpr bool kBetween = true;           // the exchange step between the two barriers
    __device__ void pre_arrive(const KParams &, CtaState &) {}
    __device__ bool next_run(const KParams &, CtaState &) { return false; }
    static constexpr int KB = 4;

    __device__ void enter(const KParams &, CtaState &) {}

    template <int BLOCK>
    __device__ void init(const KParams &p, CtaState &cs) {
        const PartParams &pp = p.part;
        const uint64_t tid = (uint64_t)cs.lid * BLOCK + threadIdx.x;
        const uint64_t nth = (uint64_t)cs.M * BLOCK;
        const int64_t s = p.source;
        const uint64_t nown = (uint64_t)(pp.ve - pp.vb);
        for (uint64_t i = tid; i < nown; i += nth) p.level_out[i] = (int64_t)i + pp.vb == s ? 0 : -1;
        const uint64_t nlw = (nown + 31) / 32;
        const bool own_s = s >= pp.vb && s < pp.ve;
        if (p.dopt) {   // owned degree-0 vertices start visited (bottom-up skips them; symmetric graph)
            const OffT *rro = static_cast<const OffT *>(pp.rro);
            const uint32_t lane = threadIdx.x & 31;
            for (uint64_t w = tid / 32; w < nlw; w += nth / 32) {
                const uint64_t v = w * 32 + lane;
                const bool d0 = v < nown && __ldg(rro + v + 1) == __ldg(rro + v);
                const uint32_t m = __ballot_sync(FULL, d0);
                if (lane == 0)
                    p.visited[w] = m | ((own_s && w == (uint64_t)((s - pp.vb) >> 5)) ? (1u << ((s - pp.vb) & 31)) : 0u);
            }
        } else {
            for (uint64_t i = tid; i < nlw; i += nth)
                p.visited[i] = (own_s && i == (uint64_t)((s - pp.vb) >> 5)) ? (1u << ((s - pp.vb) & 31)) : 0u;
        }
        const uint64_t nw = ((uint64_t)p.V + 31) / 32;
        uint32_t *F0 = pp.F[pp.rank][0], *F1 = pp.F[pp.rank][1];
        for (uint64_t i = tid; i < nw; i += nth) {     // every rank knows the source (level 0 frontier)
            F0[i] = i == (uint64_t)(s >> 5) ? (1u << (s & 31)) : 0u;
            F1[i] = 0u;
        }
        if (cs.lid == 0 && threadIdx.x == 0) {
            if (own_s && p.dopt) {   // the source's degree, summed over ranks in the init exchange
                const OffT *rro = static_cast<const OffT *>(pp.rro);
                p.ctl->pmf[0] = (unsigned long long)(rro[s - pp.vb + 1] - rro[s - pp.vb]);
            }
            p.ctl->pmode = BFS_TDB;
            p.ctl->gcount = 1;
            p.ctl->frontier_total = 1;
            p.ctl->levels = 1;
            if (p.level_cap) p.level_sizes[0] = 1;
            if (own_s) cs.reached += 1;
        }
    }

    __device__ bool empty(const KParams &p, CtaState &cs) {
        if (threadIdx.x == 0) {
            cs.app_u32[0] = p.ctl->gcount ? 1u : 0u;
            cs.app_u32[5] = p.ctl->pmode;
        }
        cta_sync();
        return cs.app_u32[0] == 0;
    }

    // claim owned targets t (local ids) -- warp-collective, batch of K per lane
    __device__ __forceinline__ void claim(const KParams &p, const int32_t (&t)[KB], uint32_t L1, uint32_t *fnext,
                                          uint32_t &won, unsigned long long &mf) {
        uint32_t *vis = p.visited;
        uint32_t cur[KB];
#pragma unroll
        for (int k = 0; k < KB; ++k) cur[k] = t[k] >= 0 ? vis[(uint32_t)t[k] >> 5] : 0xFFFFFFFFu;
#pragma unroll
        for (int k = 0; k < KB; ++k) {
            if (t[k] < 0) continue;
            const uint32_t bit = 1u << (t[k] & 31);
            if ((cur[k] & bit) || (atomicOr(vis + ((uint32_t)t[k] >> 5), bit) & bit)) continue;
            p.level_out[t[k]] = (int32_t)L1;
            const uint64_t g = (uint64_t)p.part.vb + (uint32_t)t[k];
            atomicOr(fnext + (g >> 5), 1u << (g & 31));
            ++won;
            if (p.dopt) {
                const OffT *rro = static_cast<const OffT *>(p.part.rro);
                mf += (unsigned long long)(__ldg(rro + t[k] + 1) - __ldg(rro + t[k]));
            }
        }
    }

    // bottom-up over the owned words: warp per 32 owned vertices, each unvisited
    // vertex scans its (global) neighbour list for a bit of the global frontier
    template <int BLOCK>
    __device__ void bottom_up(const KParams &p, CtaState &cs, uint64_t gw, uint64_t TW, uint64_t &edges,
                              uint32_t &won, unsigned long long &mf) {
        const PartParams &pp = p.part;
        const uint32_t lane = threadIdx.x & 31;
        const uint32_t L = cs.level, L1 = L + 1;
        const uint32_t *fcur = pp.F[pp.rank][L & 1];
        uint32_t *fnext = pp.F[pp.rank][L1 & 1];
        const OffT *rro = static_cast<const OffT *>(pp.rro);
        const int32_t *__restrict__ rcol = pp.rcol;
        const uint64_t nown = (uint64_t)(pp.ve - pp.vb);
        const uint64_t nlw = (nown + 31) / 32;
        const uint64_t gw0 = (uint64_t)pp.vb / 32;
        uint64_t scanned_total = 0;
        for (uint64_t w = gw; w < nlw; w += TW) {
            const uint32_t vw = ldcg(p.visited + w);
            if (vw == 0xFFFFFFFFu) continue;
            const uint64_t v = w * 32 + lane;
            const bool open = v < nown && !((vw >> lane) & 1u);
            OffT b = 0, e = 0;
            if (open) {
                b = __ldg(rro + v);
                e = __ldg(rro + v + 1);
            }
            const uint32_t deg = (uint32_t)(e - b);
            bool found = false;
            while (open && b < e && !found) {
                int32_t u[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) u[k] = b + k < e ? __ldg(rcol + b + k) : -1;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (u[k] >= 0 && ((ldcg(fcur + ((uint32_t)u[k] >> 5)) >> (u[k] & 31)) & 1u)) found = true;
                const uint32_t nstep = (uint32_t)min((OffT)4, (OffT)(e - b));
                scanned_total += nstep;
                b += nstep;
            }
            const uint32_t wins = __ballot_sync(FULL, found);
            if (found) {
                p.level_out[v] = (int32_t)L1;
                mf += deg;
                ++won;
            }
            if (wins && lane == 0) {
                p.visited[w] = vw | wins;
                fnext[gw0 + w] = wins;          // own slice word of the next global frontier
            }
        }
        // per-lane scans -> warp-uniform edge count (the caller adds `edges` once per warp)
#pragma unroll
        for (int s = 16; s; s >>= 1) scanned_total += __shfl_xor_sync(FULL, scanned_total, s);
        edges += scanned_total;
    }

    template <int BLOCK, int DIST = DIST_STATIC>
    __device__ uint32_t expand(const KParams &p, CtaState &cs) {
        constexpr uint32_t WPB = BLOCK / 32;
        const PartParams &pp = p.part;
        const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const uint64_t gw = (uint64_t)cs.lid * WPB + warp, TW = (uint64_t)cs.M * WPB;
        const uint32_t L = cs.level, L1 = L + 1;
        const uint32_t *fcur = pp.F[pp.rank][L & 1];
        uint32_t *fnext = pp.F[pp.rank][L1 & 1];
        const OffT *ro = static_cast<const OffT *>(p.ro);
        const int32_t *__restrict__ col = p.col;
        const uint64_t nw = ((uint64_t)p.V + 31) / 32;
        uint64_t edges = 0;
        uint32_t won = 0;
        unsigned long long mf = 0;
        if (cs.app_u32[5] == BFS_BU) {
            bottom_up<BLOCK>(p, cs, gw, TW, edges, won, mf);
        } else {
        // ---- frontier vertices from the bitmap, lane l owns word base+l
        for (uint64_t base = gw * 32; base < nw; base += TW * 32) {
            const uint64_t wi = base + lane;
            uint32_t word = wi < nw ? ldcg(fcur + wi) : 0u;
            while (__any_sync(FULL, word != 0)) {
                OffT beg = 0;
                uint32_t deg = 0;
                if (word) {
                    const uint32_t b = __ffs(word) - 1;
                    word &= word - 1;
                    const uint64_t u = wi * 32 + b;
                    beg = __ldg(ro + u);
                    deg = (uint32_t)(__ldg(ro + u + 1) - beg);
                    if (pp.nhub && deg >= pp.hub_deg) deg = 0;   // static hub: edge-balanced pass below
                }
                const uint32_t incl = warp_incl_scan(deg), excl = incl - deg;
                const uint32_t total = __shfl_sync(FULL, incl, 31);
                edges += total;
                for (uint32_t e0 = 0; e0 < total; e0 += 32 * KB) {
                    int32_t t[KB];
#pragma unroll
                    for (int k = 0; k < KB; ++k) {
                        const uint32_t e = e0 + 32 * k + lane;
                        uint32_t j = 0;
#pragma unroll
                        for (uint32_t s = 16; s >= 1; s >>= 1) {
                            const uint32_t c = j + s;
                            const uint32_t ex = __shfl_sync(FULL, excl, c);
                            if (ex <= e) j = c;
                        }
                        const OffT b = __shfl_sync(FULL, beg, j);
                        const uint32_t ex = __shfl_sync(FULL, excl, j);
                        t[k] = e < total ? __ldg(col + b + (e - ex)) : -1;
                    }
                    claim(p, t, L1, fnext, won, mf);
                }
            }
        }
        // ---- static hubs: hub edge space [0, Eh) split evenly over the warps;
        //      a hub segment is read only if the hub is in the frontier
        if (pp.nhub) {
            const uint64_t Eh = pp.hub_prefix[pp.nhub];
            const uint64_t s0 = Eh * gw / TW, s1 = Eh * (gw + 1) / TW;
            if (s0 < s1) {
                uint32_t lo = 0, hi = pp.nhub - 1;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi + 1) >> 1;
                    if (__ldg(pp.hub_prefix + mid) <= s0) lo = mid; else hi = mid - 1;
                }
                for (uint32_t h = lo; h < pp.nhub; ++h) {
                    const uint64_t hp = __ldg(pp.hub_prefix + h), hq = __ldg(pp.hub_prefix + h + 1);
                    if (hp >= s1) break;
                    const uint32_t hub = __ldg(pp.hub_ids + h);
                    if (!((ldcg(fcur + (hub >> 5)) >> (hub & 31)) & 1u)) continue;
                    const uint64_t a = hp > s0 ? hp : s0, z = hq < s1 ? hq : s1;
                    const OffT rb = __ldg(ro + hub);
                    edges += z - a;
                    for (uint64_t ws = a; ws < z; ws += 32 * KB) {
                        int32_t t[KB];
#pragma unroll
                        for (int k = 0; k < KB; ++k) {
                            const uint64_t e = ws + 32 * k + lane;
                            t[k] = e < z ? __ldg(col + rb + (e - hp)) : -1;
                        }
                        claim(p, t, L1, fnext, won, mf);
                    }
                }
            }
        }
        }   // top-down
#pragma unroll
        for (int s = 16; s; s >>= 1) {
            won += __shfl_xor_sync(FULL, won, s);
            mf += __shfl_xor_sync(FULL, mf, s);
        }
        if (lane == 0) {   // edges is warp-uniform, won / mf were per lane
            if (edges) atomicAdd(&cs.edges, (unsigned long long)edges);
            if (won) {
                atomicAdd(&cs.reached, (unsigned long long)won);
                atomicAdd(&p.ctl->pcount[L1 & 1], (unsigned long long)won);
            }
            if (mf) atomicAdd(&p.ctl->pmf[L1 & 1], mf);
            if (won || mf) __threadfence();   // REDs, read by the RB2 serial section
        }
        return ACT_CONT;
    }

    // between RB1 and RB2: recycle F[L&1], push the own slice of F[(L+1)&1]
    // to every peer (all-gather over NVLink stores)
    template <int BLOCK>
    __device__ void between(const KParams &p, CtaState &cs) {
        const PartParams &pp = p.part;
        const uint64_t tid = (uint64_t)cs.lid * BLOCK + threadIdx.x, nth = (uint64_t)cs.M * BLOCK;
        const uint32_t L = cs.level;
        const uint64_t nw = ((uint64_t)p.V + 31) / 32;
        uint32_t *fcur = pp.F[pp.rank][L & 1];
        if (pp.nccl) {
            // NCCL data plane: only the own slice of the consumed bitmap is cleared (it
            // receives level L+2's bits); the all-gather overwrites every other slice
            const uint64_t w0 = (uint64_t)pp.vb / 32;
            for (uint64_t i = tid; i < pp.slice_words; i += nth) fcur[w0 + i] = 0u;
            return;
        }
        for (uint64_t i = tid; i < nw; i += nth) fcur[i] = 0u;
        const uint32_t nb = (L + 1) & 1;
        const uint32_t *mine = pp.F[pp.rank][nb];
        const uint64_t w0 = (uint64_t)pp.vb / 32, w1 = ((uint64_t)pp.ve + 31) / 32;
        const uint64_t n = w1 - w0;
        // 16-B stores over the 4-word-aligned body, word stores at the edges
        const uint64_t a = min(n, (4 - (w0 & 3)) & 3);
        const uint64_t n4 = (n - a) / 4;
        for (int q = 0; q < pp.nranks; ++q) {
            if (q == pp.rank) continue;
            uint32_t *dst = pp.F[q][nb];
            for (uint64_t i = tid; i < a; i += nth) dst[w0 + i] = ldcg(mine + w0 + i);
            const uint4 *src4 = reinterpret_cast<const uint4 *>(mine + w0 + a);
            uint4 *dst4 = reinterpret_cast<uint4 *>(dst + w0 + a);
            for (uint64_t i = tid; i < n4; i += nth) dst4[i] = __ldcg(src4 + i);
            for (uint64_t i = a + 4 * n4 + tid; i < n; i += nth) dst[w0 + i] = ldcg(mine + w0 + i);
        }
        __threadfence_system();
    }

    // flag block of rank q: slot [r][parity] = {epoch << 32 | count, mf}; mf is
    // written first and published by the release store of the epoch word
    __device__ __forceinline__ bool exchange(const KParams &p, const CtaState &cs, uint32_t epoch,
                                             unsigned long long count, unsigned long long mf,
                                             unsigned long long *total, unsigned long long *mf_total) {
        const PartParams &pp = p.part;
        __threadfence_system();
        const unsigned long long word = ((unsigned long long)epoch << 32) | (count & 0xFFFFFFFFull);
        const uint32_t slot = (uint32_t)pp.rank * 4 + (epoch & 1) * 2;
        for (int q = 0; q < pp.nranks; ++q) {
            asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(pp.flags[q] + slot + 1), "l"(mf) : "memory");
            st_release_sys64(pp.flags[q] + slot, word);
        }
        unsigned long long sum = 0, msum = 0;
        const unsigned long long *mine = pp.flags[pp.rank];
        uint32_t spins = 0;
        for (int q = 0; q < pp.nranks; ++q) {
            const uint32_t qs = (uint32_t)q * 4 + (epoch & 1) * 2;
            unsigned long long v;
            while (((v = ld_acquire_sys64(mine + qs)) >> 32) != epoch) {
                if (spin_check(p, cs, spins)) return false;
            }
            sum += v & 0xFFFFFFFFull;
            unsigned long long m;
            asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(m) : "l"(mine + qs + 1) : "memory");
            msum += m;
        }
        *total = sum;
        *mf_total = msum;
        return true;
    }

    // NCCL data plane, RB1 of level L: publish this rank's counts for the all-gather and
    // release the comm stream (its cuStreamWaitValue32(ready >= L+1) precedes the gather)
    __device__ void nccl_publish(const KParams &p, const CtaState &cs) {
        const PartParams &pp = p.part;
        Ctl *c = p.ctl;
        const uint32_t L = cs.level, b = (L + 1) & 1;
        unsigned long long *snd = pp.cnt_send + 4 * b;
        snd[0] = c->pcount[b];
        snd[1] = c->pmf[b];
        snd[2] = L == 0 ? c->pmf[0] : 0ull;        // source degree (its owner), summed by every rank
        snd[3] = 0;
        c->pcount[b] = 0;
        c->pmf[b] = 0;
        if (L == 0) c->pmf[0] = 0;
        __threadfence_system();                      // bitmap slice + counts before the flag
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pp.ready), "r"(L + 1) : "memory");
        pp.host_ready[0] = L + 1;
    }

    // NCCL data plane, RB2 of level L (cs.level == L+1 here): wait for gather L, sum the counts
    __device__ bool nccl_collect(const KParams &p, const CtaState &cs, unsigned long long *tot,
                                 unsigned long long *mf, unsigned long long *src) {
        const PartParams &pp = p.part;
        const uint32_t L1 = cs.level;
        uint32_t spins = 0, g;
        for (;;) {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(g) : "l"(pp.gathered) : "memory");
            if (g >= L1) break;
            if (spin_check(p, cs, spins)) return false;
        }
        const unsigned long long *rcv = pp.cnt_recv + (uint64_t)(L1 & 1) * 4 * pp.nranks;
        unsigned long long a = 0, m = 0, s = 0;
        for (int q = 0; q < pp.nranks; ++q) {
            a += ldcg(rcv + 4 * q);
            m += ldcg(rcv + 4 * q + 1);
            s += ldcg(rcv + 4 * q + 2);
        }
        *tot = a;
        *mf = m;
        *src = s;
        return true;
    }

    __device__ void serial(const KParams &p, CtaState &cs, uint32_t entry, bool resizing) {
        Ctl *c = p.ctl;
        const uint32_t base = p.part.seq << 16;
        const uint64_t t0 = globaltimer();
        if (p.part.nccl) {
            if (!resizing) return;                   // init: the comm stream orders the first gather
            if (entry == ENTRY_AFTER_RB1) { nccl_publish(p, cs); return; }
            if (entry != ENTRY_AFTER_RB2) return;
            const uint32_t L = cs.level;
            unsigned long long tot = 0, mf = 0, src = 0;
            if (!nccl_collect(p, cs, &tot, &mf, &src)) return;
            if (L == 1) c->vis_edges = src;
            c->xwait_ns += globaltimer() - t0;
            next_level(p, tot, mf);
            if (!tot) {                               // every rank ends here: release any gathers enqueued ahead
                asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.part.ready), "r"(0xFFFFFFFFu) : "memory");
                p.part.host_ready[0] = 0x80000000u | L;   // final: L gathers were used
            }
            return;
        }
        if (!resizing) {   // the init global barrier: every rank cleared its bitmaps before any peer writes
            unsigned long long tot, mf;
            exchange(p, cs, base | 1u, 0, c->pmf[0], &tot, &mf);
            c->pmf[0] = 0;
            c->vis_edges = mf;                       // degree of the source
            c->xwait_ns += globaltimer() - t0;
            return;
        }
        if (entry != ENTRY_AFTER_RB2) return;
        const uint32_t L = cs.level;                 // level++ already done before RB2
        const unsigned long long mine = c->pcount[L & 1], mymf = c->pmf[L & 1];
        unsigned long long tot = 0, mf = 0;
        if (!exchange(p, cs, base | (L + 1), mine, mymf, &tot, &mf)) return;
        c->pcount[L & 1] = 0;
        c->pmf[L & 1] = 0;
        c->xwait_ns += globaltimer() - t0;
        next_level(p, tot, mf);
    }

    // global frontier size `tot` and its m_f: termination, next direction, statistics
    __device__ void next_level(const KParams &p, unsigned long long tot, unsigned long long mf) {
        Ctl *c = p.ctl;
        const uint32_t L = c->levels;                // levels counted so far (level index of `tot`)
        c->gcount = tot;
        // direction of the next level from the global n_f, m_f (same on every rank)
        const uint32_t prev = c->pmode;
        c->vis_edges += mf;
        uint32_t mode = BFS_TDB;
        if (p.dopt) {
            const unsigned long long Eg = (unsigned long long)p.part.E_global;
            const unsigned long long mu = Eg - min(Eg, c->vis_edges);
            if (prev == BFS_BU) mode = tot * p.beta < (unsigned long long)p.V ? BFS_TDB : BFS_BU;
            else mode = mf * p.alpha > mu ? BFS_BU : BFS_TDB;
            if (mode == BFS_BU) c->n_bu_levels += 1;
        }
        c->pmode = mode;
        if (tot) {
            if (L < p.level_cap) p.level_sizes[L] = (uint32_t)tot;
            c->frontier_total += tot;
            c->levels += 1;
        }
    }
};

}  // namespace coop
