/*
 * coop_protocol.cuh -- the resizing-barrier protocol of libcoop, shared by both
 * runtimes: the BFS/SSSP hot path (paper_1707_01989_b200/csrc/coop_rt.cuh) and
 * the device API for user kernels (include/coop_device.cuh).  This is the one
 * protocol oracle/barrier_model.py (O4) model-checks; the runtimes only add
 * their scheduling policy, statistics and CTA-collective plumbing around it.
 *
 * Words:
 *   W = {gen:32 | M:16 | arrived:16}  arrival word; arrivals are atomic adds, the
 *                                     CTA completing arrived == M is the last arriver
 *   R = {gen:32 | M':16 | flags:16}   release word on its own 128-B line; waiters poll it
 *                                     (flags, bit 0: a replay interval of handed-back work
 *                                     follows before the level ends -- BFS/SSSP runtime)
 * Steps (each a single atomic or ordered access, as modelled):
 *   arrive        atom.add.acq_rel W += 1          (release this CTA's interval, and for
 *                                                    the last arriver acquire everyone's)
 *   publish       W := {g+1, M', 0} (relaxed), then R := {g+1, M'} (release)
 *   wait_release  ld.acquire R until R.gen != g; killed iff R.gen != g+1 or id >= R.M
 *   kill_top      CAS W {g, M, a} -> {g, M-1, a} by id M-1 > 0, retried on concurrent
 *                 arrivals, abandoned if M or gen moved; the leaver completes
 *                 the episode on the waiters' behalf iff a == M-1
 *   add_forks     CAS W {g, M, a} -> {g, M+k, a} (bare request_fork)
 *   claim_idle    warp-collective claim of up to k set bits of the pool bitmap (parked,
 *                 forkable CTAs); each claimed CTA is handed to assign(phys, i)
 */
#ifndef COOP_PROTOCOL_CUH
#define COOP_PROTOCOL_CUH

#include <stdint.h>

namespace coop_proto {

// ---------------------------------------------------------------- ordered accesses
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_acquire32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_relaxed32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release32(uint32_t *p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed32(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long atom_add_acq_rel64(unsigned long long *p, unsigned long long v) {
    unsigned long long old;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
    return old;
}

// ---------------------------------------------------------------- the packed words
__device__ __forceinline__ uint32_t w_gen(unsigned long long w) { return (uint32_t)(w >> 32); }
__device__ __forceinline__ uint32_t w_M(unsigned long long w) { return (uint32_t)(w >> 16) & 0xFFFFu; }
__device__ __forceinline__ uint32_t w_arr(unsigned long long w) { return (uint32_t)w & 0xFFFFu; }
__device__ __forceinline__ unsigned long long pack_w(uint32_t g, uint32_t M, uint32_t a) {
    return ((unsigned long long)g << 32) | ((unsigned long long)(M & 0xFFFFu) << 16) | (a & 0xFFFFu);
}

// splitmix64 (Steele, Lea, Flood): the counter-based generator of the RANDOM policy
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// ---------------------------------------------------------------- protocol steps
__device__ __forceinline__ bool is_last(unsigned long long old);
// arrive: returns the word before this CTA's increment; last iff arrived + 1 == M
__device__ __forceinline__ unsigned long long arrive(unsigned long long *W) { return atom_add_acq_rel64(W, 1ull); }

// arrive_release: the release-only form -- a waiter acquires through the release word R, so
// only the last arriver needs the acquire, which it takes with a fence after the atomic (an
// acquire pattern: fence.acq_rel after the read of the release sequence's last value)
__device__ __forceinline__ unsigned long long arrive_release(unsigned long long *W) {
    unsigned long long old;
    asm volatile("atom.release.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(W), "l"(1ull) : "memory");
    if (is_last(old)) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    return old;
}
__device__ __forceinline__ bool is_last(unsigned long long old) { return w_arr(old) + 1u == w_M(old); }

// arrive_fenced: the same step for bodies that may leave other warps' fire-and-forget
// reductions in flight (user kernels of the device API): a full fence first, a relaxed
// add, and a fence for the last arriver before it reads everybody's results
__device__ __forceinline__ unsigned long long arrive_fenced(unsigned long long *W) {
    __threadfence();
    const unsigned long long old = atomicAdd(W, 1ull);
    if (is_last(old)) __threadfence();
    return old;
}

// publish (last arriver, or the leaver completing the episode): reset arrivals for
// generation g+1, then release every waiter (flags ride in R's low half-word)
__device__ __forceinline__ void publish(unsigned long long *W, unsigned long long *R, uint32_t g1, uint32_t Mp,
                                        uint32_t flags = 0u) {
    st_relaxed64(W, pack_w(g1, Mp, 0u));
    st_release64(R, pack_w(g1, Mp, flags));
}

// a waiter's fate once R moved on from generation g
enum : uint32_t { FATE_CONTINUE = 0, FATE_KILLED = 1 };
__device__ __forceinline__ uint32_t fate(unsigned long long r, uint32_t g, uint32_t lid) {
    return (w_gen(r) != g + 1u || lid >= w_M(r)) ? FATE_KILLED : FATE_CONTINUE;
}

// kill_top: CTA `lid` of generation g leaves if it is the top id M-1 > 0.  `w` is the
// caller's snapshot of W (updated on failed CASes).  Returns true when the CAS landed;
// *a_out = arrivals at that moment (a == M-1: every other CTA waits -> complete the
// episode on their behalf), *M_out = M before the kill.
__device__ __forceinline__ bool kill_top(unsigned long long *W, unsigned long long w, uint32_t lid, uint32_t g,
                                         uint32_t *a_out, uint32_t *M_out) {
    for (;;) {
        const uint32_t M = w_M(w);
        if (w_gen(w) != g || M != lid + 1u || M <= 1u) return false;   // a fork / kill / release moved W
        const unsigned long long prev = atomicCAS(W, w, pack_w(g, M - 1u, w_arr(w)));
        if (prev == w) {
            *a_out = w_arr(w);
            *M_out = M;
            return true;
        }
        w = prev;                                                       // arrivals raced the CAS
    }
}

// add_forks: W {g, M, a} -> {g, M+k, a}; returns M before (the first new id)
__device__ __forceinline__ uint32_t add_forks(unsigned long long *W, uint32_t k) {
    unsigned long long w = ld_relaxed64(W);
    for (;;) {
        const unsigned long long prev = atomicCAS(W, w, pack_w(w_gen(w), w_M(w) + k, w_arr(w)));
        if (prev == w) return w_M(w);
        w = prev;
    }
}

// inclusive warp scan
__device__ __forceinline__ uint32_t warp_scan(uint32_t v) {
    const uint32_t lane = threadIdx.x & 31u;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const uint32_t n = __shfl_up_sync(0xffffffffu, v, s);
        if (lane >= (uint32_t)s) v += n;
    }
    return v;
}

// claim_idle (warp-collective, every lane of the warp): clear up to k set bits of the
// pool bitmap pool[0, nwords) -- the lowest ones first -- and call assign(phys, i) for the
// i-th claimed CTA (i in [0, got), a dense numbering in claim order).  With `wait`,
// retries until k are claimed or abort() returns true (killed CTAs park promptly).
template <class Assign, class Abort>
__device__ __forceinline__ uint32_t claim_idle(uint32_t *pool, uint32_t nwords, uint32_t k, bool wait, Assign &&assign,
                                               Abort &&abort) {
    const uint32_t lane = threadIdx.x & 31u;
    uint32_t got = 0;
    while (got < k) {
        for (uint32_t w0 = 0; w0 < nwords && got < k; w0 += 32u) {
            const uint32_t wi = w0 + lane;
            uint32_t word = wi < nwords ? ld_relaxed32(&pool[wi]) : 0u;
            const uint32_t cnt = __popc(word);
            const uint32_t incl = warp_scan(cnt), excl = incl - cnt, need = k - got;
            const uint32_t want = need > excl ? min(cnt, need - excl) : 0u;
            uint32_t mask = 0u;
            for (uint32_t i = 0; i < want; ++i) {
                const uint32_t b = word & (0u - word);
                mask |= b;
                word ^= b;
            }
            uint32_t claimed = mask ? (atomicAnd(&pool[wi], ~mask) & mask) : 0u;
            const uint32_t nc = __popc(claimed);
            const uint32_t ci = warp_scan(nc);
            uint32_t r = got + ci - nc;
            while (claimed) {
                const uint32_t b = __ffs(claimed) - 1u;
                claimed &= claimed - 1u;
                assign(wi * 32u + b, r++);
            }
            got += __shfl_sync(0xffffffffu, ci, 31);
        }
        if (!wait || got >= k) break;
        uint32_t ab = 0;
        if (lane == 0) ab = abort() ? 1u : 0u;
        if (__shfl_sync(0xffffffffu, ab, 0)) break;
        __nanosleep(128);
    }
    __syncwarp();
    return got;
}

}  // namespace coop_proto

#endif  // COOP_PROTOCOL_CUH
