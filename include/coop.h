/*
 * coop.h -- C ABI of libcoop: cooperative kernels (Sorensen, Evrard, Donaldson,
 * arXiv 1707.01989) on NVIDIA B200 (sm_100a).
 *
 * The library runs the paper's hot path -- Fig. 4's cooperative graph
 * traversal as BFS and as worklist SSSP -- inside ONE
 * persistent kernel per call.  Its CTAs are the paper's workgroups: at most N
 * are resident (occupancy-bound execution), M of them are
 * active with contiguous ids [0, M).  They meet at a
 * resizing global barrier (efficient "query" form
 * PAPER.md:936-950) where the scheduler may kill the top ids (offer_kill,
 * PAPER.md:529-550) or fork new ids that receive workgroup 0's transmitted
 * state (request_fork).  Killed CTAs park in an in-kernel
 * worker loop that runs a competing non-cooperative task (megakernel,
 * PAPER.md:805-826); a scheduler CTA posts the task and the
 * resource messages.
 *
 * Conventions (all functions):
 *   - Every function returns a coop_status and never aborts or throws.  On any
 *     status other than COOP_OK, outputs are unspecified and
 *     coop_last_error() describes the failure (thread-local string).
 *   - "device" pointers are CUDA device pointers on the current device (e.g.
 *     torch tensor data_ptr()); "host" pointers are ordinary CPU memory.
 *   - The caller owns graph, output and stats buffers.  The library owns its
 *     scratch (queues, bitmaps, control words), cached per device and reused.
 *   - Blocking calls (coop_bfs, coop_sssp, ...) enqueue on opts->stream and
 *     synchronise that stream before returning.  One in-flight call per stream.
 *   - Nothing in the library falls back to the CPU.
 */
#ifndef COOP_H
#define COOP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COOP_ABI_VERSION 1

typedef enum {
    COOP_OK = 0,
    COOP_ERR_INVALID_ARG = 1,      /* bad pointer, size, source out of range, bad option */
    COOP_ERR_CUDA = 2,             /* a CUDA runtime call failed (no device, launch failure, ...) */
    COOP_ERR_NOT_CORESIDENT = 3,   /* N (+ scheduler CTA) exceeds the co-resident CTA capacity */
    COOP_ERR_FORK_BOUND = 4,       /* a grant would exceed N - M */
    COOP_ERR_NO_CAPACITY = 5,      /* a task asks for more than N - 1 workgroups (WG 0 is never killed) */
    COOP_ERR_TIMEOUT = 6,          /* in-kernel watchdog fired (a spin exceeded opts->timeout_ns) */
    COOP_ERR_OVERFLOW = 7,         /* SSSP: (V-1) * max_weight >= 2^32 - 1, distances not representable */
    COOP_ERR_NCCL = 8,             /* reserved for the partitioned multi-GPU path */
    COOP_ERR_INVARIANT = 9,        /* COOP_FLAG_CHECK: a barrier / contiguity invariant was violated */
    COOP_ERR_BUSY = 10             /* handle API: operation not valid in the handle's state */
} coop_status;

/* Resizing-barrier implementation. */
typedef enum {
    COOP_BARRIER_QUERY = 0,   /* query barrier: all W demanded WGs leave in one episode */
    COOP_BARRIER_PLAIN = 1,   /* NON-cooperative baseline: plain global barrier, all N CTAs, no scheduler
                                 interaction (Fig. 3); used for the overhead comparison */
    COOP_BARRIER_NAIVE = 2    /* naive barrier: a WG offers kill once on entry, so ~1 WG leaves per episode */
} coop_barrier_mode;

/* Who decides M' at each resizing barrier (the nondeterministic scheduler choice). */
typedef enum {
    COOP_POLICY_NEVER = 0,     /* never resize */
    COOP_POLICY_SCRIPTED = 1,  /* M' = script[episode] (0 = unchanged); waits for parked CTAs so the script is exact */
    COOP_POLICY_RANDOM = 2,    /* with probability resize_prob, M' ~ U[1, N] (counter RNG keyed by seed, episode) */
    COOP_POLICY_SCHEDULER = 3  /* scheduler CTA: periodic competing task, demand/grant resource messages */
} coop_policy;

#define COOP_FLAG_CHECK 0x1u   /* per-episode arrival / contiguity / message-passing checks -> COOP_ERR_INVARIANT */
#define COOP_FLAG_DIROPT 0x2u  /* BFS: direction-optimising levels (bottom-up on large frontiers, Beamer's
                                  alpha=14 / beta=24 switch); results are identical, only the work differs.
                                  Requires a symmetric CSR (undirected graph): bottom-up reads out-lists as
                                  in-lists. */

/* CSR graph, device memory, neighbour lists of vertex v at [row_offsets[v], row_offsets[v+1]). */
typedef struct {
    int64_t num_vertices;       /* V >= 1 */
    int64_t num_edges;          /* E = row_offsets[V] (directed entries) */
    const void *row_offsets;    /* device, V+1 entries, uint32 (offset_bits=32) or int64 (offset_bits=64) */
    int32_t offset_bits;        /* 32 or 64 */
    const int32_t *col_idx;     /* device, E entries in [0, V) */
    const uint32_t *weights;    /* device, E entries >= 1 (SSSP), NULL for BFS */
    uint32_t max_weight;        /* SSSP: max of weights (0 = unknown: the library computes it) */
    const uint64_t *probe;      /* optional device array of V probe records {degree << 32 | first neighbour}
                                   (first neighbour 0xFFFFFFFF if degree 0) built once per graph by
                                   coop_csr_probe; bottom-up BFS levels then decide degree-0 vertices and
                                   first-neighbour hits with one coalesced load.  NULL = not used. */
    const uint32_t *isolated;   /* optional device bitmap, ceil(V/32) words: bit v set iff degree(v) == 0
                                   (coop_csr_isolated); direction-optimising BFS copies it into the
                                   visited bitmap at init instead of reading the row offsets.  NULL = not used. */
} coop_csr;

typedef struct {
    uint32_t max_wgs;           /* N: 0 = max co-resident for threads_per_wg */
    uint32_t init_wgs;          /* M0 in [1, N]: 0 = N */
    uint32_t threads_per_wg;    /* 0 = 512; supported: 128, 256, 512, 1024 */
    uint32_t barrier_mode;      /* coop_barrier_mode */
    uint32_t barriers_per_level;/* 1 (fused) or 2 (Fig. 4 exactly: RB; reset; level++; RB) */
    uint32_t policy;            /* coop_policy */
    const uint32_t *script;     /* host: SCRIPTED M' per resizing episode, 0 = unchanged */
    uint32_t script_len;
    uint32_t flags;             /* COOP_FLAG_* */
    uint64_t seed;              /* RANDOM policy */
    double resize_prob;         /* RANDOM policy */
    /* SCHEDULER policy: the competing non-cooperative task (synthetic, K11 of SURVEY) */
    uint32_t task_wgs;          /* Q: workgroups demanded per task instance, 1 <= Q <= N-1 */
    uint32_t task_blocks;       /* independent blocks per instance */
    uint64_t task_block_ns;     /* busy time of one block */
    uint64_t task_period_ns;    /* P: arrival period of task instances */
    uint64_t task_first_ns;     /* delay of the first arrival after kernel start */
    uint32_t task_max;          /* max instances per call (0 = unbounded) */
    uint64_t timeout_ns;        /* watchdog for every spin loop: 0 = 20 s */
    void *stream;               /* cudaStream_t (NULL = legacy default stream) */
    void *ev_kernel_start;      /* optional cudaEvent_t recorded on `stream` right before the persistent kernel */
    void *ev_kernel_end;        /* optional cudaEvent_t recorded on `stream` right after it (kernel-only timing) */
    uint32_t workspace;         /* scratch set on the device (0..7): concurrent calls on one device need distinct ones */
    uint32_t sssp_delta;        /* SSSP near-far band width (0 = plain worklist Bellman-Ford); results identical */
    uint32_t bfs_alpha;         /* COOP_FLAG_DIROPT: top-down -> bottom-up when m_f * alpha > m_u (0 = default) */
    uint32_t bfs_beta;          /* COOP_FLAG_DIROPT: bottom-up -> top-down when n_f * beta < V (0 = default) */
} coop_opts;

/* One competing-task instance, all times from %globaltimer (ns). */
typedef struct {
    uint64_t t_arrive;          /* scheduler posted the demand */
    uint64_t t_first_surrender; /* first demanded WG killed */
    uint64_t t_last_surrender;  /* demand fully satisfied (gather time = this - t_arrive) */
    uint64_t t_first_start;     /* first task block started (kill latency = this - t_arrive) */
    uint64_t t_end;             /* last task block finished */
    uint32_t demanded;          /* Q */
    uint32_t surrendered;       /* WGs killed for this instance */
} coop_task_event;

typedef struct {
    uint64_t kernel_ns;         /* %globaltimer, WG 0 from kernel entry to termination */
    uint64_t edges_scanned;     /* sum of degrees of expanded frontier entries */
    uint64_t frontier_total;    /* sum of frontier sizes */
    uint64_t reached;           /* vertices with a finite result */
    uint32_t levels;            /* non-empty frontiers (BFS depth+1 / SSSP rounds) */
    uint32_t episodes;          /* resizing barriers executed */
    uint32_t kills, forks;      /* workgroups killed / forked */
    uint32_t min_m, max_m;      /* range of M over the run */
    uint32_t n_wgs;             /* N launched */
    uint32_t threads_per_wg;
    uint32_t tasks_posted, tasks_completed;
    uint32_t bottom_up_levels;  /* COOP_FLAG_DIROPT: levels run bottom-up */
    uint32_t mid_kills;         /* workgroups that left inside an interval (offer_kill between items) */
    uint32_t handbacks;         /* of those, workgroups that handed static items back to the survivors */
    uint32_t replays;           /* replay intervals run (the survivors ran handed-back items) */
    uint32_t reserved0;
    uint32_t *m_trace;          /* optional caller-owned HOST buffer: M after each resizing episode */
    uint32_t m_trace_cap;
    uint32_t *level_sizes;      /* optional caller-owned HOST buffer: frontier size per level */
    uint32_t level_sizes_cap;
    uint64_t *level_end_ns;     /* optional caller-owned HOST buffer: %globaltimer when each level's
                                   expand finished (its first resizing barrier released), minus kernel start */
    uint32_t level_end_ns_cap;
    coop_task_event *task_events; /* optional caller-owned HOST buffer */
    uint32_t task_events_cap;
} coop_stats;

typedef struct {
    int device;
    int sm_count;
    int max_ctas_per_sm;        /* for threads_per_wg of the query */
    int max_coresident;         /* sm_count * max_ctas_per_sm */
    int regs_per_thread;
    size_t l2_bytes;
    size_t hbm_bytes;
} coop_device_info;

typedef struct {
    uint64_t iters;             /* resizing barriers executed */
    double ns_per_barrier;      /* cudaEvent time / iters */
    uint64_t kernel_ns;
    uint32_t kills, forks;
    uint32_t violations;        /* 0 unless an invariant failed (status is then COOP_ERR_INVARIANT) */
} coop_barrier_stats;

/* ---- library ---- */
int coop_abi_version(void);
const char *coop_status_string(coop_status s);
const char *coop_last_error(void);   /* thread-local description of the last failure */

/* Build the probe records of g (probe_out: device uint64[V], caller-owned) on `stream`
 * (cudaStream_t, NULL = legacy default) and wait for them.  A graph-layout step, done once per
 * graph like building the CSR; results of coop_bfs are identical with or without it. */
coop_status coop_csr_probe(const coop_csr *g, uint64_t *probe_out, void *stream);

/* Degree-zero bitmap of g (bits_out: device uint32[ceil(V/32)], caller-owned), once per graph. */
coop_status coop_csr_isolated(const coop_csr *g, uint32_t *bits_out, void *stream);

/* Hub-first neighbour order for BFS (graph-layout step, once per graph): writes g's neighbour
 * lists to col_out (device int32[E], caller-owned) with each list sorted by descending neighbour
 * degree, so bottom-up levels probe hubs first.  BFS results are identical for any neighbour order
 * (levels are unique); use col_out as col_idx (and build the probe records from it).  Not for SSSP
 * (weights are not permuted).  COOP_ERR_INVALID_ARG if E >= 2^31 (the segmented sort's limit). */
coop_status coop_csr_hub_first(const coop_csr *g, int32_t *col_out, void *stream);

/* Co-residency capacity of the BFS/SSSP kernel for threads_per_wg on `device`. */
coop_status coop_device_query(int device, uint32_t threads_per_wg, coop_device_info *out);

/*
 * Cooperative BFS (Fig. 4; bfs of Table 1).
 * levels_out: device int32[V]; on COOP_OK levels_out[v] = hop distance from
 * `source`, -1 if unreachable.  Bit-exact for every kill/fork schedule.
 */
coop_status coop_bfs(const coop_csr *g, int64_t source, int32_t *levels_out,
                     const coop_opts *opts, coop_stats *stats);

/*
 * Cooperative worklist SSSP (l-sssp of Table 1; reading R8 of DESIGN.md).
 * dist_out: device uint32[V]; on COOP_OK dist_out[v] = min path weight,
 * 0xFFFFFFFF if unreachable.  Needs g->weights.  COOP_ERR_OVERFLOW if
 * (V-1) * max_weight >= 2^32 - 1.
 */
coop_status coop_sssp(const coop_csr *g, int64_t source, uint32_t *dist_out,
                      const coop_opts *opts, coop_stats *stats);

/*
 * End-to-end variants: graph arrays and the output are HOST pointers.  The
 * call copies the CSR to the device, runs the cooperative kernel and copies
 * the result back (all inside the call; device memory is cached between calls).
 */
coop_status coop_bfs_host(int64_t num_vertices, const void *row_offsets, int32_t offset_bits,
                          const int32_t *col_idx, int64_t source, int32_t *levels_out,
                          const coop_opts *opts, coop_stats *stats);
coop_status coop_sssp_host(int64_t num_vertices, const void *row_offsets, int32_t offset_bits,
                           const int32_t *col_idx, const uint32_t *weights, uint32_t max_weight,
                           int64_t source, uint32_t *dist_out, const coop_opts *opts, coop_stats *stats);

/*
 * Resizing-barrier microbenchmark (BASELINE.json configs[3]): n_ctas CTAs of
 * `threads` threads execute `iters` resizing barriers; with probability
 * resize_prob per episode M' ~ U[1, n_ctas].  barrier_mode QUERY or PLAIN.
 * flags COOP_FLAG_CHECK adds the arrival-count, contiguity and
 * message-passing checks.
 */
coop_status coop_barrier_bench(uint32_t n_ctas, uint32_t threads, uint64_t iters, double resize_prob,
                               uint64_t seed, uint32_t barrier_mode, uint32_t flags,
                               coop_barrier_stats *out);

/*
 * L2 atomic round trip: one thread issues `iters` dependent atomicAdd on one
 * word; returns ns per atomic (the denominator for ns/barrier).
 */
coop_status coop_l2_atomic_rtt(uint64_t iters, double *ns_per_atomic);
/* The same measurement per kind and SM: one thread on each of 8 SMs spread over both
 * dies runs a dependent chain of `iters` operations on its own line; ns_out[kind*8 + k]
 * (kinds: 0 atom.relaxed.add.u64, 1 atom.relaxed.add.u32, 2 atom.acq_rel.add.u64,
 * 3 ld.acquire.u64).  coop_l2_atomic_rtt reports the median of kind 0 over the SMs:
 * the denominator of the barrier's ns / RTT ratio. */
coop_status coop_l2_latency_profile(uint64_t iters, double *ns_out);

/* Diagnostics: barrier phase breakdown of the last call on workspace 0 (only
 * filled by a library built with -DCOOP_TRACE=1; zeros otherwise): clock64
 * cycle sums for CTA 0 -- [0..5] as a waiter, [8..13] as the last arriver:
 * entry sync, arrival, wait for release, serial section + exit, interval, count. */
coop_status coop_debug_trace(uint64_t *out16);

typedef struct coop_handle coop_handle;

/* The competing task as a standalone non-cooperative kernel (K11):
 * `blocks` CTAs of `threads` threads, each busy for block_ns; asynchronous on
 * `stream` (cudaStream_t).  Used for the measured kernel-level preemption
 * comparison (T3), where the task runs between compute launches. */
coop_status coop_spin_task(uint32_t blocks, uint32_t threads, uint64_t block_ns, void *stream);

/* Asynchronous coop_bfs with any policy: returns after enqueueing the control-block
 * copy and the launch on opts->stream; finish with coop_wait (stats, status) and
 * coop_destroy.  Calls that are in flight together need distinct opts->workspace
 * values (the scratch of a workspace belongs to one call until it is waited). */
coop_status coop_bfs_launch(const coop_csr *g, int64_t source, int32_t *levels_out, const coop_opts *opts,
                            coop_handle **handle);

/* BFS looped over sources inside ONE persistent launch -- the paper's multitasking
 * workload runs the cooperative kernel continuously while tasks arrive (P:1045,
 * P:1135-1255).  Run r traverses from sources[r % n_sources] (device int64 array);
 * a new run starts while less than loop_ns has elapsed since the kernel started
 * (each restart is a resizing barrier, so the scheduler can resize there too).
 * levels_out (device int32[V]) holds the LAST run's levels; *runs_out = runs done;
 * run_end_ns (host, optional, run_cap entries) = end of each run, ns after the
 * kernel start.  stats->reached/edges_scanned sum over all runs; the per-level
 * statistics are the last run's.  Default watchdog: loop_ns + 20 s. */
coop_status coop_bfs_loop(const coop_csr *g, const int64_t *sources, uint32_t n_sources, uint64_t loop_ns,
                          int32_t *levels_out, uint64_t *run_end_ns, uint32_t run_cap, uint32_t *runs_out,
                          const coop_opts *opts, coop_stats *stats);

/* ---- 1-D vertex-partitioned BFS across the GPUs of one node (BASELINE.json configs[4]) ----
 * Not in the paper (single iGPU).  One call per rank; every rank runs the
 * cooperative BFS kernel over its partition and the per-level frontier is
 * all-gathered INSIDE the kernel: each rank stores its slice of the next
 * frontier bitmap into every peer's copy (NVLink peer memory) and the
 * resizing barrier's serial section doubles as the cross-GPU barrier
 * (release/acquire flags at system scope).  Pointers to peer buffers come
 * from coop_ipc_* (or are plain device pointers when all ranks share a GPU). */
#define COOP_MAX_RANKS 8
typedef struct {
    int64_t num_vertices;       /* global V */
    int64_t v_begin, v_end;     /* owned vertices [v_begin, v_end); v_begin % 32 == 0 (or == V for an empty rank) */
    int32_t rank, nranks;       /* 1 <= nranks <= COOP_MAX_RANKS */
    uint32_t seq;               /* call sequence number: identical on all ranks, new for every call */
    const void *row_offsets;    /* device, V+1 offsets of the local edges (destination owned), by global source */
    int32_t offset_bits;        /* 32 or 64 */
    const int32_t *col_local;   /* device, destination - v_begin */
    int64_t num_edges;          /* local edges */
    const uint32_t *hub_ids;    /* device, ascending vertices with local degree >= hub_degree (NULL if none) */
    const uint64_t *hub_prefix; /* device, num_hubs + 1 prefix sums of the hubs' local degrees */
    uint32_t num_hubs, hub_degree;
    uint32_t *frontier[COOP_MAX_RANKS][2]; /* rank q's two frontier bitmaps, ceil(V/32) words each, device-visible */
    uint64_t *flags[COOP_MAX_RANKS];       /* rank q's flag block, 4*COOP_MAX_RANKS uint64, zeroed once when allocated */
    /* COOP_FLAG_DIROPT (bottom-up levels; symmetric graph only): */
    const void *rows_offsets;   /* device, v_end - v_begin + 1 offsets of the OWNED rows (offset_bits wide) */
    const int32_t *rows_col;    /* device, their neighbours (global ids) */
    int64_t num_edges_global;   /* directed edges of the whole graph */
} coop_part;

/* Blocking partitioned BFS of this rank.  levels_owned_out: device int32[v_end - v_begin];
 * on COOP_OK entry i = hop distance of vertex v_begin + i, -1 if unreachable. */
coop_status coop_bfs_part(const coop_part *part, int64_t source, int32_t *levels_owned_out,
                          const coop_opts *opts, coop_stats *stats);
/* Partitioned SSSP ("(vertex, dist) exchange"): the same 1-D layout
 * with weights_local (device uint32[num_edges], aligned with col_local); the
 * frontier is exchanged as (vertex, distance) pairs: part->frontier[q][0..1] are
 * rank q's two inboxes of uint64[num_vertices] (pairs of source rank r at offset
 * v_begin(r)); slices must be graphgen.part_bounds' uniform ones.  Per round:
 * relax the local edges of every rank's pairs (64-bit atomicMin on
 * {dist | round mark}, reading R8), store the owned improved vertices with their
 * final round distance into every rank's inbox, cross-GPU barrier in the second
 * resizing barrier's serial section (counts; 0 = done).  dist_owned_out: device
 * uint32[v_end - v_begin], 0xFFFFFFFF unreachable.  Blocking / asynchronous. */
coop_status coop_sssp_part(const coop_part *part, const uint32_t *weights_local, int64_t source,
                           uint32_t *dist_owned_out, const coop_opts *opts, coop_stats *stats);
coop_status coop_sssp_part_launch(const coop_part *part, const uint32_t *weights_local, int64_t source,
                                  uint32_t *dist_owned_out, const coop_opts *opts, coop_handle **handle);
/* Asynchronous variant (finish with coop_wait); several ranks may share one GPU
 * when each uses its own opts->workspace and stream. */
coop_status coop_bfs_part_launch(const coop_part *part, int64_t source, int32_t *levels_owned_out,
                                 const coop_opts *opts, coop_handle **handle);
/* North_star's NCCL data plane: the same persistent
 * cooperative kernel per rank, with the per-level frontier exchanged by
 * ncclAllGather over NVLink/NVSwitch on a comm stream instead of in-kernel peer
 * stores.  Per level L the comm stream runs cuStreamWaitValue32(ready >= L+1)
 * (released by the kernel's first resizing barrier), an in-place ncclAllGather
 * of this rank's bitmap slice plus its counts, and cuStreamWriteValue32
 * (gathered = L+1), which the second resizing barrier waits for; termination is
 * the gathered global count == 0 on every rank (no extra reduce).
 *   Layout: slices are uniform -- with sw = ceil(ceil(V/32) / nranks) words,
 *   rank q owns [32*sw*q, min(V, 32*sw*(q+1))) (graphgen.part_bounds);
 *   part->frontier[rank][0..1] are THIS rank's two bitmaps of nranks*sw words
 *   (device, zeroed once); the other frontier / flags entries are unused.
 *   nccl_comm: an ncclComm_t of nranks ranks (this rank = part->rank), from
 *   coop_nccl_comm_init or torch's ProcessGroupNCCL; every rank calls with the
 *   same source.  The default grid leaves 16 CTA slots free for NCCL's kernels.
 * Blocking; returns COOP_ERR_NCCL if NCCL or the stream memory operations are
 * unavailable or a collective fails. */
coop_status coop_bfs_part_nccl(const coop_part *part, int64_t source, int32_t *levels_owned_out,
                               void *nccl_comm, const coop_opts *opts, coop_stats *stats);
/* NCCL communicator helpers (the unique id is broadcast by the caller, e.g. over
 * torch.distributed): 128-byte ncclUniqueId; comm is an ncclComm_t. */
coop_status coop_nccl_get_unique_id(void *uid128);
coop_status coop_nccl_comm_init(int32_t nranks, const void *uid128, int32_t rank, void **comm);
coop_status coop_nccl_comm_destroy(void *comm);

/* Exchange buffers: cudaMalloc'd (so they can be shared by IPC) and zeroed; and
 * CUDA IPC helpers for the peer frontier buffers (64-byte opaque handles). */
coop_status coop_exchange_alloc(uint64_t bytes, void **dptr);
coop_status coop_exchange_free(void *dptr);
coop_status coop_ipc_get_handle(const void *dptr, void *handle64);
coop_status coop_ipc_open(const void *handle64, void **dptr);
coop_status coop_ipc_close(void *dptr);

/* ---- asynchronous handle API (host <-> GPU channel) ---- */
/* Launch cooperative BFS (kind 0) or SSSP (kind 1) asynchronously; opts->policy
 * must be COOP_POLICY_SCHEDULER.  Resource messages and tasks then come from the
 * host through a host-mapped mailbox polled by the scheduler CTA (the paper's
 * SVM channel) in addition to the periodic generator (task_period_ns
 * = 0 disables it). `out` is levels (int32*) or dist (uint32*), device. */
coop_status coop_launch(int kind, const coop_csr *g, int64_t source, void *out,
                        const coop_opts *opts, coop_handle **handle);
/* Post one task instance of task_wgs WGs (validated: 1 <= task_wgs <= N-1 else NO_CAPACITY). */
coop_status coop_submit_task(coop_handle *h, uint32_t task_wgs, uint32_t task_blocks,
                             uint64_t task_block_ns, uint64_t *task_id);
coop_status coop_demand(coop_handle *h, uint32_t kills);   /* resource message: surrender `kills` WGs */
coop_status coop_grant(coop_handle *h, uint32_t forks);    /* resource message: fork up to `forks` WGs */
coop_status coop_query(coop_handle *h, uint32_t *W);       /* outstanding demand (query) */
coop_status coop_current_m(coop_handle *h, uint32_t *M);   /* active workgroups right now */
coop_status coop_wait(coop_handle *h, coop_stats *stats);  /* wait for termination, fill stats */
void coop_destroy(coop_handle *h);


/* ---- user cooperative kernels: host half of the device API in coop_device.cuh ----
 * A kernel written against coop_device.cuh (offer_kill P:529-550, request_fork
 * P:553-592, global_barrier P:600-610, resizing_global_barrier P:612-638)
 * takes a `coop_dev *` control block.  The host creates a handle once
 * (coop_dev_create), re-arms the block before each launch (coop_dev_arm: N
 * CTAs, M0 active, the others parked in the pool), launches (coop_dev_launch in
 * coop_device.cuh, or a library app below) and reads the outcome
 * (coop_dev_collect).  coop_dev_demand / coop_dev_grant post resource messages
 * and may be called from another host thread while the kernel runs
 * (policy COOP_POLICY_SCHEDULER). */
typedef struct coop_dev coop_dev;                 /* device control block (layout in coop_device.cuh) */
typedef struct coop_dev_handle coop_dev_handle;

typedef struct {
    uint32_t max_wgs;           /* cap on N (0 = the kernel's co-resident capacity) */
    uint32_t init_wgs;          /* M0 in [1, N] (0 = N) */
    uint32_t policy;            /* coop_policy (SCHEDULER = host resource messages) */
    uint32_t flags;             /* COOP_FLAG_CHECK: arrival-count / contiguity checks at every barrier */
    uint64_t seed;              /* RANDOM */
    double resize_prob;         /* RANDOM: per resizing barrier, M' ~ U[1, N] */
    double kill_prob;           /* RANDOM: per bare offer_kill call (accepted only for id M-1 > 0) */
    double fork_prob;           /* RANDOM: per bare request_fork call, k ~ U[1, max_fork] */
    uint32_t max_fork;          /* RANDOM: 0 = 4, at most 32 */
    const uint32_t *script;     /* host, SCRIPTED: M' per resizing episode (0 = unchanged) */
    uint32_t script_len;
    uint32_t m_trace_cap;       /* M' of the first m_trace_cap resizing episodes (read by coop_dev_collect) */
    uint64_t timeout_ns;        /* watchdog for every spin (0 = 20 s) */
} coop_dev_opts;

typedef struct {
    uint64_t kernel_ns;         /* %globaltimer from CTA 0's start to the first finishing CTA */
    uint32_t n_wgs;             /* N launched */
    uint32_t kills, forks;      /* workgroups killed / forked (bare calls and barriers) */
    uint32_t episodes;          /* resizing barriers */
    uint32_t barriers;          /* all barriers */
    uint32_t offers;            /* bare offer_kill calls */
    uint32_t fork_calls;        /* bare request_fork calls */
    uint32_t min_m, max_m;      /* range of M */
    uint32_t final_m;           /* M at termination */
    uint32_t violations;        /* COOP_FLAG_CHECK failures (status is then COOP_ERR_INVARIANT) */
    uint32_t *m_trace;          /* optional caller-owned HOST buffer: M' per resizing episode */
    uint32_t m_trace_cap;
} coop_dev_stats;

coop_status coop_dev_create(const coop_dev_opts *opts, coop_dev_handle **handle);
/* Reset the control block for a launch of n_wgs CTAs (enqueued on `stream`);
 * *dev_out is the kernel argument.  COOP_ERR_INVALID_ARG if n_wgs is 0 or
 * exceeds COOP_DEV_MAX_CTAS, or init_wgs > n_wgs. */
coop_status coop_dev_arm(coop_dev_handle *h, uint32_t n_wgs, void *stream, coop_dev **dev_out);
coop_status coop_dev_demand(coop_dev_handle *h, uint32_t kills);   /* surrender `kills` WGs (query/offer_kill) */
coop_status coop_dev_grant(coop_dev_handle *h, uint32_t forks);    /* fork up to `forks` WGs */
/* Synchronise `stream`, read the control block, map its error word:
 * timeout -> COOP_ERR_TIMEOUT, invariant -> COOP_ERR_INVARIANT, overflow -> COOP_ERR_OVERFLOW. */
coop_status coop_dev_collect(coop_dev_handle *h, void *stream, coop_dev_stats *stats);
void coop_dev_destroy(coop_dev_handle *h);

/* The Pannotia applications of Table 1 as cooperative kernels on the
 * device API, with Table 1's resizing-barrier counts (color 2/2, mis 3/3, p-sssp
 * 3/3); vertex-strided loops re-chunked after every resizing barrier; the
 * iteration counter is the transmitted state.  Algorithms (R23):
 *   coop_color  Jones-Plassmann colouring with priorities (splitmix64(seed ^ v), v):
 *               colors_out[v] = iteration in which v became the highest-priority
 *               uncoloured vertex of its neighbourhood;
 *   coop_mis    Luby's maximal independent set with the same priorities (lowest
 *               undecided joins): state_out[v] = 1 in the set, 2 not;
 *   coop_psssp  Bellman-Ford over all vertices each iteration (pull form):
 *               dist_out[v] (u32, 0xFFFFFFFF unreachable).
 * 32-bit offsets, symmetric graph; device output buffers int32/uint32[V];
 * *iters_out = iterations executed.  Blocking; errors as coop_fig4_bfs. */
coop_status coop_color(coop_dev_handle *h, const coop_csr *g, uint64_t seed, int32_t *colors_out, uint32_t threads,
                       uint32_t *iters_out, coop_dev_stats *stats);
coop_status coop_mis(coop_dev_handle *h, const coop_csr *g, uint64_t seed, int32_t *state_out, uint32_t threads,
                     uint32_t *iters_out, coop_dev_stats *stats);
coop_status coop_psssp(coop_dev_handle *h, const coop_csr *g, int64_t source, uint32_t *dist_out, uint32_t threads,
                       uint32_t *iters_out, coop_dev_stats *stats);

/* Fig. 4 exactly, written on the device API: thread-strided
 * frontier with tid/stride recomputed after every resizing barrier, claims by
 * CAS on the level array, two resizing barriers per level transmitting
 * {level, in_nodes/out_nodes}.  32-bit offsets.  levels_out: device
 * int32[V], -1 unreachable.  Blocking. */
coop_status coop_fig4_bfs(coop_dev_handle *h, const coop_csr *g, int64_t source, int32_t *levels_out,
                          uint32_t threads_per_wg, coop_dev_stats *stats);

/* Cooperative work stealing (Fig. 2, adapted per §3.2):
 * per-workgroup task queues guarded by CAS mutexes, offer_kill and
 * request_fork at the head of the main loop, queue id read after the fork
 * point.  The task set is the seeded implicit tree of DESIGN.md reading R19. */
typedef struct {
    uint64_t seed;              /* root task id */
    uint32_t depth;             /* D <= 62 */
    uint32_t max_fanout;        /* B */
    uint32_t fixed;             /* 1: every inner task has exactly B children */
    uint32_t rounds;            /* R: splitmix64 rounds per lane of work */
    uint32_t queue_cap;         /* entries per queue, power of two (0 = 1024) */
} coop_ws_tree;
typedef struct {
    uint64_t count;             /* tasks processed */
    uint64_t total;             /* sum of task values mod 2^64 */
    uint64_t hist[64];          /* tasks per depth */
    uint64_t steals;            /* tasks taken from another workgroup's queue */
} coop_ws_result;
coop_status coop_work_steal(coop_dev_handle *h, const coop_ws_tree *tree, uint32_t threads_per_wg,
                            coop_ws_result *result, coop_dev_stats *stats);

#ifdef __cplusplus
}
#endif
#endif /* COOP_H */
