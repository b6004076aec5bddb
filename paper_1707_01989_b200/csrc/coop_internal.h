// coop_internal.h -- layouts shared by the host side (coop_api.cu) and the
// device runtime (coop_rt.cuh).  Not part of the public ABI.
#pragma once
#include <stdint.h>

namespace coop {

constexpr uint32_t kMaxCtas = 4096;                  // physical CTA slots (pool bitmap size)
constexpr uint32_t kPoolWords = kMaxCtas / 32;
constexpr uint32_t kHeavyDeg = 256;                  // BFS: frontier entries with deg >= this are edge-balanced
constexpr uint64_t kMask40 = (1ull << 40) - 1;

// runtime actions broadcast inside a CTA
enum : uint32_t { ACT_CONT = 0, ACT_KILLED = 1, ACT_DONE = 2, ACT_ABORT = 3, ACT_RUN_BODY = 4,
                  ACT_RUN_TASK = 5, ACT_EXIT = 6, ACT_IDLE = 7,
                  ACT_STOP = 8 };   // DIST_MID: asked to surrender mid-interval (counters flushed)
// body entry points (the paper's "designated point within the kernel")
// ENTRY_RESTART: the resizing barrier after a new run's init (BFS source loop); a CTA
// forked there starts at the loop head like ENTRY_AFTER_RB2
enum : uint32_t { ENTRY_START = 0, ENTRY_AFTER_RB1 = 1, ENTRY_AFTER_RB2 = 2, ENTRY_RESTART = 3 };
// error codes written to Ctl::err (host maps to coop_status)
enum : uint32_t { DERR_NONE = 0, DERR_TIMEOUT = 1, DERR_INVARIANT = 2, DERR_OVERFLOW = 3 };
enum : uint32_t { APP_BFS = 0, APP_SSSP = 1, APP_BARRIER = 2, APP_PBFS = 3, APP_PSSSP = 4 };
constexpr int kMaxRanks = 8;                         // partitioned BFS: GPUs of one NVSwitch node
// BFS level modes (direction optimisation): top-down over the frontier queue,
// top-down over the frontier bitmap (after a bottom-up level), bottom-up
enum : uint32_t { BFS_TDQ = 0, BFS_TDB = 1, BFS_BU = 2 };

// Transmit struct: the transmit-annotated state of Fig. 4 (level, in_nodes,
// out_nodes) plus what a forked CTA needs to join (reading R7).
struct Transmit {
    uint32_t level;
    uint32_t in_sel;
    uint32_t gen;      // barrier generation the forked CTA joins
    uint32_t M;        // active count after the episode
    uint32_t lid;      // logical id assigned to the forked CTA
    uint32_t entry;    // ENTRY_AFTER_RB1 / ENTRY_AFTER_RB2
    uint32_t pad[2];
};

struct __align__(64) Mailbox {
    uint32_t flag;     // generation of the last assignment (0 = never)
    uint32_t pad0[7];
    Transmit tx;
};

struct LightEntry { uint32_t beg; uint32_t deg; };                 // BFS frontier entry, 32-bit offsets
struct LightEntry64 { uint64_t beg; uint32_t deg; uint32_t pad; };  // 64-bit offsets
struct HeavyEntry { uint64_t beg; uint64_t prefix; uint32_t deg; uint32_t pad; };

struct TaskEventDev {
    unsigned long long t_arrive, t_first_surrender, t_last_surrender, t_first_start, t_end;
    uint32_t demanded, surrendered;
};

// Control block in device memory.  Hot words sit on their own 128-B lines.
constexpr uint32_t kClaimShards = 8;

struct __align__(128) Ctl {
    unsigned long long W;              // barrier word {gen:32 | M:16 | arrived:16} (arrivals)
    unsigned long long pad_w[15];
    unsigned long long R;              // release word {gen:32 | M':16 | 0} (waiters poll it)
    unsigned long long pad_r[15];
    // line: scheduler channel (resource messages)
    uint32_t demand;                   // WGs the scheduler wants back (query() = min(demand, M-1))
    uint32_t grant;                    // WGs the scheduler offers at the next fork point
    uint32_t pad_c[30];
    // line: frontier counters
    uint32_t qsize[2];                 // light queue sizes (in/out selected by the transmitted in_sel)
    unsigned long long heavy[2];       // packed {count:24 | edges:40}
    uint32_t pad_q[26];
    // line: status
    uint32_t done;                     // set by WG 0 at termination (parked CTAs and scheduler exit)
    uint32_t err;                      // DERR_*
    uint32_t episode;                  // resizing episodes executed
    uint32_t cur_task;                 // index of the task instance in flight (+1), 0 = none
    uint32_t pad_s[28];
    // line: transmit published by WG 0 before each arrival
    Transmit tx0;
    uint32_t pad_t[24];
    // task (competing non-cooperative kernel, megakernel worker pool P:817-826)
    uint32_t task_next;                // next block to claim
    uint32_t task_total;               // blocks of the instance in flight
    uint32_t task_done;                // blocks finished
    uint32_t task_wgs;                 // Q of the instance in flight
    unsigned long long task_block_ns;
    uint32_t pad_k[26];
    // stats (atomics at CTA exit / in serial sections)
    unsigned long long edges_scanned, frontier_total, reached, t_start, t_end;
    uint32_t kills, forks, levels, min_m, max_m, tasks_posted, tasks_completed, n_events;
    // invariant checks (COOP_FLAG_CHECK)
    uint32_t chk_arr[2];
    uint32_t violations;
    uint32_t mhist[8];                 // M' of generation g (index g & 7), written before the release of W
    uint32_t pad_x[5];
    uint32_t idmap[2][kPoolWords];
    // idle-and-forkable physical CTAs (the scheduler context's "available" set)
    uint32_t pool[kPoolWords];
    // host-mapped channel mirror: last host sequence numbers consumed
    uint32_t host_seq_seen;
    uint32_t pad_h[31];
    // BFS frontier accounting per level parity (next frontier of the level being expanded)
    uint32_t chunk[2];                 // dynamic work distribution: next chunk per level parity
    uint32_t mid_kills;                // workgroups that left at a chunk boundary (mid-interval offer_kill)
    uint32_t pad_m;
    unsigned long long nf[2];          // vertices discovered
    unsigned long long mf[2];          // sum of their degrees
    unsigned long long vis_edges;      // sum of degrees of every vertex discovered so far
    uint32_t bmode[2];                 // BFS_* mode of the level that reads parity p
    uint32_t n_bu_levels;              // statistics: bottom-up levels executed
    uint32_t pad_b[19];
    // partitioned BFS
    unsigned long long pcount[2];      // owned vertices discovered per level parity (this rank)
    unsigned long long gcount;         // vertices in the global frontier of the current level (all ranks)
    unsigned long long xwait_ns;       // time spent in the cross-GPU flag exchange
    unsigned long long pmf[2];         // sum of the degrees of the owned vertices discovered (per parity)
    uint32_t pmode;                    // BFS_TDB / BFS_BU of the next level (identical on every rank)
    uint32_t pad_p[24];
    // SSSP near-far
    unsigned long long T;              // near threshold
    unsigned long long T_lo;           // previous threshold (far entries below it are stale)
    uint32_t smode[2];                 // SSSP_* mode of the interval reading parity p
    uint32_t far_size[2];              // far pile sizes
    uint32_t far_sel;                  // far pile holding the live entries
    uint32_t far_min;                  // min distance among kept far entries (drain)
    uint32_t pad_f[24];
    unsigned long long trace[16];      // COOP_TRACE barrier breakdown (CTA 0, clock64 cycles)
    unsigned long long trace_last;
    // BFS looped over sources inside one launch (coop_bfs_loop)
    uint32_t run;                      // runs completed
    uint32_t pad_l[31];
    // partitioned SSSP: pairs per source rank in this round's inbox; own list lengths per parity
    unsigned long long qcnt[kMaxRanks];
    uint32_t list_n[2];
    uint32_t exits;                    // CTAs that left the kernel (the last one mirrors this block to the host)
    uint32_t pad_ps[13];
    // claim counters per level parity (dynamic tails of the top-down levels), one 128-B line each
    uint32_t claim[2][kClaimShards][32];
    // hand-back of a mid-interval offer_kill (SCHEDULER + query): a CTA that leaves inside an
    // interval hands the rest of its static share back; the serial section turns the handed-back
    // items into a replay interval run by the survivors before the level ends
    unsigned long long don;            // {donors:20 | items:44} handed back in the current interval
    unsigned long long rep;            // `don` of the replay interval being run
    unsigned long long rep_tw;         // warp stride M*W of the interval the items come from
    uint32_t handbacks, replays;       // statistics
    uint32_t pad_hb[26];
};

// one warp's handed-back static items: start, start + tw, ... (count of them), at flat
// offset `prefix` of the replay interval; kRepVoid in start = withdrawn (the kill-CAS failed)
struct RepEntry { uint64_t start; uint64_t prefix; uint32_t count; uint32_t pad; };
constexpr uint64_t kRepVoid = 1ull << 63;
constexpr uint64_t kMask44 = (1ull << 44) - 1;

// Partitioned BFS (1-D vertex partition).  Frontier bitmaps and
// flag blocks of every rank are device-visible here (own memory, or peer
// memory mapped through CUDA IPC over NVLink).
struct PartParams {
    int64_t vb, ve;                    // owned vertices [vb, ve), vb % 32 == 0
    int32_t rank, nranks;
    uint32_t seq;                      // call sequence number, identical on every rank
    uint32_t nhub;                     // static hubs (local degree >= hub_deg)
    uint32_t hub_deg;
    const uint32_t *hub_ids;
    const unsigned long long *hub_prefix;        // nhub + 1 local-edge prefix over the hubs
    uint32_t *F[kMaxRanks][2];         // F[q][b]: rank q's copy of global frontier bitmap b
    unsigned long long *flags[kMaxRanks];        // rank q's flag block [kMaxRanks][2 parity][2 words]
    const void *rro;                   // direction optimisation: owned rows (v_end - v_begin + 1 offsets)
    const int32_t *rcol;               //   their neighbours (global ids)
    int64_t E_global;                  //   directed edges of the whole graph (Beamer's m_u)
    // NCCL data plane (coop_bfs_part_nccl, north_star's per-level all-gather): F[rank][b]
    // is this rank's full bitmap, its own slice is all-gathered in place by ncclAllGather
    // on a comm stream that waits for `ready` and signals `gathered` (stream memory ops)
    uint32_t nccl;
    uint32_t *ready;                   // RB1 of level L: ready = L + 1 (BIG at termination)
    const uint32_t *gathered;          // written by the comm stream after gather L: L + 1
    unsigned long long *cnt_send;      // [2][4] {discovered, m_f, source degree, 0} per parity
    const unsigned long long *cnt_recv;            // [2][nranks][4], all-gathered with the slice
    volatile uint32_t *host_ready;     // host-mapped mirror of `ready` (the host enqueues ahead)
    uint64_t slice_words;              // words per rank slice (uniform: v_begin == rank * 32 * slice_words)
    // partitioned SSSP (part_sssp.cuh): F[q][b] are rank q's inboxes of (vertex, dist) pairs
    // (u64[V]), source rank r's pairs at offset qvb[r]; list[b] = own improved vertices
    int64_t qvb[kMaxRanks + 1];
    uint32_t *list[2];
};

// Host -> GPU packet channel (host-mapped pinned memory; the paper's SVM atomics).
struct HostChannel {
    volatile uint32_t seq;             // incremented by the host for every packet
    volatile uint32_t kind;            // 1 = task, 2 = demand, 3 = grant
    volatile uint32_t a, b;            // task: wgs, blocks; demand/grant: count
    volatile unsigned long long c;     // task: block ns
    volatile uint32_t ack;             // scheduler CTA: last seq consumed
    volatile uint32_t cur_m;           // scheduler CTA mirrors W.M for coop_current_m
    volatile uint32_t demand_mirror;
    volatile uint32_t done_mirror;
};

struct KParams {
    // graph (immutable kernel parameters)
    int64_t V;
    const void *ro;
    int off64;
    const int32_t *col;
    const uint32_t *w;
    const unsigned long long *probe;   // optional per-vertex {degree:32 | first neighbour:32} (coop_csr.probe)
    const uint32_t *iso;               // optional degree-zero bitmap (coop_csr.isolated)
    int64_t source;
    // outputs
    int32_t *level_out;
    uint8_t *lv8;               // BFS: level + 1 per vertex during the traversal (apps.cuh store_level)
    uint32_t *dist_out;
    // scratch
    Ctl *ctl;
    Mailbox *mb;
    uint32_t *visited;          // BFS bitmap [ceil(V/32)]
    uint32_t *qlev;             // (unused by the current SSSP)
    unsigned long long *dq;     // SSSP keys {dist:32 | ~round:32} [V]
    void *qlight[2];            // BFS light entries / SSSP vertex ids
    HeavyEntry *qheavy[2];
    uint32_t *stamp;            // barrier bench message passing [kMaxCtas]
    uint32_t *fbits[3];         // BFS direction optimisation: frontier bitmaps of levels L, L+1, L+2 (mod 3)
    uint32_t *far[2];           // SSSP near-far: far piles
    uint32_t delta;             // SSSP near-far band width (0 = plain worklist Bellman-Ford)
    uint32_t far_cap;           // entries per far pile
    uint32_t *m_trace; uint32_t m_trace_cap;
    uint32_t *level_sizes; uint32_t level_cap;
    unsigned long long *level_t;  // globaltimer at the end of each level's expand (RB1 serial section)
    TaskEventDev *events; uint32_t events_cap;
    const uint32_t *script; uint32_t script_len;
    HostChannel *host;          // host-mapped channel or nullptr
    // configuration
    uint32_t app;
    uint32_t P;                 // physical worker CTAs (N)
    uint32_t M0;
    uint32_t policy;
    uint32_t barrier_mode;
    uint32_t bpl;               // barriers per level (1 or 2)
    uint32_t flags;
    uint32_t has_sched;         // 1: CTA P is the scheduler CTA
    uint64_t seed;
    uint32_t resize_thresh;     // resize_prob * 2^32
    uint64_t timeout_ns;
    uint64_t iters;             // barrier bench
    int64_t E;                  // directed edges
    uint32_t dopt;              // BFS: direction-optimising (COOP_FLAG_DIROPT)
    PartParams part;            // APP_PBFS
    uint32_t alpha, beta;       // Beamer's switch thresholds (m_f > m_u/alpha -> BU; n_f < V/beta -> TD)
    // BFS looped over sources inside one launch (coop_bfs_loop): run r uses
    // sources[r % n_src]; a new run starts while globaltimer - t_start < loop_ns
    const int64_t *sources; uint32_t n_src;
    uint64_t loop_ns;
    unsigned long long *run_t; uint32_t run_cap;   // globaltimer at the end of each run
    // host-mapped copy of the control block, written by the last CTA to leave the kernel
    // (the call's status and statistics reach the host without a copy-back operation)
    Ctl *ctl_mirror;
    RepEntry *rep;              // hand-back entries [P][W] (W = warps per CTA)
    // periodic task generator
    uint32_t task_wgs, task_blocks, task_max;
    uint64_t task_block_ns, task_period_ns, task_first_ns;
};

__host__ __device__ inline unsigned long long pack_w(uint32_t gen, uint32_t M, uint32_t arrived) {
    return ((unsigned long long)gen << 32) | ((unsigned long long)(M & 0xFFFF) << 16) | (arrived & 0xFFFF);
}

}  // namespace coop
