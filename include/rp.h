/*
 * rp.h — C ABI of librp, a B200-native Partial All-Reduce (P-Reduce) library.
 *
 * Method: Ripples, "Heterogeneity-Aware Asynchronous Decentralized Training"
 * (arXiv 1909.08029). Citations "P:<line>" are lines of its LaTeX source
 * (PAPER.md); sections: §3 P-Reduce, §4 Group Generation,
 * §5 Smart GG, §6 Implementation.
 *
 * What one training iteration of worker i does (alg1):
 *   Step 2  x_i <- x_i - eta * grad_i                       -> rp_step
 *   Step 3  get a group G containing i                        -> rp_schedule_static[_worker]
 *                                                                or rp_group_generate
 *   Step 4  atomically x_g <- (1/|G|) sum_{g in G} x_g         -> rp_preduce (collective)
 *           and continue once *its own* group is done          -> rp_barrier_free_wait
 * Steps 2 and 4 run fused in one pass of a CUDA kernel: y_m = x_m - eta*g_m is
 * never written to memory; the mean of the members' y is written to every
 * member replica in place.
 *
 * Conventions
 *   - Every function returns int status: RP_OK (0) or a negative RP_E* code.
 *     No C++ exception or abort crosses this boundary. rp_last_error() gives
 *     a thread-local message for the last failing call on the calling thread.
 *   - Device pointers (x, g, grad) are BORROWED: the caller (e.g. a torch
 *     tensor) owns them and keeps them alive until rp_finalize. They must be
 *     16-byte aligned fp32 arrays of n_params elements on the worker's GPU.
 *   - The context, its CUDA streams, events and peer mappings are owned by the
 *     library and released by rp_finalize.
 *   - Calls for distinct workers may come from different host threads; the
 *     Group Generator is serialized internally ("generates groups in a serial
 *     manner").
 *   - Worker placement (reading R6): worker w lives on GPU w / workers_per_gpu.
 *     One process drives one GPU (rank = GPU index); that process binds and
 *     drives exactly the workers of its GPU (RP_FLAG_EMULATE: every virtual
 *     GPU's workers, one device).
 *   - One device model per process: kernel attributes, occupancy and the SM
 *     count are cached per process at first use, and the intra-GPU kernel's
 *     tile-counter ring is per device; a process may hold several contexts, on
 *     one or several identical B200s, but not on GPUs of different kinds.
 *   - rp_init loads every kernel instantiation of the library up front (CUDA
 *     lazy loading would otherwise load a kernel at its first launch, which a
 *     random schedule may first reach inside a timed region).
 */
#ifndef RP_H
#define RP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RP_ABI_VERSION 1
#define RP_MAX_WORLD 64 /* lock vector is one uint64_t, one bit per worker */
#define RP_MAX_GROUP 16 /* largest group a P-Reduce accepts */
#define RP_MAX_GPUS 8   /* GPUs of one NVSwitch node */
#define RP_MAX_LOCAL 16 /* workers per GPU in a multi-GPU job */
#define RP_IPC_HANDLE_BYTES 64

/* ---- status codes ---------------------------------------------------------- */
#define RP_OK 0
#define RP_EINVAL (-1)    /* bad argument (range, alignment, device)                    */
#define RP_ESTATE (-2)    /* call not valid in the worker's current state               */
#define RP_EPROTO (-3)    /* collective contract broken: members disagree on the group,
                             or the group is not the one the GG handed out      */
#define RP_ECONFLICT (-4) /* a member already holds an unfinished group: atomicity
                             violation. Never happens under GD / static.    */
#define RP_ETIMEOUT (-5)  /* wait timed out; rp_last_error() names missing members      */
#define RP_ECUDA (-6)     /* CUDA runtime error (message in rp_last_error)              */
#define RP_ENOMEM (-7)
#define RP_ENODEV (-8)    /* operation needs a GPU but the context is host-only         */
#define RP_EAGAIN (-9)    /* random GG: the worker's group waits in the pending queue
                             (P:728-733); call rp_group_generate again                  */

/* ---- configuration ----------------------------------------------------------- */
#define RP_FLAG_TRACE 0x1       /* keep the JSONL decision trace (rp_trace_open)       */
#define RP_FLAG_TIMING 0x2      /* bracket every kernel launch with CUDA timing events
                                   on its own stream (rp_timing_read)                   */
#define RP_FLAG_SHARED_GG 0x4   /* multi-process asynchronous runs: ONE Group Generator
                                   in POSIX shared memory "/rp_gg_<job_id>" (created by
                                   rank 0, mapped by the others), serialized by a
                                   process-shared mutex; cross-GPU groups may then be
                                   issued outside batches (launched in GG order)       */
#define RP_FLAG_RANDOM_GG 0x8   /* the basic GG of §4.1 instead of GB + GD:
                                   a random group containing the requester, the lock
                                   vector, a FIFO pending queue; k = 2 is AD-PSGD       */
#define RP_FLAG_INTER_INTRA 0x10 /* §5.2 Inter-Intra Synchronization: every Global
                                   Division queues an Inter group (Head Workers across
                                   nodes, the rest node-local) and an Intra group (whole
                                   node); nodes = cfg.nodes, or n_gpus when 0           */
#define RP_FLAG_GRAPH 0x40      /* rp_lockstep_run with a static rule on one GPU: capture one
                                   schedule period (lcm(4 or k, section length) steps) into
                                   a CUDA graph once and replay it (launch-bound small
                                   configs, e.g. configs[0]); no timing events inside   */
#define RP_FLAG_EMULATE 0x20    /* parity tool: n_gpus VIRTUAL GPUs on one device, one
                                   process (rank 0, every worker local): cross-GPU
                                   groups run the cross-GPU kernel for every virtual GPU
                                   in ONE cooperative launch (flags, staging, partial
                                   fold and pushes as across real GPUs); lockstep batches
                                   only, no NVLS, no peer export/import                 */

/* Replica / gradient storage (reading R26). Arithmetic is fp32
 * in the pinned order of reading R1 for both; bf16 widens exactly on load and rounds the mean
 * once (IEEE round-to-nearest-even) on store. bf16 contexts: plain SGD (no
 * rp_step_momentum), workers bound with rp_bind_worker_bf16; across GPUs the per-GPU partial
 * sums travel as fp32 and the rounded mean as bf16; no NVLS (rp_nvls_enable: RP_EINVAL). */
#define RP_DTYPE_F32 0
#define RP_DTYPE_BF16 1

#define RP_SCHED_PAPER4 1       /* fig:scheduler 4-phase rule, P:883-923 (reading R4)  */
#define RP_SCHED_SHIFT_K 2      /* cyclic fixed-size-k rule (reading R4)    */
#define RP_SCHED_GG (-1)        /* rp_lockstep_run: the Group Generator (GB + GD, §5)   */

typedef struct rp_config {
  int32_t world;           /* n workers, 1..RP_MAX_WORLD                                 */
  int32_t n_gpus;          /* GPUs in the job; 0 = host-only context (schedules + GG)    */
  int64_t n_params;        /* N, fp32 elements per replica (flat), > 0      */
  int32_t workers_per_gpu; /* wpg; world == n_gpus * wpg when n_gpus > 0                 */
  int32_t rank;            /* this process's GPU index in [0, n_gpus)                    */
  int32_t device;          /* CUDA device ordinal this process drives                    */
  int32_t group_size;      /* k for Global Division and SHIFT_K, 1..RP_MAX_GROUP         */
  int32_t c_thres;         /* slowdown filter c_i - c_w < C_thres; <= 0 = off   */
  int32_t nodes;           /* PAPER4 node count (world = nodes * m); 0 = n_gpus          */
  uint64_t seed_gd;        /* splitmix64 seed of the GD random partition (reading R8)    */
  int32_t flags;           /* RP_FLAG_*                                                  */
  int32_t dtype;           /* RP_DTYPE_*: storage type of replicas and gradients (0 = fp32) */
  uint64_t job_id;         /* RP_FLAG_SHARED_GG: same nonzero value on every rank        */
  int32_t watchdog_s;      /* cross-GPU flag-wait limit in seconds: 0 = default (600),
                              < 0 = wait forever; env RP_WATCHDOG_S overrides. A wait past
                              it is recorded and reported as RP_ETIMEOUT (rp_check)        */
  int32_t reserved[3];
} rp_config;

/* One group: members ascending. seq >= 0: granted by the GG (creation order);
 * seq < 0: a static-schedule group (pure function of rule, step, members). */
typedef struct rp_group {
  int64_t seq;
  int32_t size;
  int32_t members[RP_MAX_GROUP];
} rp_group;

typedef struct rp_stats {
  int64_t groups_launched;    /* P-Reduce groups executed (including singletons)       */
  int64_t singleton_groups;   /* |G| = 1: SGD only                                      */
  int64_t cross_gpu_groups;   /* groups whose members span more than one GPU           */
  int64_t kernel_launches;    /* CUDA kernels this context launched                    */
  int64_t gd_calls;           /* Global Divisions run by the GG                         */
  int64_t gg_requests;        /* rp_group_generate calls                                */
  int64_t max_gb_depth;       /* deepest Group Buffer seen                              */
  int64_t lock_assertions;    /* conflict checks performed                              */
  int64_t bytes_hbm;          /* algorithmic HBM bytes moved by launched parts          */
  int64_t bytes_nvlink;       /* algorithmic NVLink bytes stored by this GPU            */
  int64_t gg_pending;         /* random GG: requests whose group had to wait (conflicts) */
  int64_t gg_granted;         /* random GG: groups granted                              */
  int64_t nvls_groups;        /* cross-GPU groups reduced in the NVSwitch (rp_nvls_enable) */
} rp_stats;

/* Device time of this context's P-Reduce kernel launches (RP_FLAG_TIMING),
 * from CUDA events recorded on the launching stream around each launch. */
typedef struct rp_timing {
  int64_t launches;           /* completed launches accumulated                        */
  double total_ms;            /* sum of per-launch durations                           */
  double min_ms, max_ms;
  int64_t bytes_hbm;          /* algorithmic HBM bytes of those launches               */
  int64_t bytes_nvlink;       /* algorithmic NVLink bytes read by this GPU             */
  /* split by kernel: intra-GPU groups (HBM-bound) and cross-GPU parts (NVLink-bound) */
  int64_t local_launches;
  double local_ms;
  int64_t local_bytes_hbm;
  int64_t cross_launches;
  double cross_ms;
  int64_t cross_bytes_nvlink;
  int64_t cross_bytes_hbm;    /* local HBM bytes of the cross launches (incl. fused groups) */
} rp_timing;

/* One timed launch (RP_FLAG_TIMING), in launch order: rp_timing_records. */
typedef struct rp_launch_record {
  double ms;                  /* CUDA-event duration on the launching stream            */
  int64_t bytes_hbm;          /* algorithmic HBM bytes of the launch                    */
  int64_t bytes_nvlink;       /* algorithmic NVLink bytes this GPU stores into peers    */
  int64_t batch;              /* rp_batch_end calls before it (= lockstep step index)   */
  int32_t cross;              /* 1 = cross-GPU (or NVLS) kernel, 0 = intra-GPU kernel    */
  int32_t reserved;
} rp_launch_record;

typedef struct rp_ctx rp_ctx;

/* ---- lifecycle ----------------------------------------------------------------- */

/* Create a context (north star rp_init(world, n_params)). With n_gpus > 0 it
 * selects cfg->device, creates one stream per local worker and the events,
 * and zeroes the Group Generator state (Group Buffers, counters c_w, lock
 * vector, RNG = seed_gd). Errors: RP_EINVAL (world not in [1,64],
 * n_params <= 0, group_size not in [1,16], world != n_gpus*wpg, rank/device
 * out of range), RP_ECUDA, RP_ENOMEM. */
int rp_init(const rp_config* cfg, rp_ctx** out);

/* Release streams, events, peer mappings and the context. Does not free the
 * borrowed replica / gradient buffers. Waits for this context's GPU work. */
int rp_finalize(rp_ctx* ctx);

/* Register worker w's flat replica x (read-write) and default gradient
 * buffer g (read-only, may be NULL). Both are device pointers on this
 * process's GPU, 16-byte aligned, n_params fp32 each; w must belong to this
 * rank (w / wpg == rank). Errors: RP_EINVAL, RP_ENODEV. */
int rp_bind_worker(rp_ctx* ctx, int32_t w, float* x_dev, const float* g_dev);
/* The same for a cfg.dtype = RP_DTYPE_BF16 context: x and g are bfloat16 arrays (raw 16-bit
 * patterns) of n_params elements, 16-byte aligned. rp_bind_worker on a bf16 context and
 * rp_bind_worker_bf16 on an fp32 context fail with RP_EINVAL. */
int rp_bind_worker_bf16(rp_ctx* ctx, int32_t w, uint16_t* x_dev, const uint16_t* g_dev);

/* The CUDA stream (cudaStream_t as void*) on which worker w's work is
 * ordered. Producing w's gradient on this stream makes rp_preduce wait for
 * it; after rp_barrier_free_wait(w, RP_WAIT_DEVICE), work on this stream sees
 * the averaged replica. Library-owned unless replaced by rp_set_worker_stream. */
int rp_worker_stream(rp_ctx* ctx, int32_t w, void** stream_out);
int rp_set_worker_stream(rp_ctx* ctx, int32_t w, void* stream);

/* ---- multi-GPU: peer memory over NVLink / NVSwitch ----------------------------------
 * A group whose members live on several GPUs runs as one exchange step over
 * peer memory: every rank must map its peers' replicas and flag
 * arrays. After binding all local workers, each rank calls rp_peer_export,
 * the caller exchanges the records (e.g. torch.distributed.all_gather_object)
 * and every rank calls rp_peer_import with the records of ALL ranks. */
typedef struct rp_peer_info {
  int32_t rank;            /* GPU index of the exporting rank                         */
  int32_t n_local;         /* local workers exported (= workers_per_gpu)              */
  int32_t first_worker;    /* rank * workers_per_gpu                                  */
  int32_t pid;             /* exporting process id (diagnostics)                      */
  uint8_t flags_handle[RP_IPC_HANDLE_BYTES];  /* cudaIpcMemHandle_t of the flag array  */
  int64_t flags_offset;
  uint8_t stage_handle[RP_IPC_HANDLE_BYTES];  /* staging buffer (partials pushed to it)  */
  int64_t stage_offset;
  int64_t stage_region_bytes;                 /* one region per local worker            */
  uint8_t x_handle[RP_MAX_LOCAL][RP_IPC_HANDLE_BYTES]; /* allocation holding replica i */
  int64_t x_offset[RP_MAX_LOCAL];                       /* byte offset of replica i      */
} rp_peer_info;

/* Fill *out with CUDA IPC handles for this rank's flag array and the replicas
 * of its local workers (all must be bound). Errors: RP_ESTATE (unbound worker,
 * single-GPU context), RP_ECUDA (the replica memory cannot be shared). */
int rp_peer_export(rp_ctx* ctx, rp_peer_info* out);
/* Map the peers' memory (infos[i] for every rank i, own record ignored).
 * Errors: RP_EINVAL (missing / inconsistent records), RP_ECUDA. */
int rp_peer_import(rp_ctx* ctx, const rp_peer_info* infos, int32_t n);

/* ---- multi-GPU: NVLS (NVLink SHARP) P-Reduce, SURVEY §8 row f1 ------------------------
 * The averaging of alg1 step 4 for a group spanning kp GPUs, reduced INSIDE
 * the NVSwitch: every GPU writes its local partial (its members' SGD-updated replicas,
 * left-folded, reading R1) into a buffer bound to a multicast object of the group's GPU
 * set; the owner of each chunk reads the sum of all kp partials with one
 * multimem.ld_reduce, divides by |G| and writes the mean to every GPU with one
 * multimem.st. Per-GPU NVLink bytes are ~4N per direction for any kp (the push kernel
 * moves 2(kp-1)/kp * 4N). The multicast objects play the role of the paper's cached
 * per-group NCCL communicators (at most 64 cached); one object (with
 * workers_per_gpu slots of ~4N bytes) per GPU subset of >= min_gpus GPUs, created once.
 * The switch's summation order over the kp partials is its own (reading R25): results
 * are bit-exact to the oracle for kp = 2 (fp32 addition is commutative) and within the
 * north-star tolerance otherwise. */

/* *supported = 1 when this rank's GPU supports multicast objects (driver + NVSwitch
 * fabric), else 0. Errors: RP_ESTATE (not a multi-GPU context). */
int rp_nvls_supported(rp_ctx* ctx, int32_t* supported);

/* Collective-barrier callback for rp_nvls_enable: must block until every rank of the
 * context has called it the same number of times, and return 0 iff every rank passed
 * local_status == 0 (an all-reduce of the ranks' status; nonzero = some rank failed). */
typedef int (*rp_barrier_fn)(void* user, int32_t local_status);

/* Collective over ALL ranks, after rp_peer_import, before the first rp_preduce: create,
 * share (POSIX file descriptors over a Unix socket, creator = lowest GPU of the subset)
 * and bind the multicast objects of every GPU subset of >= min_gpus (2..n_gpus) GPUs,
 * then route cross-GPU groups spanning >= min_gpus GPUs through the NVLS kernel.
 * `barrier(user, status)` is called 3 times by every rank; a rank's failure makes every
 * rank stop and return an error (nobody waits on a missing member). Device memory: per subset
 * workers_per_gpu * (4 n_params + flags) bytes on every GPU of the subset.
 * Errors: RP_EINVAL (min_gpus out of range, > 64 subsets), RP_ESTATE (peers not
 * imported, already enabled), RP_ENODEV (no multicast support), RP_ECUDA, RP_ENOMEM.
 * On error NVLS stays disabled (the push kernel keeps every group). */
int rp_nvls_enable(rp_ctx* ctx, int32_t min_gpus, rp_barrier_fn barrier, void* user);

/* ---- Step 3: group determination -------------------------------------------------- */

/* Static schedule: a pure function of (rule, config, step), the
 * same on every caller. Fills group_of[w] = index of w's group in
 * this step or -1 if w skips synchronization ("-" cells), and
 * *n_groups. group_of must hold `world` entries (caller-owned).
 * RP_SCHED_PAPER4 needs world = nodes * m with m = world / nodes.
 * Errors: RP_EINVAL (unknown rule, rule incompatible with the config). */
int rp_schedule_static(rp_ctx* ctx, int32_t rule, int64_t step, int32_t* group_of,
                       int32_t* n_groups);

/* Worker w's group in this step as an rp_group (size 1 when w skips: an
 * SGD-only "singleton" P-Reduce). seq = -(1 + step*world + members[0]). */
int rp_schedule_static_worker(rp_ctx* ctx, int32_t rule, int64_t step, int32_t w,
                              rp_group* out);

/* Dynamic group generation (GG request, §5.1-§5.3): c_w += 1; if
 * w's Group Buffer is non-empty return its head, else run a Global Division
 * over workers with empty GB, passing the slowdown filter and not retired,
 * push the groups to their members' GBs (lock bits set) and return w's.
 * With RP_FLAG_RANDOM_GG (§4.1): serve the group w was notified of, else draw
 * a random group containing w; if a member's lock bit is set the group waits
 * in the pending queue and the call returns RP_EAGAIN (*out = that group) —
 * call again (a retry does not count as a new request).
 * Serialized by an internal mutex; appends {"ev":"req"} to the trace.
 * Errors: RP_ESTATE (w still holds an unfinished group, or w retired), RP_EINVAL.
 * Multi-process jobs: every rank runs the same deterministic GG; lockstep
 * callers must issue requests in the same order on every rank. */
int rp_group_generate(rp_ctx* ctx, int32_t w, rp_group* out);

/* Acknowledge completion of GG group `seq` that this process does not
 * execute: pops it from its members' Group Buffers and clears
 * their lock bits, exactly as rp_barrier_free_wait does for local groups.
 * Used by ranks that replicate the deterministic GG in lockstep runs and by
 * host-only contexts. Errors: RP_EPROTO (unknown group, not at the head of a
 * member's GB, or a member that never requested it). */
int rp_gg_release(rp_ctx* ctx, int64_t seq);

/* Lockstep convenience: rp_group_generate for workers[0..n-1] in that order
 * (one GG critical section), out[i] = the group of workers[i]. Multi-GPU
 * lockstep runs issue the same call on every rank to keep the replicated GG
 * identical. Errors as rp_group_generate (requests before the failing one
 * stay granted). */
int rp_group_generate_many(rp_ctx* ctx, const int32_t* workers, int32_t n, rp_group* out);

/* Worker w will not request again after its current group (reading R19: a
 * finished worker must never be put into a Global Division). */
int rp_retire(rp_ctx* ctx, int32_t w);

/* ---- Step 2 + 4: fused SGD + P-Reduce ---------------------------------------------- */

/* Stage worker w's SGD update x_w <- x_w - lr * grad for its next
 * rp_preduce (alg1 step 2). grad = NULL uses the bound g buffer.
 * The pointer is borrowed until w's group completes. A member without a
 * staged step contributes y = x. Errors: RP_ESTATE (already staged),
 * RP_EINVAL (misaligned / no buffer). */
int rp_step(rp_ctx* ctx, int32_t w, const float* grad_dev, float lr);
/* rp_step for a bf16 context with a bf16 gradient (grad = NULL: the bound g). On a bf16
 * context rp_step accepts only grad = NULL. Errors as rp_step, RP_EINVAL on an fp32 context. */
int rp_step_bf16(rp_ctx* ctx, int32_t w, const uint16_t* grad_dev, float lr);

/* rp_step with the paper's ResNet-50 optimizer ("Momentum optimizer is
 * used with momentum=0.9 and weight_decay=1e-4"; reading R24): inside the fused
 * kernel, per element, g' = fl(g + fl(wd*x)); v <- fl(fl(momentum*v) + g');
 * y = fl(x - fl(lr*v)). v_dev is the worker's momentum buffer (n_params fp32,
 * 16-byte aligned device memory, borrowed, zero-initialized by the caller); it
 * stays per worker (only the weights are averaged). Errors as rp_step. */
int rp_step_momentum(rp_ctx* ctx, int32_t w, const float* grad_dev, float lr, float momentum,
                     float weight_decay, float* v_dev);

/* Collective arrival of worker w at group g (alg1 step 4). Every
 * member must call with an identical group. The last local
 * arriver enqueues the fused kernel on its worker stream after the other
 * members' streams (events, no host blocking). The kernel computes, per
 * element j, y_m = x_m[j] - lr_m*g_m[j] for m in G, the pinned fp32 sum
 * (reading R1), xbar = sum / |G|, and writes xbar to every member replica;
 * non-members are untouched (F^G_uu = 1). |G| = 1 is an SGD step.
 * Errors: RP_EPROTO (w not in g, members disagree, or a GG group other than
 * the one handed to w), RP_ESTATE (w's previous group not waited),
 * RP_ECONFLICT, RP_ECUDA. */
int rp_preduce(rp_ctx* ctx, int32_t w, const rp_group* g);

/* Launch batching (one kernel per lockstep step). Between rp_batch_begin and
 * rp_batch_end, groups whose local members have all arrived are queued
 * instead of launched; rp_batch_end launches all queued groups as ONE fused
 * kernel (disjoint groups run concurrently inside it). Outside a
 * batch every ready group launches at once. A wait on a queued group before
 * rp_batch_end returns RP_ESTATE. */
int rp_batch_begin(rp_ctx* ctx);
int rp_batch_end(rp_ctx* ctx);

/* Group-local completion: never a world barrier.
 * timeout_us >= 0: block the calling host thread until w's group is done on
 *   the device (or RP_ETIMEOUT, naming members that never arrived).
 * timeout_us == RP_WAIT_DEVICE: do not block the host; w's worker stream is
 *   already ordered after the group's kernel. Requires the group launched.
 * Either way, when the last member of a group has waited, the GG releases it
 * (Group Buffer pop, lock bits clear, {"ev":"done"} in the trace). */
#define RP_WAIT_DEVICE (-1)
int rp_barrier_free_wait(rp_ctx* ctx, int32_t w, int64_t timeout_us);

/* ---- observability ------------------------------------------------------------------ */
int rp_stats_get(rp_ctx* ctx, rp_stats* out);
/* Block until every timed launch so far has completed, return their sums and
 * reset the accumulator. Errors: RP_ESTATE (context created without
 * RP_FLAG_TIMING), RP_ECUDA. */
int rp_timing_read(rp_ctx* ctx, rp_timing* out);

/* Did a cross-GPU (or NVLS) flag wait of a COMPLETED launch pass the watchdog limit
 * (rp_config.watchdog_s)? RP_OK, or RP_ETIMEOUT with rp_last_error() naming the GPU, the
 * peer, the flag kind, the chunk and the tags. After a timeout the replicas of the groups
 * of that step are undefined. rp_barrier_free_wait and rp_lockstep_run check it too. */
int rp_check(rp_ctx* ctx);
/* Start writing the JSONL decision trace (req / done / retire in GG order)
 * to `path` (truncates). The oracle replays it (tests/). */
int rp_trace_open(rp_ctx* ctx, const char* path);
const char* rp_last_error(void);
const char* rp_strerror(int status);
int rp_abi_version(void);

/* ---- synthetic inputs and compute (harness kernels, not part of the method) ----------- */

/* Enqueue a device-side busy wait of `ns` nanoseconds on `stream` (one thread
 * spinning on %globaltimer): the synthetic per-step compute time T_c of the
 * heterogeneity runs ("adding ... times the normal iteration time of sleep",
 * P:1395; reading R13). Errors: RP_EINVAL (ns < 0), RP_ECUDA. */
int rp_compute_delay(void* stream, int64_t ns);

/* Synthetic compute of worker w for the heterogeneity runs (reading R13): rp_lockstep_run
 * enqueues rp_compute_delay(ns) on w's stream at the start of each of w's steps, before its
 * rp_step (0 = none). Ordering stays group-local: a slow worker delays only the groups it
 * joins, through its arrival event. Errors: RP_EINVAL (w not local, ns < 0), RP_ENODEV. */
int rp_set_compute_delay(rp_ctx* ctx, int32_t w, int64_t ns);

/* dst[i] = xi(seed, w, t, j0 + i) for i < n on `stream` (cudaStream_t as void*),
 * the counter-based generator of DESIGN.md "Input recipe" (splitmix64
 * finalizer; bit-identical to rp_inputs/gen.py). dst must be 4-byte aligned
 * device memory. Errors: RP_EINVAL, RP_ECUDA. */
int rp_fill_xi(float* dst, int64_t n, uint64_t seed, uint64_t w, uint64_t t, uint64_t j0,
               void* stream);

/* ---- NCCL-baseline helpers (bench.py --impl nccl / nccl-group; NOT the method's path) ----
 * The paper's P-Reduce is an NCCL all-reduce on a per-group communicator;
 * with several simulated workers per GPU a baseline needs a local pre-sum and a local
 * broadcast of the mean (one NCCL rank per GPU). Buffers: device memory of the current GPU,
 * 16-byte aligned, n fp32 elements; 1 <= m <= 16 members. Errors: RP_EINVAL, RP_ECUDA.
 *   rp_bench_presum:       out = left fold over m of fl(x_i - fl(lr g_i))   (x, g read once)
 *   rp_bench_scatter_mean: x_i = fl(s / k) for every member i                (s read once) */
int rp_bench_presum(const float* const* x, const float* const* g, int32_t m, int64_t n, float lr, float* out,
                    void* stream);
int rp_bench_scatter_mean(const float* s, int64_t n, float k, float* const* x, int32_t m, void* stream);

/* Per-launch timing records (RP_FLAG_TIMING): copies up to `cap` completed launches (oldest
 * first) into out, sets *n, and drops them (like rp_timing_read, which aggregates instead).
 * Blocks until those launches completed. Errors: RP_EINVAL, RP_ESTATE (no RP_FLAG_TIMING),
 * RP_ECUDA. */
int rp_timing_records(rp_ctx* ctx, rp_launch_record* out, int32_t cap, int32_t* n);

/* Native lockstep executor (alg1, for every local worker of this rank): runs
 * `steps` iterations t = t0, t0 + 1, ... (t0 >= 1) exactly as the per-call sequence
 *   rp_step(w, NULL, lr) for every local w;
 *   step 3: t % section_length != 0 -> singleton group {w} with seq
 *           -(1 + t*world + w) (SGD only); rule RP_SCHED_PAPER4 / RP_SCHED_SHIFT_K ->
 *           rp_schedule_static_worker(rule, t, w); rule RP_SCHED_GG -> rp_group_generate_many
 *           over ALL world workers in ascending order (the replicated GG stays identical on
 *           every rank);
 *   rp_batch_begin; rp_preduce(w, its group) for every local w; rp_batch_end;
 *   rp_barrier_free_wait(w, RP_WAIT_DEVICE) for every local w; rp_gg_release of every GG
 *   group of the step with no local member (ascending seq).
 * Every rank of a multi-GPU job calls it with the same arguments. Plain SGD with the bound
 * gradients (fp32 or bf16 contexts); momentum steps use the per-call API. Returns the first
 * failing call's status (RP_EINVAL for a bad rule / t0 / steps / section_length). */
int rp_lockstep_run(rp_ctx* ctx, int32_t rule, int64_t t0, int64_t steps, float lr, int32_t section_length);

#ifdef __cplusplus
}
#endif
#endif /* RP_H */
