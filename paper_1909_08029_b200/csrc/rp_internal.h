// Internal declarations of librp (not part of the ABI; see include/rp.h).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "rp.h"

namespace rp {

// ---- errors ------------------------------------------------------------------------
// Sets the thread-local message returned by rp_last_error() and returns `code`.
int fail(int code, const std::string& msg);

// ---- static schedules (sched.cpp) ----------------------------------------------------
// Fill group_of[w] (group index, -1 = skip) for `world` workers; returns RP_OK or RP_EINVAL.
int schedule_paper4(int nodes, int m, int64_t step, int32_t* group_of, int32_t* n_groups);
int schedule_shift_k(int n, int k, int64_t step, int32_t* group_of, int32_t* n_groups);

// ---- Group Generator: Group Buffer + Global Division + filter (gg.cpp) ---------------
constexpr int kGbCap = 4;        // Group Buffer depth bound (GD alone keeps depth <= 1)
constexpr int kTableCap = 256;   // live groups

struct GGGroup {
  int64_t seq;       // -1 = free slot
  int32_t size;
  int32_t members[RP_MAX_GROUP];
  uint64_t arrived;  // members that called rp_preduce (shared GG, any process)
  int64_t ticket;    // order of complete arrival (shared GG), -1 until all members arrived
  int32_t initiator; // random GG: the requesting worker
  int32_t granted;   // random GG: lock bits held (0 while in the pending queue)
};

constexpr int32_t kPolicyGD = 0;      // Group Buffer + Global Division + filter (§5)
constexpr int32_t kPolicyRandom = 1;  // random groups + lock vector + pending queue (§4.1)

// Plain-old-data so it can live in process-shared memory.
struct GGState {
  int32_t n, k, c_thres;
  uint64_t rng;           // splitmix64 state
  int64_t next_seq;
  int32_t gb_len[RP_MAX_WORLD];
  int64_t gb[RP_MAX_WORLD][kGbCap];
  int64_t counters[RP_MAX_WORLD];
  int64_t handed[RP_MAX_WORLD];   // seq handed to w by a request, -1 = none
  uint64_t lock;
  uint64_t retired, retiring;     // reading R19
  GGGroup table[kTableCap];
  int64_t gd_calls, requests, max_depth;
  int64_t next_ticket;            // complete-arrival order of groups (shared GG)
  // Inter-Intra Synchronization (§5.2): nodes > 0 splits every division into an
  // Inter and an Intra round; head_rot[a] rotates node a's Head Worker
  int32_t nodes;
  int32_t head_rot[RP_MAX_WORLD];
  // random GG (§4.1)
  int32_t policy;
  int32_t npending;
  int64_t pending[kTableCap];     // FIFO of pending group seqs
  int64_t pending_of[RP_MAX_WORLD];
  uint8_t waiting[RP_MAX_WORLD];
  int64_t n_pending, n_granted;
};

void gg_init(GGState* s, int n, int k, int c_thres, uint64_t seed, int policy = kPolicyGD, int nodes = 0);
// Returns RP_OK and fills *out, RP_EAGAIN (random GG: the worker's group waits in the
// pending queue; *out holds it; call again), or an RP_E* code.
int gg_request(GGState* s, int w, rp_group* out);
// Group `seq` completed: pop it from its members' GBs, clear lock bits.
int gg_done(GGState* s, int64_t seq, rp_group* released);
int gg_retire(GGState* s, int w);
const GGGroup* gg_find(const GGState* s, int64_t seq);

// ---- kernels (preduce.cu, xi.cu) -------------------------------------------------------
// alg1 step 2 for one member, applied inside the fused kernels:
//   plain SGD:             y = fl(x - fl(lr g))
//   momentum + L2: g' = fl(g + fl(wd x)); v = fl(fl(mu v) + g'); y = fl(x - fl(lr v))
//   no staged step (g = nullptr): y = x
struct MemberUpdate {
  const float* g;  // gradient, or nullptr
  float* v;        // momentum buffer (read-modify-write), or nullptr for plain SGD
  float lr, mu, wd;
};
// Several disjoint groups executed by one launch: members of group gi are
// entries group_first[gi] .. group_first[gi] + group_k[gi] - 1 (packed, in
// ascending worker id). cta_begin is filled by the launcher.
constexpr int kMaxTasks = 16;
constexpr int kMaxTaskMembers = 64;
struct MultiTask {
  int32_t ngroups;
  int32_t group_k[kMaxTasks];
  int32_t group_first[kMaxTasks];
  float* x[kMaxTaskMembers];
  MemberUpdate u[kMaxTaskMembers];
  int32_t cta_begin[kMaxTasks + 1];
  int32_t reserve_sms;  // SMs left to a concurrent cross-GPU launch (0 = use every SM)
  int32_t tiles_per_cta;  // dynamic-tile kernel: CTAs retire after this many tiles (0 = persistent)
  int32_t dyn_batch;      // dynamic-tile kernel: tile ids per atomic (set by the launcher)
};

// Fused SGD + P-Reduce of groups whose members all live on the current GPU.
int launch_preduce_multi(const MultiTask& t, int64_t n, void* stream, std::string* err);
// The same with a TMA bulk-copy pipeline; RP_EINVAL for shapes it does not cover.
int launch_preduce_tma(const MultiTask& t, int64_t n, void* stream, std::string* err, int variant,
                       bool bf16 = false);
// ---- cross-GPU parts (xgpu.cu) ----------------------------------------------------------
constexpr int kMaxXParts = 8;    // cross-GPU groups one GPU takes part in, per launch
constexpr int kMaxXLocal = 8;    // local members of one cross-GPU group
constexpr int kMaxXGpus = 8;     // GPUs of one group
constexpr int kFlagSlots = 64;   // slot = lowest member of the group
constexpr int kFlagSrc = 8;      // source GPU
constexpr int kMaxChunks = 4096; // chunks per owner slice
constexpr int64_t kMinChunkF4 = 8192;  // 128 KiB per buffer and chunk (fence amortization)
constexpr int kFlagA = 0, kFlagB = 1, kFlagReady = 2;
constexpr int64_t kFlagStride = 2 * kMaxChunks + 1;  // A[chunk], B[chunk], READY
constexpr size_t kFlagWords = static_cast<size_t>(kFlagSlots) * kFlagSrc * kFlagStride;

struct XPart {
  int32_t m;          // local members (ascending worker id)
  int32_t kp;         // GPUs in the group
  int32_t me;         // this GPU's index among them (ascending GPU id)
  int32_t k_total;    // |G|
  int32_t slot;       // flag slot (lowest member of the group)
  int32_t rem;        // n mod 4
  uint64_t tag[kMaxXGpus];   // per peer: nonzero, unique per (group launch, GPU pair)
  int64_t n4, S4, CH, nch;   // geometry (xgpu_geometry): nch chunks per slice; chunks c < nch - nsmall
                             // split CH 1024-vector tiles evenly (balanced), the last nsmall chunks
                             // are tail_w tiles each (tiles CH + (c - nch + nsmall) * tail_w, ...)
  int32_t nsmall, tail_w;
  float* x[kMaxXLocal];
  MemberUpdate u[kMaxXLocal];
  float* xfirst[kMaxXGpus];               // first local member replica of each group GPU (mapped)
  float* stage[kMaxXGpus];                // staging region of each group GPU for this group (mapped)
  unsigned long long* pflags[kMaxXGpus];  // flag array of each group GPU (mapped or local)
  int32_t gpu[kMaxXGpus];                 // GPU ids, ascending
};

// Optional per-item timeline (RP_XGPU_PROFILE): 4 x u64 per item (A, B, C stage of a chunk).
struct XItemRecord {
  unsigned long long t_start, t_ready, t_end;  // %globaltimer ns: begin, wait satisfied, end
  unsigned long long meta;                     // kind (2 bits) | part (6) | cta (24) | chunk (32)
};

// A flag wait that passed the watchdog limit (host-mapped; first failure wins).
struct XErr {
  unsigned long long code;  // 0 = none, 1 = flag wait timed out
  int32_t gpu, src, kind, slot;
  int64_t chunk;
  unsigned long long tag, seen;
};

// Intra-GPU groups of the same step fused into the cross-GPU launch as "L jobs" of the
// warp-specialized kernel, so their HBM-only work fills the time the NVLink transfers leave.
constexpr int kMaxXLocalGroups = 16;
constexpr int kMaxFusedK = 4;
struct XLocalGroup {
  int32_t k;
  float* x[kMaxFusedK];
  MemberUpdate u[kMaxFusedK];
};

// Kernel parameters exceed 4 KB: CUDA >= 12.1 large-parameter launches (sm_70+).
struct XTask {
  int32_t nparts;
  int32_t my_gpu;
  int64_t n;
  unsigned long long* my_flags;
  int32_t max_ctas;                        // grid cap (0 = every resident CTA slot)
  int32_t bf16;                            // replicas / gradients are bf16 (reading R26)
  XItemRecord* prof;                       // nullptr unless profiling; [part][kind][chunk]
  unsigned long long watchdog_ns;          // flag-wait limit, 0 = wait forever
  XErr* err;                               // host-mapped error record (device address)
  int32_t nbuf;                            // shared-memory tile ring depth (launcher)
  int32_t blag;                            // warp-specialized kernel: B runs blag iterations after A
  int32_t sig2;                            // ... with two flag-posting SIG jobs per iteration (blag >= 1)
  int32_t part_major;                      // claim order: 1 = part by part, 0 = chunk-major over parts
  int32_t early_a;                         // dynamic claiming: A flags posted after the B block's first
                                           // tile, not at the iteration's end (RP_XGPU_EARLY_A)
  int32_t lookahead;                       // dynamic claiming: claim + push the next A block while a
                                           // B block's flags are not yet posted (RP_XGPU_LOOKAHEAD)
  unsigned int* claim;                     // dynamic chunk claiming: [chunk-major, part 0..7, ...,
                                           // [L tiles, done CTAs] (kXClaimWords words), zeroed
                                           // between launches by the kernel (nullptr = static lanes)
  unsigned long long* cta_stat;            // profiling: per CTA ns [ring wait, signal wait, flag wait, total]
  int32_t nlocal;                          // fused intra-GPU groups (warp-specialized kernel only)
  XLocalGroup lg[kMaxXLocalGroups];
  XPart part[kMaxXParts];
};

// Lanes of the cross-GPU kernel (chunk c runs on lane c mod kXLanes on every GPU).
constexpr int kXLanes = 296;
// RP_XGPU_PROFILE per-CTA records (u64 words, 2048 CTAs): [0, 4*2048) ns [ring wait, signal wait,
// flag wait, total]; [4*2048, 6*2048) absolute begin / end; then kCtaSig SIG times per CTA (time | 1:
// posts A flags | 2: posts B flags), kCtaWait flag waits per CTA as (start | kind, end), 2 counters
constexpr int kCtaSig = 32, kCtaWait = 32;
constexpr int64_t kCtaSigBase = 6 * 2048, kCtaWaitBase = kCtaSigBase + 2048 * kCtaSig,
                  kCtaCntBase = kCtaWaitBase + 2048 * 2 * kCtaWait, kCtaStatWords = kCtaCntBase + 2048 * 2;
constexpr int kXClaimWords = 2 * kMaxXParts + 2;  // per (virtual) GPU; the L / done words at 2 kMaxXParts
// Slice and chunk geometry of a part (kp set) for n elements (depends on n and kp only).
void xgpu_geometry(XPart& p, int64_t n);
// Bytes of one staging region (one cross-GPU group owned by one local worker).
int64_t xgpu_stage_region_bytes(int64_t n);
// This GPU's parts of the cross-GPU groups of one step, in ONE launch.
int launch_xgpu(XTask& t, void* stream, std::string* err);
// RP_XGPU_V2=1: plain-SGD steps take the register kernel of xgpu.cu instead (comparison)
bool use_v2();
// The warp-specialized cross-GPU kernel (xgpu_ws.cu; plain SGD, fp32 and bf16): TMA bulk loads
// into a staged ring, bulk stores out. emu: d_tasks holds V uploaded tasks (cooperative launch).
int launch_xgpu_ws(XTask& T, const XTask* d_tasks, int V, int max_parts, void* stream, std::string* err, int mmax,
                   int kpmax, bool emu);
// RP_FLAG_EMULATE: the tasks of V virtual GPUs (one device) in ONE cooperative launch;
// d_tasks: device buffer of V XTask (uploaded on `stream` before the launch).
int launch_xgpu_emulated(XTask* tasks, int V, XTask* d_tasks, void* stream, std::string* err);

// ---- NVLS P-Reduce (nvls.cu kernel, nvls_setup.cpp multicast objects) ---------------------
// One multicast object per GPU subset (mask of GPU ids, >= min_gpus GPUs), bound on every GPU
// of the subset to `slots` slots of slot_bytes: slot data (4 n bytes: the GPU's partial, then
// the mean) followed by flags [nch][kNvlsFlagStride] u64 (arrive[position], done).
constexpr int kNvlsFlagStride = 9;   // arrive[8] + done
constexpr int kMaxNParts = 8;        // NVLS groups one GPU takes part in, per launch
struct NvlsObj {
  uint32_t mask;         // GPU subset
  int32_t kp, me;        // |subset|, this GPU's position (ascending GPU id)
  int32_t slots;
  int64_t slot_bytes, data_bytes, nch, CH;  // CH: chunk in float4
  uint64_t mc_handle, mem_handle;           // CUmemGenericAllocationHandle
  uintptr_t uc_va, mc_va;                   // unicast / multicast mappings of the whole object
  size_t size;
  int64_t launched;      // groups launched on this subset (slot = launched % slots)
};
struct NvlsState {
  int32_t min_gpus = 0;  // 0 = disabled
  std::vector<NvlsObj> objs;
};
int nvls_supported(int device, int* out);
// Collective over all ranks (barrier called 3 times on every rank).
int nvls_setup(NvlsState* s, int rank, int n_gpus, int device, int wpg, int64_t n, int min_gpus,
               const int32_t* peer_pids, rp_barrier_fn barrier, void* user, std::string* err);
void nvls_teardown(NvlsState* s);
NvlsObj* nvls_find(NvlsState* s, uint32_t mask);
int64_t nvls_chunk_f4();

struct NPart {
  int32_t m;             // local members (ascending worker id)
  int32_t kp, me;        // GPUs in the group, this GPU's position
  int32_t k_total;       // |G|
  int32_t rem;           // n mod 4
  uint64_t tag;          // nonzero; unique per use of the slot
  int64_t n4, CH, nch, nown;
  int64_t off_P, off_R, off_S;   // first item of each phase for this part
  float* x[kMaxXLocal];
  MemberUpdate u[kMaxXLocal];
  float* uc;                     // slot data, this GPU's copy (unicast)
  float* mc;                     // slot data, multicast address
  unsigned long long* ucf;       // slot flags, unicast
  unsigned long long* mcf;       // slot flags, multicast
  unsigned long long watchdog_ns;  // flag-wait limit (0 = forever); a timeout is recorded in err
  XErr* err;                       // host-mapped error record (device address), or nullptr
  int32_t gpu;                     // this GPU's id (error record)
};
struct NTask {
  int32_t nparts;
  int32_t hbm_ctas;              // CTAs on the P/S list (launcher); 0 = one list
  int64_t total_items, n_p, n_r, off_s0, n_hbm;
  NPart part[kMaxNParts];
};
// This GPU's parts of every NVLS group of one step, in ONE launch (items P*, R*, S*).
int launch_nvls(NTask& t, void* stream, std::string* err);
int launch_delay(void* stream, int64_t ns, std::string* err);
// Force-load the kernels each launcher can pick (CUDA lazy loading would load them at their first
// launch, which a random schedule may reach only inside a timed region). Called by rp_init.
void preload_xgpu_ws();
void preload_xgpu();
void preload_preduce();
void preload_preduce_tma();
int launch_fill_xi(float* dst, int64_t n, uint64_t seed, uint64_t w, uint64_t t, uint64_t j0,
                   void* stream, std::string* err);

}  // namespace rp
